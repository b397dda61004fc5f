#!/bin/bash
# Round-2 profile refresh (GPU box, repo root, via gpurun): bench lines for
# the headline config C (+ reference arm, D, B), the ncu launch list of one
# C video with DRAM bytes per launch, `ncu --set full` captures of C's
# stem GEMM and d0 (run 1, step 0: conv launches 0 and 1), of the head
# (K8 with the fused sampler step, run 1 step 0) and of the decoder's last
# stage (K8 subpix, run 1 slice 0), the per-layer event timing of C and the
# swap timeline of C.  Outputs in gpurun_out/ (tools/collect_profiles.py
# copies the summaries into profiles/).
set -x
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
[ "${SKIP_BENCH:-0}" = 1 ] || {
python bench.py > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python bench.py --workload D > gpurun_out/bench_d.json 2> gpurun_out/bench_d.err
python bench.py --workload B --no-cpu-baseline > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err
}
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launch_c.csv python tools/profile_step.py C 2 > gpurun_out/ncu_c.log 2>&1
# launch indices count from the FIRST run (run 1, step 0): the number of
# launches per run depends on the swap schedule the host-link probe picks
for spec in "stem 0" "d0 1"; do set -- $spec
  ncu --set full --clock-control none --import-source on -k regex:conv_tc --launch-skip $2 --launch-count 1 \
      -o gpurun_out/full_c_$1 -f python tools/profile_step.py C 1 > gpurun_out/ncu_full_c_$1.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:tap_tc --launch-skip 0 --launch-count 1 \
    -o gpurun_out/full_c_head -f python tools/profile_step.py C 1 > gpurun_out/ncu_full_c_head.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tap_tc --launch-skip 25 --launch-count 1 \
    -o gpurun_out/full_c_dec -f python tools/profile_step.py C 1 > gpurun_out/ncu_full_c_dec.log 2>&1
python tools/layer_report.py C gpurun_out/layers_c.json > gpurun_out/layers_c.txt 2>&1
python tools/parity_report.py gpurun_out/parity.json > gpurun_out/parity.log 2>&1
python tools/sweep.py C gpurun_out/sweep.json > gpurun_out/sweep.log 2>&1
python tools/swap_timeline.py C > gpurun_out/swap_timeline_c.txt 2>&1
ls -la gpurun_out
# D: launch list with DRAM bytes (conv traffic per launch for bench's roofline.traffic)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launch_d.csv python tools/profile_step.py D 2 > gpurun_out/ncu_d.log 2>&1
# D's dec2 (the 288x512 sub-pixel up-conv, halo-staged) of run 1's first slice
ncu --set full --clock-control none --import-source on -k regex:conv_tc --launch-skip 2 --launch-count 1 \
    -o gpurun_out/full_d_dec2 -f python tools/profile_step.py D 1 > gpurun_out/ncu_full_d_dec2.log 2>&1
# reference arm cross-check (B, full frames per core vs the bounded sample)
timeout 1800 python tools/ref_crosscheck.py gpurun_out/ref_crosscheck.json > gpurun_out/ref_crosscheck.log 2>&1
