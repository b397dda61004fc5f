#!/bin/bash
# Round profile refresh (run on the GPU box from the repo root via gpurun):
# bench lines (B, C, D, reference arm), parity, ncu launch lists (B with
# DRAM bytes, C) and `ncu --set full` captures of the top conv launch of B
# (u0 of step 0 in run 3: 2 x 42 + 8), of the decoder's fused last stage and
# of the halo-staged decoder up-conv (dec2 of run 3's first slice: 84 + 32),
# plus the launch list of one sharded decode (D).
# Outputs land in gpurun_out/; tools/collect_profiles.py copies the
# summaries into profiles/.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err
python bench.py --workload C > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python bench.py --workload D > gpurun_out/bench_d.json 2> gpurun_out/bench_d.err
python tools/parity_report.py > gpurun_out/parity.json 2> gpurun_out/parity.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launch_b.csv python tools/profile_step.py B 3 > gpurun_out/ncu_b.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launch_c.csv python tools/profile_step.py C 2 > gpurun_out/ncu_c.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv_tc --launch-skip ${TOPIDX:-92} --launch-count 1 \
    -o gpurun_out/full_top python tools/profile_step.py B 3 > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tap_tc --launch-skip 4 --launch-count 1 \
    -o gpurun_out/full_tap python tools/profile_step.py B 1 > gpurun_out/ncu_full_tap.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv_tc --launch-skip 116 --launch-count 1 \
    -o gpurun_out/full_halo python tools/profile_step.py B 3 > gpurun_out/ncu_full_halo.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launch_d.csv python bench.py --workload D --steps 1 --warmup 3 > gpurun_out/ncu_d.log 2>&1
python tools/layer_report.py B gpurun_out/layers_b.json > gpurun_out/layers_b.txt 2>&1
python tools/layer_report.py C gpurun_out/layers_c.json > gpurun_out/layers_c.txt 2>&1
python tools/swap_timeline.py B > gpurun_out/swap_timeline_b.txt 2>&1
ls -la gpurun_out
