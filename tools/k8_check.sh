#!/bin/bash
# K8 decoder rework: parity tests touching the decoder + D / C bench + ncu of the decoder stage.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "fused_tap or sliced_decode or decode or pipeline_matches or frame0 or config_a" > gpurun_out/gputest_k8.log 2>&1
echo "rc=$?" >> gpurun_out/gputest_k8.log
timeout 600 python bench.py --workload D --no-cpu-baseline > gpurun_out/k8_bench_d.json 2> gpurun_out/k8_bench_d.err
timeout 600 python bench.py --workload B --no-cpu-baseline > gpurun_out/k8_bench_b.json 2> gpurun_out/k8_bench_b.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/k8_launch_d.csv python tools/profile_step.py D 2 > gpurun_out/k8_ncu_d.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tap_tc --launch-skip 5 --launch-count 1 \
    -o gpurun_out/k8_full_dec python tools/profile_step.py D 2 > gpurun_out/k8_ncu_full.log 2>&1
