#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
LC_K8_HEAD_TY=3 timeout 900 python -m pytest tests -m gpu -q -x -k "fused or pipeline_matches or frame0_slice" > gpurun_out/gputest_hty.log 2>&1; echo "rc=$?" >> gpurun_out/gputest_hty.log
rm -f gpurun_out/hty_*.jsonl
for rep in 1 2 3; do
  for ty in 5 3; do
    LC_K8_HEAD_TY=$ty timeout 600 python bench.py --no-cpu-baseline --steps 30 >> gpurun_out/hty_$ty.jsonl 2> /dev/null
  done
done
for ty in 5 3; do
  LC_K8_HEAD_TY=$ty ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tap_tc_kernel.1 --csv \
    --log-file gpurun_out/hty_ncu_$ty.csv python tools/profile_step.py C 2 > /dev/null 2>&1
done
