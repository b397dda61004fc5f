#!/bin/bash
# Seam / branch schedule A/B on C, interleaved repetitions on one box.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
rm -f gpurun_out/ab2_*.jsonl
for rep in 1 2 3; do
  for v in "LC_NONE=1" "LC_BRANCH_SEAM=0" "LC_SEAM_PARTS=0" "LC_BRANCH_DEEP=2"; do
    env $v timeout 600 python bench.py --no-cpu-baseline --steps 30 >> gpurun_out/ab2_$v.jsonl 2> /dev/null
  done
done
