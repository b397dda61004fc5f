#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "branch_deep" > gpurun_out/gputest_bm.log 2>&1; echo "rc=$?" >> gpurun_out/gputest_bm.log
for bd in 1 2 0 1 2 0; do
  LC_BRANCH_DEEP=$bd timeout 600 python bench.py --no-cpu-baseline --steps 30 >> gpurun_out/bm_$bd.jsonl 2> /dev/null
done
