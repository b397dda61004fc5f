#!/bin/bash
# A/B of the per-branch deep path on config C (same box, back to back).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "branch_deep or fused_sampler or ledger or swapping or tiles" > gpurun_out/gputest_bd.log 2>&1
for bd in 0 1 auto; do
  LC_BRANCH_DEEP=$bd timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c_bd$bd.json 2> gpurun_out/bench_c_bd$bd.err
done
