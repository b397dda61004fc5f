#!/bin/bash
# A/B of the seam schedule on config C (same box, back to back): whole-batch
# seam, per-branch seam, per-branch + half-entry parts (default).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "LC_BRANCH_SEAM=0" "LC_SEAM_PARTS=0" "LC_SEAM_PARTS=1" "LC_BRANCH_DEEP=0"; do
  env $v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
done
