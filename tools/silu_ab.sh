#!/bin/bash
# Parity and C timing with the approximate (tanh.approx) vs exact (ex2/rcp) SiLU epilogue.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in 0 1; do
  LC_SILU_EXACT=$v timeout 900 python tools/parity_report.py gpurun_out/parity_silu$v.json > gpurun_out/parity_silu$v.log 2>&1
  LC_SILU_EXACT=$v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/silu_c_$v.json 2> gpurun_out/silu_c_$v.err
done
