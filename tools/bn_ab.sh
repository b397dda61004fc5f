#!/bin/bash
# BN wave-model overhead constant A/B on C (power-capped clocks favour fewer operand bytes per FLOP?).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for o in 32 64 128 32; do
  LC_BN_OVERHEAD=$o timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bn_$o.json 2> gpurun_out/bn_$o.err
  LC_BN_OVERHEAD=$o python tools/layer_report.py C gpurun_out/bn_layers_$o.json > gpurun_out/bn_layers_$o.txt 2>&1
done
