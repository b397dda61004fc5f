#!/bin/bash
# K8 decoder tile height A/B (D and B benches) + decoder parity tests per variant.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for ty in 3 4 5; do
  LC_K8_TY=$ty timeout 600 python -m pytest tests -m gpu -q -x -k "fused_tap or sliced_decode or frame0_slice or config_a" > gpurun_out/k8ty_test_$ty.log 2>&1
  echo "rc=$?" >> gpurun_out/k8ty_test_$ty.log
  LC_K8_TY=$ty timeout 600 python bench.py --workload D --no-cpu-baseline > gpurun_out/k8ty_d_$ty.json 2> gpurun_out/k8ty_d_$ty.err
done
for ty in 4 5; do
  LC_K8_TY=$ty timeout 600 python bench.py --workload B --no-cpu-baseline > gpurun_out/k8ty_b_$ty.json 2> gpurun_out/k8ty_b_$ty.err
done
