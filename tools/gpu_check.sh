#!/bin/bash
# One GPU-box pass: GPU tests, the default bench (config C) and the
# reference arm, outputs under gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; lscpu > gpurun_out/lscpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "gputest rc=$?" >> gpurun_out/gputest.log
timeout 600 python bench.py > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err; echo "bench rc=$?" >> gpurun_out/bench_c.err
if [ "${REF:-1}" = 1 ]; then
  timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref_c.json 2> gpurun_out/ref_c.err
  echo "ref rc=$?" >> gpurun_out/ref_c.err
fi
