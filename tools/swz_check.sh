#!/bin/bash
# swizzled fp16 TMA-store staging: GPU tests, bench C, stem ncu
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/swz_tests.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/swz_tests.log
python bench.py > gpurun_out/swz_bench_c.json 2> gpurun_out/swz_bench_c.err; tail -1 gpurun_out/swz_bench_c.json | cut -c1-200
ncu --set full --clock-control none --import-source on -k regex:conv_tc --launch-skip 0 --launch-count 1 \
    -o gpurun_out/full_c_stem -f python tools/profile_step.py C 1 > /dev/null 2>&1
echo done
