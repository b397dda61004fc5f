#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "branch_deep or pipeline_matches or frame0_slice" > gpurun_out/gputest_hh.log 2>&1; echo "rc=$?" >> gpurun_out/gputest_hh.log
python tools/layer_report.py C gpurun_out/layers_c_hh.json > gpurun_out/layers_c_hh.txt 2>&1
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline >> gpurun_out/hh_c.jsonl 2> /dev/null; done
