#!/bin/bash
# FFMA2 epilogue candidate: parity/bit-identity subset + per-layer timing of C.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "pipeline_matches or frame0 or halo_staging or gpu_conv" > gpurun_out/gputest_ffma2.log 2>&1; echo "rc=$?" >> gpurun_out/gputest_ffma2.log
python tools/layer_report.py C gpurun_out/layers_c_ffma2.json > gpurun_out/layers_c_ffma2.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ffma2_c.json 2> gpurun_out/ffma2_c.err
