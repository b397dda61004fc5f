#!/bin/bash
# Final round-2 pass: the full GPU test suite, smoke(), then the profile refresh.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputest_final.log 2>&1; echo "rc=$?" >> gpurun_out/gputest_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
bash tools/refresh_profiles_r02.sh > gpurun_out/refresh.log 2>&1
