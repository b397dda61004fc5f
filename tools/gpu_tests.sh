#!/bin/bash
# GPU tests only (pytest -m gpu [extra args]), log under gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout ${TMO:-1500} python -m pytest tests -m gpu -q -x "$@" > gpurun_out/gputest.log 2>&1; echo "gputest rc=$?" >> gpurun_out/gputest.log
