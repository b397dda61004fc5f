#!/bin/bash
# e2e vs deferred-download gate point (B)
python -m pytest tests -m gpu -x -q -k "graph_replay or simulated or swap" > gpurun_out/dl_tests.log 2>&1
tail -2 gpurun_out/dl_tests.log
for g in off 0:stem 0:d0 0:up 1:d0 1:up 2:d0 3:d0 3:up; do
  for r in 1 2; do
    LC_DL_GATE=$g python bench.py --workload B --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/dl_$g.$r.json 2>/dev/null
    python -c "import json,sys; d=json.loads(open('gpurun_out/dl_$g.$r.json').read().strip().splitlines()[-1]); print('$g', round(d['value']), round(d['e2e']['value']), d['clocks']['sm_mhz'])"
  done
done
