#!/bin/bash
python tools/exp/subpix_ab.py > gpurun_out/subpix_ab.txt 2>&1
cat gpurun_out/subpix_ab.txt
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_all.log 2>&1; tail -3 gpurun_out/gpu_all.log
for f in 1 0; do
  for w in D B C; do
    LC_SUBPIX_FUSED=$f python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/w${w}_$f.json 2>/dev/null
    python -c "
import json
d=json.loads(open('gpurun_out/w${w}_$f.json').read().strip().splitlines()[-1]); print('$w', 'fused=$f', round(d['value'],1), round(d['e2e']['value'],1), d['clocks']['sm_mhz'])"
  done
done
