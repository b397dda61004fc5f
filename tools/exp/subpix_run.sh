#!/bin/bash
python tools/exp/subpix_ab.py > gpurun_out/subpix_ab.txt 2>&1
cat gpurun_out/subpix_ab.txt
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_all.log 2>&1; tail -3 gpurun_out/gpu_all.log
for f in 1 0; do
  LC_SUBPIX_FUSED=$f python bench.py --workload D --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/d_$f.json 2>/dev/null
  LC_SUBPIX_FUSED=$f python bench.py --workload B --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b_$f.json 2>/dev/null
  python -c "
import json
for w in 'db':
    d=json.loads(open('gpurun_out/%s_$f.json'%w).read().strip().splitlines()[-1]); print(w, 'fused=$f', round(d['value']), round(d['e2e']['value']), d['clocks']['sm_mhz'])"
done
