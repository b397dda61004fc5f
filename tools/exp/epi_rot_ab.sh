#!/bin/bash
# A/B of the epilogue column-group rotation (LC_EPI_ROT): GPU tests with it
# on, then interleaved C bench lines and per-layer stem time.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
python -m pytest tests/test_gpu_conv.py tests/test_gpu_pipeline.py -x -q 2>&1 | tail -1
for r in 1 0 1 0 1 0; do
  LC_EPI_ROT=$r python bench.py --steps 10 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('rot=$r', round(d['value'],1), 'conv_ms', round(d['roofline']['conv_ms_per_step'],2), 'clk', d['clocks']['sm_mhz'])"
done
for r in 1 0; do
  LC_EPI_ROT=$r python tools/layer_report.py C gpurun_out/rot_layers_$r.json > gpurun_out/rot_layers_$r.txt 2>&1
  python - <<PY
tot=0
for l in open('gpurun_out/rot_layers_$r.txt'):
    t=l.split()
    if len(t)>6 and t[0].isdigit() and 'K64 ' in l: tot+=float(t[1])
print('rot=$r stem us per video', round(tot,1))
PY
done
