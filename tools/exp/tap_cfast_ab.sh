#!/bin/bash
# A/B of the channel-fastest epilogue task order of the K8 tap kernels
# (LC_TAP_CFAST): GPU tests with it on, interleaved C / D bench lines, and
# the two K8 kernels' launch-list times.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for r in 1 0 1 0; do
  for w in C D; do
    LC_TAP_CFAST=$r python bench.py --workload $w --steps 10 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('cfast=$r $w', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'clk', d['clocks']['sm_mhz'])"
  done
done
for r in 1 0; do
  LC_TAP_CFAST=$r ncu --metrics gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum --clock-control none -k regex:tap_tc --csv \
      --log-file gpurun_out/tap_cfast_$r.csv python tools/profile_step.py C 1 > /dev/null 2>&1
  python - <<PY
import csv, collections
rows = list(csv.DictReader(l for l in open('gpurun_out/tap_cfast_$r.csv') if l.startswith('"')))
agg = collections.defaultdict(list)
for r in rows:
    agg[(r['Kernel Name'][:24], r['Metric Name'])].append(float(r['Metric Value'].replace(',', '')))
for k, v in sorted(agg.items()):
    print('cfast=$r', k, len(v), round(sum(v) / len(v), 1))
PY
done
