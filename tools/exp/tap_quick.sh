#!/bin/bash
python tools/exp/subpix_ab.py 2>&1 | cut -c1-60
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:tap_tc \
    --log-file gpurun_out/tapq.csv python tools/profile_step.py B 1 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=list(csv.reader(open("gpurun_out/tapq.csv")))
hi=[i for i,r in enumerate(rows) if r and r[0]=="ID"]
h=rows[hi[0]]; data=rows[hi[0]+1:]
ki=h.index("Kernel Name"); mi=h.index("Metric Name"); vi=h.index("Metric Value"); ii=h.index("ID")
per=collections.defaultdict(dict)
for r in data:
    per[int(r[ii])][r[mi]]=float(r[vi].replace(",","")); per[int(r[ii])]["name"]=r[ki]
for k in sorted(per):
    v=per[k]
    print("  %3d %-30s %7.1f us %7.1f MB" % (k, v["name"][:30], v["gpu__time_duration.sum"]/1e3, (v["dram__bytes_read.sum"]+v["dram__bytes_write.sum"])/1e6))
PY
