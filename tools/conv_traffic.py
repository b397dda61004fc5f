"""From an ncu launch list with gpu__time_duration.sum, dram__bytes_read.sum and
dram__bytes_write.sum, compute the average DRAM traffic per conv_tc launch of
the last step and update profiles/conv_traffic.json[workload]."""
import csv
import json
import os
import sys

path, workload, steps = sys.argv[1], sys.argv[2], int(sys.argv[3])
rows = list(csv.reader(open(path)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, ii, mi, vi = h.index("Kernel Name"), h.index("ID"), h.index("Metric Name"), h.index("Metric Value")
per = {}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    d = per.setdefault(int(r[ii]), {"name": r[ki]})
    d[r[mi]] = float(r[vi].replace(",", ""))
launches = [per[k] for k in sorted(per)]
last = launches[len(launches) - len(launches) // steps:]
conv = [d for d in last if "conv_tc" in d["name"]]
byts = sum(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in conv)
tms = sum(d["gpu__time_duration.sum"] for d in conv)
out_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "conv_traffic.json")
data = json.load(open(out_path)) if os.path.exists(out_path) else {}
data[workload] = byts / len(conv)
data[workload + "_detail"] = {"launches": len(conv), "dram_bytes_total": byts, "ns_total": tms,
                              "source": os.path.basename(path)}
json.dump(data, open(out_path, "w"), indent=1)
print(json.dumps(data[workload + "_detail"]), "bytes/launch", byts / len(conv))
