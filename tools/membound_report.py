"""Achieved DRAM GB/s of the non-conv (HBM/L2-bound) kernels of one run from
an ncu launch list with gpu__time_duration.sum, dram__bytes_read.sum and
dram__bytes_write.sum (tools/refresh_profiles.sh writes one).  Inputs that
were just written by the previous kernel are often still in the 126 MB L2,
so DRAM bytes can undercount the kernel's traffic; the table says so.
Usage: python tools/membound_report.py launch.csv [runs]"""
import collections
import csv
import sys

path, runs = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 3
rows = list(csv.reader(open(path)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, ii, mi, vi = h.index("Kernel Name"), h.index("ID"), h.index("Metric Name"), h.index("Metric Value")
per = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    d = per.setdefault(int(r[ii]), {"name": r[ki].split("(")[0].split("::")[-1]})
    d[r[mi]] = float(r[vi].replace(",", ""))
launches = list(per.values())
last = launches[len(launches) - len(launches) // runs:]
agg = collections.OrderedDict()
for d in last:
    if "conv_tc" in d["name"]:
        continue
    a = agg.setdefault(d["name"], [0, 0.0, 0.0])
    a[0] += 1
    a[1] += d["gpu__time_duration.sum"]
    a[2] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
print(f"{'kernel':28s} {'launches':>8s} {'us/launch':>10s} {'DRAM MB/launch':>15s} {'DRAM GB/s':>10s}")
for k, (n, ns, b) in agg.items():
    print(f"{k:28s} {n:8d} {ns / n / 1e3:10.1f} {b / n / 1e6:15.1f} {b / ns:10.0f}")
