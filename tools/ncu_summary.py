"""Summarise an ncu --metrics gpu__time_duration.sum launch list (last step)."""
import csv, collections, sys
path = sys.argv[1]; steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
rows = list(csv.reader(open(path)))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]; data = rows[hdr_i + 1:]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
mn = hdr.index("Metric Name") if "Metric Name" in hdr else None
gi = hdr.index("Grid Size") if "Grid Size" in hdr else None
recs = [(r[ki].split("(")[0].split("::")[-1], float(r[vi].replace(",", "")), r[gi] if gi else "") for r in data if len(r) > vi and (mn is None or r[mn] == "gpu__time_duration.sum")]
last = recs[len(recs) - len(recs) // steps:]
agg = collections.defaultdict(lambda: [0, 0.0])
for k, v, _ in last:
    agg[k][0] += 1; agg[k][1] += v
tot = sum(v for _, v, _ in last)
print(f"last step: {len(last)} launches, {tot/1e6:.3f} ms (ncu, serialized, clock-control none)")
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"  {v/1e6:8.3f} ms {100*v/tot:5.1f}%  x{c:<3d} {k}")
if "-v" in sys.argv:
    for k, v, g in last: print(f"    {v/1e3:9.1f} us  {k:24s} {g}")
