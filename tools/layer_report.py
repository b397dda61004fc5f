"""Per-conv-launch roofline table of one resident pipeline run (CUDA events
around every conv launch, engine conv profiler): device time, algorithmic
and executed TFLOP/s, fraction of the measured sustained tensor peak, and
the launch's tile / schedule.  Usage: python tools/layer_report.py B|C [out.json] [key=value ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2510_05367_b200 as lc  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "B"
over = dict(bench.WORKLOADS[wl])
out_json = None
for arg in sys.argv[2:]:
    if "=" in arg:
        k, v = arg.split("=", 1)
        over[k] = v
    else:
        out_json = arg
text = lc.config_text(over, base=lc.DEFAULT_CONFIG)
ctx = lc.Context(0)
ctx.configure(text)
kv = lc.parse_config(text)
ctx.upload_latent(lc.randn(lc.derive_seed(int(kv["run.seed"]), 1), ctx.latent_elems()))
for _ in range(3):
    ctx.run_resident()
ctx.set_conv_profile(True)
ctx.run_resident()
recs = ctx.conv_profile_records()
ctx.set_conv_profile(False)
peak, _ = bench.peaks()
rows = []
for i, r in enumerate(recs):
    s = r["ms"] / 1e3
    rows.append({"i": i, "us": r["ms"] * 1e3, "alg_tflops": r["alg_flops"] / s / 1e12 if s else 0,
                 "exec_tflops": r["exec_flops"] / s / 1e12 if s else 0, "desc": r["desc"]})
tot = sum(r["us"] for r in rows)
print(f"{wl}: {len(rows)} conv launches, {tot / 1e3:.3f} ms; peak (sustained) {peak} TFLOP/s")
print(f"{'#':>3} {'us':>8} {'alg TF/s':>9} {'exec TF/s':>9} {'exec/peak':>9}  launch")
for r in rows:
    print(f"{r['i']:>3} {r['us']:8.1f} {r['alg_tflops']:9.1f} {r['exec_tflops']:9.1f} {r['exec_tflops'] / peak:9.2f}  "
          f"{r['desc']}")
if out_json:
    json.dump({"workload": wl, "peak_tflops": peak, "rows": rows}, open(out_json, "w"), indent=1)
