"""Print the swap timeline of one resident run (transfer durations, host-link
GB/s, seam stalls) for a bench workload."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2510_05367_b200 as lc  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "B"
over = dict(bench.WORKLOADS[wl])
for kv in sys.argv[2:]:
    k, v = kv.split("=")
    over[k] = v
ctx = lc.Context(0)
ctx.configure(lc.config_text(over, base=lc.DEFAULT_CONFIG))
kv = lc.parse_config(lc.config_text(over, base=lc.DEFAULT_CONFIG))
ctx.upload_latent(lc.randn(lc.derive_seed(int(kv["run.seed"]), 1), ctx.latent_elems()))
for _ in range(3):
    rep = ctx.run_resident()
ev = rep["timeline"]["events"]
print("device ms", rep["device_ms"], "stall ms", rep["timeline"]["stall_ms"])
open_x, open_a = {}, None
tot_bytes, tot_ms = 0, 0.0
for kind, step, nbytes, t in ev:
    if kind == "xfer_start":
        open_x.setdefault(step, []).append(t)
    elif kind == "xfer_end":
        t0 = open_x[step].pop(0)
        tot_bytes += nbytes
        tot_ms += t - t0
        print(f"  xfer step {step}: {nbytes / 1e6:.1f} MB in {t - t0:.3f} ms = {nbytes / (t - t0) / 1e6:.1f} GB/s  [{t0:.3f}..{t:.3f}]")
    elif kind == "await_start":
        open_a = t
    elif kind == "await_end":
        print(f"  await step {step}: {t - open_a:.3f} ms at {open_a:.3f}")
    elif kind in ("compute_start", "compute_end"):
        print(f"  {kind} {step} at {t:.3f}")
