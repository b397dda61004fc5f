"""C on one box: the drop-in call (run_pipeline, pageable host buffers, one
video at a time) vs resident graph replays back to back vs the pipelined
e2e path -- ms per video each, plus the run_pipeline report's device_ms."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2510_05367_b200 as lc  # noqa: E402
import bench  # noqa: E402

text = lc.config_text(bench.WORKLOADS["C"], base=lc.DEFAULT_CONFIG)
ctx = lc.Context(0)
ctx.configure(text)
x0 = lc.PinnedArray(ctx.latent_elems())
x0.array[:] = lc.randn(lc.derive_seed(42, 1), ctx.latent_elems())
vid = lc.PinnedArray(ctx.video_elems())
out = {}
for _ in range(3):
    ctx.run_pipeline(x0.array.copy())
wall, dev = [], []
for _ in range(6):
    t = time.perf_counter()
    _, _, rep = ctx.run_pipeline(x0.array.copy())
    wall.append((time.perf_counter() - t) * 1e3)
    dev.append(rep["device_ms"]["total"])
out["run_pipeline_wall_ms"] = sorted(wall)[3]
out["run_pipeline_device_ms"] = sorted(dev)[3]
out["run_pipeline_device_ms_parts"] = rep["device_ms"]
ctx.upload_latent(x0.array)
for _ in range(3):
    ctx.run_resident()
ctx.timer_start()
for _ in range(10):
    ctx.run_resident_async()
ctx.wait()
out["resident_ms"] = ctx.timer_stop() / 10
for _ in range(2):
    ctx.run_e2e(x0, vid)
ctx.timer_start()
for _ in range(10):
    ctx.run_e2e_async(x0, vid)
ctx.wait()
out["e2e_ms"] = ctx.timer_stop() / 10
for _ in range(3):
    _, _, rep = ctx.run_pipeline(x0.array.copy())
out["run_pipeline_device_ms_after"] = rep["device_ms"]["total"]
out["stall_ms_run_pipeline"] = rep["timeline"]["stall_ms"]
print(json.dumps(out, indent=1))
