"""C with the swap off / async / sync and uncached: device ms per video
(graph replay), to bound what the swap's DMA costs the compute."""
import json
import sys

sys.path.insert(0, ".")
import paper_2510_05367_b200 as lc  # noqa: E402

C = {"run.frames": 25, "run.height": 576, "run.width": 1024, "codec.stages": 3, "codec.width": 128,
     "unet.base_channels": 320, "unet.depth": 3, "sampler.steps": 25, "cache.n": 2, "swap.mode": "async"}
ctx = lc.Context(0)
rows = {}
for label, over in [("async", {}), ("off", {"swap.mode": "off"}), ("async2", {}),
                    ("uncached", {"cache.enabled": "false", "swap.mode": "off"}), ("off2", {"swap.mode": "off"})]:
    ctx.configure(lc.config_text(dict(C, **over), base=lc.DEFAULT_CONFIG))
    for _ in range(2):
        ctx.run_pipeline()
    ms = []
    for _ in range(6):
        _, _, rep = ctx.run_pipeline()
        ms.append(rep["device_ms"]["total"])
    ms.sort()
    rows[label] = {"median_ms": ms[len(ms) // 2], "min_ms": ms[0], "hbm_peak_gb": rep["hbm_peak_bytes"] / 1e9,
                   "stall_ms": rep["timeline"]["stall_ms"]}
    print(label, json.dumps(rows[label]), flush=True)
