"""A/B check of an engine switch on a bench workload: runs the resident
pipeline once and saves the video (argv[2]); with argv[3] compares against a
saved video.  Usage: LC_X=... python tools/exp/thin_check.py B out.npy [ref.npy]"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench
import paper_2510_05367_b200 as lc
wl = sys.argv[1]
text = lc.config_text(bench.WORKLOADS[wl], base=lc.DEFAULT_CONFIG)
ctx = lc.Context(0)
ctx.configure(text)
ctx.set_decode_slice(4)
kv = lc.parse_config(text)
ctx.upload_latent(lc.randn(lc.derive_seed(int(kv["run.seed"]), 1), ctx.latent_elems()))
for _ in range(3):
    rep = ctx.run_resident()
v = ctx.download_video()
np.save(sys.argv[2], v)
print("device ms", rep["device_ms"], "launches", rep["kernel_launches"])
if len(sys.argv) > 3:
    r = np.load(sys.argv[3])
    print("rel L2 vs ref", float(np.linalg.norm(v - r) / np.linalg.norm(r)), "max abs", float(np.abs(v - r).max()))
