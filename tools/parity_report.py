"""Measured GPU-vs-oracle parity (relative L2) on the committed golden cases
and live oracle runs; writes a JSON summary (profiles/parity_<round>.json)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import lco  # noqa: E402

import paper_2510_05367_b200 as lc  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
out = {}
ctx = lc.Context(0)
for name in ["tiny", "tiny_ancestral", "tiny_ddim_m1", "tiny_halo_none", "tiny_k5", "tiny_image", "default", "config_a",
             "b_frame0", "b_frame0_ancestral", "b_frame0_ddim", "b_frame0_image", "b_frame0_fixed_k5", "c_frame0",
             "c_frame0_none_s2", "c_frame0_fixed_k5_s2", "b_frame0_none"]:
    g = np.load(os.path.join(GOLD, f"{name}.npz"))
    text = str(g["config"])
    ctx.configure(text)
    video, lat, rep = ctx.run_pipeline(want_latent=True)
    out[name] = {"latent_rel_l2": lc.rel_l2(lat, g["latent"]), "video_rel_l2": lc.rel_l2(video, g["video"]),
                 "video_max_abs": float(np.abs(video - g["video"]).max()),
                 "full_steps": rep["mac"]["full_steps"], "cached_steps": rep["mac"]["cached_steps"]}
    print(name, json.dumps(out[name]), flush=True)
path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "parity.json")
json.dump(out, open(path, "w"), indent=1)
