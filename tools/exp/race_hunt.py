"""Repeat a config in fresh processes and compare each video with the
oracle (intermittent-race hunt)."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
CFG = {"run.frames": 3, "run.height": 96, "run.width": 160, "sampler.steps": 3, "codec.width": 64}

if len(sys.argv) > 1:
    import paper_2510_05367_b200 as lc
    ctx = lc.Context(0)
    ctx.configure(lc.config_text(CFG, base=lc.DEFAULT_CONFIG))
    for k in range(int(sys.argv[2])):
        v, _, _ = ctx.run_pipeline()
        np.save(f"{sys.argv[1]}_{k}.npy", v)
    sys.exit(0)

import lco
import paper_2510_05367_b200 as lc
kv = lco.parse_text(lc.DEFAULT_CONFIG)
kv.update({k: str(v) for k, v in CFG.items()})
want, _ = lco.Restatement().run_pipeline(kv)
for fused in ("1", "0"):
    for rep in range(int(os.environ.get("RH_PROCS", "4"))):
        env = dict(os.environ, LC_SUBPIX_FUSED=fused)
        r = subprocess.run([sys.executable, __file__, "/tmp/rh", "4"], env=env, capture_output=True, text=True)
        if r.returncode:
            print("FAILED", r.stderr[-1500:])
            continue
        errs = []
        for k in range(4):
            v = np.load(f"/tmp/rh_{k}.npy")
            errs.append(round(lc.rel_l2(v, want), 6))
        print("fused", fused, "proc", rep, errs, flush=True)
