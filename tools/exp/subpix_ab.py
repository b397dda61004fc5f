"""A/B of the decoder's last stage: fused K8 (default) vs tap-to-N conv +
gather (LC_SUBPIX_FUSED=0), run in two processes; prints whether the videos
are bit-identical and their max abs difference."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

CFGS = {
    "tiny": {"run.frames": 2, "run.height": 32, "run.width": 32, "sampler.steps": 6},
    "odd": {"run.frames": 3, "run.height": 96, "run.width": 160, "sampler.steps": 3, "codec.width": 64},
    "w192": {"run.frames": 2, "run.height": 64, "run.width": 64, "sampler.steps": 2, "codec.width": 192},
    "k5": {"run.frames": 2, "run.height": 32, "run.width": 32, "sampler.steps": 3, "unet.kernel": 5},
    "headchunk": {"run.frames": 2, "run.height": 64, "run.width": 96, "sampler.steps": 3, "chunk.halo": "none",
                  "chunk.targets": "stem,u0,head", "chunk.eta": 2, "chunk.omega": 3},
    "B1": {"run.frames": 1, "run.height": 512, "run.width": 512, "codec.stages": 3, "codec.width": 128,
           "unet.base_channels": 320, "unet.depth": 3, "sampler.steps": 4, "cache.n": 2},
}

if len(sys.argv) > 2:
    import paper_2510_05367_b200 as lc
    name, path = sys.argv[1], sys.argv[2]
    ctx = lc.Context(0)
    ctx.configure(lc.config_text(CFGS[name], base=lc.DEFAULT_CONFIG))
    v, _, _ = ctx.run_pipeline()
    np.save(path, v)
    sys.exit(0)

for name in CFGS:
    outs = []
    for fused in ("1", "0"):
        path = f"/tmp/subpix_{name}_{fused}.npy"
        env = dict(os.environ, LC_SUBPIX_FUSED=fused)
        r = subprocess.run([sys.executable, __file__, name, path], env=env, capture_output=True, text=True)
        if r.returncode:
            print(name, "FAILED", r.stderr[-2000:])
            break
        outs.append(np.load(path))
    if len(outs) == 2:
        a, b = outs
        line = [name, "bit-identical" if np.array_equal(a, b) else "DIFF", float(np.abs(a - b).max()),
                float(np.abs(b).max())]
        if name != "B1":
            sys.path.insert(0, os.path.join(ROOT, "oracle"))
            import lco
            import paper_2510_05367_b200 as lc
            kv = lco.parse_text(lc.DEFAULT_CONFIG)
            kv.update({k: str(v) for k, v in CFGS[name].items()})
            want, _ = lco.Restatement().run_pipeline(kv)
            line += ["rel_l2 fused", lc.rel_l2(a, want), "old", lc.rel_l2(b, want)]
            err = np.abs(a.reshape(want.shape) - want)
            idx = np.unravel_index(np.argmax(err), err.shape)
            line += ["worst at", idx]
        print(*line)
