"""GPU stress check (not part of the suite): many seeded random
configurations -- depth 1-4, kernels 1-9, cache depths, halos, samplers,
image mode, swap modes, frame counts -- through ONE reused context (config
switching, arena re-layout, graph invalidation) against the CPU oracle at
the 1e-3 bar.  Usage: python tools/stress_random.py [n] [seed]"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import lco  # noqa: E402

import paper_2510_05367_b200 as lc  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 4242)
    oracle = lco.Restatement()
    ctx = lc.Context(0)
    worst, done, fails = 0.0, 0, []
    while done < n:
        depth = int(rng.integers(1, 5))
        stages = int(rng.integers(1, 3))
        unit = (1 << depth) * (1 << stages)
        over = {
            "run.frames": int(rng.integers(1, 6)), "run.height": unit * int(rng.integers(1, 4)),
            "run.width": unit * int(rng.integers(1, 4)), "unet.depth": depth, "codec.stages": stages,
            "unet.base_channels": int(rng.choice([8, 16, 32, 64])), "codec.width": int(rng.choice([8, 16, 64])),
            "unet.kernel": int(rng.choice([1, 3, 3, 3, 5, 7, 9])), "unet.cache_depth": int(rng.integers(0, depth)),
            "sampler.steps": int(rng.integers(2, 8)), "sampler.kind": str(rng.choice(["euler", "ddim", "ancestral"])),
            "cache.n": int(rng.integers(1, 5)), "cache.enabled": str(rng.choice(["true", "true", "false"])),
            "swap.mode": str(rng.choice(["off", "sync", "async", "async"])),
            "chunk.enabled": str(rng.choice(["true", "false"])), "chunk.halo": str(rng.choice(["exact", "none", "fixed"])),
            "chunk.halo_px": int(rng.integers(0, 4)), "chunk.eta": int(rng.choice([1, 2])),
            "chunk.omega": int(rng.choice([1, 2])),
            "chunk.targets": str(rng.choice(["u0", "stem,u0", "d0,u0,head", "stem,d0,u0,head"])),
            "decode.sliced": str(rng.choice(["true", "false"])), "run.mode": str(rng.choice(["text", "text", "image"])),
            "run.seed": int(rng.integers(0, 1000)),
        }
        text = lc.config_text(over, base=lc.DEFAULT_CONFIG)
        try:
            lc.check_config(text)
        except lc.LightCacheError:
            continue
        ctx.configure(text)
        ctx.set_decode_slice(int(rng.integers(1, 6)))
        video, lat, _ = ctx.run_pipeline(want_latent=True)
        kv = lco.parse_text(lc.DEFAULT_CONFIG)
        kv.update({k: str(v) for k, v in over.items()})
        wv, wl = oracle.run_pipeline(kv)
        ev, el = lc.rel_l2(video, wv), lc.rel_l2(lat, wl)
        worst = max(worst, ev, el)
        if not (ev < 1e-3 and el < 1e-3 and np.isfinite(video).all()):
            fails.append({"over": over, "video": ev, "latent": el})
        done += 1
        print(done, f"video {ev:.2e} latent {el:.2e}", json.dumps(over), flush=True)
    print(json.dumps({"configs": done, "worst_rel_l2": worst, "failures": fails}))
    ctx.close()
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
