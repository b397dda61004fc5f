"""Generate the committed golden fixtures from the reference itself.

Runs the UNMODIFIED reference (oracle/_ref, compiled in place from
/root/reference/proj/src by oracle/Makefile) and stores its outputs as
compressed .npz under tests/golden/.  The B/C frame-0 slices (SURVEY.md
section 8c: frame 0 of a T-frame run is bit-identical to the T=1 run) are
too slow for the single-threaded reference and are produced by the
restatement oracle/lc_oracle.c (the reference's RunResult carries only the
video, not the final latent), and their VIDEOS are then pinned against the
reference itself: `pin_b0` / `pin_c0` / `pin_bvar` run oracle/_ref's
run_pipeline on the same config (about 5 min for B, 65 min for C, single
thread), assert the restatement's video is bit-identical and record
`video_source = "oracle/_ref"` plus the reference's wall time in the npz.

Usage:  python tests/golden/make_golden.py [small|b0|c0|bvar|chunkvar|pin_b0|pin_c0|pin_bvar|pin_chunkvar|metrics|timelines|sampler]...
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import lco  # noqa: E402

DEFAULT = open(os.path.join(HERE, "default.cfg")).read()

SMALL = {
    "default": {},
    "tiny": {"run.frames": 2, "run.height": 32, "run.width": 32, "sampler.steps": 6},
    "tiny_ancestral": {"run.frames": 2, "run.height": 32, "run.width": 32, "sampler.steps": 6,
                       "sampler.kind": "ancestral"},
    "tiny_ddim_m1": {"run.frames": 2, "run.height": 32, "run.width": 32, "sampler.steps": 6,
                     "sampler.kind": "ddim", "unet.cache_depth": 1},
    "tiny_halo_none": {"run.frames": 2, "run.height": 32, "run.width": 32, "sampler.steps": 6,
                       "chunk.halo": "none", "chunk.targets": "stem,d0,u0,head"},
    "tiny_k5": {"run.frames": 2, "run.height": 32, "run.width": 32, "sampler.steps": 6, "unet.kernel": 5},
    "tiny_image": {"run.frames": 2, "run.height": 32, "run.width": 32, "sampler.steps": 6, "run.mode": "image"},
    "config_a": {"run.height": 128, "run.width": 128, "cache.n": 3, "chunk.eta": 2, "chunk.omega": 1},
}
B0 = {"run.frames": 1, "run.height": 512, "run.width": 512, "codec.stages": 3, "codec.width": 128,
      "unet.base_channels": 320, "unet.depth": 3, "sampler.steps": 4, "cache.n": 2}
C0 = {"run.frames": 1, "run.height": 576, "run.width": 1024, "codec.stages": 3, "codec.width": 128,
      "unet.base_channels": 320, "unet.depth": 3, "sampler.steps": 25, "cache.n": 2, "swap.mode": "async"}


# B frame-0 variants (samplers and image mode at the B shape)
BVAR = {
    "b_frame0_ancestral": dict(B0, **{"sampler.kind": "ancestral"}),
    "b_frame0_ddim": dict(B0, **{"sampler.kind": "ddim"}),
    "b_frame0_image": dict(B0, **{"run.mode": "image"}),
}


# halo kinds at the B / C frame-0 shapes (fixed and none halos
# at the bench shapes; C at 2 steps = one N=2 cache period)
CHUNKVAR = {
    "b_frame0_fixed_k5": dict(B0, **{"unet.kernel": 5, "chunk.halo": "fixed", "chunk.halo_px": 1}),
    "c_frame0_none_s2": dict(C0, **{"sampler.steps": 2, "chunk.halo": "none"}),
    "b_frame0_none": dict(B0, **{"chunk.halo": "none"}),
    "c_frame0_fixed_k5_s2": dict(C0, **{"sampler.steps": 2, "unet.kernel": 5, "chunk.halo": "fixed",
                                        "chunk.halo_px": 1}),
}


def kv_of(over):
    kv = lco.parse_text(DEFAULT)
    kv.update({k: str(v) for k, v in over.items()})
    return kv


def small():
    ref = lco.Reference()
    for name, over in SMALL.items():
        kv = kv_of(over)
        t = time.time()
        video, report, macs = ref.run_pipeline(kv)
        # final latent via the restatement (the reference API returns only
        # the video); the restatement's video must equal the reference's
        v2, lat = lco.Restatement().run_pipeline(kv)
        assert np.array_equal(video, v2), name
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), video=video, latent=lat,
                            macs=np.array(macs, np.int64),
                            config=np.array(lco.to_text(kv)), report=np.array(json.dumps(report)))
        print(name, f"{time.time() - t:.1f}s", flush=True)
    # integer contracts
    plans = {}
    for total in range(1, 13):
        for n in range(1, 6):
            k, f = ref.plan_steps(total, n)
            plans[f"{total}_{n}"] = np.stack([k, f])
    np.savez_compressed(os.path.join(HERE, "plans.npz"), **plans)
    splits = {}
    for (h, w) in [(8, 8), (16, 16), (32, 32), (72, 128), (9, 16), (36, 64)]:
        for eta in (1, 2, 3, 4):
            for omega in (1, 2, 4):
                if h % eta or w % omega:
                    continue
                for hk, hp in ((0, 0), (1, 1), (1, 3), (2, 0)):
                    for k in (1, 3, 5):
                        regions, halo = ref.split(h, w, eta, omega, hk, hp, k)
                        splits[f"{h}_{w}_{eta}_{omega}_{hk}_{hp}_{k}"] = np.concatenate(
                            [regions.reshape(-1), [halo]])
    np.savez_compressed(os.path.join(HERE, "splits.npz"), **splits)
    nums = {}
    for name, over in dict(SMALL, b=dict(B0, **{"run.frames": 16}), c=dict(C0, **{"run.frames": 25})).items():
        nums[name] = np.array(ref.model_numbers(kv_of(over)), np.int64)
    np.savez_compressed(os.path.join(HERE, "model_numbers.npz"), **nums)


def slice0(name, over):
    kv = kv_of(over)
    t = time.time()
    video, lat = lco.Restatement().run_pipeline(kv)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), video=video, latent=lat,
                        config=np.array(lco.to_text(kv)), seconds=np.array(time.time() - t))
    print(name, f"{time.time() - t:.1f}s", flush=True)


def pin(name, over):
    """Run the UNMODIFIED reference on a frame-0 slice config and pin the
    committed restatement video against it bit for bit."""
    path = os.path.join(HERE, f"{name}.npz")
    d = dict(np.load(path))
    kv = kv_of(over)
    assert str(d["config"]) == lco.to_text(kv), name
    t = time.time()
    video, report, macs = lco.Reference().run_pipeline(kv)
    secs = time.time() - t
    if not np.array_equal(video, d["video"]):
        diff = np.abs(video - d["video"]).max()
        raise SystemExit(f"{name}: restatement video differs from oracle/_ref (max abs {diff})")
    d["video"] = video
    d["video_source"] = np.array("oracle/_ref")
    d["ref_seconds"] = np.array(secs)
    d["macs"] = np.array(macs, np.int64)
    np.savez_compressed(path, **d)
    print(name, "pinned to oracle/_ref", f"{secs:.1f}s", flush=True)


def metrics():
    """psnr / ssim per frame (proj/src/metrics.cpp) from the reference on
    seeded videos: a perturbed pair, an identical pair, and the tiny
    baseline-vs-cached pipeline videos (the compare/sweep use)."""
    ref = lco.Reference()
    rng = np.random.default_rng(11)
    out = {}
    a = rng.random((1, 3, 3, 20, 29)).astype(np.float32)
    b = np.clip(a + 0.03 * rng.standard_normal(a.shape), 0, 1).astype(np.float32)
    for name, (x, y) in {"noise": (a, b), "same": (a, a.copy())}.items():
        ps, ss = ref.video_metrics(x[0], y[0], 1.0)
        out[name + "_a"], out[name + "_b"], out[name + "_psnr"], out[name + "_ssim"] = x, y, ps, ss
    tiny = dict(SMALL["tiny"])
    base = kv_of(dict(tiny, **{"cache.enabled": "false", "chunk.enabled": "false", "decode.sliced": "false",
                               "swap.mode": "off"}))
    var = kv_of(dict(tiny, **{"cache.n": 3}))
    va = ref.run_pipeline(base)[0]
    vb = ref.run_pipeline(var)[0]
    ps, ss = ref.video_metrics(va[0], vb[0], 1.0)
    out.update(pipe_a=va, pipe_b=vb, pipe_psnr=ps, pipe_ssim=ss)
    np.savez_compressed(os.path.join(HERE, "metrics.npz"), **out)


# sampler operator cases: (config overrides, kind, t, guidance); the schedule
# is the config's spaced one (train_steps 50 -> sampler.steps)
SAMPLER_CASES = {
    "euler_t24": ({}, 2, 24, 1.5),
    "euler_t0": ({}, 2, 0, 1.5),
    "ddim_t12": ({}, 1, 12, 2.0),
    "ddim_t0": ({}, 1, 0, 0.0),
    "ancestral_t7": ({}, 0, 7, 1.5),
    "ancestral_t0": ({}, 0, 0, 1.5),
    "euler_s6_t5": ({"sampler.steps": 6}, 2, 5, 7.5),
    "ancestral_s6_t3": ({"sampler.steps": 6, "schedule.train_steps": 1000, "schedule.beta_min": 0.00085,
                         "schedule.beta_max": 0.012}, 0, 3, 1.0),
}


def sampler():
    """cfg_combine + reverse_step_* (proj/src/sampler.cpp:95-133) from the
    reference on seeded operands: n = 1027 (a 16-byte vector body and a
    scalar tail on the device)."""
    ref = lco.Reference()
    rng = np.random.default_rng(23)
    n = 1027
    out = {}
    for name, (over, kind, t, g) in SAMPLER_CASES.items():
        kv = kv_of(over)
        x = rng.standard_normal(n).astype(np.float32)
        eu = rng.standard_normal(n).astype(np.float32)
        ec = rng.standard_normal(n).astype(np.float32)
        seed = int(rng.integers(1, 1 << 62))
        out[name + "_x"], out[name + "_eu"], out[name + "_ec"] = x, eu, ec
        out[name + "_args"] = np.array([kind, t, seed], np.uint64)
        out[name + "_g"] = np.array(g, np.float64)
        out[name + "_config"] = np.array(lco.to_text(kv))
        out[name + "_out"] = ref.sampler_step(kv, kind, t, x, eu, ec, g, seed)
    np.savez_compressed(os.path.join(HERE, "sampler.npz"), **out)


SIM_TINY = {"run.frames": 2, "run.height": 32, "run.width": 32, "sampler.steps": 6, "run.seed": 7,
            "swap.simulate": "true"}
SIM = {
    # acceptance C8 (proj/tests/acceptance_main.cpp:384-418): default config
    "c8_off": {"swap.simulate": "true", "swap.mode": "off"},
    "c8_async": {"swap.simulate": "true", "swap.mode": "async"},
    "c8_sync": {"swap.simulate": "true", "swap.mode": "sync"},
    # test_pipeline.cpp:250-260 tiny_config
    "tiny_async": dict(SIM_TINY, **{"swap.mode": "async"}),
    "tiny_sync_n3": dict(SIM_TINY, **{"swap.mode": "sync", "cache.n": 3}),
    "tiny_async_n1": dict(SIM_TINY, **{"swap.mode": "async", "cache.n": 1}),
    "slow_link": dict(SIM_TINY, **{"swap.mode": "async", "swap.bandwidth": 1e6}),
    "slow_link_sync": dict(SIM_TINY, **{"swap.mode": "sync", "swap.bandwidth": 5e6, "swap.latency": 1e-3}),
    "mid_link_n3": dict(SIM_TINY, **{"swap.mode": "async", "swap.bandwidth": 3e7, "cache.n": 3,
                                     "sampler.steps": 7}),
    "image_m1_chunks": dict(SIM_TINY, **{"swap.mode": "async", "run.mode": "image", "swap.bandwidth": 2e7,
                                         "unet.cache_depth": 1, "chunk.targets": "stem,d1,u0,u1",
                                         "chunk.eta": 4, "chunk.omega": 2}),
    "no_cache": dict(SIM_TINY, **{"swap.mode": "async", "cache.enabled": "false"}),
    "zero_latency": dict(SIM_TINY, **{"swap.mode": "async", "swap.latency": 0, "swap.mac_rate": 3e9}),
}


def timelines():
    """Simulated transfer-engine timelines (swap.simulate = true,
    proj/src/swap.cpp:141-374) from the reference's run_pipeline."""
    ref = lco.Reference()
    out = {}
    for name, over in SIM.items():
        kv = kv_of(over)
        ev, mk, st = ref.timeline(kv)
        out[name + "_events"] = ev
        out[name + "_info"] = np.array([mk, st], np.int64)
        out[name + "_config"] = np.array(lco.to_text(kv))
    np.savez_compressed(os.path.join(HERE, "timelines.npz"), **out)


if __name__ == "__main__":
    what = sys.argv[1:] or ["small"]
    if "small" in what:
        small()
    if "b0" in what:
        slice0("b_frame0", B0)
    if "c0" in what:
        slice0("c_frame0", C0)
    if "bvar" in what:
        for name, over in BVAR.items():
            slice0(name, over)
    if "pin_b0" in what:
        pin("b_frame0", B0)
    if "pin_c0" in what:
        pin("c_frame0", C0)
    if "chunkvar" in what:
        for name, over in CHUNKVAR.items():
            slice0(name, over)
    if "pin_chunkvar" in what:
        for name, over in CHUNKVAR.items():
            pin(name, over)
    if "pin_bvar" in what:
        for name, over in BVAR.items():
            pin(name, over)
    if "metrics" in what:
        metrics()
    if "sampler" in what:
        sampler()
    if "timelines" in what:
        timelines()
