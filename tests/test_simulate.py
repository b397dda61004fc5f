"""The simulated transfer engine (swap.simulate = true): a virtual ns clock
advanced by every convolution call's MACs at swap.mac_rate, one transfer
channel of latency + bytes / bandwidth per job (proj/src/swap.cpp:141-374,
driven by pipeline.cpp:119-207 and cache.cpp:43-122).

The product's host-side model (lc_simulate_timeline) is checked event by
event against the reference's own timelines: the committed fixtures
(tests/golden/timelines.npz, made by make_golden.py from oracle/_ref) and,
when oracle/_ref is built, live reference runs on seeded random configs.
The overlap laws are the reference's own: acceptance C8
(proj/tests/acceptance_main.cpp:384-418) and test_pipeline.cpp:250-260.
No GPU needed."""
import os

import numpy as np
import pytest

import lco
import paper_2510_05367_b200 as lc

GOLD = os.path.join(os.path.dirname(__file__), "golden")
DEFAULT = open(os.path.join(GOLD, "default.cfg")).read()


def _golden():
    g = np.load(os.path.join(GOLD, "timelines.npz"))
    names = sorted({k.rsplit("_", 1)[0] for k in g.files})
    return g, names


def _xfer_total(ev):
    total, open_ = 0, 0
    for kind, _, _, clock in ev.tolist():
        if kind == 2:
            open_ = clock
        elif kind == 3:
            total += clock - open_
    return total


def test_timelines_match_reference_fixtures():
    g, names = _golden()
    assert len(names) >= 10
    for name in names:
        text = str(g[name + "_config"])
        ev, mk, st = lc.simulate_timeline(text)
        want = g[name + "_events"]
        assert ev.shape == want.shape, name
        assert np.array_equal(ev, want), name
        assert [mk, st] == g[name + "_info"].tolist(), name


def test_c8_simulated_overlap_law():
    # acceptance_main.cpp:384-418: transfers far below the per-step compute
    # window -> async within 1 % of no-swap; sync = no-swap + sum(transfers)
    spans = {}
    for mode in ("off", "async", "sync"):
        text = DEFAULT + f"swap.simulate = true\nswap.mode = {mode}\n"
        ev, mk, _ = lc.simulate_timeline(text)
        spans[mode] = (ev, mk)
    xfer = _xfer_total(spans["sync"][0])
    assert xfer > 0
    assert spans["async"][1] <= 1.01 * spans["off"][1]
    assert spans["sync"][1] == spans["off"][1] + xfer


def test_virtual_makespan_lower_bound():
    # test_pipeline.cpp:250-260: total denoiser MACs at the MAC rate bound
    # the virtual makespan from below
    text = DEFAULT + ("run.frames = 2\nrun.height = 32\nrun.width = 32\nsampler.steps = 6\nrun.seed = 7\n"
                      "swap.simulate = true\nswap.mode = async\n")
    _, mk, _ = lc.simulate_timeline(text)
    mf, mc, _ = lc.model_numbers(text)
    kinds, _ = lc.plan_steps(6, 2)
    macs = sum(mf if k else mc for k in kinds)
    assert mk > 0
    assert mk / 1e9 >= macs / 5e7 * 0.99


def test_slow_link_stalls_and_event_structure():
    text = DEFAULT + ("run.frames = 2\nrun.height = 32\nrun.width = 32\nsampler.steps = 6\n"
                      "swap.simulate = true\nswap.mode = async\nswap.bandwidth = 1e6\n")
    ev, mk, st = lc.simulate_timeline(text)
    assert st > 0 and mk > st
    # matched starts/ends, sorted by clock (swap.cpp:37-56, :366-374)
    depth = {0: 0, 2: 0, 4: 0}
    for kind, *_ in ev.tolist():
        depth[kind - kind % 2] += 1 if kind % 2 == 0 else -1
        assert min(depth.values()) >= 0
    assert all(v == 0 for v in depth.values())
    assert (np.diff(ev[:, 3]) >= 0).all()
    # per branch: evict + prefetch after each full step with consumers
    # (pipeline.cpp:141-147), evict after each last consumer (:156)
    cache_bytes = lc.model_numbers(text)[2] // 2
    xs = ev[ev[:, 0] == 2]
    assert (xs[:, 2] == cache_bytes).all()
    assert len(xs) == 3 * 4 + 3 * 2


def test_simulate_rejects_nonpositive_rates():
    for bad in ("swap.bandwidth = 0", "swap.mac_rate = -1"):
        with pytest.raises(lc.ConfigError):
            lc.simulate_timeline(DEFAULT + "swap.simulate = true\n" + bad + "\n")


def _random_config(rng):
    depth = int(rng.integers(1, 4))
    m = int(rng.integers(0, depth))
    side = 8 * (1 << depth) * int(rng.integers(1, 3))
    steps = int(rng.integers(1, 9))
    kv = {
        "run.frames": int(rng.integers(1, 3)), "run.height": side, "run.width": side,
        "unet.depth": depth, "unet.cache_depth": m, "unet.base_channels": int(rng.choice([4, 8])),
        "sampler.steps": steps, "cache.n": int(rng.integers(1, 5)),
        "cache.enabled": str(bool(rng.random() < 0.85)).lower(),
        "swap.mode": str(rng.choice(["off", "sync", "async"])), "swap.simulate": "true",
        "swap.bandwidth": float(rng.choice([1e5, 1e6, 3e7, 4e9])),
        "swap.latency": float(rng.choice([0.0, 20e-6, 1e-3])),
        "swap.mac_rate": float(rng.choice([1e6, 5e7, 1e9])),
        "chunk.enabled": str(bool(rng.random() < 0.7)).lower(),
        "chunk.eta": int(rng.choice([1, 2])), "chunk.omega": int(rng.choice([1, 2])),
        "chunk.targets": str(rng.choice(["u0", "stem,u0", "d0,head", f"u{m}"])),
        "run.mode": str(rng.choice(["text", "image"])),
    }
    return kv


def test_random_configs_match_live_reference(reference):
    rng = np.random.default_rng(2510)
    checked = 0
    for _ in range(40):
        kv = lco.parse_text(DEFAULT)
        kv.update({k: str(v) for k, v in _random_config(rng).items()})
        text = lco.to_text(kv)
        try:
            want, wmk, wst = reference.timeline(kv)
        except lco.OracleError as e:
            with pytest.raises(lc.LightCacheError) as got:
                lc.simulate_timeline(text)
            assert got.value.code == e.code
            continue
        ev, mk, st = lc.simulate_timeline(text)
        assert np.array_equal(ev, want), text
        assert (mk, st) == (wmk, wst)
        checked += 1
    assert checked >= 30
