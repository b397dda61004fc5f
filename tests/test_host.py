"""Host-side contracts of the product library (liblightcache.so C-ABI),
checked bit-exactly against the reference: step plans, tile grids, MAC
closed forms, cache bytes, the config grammar and the RNG streams.
No GPU needed."""
import os

import numpy as np
import pytest

import lco
import paper_2510_05367_b200 as lc

GOLD = os.path.join(os.path.dirname(__file__), "golden")
DEFAULT = open(os.path.join(GOLD, "default.cfg")).read()


def test_plan_steps_bit_exact():
    g = np.load(os.path.join(GOLD, "plans.npz"))
    for key in g.files:
        total, n = map(int, key.split("_"))
        k, f = lc.plan_steps(total, n)
        assert np.array_equal(np.stack([k, f]), g[key]), key


def test_plan_known_answers():
    # proj/tests/test_cache.cpp:21-53
    k, _ = lc.plan_steps(8, 2)
    assert list(k) == [1, 0] * 4
    k, _ = lc.plan_steps(8, 3)
    assert [s for s in range(8) if k[s]] == [0, 3, 6]
    k, _ = lc.plan_steps(5, 1)
    assert k.all()
    with pytest.raises(lc.ConfigError):
        lc.plan_steps(0, 2)
    with pytest.raises(lc.ConfigError):
        lc.plan_steps(4, 0)


def test_split_bit_exact():
    g = np.load(os.path.join(GOLD, "splits.npz"))
    halo_names = {0: "exact", 1: "fixed", 2: "none"}
    for key in g.files:
        h, w, eta, omega, hk, hp, k = map(int, key.split("_"))
        regions, halo = lc.split(h, w, eta, omega, halo_names[hk], hp, k)
        assert np.array_equal(np.concatenate([regions.reshape(-1), [halo]]), g[key]), key


def test_split_known_answers():
    # proj/tests/test_chunk.cpp:82-116
    r, _ = lc.split(8, 8, 2, 2, "fixed", 1, 3)
    assert list(r[0, 1]) == [0, 5, 0, 5] and list(r[3, 1]) == [3, 8, 3, 8]
    with pytest.raises(lc.ShapeError):
        lc.split(9, 8, 2, 2, "none", 0, 3)


def test_model_numbers_bit_exact():
    g = np.load(os.path.join(GOLD, "model_numbers.npz"))
    import importlib.util
    spec = importlib.util.spec_from_file_location("mk", os.path.join(GOLD, "make_golden.py"))
    mk = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mk)
    cases = dict(mk.SMALL, b=dict(mk.B0, **{"run.frames": 16}), c=dict(mk.C0, **{"run.frames": 25}))
    for name, over in cases.items():
        mf, mc, cb = lc.model_numbers(lc.config_text(over, base=DEFAULT))
        want = g[name]
        assert (mf, mc, cb) == (want[0], want[1], want[7]), name


def test_model_numbers_known_answers():
    # B full 1.241 TMAC, C full 4.364 TMAC, cache 1.18 GB at C
    B = {"run.frames": 16, "run.height": 512, "run.width": 512, "codec.stages": 3, "unet.base_channels": 320}
    mf, mc, cb = lc.model_numbers(lc.config_text(B, base=DEFAULT))
    assert round(mf / 1e12, 3) == 1.241
    C = {"run.frames": 25, "run.height": 576, "run.width": 1024, "codec.stages": 3, "unet.base_channels": 320}
    mf, mc, cb = lc.model_numbers(lc.config_text(C, base=DEFAULT))
    assert round(mf / 1e12, 3) == 4.364 and cb == 1179648000


@pytest.mark.parametrize("bad,code", [
    ("nope.key = 1", 2), ("run.frames = x", 2), ("run.frames = 0", 2), ("sampler.steps = 100", 2),
    ("run.height = 40", 2), ("chunk.eta = 3", 2), ("sampler.kind = heun", 2), ("swap.mode = maybe", 2),
    ("chunk.halo = wide", 2), ("unet.kernel = 4", 2), ("unet.cache_depth = 3", 2), ("cache.enabled = yes", 2),
    ("budget.fast_bytes = -1", 2), ("run.mode = audio", 2), ("garbage line", 2),
])
def test_config_errors_match_reference(bad, code, reference):
    text = DEFAULT + "\n" + bad + "\n"
    with pytest.raises(lc.ConfigError):
        lc.check_config(text)
    assert reference.lib.ref_check_config((DEFAULT + "\n" + bad + "\n").encode()) == code


def test_config_text_round_trip():
    text = lc.normalize_config(DEFAULT + "chunk.targets = u0, u1 ,d0\ncodec.latent_channels = 4\n")
    assert "chunk.targets = u0,u1,d0" in text
    assert lc.normalize_config(text) == text


def test_randn_and_seeds_match_oracle(oracle):
    assert lc.derive_seed(42, 1) == oracle.derive_seed(42, 1)
    s = lc.derive_seed(42, 1)
    assert np.array_equal(lc.randn(s, 4096), oracle.randn(s, 4096))


def test_shard_frames_partition():
    # 25 frames over 8 GPUs -> 4 + 7x3 (balanced)
    counts = [lc.shard_frames(25, 8, r)[1] for r in range(8)]
    assert counts == [4, 3, 3, 3, 3, 3, 3, 3]
    assert [lc.shard_frames(25, 4, r)[1] for r in range(4)] == [7, 6, 6, 6]
    assert [lc.shard_frames(25, 2, r)[1] for r in range(2)] == [13, 12]
    for T in range(1, 30):
        for g in (1, 2, 4, 8):
            spans = [lc.shard_frames(T, g, r) for r in range(g)]
            covered = []
            for f0, c in spans:
                covered += list(range(f0, f0 + c))
            assert covered == list(range(T))


def _arena_configs():
    rng = np.random.default_rng(77)
    out = [{}, {"cache.enabled": "false"}, {"unet.cache_depth": 1}, {"unet.cache_depth": 2},
           {"unet.kernel": 5}, {"chunk.halo": "none"},
           {"run.frames": 25, "run.height": 576, "run.width": 1024, "codec.stages": 3, "codec.width": 128,
            "unet.base_channels": 320, "unet.depth": 3}]
    while len(out) < 40:
        depth = int(rng.integers(1, 5))
        unit = 1 << (depth + 2)
        over = {"unet.depth": depth, "run.height": unit * int(rng.integers(1, 4)),
                "run.width": unit * int(rng.integers(1, 4)), "unet.base_channels": int(rng.choice([8, 32, 320])),
                "unet.cache_depth": int(rng.integers(0, depth)), "unet.kernel": int(rng.choice([1, 3, 5])),
                "cache.enabled": str(rng.choice(["true", "false"])), "chunk.halo": str(rng.choice(["exact", "none"])),
                "run.frames": int(rng.integers(1, 6))}
        try:
            lc.check_config(lc.config_text(over, base=lc.DEFAULT_CONFIG))
        except lc.LightCacheError:
            continue
        out.append(over)
    return out


@pytest.mark.parametrize("over", _arena_configs())
def test_arena_plan_never_overlaps_live_buffers(over):
    """The lifetime packing of the denoise activations (host.cpp plan_arena,
    the arena Engine::alloc_activations lays out): buffers whose lifetimes
    within a full step overlap never share bytes, the cache keeps [0,
    cache_bytes) for the whole step, every buffer used fits below act_end."""
    p = lc.plan_arena(lc.config_text(over, base=lc.DEFAULT_CONFIG))
    bufs = [b for b in p["buffers"] if b["t1"] >= 0]
    names = [b["name"] for b in bufs]
    for must in ("patch", "stem", "D0", "U0"):
        assert must in names
    assert ("cache" in names) == (over.get("cache.enabled", "true") == "true")
    for b in bufs:
        assert 0 <= b["t0"] <= b["t1"] < p["ops"] + 1 and b["off"] % 256 == 0
        assert b["off"] + b["bytes"] <= p["act_end"]
        if b["name"] == "cache":
            assert b["off"] == 0 and b["bytes"] == p["cache_bytes"] and b["t0"] == 0 and b["t1"] >= p["ops"] - 1
        else:
            assert b["off"] >= p["cache_bytes"]
    for i, a in enumerate(bufs):
        for b in bufs[i + 1:]:
            if a["t1"] < b["t0"] or b["t1"] < a["t0"]:
                continue
            assert a["off"] + a["bytes"] <= b["off"] or b["off"] + b["bytes"] <= a["off"], (a, b)


def test_arena_plan_config_c():
    """On config C the packing holds the 1.18 GB of activations in 0.6 GB:
    the stem output's slot is reused by the deep levels and then by U_0."""
    over = {"run.frames": 25, "run.height": 576, "run.width": 1024, "codec.stages": 3, "codec.width": 128,
            "unet.base_channels": 320, "unet.depth": 3}
    p = lc.plan_arena(lc.config_text(over, base=lc.DEFAULT_CONFIG))
    bufs = {b["name"]: b for b in p["buffers"]}
    total = sum(b["bytes"] for n, b in bufs.items() if n != "cache")
    packed = p["act_end"] - p["cache_bytes"]
    assert total > 1.1e9 and packed < 0.65e9
    assert bufs["U0"]["off"] == bufs["stem"]["off"]  # U_0 reuses the stem output's storage
