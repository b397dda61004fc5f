"""End-to-end GPU parity against the CPU oracle (oracle/lc_oracle.c, itself
pinned bit-exactly to the reference in tests/test_oracle.py).

Bars (BASELINE.json north star):
  * final latents and decoded frames: relative L2 <= 1e-3 vs the fp32 oracle;
  * cache/chunk/slice schedule: bit-exact (step counts, MAC counters, cache
    bytes, transfer issue order);
  * GPU self-consistency (swap modes, decode slicing, exact-halo chunking):
    bit-identical videos, as the reference's acceptance C2 demands of the CPU
    path (proj/tests/acceptance_main.cpp:92-126).
"""
import numpy as np
import pytest

import paper_2510_05367_b200 as lc

pytestmark = pytest.mark.gpu

TOL = 1e-3

DEFAULT = lc.DEFAULT_CONFIG
# proj/tests/test_pipeline.cpp:15-23 tiny_config: 2 frames, 32x32, 6 steps
TINY = {"run.frames": 2, "run.height": 32, "run.width": 32, "sampler.steps": 6}
# Config A: 8 frames, latent 4x32x32, N=3, 2 chunks on u0
CONFIG_A = {"run.height": 128, "run.width": 128, "cache.n": 3, "chunk.eta": 2, "chunk.omega": 1}
# configs B and C
B_SHAPE = {"run.frames": 16, "run.height": 512, "run.width": 512, "codec.stages": 3, "codec.width": 128,
           "unet.base_channels": 320, "unet.depth": 3, "sampler.steps": 4, "cache.n": 2}
C_SHAPE = {"run.frames": 25, "run.height": 576, "run.width": 1024, "codec.stages": 3, "codec.width": 128,
           "unet.base_channels": 320, "unet.depth": 3, "sampler.steps": 25, "cache.n": 2, "swap.mode": "async"}


def _kv(over):
    import lco
    kv = lco.parse_text(DEFAULT)
    kv.update({k: str(v) for k, v in over.items()})
    return kv


def _run(ctx, over, **kw):
    text = lc.config_text(over, base=DEFAULT)
    ctx.configure(text)
    return ctx.run_pipeline(want_latent=True, **kw)


@pytest.mark.parametrize("over", [
    TINY,
    dict(TINY, **{"sampler.kind": "ancestral"}),
    dict(TINY, **{"sampler.kind": "ddim"}),
    dict(TINY, **{"unet.cache_depth": 1}),
    dict(TINY, **{"unet.cache_depth": 2, "cache.n": 3}),
    dict(TINY, **{"chunk.halo": "none"}),
    dict(TINY, **{"chunk.targets": "stem,d0,d1,u1,u0,head", "chunk.halo": "none", "chunk.eta": 2,
                  "chunk.omega": 2}),
    dict(TINY, **{"unet.kernel": 5}),
    dict(TINY, **{"unet.kernel": 1}),
    # odd kernels beyond 7x7 (valid in the reference, unet.cpp:139-146)
    dict(TINY, **{"unet.kernel": 9}),
    dict(TINY, **{"unet.kernel": 11, "chunk.halo": "fixed", "chunk.halo_px": 2, "sampler.steps": 3}),
    dict(TINY, **{"cache.enabled": "false", "swap.mode": "off"}),
    # image mode: encode stage + forward_noise (pipeline.cpp:108-114)
    dict(TINY, **{"run.mode": "image"}),
    dict(TINY, **{"run.mode": "image", "sampler.kind": "ancestral", "codec.stages": 3, "run.height": 64,
                  "run.width": 64}),
    # K8 (fused last decoder stage): partial tiles in x and y, one and three
    # 64-channel K blocks
    dict(TINY, **{"run.frames": 3, "run.height": 96, "run.width": 160, "sampler.steps": 3, "codec.width": 64}),
    dict(TINY, **{"run.height": 64, "run.width": 64, "sampler.steps": 2, "codec.width": 192}),
])
def test_pipeline_matches_oracle(ctx, oracle, over):
    video, lat, rep = _run(ctx, over)
    want_v, want_l = oracle.run_pipeline(_kv(over))
    assert lc.rel_l2(lat, want_l) < TOL
    assert lc.rel_l2(video, want_v) < TOL


def test_config_a_matches_oracle(ctx, oracle):
    video, lat, rep = _run(ctx, CONFIG_A)
    want_v, want_l = oracle.run_pipeline(_kv(CONFIG_A))
    assert lc.rel_l2(lat, want_l) < TOL
    assert lc.rel_l2(video, want_v) < TOL
    # schedule: 25 steps at N=3 -> 9 full / 16 cached (cache.cpp:25-33)
    assert rep["mac"]["full_steps"] == 9 and rep["mac"]["cached_steps"] == 16
    mf, mc, cb = lc.model_numbers(lc.config_text(CONFIG_A, base=DEFAULT))
    assert rep["mac"]["per_full_step"] == mf and rep["mac"]["per_cached_step"] == mc
    assert rep["mac"]["denoiser_total"] == 9 * mf + 16 * mc
    assert rep["cache_bytes"] == cb


def test_forward_full_and_cached_match_oracle(ctx, oracle):
    over = dict(TINY, **{"chunk.enabled": "false"})
    kv = _kv(over)
    rng = np.random.default_rng(5)
    x = rng.standard_normal((2, 2, 4, 8, 8)).astype(np.float32)
    ctx.configure(lc.config_text(over, base=DEFAULT))
    deep_shape = (2, 2, 16, 8, 8)
    eps, deep = ctx.forward(x, 37, want_deep=True, deep_shape=deep_shape)
    want_eps, want_deep = oracle.forward(kv, x, 37, want_deep=True)
    assert lc.rel_l2(eps, want_eps) < TOL
    assert lc.rel_l2(deep, want_deep) < TOL
    # seam exactness (proj/tests/test_unet.cpp:106-117): cached with the
    # same-step deep features equals the full pass
    eps_c, _ = ctx.forward(x, 37, deep_in=want_deep)
    want_c, _ = oracle.forward(kv, x, 37, deep_in=want_deep)
    assert lc.rel_l2(eps_c, want_c) < TOL
    assert lc.rel_l2(eps_c, eps) < TOL


def test_swap_modes_are_bit_identical(ctx):
    """Acceptance C2 on the GPU: swap off/sync/async change timing only."""
    vids = []
    for mode in ("off", "sync", "async"):
        v, _, rep = _run(ctx, dict(TINY, **{"swap.mode": mode}))
        vids.append(v)
        # reconfiguring off -> on at the same geometry must allocate the
        # slow-tier entry and really swap
        assert (rep["swap"]["calls"] > 0) == (mode != "off"), mode
        assert (rep["swap"]["bytes_moved"] > 0) == (mode != "off"), mode
    assert np.array_equal(vids[0], vids[1]) and np.array_equal(vids[0], vids[2])


_TILES_CHILD = r"""
import sys, numpy as np
import paper_2510_05367_b200 as lc
over = eval(sys.argv[1])
ctx = lc.Context(0)
res = {}
for tag, chunk in (("tiled", "true"), ("untiled", "false")):
    text = lc.config_text(dict(over, **{"chunk.enabled": chunk}), base=lc.DEFAULT_CONFIG)
    ctx.configure(text)
    v, lat, rep = ctx.run_pipeline(want_latent=True)
    res[tag + "_v"], res[tag + "_lat"] = v, lat
    res[tag + "_launches"] = rep["kernel_launches"]
np.savez(sys.argv[2], **res)
"""


@pytest.mark.parametrize("over", [
    dict(TINY, **{"chunk.targets": "stem,d0,d1,d2,u2,u1,u0,head"}),
    dict(TINY, **{"chunk.targets": "u0,head", "chunk.eta": 4, "chunk.omega": 1, "run.height": 64}),
    # C's frame-0 slice with the bench's chunking (u0 2x2, exact halo)
    dict(C_SHAPE, **{"run.frames": 1, "sampler.steps": 2}),
])
def test_exact_halo_tiles_are_bit_identical(tmp_path, over):
    """Chunked == unchunked for the lossless (exact) halo, bit for bit
    (proj/tests/test_unet.cpp:201-220, test_chunk.cpp:211-219), with every
    tile really run as its own launch over its padded window
    (LC_FORCE_TILES=1 disables the one-launch collapse of the lossless
    case)."""
    import os
    import subprocess
    import sys
    path = str(tmp_path / "tiles.npz")
    env = dict(os.environ, LC_FORCE_TILES="1")
    r = subprocess.run([sys.executable, "-c", _TILES_CHILD, repr(over), path], env=env, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    o = np.load(path)
    assert int(o["tiled_launches"]) > int(o["untiled_launches"])  # the tiles really ran separately
    assert np.array_equal(o["tiled_lat"], o["untiled_lat"])
    assert np.array_equal(o["tiled_v"], o["untiled_v"])


@pytest.mark.parametrize("over", [
    dict(TINY, **{"chunk.halo": "fixed", "chunk.halo_px": 1, "unet.kernel": 5}),
    dict(TINY, **{"chunk.halo": "fixed", "chunk.halo_px": 1, "unet.kernel": 5,
                  "chunk.targets": "stem,d0,u0,head"}),
    dict(TINY, **{"chunk.halo": "fixed", "chunk.halo_px": 2, "unet.kernel": 7, "chunk.eta": 2, "chunk.omega": 1}),
    dict(TINY, **{"chunk.halo": "fixed", "chunk.halo_px": 3, "unet.kernel": 3, "chunk.targets": "d1,u1,u0"}),
])
def test_fixed_halo_matches_oracle(ctx, oracle, over):
    """HaloMode::fixed_px (proj/src/chunk.cpp:156-160): a halo below the
    receptive radius leaves seams; the per-tile windows must reproduce the
    reference's crop-then-conv values (and above the radius it is lossless)."""
    video, lat, _ = _run(ctx, over)
    want_v, want_l = oracle.run_pipeline(_kv(over))
    assert lc.rel_l2(lat, want_l) < TOL
    assert lc.rel_l2(video, want_v) < TOL


def test_cache_off_equals_n1(ctx):
    """proj/tests/test_pipeline.cpp:75-87: cache off == N=1, bit-identical."""
    a, _, _ = _run(ctx, dict(TINY, **{"cache.enabled": "false", "swap.mode": "off"}))
    b, _, _ = _run(ctx, dict(TINY, **{"cache.enabled": "true", "cache.n": 1, "swap.mode": "off"}))
    assert np.array_equal(a, b)


def test_sliced_decode_equals_batch(ctx, oracle):
    over = dict(TINY, **{"run.frames": 5})
    ctx.configure(lc.config_text(over, base=DEFAULT))
    rng = np.random.default_rng(3)
    lat = rng.standard_normal((1, 5, 4, 8, 8)).astype(np.float32)
    outs = [ctx.decode(lat, slice_frames=g) for g in (1, 2, 5)]
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
    want = oracle.decode(_kv(over), lat)
    assert lc.rel_l2(outs[0], want) < TOL


def test_swap_issue_order(ctx):
    """Transfer issue order of SURVEY.md Appendix A P7 (N=3, 7 steps):
    | C0 X0 X0 X1 X1 | C1 A1 A1 | C2 A1 A1 X2 X2 | C3 X3 X3 X4 X4 | ..."""
    _, _, rep = _run(ctx, dict(TINY, **{"sampler.steps": 7, "cache.n": 3, "swap.mode": "sync"}))
    ev = rep["timeline"]["events"]
    starts = [(k, s) for k, s, _, _ in ev if k in ("xfer_start", "await_start", "compute_start")]
    seq = []
    for k, s in starts:
        seq.append({"compute_start": "C", "xfer_start": "X", "await_start": "A"}[k] + str(s))
    want = ("C0 X0 X0 X1 X1 C1 A1 A1 C2 A1 A1 X2 X2 C3 X3 X3 X4 X4 C4 A4 A4 C5 A4 A4 X5 X5 C6 X6 X6").split()
    assert seq == want, " ".join(seq)


def test_typed_run_result(ctx):
    """lc_get_run_result: the reference's RunResult fields for the last run,
    consistent with the JSON report (pipeline.hpp:18-39)."""
    _, _, rep = _run(ctx, dict(TINY, **{"sampler.steps": 7, "cache.n": 3, "swap.mode": "sync"}))
    r = ctx.run_result()
    assert r["full_steps"] == rep["mac"]["full_steps"] == 3 and r["cached_steps"] == 4
    assert r["denoiser_macs"] == rep["mac"]["denoiser_total"] and r["cache_bytes_planned"] == rep["cache_bytes"]
    assert r["peak_fast"] == [rep["peaks"][s]["fast"] for s in ("setup", "encode", "denoise", "decode")]
    assert abs(r["wall_total"] - rep["device_ms"]["total"] * 1e-3) < 1e-6 and r["wall_setup"] > 0
    kinds = [k for k, *_ in rep["timeline"]["events"] if k in lc.TIMELINE_KINDS]
    assert [lc.TIMELINE_KINDS[k] for k in r["timeline"][:, 0]] == kinds
    assert abs(r["stall_s"] - rep["timeline"]["stall_ms"] * 1e-3) < 1e-9 and not r["simulated"]


def test_swap_bytes_logical_and_moved(ctx):
    """Logical swap traffic is the reference's (one
    evict_all/prefetch_all call moves both entries; calls = 2 x full steps
    with consumers + last consumers + a final consumer-less full step).  Only
    dirty evictions and prefetches cross the host link: the eviction after a
    last consumer finds the host copy already valid."""
    _, _, rep = _run(ctx, dict(TINY, **{"sampler.steps": 7, "cache.n": 3, "swap.mode": "async"}))
    pair = rep["cache_bytes_physical"]  # both entries of one call
    assert rep["swap"]["calls"] == 7  # plan F c c F c c F
    assert rep["swap"]["bytes"] == 7 * pair
    assert rep["swap"]["bytes_moved"] == 5 * pair  # 3 dirty evictions + 2 prefetches


@pytest.mark.parametrize("mode,bw", [("async", 1e6), ("sync", 4e9), ("async", 4e9), ("off", 4e9)])
def test_simulated_swap_reports_the_virtual_timeline(ctx, mode, bw):
    """swap.simulate = true (proj/src/swap.cpp:141-374): the device work and
    video are unchanged, the run reports the simulated engine's virtual
    timeline (pinned to the reference in tests/test_simulate.py) and the
    ledger clock is labelled virtual (pipeline.cpp:79-82, :212-216)."""
    from paper_2510_05367_b200 import harness
    over = dict(TINY, **{"swap.mode": mode, "swap.bandwidth": bw, "run.seed": 7})
    real, _, rep_real = _run(ctx, over)
    assert rep_real["timeline"]["simulated"] is False
    text = lc.config_text(dict(over, **{"swap.simulate": "true"}), base=DEFAULT)
    res = harness.run_pipeline(ctx, text)
    assert np.array_equal(res.video, real)
    tl = res.rep["timeline"]
    assert tl["simulated"] is True
    ev, mk, st = lc.simulate_timeline(text)
    kinds = list(lc.TIMELINE_KINDS)
    assert [kinds.index(e[0]) for e in tl["events"]] == ev[:, 0].tolist()
    assert [[e[1], e[2]] for e in tl["events"]] == ev[:, 1:3].tolist()
    assert np.allclose([e[3] for e in tl["events"]], ev[:, 3] * 1e-6, rtol=1e-9, atol=1e-9)
    assert abs(tl["makespan_ms"] - mk * 1e-6) <= 1e-6 * max(1.0, mk * 1e-6)
    assert abs(tl["stall_ms"] - st * 1e-6) <= 1e-6 * max(1.0, st * 1e-6)
    rj = harness.run_report(res)
    assert rj["timeline"]["simulated"] is True
    assert harness.ledger_summary(ctx)["clock"] == "virtual"
    # the run's last ledger event (decode -> setup) carries the virtual
    # clock after the denoising drain, the timeline's last event
    last = float(harness.ledger_csv(ctx).splitlines()[-1].split(",")[1])
    assert abs(last - mk * 1e-9) <= 1e-5 * mk * 1e-9


def test_nonfinite_input_raises_shape_error(ctx):
    over = dict(TINY)
    ctx.configure(lc.config_text(over, base=DEFAULT))
    x0 = np.zeros(ctx.latent_elems(), np.float32)
    x0[3] = np.nan
    with pytest.raises(lc.ShapeError):
        ctx.run_pipeline(x0=x0)


def test_budget_error(ctx):
    with pytest.raises(lc.BudgetError):
        _run(ctx, dict(TINY, **{"budget.fast_bytes": 80000}))


@pytest.mark.parametrize("kind,extra", [("euler", {}), ("ancestral", {}), ("euler", {"cache.n": 1}),
                                        ("euler", {"swap.mode": "sync"}), ("ddim", {"cache.n": 4})])
def test_graph_replay_is_bit_identical(ctx, oracle, kind, extra):
    """Run 1 is eager, run 2 captures the body into a CUDA graph, run 3+
    replay it: all must give the same bytes (and match the oracle)."""
    over = dict(TINY, **{"sampler.kind": kind, "sampler.steps": 5}, **extra)
    outs = [_run(ctx, over) for _ in range(4)]
    for v, l, _ in outs[1:]:
        assert np.array_equal(v, outs[0][0]) and np.array_equal(l, outs[0][1])
    want_v, want_l = oracle.run_pipeline(_kv(over))
    assert lc.rel_l2(outs[-1][1], want_l) < TOL
    # resident path through the same graph
    ctx.upload_latent(lc.randn(lc.derive_seed(42, 1), ctx.latent_elems()))
    ctx.run_resident()
    assert np.array_equal(ctx.download_video().reshape(outs[0][0].shape), outs[0][0])
    # queued replays (throughput loop): same bytes, report of the last run
    for _ in range(3):
        ctx.run_resident_async()
    rep_a = ctx.wait()
    assert np.array_equal(ctx.download_video().reshape(outs[0][0].shape), outs[0][0])
    assert rep_a["kernel_launches"] == outs[-1][2]["kernel_launches"]
    # pinned host buffers: decoded slices stream out inside the body
    x0 = lc.PinnedArray(ctx.latent_elems())
    x0.array[:] = lc.randn(lc.derive_seed(42, 1), ctx.latent_elems())
    vid = lc.PinnedArray(ctx.video_elems())
    for _ in range(3):
        vid.array[:] = -1.0
        ctx.run_e2e(x0, vid)
        assert np.array_equal(vid.array.reshape(outs[0][0].shape), outs[0][0])
    # queued pinned runs: run k's video leaves inside run k+1 (deferred
    # download node) or at wait(); alternate two inputs so a download that
    # read the wrong run's video is caught
    x0b = lc.PinnedArray(ctx.latent_elems())
    x0b.array[:] = lc.randn(12345, ctx.latent_elems())
    ctx.run_e2e(x0b, vid)
    want_b = vid.array.copy()
    want_a = outs[0][0].reshape(-1)
    assert not np.array_equal(want_a, want_b)
    vids = [lc.PinnedArray(ctx.video_elems()) for _ in range(5)]
    for v in vids:
        v.array[:] = -1.0
    for k in range(5):
        ctx.run_e2e_async(x0 if k % 2 == 0 else x0b, vids[k])
    ctx.wait()
    for k in range(5):
        assert np.array_equal(vids[k].array, want_a if k % 2 == 0 else want_b), k
    # a pending download survives a different kind of launch in between
    vids[0].array[:] = -1.0
    ctx.run_e2e_async(x0b, vids[0])
    ctx.run_resident_async()
    ctx.wait()
    assert np.array_equal(vids[0].array, want_b)
    assert np.array_equal(ctx.download_video().reshape(-1), want_a)
    vids[1].array[:] = -1.0
    ctx.run_e2e_async(x0b, vids[1])
    v_sync, _, _ = ctx.run_pipeline()  # synchronous run after a queued one
    assert np.array_equal(vids[1].array, want_b)
    assert np.array_equal(v_sync.reshape(-1), want_a)
    # pageable buffers through the async entry point run synchronously (no
    # graph download node may point at pageable memory); a pinned run queued
    # before completes first
    vids[2].array[:] = -1.0
    ctx.run_e2e_async(x0, vids[2])
    xp = np.array(x0b.array)
    vp = np.full(ctx.video_elems(), -1.0, np.float32)
    import ctypes
    assert lc.lib().lc_run_pipeline_async(ctx._h, ctypes.c_void_p(xp.ctypes.data), ctypes.c_void_p(vp.ctypes.data)) == 0
    ctx.wait()
    assert np.array_equal(vids[2].array, want_a)
    assert np.array_equal(vp, want_b)
    for v in vids:
        v.free()
    x0b.free()
    x0.free()
    vid.free()


# ---------------------------------------------------------------- B / C
def _gold(name):
    import os
    return np.load(os.path.join(os.path.dirname(__file__), "golden", f"{name}.npz"))




FRAME0_GOLDENS = ["b_frame0", "c_frame0", "b_frame0_ancestral", "b_frame0_ddim", "b_frame0_image",
                  "b_frame0_fixed_k5", "c_frame0_none_s2", "c_frame0_fixed_k5_s2", "b_frame0_none"]


@pytest.mark.parametrize("name", FRAME0_GOLDENS)
def test_frame0_slice_matches_reference(ctx, name):
    """frame 0 of a T-frame run equals the T=1 run.
    The golden T=1 runs at the B / C shapes (Euler, DDIM, ancestral, image
    mode, fixed and none halos) hold the reference's own video
    (oracle/_ref run_pipeline, video_source) and the final latent of the
    restatement whose video is bit-identical to it (make_golden.py pin)."""
    g = _gold(name)
    ctx.configure(str(g["config"]))
    video, lat, rep = ctx.run_pipeline(want_latent=True)
    assert lc.rel_l2(lat, g["latent"]) < TOL
    assert lc.rel_l2(video, g["video"]) < TOL
    if "macs" in g:  # the reference's own MAC counter (RunResult::denoiser_macs)
        assert rep["mac"]["denoiser_total"] == int(g["macs"][0])


@pytest.mark.parametrize("shape", [B_SHAPE, C_SHAPE])
def test_full_shape_frame0_equals_single_frame_run(ctx, shape):
    """Frame independence on the GPU: frame 0 of the full-shape run is
    bit-identical to the 1-frame run (tile shapes change, per-pixel
    arithmetic does not)."""
    v1, l1, _ = _run(ctx, dict(shape, **{"run.frames": 1}))
    vT, lT, rep = _run(ctx, shape)
    assert np.array_equal(lT[:, :1], l1)
    assert np.array_equal(vT[:, :1], v1)
    T = shape["run.frames"]
    mf, mc, cb = lc.model_numbers(lc.config_text(shape, base=DEFAULT))
    nf = rep["mac"]["full_steps"]
    assert rep["mac"]["denoiser_total"] == nf * mf + rep["mac"]["cached_steps"] * mc
    assert rep["cache_bytes"] == cb
    # physical cache: fp16 U_{m+1} before the upsample = 1/8 of the fp32 geometry
    assert rep["cache_bytes_physical"] * 8 == cb
    assert np.isfinite(vT).all()


# ------------------------------------------------ memory ledger (§8 f1)
def _peaks(rep):
    return {s: rep["peaks"][s]["fast"] for s in ("setup", "encode", "denoise", "decode")}


def _fresh_run(over, text_only=False):
    """One run on a fresh engine (each reference run has a fresh ledger);
    returns (report, ledger summary, ledger csv)."""
    from paper_2510_05367_b200 import harness
    c = lc.Context(0)
    try:
        c.configure(lc.config_text(over, base=DEFAULT))
        rep = c.run_pipeline()[2]
        return rep, harness.ledger_summary(c), harness.ledger_csv(c)
    finally:
        c.close()


# decode-dominated geometry (codec width 128 on a base-8 U-Net): the
# unsliced decode workspace exceeds the denoise working set, as in the
# reference's C10 setting
DEC_HEAVY = dict(TINY, **{"run.frames": 12, "codec.width": 128})


def test_budget_split_aborts_in_decode():
    """Acceptance C10 (proj/tests/acceptance_main.cpp:447-478) on the HBM
    ledger: a fast-tier budget between the sliced run's overall peak and the
    unsliced decode peak lets the sliced run through and aborts the unsliced
    one in the decode stage."""
    over = dict(DEC_HEAVY, **{"swap.mode": "sync"})
    opt = _fresh_run(over)[0]
    fat = _fresh_run(dict(over, **{"decode.sliced": "false"}))[0]
    opt_peak = max(_peaks(opt).values())
    fat_decode = _peaks(fat)["decode"]
    assert fat_decode > opt_peak
    budget = (opt_peak + fat_decode) // 2
    _fresh_run(dict(over, **{"budget.fast_bytes": budget}))
    with pytest.raises(lc.BudgetError, match="stage decode"):
        _fresh_run(dict(over, **{"decode.sliced": "false", "budget.fast_bytes": budget}))


def test_slicing_changes_only_the_decode_peak():
    """Acceptance C6's slicing row (acceptance_main.cpp:322-327): -slicing
    raises the decode peak, leaves the denoise peak alone and (decode-heavy
    geometry) becomes the dominant stage of its row."""
    on = _fresh_run(dict(DEC_HEAVY, **{"swap.mode": "sync"}))[0]
    off = _fresh_run(dict(DEC_HEAVY, **{"swap.mode": "sync", "decode.sliced": "false"}))[0]
    assert _peaks(off)["decode"] > _peaks(on)["decode"]
    assert _peaks(off)["denoise"] == _peaks(on)["denoise"]
    assert _peaks(off)["decode"] > _peaks(off)["denoise"]


def test_swapping_row_frees_the_cache_in_decode():
    """Acceptance C6's -swapping row (acceptance_main.cpp:329-331) on the
    physical ledger: with the swap the final eviction leaves the entries on
    the host through decode (proj/README.md "Swap schedule"), so the decode
    peak is lower by exactly the physical cache bytes; without it they stay
    in HBM until the store's teardown.  The denoise peak does not move: the
    cache is the producing activation U_{m+1} itself (0 extra bytes, C5
    below), so there is no resident copy for the swap to free in denoise."""
    on = _fresh_run(dict(TINY, **{"swap.mode": "sync"}))[0]
    off = _fresh_run(dict(TINY, **{"swap.mode": "off"}))[0]
    cache = on["cache_bytes_physical"]
    assert cache > 0
    assert _peaks(off)["decode"] - _peaks(on)["decode"] == cache
    assert _peaks(off)["denoise"] == _peaks(on)["denoise"]


@pytest.mark.parametrize("over", [TINY, dict(TINY, **{"unet.base_channels": 64, "run.height": 64, "run.width": 64})])
def test_cache_memory_arithmetic(over):
    """Acceptance C5 (acceptance_main.cpp:276-305) on the physical ledger:
    cache-on minus cache-off denoise peak.  The reference's logical model
    pays exactly cache_bytes (fp32, upsampled) for the retained entries;
    here the entries are the U_{m+1} activation itself (fp16, pre-upsample)
    kept across steps, so they cost at most their physical bytes -- less
    when the cache-off run had no dead space to hide U_{m+1} in -- and the
    swap does not change the denoise working set (its HBM effect is in
    decode, test_swapping_row_frees_the_cache_in_decode)."""
    off = _fresh_run(dict(over, **{"cache.enabled": "false", "swap.mode": "off"}))[0]
    on = _fresh_run(dict(over, **{"swap.mode": "off"}))[0]
    swp = _fresh_run(dict(over, **{"swap.mode": "sync"}))[0]
    delta = _peaks(on)["denoise"] - _peaks(off)["denoise"]
    assert 0 <= delta <= on["cache_bytes_physical"]
    assert _peaks(swp)["denoise"] == _peaks(on)["denoise"]


@pytest.mark.parametrize("over", [TINY, dict(TINY, **{"run.mode": "image"}), dict(DEC_HEAVY, **{"decode.sliced": "false"}),
                                  dict(TINY, **{"swap.mode": "off"})])
def test_ledger_peak_is_the_physical_arena(over):
    """The per-run working sets live in one device arena sized to the peak
    of their logged lifetimes: the ledger's overall fast peak minus the
    persistent buffers equals the arena, and the tier moves of the swap
    show double residency (destination up at move_start, source down only
    at move_end, ledger.cpp:93-123) and balance out."""
    rep, summ, csv = _fresh_run(over)
    arena = rep["arena"]["bytes"]
    assert summ["overall"]["fast_peak_bytes"] - summ["current"]["fast_bytes"] == arena
    rows = [r.split(",") for r in csv.splitlines()[1:]]
    moves = [r for r in rows if r[2] in ("move_start", "move_end")]
    swapping = over.get("swap.mode", "async") != "off"
    assert bool(moves) == swapping
    occ = {"fast": 0, "slow": 0}
    for r in rows:
        kind, tier, b = r[2], r[3], int(r[4])
        if kind in ("alloc", "move_start"):
            occ[tier] += b
        elif kind in ("free", "move_end"):
            occ[tier] -= b
        assert int(r[6]) == occ[tier]
    for a, b in zip(moves[::2], moves[1::2]):
        assert a[2] == "move_start" and b[2] == "move_end" and a[5] == b[5] and a[3] != b[3]
    assert occ["slow"] == 0  # teardown: every entry left the host tier


# ------------------------------------------ randomised configurations
def _random_configs(k=16, seed=2024):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < k:
        depth = int(rng.integers(1, 4))
        stages = int(rng.integers(1, 3))
        unit = (1 << depth) * (1 << stages)
        over = {
            "run.frames": int(rng.integers(1, 5)),
            "run.height": unit * int(rng.integers(1, 5)),
            "run.width": unit * int(rng.integers(1, 5)),
            "unet.depth": depth, "codec.stages": stages,
            "unet.base_channels": int(rng.choice([8, 16, 24])),
            "codec.width": int(rng.choice([8, 16])),
            "unet.kernel": int(rng.choice([1, 3, 3, 5])),
            "unet.cache_depth": int(rng.integers(0, depth)),
            "sampler.steps": int(rng.integers(2, 7)),
            "sampler.kind": str(rng.choice(["euler", "ddim", "ancestral"])),
            "cache.n": int(rng.integers(1, 4)),
            "swap.mode": str(rng.choice(["off", "sync", "async"])),
            "chunk.enabled": str(rng.choice(["true", "false"])),
            "chunk.halo": str(rng.choice(["exact", "none", "fixed"])),
            "chunk.halo_px": int(rng.integers(0, 3)),
            "chunk.eta": int(rng.choice([1, 2])), "chunk.omega": int(rng.choice([1, 2])),
            "chunk.targets": str(rng.choice(["u0", "stem,u0", "d0,u0,head"])),
            "decode.sliced": str(rng.choice(["true", "false"])),
            "run.mode": "image" if len(out) % 4 == 3 else "text",
        }
        try:
            lc.check_config(lc.config_text(over, base=DEFAULT))
        except lc.LightCacheError:
            continue
        out.append(over)
    return out


@pytest.mark.parametrize("over", _random_configs())
def test_random_configs_match_oracle(ctx, oracle, over):
    """Seeded random shapes, depths, kernels, samplers, swap / chunk /
    slicing modes and image mode against the oracle (the tile chooser,
    schedules and epilogue variants see shapes the named tests do not)."""
    video, lat, _ = _run(ctx, over)
    want_v, want_l = oracle.run_pipeline(_kv(over))
    assert lc.rel_l2(lat, want_l) < TOL
    assert lc.rel_l2(video, want_v) < TOL


_K8_CHILD = r"""
import sys, numpy as np
import paper_2510_05367_b200 as lc
over = eval(sys.argv[1])
ctx = lc.Context(0)
ctx.configure(lc.config_text(over, base=lc.DEFAULT_CONFIG))
v, lat, _ = ctx.run_pipeline(want_latent=True)
np.savez(sys.argv[2], v=v, lat=lat)
"""


@pytest.mark.parametrize("over", [
    TINY,
    dict(TINY, **{"run.height": 64, "run.width": 96, "sampler.steps": 3, "chunk.halo": "none",
                  "chunk.targets": "stem,u0,head", "chunk.eta": 2, "chunk.omega": 3}),
    dict(TINY, **{"run.height": 64, "run.width": 64, "sampler.steps": 2, "codec.width": 192}),
])
def test_fused_tap_kernel_matches_gemm_plus_gather(tmp_path, over):
    """K8 (csrc/subpix_tc.cu) against the tap-to-N GEMM + gather pair it
    replaces (LC_SUBPIX_FUSED=0).  The head sums the same tap products in the
    same order: bit-identical latents, head chunk windows included.  The
    decoder's last stage sums its two row taps inside the MMA (fp32 tensor
    core accumulation) instead of in the gather: the videos agree to fp32
    rounding (relative L2 <= 1e-6, far inside the 1e-3 parity bar)."""
    import os
    import subprocess
    import sys
    outs = []
    for fused in ("1", "0"):
        path = str(tmp_path / f"k8_{fused}.npz")
        env = dict(os.environ, LC_SUBPIX_FUSED=fused)
        r = subprocess.run([sys.executable, "-c", _K8_CHILD, repr(over), path], env=env, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(path))
    assert np.array_equal(outs[0]["lat"], outs[1]["lat"])
    assert lc.rel_l2(outs[0]["v"], outs[1]["v"]) <= 1e-6


@pytest.mark.parametrize("over", [
    TINY,
    dict(TINY, **{"sampler.kind": "ancestral", "sampler.steps": 4}),
    dict(TINY, **{"sampler.kind": "ddim", "run.frames": 3}),
    # head chunk windows (each output pixel updated by exactly one launch)
    dict(TINY, **{"run.height": 64, "run.width": 96, "sampler.steps": 3, "chunk.halo": "none",
                  "chunk.targets": "stem,u0,head", "chunk.eta": 2, "chunk.omega": 3}),
])
def test_fused_sampler_step_is_bit_identical(tmp_path, over):
    """The CFG combine + Euler / DDIM / ancestral update applied in the K8
    head's epilogue (csrc/subpix_tc.cu, the tiles of both branches of a
    frame on one CTA) equals the separate step kernel (LC_FUSED_STEP=0) bit
    for bit: same eps values, same two-rounding order."""
    import os
    import subprocess
    import sys
    outs = []
    for fused in ("1", "0"):
        path = str(tmp_path / f"fs_{fused}.npz")
        env = dict(os.environ, LC_FUSED_STEP=fused)
        r = subprocess.run([sys.executable, "-c", _K8_CHILD, repr(over), path], env=env, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(path))
    assert np.array_equal(outs[0]["lat"], outs[1]["lat"])
    assert np.array_equal(outs[0]["v"], outs[1]["v"])


@pytest.mark.parametrize("over", [
    TINY,
    dict(TINY, **{"unet.cache_depth": 1, "sampler.steps": 5}),
    dict(TINY, **{"sampler.kind": "ancestral", "cache.n": 3, "sampler.steps": 7}),
    dict(TINY, **{"chunk.targets": "d1,u1,u0", "chunk.halo": "none"}),
])
def test_branch_deep_path_is_bit_identical(tmp_path, over):
    """The per-branch deep path of evicting full steps (forward_dev,
    chosen on slow host links) runs the same per-image arithmetic as the
    whole-batch path: bit-identical latents and videos (LC_BRANCH_DEEP=1
    vs 0)."""
    import os
    import subprocess
    import sys
    outs = []
    for bd in ("1", "2", "0"):  # per-branch deep path, per-branch up path, whole batch
        path = str(tmp_path / f"bd_{bd}.npz")
        env = dict(os.environ, LC_BRANCH_DEEP=bd)
        r = subprocess.run([sys.executable, "-c", _K8_CHILD, repr(over), path], env=env, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(path))
    for o in outs[:2]:
        assert np.array_equal(o["lat"], outs[2]["lat"])
        assert np.array_equal(o["v"], outs[2]["v"])


_HALO_CHILD = r"""
import sys, numpy as np
import paper_2510_05367_b200 as lc
over = eval(sys.argv[1])
ctx = lc.Context(0)
ctx.configure(lc.config_text(over, base=lc.DEFAULT_CONFIG))
v, lat, _ = ctx.run_pipeline(want_latent=True)
kv = lc.parse_config(lc.config_text(over, base=lc.DEFAULT_CONFIG))
ctx.upload_latent(lc.randn(lc.derive_seed(int(kv["run.seed"]), 1), ctx.latent_elems()))
ctx.set_conv_profile(True)
ctx.run_resident()
halo = sum(" halo" in r["desc"] for r in ctx.conv_profile_records())
np.savez(sys.argv[2], v=v, lat=lat, halo=halo)
"""


@pytest.mark.parametrize("over", [
    # 1024x576 video, 2 frames: decoder up-convs on 128- and 256-wide
    # lattices and the base-32 U-Net's level-0 3x3 convs (128 wide) run
    # halo-staged
    {"run.frames": 2, "run.height": 576, "run.width": 1024, "codec.stages": 3, "codec.width": 128,
     "unet.base_channels": 32, "unet.depth": 3, "sampler.steps": 2, "cache.n": 2},
    # B's frame-0 slice: dec2 (128 wide) halo-staged
    dict(B_SHAPE, **{"run.frames": 1, "sampler.steps": 2}),
    # C's frame-0 slice: d0 (320 -> 320 on the 128-wide level 0) halo-staged
    # with a streamed weight ring (no resident panel)
    dict(C_SHAPE, **{"run.frames": 1, "sampler.steps": 2}),
])
def test_halo_staging_is_bit_identical(tmp_path, over):
    """Halo operand staging (one TMA box per channel block feeding every tap
    through row-shifted descriptors, conv_tc.cu) accumulates in the same
    (segment, channel block, tap) order as per-tap staging (LC_HALO=0):
    bit-identical latents and videos."""
    import os
    import subprocess
    import sys
    outs = []
    for halo in ("1", "0"):
        path = str(tmp_path / f"halo_{halo}.npz")
        env = dict(os.environ, LC_HALO=halo)
        r = subprocess.run([sys.executable, "-c", _HALO_CHILD, repr(over), path], env=env, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(path))
    assert int(outs[0]["halo"]) > 0 and int(outs[1]["halo"]) == 0  # the switch really changed the staging
    assert np.isfinite(outs[0]["v"]).all()
    assert np.array_equal(outs[0]["lat"], outs[1]["lat"])
    assert np.array_equal(outs[0]["v"], outs[1]["v"])


def test_decode_edge_cases(ctx, oracle):
    """decode_sliced edge cases: zero frames, a slice larger than the batch,
    slices that do not divide it (ragged last slice)."""
    over = dict(TINY, **{"run.frames": 5})
    ctx.configure(lc.config_text(over, base=DEFAULT))
    empty = ctx.decode(np.zeros((1, 0, 4, 8, 8), np.float32))
    assert empty.shape == (1, 0, 3, 32, 32)
    lat = np.random.default_rng(9).standard_normal((1, 5, 4, 8, 8)).astype(np.float32)
    want = oracle.decode(_kv(over), lat)
    for g in (3, 7):  # ragged tail, slice > frames
        got = ctx.decode(lat, slice_frames=g)
        assert lc.rel_l2(got, want) < TOL
