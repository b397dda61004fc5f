"""Operator-level sampler update and all_finite on the device, against the
reference's own outputs (tests/golden/sampler.npz, made by
tests/golden/make_golden.py `sampler` from oracle/_ref).

cfg_combine + reverse_step_{ancestral,ddim,euler} (proj/src/sampler.cpp:
95-133) are fp32 elementwise work in the reference's two-rounding order, so
the bar is bit-exact; n = 1027 covers the 16-byte vector body and the scalar
tail of the kernel.
"""
import os

import numpy as np
import pytest

import paper_2510_05367_b200 as lc

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "sampler.npz")
CASES = ["euler_t24", "euler_t0", "ddim_t12", "ddim_t0", "ancestral_t7", "ancestral_t0", "euler_s6_t5",
         "ancestral_s6_t3"]


@pytest.mark.parametrize("name", CASES)
def test_sampler_step_matches_reference(ctx, name):
    g = np.load(GOLD)
    kind, t, seed = (int(v) for v in g[name + "_args"])
    ctx.configure(str(g[name + "_config"]))
    out, bad = ctx.sampler_step(kind, t, g[name + "_x"], g[name + "_eu"], g[name + "_ec"], float(g[name + "_g"]),
                                seed)
    assert not bad
    assert np.array_equal(out, g[name + "_out"])


def test_sampler_step_errors_and_nonfinite(ctx):
    ctx.configure("sampler.steps = 6")
    x = np.ones(37, np.float32)
    with pytest.raises(lc.ConfigError):  # check_t (sampler.cpp:79-84)
        ctx.sampler_step("euler", 6, x, x, x, 1.5)
    with pytest.raises(lc.ConfigError):
        ctx.sampler_step("ddim", -1, x, x, x, 1.5)
    with pytest.raises(lc.ConfigError):  # cfg_combine (sampler.cpp:130)
        ctx.sampler_step("ancestral", 2, x, x, x, -0.5)
    with pytest.raises(lc.ShapeError):  # cfg_combine (sampler.cpp:129)
        ctx.sampler_step("euler", 2, x, x[:5], x, 1.5)
    for pos in (3, 36):  # vector body, scalar tail
        e = x.copy()
        e[pos] = np.inf
        out, bad = ctx.sampler_step("euler", 2, x, x, e, 1.5)
        assert bad and not np.isfinite(out[pos])
    out, bad = ctx.sampler_step("euler", 2, x[:0], x[:0], x[:0], 1.5)
    assert out.size == 0 and not bad


def test_all_finite(ctx):
    rng = np.random.default_rng(5)
    x = rng.standard_normal(4 * 1000 + 3).astype(np.float32)
    assert ctx.all_finite(x)
    for pos, v in [(0, np.nan), (1234, np.inf), (x.size - 1, -np.inf), (x.size - 2, np.nan)]:
        y = x.copy()
        y[pos] = v
        assert not ctx.all_finite(y)
    assert ctx.all_finite(x[:0])
    assert ctx.all_finite(x[1:])  # n % 4 == 2: a two-element scalar tail
    y = x.copy()
    y[7] = np.nan
    assert not ctx.all_finite(y[1:])
