"""GPU quality metrics against the oracle pinned to the
reference (tests/golden/metrics.npz made by oracle/_ref).

Each 7x7 window's SSIM term and each squared difference are computed with
the reference's double arithmetic exactly; only the sums over windows and
pixels run as fixed-order trees, so the bar is 1e-12 relative."""
import os

import numpy as np
import pytest

import paper_2510_05367_b200 as lc

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "metrics.npz")
RTOL = 1e-12


@pytest.mark.parametrize("name", ["noise", "same", "pipe"])
def test_metrics_match_reference_golden(ctx, name):
    g = np.load(GOLD)
    ps, ss = ctx.video_metrics(g[name + "_a"][0], g[name + "_b"][0], 1.0)
    np.testing.assert_allclose(ps, g[name + "_psnr"], rtol=RTOL, atol=0)
    np.testing.assert_allclose(ss, g[name + "_ssim"], rtol=RTOL, atol=0)


def test_metrics_match_oracle_shapes(ctx, oracle):
    rng = np.random.default_rng(9)
    for shape in [(1, 1, 7, 7), (3, 3, 40, 70), (2, 3, 128, 96), (1, 2, 23, 17)]:
        a = rng.random(shape).astype(np.float32)
        b = np.clip(a + 0.05 * rng.standard_normal(shape), 0, 1).astype(np.float32)
        for L in (1.0, 255.0):
            po, so = oracle.video_metrics(a, b, L)
            pg, sg = ctx.video_metrics(a, b, L)
            np.testing.assert_allclose(pg, po, rtol=RTOL, atol=0)
            np.testing.assert_allclose(sg, so, rtol=RTOL, atol=0)
    ps, ss = ctx.video_metrics(a, a, 1.0)
    assert (ps == 99.0).all() and (ss == 1.0).all()


def test_metrics_errors(ctx):
    a = np.zeros((1, 1, 6, 9), np.float32)
    with pytest.raises(lc.ShapeError):
        ctx.video_metrics(a, a, 1.0)
    a = np.zeros((1, 1, 8, 8), np.float32)
    with pytest.raises(lc.ConfigError):
        ctx.video_metrics(a, a, -1.0)
