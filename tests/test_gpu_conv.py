"""Tensor-core conv kernel vs the CPU oracle's conv2d_window
(proj/src/tensor.cpp:155-197) on affine-conditioned inputs.

Tolerance: relative L2 <= 2e-3 per single conv (fp16 operands, fp32
accumulate); the end-to-end bar of 1e-3 is checked in test_gpu_pipeline.py.
"""
import numpy as np
import pytest

import paper_2510_05367_b200 as lc

pytestmark = pytest.mark.gpu

CONV_TOL = 2e-3


def _bank(rng, c_out, c_in, k):
    taps = rng.standard_normal((c_out, c_in, k, k)).astype(np.float32) / np.sqrt(k * k * c_in)
    bias = (0.05 * rng.standard_normal(c_out)).astype(np.float32)
    return taps, bias


def _silu(v):
    return v / (1.0 + np.exp(-v))


@pytest.mark.parametrize("shape", [
    (2, 1, 64, 8, 8, 64, 3),      # one channel block, tiny image (TI=2 tiles)
    (2, 2, 320, 16, 16, 320, 3),  # base-320 width, two N tiles of 160
    (1, 2, 128, 36, 64, 640, 3),  # non-power-of-two height, BN=224 with padding
    (2, 1, 8, 32, 32, 8, 3),      # channel padding 8 -> 64
    (1, 1, 64, 9, 16, 256, 3),    # partial row tiles (9 rows)
    (1, 1, 64, 16, 16, 64, 5),    # k = 5
    (1, 1, 64, 16, 16, 64, 1),    # k = 1
])
def test_conv2d_matches_oracle(ctx, oracle, shape):
    b, t, c, h, w, c_out, k = shape
    rng = np.random.default_rng(1)
    x = rng.standard_normal((b, t, c, h, w)).astype(np.float32)
    taps, bias = _bank(rng, c_out, c, k)
    s, o = 1.03, -0.02
    want = oracle.conv2d_window(x * np.float32(s) + np.float32(o), taps, bias, k)
    got = ctx.conv2d(x, taps, bias, s=s, o=o, silu=False)
    assert lc.rel_l2(got, want) < CONV_TOL
    got_silu = ctx.conv2d(x, taps, bias, s=s, o=o, silu=True)
    assert lc.rel_l2(got_silu, _silu(want)) < CONV_TOL


@pytest.mark.parametrize("shape", [
    (2, 1, 64, 64, 16, 16, 64),
    (1, 2, 320, 640, 32, 32, 320),
    (1, 1, 128, 128, 18, 32, 128),
])
def test_up_conv2d_subpixel_matches_oracle(ctx, oracle, shape):
    """run_up_block (proj/src/unet.cpp:101-122): conv(concat(affine(skip),
    affine(upsample2(u)))) + SiLU, upsample fused as sub-pixel taps."""
    b, t, ca, cb, h, w, c_out = shape
    rng = np.random.default_rng(2)
    skip = rng.standard_normal((b, t, ca, h, w)).astype(np.float32)
    u = rng.standard_normal((b, t, cb, h // 2, w // 2)).astype(np.float32)
    taps, bias = _bank(rng, c_out, ca + cb, 3)
    s, o = 0.97, 0.05
    up = np.repeat(np.repeat(u, 2, axis=3), 2, axis=4)
    cat = np.concatenate([skip, up], axis=2) * np.float32(s) + np.float32(o)
    want = _silu(oracle.conv2d_window(cat, taps, bias, 3))
    got = ctx.up_conv2d(skip, u, taps, bias, s=s, o=o)
    assert lc.rel_l2(got, want) < CONV_TOL
