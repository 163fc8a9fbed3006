"""Pins for the oracle's pixel-domain steps (O1, O2, Eq. 3, O11) -- CPU only.

Each check compares the oracle against something other than itself: golden examples
(tests/golden, cited), closed forms in exact integer/rational arithmetic, numpy
brute force, and textbook hexcone HSV written here with fractions.Fraction.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ------------------------------------------------------------------ O1
@pytest.mark.parametrize("levels", [2, 3, 4, 8, 256])
def test_value_channel_closed_form(levels):
    # every 8-bit max value m -> round_half_up(m (l-1) / 255), exact integer arithmetic
    m = np.arange(256, dtype=np.uint8)
    rgb = np.stack([m, m // 2, m // 3], axis=-1)
    S = oracle.value_channel(rgb, levels)
    expect = (2 * m.astype(np.int64) * (levels - 1) + 255) // 510
    assert np.array_equal(S, expect)


def test_value_channel_is_max():
    rgb = np.random.default_rng(0).integers(0, 256, size=(5000, 3), dtype=np.uint8)
    assert np.array_equal(oracle.value_channel(rgb), rgb.max(-1))


# ------------------------------------------------------------- Eq. 3
def test_histogram_golden():
    for ex in GOLD["count_histogram"]:
        h = oracle.count_histogram(np.array(ex["pixels"]), ex["levels"])
        assert h.tolist() == ex["hist"], ex["cite"]


@pytest.mark.parametrize("seed", range(5))
def test_histogram_bruteforce(seed):
    rng = np.random.default_rng(seed)
    x = rng.integers(0, 256, size=rng.integers(1, 5000))
    h = oracle.count_histogram(x, 256)
    assert np.array_equal(h, np.bincount(x, minlength=256))
    assert int(h.sum()) == x.size


def test_histogram_constant_and_permutation():
    h = oracle.count_histogram(np.full(1234, 17), 256)
    assert np.count_nonzero(h) == 1 and h[17] == 1234
    h = oracle.count_histogram(np.random.default_rng(1).permutation(256), 256)
    assert np.all(h == 1)


def test_histogram_empty_is_error():
    with pytest.raises(oracle.OracleError):
        oracle.count_histogram(np.zeros(0, np.int32), 256)


# ------------------------------------------------------------------ O2
def test_gradient_golden():
    for ex in GOLD["gradient"]:
        g = oracle.gradient_raw(np.array(ex["S"]))
        assert g.tolist() == ex["g"], ex["cite"]


def _np_gradient(S):
    S = S.astype(np.int64)
    dx = np.zeros_like(S)
    dy = np.zeros_like(S)
    dx[:, :-1] = np.diff(S, axis=1)
    dy[:-1, :] = np.diff(S, axis=0)
    return np.abs(dx) + np.abs(dy)


@pytest.mark.parametrize("shape", [(4, 4), (1, 9), (9, 1), (1, 1), (13, 7)])
def test_gradient_vs_numpy(shape):
    S = np.random.default_rng(sum(shape)).integers(0, 256, size=shape)
    assert np.array_equal(oracle.gradient_raw(S), _np_gradient(S))


def _maxnorm_exact(g, levels):
    gmax = int(g.max())
    if gmax == 0:
        return np.zeros_like(g)
    out = np.empty_like(g)
    for p, v in np.ndenumerate(g):
        q = Fraction((levels - 1) * int(v), gmax) + Fraction(1, 2)
        out[p] = q.numerator // q.denominator  # floor(x + 1/2): round half up
    return out


@pytest.mark.parametrize("gmax", [1, 2, 3, 7, 100, 509, 510])
def test_gradient_maxnorm_exact(gmax):
    rng = np.random.default_rng(gmax)
    g = rng.integers(0, gmax + 1, size=400)
    g[0] = gmax
    q = oracle.gradient_levels(g, 256, 0)
    assert np.array_equal(q, _maxnorm_exact(g, 256))
    assert q.max() == 255


def test_gradient_maxnorm_ties_round_up():
    # g=1, gmax=2 -> 127.5 -> 128 (half up)
    assert oracle.gradient_levels(np.array([0, 1, 2]), 256, 0).tolist() == [0, 128, 255]


def test_gradient_raw_clamp():
    g = np.array([0, 5, 255, 256, 510])
    assert oracle.gradient_levels(g, 256, 1).tolist() == [0, 5, 255, 255, 255]


def test_gradient_all_zero_maxnorm():
    assert np.all(oracle.gradient_levels(np.zeros(10, np.int32), 256, 0) == 0)


# ------------------------------------------------------------------ O11
def _hexcone_fraction(r, g, b, vnew):
    """Textbook hexcone RGB->HSV, V replaced, HSV->RGB, in exact Fractions, 8-bit half up."""
    r, g, b = Fraction(r, 255), Fraction(g, 255), Fraction(b, 255)
    mx, mn = max(r, g, b), min(r, g, b)
    v = Fraction(vnew, 255)
    if mx == mn:
        out = (v, v, v)
    else:
        s = (mx - mn) / mx
        d = mx - mn
        if r == mx:
            h = (g - b) / d
        elif g == mx:
            h = 2 + (b - r) / d
        else:
            h = 4 + (r - g) / d
        h = (h / 6) % 1
        i = int(h * 6)  # floor, h >= 0
        f = h * 6 - i
        p, q, t = v * (1 - s), v * (1 - s * f), v * (1 - s * (1 - f))
        out = [(v, t, p), (q, v, p), (p, v, t), (p, q, v), (t, p, v), (v, p, q)][i % 6]
    res = []
    for c in out:
        x = c * 255 + Fraction(1, 2)
        res.append(x.numerator // x.denominator)
    return tuple(res)


def test_reconstruct_vs_fraction_hexcone():
    rng = np.random.default_rng(7)
    rgb = rng.integers(0, 256, size=(3000, 3), dtype=np.uint8)
    rgb[:50] = rng.integers(0, 4, size=(50, 3))  # tiny values
    rgb[50:80, 0] = rgb[50:80, 1]  # ties between channels
    Vn = rng.integers(0, 256, size=3000)
    out = oracle.reconstruct(rgb, Vn)
    for p in range(3000):
        assert tuple(out[p]) == _hexcone_fraction(*map(int, rgb[p]), int(Vn[p])), (rgb[p], Vn[p])


def test_reconstruct_integer_closed_form_grid():
    # scaling form (R17): out_c = floor((2 c V' + V) / (2 V)), V=0 -> V'
    vals = np.array([0, 1, 2, 3, 17, 64, 127, 128, 200, 254, 255])
    R, G, B, Vn = np.meshgrid(vals, vals, vals, vals, indexing="ij")
    rgb = np.stack([R.ravel(), G.ravel(), B.ravel()], -1).astype(np.uint8)
    Vn = Vn.ravel()
    out = oracle.reconstruct(rgb, Vn).astype(np.int64)
    V = rgb.max(-1).astype(np.int64)
    c = rgb.astype(np.int64)
    Vs = np.maximum(V, 1)[:, None]
    expect = (2 * c * Vn[:, None] + Vs) // (2 * Vs)
    expect[V == 0] = Vn[V == 0, None]
    assert np.array_equal(out, expect)


def test_reconstruct_identity_when_v_unchanged():
    rgb = np.random.default_rng(3).integers(0, 256, size=(4000, 3), dtype=np.uint8)
    assert np.array_equal(oracle.reconstruct(rgb, rgb.max(-1)), rgb)


def test_hsv_golden():
    for ex in GOLD["hsv"]:
        rgb = np.array([ex["rgb"]], np.uint8)
        v = int(rgb.max())
        assert v == round(ex.get("v", ex.get("v_times_255", 0) / 255) * 255)
        # replacing V by itself reproduces the pixel; grey stays grey at any V'
        assert oracle.reconstruct(rgb, [v]).tolist() == [ex["rgb"]]
    grey = oracle.reconstruct(np.array([[128, 128, 128]], np.uint8), [200])
    assert grey.tolist() == [[200, 200, 200]]
    red = oracle.reconstruct(np.array([[255, 0, 0]], np.uint8), [100])
    assert red.tolist() == [[100, 0, 0]]


def test_edge_images_histograms_sum_to_n():
    for name, img in synth.edge_images().items():
        r = oracle.enhance(img)
        n = img.shape[0] * img.shape[1]
        assert int(r.hS.sum()) == n and int(r.hG.sum()) == n and int(r.hgraw.sum()) == n, name
