"""Oracle pins for the second workload: HE baseline and quality metrics.

Definitions: SPEC.md metrics module; HE is Eq. 5.  Every check below is
fixed by something other than the oracle's own formula: closed forms (constant images, a
single-sample difference, grey images against their inverse), exact identities (SSIM of an
image with itself is 1 exactly; LOE is invariant under strictly increasing maps) and the SPEC
examples (all-0 vs all-255 is 0 dB; a vs 255 - a has SSIM < 0.5).
"""
import math

import numpy as np
import pytest

import oracle
import synth

C1 = (0.01 * 255.0) ** 2


def test_psnr_identity_and_extremes():
    a = synth.make_image(24, 31, seed=1)
    assert oracle.psnr(a, a) == math.inf
    z = np.zeros((7, 9, 3), np.uint8)
    assert oracle.psnr(z, z + 255) == 0.0  # SPEC example: MSE == 255^2


@pytest.mark.parametrize("d", [1, 3, 17, 128])
def test_psnr_constant_difference_closed_form(d):
    a = np.full((13, 11, 3), 60, np.uint8)
    b = a + np.uint8(d)
    assert oracle.psnr(a, b) == pytest.approx(10 * math.log10(255.0 ** 2 / d ** 2), rel=1e-15)
    assert oracle.psnr(b, a) == oracle.psnr(a, b)  # symmetry


def test_psnr_single_sample():
    a = np.zeros((10, 10, 3), np.uint8)
    b = a.copy()
    b[3, 4, 1] = 9  # MSE = 81 / 300
    assert oracle.psnr(a, b) == pytest.approx(10 * math.log10(255.0 ** 2 * 300 / 81), rel=1e-15)


def test_ssim_identity_is_exactly_one():
    a = synth.make_image(40, 57, seed=2)
    assert oracle.ssim(a, a) == 1.0


@pytest.mark.parametrize("c1,c2", [(30, 33), (100, 140), (0, 255)])
def test_ssim_constant_patches_closed_form(c1, c2):
    a = np.full((16, 20, 3), c1, np.uint8)
    b = np.full((16, 20, 3), c2, np.uint8)
    ya = 0.299 * c1 + 0.587 * c1 + 0.114 * c1
    yb = 0.299 * c2 + 0.587 * c2 + 0.114 * c2
    ref = (2 * ya * yb + C1) / (ya * ya + yb * yb + C1)  # variance terms vanish
    assert oracle.ssim(a, b) == pytest.approx(ref, rel=1e-9)


def test_ssim_symmetric_bounded_and_inverse_low():
    a = synth.make_image(48, 64, seed=3, peak=0.4)
    b = synth.make_image(48, 64, seed=4, peak=0.4)
    s_ab, s_ba = oracle.ssim(a, b), oracle.ssim(b, a)
    assert abs(s_ab - s_ba) <= 1e-12 and s_ab <= 1.0
    # SPEC example: a mid-contrast image against its inverse scores below 0.5
    g = np.clip(np.linspace(40, 210, 64)[None, :, None] + np.zeros((48, 64, 3)), 0, 255).astype(np.uint8)
    g = np.ascontiguousarray(np.clip(g.astype(int) + synth.make_image(48, 64, seed=5) // 4, 0, 255).astype(np.uint8))
    assert oracle.ssim(g, 255 - g) < 0.5


def test_ssim_too_small_is_nan():
    a = np.zeros((10, 40, 3), np.uint8)
    assert math.isnan(oracle.ssim(a, a))


def test_loe_zero_for_monotone_maps():
    a = synth.make_image(60, 70, seed=6, peak=0.15)
    assert oracle.loe(a, a) == 0.0
    assert int(a.max()) <= 127
    f = (2 * np.arange(256) + 1).clip(0, 255).astype(np.uint8)  # strictly increasing on 0..127
    g = f[a]  # the same increasing map on every channel: L' = f(L), order of L preserved
    assert oracle.loe(a, g) == 0.0


@pytest.mark.parametrize("seed", [7, 8])
def test_loe_inverse_grey_closed_form(seed):
    v = (synth.make_image(50, 60, seed=seed, peak=0.35).max(-1)).astype(np.uint8)  # <= 100 x 100: no sampling
    grey = np.repeat(v[:, :, None], 3, axis=2)
    inv = 255 - grey
    m = v.size
    n = np.bincount(v.ravel(), minlength=256).astype(np.float64)
    ref = (m * m - np.sum(n * n)) / m  # pairs with different L flip order, equal L never do
    assert oracle.loe(grey, inv) == ref


def test_loe_sampling_grid():
    """Above 100 x 100 the metric samples row (i H) / 100, column (j W) / 100: an image that is
    constant on every sampled block-representative equals the small image's value."""
    small = synth.make_image(100, 100, seed=9, peak=0.3)
    big = np.repeat(np.repeat(small, 3, axis=0), 2, axis=1)  # 300 x 200, sample (3i, 2j) -> small[i, j]
    small_e = 255 - small
    big_e = np.repeat(np.repeat(small_e, 3, axis=0), 2, axis=1)
    assert oracle.loe(big, big_e) == oracle.loe(small, small_e)


def test_he_enhance_grey_follows_eq5():
    v = synth.make_image(40, 50, seed=10, peak=0.2).max(-1).astype(np.uint8)
    grey = np.repeat(v[:, :, None], 3, axis=2)
    t = oracle.he_transform(np.bincount(v.ravel(), minlength=256))
    out = oracle.he_enhance(grey)
    assert np.array_equal(out, np.repeat(t[v][:, :, None], 3, axis=2).astype(np.uint8))
    assert np.all(np.diff(t) >= 0) and t[-1] == 255
