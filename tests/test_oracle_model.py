"""Pins for the oracle's histogram-domain model: Eqs. 6-8, 11 and the index maps
(Eqs. 17-19).  CPU only.

Independent references used here: exact-integer closed forms of the nearest bin,
high-precision decimal evaluation of b_i * b_j^(1/gamma), exhaustive enumeration of
(i, j) cells in exact rationals, and brute-force enumeration of all N^2 pixel pairs
of a 4x4 image.
"""
import json
import os
from decimal import Decimal, getcontext
from fractions import Fraction

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def nearest_low_tie(x: Fraction, levels: int) -> int:
    """argmin_k |x - k/(l-1)|, smallest k on ties, exact."""
    y = x * (levels - 1)
    k = y.numerator // y.denominator  # floor
    # candidates k, k+1
    if k + 1 <= levels - 1 and (y - k) > (k + 1 - y):
        return k + 1
    return min(k, levels - 1)


# ----------------------------------------------------------- index map
@pytest.mark.parametrize("levels", [3, 4, 8, 256])
def test_index_map_closed_form(levels):
    idx = oracle.index_map(levels, 1.0)
    i = np.arange(levels)[:, None]
    j = np.arange(levels)[None, :]
    closed = (i * j + (levels - 2) // 2) // (levels - 1)
    assert np.array_equal(idx, closed)


@pytest.mark.parametrize("levels", [3, 4, 8])
def test_index_map_exact_rationals(levels):
    idx = oracle.index_map(levels, 1.0)
    for i in range(levels):
        for j in range(levels):
            x = Fraction(i, levels - 1) * Fraction(j, levels - 1)
            assert idx[i, j] == nearest_low_tie(x, levels)


def test_index_map_golden_and_monotone():
    for ex in GOLD["index_map"]:
        assert oracle.index_map(ex["levels"])[ex["i"], ex["j"]] == ex["k"], ex["cite"]
    idx = oracle.index_map(256)
    assert np.all(np.diff(idx, axis=1) >= 0) and np.all(np.diff(idx, axis=0) >= 0)
    assert np.diff(idx, axis=1).max() <= 1  # rows are steps of at most 1
    assert np.array_equal(idx, idx.T)


def _idx1_decimal(levels, gamma):
    getcontext().prec = 50
    g = Decimal(gamma)  # the exact binary value of the fp64 gamma
    inv = Decimal(1) / g
    p = [Decimal(0)] + [(Decimal(j) / (levels - 1)) ** inv for j in range(1, levels)]
    out = np.empty((levels, levels), np.int64)
    margin = 1.0
    half = Decimal(1) / 2
    for i in range(levels):
        bi = Decimal(i) / (levels - 1)
        for j in range(levels):
            y = bi * p[j] * (levels - 1)
            k = int(y)  # floor (y >= 0)
            frac = y - k
            out[i, j] = k + 1 if frac > half else k
            margin = min(margin, float(abs(frac - half)))
    return out, margin


@pytest.mark.parametrize("gamma", [1.5, 2.2, 5.0, 10.0])
def test_index1_high_precision(gamma):
    idx1 = oracle.index_map(256, gamma)
    ref, margin = _idx1_decimal(256, gamma)
    assert margin > 1e-9  # no fp64-unsafe near tie (measured: >= 1.5e-7 bins)
    assert np.array_equal(idx1, ref)


@pytest.mark.parametrize("gamma", [1.5, 2.2, 5.0, 10.0])
def test_index1_dominates_index(gamma):
    idx = oracle.index_map(256, 1.0)
    idx1 = oracle.index_map(256, gamma)
    assert np.all(idx1 >= idx)
    assert idx1[255, 255] == 255 and idx1[0, 200] == 0
    assert np.all(np.diff(idx1, axis=1) >= 0) and np.all(np.diff(idx1, axis=0) >= 0)


def test_index1_gamma1_is_index():
    assert np.array_equal(oracle.index_map(256, 1.0), oracle.index_map(256, 1.0 + 0.0))


# ----------------------------------------------------- Eqs. 6-8, 11
def test_pair_count_golden():
    for ex in GOLD["pair_count"]:
        C = oracle.pair_count(ex["hR"], ex["hL"], ex["N"])
        assert C.tolist() == ex["C"], ex["cite"]
    b = oracle.locations(3)
    assert np.outer(b, b).tolist() == GOLD["location_matrix"][0]["M"]
    for ex in GOLD["locations"]:
        assert oracle.locations(ex["levels"]).tolist() == ex["b"]


def test_weights_special_cases():
    l = 4
    idx = oracle.index_map(l)
    # single nonzero cell feeding its bin -> K = 1
    hR = np.array([0, 0, 0, 5.0])
    hL = np.array([0, 0, 5.0, 0])
    C = oracle.pair_count(hR, hL, 5.0)
    est = oracle.estimate(C, idx)
    K = oracle.weights(C, idx, est)
    assert K[3, 2] == 1.0 and np.count_nonzero(K) == 1
    # two equal cells feeding one bin -> 0.5 each (idx(1,3)=idx(3,1)=1 for l=4)
    hR = np.array([0, 2.0, 0, 2.0])
    hL = np.array([0, 2.0, 0, 2.0])
    C = oracle.pair_count(hR, hL, 4.0)
    K = oracle.weights(C, idx, oracle.estimate(C, idx))
    assert idx[1, 3] == idx[3, 1] == 1 and idx[1, 1] == 0
    assert K[1, 3] == 0.5 and K[3, 1] == 0.5
    # zero-mass cells -> 0
    assert K[0, 0] == 0.0 and K[2, 2] == 0.0


@pytest.mark.parametrize("seed", range(20))
def test_weights_partition_of_unity(seed):
    rng = np.random.default_rng(seed)
    l = int(rng.integers(2, 33))
    idx = oracle.index_map(l)
    hR = rng.random(l) * (rng.random(l) < 0.7)
    hL = rng.random(l) * (rng.random(l) < 0.7)
    hR[0] += 0.1
    hL[-1] += 0.1
    N = 50.0
    hR *= N / hR.sum()
    hL *= N / hL.sum()
    C = oracle.pair_count(hR, hL, N)
    est = oracle.estimate(C, idx)
    K = oracle.weights(C, idx, est)
    assert abs(est.sum() - N) <= 1e-9 * N  # mass conservation
    for k in range(l):
        if est[k] > 0:
            assert abs(K[idx == k].sum() - 1.0) <= 1e-12


def test_estimate_exhaustive_small_levels():
    """Eq. 8 vs exhaustive enumeration in exact rationals, l <= 8, integer masses <= 8.

    l = 7 is excluded: with l-1 = 6 the cell values b_i b_j can sit exactly half-way
    between two bins (e.g. (3/6)(3/6) = 1.5/6) while the fp64 bin locations k/6 are
    rounded, so the oracle's fp64 argmin may break such exact ties either way.  For
    l-1 odd there are no exact ties; for l-1 a power of two every location is exact.
    l = 256 (the only level count of the CUDA path) has l-1 = 255 odd: no exact ties."""
    rng = np.random.default_rng(99)
    for case in range(300):
        l = int(rng.choice([2, 3, 4, 5, 6, 8, 9]))
        hR = rng.integers(0, 9, size=l)
        hL = rng.integers(0, 9, size=l)
        if hR.sum() == 0 or hL.sum() == 0:
            continue
        N = int(hR.sum())
        idx = oracle.index_map(l)
        est = oracle.estimate(oracle.pair_count(hR, hL, N), idx)
        ref = [Fraction(0)] * l
        for i in range(l):
            for j in range(l):
                k = nearest_low_tie(Fraction(i, l - 1) * Fraction(j, l - 1), l)
                ref[k] += Fraction(int(hR[i]) * int(hL[j]), N)
        for k in range(l):
            assert abs(est[k] - float(ref[k])) <= 1e-12 * max(1.0, float(ref[k])), (case, k)


def test_estimate_spike_identity():
    # reflectance == 1 (spike at l-1) composed with an illumination spike at v -> spike at v
    l = 256
    idx = oracle.index_map(l)
    for v in [0, 1, 37, 128, 255]:
        hR = np.zeros(l)
        hR[l - 1] = 1000.0
        hL = np.zeros(l)
        hL[v] = 1000.0
        est = oracle.estimate(oracle.pair_count(hR, hL, 1000.0), idx)
        assert est[v] == 1000.0 and np.count_nonzero(est) == 1


@pytest.mark.parametrize("seed", range(6))
def test_estimate_pixel_pair_bruteforce_4x4(seed):
    """Eqs. 6-8 rebuilt by enumerating all N^2 (gradient pixel, value pixel) pairs of a
    4x4 image: Est_k = (1/N) #{(p, q) : nearest(b_G'(p) * b_S(q)) = k}."""
    rng = np.random.default_rng(seed)
    levels = [256, 8, 4][seed % 3]
    img = rng.integers(0, 256, size=(4, 4, 3), dtype=np.uint8)
    S = oracle.value_channel(img, levels)
    G = oracle.gradient_levels(oracle.gradient_raw(S), levels, seed % 2)
    hS = oracle.count_histogram(S, levels).astype(float)
    hG = oracle.count_histogram(G, levels).astype(float)
    N = 16
    est = oracle.estimate(oracle.pair_count(hG, hS, N), oracle.index_map(levels))
    ref = np.zeros(levels)
    for gp in G.ravel():
        for sq in S.ravel():
            k = (int(gp) * int(sq) + (levels - 2) // 2) // (levels - 1)
            ref[k] += 1.0 / N
    assert np.allclose(est, ref, rtol=0, atol=1e-12)
