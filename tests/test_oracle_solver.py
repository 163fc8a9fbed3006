"""Pins for the oracle's Algorithm 1 (Eqs. 10-15).  CPU only.

Independent references: the prior-dominated limits of Eqs. 12-13 (alpha, beta -> inf),
the identity-composition special case, exact coordinate minimisation of the quadratic
objective Eq. 10 (checked with finite differences of the oracle's J, a different
formula from the updates), monotone descent, support invariance, and the algebraically
factored update ("factored form") evaluated here with numpy --
a different arithmetic route to the same numbers.
"""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _rand_hists(rng, l, N=1000.0, p0=0.7):
    hS = np.floor(rng.random(l) * 50) * (rng.random(l) < p0)
    hG = np.floor(rng.random(l) * 50) * (rng.random(l) < p0)
    hS[int(rng.integers(l))] += 7
    hG[0] += 7
    hS *= N / hS.sum()
    hG *= N / hG.sum()
    return hS, hG


def test_renormalize_golden():
    for ex in GOLD["renormalize"]:
        assert oracle.renormalize(ex["h"], ex["N"]).tolist() == [float(v) for v in ex["out"]], ex["cite"]
    h = np.random.default_rng(0).random(256)
    h1 = oracle.renormalize(h, 77.0)
    assert np.allclose(oracle.renormalize(h1, 77.0), h1, rtol=1e-12, atol=0)


def test_renormalize_degenerate():
    with pytest.raises(oracle.OracleError):
        oracle.renormalize(np.zeros(4), 8.0)


def _setup(seed, l=32):
    rng = np.random.default_rng(seed)
    hS, hG = _rand_hists(rng, l)
    N = hS.sum()
    idx = oracle.index_map(l)
    hR = hG.copy()
    hL = hS.copy()
    C = oracle.pair_count(hR, hL, N)
    K = oracle.weights(C, idx, oracle.estimate(C, idx))
    return rng, hS, hG, N, idx, hR, hL, K


def test_alpha_beta_limits():
    rng, hS, hG, N, idx, hR, hL, K = _setup(1)
    hR1 = oracle.update_reflectance(hL, hS, hG, K, idx, N, beta=1e12)
    assert np.allclose(hR1, hG, rtol=1e-3, atol=1e-6)
    hL1 = oracle.update_illumination(hR1, hS, K, idx, N, alpha=1e12)
    assert np.allclose(hL1, hS, rtol=1e-3, atol=1e-6)


@pytest.mark.parametrize("alpha", [1e-3, 0.1, 10.0])
def test_identity_composition_gives_hL_equal_hS(alpha):
    """hR = spike N at l-1 (reflectance == 1): K_{l-1,j} = 1 and idx(l-1, j) = j, so
    Eq. 12 gives hL_j = (hS_j + alpha hS_j)/(1 + alpha) = hS_j."""
    l = 64
    rng = np.random.default_rng(5)
    hS, _ = _rand_hists(rng, l)
    N = hS.sum()
    idx = oracle.index_map(l)
    hR = np.zeros(l)
    hR[-1] = N
    hLprev = rng.random(l) + 0.1
    hLprev *= N / hLprev.sum()
    C = oracle.pair_count(hR, hLprev, N)
    K = oracle.weights(C, idx, oracle.estimate(C, idx))
    hL = oracle.update_illumination(hR, hS, K, idx, N, alpha)
    assert np.allclose(hL, hS, rtol=1e-13, atol=1e-12)


@pytest.mark.parametrize("seed", range(50))
def test_descent_each_update(seed):
    """J after each Eq. 13 / Eq. 12 update (K frozen) never exceeds J before."""
    rng = np.random.default_rng(1000 + seed)
    l = 32
    hS, hG = _rand_hists(rng, l)
    p = oracle.Params(levels=l, alpha=float(rng.choice([1e-3, 0.1, 1.0])),
                      beta=float(rng.choice([1e-3, 0.1, 1.0])), max_iter=6)
    hL, hR, it, trace = oracle.decompose(hS, hG, p, trace_cap=18)
    assert it == 6 and trace.size == 18
    for t in range(6):
        j0, j1, j2 = trace[3 * t: 3 * t + 3]
        assert j1 <= j0 * (1 + 1e-9) + 1e-9
        assert j2 <= j1 * (1 + 1e-9) + 1e-9
    assert abs(hL.sum() - hS.sum()) <= 1e-9 * hS.sum()
    assert abs(hR.sum() - hS.sum()) <= 1e-9 * hS.sum()


@pytest.mark.parametrize("seed", range(5))
def test_updates_are_coordinate_minimisers(seed):
    """Eq. 13 (gradient-consistent reading R7) is the exact minimiser of the quadratic
    Eq. 10 in each hR_i; Eq. 12 likewise in each hL_j.  Checked by central differences of
    the oracle's objective (a different formula)."""
    rng, hS, hG, N, idx, hR, hL, K = _setup(10 + seed, l=16)
    a, b = 0.1, 0.05
    hR1 = oracle.update_reflectance(hL, hS, hG, K, idx, N, b)
    hL1 = oracle.update_illumination(hR1, hS, K, idx, N, a)

    def J(r, l_):
        return oracle.objective(r, l_, hS, hG, K, idx, N, a, b)

    for i in range(16):
        h = 1e-3 * max(1.0, abs(hR1[i]))
        e = np.zeros(16)
        e[i] = h
        d1 = (J(hR1 + e, hL) - J(hR1 - e, hL)) / (2 * h)
        curv = (J(hR1 + e, hL) - 2 * J(hR1, hL) + J(hR1 - e, hL)) / h**2
        assert abs(d1) <= 1e-6 * max(1.0, curv * max(1.0, abs(hR1[i])))
        d1 = (J(hR1, hL1 + e) - J(hR1, hL1 - e)) / (2 * h)
        curv = (J(hR1, hL1 + e) - 2 * J(hR1, hL1) + J(hR1, hL1 - e)) / h**2
        assert abs(d1) <= 1e-6 * max(1.0, curv * max(1.0, abs(hL1[i])))


def test_frozen_k_fixed_point_stationary():
    """Alternating Eqs. 13/12 with K frozen converge to a stationary point of Eq. 10:
    finite-difference gradient <= 1e-4."""
    rng, hS, hG, N, idx, hR, hL, K = _setup(77, l=12)
    a, b = 0.5, 0.5
    for _ in range(3000):
        hR = oracle.update_reflectance(hL, hS, hG, K, idx, N, b)
        hL = oracle.update_illumination(hR, hS, K, idx, N, a)
    for v, which in ((hR, 0), (hL, 1)):
        for i in range(12):
            e = np.zeros(12)
            e[i] = 1e-4
            if which == 0:
                g = (oracle.objective(hR + e, hL, hS, hG, K, idx, N, a, b)
                     - oracle.objective(hR - e, hL, hS, hG, K, idx, N, a, b)) / 2e-4
            else:
                g = (oracle.objective(hR, hL + e, hS, hG, K, idx, N, a, b)
                     - oracle.objective(hR, hL - e, hS, hG, K, idx, N, a, b)) / 2e-4
            assert abs(g) <= 1e-4


def test_epsilon_huge_one_iteration():
    rng = np.random.default_rng(3)
    hS, hG = _rand_hists(rng, 64)
    _, _, it, _ = oracle.decompose(hS, hG, oracle.Params(levels=64, epsilon=1e12, use_epsilon=1))
    assert it == 1
    _, _, it, _ = oracle.decompose(hS, hG, oracle.Params(levels=64, epsilon=1e12, use_epsilon=0,
                                                         max_iter=7))
    assert it == 7


@pytest.mark.parametrize("form", [0, 1])
def test_supports_frozen_and_mass_conserved(form):
    rng = np.random.default_rng(8)
    hS, hG = _rand_hists(rng, 256, N=123456.0, p0=0.3)
    for T in (1, 3, 10):
        hL, hR, it, _ = oracle.decompose(hS, hG, oracle.Params(max_iter=T, update_form=form))
        assert np.array_equal(hR > 0, hG > 0) and np.array_equal(hL > 0, hS > 0)
        assert abs(hL.sum() - hS.sum()) <= 1e-9 * hS.sum()
        assert abs(hR.sum() - hS.sum()) <= 1e-9 * hS.sum()


def _factored_gc(hS, hG, alpha, beta, T, levels=256):
    """DESIGN.md section 5 factored form: Est, rho = hS/Est, row/column gathers."""
    N = hS.sum()
    i = np.arange(levels)
    idx = (i[:, None] * i[None, :] + (levels - 2) // 2) // (levels - 1)
    hR, hL = hG.copy(), hS.copy()
    for _ in range(T):
        est = np.bincount(idx.ravel(), weights=np.outer(hR, hL).ravel() / N, minlength=levels)
        rho = np.divide(hS, est, out=np.zeros(levels), where=est > 0)
        P = rho[idx]
        hR1 = (hR * (P @ (hL * hL)) / N**2 + beta * hG) / ((hL * hL).sum() / N**2 + beta)
        hL1 = (hL * (P.T @ (hR1 * hR)) / N**2 + alpha * hS) / ((hR1 * hR1).sum() / N**2 + alpha)
        hR, hL = N * hR1 / hR1.sum(), N * hL1 / hL1.sum()
    return hL, hR


@pytest.mark.parametrize("seed", range(4))
def test_literal_equals_factored(seed):
    rng = np.random.default_rng(40 + seed)
    hS, hG = _rand_hists(rng, 256, N=664000.0, p0=[0.2, 0.5, 0.9, 1.0][seed])
    p = oracle.Params(alpha=0.1, beta=[1e-3, 0.1, 1.0, 0.01][seed], max_iter=10)
    hL, hR, it, _ = oracle.decompose(hS, hG, p)
    fL, fR = _factored_gc(hS, hG, p.alpha, p.beta, 10)
    nz = hL > 0
    assert np.max(np.abs(hL[nz] - fL[nz]) / hL[nz]) < 1e-11
    nz = hR > 0
    assert np.max(np.abs(hR[nz] - fR[nz]) / hR[nz]) < 1e-11


def test_paper_literal_form_runs_and_conserves():
    rng = np.random.default_rng(11)
    hS, hG = _rand_hists(rng, 256, N=5e5, p0=0.4)
    hL, hR, it, _ = oracle.decompose(hS, hG, oracle.Params(update_form=1))
    assert it == 10 and np.all(hL >= 0) and np.all(hR >= 0)
    assert abs(hL.sum() - 5e5) < 1e-6 * 5e5
