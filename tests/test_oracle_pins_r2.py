"""Pins for the three oracle parts that round 1 left unpinned (Missing #3).  CPU only.

(a) The printed form of Eqs. 12-13 (``update_form=1`` of
    ``ho_update_illumination`` / ``ho_update_reflectance``): an exact-rational (Fraction)
    evaluation of the printed fractions on random l <= 8 integer histograms -- every sum in
    exact arithmetic, K from Eq. 11 in exact arithmetic, index(i, j) from the exact
    nearest-bin rule -- plus a hand-derived l = 2 closed form.  A ``/N*K`` for ``/(N*K)``,
    a dropped prior term, a swapped hR/hL or a missed K = 0 skip fails these.
(b) The orientation of Eqs. 17-20 (reading R4: gamma applies to the
    illumination factor j): with hR a spike at bin 255 (b_i = 1) the enhanced histogram is
    hL pushed through j -> nearest(b_j^(1/gamma)), evaluated here with 50-digit decimals;
    with hL a spike at 255 it is hR unchanged.  The swapped orientation gives the other way
    round, so both fail under a swap.
(c) The stop rule of Algorithm 1 (reading R11): stop after the first t whose
    renormalised update moved BOTH histograms by at most epsilon*N^2 (squared Euclidean
    norm), else after T.  Recomputed here from the iterates (the fixed-T runs t = 1..T) with
    numpy norms, and the suite is required to contain cases where an "or" rule, a strict
    "<", an absolute (not N^2-relative) epsilon or an off-by-one count would disagree.
"""
from decimal import Decimal, getcontext
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth


# ------------------------------------------------------------------ (a) printed Eqs. 12-13
def _nearest(x: Fraction, l: int) -> int:
    """argmin_k |x - k/(l-1)|, smallest k on ties (R5), by exhaustive exact comparison."""
    best, bd = 0, abs(x)
    for k in range(1, l):
        d = abs(x - Fraction(k, l - 1))
        if d < bd:
            best, bd = k, d
    return best


def _exact_K(hR, hL, N, l):
    """Eq. 6 cells C_ij = hR_i hL_j / N, Eq. 8 class sums, Eq. 11 K_ij = C_ij / D_idx(i,j) (0 if D = 0)."""
    idx = [[_nearest(Fraction(i, l - 1) * Fraction(j, l - 1), l) for j in range(l)] for i in range(l)]
    C = [[hR[i] * hL[j] / N for j in range(l)] for i in range(l)]
    D = [Fraction(0)] * l
    for i in range(l):
        for j in range(l):
            D[idx[i][j]] += C[i][j]
    K = [[C[i][j] / D[idx[i][j]] if D[idx[i][j]] != 0 else Fraction(0) for j in range(l)] for i in range(l)]
    return idx, K


def _printed_R(hL, hS, hG, K, idx, N, beta, l):
    """Eq. 13 as printed: (sum_j hL_j hS_idx(i,j) / (N K_ij) + beta hG_i) / (sum_j hL_j^2 / N^2 + beta),
    terms with K_ij = 0 omitted (R8: the cell carries no mass)."""
    den = sum(hL[j] * hL[j] for j in range(l)) / (N * N) + beta
    out = []
    for i in range(l):
        num = sum((hL[j] * hS[idx[i][j]] / (N * K[i][j]) for j in range(l) if K[i][j] != 0), Fraction(0))
        out.append((num + beta * hG[i]) / den)
    return out


def _printed_L(hR, hS, K, idx, N, alpha, l):
    """Eq. 12 as printed: (sum_i hR_i hS_idx(i,j) / (N K_ij) + alpha hS_j) / (sum_i hR_i^2 / N^2 + alpha)."""
    den = sum(hR[i] * hR[i] for i in range(l)) / (N * N) + alpha
    out = []
    for j in range(l):
        num = sum((hR[i] * hS[idx[i][j]] / (N * K[i][j]) for i in range(l) if K[i][j] != 0), Fraction(0))
        out.append((num + alpha * hS[j]) / den)
    return out


def _int_hists(rng, l, p0):
    """Integer histograms of one image size N: masses are exact in fp64 and in Fraction."""
    while True:
        hS = rng.integers(0, 9, l) * (rng.random(l) < p0)
        hG = rng.integers(0, 9, l) * (rng.random(l) < p0)
        if hS.sum() > 0 and hG.sum() > 0:
            break
    # same total N (hR^0 = hG must carry the image's pixel count, Alg. 1)
    N = int(max(hS.sum(), hG.sum()))
    hS[int(np.argmax(hS))] += N - hS.sum()
    hG[int(np.argmax(hG))] += N - hG.sum()
    return hS.astype(np.int64), hG.astype(np.int64), N


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray([float(x) for x in b])
    nz = b != 0
    assert np.array_equal(a == 0, b == 0)
    return float(np.max(np.abs(a[nz] - b[nz]) / np.abs(b[nz]))) if nz.any() else 0.0


@pytest.mark.parametrize("seed", range(24))
def test_printed_form_one_update_exact_rationals(seed):
    """One Eq. 13 then Eq. 12 update (raw hR', frozen K, R10) in update_form=1 equals the exact
    rational evaluation of the printed fractions within fp64 rounding (1e-12 relative)."""
    rng = np.random.default_rng(9000 + seed)
    l = [2, 3, 4, 5, 6, 8][seed % 6]
    hS, hG, N = _int_hists(rng, l, p0=[0.5, 0.8, 1.0][seed % 3])
    alpha = [Fraction(1, 10), Fraction(1, 1000), Fraction(3, 2)][seed % 3]
    beta = [Fraction(1, 1000), Fraction(1, 10), Fraction(2)][(seed // 3) % 3]
    # iterate state: start from the Alg. 1 initialisation or from a random positive pair
    if seed % 2 == 0:
        hR = [Fraction(int(v)) for v in hG]
        hL = [Fraction(int(v)) for v in hS]
    else:
        r = rng.integers(1, 20, l) * (hG > 0)
        q = rng.integers(1, 20, l) * (hS > 0)
        hR = [Fraction(int(v) * N, int(r.sum())) for v in r]
        hL = [Fraction(int(v) * N, int(q.sum())) for v in q]
    hSf = [Fraction(int(v)) for v in hS]
    hGf = [Fraction(int(v)) for v in hG]
    Nf = Fraction(N)
    idx, K = _exact_K(hR, hL, Nf, l)
    R1 = _printed_R(hL, hSf, hGf, K, idx, Nf, beta, l)
    L1 = _printed_L(R1, hSf, K, idx, Nf, alpha, l)

    # the oracle, fed the same state (its own Eq. 11 K)
    hR64 = np.array([float(v) for v in hR])
    hL64 = np.array([float(v) for v in hL])
    oidx = oracle.index_map(l)
    assert np.array_equal(oidx, np.array(idx))
    C = oracle.pair_count(hR64, hL64, float(N))
    K64 = oracle.weights(C, oidx, oracle.estimate(C, oidx))
    oR = oracle.update_reflectance(hL64, hS.astype(float), hG.astype(float), K64, oidx, float(N), float(beta), form=1)
    oL = oracle.update_illumination(oR, hS.astype(float), K64, oidx, float(N), float(alpha), form=1)
    assert _rel(oR, R1) < 1e-12
    assert _rel(oL, L1) < 1e-12


def test_printed_form_l2_closed_form():
    """Hand-derived l = 2 case (b = {0, 1}; index(i,j) = i*j: only cell (1,1) maps to bin 1).
    With r_k = hR_k, q_k = hL_k:  D_1 = r1 q1 / N, D_0 = (N^2 - r1 q1)/N, K_11 = 1,
    K_10 = r1 q0 / (N^2 - r1 q1), K_00 = r0 q0 / (N^2 - r1 q1), K_01 = r0 q1 / (N^2 - r1 q1).
    Eq. 13 printed:
      hR'_1 = (q0 hS0 (N^2 - r1 q1)/(N r1 q0) + q1 hS1 / N + beta hG1) / ((q0^2+q1^2)/N^2 + beta)
            = (hS0 (N^2 - r1 q1)/(N r1) + q1 hS1 / N + beta hG1) / den_R
      hR'_0 = (hS0 (N^2 - r1 q1)/(N r0) * 2 + beta hG0) / den_R      (cells (0,0), (0,1) both -> bin 0)
    """
    N = 10
    hS = np.array([6.0, 4.0])
    hG = np.array([7.0, 3.0])
    r0, r1 = Fraction(7), Fraction(3)
    q0, q1 = Fraction(6), Fraction(4)
    beta = Fraction(1, 10)
    den = (q0 * q0 + q1 * q1) / (N * N) + beta
    m = N * N - r1 * q1
    want1 = (Fraction(6) * m / (N * r1) + q1 * 4 / N + beta * 3) / den
    want0 = (Fraction(6) * m / (N * r0) * 2 + beta * 7) / den
    idx = oracle.index_map(2)
    C = oracle.pair_count([7.0, 3.0], [6.0, 4.0], float(N))
    K = oracle.weights(C, idx, oracle.estimate(C, idx))
    got = oracle.update_reflectance([6.0, 4.0], hS, hG, K, idx, float(N), 0.1, form=1)
    assert got[1] == pytest.approx(float(want1), rel=1e-14)
    assert got[0] == pytest.approx(float(want0), rel=1e-14)
    # the gradient-consistent form differs here (K in the numerator), so the flag is live
    gc = oracle.update_reflectance([6.0, 4.0], hS, hG, K, idx, float(N), 0.1, form=0)
    assert abs(gc[0] - got[0]) > 1e-3 * abs(got[0])


def test_printed_form_decompose_two_iterations_exact():
    """Two full Algorithm 1 iterations of the printed form (Eq. 13, Eq. 12, Eq. 15, Eq. 14, Eq. 11
    in P:249-253 order) in exact rationals equal ho_decompose(update_form=1, T=2)."""
    rng = np.random.default_rng(77)
    for l in (3, 4, 6):
        hS, hG, N = _int_hists(rng, l, p0=0.8)
        alpha, beta = Fraction(1, 10), Fraction(1, 100)
        Nf = Fraction(N)
        hR = [Fraction(int(v)) for v in hG]
        hL = [Fraction(int(v)) for v in hS]
        hSf = [Fraction(int(v)) for v in hS]
        hGf = [Fraction(int(v)) for v in hG]
        for _ in range(2):
            idx, K = _exact_K(hR, hL, Nf, l)
            R1 = _printed_R(hL, hSf, hGf, K, idx, Nf, beta, l)
            L1 = _printed_L(R1, hSf, K, idx, Nf, alpha, l)
            sR, sL = sum(R1), sum(L1)
            hR = [Nf * v / sR for v in R1]
            hL = [Nf * v / sL for v in L1]
        oL, oR, it, _ = oracle.decompose(hS.astype(float), hG.astype(float),
                                         oracle.Params(levels=l, alpha=0.1, beta=0.01, max_iter=2, update_form=1))
        assert it == 2
        assert _rel(oR, hR) < 1e-11 and _rel(oL, hL) < 1e-11


# --------------------------------------------------------------- (b) Eq. 20 orientation
def _gamma_bin(j: int, gamma: float) -> int:
    """nearest(b_j^(1/gamma)) among k/255, smallest k on ties, 50 significant digits."""
    getcontext().prec = 50
    p = (Decimal(j) / Decimal(255)) ** (Decimal(1) / Decimal(repr(gamma))) if j else Decimal(0)
    y = p * 255
    k = int(y)  # floor (y >= 0)
    return k + 1 if (y - k) > Decimal("0.5") else k


@pytest.mark.parametrize("gamma", [1.5, 2.2, 5.0])
def test_eq20_orientation_reflectance_spike(gamma):
    """hR = N at bin 255 (b_i = 1): T_k = sum of hL_j over j with nearest(b_j^(1/gamma)) = k.
    Under the swapped orientation (gamma on the reflectance factor) T would equal hL."""
    rng = np.random.default_rng(int(gamma * 10))
    N = 5000.0
    hL = rng.random(256) * (rng.random(256) < 0.6)
    hL *= N / hL.sum()
    hR = np.zeros(256)
    hR[255] = N
    T = oracle.enhanced_histogram(hR, hL, oracle.index_map(256, gamma), N)
    want = np.zeros(256)
    for j in range(256):
        want[_gamma_bin(j, gamma)] += hL[j]
    assert np.allclose(T, want, rtol=1e-13, atol=1e-9)
    assert not np.allclose(T, hL, rtol=1e-6, atol=1e-6)  # the pin discriminates


@pytest.mark.parametrize("gamma", [1.5, 2.2, 5.0])
def test_eq20_orientation_illumination_spike(gamma):
    """hL = N at bin 255 (b_j^(1/gamma) = 1): T = hR unchanged (nearest(b_i) = i)."""
    rng = np.random.default_rng(100 + int(gamma * 10))
    N = 5000.0
    hR = rng.random(256) * (rng.random(256) < 0.6)
    hR *= N / hR.sum()
    hL = np.zeros(256)
    hL[255] = N
    T = oracle.enhanced_histogram(hR, hL, oracle.index_map(256, gamma), N)
    assert np.allclose(T, hR, rtol=1e-13, atol=1e-9)


def test_eq20_pipeline_passes_reflectance_first():
    """ho_enhance feeds its Algorithm 1 outputs to Eq. 20 as (hR, hL) -- the orientation the two
    pins above fix -- and not swapped: the swapped call gives a different target here."""
    img = synth.make_image(60, 80, seed=31, peak=0.2)
    p = oracle.Params(gamma=2.2)
    r = oracle.enhance(img, p)
    N = 60.0 * 80.0
    idx1 = oracle.index_map(256, 2.2)
    assert np.array_equal(r.T, oracle.enhanced_histogram(r.hR, r.hL, idx1, N))
    assert not np.allclose(r.T, oracle.enhanced_histogram(r.hL, r.hR, idx1, N), rtol=1e-6)


# ------------------------------------------------------------------- (c) stop rule
def _iterates(hS, hG, p, T):
    """(hR^(t), hL^(t)) for t = 0..T: t = 0 is the Alg. 1 initialisation, t >= 1 the fixed-T runs."""
    R = [hG.astype(float)]
    L = [hS.astype(float)]
    for t in range(1, T + 1):
        q = oracle.Params(alpha=p.alpha, beta=p.beta, gamma=p.gamma, max_iter=t, use_epsilon=0,
                          update_form=p.update_form)
        hL, hR, it, _ = oracle.decompose(hS, hG, q)
        assert it == t
        R.append(hR)
        L.append(hL)
    return R, L


def _case_hists():
    """Histograms of synthetic images of several darkness levels (the paper's workloads' shapes)."""
    out = []
    for k, (peak, s) in enumerate([(0.05, 3.0), (0.1, 2.0), (0.2, 2.0), (0.3, 2.0), (0.4, 1.0), (0.03, 2.0)]):
        img = synth.make_image(48, 64, seed=700 + k, peak=peak, sigma_n=s)
        r = oracle.enhance(img, oracle.Params(max_iter=1))
        out.append((r.hS.astype(float), r.hG.astype(float)))
    return out


def test_stop_rule_recomputed_from_iterates():
    T = 10
    eps_list = [1e-1, 3e-2, 1e-2, 3e-3, 1e-3, 3e-4, 1e-4, 1e-5]
    disagree = {"or": 0, "strict": 0, "absolute": 0}
    checked = 0
    for hS, hG in _case_hists():
        N = hS.sum()
        for form in (0, 1):
            p = oracle.Params(update_form=form)
            R, L = _iterates(hS, hG, p, T)
            dR = [float(np.sum((R[t] - R[t - 1]) ** 2)) for t in range(1, T + 1)]
            dL = [float(np.sum((L[t] - L[t - 1]) ** 2)) for t in range(1, T + 1)]

            def first(pred):
                for t in range(1, T + 1):
                    if pred(t):
                        return t
                return T

            for eps in eps_list:
                e = eps * N * N
                want = first(lambda t: dR[t - 1] <= e and dL[t - 1] <= e)
                q = oracle.Params(update_form=form, epsilon=eps, use_epsilon=1, max_iter=T)
                hL, hR, it, _ = oracle.decompose(hS, hG, q)
                assert it == want, (form, eps, dR, dL)
                # the returned pair is the accepted iterate t = want
                assert np.array_equal(hR, R[want]) and np.array_equal(hL, L[want])
                checked += 1
                disagree["or"] += first(lambda t: dR[t - 1] <= e or dL[t - 1] <= e) != want
                disagree["strict"] += first(lambda t: dR[t - 1] < e and dL[t - 1] < e) != want or any(
                    dR[t] == e or dL[t] == e for t in range(T))
                disagree["absolute"] += first(lambda t: dR[t - 1] <= eps and dL[t - 1] <= eps) != want
    assert checked == 6 * 2 * len(eps_list)
    # the cases discriminate: an "or" rule and an absolute epsilon would fail somewhere
    assert disagree["or"] > 0 and disagree["absolute"] > 0, disagree


def test_stop_rule_never_before_first_update_and_caps_at_T():
    """t counts completed updates: the rule is tested after each update (t >= 1), never on the
    initialisation, and T caps the count even when epsilon is never met."""
    hS, hG = _case_hists()[2]
    for T in (1, 2, 5):
        _, _, it, _ = oracle.decompose(hS, hG, oracle.Params(epsilon=1e-30, use_epsilon=1, max_iter=T))
        assert it == T
        _, _, it, _ = oracle.decompose(hS, hG, oracle.Params(epsilon=1e30, use_epsilon=1, max_iter=T))
        assert it == 1
