"""CPU oracle for the HistRetinex hot path (numpy/ctypes front end of hr_oracle.c).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product package ``paper_2510_21100_b200`` never imports it and
shares no code with it (no kernels, headers, helpers, tables or constants).

Every function mirrors one C entry point of ``hr_oracle.c`` that follows
/root/reference/PAPER.md literally (see ``hr_oracle.h`` for the per-function
citation).  Pins: tests/test_oracle_*.py.  Parity unpinned by the paper: the
whole-pipeline output (the paper prints no worked example; Figs. 2-3 are
images) -- pinned only by the invariants listed in DESIGN.md section 3.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hr_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-pthread"]


def build(force: bool = False) -> str:
    """Compile hr_oracle.c into liboracle.so (gcc, no CUDA)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "hr_oracle.h"))
    ):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Params(ctypes.Structure):
    _fields_ = [
        ("levels", ctypes.c_int32),
        ("alpha", ctypes.c_double),
        ("beta", ctypes.c_double),
        ("gamma", ctypes.c_double),
        ("epsilon", ctypes.c_double),
        ("max_iter", ctypes.c_int32),
        ("use_epsilon", ctypes.c_int32),
        ("update_form", ctypes.c_int32),
        ("grad_norm", ctypes.c_int32),
    ]


@dataclass
class Params:
    """Algorithm 1 + reprocessing parameters (readings R7, R11-R14)."""

    levels: int = 256
    alpha: float = 0.1
    beta: float = 1e-3
    gamma: float = 2.2
    epsilon: float = 1e-3  # relative: ||dh||^2 <= epsilon * N^2
    max_iter: int = 10
    use_epsilon: int = 0
    update_form: int = 0  # 0 gradient-consistent, 1 paper-literal
    grad_norm: int = 0  # 0 MAXNORM, 1 RAW_CLAMP

    def c(self) -> _Params:
        return _Params(self.levels, self.alpha, self.beta, self.gamma, self.epsilon,
                       self.max_iter, self.use_epsilon, self.update_form, self.grad_norm)


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.ho_objective.restype = ctypes.c_double
        for f in ("ho_psnr", "ho_ssim", "ho_loe"):
            getattr(_lib, f).restype = ctypes.c_double
        _lib.ho_psnr.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
        _lib.ho_ssim.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32]
        _lib.ho_loe.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32]
    return _lib


class OracleError(RuntimeError):
    pass


def _ck(rc: int, what: str) -> None:
    if rc != 0:
        raise OracleError(f"{what} failed with code {rc}")


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


def _u8(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint8)


# ---------------------------------------------------------------- pixels
def value_channel(rgb: np.ndarray, levels: int = 256) -> np.ndarray:
    rgb = _u8(rgb)
    n = rgb.size // 3
    S = np.empty(rgb.shape[:-1], np.int32)
    _ck(lib().ho_value_channel(_p(rgb), ctypes.c_int64(n), levels, _p(S)), "value_channel")
    return S


def gradient_raw(S: np.ndarray) -> np.ndarray:
    S = _i32(S)
    H, W = S.shape
    g = np.empty_like(S)
    _ck(lib().ho_gradient_raw(_p(S), H, W, _p(g)), "gradient_raw")
    return g


def gradient_levels(g: np.ndarray, levels: int = 256, grad_norm: int = 0) -> np.ndarray:
    g = _i32(g)
    out = np.empty_like(g)
    _ck(lib().ho_gradient_levels(_p(g), ctypes.c_int64(g.size), levels, grad_norm, _p(out)),
        "gradient_levels")
    return out


def count_histogram(x: np.ndarray, nbins: int) -> np.ndarray:
    x = _i32(x)
    h = np.zeros(nbins, np.uint64)
    _ck(lib().ho_count_histogram(_p(x), ctypes.c_int64(x.size), nbins, _p(h)), "count_histogram")
    return h


# ------------------------------------------------------ histogram domain
def locations(levels: int) -> np.ndarray:
    b = np.empty(levels, np.float64)
    _ck(lib().ho_locations(levels, _p(b)), "locations")
    return b


def index_map(levels: int, gamma: float = 1.0) -> np.ndarray:
    idx = np.empty((levels, levels), np.int32)
    _ck(lib().ho_index_map(levels, ctypes.c_double(gamma), _p(idx)), "index_map")
    return idx


def pair_count(hR, hL, N: float) -> np.ndarray:
    hR, hL = _f64(hR), _f64(hL)
    l = hR.size
    C = np.empty((l, l), np.float64)
    _ck(lib().ho_pair_count(_p(hR), _p(hL), l, ctypes.c_double(N), _p(C)), "pair_count")
    return C


def estimate(C, idx) -> np.ndarray:
    C, idx = _f64(C), _i32(idx)
    l = C.shape[0]
    est = np.empty(l, np.float64)
    _ck(lib().ho_estimate(_p(C), _p(idx), l, _p(est)), "estimate")
    return est


def weights(C, idx, est) -> np.ndarray:
    C, idx, est = _f64(C), _i32(idx), _f64(est)
    l = C.shape[0]
    K = np.empty_like(C)
    _ck(lib().ho_weights(_p(C), _p(idx), _p(est), l, _p(K)), "weights")
    return K


def objective(hR, hL, hS, hG, K, idx, N, alpha, beta) -> float:
    hR, hL, hS, hG, K, idx = map(lambda a: a, (_f64(hR), _f64(hL), _f64(hS), _f64(hG), _f64(K), _i32(idx)))
    return lib().ho_objective(_p(hR), _p(hL), _p(hS), _p(hG), _p(K), _p(idx), hR.size,
                              ctypes.c_double(N), ctypes.c_double(alpha), ctypes.c_double(beta))


def update_reflectance(hL, hS, hG, K, idx, N, beta, form=0) -> np.ndarray:
    hL, hS, hG, K, idx = _f64(hL), _f64(hS), _f64(hG), _f64(K), _i32(idx)
    out = np.empty_like(hL)
    _ck(lib().ho_update_reflectance(_p(hL), _p(hS), _p(hG), _p(K), _p(idx), hL.size,
                                    ctypes.c_double(N), ctypes.c_double(beta), form, _p(out)),
        "update_reflectance")
    return out


def update_illumination(hR, hS, K, idx, N, alpha, form=0) -> np.ndarray:
    hR, hS, K, idx = _f64(hR), _f64(hS), _f64(K), _i32(idx)
    out = np.empty_like(hR)
    _ck(lib().ho_update_illumination(_p(hR), _p(hS), _p(K), _p(idx), hR.size,
                                     ctypes.c_double(N), ctypes.c_double(alpha), form, _p(out)),
        "update_illumination")
    return out


def renormalize(h, N: float) -> np.ndarray:
    h = _f64(h)
    out = np.empty_like(h)
    _ck(lib().ho_renormalize(_p(h), h.size, ctypes.c_double(N), _p(out)), "renormalize")
    return out


def decompose(hS, hG, params: Params, trace_cap: int = 0):
    """Algorithm 1.  Returns (hL, hR, iters, trace)."""
    hS, hG = _f64(hS), _f64(hG)
    hL = np.empty_like(hS)
    hR = np.empty_like(hS)
    it = ctypes.c_int32(0)
    trace = np.zeros(max(trace_cap, 1), np.float64)
    pc = params.c()
    _ck(lib().ho_decompose(_p(hS), _p(hG), ctypes.byref(pc), _p(hL), _p(hR), ctypes.byref(it),
                           _p(trace) if trace_cap else None, trace_cap), "decompose")
    return hL, hR, it.value, trace[: min(trace_cap, 3 * it.value)]


def enhanced_histogram(hR, hL, idx1, N) -> np.ndarray:
    hR, hL, idx1 = _f64(hR), _f64(hL), _i32(idx1)
    T = np.empty_like(hR)
    _ck(lib().ho_enhanced_histogram(_p(hR), _p(hL), _p(idx1), hR.size, ctypes.c_double(N), _p(T)),
        "enhanced_histogram")
    return T


def match_lut(hS, T, with_margin: bool = False):
    hS = np.ascontiguousarray(hS, dtype=np.uint64)
    T = _f64(T)
    lut = np.empty(hS.size, np.int32)
    margin = np.empty(hS.size, np.float64)
    _ck(lib().ho_match_lut(_p(hS), _p(T), hS.size, _p(lut), _p(margin) if with_margin else None),
        "match_lut")
    return (lut, margin) if with_margin else lut


def he_transform(hS) -> np.ndarray:
    hS = np.ascontiguousarray(hS, dtype=np.uint64)
    t = np.empty(hS.size, np.int32)
    _ck(lib().ho_he_transform(_p(hS), hS.size, _p(t)), "he_transform")
    return t


def reconstruct(rgb, Vnew) -> np.ndarray:
    rgb = _u8(rgb)
    Vnew = _i32(Vnew)
    out = np.empty_like(rgb)
    _ck(lib().ho_reconstruct(_p(rgb), ctypes.c_int64(rgb.size // 3), _p(Vnew), _p(out)), "reconstruct")
    return out


# ------------------------------------------- second workload (NEXT #4): HE and metrics
def he_enhance(rgb) -> np.ndarray:
    """HE baseline (Eq. 5): V -> round(255 CDF(V)), colour by R17.  rgb [H, W, 3] uint8."""
    rgb = _u8(rgb)
    out = np.empty_like(rgb)
    _ck(lib().ho_he_enhance(_p(rgb), rgb.shape[0], rgb.shape[1], _p(out)), "he_enhance")
    return out


def psnr(a, b) -> float:
    a, b = _u8(a), _u8(b)
    assert a.shape == b.shape
    return float(lib().ho_psnr(_p(a), _p(b), a.size // 3))


def ssim(a, b) -> float:
    a, b = _u8(a), _u8(b)
    assert a.shape == b.shape
    return float(lib().ho_ssim(_p(a), _p(b), a.shape[0], a.shape[1]))


def loe(orig, enh) -> float:
    a, b = _u8(orig), _u8(enh)
    assert a.shape == b.shape
    return float(lib().ho_loe(_p(a), _p(b), a.shape[0], a.shape[1]))


# ---------------------------------------------------------------- pipeline
@dataclass
class EnhanceResult:
    out: np.ndarray
    hS: np.ndarray
    hG: np.ndarray
    hgraw: np.ndarray
    hL: np.ndarray
    hR: np.ndarray
    T: np.ndarray
    lut: np.ndarray
    iters: int
    margin: np.ndarray


def enhance(rgb: np.ndarray, params: Params | None = None) -> EnhanceResult:
    """Whole pipeline on one [H, W, 3] uint8 image."""
    params = params or Params()
    rgb = _u8(rgb)
    H, W = rgb.shape[:2]
    out = np.empty_like(rgb)
    hS = np.zeros(256, np.uint64)
    hG = np.zeros(256, np.uint64)
    hgraw = np.zeros(511, np.uint64)
    hL, hR, T, margin = (np.zeros(256) for _ in range(4))
    lut = np.zeros(256, np.int32)
    it = ctypes.c_int32(0)
    pc = params.c()
    _ck(lib().ho_enhance(_p(rgb), H, W, ctypes.byref(pc), _p(out), _p(hS), _p(hG), _p(hgraw),
                         _p(hL), _p(hR), _p(T), _p(lut), ctypes.byref(it), _p(margin)), "enhance")
    return EnhanceResult(out, hS, hG, hgraw, hL, hR, T, lut, it.value, margin)


def enhance_batch(rgb: np.ndarray, params: Params | None = None, nthreads: int = 1,
                  want_out: bool = True):
    """Whole pipeline on a [B, H, W, 3] uint8 batch.  Returns dict of per-image arrays."""
    params = params or Params()
    rgb = _u8(rgb)
    B, H, W = rgb.shape[:3]
    r = {
        "out": np.empty_like(rgb) if want_out else None,
        "hS": np.zeros((B, 256), np.uint64),
        "hG": np.zeros((B, 256), np.uint64),
        "hL": np.zeros((B, 256)),
        "hR": np.zeros((B, 256)),
        "T": np.zeros((B, 256)),
        "lut": np.zeros((B, 256), np.int32),
        "iters": np.zeros(B, np.int32),
    }
    pc = params.c()
    _ck(lib().ho_enhance_batch(_p(rgb), ctypes.c_int64(B), H, W, ctypes.byref(pc),
                               _p(r["out"]) if want_out else None, _p(r["hS"]), _p(r["hG"]),
                               _p(r["hL"]), _p(r["hR"]), _p(r["T"]), _p(r["lut"]), _p(r["iters"]),
                               nthreads), "enhance_batch")
    return r
