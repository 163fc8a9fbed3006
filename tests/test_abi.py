"""CPU-only checks of the C-ABI library and host-side logic (no compute calls; no GPU).

* the in-tree libhistretinex.so loads and exports every symbol include/histretinex.h declares;
* calls that need no device behave (defaults, status strings, workspace sizing, NULL ctx);
* the integer constants the kernels rely on are exact over their whole domain:
  index(i,j) = ((i*j + 127) * 32897) >> 23 == (i*j + 127) div 255, and the umulhi division
  magic floor(n / 2V) == umulhi(n, floor(2^32 / 2V) + 1) for every V and n <= 2*255*255+255.
"""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2510_21100_b200 import _build, _lib

    _build.build()
    return _lib.load()


def test_header_symbols_exported(lib):
    from paper_2510_21100_b200 import _lib

    hdr = open(os.path.join(ROOT, "include", "histretinex.h")).read()
    declared = set(re.findall(r"\b(hr_[a-z_]+)\s*\(", hdr))
    declared -= {"hr_ctx"}
    assert declared, "no declarations found"
    assert declared == set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name


def test_nm_dynamic_symbols(lib):
    import subprocess

    from paper_2510_21100_b200 import _lib

    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for name in _lib.EXPORTS:
        assert re.search(rf"\bT {name}\b", out), name


def test_defaults_and_strings(lib):
    from paper_2510_21100_b200 import _lib

    p = _lib.HrParams()
    assert lib.hr_default_params(ctypes.byref(p)) == 0
    assert (p.levels, p.max_iter, p.alpha, p.beta, p.gamma, p.use_epsilon, p.update_form, p.grad_norm) == (
        256, 10, 0.1, 1e-3, 2.2, 0, 0, 0)
    assert lib.hr_default_params(None) == _lib.HR_EINVAL
    assert lib.hr_status_string(0) == b"ok"
    assert lib.hr_status_string(_lib.HR_EEMPTY) == b"empty input"
    assert b"sm_100a" in lib.hr_version()
    assert lib.hr_last_error(None) == b""


def test_workspace_sizing(lib):
    assert lib.hr_workspace_bytes(0, 10, 10) == 0
    a = lib.hr_workspace_bytes(1, 100, 100)
    b = lib.hr_workspace_bytes(64, 1080, 1920)
    assert 0 < a < b and b >= 64 * (256 * 4 + 512 * 4 + 256)


def test_null_ctx_is_einval(lib):
    from paper_2510_21100_b200 import _lib

    p = _lib.HrParams()
    lib.hr_default_params(ctypes.byref(p))
    assert lib.hr_enhance(None, None, 1, 1, 1, ctypes.byref(p), None, None, None) == _lib.HR_EINVAL
    assert lib.hr_histogram(None, None, 1, 1, 1, 0, None, None, None, None, None) == _lib.HR_EINVAL
    assert lib.hr_set_policy(None, b"groups", 2) == _lib.HR_EINVAL
    assert lib.hr_destroy(None) == 0


def test_index_magic_exhaustive():
    x = np.arange(0, 255 * 255 + 1, dtype=np.uint64)
    assert np.array_equal(((x + 127) * 32897) >> 23, (x + 127) // 255)


def test_umulhi_magic_exhaustive():
    n = np.arange(0, 2 * 255 * 255 + 255 + 1, dtype=np.uint64)
    for V in range(1, 256):
        M = np.uint64((1 << 32) // (2 * V) + 1)
        assert np.array_equal((n * M) >> np.uint64(32), n // np.uint64(2 * V)), V


def test_apply_entry_formula_exhaustive():
    """k_apply's per-channel formula, emulated in uint64: out = umulhi(c*e + V, M[V]) + (e >> 16)
    with e = 2 LUT[V] (V >= 1) or LUT[0] << 16 (V = 0), M[V] = floor(2^32/2V) + 1 (M[0] = 0),
    against floor((2 c V' + V) / 2V) (V = 0 -> V') for every V, every c <= V and every V'."""
    L = np.arange(256, dtype=np.uint64)
    for V in range(0, 256):
        c = np.arange(0, V + 1, dtype=np.uint64)[:, None]
        if V == 0:
            e = L << np.uint64(16)
            M = np.uint64(0)
        else:
            e = np.uint64(2) * L
            M = np.uint64((1 << 32) // (2 * V) + 1)
        n = (c * e[None, :] + np.uint64(V)) & np.uint64(0xFFFFFFFF)
        out = ((n * M) >> np.uint64(32)) + (e[None, :] >> np.uint64(16))
        ref = np.broadcast_to(L[None, :], out.shape) if V == 0 else (2 * c * L[None, :] + V) // (2 * V)
        assert np.array_equal(out, ref), V


def test_maxnorm_integer_formula_vs_rational():
    from fractions import Fraction

    for gmax in range(1, 511):
        for g in range(0, gmax + 1, max(1, gmax // 37)):
            q = Fraction(255 * g, gmax) + Fraction(1, 2)
            assert (510 * g + gmax) // (2 * gmax) == q.numerator // q.denominator


def test_python_binding_fails_loudly_without_cuda():
    import torch

    import paper_2510_21100_b200 as hr

    x = torch.zeros((1, 4, 4, 3), dtype=torch.uint8)  # CPU tensor
    with pytest.raises(ValueError, match="CUDA"):
        hr.hr_enhance(x)


