"""paper_2510_21100_b200 -- B200-native HistRetinex hot path (arXiv 2510.21100).

Thin Python binding over the C-ABI in include/histretinex.h.  Each function has the name
of the C entry point it calls and only marshals arguments: every step of the path runs in
the library's sm_100a kernels; there is no CPU fallback (a missing library or a non-CUDA
tensor raises).  PyTorch is used for device memory and the current CUDA stream.

    out = hr_enhance(x_u8_cuda[B, H, W, 3], Params(gamma=2.2))
    hist_s, hist_g, hist_g_raw = hr_histogram(x)
    hL, hR, target, iters = hr_solve(hist_s, hist_g, params)
    lut, status = hr_match(hist_s, target)
    out = hr_apply(x, lut)
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import HrError

__all__ = ["Params", "HrError", "hr_histogram", "hr_solve", "hr_match", "hr_apply", "hr_enhance",
           "hr_enhance_debug", "workspace_bytes", "version", "profile_enable", "profile_collect",
           "set_policy", "kernel_launches", "hr_enhance_host", "last_path", "hr_solve_trace", "hr_he",
           "hr_quality", "trace_bind"]


@dataclass
class Params:
    """Algorithm 1 + reprocessing parameters (hr_params; readings R7, R11-R14)."""

    levels: int = 256
    max_iter: int = 10
    alpha: float = 0.1
    beta: float = 1e-3
    gamma: float = 2.2
    epsilon: float = 1e-3  # relative to N^2
    use_epsilon: int = 0
    update_form: int = 0  # 0 gradient-consistent, 1 paper-literal
    grad_norm: int = 0  # 0 MAXNORM, 1 RAW_CLAMP

    def c(self) -> _lib.HrParams:
        return _lib.HrParams(self.levels, self.max_iter, self.alpha, self.beta, self.gamma,
                             self.epsilon, self.use_epsilon, self.update_form, self.grad_norm, 0)


_ctx: dict[int, ctypes.c_void_p] = {}


def _context(device: torch.device) -> ctypes.c_void_p:
    idx = device.index if device.index is not None else torch.cuda.current_device()
    c = _ctx.get(idx)
    if c is None:
        lib = _lib.load()
        c = ctypes.c_void_p()
        st = lib.hr_create(ctypes.byref(c), idx)
        if st != 0:
            raise HrError(st, f"hr_create(device={idx}) failed: {lib.hr_status_string(st).decode()}")
        _ctx[idx] = c
    return c


def _check(st: int, ctx) -> None:
    if st != 0:
        lib = _lib.load()
        raise HrError(st, f"{lib.hr_status_string(st).decode()}: {lib.hr_last_error(ctx).decode()}")


def _cuda(t: torch.Tensor, dtype: torch.dtype, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


def _buf(t: torch.Tensor, dtype: torch.dtype, shape, device: torch.device, name: str) -> torch.Tensor:
    """A caller-supplied buffer the C side will write or read: the C-ABI cannot check sizes, so
    dtype, device, contiguity and the exact shape are checked here."""
    _cuda(t, dtype, name)
    if t.device != device:
        raise ValueError(f"{name} is on {t.device}, expected {device}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    return t


def _ws_check(ws: torch.Tensor, nbytes: int, device: torch.device, name: str = "workspace") -> torch.Tensor:
    _cuda(ws, torch.uint8, name)
    if ws.device != device:
        raise ValueError(f"{name} is on {ws.device}, expected {device}")
    if ws.numel() < nbytes:
        raise ValueError(f"{name} has {ws.numel()} bytes, needs {nbytes}")
    return ws


def _hist_pair(hist_s: torch.Tensor, hist_g: torch.Tensor):
    _cuda(hist_s, torch.int32, "hist_s")
    if hist_s.dim() != 2 or hist_s.shape[1] != 256:
        raise ValueError("hist_s must be int32 [B, 256]")
    _buf(hist_g, torch.int32, hist_s.shape, hist_s.device, "hist_g")


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _stream(device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _images(x: torch.Tensor):
    _cuda(x, torch.uint8, "rgb")
    if x.dim() == 3:
        x = x.unsqueeze(0)
    if x.dim() != 4 or x.shape[-1] != 3:
        raise ValueError("rgb must be uint8 [B, H, W, 3] or [H, W, 3]")
    return x


def workspace_bytes(B: int, H: int, W: int) -> int:
    return int(_lib.load().hr_workspace_bytes(B, H, W))


def _workspace(B, H, W, device) -> torch.Tensor:
    return torch.empty(max(workspace_bytes(B, H, W), 256), dtype=torch.uint8, device=device)


def version() -> str:
    return _lib.load().hr_version().decode()


def hr_histogram(rgb: torch.Tensor, grad_norm: int = 0):
    """(1) value-channel and gradient histograms.  Returns (hist_s[B,256], hist_g[B,256],
    hist_g_raw[B,512]) as int32 tensors holding uint32 counts."""
    x = _images(rgb)
    B, H, W, _ = x.shape
    dev = x.device
    hs = torch.empty((B, 256), dtype=torch.int32, device=dev)
    hg = torch.empty((B, 256), dtype=torch.int32, device=dev)
    hgr = torch.empty((B, 512), dtype=torch.int32, device=dev)
    ws = _workspace(B, H, W, dev)
    ctx = _context(dev)
    _check(_lib.load().hr_histogram(ctx, _ptr(x), B, H, W, grad_norm, _ptr(hs), _ptr(hg), _ptr(hgr),
                                    _ptr(ws), _stream(dev)), ctx)
    return hs, hg, hgr


def hr_solve(hist_s: torch.Tensor, hist_g: torch.Tensor, params: Params | None = None):
    """(2) Algorithm 1 + Eqs. 17-20.  Returns (hL, hR, target) float64 [B,256] and iters int32 [B]."""
    p = params or Params()
    _hist_pair(hist_s, hist_g)
    B = hist_s.shape[0]
    dev = hist_s.device
    hL = torch.empty((B, 256), dtype=torch.float64, device=dev)
    hR = torch.empty_like(hL)
    tg = torch.empty_like(hL)
    it = torch.empty((B,), dtype=torch.int32, device=dev)
    pc = p.c()
    ws = _workspace(B, 1, 1, dev)
    ctx = _context(dev)
    _check(_lib.load().hr_solve(ctx, _ptr(hist_s), _ptr(hist_g), B, ctypes.byref(pc), _ptr(hL), _ptr(hR),
                                _ptr(tg), _ptr(it), _ptr(ws), _stream(dev)), ctx)
    return hL, hR, tg, it


def hr_solve_trace(hist_s: torch.Tensor, hist_g: torch.Tensor, params: Params | None = None):
    """hr_solve plus the Eq. 10 objective trace (3 values per update, K frozen).  Returns
    (hL, hR, target, iters, trace) with trace float64 [B, 3 * max_iter]."""
    p = params or Params()
    _hist_pair(hist_s, hist_g)
    B = hist_s.shape[0]
    dev = hist_s.device
    hL = torch.empty((B, 256), dtype=torch.float64, device=dev)
    hR = torch.empty_like(hL)
    tg = torch.empty_like(hL)
    it = torch.empty((B,), dtype=torch.int32, device=dev)
    stride = 3 * p.max_iter
    tr = torch.empty((B, stride), dtype=torch.float64, device=dev)
    pc = p.c()
    ws = _workspace(B, 1, 1, dev)
    ctx = _context(dev)
    _check(_lib.load().hr_solve_trace(ctx, _ptr(hist_s), _ptr(hist_g), B, ctypes.byref(pc), _ptr(hL), _ptr(hR),
                                      _ptr(tg), _ptr(it), _ptr(tr), stride, _ptr(ws), _stream(dev)), ctx)
    return hL, hR, tg, it, tr


def hr_match(hist_s: torch.Tensor, target: torch.Tensor):
    """(3) CDF + LUT.  Returns (lut uint8 [B,256], status int32 [B])."""
    _cuda(hist_s, torch.int32, "hist_s")
    if hist_s.dim() != 2 or hist_s.shape[1] != 256:
        raise ValueError("hist_s must be int32 [B, 256]")
    B = hist_s.shape[0]
    dev = hist_s.device
    _buf(target, torch.float64, (B, 256), dev, "target")
    lut = torch.empty((B, 256), dtype=torch.uint8, device=dev)
    stt = torch.empty((B,), dtype=torch.int32, device=dev)
    ctx = _context(dev)
    _check(_lib.load().hr_match(ctx, _ptr(hist_s), _ptr(target), B, _ptr(lut), _ptr(stt), _stream(dev)), ctx)
    return lut, stt


def hr_apply(rgb: torch.Tensor, lut: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """(4) per-pixel LUT + colour reconstruction."""
    x = _images(rgb)
    B, H, W, _ = x.shape
    _buf(lut, torch.uint8, (B, 256), x.device, "lut")
    out = torch.empty_like(x) if out is None else _buf(out, torch.uint8, x.shape, x.device, "out")
    ctx = _context(x.device)
    _check(_lib.load().hr_apply(ctx, _ptr(x), _ptr(lut), B, H, W, _ptr(out), _stream(x.device)), ctx)
    return out


def hr_enhance(rgb: torch.Tensor, params: Params | None = None, out: torch.Tensor | None = None,
               workspace: torch.Tensor | None = None) -> torch.Tensor:
    """(1)-(4) for the whole batch."""
    p = params or Params()
    x = _images(rgb)
    B, H, W, _ = x.shape
    out = torch.empty_like(x) if out is None else _buf(out, torch.uint8, x.shape, x.device, "out")
    if x.numel() and out.data_ptr() == x.data_ptr():
        raise ValueError("out must not alias rgb")
    ws = (_ws_check(workspace, workspace_bytes(B, H, W), x.device) if workspace is not None
          else _workspace(B, H, W, x.device))
    pc = p.c()
    ctx = _context(x.device)
    _check(_lib.load().hr_enhance(ctx, _ptr(x), B, H, W, ctypes.byref(pc), _ptr(out), _ptr(ws),
                                  _stream(x.device)), ctx)
    return out


def trace_bind(records: torch.Tensor | None, count: torch.Tensor | None, capacity: int, device=None) -> None:
    """hr_trace_bind (measurement): bind a device record buffer (48-byte records) and a uint32
    counter for the step timeline of later launches on `device`; records=None unbinds."""
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    ctx = _context(dev)
    if records is not None:
        _cuda(records, torch.uint8, "records")
        _cuda(count, torch.int32, "count")
        if records.numel() < 48 * capacity:
            raise ValueError("records holds fewer than capacity records")
    _check(_lib.load().hr_trace_bind(ctx, _ptr(records), _ptr(count), int(capacity)), ctx)


def profile_enable(device=None, on: bool = True) -> None:
    """Record per-stage CUDA events inside every hr_enhance on `device` (measurement only)."""
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    ctx = _context(dev)
    _check(_lib.load().hr_profile_enable(ctx, 1 if on else 0), ctx)


def profile_collect(device=None):
    """Summed (hist_ms, solve_ms, apply_ms) and the number of hr_enhance calls since the last
    collect (waits for the recorded events)."""
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    ctx = _context(dev)
    ms = (ctypes.c_double * 3)()
    n = ctypes.c_int32(0)
    _check(_lib.load().hr_profile_collect(ctx, ms, ctypes.byref(n)), ctx)
    return (ms[0], ms[1], ms[2]), n.value


def set_policy(key: str, value: int, device=None) -> None:
    """hr_set_policy: execution policy of hr_enhance on `device` (performance only; see
    include/histretinex.h for the keys)."""
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    ctx = _context(dev)
    _check(_lib.load().hr_set_policy(ctx, key.encode(), int(value)), ctx)


def get_policy(key: str, device=None) -> int:
    """hr_get_policy: current value of an hr_enhance policy key on `device`."""
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    ctx = _context(dev)
    v = ctypes.c_int64(0)
    _check(_lib.load().hr_get_policy(ctx, key.encode(), ctypes.byref(v)), ctx)
    return int(v.value)


def hr_enhance_host(rgb_host: torch.Tensor, params: Params | None = None, out_host: torch.Tensor | None = None,
                    device=None, chunks: int = 0, in_dev: torch.Tensor | None = None,
                    out_dev: torch.Tensor | None = None, workspace: torch.Tensor | None = None,
                    sync: bool = True) -> torch.Tensor:
    """hr_enhance_host: host [B, H, W, 3] uint8 in -> host out, copies pipelined with the
    enhancement over image chunks.  Pinned (page-locked) host tensors make the copies
    asynchronous.  Staging device buffers and the workspace are allocated when not given."""
    if rgb_host.device.type != "cpu" or rgb_host.dtype != torch.uint8 or rgb_host.dim() != 4 or rgb_host.shape[-1] != 3:
        raise ValueError("rgb_host must be a CPU uint8 tensor [B, H, W, 3]")
    x = rgb_host.contiguous()
    B, H, W, _ = x.shape
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    if out_host is None:
        out_host = torch.empty_like(x, pin_memory=x.is_pinned())
    elif (out_host.device.type != "cpu" or out_host.dtype != torch.uint8 or tuple(out_host.shape) != tuple(x.shape)
          or not out_host.is_contiguous()):
        raise ValueError(f"out_host must be a contiguous CPU uint8 tensor of shape {tuple(x.shape)}")
    in_dev = (torch.empty(x.shape, dtype=torch.uint8, device=dev) if in_dev is None
              else _buf(in_dev, torch.uint8, x.shape, dev, "in_dev"))
    out_dev = (torch.empty(x.shape, dtype=torch.uint8, device=dev) if out_dev is None
               else _buf(out_dev, torch.uint8, x.shape, dev, "out_dev"))
    ws = _workspace(B, H, W, dev) if workspace is None else _ws_check(workspace, workspace_bytes(B, H, W), dev)
    pc = (params or Params()).c()
    ctx = _context(dev)
    _check(_lib.load().hr_enhance_host(ctx, _ptr(x), B, H, W, ctypes.byref(pc), _ptr(out_host), _ptr(in_dev),
                                       _ptr(out_dev), _ptr(ws), int(chunks), _stream(dev)), ctx)
    if sync:
        torch.cuda.current_stream(dev).synchronize()
    return out_host


def last_path(device=None) -> int:
    """hr_last_path: 0 separate kernels, 3 grouped step (last hr_enhance)."""
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    return int(_lib.load().hr_last_path(_context(dev)))


def hr_he(rgb: torch.Tensor, out: torch.Tensor | None = None, return_lut: bool = False):
    """HE baseline (Eq. 5) of a [B, H, W, 3] uint8 CUDA batch."""
    x = _images(rgb)
    B, H, W, _ = x.shape
    dev = x.device
    out = torch.empty_like(x) if out is None else _buf(out, torch.uint8, x.shape, dev, "out")
    lut = torch.empty((B, 256), dtype=torch.uint8, device=dev)
    ws = _workspace(B, H, W, dev)
    ctx = _context(dev)
    _check(_lib.load().hr_he(ctx, _ptr(x), B, H, W, _ptr(out), _ptr(lut), _ptr(ws), _stream(dev)), ctx)
    return (out, lut) if return_lut else out


def hr_quality(a: torch.Tensor, b: torch.Tensor):
    """(psnr, ssim, loe) float64 [B] of image pairs (SPEC metrics; a = original for LOE)."""
    x, y = _images(a), _images(b)
    if x.shape != y.shape:
        raise ValueError("a and b must have the same shape")
    B, H, W, _ = x.shape
    dev = x.device
    ps = torch.empty((B,), dtype=torch.float64, device=dev)
    ss, lo = torch.empty_like(ps), torch.empty_like(ps)
    lib = _lib.load()
    ws = torch.empty(max(1, lib.hr_quality_workspace_bytes(B, H, W)), dtype=torch.uint8, device=dev)
    ctx = _context(dev)
    _check(lib.hr_quality(ctx, _ptr(x), _ptr(y), B, H, W, _ptr(ps), _ptr(ss), _ptr(lo), _ptr(ws), _stream(dev)), ctx)
    return ps, ss, lo


def kernel_launches(device=None) -> int:
    """hr_kernel_launches: kernels launched so far through the context of `device`."""
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    return int(_lib.load().hr_kernel_launches(_context(dev)))


def hr_enhance_debug(rgb: torch.Tensor, params: Params | None = None, full: bool = False):
    """hr_enhance also returning intermediate results of the same schedule: (out, hist_s, lut,
    iters), or with full=True a dict with out, hist_s, hist_g, lut, iters, hL, hR, target."""
    p = params or Params()
    x = _images(rgb)
    B, H, W, _ = x.shape
    dev = x.device
    out = torch.empty_like(x)
    r = {"out": out,
         "hist_s": torch.empty((B, 256), dtype=torch.int32, device=dev),
         "lut": torch.empty((B, 256), dtype=torch.uint8, device=dev),
         "iters": torch.empty((B,), dtype=torch.int32, device=dev)}
    if full:
        r["hist_g"] = torch.empty((B, 256), dtype=torch.int32, device=dev)
        for k in ("hL", "hR", "target"):
            r[k] = torch.empty((B, 256), dtype=torch.float64, device=dev)
    dbg = _lib.HrDebugOut(*[r[k].data_ptr() if k in r else None
                            for k in ("hist_s", "hist_g", "lut", "iters", "hL", "hR", "target")])
    ws = _workspace(B, H, W, dev)
    pc = p.c()
    ctx = _context(dev)
    _check(_lib.load().hr_enhance_debug(ctx, _ptr(x), B, H, W, ctypes.byref(pc), _ptr(out), _ptr(ws),
                                        ctypes.byref(dbg), _stream(dev)), ctx)
    return r if full else (out, r["hist_s"], r["lut"], r["iters"])
