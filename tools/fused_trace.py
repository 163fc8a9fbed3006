"""Timeline of one k_fused launch (measurement build tools/libhistretinex_trace.so, -DHR_FUSED_TRACE).

Prints, per config: kernel span, end of the histogram phase, per-image completion -> solve
start/end, solve durations, apply-phase spans per warp, ready-wait totals.  Not product code.
"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2510_21100_b200 import _lib  # noqa: E402

lib = ctypes.CDLL("tools/libhistretinex_trace.so")
vp = ctypes.c_void_p
lib.hr_create.argtypes = [ctypes.POINTER(vp), ctypes.c_int]
lib.hr_workspace_bytes.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32]
lib.hr_workspace_bytes.restype = ctypes.c_size_t
lib.hr_enhance.argtypes = [vp, vp, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(_lib.HrParams),
                           vp, vp, vp]
lib.hr_set_policy.argtypes = [vp, ctypes.c_char_p, ctypes.c_int64]
lib.hr_debug_fused_trace.argtypes = [vp, ctypes.c_int]
ctx = vp()
assert lib.hr_create(ctypes.byref(ctx), 0) == 0
P = _lib.HrParams()
lib.hr_default_params(ctypes.byref(P))
REC = np.dtype([("kind", "<u4"), ("cta", "<u4"), ("b", "<u4"), ("aux", "<u4"), ("t0", "<u8"), ("t1", "<u8")])
CAP = 1 << 17
buf = np.zeros(CAP, dtype=REC)


def pct(a, qs=(0, 50, 90, 100)):
    return " ".join(f"p{q}={np.percentile(a, q):.1f}" for q in qs) if len(a) else "-"


def run(cfg, policy):
    x = torch.from_numpy(synth.make_config(cfg)).cuda()
    B, H, W, _ = x.shape
    out = torch.empty_like(x)
    ws = torch.empty(lib.hr_workspace_bytes(B, H, W), dtype=torch.uint8, device="cuda")
    for k, v in policy.items():
        assert lib.hr_set_policy(ctx, k.encode(), v) == 0
    for _ in range(3):
        assert lib.hr_enhance(ctx, vp(x.data_ptr()), B, H, W, ctypes.byref(P), vp(out.data_ptr()), vp(ws.data_ptr()), None) == 0
    torch.cuda.synchronize()
    lib.hr_debug_fused_trace(vp(buf.ctypes.data), CAP)
    assert lib.hr_enhance(ctx, vp(x.data_ptr()), B, H, W, ctypes.byref(P), vp(out.data_ptr()), vp(ws.data_ptr()), None) == 0
    torch.cuda.synchronize()
    n = lib.hr_debug_fused_trace(vp(buf.ctypes.data), CAP)
    r = buf[:n].copy()
    t00 = r["t0"].min()
    us = lambda t: (t.astype(np.int64) - int(t00)) / 1e3  # noqa: E731
    k = r["kind"]
    start, hist, solve, app, wait = r[k == 4], r[k == 0], r[k == 1], r[k == 2], r[k == 3]
    print(f"== {cfg} B={B} {H}x{W} policy={policy}  records={n}")
    print(f"  CTA starts: {pct(us(start['t0']))} us")
    print(f"  kernel span: {us(np.array([r['t1'].max()]))[0]:.1f} us")
    hd = us(hist["t1"])
    print(f"  hist bands: n={len(hist)} dur {pct((hist['t1'] - hist['t0']) / 1e3)} us; phase end {hd.max():.1f} us")
    img_done = np.array([hd[hist["b"] == b].max() for b in range(B)])
    print(f"  image hist complete: first {img_done.min():.1f} last {img_done.max():.1f} us")
    sd = (solve["t1"] - solve["t0"]) / 1e3
    print(f"  solves: n={len(solve)} dur {pct(sd)} us; start {pct(us(solve['t0']))}; end {pct(us(solve['t1']))}")
    print(f"  CTA-us in solves: {sd.sum():.0f} (= {sd.sum() / max(len(start), 1):.1f} us per CTA)")
    a0, a1 = us(app["t0"]), us(app["t1"])
    print(f"  apply warps: n={len(app)} start {pct(a0)} end {pct(a1)}")
    wd = (wait["t1"] - wait["t0"]) / 1e3
    print(f"  ready waits: n={len(wait)} total {wd.sum():.0f} warp-us, dur {pct(wd)}; images {np.unique(wait['b'])[:12]}")


for cfg in sys.argv[1:] or ["C3", "C5"]:
    run(cfg, {"fused_min_b": 2, "fused_max_b": 1 << 20, "fused_bands": 2, "fused_gs": 8, "fused_cpsm": 2})
