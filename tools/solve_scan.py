"""Per-image solver latency over whole batches (measurement build tools/libhistretinex_prof.so).

Each image is solved alone (one CTA) with the phase clocks on; prints the latency
distribution and the slowest images with their support sizes and phase split.  The batch's
solve stage is gated by its slowest image.  Not product code."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2510_21100_b200 import _lib  # noqa: E402

lib = ctypes.CDLL(os.environ.get("HR_PROF_LIB", "tools/libhistretinex_prof.so"))
vp = ctypes.c_void_p
ctx = vp()
assert lib.hr_create(ctypes.byref(ctx), 0) == 0
P = _lib.HrParams()
lib.hr_default_params(ctypes.byref(P))
GHZ = 1.965

for cfg, nimg in (("C3", 64), ("C5", 64), ("C2", 1), ("C4", 1)):
    x = torch.from_numpy(synth.make_config(cfg, batch=nimg)).cuda()
    B, H, W, _ = x.shape
    ws = torch.empty(lib.hr_workspace_bytes(ctypes.c_int64(B), H, W) if False else 1 << 26, dtype=torch.uint8,
                     device="cuda")
    hs = torch.empty((B, 256), dtype=torch.int32, device="cuda")
    hg = torch.empty_like(hs)
    hgr = torch.empty((B, 512), dtype=torch.int32, device="cuda")
    lib.hr_histogram(ctx, vp(x.data_ptr()), ctypes.c_int64(B), H, W, 0, vp(hs.data_ptr()), vp(hg.data_ptr()),
                     vp(hgr.data_ptr()), vp(ws.data_ptr()), None)
    torch.cuda.synchronize()
    out = [torch.empty((1, 256), dtype=torch.float64, device="cuda") for _ in range(3)]
    it = torch.empty(1, dtype=torch.int32, device="cuda")
    rows = []
    for b in range(B):
        buf = (ctypes.c_longlong * 1024)()
        for rep in range(2):
            lib.hr_debug_solve_clocks(buf, 1024)
            lib.hr_solve(ctx, vp(hs[b:].data_ptr()), vp(hg[b:].data_ptr()), ctypes.c_int64(1), ctypes.byref(P),
                         vp(out[0].data_ptr()), vp(out[1].data_ptr()), vp(out[2].data_ptr()), vp(it.data_ptr()),
                         vp(ws.data_ptr()), None)
            torch.cuda.synchronize()
            n = lib.hr_debug_solve_clocks(buf, 1024)
        c = np.array(buf[:n], dtype=np.int64)
        d = np.diff(c)
        full = (ctypes.c_longlong * 1024)()
        lib.hr_debug_solve_clocks_all(full)
        nL, nR = int((hs[b] > 0).sum()), int((hg[b] > 0).sum())
        sl = [int(v) for v in full[600:621]]
        rb1 = [sl[i + 1] - sl[i] for i in range(6)]
        rb2 = [sl[11 + i] - sl[10 + i] for i in range(6)]
        rows.append((int(c[-1] - c[0]), b, nL, nR, d.tolist(), [int(v) for v in full[512:528]], int(it.item()),
                     rb1, rb2))
    tot = np.array([r[0] for r in rows]) / GHZ / 1e3
    print(f"== {cfg}: {B} images, solve latency us: min {tot.min():.1f} p50 {np.median(tot):.1f} "
          f"p90 {np.percentile(tot, 90):.1f} max {tot.max():.1f}")
    for r in sorted(rows, reverse=True)[:6]:
        print(f"   img {r[1]:3d} nL={r[2]:3d} nR={r[3]:3d} E={r[2] * r[3]:5d} iters={r[6]:2d} "
              f"total {r[0] / GHZ / 1e3:6.1f} us  [hist,supp,runs,iters,eq20]={r[4]}  per-iter [E1,E2,R,L]="
              f"{[round(v / max(r[6], 1)) for v in r[5][:4]]}")
        print("      sub-phases per iter: E1[renorm,pieces,slot,bar]=%s E2[stopchk,bins,rcp,bar]=%s R[walk,shfl+v,slot,bar]=%s "
              "L[walk,shfl+u,slot,bar]=%s" % tuple(
                  str([round(r[5][i] / max(r[6], 1)) for i in ix]) for ix in ((7, 8, 9, 0), (14, 15, 10, 1), (4, 5, 6, 2),
                                                                              (11, 12, 13, 3))))
        print(f"      run_build steps [count+scan, desc, fix+mask, keyscan, slots, pieces+scan/write]: {r[7]}"
              f"  tail [idx1 keys, scan+zero, row walks, bin sums, target store, cdf+lut]: {r[8]}")
