"""Per-phase clock64 breakdown of k_solve (measurement build tools/libhistretinex_prof.so)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2510_21100_b200 import _lib  # noqa: E402

lib = ctypes.CDLL("tools/libhistretinex_prof.so")
vp = ctypes.c_void_p
ctx = vp()
assert lib.hr_create(ctypes.byref(ctx), 0) == 0
P = _lib.HrParams()
lib.hr_default_params(ctypes.byref(P))
names = ["start", "hist", "supp", "list"]
it_names = ["E1", "E2", "R1", "R2", "L1", "L2", "RN"]
tail = ["T0", "T1", "T2", "end"]

for cfg, sel in (("C3", 0), ("C3", 2), ("C5", 0), ("C2", 0), ("C4", 0)):
    x = torch.from_numpy(synth.make_config(cfg, batch=sel + 1)[sel:sel + 1]).cuda()
    B, H, W, _ = x.shape
    ws = torch.empty(1 << 22, dtype=torch.uint8, device="cuda")
    hs = torch.empty((1, 256), dtype=torch.int32, device="cuda")
    hg = torch.empty_like(hs)
    hgr = torch.empty((1, 512), dtype=torch.int32, device="cuda")
    lib.hr_histogram(ctx, vp(x.data_ptr()), ctypes.c_int64(1), H, W, 0, vp(hs.data_ptr()), vp(hg.data_ptr()),
                     vp(hgr.data_ptr()), vp(ws.data_ptr()), None)
    out = [torch.empty((1, 256), dtype=torch.float64, device="cuda") for _ in range(3)]
    it = torch.empty(1, dtype=torch.int32, device="cuda")
    for rep in range(3):
        buf = (ctypes.c_longlong * 1024)()
        lib.hr_debug_solve_clocks(buf, 1024)
        lib.hr_solve(ctx, vp(hs.data_ptr()), vp(hg.data_ptr()), ctypes.c_int64(1), ctypes.byref(P),
                     vp(out[0].data_ptr()), vp(out[1].data_ptr()), vp(out[2].data_ptr()), vp(it.data_ptr()),
                     vp(ws.data_ptr()), None)
        torch.cuda.synchronize()
        n = lib.hr_debug_solve_clocks(buf, 1024)
    c = np.array(buf[:n], dtype=np.int64)
    d = np.diff(c)
    nL, nR = int((hs > 0).sum()), int((hg > 0).sum())
    print(f"{cfg}[{sel}] nL={nL} nR={nR} E={nL*nR} total={c[-1]-c[0]} cycles ({(c[-1]-c[0])/1.965e3:.1f} us @1.965GHz), marks={n}")
    # marks: start, hist, supp, runs, iterations (all), tail (Eq. 20 + target)
    print("  deltas [hist, supp, runs, iterations, eq20]:", d.tolist())
    wc = (ctypes.c_longlong * 16)()
    lib.hr_debug_solve_warp_clocks(wc)
    print("  warp kernel [load, supports, runs, E1 work, E1 reduce, Est, R work, R reduce, L work, L reduce+, after-loop, T+out]:",
          list(wc[:12]))
    full = (ctypes.c_longlong * 1024)()
    lib.hr_debug_solve_clocks_all(full)
    print("  iteration phase sums, each ending at its barrier [E1, E2, R, L]:", list(full[512:516]),
          "per iteration:", [round(x / 10) for x in full[512:516]])
