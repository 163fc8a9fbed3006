"""Phase clocks of the cluster solver on one large image (measurement build
tools/libhistretinex_prof.so, -DHR_SOLVE_PROFILE; slots in solve_cluster_dev.cuh).

    HR_LIB=tools/libhistretinex_prof.so python tools/cluster_scan.py [C4]
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2510_21100_b200 as hr  # noqa: E402
from paper_2510_21100_b200 import _lib  # noqa: E402

GHZ = 1.965
cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
lib = _lib.load()
x = torch.from_numpy(synth.make_config(cfg)).cuda()
hr.set_policy("graph_b1", 0)
for _ in range(3):
    out = hr.hr_enhance(x)
torch.cuda.synchronize()
full = (ctypes.c_longlong * 1024)()
lib.hr_debug_solve_clocks_all(full)
c = np.array(full[700:711], dtype=np.int64)
ph = np.array(full[720:725], dtype=np.int64)
names = ["supports", "keys", "runs", "iterations", "eq20+lut"]
print(f"{cfg}: cluster solve {(c[5] - c[0]) / GHZ / 1e3:.1f} us: " +
      " ".join(f"{n}={d}" for n, d in zip(names, np.diff(c).tolist())))
print("  per-iteration sums E1/E2+sync/E3/R+sync/L+sync (cycles, all iterations):", ph.tolist())
print("  tail: idx1 keys %d, row walks %d, bin sums + sync %d, combine %d, lut %d, final sync %d" % (
    c[6] - c[4], c[7] - c[6], c[8] - c[7], c[9] - c[8], c[10] - c[9], c[5] - c[10]))
