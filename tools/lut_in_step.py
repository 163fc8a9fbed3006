"""Cycles of the CDF + LUT tail inside k_solve during hr_enhance (measurement build
tools/libhistretinex_prof.so; slots 15 -> 16 of the solver's fixed-slot clock marks).

    HR_LIB=tools/libhistretinex_prof.so python tools/lut_in_step.py [C2]
"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2510_21100_b200 as hr  # noqa: E402
from paper_2510_21100_b200 import _lib  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
lib = _lib.load()
x = torch.from_numpy(synth.make_config(cfg)).cuda()
hr.set_policy("graph_b1", 0)
hr.set_policy("solve_cluster", 0)
for _ in range(3):
    out = hr.hr_enhance(x)
torch.cuda.synchronize()
full = (ctypes.c_longlong * 1024)()
lib.hr_debug_solve_clocks_all(full)
sl = np.array(full[610:617], dtype=np.int64)
print(cfg, "tail [idx1 keys, scan+zero, row walks, bin sums, target store, cdf+lut] cycles:", np.diff(sl).tolist())
