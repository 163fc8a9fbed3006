"""One hr_solve launch on one config's histograms (a short command for ncu captures of k_solve).

    python tools/solve_one.py C5 [images]
"""
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2510_21100_b200 as hr  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 0
x = torch.from_numpy(synth.make_config(cfg, batch=n or None)).cuda()
hs, hg, _ = hr.hr_histogram(x)
for _ in range(3):
    hr.hr_solve(hs, hg)
torch.cuda.synchronize()
print("ok", cfg, tuple(x.shape))
