"""Small cases of every hr_enhance path for compute-sanitizer (memcheck / racecheck / synccheck)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2510_21100_b200 as hr  # noqa: E402
import synth  # noqa: E402


def batch(B, H, W, s0=0):
    return torch.from_numpy(np.stack([synth.make_image(H, W, seed=s0 + b, peak=(0.05, 0.3)[b % 2]) for b in range(B)])).cuda()


cases = [(2, 32, 48), (3, 17, 40), (2, 16, 17), (1, 64, 96), (4, 30, 24)]
for B, H, W in cases:
    x = batch(B, H, W)
    for fused in (0, 2):
        hr.set_policy("fused_min_b", fused)
        hr.set_policy("fused_max_b", 1 << 20)
        out = hr.hr_enhance(x)
        torch.cuda.synchronize()
    hr.set_policy("fused_min_b", 0)
    hr.set_policy("hist_overlap", 1)
    out2 = hr.hr_enhance(x)
    hr.set_policy("hist_overlap", 0)
    torch.cuda.synchronize()
    assert torch.equal(out, out2)
    hs, hg, graw = hr.hr_histogram(x)
    hL, hR, T, it = hr.hr_solve(hs, hg)
    lut, _st = hr.hr_match(hs, T)
    o3 = hr.hr_apply(x, lut)
    torch.cuda.synchronize()
    h = hr.hr_enhance_host(x.cpu(), chunks=2)
    print("case", B, H, W, "ok", flush=True)
print("all cases ok")
