"""Fused vs separate-kernel hr_enhance time over batch size (1080p images, CUDA events)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2510_21100_b200 as hr  # noqa: E402
import synth  # noqa: E402

x_all = torch.from_numpy(synth.make_config("C3")).cuda()
p = hr.Params()
for B in (2, 4, 8, 12, 16, 24, 32, 48, 64):
    x = x_all[:B].contiguous()
    out = torch.empty_like(x)
    ws = torch.empty(hr.workspace_bytes(B, 1080, 1920), dtype=torch.uint8, device="cuda")
    res = {}
    for name, fmin in (("fused", 2), ("separate", 0)):
        hr.set_policy("fused_min_b", fmin)
        hr.set_policy("fused_max_b", 1 << 20)
        for _ in range(5):
            hr.hr_enhance(x, p, out=out, workspace=ws)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            hr.hr_enhance(x, p, out=out, workspace=ws)
        e1.record()
        torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / 20 * 1e3
    print(f"B={B:3d}  fused {res['fused']:8.1f} us  separate {res['separate']:8.1f} us  "
          f"-> {'fused' if res['fused'] < res['separate'] else 'separate'}", flush=True)
