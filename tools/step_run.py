"""K hr_enhance steps of one config on a stream of its own, the way bench.py runs them (a short
command for ncu launch lists and captures).

    python tools/step_run.py C3 [K] [groups]
"""
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2510_21100_b200 as hr  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 4
if len(sys.argv) > 3:
    hr.set_policy("groups", int(sys.argv[3]))
c = synth.CONFIGS[cfg]
x = torch.from_numpy(synth.make_config(cfg)).cuda()
out = torch.empty_like(x)
ws = torch.empty(hr.workspace_bytes(*x.shape[:3]), dtype=torch.uint8, device="cuda")
p = hr.Params(use_epsilon=c.use_epsilon)
s = torch.cuda.Stream()
torch.cuda.synchronize()
with torch.cuda.stream(s):
    for _ in range(K):
        hr.hr_enhance(x, p, out=out, workspace=ws)
    s.synchronize()
print("ok", cfg, K, "launches", hr.kernel_launches())
