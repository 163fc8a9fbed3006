"""Solver latency probe: hr_solve / hr_match time vs iteration count and batch (GPU)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2510_21100_b200 as hr  # noqa: E402
import synth  # noqa: E402


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us


res = {}
for cfg in ("C3", "C5", "C2", "C4"):
    x = torch.from_numpy(synth.make_config(cfg)).cuda()
    hs, hg, _ = hr.hr_histogram(x)
    nz = [(int((hs[b] > 0).sum()), int((hg[b] > 0).sum())) for b in range(min(4, hs.shape[0]))]
    r = {"supports(nL,nR)": nz}
    for B in sorted({1, hs.shape[0]}):
        for T in (1, 2, 10):
            p = hr.Params(max_iter=T)
            r[f"solve_B{B}_T{T}_us"] = round(timeit(lambda: hr.hr_solve(hs[:B], hg[:B], p)), 2)
    tg = hr.hr_solve(hs, hg)[2]
    r["match_us"] = round(timeit(lambda: hr.hr_match(hs, tg)), 2)
    res[cfg] = r
    print(cfg, json.dumps(r), flush=True)
