"""Per-CTA end times of the histogram kernel vs its segment count (step trace via
hr_trace_bind; not product code).

    python tools/hist_balance.py C5
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2510_21100_b200 as hr  # noqa: E402
from paper_2510_21100_b200 import _lib  # noqa: E402

REC = np.dtype([("kind", "<u4"), ("cta", "<u4"), ("sm", "<u4"), ("aux", "<u4"), ("t0", "<u8"), ("mid", "<u8"),
                ("t1", "<u8"), ("pad", "<u8")])
cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
lib = _lib.load()
cap = 1 << 16
buf = torch.zeros(cap * REC.itemsize, dtype=torch.uint8, device="cuda")
cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
x = torch.from_numpy(synth.make_config(cfg)).cuda()
B, H, W, _ = x.shape
hs, hg, hgr = hr.hr_histogram(x)
hr.trace_bind(buf, cnt, cap)
ends = []
for rep in range(5):
    cnt.zero_()
    torch.cuda.synchronize()
    hr.hr_histogram(x)
    torch.cuda.synchronize()
    n = min(int(cnt.item()), cap)
    r = np.frombuffer(buf.cpu().numpy().tobytes(), dtype=REC)[:n]
    r = r[r["kind"] == 1]
    ends.append(r)
G = 296
R = B * H
for r in ends[-2:]:
    T0 = r["t0"].min()
    seg = np.array([len({(row // H) for row in (R * c // G, (R * (c + 1) // G) - 1)}) for c in r["cta"]])
    dur = (r["t1"] - T0) / 1e3
    sm = r["sm"]
    print(f"{cfg}: end p0 {dur.min():.1f} p50 {np.median(dur):.1f} p100 {dur.max():.1f} us")
    for k in (1, 2):
        m = seg == k
        if m.any():
            print(f"  {k} segment(s): {m.sum():3d} CTAs, end mean {dur[m].mean():.1f} us, max {dur[m].max():.1f}")
    # by SM: do the two CTAs of an SM end together?  by SM id range (GPC / die)
    order = np.argsort(sm)
    per_sm = {}
    for s_, d_ in zip(sm, dur):
        per_sm.setdefault(int(s_), []).append(d_)
    sm_end = np.array([max(v) for k, v in sorted(per_sm.items())])
    print("  SM end (max of its CTAs) by SM id deciles:", " ".join(f"{np.mean(c):.1f}" for c in np.array_split(sm_end, 10)))
