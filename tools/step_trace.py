"""Timeline of one hr_enhance step (step trace via hr_trace_bind): per kernel the CTA
start/end spread, per solver CTA its wait for the image's histogram and its solve, and when the
apply CTAs start.  Not product code.

    python tools/step_trace.py C3 [ENV=VAL ...]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2510_21100_b200 as hr  # noqa: E402
from paper_2510_21100_b200 import _lib  # noqa: E402

REC = np.dtype([("kind", "<u4"), ("cta", "<u4"), ("sm", "<u4"), ("aux", "<u4"), ("t0", "<u8"), ("mid", "<u8"),
                ("t1", "<u8"), ("pad", "<u8")])
NAMES = {1: "k_hist", 3: "k_solve", 4: "k_apply"}


def pct(a, qs=(0, 10, 50, 90, 100)):
    return " ".join(f"p{q}={np.percentile(a, q):7.1f}" for q in qs) if len(a) else "-"


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
    lib = _lib.load()
    cap = 1 << 16
    buf = torch.zeros(cap * REC.itemsize, dtype=torch.uint8, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    x = torch.from_numpy(synth.make_config(cfg)).cuda()
    out = torch.empty_like(x)
    ws = hr._workspace(*x.shape[:3], x.device)
    for _ in range(5):
        hr.hr_enhance(x, out=out, workspace=ws)
    torch.cuda.synchronize()
    hr.trace_bind(buf, cnt, cap)
    for _ in range(3):  # keep the last of three back-to-back steps (as in the bench loop)
        cnt.zero_()
        torch.cuda.synchronize()
        hr.hr_enhance(x, out=out, workspace=ws)
        hr.hr_enhance(x, out=out, workspace=ws)
        torch.cuda.synchronize()
    n = min(int(cnt.item()), cap)
    r = np.frombuffer(buf.cpu().numpy().tobytes(), dtype=REC)[:n]
    # the second of the two steps: records after the last k_hist* start of the second launch
    hs = np.sort(r[(r["kind"] == 1) | (r["kind"] == 2)]["t0"])
    t_step2 = hs[len(hs) // 2] if len(hs) else r["t0"].min()
    r = r[r["t0"] >= t_step2 - 1000] if len(hs) else r
    T0 = r["t0"].min()
    print(f"{cfg}: {n} records, step span {(r['t1'].max() - T0) / 1e3:.1f} us  (env: {sys.argv[2:]})")
    groups = []  # (kind, launch label): histogram / solver launches are told apart by aux
    for k in sorted(set(r["kind"])):
        q = r[r["kind"] == k]
        if k in (1, 3):
            for a in sorted(set(q["aux"]), key=lambda a: q[q["aux"] == a]["t0"].min()):
                groups.append((k, q[q["aux"] == a]))
        else:
            groups.append((k, q))
    for k, q in groups:
        print(f"  {NAMES.get(k, k):11s} CTAs {len(q):4d}  start[us] {pct((q['t0'] - T0) / 1e3)}")
        print(f"  {'':11s}            end[us] {pct((q['t1'] - T0) / 1e3)}")
        if k == 3:
            wait = (q["mid"] - q["t0"]) / 1e3
            solve = (q["t1"] - q["mid"]) / 1e3
            print(f"  {'':11s}        solve start {pct((q['mid'] - T0) / 1e3)}")
            print(f"  {'':11s}         wait[us] {pct(wait)}")
            print(f"  {'':11s}        solve[us] {pct(solve)}")


if __name__ == "__main__":
    for kv in sys.argv[2:]:
        k, v = kv.split("=")
        os.environ[k] = v
    main()
