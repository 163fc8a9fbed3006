"""A/B: hr_enhance launched directly vs replayed from a CUDA graph captured from the same calls
(stream capture keeps the programmatic-dependent-launch edges).  Per config: steps timed the
bench way (back to back; configs whose input fits in L2 each after a 256 MB flush), median of
5 rounds.  Not product code.

    python tools/graph_ab.py [C1 C2 C3 C5 ...]
"""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import synth  # noqa: E402
import paper_2510_21100_b200 as hr  # noqa: E402

cfgs = sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"]
for cfg in cfgs:
    c = synth.CONFIGS[cfg]
    x = torch.from_numpy(synth.make_config(cfg)).cuda()
    out = torch.empty_like(x)
    ws = torch.empty(hr.workspace_bytes(*x.shape[:3]), dtype=torch.uint8, device="cuda")
    p = hr.Params(use_epsilon=c.use_epsilon)

    def step():
        hr.hr_enhance(x, p, out=out, workspace=ws)

    for _ in range(5):
        step()
    torch.cuda.synchronize()
    ref = out.clone()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            step()
    torch.cuda.current_stream().wait_stream(s)
    with torch.cuda.graph(g):
        step()
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref), "graph replay output differs"
    flush = torch.empty(bench.L2_FLUSH_BYTES, dtype=torch.uint8, device="cuda") if bench.flush_l2(*x.shape[:3]) else None
    st = torch.cuda.current_stream()

    def timed(fn, n):
        if flush is not None:
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
            for a, b in ev:
                flush.fill_(1)
                a.record(st)
                fn()
                b.record(st)
            torch.cuda.synchronize()
            return statistics.median(a.elapsed_time(b) for a, b in ev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(n):
            fn()
        e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n

    n = 200 if flush is None else 100
    rd, rg = [], []
    for _ in range(5):
        rd.append(timed(step, n))
        rg.append(timed(g.replay, n))
    print(f"{cfg}: direct {statistics.median(rd):.4f} ms  graph {statistics.median(rg):.4f} ms  "
          f"(rounds direct {[round(v, 4) for v in rd]} graph {[round(v, 4) for v in rg]})", flush=True)
