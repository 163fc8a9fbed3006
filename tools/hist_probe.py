"""Histogram-kernel throughput vs image content (measurement only, not product code).

Times hr_histogram (zeroing + k_hist) with preallocated buffers on: a C3/C5 batch, a constant
image (every pixel the same V, gradient 0), uniform RGB noise, and a 'dark noise' image (V in
0..15).  Same shapes, so any difference is content-dependent (same-address shared atomics)."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2510_21100_b200 import _lib  # noqa: E402
import paper_2510_21100_b200 as hr  # noqa: E402

lib = _lib.load()
vp = ctypes.c_void_p


def run(name, x, reps=20):
    B, H, W, _ = x.shape
    ctx = hr._context(x.device)
    hs = torch.empty((B, 256), dtype=torch.int32, device="cuda")
    hg = torch.empty_like(hs)
    hgr = torch.empty((B, 512), dtype=torch.int32, device="cuda")
    ws = torch.empty(max(hr.workspace_bytes(B, H, W), 256), dtype=torch.uint8, device="cuda")
    st = vp(torch.cuda.current_stream().cuda_stream)

    def f():
        lib.hr_histogram(ctx, vp(x.data_ptr()), ctypes.c_int64(B), H, W, 0, vp(hs.data_ptr()), vp(hg.data_ptr()),
                         vp(hgr.data_ptr()), vp(ws.data_ptr()), st)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / reps * 1e3
    print(f"{name:12s} {tuple(x.shape)}  {us:7.1f} us  {x.numel() / us / 1e3:6.2f} TB/s", flush=True)


for cfg in sys.argv[1:] or ["C3", "C5"]:
    x = torch.from_numpy(synth.make_config(cfg)).cuda()
    run(cfg, x)
    g = torch.Generator(device="cuda").manual_seed(1)
    run(cfg + "-const", torch.full_like(x, 9))
    run(cfg + "-noise", torch.randint(0, 256, x.shape, dtype=torch.uint8, device="cuda", generator=g))
    run(cfg + "-dark16", torch.randint(0, 16, x.shape, dtype=torch.uint8, device="cuda", generator=g))
    del x

if len(sys.argv) > 1 and sys.argv[1] == "C5":
    x = torch.from_numpy(synth.make_config("C5")).cuda()
    run("C5-W592", x[:, :, :592].contiguous())
    run("C5-W576", x[:, :, :576].contiguous())
    run("C5-H200x2", x.reshape(512, 200, 600, 3))
    run("C5-2img", x.reshape(128, 800, 600, 3))
