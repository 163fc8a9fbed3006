"""γ sweep diagnostic on the GPU (after Table III's methodology).

For synthetic low-light batches (C5-like dark 600x400 and C3-like 1920x1080), enhance with
γ in {1, 1.5, 2.2, 3, 5, 7, 10} and report mean output V and PSNR / SSIM / LOE against the
input (hr_quality), next to the HE baseline (hr_he).  Metrics against the low-light input
measure change, not quality (the paper scores against references or no-reference NIQE, which
are out of scope); the table shows the γ trend and the order-preservation (LOE) contrast with
HE.  Also times hr_he and hr_quality.  Not product code; prints a table.
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2510_21100_b200 as hr  # noqa: E402
import synth  # noqa: E402


def fmean(t):  # mean over finite values (identical pairs have PSNR = +inf), and their count
    f = torch.isfinite(t)
    return (t[f].mean().item() if f.any() else float("inf")), int((~f).sum())


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for cfg, n in (("C5", 32), ("C3", 8)):
    x = torch.from_numpy(synth.make_config(cfg, batch=n)).cuda()
    B, H, W, _ = x.shape
    print(f"== {cfg}-like batch: {B} x {W}x{H}, mean input V {x.max(-1).values.float().mean():.1f}")
    print(f"{'method':>12s} {'mean V':>8s} {'PSNR dB':>8s} {'(=inf)':>6s} {'SSIM':>7s} {'LOE':>8s}")
    for g in (1.0, 1.5, 2.2, 3.0, 5.0, 7.0, 10.0):
        y = hr.hr_enhance(x, hr.Params(gamma=g))
        ps, ss, lo = hr.hr_quality(x, y)
        pm, ninf = fmean(ps)
        print(f"{'γ=' + str(g):>12s} {y.max(-1).values.float().mean():8.1f} {pm:8.2f} {ninf:6d} {ss.mean():7.4f} "
              f"{lo.mean():8.1f}")
    h = hr.hr_he(x)
    ps, ss, lo = hr.hr_quality(x, h)
    pm, ninf = fmean(ps)
    print(f"{'HE (Eq. 5)':>12s} {h.max(-1).values.float().mean():8.1f} {pm:8.2f} {ninf:6d} {ss.mean():7.4f} "
          f"{lo.mean():8.1f}")
    y = hr.hr_enhance(x)
    t_he = timed(lambda: hr.hr_he(x))
    t_q = timed(lambda: hr.hr_quality(x, y))
    mp = B * H * W / 1e6
    print(f"throughput: hr_he {mp / (t_he / 1e3):,.0f} MP/s ({t_he:.3f} ms), "
          f"hr_quality {mp / (t_q / 1e3):,.0f} MP/s ({t_q:.3f} ms)\n")
