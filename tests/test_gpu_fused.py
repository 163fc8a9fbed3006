"""The persistent fused kernel (csrc/k_fused.cu) against the separate-kernel path and the oracle.

hr_enhance picks the fused kernel for B >= fused_min_b (hr_set_policy); the policy is
performance-only, so every output (pixels, hist_s, LUT, iteration counts) must be
bit-identical to the unfused kernels for every knob value, and both must match the oracle.
Shapes cover the three hist template paths (W % 16 == 0, W % 8 == 0, scalar loads), the
scalar column tail, H = 1 / W = 1 degenerate rows, and shapes the fused kernel rejects
(H*W % 16 != 0 -> separate kernels).
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


def hr():
    import paper_2510_21100_b200 as m

    return m


def batch(B, H, W, seed0=0):
    return np.stack([synth.make_image(H, W, seed=seed0 + 97 * b, peak=(0.03, 0.3, 0.08)[b % 3]) for b in range(B)])


def run(x, params=None, **policy):
    m = hr()
    defaults = dict(fused_min_b=2, fused_max_b=1 << 20, fused_cpsm=2, fused_bands=2, fused_gs=8)
    defaults.update(policy)
    for k, v in defaults.items():
        m.set_policy(k, v)
    try:
        out, hs, lut, it = m.hr_enhance_debug(torch.from_numpy(x).cuda(), params)
        torch.cuda.synchronize()
        return out.cpu().numpy(), hs.cpu().numpy(), lut.cpu().numpy(), it.cpu().numpy()
    finally:
        for k, v in dict(fused_min_b=0, fused_max_b=0, fused_cpsm=2, fused_bands=2, fused_gs=8).items():
            m.set_policy(k, v)


SHAPES = [
    (2, 4, 4),      # one band, one chunk per image
    (3, 37, 112),   # W % 16 == 0: 16-px strips, ragged band rows
    (4, 30, 24),    # W % 8 == 0: 8-px strips
    (2, 16, 17),    # H*W % 16 == 0 with odd W: scalar-load strips + column tail
    (3, 16, 1),     # W = 1: all pixels in the scalar tail
    (2, 1, 48),     # H = 1: no dy anywhere
    (5, 64, 48),
    (2, 37, 101),   # H*W % 16 != 0: the fused kernel is not used (separate kernels)
]


@pytest.mark.parametrize("shape", SHAPES)
def test_fused_equals_unfused(shape):
    x = batch(*shape)
    f = run(x, fused_min_b=2)
    u = run(x, fused_min_b=0)
    for a, b, what in zip(f, u, ("pixels", "hist_s", "lut", "iters")):
        assert np.array_equal(a, b), f"{what} differ between fused and unfused"


@pytest.mark.parametrize("shape", [(3, 37, 112), (4, 30, 24), (2, 16, 17)])
def test_fused_vs_oracle(shape):
    x = batch(*shape, seed0=11)
    out, hs, lut, it = run(x)
    op = oracle.Params()
    for b in range(x.shape[0]):
        r = oracle.enhance(x[b], op)
        assert np.array_equal(hs[b].astype(np.uint64), r.hS)
        assert it[b] == r.iters
        assert np.array_equal(lut[b].astype(np.int32), r.lut)
        assert np.array_equal(out[b], r.out)


@pytest.mark.parametrize("knob,values", [
    ("fused_bands", [1, 2, 64, 4096]),   # one band per image .. one row per band
    ("fused_gs", [1, 3, 64, 100000]),    # tiny apply tickets .. one ticket for everything
    ("fused_cpsm", [1]),
])
def test_fused_policy_invariance(knob, values):
    x = batch(6, 90, 160, seed0=5)
    ref = run(x, fused_min_b=0)
    for v in values:
        got = run(x, **{knob: v})
        for a, b, what in zip(got, ref, ("pixels", "hist_s", "lut", "iters")):
            assert np.array_equal(a, b), f"{knob}={v}: {what} differ"


def test_fused_param_sets():
    x = batch(3, 48, 64, seed0=21)
    for kw in (dict(update_form=1), dict(use_epsilon=1, epsilon=1e-3), dict(grad_norm=1, beta=0.1), dict(gamma=1.0)):
        f = run(x, hr().Params(**kw), fused_min_b=2)
        u = run(x, hr().Params(**kw), fused_min_b=0)
        for a, b, what in zip(f, u, ("pixels", "hist_s", "lut", "iters")):
            assert np.array_equal(a, b), f"{kw}: {what} differ"


def test_fused_degenerate_images_in_batch():
    """All-black and constant images (solver's degenerate exits) next to normal ones."""
    x = batch(4, 32, 48, seed0=3)
    x[1] = 0
    x[2] = 77
    f = run(x, fused_min_b=2)
    u = run(x, fused_min_b=0)
    for a, b, what in zip(f, u, ("pixels", "hist_s", "lut", "iters")):
        assert np.array_equal(a, b), f"{what} differ"


def test_fused_repeat_and_large_batch():
    """Back-to-back launches reuse the zeroed control block; B = 300 > the grid's CTA count."""
    x = batch(300, 16, 32, seed0=9)
    a = run(x)
    b = run(x)
    u = run(x, fused_min_b=0)
    for p, q, r, what in zip(a, b, u, ("pixels", "hist_s", "lut", "iters")):
        assert np.array_equal(p, q) and np.array_equal(p, r), what


def test_set_policy_rejects_bad_keys():
    m = hr()
    with pytest.raises(m.HrError):
        m.set_policy("no_such_knob", 1)
    with pytest.raises(m.HrError):
        m.set_policy("fused_cpsm", 3)
    with pytest.raises(m.HrError):
        m.set_policy("fused_gs", 0)


@pytest.mark.parametrize("chunks", [0, 1, 3, 5])
def test_enhance_host_equals_device(chunks):
    """hr_enhance_host (pinned host in/out, copies pipelined over image chunks) gives exactly
    hr_enhance's output; pageable host memory works too."""
    m = hr()
    x = batch(5, 40, 64, seed0=31)
    ref = m.hr_enhance(torch.from_numpy(x).cuda()).cpu().numpy()
    xp = torch.from_numpy(x).pin_memory()
    got = m.hr_enhance_host(xp, chunks=chunks).numpy()
    assert np.array_equal(got, ref)
    got2 = m.hr_enhance_host(torch.from_numpy(x), chunks=chunks).numpy()  # pageable
    assert np.array_equal(got2, ref)


def test_enhance_host_rejects_bad_args():
    m = hr()
    with pytest.raises(ValueError):
        m.hr_enhance_host(torch.zeros((2, 4, 4, 3), dtype=torch.uint8, device="cuda"))


@pytest.mark.parametrize("knob", ["apply_dyn", "apply_dyn=2", "apply_dyn=3", "hist_overlap", "groups=2", "groups=3",
                                  "groups=7", "groups=2,group_apply=0", "groups=3,apply_gs=1",
                                  "solve_waves", "solve_waves,solve_waves_ag=2", "solve_wide_px=1",
                                  "groups=2,group_first_pct=0", "groups=2,group_first_pct=99",
                                  "groups=2,group_apply=2", "groups=3,group_apply=2,apply_gs=1",
                                  "groups=2,apply_tail_pct=30", "groups=2,apply_tail_pct=100",
                                  "solve_queue", "groups=3,solve_queue"])
@pytest.mark.parametrize("shape", [(2, 4, 4), (3, 37, 112), (4, 30, 24), (40, 16, 32), (300, 8, 16), (2, 37, 101),
                                   (2, 37, 264), (20, 45, 256), (5, 120, 600), (1, 300, 1920), (150, 16, 256)])
def test_policy_options_bit_exact(knob, shape):
    """The optional schedules (completion-order or flag-gated ticketed apply; solvers starting per
    image during the histogram pass; the grouped step, histograms of one group beside the solves
    of the previous one) change only the schedule.  The last
    five shapes take the TMA histogram kernel in image waves under hist_overlap (W % 16 == 8 with
    odd H; several waves; one image; more images than SMs)."""
    m = hr()
    x = torch.from_numpy(batch(*shape, seed0=17)).cuda()
    ref = [t.cpu() for t in m.hr_enhance_debug(x)]
    kv = [(k, int(v or 1)) for k, _, v in (item.partition("=") for item in knob.split(","))]
    saved = [(k, m.get_policy(k)) for k, _ in kv]
    for k, v in kv:
        m.set_policy(k, v)
    try:
        got = [t.cpu() for t in m.hr_enhance_debug(x)]
        got2 = [t.cpu() for t in m.hr_enhance_debug(x)]  # back-to-back: the queue state resets
    finally:
        for k, v in saved:
            m.set_policy(k, v)
    for a, b, c in zip(ref, got, got2):
        assert torch.equal(a, b) and torch.equal(a, c)
