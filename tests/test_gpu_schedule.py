"""hr_enhance's schedules (separate kernels, the grouped step) and the host-memory entry point.

The execution policy (hr_set_policy) is performance-only: every output (pixels, hist_s, LUT,
iteration counts) must be bit-identical whatever the knobs, and equal to the oracle.  Shapes
cover the histogram kernel's template paths (W % 16 == 0: 16-px strips, W % 8 == 0: 8-px strips,
byte loads), H*W % 16 != 0 (the scalar apply), one-row images, batches larger than the grid,
and degenerate images next to normal ones.
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
    saved = [(k, m.get_policy(k)) for k in policy]
    for k, v in policy.items():
        m.set_policy(k, v)
    try:
        out, hs, lut, it = m.hr_enhance_debug(torch.from_numpy(x).cuda(), params)
        torch.cuda.synchronize()
        return out.cpu().numpy(), hs.cpu().numpy(), lut.cpu().numpy(), it.cpu().numpy()
    finally:
        for k, v in saved:
            m.set_policy(k, v)


SHAPES = [(2, 4, 4), (3, 37, 112), (4, 30, 24), (2, 16, 17), (3, 16, 1), (2, 1, 48), (5, 64, 48), (2, 37, 101),
          (5, 120, 600), (40, 16, 32), (300, 8, 16), (20, 45, 256), (150, 16, 256)]


@pytest.mark.parametrize("shape", SHAPES)
def test_grouped_equals_separate_and_oracle(shape):
    x = batch(*shape, seed0=17)
    g = run(x)  # default: the grouped step for B >= 2
    assert hr().last_path() == 3
    s = run(x, groups=0)
    assert hr().last_path() == 0
    for a, b, what in zip(g, s, ("pixels", "hist_s", "lut", "iters")):
        assert np.array_equal(a, b), f"{what}: grouped step != separate kernels"
    op = oracle.Params()
    for b in range(min(3, x.shape[0])):
        r = oracle.enhance(x[b], op)
        assert np.array_equal(g[1][b].astype(np.uint64), r.hS)
        assert g[3][b] == r.iters
        assert np.array_equal(g[2][b].astype(np.int32), r.lut)
        assert np.array_equal(g[0][b], r.out)


@pytest.mark.parametrize("knob", ["groups=3", "groups=7", "groups=2,group_first_pct=1", "groups=2,group_first_pct=99",
                                  "groups=3,apply_gs=1", "groups=2,apply_gs=1000", "solve_wide_px=1",
                                  "groups=0,solve_wide_px=1", "solve_cpsm=1", "solve_cpsm=2", "hist_cpsm=1",
                                  "apply_cpsm=1", "groups=0,solve_cpsm=2,hist_cpsm=1,apply_cpsm=1",
                                  "apply_full_grid=1", "apply_full_grid=0", "groups=3,apply_full_grid=1"])
@pytest.mark.parametrize("shape", [(2, 4, 4), (3, 37, 112), (40, 16, 32), (2, 37, 264), (5, 120, 600), (1, 300, 1920),
                                   (150, 16, 256)])
def test_policy_options_bit_exact(knob, shape):
    x = batch(*shape, seed0=17)
    ref = run(x)
    kv = {k: int(v) for k, _, v in (item.partition("=") for item in knob.split(","))}
    got = run(x, **kv)
    got2 = run(x, **kv)  # back to back: the control block is re-zeroed every step
    for a, b, c, what in zip(ref, got, got2, ("pixels", "hist_s", "lut", "iters")):
        assert np.array_equal(a, b) and np.array_equal(a, c), f"{knob}: {what}"


def test_param_sets_both_schedules():
    x = batch(3, 48, 64, seed0=21)
    for kw in (dict(update_form=1), dict(use_epsilon=1, epsilon=1e-3), dict(grad_norm=1, beta=0.1), dict(gamma=1.0)):
        g = run(x, hr().Params(**kw))
        s = run(x, hr().Params(**kw), groups=0)
        for a, b, what in zip(g, s, ("pixels", "hist_s", "lut", "iters")):
            assert np.array_equal(a, b), f"{kw}: {what}"


def test_degenerate_images_in_batch():
    """All-black and constant images (the solver's degenerate exits) next to normal ones."""
    x = batch(4, 32, 48, seed0=3)
    x[1] = 0
    x[2] = 77
    g = run(x)
    s = run(x, groups=0)
    for a, b, what in zip(g, s, ("pixels", "hist_s", "lut", "iters")):
        assert np.array_equal(a, b), what
    for b in (1, 2):
        r = oracle.enhance(x[b], oracle.Params())
        assert np.array_equal(g[0][b], r.out)


def test_set_policy_rejects_bad_keys():
    m = hr()
    with pytest.raises(m.HrError):
        m.set_policy("no_such_knob", 1)
    with pytest.raises(m.HrError):
        m.set_policy("hist_cpsm", 3)
    with pytest.raises(m.HrError):
        m.set_policy("apply_gs", 0)
    for gone in ("fused_min_b", "chunks", "warp_solver", "hist_tma", "apply_dyn", "solve_queue"):
        with pytest.raises(m.HrError):
            m.set_policy(gone, 1)


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


def test_caller_buffers_are_checked():
    """Buffers the C side cannot size-check are checked by the binding (ValueError, nothing
    launched): a workspace for a smaller batch, a mis-shaped out / lut / hist / target."""
    m = hr()
    x = torch.from_numpy(batch(4, 40, 64)).cuda()
    small = torch.empty(m.workspace_bytes(1, 40, 64), dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError):
        m.hr_enhance(x, workspace=small)
    with pytest.raises(ValueError):
        m.hr_enhance(x, out=torch.empty((4, 40, 63, 3), dtype=torch.uint8, device="cuda"))
    with pytest.raises(ValueError):
        m.hr_enhance(x, out=x)
    with pytest.raises(ValueError):
        m.hr_apply(x, torch.zeros((3, 256), dtype=torch.uint8, device="cuda"))
    hs = torch.zeros((4, 256), dtype=torch.int32, device="cuda")
    with pytest.raises(ValueError):
        m.hr_solve(hs, torch.zeros((3, 256), dtype=torch.int32, device="cuda"))
    with pytest.raises(ValueError):
        m.hr_match(hs, torch.zeros((4, 255), dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        m.hr_enhance_host(x.cpu(), in_dev=torch.empty((4, 40, 64, 2), dtype=torch.uint8, device="cuda"))
    with pytest.raises(ValueError):
        m.hr_enhance_host(x.cpu(), out_host=torch.empty((4, 40, 64, 2), dtype=torch.uint8))


def test_enhance_host_rejects_bad_args():
    m = hr()
    with pytest.raises(ValueError):
        m.hr_enhance_host(torch.zeros((2, 4, 4, 3), dtype=torch.uint8, device="cuda"))


def test_many_gammas_reuse_index1_tables():
    """More distinct gammas than the context caches (64): slots are reused after their readers
    finished; every result still matches a fresh computation at the same gamma."""
    m = hr()
    x = torch.from_numpy(batch(2, 24, 32, seed0=5)).cuda()
    gammas = [1.0 + 0.05 * i for i in range(70)]
    outs = [m.hr_enhance(x, m.Params(gamma=g)) for g in gammas]
    torch.cuda.synchronize()
    for g, o in list(zip(gammas, outs))[::9]:
        r = oracle.enhance(x[0].cpu().numpy(), oracle.Params(gamma=g))
        assert np.array_equal(o[0].cpu().numpy(), r.out), g


def test_single_image_graph_replay():
    """One image on a non-default stream: hr_enhance captures its step into a cached CUDA graph
    and replays it; outputs equal the direct launches, a new buffer or parameter set captures
    anew, and the kernel counter counts the replayed kernels."""
    m = hr()
    x = torch.from_numpy(batch(1, 90, 160, seed0=41)).cuda()
    ref = m.hr_enhance(x)  # legacy default stream: direct launches
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        outs = []
        out = torch.empty_like(x)
        ws = torch.empty(m.workspace_bytes(1, 90, 160), dtype=torch.uint8, device="cuda")
        for g in (2.2, 2.2, 1.5, 2.2):
            k0 = m.kernel_launches()
            m.hr_enhance(x, m.Params(gamma=g), out=out, workspace=ws)
            outs.append((g, out.clone(), m.kernel_launches() - k0))
        s.synchronize()
    assert torch.equal(outs[0][1], ref) and torch.equal(outs[1][1], ref) and torch.equal(outs[3][1], ref)
    assert outs[0][2] == outs[1][2] == outs[3][2] > 0
    r15 = oracle.enhance(x[0].cpu().numpy(), oracle.Params(gamma=1.5))
    assert np.array_equal(outs[2][1][0].cpu().numpy(), r15.out)


def test_graphs_with_many_gammas():
    """One image on a side stream with more gammas than cached index_1 tables: evicting a table
    also drops the cached step graphs that read it; every output matches the oracle."""
    m = hr()
    x = torch.from_numpy(batch(1, 24, 32, seed0=6)).cuda()
    s = torch.cuda.Stream()
    gammas = [1.0 + 0.04 * i for i in range(70)] + [1.0, 1.04, 3.76]
    with torch.cuda.stream(s):
        out = torch.empty_like(x)
        ws = torch.empty(m.workspace_bytes(1, 24, 32), dtype=torch.uint8, device="cuda")
        res = []
        for g in gammas:
            m.hr_enhance(x, m.Params(gamma=g), out=out, workspace=ws)
            res.append(out.clone())
        s.synchronize()
    for g, o in list(zip(gammas, res))[::7] + list(zip(gammas, res))[-3:]:
        r = oracle.enhance(x[0].cpu().numpy(), oracle.Params(gamma=g))
        assert np.array_equal(o[0].cpu().numpy(), r.out), g
