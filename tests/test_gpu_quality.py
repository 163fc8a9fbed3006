"""Second workload on the GPU: HE baseline and quality metrics vs the oracle.

HE (Eq. 5) pixels and tables are bit-exact; LOE counts are exact; PSNR and SSIM are fp64 and
equal to the oracle up to rounding order (PSNR from an exact integer SSE: 1e-12 relative; SSIM
from separable Gaussian sums: 1e-10 absolute).  Pairs cover an image against its HistRetinex
enhancement, against its HE baseline and against itself; shapes cover LOE's sampling grid
(> 100 px per side), SSIM's lower size limit (< 11 px: NaN) and ragged tiles.
"""
import math

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
    return np.stack([synth.make_image(H, W, seed=seed0 + 13 * b, peak=(0.05, 0.3, 0.12)[b % 3]) for b in range(B)])


@pytest.mark.parametrize("shape", [(3, 37, 112), (2, 64, 48), (1, 100, 100), (2, 17, 16), (4, 400, 600)])
def test_he_vs_oracle(shape):
    x = batch(*shape, seed0=1)
    out, lut = hr().hr_he(torch.from_numpy(x).cuda(), return_lut=True)
    out, lut = out.cpu().numpy(), lut.cpu().numpy()
    for b in range(x.shape[0]):
        t = oracle.he_transform(np.bincount(x[b].max(-1).ravel(), minlength=256))
        assert np.array_equal(lut[b].astype(np.int32), t), f"HE table image {b}"
        assert np.array_equal(out[b], oracle.he_enhance(x[b])), f"HE pixels image {b}"


@pytest.mark.parametrize("shape", [(3, 37, 112), (2, 64, 48), (2, 120, 333), (1, 300, 200), (2, 8, 40)])
def test_quality_vs_oracle(shape):
    x = batch(*shape, seed0=2)
    xd = torch.from_numpy(x).cuda()
    pairs = {
        "enhanced": hr().hr_enhance(xd),
        "he": hr().hr_he(xd),
        "identical": xd.clone(),
    }
    for name, y in pairs.items():
        ps, ss, lo = (t.cpu().numpy() for t in hr().hr_quality(xd, y))
        yh = y.cpu().numpy()
        for b in range(x.shape[0]):
            rp, rs, rl = oracle.psnr(x[b], yh[b]), oracle.ssim(x[b], yh[b]), oracle.loe(x[b], yh[b])
            if math.isinf(rp):
                assert math.isinf(ps[b]) and ps[b] > 0, (name, b)
            else:
                assert ps[b] == pytest.approx(rp, rel=1e-12), (name, b)
            if math.isnan(rs):
                assert math.isnan(ss[b]), (name, b)
            else:
                assert abs(ss[b] - rs) <= 1e-10, (name, b, ss[b], rs)
            assert lo[b] == rl, (name, b, lo[b], rl)


def test_quality_batch_equals_single():
    x = batch(5, 90, 130, seed0=3)
    xd = torch.from_numpy(x).cuda()
    y = hr().hr_enhance(xd)
    full = [t.cpu().numpy() for t in hr().hr_quality(xd, y)]
    for b in range(5):
        one = [t.cpu().numpy() for t in hr().hr_quality(xd[b:b + 1].contiguous(), y[b:b + 1].contiguous())]
        for f, o in zip(full, one):
            assert f[b] == o[0]


def test_he_improves_contrast_but_histretinex_preserves_order():
    """Diagnostic sanity on a dark batch: both brighten; HistRetinex keeps LOE low."""
    x = torch.from_numpy(batch(3, 120, 160, seed0=4)).cuda()
    y, h = hr().hr_enhance(x), hr().hr_he(x)
    assert float(y.float().mean()) > float(x.float().mean()) and float(h.float().mean()) > float(x.float().mean())
    _, _, lo_y = hr().hr_quality(x, y)
    assert torch.all(lo_y >= 0)
