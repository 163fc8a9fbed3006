"""Host check of the arithmetic claim behind the streaming apply kernel (apply_dev.cuh): the
colour reconstruction out_c = floor((2 c V' + V) / (2 V)) (reading R17) equals
rn(c * alpha + beta) in fp32 with alpha = fl(V'/V), beta = fl(1/(4V)), for EVERY level V >= 1,
channel value c <= V and matched level V' -- the fused multiply-add emulated exactly (the 8 x 24
bit product and the sum are exact in float64, one rounding to fp32), the rounding to nearest by
adding 1.5 * 2^23 as the kernel does.  The GPU tests compare the kernel itself with the oracle.
"""
import numpy as np


def test_fp32_colour_formula_exhaustive():
    V = np.arange(1, 256)
    Vf = V.astype(np.float32)
    beta = (np.float32(0.25) / Vf).astype(np.float32)      # correctly rounded fp32 division
    c = np.arange(256)
    ok = c[None, :] <= V[:, None]                          # a channel never exceeds the value channel
    cf = c.astype(np.float64)[None, :]
    for Vp in range(256):
        alpha = (np.float32(Vp) / Vf).astype(np.float32)
        y = (cf * alpha.astype(np.float64)[:, None] + beta.astype(np.float64)[:, None]).astype(np.float32)
        t = (y + np.float32(12582912.0)).astype(np.float32)
        out = (t.view(np.uint32) & 0xFF).astype(np.int64)
        ref = (2 * c[None, :] * Vp + V[:, None]) // (2 * V[:, None])
        assert np.array_equal(out[ok], ref[ok]), Vp
    # the distance of (2cV' + V + 1/2) / 2V from the integers that makes the rounding safe
    assert 0.5 / (2 * 255) > 9.8e-4
