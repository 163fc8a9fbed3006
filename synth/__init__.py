"""Seeded synthetic low-light RGB8 images (harness code; none of the method's arithmetic).

This module is the ONLY code shared by the oracle side and the CUDA side: it makes
input bytes.  It holds no histogram, solver, matching or colour arithmetic of the
method.  Recipe (from BASELINE.json "configs" and SURVEY.md 8(d)):

* illumination: sum of 3 isotropic 2-D Gaussians (centre ~ U[0,H) x U[0,W),
  sigma ~ U[0.15,0.5]*min(H,W), amplitude ~ U[0.5,1]), min-max normalised and mapped
  affinely to [peak*0.04/0.3, peak]  ([0.04, 0.3] at the default peak 0.3);
* reflectance: per channel i.i.d. U[0.2,1.0], smoothed by a 5x5 box mean (edge replicate);
* image = reflectance * illumination * 255 + N(0, sigma_n^2), clipped to [0,255], rint;
* optional bright spots (config C4): discs of radius U[0.003,0.01]*min(H,W) at uniform
  centres until >= spot_frac of the pixels are covered, set to U{240..255} per channel.

These images stand in for the paper's datasets (MEF/NPE/LOL/LSRW/ExDark),
which are not available; only their shapes are mirrored.  Layout [B][H][W][3] (HWC).
numpy PCG64 ``default_rng(seed)``, fixed draw order, float32 arithmetic.
"""
from __future__ import annotations

import hashlib
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np


def _box5(a: np.ndarray) -> np.ndarray:
    """5x5 box mean over axes (0, 1) with edge replication."""
    p = np.pad(a, ((2, 2), (2, 2), (0, 0)), mode="edge")
    H, W = a.shape[:2]
    s = p[0:H] + p[1:H + 1] + p[2:H + 2] + p[3:H + 3] + p[4:H + 4]
    t = s[:, 0:W] + s[:, 1:W + 1] + s[:, 2:W + 2] + s[:, 3:W + 3] + s[:, 4:W + 4]
    return t * np.float32(1.0 / 25.0)


def make_image(H: int, W: int, seed: int, peak: float = 0.3, sigma_n: float = 2.0,
               spot_frac: float = 0.0) -> np.ndarray:
    """One seeded synthetic low-light image, uint8 [H, W, 3]."""
    rng = np.random.default_rng(seed)
    m = float(min(H, W))
    ys = np.arange(H, dtype=np.float64)[:, None]
    xs = np.arange(W, dtype=np.float64)[None, :]
    illum = np.zeros((H, W), np.float64)
    for _ in range(3):
        cy = rng.uniform(0.0, H)
        cx = rng.uniform(0.0, W)
        sig = rng.uniform(0.15, 0.5) * m
        amp = rng.uniform(0.5, 1.0)
        gy = np.exp(-((ys - cy) ** 2) / (2.0 * sig * sig))
        gx = np.exp(-((xs - cx) ** 2) / (2.0 * sig * sig))
        illum += amp * (gy * gx)
    lo, hi = illum.min(), illum.max()
    illum = (illum - lo) / (hi - lo) if hi > lo else np.zeros_like(illum)
    low = peak * 0.04 / 0.3
    illum = (low + (peak - low) * illum).astype(np.float32)

    mask = None
    if spot_frac > 0:
        mask = np.zeros((H, W), bool)
        need = spot_frac * H * W
        covered = 0
        while covered < need:
            cy = rng.uniform(0.0, H)
            cx = rng.uniform(0.0, W)
            r = rng.uniform(0.003, 0.01) * m
            y0, y1 = max(0, int(np.floor(cy - r))), min(H, int(np.ceil(cy + r)) + 1)
            x0, x1 = max(0, int(np.floor(cx - r))), min(W, int(np.ceil(cx + r)) + 1)
            yy = np.arange(y0, y1)[:, None] + 0.5
            xx = np.arange(x0, x1)[None, :] + 0.5
            disc = (yy - cy) ** 2 + (xx - cx) ** 2 <= r * r
            sub = mask[y0:y1, x0:x1]
            covered += int(np.count_nonzero(disc & ~sub))
            sub |= disc

    refl = rng.random((H, W, 3), dtype=np.float32) * np.float32(0.8) + np.float32(0.2)
    refl = _box5(refl)
    noise = rng.standard_normal((H, W, 3), dtype=np.float32) * np.float32(sigma_n)
    img = refl * (illum[:, :, None] * np.float32(255.0)) + noise
    np.clip(img, 0.0, 255.0, out=img)
    out = np.rint(img).astype(np.uint8)
    if mask is not None:
        n = int(np.count_nonzero(mask))
        out[mask] = rng.integers(240, 256, size=(n, 3), dtype=np.uint8)
    return out


@dataclass(frozen=True)
class Config:
    name: str
    B: int
    H: int
    W: int
    use_epsilon: int  # Alg. 1 stop rule (C1) or fixed T (others)
    note: str

    @property
    def pixels(self) -> int:
        return self.B * self.H * self.W


# BASELINE.json "configs" (widths x heights as written there: "1000x664" = W 1000, H 664).
CONFIGS = {
    "C1": Config("C1", 1, 100, 100, 1, "single 100x100, seed 1, peak 0.3, sigma 2"),
    "C2": Config("C2", 1, 664, 1000, 0, "single 1000x664 (Table IV timing resolution), seed 2"),
    "C3": Config("C3", 64, 1080, 1920, 0, "64 x 1920x1080, seed 3000+b, peak ~ U[0.03,0.4] from rng(3)"),
    "C4": Config("C4", 1, 4320, 7680, 0, "single 7680x4320 + 0.5% bright spots, seed 4"),
    "C5": Config("C5", 256, 400, 600, 0, "256 x 600x400, very dark: peak 0.05, sigma 3, seed 5000+b"),
}


def image_params(cfg: str, b: int) -> dict:
    """Per-image generator arguments of config `cfg`, image b."""
    if cfg == "C1":
        return dict(seed=1, peak=0.3, sigma_n=2.0)
    if cfg == "C2":
        return dict(seed=2, peak=0.3, sigma_n=2.0)
    if cfg == "C3":
        peaks = np.random.default_rng(3).uniform(0.03, 0.4, size=CONFIGS["C3"].B)
        return dict(seed=3000 + b, peak=float(peaks[b]), sigma_n=2.0)
    if cfg == "C4":
        return dict(seed=4, peak=0.3, sigma_n=2.0, spot_frac=0.005)
    if cfg == "C5":
        return dict(seed=5000 + b, peak=0.05, sigma_n=3.0)
    raise KeyError(cfg)


def make_config(cfg: str, batch: int | None = None, out: np.ndarray | None = None,
                threads: int = 8, first: int = 0) -> np.ndarray:
    """The [B, H, W, 3] uint8 batch of config `cfg` (optionally only `batch` images), starting
    at image `first` of the config's seeded image sequence (a data-parallel rank's shard).

    `out` may be a preallocated (e.g. pinned) uint8 array of the right shape."""
    c = CONFIGS[cfg]
    B = c.B if batch is None else batch
    if out is None:
        out = np.empty((B, c.H, c.W, 3), np.uint8)

    def one(b):
        out[b] = make_image(c.H, c.W, **image_params(cfg, first + b))

    if B == 1 or threads <= 1:
        for b in range(B):
            one(b)
    else:
        with ThreadPoolExecutor(max_workers=threads) as ex:
            list(ex.map(one, range(B)))
    return out


def sha256(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8)).hexdigest()


def edge_images() -> dict:
    """Parity-only inputs for the edge cases the five configs miss."""
    rng = np.random.default_rng(12345)
    e = {}
    e["uniform_noise"] = rng.integers(0, 256, size=(64, 96, 3), dtype=np.uint8)  # dense supports
    e["constant"] = np.full((33, 47, 3), (40, 25, 10), np.uint8)
    e["black"] = np.zeros((20, 30, 3), np.uint8)
    e["one_pixel"] = np.array([[[7, 200, 3]]], np.uint8)
    e["one_row"] = make_image(1, 173, seed=11)
    e["one_col"] = make_image(157, 1, seed=12)
    e["ragged_101x37"] = make_image(37, 101, seed=13)
    e["clamp_case"] = np.array([[[255, 255, 255], [0, 0, 0]], [[0, 0, 0], [0, 0, 0]]], np.uint8)
    return e
