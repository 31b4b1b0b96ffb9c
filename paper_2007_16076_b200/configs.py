"""Seeded synthetic images for the five BASELINE.json configurations.

There is no public dataset behind BASELINE.json; these generators are the
stand-ins.  Every detail the recipes leave open is pinned
here and recorded in DESIGN.md:

cfg1  32x32 fp32 U[0,1) (``rng.random(dtype=float32)``), 8-conn, naive.
cfg2  64x64 uint8 U{0..255} (``rng.integers(0, 256)``), zeros remapped to 1
      (the reference's own ``remap_zero`` rule, pgm.py:42-47), 8-conn,
      filling-rate.
cfg3  128x128: standard-normal white noise, Gaussian sigma=2 px (separable,
      scipy-compatible 'reflect' boundary, truncate=4.0 -> radius 8), min-max
      to [0,1] in float64 then cast to fp32; 4-conn, filling-rate.
cfg4  128x128 uint8: 32 Voronoi sites uniform in [0,128)^2 (float coords,
      nearest to the pixel centre (r, c) by squared Euclidean distance, ties to
      the lowest site index), site values U{0..255}, plus per-pixel noise
      U{-8..8}, clipped to [0,255], zeros remapped to 1; 8-conn, filling-rate.
cfg5  256x256: value noise, octaves with cell sizes 64/16/4 px and weights
      0.6/0.3/0.1; each octave is a (256/cell+1)^2 lattice of U[0,1) values
      interpolated bilinearly at (r/cell, c/cell); the weighted sum is min-max
      rescaled to [0,1] in float64 then cast to fp32; 8-conn, filling-rate.

Only numpy is used, so the same images are produced on the GPU box.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SEEDS = {1: 20071601, 2: 20071602, 3: 20071603, 4: 20071604, 5: 20071605}


@dataclass(frozen=True)
class ConfigSpec:
    index: int
    name: str
    shape: tuple[int, int]
    conn: int
    strategy: str  # "naive" | "filling-rate"
    dtype: str     # "f32" | "u8"

    @property
    def n(self) -> int:
        return self.shape[0] * self.shape[1]

    @property
    def total_pairs(self) -> int:
        return (self.n * self.n - self.n) // 2


CONFIGS = {
    1: ConfigSpec(1, "cfg1_32x32_f32_u01_8c_naive", (32, 32), 8, "naive", "f32"),
    2: ConfigSpec(2, "cfg2_64x64_u8_uniform_8c_fillrate", (64, 64), 8, "filling-rate", "u8"),
    3: ConfigSpec(3, "cfg3_128x128_f32_gauss2_4c_fillrate", (128, 128), 4, "filling-rate", "f32"),
    4: ConfigSpec(4, "cfg4_128x128_u8_voronoi32_8c_fillrate", (128, 128), 8, "filling-rate", "u8"),
    5: ConfigSpec(5, "cfg5_256x256_f32_valuenoise_8c_fillrate", (256, 256), 8, "filling-rate", "f32"),
}


def _gauss_kernel(sigma: float, truncate: float = 4.0) -> np.ndarray:
    radius = int(truncate * sigma + 0.5)
    x = np.arange(-radius, radius + 1, dtype=np.float64)
    k = np.exp(-0.5 * (x / sigma) ** 2)
    return k / k.sum()


def _filter1d_reflect(a: np.ndarray, k: np.ndarray, axis: int) -> np.ndarray:
    r = (len(k) - 1) // 2
    pad = [(0, 0)] * a.ndim
    pad[axis] = (r, r)
    p = np.pad(a, pad, mode="symmetric")  # scipy.ndimage 'reflect' == numpy 'symmetric'
    out = np.zeros_like(a)
    n = a.shape[axis]
    for i, kv in enumerate(k):
        sl = [slice(None)] * a.ndim
        sl[axis] = slice(i, i + n)
        out += kv * p[tuple(sl)]
    return out


def gaussian_filter(a: np.ndarray, sigma: float, truncate: float = 4.0) -> np.ndarray:
    k = _gauss_kernel(sigma, truncate)
    return _filter1d_reflect(_filter1d_reflect(np.asarray(a, np.float64), k, 0), k, 1)


def _minmax01_f32(a: np.ndarray) -> np.ndarray:
    lo, hi = a.min(), a.max()
    return ((a - lo) / (hi - lo)).astype(np.float32)


def make_image(index: int, seed: int | None = None) -> np.ndarray:
    """The synthetic image of config ``index`` (uint8 for int configs, fp32 else)."""
    spec = CONFIGS[index]
    rng = np.random.default_rng(SEEDS[index] if seed is None else seed)
    H, W = spec.shape
    if index == 1:
        return rng.random((H, W), dtype=np.float32)
    if index == 2:
        img = rng.integers(0, 256, (H, W)).astype(np.uint8)
        return np.maximum(img, 1).astype(np.uint8)
    if index == 3:
        noise = rng.standard_normal((H, W))
        return _minmax01_f32(gaussian_filter(noise, 2.0, 4.0))
    if index == 4:
        sites = rng.uniform(0.0, float(H), (32, 2))
        vals = rng.integers(0, 256, 32)
        rr, cc = np.mgrid[0:H, 0:W]
        d2 = (rr[..., None] - sites[:, 0]) ** 2 + (cc[..., None] - sites[:, 1]) ** 2
        label = np.argmin(d2, axis=-1)
        img = vals[label] + rng.integers(-8, 9, (H, W))
        img = np.clip(img, 0, 255).astype(np.uint8)
        return np.maximum(img, 1).astype(np.uint8)
    if index == 5:
        acc = np.zeros((H, W), dtype=np.float64)
        rr, cc = np.mgrid[0:H, 0:W].astype(np.float64)
        for cell, weight in ((64, 0.6), (16, 0.3), (4, 0.1)):
            lat = rng.random((H // cell + 1, W // cell + 1))
            y, x = rr / cell, cc / cell
            y0, x0 = np.floor(y).astype(int), np.floor(x).astype(int)
            fy, fx = y - y0, x - x0
            y1 = np.minimum(y0 + 1, lat.shape[0] - 1)
            x1 = np.minimum(x0 + 1, lat.shape[1] - 1)
            v = (lat[y0, x0] * (1 - fy) * (1 - fx) + lat[y0, x1] * (1 - fy) * fx
                 + lat[y1, x0] * fy * (1 - fx) + lat[y1, x1] * fy * fx)
            acc += weight * v
        return _minmax01_f32(acc)
    raise ValueError(f"unknown config {index}")
