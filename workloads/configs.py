"""The five BASELINE.json configurations and their seeded image generators.

Readings of the config strings (SURVEY.md §8(d) "Synthetic inputs"; recorded in
DESIGN.md §3 "Input recipe"):

* structure (patch colours, Voronoi seeds/colours, sinusoid parameters, disks)
  is drawn from ``numpy.random.default_rng(seed)`` in the order listed in each
  generator;
* the additive Gaussian noise is drawn per 64-row block from
  ``default_rng([seed, 0x5EED, block])`` in float32, so any row band of the
  8192x8192 image can be regenerated exactly without building the whole image;
* every image is clipped to its nominal range ([0,255], or [0,1] for config 4)
  and returned as planar float32 ``(d, rows, W)``.

Nothing in this module computes any part of the filter.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

NOISE_BLOCK = 64


@dataclasses.dataclass(frozen=True)
class Config:
    index: int            # 1-based, as in BASELINE.json configs[index-1]
    name: str
    H: int
    W: int
    d: int
    sigma_s: float
    C: tuple              # d x d covariance, row-major tuple of tuples
    N: int                # raised-cosine order
    M: int                # Monte Carlo samples (the paper's T)
    seed: int
    value_range: float    # nominal range R: 255, or 1 for config 4
    kind: str             # generator kind
    noise_sigma: float
    n_regions: int = 0    # Voronoi seeds / patches

    @property
    def radius(self) -> int:
        # ceil(3 sigma_s): PAPER.md:46 window [-3s,3s]^2, SPEC.md:242 ceiling.
        return int(math.ceil(3.0 * self.sigma_s - 1e-12))

    @property
    def C_array(self) -> np.ndarray:
        return np.array(self.C, dtype=np.float64)

    @property
    def pixels(self) -> int:
        return self.H * self.W

    @property
    def pixel_samples(self) -> int:
        return self.H * self.W * self.M


def _diag(v, d):
    return tuple(tuple(float(v) if i == j else 0.0 for j in range(d)) for i in range(d))


_C3 = tuple(tuple(35.0 ** 2 * x for x in row)
            for row in ((1.0, 0.5, 0.3), (0.5, 1.0, 0.5), (0.3, 0.5, 1.0)))

CONFIGS = {
    1: Config(1, "cfg1_patches_64x64_rgb", 64, 64, 3, 2.0, _diag(40.0 ** 2, 3), 20, 32, 0,
              255.0, "patches", 10.0, 64),
    2: Config(2, "cfg2_voronoi_512x512_rgb", 512, 512, 3, 5.0, _diag(30.0 ** 2, 3), 30, 64, 1,
              255.0, "voronoi", 15.0, 64),
    3: Config(3, "cfg3_sinusoid_disks_1080x1920_rgb", 1080, 1920, 3, 10.0, _C3, 40, 128, 2,
              255.0, "sinusoid_disks", 8.0, 200),
    4: Config(4, "cfg4_voronoi_1024x1024_d8", 1024, 1024, 8, 8.0, _diag(0.15 ** 2, 8), 30, 256, 3,
              1.0, "voronoi", 0.03, 32),
    5: Config(5, "cfg5_voronoi_8192x8192_rgb", 8192, 8192, 3, 16.0, _diag(30.0 ** 2, 3), 40, 512, 4,
              255.0, "voronoi", 12.0, 4096),
}


def get_config(i: int) -> Config:
    return CONFIGS[int(i)]


# --------------------------------------------------------------------------
# structure (drawn once from default_rng(seed), in the listed order)
# --------------------------------------------------------------------------
def _structure(cfg: Config):
    rng = np.random.default_rng(cfg.seed)
    R = cfg.value_range
    if cfg.kind == "patches":
        # 8x8 grid of 8x8-pixel constant patches, colours U[0,255]^3 per patch.
        gy, gx = cfg.H // 8, cfg.W // 8
        return {"colours": rng.uniform(0.0, R, size=(gy, gx, cfg.d))}
    if cfg.kind == "voronoi":
        seeds = rng.uniform([0.0, 0.0], [cfg.H, cfg.W], size=(cfg.n_regions, 2))  # (y, x)
        colours = rng.uniform(0.0, R, size=(cfg.n_regions, cfg.d))
        return {"seeds": seeds, "colours": colours}
    if cfg.kind == "sinusoid_disks":
        u = rng.uniform(0.0, 8.0, size=cfg.d)
        v = rng.uniform(0.0, 8.0, size=cfg.d)
        phi = rng.uniform(0.0, 2.0 * np.pi, size=cfg.d)
        centres = rng.uniform([0.0, 0.0], [cfg.H, cfg.W], size=(cfg.n_regions, 2))
        radii = rng.uniform(8.0, 64.0, size=cfg.n_regions)
        colours = rng.uniform(0.0, R, size=(cfg.n_regions, cfg.d))
        return {"u": u, "v": v, "phi": phi, "centres": centres, "radii": radii, "colours": colours}
    raise ValueError(cfg.kind)


_STRUCT_CACHE: dict = {}


def _cached_structure(cfg: Config):
    key = cfg.index
    if key not in _STRUCT_CACHE:
        st = _structure(cfg)
        if cfg.kind == "voronoi":
            from scipy.spatial import cKDTree
            st["tree"] = cKDTree(st["seeds"])
        _STRUCT_CACHE[key] = st
    return _STRUCT_CACHE[key]


def _base_rows(cfg: Config, y0: int, y1: int) -> np.ndarray:
    """Noise-free image rows [y0, y1) as float64 (d, y1-y0, W)."""
    st = _cached_structure(cfg)
    rows = y1 - y0
    ys = np.arange(y0, y1, dtype=np.float64)
    xs = np.arange(cfg.W, dtype=np.float64)
    if cfg.kind == "patches":
        iy = (np.arange(y0, y1) // 8)[:, None]
        ix = (np.arange(cfg.W) // 8)[None, :]
        img = st["colours"][iy, ix]                      # (rows, W, d)
        return np.ascontiguousarray(np.moveaxis(img, -1, 0))
    if cfg.kind == "voronoi":
        out = np.empty((cfg.d, rows, cfg.W), dtype=np.float64)
        step = max(1, (1 << 21) // cfg.W)
        for a in range(0, rows, step):
            b = min(rows, a + step)
            yy, xx = np.meshgrid(ys[a:b] + 0.5, xs + 0.5, indexing="ij")
            _, lab = st["tree"].query(np.stack([yy.ravel(), xx.ravel()], 1), workers=-1)
            out[:, a:b, :] = st["colours"][lab].T.reshape(cfg.d, b - a, cfg.W)
        return out
    if cfg.kind == "sinusoid_disks":
        u, v, phi = st["u"], st["v"], st["phi"]
        img = np.empty((cfg.d, rows, cfg.W), dtype=np.float64)
        for c in range(cfg.d):
            img[c] = 127.5 + 100.0 * np.sin(
                2.0 * np.pi * (u[c] * xs[None, :] / cfg.W + v[c] * ys[:, None] / cfg.H) + phi[c])
        yy = ys[:, None] + 0.5
        xx = xs[None, :] + 0.5
        for (cy, cx), rad, col in zip(st["centres"], st["radii"], st["colours"]):
            if cy + rad < y0 or cy - rad > y1:
                continue
            inside = (yy - cy) ** 2 + (xx - cx) ** 2 <= rad * rad
            for c in range(cfg.d):
                img[c][inside] = col[c]
        return img
    raise ValueError(cfg.kind)


def _noise_rows(cfg: Config, y0: int, y1: int) -> np.ndarray:
    out = np.empty((cfg.d, y1 - y0, cfg.W), dtype=np.float32)
    b0, b1 = y0 // NOISE_BLOCK, (y1 - 1) // NOISE_BLOCK
    for b in range(b0, b1 + 1):
        r0 = b * NOISE_BLOCK
        r1 = min(cfg.H, r0 + NOISE_BLOCK)
        rng = np.random.default_rng([cfg.seed, 0x5EED, b])
        blk = rng.standard_normal(size=(cfg.d, r1 - r0, cfg.W), dtype=np.float32)
        a, e = max(y0, r0), min(y1, r1)
        out[:, a - y0:e - y0, :] = blk[:, a - r0:e - r0, :]
    return out * np.float32(cfg.noise_sigma)


def make_image_rows(cfg: Config, y0: int, y1: int) -> np.ndarray:
    """Rows [y0, y1) of the config's image, planar float32 (d, y1-y0, W)."""
    if not (0 <= y0 < y1 <= cfg.H):
        raise ValueError("bad row range")
    img = _base_rows(cfg, y0, y1) + _noise_rows(cfg, y0, y1)
    np.clip(img, 0.0, cfg.value_range, out=img)
    return img.astype(np.float32)


def make_image(cfg: Config) -> np.ndarray:
    """The full image, planar float32 (d, H, W)."""
    return make_image_rows(cfg, 0, cfg.H)


def small_config(d=3, H=24, W=20, sigma_s=1.0, sigma_r=40.0, N=10, M=6, seed=0, C=None,
                 value_range=255.0) -> Config:
    """A tiny ad-hoc configuration for oracle / parity tests."""
    if C is None:
        C = _diag(sigma_r ** 2, d)
    else:
        C = tuple(tuple(float(x) for x in row) for row in np.asarray(C, dtype=np.float64))
    return Config(0, f"small_{H}x{W}_d{d}", H, W, d, float(sigma_s), C, N, M, seed,
                  value_range, "random", 0.0)


def random_image(H, W, d, seed=0, value_range=255.0, smooth=False) -> np.ndarray:
    """Uniform random planar float32 image (d, H, W) for small tests."""
    rng = np.random.default_rng(seed)
    img = rng.uniform(0.0, value_range, size=(d, H, W))
    if smooth:
        img = np.cumsum(img, axis=2) / np.arange(1, W + 1)
    return img.astype(np.float32)
