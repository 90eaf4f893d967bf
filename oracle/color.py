"""sRGB <-> CIE-Lab (D65) for the Lab-space filtering of PAPER.md:305-308 ("we first performed a
color transformation from the RGB to the CIE-Lab space, performed the filtering in the CIE-Lab
space, and then transformed back to the RGB space"). TEST INFRASTRUCTURE ONLY.

Plain fp64 from the defining constants (reading R18):
  * sRGB transfer (IEC 61966-2-1): c <= 0.04045 -> c / 12.92, else ((c + 0.055) / 1.055)^2.4,
    c = v / 255; inverse c <= 0.0031308 -> 12.92 c, else 1.055 c^(1/2.4) - 0.055;
  * linear RGB -> XYZ: the matrix whose columns are the primaries' XYZ (chromaticities
    R (0.64, 0.33), G (0.30, 0.60), B (0.15, 0.06)) scaled so that RGB = (1, 1, 1) maps to the
    D65 white (x, y) = (0.3127, 0.3290), Y = 1;
  * CIE 1976 L*a*b* relative to that white: f(t) = t^(1/3) if t > (6/29)^3 else
    t / (3 (6/29)^2) + 4/29; L = 116 f(Y/Yn) - 16, a = 500 (f(X/Xn) - f(Y/Yn)),
    b = 200 (f(Y/Yn) - f(Z/Zn)).
Planar images (3, ...) in and out.
"""
import numpy as np

DELTA = 6.0 / 29.0
PRIMARIES = np.array([[0.64, 0.33], [0.30, 0.60], [0.15, 0.06]])
WHITE_XY = np.array([0.3127, 0.3290])


def _xyz(xy):
    x, y = xy
    return np.array([x / y, 1.0, (1.0 - x - y) / y])


def rgb_to_xyz_matrix():
    P = np.stack([_xyz(p) for p in PRIMARIES], axis=1)       # columns: primaries at Y = 1
    S = np.linalg.solve(P, _xyz(WHITE_XY))                      # scale so that M (1,1,1) = white
    return P * S[None, :]


def white():
    return _xyz(WHITE_XY)


def srgb_to_linear(v):
    c = np.asarray(v, dtype=np.float64) / 255.0
    return np.where(c <= 0.04045, c / 12.92, ((c + 0.055) / 1.055) ** 2.4)


def linear_to_srgb(c):
    c = np.asarray(c, dtype=np.float64)
    return 255.0 * np.where(c <= 0.0031308, 12.92 * c, 1.055 * np.sign(c) * np.abs(c) ** (1.0 / 2.4) - 0.055)


def _f(t):
    return np.where(t > DELTA ** 3, np.cbrt(t), t / (3 * DELTA ** 2) + 4.0 / 29.0)


def _finv(t):
    return np.where(t > DELTA, t ** 3, 3 * DELTA ** 2 * (t - 4.0 / 29.0))


def srgb_to_lab(rgb):
    """(3, ...) sRGB in [0, 255] -> (3, ...) L*, a*, b*."""
    lin = srgb_to_linear(rgb)
    xyz = np.tensordot(rgb_to_xyz_matrix(), lin, axes=([1], [0]))
    w = white()
    fx, fy, fz = (_f(xyz[i] / w[i]) for i in range(3))
    return np.stack([116.0 * fy - 16.0, 500.0 * (fx - fy), 200.0 * (fy - fz)])


def lab_to_srgb(lab):
    """Inverse of srgb_to_lab (no clipping)."""
    lab = np.asarray(lab, dtype=np.float64)
    fy = (lab[0] + 16.0) / 116.0
    fx = fy + lab[1] / 500.0
    fz = fy - lab[2] / 200.0
    w = white()
    xyz = np.stack([w[0] * _finv(fx), w[1] * _finv(fy), w[2] * _finv(fz)])
    lin = np.tensordot(np.linalg.inv(rgb_to_xyz_matrix()), xyz, axes=([1], [0]))
    return linear_to_srgb(lin)
