"""Brute-force windowed filters (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

These evaluate the filter by its plain definition, summing over the window
j in [-r, r]^2 with half-sample symmetric reflection at the
image border (reading R1):

  O1  mc_filter_bruteforce / mc_filter_pixels: Eq. (5)-(6)
      with psi replaced by Eq. (14), taking real parts of
      the numerator and denominator before dividing (reading R4). The common
      1/T factor cancels and is omitted (reading R13).
  kernel_filter_bruteforce: Eq. (5)-(6) with any range kernel psi of the
      rotated difference g(i-j) - g(i) (used with Eq. (7), (9), (10)).
  direct_bruteforce: Eq. (2)-(3) with phi of Eq. (1).
"""
import numpy as np

from . import plan as _plan


def reflect(i, n):
    """Half-sample symmetric reflection into [0, n), period 2n (reading R1)."""
    i = np.asarray(i)
    p = 2 * n
    i = np.mod(i, p)
    return np.where(i < n, i, p - 1 - i)


def _shift(img, jy, jx):
    """img(rho(i - j)) for all pixels i: planar (c, H, W) -> (c, H, W)."""
    _, H, W = img.shape
    ys = reflect(np.arange(H) - jy, H)
    xs = reflect(np.arange(W) - jx, W)
    return img[:, ys][:, :, xs]


def _rotate(f, Q):
    """g(i) = Q^T f(i)."""
    return np.einsum("ck,chw->khw", np.asarray(Q, dtype=np.float64), f.astype(np.float64))


def mc_filter_bruteforce(f, Q, alpha, N, Y, sigma_s, spatial="gaussian"):
    """O1 over the whole image. Returns (S, P, Z): S (d,H,W), P (d,H,W), Z (H,W)."""
    f64 = np.asarray(f, dtype=np.float64)
    d, H, W = f64.shape
    w = _plan.spatial_window(sigma_s, spatial)
    r = (len(w) - 1) // 2
    g = _rotate(f64, Q)
    Yg = np.asarray(Y, dtype=np.float64) * _plan.gammas(alpha, N)[None, :]   # (T, d)
    P = np.zeros((d, H, W))
    Z = np.zeros((H, W))
    for jy in range(-r, r + 1):
        for jx in range(-r, r + 1):
            om = w[jy + r] * w[jx + r]
            fj = _shift(f64, jy, jx)
            dg = _shift(g, jy, jx) - g                                        # g(i-j) - g(i)
            # Re sum_t prod_k exp(iota Y_k gamma_k dg_k) = sum_t cos(sum_k Y_k gamma_k dg_k)
            psi = np.cos(np.tensordot(Yg, dg, axes=([1], [0]))).sum(axis=0)   # (H, W)
            Z += om * psi
            P += om * psi[None] * fj
    return P / Z[None], P, Z


def mc_filter_pixels(get_rows, H, W, pixels, Q, alpha, N, Y, sigma_s, spatial="gaussian"):
    """O1 at selected pixels of an image of any size.

    get_rows(y0, y1) must return planar rows [y0, y1) of the full image.
    pixels: iterable of (y, x). Returns (S (n,d), P (n,d), Z (n,))."""
    w = _plan.spatial_window(sigma_s, spatial)
    r = (len(w) - 1) // 2
    om = np.outer(w, w)                                                       # (2r+1, 2r+1)
    Yg = np.asarray(Y, dtype=np.float64) * _plan.gammas(alpha, N)[None, :]
    Q = np.asarray(Q, dtype=np.float64)
    out_S, out_P, out_Z = [], [], []
    cache = {}
    for (y, x) in pixels:
        ys = reflect(np.arange(y + r, y - r - 1, -1), H)      # rho(y - jy), jy = -r..r
        xs = reflect(np.arange(x + r, x - r - 1, -1), W)
        y0, y1 = int(ys.min()), int(ys.max()) + 1
        key = (y0, y1)
        if key not in cache:
            cache.clear()
            cache[key] = np.asarray(get_rows(y0, y1), dtype=np.float64)
        rows = cache[key]
        fw = rows[:, ys - y0][:, :, xs]                                       # (d, 2r+1, 2r+1)
        fi = rows[:, y - y0, x]
        dg = np.einsum("ck,cab->kab", Q, fw - fi[:, None, None])              # Q^T (f(i-j) - f(i))
        psi = np.cos(np.tensordot(Yg, dg, axes=([1], [0]))).sum(axis=0)
        Zp = np.sum(om * psi)
        Pp = np.einsum("ab,cab->c", om * psi, fw)
        out_S.append(Pp / Zp)
        out_P.append(Pp)
        out_Z.append(Zp)
    return np.array(out_S), np.array(out_P), np.array(out_Z)


def kernel_filter_bruteforce(f, Q, sigma_s, psi_fn, spatial="gaussian"):
    """Eq. (5)-(6) with range kernel psi_fn(dg) where dg has shape (H, W, d).
    psi_fn may return complex values; real parts are taken (reading R4)."""
    f64 = np.asarray(f, dtype=np.float64)
    d, H, W = f64.shape
    w = _plan.spatial_window(sigma_s, spatial)
    r = (len(w) - 1) // 2
    g = _rotate(f64, Q)
    P = np.zeros((d, H, W))
    Z = np.zeros((H, W))
    for jy in range(-r, r + 1):
        for jx in range(-r, r + 1):
            om = w[jy + r] * w[jx + r]
            dg = np.moveaxis(_shift(g, jy, jx) - g, 0, -1)
            psi = np.real(psi_fn(dg))
            Z += om * psi
            P += om * psi[None] * _shift(f64, jy, jx)
    return P / Z[None], P, Z


def direct_bruteforce(f, C, sigma_s, spatial="gaussian"):
    """Eq. (2)-(3): phi(x) = exp(-x^T C^-1 x / 2) on x = f(i-j) - f(i)."""
    f64 = np.asarray(f, dtype=np.float64)
    d, H, W = f64.shape
    w = _plan.spatial_window(sigma_s, spatial)
    r = (len(w) - 1) // 2
    Cinv = np.linalg.inv(np.asarray(C, dtype=np.float64))
    num = np.zeros((d, H, W))
    den = np.zeros((H, W))
    for jy in range(-r, r + 1):
        for jx in range(-r, r + 1):
            fj = _shift(f64, jy, jx)
            x = fj - f64
            q = np.einsum("ahw,ab,bhw->hw", x, Cinv, x)
            wt = w[jy + r] * w[jx + r] * np.exp(-0.5 * q)
            den += wt
            num += wt[None] * fj
    return num / den[None]
