"""Setup steps of Algorithm 1 for the oracle (TEST INFRASTRUCTURE ONLY).

Alg. 1: diagonalise C -> Q, alpha  (Eq. (4))
Alg. 1: spatial filter omega        (Eq. (1))
Alg. 1:            gamma_k = alpha_k / sqrt(N)
"""
import math

import numpy as np


def radius(sigma_s: float) -> int:
    """Window half-width: [-3 sigma_s, 3 sigma_s]^2, ceiling (reading R2)."""
    return int(math.ceil(3.0 * float(sigma_s) - 1e-12))


def spatial_taps(sigma_s: float) -> np.ndarray:
    """1-D taps w(m) = exp(-m^2 / 2 sigma_s^2), m in [-r, r], normalised to sum 1.

    omega(j) = w(j_y) w(j_x) is Eq. (1)'s exp(-||j||^2 / 2 sigma_s^2) up to a
    constant factor, which cancels in the filter (reading R3)."""
    r = radius(sigma_s)
    m = np.arange(-r, r + 1, dtype=np.float64)
    w = np.exp(-(m * m) / (2.0 * float(sigma_s) ** 2))
    return w / w.sum()


def spatial_window(sigma_s: float, kind: str = "gaussian") -> np.ndarray:
    """1-D taps w(m), m in [-r, r], normalised to sum 1, for the separable spatial kernel
    omega(j) = w(j_y) w(j_x).

    gaussian: Eq. (1) on r = ceil(3 sigma_s) (``spatial_taps``).
    box, hat: "replace the spatial filter ... with any arbitrary spatial filter
    (such as a box or hat filter)"; reading R15 keeps the window r = ceil(3 sigma_s):
    box w(m) = 1, hat w(m) = r + 1 - |m|.
    deriche: the recursive engine's kernel (``deriche_window``, reading R16)."""
    if kind == "gaussian":
        return spatial_taps(sigma_s)
    if kind == "deriche":
        return deriche_window(sigma_s)
    r = radius(sigma_s)
    m = np.arange(-r, r + 1, dtype=np.float64)
    if kind == "box":
        w = np.ones_like(m)
    elif kind == "hat":
        w = (r + 1) - np.abs(m)
    else:
        raise ValueError(f"unknown spatial kernel {kind!r}")
    return w / w.sum()


SPATIAL_KINDS = {"gaussian": 0, "box": 1, "hat": 2}

# Deriche's 4th-order recursive approximation of the Gaussian (PAPER.md:204 cites
# Deriche 1993 for the O(1)-in-sigma_s convolutions of Alg. 1 step 10):
# h(x) = (a0 cos(w0 x/s) + a1 sin(w0 x/s)) e^{-b0 x/s} + (c0 cos(w1 x/s) + c1 sin(w1 x/s)) e^{-b1 x/s},
# x >= 0, the published smoothing-filter constants (reading R16).
DERICHE = {"a0": 1.68, "a1": 3.735, "b0": 1.783, "b1": 1.723,
           "c0": -0.6803, "c1": -0.2598, "w0": 0.6318, "w1": 1.997}


def deriche_h(x, sigma_s: float) -> np.ndarray:
    """Deriche's causal impulse response h(x), x >= 0 (unnormalised, h(0) = a0 + c0)."""
    D = DERICHE
    x = np.asarray(x, dtype=np.float64) / float(sigma_s)
    return ((D["a0"] * np.cos(D["w0"] * x) + D["a1"] * np.sin(D["w0"] * x)) * np.exp(-D["b0"] * x)
            + (D["c0"] * np.cos(D["w1"] * x) + D["c1"] * np.sin(D["w1"] * x)) * np.exp(-D["b1"] * x))


def deriche_radius(sigma_s: float) -> int:
    """Support at which the tail is below 1e-17 of the peak: |h(x)| <= (|a0|+|a1|) e^{-b0 x/s}
    + (|c0|+|c1|) e^{-b1 x/s} <= sum|.| e^{-min(b) x/s}."""
    D = DERICHE
    amp = abs(D["a0"]) + abs(D["a1"]) + abs(D["c0"]) + abs(D["c1"])
    return int(math.ceil(float(sigma_s) * math.log(amp / 1e-17) / min(D["b0"], D["b1"])))


def deriche_window(sigma_s: float) -> np.ndarray:
    """The symmetric recursive-Gaussian kernel g(m) = h(|m|) / sum, m in [-L, L] (L = deriche_radius):
    the spatial filter the recursive engine applies (reading R16), written out as plain taps."""
    L = deriche_radius(sigma_s)
    g = deriche_h(np.abs(np.arange(-L, L + 1)), sigma_s)
    return g / g.sum()


def diagonalize(C):
    """Q (orthogonal, columns q_k) and alpha (> 0) with x^T C^-1 x = sum_k alpha_k^2 y_k^2,
    y = Q^T x (Eq. (4)).

    Canonical choice (paper silent, reading R8): diagonal C -> Q = I,
    alpha_k = C_kk^-1/2 with no reordering; otherwise numpy ``eigh`` eigenvectors
    sorted by alpha descending (C-eigenvalues ascending) and each column signed
    so its first component with |q| > 1e-6 max|q| is positive."""
    C = np.asarray(C, dtype=np.float64)
    d = C.shape[0]
    if C.shape != (d, d):
        raise ValueError("C must be square")
    if np.max(np.abs(C - C.T)) > 1e-12 * max(1.0, np.max(np.abs(C))):
        raise ValueError("C not symmetric")
    off = C - np.diag(np.diag(C))
    if not np.any(off):
        lam = np.diag(C).copy()
        if np.any(lam <= 1e-12 * lam.max()):
            raise ValueError("C not positive definite")
        return np.eye(d), 1.0 / np.sqrt(lam)
    lam, V = np.linalg.eigh(C)
    if np.any(lam <= 1e-12 * lam.max()):
        raise ValueError("C not positive definite")
    order = np.argsort(lam, kind="stable")          # ascending eigenvalue = alpha descending
    lam, V = lam[order], V[:, order]
    for k in range(d):
        col = V[:, k]
        thr = 1e-6 * np.max(np.abs(col))
        first = np.nonzero(np.abs(col) > thr)[0][0]
        if col[first] < 0:
            V[:, k] = -col
    return V, 1.0 / np.sqrt(lam)


def gammas(alpha, N: int) -> np.ndarray:
    """gamma_k = alpha_k / sqrt(N) (Alg. 1)."""
    return np.asarray(alpha, dtype=np.float64) / math.sqrt(N)
