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
