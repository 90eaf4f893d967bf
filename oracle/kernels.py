"""Range-kernel identities of Section 2 (TEST INFRASTRUCTURE ONLY).

Eq. (7)  psi(y) = prod_k exp(-alpha_k^2 y_k^2 / 2)
Eq. (9) psi(y) ~ prod_k cos(alpha_k y_k / sqrt(N))^N     (Prop. 1)
Eq. (11) cos^N(theta) = sum_n 2^-N C(N,n) exp(iota (N-2n) theta)
Eq. (10) psi(y) = E prod_k exp(iota (N - 2X_k) gamma_k y_k)
Eq. (14) MC estimate (1/T) sum_t prod_k exp(iota Y_k^(t) gamma_k y_k)
"""
import itertools
import math

import numpy as np


def gaussian_range(y, alpha):
    """Eq. (7): product of 1-D Gaussians in the rotated coordinates."""
    y = np.asarray(y, dtype=np.float64)
    a = np.asarray(alpha, dtype=np.float64)
    return np.exp(-0.5 * np.sum((a * y) ** 2, axis=-1))


def raised_cosine(y, alpha, N):
    """Eq. (9): prod_k [cos(alpha_k y_k / sqrt(N))]^N."""
    y = np.asarray(y, dtype=np.float64)
    a = np.asarray(alpha, dtype=np.float64)
    return np.prod(np.cos(a * y / math.sqrt(N)) ** N, axis=-1)


def binomial_pmf(N):
    """P(X = n) for X ~ B(N, 1/2): 2^-N C(N, n)."""
    return np.array([math.comb(N, n) for n in range(N + 1)], dtype=np.float64) / 2.0 ** N


def cosN_binomial_expectation(theta, N):
    """Eq. (11): sum_n 2^-N C(N,n) exp(iota (N-2n) theta), complex."""
    theta = np.asarray(theta, dtype=np.float64)
    p = binomial_pmf(N)
    n = np.arange(N + 1)
    return np.sum(p * np.exp(1j * (N - 2 * n) * theta[..., None]), axis=-1)


def exhaustive_kernel(y, alpha, N):
    """Eq. (10) evaluated exactly: all (N+1)^d outcomes of X weighted by the
    product binomial pmf (independent components)."""
    y = np.asarray(y, dtype=np.float64)
    a = np.asarray(alpha, dtype=np.float64)
    d = a.shape[0]
    g = a / math.sqrt(N)
    p = binomial_pmf(N)
    acc = np.zeros(y.shape[:-1], dtype=np.complex128)
    for xs in itertools.product(range(N + 1), repeat=d):
        wgt = np.prod([p[x] for x in xs])
        Yv = N - 2 * np.array(xs)
        acc = acc + wgt * np.exp(1j * np.sum(Yv * g * y, axis=-1))
    return acc


def sampled_kernel(y, Y, gamma):
    """Eq. (14): (1/T) sum_t prod_k exp(iota Y_k^(t) gamma_k y_k), complex."""
    y = np.asarray(y, dtype=np.float64)
    Y = np.asarray(Y, dtype=np.float64)
    g = np.asarray(gamma, dtype=np.float64)
    ph = np.tensordot(y, (Y * g).T, axes=([-1], [0]))          # (..., T)
    return np.mean(np.exp(1j * ph), axis=-1)
