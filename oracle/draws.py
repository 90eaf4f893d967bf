"""Monte Carlo draws for the oracle (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

PAPER.md:109-117 (Prop. 2): X_k ~ B(N, 1/2) independent
(Eq. (13)-(14)): T draws X^(1..T), Y^(t) = N - 2 X^(t). The paper does not name
a generator (reading R9 in DESIGN.md): word w of the stream is the raw output
of Philox4x64-10 (Salmon et al., SC'11) with key (seed, 0), counter starting
at 1 -- exactly numpy's ``Philox(key=seed).random_raw()``, a library routine
pinned to the Random123 known-answer vectors in tests/golden/. A binomial
B(N, 1/2) variate is the number of set bits among the low N bits of one word
(a sum of N fair Bernoulli bits). Draw (t, k) uses word t*d + k.
"""
import math

import numpy as np


def philox_words(seed: int, n: int) -> np.ndarray:
    """First n raw 64-bit words of Philox4x64-10 with key (seed, 0)."""
    return np.random.Philox(key=int(seed)).random_raw(int(n)).astype(np.uint64)


def binomial_draws(seed: int, T: int, d: int, N: int) -> np.ndarray:
    """X (T, d) int64: X[t, k] = popcount(word[t*d + k] & (2^N - 1))."""
    if not (1 <= N <= 64):
        raise ValueError("N must be in [1, 64]")
    words = philox_words(seed, T * d)
    mask = np.uint64((1 << N) - 1) if N < 64 else np.uint64(0xFFFFFFFFFFFFFFFF)
    X = np.array([bin(int(wd & mask)).count("1") for wd in words], dtype=np.int64)
    return X.reshape(T, d)


def y_draws(seed: int, T: int, d: int, N: int) -> np.ndarray:
    """Y (T, d) = N - 2X."""
    return N - 2 * binomial_draws(seed, T, d, N)


def philox_words_key(seed: int, key1: int, n: int) -> np.ndarray:
    """First n raw words of Philox4x64-10 with key (seed, key1) (numpy's 128-bit key
    seed + key1 * 2^64)."""
    return np.random.Philox(key=int(seed) + (int(key1) << 64)).random_raw(int(n)).astype(np.uint64)


def binomial_cdf_table(N: int) -> np.ndarray:
    """cdf(n) = sum_{m <= n} C(N, m) 2^-N for n < N, as fp64 (exact integers, one rounding)."""
    cum, out = 0, []
    for n in range(N):
        cum += math.comb(N, n)
        out.append(np.float64(cum) * np.float64(2.0) ** -N)
    return np.array(out, dtype=np.float64)


def stratified_binomial_draws(seed: int, M: int, d: int, N: int) -> np.ndarray:
    """Stratified X (M, d) (reading R17; "improving the Monte Carlo integration"):
    per dimension c, sample k takes stratum pi_c(k) of M equal strata of [0, 1) -- pi_c(k) the
    rank of word (k d + c) of key (seed, 1) among dimension c's M words, ties by k -- and
    u = (pi_c(k) + (word (k d + c) of key (seed, 2) >> 11) 2^-53) / M, X = F^-1(u) the
    B(N, 1/2) quantile: min{n < N : u < cdf(n)}, else N."""
    keys = philox_words_key(seed, 1, M * d).reshape(M, d)
    v = philox_words_key(seed, 2, M * d).reshape(M, d)
    rank = np.empty((M, d), dtype=np.int64)
    for c in range(d):
        order = np.argsort(keys[:, c], kind="stable")
        rank[order, c] = np.arange(M)
    u = (rank.astype(np.float64) + (v >> np.uint64(11)).astype(np.float64) * 2.0 ** -53) / np.float64(M)
    cdf = binomial_cdf_table(N)
    return np.searchsorted(cdf, u, side="right").astype(np.int64)


def stratified_y_draws(seed: int, M: int, d: int, N: int) -> np.ndarray:
    return N - 2 * stratified_binomial_draws(seed, M, d, N)
