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
