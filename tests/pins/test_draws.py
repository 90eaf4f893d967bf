"""Pins for oracle/draws.py: Philox known answers (library routine vs published
vectors) and the binomial law of the popcount sampler (Prop. 2)."""
import math

import numpy as np
import pytest
from scipy import stats

from oracle import draws
from tests.conftest import golden_lines


def _numpy_philox_block(ctr, key):
    # numpy pre-increments the 256-bit counter before each block, so start one below.
    c = list(ctr)
    for i in range(4):
        if c[i] > 0:
            c[i] -= 1
            break
        c[i] = (1 << 64) - 1
    g = np.random.Philox(counter=c, key=list(key))
    return [int(v) for v in g.random_raw(4)]


def test_philox_known_answers():
    lines = golden_lines("philox4x64_10_kat.txt")
    assert len(lines) >= 2
    for ln in lines:
        h = [int(x, 16) for x in ln.split()]
        ctr, key, want = h[0:4], h[4:6], h[6:10]
        assert _numpy_philox_block(ctr, key) == want


def test_stream_is_counter_from_one():
    # word w = lane w%4 of block counter (w//4 + 1, 0, 0, 0), key (seed, 0)  (reading R9)
    seed = 1234
    words = draws.philox_words(seed, 12)
    for blk in range(3):
        g = np.random.Philox(counter=[blk, 0, 0, 0], key=[seed, 0])
        assert [int(v) for v in g.random_raw(4)] == [int(v) for v in words[4 * blk:4 * blk + 4]]


def test_binomial_draws_popcount_definition():
    seed, T, d, N = 5, 7, 3, 20
    X = draws.binomial_draws(seed, T, d, N)
    words = draws.philox_words(seed, T * d)
    for t in range(T):
        for k in range(d):
            assert X[t, k] == bin(int(words[t * d + k]) & ((1 << N) - 1)).count("1")
    Y = draws.y_draws(seed, T, d, N)
    assert np.array_equal(Y, N - 2 * X)
    assert np.all((Y - N) % 2 == 0) and np.all(np.abs(Y) <= N)


@pytest.mark.parametrize("N", [2, 10, 20, 40])
def test_binomial_law_chi_square(N):
    n = 60000
    X = draws.binomial_draws(99 + N, n, 1, N).ravel()
    pmf = np.array([math.comb(N, k) for k in range(N + 1)]) / 2.0 ** N
    obs = np.bincount(X, minlength=N + 1).astype(float)
    exp = n * pmf
    keep = exp >= 5                       # pool sparse tails
    o = np.append(obs[keep], obs[~keep].sum())
    e = np.append(exp[keep], exp[~keep].sum())
    if e[-1] == 0:
        o, e = o[:-1], e[:-1]
    chi2 = ((o - e) ** 2 / e).sum()
    assert stats.chi2.sf(chi2, len(o) - 1) > 1e-4
    assert abs(X.mean() - N / 2) < 5 * math.sqrt(N / 4 / n)
    assert abs(X.var() - N / 4) < 0.05 * N / 4
    Y = N - 2 * X
    assert abs(Y.mean()) < 5 * math.sqrt(N / n)


def test_determinism():
    a = draws.y_draws(3, 64, 8, 30)
    b = draws.y_draws(3, 64, 8, 30)
    assert np.array_equal(a, b)
    assert not np.array_equal(a, draws.y_draws(4, 64, 8, 30))


# ---- stratified draws (reading R17) ------------------------------------------------------------
def test_stratified_reproduces_the_pmf_exactly_when_strata_align():
    """M = 2^N strata: every CDF breakpoint cum(n)/2^N is a stratum edge, so each stratum maps to
    one value and the counts are exactly C(N, n) (the binomial pmf times M)."""
    import math
    for N, d, seed in [(4, 2, 0), (6, 3, 1), (8, 1, 2)]:
        X = draws.stratified_binomial_draws(seed, 2 ** N, d, N)
        for c in range(d):
            assert list(np.bincount(X[:, c], minlength=N + 1)) == [math.comb(N, n) for n in range(N + 1)]


def test_stratified_counts_within_one_of_expected_and_strata_are_a_permutation():
    import math
    N, M, d = 40, 512, 3
    X = draws.stratified_binomial_draws(4, M, d, N)
    pmf = np.array([math.comb(N, n) for n in range(N + 1)], dtype=np.float64) / 2.0 ** N
    for c in range(d):
        counts = np.bincount(X[:, c], minlength=N + 1)
        # stratum j holds u in [j/M, (j+1)/M): the count of value n is the number of strata
        # meeting [cdf(n-1), cdf(n)), i.e. M pmf(n) rounded either way (+-1 at each edge)
        assert np.all(np.abs(counts - M * pmf) <= 2.0)
    keys = draws.philox_words_key(4, 1, M * d).reshape(M, d)
    for c in range(d):
        assert len(set(keys[:, c].tolist())) == M          # distinct keys: ranks are a permutation


def test_stratified_marginal_is_binomial_over_seeds():
    """Averaged over realisations, each sample is B(N, 1/2): chi^2 of the pooled draws of one
    sample index against the pmf."""
    import math
    N, M = 10, 8
    X = np.array([draws.stratified_binomial_draws(s, M, 1, N)[3, 0] for s in range(4000)])
    pmf = np.array([math.comb(N, n) for n in range(N + 1)]) / 2.0 ** N
    obs = np.bincount(X, minlength=N + 1)
    exp = 4000 * pmf
    keep = exp >= 5
    chi2 = (((obs - exp) ** 2 / exp)[keep]).sum() + ((obs[~keep].sum() - exp[~keep].sum()) ** 2 / exp[~keep].sum())
    assert chi2 < 30.0, chi2             # ~10 dof; 30 is p < 0.001
