"""Pins for the oracle filters: O1 (numpy brute force, Eq. (5)-(6) with Eq. (14)),
O2 (C, Algorithm 1) and O3 (C, exact Eq. (2)-(3)).

What pins them (none of these re-types the function under test):
  * keystone: O2 (separable, Alg. 1) == O1 (windowed definition), an exact
    rearrangement (Eq. (15)-(19));
  * Prop. 2 transfer: feeding O1/O2 every outcome of X in proportion to its
    binomial probability gives the raised-cosine filter (Eq. (9)) exactly;
  * Prop. 1: raised-cosine filter -> exact Gaussian filter as N grows;
  * special cases: constant image, C -> infinity and Y = 0 (pure Gaussian blur,
    compared with scipy.ndimage.correlate1d mode='reflect'), translation and
    flip equivariance, range containment, d = 1 scalar bilateral by hand.
"""
import itertools
import math

import numpy as np
import pytest
from scipy import ndimage

from oracle import draws, filters, kernels, native, plan
from workloads.configs import random_image


def _blur(f, sigma_s):
    """Truncated normalised Gaussian blur via scipy (library routine), reflect boundary."""
    w = plan.spatial_taps(sigma_s)
    out = ndimage.correlate1d(f.astype(np.float64), w, axis=1, mode="reflect")
    return ndimage.correlate1d(out, w, axis=2, mode="reflect")


def _random_spd(d, scale, seed):
    rng = np.random.default_rng(seed)
    A = rng.normal(size=(d, d))
    return scale ** 2 * (A @ A.T / d + np.eye(d))


CASES = [  # (H, W, d, sigma_s, N, T, seed, diagonal)
    (12, 10, 1, 1.0, 4, 8, 0, True),
    (9, 14, 2, 1.5, 10, 16, 1, False),
    (16, 16, 3, 1.0, 10, 12, 2, True),
    (11, 13, 3, 2.0, 4, 5, 3, False),
    (5, 7, 3, 2.3, 20, 9, 4, False),      # window larger than the image: multi-fold reflection
    (3, 3, 2, 1.0, 6, 4, 5, True),
    (1, 8, 3, 1.0, 10, 3, 6, True),       # single row
]


@pytest.mark.parametrize("case", CASES)
def test_keystone_alg1_equals_windowed_definition(case):
    H, W, d, s, N, T, seed, diag = case
    f = random_image(H, W, d, seed=seed)
    C = np.diag(np.full(d, 40.0 ** 2)) if diag else _random_spd(d, 40.0, seed)
    Q, a = plan.diagonalize(C)
    Y = draws.y_draws(seed, T, d, N)
    S1, P1, Z1 = filters.mc_filter_bruteforce(f, Q, a, N, Y, s)
    S2, P2, Z2 = native.mcsf_full(f, Q, a, N, Y, s)
    np.testing.assert_allclose(Z2, Z1, atol=1e-10 * T)
    np.testing.assert_allclose(P2, P1, atol=1e-10 * T * 255)
    ok = np.abs(Z1) > 1e-3 * T
    assert np.abs(S2 - S1)[:, ok].max() < 1e-9


def test_pixel_evaluator_matches_full():
    H, W, d, s, N, T = 14, 11, 3, 1.5, 10, 7
    f = random_image(H, W, d, seed=11)
    C = _random_spd(d, 35.0, 11)
    Q, a = plan.diagonalize(C)
    Y = draws.y_draws(11, T, d, N)
    S, P, Z = filters.mc_filter_bruteforce(f, Q, a, N, Y, s)
    pix = [(0, 0), (13, 10), (5, 3), (0, 10), (7, 0)]
    Sp, Pp, Zp = filters.mc_filter_pixels(lambda y0, y1: f[:, y0:y1], H, W, pix, Q, a, N, Y, s)
    for n, (y, x) in enumerate(pix):
        assert abs(Zp[n] - Z[y, x]) < 1e-11
        np.testing.assert_allclose(Pp[n], P[:, y, x], atol=1e-9)


def _all_outcomes_Y(N, d):
    """Every outcome of X ~ B(N,1/2)^d repeated C(N,n1)...C(N,nd) times: the
    unweighted mean over this list IS the expectation of Eq. (10)."""
    one = [N - 2 * n for n in range(N + 1) for _ in range(math.comb(N, n))]
    return np.array(list(itertools.product(one, repeat=d)), dtype=np.int64)


@pytest.mark.parametrize("d,N", [(1, 4), (2, 2), (3, 2)])
def test_prop2_transfer_to_filter(d, N):
    f = random_image(8, 8, d, seed=d)
    C = np.diag(np.full(d, 30.0 ** 2)) if d != 2 else _random_spd(d, 30.0, 9)
    Q, a = plan.diagonalize(C)
    Y = _all_outcomes_Y(N, d)
    S_all, _, _ = native.mcsf_full(f, Q, a, N, Y, 1.0)
    S_rc, _, _ = filters.kernel_filter_bruteforce(f, Q, 1.0, lambda y: kernels.raised_cosine(y, a, N))
    np.testing.assert_allclose(S_all, S_rc, atol=1e-9)
    S_ex, _, _ = filters.kernel_filter_bruteforce(f, Q, 1.0, lambda y: kernels.exhaustive_kernel(y, a, N))
    np.testing.assert_allclose(S_ex, S_rc, atol=1e-9)


def test_prop1_filter_limit():
    f = random_image(10, 10, 3, seed=3)
    C = _random_spd(3, 60.0, 3)
    Q, a = plan.diagonalize(C)
    exact = filters.direct_bruteforce(f, C, 1.0)
    errs = []
    for N in (50, 200, 800):
        S, _, _ = filters.kernel_filter_bruteforce(f, Q, 1.0, lambda y: kernels.raised_cosine(y, a, N))
        errs.append(np.abs(S - exact).max())
    assert errs[0] > errs[1] > errs[2]
    assert errs[2] < 0.05


def test_constant_image_is_fixed_point():
    f = np.full((3, 9, 12), 77.25, dtype=np.float32)
    C = _random_spd(3, 40.0, 1)
    Q, a = plan.diagonalize(C)
    Y = draws.y_draws(1, 10, 3, 10)
    S, P, Z = native.mcsf_full(f, Q, a, 10, Y, 1.5)
    assert np.abs(S - 77.25).max() < 1e-12
    np.testing.assert_allclose(Z, 10.0, rtol=1e-14)        # z = T * sum(taps) * 1
    assert np.abs(native.direct_full(f, C, 1.5) - 77.25).max() < 1e-12
    S1, _, _ = filters.mc_filter_bruteforce(f, Q, a, 10, Y, 1.5)
    assert np.abs(S1 - 77.25).max() < 1e-12


def test_infinite_covariance_is_gaussian_blur():
    f = random_image(13, 17, 3, seed=4)
    C = np.diag(np.full(3, 1e12))
    Q, a = plan.diagonalize(C)
    Y = draws.y_draws(2, 6, 3, 10)
    S, _, _ = native.mcsf_full(f, Q, a, 10, Y, 2.0)
    np.testing.assert_allclose(S, _blur(f, 2.0), atol=1e-6)
    np.testing.assert_allclose(native.direct_full(f, C, 2.0), _blur(f, 2.0), atol=1e-6)


def test_zero_frequency_sample_is_gaussian_blur():
    f = random_image(11, 9, 2, seed=5)
    Q, a = plan.diagonalize(_random_spd(2, 20.0, 5))
    Y = np.zeros((1, 2), dtype=np.int64)
    S, _, Z = native.mcsf_full(f, Q, a, 10, Y, 1.0)
    np.testing.assert_allclose(S, _blur(f, 1.0), atol=1e-10)
    np.testing.assert_allclose(Z, 1.0, rtol=1e-14)


def test_translation_equivariance():
    f = np.round(random_image(10, 12, 3, seed=6) * 2) / np.float32(4)   # exact in fp32 after +c
    Q, a = plan.diagonalize(_random_spd(3, 40.0, 6))
    Y = draws.y_draws(6, 8, 3, 10)
    S0, _, Z0 = native.mcsf_full(f, Q, a, 10, Y, 1.0)
    c = np.array([100.0, -37.5, 64.0], dtype=np.float32)
    S1, _, _ = native.mcsf_full(f + c[:, None, None], Q, a, 10, Y, 1.0)
    ok = np.abs(Z0) > 0.05 * 8
    assert np.abs(S1 - S0 - c[:, None, None].astype(np.float64))[:, ok].max() < 1e-8


def test_flip_equivariance():
    f = random_image(9, 13, 3, seed=7)
    C = _random_spd(3, 40.0, 7)
    Q, a = plan.diagonalize(C)
    Y = draws.y_draws(7, 6, 3, 10)
    S0, _, _ = native.mcsf_full(f, Q, a, 10, Y, 1.5)
    S1, _, _ = native.mcsf_full(np.ascontiguousarray(f[:, :, ::-1]), Q, a, 10, Y, 1.5)
    np.testing.assert_allclose(S1[:, :, ::-1], S0, atol=1e-9)
    D0 = native.direct_full(f, C, 1.5)
    D1 = native.direct_full(np.ascontiguousarray(f[:, ::-1, :]), C, 1.5)
    np.testing.assert_allclose(D1[:, ::-1, :], D0, atol=1e-10)


def test_slab_band_equals_full():
    f = random_image(40, 16, 3, seed=8)
    Q, a = plan.diagonalize(np.diag([900.0] * 3))
    Y = draws.y_draws(8, 5, 3, 10)
    S, P, Z = native.mcsf_full(f, Q, a, 10, Y, 2.0)
    r = plan.radius(2.0)
    for (y0, n) in [(0, 5), (17, 6), (33, 7)]:
        s0, s1 = native.slab_bounds(40, y0, n, r)
        Sb, Pb, Zb = native.mcsf_alg1(f[:, s0:s1], 40, s0, y0, n, Q, a, 10, Y, 2.0)
        np.testing.assert_array_equal(Zb, Z[y0:y0 + n])
        np.testing.assert_array_equal(Pb, P[:, y0:y0 + n])
        Db = native.direct(f[:, s0:s1], 40, s0, y0, n, np.diag([900.0] * 3), 2.0)
        D = native.direct_full(f, np.diag([900.0] * 3), 2.0)
        np.testing.assert_array_equal(Db, D[:, y0:y0 + n])


def test_direct_scalar_bilateral_by_hand():
    H, W, s, sr = 7, 8, 1.0, 25.0
    f = random_image(H, W, 1, seed=9)
    out = native.direct_full(f, np.array([[sr * sr]]), s)
    r = plan.radius(s)
    for y in range(H):
        for x in range(W):
            num = den = 0.0
            for jy in range(-r, r + 1):
                for jx in range(-r, r + 1):
                    yy = int(filters.reflect(y - jy, H))
                    xx = int(filters.reflect(x - jx, W))
                    v = float(f[0, yy, xx])
                    wt = math.exp(-(jy * jy + jx * jx) / (2 * s * s)) * \
                        math.exp(-(v - float(f[0, y, x])) ** 2 / (2 * sr * sr))
                    num += wt * v
                    den += wt
            assert abs(out[0, y, x] - num / den) < 1e-10


def test_direct_range_containment_and_bruteforce():
    f = random_image(10, 11, 3, seed=10)
    C = _random_spd(3, 30.0, 10)
    D = native.direct_full(f, C, 1.5)
    for c in range(3):
        assert D[c].min() >= f[c].min() - 1e-9 and D[c].max() <= f[c].max() + 1e-9
    np.testing.assert_allclose(D, filters.direct_bruteforce(f, C, 1.5), atol=1e-10)


def test_reflect_boundary_definition():
    # half-sample reflection: -1 -> 0, n -> n-1, period 2n (reading R1)
    assert list(filters.reflect(np.arange(-4, 8), 3)) == [2, 2, 1, 0, 0, 1, 2, 2, 1, 0, 0, 1]
    assert list(filters.reflect(np.arange(-3, 4), 1)) == [0] * 7


def test_mc_converges_to_raised_cosine_filter():
    """Unbiasedness (Prop. 2 + Eq. (13)): mean of P and Z over independent seeds
    approaches the raised-cosine numerator/denominator at rate 1/sqrt(#draws)."""
    f = random_image(8, 8, 2, seed=12)
    Q, a = plan.diagonalize(np.diag([50.0 ** 2] * 2))
    N, T, n_seeds = 10, 50, 40
    _, Prc, Zrc = filters.kernel_filter_bruteforce(f, Q, 1.0, lambda y: kernels.raised_cosine(y, a, N))
    Zs = []
    for sd in range(n_seeds):
        Y = draws.y_draws(1000 + sd, T, 2, N)
        _, P, Z = native.mcsf_full(f, Q, a, N, Y, 1.0)
        Zs.append(Z / T)
    Zm = np.mean(Zs, axis=0)
    se = np.std(Zs, axis=0) / math.sqrt(n_seeds)
    assert np.all(np.abs(Zm - Zrc) < 5 * se + 1e-12)
