"""Pins for the recursive (O(1)-in-sigma_s) engine's spatial kernel (PAPER.md:204,
"we can efficiently compute the Gaussian convolutions in step 10 using separability and
recursion ... at O(1) cost with respect to sigma_s [Deriche 1993]"; reading R16).

The oracle writes that kernel out as plain taps (oracle.plan.deriche_window) and convolves
with them directly (O1 / O2 with spatial="deriche"). What pins it:
  * the constants: Deriche's h(x) must reproduce the closed-form Gaussian it approximates
    (normalised, max deviation <= 1e-3 of the peak for sigma_s from 1 to 50) and its sum
    must match sigma_s sqrt(2 pi) -- a misprinted constant fails both;
  * normalisation, symmetry and the 1e-17 tail bound of the truncation;
  * C -> infinity: MCSF with the Deriche kernel reduces to the separable blur, checked
    against an FFT circular convolution of the even (reflected) extension -- a library
    route independent of the oracle's reflected-index sums;
  * the keystone (Alg. 1 separable form == windowed definition) with this kernel;
  * the recursion the GPU runs: a test-local fp64 implementation of the complex
    first-order recursions with the closed-form reflected-periodic initial state equals
    the direct convolution with the taps (this pins the derivation in DESIGN.md §11,
    not the oracle).
"""
import cmath
import math

import numpy as np
import pytest

from oracle import draws, filters, native, plan
from workloads.configs import random_image

D = plan.DERICHE


@pytest.mark.parametrize("sigma_s", [1.0, 2.0, 5.0, 16.0, 50.0])
def test_deriche_reproduces_the_gaussian(sigma_s):
    L = plan.deriche_radius(sigma_s)
    m = np.arange(-L, L + 1)
    g = plan.deriche_window(sigma_s)
    gauss = np.exp(-m * m / (2 * sigma_s ** 2))
    gauss /= gauss.sum()
    assert np.abs(g - gauss).max() <= 1e-3 * gauss.max()
    h = plan.deriche_h(np.abs(m), sigma_s)
    assert abs(h.sum() / (sigma_s * math.sqrt(2 * math.pi)) - 1.0) < 5e-4


@pytest.mark.parametrize("sigma_s", [0.7, 3.0, 16.0])
def test_window_normalised_symmetric_and_tail_negligible(sigma_s):
    g = plan.deriche_window(sigma_s)
    L = (len(g) - 1) // 2
    assert abs(g.sum() - 1.0) < 1e-14
    np.testing.assert_array_equal(g, g[::-1])
    assert abs(plan.deriche_h(L, sigma_s)) < 1e-17
    assert abs(plan.deriche_h(0.0, sigma_s) - (D["a0"] + D["c0"])) < 1e-15


def _fft_reflect_blur_1d(x, g):
    """Convolution of the half-sample-reflected periodic extension of x (period 2n) with the
    symmetric taps g, via numpy's FFT on one period of the even extension."""
    n = len(x)
    ext = np.concatenate([x, x[::-1]])
    L = (len(g) - 1) // 2
    ker = np.zeros(2 * n)
    for m in range(-L, L + 1):
        ker[m % (2 * n)] += g[m + L]
    return np.real(np.fft.ifft(np.fft.fft(ext) * np.fft.fft(ker)))[:n]


@pytest.mark.parametrize("H,W,sigma_s", [(11, 13, 1.0), (6, 9, 2.5), (30, 4, 1.5)])
def test_c_to_infinity_is_the_recursive_gaussian_blur(H, W, sigma_s):
    d, N, T = 3, 10, 3
    f = random_image(H, W, d, seed=7)
    g = plan.deriche_window(sigma_s)
    ref = np.apply_along_axis(_fft_reflect_blur_1d, 1, f.astype(np.float64), g)
    ref = np.apply_along_axis(_fft_reflect_blur_1d, 2, ref, g)
    Q, a = plan.diagonalize(np.eye(d) * 1e16)
    S, P, Z = native.mcsf_full(f, Q, a, N, draws.y_draws(1, T, d, N), sigma_s, spatial="deriche")
    np.testing.assert_allclose(S, ref, atol=1e-8)
    np.testing.assert_allclose(Z, T, atol=1e-9)


@pytest.mark.parametrize("case", [(7, 9, 3, 1.0, 10, 4, 0), (1, 12, 2, 0.8, 20, 3, 1)])
def test_keystone_with_recursive_kernel(case):
    H, W, d, s, N, T, seed = case
    f = random_image(H, W, d, seed=seed)
    Q, a = plan.diagonalize(np.diag(np.full(d, 40.0 ** 2)))
    Y = draws.y_draws(seed, T, d, N)
    S1, P1, Z1 = filters.mc_filter_bruteforce(f, Q, a, N, Y, s, spatial="deriche")
    S2, P2, Z2 = native.mcsf_full(f, Q, a, N, Y, s, spatial="deriche")
    np.testing.assert_allclose(Z2, Z1, atol=1e-10 * T)
    np.testing.assert_allclose(P2, P1, atol=1e-10 * T * 255)


# ---- the recursion the GPU implements (test-local reference of DESIGN.md §11) --------------
def _poles(sigma_s):
    z = [cmath.exp(complex(-D["b0"], D["w0"]) / sigma_s), cmath.exp(complex(-D["b1"], D["w1"]) / sigma_s)]
    A = [complex(D["a0"], -D["a1"]), complex(D["c0"], -D["c1"])]
    # sum over all integers m of h(|m|) = 2 Re sum_j A_j / (1 - z_j) - h(0)
    S = 2 * sum(Aj / (1 - zj) for Aj, zj in zip(A, z)).real - (D["a0"] + D["c0"])
    A = [Aj / S for Aj in A]
    return z, A, (D["a0"] + D["c0"]) / S


def _recursive_1d(x, sigma_s):
    """y[k] = sum_j Re[A_j (u_j[k] + v_j[k])] - g0 x[k]; u_j[k] = x[k] + z_j u_j[k-1],
    v_j[k] = x[k] + z_j v_j[k+1]; reflected-periodic initial state
    u[-1] = (S_head + z^n S_tail) / (1 - z^2n), v[n] = u[n-1]."""
    z, A, g0 = _poles(sigma_s)
    n = len(x)
    y = -g0 * np.asarray(x, dtype=np.float64)
    for zj, Aj in zip(z, A):
        s_head = sum(zj ** m * x[m] for m in range(n))
        s_tail = sum(zj ** (n - 1 - m) * x[m] for m in range(n))
        u = (s_head + zj ** n * s_tail) / (1 - zj ** (2 * n))
        us = []
        for k in range(n):
            u = x[k] + zj * u
            us.append(u)
        v = us[-1]                                   # v[n] = u[n-1]
        for k in range(n - 1, -1, -1):
            v = x[k] + zj * v
            y[k] += (Aj * (us[k] + v)).real
    return y


@pytest.mark.parametrize("n,sigma_s", [(1, 1.0), (2, 3.0), (5, 2.0), (17, 1.3), (64, 4.0), (200, 16.0)])
def test_recursion_with_closed_form_init_equals_direct_convolution(n, sigma_s):
    x = np.random.default_rng(n).uniform(-128, 128, n)
    np.testing.assert_allclose(_recursive_1d(x, sigma_s), _fft_reflect_blur_1d(x, plan.deriche_window(sigma_s)),
                               atol=1e-9)
