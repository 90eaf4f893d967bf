"""Pins for oracle/kernels.py: Prop. 1, Prop. 2 / Eq. (10)-(12)
(PAPER.md:109-132), Fig. 1 regime."""
import math

import numpy as np
import pytest

from oracle import kernels


def test_prop2_scalar_identity():
    th = np.linspace(-math.pi, math.pi, 1001)
    for N in range(1, 13):
        v = kernels.cosN_binomial_expectation(th, N)
        np.testing.assert_allclose(v.real, np.cos(th) ** N, atol=1e-12)
        assert np.abs(v.imag).max() < 1e-12        # symmetric pmf: imaginary parts cancel


def test_prop2_worked_value():
    # theta = pi/3, N = 2: 1/4 cos(2pi/3) + 1/2 + 1/4 cos(-2pi/3) = 1/4 = cos^2(pi/3)
    assert abs(kernels.cosN_binomial_expectation(np.array(math.pi / 3), 2).real - 0.25) < 1e-15


@pytest.mark.parametrize("d,N", [(1, 6), (2, 4), (3, 2)])
def test_prop2_multivariate_exhaustive(d, N):
    rng = np.random.default_rng(d)
    alpha = rng.uniform(0.01, 0.05, size=d)
    y = rng.uniform(-200, 200, size=(50, d))
    ex = kernels.exhaustive_kernel(y, alpha, N)
    np.testing.assert_allclose(ex.real, kernels.raised_cosine(y, alpha, N), atol=1e-12)
    assert np.abs(ex.imag).max() < 1e-12


def test_prop1_fig1_regime():
    # Fig. 1: alpha = 1/30, N = 20, range [-255, 255].
    t = np.arange(-255, 256, dtype=float)[:, None]
    a = np.array([1 / 30])
    errs = {N: np.abs(kernels.raised_cosine(t, a, N) - kernels.gaussian_range(t, a)).max()
            for N in (10, 20, 40, 80, 160)}
    assert errs[20] < 0.02
    assert errs[10] > errs[20] > errs[40] > errs[80] > errs[160]
    # O(1/N) convergence: the sup error scales like c/N with c ~ 0.18 (2nd-order Taylor term)
    for N in (40, 80, 160):
        assert 0.1 / N < errs[N] < 0.25 / N


def test_prop1_limit_pointwise():
    a = np.array([0.03, 0.05])
    y = np.array([[10.0, -25.0], [40.0, 3.0]])
    g = kernels.gaussian_range(y, a)
    rc = kernels.raised_cosine(y, a, 100000)
    np.testing.assert_allclose(rc, g, rtol=1e-4)


def test_gaussian_range_values():
    assert kernels.gaussian_range(np.zeros(3), np.ones(3) / 30) == 1.0
    assert abs(kernels.gaussian_range(np.array([30.0]), np.array([1 / 30])) - math.exp(-0.5)) < 1e-15
    assert abs(kernels.gaussian_range(np.array([10.0, 20.0]), np.array([0.1, 0.05])) - math.exp(-1)) < 1e-15


def test_sampled_kernel_special_cases():
    Y = np.array([[0]])
    assert abs(kernels.sampled_kernel(np.array([123.0]), Y, [0.1]) - 1.0) < 1e-15
    Y = np.array([[4, -2], [0, 2]])
    assert abs(kernels.sampled_kernel(np.zeros(2), Y, [0.1, 0.2]) - 1.0) < 1e-15
    # all outcomes of B(2, 1/2) in proportion {2:1, 0:2, -2:1} reproduce cos^2 exactly
    Y = np.array([[2], [0], [0], [-2]])
    y = np.array([[37.0]])
    v = kernels.sampled_kernel(y, Y, [0.01])
    assert abs(v.real - math.cos(0.37) ** 2) < 1e-15 and abs(v.imag) < 1e-15
