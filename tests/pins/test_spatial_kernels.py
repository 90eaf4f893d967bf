"""Pins for the non-Gaussian spatial kernels ("we can replace the spatial
filter omega(i) in (1) with any arbitrary spatial filter (such as a box or hat filter),
and the above reductions would still hold"; reading R15).

What pins them:
  * box taps against the textbook moving average: the C -> infinity MC filter (and the
    exact filter) must equal scipy.ndimage.uniform_filter with mode='reflect';
  * hat taps against their construction as a box convolved with itself (np.convolve of
    two length-(r+1) boxes), independent of the closed form r + 1 - |m|;
  * the keystone (Alg. 1 separable form == windowed definition) with box and hat taps:
    the reduction of Eq. (15)-(19) holds for any separable omega.
"""
import numpy as np
import pytest
from scipy import ndimage

from oracle import draws, filters, native, plan
from workloads.configs import random_image


@pytest.mark.parametrize("sigma_s", [0.4, 1.0, 2.0, 5.0, 16.0])
def test_box_taps_are_a_moving_average(sigma_s):
    r = plan.radius(sigma_s)
    w = plan.spatial_window(sigma_s, "box")
    assert len(w) == 2 * r + 1
    assert abs(w.sum() - 1.0) < 1e-15
    assert np.ptp(w) == 0.0


@pytest.mark.parametrize("sigma_s", [0.4, 1.0, 2.0, 5.0, 16.0])
def test_hat_taps_are_box_convolved_with_box(sigma_s):
    r = plan.radius(sigma_s)
    box = np.ones(r + 1)
    tri = np.convolve(box, box)            # support 2r+1, peak r+1 at the centre
    np.testing.assert_allclose(plan.spatial_window(sigma_s, "hat"), tri / tri.sum(), rtol=0, atol=1e-16)


def test_unknown_kind_rejected():
    with pytest.raises(ValueError):
        plan.spatial_window(1.0, "lanczos")


@pytest.mark.parametrize("H,W,sigma_s", [(13, 17, 1.0), (9, 6, 2.0), (4, 5, 1.7)])
def test_box_c_to_infinity_is_uniform_filter(H, W, sigma_s):
    """With C -> infinity every range weight is 1: MCSF and the exact filter reduce to
    the box blur, i.e. scipy's uniform_filter (library routine), reflect boundary."""
    d, N, T = 3, 10, 4
    f = random_image(H, W, d, seed=3)
    r = plan.radius(sigma_s)
    ref = ndimage.uniform_filter(f.astype(np.float64), size=(1, 2 * r + 1, 2 * r + 1), mode="reflect")
    C = np.eye(d) * 1e16
    Q, a = plan.diagonalize(C)
    Y = draws.y_draws(5, T, d, N)
    S, P, Z = native.mcsf_full(f, Q, a, N, Y, sigma_s, spatial="box")
    np.testing.assert_allclose(S, ref, atol=1e-7)
    np.testing.assert_allclose(Z, T, atol=1e-9)
    np.testing.assert_allclose(native.direct_full(f, C, sigma_s, spatial="box"), ref, atol=1e-7)


@pytest.mark.parametrize("kind", ["box", "hat"])
@pytest.mark.parametrize("case", [(12, 10, 3, 1.0, 10, 6, 0), (7, 9, 2, 2.0, 20, 5, 1), (1, 8, 3, 1.0, 10, 3, 2)])
def test_keystone_holds_for_any_separable_window(kind, case):
    H, W, d, s, N, T, seed = case
    f = random_image(H, W, d, seed=seed)
    C = np.diag(np.full(d, 40.0 ** 2))
    Q, a = plan.diagonalize(C)
    Y = draws.y_draws(seed, T, d, N)
    S1, P1, Z1 = filters.mc_filter_bruteforce(f, Q, a, N, Y, s, spatial=kind)
    S2, P2, Z2 = native.mcsf_full(f, Q, a, N, Y, s, spatial=kind)
    np.testing.assert_allclose(Z2, Z1, atol=1e-10 * T)
    np.testing.assert_allclose(P2, P1, atol=1e-10 * T * 255)


def test_hat_exact_filter_matches_bruteforce():
    f = random_image(8, 9, 3, seed=4)
    C = np.diag([30.0 ** 2, 40.0 ** 2, 50.0 ** 2])
    np.testing.assert_allclose(native.direct_full(f, C, 1.0, spatial="hat"),
                               filters.direct_bruteforce(f, C, 1.0, spatial="hat"), atol=1e-9)
