"""Pins for the accuracy-experiment oracle (Eq. (20), Fig. 5 of PAPER.md):
  * Eq. (20) against a hand-computed value and its invariants (zero for identical images,
    symmetric, scales with the square of a uniform offset);
  * the Monte Carlo error shrinks with T: averaged over realisations, the MSE between the
    MC filter and the raised-cosine filter it estimates (Prop. 2: the all-outcomes filter,
    tests/pins/test_filters.py) falls roughly like 1/T (variance of an unbiased mean);
  * prefixes: the curve's checkpoint T uses exactly the first T draws of the realisation.
"""
import numpy as np

from oracle import draws, experiments, native, plan
from workloads.configs import random_image


def test_mse_hand_value_and_invariants():
    B = np.zeros((3, 2, 2))
    S = np.zeros((3, 2, 2))
    S[0, 0, 0] = 2.0
    S[2, 1, 1] = -4.0
    assert experiments.mse(B, S) == (4.0 + 16.0) / 12.0
    assert experiments.mse(S, S) == 0.0
    assert experiments.mse(B, S) == experiments.mse(S, B)
    assert experiments.mse(B, B + 3.0) == 9.0


def test_curve_uses_draw_prefixes():
    f = random_image(10, 12, 3, seed=2)
    Q, a = plan.diagonalize(np.eye(3) * 50.0 ** 2)
    ref = native.direct_full(f, np.eye(3) * 50.0 ** 2, 1.0)
    curve = experiments.mse_curve(f, ref, Q, a, 10, [7], [3, 5], 1.0)
    Y = draws.y_draws(7, 5, 3, 10)
    S3, _, _ = native.mcsf_full(f, Q, a, 10, Y[:3], 1.0)
    assert curve[0, 0] == experiments.mse(ref, S3)


def test_mc_error_falls_like_one_over_t():
    """Against the exact raised-cosine filter (the MC estimator's mean), the average MSE at
    T = 64 is well below the average at T = 4 (ideal ratio 16 for an unbiased mean)."""
    H, W, d, s, N = 12, 12, 2, 1.0, 6
    f = random_image(H, W, d, seed=5)
    C = np.eye(d) * 40.0 ** 2
    Q, a = plan.diagonalize(C)
    # raised-cosine filter by exhaustive weighting of the outcomes (Prop. 2): 2^(N d) = 4096 rows
    from tests.pins.test_filters import _all_outcomes_Y
    Yall = _all_outcomes_Y(N, d)
    S_rc, _, _ = native.mcsf_full(f, Q, a, N, Yall, s)
    curve = experiments.mse_curve(f, S_rc, Q, a, N, list(range(40)), [4, 64], s)
    m4, m64 = curve.mean(axis=0)
    assert m64 < m4 / 6.0, (m4, m64)


def test_stratified_draws_reduce_the_mc_error():
    """Variance reduction (reading R17): at the same T, the average MSE to the raised-cosine
    filter is lower with stratified draws than with iid draws."""
    H, W, d, s, N, T = 12, 12, 2, 1.0, 6, 16
    f = random_image(H, W, d, seed=5)
    Q, a = plan.diagonalize(np.eye(d) * 40.0 ** 2)
    from tests.pins.test_filters import _all_outcomes_Y
    S_rc, _, _ = native.mcsf_full(f, Q, a, N, _all_outcomes_Y(N, d), s)
    iid, strat = [], []
    for seed in range(30):
        S1, _, _ = native.mcsf_full(f, Q, a, N, draws.y_draws(seed, T, d, N), s)
        S2, _, _ = native.mcsf_full(f, Q, a, N, draws.stratified_y_draws(seed, T, d, N), s)
        iid.append(experiments.mse(S_rc, S1))
        strat.append(experiments.mse(S_rc, S2))
    assert np.mean(strat) < 0.8 * np.mean(iid), (np.mean(strat), np.mean(iid))
