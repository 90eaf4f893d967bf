"""GPU stratified sampler (option "sampler" = 1, reading R17): draws bit-exact against the
oracle's stratified_binomial_draws, t within one fp32 ulp, and the error sweep with stratified
draws against the oracle curve."""
import numpy as np
import pytest
import torch

from oracle import draws, experiments, native
from oracle import plan as oplan
from workloads.configs import random_image

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("M,d,N,seed", [(16, 2, 4, 0), (512, 3, 40, 4), (1000, 8, 30, 3), (37, 1, 64, 9),
                                        (1, 3, 10, 2), (300, 3, 2, 5)])
def test_stratified_draws_bit_exact(M, d, N, seed):
    from paper_1605_02164_b200 import Plan
    rng = np.random.default_rng(seed)
    A = rng.normal(size=(d, d))
    C = 30.0 ** 2 * (A @ A.T / d + np.eye(d))
    p = Plan(8, 8, d, 1.0, C, N, M, seed)
    p.set_option("sampler", 1)
    p.sample_freqs()
    X, t, Q, a = p.get_draws()
    Xo = draws.stratified_binomial_draws(seed, M, d, N)
    assert np.array_equal(X, Xo)
    Qo, ao = oplan.diagonalize(C)
    t64 = ((N - 2 * Xo) * oplan.gammas(ao, N)[None, :]) @ Qo.T
    ulp = np.spacing(np.abs(t64).astype(np.float32)).astype(np.float64)
    assert np.all(np.abs(t.astype(np.float64) - t64) <= ulp)


def test_sweep_with_stratified_draws():
    from paper_1605_02164_b200 import Plan
    d, Hh, W, s, N, M = 3, 40, 48, 1.0, 10, 32
    C = np.eye(d) * 30.0 ** 2
    f = random_image(Hh, W, d, seed=4, smooth=True)
    ref = native.direct_full(f, C, s).astype(np.float32)
    seeds, t_list = [21, 22], [8, 32]
    Q, a = oplan.diagonalize(C)
    o = experiments.mse_curve(f, ref, Q, a, N, seeds, t_list, s, sampler="stratified", M=M)
    p = Plan(Hh, W, d, s, C, N, M, 0)
    p.set_option("sampler", 1)
    p.sample_freqs()
    g = p.mse_sweep(torch.from_numpy(f).cuda(), torch.from_numpy(ref).cuda(), seeds, t_list)
    np.testing.assert_allclose(g, o, rtol=2e-3)
