"""GPU parity of the on-device error-vs-T experiment (bf_vec_mse_sweep; Fig. 5,
Eq. (20)) against the oracle's mse_curve on the same image, reference and seeds."""
import numpy as np
import pytest
import torch

from oracle import experiments, native
from oracle import plan as oplan
from workloads.configs import random_image, small_config

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("engine,d", [(0, 3), (1, 3), (0, 8)])
def test_sweep_matches_oracle_curve(engine, d):
    """d = 8 runs the realisation-batched sweep through the 8-channel kernel (variant 8)."""
    from paper_1605_02164_b200 import Plan
    Hh, W, s, N = 48, 64, 1.0, 10                # the Fig. 5 setting: sigma_s = 1, sigma_r = 30
    C = np.eye(d) * 30.0 ** 2
    cfg = small_config(d=d, H=Hh, W=W, sigma_s=s, N=N, M=64, seed=0, C=C)
    f = random_image(Hh, W, d, seed=3, smooth=True)
    ref = native.direct_full(f, C, s).astype(np.float32)
    seeds, t_list = [11, 12, 13], [4, 16, 64]
    Q, a = oplan.diagonalize(C)
    spatial = "deriche" if engine == 1 else "gaussian"
    o = experiments.mse_curve(f, ref, Q, a, N, seeds, t_list, s, spatial=spatial)
    p = Plan(Hh, W, d, s, C, N, 64, 0)
    p.set_option("engine", engine)
    p.sample_freqs()
    fg = torch.from_numpy(f).cuda()
    g = p.mse_sweep(fg, torch.from_numpy(ref).cuda(), seeds, t_list)
    print(engine, o, g)
    np.testing.assert_allclose(g, o, rtol=2e-3)
    # the plan's own draws are restored
    X, _, _, _ = p.get_draws()
    from oracle import draws
    assert np.array_equal(X, draws.binomial_draws(0, 64, d, N))


def test_sweep_argument_checks():
    from paper_1605_02164_b200 import BfVecError, Plan
    p = Plan(16, 16, 3, 1.0, np.eye(3) * 900.0, 10, 8, 0)
    p.sample_freqs()
    f = torch.zeros((3, 16, 16), device="cuda")
    for tl in ([0, 4], [4, 4], [4, 9]):
        with pytest.raises(BfVecError):
            p.mse_sweep(f, f, [1], tl)
