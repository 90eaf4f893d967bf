"""GPU parity of the non-Gaussian spatial kernels (option "spatial_kernel"; PAPER.md:205,
DESIGN.md reading R15): the CUDA path against the oracle with the same box / hat taps."""
import numpy as np
import pytest
import torch

from oracle import native
from oracle import plan as oplan
from tests.gpu import helpers as H
from tests.gpu.test_parity import _edge_cfg
from workloads import CONFIGS, make_image
from workloads.configs import random_image

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind", ["box", "hat"])
@pytest.mark.parametrize("i", [1, 2])
def test_config_parity(kind, i):
    cfg = CONFIGS[i]
    f = make_image(cfg)
    Q, a, Y = H.oracle_draws(cfg)
    S_o, P_o, Z_o = native.mcsf_full(f, Q, a, cfg.N, Y, cfg.sigma_s, spatial=kind)
    p = H.gpu_plan(cfg)
    p.set_option("spatial_kernel", oplan.SPATIAL_KINDS[kind])
    assert p.info("spatial_kernel") == oplan.SPATIAL_KINDS[kind]
    S_g, P_g, Z_g = H.gpu_run(p, f)
    res = H.gates(cfg, S_g, P_g, Z_g, S_o, P_o, Z_o)
    print(kind, i, res)
    H.assert_gates(res)


@pytest.mark.parametrize("kind", ["box", "hat"])
@pytest.mark.parametrize("case", [(64, 96, 8, 2.0, 30, 6, 7, "diag"), (131, 77, 3, 5.0, 30, 17, 9, "full"),
                                  (1, 37, 3, 1.0, 10, 5, 1, "diag")])
def test_edge_parity(kind, case):
    cfg = _edge_cfg(case)
    f = random_image(cfg.H, cfg.W, cfg.d, seed=cfg.seed, smooth=True)
    Q, a, Y = H.oracle_draws(cfg)
    S_o, P_o, Z_o = native.mcsf_full(f, Q, a, cfg.N, Y, cfg.sigma_s, spatial=kind)
    p = H.gpu_plan(cfg)
    p.set_option("spatial_kernel", oplan.SPATIAL_KINDS[kind])
    res = H.gates(cfg, *H.gpu_run(p, f), S_o, P_o, Z_o)
    print(kind, case, res)
    H.assert_gates(res)


@pytest.mark.parametrize("kind", ["box", "hat"])
def test_direct_parity(kind):
    cfg = CONFIGS[1]
    f = make_image(cfg)
    p = H.gpu_plan(cfg)
    p.set_option("spatial_kernel", oplan.SPATIAL_KINDS[kind])
    g = p.direct(torch.from_numpy(f).cuda()).cpu().numpy()
    o = native.direct_full(f, cfg.C_array, cfg.sigma_s, spatial=kind)
    assert np.abs(g - o).max() < 1e-3


def test_invalid_spatial_kernel_rejected():
    from paper_1605_02164_b200 import BfVecError
    p = H.gpu_plan(CONFIGS[1])
    with pytest.raises(BfVecError):
        p.set_option("spatial_kernel", 3)
