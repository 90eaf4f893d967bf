"""Every compiled fused-kernel variant (option "variant": 1 shared-memory ring, 2 TMEM ring,
3 TMEM ring with two consumer warps per pair, 4 TMEM ring with two samples per pass) against the
oracle on the same inputs and draws, incl. an odd sample count (variant 4's one-sample tail)."""
import dataclasses

import numpy as np
import pytest

from oracle import native
from tests.gpu import helpers as H
from tests.gpu.test_parity import _edge_cfg
from workloads import CONFIGS, make_image
from workloads.configs import random_image

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("variant", [1, 2, 3, 4, 5, 6])
def test_config2_parity(variant):
    cfg = CONFIGS[2]
    f = make_image(cfg)
    Q, a, Y = H.oracle_draws(cfg)
    S_o, P_o, Z_o = native.mcsf_full(f, Q, a, cfg.N, Y, cfg.sigma_s)
    p = H.gpu_plan(cfg)
    p.set_option("variant", variant)
    res = H.gates(cfg, *H.gpu_run(p, f), S_o, P_o, Z_o)
    print(variant, p.info("variant"), res)
    H.assert_gates(res)


@pytest.mark.parametrize("variant", [2, 4, 5, 6])
@pytest.mark.parametrize("case", [(131, 77, 3, 5.0, 30, 17, 9, "full"), (70, 96, 3, 16.0, 40, 7, 2, "diag"),
                                  (40, 33, 3, 8.0, 20, 5, 4, "full")])
def test_edge_parity(variant, case):
    cfg = _edge_cfg(case)
    f = random_image(cfg.H, cfg.W, cfg.d, seed=cfg.seed, smooth=True)
    Q, a, Y = H.oracle_draws(cfg)
    S_o, P_o, Z_o = native.mcsf_full(f, Q, a, cfg.N, Y, cfg.sigma_s)
    p = H.gpu_plan(cfg)
    p.set_option("variant", variant)
    for tr, g in [(0, 0), (32, 2), (64, 3)]:
        p.set_option("tile_rows", tr)
        p.set_option("groups", g)
        res = H.gates(cfg, *H.gpu_run(p, f), S_o, P_o, Z_o)
        print(variant, case, tr, g, res)
        H.assert_gates(res)
