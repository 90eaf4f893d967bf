"""GPU sRGB <-> CIE-Lab transforms and Lab-space filtering (option "colorspace" = 1;
PAPER.md:305-308, reading R18) against the oracle (oracle/color.py, fp64)."""
import numpy as np
import pytest
import torch

from oracle import color, native
from tests.gpu import helpers as H
from workloads import CONFIGS, make_image
from workloads.configs import small_config

pytestmark = pytest.mark.gpu


def _rgb_samples():
    rng = np.random.default_rng(0)
    x = rng.uniform(0, 255, (3, 200000))
    edges = np.array([0.0, 255.0, 10.31475, 10.3148, 0.5, 254.5, 128.0])   # incl. the 0.04045 knee
    e = np.stack(np.meshgrid(edges, edges, edges)).reshape(3, -1)
    return np.concatenate([x, e], axis=1).astype(np.float32)


def test_conversions_match_oracle():
    from paper_1605_02164_b200 import lab_to_srgb, srgb_to_lab
    rgb = _rgb_samples()
    lab_g = srgb_to_lab(torch.from_numpy(rgb).cuda()).cpu().numpy()
    lab_o = color.srgb_to_lab(rgb.astype(np.float64))
    assert np.abs(lab_g - lab_o).max() < 2e-3
    back_g = lab_to_srgb(torch.from_numpy(lab_o.astype(np.float32)).cuda()).cpu().numpy()
    back_o = color.lab_to_srgb(lab_o.astype(np.float32).astype(np.float64))
    assert np.abs(back_g - back_o).max() < 2e-3
    # in place and round trip
    t = torch.from_numpy(rgb).cuda()
    srgb_to_lab(t, out=t)
    lab_to_srgb(t, out=t)
    assert np.abs(t.cpu().numpy() - rgb).max() < 5e-3


@pytest.mark.parametrize("engine", [0, 1])
def test_lab_space_filter_parity(engine):
    base = CONFIGS[1]
    cfg = small_config(d=3, H=base.H, W=base.W, sigma_s=2.0, N=20, M=32, seed=0, C=np.eye(3) * 20.0 ** 2)
    f = make_image(base)
    lab_o = color.srgb_to_lab(f.astype(np.float64)).astype(np.float32)
    Q, a, Y = H.oracle_draws(cfg)
    S_o, P_o, Z_o = native.mcsf_full(lab_o, Q, a, cfg.N, Y, cfg.sigma_s,
                                     spatial="deriche" if engine == 1 else "gaussian")
    p = H.gpu_plan(cfg)
    p.set_option("engine", engine)
    p.set_option("colorspace", 1)
    p.set_option("value_range", 100.0)
    S_g, P_g, Z_g = H.gpu_run(p, f)      # S back in sRGB, P / Z in Lab space
    Rlab = 100.0
    assert np.abs(Z_g - Z_o).max() / cfg.M <= H.GATE_A
    assert np.abs(P_g - P_o).max() / cfg.M / Rlab <= H.GATE_A
    ok = Z_o / cfg.M >= H.Z_FLOOR
    # Gate B in the filtering space (Lab, R = 100): the raw sums' quotient
    err_lab = np.abs(P_g / Z_g[None] - S_o)[:, ok].max()
    assert err_lab <= H.GATE_B * Rlab / 255.0, err_lab
    # the sRGB output adds the fp32 back-transform (same bound as the transform's own parity,
    # test_conversions_match_oracle: its error grows with the sRGB curve's slope near black)
    S_rgb_o = color.lab_to_srgb(S_o)
    err = np.abs(S_g - S_rgb_o)[:, ok].max()
    print(engine, err_lab, err, int((~ok).sum()))
    assert err <= 3e-3


def test_colorspace_requires_three_channels():
    from paper_1605_02164_b200 import BfVecError, Plan
    p = Plan(8, 8, 2, 1.0, np.eye(2) * 100.0, 10, 4, 0)
    with pytest.raises(BfVecError):
        p.set_option("colorspace", 1)
