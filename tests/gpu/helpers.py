"""Shared helpers of the GPU parity tests: run the CUDA path through the C ABI
and the oracle on the same seeded inputs and draws, and evaluate the gates of
DESIGN.md §5 (readings R5):

  Gate A (every pixel): |Z_gpu - Z_orc| / M <= 1e-5 and |P_gpu - P_orc| / M <= 1e-5 R
  Gate B (output):      max |S_gpu - S_orc| <= 1e-3 R/255 over pixels with Z_orc/M >= 0.05
"""
import numpy as np
import torch

from oracle import draws, native
from oracle import plan as oplan

GATE_A = 1e-5
GATE_B = 1e-3
Z_FLOOR = 0.05


def oracle_draws(cfg):
    Q, a = oplan.diagonalize(cfg.C_array)
    Y = draws.y_draws(cfg.seed, cfg.M, cfg.d, cfg.N)
    return Q, a, Y


def gpu_plan(cfg):
    from paper_1605_02164_b200 import Plan
    p = Plan(cfg.H, cfg.W, cfg.d, cfg.sigma_s, cfg.C_array, cfg.N, cfg.M, cfg.seed,
             value_range=cfg.value_range)
    p.sample_freqs()
    return p


def gpu_run(p, f_np):
    """(S, P, Z) from the CUDA path: S via bf_vec_filter, raw P/Z via bf_vec_filter_partial."""
    dev = torch.device("cuda:0")
    f = torch.from_numpy(np.ascontiguousarray(f_np)).to(dev)
    S = p.filter(f)
    PZ = p.filter_partial(f, 0, p.M)
    torch.cuda.synchronize()
    PZ = PZ.cpu().numpy().reshape(p.d + 1, p.H, p.W).astype(np.float64)
    return S.cpu().numpy().astype(np.float64), PZ[:p.d], PZ[p.d]


def gates(cfg, S_g, P_g, Z_g, S_o, P_o, Z_o):
    M, R = cfg.M, cfg.value_range
    ga_z = np.abs(Z_g - Z_o).max() / M
    ga_p = np.abs(P_g - P_o).max() / M / R
    ok = Z_o / M >= Z_FLOOR
    gb = np.abs(S_g - S_o)[..., ok].max() / (R / 255.0) if ok.any() else 0.0
    return {"gate_a_z": ga_z, "gate_a_p": ga_p, "gate_b": gb, "excluded": int((~ok).sum()),
            "all_max": float(np.nanmax(np.abs(S_g - S_o)))}


def assert_gates(res):
    assert res["gate_a_z"] <= GATE_A, res
    assert res["gate_a_p"] <= GATE_A, res
    assert res["gate_b"] <= GATE_B, res


def oracle_band(cfg, get_rows, Q, a, Y, y0, n):
    r = cfg.radius
    s0, s1 = native.slab_bounds(cfg.H, y0, n, r)
    slab = get_rows(s0, s1)
    return native.mcsf_alg1(slab, cfg.H, s0, y0, n, Q, a, cfg.N, Y, cfg.sigma_s)
