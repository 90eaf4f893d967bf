"""GPU parity of the recursive O(1)-in-sigma_s engine (option "engine" = 1; PAPER.md:204,
DESIGN.md reading R16 / §11) against the oracle's plain definition: Algorithm 1 with the
Deriche kernel written out as taps (oracle.plan.deriche_window) on the reflected image.
Gates as for the FIR engine (tests/gpu/helpers.py)."""
import dataclasses

import numpy as np
import pytest
import torch

from oracle import filters, native
from tests.gpu import helpers as H
from tests.gpu.test_parity import _edge_cfg
from workloads import CONFIGS, make_image
from workloads.configs import random_image, small_config

pytestmark = pytest.mark.gpu


_IMPL = {"rec_impl": 1, "rec_tc": 0, "rec_vtc": 0}


@pytest.fixture(autouse=True, params=[(2, 0, 0), (2, 1, 0), (2, 1, 1), (1, 0, 0), (1, 1, 0), (0, 0, 0)],
                ids=["vlines", "vlines_tc", "vlines_tc_vscan", "tiled", "tiled_tc", "staged"])
def rec_impl(request):
    """Every test runs on every implementation of the engine (option "rec_impl"; "rec_tc" = 1: the
    tiles' pass-2 blurs on the tensor cores, d = 3; "rec_vtc" = 1: the column scan's virtual-line
    blurs too, W a multiple of 32)."""
    _IMPL["rec_impl"], _IMPL["rec_tc"], _IMPL["rec_vtc"] = request.param
    yield request.param[0]


def _rec_plan(cfg, batch=0):
    p = H.gpu_plan(cfg)
    p.set_option("engine", 1)
    p.set_option("rec_impl", _IMPL["rec_impl"])
    p.set_option("rec_tc", _IMPL["rec_tc"])
    p.set_option("rec_vtc", _IMPL["rec_vtc"])
    if batch:
        p.set_option("rec_batch", batch)
    return p


@pytest.mark.parametrize("i", [1, 2])
def test_config_full_parity(i):
    cfg = CONFIGS[i]
    f = make_image(cfg)
    Q, a, Y = H.oracle_draws(cfg)
    S_o, P_o, Z_o = native.mcsf_full(f, Q, a, cfg.N, Y, cfg.sigma_s, spatial="deriche")
    p = _rec_plan(cfg)
    S_g, P_g, Z_g = H.gpu_run(p, f)
    res = H.gates(cfg, S_g, P_g, Z_g, S_o, P_o, Z_o)
    print(f"recursive config {i} impl {p.info('rec_impl')}: {res} batch {p.info('rec_batch')}")
    H.assert_gates(res)


EDGE = [
    (1, 1, 3, 1.0, 10, 4, 0, "diag"),
    (1, 37, 3, 1.0, 10, 5, 1, "diag"),
    (37, 1, 2, 1.3, 10, 5, 2, "full"),
    (5, 7, 3, 4.0, 20, 6, 3, "full"),         # kernel support (24 sigma) >> image: multi-fold reflection
    (33, 45, 1, 2.0, 16, 9, 4, "diag"),
    (64, 96, 8, 2.0, 30, 6, 7, "diag"),
    (29, 66, 5, 1.0, 12, 7, 6, "full"),
    (131, 77, 3, 5.0, 30, 17, 9, "full"),     # ragged 32-tiles in both axes
    (50, 50, 3, 0.7, 10, 1, 8, "full"),       # M = 1
    (40, 200, 3, 30.0, 20, 4, 11, "diag"),    # r = 90 > 64: only the recursive engine runs
]


@pytest.mark.parametrize("case", EDGE)
def test_edge_cases_parity(case):
    cfg = _edge_cfg(case)
    f = random_image(cfg.H, cfg.W, cfg.d, seed=cfg.seed, smooth=True)
    Q, a, Y = H.oracle_draws(cfg)
    S_o, P_o, Z_o = native.mcsf_full(f, Q, a, cfg.N, Y, cfg.sigma_s, spatial="deriche")
    p = _rec_plan(cfg, batch=3)
    res = H.gates(cfg, *H.gpu_run(p, f), S_o, P_o, Z_o)
    print(case, res)
    H.assert_gates(res)


def test_fir_engine_rejects_large_radius():
    from paper_1605_02164_b200 import BfVecError
    cfg = _edge_cfg((40, 200, 3, 30.0, 20, 4, 11, "diag"))
    p = H.gpu_plan(cfg)
    assert p.info("fir_supported") == 0
    f = torch.from_numpy(random_image(cfg.H, cfg.W, 3, seed=0)).cuda()
    with pytest.raises(BfVecError) as e:
        p.filter(f)
    assert e.value.status == -4
    with pytest.raises(BfVecError):
        p.direct(f)


def test_batch_schedules_agree_and_are_deterministic():
    cfg = CONFIGS[2]
    f = make_image(cfg)
    base = H.gpu_run(_rec_plan(cfg, batch=64), f)
    for nb in (1, 5, 16):
        S, P, Z = H.gpu_run(_rec_plan(cfg, batch=nb), f)
        np.testing.assert_allclose(Z, base[2], atol=1e-5 * cfg.M)
        np.testing.assert_allclose(P, base[1], atol=1e-5 * cfg.M * 255)
    p = _rec_plan(cfg, batch=5)
    ft = torch.from_numpy(f).cuda()
    a = p.filter(ft).clone()
    b = p.filter(ft).clone()
    assert torch.equal(a, b)


def test_partial_shards_and_host_entry():
    cfg = CONFIGS[1]
    f_np = make_image(cfg)
    f = torch.from_numpy(f_np).cuda()
    p = _rec_plan(cfg, batch=4)
    full = p.filter_partial(f, 0, cfg.M).cpu().numpy()
    acc = sum(p.filter_partial(f, g * cfg.M // 3, (g + 1) * cfg.M // 3).cpu().numpy().astype(np.float64)
              for g in range(3))
    np.testing.assert_allclose(acc, full, atol=1e-5 * cfg.M * 255)
    dev = p.filter(f).cpu()
    host = p.filter_host(torch.from_numpy(f_np).pin_memory())
    assert torch.equal(dev, host)


def test_band_entry_rejected_for_proper_band():
    from paper_1605_02164_b200 import BfVecError
    cfg = CONFIGS[1]
    f = torch.from_numpy(make_image(cfg)).cuda()
    p = _rec_plan(cfg)
    with pytest.raises(BfVecError):
        p.filter_rows(f[:, 0:40].contiguous(), 0, 0, 20)
    whole = p.filter_rows(f, 0, 0, cfg.H)
    assert torch.equal(whole, p.filter(f))


def test_full_size_config5_sampled_pixels():
    """The full 8192^2 image at the bench's sigma_s, with M = 4 samples so the oracle's
    windowed definition (769^2 taps per pixel) stays cheap: 12 sampled pixels incl. corners."""
    cfg = dataclasses.replace(CONFIGS[5], M=4)
    f = make_image(CONFIGS[5])
    Q, a, Y = H.oracle_draws(cfg)
    p = _rec_plan(cfg)
    S_g, P_g, Z_g = H.gpu_run(p, f)
    rng = np.random.default_rng(5)
    pix = [(int(y), int(x)) for y, x in zip(rng.integers(0, cfg.H, 8), rng.integers(0, cfg.W, 8))]
    pix += [(0, 0), (cfg.H - 1, cfg.W - 1), (0, cfg.W - 1), (cfg.H - 1, 0)]
    S_o, P_o, Z_o = filters.mc_filter_pixels(lambda y0, y1: f[:, y0:y1], cfg.H, cfg.W, pix, Q, a, cfg.N, Y,
                                             cfg.sigma_s, spatial="deriche")
    ys, xs = np.array(pix).T
    res = H.gates(cfg, S_g[:, ys, xs], P_g[:, ys, xs], Z_g[ys, xs], S_o.T, P_o.T, Z_o)
    print("config 5 (M=4) pixels:", res)
    H.assert_gates(res)


@pytest.mark.parametrize("shape", [(256, 256), (200, 328), (64, 1024)])
def test_tensor_core_pass2_equals_fp32_pass2(shape, rec_impl):
    """Option rec_tc: pass 2's tile blurs as tf32 x3 GEMMs on the tensor cores give the
    FP32 recursion's partial sums to fp32 rounding -- on full-tile images and on ragged ones (full
    tiles on the tensor cores, the rest on the FP32 path). Relative to the largest sum: 2e-6."""
    if rec_impl == 0 or _IMPL["rec_tc"]:
        pytest.skip("the staged engine has no pass 2; the _tc fixtures repeat the same comparison")
    Hh, Ww = shape
    cfg = dataclasses.replace(CONFIGS[2], H=Hh, W=Ww, M=12)
    f = torch.from_numpy(random_image(Hh, Ww, 3, seed=Hh + Ww, smooth=True)).cuda()
    out = {}
    for tc in (0, 1):
        p = H.gpu_plan(cfg)
        p.set_option("engine", 1)
        p.set_option("rec_impl", rec_impl)
        p.set_option("rec_tc", tc)
        out[tc] = p.filter_partial(f, 0, cfg.M).cpu().numpy().astype(np.float64)
    scale = np.abs(out[0]).max()
    err = np.abs(out[1] - out[0]).max() / scale
    print(f"{shape} rec_impl {rec_impl}: max |tc - fp32| / max = {err:.2e}")
    assert err <= 2e-6


@pytest.mark.parametrize("d", [1, 2, 4, 5, 7])
@pytest.mark.parametrize("shape", [(96, 160), (100, 150)])
def test_tensor_core_recursion_other_channel_counts(d, shape, rec_impl):
    """The tensor-core segment blurs for d != 3 (pass 2 in ceil(2(d+1)/4) M halves, the last one
    padded for even d; the column scan's virtual lines for any d when W is a multiple of 32): the
    same partial sums as the FP32 recursion to fp32 rounding (2e-6 of the largest sum), and Gate A
    against the oracle."""
    if rec_impl != 2 or not _IMPL["rec_tc"] or not _IMPL["rec_vtc"]:
        pytest.skip("one fixture instance is enough")
    Hh, Ww = shape
    cfg = small_config(d=d, H=Hh, W=Ww, sigma_s=3.0, N=12, M=5, seed=d + Hh)
    f_np = random_image(Hh, Ww, d, seed=d + Ww, smooth=True)
    f = torch.from_numpy(f_np).cuda()
    out = {}
    for tc in (0, 1):
        p = H.gpu_plan(cfg)
        p.set_option("engine", 1)
        p.set_option("rec_impl", 2)
        p.set_option("rec_tc", tc)
        out[tc] = p.filter_partial(f, 0, cfg.M).cpu().numpy().astype(np.float64)
    err = np.abs(out[1] - out[0]).max() / np.abs(out[0]).max()
    Q, a, Y = H.oracle_draws(cfg)
    S_o, P_o, Z_o = native.mcsf_full(f_np, Q, a, cfg.N, Y, cfg.sigma_s, spatial="deriche")
    p = _rec_plan(cfg)
    res = H.gates(cfg, *H.gpu_run(p, f_np), S_o, P_o, Z_o)
    print(f"d {d} {shape}: max |tc - fp32| / max = {err:.2e}, {res}")
    assert err <= 2e-6
    H.assert_gates(res)


@pytest.mark.parametrize("overlap", [1, 2])
@pytest.mark.parametrize("shape", [(96, 128, 3, 2.0, 20, 11, 12), (131, 77, 3, 5.0, 30, 17, 13)],
                         ids=["full_tiles", "ragged"])
def test_overlap_schedule_bitwise(overlap, shape):
    """Option "rec_overlap": batch k + 1's pass 0 on the plan's stream while batch
    k's scans run on an auxiliary stream, two scratch sets. Every kernel does the same arithmetic on
    the same inputs, so the output must be bitwise that of the one-stream schedule, over several
    batches (incl. a short last one), through both the eager and the graph-replayed call; and it
    passes the gates against the oracle."""
    if _IMPL["rec_impl"] == 0:
        pytest.skip("the staged engine has one schedule")
    cfg = _edge_cfg(shape + ("full",))
    f = random_image(cfg.H, cfg.W, cfg.d, seed=cfg.seed, smooth=True)
    outs = {}
    for ov in (0, overlap):
        p = _rec_plan(cfg, batch=4)   # 17 or 11 samples: 3-5 batches, the last one short
        p.set_option("rec_overlap", ov)
        ft = torch.from_numpy(np.ascontiguousarray(f)).cuda()
        out = torch.empty((cfg.d, cfg.H, cfg.W), dtype=torch.float32, device="cuda")
        runs = [p.filter(ft, out).cpu().numpy() for _ in range(3)]   # eager, capture, replay
        for r in runs[1:]:
            assert np.array_equal(r, runs[0])
        outs[ov] = (runs[0], H.gpu_run(p, f))
    assert np.array_equal(outs[0][0], outs[overlap][0])
    for a, b in zip(outs[0][1], outs[overlap][1]):
        assert np.array_equal(a, b)
    Q, a, Y = H.oracle_draws(cfg)
    S_o, P_o, Z_o = native.mcsf_full(f, Q, a, cfg.N, Y, cfg.sigma_s, spatial="deriche")
    H.assert_gates(H.gates(cfg, *outs[overlap][1], S_o, P_o, Z_o))
