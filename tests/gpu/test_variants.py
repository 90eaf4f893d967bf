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
    if p.info("variant") != variant:
        pytest.skip(f"variant {variant} at r = {cfg.radius} is a comparison instance "
                    "(build with -DBFVEC_COMPARISON_VARIANTS)")
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
    if p.info("variant") != variant:
        pytest.skip(f"variant {variant} at r = {cfg.radius} is a comparison instance "
                    "(build with -DBFVEC_COMPARISON_VARIANTS)")
    for tr, g in [(0, 0), (32, 2), (64, 3)]:
        p.set_option("tile_rows", tr)
        p.set_option("groups", g)
        res = H.gates(cfg, *H.gpu_run(p, f), S_o, P_o, Z_o)
        print(variant, case, tr, g, res)
        H.assert_gates(res)


# variant 8: the tensor-memory ring for 5 <= d <= 8 (two launches: {Z, P0..P6} two pairs per TMEM
# quarter, then P7 for four samples at once). Sample counts that leave the last four-sample pass partly empty (5, 7, 9),
# ragged tiles, d = 5 (channels 5..7 zero), forced schedules.
@pytest.mark.parametrize("case", [(96, 70, 8, 8.0, 30, 9, 12, "full"), (64, 96, 8, 2.0, 30, 7, 7, "diag"),
                                  (29, 66, 5, 1.0, 12, 5, 6, "full"), (50, 41, 6, 5.0, 20, 6, 3, "diag")])
def test_variant8_edge_parity(case):
    cfg = _edge_cfg(case)
    f = random_image(cfg.H, cfg.W, cfg.d, seed=cfg.seed, smooth=True)
    Q, a, Y = H.oracle_draws(cfg)
    S_o, P_o, Z_o = native.mcsf_full(f, Q, a, cfg.N, Y, cfg.sigma_s)
    p = H.gpu_plan(cfg)
    p.set_option("variant", 8)
    assert p.info("variant") == 8
    for tr, g in [(0, 0), (32, 2), (48, 3)]:
        p.set_option("tile_rows", tr)
        p.set_option("groups", g)
        res = H.gates(cfg, *H.gpu_run(p, f), S_o, P_o, Z_o)
        print(case, tr, g, res)
        H.assert_gates(res)


def test_variant8_config4_bands():
    """Config 4 at full size with variant 8, checked on two row bands against the oracle."""
    cfg = CONFIGS[4]
    f = make_image(cfg)
    Q, a, Y = H.oracle_draws(cfg)
    p = H.gpu_plan(cfg)
    p.set_option("variant", 8)
    S_g, P_g, Z_g = H.gpu_run(p, f)
    get_rows = lambda y0, y1: f[:, y0:y1]
    for y0 in (0, cfg.H - 16):
        S_o, P_o, Z_o = H.oracle_band(cfg, get_rows, Q, a, Y, y0, 16)
        res = H.gates(cfg, S_g[:, y0:y0 + 16], P_g[:, y0:y0 + 16], Z_g[y0:y0 + 16], S_o, P_o, Z_o)
        print("config 4 variant 8 band", y0, res)
        H.assert_gates(res)


@pytest.mark.parametrize("case", [(96, 70, 8, 8.0, 30, 9, 12, "full"), (29, 66, 5, 1.0, 12, 5, 6, "full")])
def test_variant1_d8_parity(case):
    """The shared-memory-ring kernel (variant 1) for d = 8, no longer the default there."""
    cfg = _edge_cfg(case)
    f = random_image(cfg.H, cfg.W, cfg.d, seed=cfg.seed, smooth=True)
    Q, a, Y = H.oracle_draws(cfg)
    S_o, P_o, Z_o = native.mcsf_full(f, Q, a, cfg.N, Y, cfg.sigma_s)
    p = H.gpu_plan(cfg)
    p.set_option("variant", 1)
    assert p.info("variant") == 1
    res = H.gates(cfg, *H.gpu_run(p, f), S_o, P_o, Z_o)
    print(case, res)
    H.assert_gates(res)


# The persistent schedule of the v6 kernel (option "persistent": one CTA per SM, each an equal share
# of the (strip, pass, chunk) work line, items starting / ending mid-pass, per-strip slots, zeroed
# unused rows and slots): forced on against the oracle, on shapes whose shares start mid-pass,
# span several strips, cover less than one pass, and with odd sample counts (one-sample passes).
@pytest.mark.parametrize("case", [(131, 77, 3, 5.0, 30, 17, 9, "full"), (70, 96, 3, 16.0, 40, 7, 2, "diag"),
                                  (512, 70, 3, 2.0, 20, 9, 5, "diag"), (300, 200, 1, 3.3, 20, 6, 7, "full"),
                                  (40, 33, 2, 8.0, 20, 5, 4, "full"),
                                  (40, 320, 3, 1.0, 10, 1500, 6, "diag")])   # shares of >= 50 passes: whole-pass cuts
def test_persistent_schedule_parity(case):
    cfg = _edge_cfg(case)
    f = random_image(cfg.H, cfg.W, cfg.d, seed=cfg.seed, smooth=True)
    Q, a, Y = H.oracle_draws(cfg)
    S_o, P_o, Z_o = native.mcsf_full(f, Q, a, cfg.N, Y, cfg.sigma_s)
    p = H.gpu_plan(cfg)
    p.set_option("persistent", 2)
    res = H.gates(cfg, *H.gpu_run(p, f), S_o, P_o, Z_o)
    print(case, "persistent", p.info("last_persistent"), "groups", p.info("groups"), res)
    assert p.info("last_persistent") == 1
    H.assert_gates(res)
    p.set_option("persistent", 0)
    res0 = H.gates(cfg, *H.gpu_run(p, f), S_o, P_o, Z_o)
    assert p.info("last_persistent") == 0
    H.assert_gates(res0)


def test_persistent_config2_default_and_graph():
    """Config 2 picks the persistent schedule by default (its 128 classic CTAs leave 20 SMs idle);
    the result passes the gates, repeats bitwise, and graph replay equals eager."""
    import torch
    cfg = CONFIGS[2]
    f = make_image(cfg)
    Q, a, Y = H.oracle_draws(cfg)
    S_o, P_o, Z_o = native.mcsf_full(f, Q, a, cfg.N, Y, cfg.sigma_s)
    p = H.gpu_plan(cfg)
    S_g, P_g, Z_g = H.gpu_run(p, f)
    assert p.info("last_persistent") == 1
    H.assert_gates(H.gates(cfg, S_g, P_g, Z_g, S_o, P_o, Z_o))
    fg = torch.from_numpy(f).cuda()
    p.set_option("graph", 0)
    e1 = p.filter(fg).clone()
    e2 = p.filter(fg).clone()
    assert torch.equal(e1, e2)
    p.set_option("graph", 1)
    s = torch.cuda.Stream()
    out = torch.empty_like(fg)
    with torch.cuda.stream(s):
        for _ in range(4):
            p.filter(fg, out)
    s.synchronize()
    assert p.info("graph_ready") == 1
    assert torch.equal(out, e1)


def test_persistent_tables_rewritten_invalidate_graph():
    """A call of another shape rewrites the persistent item tables; a CUDA graph captured for the
    first shape must then re-capture (plan generation), not replay against the rewritten tables."""
    import torch
    cfg = CONFIGS[2]
    fg = torch.from_numpy(make_image(cfg)).cuda()
    p = H.gpu_plan(cfg)
    p.set_option("graph", 0)
    ref = p.filter(fg).clone()
    p.set_option("graph", 1)
    s = torch.cuda.Stream()
    out = torch.empty_like(fg)
    with torch.cuda.stream(s):
        for _ in range(3):
            p.filter(fg, out)
    s.synchronize()
    assert p.info("graph_ready") == 1 and p.info("last_persistent") == 1
    with torch.cuda.stream(s):
        p.filter_partial(fg, 0, cfg.M // 2 + 7)          # another pass count: new tables
        for _ in range(3):
            out.zero_()
            p.filter(fg, out)
    s.synchronize()
    assert torch.equal(out, ref)
