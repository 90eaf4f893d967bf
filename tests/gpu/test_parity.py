"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs and draws. Gates in tests/gpu/helpers.py."""
import dataclasses
import math

import numpy as np
import pytest
import torch

from oracle import draws, filters, native
from oracle import plan as oplan
from paper_1605_02164_b200 import BfVecError
from tests.gpu import helpers as H
from workloads import CONFIGS, make_image, make_image_rows
from workloads.configs import random_image, small_config

pytestmark = pytest.mark.gpu


def test_sampler_bit_exact():
    for i in (1, 2, 3, 4, 5):
        cfg = CONFIGS[i]
        p = H.gpu_plan(cfg)
        X, t, Q, a = p.get_draws()
        Xo = draws.binomial_draws(cfg.seed, cfg.M, cfg.d, cfg.N)
        assert np.array_equal(X, Xo), i
        Qo, ao, Yo = H.oracle_draws(cfg)
        t64 = (Yo * oplan.gammas(ao, cfg.N)[None, :]) @ Qo.T           # t_k = Q (Y o gamma)
        ulp = np.spacing(np.abs(t64).astype(np.float32)).astype(np.float64)
        assert np.all(np.abs(t.astype(np.float64) - t64) <= ulp), i
        p.close()


@pytest.mark.parametrize("i", [1, 2])
def test_config_full_parity(i):
    cfg = CONFIGS[i]
    f = make_image(cfg)
    Q, a, Y = H.oracle_draws(cfg)
    S_o, P_o, Z_o = native.mcsf_full(f, Q, a, cfg.N, Y, cfg.sigma_s)
    p = H.gpu_plan(cfg)
    S_g, P_g, Z_g = H.gpu_run(p, f)
    res = H.gates(cfg, S_g, P_g, Z_g, S_o, P_o, Z_o)
    print(f"config {i}: {res}")
    H.assert_gates(res)
    zmin, nsmall = p.diag()
    assert abs(zmin - (Z_g.min() / cfg.M)) < 1e-5
    assert nsmall == int((Z_g / cfg.M < H.Z_FLOOR).sum())


@pytest.mark.parametrize("i", [3, 4, 5])
def test_config_bands_parity(i):
    """Full-size launch (the bench's configuration), checked on three row bands
    (top, middle, bottom) against Algorithm 1 on a row slab, and on sampled
    pixels against the windowed definition."""
    cfg = CONFIGS[i]
    f = make_image(cfg)
    Q, a, Y = H.oracle_draws(cfg)
    p = H.gpu_plan(cfg)
    S_g, P_g, Z_g = H.gpu_run(p, f)
    get_rows = lambda y0, y1: f[:, y0:y1]
    nb = 8 if i == 5 else 16
    bands = [0, cfg.H // 2 - nb // 2, cfg.H - nb]   # top / middle / bottom (config 5: ~40 s of oracle each)
    worst = {}
    for y0 in bands:
        S_o, P_o, Z_o = H.oracle_band(cfg, get_rows, Q, a, Y, y0, nb)
        res = H.gates(cfg, S_g[:, y0:y0 + nb], P_g[:, y0:y0 + nb], Z_g[y0:y0 + nb], S_o, P_o, Z_o)
        print(f"config {i} band {y0}: {res}")
        H.assert_gates(res)
    rng = np.random.default_rng(100 + i)
    pix = [(int(y), int(x)) for y, x in zip(rng.integers(0, cfg.H, 24), rng.integers(0, cfg.W, 24))]
    pix += [(0, 0), (cfg.H - 1, cfg.W - 1), (cfg.H // 2, 0), (0, cfg.W - 1)]
    S_o, P_o, Z_o = filters.mc_filter_pixels(get_rows, cfg.H, cfg.W, pix, Q, a, cfg.N, Y, cfg.sigma_s)
    ys, xs = np.array(pix).T
    res = H.gates(cfg, S_g[:, ys, xs], P_g[:, ys, xs], Z_g[ys, xs], S_o.T, P_o.T, Z_o)
    print(f"config {i} pixels: {res}")
    H.assert_gates(res)


EDGE = [
    # (H, W, d, sigma_s, N, M, seed, C kind)
    (1, 1, 3, 1.0, 10, 4, 0, "diag"),         # single pixel
    (1, 37, 3, 1.0, 10, 5, 1, "diag"),        # single row, ragged width
    (37, 1, 2, 1.3, 10, 5, 2, "full"),        # single column
    (5, 7, 3, 4.0, 20, 6, 3, "full"),         # window much larger than the image
    (33, 45, 1, 2.0, 16, 9, 4, "diag"),       # d = 1, ragged tiles
    (40, 70, 2, 1.5, 10, 12, 5, "full"),      # d = 2
    (29, 66, 5, 1.0, 12, 7, 6, "full"),       # d = 5 (padded to the D = 8 kernel)
    (64, 96, 8, 2.0, 30, 6, 7, "diag"),       # d = 8
    (50, 50, 3, 0.7, 10, 1, 8, "full"),       # M = 1, r = 3 (padded radius)
    (131, 77, 3, 5.0, 30, 17, 9, "full"),     # several tiles and a ragged tail
    (70, 40, 4, 3.3, 20, 10, 10, "diag"),     # d = 4, r = 10 (padded radius)
    (150, 90, 3, 21.3, 40, 5, 11, "diag"),    # r = 64: the largest FIR radius (v3 instance)
    (96, 70, 8, 8.0, 30, 4, 12, "full"),      # d = 8 at config 4's r = 24
    (90, 64, 4, 16.0, 40, 3, 13, "diag"),     # d = 4, r = 48 (v3)
    (64, 64, 3, 16.0, 40, 3, 14, "full"),     # r = 48 default kernel (v5): one sample pair + a one-sample tail
    (64, 64, 3, 10.0, 40, 2, 15, "full"),     # v5 at r = 30 with a single pass
    (77, 100, 3, 1.0, 10, 7, 16, "full"),     # two-sample kernel at R = 3 (d = 3): several strips, odd M
    (45, 70, 1, 2.0, 16, 5, 17, "diag"),      # two-sample kernel at R = 6, d = 1
    (60, 50, 2, 3.3, 20, 6, 18, "full"),      # two-sample kernel at R = 10, d = 2
]


def _edge_cfg(case):
    Hh, W, d, s, N, M, seed, kind = case
    if kind == "diag":
        C = np.diag(np.full(d, 40.0 ** 2))
    else:
        rng = np.random.default_rng(seed)
        A = rng.normal(size=(d, d))
        C = 40.0 ** 2 * (A @ A.T / d + np.eye(d))
    return small_config(d=d, H=Hh, W=W, sigma_s=s, N=N, M=M, seed=seed, C=C)


@pytest.mark.parametrize("case", EDGE)
def test_edge_cases_parity(case):
    cfg = _edge_cfg(case)
    f = random_image(cfg.H, cfg.W, cfg.d, seed=cfg.seed, smooth=True)
    Q, a, Y = H.oracle_draws(cfg)
    S_o, P_o, Z_o = native.mcsf_full(f, Q, a, cfg.N, Y, cfg.sigma_s)
    p = H.gpu_plan(cfg)
    S_g, P_g, Z_g = H.gpu_run(p, f)
    res = H.gates(cfg, S_g, P_g, Z_g, S_o, P_o, Z_o)
    print(case, res)
    H.assert_gates(res)


def test_constant_image_and_zero_noise():
    cfg = small_config(d=3, H=48, W=64, sigma_s=2.0, N=20, M=16, seed=3)
    f = np.full((3, 48, 64), 123.5, dtype=np.float32)
    p = H.gpu_plan(cfg)
    S_g, P_g, Z_g = H.gpu_run(p, f)
    assert np.abs(S_g - 123.5).max() < 1e-3
    np.testing.assert_allclose(Z_g, cfg.M, rtol=1e-5)


def test_forced_schedules_agree():
    """Different (tile_rows, groups) schedules compute the same sums."""
    cfg = CONFIGS[2]
    f = make_image(cfg)
    p = H.gpu_plan(cfg)
    base = H.gpu_run(p, f)
    for tr, g in [(32, 1), (64, 3), (512, 7), (96, 64)]:
        p.set_option("tile_rows", tr)
        p.set_option("groups", g)
        S, P, Z = H.gpu_run(p, f)
        assert p.info("groups") == g
        np.testing.assert_allclose(Z, base[2], atol=1e-5 * cfg.M)
        ok = base[2] / cfg.M >= H.Z_FLOOR            # conditioned pixels (reading R5)
        assert np.abs(S - base[0])[:, ok].max() < 2e-3


def test_determinism_bitwise():
    cfg = CONFIGS[2]
    f = torch.from_numpy(make_image(cfg)).cuda()
    p = H.gpu_plan(cfg)
    a = p.filter(f).clone()
    b = p.filter(f).clone()
    torch.cuda.synchronize()
    assert torch.equal(a, b)


def test_filter_rows_band_equals_full():
    cfg = CONFIGS[2]
    f_np = make_image(cfg)
    f = torch.from_numpy(f_np).cuda()
    p = H.gpu_plan(cfg)
    full = p.filter(f).cpu().numpy()
    Z = p.filter_partial(f, 0, cfg.M).cpu().numpy().reshape(cfg.d + 1, cfg.H, cfg.W)[cfg.d]
    r = cfg.radius
    for (y0, y1) in [(0, 100), (200, 333), (480, 512)]:
        s0, s1 = native.slab_bounds(cfg.H, y0, y1 - y0, r)
        out = p.filter_rows(f[:, s0:s1].contiguous(), s0, y0, y1).cpu().numpy()
        ok = Z[y0:y1] / cfg.M >= H.Z_FLOOR           # conditioned pixels (reading R5)
        assert np.abs(out - full[:, y0:y1])[:, ok].max() < 2e-3


@pytest.mark.parametrize("groups", [1, 4])
def test_band_sharding_bitwise_equals_full(groups):
    """row-band sharding reproduces the single-GPU output BITWISE. Each output
    pixel's sums are formed by one CTA in a fixed order (H-pass taps, V-pass taps, samples in
    pass order within a group, groups summed in order by the normaliser), none of which depends
    on where a band or a row tile starts -- so with the same sample-group count the band entry
    (its own slab, reflection only at true image edges) must give identical bits, for bands
    aligned to the 16-row chunk grid and for ragged ones."""
    cfg = CONFIGS[2]
    f = torch.from_numpy(make_image(cfg)).cuda()
    p = H.gpu_plan(cfg)
    p.set_option("groups", groups)
    full = p.filter(f).cpu().numpy()
    r = cfg.radius
    for (y0, y1) in [(0, 128), (128, 256), (256, 512), (0, 100), (211, 333), (497, 512), (0, 512)]:
        s0, s1 = native.slab_bounds(cfg.H, y0, y1 - y0, r)
        out = p.filter_rows(f[:, s0:s1].contiguous(), s0, y0, y1).cpu().numpy()
        assert p.info("groups") == groups
        np.testing.assert_array_equal(out, full[:, y0:y1], err_msg=f"band [{y0},{y1}) groups {groups}")


def test_sample_shards_sum_to_full():
    cfg = CONFIGS[2]
    f = torch.from_numpy(make_image(cfg)).cuda()
    p = H.gpu_plan(cfg)
    full = p.filter_partial(f, 0, cfg.M).cpu().numpy()
    G = 3
    acc = np.zeros_like(full, dtype=np.float64)
    for g in range(G):
        acc += p.filter_partial(f, g * cfg.M // G, (g + 1) * cfg.M // G).cpu().numpy()
    np.testing.assert_allclose(acc, full, atol=1e-5 * cfg.M * 255)
    # banded layout: the band blocks hold the same numbers
    rpb = 200
    banded = p.filter_partial(f, 0, cfg.M, rows_per_band=rpb).cpu().numpy()
    d, Hh, W = cfg.d, cfg.H, cfg.W
    plain = full.reshape(d + 1, Hh, W)
    off = 0
    for b0 in range(0, Hh, rpb):
        n = min(rpb, Hh - b0)
        blk = banded[off:off + (d + 1) * n * W].reshape(d + 1, n, W)
        np.testing.assert_array_equal(blk, plain[:, b0:b0 + n])
        off += (d + 1) * n * W
        S_band = p.normalize(torch.from_numpy(np.ascontiguousarray(blk)).cuda(), b0, b0 + n)
        np.testing.assert_allclose(S_band.cpu().numpy(), plain[:d, b0:b0 + n] / plain[d, b0:b0 + n], rtol=1e-6)


def test_filter_host_async_frames_bitwise():
    """bf_vec_filter_host_async: five different frames enqueued back to back (copies of frame i+1 / i-1
    overlapping frame i), then one bf_vec_host_sync: each frame's output equals bf_vec_filter_host
    bit for bit (the alternating device slots are never overwritten while in use)."""
    cfg = CONFIGS[2]
    base = make_image(cfg)
    frames = [np.ascontiguousarray(np.roll(base, 37 * i, axis=2)) for i in range(5)]
    p = H.gpu_plan(cfg)
    ref = [p.filter_host(torch.from_numpy(fr).pin_memory()).clone() for fr in frames]
    fin = [torch.from_numpy(fr).pin_memory() for fr in frames]
    outs = [torch.empty((cfg.d, cfg.H, cfg.W), dtype=torch.float32).pin_memory() for _ in frames]
    s = torch.cuda.Stream()
    for fr, o in zip(fin, outs):
        p.filter_host_async(fr, o, stream=s)
    p.host_sync()
    for i, (o, r) in enumerate(zip(outs, ref)):
        assert torch.equal(o, r), f"frame {i}"
    # again, with a sync between every second frame and the default stream
    outs2 = [torch.empty_like(o) for o in outs]
    for i, (fr, o) in enumerate(zip(fin, outs2)):
        p.filter_host_async(fr, o)
        if i % 2:
            p.host_sync()
    p.host_sync()
    for o, r in zip(outs2, ref):
        assert torch.equal(o, r)
    p.close()


def test_filter_host_matches_device():
    cfg = CONFIGS[1]
    f_np = make_image(cfg)
    p = H.gpu_plan(cfg)
    dev = p.filter(torch.from_numpy(f_np).cuda()).cpu()
    host = p.filter_host(torch.from_numpy(f_np).pin_memory())
    assert torch.equal(dev, host)


@pytest.mark.parametrize("i", [1, 2])
def test_direct_filter_parity(i):
    cfg = CONFIGS[i]
    f = make_image(cfg)
    p = H.gpu_plan(cfg)
    g = p.direct(torch.from_numpy(f).cuda()).cpu().numpy()
    if i == 1:
        o = native.direct_full(f, cfg.C_array, cfg.sigma_s)
        assert np.abs(g - o).max() < 1e-3
    else:
        for y0 in (0, 250, 500):
            s0, s1 = native.slab_bounds(cfg.H, y0, 12, cfg.radius)
            o = native.direct(f[:, s0:s1], cfg.H, s0, y0, 12, cfg.C_array, cfg.sigma_s)
            assert np.abs(g[:, y0:y0 + 12] - o).max() < 1e-3


def test_direct_small_nondiagonal():
    cfg = _edge_cfg((37, 53, 3, 1.5, 10, 4, 3, "full"))
    f = random_image(cfg.H, cfg.W, 3, seed=1)
    p = H.gpu_plan(cfg)
    g = p.direct(torch.from_numpy(f).cuda()).cpu().numpy()
    o = native.direct_full(f, cfg.C_array, cfg.sigma_s)
    assert np.abs(g - o).max() < 1e-3


def test_p2p_sample_exchange_world1_matches_filter():
    """bf_vec_filter_partial_p2p + bf_vec_normalize_slots on one rank (the peer table is this
    rank's own receive buffer): the same result as bf_vec_filter up to fp32 summation order."""
    from paper_1605_02164_b200 import shard
    cfg = CONFIGS[2]
    f = torch.from_numpy(make_image(cfg)).cuda()
    p = H.gpu_plan(cfg)
    ref = p.filter(f).cpu().numpy()
    Z = p.filter_partial(f, 0, cfg.M).cpu().numpy().reshape(cfg.d + 1, cfg.H, cfg.W)[cfg.d]
    slots = shard.P2PSlots(p, 1, 0, slots_per_rank=4)
    try:
        with pytest.raises(BfVecError):         # before any p2p call: BF_E_STATE
            p.normalize_slots(slots.ptr, 4, 0, cfg.H, device=f.device)
        out, y0, y1 = shard.filter_samples_p2p(p, f, slots)
        got = out.cpu().numpy()
        # the band must be the owner's band of that call: a larger or shifted band
        # or more slots than were written is refused instead of reading past the buffer
        for bad in ((4, 0, cfg.H // 2), (4, 1, cfg.H), (5, 0, cfg.H)):
            with pytest.raises(BfVecError):
                p.normalize_slots(slots.last_ptr, bad[0], bad[1], bad[2], device=f.device)
    finally:
        slots.close()
    assert (y0, y1) == (0, cfg.H)
    ok = Z / cfg.M >= H.Z_FLOOR
    assert np.abs(got - ref)[:, ok].max() < 2e-3


def test_filter_partial_rejects_short_pz_before_launch():
    """an undersized PZ is refused before the kernel could write past it."""
    cfg = CONFIGS[1]
    f = torch.from_numpy(make_image(cfg)).cuda()
    p = H.gpu_plan(cfg)
    n = (cfg.d + 1) * cfg.H * cfg.W
    guard = torch.full((n + 4096,), 7.0, device=f.device)
    short = guard[: n - 1]
    with pytest.raises(ValueError):
        p.filter_partial(f, 0, cfg.M, PZ=short)
    torch.cuda.synchronize()
    assert bool((guard == 7.0).all())          # nothing was written
    with pytest.raises(ValueError):
        p.filter_partial(f, 0, cfg.M, PZ=guard[:n].view(cfg.d + 1, cfg.H, cfg.W).transpose(1, 2))
    p.close()


def test_graph_replay_bitwise_equals_eager():
    """Option "graph": on a created stream the second bf_vec_filter call captures a CUDA graph and
    later calls replay it; the output is bit-identical to eager launches, and an option change
    re-captures."""
    cfg = CONFIGS[2]
    f = torch.from_numpy(make_image(cfg)).cuda()
    p = H.gpu_plan(cfg)
    p.set_option("graph", 0)
    eager = p.filter(f).clone()
    p.set_option("graph", 1)
    s = torch.cuda.Stream()
    out = torch.empty_like(f)
    with torch.cuda.stream(s):
        for _ in range(4):
            p.filter(f, out)
    s.synchronize()
    assert p.info("graph_ready") == 1
    assert torch.equal(out, eager)
    with torch.cuda.stream(s):
        p.set_option("spatial_kernel", 1)        # new kernel arguments -> eager, then re-capture
        p.filter(f, out)
        p.filter(f, out)
        p.filter(f, out)
    s.synchronize()
    p.set_option("graph", 0)
    box = p.filter(f).clone()
    assert torch.equal(out, box)
    # another entry point that grows the plan's scratch (partial planes of 4 images) frees the
    # buffers the captured graph points at: the next call must re-capture, not replay stale pointers
    p.set_option("graph", 1)
    with torch.cuda.stream(s):
        for _ in range(3):
            p.filter(f, out)
    s.synchronize()
    assert p.info("graph_ready") == 1
    p.filter_batch(torch.stack([f] * 4))
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        for _ in range(3):
            out.zero_()
            p.filter(f, out)
    s.synchronize()
    assert torch.equal(out, box)


@pytest.mark.parametrize("case", [(3, 64, 64, 3, 2.0, 20, 32), (5, 37, 45, 3, 5.0, 30, 9), (2, 96, 64, 8, 3.0, 20, 6),
                                  (4, 40, 33, 1, 16.0, 40, 5)])
def test_filter_batch_matches_single_images(case):
    """bf_vec_filter_batch (one fused launch over all images) equals per-image filtering up to the
    fp32 summation order of the sample groups, and each image matches the oracle."""
    nimg, Hh, W, d, s, N, M = case
    cfg = _edge_cfg((Hh, W, d, s, N, M, 40 + nimg, "diag"))
    imgs = np.stack([random_image(Hh, W, d, seed=100 + i, smooth=bool(i % 2)) for i in range(nimg)])
    p = H.gpu_plan(cfg)
    fb = torch.from_numpy(imgs).cuda()
    batch = p.filter_batch(fb).cpu().numpy()
    Q, a, Y = H.oracle_draws(cfg)
    for i in range(nimg):
        single = p.filter(torch.from_numpy(imgs[i]).cuda()).cpu().numpy()
        S_o, P_o, Z_o = native.mcsf_full(imgs[i], Q, a, N, Y, s)
        ok = Z_o / M >= H.Z_FLOOR
        assert np.abs(batch[i] - single)[:, ok].max() < 2e-3, i
        assert np.abs(batch[i] - S_o)[:, ok].max() <= H.GATE_B * cfg.value_range / 255.0, i
