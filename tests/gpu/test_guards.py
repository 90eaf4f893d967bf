"""Memory-safety and race checks of every device entry point without compute-sanitizer (which
this GPU pool does not run: profiles/r02_compute_sanitizer_refused.txt).

* Guard bands: each output is a view into the middle of a larger buffer whose other bytes hold a
  NaN sentinel; after the call the sentinel must be intact (an out-of-bounds store anywhere past
  either end of an output shows up), and inputs are checked unmodified.
* Races across streams and plans: two plans on two streams, launched back to back so their kernels
  overlap, must give bitwise the results of isolated runs.
* Repetition: the default kernels run many times on one input give identical bits (a data race in
  a ring-buffer protocol shows up as rare run-to-run differences).
The checked build (tools/checked_build.sh: -DBFVEC_CHECKED, mbarrier watchdogs and ring-slot row
tags) runs the whole GPU suite, this file included, on top of these."""
import numpy as np
import pytest
import torch

from paper_1605_02164_b200 import Plan, lab_to_srgb, srgb_to_lab
from tests.gpu import helpers as H
from workloads import CONFIGS, make_image
from workloads.configs import random_image, small_config

pytestmark = pytest.mark.gpu

GUARD = 4099          # floats on each side (not a multiple of any tile)
SENTINEL = np.array([0x7FC0DEAD], dtype=np.uint32).view(np.float32)[0]


def guarded(shape, dev="cuda"):
    n = int(np.prod(shape))
    buf = torch.full((n + 2 * GUARD,), float("nan"), device=dev)
    buf.view(torch.int32).fill_(int(np.array(SENTINEL).view(np.int32)))
    return buf, buf[GUARD:GUARD + n].view(*shape)


def assert_intact(buf, n, what):
    torch.cuda.synchronize()
    bits = buf.view(torch.int32)
    s = int(np.array(SENTINEL).view(np.int32))
    assert bool((bits[:GUARD] == s).all()), f"{what}: store before the output"
    assert bool((bits[GUARD + n:] == s).all()), f"{what}: store past the output"


def _plan(cfg, **opts):
    p = H.gpu_plan(cfg)
    for k, v in opts.items():
        p.set_option(k, v)
    return p


CASES = [  # (name, cfg, options)
    ("v6_r15", CONFIGS[2], {}),
    ("v6_r6_ragged", small_config(d=3, H=77, W=100, sigma_s=2.0, N=20, M=5, seed=1), {}),
    ("box", small_config(d=3, H=70, W=90, sigma_s=5.0, N=20, M=4, seed=2), {"spatial_kernel": 1}),
    ("v8_d8", small_config(d=8, H=50, W=70, sigma_s=2.0, N=20, M=5, seed=3, C=np.eye(8) * 0.3 ** 2,
                           value_range=1.0), {}),
    ("v3_r64", small_config(d=3, H=60, W=50, sigma_s=21.3, N=20, M=3, seed=4), {}),
    ("rec_tiled", small_config(d=3, H=70, W=90, sigma_s=4.0, N=20, M=5, seed=5), {"engine": 1}),
    ("rec_staged", small_config(d=3, H=70, W=90, sigma_s=4.0, N=20, M=5, seed=6), {"engine": 1, "rec_impl": 0}),
]


@pytest.mark.parametrize("name,cfg,opts", CASES, ids=[c[0] for c in CASES])
def test_guard_bands_filter_partial_normalize(name, cfg, opts):
    f_np = random_image(cfg.H, cfg.W, cfg.d, seed=9, value_range=cfg.value_range, smooth=True)
    f = torch.from_numpy(f_np).cuda()
    f_copy = f.clone()
    p = _plan(cfg, graph=0, **opts)
    shp = (cfg.d, cfg.H, cfg.W)
    n = cfg.d * cfg.H * cfg.W
    buf, out = guarded(shp)
    p.filter(f, out)
    assert_intact(buf, n, f"{name} filter")
    # partial sums, plain and band-major layouts
    npz = (cfg.d + 1) * cfg.H * cfg.W
    bufz, pz = guarded((npz,))
    p.filter_partial(f, 0, cfg.M, PZ=pz)
    assert_intact(bufz, npz, f"{name} filter_partial")
    if opts.get("engine", 0) == 0:
        rpb = max(1, cfg.H // 3)
        bufb, pzb = guarded((npz,))
        p.filter_partial(f, 0, cfg.M, PZ=pzb, rows_per_band=rpb)
        assert_intact(bufb, npz, f"{name} filter_partial banded")
        # a band through bf_vec_filter_rows (slab = the whole image)
        y0, y1 = cfg.H // 3, cfg.H // 3 + max(1, cfg.H // 4)
        bufr, outr = guarded((cfg.d, y1 - y0, cfg.W))
        p.filter_rows(f, 0, y0, y1, out=outr)
        assert_intact(bufr, cfg.d * (y1 - y0) * cfg.W, f"{name} filter_rows")
    # normalise a band of the raw sums
    y0, y1 = 0, max(1, cfg.H // 2)
    band = pz.view(cfg.d + 1, cfg.H, cfg.W)[:, y0:y1].contiguous()
    bufn, outn = guarded((cfg.d, y1 - y0, cfg.W))
    p.normalize(band, y0, y1, out=outn)
    assert_intact(bufn, cfg.d * (y1 - y0) * cfg.W, f"{name} normalize")
    assert torch.equal(f, f_copy), f"{name}: input modified"
    p.close()


@pytest.mark.parametrize("d,H_,W_,sigma", [(3, 37, 53, 2.0), (3, 64, 130, 10.0), (8, 33, 41, 1.5), (1, 1, 1, 3.0)])
def test_guard_bands_direct(d, H_, W_, sigma):
    cfg = small_config(d=d, H=H_, W=W_, sigma_s=sigma, N=10, M=2, seed=1)
    f = torch.from_numpy(random_image(H_, W_, d, seed=3)).cuda()
    p = H.gpu_plan(cfg)
    buf, out = guarded((d, H_, W_))
    p.direct(f, out)
    assert_intact(buf, d * H_ * W_, "direct")
    assert bool(torch.isfinite(out).all())
    p.close()


def test_guard_bands_batch_and_lab():
    cfg = small_config(d=3, H=48, W=70, sigma_s=2.0, N=20, M=4, seed=2)
    nimg = 3
    fb = torch.from_numpy(np.stack([random_image(cfg.H, cfg.W, 3, seed=s, smooth=True) for s in range(nimg)])).cuda()
    p = H.gpu_plan(cfg)
    n = nimg * 3 * cfg.H * cfg.W
    buf, out = guarded((nimg, 3, cfg.H, cfg.W))
    p.filter_batch(fb, out)
    assert_intact(buf, n, "filter_batch")
    rgb = fb[0].contiguous()
    bufl, lab = guarded(tuple(rgb.shape))
    srgb_to_lab(rgb, lab)
    assert_intact(bufl, rgb.numel(), "srgb_to_lab")
    bufs, back = guarded(tuple(rgb.shape))
    lab_to_srgb(lab, back)
    assert_intact(bufs, rgb.numel(), "lab_to_srgb")
    p.close()


def test_one_plan_two_streams_is_ordered():
    """One plan driven from the legacy default stream and a non-blocking stream back to back, no
    host sync in between: the library orders the calls on the device (StreamOrder), so the shared
    scratch is never raced (the checked build's slower kernels exposed the unordered case)."""
    cfg = CONFIGS[2]
    f = torch.from_numpy(make_image(cfg)).cuda()
    g = f.flip(2).contiguous()
    p = H.gpu_plan(cfg)
    p.set_option("graph", 0)
    rf = p.filter(f).clone()
    rg = p.filter(g).clone()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    outs = []
    for i in range(6):
        o = torch.empty_like(f)
        src = f if i % 2 == 0 else g
        if i % 3 == 0:
            p.filter(src, o)                 # legacy default stream
        else:
            p.filter(src, o, stream=s)       # non-blocking stream, no sync with the previous call
        outs.append((o, rf if i % 2 == 0 else rg))
    torch.cuda.synchronize()
    for i, (o, r) in enumerate(outs):
        assert torch.equal(o, r), f"call {i}"
    p.close()


def test_two_streams_two_plans_bitwise():
    """Two plans (different kernels: v6 at r = 15 and the recursive engine) on two streams, their
    launches interleaved so the kernels overlap on the device: each result equals its isolated run
    bit for bit."""
    c2 = CONFIGS[2]
    f2 = torch.from_numpy(make_image(c2)).cuda()
    c3 = small_config(d=3, H=300, W=400, sigma_s=3.0, N=20, M=16, seed=7)
    f3 = torch.from_numpy(random_image(c3.H, c3.W, 3, seed=4, smooth=True)).cuda()
    pa = H.gpu_plan(c2)
    pb = _plan(c3, engine=1)
    ra = pa.filter(f2).clone()
    rb = pb.filter(f3).clone()
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    torch.cuda.synchronize()
    for _ in range(4):
        oa = torch.empty_like(f2)
        ob = torch.empty_like(f3)
        pa.filter(f2, oa, stream=sa)
        pb.filter(f3, ob, stream=sb)
        outs.append((oa, ob))
    torch.cuda.synchronize()
    for oa, ob in outs:
        assert torch.equal(oa, ra)
        assert torch.equal(ob, rb)
    pa.close()
    pb.close()


@pytest.mark.parametrize("cfg_i,reps", [(2, 30), (3, 4)])
def test_repeated_runs_bitwise(cfg_i, reps):
    cfg = CONFIGS[cfg_i]
    f = torch.from_numpy(make_image(cfg)).cuda()
    p = H.gpu_plan(cfg)
    ref = p.filter(f).clone()
    for _ in range(reps):
        assert torch.equal(p.filter(f), ref)
    p.close()
