"""Small driver for ncu captures: filters `--rows` output rows of config `--config`
(band sharding entry, same fused kernel and schedule logic as the bench) `--reps` times."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from oracle import native  # noqa: E402  (slab bounds only)
from paper_1605_02164_b200 import Plan  # noqa: E402
from workloads import CONFIGS, make_image_rows  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--rows", type=int, default=0)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--samples", type=int, default=0)
ap.add_argument("--tile-rows", type=int, default=0)
ap.add_argument("--groups", type=int, default=0)
ap.add_argument("--variant", type=int, default=0)
ap.add_argument("--engine", type=int, default=0)
ap.add_argument("--sigma", type=float, default=0.0, help="override sigma_s (recursive engine sweeps)")
ap.add_argument("--rec-impl", type=int, default=-1, help="recursive engine: 0 staged, 1 tiled, 2 virtual lines (default)")
ap.add_argument("--rec-tc", type=int, default=-1, help="recursive engine, d = 3: 1 tensor-core pass 2")
ap.add_argument("--rec-overlap", type=int, default=-1, help="recursive engine: pass 0 / scan overlap mode")
ap.add_argument("--rec-batch", type=int, default=-1, help="recursive engine: samples per batch (0 auto)")
ap.add_argument("--rec-vtc", type=int, default=-1, help="recursive engine: 1 tensor-core virtual-line blurs")
a = ap.parse_args()
cfg = CONFIGS[a.config]
if a.sigma:
    import dataclasses
    cfg = dataclasses.replace(cfg, sigma_s=a.sigma)
rows = a.rows or cfg.H
y0 = (cfg.H - rows) // 2
s0, s1 = native.slab_bounds(cfg.H, y0, rows, cfg.radius)
M = a.samples or cfg.M
p = Plan(cfg.H, cfg.W, cfg.d, cfg.sigma_s, cfg.C_array, cfg.N, M, cfg.seed, value_range=cfg.value_range)
p.sample_freqs()
if a.tile_rows:
    p.set_option('tile_rows', a.tile_rows)
if a.groups:
    p.set_option('groups', a.groups)
if a.variant:
    p.set_option('variant', a.variant)
if a.engine:
    p.set_option('engine', a.engine)
if a.rec_impl >= 0:
    p.set_option('rec_impl', a.rec_impl)
if a.rec_tc >= 0:
    p.set_option('rec_tc', a.rec_tc)
if a.rec_vtc >= 0:
    p.set_option('rec_vtc', a.rec_vtc)
if a.rec_overlap >= 0:
    p.set_option('rec_overlap', a.rec_overlap)
if a.rec_batch >= 0:
    p.set_option('rec_batch', a.rec_batch)
slab = torch.from_numpy(make_image_rows(cfg, s0, s1)).cuda()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for i in range(a.reps):
    ev[0].record()
    out = p.filter_rows(slab, s0, y0, y0 + rows)
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1])
    print(f"rep {i}: {ms:.3f} ms  {rows * cfg.W * M / ms * 1e3:.3e} px*samples/s  "
          f"tile_rows={p.info('tile_rows')} groups={p.info('groups')} ctas={p.info('ctas')} rec_batch={p.info('rec_batch')}")
