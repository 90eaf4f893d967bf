"""Per-call host and device timing of bf_vec_filter for one config and kernel variant."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1605_02164_b200 import Plan
from workloads import CONFIGS, make_image
cfg = CONFIGS[int(sys.argv[1])]
f = torch.from_numpy(make_image(cfg)).cuda()
for variant in (1, 2):
    p = Plan(cfg.H, cfg.W, cfg.d, cfg.sigma_s, cfg.C_array, cfg.N, cfg.M, cfg.seed, value_range=cfg.value_range)
    p.sample_freqs()
    p.set_option("variant", variant)
    out = p.filter(f)
    torch.cuda.synchronize()
    p.set_option("profile", 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    host = []
    e0.record()
    for _ in range(10):
        t0 = time.perf_counter(); p.filter(f, out); host.append(time.perf_counter() - t0)
    e1.record(); torch.cuda.synchronize()
    print(f"variant {variant} (info {p.info('variant')}): device {e0.elapsed_time(e1)/10:.3f} ms/call, "
          f"fused {p.info('fused_ns_total')/1e6/p.info('fused_calls'):.3f} ms, host {1e3*sum(host)/10:.3f} ms/call, "
          f"tile {p.info('tile_rows')} groups {p.info('groups')} occ {p.info('occupancy')}")
    p.close()
