import sys, os, time, statistics
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1605_02164_b200 import Plan
from workloads import CONFIGS, make_image
f = torch.from_numpy(make_image(CONFIGS[2])).cuda()
out = torch.empty_like(f)
for s in (3.0, 4.0, 4.5, 5.0, 4.0):
    p = Plan(512, 512, 3, s, np.eye(3) * 1600.0, 10, 300, 1)
    p.sample_freqs()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < 0.3:
        p.filter(f, out); torch.cuda.synchronize()
    ts = []
    for _ in range(7):
        ev[0].record(); p.filter(f, out); ev[1].record(); torch.cuda.synchronize(); ts.append(ev[0].elapsed_time(ev[1]))
    print(s, p.info("radius"), p.info("kernel_R"), p.info("variant"), p.info("tile_rows"), p.info("groups"), p.info("ctas"), ["%.2f" % t for t in ts], flush=True)
    p.close()
