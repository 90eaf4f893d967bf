"""Diagnostic: per-call times of one short fused launch repeated for a few seconds, with NVML SM clock
and throttle reasons sampled alongside (explains outliers in short-kernel timings)."""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import pynvml  # noqa: E402
import torch  # noqa: E402

from paper_1605_02164_b200 import Plan  # noqa: E402
from workloads import CONFIGS, make_image  # noqa: E402

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
samples = []
stop = threading.Event()


def sampler():
    while not stop.is_set():
        samples.append((time.perf_counter(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
        time.sleep(0.01)


f = torch.from_numpy(make_image(CONFIGS[2])).cuda()
out = torch.empty_like(f)
p = Plan(512, 512, 3, float(sys.argv[1]) if len(sys.argv) > 1 else 5.0, np.eye(3) * 1600.0, 10, 300, 1)
p.sample_freqs()
th = threading.Thread(target=sampler, daemon=True)
th.start()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
rec = []
t_end = time.perf_counter() + 4.0
while time.perf_counter() < t_end:
    t0 = time.perf_counter()
    ev[0].record()
    p.filter(f, out)
    t_host = time.perf_counter() - t0
    ev[1].record()
    torch.cuda.synchronize()
    rec.append((t0, ev[0].elapsed_time(ev[1]), t_host * 1e3))
stop.set()
th.join()
ts = np.array([r[1] for r in rec])
print(f"calls {len(ts)} median {np.median(ts):.3f} ms p10 {np.percentile(ts, 10):.3f} p90 {np.percentile(ts, 90):.3f} "
      f"max {ts.max():.3f}")
slow = [r for r in rec if r[1] > 2 * np.median(ts)]
print(f"slow calls: {len(slow)}")
clk = np.array([s[1] for s in samples])
print(f"sm clock MHz: min {clk.min()} median {np.median(clk)} max {clk.max()}; reasons seen: "
      f"{sorted(set(hex(s[2]) for s in samples))}")
hosts = np.array([r[2] for r in rec])
print(f"host enqueue ms: median {np.median(hosts):.3f} max {hosts.max():.3f}")
for t0, ms, hms in slow[:10]:
    near = [s for s in samples if abs(s[0] - t0) < 0.03]
    print(f"  slow {ms:.2f} ms (host enqueue {hms:.2f} ms) at +{t0 - rec[0][0]:.3f} s; "
          f"clocks nearby {sorted(set((s[1], hex(s[2])) for s in near))}")
