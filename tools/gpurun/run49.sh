mkdir -p gpurun_out
timeout 900 python -m pytest tests/gpu/test_spatial_parity.py tests/gpu/test_variants.py -q -x > gpurun_out/pytest49.log 2>&1
echo "pytest exit $?"
cat > /tmp/boxbench.py <<'PY'
import sys, os, time, statistics
sys.path.insert(0, os.getcwd())
import torch
from paper_1605_02164_b200 import Plan
from workloads import CONFIGS, make_image
for ci in (5, 3, 2):
    cfg = CONFIGS[ci]
    f = torch.from_numpy(make_image(cfg)).cuda(); out = torch.empty_like(f)
    s = torch.cuda.Stream()
    for kind in (0, 1, 2):
        p = Plan(cfg.H, cfg.W, cfg.d, cfg.sigma_s, cfg.C_array, cfg.N, cfg.M, cfg.seed)
        p.set_option("spatial_kernel", kind); p.sample_freqs()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        with torch.cuda.stream(s):
            t0 = time.perf_counter()
            while time.perf_counter() - t0 < 0.5:
                p.filter(f, out); s.synchronize()
            ts = []
            for _ in range(5):
                ev[0].record(s); p.filter(f, out); ev[1].record(s); s.synchronize(); ts.append(ev[0].elapsed_time(ev[1]))
        ms = statistics.median(ts)
        print(f"config {ci} spatial {kind} variant {p.info('variant')}: {ms:.3f} ms {cfg.H*cfg.W*cfg.M/ms*1e3:.4e} px*samples/s", flush=True)
        p.close()
PY
timeout 600 python /tmp/boxbench.py > gpurun_out/boxbench49.log 2>&1
echo done
