import sys, torch, numpy as np
sys.path.insert(0, '.')
from tests.gpu import helpers as H
from workloads import CONFIGS, make_image
cfg = CONFIGS[2]
f = torch.from_numpy(make_image(cfg)).cuda()
p = H.gpu_plan(cfg)
p.set_option("graph", 0)
eager = p.filter(f).clone()
eager2 = p.filter(f).clone()
print("eager vs eager2 equal", torch.equal(eager, eager2))
p.set_option("graph", 1)
s = torch.cuda.Stream()
out = torch.empty_like(f)
for i in range(4):
    with torch.cuda.stream(s):
        p.filter(f, out)
    s.synchronize()
    d = (out - eager).abs()
    print(i, "graph_ready", p.info("graph_ready"), "groups", p.info("groups"), "max diff", float(d.max()), "n diff", int((d > 0).sum()))
