"""Config 5's random half (length 5 x diameter on the 1 M-face torus) in start-face order: per-lane loads vs cooperative gather (dev)."""
import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2603_15780_b200 as dg
from paper_2603_15780_b200 import workloads as W
n = int(sys.argv[1]) if len(sys.argv) > 1 else 500_000
xyz, tri = W.torus(1 / 3, 1 / 6, 1000, 500)
mesh = dg.Mesh(xyz, tri, device=0)
diam = 2 * (1 / 3 + 1 / 6)
dev = torch.device("cuda", 0)
t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dtype=dt)
for mult in [float(x) for x in (sys.argv[2].split(',') if len(sys.argv) > 2 else ('0.5', '5.0'))]:
    f, b, d = W.sample_queries(xyz, tri, n, mult * diam, seed=9)
    F, B, D = t(f, torch.int32), t(b, torch.float64), t(d, torch.float64)
    o = dict(face=torch.empty(n, dtype=torch.int32, device=dev), bary=torch.empty(n, 3, dtype=torch.float64, device=dev),
             dir=torch.empty(n, 3, dtype=torch.float64, device=dev), total_crossings=torch.zeros(1, dtype=torch.int64, device=dev))
    for name, kw in (("sorted loads", dict(sort_by_face=True, walker="loads")), ("sorted coop", dict(sort_by_face=True, walker="coop")),
                     ("plain coop", dict(sort_by_face=False, walker="coop")), ("auto", {}), ("sorted coop", dict(sort_by_face=True, walker="coop")), ("auto", {})):
        ts = []
        for _ in range(3):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); mesh.trace_batch_device(F, B, D, o, max_steps=200000, **kw); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
        cr = int(o["total_crossings"].item())
        print(f"length {mult} x diameter  {name:13s} {min(ts):9.2f} ms  {cr/n:8.1f} crossings/trace  {cr/min(ts)/1e6:6.2f} Gcross/s", flush=True)
