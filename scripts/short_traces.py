"""Device-resident timing of short traces (icosphere-4, 100 k traces of length 0.1 .. pi/2: the reference's
benchmark protocol), where start-up and finish are a tenth of the work. usage: python scripts/short_traces.py"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_15780_b200 as dg
from paper_2603_15780_b200 import workloads as W
n = 100000
xyz, tri = W.icosphere(4)
f, b, d = W.sample_queries(xyz, tri, n, (0.1, np.pi / 2), seed=42)
mesh = dg.Mesh(xyz, tri, device=0)
dev = torch.device("cuda", 0)
t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dtype=dt)
F, B, D = t(f, torch.int32), t(b, torch.float64), t(d, torch.float64)
o = dict(face=torch.empty(n, dtype=torch.int32, device=dev), bary=torch.empty(n, 3, dtype=torch.float64, device=dev),
         dir=torch.empty(n, 3, dtype=torch.float64, device=dev), total_crossings=torch.zeros(1, dtype=torch.int64, device=dev))
ts = []
for _ in range(20):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); mesh.trace_batch_device(F, B, D, o); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
cr = int(o["total_crossings"].item())
import time
h = []
for _ in range(10):
    t0 = time.perf_counter(); mesh.trace_batch(f, b, d); h.append((time.perf_counter() - t0) * 1e3)
print(f"{os.path.basename(os.environ.get('DG_B200_LIB', 'default'))}: device {min(ts):.4f} ms ({cr / n:.1f} crossings/trace, {cr / min(ts) / 1e6:.2f} Gcross/s); host-mode call {min(h):.3f} ms")
