"""c5 vertex-to-vertex walkers alone: rate by walker (diagnostic)."""
import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2603_15780_b200 as dg
from paper_2603_15780_b200 import workloads as W
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
xyz, tri = W.torus(1 / 3, 1 / 6, 1000, 500)
mesh = dg.Mesh(xyz, tri, device=0)
f, b, d = W.vertex_edge_queries(xyz, tri, n, 5.0, seed=5, meridian=True)
dev = torch.device("cuda", 0)
t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dtype=dt)
F, B, D = t(f, torch.int32), t(b, torch.float64), t(d, torch.float64)
o = dict(face=torch.empty(n, dtype=torch.int32, device=dev), bary=torch.empty(n, 3, dtype=torch.float64, device=dev),
         dir=torch.empty(n, 3, dtype=torch.float64, device=dev), npoints=torch.empty(n, dtype=torch.int32, device=dev),
         crossings=torch.empty(n, dtype=torch.int32, device=dev), total_crossings=torch.zeros(1, dtype=torch.int64, device=dev))
for name, kw in (("auto", {}), ("generic", dict(generic_walker=True)), ("loads", dict(walker="loads")), ("auto bps=2", dict(blocks_per_sm=2))):
    ts = []
    for _ in range(2):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); mesh.trace_batch_device(F, B, D, o, max_steps=200000, sort_by_face=False, **kw); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    cr = int(o["total_crossings"].item()); pts = int(o["npoints"].sum().item())
    print(f"{name:12s} {min(ts):9.2f} ms  crossings/trace {cr/n:8.1f} points/trace {pts/n:8.1f}  {cr/min(ts)/1e6:6.2f} Gcross/s  {pts/min(ts)/1e6:6.2f} Gpoints/s", flush=True)
