"""config-5 vertex walkers through the GENERAL walker only (profiling target: its code is inlined in one kernel)."""
import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2603_15780_b200 as dg
from paper_2603_15780_b200 import workloads as W
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
xyz, tri = W.torus(1 / 3, 1 / 6, 1000, 500)
mesh = dg.Mesh(xyz, tri, device=0)
f, b, d = W.vertex_edge_queries(xyz, tri, n, 5.0, seed=5, meridian=True)
dev = torch.device("cuda", 0)
t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dtype=dt)
F, B, D = t(f, torch.int32), t(b, torch.float64), t(d, torch.float64)
o = dict(face=torch.empty(n, dtype=torch.int32, device=dev), bary=torch.empty(n, 3, dtype=torch.float64, device=dev),
         total_crossings=torch.zeros(1, dtype=torch.int64, device=dev))
for _ in range(3):
    mesh.trace_batch_device(F, B, D, o, max_steps=200000, sort_by_face=False, generic_walker=True)
    torch.cuda.synchronize()
print("crossings", int(o["total_crossings"].item()))
