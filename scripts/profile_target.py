"""One bench workload, one call shape, three launches: the target of the ncu captures under profiles/ (round 2).
usage: python scripts/profile_target.py c2|c3|c4|c5 forward|fused [exact|fast] [n]
Runs the call three times; `ncu -k regex:<kernel> -s 2 -c 1` then captures the warm third launch."""
import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_15780_b200 as dg
from bench import WORKLOADS, make_workload
key, mode = sys.argv[1], sys.argv[2]
lane = sys.argv[3] if len(sys.argv) > 3 else "exact"
n = int(sys.argv[4]) if len(sys.argv) > 4 else WORKLOADS[key]["n"]
xyz, tri, f, b, d, q = make_workload(key, n, 42)
n = len(f)
mesh = dg.Mesh(xyz, tri, device=0)
eps = mesh.default_gfd_eps()
dev = torch.device("cuda", 0)
t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dtype=dt)
F, B, D = t(f, torch.int32), t(b, torch.float64), t(d, torch.float64)
o = dict(face=torch.empty(n, dtype=torch.int32, device=dev), bary=torch.empty(n, 3, dtype=torch.float64, device=dev),
         dir=torch.empty(n, 3, dtype=torch.float64, device=dev), traced=torch.empty(n, dtype=torch.float64, device=dev),
         term=torch.empty(n, dtype=torch.uint8, device=dev), status=torch.empty(n, dtype=torch.uint8, device=dev),
         total_crossings=torch.zeros(1, dtype=torch.int64, device=dev))
jv = torch.empty(n, 4, dtype=torch.float64, device=dev); jp = torch.empty(n, 4, dtype=torch.float64, device=dev)
for _ in range(3):
    if mode == "forward":
        mesh.trace_batch_device(F, B, D, o, max_steps=WORKLOADS[key]["max_steps"], lane=lane)
    else:
        mesh.trace_gfd_device(F, B, D, o, eps, eps, jv, jp, lane=lane)
    torch.cuda.synchronize()
print(key, mode, lane, "n =", n, "crossings =", int(o["total_crossings"].item()), "plan =", mesh.trace_plan(n))
