"""Where per-lane loads lose to the cooperative gather under start-face order, on tori of several sizes (dev).
Lengths are chosen so that the expected crossings per trace are 0.5 ... 2.5 sqrt(F)."""
import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2603_15780_b200 as dg
from paper_2603_15780_b200 import workloads as W
dev = torch.device("cuda", 0)
t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dtype=dt)
cases = [(int(a), int(b), int(c)) for a, b, c in (x.split(":") for x in sys.argv[1].split(","))] if len(sys.argv) > 1 else [(1500, 750, 500000), (2000, 1000, 500000)]
mults = [float(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0.5, 1.0, 1.5, 2.5]
for nu, nv, n in cases:
    xyz, tri = W.torus(1 / 3, 1 / 6, nu, nv)
    mesh = dg.Mesh(xyz, tri, device=0)
    F = len(tri)
    for mult in mults:
        length = mult * np.sqrt(F) * mesh.mean_edge / 2.2
        f, b, d = W.sample_queries(xyz, tri, n, length, seed=9)
        Fq, B, D = t(f, torch.int32), t(b, torch.float64), t(d, torch.float64)
        o = dict(face=torch.empty(n, dtype=torch.int32, device=dev), bary=torch.empty(n, 3, dtype=torch.float64, device=dev),
                 dir=torch.empty(n, 3, dtype=torch.float64, device=dev), total_crossings=torch.zeros(1, dtype=torch.int64, device=dev))
        row = []
        for name, kw in (("loads", dict(sort_by_face=True, walker="loads")), ("coop", dict(sort_by_face=True, walker="coop")), ("auto", {})):
            ts = []
            for _ in range(2):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record(); mesh.trace_batch_device(Fq, B, D, o, max_steps=200000, **kw); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
            row.append(f"{name} {min(ts):8.2f} ms")
        cr = int(o["total_crossings"].item())
        print(f"F {F:8d} n {n:8d}  target {mult:3.1f} sqrt(F)  measured {cr / n / np.sqrt(F):4.2f} sqrt(F) crossings/trace   " + "   ".join(row), flush=True)
    del mesh
