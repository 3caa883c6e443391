"""Fused forward + GFD on big tori: the sibling launch's gather (run with DG_FAST_GATHER=coop for the other one) (dev)."""
import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2603_15780_b200 as dg
from paper_2603_15780_b200 import workloads as W
dev = torch.device("cuda", 0)
t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dtype=dt)
n = 500_000
for nu, nv in ((1000, 500), (2000, 1000)):
    xyz, tri = W.torus(1 / 3, 1 / 6, nu, nv)
    mesh = dg.Mesh(xyz, tri, device=0)
    F = len(tri); eps = mesh.default_gfd_eps()
    for mult in (0.3, 0.6, 1.0):
        length = mult * np.sqrt(F) * mesh.mean_edge / 2.2
        f, b, d = W.sample_queries(xyz, tri, n, length, seed=9)
        Fq, B, D = t(f, torch.int32), t(b, torch.float64), t(d, torch.float64)
        o = dict(face=torch.empty(n, dtype=torch.int32, device=dev), bary=torch.empty(n, 3, dtype=torch.float64, device=dev),
                 dir=torch.empty(n, 3, dtype=torch.float64, device=dev), total_crossings=torch.zeros(1, dtype=torch.int64, device=dev))
        jv = torch.empty(n, 4, dtype=torch.float64, device=dev); jp = torch.empty(n, 4, dtype=torch.float64, device=dev)
        ts = []
        for _ in range(2):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); mesh.trace_gfd_device(Fq, B, D, o, eps, eps, jv, jp); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
        cr = int(o["total_crossings"].item())
        print(f"F {F:8d}  {cr / n:7.0f} crossings/trace ({cr / n / np.sqrt(F):4.2f} sqrt(F))  fused fwd+GFD {min(ts):8.2f} ms  gather {os.environ.get('DG_FAST_GATHER', 'default')}", flush=True)
    del mesh
