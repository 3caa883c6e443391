"""exact lane vs tolerance lane: forward time on c2 / c3 and the fused forward + GFD on c3 (diagnostic)."""
import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2603_15780_b200 as dg
from bench import make_workload
dev = torch.device("cuda", 0)
t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dtype=dt)
for key, n in (("c2", 1_000_000), ("c3", 1_000_000)):
    xyz, tri, f, b, d, q = make_workload(key, n, 42)
    mesh = dg.Mesh(xyz, tri, device=0)
    eps = mesh.default_gfd_eps()
    F, B, D = t(f, torch.int32), t(b, torch.float64), t(d, torch.float64)
    o = dict(face=torch.empty(n, dtype=torch.int32, device=dev), bary=torch.empty(n, 3, dtype=torch.float64, device=dev),
             dir=torch.empty(n, 3, dtype=torch.float64, device=dev), term=torch.empty(n, dtype=torch.uint8, device=dev),
             status=torch.empty(n, dtype=torch.uint8, device=dev), total_crossings=torch.zeros(1, dtype=torch.int64, device=dev))
    jv = torch.empty(n, 4, dtype=torch.float64, device=dev); jp = torch.empty(n, 4, dtype=torch.float64, device=dev)
    for lane in ("exact", "fast"):
        for label, fn in (("forward", lambda: mesh.trace_batch_device(F, B, D, o, lane=lane)),
                          ("fused fwd+GFD", lambda: mesh.trace_gfd_device(F, B, D, o, eps, eps, jv, jp, lane=lane))):
            ts = []
            for _ in range(5):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
            cr = int(o["total_crossings"].item())
            print(f"{key} {lane:6s} {label:14s} {min(ts):8.3f} ms {cr/min(ts)/1e6:7.2f} Gcross/s", flush=True)
