"""c3 at 10 M: plain vs start-face order, lone forward and fused forward + GFD (diagnostic)."""
import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2603_15780_b200 as dg
from bench import make_workload
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
xyz, tri, f, b, d, q = make_workload("c3", n, 42)
mesh = dg.Mesh(xyz, tri, device=0)
eps = mesh.default_gfd_eps()
dev = torch.device("cuda", 0)
t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dtype=dt)
def run(name, f, b, d, **kw):
    F, B, D = t(f, torch.int32), t(b, torch.float64), t(d, torch.float64)
    k = len(f)
    o = dict(face=torch.empty(k, dtype=torch.int32, device=dev), bary=torch.empty(k, 3, dtype=torch.float64, device=dev),
             dir=torch.empty(k, 3, dtype=torch.float64, device=dev), term=torch.empty(k, dtype=torch.uint8, device=dev),
             status=torch.empty(k, dtype=torch.uint8, device=dev), total_crossings=torch.zeros(1, dtype=torch.int64, device=dev))
    jv = torch.empty(k, 4, dtype=torch.float64, device=dev); jp = torch.empty(k, 4, dtype=torch.float64, device=dev)
    for label, fn in (("forward", lambda: mesh.trace_batch_device(F, B, D, o, **kw)),
                      ("fused fwd+GFD", lambda: mesh.trace_gfd_device(F, B, D, o, eps, eps, jv, jp))):
        ts = []
        for _ in range(3):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
        cr = int(o["total_crossings"].item())
        print(f"{name:28s} {label:14s} {min(ts):8.2f} ms {cr/min(ts)/1e6:7.2f} Gcross/s", flush=True)
run("plain order", f, b, d)
run("sort_by_face (device)", f, b, d, sort_by_face=True)
order = np.argsort(f, kind="stable")
run("pre-sorted by face", f[order], b[order], d[order])
run("pre-sorted, loads", f[order], b[order], d[order], walker="loads")
