"""Config-5 style stress: 1M-face torus, half the starts exactly at vertices aimed along an
incident edge, length 5 x outer diameter, max_steps 200000, scaled to one GPU."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_15780_b200 as dg
from paper_2603_15780_b200 import workloads as W
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
xyz, tri = W.torus(1 / 3, 1 / 6, 1000, 500)
mesh = dg.Mesh(xyz, tri, device=0)
fv, bv, dv = W.vertex_edge_queries(xyz, tri, n // 2, 5.0)
fr, br, dr = W.sample_queries(xyz, tri, n - n // 2, 5.0, seed=9)
dev = torch.device("cuda", 0)
t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dtype=dt)
def run(name, f, b, d):
    k = len(f)
    F, B, D = t(f, torch.int32), t(b, torch.float64), t(d, torch.float64)
    o = dict(face=torch.empty(k, dtype=torch.int32, device=dev), bary=torch.empty(k, 3, dtype=torch.float64, device=dev),
             dir=torch.empty(k, 3, dtype=torch.float64, device=dev), term=torch.empty(k, dtype=torch.uint8, device=dev),
             npoints=torch.empty(k, dtype=torch.int32, device=dev), total_crossings=torch.zeros(1, dtype=torch.int64, device=dev))
    ts = []
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); mesh.trace_batch_device(F, B, D, o, max_steps=200000); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    cr = int(o["total_crossings"].item()); seg = int(o["npoints"].sum().item()) - k
    print(f"{name:22s} n={k} {min(ts):9.2f} ms  crossings/trace {cr/k:8.1f} segments/trace {seg/k:8.1f}  "
          f"{cr/min(ts)/1e6:6.2f} Gcross/s {seg/min(ts)/1e6:6.2f} Gseg/s  term!=0: {int((o['term']!=0).sum())}", flush=True)
run("random starts", fr, br, dr)
run("vertex-edge starts", fv, bv, dv)
run("mixed (config 5)", np.concatenate([fv, fr]), np.concatenate([bv, br]), np.concatenate([dv, dr]))
