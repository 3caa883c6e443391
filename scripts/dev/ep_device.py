"""EP backward alone, device-resident, on config 2 (dev)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2603_15780_b200 as dg
from bench import make_workload
n = 1_000_000
xyz, tri, f, b, d, q = make_workload("c2", n, 42)
mesh = dg.Mesh(xyz, tri, device=0)
dev = torch.device("cuda", 0)
t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dtype=dt)
F, B, D, G = t(f, torch.int32), t(b, torch.float64), t(d, torch.float64), t(q, torch.float64)
o = dict(face=torch.empty(n, dtype=torch.int32, device=dev), bary=torch.empty(n, 3, dtype=torch.float64, device=dev),
         dir=torch.empty(n, 3, dtype=torch.float64, device=dev))
mesh.trace_batch_device(F, B, D, o)
gv = torch.empty(n, 3, dtype=torch.float64, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ts = []
for _ in range(8):
    flush.zero_()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); mesh.ep_backward_device(F, D, o["face"], o["dir"], G, gv); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
print(f"ep_backward device-resident, L2 flushed: {min(ts):.4f} / {sorted(ts)[4]:.4f} ms  checksum {float(gv.sum()):.17g}", flush=True)
