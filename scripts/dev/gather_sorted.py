"""Which gather wins under start-face scheduling, c3 and c4 (diagnostic)."""
import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2603_15780_b200 as dg
from bench import make_workload
dev = torch.device("cuda", 0)
t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dtype=dt)
for key, n in (("c3", 1_000_000), ("c3", 4_000_000), ("c4", 64 * 65536)):
    xyz, tri, f, b, d, q = make_workload(key, n, 42)
    mesh = dg.Mesh(xyz, tri, device=0)
    F, B, D = t(f, torch.int32), t(b, torch.float64), t(d, torch.float64)
    k = len(f)
    o = dict(face=torch.empty(k, dtype=torch.int32, device=dev), bary=torch.empty(k, 3, dtype=torch.float64, device=dev),
             total_crossings=torch.zeros(1, dtype=torch.int64, device=dev))
    for sort in (None, False):
        for w in ("auto", "loads", "coop", "tma"):
            ts = []
            for _ in range(3):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record(); mesh.trace_batch_device(F, B, D, o, walker=w, sort_by_face=sort); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
            cr = int(o["total_crossings"].item())
            print(f"{key} n={k} sort={'auto' if sort is None else 'off'} walker={w:6s} {min(ts):8.2f} ms {cr/min(ts)/1e6:7.2f} Gcross/s", flush=True)
    del mesh
