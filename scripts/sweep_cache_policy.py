"""Forward-only timing of the fast walker with and without crossing records over mesh sizes
(noisy tori, device-resident inputs): finds where the transport cache stops paying off."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_15780_b200 as dg
from paper_2603_15780_b200 import workloads as W

dev = torch.device("cuda", 0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 400_000
for na, nb in ((200, 100), (300, 150), (400, 200), (500, 250), (600, 300), (700, 350), (800, 400), (1000, 500)):
    xyz, tri = W.torus(1.0 / 3.0, 1.0 / 6.0, na, nb, noise=0.1, seed=7)
    f, b, d = W.sample_queries(xyz, tri, n, 0.5 * W.bbox_diagonal(xyz), seed=42)
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dtype=dt)
    F, B, D = t(f, torch.int32), t(b, torch.float64), t(d, torch.float64)
    o = dict(face=torch.empty(n, dtype=torch.int32, device=dev), bary=torch.empty(n, 3, dtype=torch.float64, device=dev),
             dir=torch.empty(n, 3, dtype=torch.float64, device=dev), total_crossings=torch.zeros(1, dtype=torch.int64, device=dev))
    row = [f"faces {len(tri):8d}"]
    for cache in (True, False):
        mesh = dg.Mesh(xyz, tri, device=0, transport_cache=cache)
        for _ in range(2): mesh.trace_batch_device(F, B, D, o)
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); mesh.trace_batch_device(F, B, D, o); e.record(); torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        cr = int(o["total_crossings"].item())
        row.append(f"{'cached' if cache else 'uncached'} {mesh.device_bytes/1e6:7.1f} MB {min(ts):8.3f} ms {cr/min(ts)/1e6:6.2f} Gcross/s")
        del mesh
    print(" | ".join(row), flush=True)
