"""Fan-walk prefetch (DG_FAN_PREFETCH) on config 5's vertex-to-vertex walkers: time and bits, off against on."""
import os, sys, subprocess
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import torch
    sys.path.insert(0, ROOT)
    import paper_2603_15780_b200 as dg
    from paper_2603_15780_b200 import workloads as W
    n = int(sys.argv[2])
    xyz, tri = W.torus(1 / 3, 1 / 6, 1000, 500)
    mesh = dg.Mesh(xyz, tri, device=0)
    f, b, d = W.vertex_edge_queries(xyz, tri, n, 5.0, seed=5, meridian=True)
    dev = torch.device("cuda", 0)
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dtype=dt)
    F, B, D = t(f, torch.int32), t(b, torch.float64), t(d, torch.float64)
    o = dict(face=torch.empty(n, dtype=torch.int32, device=dev), bary=torch.empty(n, 3, dtype=torch.float64, device=dev),
             dir=torch.empty(n, 3, dtype=torch.float64, device=dev), npoints=torch.empty(n, dtype=torch.int32, device=dev),
             crossings=torch.empty(n, dtype=torch.int32, device=dev), total_crossings=torch.zeros(1, dtype=torch.int64, device=dev))
    ts = []
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); mesh.trace_batch_device(F, B, D, o, max_steps=200000, sort_by_face=False); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    import hashlib
    h = hashlib.sha256()
    for k in ("face", "bary", "dir", "crossings"):
        h.update(o[k].cpu().numpy().tobytes())
    print(f"DG_FAN_PREFETCH={os.environ.get('DG_FAN_PREFETCH','-')} n={n} min {min(ts):.2f} ms  all {[round(x,1) for x in ts]}  sha {h.hexdigest()[:16]}", flush=True)
else:
    n = sys.argv[1] if len(sys.argv) > 1 else "200000"
    for v in ("0", "1", "0", "1"):
        subprocess.run([sys.executable, __file__, "child", n], env=dict(os.environ, DG_FAN_PREFETCH=v))
