"""Fan-walk prefetch (DG_FAN_PREFETCH) on config 5's vertex-to-vertex walkers, the general walker on the same, and
the controls (c2 forward, 1 M-face torus): time and bits, off against on (same library, runtime flag)."""
import os, sys, subprocess, hashlib
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import torch
    sys.path.insert(0, ROOT)
    import paper_2603_15780_b200 as dg
    from paper_2603_15780_b200 import workloads as W
    dev = torch.device("cuda", 0)
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dtype=dt)
    tag = "prefetch=" + os.environ.get("DG_FAN_PREFETCH", "-")
    def run(name, mesh, f, b, d, **kw):
        n = len(f)
        F, B, D = t(f, torch.int32), t(b, torch.float64), t(d, torch.float64)
        o = dict(face=torch.empty(n, dtype=torch.int32, device=dev), bary=torch.empty(n, 3, dtype=torch.float64, device=dev),
                 dir=torch.empty(n, 3, dtype=torch.float64, device=dev), npoints=torch.empty(n, dtype=torch.int32, device=dev),
                 crossings=torch.empty(n, dtype=torch.int32, device=dev), total_crossings=torch.zeros(1, dtype=torch.int64, device=dev))
        ts = []
        for _ in range(4):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); mesh.trace_batch_device(F, B, D, o, **kw); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
        h = hashlib.sha256()
        for k in ("face", "bary", "dir", "crossings"):
            h.update(o[k].cpu().numpy().tobytes())
        print(f"{tag:12s} {name:30s} min {min(ts[1:]):9.3f} ms  sha {h.hexdigest()[:12]}", flush=True)
    xyz, tri = W.torus(1 / 3, 1 / 6, 1000, 500)
    mesh = dg.Mesh(xyz, tri, device=0)
    f, b, d = W.vertex_edge_queries(xyz, tri, 200_000, 5.0, seed=5, meridian=True)
    run("c5 vertex walkers 200k", mesh, f, b, d, max_steps=200000, sort_by_face=False)
    run("c5 vertex walkers, generic", mesh, f, b, d, max_steps=200000, sort_by_face=False, generic_walker=True)
    f2, b2, d2 = W.sample_queries(xyz, tri, 1_000_000, 0.5 * float(np.linalg.norm(xyz.max(0) - xyz.min(0))), seed=42)
    run("torus random 1M x 0.5 diag", mesh, f2, b2, d2)
    del mesh
    xyz, tri = W.bumpy_sphere(6)
    mesh = dg.Mesh(xyz, tri, device=0)
    f2, b2, d2 = W.sample_queries(xyz, tri, 1_000_000, 0.5 * float(np.linalg.norm(xyz.max(0) - xyz.min(0))), seed=42)
    run("c2 forward 1M", mesh, f2, b2, d2)
else:
    for v in ("0", "1", "0", "1"):
        subprocess.run([sys.executable, __file__, "child"], env=dict(os.environ, DG_FAN_PREFETCH=v))
