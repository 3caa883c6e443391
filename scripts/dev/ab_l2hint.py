"""A/B of the record load's L2 prefetch-size hint (build/variants/l2_128.so against the in-tree build) on meshes
beyond the L2: noisy 1 M-face torus (config 3) in request and start-face order, per-lane loads and AUTO; config 4."""
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
        print(f"{sys.argv[2]:8s} {name:44s} min {min(ts[1:]):9.3f} ms  sha {h.hexdigest()[:12]}", flush=True)
    xyz, tri = W.torus(1 / 3, 1 / 6, 1000, 500, noise=0.1)
    mesh = dg.Mesh(xyz, tri, device=0)
    L = 0.5 * float(np.linalg.norm(xyz.max(0) - xyz.min(0)))
    f, b, d = W.sample_queries(xyz, tri, 1_000_000, L, seed=42)
    for sort in (False, True):
        for walker in ("auto", "loads", "coop"):
            run(f"c3 1M sort_by_face={sort} walker={walker}", mesh, f, b, d, sort_by_face=sort, walker=walker)
    run("c3 1M tolerance lane, face order", mesh, f, b, d, sort_by_face=True, lane="fast")
    f5, b5, d5 = W.sample_queries(xyz, tri, 200_000, 5.0, seed=9)
    for walker in ("loads", "coop"):
        run(f"torus 200k x 5 diameters walker={walker}", mesh, f5, b5, d5, sort_by_face=True, walker=walker, max_steps=200000)
    del mesh
    torch.cuda.empty_cache()
    xyz, tri, f, b, d, _ = W.config4()
    mesh = dg.Mesh(xyz, tri, device=0)
    for walker in ("auto", "loads", "coop"):
        run(f"c4 4.2M walker={walker}", mesh, f, b, d, walker=walker)
else:
    for name, lib in (("head", ""), ("l2_128", "build/variants/l2_128.so"), ("head", ""), ("l2_128", "build/variants/l2_128.so")):
        env = dict(os.environ)
        if lib: env["DG_B200_LIB"] = os.path.join(ROOT, lib)
        subprocess.run([sys.executable, __file__, "child", name], env=env)
