"""EP backward of the resident batch on pinned buffers by slice shape (dev)."""
import os, sys, time, subprocess
if len(sys.argv) > 1:
    import numpy as np, torch
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
    import paper_2603_15780_b200 as dg
    from bench import make_workload
    n = 1_000_000
    xyz, tri, f, b, d, q = make_workload("c2", n, 42)
    mesh = dg.Mesh(xyz, tri, device=0)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
    hf, hb, hd, hg = pin(f), pin(b), pin(d), pin(q)
    gv = torch.empty((n, 3), dtype=torch.float64).pin_memory().numpy()
    batch = dg.Batch(mesh, n)
    batch.trace(hf, hb, hd)
    ts = []
    for _ in range(12):
        t0 = time.perf_counter(); batch.ep_backward(hg, grad_v=gv); ts.append((time.perf_counter() - t0) * 1e3)
    print(sys.argv[1], f"ep_backward {min(ts):.3f} / {sorted(ts)[len(ts)//2]:.3f} ms", flush=True)
else:
    for shape in ("", "1,3,3,1", "1,2,2,1", "1,4,4,1", "2,3,3,1", "1,2,4,2"):
        env = dict(os.environ)
        if shape: env["DG_BATCH_EP_SHAPE"] = shape
        subprocess.run([sys.executable, __file__, shape or "equal"], env=env)
