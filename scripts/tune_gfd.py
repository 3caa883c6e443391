"""Device-resident timing of the GFD backward (with the forward results as its base traces) on the c2 / c3
workloads: usage python scripts/tune_gfd.py [c2|c3] [geodesics]. DG_GFD_SIBLINGS=0 / DG_FAST_GATHER=loads|tma|coop select
the round-2 schedule and the gather."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_15780_b200 as dg
from bench import make_workload
key = sys.argv[1] if len(sys.argv) > 1 else "c3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1000000
if key.startswith("torus:"):   # torus:NA = noisy NA x NA/2 torus, NA^2 faces
    from paper_2603_15780_b200 import workloads as W
    na = int(key.split(":")[1])
    xyz, tri = W.torus(1 / 3, 1 / 6, na, na // 2, noise=0.1, seed=7)
    f, b, d = W.sample_queries(xyz, tri, n, 0.5 * W.bbox_diagonal(xyz), seed=42)
    q = np.random.default_rng(43).normal(size=(n, 3))
else:
    xyz, tri, f, b, d, q = make_workload(key, n, 42)
mesh = dg.Mesh(xyz, tri, device=0)
dev = torch.device("cuda", 0)
t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dtype=dt)
F, B, D, G = t(f, torch.int32), t(b, torch.float64), t(d, torch.float64), t(q, torch.float64)
o = dict(face=torch.empty(n, dtype=torch.int32, device=dev), bary=torch.empty(n, 3, dtype=torch.float64, device=dev),
         dir=torch.empty(n, 3, dtype=torch.float64, device=dev), term=torch.empty(n, dtype=torch.uint8, device=dev),
         status=torch.empty(n, dtype=torch.uint8, device=dev), total_crossings=torch.zeros(1, dtype=torch.int64, device=dev))
jv, jp = (torch.empty(n, 4, dtype=torch.float64, device=dev) for _ in range(2))
gv, gp = (torch.empty(n, 3, dtype=torch.float64, device=dev) for _ in range(2))
eps = mesh.default_gfd_eps()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
tf, tg, tn = [], [], []
for _ in range(4):
    flush.fill_(1)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record(); mesh.trace_batch_device(F, B, D, o); e[1].record()
    mesh.gfd_device(F, B, D, eps, eps, G, jv, jp, gv, gp, base=o); e[2].record(); torch.cuda.synchronize()
    tf.append(e[0].elapsed_time(e[1])); tg.append(e[1].elapsed_time(e[2]))
    check = float(jv.sum() + jp.sum())
    flush.fill_(1)
    e[0].record(); mesh.gfd_device(F, B, D, eps, eps, G, jv, jp, gv, gp); e[1].record(); torch.cuda.synchronize()
    tn.append(e[0].elapsed_time(e[1]))
    assert float(jv.sum() + jp.sum()) == check
cr = int(o["total_crossings"].item()) // 1
print(f"{key} n={n} gather={os.environ.get('DG_FAST_GATHER', mesh.gather)} siblings={os.environ.get('DG_GFD_SIBLINGS', '3')} "
      f"forward {min(tf):.2f} ms  gfd with base {min(tg):.2f} ms  gfd alone {min(tn):.2f} ms  checksum {check:.17g}", flush=True)
