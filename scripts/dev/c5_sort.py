"""c5 (half vertex walkers, half random): scheduling order (diagnostic)."""
import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2603_15780_b200 as dg
from paper_2603_15780_b200 import workloads as W
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
xyz, tri, f, b, d = W.config5(n)
mesh = dg.Mesh(xyz, tri, device=0)
dev = torch.device("cuda", 0)
t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dtype=dt)
def run(name, f, b, d, **kw):
    F, B, D = t(f, torch.int32), t(b, torch.float64), t(d, torch.float64)
    k = len(f)
    o = dict(face=torch.empty(k, dtype=torch.int32, device=dev), bary=torch.empty(k, 3, dtype=torch.float64, device=dev),
             total_crossings=torch.zeros(1, dtype=torch.int64, device=dev))
    ts = []
    for _ in range(2):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); mesh.trace_batch_device(F, B, D, o, max_steps=200000, **kw); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    cr = int(o["total_crossings"].item())
    print(f"{name:44s} {min(ts):9.2f} ms {cr/min(ts)/1e6:7.2f} Gcross/s", flush=True)
run("sort AUTO (by face)", f, b, d)
run("sort off (vertex half first)", f, b, d, sort_by_face=False)
h = n // 2
run("vertex half alone", f[:h], b[:h], d[:h], sort_by_face=False)
run("random half alone, sorted", f[h:], b[h:], d[h:])
run("random half alone, unsorted", f[h:], b[h:], d[h:], sort_by_face=False)
perm = np.random.default_rng(0).permutation(n)
run("shuffled, sort off", f[perm], b[perm], d[perm], sort_by_face=False)
run("shuffled, sort AUTO", f[perm], b[perm], d[perm])
