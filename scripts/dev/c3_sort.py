"""c3 lone forward: plain order vs start-face order (diagnostic)."""
import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2603_15780_b200 as dg
from bench import make_workload
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
xyz, tri, f, b, d, q = make_workload("c3", n, 42)
mesh = dg.Mesh(xyz, tri, device=0)
dev = torch.device("cuda", 0)
t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dtype=dt)
def run(name, f, b, d, **kw):
    F, B, D = t(f, torch.int32), t(b, torch.float64), t(d, torch.float64)
    k = len(f)
    o = dict(face=torch.empty(k, dtype=torch.int32, device=dev), bary=torch.empty(k, 3, dtype=torch.float64, device=dev),
             dir=torch.empty(k, 3, dtype=torch.float64, device=dev), total_crossings=torch.zeros(1, dtype=torch.int64, device=dev))
    ts = []
    for _ in range(4):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); mesh.trace_batch_device(F, B, D, o, **kw); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    cr = int(o["total_crossings"].item())
    print(f"{name:40s} {min(ts):8.2f} ms {cr/min(ts)/1e6:7.2f} Gcross/s", flush=True)
    return o
run("plain order", f, b, d)
run("sort_by_face (device radix sort)", f, b, d, sort_by_face=True)
order = np.argsort(f, kind="stable")
run("pre-sorted by face on host", f[order], b[order], d[order])
for w in ("loads", "coop", "tma"):
    run(f"pre-sorted, walker={w}", f[order], b[order], d[order], walker=w)
# Morton order of face centroids in (alpha, beta) parameter space of the torus grid
i = (np.arange(len(tri)) // 2) // 500; j = (np.arange(len(tri)) // 2) % 500
def part1by1(x):
    x = x.astype(np.uint64) & 0xffff
    x = (x | (x << 8)) & 0x00FF00FF; x = (x | (x << 4)) & 0x0F0F0F0F; x = (x | (x << 2)) & 0x33333333; x = (x | (x << 1)) & 0x55555555
    return x
key = part1by1(i) | (part1by1(j) << 1)
order = np.argsort(key[f], kind="stable")
run("queries in Morton order of start face", f[order], b[order], d[order])
for w in ("loads", "coop"):
    run(f"Morton, walker={w}", f[order], b[order], d[order], walker=w)
