"""Wall-clock breakdown of the host-facing training step (resident batch) on pinned buffers.
usage: python scripts/e2e_breakdown.py [c2|c3] [n]"""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_15780_b200 as dg
from bench import make_workload

key = sys.argv[1] if len(sys.argv) > 1 else "c2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
xyz, tri, f, b, d, q = make_workload(key, n, 42)
mesh = dg.Mesh(xyz, tri, device=0)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
pe = lambda shape, dt: torch.empty(shape, dtype=dt).pin_memory().numpy()
hf, hb, hd, hg = pin(f), pin(b), pin(d), pin(q)
res = dg.TraceResult(face=pe(n, torch.int32), bary=pe((n, 3), torch.float64), dir=pe((n, 3), torch.float64),
                     traced=pe(n, torch.float64), requested=pe(n, torch.float64), term=pe(n, torch.uint8),
                     status=pe(n, torch.uint8), stall=pe(n, torch.uint8), npoints=pe(n, torch.int32),
                     crossings=pe(n, torch.int32))
gv = pe((n, 3), torch.float64)
batch = dg.Batch(mesh, n)

def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter(); fn(); ts.append((time.perf_counter() - t0) * 1e3)
    return min(ts), float(np.median(ts))

for s, bps in (("1", 0), ("4", 0), ("4", 3), ("6", 3), ("8", 3), ("8", 2), ("6", 2), ("5", 3)):
    os.environ["DG_BATCH_SLICES"] = s
    print(f"slices {s} blocks/SM {bps}: batch.trace {timed(lambda: batch.trace(hf, hb, hd, blocks_per_sm=bps, out=res))}  "
          f"batch.ep_backward {timed(lambda: batch.ep_backward(hg, grad_v=gv))}  "
          f"mesh.trace_batch {timed(lambda: mesh.trace_batch(hf, hb, hd, out=res))}", flush=True)
# copy-only references
dev = torch.device("cuda", 0)
tin = [torch.from_numpy(a) for a in (hf, hb, hd)]
din = [torch.empty_like(t, device=dev) for t in tin]
def h2d():
    for a, c in zip(tin, din): c.copy_(a, non_blocking=True)
    torch.cuda.synchronize()
print("H2D 52 B/geodesic:", timed(h2d))
outs = [torch.from_numpy(getattr(res, k)) for k in ("face", "bary", "dir", "traced", "requested", "term", "status", "stall", "npoints", "crossings")]
douts = [torch.empty_like(t, device=dev) for t in outs]
def d2h():
    for a, c in zip(outs, douts): a.copy_(c, non_blocking=True)
    torch.cuda.synchronize()
print("D2H 79 B/geodesic:", timed(d2h))
