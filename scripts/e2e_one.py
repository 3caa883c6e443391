"""One measurement of the host-facing forward call (resident batch, pinned buffers, c2) under the current
DG_BATCH_SLICES / DG_BATCH_SLICE_SHAPE; driven by scripts/slice_sweep.py."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_15780_b200 as dg
from bench import make_workload
n = 1_000_000
xyz, tri, f, b, d, q = make_workload("c2", n, 42)
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
def timed(fn, reps=7):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter(); fn(); ts.append((time.perf_counter() - t0) * 1e3)
    return min(ts), float(np.median(ts))
t = timed(lambda: batch.trace(hf, hb, hd, out=res)); e = timed(lambda: batch.ep_backward(hg, grad_v=gv))
print(f"batch.trace min {t[0]:.3f} median {t[1]:.3f} ms   batch.ep_backward min {e[0]:.3f} median {e[1]:.3f} ms")
