"""Host-facing training step on pinned buffers: streamed forward (default) against the sliced pipeline (dev)."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
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
def timed(fn, reps=7):
    fn(); fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter(); fn(); ts.append((time.perf_counter() - t0) * 1e3)
    return f"{min(ts):.3f} / {float(np.median(ts)):.3f}"
def step():
    batch.trace(hf, hb, hd, out=res); batch.ep_backward(hg, grad_v=gv)
for label, env in (("streamed", None), ("sliced x4", "4"), ("streamed", None)):
    if env: os.environ["DG_BATCH_SLICES"] = env
    else: os.environ.pop("DG_BATCH_SLICES", None)
    print(f"{label:10s} batch.trace {timed(lambda: batch.trace(hf, hb, hd, out=res))} ms   forward + EP step {timed(step)} ms (min / median)", flush=True)
