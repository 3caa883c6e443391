"""Where the host-facing (DG_MEM_HOST) step spends its time."""
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
hf, hb, hd, hq = pin(f), pin(b), pin(d), pin(q)
res = dg.TraceResult(face=pe(n, torch.int32), bary=pe((n, 3), torch.float64), dir=pe((n, 3), torch.float64),
                     traced=pe(n, torch.float64), requested=pe(n, torch.float64), term=pe(n, torch.uint8),
                     status=pe(n, torch.uint8), stall=pe(n, torch.uint8), npoints=pe(n, torch.int32),
                     crossings=pe(n, torch.int32))
hg, hgv = pe((n, 3), torch.float64), pe((n, 3), torch.float64)
Xh = xyz[tri]
for it in range(4):
    t0 = time.perf_counter(); r = mesh.trace_batch(hf, hb, hd, out=res)
    t1 = time.perf_counter(); np.einsum("nk,nkd->nd", r.bary, Xh[r.face], out=hg); np.subtract(hg, hq, out=hg); np.multiply(hg, 2.0, out=hg)
    t2 = time.perf_counter(); mesh.ep_backward(hf, hd, r.face, r.dir, hg, grad_v=hgv)
    t3 = time.perf_counter()
    print(f"trace_batch(host) {1e3*(t1-t0):7.2f} ms | loss-gradient glue (numpy) {1e3*(t2-t1):7.2f} ms | ep_backward(host) {1e3*(t3-t2):7.2f} ms")
# pageable
t0 = time.perf_counter(); r = mesh.trace_batch(f, b, d); t1 = time.perf_counter()
print(f"trace_batch pageable in/out {1e3*(t1-t0):.2f} ms")
