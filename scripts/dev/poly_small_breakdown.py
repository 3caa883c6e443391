"""Where a small polyline batch spends its time: Python harness vs the C call, both sides (dev diagnostic)."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import refapi
import paper_2603_15780_b200 as dg
from paper_2603_15780_b200 import capi

acc = {}
def wrap(L, name):
    fn = getattr(L, name)
    def w(*a):
        t0 = time.perf_counter(); r = fn(*a); acc[name] = acc.get(name, 0.0) + time.perf_counter() - t0
        return r
    setattr(L, name, w)

wrap(capi.lib(), "dg_trace_polylines"); wrap(capi.lib(), "dg_trace_batch"); wrap(refapi.lib(), "ref_trace_batch")
rm = refapi.RefMesh.icosphere(4)
a = rm.arrays()
m = dg.Mesh(a["xyz"], a["tri"])
for batch in (1, 100, 300, 1000, 2000, 10000, 100000):
    f, b, d = rm.sample_queries(42, batch, 0.1, np.pi / 2)
    fns = {"ref_parallel": lambda: rm.trace_batch(f, b, d, record_polyline=True, workers=0),
           "gpu_poly": lambda: m.trace_batch(f, b, d, record_polyline=True, poly_views=True),
           "gpu_nopoly": lambda: m.trace_batch(f, b, d)}
    for k, fn in fns.items():
        fn(); fn()
        reps = 20 if batch <= 10000 else 5
        ts, cs = [], []
        for _ in range(reps):
            acc.clear()
            t0 = time.perf_counter(); r = fn(); ts.append(time.perf_counter() - t0); cs.append(sum(acc.values()))
        extra = f" points {int(r.npoints.sum())}" if k == "gpu_poly" else ""
        print(f"batch {batch:6d} {k:13s} total {np.median(ts)*1e3:8.3f} ms   C call {np.median(cs)*1e3:8.3f} ms{extra}", flush=True)
