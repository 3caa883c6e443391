"""Kernel durations of one small polyline call (run under ncu --metrics gpu__time_duration.sum)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import refapi
import paper_2603_15780_b200 as dg
rm = refapi.RefMesh.icosphere(4)
a = rm.arrays()
m = dg.Mesh(a["xyz"], a["tri"])
for batch in (1, 100, 1000, 100000):
    f, b, d = rm.sample_queries(42, batch, 0.1, np.pi / 2)
    for _ in range(2):
        m.trace_batch(f, b, d, record_polyline=True, poly_views=True)
        m.trace_batch(f, b, d)
