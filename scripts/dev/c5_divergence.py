"""Where do GPU and reference part ways on config 5's vertex-to-vertex walks? (diagnostic)"""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2603_15780_b200 as dg, refapi
from paper_2603_15780_b200 import workloads as W
n = 2_000_000
xyz, tri, f, b, d = W.config5(n)
m = dg.Mesh(xyz, tri); rm = refapi.RefMesh.build(xyz, tri)
k = 600
idx = np.arange(k)
o = m.trace_batch(f[idx], b[idx], d[idx], record_polyline=True, max_steps=200000)
t = rm.trace_batch(f[idx], b[idx], d[idx], record_polyline=True, max_steps=200000)
same = 0; first = []; prev_vertex = 0; pos_ok = 0
diag = W.bbox_diagonal(xyz)
for i in range(k):
    a0, a1 = o.poly_offsets[i], o.poly_offsets[i + 1]; b0, b1 = t.poly_offsets[i], t.poly_offsets[i + 1]
    fa, fb = o.poly_face[a0:a1], t.poly_face[b0:b1]
    L = min(len(fa), len(fb))
    neq = np.nonzero(fa[:L] != fb[:L])[0]
    if len(neq) == 0 and len(fa) == len(fb):
        same += 1; continue
    j = int(neq[0]) if len(neq) else L
    first.append(j)
    pb = t.poly_bary[b0 + max(j - 1, 0)]
    pa = o.poly_bary[a0 + max(j - 1, 0)]
    prev_vertex += int((pb == 1.0).any() or (pa == 1.0).any() or (t.poly_bary[b0 + min(j, len(fb) - 1)] == 1.0).any() or (o.poly_bary[a0 + min(j, len(fa) - 1)] == 1.0).any())
    ea = m.embed(fa[:j], o.poly_bary[a0:a0 + j]); eb = m.embed(fb[:j], t.poly_bary[b0:b0 + j])
    pos_ok += int(np.abs(ea - eb).max() <= 1e-9 * diag) if j else 1
print("identical", same, "of", k, "; divergent", len(first), "first mismatch idx median", np.median(first) if first else None,
      "min", min(first) if first else None, "; mismatch adjacent to a vertex point:", prev_vertex, "; positions equal before it:", pos_ok)
vp_o = (o.poly_bary == 1.0).any(1).sum(); vp_t = (t.poly_bary == 1.0).any(1).sum()
print("vertex points ours", vp_o, "theirs", vp_t, "end distance median", np.median(np.linalg.norm(m.embed(o.face, o.bary) - m.embed(t.face, t.bary), axis=1)))
