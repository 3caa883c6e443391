import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))); sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "scripts"))
import paper_2603_15780_b200 as dg
from paper_2603_15780_b200 import workloads as W
import fuzz_walkers as FZ
rng = np.random.default_rng(11)
n = 30000
for r in range(300):
    unit_xyz, tri, scale = FZ.random_mesh(rng)
    xyz = unit_xyz * scale
    try:
        meshes = [dg.Mesh(xyz, tri, transport_cache=c) for c in (True, False)]
    except dg.DgError:
        continue
    diag = W.bbox_diagonal(unit_xyz)
    f, b, d = W.sample_queries(unit_xyz, tri, n, (1e-9 * diag, 3.0 * diag), seed=int(rng.integers(1 << 30)))
    k = n // 20
    b[:k] = np.eye(3)[rng.integers(0, 3, k)]
    b[k:2 * k] = np.array([0.5, 0.5, 0.0])[rng.permuted(np.tile(np.arange(3), (k, 1)), axis=1)]
    e = unit_xyz[tri[f[2 * k:3 * k], 1]] - unit_xyz[tri[f[2 * k:3 * k], 0]]
    d[2 * k:3 * k] = e * (np.linalg.norm(d[2 * k:3 * k], axis=1) / np.linalg.norm(e, axis=1))[:, None]
    d *= scale
    d[3 * k] = 0.0; f[3 * k + 1] = -5; b[3 * k + 2] = [2.0, -0.5, -0.5]; d[3 * k + 3] = [np.nan, 1.0, 0.0]
    max_steps = int(rng.choice([0, 0, 5, 60]))
    pay = rng.normal(size=(n, 3)) * scale
    eff = max_steps if max_steps > 0 else int(10 * np.sqrt(len(tri))) + 100
    m = meshes[0]
    for hole in (False, True):
        t = m.trace_batch(f, b, d, max_steps=max_steps, hole_avoidance=hole, walker="generic")
        over = t.npoints - (eff + 2)
        if over.max() > 0:
            i = int(np.argmax(over))
            print(f"round {r} faces {len(tri)} scale {scale:g} max_steps {eff} hole {hole}: npoints {t.npoints[i]} at query {i} (kind: {'vertex' if i < k else 'edge' if i < 2*k else 'along-edge' if i < 3*k else 'random'}) term {t.term[i]} status {t.status[i]} bary {b[i]} ", flush=True)
print("done")
