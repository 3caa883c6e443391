"""Config-4 style stress: 64 meshes of 10 k - 200 k faces, 65 536 queries per mesh,
lengths log-uniform in [0.01, 2] x each mesh's bbox diagonal (divergence stress). Two ways to run it:
 (a) the reference's way -- concat_meshes (mesh.cpp:199-206) into ONE mesh, one batch;
 (b) one device mesh per component (each small enough for crossing records), one batch per mesh.
usage: python scripts/bench_c4.py [meshes=64] [queries_per_mesh=65536]"""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_15780_b200 as dg
from paper_2603_15780_b200 import workloads as W

M = int(sys.argv[1]) if len(sys.argv) > 1 else 64
Q = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
rng = np.random.default_rng(4)
parts = []
for i in range(M):
    kind = i % 3
    if kind == 0:
        na = int(rng.integers(100, 448)); xyz, tri = W.torus(1 / 3, 1 / 6, na, na // 2, noise=0.05, seed=i)   # 10 k - 200 k faces
    elif kind == 1:
        xyz, tri = W.bumpy_sphere(int(rng.integers(5, 7)), amplitude=0.05 + 0.05 * rng.random())            # 20 k / 82 k faces
    else:
        xyz, tri = W.icosphere(int(rng.integers(5, 7)))
    parts.append((xyz * (0.5 + rng.random()), tri))
faces = [len(t) for _, t in parts]
print(f"{M} meshes, faces {min(faces)}..{max(faces)}, total {sum(faces)}", flush=True)
queries = []
for i, (xyz, tri) in enumerate(parts):
    d = W.bbox_diagonal(xyz)
    queries.append(W.sample_queries(xyz, tri, Q, (0.01 * d, 2.0 * d), seed=100 + i))

dev = torch.device("cuda", 0)
t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dtype=dt)
def outs(k):
    return dict(face=torch.empty(k, dtype=torch.int32, device=dev), bary=torch.empty(k, 3, dtype=torch.float64, device=dev),
                dir=torch.empty(k, 3, dtype=torch.float64, device=dev), term=torch.empty(k, dtype=torch.uint8, device=dev),
                total_crossings=torch.zeros(1, dtype=torch.int64, device=dev))

# (a) one concatenated mesh
t0 = time.perf_counter()
voff = np.cumsum([0] + [len(x) for x, _ in parts])
foff = np.cumsum([0] + faces)
XYZ = np.concatenate([x for x, _ in parts]); TRI = np.concatenate([tr + voff[i] for i, (_, tr) in enumerate(parts)]).astype(np.int32)
big = dg.Mesh(XYZ, TRI, device=0)
print(f"(a) concatenated: derive + upload {time.perf_counter() - t0:.1f} s, {big.device_bytes / 1e6:.0f} MB on device, "
      f"crossing records: {big.has_transport_cache}", flush=True)
F = t(np.concatenate([q[0] + foff[i] for i, q in enumerate(queries)]), torch.int32)
B = t(np.concatenate([q[1] for q in queries]), torch.float64); D = t(np.concatenate([q[2] for q in queries]), torch.float64)
o = outs(len(F))
ts = []
for _ in range(3):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); big.trace_batch_device(F, B, D, o); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
cr_a = int(o["total_crossings"].item())
print(f"(a) {len(F)} geodesics, {cr_a / len(F):.1f} crossings/trace: {min(ts):.2f} ms = {cr_a / min(ts) / 1e6:.2f} Gcross/s, "
      f"terminated by max_steps: {int((o['term'] == 2).sum())}", flush=True)
ref_face, ref_bary = o["face"].clone(), o["bary"].clone()
del big

# (b) one device mesh per component, batches on separate streams
meshes = [dg.Mesh(x, tr, device=0) for x, tr in parts]
ins = [(t(q[0], torch.int32), t(q[1], torch.float64), t(q[2], torch.float64)) for q in queries]
os_ = [outs(Q) for _ in range(M)]
streams = [torch.cuda.Stream() for _ in range(8)]
maxs = int(10 * np.sqrt(sum(faces))) + 100   # the step limit the concatenated mesh implies (tracer.cpp:543)
ts = []
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i, m in enumerate(meshes):
        with torch.cuda.stream(streams[i % 8]):
            m.trace_batch_device(*ins[i], os_[i], max_steps=maxs)
    torch.cuda.synchronize(); ts.append((time.perf_counter() - t0) * 1e3)
cr_b = sum(int(x["total_crossings"].item()) for x in os_)
same = all(torch.equal(os_[i]["bary"], ref_bary[i * Q:(i + 1) * Q]) and
           torch.equal(os_[i]["face"] + int(foff[i]), ref_face[i * Q:(i + 1) * Q]) for i in range(M))
print(f"(b) per-mesh, {sum(m.has_transport_cache for m in meshes)}/{M} with crossing records: {min(ts):.2f} ms = "
      f"{cr_b / min(ts) / 1e6:.2f} Gcross/s; crossings equal: {cr_a == cr_b}; results bit-equal to (a): {same}", flush=True)
