"""Synthetic meshes and query batches of the BASELINE.json configurations.

Pure numpy, host side, build-once data generation -- not part of the compute path. The
generators produce the same surfaces as the reference's fixtures (make_icosphere / make_torus,
proj/src/oracles.cpp:183-247) but vectorised; the samplers draw area-uniform starts with an
O(log F) CDF search instead of the reference's O(F) scan (io.cpp:168-178) and the same
in-plane direction construction as sample_tangent (io.cpp:184-197).
"""
from __future__ import annotations

import numpy as np


def icosphere(subdiv: int):
    t = (1.0 + np.sqrt(5.0)) / 2.0
    v = np.array([[-1, t, 0], [1, t, 0], [-1, -t, 0], [1, -t, 0], [0, -1, t], [0, 1, t], [0, -1, -t], [0, 1, -t],
                  [t, 0, -1], [t, 0, 1], [-t, 0, -1], [-t, 0, 1]], float)
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    f = np.array([[0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11], [1, 5, 9], [5, 11, 4], [11, 10, 2],
                  [10, 7, 6], [7, 1, 8], [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9], [4, 9, 5],
                  [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]], np.int64)
    for _ in range(subdiv):
        nv = len(v)
        e = np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]])
        key = np.minimum(e[:, 0], e[:, 1]) * nv + np.maximum(e[:, 0], e[:, 1])
        uniq, inv = np.unique(key, return_inverse=True)
        a, b = uniq // nv, uniq % nv
        mid = v[a] + v[b]
        mid /= np.linalg.norm(mid, axis=1, keepdims=True)
        v = np.concatenate([v, mid])
        m = nv + inv.reshape(3, -1)  # ab, bc, ca per face
        ab, bc, ca = m[0], m[1], m[2]
        f = np.concatenate([np.stack([f[:, 0], ab, ca], 1), np.stack([f[:, 1], bc, ab], 1),
                            np.stack([f[:, 2], ca, bc], 1), np.stack([ab, bc, ca], 1)])
    return v, f.astype(np.int32)


def bumpy_sphere(subdiv: int = 6, amplitude: float = 0.08):
    """Config 2: icosphere scaled radially by 1 + a sin(5x) sin(4y) cos(3z)."""
    v, f = icosphere(subdiv)
    s = 1.0 + amplitude * np.sin(5 * v[:, 0]) * np.sin(4 * v[:, 1]) * np.cos(3 * v[:, 2])
    return v * s[:, None], f


def torus(r_major: float, r_minor: float, n_alpha: int, n_beta: int, noise: float = 0.0, seed: int = 7):
    """make_torus connectivity; `noise` displaces each vertex along its analytic normal by
    U(-noise, noise) x mean edge length (config 3)."""
    a = 2.0 * np.pi * np.arange(n_alpha) / n_alpha
    b = 2.0 * np.pi * np.arange(n_beta) / n_beta
    A, B = np.meshgrid(a, b, indexing="ij")
    ring = r_major + r_minor * np.cos(B)
    v = np.stack([ring * np.cos(A), ring * np.sin(A), r_minor * np.sin(B)], -1).reshape(-1, 3)
    i, j = np.meshgrid(np.arange(n_alpha), np.arange(n_beta), indexing="ij")
    vid = lambda ii, jj: (ii % n_alpha) * n_beta + (jj % n_beta)
    f0 = np.stack([vid(i, j), vid(i + 1, j), vid(i + 1, j + 1)], -1).reshape(-1, 3)
    f1 = np.stack([vid(i, j), vid(i + 1, j + 1), vid(i, j + 1)], -1).reshape(-1, 3)
    f = np.stack([f0, f1], 1).reshape(-1, 3).astype(np.int32)
    if noise > 0:
        nrm = np.stack([np.cos(B) * np.cos(A), np.cos(B) * np.sin(A), np.sin(B)], -1).reshape(-1, 3)
        e = v[f[:, [1, 2, 0]]] - v[f]
        mean_edge = np.linalg.norm(e, axis=-1).mean()
        rng = np.random.default_rng(seed)
        v = v + nrm * (rng.uniform(-noise, noise, len(v)) * mean_edge)[:, None]
    return v, f


def bbox_diagonal(xyz):
    return float(np.linalg.norm(xyz.max(0) - xyz.min(0)))


def sample_queries(xyz, tri, n: int, length, seed: int = 42, face_normals=None):
    """n area-uniform starts with uniform in-plane directions; `length` is a scalar or a
    (lo, hi) range sampled log-uniformly. Returns face[int32 n], bary[n,3], dir[n,3]."""
    rng = np.random.default_rng(seed)
    X = xyz[tri]
    e1, e2 = X[:, 1] - X[:, 0], X[:, 2] - X[:, 0]
    nrm = np.cross(e1, e2)
    area2 = np.linalg.norm(nrm, axis=1)
    cdf = np.cumsum(area2)
    face = np.searchsorted(cdf, rng.uniform(0, cdf[-1], n)).clip(0, len(tri) - 1).astype(np.int32)
    r1 = np.sqrt(rng.uniform(size=n))
    r2 = rng.uniform(size=n)
    bary = np.stack([1.0 - r1, r1 * (1.0 - r2), r1 * r2], 1)
    nf = nrm[face] / area2[face, None] if face_normals is None else face_normals[face]
    t1 = e1[face] / np.linalg.norm(e1[face], axis=1, keepdims=True)
    t1 = t1 - nf * np.einsum("nd,nd->n", t1, nf)[:, None]
    t1 /= np.linalg.norm(t1, axis=1, keepdims=True)
    t2 = np.cross(nf, t1)
    phi = 2.0 * np.pi * rng.uniform(size=n)
    if np.isscalar(length):
        ln = np.full(n, float(length))
    else:
        lo, hi = length
        ln = np.exp(rng.uniform(np.log(lo), np.log(hi), n))
    d = (t1 * np.cos(phi)[:, None] + t2 * np.sin(phi)[:, None]) * ln[:, None]
    return face, bary, d


def vertex_edge_queries(xyz, tri, n: int, length: float, seed: int = 5, meridian: bool = False):
    """Config-5 style starts: exactly at a vertex, aimed exactly along an incident edge. meridian=True (torus()
    connectivity only): the odd faces' edge corner 0 -> corner 2, which runs along a meridian circle -- a chain of
    edges the straightest geodesic follows vertex to vertex (reference, 1000 x 500 torus, length 5: median 2 388
    vertex points of ~3 000 per trace); the default edge corner 0 -> corner 1 of a random face is left after the
    first vertex on most faces."""
    rng = np.random.default_rng(seed)
    if meridian:
        face = (2 * rng.integers(0, len(tri) // 2, n) + 1).astype(np.int32)
        to = 2
    else:
        face = rng.integers(0, len(tri), n).astype(np.int32)
        to = 1
    bary = np.zeros((n, 3))
    bary[:, 0] = 1.0
    d = xyz[tri[face, to]] - xyz[tri[face, 0]]
    d *= (length / np.linalg.norm(d, axis=1))[:, None]
    return face, bary, d


def concat(parts):
    """concat_meshes semantics (mesh.cpp:199-206) on arrays: vertices appended, face vertex ids offset,
    faces in part order. Returns xyz, tri, vertex offsets [len+1], face offsets [len+1]."""
    voff = np.cumsum([0] + [len(x) for x, _ in parts])
    foff = np.cumsum([0] + [len(t) for _, t in parts])
    xyz = np.concatenate([x for x, _ in parts])
    tri = np.concatenate([t.astype(np.int64) + voff[i] for i, (_, t) in enumerate(parts)]).astype(np.int32)
    return xyz, tri, voff, foff


def config4(meshes: int = 64, queries_per_mesh: int = 65536, seed: int = 4):
    """Config 4: `meshes` components of 10 k - 200 k faces (six noisy tori of uniformly drawn
    face count to one bumpy sphere and one icosphere; a fixed seed-chosen list, about 6 M faces in all, each scaled by a factor in [0.5, 1.5]) concatenated into ONE
    mesh; `queries_per_mesh` queries on each, lengths log-uniform in [0.01, 2] x that component's bbox
    diagonal (divergence stress). Returns xyz, tri, face, bary, dir, face offsets."""
    rng = np.random.default_rng(seed)
    parts = []
    for i in range(meshes):
        kind = i % 8
        if kind == 0:
            xyz, tri = icosphere(int(rng.integers(5, 7)))                         # 20 k / 82 k faces
        elif kind == 1:
            xyz, tri = bumpy_sphere(6, amplitude=0.05 + 0.05 * rng.random())      # 82 k
        else:
            na = int(round(np.sqrt(rng.uniform(10_000, 200_000))))                # na x na/2 x 2 = 10 k - 200 k faces
            xyz, tri = torus(1 / 3, 1 / 6, na, na // 2, noise=0.05, seed=i)
        parts.append((xyz * (0.5 + rng.random()), tri))
    xyz, tri, voff, foff = concat(parts)
    fs, bs, ds = [], [], []
    for i, (x, t) in enumerate(parts):
        diag = bbox_diagonal(x)
        f, b, d = sample_queries(x, t, queries_per_mesh, (0.01 * diag, 2.0 * diag), seed=100 + i)
        fs.append(f + np.int32(foff[i])); bs.append(b); ds.append(d)
    return xyz, tri, np.concatenate(fs).astype(np.int32), np.concatenate(bs), np.concatenate(ds), foff


def config5(n: int, seed: int = 5, noise: float = 0.0):
    """Config 5: the 1 M-face torus, n queries of length 5 x the outer diameter (= 5.0
    for make_torus(1/3, 1/6)), the first half exactly at vertices aimed exactly along an incident (meridian) edge -- vertex-to-vertex walks --,
    the second half random. To be traced with max_steps = 200 000 on both sides."""
    xyz, tri = torus(1 / 3, 1 / 6, 1000, 500, noise=noise, seed=7)
    fv, bv, dv = vertex_edge_queries(xyz, tri, n // 2, 5.0, seed=seed, meridian=True)
    fr, br, dr = sample_queries(xyz, tri, n - n // 2, 5.0, seed=seed + 4)
    return xyz, tri, np.concatenate([fv, fr]), np.concatenate([bv, br]), np.concatenate([dv, dr])


C5_MAX_STEPS = 200_000
