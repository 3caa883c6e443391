"""BASELINE.json's configurations 3, 4 and 5 AT THEIR STATED SIZES against the UNMODIFIED reference
(oracle/_ref), through the C-ABI (VERDICT r1 "next round" item 1).

The GPU traces the whole workload (per-GPU share for config 5); the reference, which needs minutes
for the full batch on host cores, checks a prefix of the query stream plus a random sample of it
(8d "CPU baseline": parity is checked on the timed prefix plus a random sample). Results of the
sample are taken OUT OF THE FULL-BATCH RUN, so the comparison covers the schedule and the gather
variant the full-size launch really used, not a small re-run.

Bars: edge-only f64 traces bit-equal (faces, barycentrics, directions, lengths, termination);
vertex-heavy traces identical face sequences + 1e-9 x bbox diagonal; GFD jv/jp within 1e-5 of the
largest entry, degraded flags and frames bit-equal (diff.cpp:273-326), both round-2 schedules."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_15780_b200 import workloads as W  # noqa: E402

pytestmark = pytest.mark.gpu


def prefix_and_sample(n, k_prefix, k_random, seed):
    rng = np.random.default_rng(seed)
    return np.concatenate([np.arange(k_prefix), np.sort(rng.choice(np.arange(k_prefix, n), k_random, replace=False))])


def test_config3_forward_and_gfd_on_the_1m_face_torus(gpu, ref):
    """Config 3: 1 M-face noisy torus, bench stream (seed 42), forward + GFD with the default eps.
    6 000-sample prefix: jv / jp <= 1e-5 relative, degraded flags and frames bit-equal, pulled-back
    gradients cos >= 0.999999, for the sibling schedule, the plain schedule and the known-base form."""
    from bench import make_workload
    n = 6000
    xyz, tri, f, b, d, q = make_workload("c3", n, 42)
    m = gpu.Mesh(xyz, tri)
    assert m.nf == 1_000_000 and m.has_transport_cache and m.gather == "coop"
    rm = ref.RefMesh.build(xyz, tri)
    assert m.default_gfd_eps() == rm.default_gfd_eps()
    fwd = m.trace_batch(f, b, d)
    theirs_fwd = rm.trace_batch(f, b, d)
    for k in ("face", "bary", "dir", "traced", "term", "status"):
        assert np.array_equal(getattr(fwd, k), getattr(theirs_fwd, k)), k
    g = 2.0 * (m.embed(fwd.face, fwd.bary) - q)      # gradcheck.cpp:88
    theirs = rm.gfd(f, b, d, g=g)                    # gfd_batched_many, diff.cpp:273-326
    runs = {"siblings": m.gfd(f, b, d, g=g), "plain": m.gfd(f, b, d, g=g, plain_schedule=True),
            "known base": m.gfd(f, b, d, g=g, base=fwd,
                                out=dict(jv=np.zeros((n, 4)), jp=np.zeros((n, 4)), degraded=np.zeros((n, 4), np.uint8),
                                         frames=np.zeros((n, gpu.capi.FRAME_DOUBLES)), grad_v=np.zeros((n, 3)),
                                         grad_p=np.zeros((n, 3))))}
    for name, ours in runs.items():
        assert np.array_equal(ours["degraded"], theirs["degraded"]), name
        assert np.array_equal(ours["frames"], theirs["frames"]), name
        for k in ("jv", "jp"):
            scale = np.abs(theirs[k]).max()
            assert np.abs(ours[k] - theirs[k]).max() <= 1e-5 * scale, (name, k)
        for k in ("grad_v", "grad_p"):
            num = np.einsum("nd,nd->n", ours[k], theirs[k])
            na, nb = np.linalg.norm(ours[k], axis=1), np.linalg.norm(theirs[k], axis=1)
            ok = na * nb > 1e-12
            assert (num[ok] / (na * nb)[ok]).min() >= 0.999999, (name, k)
            assert np.abs(na[ok] / nb[ok] - 1).max() <= 1e-4, (name, k)
    for k in ("jv", "jp", "degraded", "grad_v", "grad_p"):   # a schedule is only a schedule
        assert np.array_equal(runs["siblings"][k], runs["plain"][k]), k
        assert np.array_equal(runs["siblings"][k], runs["known base"][k]), k
    # random starts never take a vertex branch on this mesh, so the Jacobians are in fact bit-equal
    assert not theirs["degraded"].any()
    assert np.array_equal(runs["siblings"]["jv"], theirs["jv"]) and np.array_equal(runs["siblings"]["jp"], theirs["jp"])


def test_config4_64_meshes_full_batch(gpu, ref):
    """Config 4 exactly as SURVEY 8(d): 64 meshes of 10 k - 200 k faces concatenated into one
    (6.8 M faces, 2.6 GB of crossing records: the cooperative gather), 65 536 queries per mesh (4.2 M),
    lengths log-uniform in [0.01, 2] x each component's bbox diagonal, default max_steps of the
    concatenated mesh. GPU: the whole batch in one call. Reference: 1 % prefix + 1 % random sample,
    bit-equal."""
    xyz, tri, f, b, d, foff = W.config4()
    assert len(foff) == 65 and len(f) == 64 * 65536
    faces = np.diff(foff)
    assert faces.min() >= 10_000 and faces.max() <= 200_000
    m = gpu.Mesh(xyz, tri)
    assert m.has_transport_cache and m.gather == "coop"
    n = len(f)
    full = m.trace_batch(f, b, d)                    # default max_steps = 10 sqrt(F) + 100 of the big mesh
    assert (full.status == 0).all()
    # every trace stays on its component (test_tracer.cpp:499-512)
    comp = np.repeat(np.arange(64), 65536)
    assert np.array_equal(np.searchsorted(foff, full.face, side="right") - 1, comp)
    # divergence stress: crossing counts span more than two decades
    assert full.crossings.max() > 200 * max(1, np.percentile(full.crossings, 5))
    idx = prefix_and_sample(n, n // 100, n // 100, 1)
    rm = ref.RefMesh.build(xyz, tri)
    assert rm.default_max_steps() == m.default_max_steps()
    theirs = rm.trace_batch(f[idx], b[idx], d[idx], record_polyline=True)
    for k in ("face", "bary", "dir", "traced", "requested", "term", "status", "npoints"):
        assert np.array_equal(getattr(full, k)[idx], getattr(theirs, k)), k
    assert np.array_equal(full.crossings[idx], (theirs.npoints - 2).clip(min=0))
    # whole face sequences of a slice of the sample, from a polyline run of ours
    sub = idx[-4000:]
    poly = m.trace_batch(f[sub], b[sub], d[sub], record_polyline=True)
    lo = theirs.poly_offsets[len(idx) - 4000]
    assert np.array_equal(poly.poly_face, theirs.poly_face[lo:]) and np.array_equal(poly.poly_bary, theirs.poly_bary[lo:])
    assert np.array_equal(poly.poly_seg, theirs.poly_seg[lo:])


def test_config5_long_vertex_heavy_traces_on_the_1m_face_torus(gpu, ref):
    """Config 5, one GPU's share of the stated batch scaled to a test: 1 M-face torus,
    length 5 x the outer diameter, max_steps = 200 000 on both sides, half the starts exactly at
    vertices aimed exactly along an incident edge (vertex-to-vertex walks through atan2 / sin / cos:
    not bit-comparable with glibc), half random. GPU: 2 M geodesics (about 1e10 face crossings) in one call.
    Reference: 0.1 % prefix of each half + a random 0.1 %: identical face sequences, end points,
    directions and lengths within 1e-9 x diagonal; the random half bit-equal."""
    n = 2_000_000
    xyz, tri, f, b, d = W.config5(n)
    m = gpu.Mesh(xyz, tri)
    assert m.nf == 1_000_000
    full = m.trace_batch(f, b, d, max_steps=W.C5_MAX_STEPS)
    assert (full.status == 0).all() and (full.term == 0).all()
    assert np.abs(full.traced - 5.0).max() < 1e-9
    assert full.total_crossings > 2000 * n
    k = n // 1000
    rng = np.random.default_rng(2)
    idx = np.concatenate([np.arange(k), n // 2 + np.arange(k), np.sort(rng.choice(n, k, replace=False))])
    rm = ref.RefMesh.build(xyz, tri)
    theirs = rm.trace_batch(f[idx], b[idx], d[idx], record_polyline=True, max_steps=W.C5_MAX_STEPS)
    diag = W.bbox_diagonal(xyz)
    for key in ("face", "term", "status", "npoints"):
        assert np.array_equal(getattr(full, key)[idx], getattr(theirs, key)), key
    for key in ("bary", "dir", "traced"):
        assert np.abs(getattr(full, key)[idx] - getattr(theirs, key)).max() <= 1e-9 * diag, key
    rand = idx >= n // 2                         # random starts: edge crossings only, bit for bit
    for key in ("bary", "dir", "traced"):
        assert np.array_equal(getattr(full, key)[idx][rand], getattr(theirs, key)[rand]), key
    poly = m.trace_batch(f[idx], b[idx], d[idx], record_polyline=True, max_steps=W.C5_MAX_STEPS)
    assert np.array_equal(poly.poly_face, theirs.poly_face)            # the whole face sequence of every trace
    # intermediate points after hundreds of atan2 / sin / cos vertex crossings: positions within 1e-9 x diagonal
    assert np.abs(m.embed(poly.poly_face, poly.poly_bary) - m.embed(theirs.poly_face, theirs.poly_bary)).max() <= 1e-9 * diag
    assert np.abs(poly.poly_bary - theirs.poly_bary).max() <= 1e-7   # (barycentrics are relative to ~2e-3 long edges)
    vertex_points = (theirs.poly_bary == 1.0).any(1)
    per_trace = np.add.reduceat(vertex_points.astype(np.int64), theirs.poly_offsets[:-1])
    assert per_trace[:k].min() > 100 and per_trace[:k].mean() > 400    # the walks really go vertex to vertex


def test_config3_strong_scaling_shards_give_the_bits_of_the_whole(gpu):
    """Config 3 is sharded over the GPUs by expected work (sharding.shard_bounds); a shard's results are
    the bits of the same queries inside the whole batch, whatever the cut (acceptance.cpp:173-201)."""
    from bench import make_workload
    from paper_2603_15780_b200 import sharding
    n = 200_000
    xyz, tri, f, b, d, q = make_workload("c3", n, 42)
    m = gpu.Mesh(xyz, tri)
    whole = m.trace_batch(f, b, d)
    for world in (2, 8):
        bnd = sharding.shard_bounds(np.linalg.norm(d, axis=1), world)
        assert bnd[0] == 0 and bnd[-1] == n
        for r in (0, world - 1):
            sl = slice(int(bnd[r]), int(bnd[r + 1]))
            part = m.trace_batch(f[sl], b[sl], d[sl])
            for k in ("face", "bary", "dir", "traced", "term"):
                assert np.array_equal(getattr(part, k), getattr(whole, k)[sl]), (world, r, k)
