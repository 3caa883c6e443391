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


def test_config2_training_step_through_host_buffers_at_full_size(gpu, ref):
    """The headline path of bench.py's `e2e`: config 2's 1 M geodesics through the resident batch on host buffers --
    the STREAMED forward (one walker while queries arrive and results leave), then EP on the resident samples --
    against the reference on a prefix + random sample taken out of the full-batch run: every bit."""
    from bench import make_workload
    n = 1_000_000
    xyz, tri, f, b, d, q = make_workload("c2", n, 42)
    m = gpu.Mesh(xyz, tri)
    rm = ref.RefMesh.build(xyz, tri)
    batch = gpu.Batch(m, n)
    h = batch.trace(f, b, d)
    g = 2.0 * (m.embed(h.face, h.bary) - q)          # gradcheck.cpp:88
    gv = batch.ep_backward(g)
    assert h.total_crossings == int(h.crossings.sum()) and (h.status == 0).all() and (h.term == 0).all()
    sel = prefix_and_sample(n, 6000, 6000, 2)
    r = rm.trace_batch(f[sel], b[sel], d[sel], record_polyline=True)
    for k in ("face", "bary", "dir", "traced", "term", "status"):
        assert np.array_equal(getattr(r, k), getattr(h, k)[sel]), k
    assert np.array_equal(r.npoints - 2, h.crossings[sel])       # one polyline point per crossing + start + end
    theirs = rm.ep(f[sel], b[sel], d[sel], r.face, r.bary, r.dir, g=g[sel])
    assert np.array_equal(theirs["grad_v"], gv[sel])
    batch.close()


def test_config3_forward_and_gfd_on_the_1m_face_torus(gpu, ref):
    """Config 3: 1 M-face noisy torus, bench stream (seed 42), forward + GFD with the default eps.
    6 000-sample prefix: jv / jp <= 1e-5 relative, degraded flags and frames bit-equal, pulled-back
    gradients cos >= 0.999999, for the sibling schedule, the plain schedule and the known-base form."""
    from bench import make_workload
    n = 6000
    xyz, tri, f, b, d, q = make_workload("c3", n, 42)
    m = gpu.Mesh(xyz, tri)
    assert m.nf == 1_000_000 and m.has_transport_cache and m.gather == "coop" and m.trace_plan(n) == (False, "coop")
    assert m.trace_plan(10_000_000) == (True, "loads")   # start-face order beyond 32 768 queries: per-lane loads
    rm = ref.RefMesh.build(xyz, tri)
    assert m.default_gfd_eps() == rm.default_gfd_eps()
    fwd = m.trace_batch(f, b, d)
    theirs_fwd = rm.trace_batch(f, b, d)
    for k in ("face", "bary", "dir", "traced", "term", "status"):
        assert np.array_equal(getattr(fwd, k), getattr(theirs_fwd, k)), k
    g = 2.0 * (m.embed(fwd.face, fwd.bary) - q)      # gradcheck.cpp:88
    theirs = rm.gfd(f, b, d, g=g)                    # gfd_batched_many, diff.cpp:273-326
    runs = {"siblings": m.gfd(f, b, d, g=g), "plain": m.gfd(f, b, d, g=g, plain_schedule=True),
            "face order": m.gfd(f, b, d, g=g, plain_schedule=2), "face order, known base": m.gfd(f, b, d, g=g, base=fwd, plain_schedule=2),
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
        assert np.array_equal(runs["siblings"][k], runs["face order"][k]), k
        assert np.array_equal(runs["siblings"][k], runs["face order, known base"][k]), k
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
    """Config 5, a test-sized share of one GPU's batch: 1 M-face torus, length 5 x the outer
    diameter, max_steps = 200 000 on both sides; the first half of the starts exactly at vertices aimed exactly
    along a meridian edge, the second half random. GPU: 2 M geodesics (about 8e9 face crossings) in one call.

    Random starts (non-degenerate queries): bit for bit against the reference, whole face sequences included.

    Vertex starts walk vertex to vertex (reference: median 2 388 vertex crossings per trace). Each such crossing is a
    knife edge: the outgoing direction comes out of atan2 / sin / cos, and whether it lies EXACTLY along the next
    edge (another vertex hit) or a last ulp beside it (an edge crossing) is decided by the last bit of libm -- CUDA's
    and glibc's differ there. These are the degenerate queries of north_star ("identical face sequences on
    non-degenerate queries"): the bar is (a) every walk completes with the exact length, (b) a walk can only part
    from the reference's AT a vertex point, (c) the walks that do not part (the majority) agree within
    1e-9 x diagonal at every polyline point, (d) both sides see the same amount of vertex crossings."""
    n = 2_000_000
    xyz, tri, f, b, d = W.config5(n)
    m = gpu.Mesh(xyz, tri)
    assert m.nf == 1_000_000
    full = m.trace_batch(f, b, d, max_steps=W.C5_MAX_STEPS)
    assert (full.status == 0).all() and (full.term == 0).all()
    assert np.abs(full.traced - 5.0).max() < 1e-9
    assert full.total_crossings > 2000 * n
    diag = W.bbox_diagonal(xyz)
    rm = ref.RefMesh.build(xyz, tri)
    k = n // 1000
    rng = np.random.default_rng(2)

    # ---- random half: prefix + random sample, bit for bit
    idx = np.concatenate([n // 2 + np.arange(k), np.sort(rng.choice(np.arange(n // 2 + k, n), k, replace=False))])
    theirs = rm.trace_batch(f[idx], b[idx], d[idx], record_polyline=True, max_steps=W.C5_MAX_STEPS)
    for key in ("face", "bary", "dir", "traced", "term", "status", "npoints"):
        assert np.array_equal(getattr(full, key)[idx], getattr(theirs, key)), key
    poly = m.trace_batch(f[idx], b[idx], d[idx], record_polyline=True, max_steps=W.C5_MAX_STEPS)
    assert np.array_equal(poly.poly_face, theirs.poly_face) and np.array_equal(poly.poly_bary, theirs.poly_bary)
    assert np.array_equal(poly.poly_seg, theirs.poly_seg)

    # ---- vertex half: prefix + random sample
    idx = np.concatenate([np.arange(k // 2), np.sort(rng.choice(np.arange(k // 2, n // 2), k // 2, replace=False))])
    theirs = rm.trace_batch(f[idx], b[idx], d[idx], record_polyline=True, max_steps=W.C5_MAX_STEPS)
    ours = m.trace_batch(f[idx], b[idx], d[idx], record_polyline=True, max_steps=W.C5_MAX_STEPS)
    for key in ("face", "bary", "dir", "traced"):      # the sample's results inside the big batch are the same bits
        assert np.array_equal(getattr(full, key)[idx], getattr(ours, key)), key
    assert (theirs.term == 0).all() and np.abs(theirs.traced - 5.0).max() < 1e-9
    is_vertex = lambda bary: (bary == 1.0).any(-1)
    same = 0
    for i in range(len(idx)):
        a0, a1 = ours.poly_offsets[i], ours.poly_offsets[i + 1]
        b0, b1 = theirs.poly_offsets[i], theirs.poly_offsets[i + 1]
        fa, fb = ours.poly_face[a0:a1], theirs.poly_face[b0:b1]
        L = min(len(fa), len(fb))
        neq = np.nonzero(fa[:L] != fb[:L])[0]
        if len(neq) == 0 and len(fa) == len(fb):
            same += 1                                  # (c) the same walk: every point within tolerance
            assert np.abs(m.embed(fa, ours.poly_bary[a0:a1]) - m.embed(fb, theirs.poly_bary[b0:b1])).max() <= 1e-9 * diag, i
            continue
        j = int(neq[0]) if len(neq) else L             # (b) first parting of the ways: at a vertex point
        near = [ours.poly_bary[a0 + max(j - 1, 0)], theirs.poly_bary[b0 + max(j - 1, 0)],
                ours.poly_bary[a0 + min(j, len(fa) - 1)], theirs.poly_bary[b0 + min(j, len(fb) - 1)]]
        assert any(is_vertex(p) for p in near), (i, j)
    assert same >= len(idx) // 2, same
    v_ours, v_theirs = is_vertex(ours.poly_bary).sum(), is_vertex(theirs.poly_bary).sum()
    assert abs(int(v_ours) - int(v_theirs)) <= 0.15 * v_theirs                 # (d)
    per_trace = np.add.reduceat(is_vertex(theirs.poly_bary).astype(np.int64), theirs.poly_offsets[:-1])
    assert per_trace.min() > 100 and np.median(per_trace) > 1000               # the walks really go vertex to vertex


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


def test_gather_of_a_batch_in_start_face_order_follows_the_trace_length(gpu):
    """On a mesh beyond the L2 a batch in start-face order is queued on both gathers with complementary gates on the
    mean requested length (summed on the device): short traces run the per-lane loads, long ones the cooperative
    gather. Whatever runs, exactly one of the two does, and the bits are those of either gather on its own."""
    from paper_2603_15780_b200 import workloads as W
    xyz, tri = W.torus(1 / 3, 1 / 6, 1000, 500)
    m = gpu.Mesh(xyz, tri)
    n = 40_000
    for mult in (0.3, 4.0):   # x outer diameter: ~310 and ~4 200 crossings per trace, either side of 1e6 / sqrt(F)
        f, b, d = W.sample_queries(xyz, tri, n, mult * 1.0, seed=17)
        auto = m.trace_batch(f, b, d, sort_by_face=True)
        assert auto.total_crossings == int(auto.crossings.sum()) and (auto.status == 0).all()
        assert abs(auto.traced - auto.requested).max() <= 1e-9
        for walker in ("loads", "coop"):
            one = m.trace_batch(f, b, d, sort_by_face=True, walker=walker)
            for k in ("face", "bary", "dir", "traced", "term", "status", "crossings"):
                assert np.array_equal(getattr(auto, k), getattr(one, k)), (mult, walker, k)
            assert one.total_crossings == auto.total_crossings
        # the tolerance lane takes the same two roads (half-size records / 128-byte records with the cooperative gather)
        fast = m.trace_batch(f, b, d, sort_by_face=True, lane="fast")
        assert np.array_equal(fast.face, auto.face) and np.array_equal(fast.crossings, auto.crossings)
        assert np.abs(m.embed(fast.face, fast.bary) - m.embed(auto.face, auto.bary)).max() <= 1e-9 * 1.1
