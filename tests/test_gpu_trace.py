"""Parity of the CUDA tracer (through the C-ABI) with the UNMODIFIED reference
(oracle/_ref/libdigeo_ref.so) on the same seeded inputs. Mirrors the reference's own tracer
tests (proj/tests/test_tracer.cpp) and BASELINE.json's configurations.

Bar: the f64 lane is compiled without FMA contraction in the reference's operation order, so
traces that never take a vertex branch must be BIT-IDENTICAL (faces, points, directions,
lengths, polylines). Vertex branches call atan2/sin/cos, where CUDA's libm may differ from
glibc in the last ulp: there the face sequence must be identical and positions agree to
1e-9 x bbox diagonal.
"""
import numpy as np
import pytest

from conftest import assert_trace_equal, gpu_mesh

pytestmark = pytest.mark.gpu


def both(ref_mesh, mesh, f, b, d, **kw):
    r = ref_mesh.trace_batch(f, b, d, record_polyline=True, **kw)
    h = mesh.trace_batch(f, b, d, record_polyline=True, **kw)
    return r, h


def test_config1_icosphere4_unit_vectors(gpu, ref):
    """BASELINE config 1: ico-4 (5 120 F), 10 k unit-length tangents, vs closed-form sphere."""
    rm = ref.RefMesh.icosphere(4)
    m = gpu_mesh(gpu, rm)
    f, b, d = rm.sample_queries(42, 10000, 1.0, 1.0)
    r, h = both(rm, m, f, b, d)
    assert_trace_equal(r, h, len(f))
    assert h.total_crossings == int(h.crossings.sum())
    assert np.array_equal(h.crossings, h.npoints - 2)  # one point per advance + the start point
    # accuracy against the closed-form sphere exponential map (reference: 2.24e-3 mean)
    P = m.embed(f, b)
    Pn = P / np.linalg.norm(P, axis=1, keepdims=True)
    dt = d - Pn * np.einsum("nd,nd->n", d, Pn)[:, None]
    dt /= np.linalg.norm(dt, axis=1, keepdims=True)
    exact = Pn * np.cos(1.0) + dt * np.sin(1.0)
    err = np.linalg.norm(m.embed(h.face, h.bary) - exact, axis=1).mean()
    assert err < 5e-3


@pytest.mark.parametrize("kw", [dict(), dict(want_q=True), dict(use_f32=True), dict(max_steps=7),
                                dict(sort_by_face=True), dict(refill_min=8), dict(blocks_per_sm=1)])
def test_icosphere_variants(gpu, ref, kw):
    rm = ref.RefMesh.icosphere(3)
    m = gpu_mesh(gpu, rm)
    f, b, d = rm.sample_queries(1, 4000, 0.1, 3.0)
    rng = np.random.default_rng(0)
    pay = rng.normal(size=(len(f), 3))
    pay[::3] = 0  # zero payload rows mean "no payload" (tracer.cpp:582)
    ref_kw = {k: v for k, v in kw.items() if k not in ("sort_by_face", "refill_min", "blocks_per_sm")}
    r = rm.trace_batch(f, b, d, payload=pay, record_polyline=True, **ref_kw)
    h = m.trace_batch(f, b, d, payload=pay, record_polyline=True, **kw)
    assert_trace_equal(r, h, len(f), payload=True, q=kw.get("want_q", False))
    assert np.array_equal(r.has_payload, h.has_payload)


@pytest.mark.parametrize("cache", [True, False])
def test_torus_long_traces_bit_exact(gpu, ref, cache):
    rm = ref.RefMesh.torus(1 / 3, 1 / 6, 200, 100)
    m = gpu_mesh(gpu, rm, transport_cache=cache)
    assert m.has_transport_cache == cache
    f, b, d = rm.sample_queries(7, 20000, 0.05, 1.5)
    r, h = both(rm, m, f, b, d)
    assert_trace_equal(r, h, len(f))


@pytest.mark.parametrize("cache", [True, False])
def test_vertex_paths(gpu, ref, cache):
    """Vertex-to-vertex walks (config-5 style starts) and random departures from vertices."""
    rm = ref.RefMesh.torus(1 / 3, 1 / 6, 64, 32)
    m = gpu_mesh(gpu, rm, transport_cache=cache)
    a = rm.arrays()
    X, T = a["xyz"], a["tri"]
    rng = np.random.default_rng(3)
    n = 4000
    fs = rng.integers(0, rm.nf, n).astype(np.int32)
    corner = rng.integers(0, 3, n)
    bs = np.zeros((n, 3))
    bs[np.arange(n), corner] = 1
    nxt = (corner + rng.integers(1, 3, n)) % 3
    ds = X[T[fs, nxt]] - X[T[fs, corner]]
    ds = ds / np.linalg.norm(ds, axis=1, keepdims=True) * rng.uniform(0.2, 2.0, (n, 1))
    pay = rng.normal(size=(n, 3))
    diag = np.linalg.norm(X.max(0) - X.min(0))
    for dirs in (ds, rng.normal(size=(n, 3))):
        r = rm.trace_batch(fs, bs, dirs, payload=pay, want_q=True, record_polyline=True, max_steps=5000)
        h = m.trace_batch(fs, bs, dirs, payload=pay, want_q=True, record_polyline=True, max_steps=5000)
        assert_trace_equal(r, h, n, payload=True, q=True, exact=False, tol=1e-9 * diag)
        assert (h.crossings > 0).any()


def test_cone_apex_and_icosahedron_vertices(gpu, ref):
    for rm in (ref.RefMesh.cone(1.0, 1.0, 16), ref.RefMesh.icosphere(0), ref.RefMesh.icosphere(2)):
        m = gpu_mesh(gpu, rm)
        a = rm.arrays()
        X = a["xyz"]
        apex = int(np.argmax(np.diff(a["csr_off"])))
        f, b, d = rm.sample_queries(12, 3000, 1.0, 1.0)
        P = rm.embed(f, b)
        d = X[apex] - P
        d = d / np.linalg.norm(d, axis=1, keepdims=True) * 2.5
        rng = np.random.default_rng(5)
        pay = rng.normal(size=(len(f), 3))
        for hole in (False, True):
            r = rm.trace_batch(f, b, d, payload=pay, want_q=True, record_polyline=True, hole_avoidance=hole)
            h = m.trace_batch(f, b, d, payload=pay, want_q=True, record_polyline=True, hole_avoidance=hole)
            assert_trace_equal(r, h, len(f), payload=True, q=True, exact=False, tol=1e-9)


@pytest.mark.parametrize("hole", [False, True])
def test_open_meshes_boundary_and_hole_avoidance(gpu, ref, hole):
    rng = np.random.default_rng(11)
    for rm, seed in ((ref.RefMesh.plane(12, 9, 1.0, 3), 5), (ref.RefMesh.cylinder(0.5, 1.0, 24, 6), 9)):
        m = gpu_mesh(gpu, rm)
        f, b, d = rm.sample_queries(seed, 6000, 0.05, 3.0)
        pay = rng.normal(size=(len(f), 3))
        r = rm.trace_batch(f, b, d, payload=pay, want_q=True, record_polyline=True, hole_avoidance=hole)
        h = m.trace_batch(f, b, d, payload=pay, want_q=True, record_polyline=True, hole_avoidance=hole)
        # boundary slides visit vertices only through exact arithmetic; everything is bit-equal
        assert_trace_equal(r, h, len(f), payload=True, q=True, exact=False, tol=1e-12)
        if not hole:
            assert (h.term == 1).any()


def test_square_known_answers_and_error_slots(gpu, ref):
    """Appendix-B known answers of the reference (golden trace_square.json case first)."""
    sq = ref.RefMesh.build([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0]], [[0, 1, 2], [0, 2, 3]])
    m = gpu_mesh(gpu, sq)
    F = np.array([0, 0, 0, 0, 0, 0, 7, 0, 0, -1], np.int32)
    B = np.array([[.5, .25, .25], [.5, 0, .5], [1, 0, 0], [.5, .25, .25], [.5, .25, .25], [.5, .25, .25],
                  [.3, .3, .4], [.5, .25, .25], [.5, .5, .5], [1, 0, 0]])
    D = np.array([[.25, .5, 0], [-.2, .1, 0], [.1, .3, 0], [2, .1, 0], [0, 0, .5], [0, 0, 0], [1, 0, 0],
                  [0, 0, 0], [1, 0, 0], [1, 0, 0]], float)
    for hole in (False, True):
        r = sq.trace_batch(F, B, D, record_polyline=True, hole_avoidance=hole)
        h = m.trace_batch(F, B, D, record_polyline=True, hole_avoidance=hole)
        assert_trace_equal(r, h, len(F))
        assert r.errors == h.errors
    h = m.trace_batch(F, B, D, record_polyline=True)
    # golden: final bary and the 1.1e-16 second segment (tests/golden/trace_square.json)
    assert h.bary[0].tolist() == [0.24999999999999992, 0.75000000000000011, 0.0]
    assert h.poly_seg[h.poly_offsets[0]:h.poly_offsets[1]].tolist() == [0.0, 0.55901699437494734, 1.1102230246251565e-16]
    assert h.term[3] == 1 and h.traced[3] == 0.50062460986251966
    assert h.errors == [(4, "initial direction is normal to the anchor face"), (6, "trace: start face out of range"),
                        (8, "trace: start barycentric coordinates not in the simplex"),
                        (9, "trace: start face out of range")]


def test_concat_meshes_stay_on_component(gpu, ref):
    ra, rb = ref.RefMesh.icosphere(2), ref.RefMesh.torus(1 / 3, 1 / 6, 24, 12)
    rm = ref.RefMesh.concat(ra, rb)
    m = gpu_mesh(gpu, rm)
    f, b, d = rm.sample_queries(2, 5000, 0.1, 2.0)
    r, h = both(rm, m, f, b, d)
    assert_trace_equal(r, h, len(f))
    assert ((f < ra.nf) == (h.face < ra.nf)).all()


def test_empty_and_single(gpu, ref):
    rm = ref.RefMesh.icosphere(1)
    m = gpu_mesh(gpu, rm)
    e = m.trace_batch(np.empty(0, np.int32), np.empty((0, 3)), np.empty((0, 3)), record_polyline=True)
    assert len(e.face) == 0 and e.total_crossings == 0
    f, b, d = rm.sample_queries(3, 1, 1.0, 1.0)
    r, h = both(rm, m, f, b, d)
    assert_trace_equal(r, h, 1)


def test_host_mode_paths_by_batch_size_agree(gpu, ref):
    """Host-mode dg_trace_batch picks its plumbing by batch size -- up to 256 queries the kernel works
    on the mapped pinned block (alternating work cursors, no copies), up to 8 192 one packed copy
    each way, from 65 536 the sliced copy/compute pipeline -- and none of it may show in the
    results: every prefix of a batch equals the same rows of the whole batch, call after call
    (both cursor parities), with and without the transport matrix, totals included."""
    rm = ref.RefMesh.torus(1 / 3, 1 / 6, 48, 24)
    m = gpu_mesh(gpu, rm)
    f, b, d = rm.sample_queries(77, 70000, 0.05, 1.5)
    fields = ("face", "bary", "dir", "traced", "requested", "term", "status", "stall", "crossings")
    for want_q in (False, True):
        whole = m.trace_batch(f, b, d, want_q=want_q)
        assert whole.total_crossings == int(whole.crossings.sum())
        for k in (1, 2, 50, 255, 256, 257, 300, 8192, 8193, 65536):
            for _ in range(3 if k <= 300 else 1):
                part = m.trace_batch(f[:k], b[:k], d[:k], want_q=want_q)
                for key in fields + (("q",) if want_q else ()):
                    assert np.array_equal(getattr(part, key), getattr(whole, key)[:k], equal_nan=True), (k, key)
                assert part.total_crossings == int(whole.crossings[:k].sum()), k
    theirs = rm.trace_batch(f[:300], b[:300], d[:300])
    part = m.trace_batch(f[:300], b[:300], d[:300])
    assert np.array_equal(part.face, theirs.face) and np.array_equal(part.term, theirs.term)


def test_invalid_batch_arguments(gpu, ref):
    m = gpu_mesh(gpu, ref.RefMesh.icosphere(1))
    with pytest.raises(gpu.DgError) as e:
        m.trace_batch(np.zeros(3, np.int32), np.zeros((2, 3)), np.zeros((3, 3)))
    assert e.value.klass == "InvalidArgs"
    with pytest.raises(gpu.DgError):
        m.trace_batch(np.zeros(3, np.int32), np.zeros((3, 3)), np.zeros((3, 3)), payload=np.zeros((2, 3)))


def test_run_to_run_and_shape_determinism(gpu, ref):
    """Results are bitwise independent of the launch shape (the reference's worker-count contract)."""
    rm = ref.RefMesh.icosphere(5)
    m = gpu_mesh(gpu, rm)
    f, b, d = rm.sample_queries(8, 30000, 0.05, 4.0)
    base = m.trace_batch(f, b, d)
    for kw in (dict(), dict(blocks_per_sm=1), dict(refill_min=16), dict(sort_by_face=True)):
        o = m.trace_batch(f, b, d, **kw)
        for k in ("face", "bary", "dir", "traced", "term", "status", "crossings"):
            assert np.array_equal(getattr(base, k), getattr(o, k)), (k, kw)


def test_full_size_invariants_1m_face_torus(gpu):
    """BASELINE-size mesh (1 M faces): size-independent properties of the exponential map --
    requested length is consumed exactly, barycentrics stay on the simplex, directions are unit
    and tangent, and reversing the final direction returns to the start (geodesic reversibility)."""
    from paper_2603_15780_b200 import workloads as W
    xyz, tri = W.torus(1 / 3, 1 / 6, 1000, 500)
    m = gpu.Mesh(xyz, tri)
    n = 200000
    diag = W.bbox_diagonal(xyz)
    f, b, d = W.sample_queries(xyz, tri, n, 0.25 * diag, seed=4)
    h = m.trace_batch(f, b, d)
    assert (h.status == 0).all() and (h.term == 0).all()
    assert np.abs(h.traced - h.requested).max() <= 1e-12 * diag
    assert np.abs(h.bary.sum(1) - 1).max() <= 1e-12 and h.bary.min() >= 0
    assert np.abs(np.linalg.norm(h.dir, axis=1) - 1).max() <= 1e-12
    assert np.abs(np.einsum("nd,nd->n", h.dir, m.fnormal[h.face])).max() <= 1e-9
    back = m.trace_batch(h.face, h.bary, -h.dir * h.requested[:, None])
    ok = back.status == 0
    err = np.linalg.norm(m.embed(back.face[ok], back.bary[ok]) - m.embed(f[ok], b[ok]), axis=1)
    # vertex-free straightest geodesics are reversible up to rounding
    assert np.quantile(err, 0.999) <= 1e-9 * diag
    assert h.total_crossings > 300 * n


def test_config4_style_heterogeneous_batch_mixed_lengths(gpu, ref):
    """BASELINE config 4 (scaled down): several meshes concatenated into one (mesh.cpp:199-206),
    queries on every component, lengths log-uniform over two decades (divergence stress)."""
    parts = [ref.RefMesh.icosphere(3), ref.RefMesh.torus(1 / 3, 1 / 6, 40, 20), ref.RefMesh.icosphere(2),
             ref.RefMesh.torus(0.5, 0.2, 24, 12)]
    rm = parts[0]
    for p in parts[1:]:
        rm = ref.RefMesh.concat(rm, p)
    m = gpu_mesh(gpu, rm)
    f, b, d = rm.sample_queries(21, 20000, 1.0, 1.0)
    rng = np.random.default_rng(4)
    d *= np.exp(rng.uniform(np.log(0.01), np.log(4.0), len(f)))[:, None]
    r, h = both(rm, m, f, b, d)
    assert_trace_equal(r, h, len(f))
    assert h.crossings.max() > 50 * max(1, np.median(h.crossings)) / 10


def test_config5_style_long_vertex_heavy_traces(gpu, ref):
    """BASELINE config 5 (scaled down): starts exactly at vertices aimed exactly along an edge,
    length 5 x the outer diameter, explicit max_steps on both sides; half random starts."""
    rm = ref.RefMesh.torus(1 / 3, 1 / 6, 100, 50)
    m = gpu_mesh(gpu, rm)
    a = rm.arrays()
    X, T = a["xyz"], a["tri"]
    n = 600
    rng = np.random.default_rng(6)
    fs = rng.integers(0, rm.nf, n).astype(np.int32)
    bs = np.zeros((n, 3))
    bs[:, 0] = 1
    ds = X[T[fs, 1]] - X[T[fs, 0]]
    ds *= (5.0 / np.linalg.norm(ds, axis=1))[:, None]
    f2, b2, d2 = rm.sample_queries(3, n, 5.0, 5.0)
    F, B, D = np.concatenate([fs, f2]), np.concatenate([bs, b2]), np.concatenate([ds, d2])
    r = rm.trace_batch(F, B, D, record_polyline=True, max_steps=200000)
    h = m.trace_batch(F, B, D, record_polyline=True, max_steps=200000)
    diag = np.linalg.norm(X.max(0) - X.min(0))
    assert_trace_equal(r, h, len(F), exact=False, tol=1e-9 * diag)
    vertex_points = (h.poly_bary == 1).any(1).sum()
    assert vertex_points > 3 * n           # the walks really pass through vertices
    assert (h.term == 0).all() and np.abs(h.traced - 5.0).max() < 1e-9


def test_default_max_steps_termination_matches(gpu, ref):
    """MaxSteps must trigger on the same step as the reference (a vertex crossing costs 2 steps)."""
    rm = ref.RefMesh.icosphere(2)
    m = gpu_mesh(gpu, rm)
    f, b, d = rm.sample_queries(13, 3000, 30.0, 60.0)   # far longer than 10*sqrt(F)+100 crossings
    r, h = both(rm, m, f, b, d)
    assert (h.term == 2).any()
    assert_trace_equal(r, h, len(f))


def test_transport_cache_is_bit_identical(gpu, ref):
    """The per-half-edge transport cache (layout choice, on when it fits in L2) must not change a
    single bit of any output: payload, Q, polylines, hole avoidance included."""
    rng = np.random.default_rng(17)
    for rm, seed in ((ref.RefMesh.icosphere(4), 31), (ref.RefMesh.plane(14, 11, 1.0, 3), 32)):
        on, off = gpu_mesh(gpu, rm, True), gpu_mesh(gpu, rm, False)
        assert on.has_transport_cache and not off.has_transport_cache
        assert on.device_bytes > off.device_bytes
        f, b, d = rm.sample_queries(seed, 20000, 0.05, 2.5)
        pay = rng.normal(size=(len(f), 3))
        for kw in (dict(), dict(payload=pay, want_q=True, hole_avoidance=True)):
            x = on.trace_batch(f, b, d, record_polyline=True, **kw)
            y = off.trace_batch(f, b, d, record_polyline=True, **kw)
            for k in ("face", "bary", "dir", "traced", "term", "status", "npoints", "crossings", "poly_face",
                      "poly_bary", "poly_seg") + (("payload", "q") if kw else ()):
                assert np.array_equal(getattr(x, k), getattr(y, k)), k


def test_one_call_polylines_give_the_bits_of_the_two_call_form(gpu, ref):
    """dg_trace_polylines (capped first pass, device scan, compaction, second pass for the traces that outgrew
    their slots) against the count call + host scan + fill call, and against the reference: every polyline bit.
    Covers: slots that always suffice (small batch), a slot budget so tight that most traces need pass 2, payload +
    transport matrix + hole avoidance on an open mesh, rejected starts and zero-length requests (0 / 1 points)."""
    import os
    rm = ref.RefMesh.icosphere(4)
    m = gpu_mesh(gpu, rm)
    f, b, d = rm.sample_queries(5, 30000, 0.02, 3.0)
    f[7] = -1
    d[11] = 0.0
    for count in (1, 60, 30000):
        a = m.trace_batch(f[:count], b[:count], d[:count], record_polyline=True)
        t = m.trace_batch(f[:count], b[:count], d[:count], record_polyline=True, two_call_polylines=True)
        r = rm.trace_batch(f[:count], b[:count], d[:count], record_polyline=True)
        for k in ("npoints", "poly_face", "poly_bary", "poly_seg", "face", "bary", "dir", "traced", "crossings"):
            assert np.array_equal(getattr(a, k), getattr(t, k)), (count, k)
        assert np.array_equal(a.poly_offsets, np.concatenate([[0], np.cumsum(a.npoints)]))
        assert_trace_equal(r, a, count)
        assert a.total_crossings == t.total_crossings
    # pass 2 for most traces: 16 points of slot per trace at this batch size
    os.environ["DG_POLY_SLOT_BUDGET"] = "1024"
    pm = ref.RefMesh.plane(14, 11, 1.0, 3)
    mp = gpu_mesh(gpu, pm)
    f, b, d = pm.sample_queries(6, 20000, 0.05, 2.5)
    pay = np.random.default_rng(3).normal(size=(len(f), 3))
    kw = dict(payload=pay, want_q=True, hole_avoidance=True)
    a = mp.trace_batch(f, b, d, record_polyline=True, **kw)
    t = mp.trace_batch(f, b, d, record_polyline=True, two_call_polylines=True, **kw)
    r = pm.trace_batch(f, b, d, record_polyline=True, **kw)
    for k in ("npoints", "poly_face", "poly_bary", "poly_seg", "payload", "q"):
        assert np.array_equal(getattr(a, k), getattr(t, k)), k
    assert_trace_equal(r, a, len(f), payload=True, q=True)
    del os.environ["DG_POLY_SLOT_BUDGET"]


def test_new_entry_points_on_empty_and_odd_requests(gpu, ref):
    """n = 0 and n = 1 through the one-call polylines, the fused forward + GFD and the pull-back; the tolerance lane
    asked for where it does not apply (payload, a mesh without crossing records, f32) runs the exact lane."""
    rm = ref.RefMesh.icosphere(2)
    a = rm.arrays()
    m = gpu.Mesh(a["xyz"], a["tri"])
    f, b, d = rm.sample_queries(1, 300, 0.2, 1.0)
    z = lambda *shape: np.empty(shape)
    e = m.trace_batch(f[:0], b[:0], d[:0], record_polyline=True)
    assert len(e.face) == 0 and e.poly_offsets.tolist() == [0] and len(e.poly_face) == 0 and e.total_crossings == 0
    r, jac = m.trace_gfd(f[:0], b[:0], d[:0])
    assert len(r.face) == 0 and jac["jv"].shape == (0, 4)
    assert m.gfd_pullback(f[:0], d[:0], f[:0], z(0, 4), z(0, 4), z(0, 3))["grad_v"].shape == (0, 3)
    one, jac1 = m.trace_gfd(f[:1], b[:1], d[:1])
    sep = m.gfd(f[:1], b[:1], d[:1])
    assert np.array_equal(jac1["jv"], sep["jv"]) and np.array_equal(one.bary, m.trace_batch(f[:1], b[:1], d[:1]).bary)
    # the lane is the plain forward map's: a payload request runs the exact lane whatever `lane` says
    pay = np.random.default_rng(0).normal(size=(len(f), 3))
    x = m.trace_batch(f, b, d, payload=pay, lane="fast")
    y = m.trace_batch(f, b, d, payload=pay)
    assert np.array_equal(x.bary, y.bary) and np.array_equal(x.payload, y.payload)
    # no crossing records on the mesh: nothing for the lane to walk over -> exact bits
    plain = gpu.Mesh(a["xyz"], a["tri"], transport_cache=False)
    assert np.array_equal(plain.trace_batch(f, b, d, lane="fast").bary, y.bary)
    # and where it applies it is the same walk, within tolerance, on a big enough batch for every code path
    f2, b2, d2 = rm.sample_queries(2, 40000, 0.2, 3.0)
    ex, fa = m.trace_batch(f2, b2, d2), m.trace_batch(f2, b2, d2, lane="fast")
    assert np.array_equal(ex.face, fa.face) and np.array_equal(ex.crossings, fa.crossings)
    assert np.abs(m.embed(ex.face, ex.bary) - m.embed(fa.face, fa.bary)).max() <= 1e-9 * 2.0


def test_polyline_slots_hold_two_points_per_step_under_hole_avoidance(gpu, ref):
    """One-call polylines with hole avoidance under a tight step limit (all three size paths) against the reference."""
    # hole avoidance under a tight step limit: a step that reaches a boundary edge pushes TWO points (its advance and the
    # slide along the boundary), so a trace can record up to 2 max_steps + 2 points -- the slots must hold them
    # (found by scripts/fuzz_walkers.py: "a trace recorded more points than its step limit allows")
    rng = np.random.default_rng(5)
    nx, ny = 12, 9
    gx, gy = np.meshgrid(np.arange(nx + 1.0), np.arange(ny + 1.0), indexing="ij")
    xyz = np.stack([gx.ravel(), gy.ravel(), np.zeros(gx.size)], 1)
    xyz[:, :2] += 0.3 * rng.uniform(-0.5, 0.5, (len(xyz), 2))      # jittered open grid
    idx = lambda i, j: i * (ny + 1) + j
    tri = np.array([[idx(i, j), idx(i + 1, j), idx(i + 1, j + 1)] for i in range(nx) for j in range(ny)] +
                   [[idx(i, j), idx(i + 1, j + 1), idx(i, j + 1)] for i in range(nx) for j in range(ny)], np.int32)
    gm, gr = gpu.Mesh(xyz, tri), ref.RefMesh.build(xyz, tri)
    from paper_2603_15780_b200 import workloads as W
    diag = W.bbox_diagonal(xyz)
    f, b, d = W.sample_queries(xyz, tri, 30000, (0.5 * diag, 3 * diag), seed=3)
    for steps in (5, 60):
        r = gr.trace_batch(f, b, d, record_polyline=True, hole_avoidance=True, max_steps=steps)
        hot = np.nonzero(r.npoints > steps + 2)[0]
        assert len(hot) > 0                                          # the case is in the batch
        a = gm.trace_batch(f, b, d, record_polyline=True, hole_avoidance=True, max_steps=steps)     # large path
        assert_trace_equal(r, a, len(f))
        sub = np.concatenate([hot, np.arange(1000)])                 # one-block small path (<= 2 048 traces)
        a = gm.trace_batch(f[sub], b[sub], d[sub], record_polyline=True, hole_avoidance=True, max_steps=steps)
        rs = gr.trace_batch(f[sub], b[sub], d[sub], record_polyline=True, hole_avoidance=True, max_steps=steps)
        assert_trace_equal(rs, a, len(sub))
        a = gm.trace_batch(f[sub[:200]], b[sub[:200]], d[sub[:200]], record_polyline=True, hole_avoidance=True, max_steps=steps)   # mapped
        assert np.array_equal(a.poly_bary, rs.poly_bary[:rs.poly_offsets[200]])
