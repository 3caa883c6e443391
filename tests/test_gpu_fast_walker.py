"""The fast walker (csrc/dg_fast_walk.cuh) against the general state machine it shortcuts
(csrc/dg_tracer_core.cuh, i.e. proj/src/tracer.cpp:44-529), through the C-ABI with the walker
selector of dg_trace_cfg. Bar: EVERY output bit-identical -- faces, barycentrics, directions,
lengths, termination / status / stall bytes, crossing and point counts -- on every mesh family,
both mesh layouts, and on the inputs that exercise each exit from the fast path: vertex hits,
boundaries, step limits, exact zeros, rejected starts, zero-length requests."""
import numpy as np
import pytest

from paper_2603_15780_b200 import workloads as W

pytestmark = pytest.mark.gpu

FIELDS = ("face", "bary", "dir", "traced", "requested", "term", "status", "stall", "npoints", "crossings")


def both_walkers(m, f, b, d, **kw):
    """General walker vs the fast walker with each gather of the crossing records (per-lane 256-bit
    loads, TMA tile::gather4, cooperative loads; on a mesh without records every selector runs the
    face-record walker)."""
    slow = m.trace_batch(f, b, d, walker="generic", **kw)
    for walker in ("loads", "tma", "coop", "auto"):
        fast = m.trace_batch(f, b, d, walker=walker, **kw)
        for k in FIELDS:
            x, y = getattr(fast, k), getattr(slow, k)
            same = (x == y) | ((x != x) & (y != y))
            bad = np.nonzero(~same.reshape(len(f), -1).all(1))[0]
            assert len(bad) == 0, f"{walker} {k}: {len(bad)}/{len(f)} differ, first {bad[:5]}: fast {x[bad[:3]]} generic {y[bad[:3]]}"
        assert fast.total_crossings == slow.total_crossings == int(slow.crossings.sum())
    return fast


@pytest.mark.parametrize("cache", [True, False])
def test_payload_lane_of_the_fast_walker(gpu, ref, cache):
    """A payload to transport and nothing else of the full variant runs on the fast walker (kPay):
    transported payload and end states bit-identical to the general walker with every gather, on
    closed and open meshes, with payload-free (zero) elements, vertex starts and a tight step
    limit; and bit-identical to the reference where no vertex branch is taken."""
    rng = np.random.default_rng(8)
    for rm, seed, max_steps in ((ref.RefMesh.icosphere(4), 41, 0), (ref.RefMesh.torus(1 / 3, 1 / 6, 60, 30), 42, 0),
                                (ref.RefMesh.plane(12, 9, 1.0, 2), 43, 0), (ref.RefMesh.icosphere(3), 44, 11)):
        a = rm.arrays()
        m = gpu.Mesh(a["xyz"], a["tri"], transport_cache=cache)
        f, b, d = rm.sample_queries(seed, 12000, 0.05, 2.5)
        pay = rng.normal(size=(len(f), 3)) * 10.0 ** rng.uniform(-3, 3, (len(f), 1))
        pay[::7] = 0.0                      # zero payload = no payload (tracer.cpp:580-583)
        b[100:200] = [0.0, 1.0, 0.0]        # vertex starts: the generic path carries the payload over the fan
        slow = m.trace_batch(f, b, d, payload=pay, max_steps=max_steps, walker="generic")
        for walker in ("loads", "tma", "coop", "auto"):
            fast = m.trace_batch(f, b, d, payload=pay, max_steps=max_steps, walker=walker)
            for k in FIELDS + ("payload",):
                x, y = getattr(fast, k), getattr(slow, k)
                assert np.array_equal(x, y, equal_nan=True), (walker, k)
        theirs = rm.trace_batch(f, b, d, payload=pay, max_steps=max_steps, record_polyline=True)
        no_vertex = np.ones(len(f), bool)
        at_vertex = (theirs.poly_bary == 1.0).any(1)
        np.logical_and.at(no_vertex, np.repeat(np.arange(len(f)), np.diff(theirs.poly_offsets)), ~at_vertex)
        assert np.array_equal(fast.face, theirs.face) and np.array_equal(fast.term, theirs.term)
        assert np.array_equal(fast.payload[no_vertex], theirs.payload[no_vertex])
        assert np.abs(fast.payload - theirs.payload).max() <= 1e-9 * np.abs(pay).max()
        keep = np.linalg.norm(pay, axis=1) > 0
        assert np.abs(np.linalg.norm(fast.payload[keep], axis=1) / np.linalg.norm(pay[keep], axis=1) - 1).max() < 1e-10


@pytest.mark.parametrize("cache", [True, False])
def test_transport_matrix_lane_of_the_fast_walker(gpu, ref, cache):
    """want_transport_matrix requests (tracer.cpp:99-102, the opt.cpp:298-323 use) run on the fast
    walker's kPay = 2 lane: Q, payload and end states bit-identical to the general walker with
    every gather, on closed and open meshes, with vertex starts, hole avoidance and a tight step
    limit; bit-identical to the reference where no vertex branch is taken; Q stays an isometry of
    the tangent planes (columns of a rotation restricted to the end plane)."""
    rng = np.random.default_rng(10)
    for rm, seed, max_steps, hole in ((ref.RefMesh.icosphere(4), 61, 0, False), (ref.RefMesh.torus(1 / 3, 1 / 6, 48, 24), 62, 0, False),
                                      (ref.RefMesh.plane(11, 8, 1.0, 3), 63, 0, True), (ref.RefMesh.icosphere(3), 64, 9, False)):
        a = rm.arrays()
        m = gpu.Mesh(a["xyz"], a["tri"], transport_cache=cache)
        f, b, d = rm.sample_queries(seed, 9000, 0.05, 2.5)
        pay = rng.normal(size=(len(f), 3))
        pay[::6] = 0.0
        b[50:120] = [0.0, 0.0, 1.0]
        for kw in (dict(), dict(payload=pay)):
            kw = dict(kw, want_q=True, max_steps=max_steps, hole_avoidance=hole)
            slow = m.trace_batch(f, b, d, walker="generic", **kw)
            for walker in ("loads", "tma", "coop", "auto"):
                fast = m.trace_batch(f, b, d, walker=walker, **kw)
                for k in FIELDS + ("q",) + (("payload",) if "payload" in kw else ()):
                    assert np.array_equal(getattr(fast, k), getattr(slow, k), equal_nan=True), (walker, k)
        theirs = rm.trace_batch(f, b, d, record_polyline=True, **kw)
        no_vertex = np.ones(len(f), bool)
        at_vertex = (theirs.poly_bary == 1.0).any(1)
        np.logical_and.at(no_vertex, np.repeat(np.arange(len(f)), np.diff(theirs.poly_offsets)), ~at_vertex)
        assert np.array_equal(fast.face, theirs.face) and np.array_equal(fast.term, theirs.term)
        assert np.array_equal(fast.q[no_vertex], theirs.q[no_vertex])
        assert np.abs(fast.q - theirs.q).max() <= 1e-9
        ok = (fast.status == 0) & (fast.crossings >= 1) & no_vertex
        Q = fast.q[ok].reshape(-1, 3, 3)
        n0 = a["fnormal"][f[ok]]
        # the columns start as the ambient basis (tracer.cpp:60); the first fold drops the start normal and
        # every fold is an isometry of the tangent planes: Q^T Q = I - n n^T
        want = np.eye(3)[None] - n0[:, :, None] * n0[:, None, :]
        assert np.abs(np.einsum("nki,nkj->nij", Q, Q) - want).max() < 1e-9


@pytest.mark.parametrize("cache", [True, False])
def test_hole_avoidance_on_the_fast_walker(gpu, ref, cache):
    """hole_avoidance requests (without polyline / transport matrix) run on the fast walker with
    the full Tracer behind it: boundary edges and boundary vertices -- where hole avoidance acts --
    are exactly what the fast step hands over. Bit-identical to the general walker, with and
    without a payload; end states equal to the reference."""
    rng = np.random.default_rng(9)
    for rm, seed in ((ref.RefMesh.plane(10, 7, 1.0, 4), 51), (ref.RefMesh.cylinder(0.5, 1.5, 20, 6), 52),
                     (ref.RefMesh.icosphere(3), 53)):
        a = rm.arrays()
        m = gpu.Mesh(a["xyz"], a["tri"], transport_cache=cache)
        f, b, d = rm.sample_queries(seed, 8000, 0.1, 4.0)
        pay = rng.normal(size=(len(f), 3))
        for kw in (dict(), dict(payload=pay)):
            slow = m.trace_batch(f, b, d, hole_avoidance=True, walker="generic", **kw)
            for walker in ("loads", "tma", "coop", "auto"):
                fast = m.trace_batch(f, b, d, hole_avoidance=True, walker=walker, **kw)
                for k in FIELDS + (("payload",) if kw else ()):
                    assert np.array_equal(getattr(fast, k), getattr(slow, k), equal_nan=True), (walker, k)
            theirs = rm.trace_batch(f, b, d, hole_avoidance=True, record_polyline=True, **kw)
            assert np.array_equal(fast.face, theirs.face) and np.array_equal(fast.term, theirs.term)
            assert np.abs(fast.bary - theirs.bary).max() < 1e-9 and np.abs(fast.traced - theirs.traced).max() < 1e-9
        if a["vboundary"].any():
            plain = m.trace_batch(f, b, d)
            assert (plain.term == 1).any() and (fast.term == 0).all()   # what stopped at the boundary now slides along it


@pytest.mark.parametrize("cache", [True, False])
def test_bumpy_sphere_config2_style(gpu, cache):
    xyz, tri = W.bumpy_sphere(5)
    m = gpu.Mesh(xyz, tri, transport_cache=cache)
    assert m.has_transport_cache == cache
    f, b, d = W.sample_queries(xyz, tri, 150_000, 0.5 * W.bbox_diagonal(xyz), seed=3)
    r = both_walkers(m, f, b, d)
    assert (r.term == 0).all() and (r.status == 0).all() and np.abs(r.traced - r.requested).max() < 1e-9


@pytest.mark.parametrize("cache", [True, False])
def test_noisy_torus_mixed_lengths_and_step_limit(gpu, cache):
    xyz, tri = W.torus(1 / 3, 1 / 6, 300, 150, noise=0.1, seed=7)
    m = gpu.Mesh(xyz, tri, transport_cache=cache)
    n = 60_000
    diag = W.bbox_diagonal(xyz)
    f, b, d = W.sample_queries(xyz, tri, n, (1e-4 * diag, 2.0 * diag), seed=9)  # log-uniform lengths: divergence stress
    both_walkers(m, f, b, d)
    r = both_walkers(m, f, b, d, max_steps=37)  # MaxSteps terminations leave through the generic funnel
    assert (r.term == 2).any() and (r.term == 0).any()


@pytest.mark.parametrize("cache", [True, False])
def test_vertex_to_vertex_walks(gpu, cache):
    xyz, tri = W.torus(1 / 3, 1 / 6, 64, 32)
    m = gpu.Mesh(xyz, tri, transport_cache=cache)
    f, b, d = W.vertex_edge_queries(xyz, tri, 4000, 1.0, seed=5)
    f2, b2, d2 = W.sample_queries(xyz, tri, 4000, 1.0, seed=6)
    both_walkers(m, np.concatenate([f, f2]), np.concatenate([b, b2]), np.concatenate([d, d2]))


@pytest.mark.parametrize("cache", [True, False])
def test_flat_grid_exact_zeros_and_boundary(gpu, ref, cache):
    """Axis-aligned directions on a planar grid: zero numerators in every quotient, vertex hits,
    edge-tangent slides and boundary stops."""
    rm = ref.RefMesh.plane(12, 12, 1.0, 0)
    a = rm.arrays()
    m = gpu.Mesh(a["xyz"], a["tri"], transport_cache=cache)
    f, b, d = rm.sample_queries(21, 6000, 0.05, 3.0)
    d[:1500] = np.array([1.0, 0.0, 0.0]) * np.linalg.norm(d[:1500], axis=1, keepdims=True)
    d[1500:3000] = np.array([0.0, -1.0, 0.0]) * np.linalg.norm(d[1500:3000], axis=1, keepdims=True)
    b[3000:3300] = np.array([0.5, 0.5, 0.0])       # starts on an edge
    b[3300:3600] = np.array([0.0, 0.0, 1.0])       # starts at a vertex
    r = both_walkers(m, f, b, d)
    assert (r.term == 1).any()                      # some leave through the boundary
    ours = m.trace_batch(f, b, d, record_polyline=True)
    theirs = rm.trace_batch(f, b, d, record_polyline=True)
    assert np.array_equal(ours.face, theirs.face) and np.array_equal(ours.poly_face, theirs.poly_face)
    # bit-equal to the reference wherever no vertex branch (libm atan2 / sincos) was taken
    no_vertex = np.ones(len(f), bool)
    at_vertex = (theirs.poly_bary == 1.0).any(1)
    np.logical_and.at(no_vertex, np.repeat(np.arange(len(f)), np.diff(theirs.poly_offsets)), ~at_vertex)
    assert no_vertex.sum() > 3000
    assert np.array_equal(r.face, theirs.face)
    assert np.array_equal(r.bary[no_vertex], theirs.bary[no_vertex]) and np.array_equal(r.dir[no_vertex], theirs.dir[no_vertex])
    assert np.abs(r.bary - theirs.bary).max() < 1e-9 and np.abs(r.dir - theirs.dir).max() < 1e-9


def test_rejected_and_degenerate_starts(gpu):
    xyz, tri = W.icosphere(3)
    m = gpu.Mesh(xyz, tri)
    f, b, d = W.sample_queries(xyz, tri, 2000, 1.0, seed=1)
    f[10] = -1; f[11] = len(tri)                   # face out of range
    b[20] = [0.7, 0.7, 0.7]                        # not in the simplex
    d[30] = 0.0                                    # zero-length request
    n = np.cross(xyz[tri[f[40], 1]] - xyz[tri[f[40], 0]], xyz[tri[f[40], 2]] - xyz[tri[f[40], 0]])
    d[40] = n / np.linalg.norm(n)                  # normal to the anchor face
    d[50] *= 1e-300                                # tiny but positive length
    b[60] = [np.nan, 0.5, 0.5]
    d[70] = [np.nan, 0.0, 1.0]
    r = both_walkers(m, f, b, d)
    assert list(r.stall[[10, 11, 20, 40]]) == [4, 4, 5, 3] and r.traced[30] == 0.0


@pytest.mark.parametrize("key,n", [("c2", 60_000), ("c3", 12_000)])
def test_baseline_configs_against_the_reference(gpu, ref, key, n):
    """BASELINE.json's meshes at full size (config 2: 81 920 faces, crossing records gathered with
    256-bit loads; config 3: 1 M faces, 384 MB of crossing records gathered through TMA
    tile::gather4) on a prefix of the benchmark's own query stream: final face,
    barycentrics, direction, traced length and the whole face sequence against the UNMODIFIED
    reference -- bit for bit (random starts never take a vertex branch), plus EP gradients."""
    import sys, os
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from bench import make_workload
    xyz, tri, f, b, d, q = make_workload(key, n, 42)
    m = gpu.Mesh(xyz, tri)
    assert m.has_transport_cache
    rm = ref.RefMesh.build(xyz, tri)
    ours = both_walkers(m, f, b, d)
    theirs = rm.trace_batch(f, b, d, record_polyline=True)
    for k in ("face", "bary", "dir", "traced", "requested", "term", "status"):
        assert np.array_equal(getattr(ours, k), getattr(theirs, k)), k
    assert np.array_equal(ours.npoints, theirs.npoints)
    assert ours.total_crossings == int((theirs.npoints - 2).sum())  # one polyline point per advance + the start
    poly = m.trace_batch(f[:2000], b[:2000], d[:2000], record_polyline=True)
    keep = theirs.poly_offsets[2000]
    assert np.array_equal(poly.poly_face, theirs.poly_face[:keep]) and np.array_equal(poly.poly_bary, theirs.poly_bary[:keep])
    g = 2.0 * (m.embed(ours.face, ours.bary) - q)  # gradcheck.cpp:88
    assert np.array_equal(m.ep_backward(f, d, ours.face, ours.dir, g),
                          rm.ep(f, b, d, theirs.face, theirs.bary, theirs.dir, g=g)["grad_v"])


def test_randomised_meshes_scales_and_starts(gpu):
    """scripts/fuzz_walkers.py, a short run: random mesh families at scales from 1e-160 to 1e+160
    (the operand-range guards of the hand-expanded divisions), slivers, lengths over 9 decades,
    vertex / edge / along-edge / rejected starts, tight step limits -- fast walker == general walker
    bit for bit on both layouts, and the two layouts agree."""
    import os, sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))
    import fuzz_walkers
    assert fuzz_walkers.main(rounds=24, n=6000, seed=11) == 0


@pytest.mark.parametrize("records", ["half-size", "128-byte"])
@pytest.mark.parametrize("key,n", [("c1", 10_000), ("c2", 200_000), ("c3", 60_000)])
def test_tolerance_lane_parity_gate(gpu, ref, key, n, records, monkeypatch):
    """DG_LANE_FAST, the opt-in tolerance lane of the plain forward map: the intrinsic fold over half-size (64-byte)
    crossing records -- no in_from, no Gram solve, rsqrt normalisation -- and, where a mesh has no such records
    (DG_LANE_FAST_128 forces it here), the fast step over the 128-byte records with reciprocal-multiply quotients, one
    reciprocal for the exit parameter, no second renormalising snap, first-order renormalisation. Its bar is
    north_star's, stated here: identical face sequences and end faces on the (non-degenerate) random queries of
    configs 1-3, end points within 1e-9 x bbox diagonal, directions within 1e-9, traced length within 1e-9 relative --
    against the EXACT lane and against the UNMODIFIED reference; GFD Jacobians through the lane within 1e-5 relative
    to the largest entry of the reference's, pulled-back gradients cos >= 0.999999."""
    import sys, os
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from bench import make_workload
    if key == "c1":
        xyz, tri = W.icosphere(4)
        f, b, d = W.sample_queries(xyz, tri, n, 1.0, seed=42)
    else:
        xyz, tri, f, b, d, _ = make_workload(key, n, 42)
    if records == "128-byte":
        monkeypatch.setenv("DG_LANE_FAST_128", "1")
    m = gpu.Mesh(xyz, tri)
    diag = W.bbox_diagonal(xyz)
    exact = m.trace_batch(f, b, d, sort_by_face=False)
    fast = m.trace_batch(f, b, d, lane="fast", sort_by_face=False)
    assert np.array_equal(fast.face, exact.face) and np.array_equal(fast.crossings, exact.crossings)
    assert np.array_equal(fast.term, exact.term) and np.array_equal(fast.status, exact.status)
    assert not np.array_equal(fast.bary, exact.bary)            # it IS another arithmetic
    assert np.abs(m.embed(fast.face, fast.bary) - m.embed(exact.face, exact.bary)).max() <= 1e-9 * diag
    assert np.abs(fast.dir - exact.dir).max() <= 1e-9
    assert np.abs(fast.traced - exact.traced).max() <= 1e-9 * np.abs(exact.traced).max()
    k = min(n, 20_000)
    rm = ref.RefMesh.build(xyz, tri)
    theirs = rm.trace_batch(f[:k], b[:k], d[:k], record_polyline=True)
    assert np.array_equal(fast.face[:k], theirs.face)
    assert np.array_equal(fast.crossings[:k], (theirs.npoints - 2).clip(min=0))   # as many crossings, i.e. the same walk
    assert np.abs(m.embed(fast.face[:k], fast.bary[:k]) - rm.embed(theirs.face, theirs.bary)).max() <= 1e-9 * diag
    assert np.abs(fast.dir[:k] - theirs.dir).max() <= 1e-9
    # GFD through the lane (fused forward + Jacobians): forward record as above, Jacobians within the GFD tolerance
    s = min(n, 4000)
    g = np.random.default_rng(3).normal(size=(s, 3))
    r, jac = m.trace_gfd(f[:s], b[:s], d[:s], lane="fast")
    assert np.array_equal(r.face, exact.face[:s])
    rg = rm.gfd(f[:s], b[:s], d[:s], g=g)
    for name in ("jv", "jp"):
        assert np.abs(jac[name] - rg[name]).max() <= 1e-5 * np.abs(rg[name]).max(), name
    assert np.array_equal(jac["degraded"], rg["degraded"])
    pb = m.gfd_pullback(f[:s], d[:s], r.face, jac["jv"], jac["jp"], g)
    for name in ("grad_v", "grad_p"):
        num = np.einsum("nd,nd->n", pb[name], rg[name])
        den = np.linalg.norm(pb[name], axis=1) * np.linalg.norm(rg[name], axis=1)
        ok = den > 1e-12
        assert (num[ok] / den[ok]).min() >= 0.999999, name


def test_corner_angle_table_changes_no_bit(gpu, monkeypatch):
    """The fan walk (tracer.cpp:252-311) takes the interior angle of every fan face from a table built at upload by
    the function it would call itself: vertex-to-vertex walks with and without the table, every bit, both walkers."""
    from paper_2603_15780_b200 import workloads as W
    xyz, tri = W.torus(1 / 3, 1 / 6, 96, 48, noise=0.05, seed=3)
    f, b, d = W.vertex_edge_queries(xyz, tri, 20_000, 3.0, seed=5, meridian=True)
    fr, br, dr = W.sample_queries(xyz, tri, 5_000, 1.5, seed=6)
    br[::3] = [1.0, 0.0, 0.0]                       # vertex starts in arbitrary directions
    f, b, d = np.concatenate([f, fr]), np.concatenate([b, br]), np.concatenate([d, dr])
    with_table = gpu.Mesh(xyz, tri)
    monkeypatch.setenv("DG_CORNER_ANGLES", "0")
    without = gpu.Mesh(xyz, tri)
    monkeypatch.delenv("DG_CORNER_ANGLES")
    assert with_table.device_bytes - without.device_bytes == 3 * len(tri) * 8
    for kw in (dict(), dict(walker="generic"), dict(record_polyline=True)):
        x, y = with_table.trace_batch(f, b, d, **kw), without.trace_batch(f, b, d, **kw)
        for k in FIELDS + (("poly_face", "poly_bary", "poly_seg") if kw.get("record_polyline") else ()):
            assert np.array_equal(getattr(x, k), getattr(y, k), equal_nan=True), (kw, k)
        assert x.total_crossings == y.total_crossings and (x.npoints > 50).any()
