"""Parity of the EP / GFD differentials and the single-transition operations with the
UNMODIFIED reference (proj/src/diff.cpp, tracer.cpp:630-735) through the C-ABI.
Mirrors proj/tests/test_diff.cpp.

Bar: EP is pure f64 arithmetic in the reference's operation order -> bit-identical given the
same forward result. GFD Jacobians are finite differences of end points divided by
eps ~ 1e-4 x mean edge, so last-ulp differences of vertex-branch traces are amplified:
tolerance 1e-5 relative to the largest entry; on traces without vertex
branches they are bit-identical too."""
import numpy as np
import pytest

from conftest import gpu_mesh

pytestmark = pytest.mark.gpu


def unit_rows(rng, n):
    q = rng.normal(size=(n, 3))
    return q / np.linalg.norm(q, axis=1, keepdims=True)


@pytest.mark.parametrize("fixture", ["ico4", "torus", "plane"])
def test_ep_bit_exact(gpu, ref, fixture):
    rm = {"ico4": lambda: ref.RefMesh.icosphere(4), "torus": lambda: ref.RefMesh.torus(1 / 3, 1 / 6, 64, 32),
          "plane": lambda: ref.RefMesh.plane(10, 10, 1.0, 3)}[fixture]()
    m = gpu_mesh(gpu, rm)
    f, b, d = rm.sample_queries(42, 10000, 0.1, 1.0)
    h = m.trace_batch(f, b, d)
    rng = np.random.default_rng(1)
    g = 2.0 * (m.embed(h.face, h.bary) - unit_rows(rng, len(f)))  # gradcheck.cpp:88
    ours = m.ep(f, b, d, h.face, h.bary, h.dir, g=g)
    theirs = rm.ep(f, b, d, h.face, h.bary, h.dir, g=g)
    for k in ("rot", "frames", "grad_v", "grad_p"):
        assert np.array_equal(ours[k], theirs[k]), k
    assert not ours["grad_p"].any()  # EP: grad_p is exactly zero (test_diff.cpp:361)
    # R is a rotation (test_diff.cpp:65-79)
    R = ours["rot"].reshape(-1, 3, 3)
    assert np.abs(R @ R.transpose(0, 2, 1) - np.eye(3)).max() < 1e-9
    assert np.abs(np.linalg.det(R) - 1).max() < 1e-9
    if fixture == "plane":
        assert np.abs(R - np.eye(3)).max() < 1e-12  # EP on a plane is the identity (test_diff.cpp:50-63)


def test_ep_degenerate_direction_errors(gpu, ref):
    rm = ref.RefMesh.icosphere(2)
    m = gpu_mesh(gpu, rm)
    f, b, d = rm.sample_queries(3, 16, 1.0, 1.0)
    h = m.trace_batch(f, b, d)
    d2 = d.copy()
    d2[5] = 0
    with pytest.raises(gpu.DgError) as e:
        m.ep(f, b, d2, h.face, h.bary, h.dir)
    assert e.value.klass == "DegenerateDirection" and e.value.index == 5 and "too small" in e.value.msg
    with pytest.raises(ref.RefError) as er:
        rm.ep(f, b, d2, h.face, h.bary, h.dir)
    assert er.value.klass == "DegenerateDirection" and er.value.index == 5
    d3 = d.copy()
    d3[7] = rm.arrays()["fnormal"][f[7]]
    with pytest.raises(gpu.DgError) as e:
        m.ep(f, b, d3, h.face, h.bary, h.dir)
    assert e.value.klass == "DegenerateDirection" and e.value.index == 7 and "normal to the face" in e.value.msg


@pytest.mark.parametrize("fixture,n", [("ico4", 4000), ("torus", 3000), ("cyl", 2000)])
def test_gfd_matches_reference(gpu, ref, fixture, n):
    rm = {"ico4": lambda: ref.RefMesh.icosphere(4), "torus": lambda: ref.RefMesh.torus(1 / 3, 1 / 6, 64, 32),
          "cyl": lambda: ref.RefMesh.cylinder(0.5, 4.0, 24, 24)}[fixture]()
    m = gpu_mesh(gpu, rm)
    f, b, d = rm.sample_queries(9, n, 0.1, 0.8)
    if fixture == "cyl":  # keep base traces on the open cylinder
        base = rm.trace_batch(f, b, d)
        keep = (base.term == 0) & (base.status == 0)
        f, b, d = f[keep], b[keep], d[keep]
    rng = np.random.default_rng(2)
    g = unit_rows(rng, len(f))
    assert m.default_gfd_eps() == rm.default_gfd_eps()
    ours = m.gfd(f, b, d, g=g)
    theirs = rm.gfd(f, b, d, g=g)
    assert np.array_equal(ours["degraded"], theirs["degraded"])
    assert np.array_equal(ours["frames"], theirs["frames"])
    for k in ("jv", "jp"):
        scale = np.abs(theirs[k]).max()
        assert np.abs(ours[k] - theirs[k]).max() <= 1e-5 * scale, k
    for k in ("grad_v", "grad_p"):
        num = np.einsum("nd,nd->n", ours[k], theirs[k])
        den = np.linalg.norm(ours[k], axis=1) * np.linalg.norm(theirs[k], axis=1)
        ok = den > 1e-12
        assert (num[ok] / den[ok]).min() >= 0.999999, k
        assert np.abs(np.linalg.norm(ours[k], axis=1)[ok] / np.linalg.norm(theirs[k], axis=1)[ok] - 1).max() <= 1e-4
    # the base end states are the forward trace
    h = m.trace_batch(f, b, d)
    assert np.array_equal(ours["base_face"], h.face) and np.array_equal(ours["base_bary"], h.bary)
    # batched == unbatched exactly (test_diff.cpp:139-171): same kernel, any batch composition
    sub = m.gfd(f[:64], b[:64], d[:64], g=g[:64])
    assert np.array_equal(sub["jv"], ours["jv"][:64]) and np.array_equal(sub["jp"], ours["jp"][:64])


@pytest.mark.parametrize("cache", [True, False])
def test_gfd_sibling_schedule_and_known_base_change_no_bit(gpu, ref, cache):
    """Round 2 of GFD runs the full-length re-traces of a sample as sibling lanes of one warp
    (dg_diff_cfg.schedule, TraceParams::siblings: groups of 3 with the caller's forward results as
    base traces, of 4 without). It is a schedule, not an algorithm: every output is bit-identical
    to the plain job order, with and without a known base, on both mesh layouts, for batch sizes
    that do not fill the last group or warp, and on an open mesh where some columns take the
    one-sided fallback."""
    for rm, n, eps in ((ref.RefMesh.torus(1 / 3, 1 / 6, 64, 32), 5003, None), (ref.RefMesh.icosphere(3), 61, None),
                       (ref.RefMesh.plane(6, 6, 1.0, 0), 2500, 1e-3)):
        a = rm.arrays()
        m = gpu.Mesh(a["xyz"], a["tri"], transport_cache=cache)
        f, b, d = rm.sample_queries(21, n, 0.05, 0.7)
        base = m.trace_batch(f, b, d)
        if eps is not None:   # traces that hit the boundary end 1e-9 before it instead: their + perturbations leave the mesh
            hit = base.term == 1
            d[hit] *= ((base.traced[hit] - 1e-9) / base.requested[hit])[:, None]
            base = m.trace_batch(f, b, d)
        keep = (base.term == 0) & (base.status == 0)
        if eps is not None:   # seeds (eps-length) must stay on the open mesh
            P = rm.embed(f, b)
            keep &= (P[:, :2].min(1) > 0.02) & (P[:, :2].max(1) < 0.98)
        f, b, d = f[keep], b[keep], d[keep]
        base = m.trace_batch(f, b, d)
        g = unit_rows(np.random.default_rng(3), len(f))
        kw = dict(g=g) if eps is None else dict(g=g, eps_v=eps, eps_p=eps)
        want = m.gfd(f, b, d, plain_schedule=True, **kw)
        # plain_schedule = 2: DG_GFD_SCHEDULE_FACE_ORDER, the sibling groups in start-face order of their samples
        # (groups of 4, and groups of 3 + a plain tail with a known base)
        for got in (m.gfd(f, b, d, **kw), m.gfd(f, b, d, base=base, **kw), m.gfd(f, b, d, base=base, plain_schedule=True, **kw),
                    m.gfd(f, b, d, plain_schedule=2, **kw), m.gfd(f, b, d, base=base, plain_schedule=2, **kw)):
            for k in ("jv", "jp", "degraded", "frames", "grad_v", "grad_p"):
                assert np.array_equal(got[k], want[k], equal_nan=True), k
        if eps is not None:
            assert want["degraded"].any(), "fixture must exercise the fallback"


def test_gfd_plane_is_identity(gpu, ref):
    """test_diff.cpp:89-112: on a flat mesh both Jacobians are the frame change of the identity."""
    rm = ref.RefMesh.plane(12, 12, 4.0, 5)
    m = gpu_mesh(gpu, rm)
    f, b, d = rm.sample_queries(4, 500, 0.05, 0.3)
    base = rm.trace_batch(f, b, d)
    keep = (base.term == 0) & (base.status == 0)
    f, b, d = f[keep], b[keep], d[keep]
    ours, theirs = m.gfd(f, b, d), rm.gfd(f, b, d)
    assert np.abs(ours["jv"] - theirs["jv"]).max() <= 1e-6
    assert np.abs(ours["jp"] - theirs["jp"]).max() <= 1e-6


def test_gfd_one_sided_fallback_near_boundary(gpu, ref):
    """Columns whose + perturbation leaves an open mesh fall back to the - side and are flagged
    (diff.cpp:130-137)."""
    rm = ref.RefMesh.plane(6, 6, 1.0, 0)
    m = gpu_mesh(gpu, rm)
    a = rm.arrays()
    # traces that end exactly on / next to the boundary: aim at boundary points with full length
    rng = np.random.default_rng(6)
    f, b, d = rm.sample_queries(5, 3000, 0.05, 0.6)
    base = rm.trace_batch(f, b, d)
    P = rm.embed(f, b)
    # shorten traces that hit the boundary so that they end 1e-9 before it
    hit = base.term == 1
    d[hit] *= ((base.traced[hit] - 1e-9) / base.requested[hit])[:, None]
    base = rm.trace_batch(f, b, d)
    P = rm.embed(f, b)
    inside = (P[:, :2].min(1) > 0.02) & (P[:, :2].max(1) < 0.98)  # seeds (eps-length) must stay on the mesh
    keep = (base.term == 0) & (base.status == 0) & inside
    f, b, d = f[keep], b[keep], d[keep]
    eps = 1e-3
    theirs = rm.gfd(f, b, d, eps_v=eps, eps_p=eps)
    ours = m.gfd(f, b, d, eps_v=eps, eps_p=eps)
    assert theirs["degraded"].any(), "fixture must exercise the fallback"
    assert np.array_equal(ours["degraded"], theirs["degraded"])
    assert np.abs(ours["jv"] - theirs["jv"]).max() <= 1e-6
    assert np.abs(ours["jp"] - theirs["jp"]).max() <= 1e-6


def test_gfd_whole_call_errors(gpu, ref):
    rm = ref.RefMesh.plane(4, 4, 1.0, 0)
    m = gpu_mesh(gpu, rm)
    f, b, d = rm.sample_queries(5, 64, 3.0, 4.0)  # every base trace leaves the unit square
    with pytest.raises(gpu.DgError) as e:
        m.gfd(f, b, d)
    assert e.value.klass == "Error" and e.value.msg == "gfd: the base trace did not reach its requested length"
    with pytest.raises(ref.RefError) as er:
        rm.gfd(f, b, d)
    assert er.value.msg == e.value.msg
    d[:] = 0
    with pytest.raises(gpu.DgError) as e:
        m.gfd(f, b, d)
    assert e.value.klass == "DegenerateDirection"


def test_gradcheck_medians_on_sphere(gpu, ref):
    """run_gradcheck's criteria (gradcheck.cpp:46-131, test_diff.cpp:350-361) on the GPU path:
    pullback of |Exp - q|^2 against the closed-form sphere gradient is checked indirectly by
    requiring our pulled-back gradients to reproduce the reference's medians."""
    rm = ref.RefMesh.icosphere(4)
    m = gpu_mesh(gpu, rm)
    f, b, d = rm.sample_queries(11, 2000, 0.2, 1.0)
    rng = np.random.default_rng(3)
    q = unit_rows(rng, len(f))
    h = m.trace_batch(f, b, d)
    g = 2.0 * (m.embed(h.face, h.bary) - q)
    ours, theirs = m.gfd(f, b, d, g=g), rm.gfd(f, b, d, g=g)
    cos = np.einsum("nd,nd->n", ours["grad_v"], theirs["grad_v"]) / (
        np.linalg.norm(ours["grad_v"], axis=1) * np.linalg.norm(theirs["grad_v"], axis=1))
    assert np.median(cos) >= 0.9999999


def test_single_transitions(gpu, ref):
    """geodesic_step / transport_over_edge / transport_over_vertex / boundary_continue."""
    rm = ref.RefMesh.icosphere(2)
    m = gpu_mesh(gpu, rm)
    rng = np.random.default_rng(8)
    n = 300
    f, b, d = rm.sample_queries(2, n, 1.0, 1.0)
    rem = rng.uniform(0.01, 0.5, n)
    o = m.transition(0, f, b, d, remaining=rem)
    for i in range(n):
        r = rm.geodesic_step(f[i], b[i], d[i], rem[i])
        assert o["rc"][i] == 0 and r["face"] == o["face"][i] and r["event"] == o["event"][i]
        assert np.array_equal(r["bary"], o["bary"][i]) and np.array_equal(r["dir"], o["v"][i])
        assert r["step_length"] == o["step_length"][i] and r["finished"] == bool(o["finished"][i])
    # edge points
    be = b.copy()
    k = rng.integers(0, 3, n)
    be[np.arange(n), k] = 0
    be /= be.sum(1, keepdims=True)
    o = m.transition(1, f, be, d)
    for i in range(n):
        rf, rb, rv = rm.transition(0, f[i], be[i], d[i])
        assert o["rc"][i] == 0 and rf == o["face"][i]
        assert np.array_equal(rb, o["bary"][i]) and np.array_equal(rv, o["v"][i])
    # vertex points
    bv = np.zeros((n, 3))
    bv[np.arange(n), k] = 1
    o = m.transition(2, f, bv, d)
    for i in range(n):
        rf, rb, rv = rm.transition(1, f[i], bv[i], d[i])
        assert o["rc"][i] == 0 and rf == o["face"][i]
        assert np.abs(rb - o["bary"][i]).max() <= 1e-12 and np.abs(rv - o["v"][i]).max() <= 1e-9
    # wrong point class -> InvalidArgs per element
    o = m.transition(1, f[:4], b[:4], d[:4])
    assert (o["rc"] == 1).all()
    with pytest.raises(ref.RefError):
        rm.transition(0, f[0], b[0], d[0])
    # boundary_continue on an open mesh
    pm = ref.RefMesh.plane(5, 5, 1.0, 0)
    mp = gpu_mesh(gpu, pm)
    a = pm.arrays()
    fb, kb = np.nonzero(a["adj"] < 0)
    nb = len(fb)
    tpar = rng.uniform(0.1, 0.9, nb)
    bb = np.zeros((nb, 3))
    bb[np.arange(nb), (kb + 1) % 3] = tpar
    bb[np.arange(nb), (kb + 2) % 3] = 1 - tpar
    dv = rng.normal(size=(nb, 3))
    dv[:, 2] = 0
    o = mp.transition(3, fb.astype(np.int32), bb, dv)
    for i in range(nb):
        rf, rb, rv = pm.transition(2, fb[i], bb[i], dv[i])
        assert o["rc"][i] == 0 and rf == o["face"][i]
        assert np.array_equal(rb, o["bary"][i]) and np.array_equal(rv, o["v"][i])


def test_fused_forward_gfd_and_pullback_give_the_bits_of_the_separate_calls(gpu, ref):
    """dg_trace_gfd: the forward traces ride in GFD's round 2 as the fourth sibling of their sample's re-traces and
    write the forward result record; dg_gfd_pullback pulls an upstream gradient back through the resident Jacobians.
    Forward results == dg_trace_batch, Jacobians == dg_gfd_jacobians, gradients == dg_gfd_jacobians with g -- all
    bit for bit, on both mesh layouts, incl. a batch with rejected / stalled / zero-length starts in the forward
    record and an open mesh where the one-sided fallback rounds run; and through the resident batch."""
    rng = np.random.default_rng(8)
    for rm, n, cache in ((ref.RefMesh.torus(1 / 3, 1 / 6, 64, 32), 5003, True), (ref.RefMesh.icosphere(3), 2000, False)):
        a = rm.arrays()
        m = gpu.Mesh(a["xyz"], a["tri"], transport_cache=cache)
        f, b, d = rm.sample_queries(31, n, 0.05, 0.9)
        g = unit_rows(rng, n)
        fwd = m.trace_batch(f, b, d)
        sep = m.gfd(f, b, d, g=g)
        r, jac = m.trace_gfd(f, b, d)
        for k in ("face", "bary", "dir", "traced", "requested", "term", "status", "stall", "npoints", "crossings"):
            assert np.array_equal(getattr(r, k), getattr(fwd, k)), k
        assert r.total_crossings == fwd.total_crossings
        for k in ("jv", "jp", "degraded", "frames"):
            assert np.array_equal(jac[k], sep[k]), k
        pb = m.gfd_pullback(f, d, r.face, jac["jv"], jac["jp"], g)
        assert np.array_equal(pb["grad_v"], sep["grad_v"]) and np.array_equal(pb["grad_p"], sep["grad_p"])
        # resident batch: forward with gfd=True, then the backward is the pull-back
        bt = gpu.Batch(m, n)
        rb = bt.trace(f, b, d, gfd=True)
        for k in ("face", "bary", "dir", "traced", "requested", "term", "status", "stall", "npoints", "crossings"):
            assert np.array_equal(getattr(rb, k), getattr(fwd, k)), k
        out = bt.gfd(g=g)
        for k in ("jv", "jp", "degraded", "grad_v", "grad_p"):
            assert np.array_equal(out[k], sep[k]), k
        out2 = bt.gfd(g=2 * g)   # another upstream gradient, same Jacobians
        assert np.array_equal(out2["grad_v"], m.gfd(f, b, d, g=2 * g)["grad_v"])
        bt.close()
    # the forward record of starts GFD cannot differentiate: the whole-call error comes with valid forward results
    rm = ref.RefMesh.icosphere(2)
    m = gpu_mesh(gpu, rm)
    f, b, d = rm.sample_queries(3, 64, 0.3, 1.0)
    d[5] = 0.0                                   # zero-length request: DegenerateDirection for GFD
    d[9] = rm.arrays()["fnormal"][f[9]]          # normal to the anchor face: stalls in the forward
    fwd = m.trace_batch(f, b, d)
    with pytest.raises(gpu.DgError) as e:
        m.trace_gfd(f, b, d)
    assert e.value.klass == "DegenerateDirection" and e.value.index == 5
    for k in ("face", "bary", "dir", "traced", "requested", "term", "status", "stall"):
        assert np.array_equal(getattr(e.value.forward, k), getattr(fwd, k)), k
    # open mesh: base traces that leave the mesh -> "gfd: the base trace did not reach its requested length"
    pm = ref.RefMesh.plane(6, 6, 1.0, 0)
    mp = gpu_mesh(gpu, pm)
    f, b, d = pm.sample_queries(4, 500, 0.5, 2.0)
    fwd = mp.trace_batch(f, b, d)
    assert (fwd.term == 1).any()
    with pytest.raises(gpu.DgError) as e:
        mp.trace_gfd(f, b, d)
    assert e.value.klass == "Error" and "base trace" in e.value.msg
    assert np.array_equal(e.value.forward.bary, fwd.bary) and np.array_equal(e.value.forward.term, fwd.term)
    keep = (fwd.term == 0) & (fwd.status == 0)
    P = pm.embed(f, b)
    keep &= (P[:, :2].min(1) > 0.02) & (P[:, :2].max(1) < 0.98)
    f, b, d = f[keep], b[keep], d[keep]
    sep = mp.gfd(f, b, d)
    r, jac = mp.trace_gfd(f, b, d)
    for k in ("jv", "jp", "degraded"):
        assert np.array_equal(jac[k], sep[k]), k
