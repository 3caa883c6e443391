"""CPU tier: pins the plain-C oracle (oracle/digeo_oracle.c) and the host-compiled device state
machine (tests/hostcheck) against (1) the golden fixtures generated from the unmodified
reference (tests/golden/*.npz, made by tests/golden/make_golden.py), (2) the reference's own
golden trace values (proj/tests/golden/trace_square.json, restated below) and (3) -- when
oracle/_ref is present -- the reference itself on fresh seeded inputs."""
import glob
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
TRACE_FIXTURES = sorted(p for p in glob.glob(os.path.join(HERE, "golden", "*.npz")) if "diff" not in p)


@pytest.fixture(scope="session")
def oracle():
    import __graft_entry__  # noqa: F401
    import oracle_api
    if not oracle_api.available():
        import subprocess
        subprocess.check_call(["make", "-C", os.path.join(os.path.dirname(HERE), "oracle"), "liboracle.so"])
    return oracle_api


@pytest.fixture(scope="session")
def hostcheck():
    import hostcheck_api
    hostcheck_api.build()
    return hostcheck_api


def _equal(a, b):
    return bool(((a == b) | (np.isnan(a) & np.isnan(b))).all())


def check_against_fixture(z, r, exact):
    n = len(z["face"])
    for k in ("face", "term", "status", "npoints"):
        assert np.array_equal(z["o_" + k], getattr(r, k)), k
    assert np.array_equal(z["poly_face"], r.poly_face), "face sequence"
    pairs = [("o_bary", r.bary), ("o_dir", r.dir), ("o_traced", r.traced), ("o_requested", r.requested),
             ("poly_bary", r.poly_bary), ("poly_seg", r.poly_seg)]
    if z["payload"].size:
        pairs.append(("o_payload", r.payload))
    if z["cfg"][2]:
        pairs.append(("o_q", r.q))
    for k, got in pairs:
        if exact:
            assert _equal(z[k], got), f"{k} not bit-equal ({n} traces)"
        else:
            assert np.nanmax(np.abs(z[k] - got)) <= 1e-12, k


@pytest.mark.parametrize("path", TRACE_FIXTURES, ids=[os.path.basename(p)[:-4] for p in TRACE_FIXTURES])
def test_oracle_matches_reference_fixtures(oracle, path):
    z = np.load(path)
    m = oracle.OracleMesh(z["xyz"], z["tri"])
    assert np.array_equal(m.arrays()["adj"], z["adj"]) and np.array_equal(m.arrays()["vangle"], z["vangle"])
    assert m.mean_edge == float(z["mean_edge"])
    pay = z["payload"] if z["payload"].size else None
    r = m.trace_batch(z["face"], z["bary"], z["dir"], payload=pay, max_steps=int(z["cfg"][0]),
                      hole_avoidance=bool(z["cfg"][1]), want_q=bool(z["cfg"][2]), record_polyline=True)
    check_against_fixture(z, r, exact=True)  # same libm on the host: bit-exact including vertex branches


@pytest.mark.parametrize("path", TRACE_FIXTURES, ids=[os.path.basename(p)[:-4] for p in TRACE_FIXTURES])
def test_device_state_machine_on_host_matches_fixtures(hostcheck, oracle, path):
    """The kernel's state machine (dg_tracer_core.cuh) compiled for the host reproduces the
    reference fixtures bit for bit -- control flow and arithmetic are checked before any GPU time."""
    z = np.load(path)
    a = oracle.OracleMesh(z["xyz"], z["tri"]).arrays()
    hm = hostcheck.HostMesh(a)
    pay = z["payload"] if z["payload"].size else None
    r = hm.trace_batch(z["face"], z["bary"], z["dir"], payload=pay, max_steps=int(z["cfg"][0]),
                       hole_avoidance=bool(z["cfg"][1]), want_q=bool(z["cfg"][2]), record_polyline=True)
    check_against_fixture(z, r, exact=True)


@pytest.mark.parametrize("cached", [False, True], ids=["face-records", "crossing-records"])
@pytest.mark.parametrize("path", TRACE_FIXTURES, ids=[os.path.basename(p)[:-4] for p in TRACE_FIXTURES])
def test_fast_walker_on_host_matches_fixtures(hostcheck, oracle, path, cached):
    """The fast walker (csrc/dg_fast_walk.cuh: lean start-up, fast step, finish, and the generic
    paths it hands everything else to) compiled for the host and driven the way the kernel drives
    a lane: end states and counters of the reference fixtures, bit for bit, on both mesh layouts.
    (Fixtures with a payload run the payload lane of the fast walker and pin the transported
    payload as well; hole-avoidance fixtures run it with the full Tracer behind the fast step;
    transport-matrix fixtures run the variant that carries the three matrix columns.)"""
    z = np.load(path)
    a = oracle.OracleMesh(z["xyz"], z["tri"]).arrays()
    hm = hostcheck.HostMesh(a)
    pay = z["payload"] if z["payload"].size else None
    r = hm.trace_batch_fast(z["face"], z["bary"], z["dir"], max_steps=int(z["cfg"][0]), cached=cached, payload=pay,
                            hole_avoidance=bool(z["cfg"][1]), record_polyline=True, want_q=bool(z["cfg"][2]))
    assert np.array_equal(z["poly_face"], r.poly_face), "face sequence"
    assert _equal(z["poly_bary"], r.poly_bary) and _equal(z["poly_seg"], r.poly_seg)
    for k in ("face", "term", "status", "npoints"):
        assert np.array_equal(z["o_" + k], getattr(r, k)), k
    pairs = [("o_bary", r.bary), ("o_dir", r.dir), ("o_traced", r.traced), ("o_requested", r.requested)]
    if pay is not None:
        pairs.append(("o_payload", r.payload))   # the payload lane of the fast walker (kPay)
    if z["cfg"][2]:
        pairs.append(("o_q", r.q))               # the transport-matrix lane (kPay == 2)
    for k, got in pairs:
        assert _equal(z[k], got), f"{k} not bit-equal"
    g = hm.trace_batch(z["face"], z["bary"], z["dir"], max_steps=int(z["cfg"][0]), hole_avoidance=bool(z["cfg"][1]))
    assert np.array_equal(g.crossings, r.crossings) and np.array_equal(g.stall, r.stall)


@pytest.mark.parametrize("cached", [False, True], ids=["face-records", "crossing-records"])
def test_fast_walker_on_host_vs_reference_fresh_inputs(hostcheck, ref, cached):
    """Differential check of the host-compiled fast walker against the unmodified reference on
    meshes and inputs that are not in the fixtures, including every way out of the fast step:
    vertex starts, edge starts, axis-aligned directions on a flat grid (exact zeros), boundary
    stops, a tight step limit, rejected and zero-length starts."""
    cases = [(ref.RefMesh.icosphere(4), 81, 0.1, 3.0, 0), (ref.RefMesh.torus(1 / 3, 1 / 6, 48, 24), 82, 0.05, 2.0, 0),
             (ref.RefMesh.plane(10, 8, 1.0, 0), 83, 0.05, 2.0, 0), (ref.RefMesh.cylinder(0.5, 1.0, 16, 4), 84, 0.05, 3.0, 0),
             (ref.RefMesh.icosphere(3), 85, 1.0, 6.0, 9)]
    for rm, seed, lo, hi, max_steps in cases:
        hm = hostcheck.HostMesh(rm.arrays())
        f, b, d = rm.sample_queries(seed, 4000, lo, hi)
        d[:400] = np.array([1.0, 0.0, 0.0]) * np.linalg.norm(d[:400], axis=1, keepdims=True)   # may leave the face plane: projected
        b[400:500] = [0.5, 0.5, 0.0]
        b[500:600] = [0.0, 1.0, 0.0]
        f[600] = -1; b[601] = [0.9, 0.9, 0.9]; d[602] = 0.0
        theirs = rm.trace_batch(f, b, d, record_polyline=True, max_steps=max_steps)
        ours = hm.trace_batch_fast(f, b, d, max_steps=max_steps or rm.default_max_steps(), cached=cached)
        for k in ("face", "term", "status", "npoints"):
            assert np.array_equal(getattr(theirs, k), getattr(ours, k)), k
        for k in ("bary", "dir", "traced", "requested"):
            assert _equal(getattr(theirs, k), getattr(ours, k)), k   # same libm on the host: exact on vertex branches too
        assert (ours.crossings[ours.term == 0] >= 0).all()


def test_golden_square_trace_values(oracle):
    """proj/tests/golden/trace_square.json, compared bit-for-bit by the reference (test_io.cpp:71-82)."""
    m = oracle.OracleMesh([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0]], [[0, 1, 2], [0, 2, 3]])
    r = m.trace_batch([0], [[.5, .25, .25]], [[.25, .5, 0]], record_polyline=True)
    assert r.face[0] == 1 and r.bary[0].tolist() == [0.24999999999999992, 0.75000000000000011, 0.0]
    assert r.poly_face.tolist() == [0, 0, 1]
    assert r.poly_bary.tolist() == [[.5, .25, .25], [.25, 0.0, .75], [0.24999999999999992, 0.75000000000000011, 0.0]]
    assert r.poly_seg.tolist() == [0.0, 0.55901699437494734, 1.1102230246251565e-16]
    assert r.dir[0].tolist() == [0.44721359549995771, 0.89442719099991608, 0.0]
    assert r.term[0] == 0 and r.status[0] == 0
    # boundary stop known answer
    r = m.trace_batch([0], [[.5, .25, .25]], [[2, .1, 0]])
    assert r.term[0] == 1 and r.bary[0].tolist() == [0.0, 0.72500000000000009, 0.27499999999999997]
    assert r.traced[0] == 0.50062460986251966 and r.requested[0] == 2.0024984394500787


def test_oracle_differentials_match_fixture(oracle):
    z = np.load(os.path.join(HERE, "golden", "ico3_diff.npz"))
    m = oracle.OracleMesh(z["xyz"], z["tri"])
    ep = m.ep(z["face"], z["bary"], z["dir"], z["end_face"], z["end_bary"], z["end_dir"], g=z["g"])
    assert np.array_equal(ep["rot"], z["ep_rot"]) and np.array_equal(ep["frames"], z["ep_frames"])
    assert np.array_equal(ep["grad_v"], z["ep_grad_v"]) and not ep["grad_p"].any()
    assert m.default_gfd_eps() == float(z["eps"])
    gfd = m.gfd(z["face"], z["bary"], z["dir"], g=z["g"])
    for k in ("jv", "jp", "degraded", "frames", "grad_v", "grad_p"):
        assert np.array_equal(gfd[k], z["gfd_" + k]), k


def test_oracle_error_classes(oracle):
    with pytest.raises(oracle.OracleError) as e:
        oracle.OracleMesh([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [0, -1, 0]], [[0, 1, 2], [0, 1, 3], [1, 0, 4]])
    assert e.value.klass == "NonManifoldError" and e.value.msg == "edge (0,1) incident to 3+ faces"
    with pytest.raises(oracle.OracleError) as e:
        oracle.OracleMesh([[0, 0, 0], [1, 0, 0], [2, 0, 0]], [[0, 1, 2]])
    assert e.value.klass == "DegenerateFaceError" and e.value.msg == "face 0 has zero area"


def test_oracle_vs_reference_fresh_inputs(oracle, ref):
    """Differential check against the unmodified reference on inputs that are not in the fixtures."""
    for rm, seed, lo, hi in ((ref.RefMesh.icosphere(3), 77, 0.1, 3.0), (ref.RefMesh.torus(1 / 3, 1 / 6, 40, 20), 78, 0.05, 2.0),
                             (ref.RefMesh.cylinder(0.5, 1.0, 16, 4), 79, 0.05, 3.0)):
        a = rm.arrays()
        m = oracle.OracleMesh(a["xyz"], a["tri"])
        for k in ("adj", "fnormal", "farea", "vangle", "varea", "vboundary", "csr_off", "csr_list"):
            assert np.array_equal(m.arrays()[k], a[k]), k
        f, b, d = rm.sample_queries(seed, 3000, lo, hi)
        pay = np.random.default_rng(seed).normal(size=(len(f), 3))
        for hole in (False, True):
            r = rm.trace_batch(f, b, d, payload=pay, want_q=True, record_polyline=True, hole_avoidance=hole)
            o = m.trace_batch(f, b, d, payload=pay, want_q=True, record_polyline=True, hole_avoidance=hole)
            for k in ("face", "bary", "dir", "traced", "term", "status", "npoints", "payload", "q", "poly_face",
                      "poly_bary", "poly_seg"):
                assert _equal(np.asarray(getattr(r, k), float), np.asarray(getattr(o, k), float)), (k, hole)
            assert r.errors == o.errors


@pytest.mark.parametrize("records", [1, 2], ids=["128-byte records", "half-size records"])
def test_tolerance_lane_on_host_vs_reference(hostcheck, ref, records):
    """DG_LANE_FAST (the opt-in tolerance lane of the fast step: reciprocal-multiply quotients, one reciprocal for the
    exit parameter, no second renormalising snap, first-order direction renormalisation), compiled for the host and
    driven the way the kernel drives a lane, against the unmodified reference: identical end faces, termination and
    point counts -- i.e. the same walks, every way out of the fast step included --, end points within 1e-9 x bbox
    diagonal, directions within 1e-9, lengths within 1e-9 relative; and it really is another arithmetic (not
    bit-equal on plain traces)."""
    cases = [(ref.RefMesh.icosphere(4), 91, 0.1, 3.0), (ref.RefMesh.torus(1 / 3, 1 / 6, 48, 24), 92, 0.05, 2.0),
             (ref.RefMesh.plane(10, 8, 1.0, 0), 93, 0.05, 2.0)]
    for rm, seed, lo, hi in cases:
        hm = hostcheck.HostMesh(rm.arrays())
        f, b, d = rm.sample_queries(seed, 4000, lo, hi)
        b[400:500] = [0.5, 0.5, 0.0]        # edge starts
        b[500:600] = [0.0, 1.0, 0.0]        # vertex starts
        f[600] = -1; d[602] = 0.0
        theirs = rm.trace_batch(f, b, d, record_polyline=True)
        ours = hm.trace_batch_fast(f, b, d, max_steps=rm.default_max_steps(), cached=True, lane_fast=records)
        for k in ("face", "term", "status", "npoints"):
            assert np.array_equal(getattr(theirs, k), getattr(ours, k)), k
        diag = np.linalg.norm(rm.xyz.max(0) - rm.xyz.min(0))
        ok = theirs.face >= 0
        assert np.abs(rm.embed(ours.face[ok], ours.bary[ok]) - rm.embed(theirs.face[ok], theirs.bary[ok])).max() <= 1e-9 * diag
        assert np.abs(ours.dir - theirs.dir).max() <= 1e-9
        assert np.abs(ours.traced - theirs.traced).max() <= 1e-9 * max(1.0, np.abs(theirs.traced).max())
        plain = ok & (theirs.npoints > 3)
        assert not np.array_equal(ours.bary[plain], theirs.bary[plain])
