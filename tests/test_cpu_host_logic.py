"""CPU tier: the C-ABI library loads and exports every declared symbol, fails loudly without a
device, the host-side mesh derivation matches the reference, workload generators are sane, and
the query-sharding logic is exact under a 2-rank gloo run."""
import ctypes
import os
import re
import subprocess
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def test_capi_exports_every_declared_symbol(dg):
    hdr = open(os.path.join(ROOT, "include", "dg_b200.h")).read()
    declared = set(re.findall(r"DG_API\s+[\w\s\*]+?\b(dg_\w+)\s*\(", hdr))
    assert len(declared) >= 18
    lib = ctypes.CDLL(dg.capi.LIB_PATH)
    for name in sorted(declared):
        assert hasattr(lib, name), f"{name} declared in include/dg_b200.h but not exported"
    assert set(dg.capi.EXPORTS) <= declared
    lib.dg_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.dg_version()


def test_library_is_sm100a_only():
    so = os.path.join(ROOT, "paper_2603_15780_b200", "lib", "libdigeo_b200.so")
    out = subprocess.run(["cuobjdump", "-lelf", so], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+\w?)", out))
    assert archs == {"100a"}, archs


def test_no_device_is_a_loud_error(dg):
    if dg.device_count() > 0:
        pytest.skip("a GPU is present")
    m = dg.Mesh([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0]], [[0, 1, 2], [0, 2, 3]], upload=False)
    with pytest.raises(dg.DgError) as e:
        m.upload()
    assert e.value.klass == "NoDevice" and "no CPU fallback" in e.value.msg
    with pytest.raises(dg.DgError):
        m.trace_batch(np.zeros(1, np.int32), [[.3, .3, .4]], [[1, 0, 0]])


def test_mesh_derive_matches_reference(dg, ref):
    for rm in (ref.RefMesh.icosphere(4), ref.RefMesh.torus(1 / 3, 1 / 6, 50, 20), ref.RefMesh.plane(9, 7, 1.0, 3),
               ref.RefMesh.cone(1, 1, 9), ref.RefMesh.cylinder(.5, 1, 12, 3)):
        a = rm.arrays()
        m = dg.Mesh(a["xyz"], a["tri"], upload=False)
        for k in ("adj", "fnormal", "farea", "vangle", "varea", "vboundary", "csr_off", "csr_list"):
            assert np.array_equal(a[k], getattr(m, k).reshape(a[k].shape)), k
        assert m.mean_edge == a["mean_edge"] and m.total_area == a["total_area"]
        assert m.default_max_steps() == rm.default_max_steps()


@pytest.mark.parametrize("xyz,tri,klass,msg", [
    ([[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[0, 1, 3]], "ParseError", "face 0 references vertex out of range"),
    ([[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[0, 1, 1]], "DegenerateFaceError", "face 0 has repeated vertices"),
    ([[0, 0, 0], [1, 0, 0], [2, 0, 0]], [[0, 1, 2]], "DegenerateFaceError", "face 0 has zero area"),
    ([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [0, -1, 0]], [[0, 1, 2], [0, 1, 3], [1, 0, 4]], "NonManifoldError",
     "edge (0,1) incident to 3+ faces"),
])
def test_mesh_derive_errors_match_reference(dg, ref, xyz, tri, klass, msg):
    with pytest.raises(dg.DgError) as e:
        dg.Mesh(xyz, tri, upload=False)
    assert e.value.klass == klass and e.value.msg == msg
    with pytest.raises(ref.RefError) as r:
        ref.RefMesh.build(xyz, tri)
    assert r.value.klass == klass and r.value.msg == msg


def test_workload_generators(dg, ref):
    from paper_2603_15780_b200 import workloads as W
    xyz, tri = W.icosphere(3)
    a = ref.RefMesh.icosphere(3).arrays()
    assert tri.shape == a["tri"].shape and np.allclose(np.linalg.norm(xyz, axis=1), 1)
    m = dg.Mesh(xyz, tri, upload=False)
    assert not m.vboundary.any() and (m.adj >= 0).all() and abs(m.total_area - a["total_area"]) < 1e-9
    xyz, tri = W.torus(1 / 3, 1 / 6, 40, 20, noise=0.1)
    mt = dg.Mesh(xyz, tri, upload=False)
    assert mt.nf == 1600 and (mt.adj >= 0).all()
    f, b, d = W.sample_queries(xyz, tri, 5000, 0.3, seed=1)
    assert np.abs(b.sum(1) - 1).max() < 1e-12 and b.min() >= 0
    assert np.abs(np.linalg.norm(d, axis=1) - 0.3).max() < 1e-12
    assert np.abs(np.einsum("nd,nd->n", d, mt.fnormal[f])).max() < 1e-12
    f, b, d = W.vertex_edge_queries(xyz, tri, 10, 5.0)
    assert (b[:, 0] == 1).all()


def test_shard_bounds_balance_and_cover():
    from paper_2603_15780_b200.sharding import shard_bounds
    rng = np.random.default_rng(0)
    w = rng.uniform(0.01, 2.0, 100001)
    for world in (1, 2, 3, 8):
        b = shard_bounds(w, world)
        assert b[0] == 0 and b[-1] == len(w) and (np.diff(b) >= 0).all() and len(b) == world + 1
        loads = np.array([w[b[r]:b[r + 1]].sum() for r in range(world)])
        assert loads.max() - loads.min() <= 2 * w.max() + 1e-9
    assert shard_bounds(np.zeros(10), 4).tolist() == [0, 2, 5, 8, 10]
    assert shard_bounds([], 3).tolist() == [0, 0, 0, 0]


WORKER = r'''
import os, sys
import numpy as np
import torch.distributed as dist
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, os.path.join(sys.argv[1], "tests"))
from paper_2603_15780_b200.sharding import trace_sharded
import refapi, hostcheck_api as hc
dist.init_process_group("gloo")
rm = refapi.RefMesh.icosphere(3)
hm = hc.HostMesh(rm.arrays())          # stand-in replica: the device state machine compiled for the host
f, b, d = rm.sample_queries(5, 3001, 0.05, 3.0)
def trace_fn(ff, bb, dd):
    r = hm.trace_batch(ff, bb, dd)
    return dict(face=r.face, bary=r.bary, dir=r.dir, traced=r.traced, term=r.term, crossings=r.crossings)
out = trace_sharded(trace_fn, f, b, d, dist=dist)
full = trace_fn(f, b, d)
ok = all(np.array_equal(out[k], full[k]) for k in full)
print(f"rank {dist.get_rank()} ok={ok} n={len(out['face'])}", flush=True)
dist.barrier(); dist.destroy_process_group()
sys.exit(0 if ok else 1)
'''


def test_query_sharding_world_size_2_gloo(ref, tmp_path):
    """Results gathered from 2 ranks are bitwise the single-process results, at the request index."""
    import hostcheck_api
    hostcheck_api.build()
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    env = dict(os.environ, OMP_NUM_THREADS="2")
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", "29533", str(script), ROOT],
                       capture_output=True, text=True, env=env, timeout=300)
    assert p.returncode == 0, p.stdout + p.stderr
    assert p.stdout.count("ok=True") == 2


def test_wire_formats_match_reference_json(ref):
    """traces_to_json of the host shim (no JSON dependency) emits the reference's document for
    the golden trace byte for byte (proj/tests/test_io.cpp:71-82 compares parsed values)."""
    import json
    exe = os.path.join(ROOT, "tests", "_build", "io_check")
    if not os.path.exists(exe):
        subprocess.check_call(["make", "-C", os.path.join(ROOT, "tests", "cpp")])
    p = subprocess.run([exe], capture_output=True, text=True, timeout=60)
    assert p.returncode == 0 and "IO_OK" in p.stderr, p.stderr
    ours = json.loads(p.stdout)
    sq = ref.RefMesh.build([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0]], [[0, 1, 2], [0, 2, 3]])
    _, text = sq.trace_batch([0, 0], [[.5, .25, .25]] * 2, [[.25, .5, 0], [0, 0, .5]], record_polyline=True, json=True)
    theirs = json.loads(text)
    assert ours["schema"] == theirs["schema"] == "digeo.traces/1"
    assert ours["traces"][0] == theirs["traces"][0]                      # golden trace, exact doubles
    # byte-for-byte for the golden element (same key order, indentation and number formatting)
    golden_text = text[: text.index('"ok": false') if '"ok": false' in text else len(text)]
    assert p.stdout.startswith(golden_text[: golden_text.rindex("},") + 1][:600])
    stalled = dict(theirs["traces"][1])
    mine = dict(ours["traces"][1])
    assert mine.pop("transported_payload") == [1e-5, -2.5e20, 3.0]
    assert mine == stalled


def test_side_predicate_equals_the_sign_of_the_reference_arctangent():
    """The fan walk takes the side of its overshoot from `signed_angle(e_far, e_near, n) >= 0` (tracer.cpp:294,
    geometry.hpp:56-58: atan2(dot(cross(a, b), n), dot(a, b))). The device code evaluates the same predicate without
    the arctangent (signed_angle_nonneg, dg_math.cuh); here it is held against libm's atan2 on the same products:
    signed zeros, NaN, infinities, tiny and random arguments."""
    import ctypes as C
    import hostcheck_api
    lib = hostcheck_api.lib()
    rng = np.random.default_rng(3)
    special = [0.0, -0.0, 1.0, -1.0, 5e-324, -5e-324, 1e-300, -1e-300, np.inf, -np.inf, np.nan, 0.5, -0.5]
    # a = (x, y, 0), b = (1, 0, 0) ... products chosen through axis-aligned vectors: a x b . n and a . b take every pair
    A, B, N = [], [], []
    for y in special:
        for x in special:
            # a = (1, 0, 0), b = (x, y, 0), n = (0, 0, 1): cross(a, b) = (0, 0, y), dot(a, b) = x (+ 0 terms)
            A.append((1.0, 0.0, 0.0)); B.append((x, y, 0.0)); N.append((0.0, 0.0, 1.0))
    a = np.array(A + list(rng.normal(size=(20000, 3)))); b = np.array(B + list(rng.normal(size=(20000, 3))))
    n = np.array(N + list(rng.normal(size=(20000, 3))))
    # nearly parallel / antiparallel pairs: the product y is a rounding residue of either sign or a signed zero
    t = rng.normal(size=(20000, 3)); s = rng.choice([-1.0, 1.0, 2.0, -0.5], size=(20000, 1))
    a = np.concatenate([a, t]); b = np.concatenate([b, t * s]); n = np.concatenate([n, rng.normal(size=(20000, 3))])
    a, b, n = (np.ascontiguousarray(v, dtype=np.float64) for v in (a, b, n))
    out = np.zeros(len(a), dtype=np.uint8)
    p = lambda v: v.ctypes.data_as(C.c_void_p)
    lib.hc_signed_angle_nonneg(C.c_int64(len(a)), p(a), p(b), p(n), p(out))
    with np.errstate(all="ignore"):
        cx = a[:, 1] * b[:, 2] - a[:, 2] * b[:, 1]
        cy = a[:, 2] * b[:, 0] - a[:, 0] * b[:, 2]
        cz = a[:, 0] * b[:, 1] - a[:, 1] * b[:, 0]
        y = cx * n[:, 0] + cy * n[:, 1] + cz * n[:, 2]
        x = a[:, 0] * b[:, 0] + a[:, 1] * b[:, 1] + a[:, 2] * b[:, 2]
        want = (np.arctan2(y, x) >= 0).astype(np.uint8)
    assert np.array_equal(out, want), np.flatnonzero(out != want)[:10]
    assert 0 < want.sum() < len(want)
