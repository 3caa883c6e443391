"""Multi-GPU behind the C-ABI (dg_set_devices / dg_set_device_list): one request fanned out over the
devices of the mesh's set, results at the request index, BITWISE independent of the set -- the reference's
determinism contract with devices in the place of workers (tracer.cpp:596-603, acceptance.cpp:173-201).

The lease box has one GPU, so the device set lists GPU 0 two and three times: every device gets its own copy of
the mesh, its own host thread, streams, staging and (device mode) peer copies -- the whole fork/join path runs,
only the copies share one GPU."""
import numpy as np
import pytest

from paper_2603_15780_b200 import workloads as W

pytestmark = pytest.mark.gpu

FIELDS = ("face", "bary", "dir", "traced", "requested", "term", "status", "stall", "npoints", "crossings")


def setup(gpu, copies, n=70_000, seed=3):
    xyz, tri = W.icosphere(4)
    one = gpu.Mesh(xyz, tri, device=0)
    many = gpu.Mesh(xyz, tri, devices=[0] * copies)
    assert one.device_count == 1 and many.device_count == copies
    f, b, d = W.sample_queries(xyz, tri, n, (0.01, 2.0), seed=seed)   # mixed lengths: shards of unequal counts
    return one, many, f, b, d


@pytest.mark.parametrize("copies", [2, 3])
def test_host_mode_trace_is_independent_of_the_device_set(gpu, copies):
    one, many, f, b, d = setup(gpu, copies)
    a, c = one.trace_batch(f, b, d), many.trace_batch(f, b, d)
    for k in FIELDS:
        assert np.array_equal(getattr(a, k), getattr(c, k)), k
    assert a.total_crossings == c.total_crossings
    # payload + transport matrix + hole avoidance + polylines (the full walker, the staged path)
    pay = np.random.default_rng(1).normal(size=(len(f), 3))
    kw = dict(payload=pay, want_q=True, hole_avoidance=True, record_polyline=True)
    a, c = one.trace_batch(f, b, d, **kw), many.trace_batch(f, b, d, **kw)
    for k in FIELDS + ("payload", "q", "poly_offsets", "poly_face", "poly_bary", "poly_seg"):
        assert np.array_equal(getattr(a, k), getattr(c, k)), k
    # a request below the fan-out size stays on the primary device and still agrees
    a, c = one.trace_batch(f[:5000], b[:5000], d[:5000]), many.trace_batch(f[:5000], b[:5000], d[:5000])
    assert np.array_equal(a.bary, c.bary)


def test_rejected_starts_keep_their_request_index_across_shards(gpu):
    one, many, f, b, d = setup(gpu, 2)
    f = f.copy()
    bad = np.array([5, 30_000, 69_999])
    f[bad] = -1
    a, c = one.trace_batch(f, b, d), many.trace_batch(f, b, d)
    assert np.array_equal(a.stall, c.stall) and list(np.nonzero(c.status)[0]) == list(bad)
    assert [i for i, _ in c.errors] == list(bad)


@pytest.mark.parametrize("copies", [2, 3])
def test_differentials_are_independent_of_the_device_set(gpu, copies):
    one, many, f, b, d = setup(gpu, copies)
    fwd = one.trace_batch(f, b, d)
    g = np.random.default_rng(2).normal(size=(len(f), 3))
    a, c = one.ep(f, b, d, fwd.face, fwd.bary, fwd.dir, g=g), many.ep(f, b, d, fwd.face, fwd.bary, fwd.dir, g=g)
    for k in ("rot", "frames", "grad_v", "grad_p"):
        assert np.array_equal(a[k], c[k]), k
    a, c = one.gfd(f, b, d, g=g), many.gfd(f, b, d, g=g)
    for k in ("jv", "jp", "degraded", "frames", "grad_v", "grad_p", "base_face", "base_bary", "base_dir"):
        assert np.array_equal(a[k], c[k]), k
    out = lambda: dict(jv=np.zeros((len(f), 4)), jp=np.zeros((len(f), 4)), degraded=np.zeros((len(f), 4), np.uint8),
                       grad_v=np.zeros((len(f), 3)), grad_p=np.zeros((len(f), 3)))
    kb = many.gfd(f, b, d, g=g, base=fwd, out=out())
    for k in ("jv", "jp", "degraded", "grad_v", "grad_p"):
        assert np.array_equal(a[k], kb[k]), k
    # whole-call errors carry the REQUEST index of the first offending sample, whichever shard it fell into
    d2 = d.copy()
    d2[60_000] = 0
    for m in (one, many):
        with pytest.raises(gpu.DgError) as e:
            m.ep(f, b, d2, fwd.face, fwd.bary, fwd.dir)
        assert e.value.klass == "DegenerateDirection" and e.value.index == 60_000
        with pytest.raises(gpu.DgError) as e:
            m.gfd(f, b, d2, g=g)
        assert e.value.klass == "DegenerateDirection" and e.value.index == 60_000


def test_resident_batch_on_a_device_set(gpu):
    one, many, f, b, d = setup(gpu, 2)
    g = np.random.default_rng(4).normal(size=(len(f), 3))
    ba, bc = gpu.Batch(one, len(f)), gpu.Batch(many, len(f))
    ra, rc = ba.trace(f, b, d), bc.trace(f, b, d)
    for k in FIELDS:
        assert np.array_equal(getattr(ra, k), getattr(rc, k)), k
    assert ra.total_crossings == rc.total_crossings
    assert np.array_equal(ba.ep_backward(g), bc.ep_backward(g))
    ga, gc = ba.gfd(g=g), bc.gfd(g=g)
    for k in ("jv", "jp", "degraded", "grad_v", "grad_p"):
        assert np.array_equal(ga[k], gc[k]), k
    ba.close(); bc.close()


def test_streamed_forward_on_a_device_set(gpu):
    """Shards of >= 2^18 queries each run the STREAMED forward (one persistent walker per device, upload cursor and
    completion flags of its own): two of them side by side -- here on one GPU -- give the bits of one device."""
    one, many, f, b, d = setup(gpu, 2, n=2 * (1 << 18) + 70_001)
    ba, bc = gpu.Batch(one, len(f)), gpu.Batch(many, len(f))
    ra, rc = ba.trace(f, b, d), bc.trace(f, b, d)
    for k in FIELDS:
        assert np.array_equal(getattr(ra, k), getattr(rc, k)), k
    assert ra.total_crossings == rc.total_crossings == int(ra.crossings.sum())
    g = np.random.default_rng(4).normal(size=(len(f), 3))
    assert np.array_equal(ba.ep_backward(g), bc.ep_backward(g))
    ba.close(); bc.close()


def test_device_mode_fans_out_through_peer_copies(gpu):
    import torch
    one, many, f, b, d = setup(gpu, 3, n=90_000)
    dev = torch.device("cuda", 0)
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dtype=dt)
    F, B, D = t(f, torch.int32), t(b, torch.float64), t(d, torch.float64)
    n = len(f)

    def outs():
        return dict(face=torch.empty(n, dtype=torch.int32, device=dev), bary=torch.empty(n, 3, dtype=torch.float64, device=dev),
                    dir=torch.empty(n, 3, dtype=torch.float64, device=dev), traced=torch.empty(n, dtype=torch.float64, device=dev),
                    term=torch.empty(n, dtype=torch.uint8, device=dev), status=torch.empty(n, dtype=torch.uint8, device=dev),
                    crossings=torch.empty(n, dtype=torch.int32, device=dev), total_crossings=torch.zeros(1, dtype=torch.int64, device=dev))
    oa, oc = outs(), outs()
    one.trace_batch_device(F, B, D, oa)
    many.trace_batch_device(F, B, D, oc)
    torch.cuda.synchronize()
    for k in oa:
        assert torch.equal(oa[k], oc[k]), k
    G = t(np.random.default_rng(5).normal(size=(n, 3)), torch.float64)
    ga, gc = torch.empty(n, 3, dtype=torch.float64, device=dev), torch.empty(n, 3, dtype=torch.float64, device=dev)
    one.ep_backward_device(F, D, oa["face"], oa["dir"], G, ga)
    many.ep_backward_device(F, D, oc["face"], oc["dir"], G, gc)
    assert torch.equal(ga, gc)
    eps = one.default_gfd_eps()
    ja, jc = [torch.empty(n, 4, dtype=torch.float64, device=dev) for _ in range(2)], [torch.empty(n, 4, dtype=torch.float64, device=dev) for _ in range(2)]
    va, vc = torch.empty(n, 3, dtype=torch.float64, device=dev), torch.empty(n, 3, dtype=torch.float64, device=dev)
    one.gfd_device(F, B, D, eps, eps, G, ja[0], ja[1], va, base=oa)
    many.gfd_device(F, B, D, eps, eps, G, jc[0], jc[1], vc, base=oc)
    torch.cuda.synchronize()
    assert torch.equal(ja[0], jc[0]) and torch.equal(ja[1], jc[1]) and torch.equal(va, vc)
