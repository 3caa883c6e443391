"""Resident batch (dg_batch_*): forward + EP / GFD backward on device-resident samples.
Bar: the same bits as the separate host-mode calls (it runs their device-mode paths), and parity
with the UNMODIFIED reference on the forward results and the EP gradient; every slice count of
the copy/compute pipeline gives the same bits."""
import os

import numpy as np
import pytest

from conftest import assert_trace_equal, gpu_mesh

pytestmark = pytest.mark.gpu


def unit_rows(rng, n):
    q = rng.normal(size=(n, 3))
    return q / np.linalg.norm(q, axis=1, keepdims=True)


@pytest.mark.parametrize("slices", ["1", "2", "4"])
def test_batch_forward_ep_matches_reference_and_separate_calls(gpu, ref, slices, monkeypatch):
    monkeypatch.setenv("DG_BATCH_SLICES", slices)
    rm = ref.RefMesh.icosphere(4)
    m = gpu_mesh(gpu, rm)
    n = 20011
    f, b, d = rm.sample_queries(7, n, 0.2, 1.5)
    batch = gpu.Batch(m, n + 5)
    h = batch.trace(f, b, d)
    r = rm.trace_batch(f, b, d, record_polyline=True)  # the reference counts points only when it records them
    assert_trace_equal(r, h, n, check_poly=False)
    h2 = m.trace_batch(f, b, d)
    for k in ("face", "bary", "dir", "traced", "requested", "term", "status", "stall", "npoints", "crossings"):
        assert np.array_equal(getattr(h, k), getattr(h2, k)), k
    assert h.total_crossings == h2.total_crossings == int(h2.crossings.sum())
    g = 2.0 * (m.embed(h.face, h.bary) - unit_rows(np.random.default_rng(1), n))  # gradcheck.cpp:88
    gp = np.full((n, 3), np.nan)
    gv = batch.ep_backward(g, grad_p=gp)
    theirs = rm.ep(f, b, d, h.face, h.bary, h.dir, g=g)
    assert np.array_equal(gv, theirs["grad_v"]) and not gp.any()
    assert np.array_equal(gv, m.ep_backward(f, d, h.face, h.dir, g))


def test_batch_gfd_matches_separate_call(gpu, ref):
    rm = ref.RefMesh.torus(1 / 3, 1 / 6, 64, 32)
    m = gpu_mesh(gpu, rm)
    n = 3000
    f, b, d = rm.sample_queries(11, n, 0.05, 0.4)
    batch = gpu.Batch(m, n)
    h = batch.trace(f, b, d)
    g = unit_rows(np.random.default_rng(2), n)
    ours = batch.gfd(g=g)
    sep = m.gfd(f, b, d, g=g)
    for k in ("jv", "jp", "degraded", "grad_v", "grad_p"):
        assert np.array_equal(ours[k], sep[k]), k
    theirs = rm.gfd(f, b, d, g=g)
    scale = np.abs(theirs["jv"]).max()
    assert np.abs(ours["jv"] - theirs["jv"]).max() <= 1e-5 * scale  # SURVEY.md 8c tolerance


def test_batch_gfd_takes_over_the_forward_traces(gpu, ref, monkeypatch):
    """The resident GFD reuses the forward results as its base traces: same bits as a re-trace,
    same whole-call failure when a base trace leaves the mesh (diff.cpp:121-124)."""
    rm = ref.RefMesh.icosphere(4)
    m = gpu_mesh(gpu, rm)
    n = 2500
    f, b, d = rm.sample_queries(5, n, 0.1, 1.0)
    g = unit_rows(np.random.default_rng(4), n)
    batch = gpu.Batch(m, n)
    batch.trace(f, b, d)
    reused = batch.gfd(g=g)
    monkeypatch.setenv("DG_BATCH_GFD_RETRACE", "1")
    retraced = batch.gfd(g=g)
    monkeypatch.delenv("DG_BATCH_GFD_RETRACE")
    for k in ("jv", "jp", "degraded", "grad_v", "grad_p"):
        assert np.array_equal(reused[k], retraced[k]), k
    h = m.trace_batch(f, b, d)
    given = m.gfd(f, b, d, g=g, base=h)  # dg_gfd_jacobians_with_base: gfd_batched's `trace` argument
    for k in ("jv", "jp", "degraded", "grad_v", "grad_p", "frames"):
        assert np.array_equal(given[k], m.gfd(f, b, d, g=g)[k]), k
    batch.trace(f, b, d, max_steps=7)  # a different step limit: the forward traces are not GFD's base traces
    limited = batch.gfd(g=g)
    assert np.array_equal(limited["jv"], reused["jv"])
    pl = ref.RefMesh.plane(6, 6, 1.0, 0)
    mp = gpu_mesh(gpu, pl)
    fp, bp, dp = pl.sample_queries(2, 64, 0.01, 0.05)
    dp[17] *= 1e3  # leaves through the boundary
    bt = gpu.Batch(mp, 64)
    h = bt.trace(fp, bp, dp)
    assert h.term[17] == 1
    with pytest.raises(gpu.DgError) as e:
        bt.gfd()
    assert "base trace did not reach" in e.value.msg and e.value.index == 17


def test_batch_contract_errors(gpu, ref):
    rm = ref.RefMesh.icosphere(2)
    m = gpu_mesh(gpu, rm)
    batch = gpu.Batch(m, 16)
    with pytest.raises(gpu.DgError) as e:
        batch.ep_backward(np.zeros((4, 3)))
    assert e.value.klass == "InvalidArgs"
    f, b, d = rm.sample_queries(3, 32, 1.0, 1.0)
    with pytest.raises(gpu.DgError) as e:
        batch.trace(f, b, d)  # exceeds the capacity
    assert e.value.klass == "InvalidArgs"
    h = batch.trace(f[:16], b[:16], d[:16])
    d0 = d[:16].copy()
    d0[5] = 0.0
    h = batch.trace(f[:16], b[:16], d0)  # zero-length request: a valid trace, a degenerate EP direction
    assert h.traced[5] == 0.0
    with pytest.raises(gpu.DgError) as e:
        batch.ep_backward(np.ones((16, 3)))
    assert e.value.klass == "DegenerateDirection" and e.value.index == 5


def test_resident_batch_in_the_tolerance_lane(gpu, ref):
    """dg_trace_cfg.lane = DG_LANE_FAST through the resident batch: forward (plain and as the forward of a GFD step) and
    the pull-back agree with the exact lane's within the lane's bar -- same end faces, 1e-9 x diagonal, GFD gradients
    cos >= 0.999999 -- and with the lane's own device-mode calls bit for bit."""
    rm = ref.RefMesh.torus(1 / 3, 1 / 6, 64, 32)
    a = rm.arrays()
    m = gpu.Mesh(a["xyz"], a["tri"])
    f, b, d = rm.sample_queries(17, 70000, 0.05, 0.9)
    g = np.random.default_rng(1).normal(size=(len(f), 3))
    bt = gpu.Batch(m, len(f))
    exact = bt.trace(f, b, d)
    fast = bt.trace(f, b, d, lane="fast")
    direct = m.trace_batch(f, b, d, lane="fast")
    assert np.array_equal(fast.bary, direct.bary) and np.array_equal(fast.dir, direct.dir)
    assert np.array_equal(fast.face, exact.face) and not np.array_equal(fast.bary, exact.bary)
    diag = np.linalg.norm(a["xyz"].max(0) - a["xyz"].min(0))
    assert np.abs(m.embed(fast.face, fast.bary) - m.embed(exact.face, exact.bary)).max() <= 1e-9 * diag
    fused = bt.trace(f, b, d, gfd=True, lane="fast")
    assert np.array_equal(fused.bary, fast.bary)
    out = bt.gfd(g=g)
    sep = m.gfd(f, b, d, g=g)
    for k in ("grad_v", "grad_p"):
        num = np.einsum("nd,nd->n", out[k], sep[k])
        den = np.linalg.norm(out[k], axis=1) * np.linalg.norm(sep[k], axis=1)
        ok = den > 1e-12
        assert (num[ok] / den[ok]).min() >= 0.999999, k
    assert np.abs(out["jv"] - sep["jv"]).max() <= 1e-5 * np.abs(sep["jv"]).max()
    bt.close()


def test_streamed_forward_gives_the_bits_of_the_sliced_pipeline(gpu, ref, monkeypatch):
    """>= 2^18 queries in plain order run as ONE walker while the queries arrive and the results leave (upload cursor,
    per-chunk completion flags). Same bits as the sliced pipeline and the reference; covers a ragged last chunk,
    rejected starts, zero-length requests and vertex starts (every way a trace can end), then EP on the resident batch."""
    rm = ref.RefMesh.icosphere(5)
    m = gpu_mesh(gpu, rm)
    n = 4 * 65536 + 40017
    f, b, d = rm.sample_queries(3, n, 0.01, 1.2)
    f[5] = -1; f[70000] = rm.nf + 3          # rejected starts
    d[9] = 0.0; d[131072] = 0.0              # zero-length requests
    b[11] = [1.0, 0.0, 0.0]; b[200001] = [0.0, 1.0, 0.0]   # vertex starts
    b[13] = [0.7, 0.7, -0.4]                 # rejected barycentrics
    batch = gpu.Batch(m, n)
    for rep in range(2):                     # twice: the counters and flags of the batch are reused
        h = batch.trace(f, b, d)
    monkeypatch.setenv("DG_BATCH_SLICES", "4")
    s = batch.trace(f, b, d)
    monkeypatch.delenv("DG_BATCH_SLICES")
    for k in ("face", "bary", "dir", "traced", "requested", "term", "status", "stall", "npoints", "crossings"):
        assert np.array_equal(getattr(h, k), getattr(s, k)), k
    assert h.total_crossings == s.total_crossings == int(h.crossings.sum())
    k = 30000
    sel = np.r_[100:k, n - k:n]              # (clear of the doctored entries: the reference leaves rejected slots unset,
                                             # and a vertex start goes through atan2, CUDA's against glibc's)
    r = rm.trace_batch(f[sel], b[sel], d[sel], record_polyline=True)
    for name in ("face", "bary", "dir", "traced", "term", "status"):
        assert np.array_equal(getattr(r, name), getattr(h, name)[sel]), name
    # EP on a streamed resident batch (clean samples: EP rejects a zero direction for the whole call)
    f2, b2, d2 = f[100:], b[100:].copy(), d[100:].copy()
    bad = (np.abs(d2).sum(1) == 0) | (f2 < 0) | (f2 >= rm.nf)
    f2, b2, d2 = f2[~bad], b2[~bad], d2[~bad]
    h2 = batch.trace(f2, b2, d2)
    g = unit_rows(np.random.default_rng(1), len(f2))
    gv = batch.ep_backward(g)
    sep = m.ep_backward(f2[:5000], d2[:5000], h2.face[:5000], h2.dir[:5000], g[:5000])
    assert np.array_equal(gv[:5000], sep)
    # a request of exactly 2^18 queries: whole chunks, whole pieces, the smallest streamed call
    m18 = 1 << 18
    e = batch.trace(f2[:m18], b2[:m18], d2[:m18])
    for k in ("face", "bary", "dir", "traced", "crossings"):
        assert np.array_equal(getattr(e, k), getattr(h2, k)[:m18]), k
    assert e.total_crossings == int(h2.crossings[:m18].sum())
    # EP on the streamed batch reports a degenerate direction with its request index (diff.cpp:46)
    d3 = d2.copy()
    d3[200_000] = 0.0
    batch.trace(f2, b2, d3)
    with pytest.raises(gpu.DgError) as err:
        batch.ep_backward(g)
    assert err.value.klass == "DegenerateDirection" and err.value.index == 200_000
    # the host-mode dg_trace_batch of a large plain request runs on the same pipeline
    t = m.trace_batch(f, b, d)
    assert np.array_equal(t.bary, h.bary) and np.array_equal(t.face, h.face)
