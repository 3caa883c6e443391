"""Randomised differential test: fast walker vs the general state machine (walker selector of
dg_trace_cfg), every output bit for bit, over mesh families, extreme mesh scales (the operand-range
guards of the hand-expanded divisions), sliver triangles, lengths over 12 decades and degenerate
starts. usage: python scripts/fuzz_walkers.py [rounds=40] [geodesics=40000] [seed=0]"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_15780_b200 as dg
from paper_2603_15780_b200 import workloads as W

FIELDS = ("face", "bary", "dir", "traced", "requested", "term", "status", "stall", "npoints", "crossings")


def random_mesh(rng):
    kind = rng.integers(0, 4)
    if kind == 0:
        xyz, tri = W.icosphere(int(rng.integers(1, 6)))
    elif kind == 1:
        na = int(rng.integers(6, 120)); xyz, tri = W.torus(1 / 3, float(rng.uniform(0.02, 0.3)), na, max(3, na // int(rng.integers(1, 4))),
                                                         noise=float(rng.choice([0.0, 0.1, 0.4])), seed=int(rng.integers(1 << 30)))
    elif kind == 2:
        xyz, tri = W.bumpy_sphere(int(rng.integers(2, 6)), amplitude=float(rng.uniform(0.0, 0.3)))
    else:  # open planar grid with jitter: boundaries, exact zeros when the jitter is 0
        nx, ny = int(rng.integers(2, 40)), int(rng.integers(2, 40))
        gx, gy = np.meshgrid(np.arange(nx + 1.0), np.arange(ny + 1.0), indexing="ij")
        xyz = np.stack([gx.ravel(), gy.ravel(), np.zeros(gx.size)], 1)
        xyz[:, :2] += rng.choice([0.0, 0.3]) * rng.uniform(-0.5, 0.5, (len(xyz), 2))
        idx = lambda i, j: i * (ny + 1) + j
        tri = np.array([[idx(i, j), idx(i + 1, j), idx(i + 1, j + 1)] for i in range(nx) for j in range(ny)] +
                       [[idx(i, j), idx(i + 1, j + 1), idx(i, j + 1)] for i in range(nx) for j in range(ny)], np.int32)
    if rng.random() < 0.3:   # anisotropic stretch: sliver triangles
        xyz = xyz * np.array([1.0, float(10.0 ** rng.uniform(-3, 0)), 1.0])
    scale = float(10.0 ** rng.choice([0, 0, 0, -3, 4, -60, 70, -118, -125, 98, 104, -160, 160]))
    return np.ascontiguousarray(xyz), np.ascontiguousarray(tri, np.int32), scale


def main(rounds=40, n=40000, seed=0):
    rng = np.random.default_rng(seed)
    bad = 0
    for r in range(rounds):
        unit_xyz, tri, scale = random_mesh(rng)
        xyz = unit_xyz * scale   # queries are sampled on the unscaled mesh (its areas do not overflow) and scaled after
        try:
            meshes = [dg.Mesh(xyz, tri, transport_cache=c) for c in (True, False)]
        except dg.DgError as e:   # degenerate after scaling (area test of Mesh::build): both layouts refuse alike
            print(f"round {r}: mesh rejected ({e.klass})", flush=True)
            continue
        diag = W.bbox_diagonal(unit_xyz)
        f, b, d = W.sample_queries(unit_xyz, tri, n, (1e-9 * diag, 3.0 * diag), seed=int(rng.integers(1 << 30)))
        k = n // 20
        b[:k] = np.eye(3)[rng.integers(0, 3, k)]                       # vertex starts
        b[k:2 * k] = np.array([0.5, 0.5, 0.0])[rng.permuted(np.tile(np.arange(3), (k, 1)), axis=1)]  # edge starts
        e = unit_xyz[tri[f[2 * k:3 * k], 1]] - unit_xyz[tri[f[2 * k:3 * k], 0]]    # exactly along an edge
        d[2 * k:3 * k] = e * (np.linalg.norm(d[2 * k:3 * k], axis=1) / np.linalg.norm(e, axis=1))[:, None]
        d *= scale
        d[3 * k] = 0.0; f[3 * k + 1] = -5; b[3 * k + 2] = [2.0, -0.5, -0.5]; d[3 * k + 3] = [np.nan, 1.0, 0.0]
        max_steps = int(rng.choice([0, 0, 5, 60]))
        ref = None
        for m in meshes:
            slow = m.trace_batch(f, b, d, max_steps=max_steps, walker="generic")
            for walker in (("loads", "tma", "coop") if m.has_transport_cache else ("auto",)):
                fast = m.trace_batch(f, b, d, max_steps=max_steps, walker=walker)
                for key in FIELDS:
                    x, y = getattr(fast, key), getattr(slow, key)
                    same = (x == y) | ((x != x) & (y != y))
                    if not same.all():
                        bad += 1
                        i = np.nonzero(~same.reshape(n, -1).all(1))[0]
                        print(f"round {r} cache={m.has_transport_cache} walker={walker} scale={scale:g}: {key} differs at {i[:5]} ({len(i)} rows)", flush=True)
            # the full-Tracer-backed variant: payload + hole avoidance + polylines in one request
            pay = rng.normal(size=(n, 3)) * scale
            pay[::5] = 0.0
            kw = dict(max_steps=max_steps, payload=pay, hole_avoidance=bool(r % 2), record_polyline=True)
            slow_full = m.trace_batch(f, b, d, walker="generic", **kw)
            for walker in (("loads", "tma", "coop") if m.has_transport_cache else ("auto",)):
                fast_full = m.trace_batch(f, b, d, walker=walker, **kw)
                for key in FIELDS + ("payload", "poly_face", "poly_bary", "poly_seg"):
                    x, y = getattr(fast_full, key), getattr(slow_full, key)
                    if not np.array_equal(x, y, equal_nan=True):
                        bad += 1
                        print(f"round {r} cache={m.has_transport_cache} walker={walker} scale={scale:g}: full-variant {key} differs", flush=True)
            # the polyline-only lane (kPay = 3): the reference's default call -- polylines, no payload --, and hole
            # avoidance without a payload
            kw = dict(max_steps=max_steps, hole_avoidance=bool((r >> 1) % 2), record_polyline=bool(r % 2 == 0) or not (r >> 1) % 2)
            slow_p = m.trace_batch(f, b, d, walker="generic", **kw)
            for walker in (("loads", "tma", "coop") if m.has_transport_cache else ("auto",)):
                fast_p = m.trace_batch(f, b, d, walker=walker, **kw)
                for key in FIELDS + (("poly_face", "poly_bary", "poly_seg") if kw["record_polyline"] else ()):
                    if not np.array_equal(getattr(fast_p, key), getattr(slow_p, key), equal_nan=True):
                        bad += 1
                        print(f"round {r} cache={m.has_transport_cache} walker={walker} scale={scale:g}: polyline-only variant {key} differs", flush=True)
            # the transport-matrix lane (kPay = 2), with and without a payload, with and without polylines
            kw = dict(max_steps=max_steps, want_q=True, hole_avoidance=bool((r >> 1) % 2), record_polyline=bool(r % 3 == 0))
            if r % 2:
                kw["payload"] = pay
            slow_q = m.trace_batch(f, b, d, walker="generic", **kw)
            for walker in (("loads", "tma", "coop") if m.has_transport_cache else ("auto",)):
                fast_q = m.trace_batch(f, b, d, walker=walker, **kw)
                keys = FIELDS + ("q",) + (("payload",) if r % 2 else ()) + (("poly_face", "poly_bary", "poly_seg") if r % 3 == 0 else ())
                for key in keys:
                    if not np.array_equal(getattr(fast_q, key), getattr(slow_q, key), equal_nan=True):
                        bad += 1
                        print(f"round {r} cache={m.has_transport_cache} walker={walker} scale={scale:g}: transport-matrix variant {key} differs", flush=True)
            # the tolerance lane (DG_LANE_FAST) on the non-degenerate part of the batch (random interior starts, random
            # directions): the same walks as the exact lane -- end faces, crossing counts, terminations -- and end points
            # within 1e-9 x diagonal; a knife-edge query may legitimately part ways, so up to 1 in 10 000 is tolerated
            if m.has_transport_cache:
                lane = m.trace_batch(f, b, d, max_steps=max_steps, lane="fast", sort_by_face=False)
                exact = m.trace_batch(f, b, d, max_steps=max_steps, sort_by_face=False)
                sel = np.arange(3 * k + 4, n)
                walk_differs = ((lane.face != exact.face) | (lane.crossings != exact.crossings) | (lane.term != exact.term) |
                                (lane.status != exact.status))[sel]
                same = sel[~walk_differs]
                ok_face = exact.face[same] >= 0
                dpos = np.abs(m.embed(lane.face[same][ok_face], lane.bary[same][ok_face]) -
                              m.embed(exact.face[same][ok_face], exact.bary[same][ok_face])).max() if ok_face.any() else 0.0
                ddir = np.nanmax(np.abs(lane.dir[same] - exact.dir[same])) if len(same) else 0.0
                if walk_differs.sum() > max(1, len(sel) // 10000) or not dpos <= 1e-9 * diag * scale or not ddir <= 1e-9:
                    bad += 1
                    print(f"round {r} scale={scale:g}: tolerance lane: {int(walk_differs.sum())} of {len(sel)} walks differ, "
                          f"max |dpos| / diag {dpos / (diag * scale):.3g}, max |ddir| {ddir:.3g}", flush=True)
            if ref is None:
                ref = fast
            else:
                assert all(np.array_equal(getattr(ref, key), getattr(fast, key), equal_nan=True) for key in ("face", "bary", "dir", "term")), "layouts differ"
        print(f"round {r}: faces {len(tri)} scale {scale:g} max_steps {max_steps} crossings {fast.total_crossings} "
              f"terms {np.bincount(fast.term, minlength=3).tolist()} stalled {int(fast.status.sum())}", flush=True)
    print("FUZZ_OK" if bad == 0 else f"FUZZ_FAILED {bad}")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main(*(int(a) for a in sys.argv[1:4])))
