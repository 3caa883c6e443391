"""Generates tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref/libdigeo_ref.so, built
from /root/reference by oracle/Makefile). Run in the build container:  python tests/golden/make_golden.py
The fixtures travel to the GPU box, where /root/reference does not exist."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import refapi  # noqa: E402


def trace_fields(r):
    return dict(o_face=r.face, o_bary=r.bary, o_dir=r.dir, o_traced=r.traced, o_requested=r.requested,
                o_term=r.term, o_status=r.status, o_npoints=r.npoints, o_payload=r.payload,
                o_q=r.q if r.q is not None else np.zeros((len(r.face), 9)), poly_face=r.poly_face,
                poly_bary=r.poly_bary, poly_seg=r.poly_seg)


def save(name, rm, f, b, d, payload=None, **kw):
    a = rm.arrays()
    r = rm.trace_batch(f, b, d, payload=payload, record_polyline=True, **kw)
    cfg = dict(max_steps=0, hole_avoidance=False, want_q=False)
    cfg.update(kw)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), xyz=a["xyz"], tri=a["tri"], adj=a["adj"],
                        vangle=a["vangle"], mean_edge=a["mean_edge"], face=f, bary=b, dir=d,
                        payload=payload if payload is not None else np.zeros((0, 3)),
                        cfg=np.array([cfg["max_steps"], int(cfg["hole_avoidance"]), int(cfg["want_q"])]),
                        **trace_fields(r))
    return r


def main():
    rng = np.random.default_rng(2026)
    # 1. the reference's own golden case + the Appendix-B square cases
    sq = refapi.RefMesh.build([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0]], [[0, 1, 2], [0, 2, 3]])
    F = np.array([0, 0, 0, 0, 0, 0, 7, 0, 0, -1], np.int32)
    B = np.array([[.5, .25, .25], [.5, 0, .5], [1, 0, 0], [.5, .25, .25], [.5, .25, .25], [.5, .25, .25],
                  [.3, .3, .4], [.5, .25, .25], [.5, .5, .5], [1, 0, 0]])
    D = np.array([[.25, .5, 0], [-.2, .1, 0], [.1, .3, 0], [2, .1, 0], [0, 0, .5], [0, 0, 0], [1, 0, 0],
                  [0, 0, 0], [1, 0, 0], [1, 0, 0]], float)
    save("square_cases", sq, F, B, D)
    save("square_cases_hole", sq, F, B, D, hole_avoidance=True)
    # 2. config 1 (ico-4, unit tangents), a 600-query prefix with payload + Q
    ico = refapi.RefMesh.icosphere(4)
    f, b, d = ico.sample_queries(42, 600, 1.0, 1.0)
    save("ico4_config1", ico, f, b, d, payload=rng.normal(size=(600, 3)), want_q=True)
    # 3. torus vertex-to-vertex walks (config-5 style) and random departures from vertices
    tor = refapi.RefMesh.torus(1 / 3, 1 / 6, 32, 16)
    a = tor.arrays()
    X, T = a["xyz"], a["tri"]
    n = 300
    fs = rng.integers(0, tor.nf, n).astype(np.int32)
    c = rng.integers(0, 3, n)
    bs = np.zeros((n, 3))
    bs[np.arange(n), c] = 1
    ds = X[T[fs, (c + 1) % 3]] - X[T[fs, c]]
    ds = ds / np.linalg.norm(ds, axis=1, keepdims=True) * rng.uniform(0.2, 1.5, (n, 1))
    ds[n // 2:] = rng.normal(size=(n - n // 2, 3))
    save("torus_vertex_walks", tor, fs, bs, ds, payload=rng.normal(size=(n, 3)), want_q=True, max_steps=5000)
    # 4. open meshes: boundary stop and hole avoidance
    pl = refapi.RefMesh.plane(7, 5, 1.0, 3)
    f, b, d = pl.sample_queries(5, 400, 0.05, 2.0)
    save("plane_boundary", pl, f, b, d)
    save("plane_hole_avoidance", pl, f, b, d, payload=rng.normal(size=(400, 3)), hole_avoidance=True, want_q=True)
    # 5. cone apex crossings
    co = refapi.RefMesh.cone(1.0, 1.0, 12)
    ac = co.arrays()
    apex = int(np.argmax(np.diff(ac["csr_off"])))
    f, b, d = co.sample_queries(12, 300, 1.0, 1.0)
    P = co.embed(f, b)
    d = ac["xyz"][apex] - P
    d = d / np.linalg.norm(d, axis=1, keepdims=True) * 1.7
    save("cone_apex", co, f, b, d, payload=rng.normal(size=(300, 3)), want_q=True)
    # 6. differentials on ico-3: EP (bit-exact) and GFD
    i3 = refapi.RefMesh.icosphere(3)
    f, b, d = i3.sample_queries(9, 300, 0.2, 1.0)
    r = i3.trace_batch(f, b, d)
    g = rng.normal(size=(300, 3))
    ep = i3.ep(f, b, d, r.face, r.bary, r.dir, g=g)
    gfd = i3.gfd(f, b, d, g=g)
    a3 = i3.arrays()
    np.savez_compressed(os.path.join(HERE, "ico3_diff.npz"), xyz=a3["xyz"], tri=a3["tri"], face=f, bary=b, dir=d, g=g,
                        end_face=r.face, end_bary=r.bary, end_dir=r.dir, ep_rot=ep["rot"], ep_frames=ep["frames"],
                        ep_grad_v=ep["grad_v"], gfd_jv=gfd["jv"], gfd_jp=gfd["jp"], gfd_degraded=gfd["degraded"],
                        gfd_frames=gfd["frames"], gfd_grad_v=gfd["grad_v"], gfd_grad_p=gfd["grad_p"],
                        eps=i3.default_gfd_eps())
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
