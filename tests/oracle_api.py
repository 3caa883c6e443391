"""ctypes binding of oracle/liboracle.so, the plain-C restatement of the reference algorithm.
TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from refapi import TraceResult, _f64, _i32, _p

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "oracle", "liboracle.so")
ERR = {1: "InvalidArgs", 3: "ParseError", 4: "NonManifoldError", 5: "DegenerateFaceError",
       6: "DegenerateDirection", 7: "Error", 10: "NumericalStall"}
STALL = {1: "degenerate direction in face", 2: "no positive exit parameter",
         3: "initial direction is normal to the anchor face", 4: "trace: start face out of range",
         5: "trace: start barycentric coordinates not in the simplex"}


class OracleError(RuntimeError):
    def __init__(self, klass, msg):
        super().__init__(f"{klass}: {msg}")
        self.klass, self.msg, self.index = klass, msg, -1


class Cfg(C.Structure):
    _fields_ = [("max_steps", C.c_int), ("hole_avoidance", C.c_int), ("want_q", C.c_int), ("threads", C.c_int)]


_lib = None


def available():
    return os.path.exists(SO)


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(SO)
        _lib.og_mesh_build.restype = C.c_void_p
        _lib.og_mesh_mean_edge.restype = C.c_double
        _lib.og_mesh_mean_edge.argtypes = [C.c_void_p]
        _lib.og_mesh_free.argtypes = [C.c_void_p]
        _lib.og_mesh_get.argtypes = [C.c_void_p] * 9
        _lib.og_trace_batch.argtypes = [C.c_void_p, C.c_int64] + [C.c_void_p] * 20
        _lib.og_ep.argtypes = [C.c_void_p, C.c_int64] + [C.c_void_p] * 10
        _lib.og_gfd.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_double] + \
                               [C.c_void_p] * 7 + [C.c_int, C.c_void_p, C.c_int]
    return _lib


class OracleMesh:
    def __init__(self, xyz, tri):
        self.xyz = _f64(xyz).reshape(-1, 3)
        self.tri = _i32(tri).reshape(-1, 3)
        self.nv, self.nf = len(self.xyz), len(self.tri)
        ec = C.c_int(0)
        buf = C.create_string_buffer(256)
        h = lib().og_mesh_build(_p(self.xyz), self.nv, _p(self.tri), self.nf, C.byref(ec), buf, 256)
        if not h:
            raise OracleError(ERR.get(ec.value, "?"), buf.value.decode())
        self.h = C.c_void_p(h)
        self.mean_edge = lib().og_mesh_mean_edge(self.h)

    def __del__(self):
        try:
            lib().og_mesh_free(self.h)
        except Exception:
            pass

    def arrays(self):
        nv, nf = self.nv, self.nf
        d = dict(adj=np.empty((nf, 3), np.int32), fnormal=np.empty((nf, 3)), farea=np.empty(nf), vangle=np.empty(nv),
                 varea=np.empty(nv), vboundary=np.empty(nv, np.uint8), csr_off=np.empty(nv + 1, np.int32),
                 csr_list=np.empty(3 * nf, np.int32))
        lib().og_mesh_get(self.h, *[_p(d[k]) for k in ("adj", "fnormal", "farea", "vangle", "varea", "vboundary",
                                                      "csr_off", "csr_list")])
        d["xyz"], d["tri"], d["mean_edge"] = self.xyz, self.tri, self.mean_edge
        return d

    def embed(self, face, bary):
        return np.einsum("nk,nkd->nd", bary, self.xyz[self.tri[face]])

    def default_gfd_eps(self):
        return 1e-4 * self.mean_edge

    def trace_batch(self, face, bary, dirs, payload=None, max_steps=0, hole_avoidance=False, want_q=False,
                    record_polyline=False, threads=0):
        face, bary, dirs, payload = _i32(face), _f64(bary), _f64(dirs), _f64(payload)
        n = len(face)
        r = TraceResult(face=np.empty(n, np.int32), bary=np.empty((n, 3)), dir=np.empty((n, 3)), traced=np.empty(n),
                        requested=np.empty(n), term=np.empty(n, np.uint8), status=np.empty(n, np.uint8),
                        payload=np.empty((n, 3)), q=np.empty((n, 9)), npoints=np.empty(n, np.int32))
        r.stall = np.empty(n, np.uint8)
        cfg = Cfg(int(max_steps), int(hole_avoidance), int(want_q), int(threads))

        def call(off, pf, pb, ps):
            lib().og_trace_batch(self.h, n, _p(face), _p(bary), _p(dirs), _p(payload), C.addressof(cfg), _p(r.face),
                                 _p(r.bary), _p(r.dir), _p(r.traced), _p(r.requested), _p(r.term), _p(r.status),
                                 _p(r.stall), _p(r.payload), _p(r.q), _p(r.npoints), _p(off), _p(pf), _p(pb), _p(ps))
        call(None, None, None, None)
        if record_polyline:
            off = np.zeros(n + 1, np.int64)
            np.cumsum(r.npoints, out=off[1:])
            tot = int(off[-1])
            r.poly_offsets, r.poly_face = off, np.empty(tot, np.int32)
            r.poly_bary, r.poly_seg = np.empty((tot, 3)), np.empty(tot)
            call(off, r.poly_face, r.poly_bary, r.poly_seg)
        if payload is not None:
            r.has_payload = (np.square(payload.reshape(n, 3)).sum(1) > 0).astype(np.uint8)
        r.errors = [(int(i), STALL[int(r.stall[i])]) for i in np.nonzero(r.status)[0]]
        return r

    def ep(self, face, bary, v, end_face, end_bary, end_dir, g=None):
        n = len(face)
        out = dict(rot=np.empty((n, 9)), frames=np.empty((n, 33)), grad_v=np.zeros((n, 3)), grad_p=np.zeros((n, 3)))
        ei = C.c_int64(-1)
        rc = lib().og_ep(self.h, n, _p(_i32(face)), _p(_f64(v)), _p(_i32(end_face)), _p(_f64(end_dir)), _p(_f64(g)),
                         _p(out["rot"]), _p(out["frames"]), _p(out["grad_v"]), _p(out["grad_p"]), C.addressof(ei))
        if rc:
            e = OracleError(ERR.get(rc, "?"), "degenerate direction")
            e.index = ei.value
            raise e
        return out

    def gfd(self, face, bary, v, eps_v=None, eps_p=None, g=None, threads=0):
        n = len(face)
        eps = self.default_gfd_eps()
        eps_v = eps if eps_v is None else eps_v
        eps_p = eps if eps_p is None else eps_p
        out = dict(jv=np.zeros((n, 4)), jp=np.zeros((n, 4)), degraded=np.zeros((n, 4), np.uint8),
                   frames=np.zeros((n, 33)), grad_v=np.zeros((n, 3)), grad_p=np.zeros((n, 3)))
        buf = C.create_string_buffer(256)
        rc = lib().og_gfd(self.h, n, _p(_i32(face)), _p(_f64(bary)), _p(_f64(v)), float(eps_v), float(eps_p),
                          _p(_f64(g)), _p(out["jv"]), _p(out["jp"]), _p(out["degraded"]), _p(out["frames"]),
                          _p(out["grad_v"]), _p(out["grad_p"]), int(threads), buf, 256)
        if rc:
            raise OracleError(ERR.get(rc, "?"), buf.value.decode())
        return out


def check_trace(xyz, tri, f, b, d, h):
    """smoke()'s checker when oracle/_ref is absent: bit parity of a product result with the C oracle."""
    o = OracleMesh(xyz, tri).trace_batch(f, b, d, record_polyline=True)
    assert np.array_equal(o.face, h.face) and np.array_equal(o.bary, h.bary) and np.array_equal(o.dir, h.dir)
    assert np.array_equal(o.poly_face, h.poly_face)
