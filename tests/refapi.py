"""ctypes binding of oracle/_ref/libdigeo_ref.so -- the UNMODIFIED reference behind
oracle/ref_shim.cpp. TEST INFRASTRUCTURE: imported by tests/ and by bench.py's
cpu_baseline / --impl reference legs only, never by the product package."""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libdigeo_ref.so")

ERR_CLASS = {0: None, 1: "InvalidArgs", 3: "ParseError", 4: "NonManifoldError",
             5: "DegenerateFaceError", 6: "DegenerateDirection", 7: "Error",
             10: "NumericalStall", 11: "BoundaryHit", 99: "std::exception"}


class RefError(RuntimeError):
    def __init__(self, klass, msg):
        super().__init__(f"{klass}: {msg}")
        self.klass = klass
        self.msg = msg


def available() -> bool:
    return os.path.exists(REF_SO)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"{REF_SO} missing: run `make -C oracle ref` where /root/reference exists")
        _lib = C.CDLL(REF_SO, mode=os.RTLD_LOCAL)
        vp = C.c_void_p
        for name in ("ref_mesh_build", "ref_mesh_load_obj", "ref_concat_meshes", "ref_make_icosphere",
                     "ref_make_torus", "ref_make_plane", "ref_make_cylinder", "ref_make_cone",
                     "ref_trace_batch", "ref_trace_single"):
            getattr(_lib, name).restype = vp
        _lib.ref_mesh_mean_edge.restype = C.c_double
        _lib.ref_mesh_total_area.restype = C.c_double
        _lib.ref_default_gfd_eps.restype = C.c_double
        _lib.ref_result_size.restype = C.c_int64
        _lib.ref_traces_json.restype = C.c_char_p
        _lib.ref_last_error.restype = C.c_char_p
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.int32)


@dataclass
class TraceResult:
    face: np.ndarray
    bary: np.ndarray
    dir: np.ndarray
    traced: np.ndarray
    requested: np.ndarray
    term: np.ndarray       # 0 LengthReached, 1 Boundary, 2 MaxSteps
    status: np.ndarray     # 0 Ok, 1 Stalled
    payload: np.ndarray | None = None
    has_payload: np.ndarray | None = None
    q: np.ndarray | None = None
    npoints: np.ndarray | None = None
    errors: list = field(default_factory=list)
    poly_offsets: np.ndarray | None = None
    poly_face: np.ndarray | None = None
    poly_bary: np.ndarray | None = None
    poly_seg: np.ndarray | None = None
    crossings: np.ndarray | None = None
    stall: np.ndarray | None = None


class RefMesh:
    def __init__(self, handle):
        if not handle:
            raise RuntimeError("null reference mesh handle")
        self.h = C.c_void_p(handle)
        L = lib()
        self.nv = L.ref_mesh_nv(self.h)
        self.nf = L.ref_mesh_nf(self.h)
        self._arrays = None

    def __del__(self):
        try:
            lib().ref_mesh_free(self.h)
        except Exception:
            pass

    # ---- constructors
    @staticmethod
    def build(xyz, tri):
        xyz = _f64(xyz).reshape(-1, 3)
        tri = _i32(tri).reshape(-1, 3)
        ec = C.c_int(0)
        buf = C.create_string_buffer(512)
        h = lib().ref_mesh_build(_p(xyz), len(xyz), _p(tri), len(tri), C.byref(ec), buf, 512)
        if not h:
            raise RefError(ERR_CLASS.get(ec.value, "?"), buf.value.decode())
        return RefMesh(h)

    @staticmethod
    def icosphere(subdiv):
        return RefMesh(lib().ref_make_icosphere(int(subdiv)))

    @staticmethod
    def torus(R, r, na, nb):
        return RefMesh(lib().ref_make_torus(C.c_double(R), C.c_double(r), int(na), int(nb)))

    @staticmethod
    def plane(nx, ny, size=1.0, seed=0):
        return RefMesh(lib().ref_make_plane(int(nx), int(ny), C.c_double(size), C.c_uint64(seed)))

    @staticmethod
    def cylinder(radius, height, na, nh):
        return RefMesh(lib().ref_make_cylinder(C.c_double(radius), C.c_double(height), int(na), int(nh)))

    @staticmethod
    def cone(radius, height, na):
        return RefMesh(lib().ref_make_cone(C.c_double(radius), C.c_double(height), int(na)))

    @staticmethod
    def concat(a, b):
        return RefMesh(lib().ref_concat_meshes(a.h, b.h))

    # ---- data
    def arrays(self):
        if self._arrays is None:
            nv, nf = self.nv, self.nf
            d = dict(
                xyz=np.empty((nv, 3)), tri=np.empty((nf, 3), np.int32), adj=np.empty((nf, 3), np.int32),
                fnormal=np.empty((nf, 3)), farea=np.empty(nf), vangle=np.empty(nv), varea=np.empty(nv),
                vboundary=np.empty(nv, np.uint8), csr_off=np.empty(nv + 1, np.int32),
                csr_list=np.empty(3 * nf, np.int32))
            lib().ref_mesh_get(self.h, *[_p(d[k]) for k in ("xyz", "tri", "adj", "fnormal", "farea", "vangle",
                                                           "varea", "vboundary", "csr_off", "csr_list")])
            d["mean_edge"] = lib().ref_mesh_mean_edge(self.h)
            d["total_area"] = lib().ref_mesh_total_area(self.h)
            self._arrays = d
        return self._arrays

    @property
    def xyz(self):
        return self.arrays()["xyz"]

    @property
    def tri(self):
        return self.arrays()["tri"]

    def default_max_steps(self):
        return lib().ref_default_max_steps(self.h)

    def default_gfd_eps(self):
        return lib().ref_default_gfd_eps(self.h)

    def sample_queries(self, seed, n, min_len, max_len):
        face = np.empty(n, np.int32)
        bary = np.empty((n, 3))
        d = np.empty((n, 3))
        lib().ref_sample_queries(self.h, C.c_uint64(seed), int(n), C.c_double(min_len), C.c_double(max_len),
                                 _p(face), _p(bary), _p(d))
        return face, bary, d

    def embed(self, face, bary):
        a = self.arrays()
        X = a["xyz"][a["tri"][face]]            # n,3,3
        return np.einsum("nk,nkd->nd", bary, X)

    # ---- tracing
    def _collect(self, h, record_polyline, keep_handle=False):
        L = lib()
        n = L.ref_result_size(h)
        r = TraceResult(face=np.empty(n, np.int32), bary=np.empty((n, 3)), dir=np.empty((n, 3)),
                        traced=np.empty(n), requested=np.empty(n), term=np.empty(n, np.uint8),
                        status=np.empty(n, np.uint8), payload=np.empty((n, 3)),
                        has_payload=np.empty(n, np.uint8), q=np.empty((n, 9)), npoints=np.empty(n, np.int32))
        has_q = np.empty(n, np.uint8)
        L.ref_result_soa(h, _p(r.face), _p(r.bary), _p(r.dir), _p(r.traced), _p(r.requested), _p(r.term),
                         _p(r.status), _p(r.payload), _p(r.has_payload), _p(r.q), _p(has_q), _p(r.npoints))
        if not has_q.any():
            r.q = None
        buf = C.create_string_buffer(256)
        r.errors = []
        for i in np.nonzero(r.status)[0]:
            L.ref_result_error(h, C.c_int64(int(i)), buf, 256)
            r.errors.append((int(i), buf.value.decode()))
        if record_polyline:
            off = np.zeros(n + 1, np.int64)
            np.cumsum(r.npoints, out=off[1:])
            tot = int(off[-1])
            r.poly_offsets = off
            r.poly_face = np.empty(tot, np.int32)
            r.poly_bary = np.empty((tot, 3))
            r.poly_seg = np.empty(tot)
            L.ref_result_polyline(h, _p(off), _p(r.poly_face), _p(r.poly_bary), _p(r.poly_seg))
        if keep_handle:
            return r, h
        L.ref_result_free(h)
        return r

    def trace_batch(self, face, bary, dirs, payload=None, max_steps=0, hole_avoidance=False, want_q=False,
                    record_polyline=False, use_f32=False, workers=0, json=False):
        face, bary, dirs, payload = _i32(face), _f64(bary), _f64(dirs), _f64(payload)
        ec = C.c_int(0)
        buf = C.create_string_buffer(512)
        h = lib().ref_trace_batch(self.h, C.c_int64(len(face)), _p(face), _p(bary), _p(dirs), _p(payload),
                                  int(max_steps), int(hole_avoidance), int(want_q), int(record_polyline),
                                  int(use_f32), int(workers), C.byref(ec), buf, 512)
        if not h:
            raise RefError(ERR_CLASS.get(ec.value, "?"), buf.value.decode())
        h = C.c_void_p(h)
        if json:
            r, h = self._collect(h, record_polyline, keep_handle=True)
            s = lib().ref_traces_json(h).decode()
            lib().ref_result_free(h)
            return r, s
        return self._collect(h, record_polyline)

    def trace(self, face, bary, d, payload=None, max_steps=0, hole_avoidance=False, want_q=False,
              record_polyline=True, use_f32=False):
        """digeo::trace: throws NumericalStall for stalled traces."""
        bary, d, payload = _f64(bary), _f64(d), _f64(payload)
        ec = C.c_int(0)
        buf = C.create_string_buffer(512)
        h = lib().ref_trace_single(self.h, int(face), _p(bary), _p(d), _p(payload), int(max_steps),
                                   int(hole_avoidance), int(want_q), int(record_polyline), int(use_f32),
                                   C.byref(ec), buf, 512)
        if not h:
            raise RefError(ERR_CLASS.get(ec.value, "?"), buf.value.decode())
        return self._collect(C.c_void_p(h), record_polyline)

    # ---- single transitions
    def geodesic_step(self, face, bary, v_unit, remaining, hole_avoidance=False):
        bary, v_unit = _f64(bary), _f64(v_unit)
        of = C.c_int32(0)
        ob, od = np.empty(3), np.empty(3)
        sl = C.c_double(0)
        fin, ev = C.c_int(0), C.c_int(0)
        buf = C.create_string_buffer(512)
        rc = lib().ref_geodesic_step(self.h, int(face), _p(bary), _p(v_unit), C.c_double(remaining),
                                     int(hole_avoidance), C.byref(of), _p(ob), _p(od), C.byref(sl),
                                     C.byref(fin), C.byref(ev), buf, 512)
        if rc:
            raise RefError(ERR_CLASS.get(rc, "?"), buf.value.decode())
        return dict(face=of.value, bary=ob, dir=od, step_length=sl.value, finished=bool(fin.value), event=ev.value)

    def transition(self, which, face, bary, v):
        """which: 0 transport_over_edge, 1 transport_over_vertex, 2 boundary_continue."""
        bary, v = _f64(bary), _f64(v)
        of = C.c_int32(0)
        ob, ov = np.empty(3), np.empty(3)
        buf = C.create_string_buffer(512)
        rc = lib().ref_transition(self.h, int(which), int(face), _p(bary), _p(v), C.byref(of), _p(ob), _p(ov),
                                  buf, 512)
        if rc:
            raise RefError(ERR_CLASS.get(rc, "?"), buf.value.decode())
        return of.value, ob, ov

    # ---- differentials
    def ep(self, face, bary, v, end_face, end_bary, end_dir, g=None):
        n = len(face)
        fd = lib().ref_frame_doubles()
        out = dict(rot=np.empty((n, 9)), frames=np.empty((n, fd)), grad_v=np.zeros((n, 3)), grad_p=np.zeros((n, 3)))
        ei = C.c_int64(-1)
        buf = C.create_string_buffer(512)
        rc = lib().ref_ep(self.h, C.c_int64(n), _p(_i32(face)), _p(_f64(bary)), _p(_f64(v)), _p(_i32(end_face)),
                          _p(_f64(end_bary)), _p(_f64(end_dir)), _p(_f64(g)), _p(out["rot"]), _p(out["frames"]),
                          _p(out["grad_v"]), _p(out["grad_p"]), C.byref(ei), buf, 512)
        if rc:
            e = RefError(ERR_CLASS.get(rc, "?"), buf.value.decode())
            e.index = ei.value
            raise e
        return out

    def gfd(self, face, bary, v, eps_v=None, eps_p=None, workers=0, g=None, mode=0):
        n = len(face)
        eps = self.default_gfd_eps()
        eps_v = eps if eps_v is None else eps_v
        eps_p = eps if eps_p is None else eps_p
        fd = lib().ref_frame_doubles()
        out = dict(jv=np.empty((n, 4)), jp=np.empty((n, 4)), degraded=np.empty((n, 4), np.uint8),
                   frames=np.empty((n, fd)), grad_v=np.zeros((n, 3)), grad_p=np.zeros((n, 3)))
        buf = C.create_string_buffer(512)
        rc = lib().ref_gfd(self.h, int(mode), C.c_int64(n), _p(_i32(face)), _p(_f64(bary)), _p(_f64(v)),
                           C.c_double(eps_v), C.c_double(eps_p), int(workers), _p(_f64(g)), _p(out["jv"]),
                           _p(out["jp"]), _p(out["degraded"]), _p(out["frames"]), _p(out["grad_v"]),
                           _p(out["grad_p"]), buf, 512)
        if rc:
            raise RefError(ERR_CLASS.get(rc, "?"), buf.value.decode())
        return out

    def gradcheck(self, scheme, n, seed, min_len, max_len, workers=0):
        out = np.empty(5)
        buf = C.create_string_buffer(512)
        rc = lib().ref_gradcheck(self.h, 1 if scheme == "gfd" else 0, int(n), C.c_uint64(seed),
                                 C.c_double(min_len), C.c_double(max_len), int(workers), _p(out), buf, 512)
        if rc:
            raise RefError(ERR_CLASS.get(rc, "?"), buf.value.decode())
        return dict(median_cos_v=out[0], median_norm_ratio_v=out[1], median_cos_p=out[2],
                    median_norm_ratio_p=out[3], max_p_grad_norm=out[4])


def resolve_workers(requested=0):
    return lib().ref_resolve_workers(int(requested))
