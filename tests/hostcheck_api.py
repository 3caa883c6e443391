"""ctypes binding of tests/_build/libdg_hostcheck.so: the device state machine compiled for the
host (tests/hostcheck/hostcheck.cu). TEST INFRASTRUCTURE for the CPU-only tier."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from refapi import TraceResult, _f64, _i32, _p

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_build", "libdg_hostcheck.so")
SRC = os.path.join(HERE, "hostcheck", "hostcheck.cu")
CORE = os.path.join(HERE, "..", "paper_2603_15780_b200", "csrc")


def build(force=False):
    deps = [SRC] + [os.path.join(CORE, f) for f in ("dg_tracer_core.cuh", "dg_mesh_view.cuh", "dg_math.cuh",
                                                     "dg_fast_walk.cuh", "dg_kernels.cuh")]
    if not force and os.path.exists(SO) and all(os.path.getmtime(SO) >= os.path.getmtime(d) for d in deps):
        return SO
    os.makedirs(os.path.dirname(SO), exist_ok=True)
    subprocess.check_call(["nvcc", "-x", "cu", "-O2", "-std=c++17", "-Wno-deprecated-gpu-targets", "-Xcompiler",
                           "-fPIC,-fopenmp,-fvisibility=hidden", "-shared", "-o", SO, SRC, "-lgomp"])
    return SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.hc_mesh_create.restype = C.c_void_p
    return _lib


class HostMesh:
    def __init__(self, arrays):
        a = arrays
        self.a = a
        self.nf = len(a["tri"])
        self.nv = len(a["xyz"])
        self.h = C.c_void_p(lib().hc_mesh_create(
            _p(_f64(a["xyz"])), self.nv, _p(_i32(a["tri"])), self.nf, _p(_i32(a["adj"])), _p(_f64(a["fnormal"])),
            _p(_f64(a["vangle"])), _p(np.ascontiguousarray(a["vboundary"], np.uint8)), _p(_i32(a["csr_off"])),
            _p(_i32(a["csr_list"]))))

    def __del__(self):
        try:
            lib().hc_mesh_free(self.h)
        except Exception:
            pass

    def trace_batch(self, face, bary, dirs, payload=None, max_steps=0, hole_avoidance=False, want_q=False,
                    record_polyline=False, use_f32=False):
        face, bary, dirs, payload = _i32(face), _f64(bary), _f64(dirs), _f64(payload)
        n = len(face)
        if max_steps <= 0:
            max_steps = int(10.0 * np.sqrt(float(self.nf))) + 100
        r = TraceResult(face=np.empty(n, np.int32), bary=np.empty((n, 3)), dir=np.empty((n, 3)),
                        traced=np.empty(n), requested=np.empty(n), term=np.empty(n, np.uint8),
                        status=np.empty(n, np.uint8), payload=np.empty((n, 3)), q=np.empty((n, 9)),
                        npoints=np.empty(n, np.int32))
        r.stall = np.empty(n, np.uint8)
        r.crossings = np.empty(n, np.int32)

        def call(off, pf, pb, ps):
            lib().hc_trace_batch(self.h, C.c_int64(n), _p(face), _p(bary), _p(dirs), _p(payload), int(max_steps),
                                 int(hole_avoidance), int(want_q), int(use_f32), _p(r.face), _p(r.bary), _p(r.dir),
                                 _p(r.traced), _p(r.requested), _p(r.term), _p(r.status), _p(r.stall), _p(r.payload),
                                 _p(r.q), _p(r.npoints), _p(r.crossings), _p(off), _p(pf), _p(pb), _p(ps))
        call(None, None, None, None)
        if record_polyline:
            off = np.zeros(n + 1, np.int64)
            np.cumsum(r.npoints, out=off[1:])
            tot = int(off[-1])
            r.poly_offsets = off
            r.poly_face = np.empty(tot, np.int32)
            r.poly_bary = np.empty((tot, 3))
            r.poly_seg = np.empty(tot)
            call(off, r.poly_face, r.poly_bary, r.poly_seg)
        if payload is not None:
            r.has_payload = (np.square(payload).sum(1) > 0).astype(np.uint8)
        return r

    def trace_batch_fast(self, face, bary, dirs, max_steps=0, cached=False, payload=None, hole_avoidance=False,
                         record_polyline=False, want_q=False, lane_fast=False):
        """The fast walker (csrc/dg_fast_walk.cuh: fast_init / fast_step / fast_finish + the generic
        paths behind them) driven on the host the way trace_fast_kernel drives a lane."""
        face, bary, dirs, payload = _i32(face), _f64(bary), _f64(dirs), _f64(payload)
        n = len(face)
        if max_steps <= 0:
            max_steps = int(10.0 * np.sqrt(float(self.nf))) + 100
        r = TraceResult(face=np.empty(n, np.int32), bary=np.empty((n, 3)), dir=np.empty((n, 3)),
                        traced=np.empty(n), requested=np.empty(n), term=np.empty(n, np.uint8),
                        status=np.empty(n, np.uint8), npoints=np.empty(n, np.int32))
        r.stall = np.empty(n, np.uint8)
        r.crossings = np.empty(n, np.int32)
        if payload is not None:
            r.payload = np.empty((n, 3))
        if want_q:
            r.q = np.empty((n, 9))

        lib().hc_set_lane_fast(int(lane_fast))

        def call(off, pf, pb, ps):
            lib().hc_trace_batch_fast(self.h, C.c_int64(n), _p(face), _p(bary), _p(dirs), _p(payload), _p(r.payload),
                                      int(hole_avoidance), int(want_q), _p(r.q), int(max_steps), int(cached), _p(r.face), _p(r.bary), _p(r.dir),
                                      _p(r.traced), _p(r.requested), _p(r.term), _p(r.status), _p(r.stall), _p(r.npoints),
                                      _p(r.crossings), _p(off), _p(pf), _p(pb), _p(ps))
        call(None, None, None, None)
        if lane_fast:
            lib().hc_set_lane_fast(0)
        if record_polyline:   # the two passes of the C-ABI: count, scan, fill
            off = np.zeros(n + 1, np.int64)
            np.cumsum(r.npoints, out=off[1:])
            tot = int(off[-1])
            r.poly_offsets = off
            r.poly_face = np.empty(tot, np.int32)
            r.poly_bary = np.empty((tot, 3))
            r.poly_seg = np.empty(tot)
            call(off, r.poly_face, r.poly_bary, r.poly_seg)
        return r
