"""Array-level mirror of the reference's operator interface for this path, over the C-ABI.

Names and argument meaning follow proj/include/digeo/{mesh,tracer,diff}.hpp (Mesh::build,
trace_batch, geodesic_step ..., ep_jacobians, gfd_batched_many, pullback_ambient); the
object-level C++ mirror lives in include/digeo/. Inputs/outputs are numpy arrays (host mode:
the library stages them) or torch CUDA tensors (device mode: zero-copy, asynchronous on the
current torch stream).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import capi
from .capi import DgError, DiffCfg, TraceCfg, TraceIn, TraceOut, check, lib, ptr


def _f64(a, shape=None):
    if a is None:
        return None
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a.reshape(shape) if shape else a


def _i32(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.int32)


def _is_torch(a):
    return a is not None and not isinstance(a, np.ndarray) and hasattr(a, "data_ptr")


@dataclass
class TraceResult:
    face: np.ndarray
    bary: np.ndarray
    dir: np.ndarray
    traced: np.ndarray
    requested: np.ndarray
    term: np.ndarray       # 0 LengthReached, 1 Boundary, 2 MaxSteps
    status: np.ndarray     # 0 Ok, 1 Stalled
    stall: np.ndarray      # DG_STALL_*
    npoints: np.ndarray
    crossings: np.ndarray
    total_crossings: int = 0
    payload: np.ndarray | None = None
    has_payload: np.ndarray | None = None
    q: np.ndarray | None = None
    poly_offsets: np.ndarray | None = None
    poly_face: np.ndarray | None = None
    poly_bary: np.ndarray | None = None
    poly_seg: np.ndarray | None = None
    errors: list = field(default_factory=list)


class Mesh:
    """Immutable triangle mesh: host-side derived arrays (Mesh::build, mesh.cpp:34-130) plus
    the GPU-resident fat-record store (dg_mesh_create)."""

    def __init__(self, xyz, tri, device=None, upload=True, transport_cache="auto", devices=None):
        """device: the CUDA ordinal the mesh lives on; devices: a LIST of ordinals (multi-GPU, dg_set_device_list):
        the mesh is replicated on each of them and large batched calls fan out over the set, results at the request
        index, bitwise independent of the set. An ordinal may repeat (several copies on one GPU, for tests)."""
        L = lib()
        self.devices = None if devices is None else [int(x) for x in devices]
        self.transport_cache = transport_cache
        self.has_transport_cache = False
        self.uses_tma_gather = False
        self.gather = "loads"      # how lone traces fetch the crossing records: loads | tma | coop
        self.xyz = _f64(xyz).reshape(-1, 3)
        self.tri = _i32(tri).reshape(-1, 3)
        nv, nf = len(self.xyz), len(self.tri)
        self.nv, self.nf = nv, nf
        self.adj = np.empty((nf, 3), np.int32)
        self.fnormal = np.empty((nf, 3))
        self.farea = np.empty(nf)
        self.vangle = np.empty(nv)
        self.varea = np.empty(nv)
        self.vboundary = np.empty(nv, np.uint8)
        self.csr_off = np.empty(nv + 1, np.int32)
        self.csr_list = np.empty(3 * nf, np.int32)
        me, ta, ei = C.c_double(0), C.c_double(0), C.c_int64(-1)
        check(L.dg_mesh_derive(ptr(self.xyz), nv, ptr(self.tri), nf, ptr(self.adj), ptr(self.fnormal),
                               ptr(self.farea), ptr(self.vangle), ptr(self.varea), ptr(self.vboundary),
                               ptr(self.csr_off), ptr(self.csr_list), C.addressof(me), C.addressof(ta),
                               C.addressof(ei)), ei)
        self.mean_edge = me.value
        self.total_area = ta.value
        self.h = None
        if upload:
            self.upload(device)

    build = classmethod(lambda cls, xyz, tri, **kw: cls(xyz, tri, **kw))

    def upload(self, device=None):
        L = lib()
        capi.require_device()
        if self.devices:
            arr = np.asarray(self.devices, np.int32)
            check(L.dg_set_device_list(ptr(arr), len(arr)))
        elif device is not None:
            check(L.dg_set_device(int(device)))
        h = C.c_void_p(0)
        flags = {"auto": 0, None: 0, True: 1, "on": 1, False: 2, "off": 2}[self.transport_cache]
        check(L.dg_mesh_create_ex(ptr(self.xyz), self.nv, ptr(self.tri), self.nf, ptr(self.adj), ptr(self.fnormal),
                                  ptr(self.vangle), ptr(self.vboundary), ptr(self.csr_off), ptr(self.csr_list),
                                  flags, C.addressof(h)))
        self.h = h
        if self.devices:   # the device set is per creating thread: go back to a single device for later meshes
            check(L.dg_set_device(self.devices[0]))
        self.device_count = int(L.dg_mesh_device_count(h))
        self.has_transport_cache = bool(L.dg_mesh_has_transport_cache(h))
        self.uses_tma_gather = bool(L.dg_mesh_uses_tma_gather(h))
        self.gather = ("loads", "tma", "coop")[L.dg_mesh_gather_mode(h)]
        return self

    def __del__(self):
        try:
            if self.h:
                lib().dg_mesh_destroy(self.h)
                self.h = None
        except Exception:
            pass

    @property
    def device_bytes(self):
        return lib().dg_mesh_device_bytes(self.h)

    def trace_plan(self, n, device_mode=True):
        """(face_order, gather) a plain f64 forward request of n queries gets by default (dg_trace_plan)."""
        fo, ga = C.c_int(0), C.c_int(0)
        cfg = TraceCfg(memory=capi.MEM_DEVICE if device_mode else capi.MEM_HOST)
        check(lib().dg_trace_plan(self._handle(), int(n), C.addressof(cfg), C.addressof(fo), C.addressof(ga)))
        return bool(fo.value), ("loads", "tma", "coop")[ga.value]

    def default_max_steps(self):
        return int(10.0 * np.sqrt(float(self.nf))) + 100

    def default_gfd_eps(self):
        return 1e-4 * self.mean_edge

    def embed(self, face, bary):
        X = self.xyz[self.tri[face]]
        return np.einsum("nk,nkd->nd", bary, X)

    def _handle(self):
        if not self.h:
            raise DgError(capi.DG_ERR_NO_DEVICE, "mesh is not resident on a GPU (there is no CPU fallback)")
        return self.h

    # ------------------------------------------------------------------ forward tracing
    def trace_batch(self, face, bary, dirs, payload=None, max_steps=0, hole_avoidance=False, want_q=False,
                    record_polyline=False, use_f32=False, sort_by_face=None, refill_min=0, blocks_per_sm=0,
                    out=None, generic_walker=False, walker="auto", two_call_polylines=False, poly_views=False, lane="exact"):
        """trace_batch (tracer.cpp:596) on host arrays; results at the request index. `out`: a
        TraceResult of a previous call of the same size whose (e.g. pinned) arrays are reused.
        record_polyline: ONE call (dg_trace_polylines: capped first pass, device scan, compaction); the polylines
        are copied out of the mesh's pinned arrays unless poly_views=True (views: valid until the next recording
        call on this mesh). two_call_polylines=True runs the count call + host scan + fill call instead."""
        h = self._handle()
        face, bary, dirs, payload = _i32(face), _f64(bary), _f64(dirs), _f64(payload)
        n = len(face)
        if bary.size != 3 * n or dirs.size != 3 * n:
            raise DgError(1, "trace_batch: starts and dirs differ in length")
        if payload is not None and payload.size != 3 * n:
            raise DgError(1, "trace_batch: payloads must be empty or match the batch size")
        r = out if out is not None else TraceResult(
            face=np.empty(n, np.int32), bary=np.empty((n, 3)), dir=np.empty((n, 3)),
            traced=np.empty(n), requested=np.empty(n), term=np.empty(n, np.uint8),
            status=np.empty(n, np.uint8), stall=np.empty(n, np.uint8),
            npoints=np.empty(n, np.int32), crossings=np.empty(n, np.int32))
        if payload is not None:
            r.payload = np.empty((n, 3))
            r.has_payload = (np.square(payload.reshape(n, 3)).sum(1) > 0).astype(np.uint8)
        if want_q:
            r.q = np.empty((n, 9))
        cfg = TraceCfg(max_steps=int(max_steps), hole_avoidance=int(hole_avoidance),
                       want_transport_matrix=int(want_q), use_f32=int(use_f32), memory=capi.MEM_HOST,
                       sort_by_face=SORT[sort_by_face], refill_min=int(refill_min), blocks_per_sm=int(blocks_per_sm),
                       walker=1 if generic_walker else WALKERS[walker], lane=LANES[lane])
        tin = TraceIn(ptr(face), ptr(bary), ptr(dirs), ptr(payload))
        total = C.c_uint64(0)

        def call(off, pf, pb, ps, tot):
            out = TraceOut(ptr(r.face), ptr(r.bary), ptr(r.dir), ptr(r.traced), ptr(r.requested), ptr(r.term),
                           ptr(r.status), ptr(r.stall), ptr(r.payload), ptr(r.q), ptr(r.npoints), ptr(r.crossings),
                           C.addressof(total), ptr(off), tot, ptr(pf), ptr(pb), ptr(ps))
            check(lib().dg_trace_batch(h, n, C.addressof(tin), C.addressof(cfg), C.addressof(out)))

        if record_polyline and not two_call_polylines and sort_by_face is not True:
            out_s = TraceOut(ptr(r.face), ptr(r.bary), ptr(r.dir), ptr(r.traced), ptr(r.requested), ptr(r.term),
                             ptr(r.status), ptr(r.stall), ptr(r.payload), ptr(r.q), ptr(r.npoints), ptr(r.crossings),
                             C.addressof(total), None, 0, None, None, None)
            pl = capi.Polylines()
            check(lib().dg_trace_polylines(h, n, C.addressof(tin), C.addressof(cfg), C.addressof(out_s), C.addressof(pl)))
            tot = int(pl.total)
            view = lambda p, count, shape: (np.ctypeslib.as_array(p, shape=(count,)).reshape(shape) if count else
                                            np.empty(shape, np.ctypeslib.as_array(p, shape=(1,)).dtype if p else np.float64))
            keep = (lambda a: a) if poly_views else (lambda a: a.copy())
            r.poly_offsets = keep(np.ctypeslib.as_array(pl.offsets, shape=(n + 1,)))
            r.poly_face = keep(view(pl.face, tot, (tot,))) if tot else np.empty(0, np.int32)
            r.poly_bary = keep(view(pl.bary, 3 * tot, (tot, 3))) if tot else np.empty((0, 3))
            r.poly_seg = keep(view(pl.seg, tot, (tot,))) if tot else np.empty(0)
            r.total_crossings = int(total.value)
            r.errors = [(int(i), capi.STALL_MESSAGES[int(r.stall[i])]) for i in np.nonzero(r.status)[0]]
            return r
        call(None, None, None, None, 0)
        if record_polyline:
            # two passes: the first sized the polylines (npoints), the second writes them
            off = np.zeros(n + 1, np.int64)
            np.cumsum(r.npoints, out=off[1:])
            tot = int(off[-1])
            r.poly_offsets = off
            r.poly_face = np.empty(tot, np.int32)
            r.poly_bary = np.empty((tot, 3))
            r.poly_seg = np.empty(tot)
            if n:
                call(off, r.poly_face, r.poly_bary, r.poly_seg, tot)
        r.total_crossings = int(total.value)
        r.errors = [(int(i), capi.STALL_MESSAGES[int(r.stall[i])]) for i in np.nonzero(r.status)[0]]
        return r

    def trace_batch_device(self, face, bary, dirs, out, payload=None, max_steps=0, hole_avoidance=False,
                           want_q=False, stream=None, sort_by_face=None, refill_min=0, blocks_per_sm=0,
                           generic_walker=False, walker="auto", lane="exact"):
        """Zero-copy entry point: every array is a torch CUDA tensor on the mesh's device;
        `out` maps dg_trace_out field names to preallocated tensors. Asynchronous on `stream`."""
        import torch
        h = self._handle()
        n = int(face.numel())
        cfg = TraceCfg(max_steps=int(max_steps), hole_avoidance=int(hole_avoidance),
                       want_transport_matrix=int(want_q), memory=capi.MEM_DEVICE, sort_by_face=SORT[sort_by_face],
                       refill_min=int(refill_min), blocks_per_sm=int(blocks_per_sm),
                       walker=1 if generic_walker else WALKERS[walker], lane=LANES[lane],
                       stream=(stream if stream is not None else torch.cuda.current_stream().cuda_stream))
        tin = TraceIn(ptr(face), ptr(bary), ptr(dirs), ptr(payload))
        o = TraceOut()
        for k, v in out.items():
            if k == "poly_total":
                o.poly_total = int(v)
            else:
                setattr(o, k, ptr(v))
        check(lib().dg_trace_batch(h, n, C.addressof(tin), C.addressof(cfg), C.addressof(o)))

    # ------------------------------------------------------- single-transition operations
    def transition(self, which, face, bary, v, remaining=None, hole_avoidance=False):
        """which: 0 geodesic_step, 1 transport_over_edge, 2 transport_over_vertex,
        3 boundary_continue (tracer.cpp:630-735), on n independent states."""
        h = self._handle()
        face, bary, v = _i32(np.atleast_1d(face)), _f64(bary).reshape(-1, 3), _f64(v).reshape(-1, 3)
        n = len(face)
        rem = _f64(np.broadcast_to(np.asarray(0.0 if remaining is None else remaining, float), (n,)))
        o = dict(face=np.empty(n, np.int32), bary=np.empty((n, 3)), v=np.empty((n, 3)), step_length=np.zeros(n),
                 finished=np.zeros(n, np.uint8), event=np.zeros(n, np.uint8), stall=np.zeros(n, np.uint8),
                 rc=np.zeros(n, np.int32))
        check(lib().dg_transition(h, int(which), n, ptr(face), ptr(bary), ptr(v), ptr(rem), int(hole_avoidance),
                                  ptr(o["face"]), ptr(o["bary"]), ptr(o["v"]), ptr(o["step_length"]),
                                  ptr(o["finished"]), ptr(o["event"]), ptr(o["stall"]), ptr(o["rc"])))
        return o

    # --------------------------------------------------------------------- differentials
    def ep(self, face, bary, v, end_face, end_bary, end_dir, g=None):
        """ep_jacobians (+ pullback_ambient when g is given), diff.cpp:44-66, :347-354."""
        h = self._handle()
        face, end_face = _i32(face), _i32(end_face)
        n = len(face)
        bary, v, end_bary, end_dir, g = _f64(bary), _f64(v), _f64(end_bary), _f64(end_dir), _f64(g)
        out = dict(rot=np.empty((n, 9)), frames=np.empty((n, capi.FRAME_DOUBLES)), grad_v=np.zeros((n, 3)),
                   grad_p=np.zeros((n, 3)))
        ei = C.c_int64(-1)
        cfg = DiffCfg(memory=capi.MEM_HOST)
        check(lib().dg_ep_jacobians(h, n, ptr(face), ptr(bary), ptr(v), ptr(end_face), ptr(end_bary), ptr(end_dir),
                                    C.addressof(cfg), ptr(out["rot"]), ptr(out["frames"]), C.addressof(ei)), ei)
        if g is not None:
            check(lib().dg_ep_backward(h, n, ptr(face), ptr(v), ptr(end_face), ptr(end_dir), ptr(g),
                                       C.addressof(cfg), ptr(out["grad_v"]), ptr(out["grad_p"]), C.addressof(ei)), ei)
        return out

    def ep_backward(self, face, v, end_face, end_dir, g, grad_v=None):
        """Fused ep_jacobians + pullback_ambient on host arrays: returns grad_v (grad_p == 0)."""
        face, end_face = _i32(face), _i32(end_face)
        n = len(face)
        v, end_dir, g = _f64(v), _f64(end_dir), _f64(g)
        if grad_v is None:
            grad_v = np.empty((n, 3))
        ei = C.c_int64(-1)
        cfg = DiffCfg(memory=capi.MEM_HOST)
        check(lib().dg_ep_backward(self._handle(), n, ptr(face), ptr(v), ptr(end_face), ptr(end_dir), ptr(g),
                                   C.addressof(cfg), ptr(grad_v), None, C.addressof(ei)), ei)
        return grad_v

    def ep_backward_device(self, face, v, end_face, end_dir, g, grad_v, grad_p=None, stream=None):
        import torch
        cfg = DiffCfg(memory=capi.MEM_DEVICE,
                      stream=(stream if stream is not None else torch.cuda.current_stream().cuda_stream))
        ei = C.c_int64(-1)
        check(lib().dg_ep_backward(self._handle(), int(face.numel()), ptr(face), ptr(v), ptr(end_face), ptr(end_dir),
                                   ptr(g), C.addressof(cfg), ptr(grad_v), ptr(grad_p), C.addressof(ei)), ei)

    def gfd(self, face, bary, v, eps_v=None, eps_p=None, g=None, max_steps=0, out=None, base=None, plain_schedule=False):
        """gfd_batched_many (+ pullback_ambient when g is given), diff.cpp:273-326. plain_schedule: False = AUTO,
        True = plain job order, 2 = sibling groups in start-face order of their samples (dg_diff_cfg.schedule). `out`: a dict
        of preallocated (e.g. pinned) arrays; only the keys present are computed and copied back
        (jv, jp, degraded, frames, grad_v, grad_p, base_face, base_bary, base_dir)."""
        h = self._handle()
        face = _i32(face)
        n = len(face)
        bary, v, g = _f64(bary), _f64(v), _f64(g)
        eps = self.default_gfd_eps()
        eps_v = eps if eps_v is None else eps_v
        eps_p = eps if eps_p is None else eps_p
        if out is None:
            out = dict(jv=np.zeros((n, 4)), jp=np.zeros((n, 4)), degraded=np.zeros((n, 4), np.uint8),
                       frames=np.zeros((n, capi.FRAME_DOUBLES)), grad_v=np.zeros((n, 3)), grad_p=np.zeros((n, 3)),
                       base_face=np.empty(n, np.int32), base_bary=np.empty((n, 3)), base_dir=np.empty((n, 3)))
        ei = C.c_int64(-1)
        cfg = DiffCfg(memory=capi.MEM_HOST, max_steps=int(max_steps), schedule=int(plain_schedule))
        o = lambda k: ptr(out.get(k))
        if base is not None:  # a TraceResult of trace_batch on the same samples (gfd_batched's `trace` argument)
            # converted copies are bound to locals: they must outlive the C call
            bface, bbary, bdir = _i32(base.face), _f64(base.bary), _f64(base.dir)
            bterm, bstatus = np.ascontiguousarray(base.term, np.uint8), np.ascontiguousarray(base.status, np.uint8)
            check(lib().dg_gfd_jacobians_with_base(
                h, n, ptr(face), ptr(bary), ptr(v), ptr(bface), ptr(bbary), ptr(bdir),
                ptr(bterm), ptr(bstatus), float(eps_v), float(eps_p), ptr(g), C.addressof(cfg), o("jv"), o("jp"),
                o("degraded"), o("frames"), o("grad_v") if g is not None else None,
                o("grad_p") if g is not None else None, C.addressof(ei)), ei)
            return out
        check(lib().dg_gfd_jacobians(h, n, ptr(face), ptr(bary), ptr(v), float(eps_v), float(eps_p), ptr(g),
                                     C.addressof(cfg), o("jv"), o("jp"), o("degraded"), o("frames"),
                                     o("grad_v") if g is not None else None, o("grad_p") if g is not None else None,
                                     o("base_face"), o("base_bary"), o("base_dir"), C.addressof(ei)), ei)
        return out

    def gfd_device(self, face, bary, v, eps_v, eps_p, g, jv, jp, grad_v=None, grad_p=None, degraded=None,
                   stream=None, max_steps=0, base=None, plain_schedule=False):
        """`base`: the forward results of the same samples (dict of device tensors face / bary / dir /
        term / status, as trace_batch_device writes them): GFD then takes them as its base traces
        (the `trace` argument of gfd_batched, diff.hpp:73) instead of re-tracing them."""
        import torch
        cfg = DiffCfg(memory=capi.MEM_DEVICE, max_steps=int(max_steps), schedule=int(plain_schedule),
                      stream=(stream if stream is not None else torch.cuda.current_stream().cuda_stream))
        ei = C.c_int64(-1)
        if base is not None:
            check(lib().dg_gfd_jacobians_with_base(
                self._handle(), int(face.numel()), ptr(face), ptr(bary), ptr(v), ptr(base["face"]), ptr(base["bary"]),
                ptr(base["dir"]), ptr(base["term"]), ptr(base["status"]), float(eps_v), float(eps_p), ptr(g),
                C.addressof(cfg), ptr(jv), ptr(jp), ptr(degraded), None, ptr(grad_v), ptr(grad_p), C.addressof(ei)), ei)
            return
        check(lib().dg_gfd_jacobians(self._handle(), int(face.numel()), ptr(face), ptr(bary), ptr(v), float(eps_v),
                                     float(eps_p), ptr(g), C.addressof(cfg), ptr(jv), ptr(jp), ptr(degraded), None,
                                     ptr(grad_v), ptr(grad_p), None, None, None, C.addressof(ei)), ei)


    # ------------------------------------------ fused forward + GFD Jacobians, pull-back only backward
    def trace_gfd(self, face, bary, dirs, eps_v=None, eps_p=None, max_steps=0, plain_schedule=False, lane="exact"):
        """dg_trace_gfd on host arrays: the forward exp map and the GFD Jacobians of the same samples in one call
        (the forward traces ride in GFD's round 2 as the fourth sibling). Returns (TraceResult, dict jv/jp/degraded/
        frames). A whole-call GFD failure raises AFTER the forward results are in place (`.forward` of the error)."""
        h = self._handle()
        face, bary, dirs = _i32(face), _f64(bary), _f64(dirs)
        n = len(face)
        eps = self.default_gfd_eps()
        eps_v = eps if eps_v is None else eps_v
        eps_p = eps if eps_p is None else eps_p
        r = TraceResult(face=np.empty(n, np.int32), bary=np.empty((n, 3)), dir=np.empty((n, 3)), traced=np.empty(n),
                        requested=np.empty(n), term=np.empty(n, np.uint8), status=np.empty(n, np.uint8),
                        stall=np.empty(n, np.uint8), npoints=np.empty(n, np.int32), crossings=np.empty(n, np.int32))
        jac = dict(jv=np.zeros((n, 4)), jp=np.zeros((n, 4)), degraded=np.zeros((n, 4), np.uint8),
                   frames=np.zeros((n, capi.FRAME_DOUBLES)))
        total = C.c_uint64(0)
        o = TraceOut(ptr(r.face), ptr(r.bary), ptr(r.dir), ptr(r.traced), ptr(r.requested), ptr(r.term), ptr(r.status),
                     ptr(r.stall), None, None, ptr(r.npoints), ptr(r.crossings), C.addressof(total), None, 0, None, None, None)
        cfg = DiffCfg(memory=capi.MEM_HOST, max_steps=int(max_steps), schedule=int(plain_schedule), lane=LANES[lane])
        ei = C.c_int64(-1)
        rc = lib().dg_trace_gfd(h, n, ptr(face), ptr(bary), ptr(dirs), float(eps_v), float(eps_p), C.addressof(cfg),
                                C.addressof(o), ptr(jac["jv"]), ptr(jac["jp"]), ptr(jac["degraded"]), ptr(jac["frames"]),
                                C.addressof(ei))
        r.total_crossings = int(total.value)
        r.errors = [(int(i), capi.STALL_MESSAGES[int(r.stall[i])]) for i in np.nonzero(r.status)[0]]
        if rc != capi.DG_OK:
            e = DgError(rc, lib().dg_last_error().decode())
            e.index = ei.value
            e.forward = r
            raise e
        return r, jac

    def trace_gfd_device(self, face, bary, dirs, out, eps_v, eps_p, jv, jp, degraded=None, stream=None, max_steps=0,
                         lane="exact"):
        """dg_trace_gfd on torch CUDA tensors; `out` as trace_batch_device."""
        import torch
        cfg = DiffCfg(memory=capi.MEM_DEVICE, max_steps=int(max_steps), lane=LANES[lane],
                      stream=(stream if stream is not None else torch.cuda.current_stream().cuda_stream))
        o = TraceOut()
        for k, v in out.items():
            setattr(o, k, ptr(v))
        ei = C.c_int64(-1)
        check(lib().dg_trace_gfd(self._handle(), int(face.numel()), ptr(face), ptr(bary), ptr(dirs), float(eps_v), float(eps_p),
                                 C.addressof(cfg), C.addressof(o), ptr(jv), ptr(jp), ptr(degraded), None, C.addressof(ei)), ei)

    def gfd_pullback(self, face, v, end_face, jv, jp, g):
        """pullback_ambient of g through Jacobians that are already there (dg_gfd_pullback), host arrays."""
        face, end_face, v, jv, jp, g = _i32(face), _i32(end_face), _f64(v), _f64(jv), _f64(jp), _f64(g)
        n = len(face)
        out = dict(grad_v=np.zeros((n, 3)), grad_p=np.zeros((n, 3)))
        cfg = DiffCfg(memory=capi.MEM_HOST)
        check(lib().dg_gfd_pullback(self._handle(), n, ptr(face), ptr(v), ptr(end_face), ptr(jv), ptr(jp), ptr(g),
                                    C.addressof(cfg), ptr(out["grad_v"]), ptr(out["grad_p"])))
        return out

    def gfd_pullback_device(self, face, v, end_face, jv, jp, g, grad_v, grad_p=None, stream=None):
        import torch
        cfg = DiffCfg(memory=capi.MEM_DEVICE,
                      stream=(stream if stream is not None else torch.cuda.current_stream().cuda_stream))
        check(lib().dg_gfd_pullback(self._handle(), int(face.numel()), ptr(face), ptr(v), ptr(end_face), ptr(jv), ptr(jp), ptr(g),
                                    C.addressof(cfg), ptr(grad_v), ptr(grad_p)))


# dg_trace_cfg.lane / dg_diff_cfg.lane (DG_LANE_*)
LANES = {"exact": 1, "default": 0, None: 0, "fast": 2}
# dg_trace_cfg.sort_by_face (DG_SORT_*): None = the library decides
SORT = {None: 0, "auto": 0, True: 1, False: 2, 1: 1, 0: 2}
# dg_trace_cfg.walker (DG_WALKER_*): which kernel traces a plain f64 forward request
WALKERS = {"auto": 0, "generic": 1, "loads": 2, "tma": 3, "coop": 4}


class Batch:
    """Resident batch (dg_batch_*): forward exp map, then EP or GFD backward on the same samples,
    with the forward state kept on the GPU between the calls. Host arrays in, host arrays out."""

    def __init__(self, mesh, capacity):
        self.mesh = mesh
        self.capacity = int(capacity)
        h = C.c_void_p()
        check(lib().dg_batch_create(mesh._handle(), self.capacity, C.addressof(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().dg_batch_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown: the library handle may already be gone
            pass

    def trace(self, face, bary, dirs, max_steps=0, refill_min=0, blocks_per_sm=0, out=None, gfd=False, eps_v=None,
              eps_p=None, lane="exact"):
        """gfd=True: the forward of a step whose backward will be GFD (dg_batch_trace_gfd): the Jacobians are
        computed with the forward traces (fourth sibling of GFD's round 2) and stay on the GPU; the following
        Batch.gfd(g=...) with the same eps only pulls g back."""
        face, bary, dirs = _i32(face), _f64(bary), _f64(dirs)
        n = len(face)
        if bary.size != 3 * n or dirs.size != 3 * n:
            raise DgError(1, "trace_batch: starts and dirs differ in length")
        r = out if out is not None else TraceResult(
            face=np.empty(n, np.int32), bary=np.empty((n, 3)), dir=np.empty((n, 3)),
            traced=np.empty(n), requested=np.empty(n), term=np.empty(n, np.uint8),
            status=np.empty(n, np.uint8), stall=np.empty(n, np.uint8),
            npoints=np.empty(n, np.int32), crossings=np.empty(n, np.int32))
        cfg = TraceCfg(max_steps=int(max_steps), memory=capi.MEM_HOST, refill_min=int(refill_min),
                       blocks_per_sm=int(blocks_per_sm), lane=LANES[lane])
        tin = TraceIn(ptr(face), ptr(bary), ptr(dirs), None)
        total = C.c_uint64(0)
        o = TraceOut(ptr(r.face), ptr(r.bary), ptr(r.dir), ptr(r.traced), ptr(r.requested), ptr(r.term),
                     ptr(r.status), ptr(r.stall), None, None, ptr(r.npoints), ptr(r.crossings),
                     C.addressof(total), None, 0, None, None, None)
        if gfd:
            eps = self.mesh.default_gfd_eps()
            check(lib().dg_batch_trace_gfd(self._h, n, C.addressof(tin), C.addressof(cfg), float(eps if eps_v is None else eps_v),
                                           float(eps if eps_p is None else eps_p), C.addressof(o)))
        else:
            check(lib().dg_batch_trace(self._h, n, C.addressof(tin), C.addressof(cfg), C.addressof(o)))
        r.total_crossings = int(total.value)
        return r

    def ep_backward(self, g, grad_v=None, grad_p=None):
        n = int(lib().dg_batch_size(self._h))
        g = _f64(g)
        if grad_v is None:
            grad_v = np.empty((n, 3))
        ei = C.c_int64(-1)
        check(lib().dg_batch_ep_backward(self._h, ptr(g), ptr(grad_v), ptr(grad_p), C.addressof(ei)), ei)
        return grad_v

    def gfd(self, eps_v=None, eps_p=None, g=None, max_steps=0, out=None):
        n = int(lib().dg_batch_size(self._h))
        g = _f64(g)
        eps = self.mesh.default_gfd_eps()
        eps_v = eps if eps_v is None else eps_v
        eps_p = eps if eps_p is None else eps_p
        if out is None:
            out = dict(jv=np.zeros((n, 4)), jp=np.zeros((n, 4)), degraded=np.zeros((n, 4), np.uint8),
                       grad_v=np.zeros((n, 3)), grad_p=np.zeros((n, 3)))
        ei = C.c_int64(-1)
        o = lambda k: ptr(out.get(k))
        check(lib().dg_batch_gfd(self._h, float(eps_v), float(eps_p), ptr(g), int(max_steps), o("jv"), o("jp"),
                                 o("degraded"), o("grad_v") if g is not None else None,
                                 o("grad_p") if g is not None else None, C.addressof(ei)), ei)
        return out


def kernel_info(use_f32=False, full=False, cached=False, tma=False, coop=False, dense=False):
    regs, bps, bt = C.c_int(0), C.c_int(0), C.c_int(0)
    lib().dg_trace_kernel_info(int(use_f32), int(full) | (int(cached) << 1) | (int(tma) << 2) | (int(coop) << 3) | (int(dense) << 4),
                               C.addressof(regs), C.addressof(bps),
                               C.addressof(bt))
    return dict(registers=regs.value, blocks_per_sm=bps.value, block_threads=bt.value)
