"""ctypes binding of libdigeo_b200.so (include/dg_b200.h).

This is the only way Python reaches the compute path: every function here is a thin call
into the C-ABI. There is no Python or CPU implementation behind it -- if the shared library
is missing the import fails, and if no CUDA device is usable every compute call raises
DgError(DG_ERR_NO_DEVICE).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DG_B200_LIB") or os.path.join(PKG, "lib", "libdigeo_b200.so")

DG_OK = 0
ERR_NAMES = {1: "InvalidArgs", 2: "CudaError", 3: "ParseError", 4: "NonManifoldError",
             5: "DegenerateFaceError", 6: "DegenerateDirection", 7: "Error", 8: "NoDevice",
             10: "NumericalStall", 11: "BoundaryHit"}
DG_ERR_NO_DEVICE = 8
MEM_HOST, MEM_DEVICE = 0, 1
FRAME_DOUBLES = 33

# messages of the per-element stall codes (reference strings, tracer.cpp:183,197,474,459,461)
STALL_MESSAGES = {
    0: "",
    1: "degenerate direction in face",
    2: "no positive exit parameter",
    3: "initial direction is normal to the anchor face",
    4: "trace: start face out of range",
    5: "trace: start barycentric coordinates not in the simplex",
}

EXPORTS = [
    "dg_last_error", "dg_version", "dg_device_count", "dg_set_device", "dg_set_devices", "dg_set_device_list",
    "dg_mesh_device_count", "dg_device_sm_count", "dg_trim",
    "dg_mesh_derive", "dg_mesh_create", "dg_mesh_create_ex", "dg_mesh_has_transport_cache", "dg_mesh_uses_tma_gather", "dg_mesh_gather_mode", "dg_mesh_destroy", "dg_mesh_face_count", "dg_mesh_vertex_count",
    "dg_mesh_device_bytes", "dg_mesh_device", "dg_trace_batch", "dg_trace_polylines", "dg_trace_plan", "dg_transition", "dg_ep_jacobians",
    "dg_ep_backward", "dg_gfd_jacobians", "dg_gfd_jacobians_with_base", "dg_trace_gfd", "dg_gfd_pullback", "dg_trace_kernel_info",
    "dg_batch_create", "dg_batch_destroy", "dg_batch_size", "dg_batch_trace", "dg_batch_trace_gfd", "dg_batch_ep_backward", "dg_batch_gfd",
]


class DgError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERR_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.klass = ERR_NAMES.get(code, str(code))
        self.msg = msg
        self.index = -1


class TraceCfg(C.Structure):
    _fields_ = [("max_steps", C.c_int32), ("hole_avoidance", C.c_uint8), ("want_transport_matrix", C.c_uint8),
                ("use_f32", C.c_uint8), ("lane", C.c_uint8), ("memory", C.c_uint8), ("sort_by_face", C.c_uint8),
                ("refill_min", C.c_uint8), ("blocks_per_sm", C.c_uint8), ("walker", C.c_uint8),
                ("reserved", C.c_uint8 * 3), ("stream", C.c_void_p)]


class TraceIn(C.Structure):
    _fields_ = [("face", C.c_void_p), ("bary", C.c_void_p), ("dir", C.c_void_p), ("payload", C.c_void_p)]


class TraceOut(C.Structure):
    _fields_ = [("face", C.c_void_p), ("bary", C.c_void_p), ("dir", C.c_void_p), ("traced", C.c_void_p),
                ("requested", C.c_void_p), ("term", C.c_void_p), ("status", C.c_void_p), ("stall", C.c_void_p),
                ("payload", C.c_void_p), ("transport", C.c_void_p), ("npoints", C.c_void_p),
                ("crossings", C.c_void_p), ("total_crossings", C.c_void_p), ("poly_offsets", C.c_void_p),
                ("poly_total", C.c_int64), ("poly_face", C.c_void_p), ("poly_bary", C.c_void_p),
                ("poly_seg", C.c_void_p)]


class Polylines(C.Structure):
    _fields_ = [("total", C.c_int64), ("offsets", C.POINTER(C.c_int64)), ("face", C.POINTER(C.c_int32)),
                ("bary", C.POINTER(C.c_double)), ("seg", C.POINTER(C.c_double))]


class DiffCfg(C.Structure):
    _fields_ = [("memory", C.c_uint8), ("lane", C.c_uint8), ("schedule", C.c_uint8), ("reserved", C.c_uint8 * 5), ("stream", C.c_void_p),
                ("max_steps", C.c_int32)]


_lib = None


def lib():
    """Loads the shared library; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                              f"g.build()'` or `make -C paper_2603_15780_b200/csrc` (there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.dg_last_error.restype = C.c_char_p
        L.dg_version.restype = C.c_char_p
        L.dg_mesh_device_bytes.restype = C.c_int64
        L.dg_mesh_destroy.restype = None
        L.dg_mesh_destroy.argtypes = [C.c_void_p]
        for name in ("dg_mesh_face_count", "dg_mesh_vertex_count", "dg_mesh_device_bytes", "dg_mesh_device"):
            getattr(L, name).argtypes = [C.c_void_p]
        vp, i32, i64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_double
        L.dg_set_devices.argtypes = [C.c_uint64]
        L.dg_set_device_list.argtypes = [vp, i32]
        L.dg_mesh_device_count.argtypes = [vp]
        L.dg_trim.argtypes = [vp]
        L.dg_mesh_derive.argtypes = [vp, i32, vp, i32] + [vp] * 11
        L.dg_mesh_create.argtypes = [vp, i32, vp, i32] + [vp] * 7
        L.dg_mesh_create_ex.argtypes = [vp, i32, vp, i32] + [vp] * 6 + [C.c_uint32, vp]
        L.dg_mesh_has_transport_cache.argtypes = [vp]
        L.dg_mesh_uses_tma_gather.argtypes = [vp]
        L.dg_mesh_gather_mode.argtypes = [vp]
        L.dg_trace_batch.argtypes = [vp, i64, vp, vp, vp]
        L.dg_trace_plan.argtypes = [vp, i64, vp, vp, vp]
        L.dg_trace_polylines.argtypes = [vp, i64, vp, vp, vp, vp]
        L.dg_transition.argtypes = [vp, C.c_int, i64, vp, vp, vp, vp, C.c_int] + [vp] * 8
        L.dg_ep_jacobians.argtypes = [vp, i64] + [vp] * 10
        L.dg_ep_backward.argtypes = [vp, i64] + [vp] * 9
        L.dg_gfd_jacobians.argtypes = [vp, i64, vp, vp, vp, dbl, dbl] + [vp] * 12
        L.dg_gfd_jacobians_with_base.argtypes = [vp, i64] + [vp] * 8 + [dbl, dbl] + [vp] * 9
        L.dg_trace_gfd.argtypes = [vp, i64, vp, vp, vp, dbl, dbl] + [vp] * 7
        L.dg_gfd_pullback.argtypes = [vp, i64] + [vp] * 9
        L.dg_batch_trace_gfd.argtypes = [vp, i64, vp, vp, dbl, dbl, vp]
        L.dg_trace_kernel_info.argtypes = [C.c_int, C.c_int, vp, vp, vp]
        L.dg_trace_kernel_info.restype = None
        L.dg_batch_create.argtypes = [vp, i64, vp]
        L.dg_batch_destroy.argtypes = [vp]
        L.dg_batch_destroy.restype = None
        L.dg_batch_size.argtypes = [vp]
        L.dg_batch_size.restype = i64
        L.dg_batch_trace.argtypes = [vp, i64, vp, vp, vp]
        L.dg_batch_ep_backward.argtypes = [vp] * 5
        L.dg_batch_gfd.argtypes = [vp, dbl, dbl, vp, i32] + [vp] * 6
        _lib = L
    return _lib


def check(rc, index=None):
    if rc != DG_OK:
        e = DgError(rc, lib().dg_last_error().decode())
        if index is not None:
            e.index = index.value
        raise e


def ptr(a):
    """Raw address of a numpy array, a torch tensor, or None."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("ptr(): array is not C-contiguous")
        return a.ctypes.data
    if not a.is_contiguous():  # torch.Tensor
        raise ValueError("ptr(): tensor is not contiguous")
    return a.data_ptr()


def device_count() -> int:
    return lib().dg_device_count()


def require_device():
    if device_count() == 0:
        raise DgError(DG_ERR_NO_DEVICE, "no usable CUDA device: there is no CPU fallback")
