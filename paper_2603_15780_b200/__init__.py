"""B200-native batched straightest-geodesic exponential map and its EP / GFD differentials.

Python surface over libdigeo_b200.so (hand-written sm_100a CUDA behind a C-ABI). Importing the
package loads the shared library and raises if it has not been built: there is no CPU path.
"""
from . import capi
from .api import Batch, Mesh, TraceResult, kernel_info
from .capi import DgError, device_count

capi.lib()  # fail loudly at import time when the native library is absent

__all__ = ["Batch", "Mesh", "TraceResult", "DgError", "device_count", "kernel_info", "capi"]
