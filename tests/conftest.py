import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (HERE, ROOT):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box with `-m gpu`)")


def _ensure_built():
    import __graft_entry__ as g
    so = os.path.join(ROOT, "paper_2603_15780_b200", "lib", "libdigeo_b200.so")
    ref = os.path.join(ROOT, "oracle", "_ref", "libdigeo_ref.so")
    if not (os.path.exists(so) and os.path.exists(ref)):
        g.build()


@pytest.fixture(scope="session")
def dg():
    _ensure_built()
    import paper_2603_15780_b200 as dg
    return dg


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference behind oracle/_ref/libdigeo_ref.so (the checker)."""
    _ensure_built()
    import refapi
    if not refapi.available():
        pytest.skip("oracle/_ref/libdigeo_ref.so not built (needs /root/reference at build time)")
    return refapi


@pytest.fixture(scope="session")
def gpu(dg):
    if dg.device_count() == 0:
        pytest.fail("GPU test selected but no CUDA device is usable (there is no CPU fallback)")
    return dg


def gpu_mesh(dg, rm, transport_cache="auto"):
    """Uploads a reference-built mesh through OUR derive + create path."""
    a = rm.arrays()
    return dg.Mesh(a["xyz"], a["tri"], transport_cache=transport_cache)


def assert_trace_equal(r, h, n, check_poly=True, payload=False, q=False, exact=True, tol=1e-9):
    """r: reference result, h: ours. exact=True demands bit equality (edge-only f64 traces)."""
    for k in ("face", "term", "status", "npoints"):
        a, b = getattr(r, k), getattr(h, k)
        bad = np.nonzero(a != b)[0]
        assert len(bad) == 0, f"{k}: {len(bad)}/{n} differ, first {bad[:5]} ref={a[bad[:5]]} ours={b[bad[:5]]}"
    fields = ["bary", "dir", "traced", "requested"]
    if payload:
        fields.append("payload")
    if q:
        fields.append("q")
    for k in fields:
        a, b = getattr(r, k), getattr(h, k)
        if exact:
            same = (a == b) | (np.isnan(a) & np.isnan(b))
            bad = np.nonzero(~same.reshape(n, -1).all(1))[0]
            assert len(bad) == 0, f"{k}: {len(bad)}/{n} not bit-equal, first {bad[:5]}, max|d|={np.nanmax(np.abs(a - b))}"
        else:
            d = np.nanmax(np.abs(a - b)) if a.size else 0.0
            assert d <= tol, f"{k}: max|d|={d} > {tol}"
    if check_poly and r.poly_face is not None:
        assert np.array_equal(r.poly_face, h.poly_face), "polyline face sequence differs"
        if exact:
            assert np.array_equal(r.poly_bary, h.poly_bary), "polyline points differ"
            assert np.array_equal(r.poly_seg, h.poly_seg), "polyline segment lengths differ"
        else:
            assert np.abs(r.poly_bary - h.poly_bary).max() <= tol
            assert np.abs(r.poly_seg - h.poly_seg).max() <= tol
