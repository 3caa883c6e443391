"""Sphere gradient-check harness over the GPU path: a host driver with the
protocol of the reference's run_gradcheck (proj/src/gradcheck.cpp:46-131) -- deterministic
samples, forward batch, EP or GFD Jacobians, pullback of |Exp - q|^2, comparison with the
closed-form sphere gradients -- issuing ONE batched forward call and ONE batched backward call
instead of the reference's per-sample loop. The sampler reproduces the reference's Rng
(xoshiro256** seeded by splitmix64, geometry.hpp:146-185) and its draw order, so a report is
comparable number for number with the reference's for the same (mesh, n, seed)."""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

_M = (1 << 64) - 1


class Rng:
    """geometry.hpp:146-185."""

    def __init__(self, seed: int):
        s = seed & _M
        st = []
        for _ in range(4):
            s = (s + 0x9E3779B97F4A7C15) & _M
            z = s
            z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M
            z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M
            st.append(z ^ (z >> 31))
        self.s = st

    @staticmethod
    def _rotl(x, k):
        return ((x << k) | (x >> (64 - k))) & _M

    def next_u64(self):
        s0, s1, s2, s3 = self.s
        result = (self._rotl((s1 * 5) & _M, 7) * 9) & _M
        t = (s1 << 17) & _M
        s2 ^= s0
        s3 ^= s1
        s1 ^= s2
        s0 ^= s3
        s2 ^= t
        s3 = self._rotl(s3, 45)
        self.s = [s0, s1, s2, s3]
        return result

    def uniform(self, lo=None, hi=None):
        u = float(self.next_u64() >> 11) * 2.0 ** -53
        return u if lo is None else lo + (hi - lo) * u


def sample_surface_point(mesh, cum_area, rng):
    """io.cpp:168-182 (first face whose running area reaches the pick; sqrt trick)."""
    pick = rng.uniform() * mesh.total_area
    f = int(np.searchsorted(cum_area, pick, side="left"))
    f = min(f, mesh.nf - 1)
    r1 = math.sqrt(rng.uniform())
    r2 = rng.uniform()
    return f, np.array([1.0 - r1, r1 * (1.0 - r2), r1 * r2])


def _unit(v):
    n = math.sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2])
    return v / n if n > 0 else v * 0.0


def sample_tangent(mesh, f, rng, min_len, max_len):
    """io.cpp:184-197."""
    c = mesh.tri[f]
    n = mesh.fnormal[f]
    t1 = _unit(mesh.xyz[c[1]] - mesh.xyz[c[0]])
    t1 = _unit(t1 - n * (t1[0] * n[0] + t1[1] * n[1] + t1[2] * n[2]))
    t2 = np.cross(n, t1)
    phi = 2.0 * math.pi * rng.uniform()
    ln = rng.uniform(min_len, max_len)
    return (t1 * math.cos(phi) + t2 * math.sin(phi)) * ln


def random_unit(rng):
    z = rng.uniform(-1.0, 1.0)
    phi = 2.0 * math.pi * rng.uniform()
    r = math.sqrt(max(0.0, 1.0 - z * z))
    return np.array([r * math.cos(phi), r * math.sin(phi), z])


def draw_samples(mesh, n, seed, min_len, max_len, with_targets=True):
    rng = Rng(seed)
    cum = np.cumsum(mesh.farea)
    face = np.empty(n, np.int32)
    bary, v, q = np.empty((n, 3)), np.empty((n, 3)), np.empty((n, 3))
    for i in range(n):
        face[i], bary[i] = sample_surface_point(mesh, cum, rng)
        v[i] = sample_tangent(mesh, face[i], rng, min_len, max_len)
        if with_targets:
            q[i] = random_unit(rng)
    return face, bary, v, q


@dataclass
class GradCheckReport:
    scheme: str
    median_cos_v: float
    median_norm_ratio_v: float
    median_cos_p: float
    median_norm_ratio_p: float
    max_p_grad_norm: float
    cos_v: np.ndarray
    cos_p: np.ndarray


def _rows(a):
    return np.linalg.norm(a, axis=1)


def _median(x):
    x = x[np.isfinite(x)]
    return float(np.median(x)) if len(x) else float("nan")


def sphere_closed_form(p_s, v_s, q):
    """Closed-form pulled-back gradients of |Exp_p(v) - q|^2 on the unit sphere
    (sphere_exp / sphere_jacobians, oracles.cpp:10-40; Jacobi fields for the start point)."""
    ln = _rows(v_s)[:, None]
    c, s = np.cos(ln), np.sin(ln)
    y = p_s * c + v_s * (s / ln)
    g = 2.0 * (y - q)
    # J_v^T g with J_v = [(I - p v^T)/|v| - v v^T/|v|^3] sin|v| + v v^T/|v|^2 cos|v|
    vg = np.einsum("nd,nd->n", v_s, g)[:, None]
    pg = np.einsum("nd,nd->n", p_s, g)[:, None]
    jt_g = (g - v_s * pg) / ln * s - v_s * vg / ln ** 3 * s + v_s * vg / ln ** 2 * c
    cf_v = jt_g - p_s * np.einsum("nd,nd->n", jt_g, p_s)[:, None]
    v_par = v_s / ln
    e_perp = np.cross(p_s, v_par)
    gamma_dot = -p_s * s + v_par * c
    cf_p = v_par * np.einsum("nd,nd->n", g, gamma_dot)[:, None] + e_perp * (c * np.einsum("nd,nd->n", g, e_perp)[:, None])
    return cf_v, cf_p


def run_gradcheck(mesh, scheme: str, n: int, seed: int, min_len: float, max_len: float) -> GradCheckReport:
    face, bary, v, q = draw_samples(mesh, n, seed, min_len, max_len)
    base = mesh.trace_batch(face, bary, v)                       # one batched forward launch
    y = mesh.embed(base.face, base.bary)
    g = 2.0 * (y - q)
    if scheme == "gfd":
        out = mesh.gfd(face, bary, v, g=g)                       # two batched rounds
        grad_v, grad_p = out["grad_v"], out["grad_p"]
    else:
        grad_v = mesh.ep_backward(face, v, base.face, base.dir, g)   # one fused launch
        grad_p = np.zeros_like(grad_v)
    p0 = mesh.embed(face, bary)
    p_s = p0 / _rows(p0)[:, None]
    v_t = v - p_s * np.einsum("nd,nd->n", v, p_s)[:, None]
    v_s = v_t / _rows(v_t)[:, None] * _rows(v)[:, None]
    cf_v, cf_p = sphere_closed_form(p_s, v_s, q)

    def cosine(a, b):
        na, nb = _rows(a), _rows(b)
        with np.errstate(invalid="ignore", divide="ignore"):
            return np.where((na > 0) & (nb > 0), np.einsum("nd,nd->n", a, b) / (na * nb), np.nan)
    with np.errstate(invalid="ignore", divide="ignore"):
        ratio_v = np.where(_rows(cf_v) > 0, _rows(grad_v) / _rows(cf_v), np.nan)
        ratio_p = np.where(_rows(cf_p) > 0, _rows(grad_p) / _rows(cf_p), np.nan)
    cv, cp = cosine(grad_v, cf_v), cosine(grad_p, cf_p)
    return GradCheckReport(scheme, _median(cv), _median(ratio_v), _median(cp), _median(ratio_p),
                           float(_rows(grad_p).max()), cv, cp)
