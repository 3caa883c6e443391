"""Multi-GPU plumbing: one process per GPU, mesh replicated, query batch sharded.

The path has no exchange step: queries are independent and the mesh is read-only,
so every rank traces a contiguous slice of the request and the SoA results are gathered at the
request index -- no reduction. Slices are cut by equal expected work (weight = requested
length, a proxy for the number of face crossings), not by equal counts. `torch.distributed` is
only the plumbing: NCCL over NVLink on the GPU box, gloo in the CPU tests.
"""
from __future__ import annotations

import numpy as np


def shard_bounds(weights, world: int) -> np.ndarray:
    """Cut points b[0..world] of `world` contiguous slices with (nearly) equal total weight.
    Deterministic and independent of the rank that evaluates it."""
    w = np.asarray(weights, dtype=np.float64)
    n = len(w)
    if world <= 1 or n == 0:
        return np.array([0] + [n] * max(world, 1), dtype=np.int64)
    c = np.cumsum(np.maximum(w, 0.0))
    total = c[-1]
    if not np.isfinite(total) or total <= 0:
        return np.linspace(0, n, world + 1).round().astype(np.int64)
    cuts = np.searchsorted(c, total * np.arange(1, world) / world, side="left") + 1
    b = np.concatenate([[0], np.minimum(cuts, n), [n]]).astype(np.int64)
    return np.maximum.accumulate(b)


def my_slice(weights, rank: int, world: int) -> slice:
    b = shard_bounds(weights, world)
    return slice(int(b[rank]), int(b[rank + 1]))


def gather_rows(local, bounds, dist, device=None):
    """All-gathers ragged row blocks (one per rank, in rank order) into the full array at the
    request index. `local`: torch tensor [n_r, ...]; returns a tensor [n, ...] on every rank."""
    import torch
    world = dist.get_world_size()
    sizes = [int(bounds[r + 1] - bounds[r]) for r in range(world)]
    pad = max(sizes) if sizes else 0
    shape = (pad,) + tuple(local.shape[1:])
    buf = torch.zeros(shape, dtype=local.dtype, device=local.device)
    buf[: local.shape[0]] = local
    out = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(out, buf)
    return torch.cat([o[:s] for o, s in zip(out, sizes)], dim=0)


def trace_sharded(trace_fn, face, bary, dirs, dist=None, to_tensor=None):
    """Runs `trace_fn(face, bary, dirs) -> dict of per-query numpy arrays` on this rank's slice and
    gathers every output at the request index. With dist=None (single process) it is the identity
    wrapper. The mesh handle lives inside trace_fn (one replica per rank)."""
    import torch
    n = len(face)
    if dist is None or dist.get_world_size() == 1:
        return trace_fn(face, bary, dirs)
    rank, world = dist.get_rank(), dist.get_world_size()
    weights = np.linalg.norm(np.asarray(dirs, float).reshape(n, 3), axis=1)
    bounds = shard_bounds(weights, world)
    sl = slice(int(bounds[rank]), int(bounds[rank + 1]))
    local = trace_fn(face[sl], bary[sl], dirs[sl])
    to_tensor = to_tensor or (lambda a: torch.from_numpy(np.ascontiguousarray(a)))
    out = {}
    for k in sorted(local):
        g = gather_rows(to_tensor(local[k]), bounds, dist)
        out[k] = g.cpu().numpy()
    return out
