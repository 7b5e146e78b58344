"""Exact nearest-neighbour queries on the GPU.

Replaces the reference's ``scipy.spatial.cKDTree`` uses on the field-expansion
path: ``SpatialIndex`` / ``filter_new_points`` (field.py:111-151),
``median_nn_spacing`` (field.py:154-161) and the 3-NN scale init of
``insert_points`` (field.py:279-289).  Distances are float64, computed by the
``ssr_knn`` kernel on a dense uniform grid (exact, not approximate: the novelty
filter's contract needs exact distances).
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import _lib
from .errors import InvalidParameter

MAX_CELLS = 1 << 24


def _as_points(x, dev) -> torch.Tensor:
    t = torch.as_tensor(x if torch.is_tensor(x) else np.asarray(x, dtype=np.float64))
    return t.to(device=dev, dtype=torch.float64).reshape(-1, 3).contiguous()


def knn_distances(pool, queries, k: int) -> torch.Tensor:
    """(n_q, k) ascending float64 distances from each query to its k nearest pool points."""
    dev = _lib.require_cuda()
    pool = _as_points(pool, dev)
    queries = _as_points(queries, dev)
    n, nq = pool.shape[0], queries.shape[0]
    out = torch.empty((nq, k), dtype=torch.float64, device=dev)
    if nq == 0:
        return out
    both = torch.cat([pool, queries]) if n else queries
    lo = both.min(dim=0).values
    hi = both.max(dim=0).values
    lo_h, hi_h = lo.cpu().numpy(), hi.cpu().numpy()
    ext = np.maximum(hi_h - lo_h, 1e-9)
    # about two pool points per cell for uniform data, capped at MAX_CELLS
    h = float(np.cbrt(np.prod(ext) / max(n / 2.0, 1.0)))
    h = max(h, float(ext.max()) / 1024.0, 1e-12)
    while True:
        dims = np.maximum(np.ceil(ext / h).astype(np.int64), 1)
        if int(np.prod(dims)) <= MAX_CELLS:
            break
        h *= 1.26
    grid = (ctypes.c_double * 4)(float(lo_h[0]), float(lo_h[1]), float(lo_h[2]), h)
    cdims = (ctypes.c_int32 * 3)(*(int(d) for d in dims))
    ws = torch.empty(_lib.query("ssr_knn_workspace", n, int(np.prod(dims))), dtype=torch.uint8, device=dev)
    _lib.call("ssr_knn", pool.data_ptr() if n else None, n, queries.data_ptr(), nq, int(k), grid, cdims,
              out.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_ptr())
    return out


class SpatialIndex:
    """Exact nearest-neighbour distances over a fixed point set (field.py:111-136)."""

    def __init__(self, points):
        self._dev = _lib.require_cuda()
        self._pts = _as_points(points, self._dev)

    def __len__(self):
        return int(self._pts.shape[0])

    def min_distance(self, queries) -> torch.Tensor:
        q = _as_points(queries, self._dev)
        if len(self) == 0:
            return torch.full((q.shape[0],), math.inf, dtype=torch.float64, device=self._dev)
        return knn_distances(self._pts, q, 1)[:, 0]


def filter_new_points(existing: SpatialIndex, candidates, threshold):
    """Candidates strictly farther than ``threshold`` from every existing point (field.py:139-151)."""
    if threshold <= 0:
        raise InvalidParameter(f"novelty threshold must be positive, got {threshold}")
    if not candidates:
        return []
    pos = np.stack([c.position for c in candidates])
    dist = existing.min_distance(pos).cpu().numpy()
    return [c for c, d in zip(candidates, dist) if d > threshold]


def median_nn_spacing(points) -> float:
    """Median nearest-neighbour distance within a point set (field.py:154-161)."""
    dev = _lib.require_cuda()
    pts = _as_points(points, dev)
    if pts.shape[0] < 2:
        return 0.0
    d = knn_distances(pts, pts, 2)[:, 1]
    return float(torch.quantile(d, 0.5)) if d.numel() <= 16_000_000 else float(np.median(d.cpu().numpy()))


def mean_knn_scale(existing_positions, new_positions) -> torch.Tensor:
    """field.py:279-289: mean distance of each new point to its 3 nearest in
    (existing centres + new points), floored at 1e-7; 0.1 for a lone point."""
    dev = _lib.require_cuda()
    new = _as_points(new_positions, dev)
    ex = _as_points(existing_positions, dev) if existing_positions is not None else new[:0]
    pool = torch.cat([ex, new])
    n_new = new.shape[0]
    if pool.shape[0] > 1:
        k = min(4, pool.shape[0])
        d = knn_distances(pool, new, k)
        # column 0 is the point itself (distance 0)
        return torch.clamp(d[:, 1:].mean(dim=1), min=1e-7)
    return torch.full((n_new,), 0.1, dtype=torch.float64, device=dev)
