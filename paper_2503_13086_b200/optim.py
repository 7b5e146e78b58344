"""Fused dense Adam over the flat field buffer (mirrors optim.py:17-130).

Every row is updated every step (invisible rows included), one step counter
per parameter class, positions at ``position_rate * scene_extent``, SH rest
coefficients at 1/20 of the DC rate, eps 1e-15.  m and v share the field's
flat class-major layout so one kernel pass updates all 59 floats per row.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import _lib
from .errors import InvalidParameter, StaleFieldError
from .field import CLASSES, alloc_growing, class_slices, flat_size, pack_classes, row_stride

BETA1 = 0.9
BETA2 = 0.999
EPS = 1e-15
ROTATION_LR = 1e-3
SCALE_LR = 5e-3
OPACITY_LR = 0.05
SH_DC_LR = 2.5e-3
SH_REST_LR = SH_DC_LR / 20.0


class FieldOptimizer:
    """Steps a GaussianField from FieldGrads with per-class rates."""

    def __init__(self, fld, scene_extent=1.0):
        if not (scene_extent > 0) or not math.isfinite(scene_extent):
            raise InvalidParameter(f"scene_extent must be finite and > 0, got {scene_extent}")
        self.scene_extent = float(scene_extent)
        self.m = torch.zeros_like(fld.flat)
        self.v = torch.zeros_like(fld.flat)
        self.steps = {k: 0 for k in CLASSES}
        self.n_rows = len(fld)
        self.sh_degree = fld.sh_degree
        self._generation = fld.generation

    def _moment_view(self, buf, name):
        n, k = self.n_rows, (self.sh_degree + 1) ** 2
        i = CLASSES.index(name)
        off, w = class_slices(n, k)[i]
        return buf[off: off + w * n].view(((n, 3), (n, 4), (n, 3), (n,), (n, 3, k))[i])

    def moments(self, name):
        return self._moment_view(self.m, name), self._moment_view(self.v, name)

    def _adopt(self, fld, new_m, new_v):
        self.m, self.v = new_m, new_v
        self.n_rows = len(fld)
        self._generation = fld.generation

    def sync(self, fld, keep_mask, n_added):
        """Track a densify/prune: kept rows keep their moments, new rows start cold (optim.py:101-111)."""
        keep_np = np.asarray(keep_mask, dtype=bool)
        if keep_np.all():  # pure growth (field expansion): copy the regions, new rows start cold
            self.m, self.v = self._grow(self.m, int(n_added)), self._grow(self.v, int(n_added))
            self.n_rows += int(n_added)
            self._generation = fld.generation
            if self.n_rows != len(fld):
                raise InvalidParameter(f"remap produced {self.n_rows} rows, field has {len(fld)}")
            return
        keep = torch.as_tensor(keep_np, device=self.m.device)
        n_new = int(keep.sum().item()) + int(n_added)
        newm, newv = [], []
        for name in CLASSES:
            for src, dst in ((self.m, newm), (self.v, newv)):
                mv = self._moment_view(src, name)
                kept = mv[keep]
                dst.append(torch.cat([kept, torch.zeros((int(n_added),) + tuple(mv.shape[1:]), device=mv.device)]))
        k = (self.sh_degree + 1) ** 2
        self.m, self.v = pack_classes(newm, n_new, k, self.m.device), pack_classes(newv, n_new, k, self.m.device)
        self.n_rows = n_new
        self._generation = fld.generation
        if self.n_rows != len(fld):
            raise InvalidParameter(f"remap produced {self.n_rows} rows, field has {len(fld)}")

    def _grow(self, buf, n_added):
        n, k = self.n_rows, (self.sh_degree + 1) ** 2
        n_tot = n + n_added
        out = alloc_growing(flat_size(n_tot, k), buf.device, buf.dtype)
        for (o_off, w), (n_off, _) in zip(class_slices(n, k), class_slices(n_tot, k)):
            out[n_off: n_off + w * n] = buf[o_off: o_off + w * n]
            out[n_off + w * n: n_off + w * row_stride(n_tot)] = 0.0  # new rows start cold; padding zero
        return out

    def step(self, fld, grads, position_rate):
        """Apply one update; position_rate comes from the lr scheduler (optim.py:113-130)."""
        if fld.generation != self._generation:
            raise StaleFieldError("field changed shape since the optimizer last synced")
        if tuple(grads.positions.shape) != tuple(fld.positions.shape):
            raise InvalidParameter("gradient dimensions do not match field")
        n = len(fld)
        if n == 0:
            return
        g = grads.flat_params(fld.flat.device)
        lr, bc1, bc2 = self.advance(position_rate)
        fld.version += 1
        _lib.call("ssr_adam", n, fld.sh_degree, fld.flat.data_ptr(), g.data_ptr(), self.m.data_ptr(),
                  self.v.data_ptr(), lr, SH_REST_LR, bc1, bc2, _lib.stream_ptr())

    def check(self, fld):
        if fld.generation != self._generation:
            raise StaleFieldError("field changed shape since the optimizer last synced")

    def advance(self, position_rate):
        """Count one step for every class; (lr, bc1, bc2) host arrays for the kernels."""
        for k in CLASSES:
            self.steps[k] += 1
        lr = (ctypes.c_double * 5)(position_rate * self.scene_extent, ROTATION_LR, SCALE_LR, OPACITY_LR, SH_DC_LR)
        bc1 = (ctypes.c_double * 5)(*[1.0 - BETA1 ** self.steps[k] for k in CLASSES])
        bc2 = (ctypes.c_double * 5)(*[1.0 - BETA2 ** self.steps[k] for k in CLASSES])
        return lr, bc1, bc2
