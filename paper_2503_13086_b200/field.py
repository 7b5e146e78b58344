"""GPU-resident Gaussian field (mirrors field.py:164-375 of the reference).

Parameters live in ONE flat float32 CUDA buffer, class-major:
``[positions 3N | rotations 4N | log_scales 3N | opacity_logits N | sh 3KN]``.
The reference attribute names (``positions``, ``rotations``, ``log_scales``,
``opacity_logits``, ``sh``) are views into it with the reference shapes
((N,3), (N,4), (N,3), (N,), (N,3,K) channel-major).  ``generation`` counts
structural changes exactly like the reference so stale renders are rejected.
"""

from __future__ import annotations

import ctypes
import hashlib
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import InvalidParameter

SH_C0 = 0.28209479177387814
CLASSES = ("positions", "rotations", "log_scales", "opacity_logits", "sh")


def row_floats(sh_degree: int) -> int:
    """Parameter floats per Gaussian: 11 + 3K (59 at SH3)."""
    return 11 + 3 * (sh_degree + 1) ** 2


def row_stride(n: int) -> int:
    """Rows reserved per class region: n rounded up to a multiple of 4, so every
    class starts 16-byte aligned (float4 / TMA paths) for any n (ssr_common.cuh)."""
    return (int(n) + 3) & ~3


def class_slices(n: int, k: int):
    """(start, width) of each class inside the flat buffer of n rows."""
    w = (3, 4, 3, 1, 3 * k)
    ns = row_stride(n)
    out, off = [], 0
    for wi in w:
        out.append((off, wi))
        off += wi * ns
    return out


def flat_size(n: int, k: int, extra: int = 0) -> int:
    """Floats of a flat buffer of n rows: the 5 classes (+ ``extra`` 1-wide regions)."""
    return (11 + 3 * k + extra) * row_stride(n)


def alloc_growing(numel: int, device, dtype=torch.float32) -> torch.Tensor:
    """Uninitialised 1-D buffer of ``numel`` elements whose allocation is rounded
    up to 1/16 of the size's leading power of two, so a buffer that grows by a
    little every event (field expansion) reuses the block its predecessor
    freed instead of a fresh device allocation each time."""
    step = 1 << max(20, int(numel).bit_length() - 4)
    cap = (int(numel) + step - 1) // step * step
    return torch.empty(cap, dtype=dtype, device=device)[:numel]


def pack_classes(parts, n: int, k: int, device, dtype=torch.float32) -> torch.Tensor:
    """Flat, padded class-major buffer from the five class arrays (each n rows)."""
    flat = torch.zeros(flat_size(n, k), dtype=dtype, device=device)
    for (off, w), part in zip(class_slices(n, k), parts):
        flat[off: off + w * n] = part.reshape(-1).to(device=device, dtype=dtype)
    return flat


@dataclass
class DensifyOptions:
    grad_threshold: float = 2e-4
    percent_dense: float = 0.01
    scene_extent: float = 1.0
    prune_opacity: float = 0.005
    split_scale_shrink: float = 1.6


@dataclass
class DensifySummary:
    cloned: int
    split: int
    pruned: int
    keep_mask: np.ndarray  # over the pre-call rows; False = removed
    n_added: int

    @property
    def changed(self) -> bool:
        return self.cloned > 0 or self.split > 0 or self.pruned > 0


@dataclass
class SparsePoint:
    position: np.ndarray
    color: np.ndarray

    def __post_init__(self):
        self.position = np.asarray(self.position, dtype=np.float64).reshape(3)
        self.color = np.asarray(self.color, dtype=np.float64).reshape(3)

    @property
    def finite(self) -> bool:
        return bool(np.isfinite(self.position).all() and np.isfinite(self.color).all())


class GaussianField:
    """Growable set of Gaussians stored struct-of-arrays in one flat CUDA buffer."""

    def __init__(self, sh_degree: int = 0, device=None):
        if not 0 <= sh_degree <= 3:
            raise InvalidParameter(f"sh_degree must be in 0..3, got {sh_degree}")
        self.sh_degree = int(sh_degree)
        self.device = _lib.require_cuda() if device is None else torch.device(device)
        self._n = 0
        self._flat = torch.zeros(0, dtype=torch.float32, device=self.device)
        self.generation = 0
        # bumped by every in-place parameter update (optimizer steps, assignment);
        # a projection's lazily computed aux fields check it (ProjectedSplats._aux)
        self.version = 0

    # ------------------------------------------------------------ construction
    @classmethod
    def from_arrays(cls, positions, rotations, log_scales, opacity_logits, sh, device=None) -> "GaussianField":
        sh_t = torch.as_tensor(np.asarray(sh) if not torch.is_tensor(sh) else sh)
        k = sh_t.shape[2]
        deg = int(round(math.sqrt(k))) - 1
        f = cls(sh_degree=deg, device=device)
        arrs = [torch.as_tensor(a if torch.is_tensor(a) else np.asarray(a)) for a in
                (positions, rotations, log_scales, opacity_logits, sh)]
        n = arrs[0].shape[0]
        if sum(a.numel() for a in arrs) != n * row_floats(deg):
            raise InvalidParameter("parameter arrays have inconsistent shapes")
        f._flat = pack_classes(arrs, n, k, f.device)
        f._n = n
        return f

    @classmethod
    def from_host(cls, hp, device=None) -> "GaussianField":
        """From a scenes.HostParams / any object with the five attributes."""
        return cls.from_arrays(*(getattr(hp, k) for k in CLASSES), device=device)

    # ------------------------------------------------------------ views
    def __len__(self):
        return self._n

    @property
    def n_sh_coeffs(self) -> int:
        return (self.sh_degree + 1) ** 2

    @property
    def flat(self) -> torch.Tensor:
        return self._flat

    def _view(self, i):
        n, k = self._n, self.n_sh_coeffs
        off, w = class_slices(n, k)[i]
        v = self._flat[off: off + w * n]
        shape = ((n, 3), (n, 4), (n, 3), (n,), (n, 3, k))[i]
        return v.view(shape)

    def _assign(self, i, value):
        dst = self._view(i)
        src = torch.as_tensor(value if torch.is_tensor(value) else np.asarray(value))
        if tuple(src.shape) != tuple(dst.shape):
            raise InvalidParameter(f"{CLASSES[i]} must have shape {tuple(dst.shape)}, got {tuple(src.shape)}")
        dst.copy_(src.to(dtype=torch.float32))
        self.version += 1

    positions = property(lambda s: s._view(0), lambda s, v: s._assign(0, v))
    rotations = property(lambda s: s._view(1), lambda s, v: s._assign(1, v))
    log_scales = property(lambda s: s._view(2), lambda s, v: s._assign(2, v))
    opacity_logits = property(lambda s: s._view(3), lambda s, v: s._assign(3, v))
    sh = property(lambda s: s._view(4), lambda s, v: s._assign(4, v))

    def opacities(self):
        return torch.sigmoid(self.opacity_logits)

    def scales(self):
        return torch.exp(self.log_scales)

    def covariances(self):
        """Sigma = R S S^T R^T per Gaussian (field.py:71-75), float64."""
        q = self.rotations.double()
        q = q / q.norm(dim=1, keepdim=True)
        w, x, y, z = q.unbind(1)
        r = torch.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                         2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                         2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], 1).view(-1, 3, 3)
        m = r * torch.exp(self.log_scales.double())[:, None, :]
        return m @ m.transpose(1, 2)

    def to_numpy(self) -> dict:
        return {k: getattr(self, k).detach().cpu().numpy() for k in CLASSES}

    def checksum(self) -> str:
        h = hashlib.sha256()
        for k in CLASSES:
            h.update(np.ascontiguousarray(getattr(self, k).detach().cpu().numpy()).tobytes())
        return h.hexdigest()

    def _check_finite(self):
        # real rows only: the up-to-3 padding rows per class region are not parameters
        if not all(bool(torch.isfinite(self._view(i)).all()) for i in range(len(CLASSES))):
            raise InvalidParameter("non-finite values in field parameters")

    # ------------------------------------------------------------ structure
    def insert_points(self, points, init_opacity: float = 0.1) -> int:
        """Append one Gaussian per sparse point (field.py:258-301).

        Scale init = mean distance to the 3 nearest points of the union of the
        existing centres and the new points (exact k-NN on the GPU grid index,
        spatial.py); identity rotation; logit(init_opacity); DC from colour.
        """
        usable = [p for p in points if p.finite]
        if not usable:
            return 0
        return self.insert_arrays(np.stack([p.position for p in usable]), np.stack([p.color for p in usable]),
                                  init_opacity)

    def insert_arrays(self, positions, colors, init_opacity: float = 0.1) -> int:
        """insert_points for (n, 3) position / colour arrays (host or device);
        rows with a non-finite value are skipped like non-finite SparsePoints."""
        from .spatial import mean_knn_scale

        dev = self.device
        as_t = lambda x: (x if torch.is_tensor(x) else torch.as_tensor(np.asarray(x, dtype=np.float64))).to(
            device=dev, dtype=torch.float64).reshape(-1, 3)
        new_pos, cols = as_t(positions), as_t(colors)
        if new_pos.shape[0] != cols.shape[0]:
            raise InvalidParameter("positions and colors must have the same number of rows")
        ok = torch.isfinite(new_pos).all(dim=1) & torch.isfinite(cols).all(dim=1)
        if not bool(ok.all()):
            new_pos, cols = new_pos[ok], cols[ok]
        n_new = int(new_pos.shape[0])
        if n_new == 0:
            return 0
        # exact 3-NN over (existing centres + new points) on the GPU grid index
        mean_d = mean_knn_scale(self.positions.double() if self._n else None, new_pos)
        K = self.n_sh_coeffs
        log_scales = torch.log(mean_d)[:, None].repeat(1, 3)
        rot = torch.zeros(n_new, 4, dtype=torch.float64, device=dev)
        rot[:, 0] = 1.0
        logit = torch.full((n_new,), math.log(init_opacity / (1.0 - init_opacity)), dtype=torch.float64, device=dev)
        sh = torch.zeros(n_new, 3, K, dtype=torch.float64, device=dev)
        sh[:, :, 0] = (cols - 0.5) / SH_C0
        self._append([new_pos, rot, log_scales, logit, sh])
        self.generation += 1
        self._check_finite()
        return n_new

    def _append(self, parts):
        """Grow the flat buffer by parts' rows (each class region copied once)."""
        n_add = parts[0].shape[0]
        n_old, k = self._n, self.n_sh_coeffs
        n_tot = n_old + n_add
        flat = alloc_growing(flat_size(n_tot, k), self.device)
        old_sl, new_sl = class_slices(n_old, k), class_slices(n_tot, k)
        for (o_off, w), (n_off, _), part in zip(old_sl, new_sl, parts):
            if n_old:
                flat[n_off: n_off + w * n_old] = self._flat[o_off: o_off + w * n_old]
            flat[n_off + w * n_old: n_off + w * n_tot] = part.reshape(-1).to(dtype=torch.float32)
            flat[n_off + w * n_tot: n_off + w * row_stride(n_tot)] = 0.0  # padding rows: no stale bytes
        self._flat = flat
        self._n = n_tot
        self.version += 1

    def densify_and_prune(self, grad_stats, opts: DensifyOptions, rng, optimizer=None) -> DensifySummary:
        """Clone/split hot Gaussians and prune transparent ones (field.py:303-375).

        ``grad_stats`` is the averaged screen-gradient statistic (N,).  Split
        children draw ``rng.standard_normal((2*n_split, 3))`` from the session
        generator on the host (field.py:340) so RNG streams stay aligned.  When
        ``optimizer`` is given its moments are remapped in the same kernel pass
        (equivalent to optimizer.sync(...)).
        """
        stats = torch.as_tensor(grad_stats if torch.is_tensor(grad_stats) else np.asarray(grad_stats))
        if stats.shape[0] != self._n:
            raise InvalidParameter(f"grad_stats length {stats.shape[0]} != field size {self._n}")
        n = self._n
        if n == 0:
            return DensifySummary(0, 0, 0, np.ones(0, dtype=bool), 0)
        stats = stats.to(device=self.device, dtype=torch.float32).contiguous()
        flags = torch.empty(n, dtype=torch.uint8, device=self.device)
        counts = torch.empty(3, dtype=torch.int32, device=self.device)
        st = _lib.stream_ptr()
        _lib.call("ssr_densify_masks", n, self._flat.data_ptr(), self.sh_degree, stats.data_ptr(),
                  float(opts.grad_threshold), float(opts.percent_dense * opts.scene_extent),
                  float(opts.prune_opacity), flags.data_ptr(), counts.data_ptr(), st)
        cl, sp, pr = (int(v) for v in counts.cpu().tolist())
        keep = (flags & 1).bool()
        keep_np = keep.cpu().numpy()
        n_added = cl + 2 * sp
        if not (cl or sp or pr):
            return DensifySummary(0, 0, 0, keep_np, 0)
        eps = torch.as_tensor(rng.standard_normal((2 * sp, 3)) if sp else np.zeros((1, 3)),
                              dtype=torch.float64).to(self.device)
        n_new = int(keep_np.sum()) + n_added
        new = torch.zeros(flat_size(n_new, self.n_sh_coeffs), dtype=torch.float32, device=self.device)
        ws = torch.empty(_lib.query("ssr_densify_workspace", n), dtype=torch.uint8, device=self.device)
        m_old = v_old = new_m = new_v = None
        if optimizer is not None:
            m_old, v_old = optimizer.m, optimizer.v
            new_m, new_v = torch.zeros_like(new), torch.zeros_like(new)
        _lib.call("ssr_densify_apply", n, n_new, self.sh_degree, self._flat.data_ptr(), _lib.ptr(m_old),
                  _lib.ptr(v_old), flags.data_ptr(), eps.data_ptr(), float(math.log(opts.split_scale_shrink)),
                  new.data_ptr(), _lib.ptr(new_m), _lib.ptr(new_v), ws.data_ptr(), ws.numel(), st)
        self._flat = new
        self._n = n_new
        self.generation += 1
        self.version += 1
        if optimizer is not None:
            optimizer._adopt(self, new_m, new_v)
        self._check_finite()
        return DensifySummary(cl, sp, pr, keep_np, n_added)
