"""Training objective on device (mirrors losses.py:37-182 of the reference).

``total_loss`` runs the fused L1 + (1 - SSIM) + load-balance kernels and
returns device gradients; the scalar terms stay in a device buffer until read
(reading a property synchronises), so a training loop needs no host round
trip per iteration.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from . import _lib
from .errors import InvalidParameter


@dataclass
class LossWeights:
    l1: float = 0.47
    ssim: float = 0.12
    load: float = 0.41

    def __post_init__(self):
        for name in ("l1", "ssim", "load"):
            v = getattr(self, name)
            if not math.isfinite(v) or v < 0:
                raise InvalidParameter(f"loss weight {name} must be finite and >= 0, got {v}")


class LossBreakdown:
    """d_image (H,W,3) / d_soft (H,W) device tensors plus lazily-read scalars."""

    def __init__(self, values: torch.Tensor, d_image: torch.Tensor, d_soft: torch.Tensor, ready=None):
        self.values = values  # float64 (device, or pinned host): l1, ssim_loss, load, total, hard_count_std
        self.d_image = d_image
        self.d_soft = d_soft
        self._ready = ready  # event after the write when values is pinned host memory
        self._host = None

    def _get(self, i):
        if self._host is None:
            if self._ready is not None:
                self._ready.synchronize()
            self._host = self.values.cpu().tolist()
        return float(self._host[i])

    l1 = property(lambda s: s._get(0))
    ssim_loss = property(lambda s: s._get(1))
    load = property(lambda s: s._get(2))
    total = property(lambda s: s._get(3))
    hard_count_std = property(lambda s: s._get(4))


class _Workspace:
    cache = {}

    @classmethod
    def get(cls, w, h, dev):
        key = (w, h, str(dev))
        if key not in cls.cache:
            cls.cache[key] = torch.empty(_lib.query("ssr_loss_workspace", w, h), dtype=torch.uint8, device=dev)
        return cls.cache[key]


def total_loss(rendered, target, output, weights: LossWeights, values_out: torch.Tensor | None = None
               ) -> LossBreakdown:
    """Weighted objective over one rendered view (losses.py:147-173).

    ``target`` is float in [0, 1] or uint8 (value / 255, as the reference's
    io/images.py loads its 8-bit image files).  ``values_out`` (optional): a
    pinned host float64 tensor of 5 the kernel writes the scalar terms into
    directly (mapped host memory), so reading them back needs no copy on the
    stream; the breakdown's properties wait for that write."""
    rendered = torch.as_tensor(rendered)
    target = torch.as_tensor(target)
    if tuple(rendered.shape) != tuple(target.shape) or rendered.dim() != 3 or rendered.shape[2] != 3:
        raise InvalidParameter(f"shape mismatch {tuple(rendered.shape)} vs {tuple(target.shape)}")
    h, w = int(rendered.shape[0]), int(rendered.shape[1])
    if h < 11 or w < 11:
        raise InvalidParameter(f"image {h}x{w} smaller than the 11-tap SSIM window")
    dev = output.image.device
    x = rendered.to(device=dev, dtype=torch.float32).contiguous()
    # an 8-bit target (the reference's image files; value / 255) is read as is
    u8 = target.dtype == torch.uint8
    y = target.to(device=dev).contiguous() if u8 else target.to(device=dev, dtype=torch.float32).contiguous()
    if output.soft_count is None:
        # render(soft_count=False): only a loss without the load term can use it
        if weights.load > 0:
            raise InvalidParameter("the load-balance term needs soft counts; render with soft_count=True")
        soft = None
    else:
        soft = output.soft_count.to(dtype=torch.float64).contiguous()
    hard = output.hard_count.to(dtype=torch.int32).contiguous()
    d_image = torch.empty_like(x)
    d_soft = None if soft is None else torch.empty(soft.shape, dtype=torch.float32, device=dev)
    if values_out is not None:
        if values_out.device.type != "cpu" or not values_out.is_pinned() or values_out.dtype != torch.float64 \
                or values_out.numel() < 5 or not values_out.is_contiguous():
            raise InvalidParameter("values_out must be a contiguous pinned host float64 tensor of >= 5 elements")
        vals = values_out
    else:
        vals = torch.empty(5, dtype=torch.float64, device=dev)
    ws = _Workspace.get(w, h, dev)
    _lib.call("ssr_loss", w, h, x.data_ptr(), y.data_ptr(), 1 if u8 else 0, _lib.ptr(soft), hard.data_ptr(),
              float(weights.l1),
              float(weights.ssim), float(weights.load), d_image.data_ptr(), _lib.ptr(d_soft), vals.data_ptr(),
              ws.data_ptr(), ws.numel(), _lib.stream_ptr())
    ready = None
    if values_out is not None:
        ready = torch.cuda.Event()
        ready.record()
    return LossBreakdown(vals, d_image, d_soft, ready)


def psnr(rendered, target) -> float:
    rendered = torch.as_tensor(rendered).double()
    target = torch.as_tensor(target).to(rendered.device).double()
    mse = float(((rendered - target) ** 2).mean())
    return float("inf") if mse == 0.0 else -10.0 * math.log10(mse)
