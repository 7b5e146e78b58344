"""Stage 4 host wrapper: ``backward`` and ``FieldGrads`` (backward.py:28-129)."""

from __future__ import annotations

import threading

import numpy as np
import torch

from .. import _lib
from ..errors import InvalidParameter, StaleFieldError
from ..field import class_slices, flat_size, pack_classes, row_stride
from .forward import RenderOutput

LAYOUTS = {"splat": 0, "pixel": 1}

_ROWS: dict = {}


_LISTS: dict = {}


def _row_list(dev, n: int) -> torch.Tensor:
    """N + 1 uint32 of scratch for ssr_chain's visible-row list (per device,
    stream and host thread, like the rows workspace; grown on demand)."""
    key = (dev.index if dev.index is not None else torch.cuda.current_device(), _lib.stream_ptr(),
           threading.get_ident())
    buf = _LISTS.get(key)
    if buf is None or buf.numel() < n + 1:
        buf = torch.empty(n + 1 + (n + 1) // 8, dtype=torch.int32, device=dev)
        _LISTS[key] = buf
    return buf


def rows_workspace(dev, m: int) -> torch.Tensor:
    """The ``inst_rows`` workspace of ssr_backward / ssr_chain (include/ssr.h)
    for the current device, stream and host thread: zero-filled when (re)allocated, then
    reused by every call -- its generation tags mark which rows the last
    backward wrote, so rows of unwalked slots are never zero-filled."""
    need = int(_lib.load().ssr_rows_floats(m))
    # one per device, stream and host thread: a backward and its chain are
    # separate calls, so calls of two threads on one stream must not share it
    key = (dev.index if dev.index is not None else torch.cuda.current_device(), _lib.stream_ptr(),
           threading.get_ident())
    buf = _ROWS.get(key)
    if buf is None or buf.numel() < need:
        _ROWS.pop(key, None)
        buf = torch.zeros(need + need // 8, dtype=torch.float32, device=dev)
        _ROWS[key] = buf
    return buf


class FieldGrads:
    """Gradients aligned with the field's parameter arrays.

    When produced by ``backward`` every array is a view into one flat buffer
    ``[pos 3N | rot 4N | logscale 3N | logit N | sh 3KN | screen_norms N |
    visible N]`` (the allreduce unit of view-sharded batches); constructed
    from arrays it packs them lazily for the optimizer.
    """

    def __init__(self, positions=None, rotations=None, log_scales=None, opacity_logits=None, sh=None,
                 screen_norms=None, visible=None, *, _flat=None, _n=None, _k=None):
        if _flat is not None:
            self._flat, self._n, self._k = _flat, _n, _k
            return
        self._flat = None
        self._arrays = dict(positions=positions, rotations=rotations, log_scales=log_scales,
                            opacity_logits=opacity_logits, sh=sh, screen_norms=screen_norms, visible=visible)
        self._n = int(np.asarray(positions.shape)[0])
        self._k = int(sh.shape[2])

    @classmethod
    def zeros(cls, n: int, sh_degree: int, device) -> "FieldGrads":
        k = (sh_degree + 1) ** 2
        flat = torch.zeros(flat_size(n, k, extra=2), dtype=torch.float32, device=device)
        return cls(_flat=flat, _n=n, _k=k)

    def _view(self, i):
        n, k = self._n, self._k
        if i < 5:
            off, w = class_slices(n, k)[i]
            return self._flat[off: off + w * n].view(((n, 3), (n, 4), (n, 3), (n,), (n, 3, k))[i])
        s, ns = 11 + 3 * k, row_stride(n)
        return self._flat[(s + i - 5) * ns: (s + i - 5) * ns + n]

    def _get(self, name, i):
        if self._flat is not None:
            return self._view(i)
        return self._arrays[name]

    positions = property(lambda s: s._get("positions", 0))
    rotations = property(lambda s: s._get("rotations", 1))
    log_scales = property(lambda s: s._get("log_scales", 2))
    opacity_logits = property(lambda s: s._get("opacity_logits", 3))
    sh = property(lambda s: s._get("sh", 4))
    screen_norms = property(lambda s: s._get("screen_norms", 5))

    @property
    def visible(self):
        if self._flat is not None:
            return self._view(6) > 0
        return self._arrays["visible"]

    @property
    def visible_count(self) -> torch.Tensor:
        """Per-row number of views that saw the Gaussian (float; batches)."""
        return self._view(6)

    def flat_params(self, device) -> torch.Tensor:
        """Parameter-gradient part of the flat buffer (packs user-built grads)."""
        if self._flat is not None:
            return self._flat
        parts = [torch.as_tensor(self._arrays[k] if torch.is_tensor(self._arrays[k]) else
                                 np.asarray(self._arrays[k]))
                 for k in ("positions", "rotations", "log_scales", "opacity_logits", "sh")]
        return pack_classes(parts, self._n, self._k, device)

    @property
    def flat(self):
        return self._flat


def _as_dev(x, shape, dev):
    t = torch.as_tensor(x if torch.is_tensor(x) else np.asarray(x))
    if t.numel() != int(np.prod(shape)):
        raise InvalidParameter(f"gradient has {t.numel()} elements, expected shape {shape}")
    return t.to(device=dev, dtype=torch.float32).reshape(shape).contiguous()


def backward(field, out: RenderOutput, d_image, d_soft=None, layout: str = "splat", workers: int = 1,
             grads: FieldGrads | None = None, accumulate: bool = False, stats: torch.Tensor | None = None
             ) -> FieldGrads:
    """Gradients of a scalar loss given dL/d(image) and dL/d(soft_count).

    Extensions beyond the reference signature (all optional): ``grads`` +
    ``accumulate`` sum several views into one FieldGrads (semi-global view
    batches); ``stats`` (2N float: grad_accum, grad_count) receives the
    densify statistics of pipeline.py:201-202 in the same kernel pass.
    """
    if out.generation != field.generation:
        raise StaleFieldError(f"render saw generation {out.generation}, field is at {field.generation}")
    if out.ckpt is None or (out.ckpt.numel() == 0 and out.splats.n_instances > 0):
        raise InvalidParameter("this RenderOutput came from render(for_backward=False) and cannot be differentiated")
    if layout not in LAYOUTS:
        raise ValueError(f"unknown backward layout {layout!r}")
    cam, sp = out.cam, out.splats
    h, w = cam.height, cam.width
    dev = out.image.device
    d_image = _as_dev(d_image, (h, w, 3), dev)
    d_soft = None if d_soft is None else _as_dev(d_soft, (h, w), dev)
    n, k = len(field), field.n_sh_coeffs
    if grads is None:
        grads = FieldGrads(_flat=torch.empty(flat_size(n, k, extra=2), dtype=torch.float32, device=dev), _n=n, _k=k)
        accumulate = False
    elif grads._flat is None or grads._n != n:
        raise InvalidParameter("grads buffer does not match the field")
    m = sp.n_instances
    st = _lib.stream_ptr()
    s = sp.struct()
    rows = rows_workspace(dev, m)
    if m:
        _lib.call("ssr_backward", LAYOUTS[layout], m, s, sp.inst_gauss.data_ptr(), sp.tile_ranges.data_ptr(),
                  out.frame_struct(), d_image.data_ptr(), _lib.ptr(d_soft), rows.data_ptr(), st)
    if n:
        flat = field.flat
        sl = class_slices(n, k)
        # accumulating (view batches): scratch for the list of the rows this view sees
        row_list = _row_list(dev, n) if accumulate else None
        _lib.call("ssr_chain", _lib.camera_struct(cam), n, field.sh_degree, flat[sl[0][0]:].data_ptr(),
                  flat[sl[1][0]:].data_ptr(), flat[sl[2][0]:].data_ptr(), flat[sl[4][0]:].data_ptr(), s,
                  rows.data_ptr(), grads.flat.data_ptr(), 1 if accumulate else 0, _lib.ptr(stats),
                  _lib.ptr(row_list), st)
    return grads


def backward_and_step(field, out: RenderOutput, d_image, d_soft, optimizer, position_rate: float,
                      layout: str = "splat", stats: torch.Tensor | None = None) -> None:
    """``backward`` followed by ``optimizer.step`` without materialising FieldGrads.

    Same results as the two reference calls (backward.py:41-129 then
    optim.py:113-130) up to fp32 rounding order; the chain kernels apply the
    dense Adam update in place (ssr_chain_adam), saving the gradient buffer's
    write and read (~0.5 GB per iteration at config 2).
    """
    from ..optim import SH_REST_LR

    if out.generation != field.generation:
        raise StaleFieldError(f"render saw generation {out.generation}, field is at {field.generation}")
    if out.ckpt is None or (out.ckpt.numel() == 0 and out.splats.n_instances > 0):
        raise InvalidParameter("this RenderOutput came from render(for_backward=False) and cannot be differentiated")
    if layout not in LAYOUTS:
        raise ValueError(f"unknown backward layout {layout!r}")
    optimizer.check(field)
    cam, sp = out.cam, out.splats
    h, w = cam.height, cam.width
    dev = out.image.device
    d_image = _as_dev(d_image, (h, w, 3), dev)
    d_soft = None if d_soft is None else _as_dev(d_soft, (h, w), dev)
    n = len(field)
    m = sp.n_instances
    st = _lib.stream_ptr()
    s = sp.struct()
    rows = rows_workspace(dev, m)
    if m:
        _lib.call("ssr_backward", LAYOUTS[layout], m, s, sp.inst_gauss.data_ptr(), sp.tile_ranges.data_ptr(),
                  out.frame_struct(), d_image.data_ptr(), _lib.ptr(d_soft), rows.data_ptr(), st)
    if n:
        lr, bc1, bc2 = optimizer.advance(position_rate)
        field.version += 1
        _lib.call("ssr_chain_adam", _lib.camera_struct(cam), n, field.sh_degree, field.flat.data_ptr(),
                  optimizer.m.data_ptr(), optimizer.v.data_ptr(), s, rows.data_ptr(), _lib.ptr(stats), lr,
                  SH_REST_LR, bc1, bc2, st)
