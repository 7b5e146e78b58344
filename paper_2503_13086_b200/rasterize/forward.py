"""Stage 3 host wrapper: ``render`` (forward.py:21-114 of the reference)."""

from __future__ import annotations

from dataclasses import dataclass, field as dc_field

import numpy as np
import torch

from .. import _lib
from ..camera import CameraFrame
from ..errors import InvalidParameter
from .projection import ProjectedSplats, project_begin, project_end, project_field  # noqa: F401

# Relative guard bands of the fp32 walk's discrete decisions; pixels inside
# either are re-walked in float64.  GUARD_BAND covers the
# alpha >= 1/255 gate and the 0.99 cap, GUARD_BAND_T the T(1-alpha) < 1e-4
# termination (whose fp32 error accumulates over the walk).
GUARD_BAND = 1e-5
GUARD_BAND_T = 1e-4


@dataclass
class RenderOutput:
    """Rendered image plus the retained state the backward pass replays."""

    image: torch.Tensor  # (H, W, 3) float32
    t_final: torch.Tensor  # (H, W)
    n_walk: torch.Tensor  # (H, W) int32
    terminated: torch.Tensor  # (H, W) uint8
    hard_count: torch.Tensor  # (H, W) int32
    soft_count: torch.Tensor  # (H, W) float64; None for render(soft_count=False)
    splats: ProjectedSplats
    cam: CameraFrame
    bg: np.ndarray
    generation: int
    workers: int = dc_field(default=1, repr=False)
    flagged: torch.Tensor = dc_field(default=None, repr=False)  # (H, W) uint8 guard-band pixels
    tile_info: torch.Tensor = dc_field(default=None, repr=False)  # (n_tiles, 4) int32
    ckpt: torch.Tensor = dc_field(default=None, repr=False)  # bucket checkpoints (T, C_front)
    fix_list: torch.Tensor = dc_field(default=None, repr=False)  # compact flagged pixel / tile lists

    @property
    def n_visible(self) -> int:
        return self.splats.n_visible

    def frame_struct(self) -> _lib.SsrFrame:
        f = _lib.SsrFrame()
        f.width, f.height = self.cam.width, self.cam.height
        f.tiles_x, f.tiles_y = self.splats.tiles_x, self.splats.tiles_y
        for i in range(3):
            f.bg[i] = float(self.bg[i])
        for k in ("image", "t_final", "n_walk", "terminated", "hard_count", "soft_count", "flagged", "tile_info",
                  "ckpt", "fix_list"):
            t = getattr(self, k)
            setattr(f, k, t.data_ptr() if t is not None and t.numel() else None)
        return f


def render(field, cam: CameraFrame, bg=(0.0, 0.0, 0.0), workers: int = 1, band: float = None,
           band_t: float = None, *, for_backward: bool = True, soft_count: bool = True) -> RenderOutput:
    """Render the field from ``cam`` over a constant background colour.

    ``for_backward=False`` is the render-only path (view_psnr, pipeline.py:180-182):
    identical outputs, but the bucket checkpoints the backward seeds from are not
    written (~16 B per live pixel-bucket, ~320 MB at 1M Gaussians / 1080p), so the
    result cannot be passed to ``backward``.

    ``soft_count=False`` skips the soft blend count (``RenderOutput.soft_count``
    is None): a loss whose load weight is 0 never reads it (losses.py:155-160),
    and without it the walk culls pairs certain to stay below 1/255 at the
    packed far test.  Every other output is identical; such a render feeds
    ``total_loss`` only with ``weights.load == 0``."""
    if workers < 1:
        raise InvalidParameter(f"workers must be >= 1, got {workers}")
    band = GUARD_BAND if band is None else float(band)
    band_t = GUARD_BAND_T if band_t is None else float(band_t)
    bg = np.asarray(bg, dtype=np.float64).reshape(3)
    splats, ctx = project_begin(field, cam)
    # the outputs do not depend on the instance count: allocated while the
    # device runs the preprocess, before the host waits for that count
    dev = splats.tile_ranges.device
    h, w = cam.height, cam.width
    n_tiles = splats.tiles_x * splats.tiles_y
    e = lambda *s, dt=torch.float32: torch.empty(s, dtype=dt, device=dev)
    image, t_final, n_walk = e(h, w, 3), e(h, w), e(h, w, dt=torch.int32)
    terminated, hard = e(h, w, dt=torch.uint8), e(h, w, dt=torch.int32)
    soft = e(h, w, dt=torch.float64) if soft_count else None
    flagged, tile_info = e(h, w, dt=torch.uint8), e(n_tiles, 4, dt=torch.int32)
    fix_list = e(int(_lib.load().ssr_fix_list_ints(w, h, n_tiles)), dt=torch.int32)
    project_end(splats, ctx, field)
    m = splats.n_instances
    out = RenderOutput(
        image=image, t_final=t_final, n_walk=n_walk, terminated=terminated, hard_count=hard, soft_count=soft,
        splats=splats, cam=cam, bg=bg, generation=field.generation, workers=workers, flagged=flagged,
        tile_info=tile_info,
        ckpt=e(int(_lib.load().ssr_ckpt_floats(max(m, splats._cap), n_tiles)) if for_backward else 0),
        fix_list=fix_list,
    )
    _lib.call("ssr_forward", m, splats.struct(), splats.inst_gauss.data_ptr() if m else None,
              splats.tile_ranges.data_ptr(), out.frame_struct(), band, band_t, _lib.stream_ptr())
    return out
