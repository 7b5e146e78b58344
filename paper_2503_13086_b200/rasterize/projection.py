"""Stage 1-2 host wrapper: preprocess + tile binning (projection.py:24-191).

``project_field`` returns a ``ProjectedSplats`` whose reference-named fields
(``gauss_index``, ``means2d``, ``conics``, ``inst_splat``, ``tile_starts`` ...)
are computed lazily from the device buffers the kernels use; the hot path
itself only touches the N-indexed device arrays and the sorted instance list.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field as dc_field

import torch

from .. import _lib
from ..camera import CameraFrame
from ..errors import InvalidParameter, StaleFieldError

TILE = 16
ZNEAR = 0.2
COV2D_DILATION = 0.3
FRUSTUM_EXPAND = 1.3


def tile_grid(width: int, height: int):
    return (width + TILE - 1) // TILE, (height + TILE - 1) // TILE


@dataclass
class ProjectedSplats:
    """Device state of one projection (N-indexed) plus the sorted instances."""

    n: int
    sh_degree: int
    tiles_x: int
    tiles_y: int
    bufs: dict  # name -> tensor (see ssr_splats in include/ssr.h)
    inst_gauss: torch.Tensor  # (M,) int32 field row per sorted instance
    tile_ranges: torch.Tensor  # (n_tiles, 2) int32 (start, end)
    cam: CameraFrame
    _src: tuple = dc_field(default=None, repr=False)  # (field, field.version, n, K) for aux
    _cap: int = dc_field(default=0, repr=False)  # instance capacity of the buffers sized by M
    _cache: dict = dc_field(default_factory=dict, repr=False)

    def struct(self) -> _lib.SsrSplats:
        s = _lib.SsrSplats()
        for k in ("mean", "conic_opa", "color", "conic_opa64", "color64", "depth", "rect", "tiles", "offset",
                  "row_offset", "depth_order"):
            setattr(s, k, self.bufs[k].data_ptr() if self.bufs[k].numel() else None)
        return s

    # ---------------------------------------------------------- reference-named views
    @property
    def n_instances(self) -> int:
        return int(self.inst_gauss.numel())

    @property
    def visible_mask(self) -> torch.Tensor:
        return self.bufs["tiles"][: self.n] > 0

    @property
    def gauss_index(self) -> torch.Tensor:
        if "gi" not in self._cache:
            self._cache["gi"] = torch.nonzero(self.visible_mask).flatten()
        return self._cache["gi"]

    @property
    def n_visible(self) -> int:
        return int(self.gauss_index.numel())

    def _rows(self, name, cols, dtype=None):
        t = self.bufs[name].view(self.n, -1)[self.gauss_index][:, cols]
        return t if dtype is None else t.to(dtype)

    means2d = property(lambda s: s._rows("mean", slice(0, 2)))
    conics = property(lambda s: s._rows("conic_opa64", slice(0, 3)))
    opacities = property(lambda s: s._rows("conic_opa64", 3))
    colors = property(lambda s: s._rows("color64", slice(0, 3)))
    depths = property(lambda s: s.bufs["depth"][s.gauss_index])

    @property
    def inst_splat(self) -> torch.Tensor:
        """Visible-splat index per sorted instance (projection.py:50)."""
        rank = torch.cumsum(self.visible_mask.to(torch.int64), 0) - 1
        return rank[self.inst_gauss.long()]

    @property
    def tile_starts(self) -> torch.Tensor:
        return self.tile_ranges[:, 0].long()

    @property
    def tile_ends(self) -> torch.Tensor:
        return self.tile_ranges[:, 1].long()

    def _aux(self):
        if "aux" in self._cache:
            return self._cache["aux"]
        fld, version, n, k = self._src
        if fld.version != version or len(fld) != n:
            # the aux fields are recomputed from the live parameters; after an
            # in-place update they would describe a different field than this render
            raise StaleFieldError("field parameters changed since this projection; aux fields are unavailable")
        flat = fld.flat
        from ..field import class_slices

        sl = class_slices(n, k)
        dev = flat.device
        f64 = lambda *s: torch.zeros(s, dtype=torch.float64, device=dev)
        a = dict(cam_points=f64(n, 3), clamp_mul=f64(n, 2), cov2d=f64(n, 3), cov3d_cam=f64(n, 3, 3),
                 sh_dirs=f64(n, 3), sh_radii=f64(n), sh_lo=torch.zeros(n, 3, dtype=torch.uint8, device=dev),
                 sh_hi=torch.zeros(n, 3, dtype=torch.uint8, device=dev), radii=f64(n))
        cam = _lib.camera_struct(self.cam)
        _lib.call("ssr_project_aux", cam, n, self.sh_degree, flat[sl[0][0]:].data_ptr(),
                  flat[sl[1][0]:].data_ptr(), flat[sl[2][0]:].data_ptr(), flat[sl[4][0]:].data_ptr(),
                  self.bufs["tiles"].data_ptr(), *[a[x].data_ptr() for x in (
                      "cam_points", "clamp_mul", "cov2d", "cov3d_cam", "sh_dirs", "sh_radii", "sh_lo", "sh_hi",
                      "radii")], _lib.stream_ptr())
        gi = self.gauss_index
        out = {k2: v[gi] for k2, v in a.items()}
        out["sh_lo"] = out["sh_lo"].bool()
        out["sh_hi"] = out["sh_hi"].bool()
        self._cache["aux"] = out
        return out

    cam_points = property(lambda s: s._aux()["cam_points"])
    clamp_mul = property(lambda s: s._aux()["clamp_mul"])
    cov2d = property(lambda s: s._aux()["cov2d"])
    cov3d_cam = property(lambda s: s._aux()["cov3d_cam"])
    sh_dirs = property(lambda s: s._aux()["sh_dirs"])
    sh_radii = property(lambda s: s._aux()["sh_radii"])
    sh_lo = property(lambda s: s._aux()["sh_lo"])
    sh_hi = property(lambda s: s._aux()["sh_hi"])
    radii = property(lambda s: s._aux()["radii"])


def _alloc_splats(n: int, dev) -> dict:
    e = lambda *s, dt=torch.float32: torch.empty(s, dtype=dt, device=dev)
    return dict(mean=e(n, 2, dt=torch.float64), conic_opa=e(n, 4), color=e(n, 4),
                conic_opa64=e(n, 4, dt=torch.float64), color64=e(n, 4, dt=torch.float64),
                depth=e(n, dt=torch.float64), rect=e(n, 4, dt=torch.int32), tiles=e(n, dt=torch.int32),
                offset=e(n, dt=torch.int32), row_offset=e(n, dt=torch.int32), depth_order=e(n, dt=torch.int32))


_CAM_ATTRS = ("rotation", "translation", "center", "fx", "fy", "cx", "cy", "width", "height")


def check_camera(cam) -> None:
    """Accept any camera object with the reference CameraFrame's attributes
    (camera.py:11-60): this package's CameraFrame, the reference's own, or a
    duck-typed equivalent.  Only those attributes are read (_lib.camera_struct)."""
    missing = [a for a in _CAM_ATTRS if not hasattr(cam, a)]
    if missing:
        raise InvalidParameter(f"cam lacks camera attributes {missing}")
    if int(cam.width) < 1 or int(cam.height) < 1:
        raise InvalidParameter(f"camera size must be positive, got {cam.width}x{cam.height}")


def project_field(field, cam: CameraFrame) -> ProjectedSplats:
    """Project every Gaussian, cull, bin into tiles and depth-sort (projection.py:69-191)."""
    sp, ctx = project_begin(field, cam)
    project_end(sp, ctx, field)
    return sp


def project_begin(field, cam: CameraFrame):
    """Launch the preprocess and the per-Gaussian scans; returns (splats, ctx).

    Nothing here waits for the device.  The instance buffers are allocated
    speculatively from the field's last instance count (``_m_hint``), so that
    after the one host synchronisation of the path (the instance total M, in
    ``project_end``) the binning launches without further host work.
    """
    from ..field import class_slices

    dev = _lib.require_cuda()
    check_camera(cam)
    n, k = len(field), field.n_sh_coeffs
    tiles_x, tiles_y = tile_grid(cam.width, cam.height)
    n_tiles = tiles_x * tiles_y
    st = _lib.stream_ptr()
    bufs = _alloc_splats(n, dev)
    # every tile's range is written by ssr_bin_tiles (empty tiles included)
    sp = ProjectedSplats(n, field.sh_degree, tiles_x, tiles_y, bufs,
                         torch.empty(0, dtype=torch.int32, device=dev),
                         torch.empty(n_tiles, 2, dtype=torch.int32, device=dev), cam, (field, field.version, n, k))
    if n == 0:
        sp.tile_ranges.zero_()
        return sp, None
    flat = field.flat
    sl = class_slices(n, k)
    cstruct = _lib.camera_struct(cam)
    s = sp.struct()
    _lib.call("ssr_preprocess", cstruct, n, field.sh_degree, flat[sl[0][0]:].data_ptr(), flat[sl[1][0]:].data_ptr(),
              flat[sl[2][0]:].data_ptr(), flat[sl[3][0]:].data_ptr(), flat[sl[4][0]:].data_ptr(), s, st)
    ws = torch.empty(_lib.query("ssr_scan_workspace", n), dtype=torch.uint8, device=dev)
    total = torch.empty(1, dtype=torch.int64, device=dev)
    _lib.call("ssr_scan_tiles", n, s, ws.data_ptr(), ws.numel(), total.data_ptr(), st)
    cap = int(getattr(field, "_m_hint", 0) or 0)
    inst_cap = ws_cap = None
    if cap > 0:
        inst_cap = torch.empty(cap, dtype=torch.int32, device=dev)
        ws_cap = torch.empty(_lib.query("ssr_bin_workspace", cap, n_tiles), dtype=torch.uint8, device=dev)
    return sp, (total, cap, inst_cap, ws_cap, s, st, ws)


def project_end(sp: ProjectedSplats, ctx, field=None) -> ProjectedSplats:
    """Read the instance total (the path's one host synchronisation) and bin."""
    if ctx is None:
        return sp
    total, cap, inst_cap, ws_cap, s, st, _ = ctx
    dev = total.device
    n_tiles = sp.tiles_x * sp.tiles_y
    m = -1
    if cap > 0:
        # read M and launch the binning in one native call (no host-language
        # work between the synchronisation and the first binning kernel)
        m_out = ctypes.c_int64(0)
        rc = _lib.call_rc("ssr_bin_tiles_capacity", sp.n, cap, sp.tiles_x, sp.tiles_y, s, total.data_ptr(),
                          ctypes.byref(m_out), inst_cap.data_ptr(), sp.tile_ranges.data_ptr(), ws_cap.data_ptr(),
                          ws_cap.numel(), st)
        m = int(m_out.value)
        if rc == 0:
            sp.inst_gauss = inst_cap[:m]
            sp._cap = cap
            return sp
        if rc != 3 or m <= cap:
            _lib.raise_last("ssr_bin_tiles_capacity", rc)
    if m < 0:
        m = int(total.item())  # host needs M to size the instance buffers
    if m < 0 or m >= 1 << 30:
        raise InvalidParameter(f"instance count {m} exceeds the 2^30 - 1 limit of the tile sort")
    sp.inst_gauss = torch.empty(m, dtype=torch.int32, device=dev)
    ws = torch.empty(_lib.query("ssr_bin_workspace", m, n_tiles), dtype=torch.uint8, device=dev)
    sp._cap = m
    if field is not None:
        # capacity for the next renders: M + 6%, rounded up to 1/16 of M's leading
        # power of two, so the buffer sizes repeat and the allocator reuses its blocks
        step = 1 << max(12, m.bit_length() - 4)
        field._m_hint = (m + m // 16 + step) // step * step
    _lib.call("ssr_bin_tiles", sp.n, m, sp.tiles_x, sp.tiles_y, s, sp.inst_gauss.data_ptr() if m else None,
              sp.tile_ranges.data_ptr(), ws.data_ptr(), ws.numel(), st)
    return sp
