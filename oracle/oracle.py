"""TEST INFRASTRUCTURE ONLY -- CPU oracle for the splat rasterizer hot path.

numpy glue over ``liboracle.so`` (plain-C float64 restatement in
``splat_oracle.c``) that mirrors the reference package's operator API:
``project_field`` / ``render`` / ``backward`` / ``total_loss`` /
``FieldOptimizer`` / ``densify_and_prune``.  Citations are to
``/root/reference/pkg/src/splatstream/<file>:<line>``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module; it is the checker, never the thing shipped.  It is pinned
against golden vectors produced by the reference itself
(``tests/golden/make_golden.py`` -> ``tests/test_oracle_golden.py``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

TILE = 16
ALPHA_MIN = 1.0 / 255.0
ALPHA_CAP = 0.99
T_EPS = 1e-4
SOFT_TAU = 0.01

# optim.py:17-25
BETA1, BETA2, EPS = 0.9, 0.999, 1e-15
ROTATION_LR, SCALE_LR, OPACITY_LR = 1e-3, 5e-3, 0.05
SH_DC_LR = 2.5e-3
SH_REST_LR = SH_DC_LR / 20.0


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "splat_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    return _LIB_PATH


class _Cam(ctypes.Structure):
    _fields_ = [
        ("R", ctypes.c_double * 9),
        ("t", ctypes.c_double * 3),
        ("fx", ctypes.c_double),
        ("fy", ctypes.c_double),
        ("cx", ctypes.c_double),
        ("cy", ctypes.c_double),
        ("center", ctypes.c_double * 3),
        ("width", ctypes.c_int64),
        ("height", ctypes.c_int64),
    ]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = ctypes.CDLL(_LIB_PATH)
        _lib.orc_num_threads.restype = ctypes.c_int
        _lib.orc_ssim.restype = ctypes.c_double
    return _lib


def set_threads(n: int) -> None:
    lib().orc_set_threads(int(n))


def num_threads() -> int:
    return int(lib().orc_num_threads())


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _cam(cam) -> _Cam:
    c = _Cam()
    R = np.asarray(cam.rotation, dtype=np.float64).reshape(9)
    t = np.asarray(cam.translation, dtype=np.float64).reshape(3)
    center = -np.asarray(cam.rotation, np.float64).reshape(3, 3).T @ t
    for i in range(9):
        c.R[i] = R[i]
    for i in range(3):
        c.t[i] = t[i]
        c.center[i] = center[i]
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    c.width, c.height = int(cam.width), int(cam.height)
    return c


@dataclass
class Params:
    """float64 SoA Gaussian parameters (field.py:186-245 layout)."""

    positions: np.ndarray
    rotations: np.ndarray
    log_scales: np.ndarray
    opacity_logits: np.ndarray
    sh: np.ndarray  # (N, 3, K) channel-major

    @property
    def sh_degree(self) -> int:
        return int(round(np.sqrt(self.sh.shape[2]))) - 1

    def __len__(self):
        return self.positions.shape[0]

    def copy(self) -> "Params":
        return Params(*(np.array(a, dtype=np.float64, copy=True) for a in (
            self.positions, self.rotations, self.log_scales, self.opacity_logits, self.sh)))

    @classmethod
    def from_any(cls, obj) -> "Params":
        return cls(*(np.ascontiguousarray(np.asarray(getattr(obj, k)), dtype=np.float64) for k in (
            "positions", "rotations", "log_scales", "opacity_logits", "sh")))


def tile_grid(width, height):
    return (width + TILE - 1) // TILE, (height + TILE - 1) // TILE


def project_field(params: Params, cam) -> dict:
    """projection.py:69-191 -- returns the ProjectedSplats fields as a dict."""
    P = params
    n = len(P)
    K = P.sh.shape[2]
    tiles_x, tiles_y = tile_grid(cam.width, cam.height)
    n_tiles = tiles_x * tiles_y
    keep = np.zeros(n, np.uint8)
    f = lambda *s: np.zeros(s, np.float64)
    means2d, conics, depths, radii = f(n, 2), f(n, 3), f(n), f(n)
    colors, opac, cam_pts, clamp_mul = f(n, 3), f(n), f(n, 3), f(n, 2)
    cov2d, cov3d, dirs, rsafe = f(n, 3), f(n, 3, 3), f(n, 3), f(n)
    lo, hi = np.zeros((n, 3), np.uint8), np.zeros((n, 3), np.uint8)
    rect = np.zeros((n, 4), np.int64)
    c = _cam(cam)
    arrs = [np.ascontiguousarray(a, np.float64) for a in (P.positions, P.rotations, P.log_scales, P.opacity_logits, P.sh)]
    if n:
        lib().orc_project(ctypes.c_int64(n), ctypes.c_int(int(round(np.sqrt(K))) - 1), *[_p(a) for a in arrs],
                          ctypes.byref(c), _p(keep), _p(means2d), _p(conics), _p(depths), _p(radii), _p(colors),
                          _p(opac), _p(cam_pts), _p(clamp_mul), _p(cov2d), _p(cov3d), _p(dirs), _p(rsafe),
                          _p(lo), _p(hi), _p(rect))
    gi = np.nonzero(keep)[0].astype(np.int64)
    out = dict(
        gauss_index=gi, means2d=means2d[gi], conics=conics[gi], depths=depths[gi], radii=radii[gi],
        colors=colors[gi], opacities=opac[gi], cam_points=cam_pts[gi], clamp_mul=clamp_mul[gi],
        cov2d=cov2d[gi], cov3d_cam=cov3d[gi], sh_dirs=dirs[gi], sh_radii=rsafe[gi],
        sh_lo=lo[gi].astype(bool), sh_hi=hi[gi].astype(bool), tiles_x=tiles_x, tiles_y=tiles_y,
    )
    r = np.ascontiguousarray(rect[gi])
    counts = (r[:, 2] - r[:, 0]) * (r[:, 3] - r[:, 1])
    M = int(counts.sum())
    inst = np.zeros(M, np.int64)
    ts, te = np.zeros(n_tiles, np.int64), np.zeros(n_tiles, np.int64)
    if M:
        lib().orc_bin_tiles(ctypes.c_int64(gi.size), ctypes.c_int64(tiles_x), ctypes.c_int64(n_tiles), _p(r),
                            _p(np.ascontiguousarray(out["depths"])), ctypes.c_int64(M), _p(inst), _p(ts), _p(te))
    out.update(inst_splat=inst, tile_starts=ts, tile_ends=te, rect=r)
    return out


def render(params: Params, cam, bg=(0.0, 0.0, 0.0)) -> dict:
    """forward.py:66-114 + kernels.py:31-103."""
    sp = project_field(params, cam)
    h, w = cam.height, cam.width
    bg = np.asarray(bg, np.float64).reshape(3)
    img = np.empty((h, w, 3))
    t_final = np.ones((h, w))
    n_walk = np.zeros((h, w), np.int64)
    term = np.zeros((h, w), np.uint8)
    hard = np.zeros((h, w), np.int64)
    soft = np.zeros((h, w))
    n_tiles = sp["tiles_x"] * sp["tiles_y"]
    lib().orc_forward(ctypes.c_int64(sp["tiles_x"]), ctypes.c_int64(w), ctypes.c_int64(h), ctypes.c_int64(n_tiles),
                      _p(sp["tile_starts"]), _p(sp["tile_ends"]), _p(sp["inst_splat"]),
                      _p(np.ascontiguousarray(sp["means2d"])), _p(np.ascontiguousarray(sp["conics"])),
                      _p(np.ascontiguousarray(sp["opacities"])), _p(np.ascontiguousarray(sp["colors"])), _p(bg),
                      _p(img), _p(t_final), _p(n_walk), _p(term), _p(hard), _p(soft))
    return dict(image=img, t_final=t_final, n_walk=n_walk, terminated=term, hard_count=hard,
                soft_count=soft, splats=sp, bg=bg, cam=cam)


def backward_rows(out: dict, d_image, d_soft=None, layout="splat") -> np.ndarray:
    """kernels.py:106-353 per-instance rows (M, 9)."""
    sp, cam = out["splats"], out["cam"]
    h, w = cam.height, cam.width
    d_image = np.ascontiguousarray(np.asarray(d_image, np.float64).reshape(h, w, 3))
    d_soft = np.zeros((h, w)) if d_soft is None else np.ascontiguousarray(np.asarray(d_soft, np.float64).reshape(h, w))
    M = sp["inst_splat"].size
    rows = np.zeros((M, 9))
    fn = lib().orc_backward_splat if layout == "splat" else lib().orc_backward_pixel
    n_tiles = sp["tiles_x"] * sp["tiles_y"]
    if M:
        fn(ctypes.c_int64(sp["tiles_x"]), ctypes.c_int64(w), ctypes.c_int64(h), ctypes.c_int64(n_tiles),
           _p(sp["tile_starts"]), _p(sp["tile_ends"]), _p(sp["inst_splat"]),
           _p(np.ascontiguousarray(sp["means2d"])), _p(np.ascontiguousarray(sp["conics"])),
           _p(np.ascontiguousarray(sp["opacities"])), _p(np.ascontiguousarray(sp["colors"])), _p(out["bg"]),
           _p(d_image), _p(d_soft), _p(out["t_final"]), _p(out["n_walk"]), _p(out["terminated"]), _p(rows))
    return rows


def backward(params: Params, out: dict, d_image, d_soft=None, layout="splat") -> dict:
    """backward.py:41-129 -- FieldGrads as a dict of float64 arrays."""
    if layout not in ("splat", "pixel"):
        raise ValueError(f"unknown backward layout {layout!r}")
    sp, cam = out["splats"], out["cam"]
    h, w = cam.height, cam.width
    n = len(params)
    K = params.sh.shape[2]
    g = dict(positions=np.zeros((n, 3)), rotations=np.zeros((n, 4)), log_scales=np.zeros((n, 3)),
             opacity_logits=np.zeros(n), sh=np.zeros((n, 3, K)), screen_norms=np.zeros(n),
             visible=np.zeros(n, bool))
    gi = sp["gauss_index"]
    V = gi.size
    if V == 0:
        return g
    g["visible"][gi] = True
    rows = backward_rows(out, d_image, d_soft, layout)
    per = np.zeros((V, 9))
    M = sp["inst_splat"].size
    if M:
        lib().orc_merge(ctypes.c_int64(M), ctypes.c_int64(V), _p(sp["inst_splat"]), _p(rows), _p(per))
    d_pos, d_quat, d_ls, d_sh = np.zeros((V, 3)), np.zeros((V, 4)), np.zeros((V, 3)), np.zeros((V, 3, K))
    c = _cam(cam)
    C = lambda a: np.ascontiguousarray(a, np.float64)
    lib().orc_chain(ctypes.c_int64(V), ctypes.c_int(int(round(np.sqrt(K))) - 1), ctypes.byref(c),
                    _p(C(params.sh[gi])), _p(C(params.rotations[gi])), _p(C(params.log_scales[gi])),
                    _p(C(sp["conics"])), _p(C(sp["cam_points"])), _p(C(sp["clamp_mul"])), _p(C(sp["cov3d_cam"])),
                    _p(C(sp["sh_dirs"])), _p(C(sp["sh_radii"])), _p(np.ascontiguousarray(sp["sh_lo"], np.uint8)),
                    _p(np.ascontiguousarray(sp["sh_hi"], np.uint8)), _p(per), _p(d_pos), _p(d_quat), _p(d_ls), _p(d_sh))
    g["positions"][gi] = d_pos
    g["rotations"][gi] = d_quat
    g["log_scales"][gi] = d_ls
    g["opacity_logits"][gi] = per[:, 3]
    g["sh"][gi] = d_sh
    g["screen_norms"][gi] = np.linalg.norm(per[:, 4:6], axis=1) * (0.5 * max(w, h))
    return g


# ---------------------------------------------------------------- losses.py


@dataclass
class LossWeights:
    l1: float = 0.47
    ssim: float = 0.12
    load: float = 0.41


def ssim_value_and_grad(x, y):
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    if x.ndim == 2:
        x, y = x[:, :, None], y[:, :, None]
    h, w, nch = x.shape
    grad = np.zeros_like(x)
    val = lib().orc_ssim(ctypes.c_int64(h), ctypes.c_int64(w), ctypes.c_int64(nch), _p(x), _p(y), _p(grad))
    return float(val), grad


def total_loss(rendered, target, soft_count, hard_count, weights: LossWeights) -> dict:
    """losses.py:55-173."""
    rendered = np.asarray(rendered, np.float64)
    target = np.asarray(target, np.float64)
    diff = rendered - target
    v_l1 = float(np.abs(diff).mean())
    g_l1 = np.sign(diff) / diff.size
    v_s, g_s = ssim_value_and_grad(rendered, target)
    v_ssim, g_ssim = 1.0 - v_s, -g_s
    s = np.asarray(soft_count, np.float64)
    if weights.load > 0.0:
        if s.size == 0 or s.min() == s.max():
            v_load, g_load = 0.0, np.zeros_like(s)
        else:
            dev = s - s.mean()
            std = float((dev * dev).mean()) ** 0.5
            v_load, g_load = (0.0, np.zeros_like(s)) if std == 0.0 else (std, dev / (s.size * std))
        d_soft = weights.load * g_load
    else:
        v_load, d_soft = 0.0, np.zeros_like(s)
    total = weights.l1 * v_l1 + weights.ssim * v_ssim + weights.load * v_load
    d_image = weights.l1 * g_l1 + weights.ssim * g_ssim
    return dict(l1=v_l1, ssim_loss=v_ssim, load=v_load, total=total, d_image=d_image, d_soft=d_soft,
                hard_count_std=float(np.asarray(hard_count, np.float64).std()))


# ---------------------------------------------------------------- optim.py / field.py


class Optimizer:
    """optim.py:78-130 -- dense bias-corrected Adam, one step counter per class."""

    CLASSES = ("positions", "rotations", "log_scales", "opacity_logits", "sh")

    def __init__(self, params: Params, scene_extent=1.0):
        self.scene_extent = float(scene_extent)
        self.m = {k: np.zeros_like(getattr(params, k)) for k in self.CLASSES}
        self.v = {k: np.zeros_like(getattr(params, k)) for k in self.CLASSES}
        self.steps = {k: 0 for k in self.CLASSES}

    def step(self, params: Params, grads: dict, position_rate: float):
        K = params.sh.shape[2]
        sh_lr = np.full((1, 1, K), SH_REST_LR)
        sh_lr[0, 0, 0] = SH_DC_LR
        lrs = dict(positions=position_rate * self.scene_extent, rotations=ROTATION_LR, log_scales=SCALE_LR,
                   opacity_logits=OPACITY_LR, sh=sh_lr)
        for k in self.CLASSES:
            p = getattr(params, k)
            self.steps[k] += 1
            lr = np.ascontiguousarray(np.broadcast_to(lrs[k], p.shape), np.float64)
            gr = np.ascontiguousarray(grads[k], np.float64)
            lib().orc_adam(ctypes.c_int64(p.size), _p(p), _p(gr), _p(self.m[k]), _p(self.v[k]), _p(lr),
                           ctypes.c_int64(self.steps[k]))

    def sync(self, keep_mask, n_added):
        """optim.py:49-54,101-111."""
        for k in self.CLASSES:
            for d in (self.m, self.v):
                a = d[k]
                d[k] = np.concatenate([a[keep_mask], np.zeros((n_added,) + a.shape[1:])], axis=0)


@dataclass
class DensifyOptions:
    grad_threshold: float = 2e-4
    percent_dense: float = 0.01
    scene_extent: float = 1.0
    prune_opacity: float = 0.005
    split_scale_shrink: float = 1.6


def _quat_to_rotmat(q):
    q = np.asarray(q, np.float64)
    norm = np.linalg.norm(q, axis=-1, keepdims=True)
    w, x, y, z = np.moveaxis(q / norm, -1, 0)
    rot = np.empty(q.shape[:-1] + (3, 3))
    rot[..., 0, 0] = 1 - 2 * (y * y + z * z)
    rot[..., 0, 1] = 2 * (x * y - w * z)
    rot[..., 0, 2] = 2 * (x * z + w * y)
    rot[..., 1, 0] = 2 * (x * y + w * z)
    rot[..., 1, 1] = 1 - 2 * (x * x + z * z)
    rot[..., 1, 2] = 2 * (y * z - w * x)
    rot[..., 2, 0] = 2 * (x * z - w * y)
    rot[..., 2, 1] = 2 * (y * z + w * x)
    rot[..., 2, 2] = 1 - 2 * (x * x + y * y)
    return rot


def densify_and_prune(params: Params, grad_stats, opts: DensifyOptions, rng):
    """field.py:303-375 -- returns (new_params, cloned, split, pruned, keep_mask, n_added)."""
    grad_stats = np.asarray(grad_stats, np.float64)
    P = params
    scales = np.exp(P.log_scales)
    max_scale = scales.max(axis=1)
    hot = grad_stats > opts.grad_threshold
    prune = (1.0 / (1.0 + np.exp(-P.opacity_logits))) < opts.prune_opacity
    big = max_scale > opts.percent_dense * opts.scene_extent
    clone = hot & ~big & ~prune
    split = hot & big & ~prune
    adds = {k: [] for k in Optimizer.CLASSES}
    if clone.any():
        for k in Optimizer.CLASSES:
            adds[k].append(getattr(P, k)[clone].copy())
    if split.any():
        idx = np.nonzero(split)[0]
        rep = np.repeat(idx, 2)
        rot = _quat_to_rotmat(P.rotations[rep])
        eps = rng.standard_normal((rep.size, 3))
        offsets = np.einsum("nij,nj->ni", rot, scales[rep] * eps)
        adds["positions"].append(P.positions[rep] + offsets)
        adds["rotations"].append(P.rotations[rep].copy())
        adds["log_scales"].append(P.log_scales[rep] - np.log(opts.split_scale_shrink))
        adds["opacity_logits"].append(P.opacity_logits[rep].copy())
        adds["sh"].append(P.sh[rep].copy())
    keep = ~(split | prune)
    n_added = int(sum(a.shape[0] for a in adds["positions"]))
    changed = clone.any() or split.any() or prune.any()
    if not changed:
        return P, 0, 0, 0, keep, 0
    new = Params(*(np.concatenate([getattr(P, k)[keep]] + adds[k]) for k in Optimizer.CLASSES))
    return new, int(clone.sum()), int(split.sum()), int(prune.sum()), keep, n_added
