"""Generate golden vectors from the REFERENCE implementation (splatstream).

Run in the builder container only (needs /root/reference, read-only):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Each case writes ``tests/golden/<name>.npz`` holding the float32-rounded
inputs (upcast to float64, exactly what the reference consumed), the float64
camera, and the reference's outputs for project_field / render / total_loss /
backward (both layouts) / FieldOptimizer.step / densify_and_prune.  The oracle
(``oracle/``) is pinned against these in ``tests/test_oracle_golden.py``; the
GPU path is checked against the oracle and these fixtures in the -m gpu tests.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from splatstream.camera import CameraFrame as RefCam  # noqa: E402
from splatstream.field import DensifyOptions, GaussianField  # noqa: E402
from splatstream.losses import LossWeights, total_loss  # noqa: E402
from splatstream.optim import FieldOptimizer  # noqa: E402
from splatstream.rasterize import backward, project_field, render  # noqa: E402

from paper_2503_13086_b200 import scenes  # noqa: E402
from paper_2503_13086_b200.camera import look_at  # noqa: E402

PROJ_KEYS = ("gauss_index", "means2d", "conics", "depths", "radii", "colors", "opacities",
             "cam_points", "clamp_mul", "cov2d", "cov3d_cam", "sh_dirs", "sh_radii", "sh_lo",
             "sh_hi", "inst_splat", "tile_starts", "tile_ends")
OUT_KEYS = ("image", "t_final", "n_walk", "terminated", "hard_count", "soft_count")
GRAD_KEYS = ("positions", "rotations", "log_scales", "opacity_logits", "sh", "screen_norms", "visible")
PARAM_KEYS = ("positions", "rotations", "log_scales", "opacity_logits", "sh")


def _field(p):
    f = GaussianField(sh_degree=p.sh_degree)
    for k in PARAM_KEYS:
        setattr(f, k, np.array(getattr(p, k), dtype=np.float64))
    return f


def run_case(name, params, cam, bg, weights=LossWeights(), target_seed=99, densify=True, extras=True):
    field = _field(params)
    rcam = RefCam(cam.image_id, cam.width, cam.height, cam.fx, cam.fy, cam.cx, cam.cy,
                  cam.rotation, cam.translation)
    rec = {f"in_{k}": getattr(field, k).copy() for k in PARAM_KEYS}
    rec.update(cam_R=rcam.rotation, cam_t=rcam.translation,
               cam_intr=np.array([rcam.fx, rcam.fy, rcam.cx, rcam.cy]),
               cam_wh=np.array([rcam.width, rcam.height]), bg=np.asarray(bg, np.float64))
    sp = project_field(field, rcam)
    for k in PROJ_KEYS:
        rec[f"proj_{k}"] = np.asarray(getattr(sp, k))
    out = render(field, rcam, bg=bg)
    for k in OUT_KEYS:
        rec[f"out_{k}"] = np.asarray(getattr(out, k))
    rng = np.random.default_rng(target_seed)
    target = np.clip(out.image + rng.normal(0.0, 0.15, out.image.shape), 0.0, 1.0)
    rec["target"] = target
    rec["loss_weights"] = np.array([weights.l1, weights.ssim, weights.load])
    if min(cam.width, cam.height) >= 11:
        br = total_loss(out.image, target, out, weights)
        rec.update(loss_l1=br.l1, loss_ssim=br.ssim_loss, loss_load=br.load, loss_total=br.total,
                   loss_d_image=br.d_image, loss_d_soft=br.d_soft)
        d_img, d_soft = br.d_image, br.d_soft
    else:
        d_img = rng.standard_normal(out.image.shape) * 1e-3
        d_soft = rng.standard_normal(out.soft_count.shape) * 1e-4
    rec["bwd_d_image"], rec["bwd_d_soft"] = d_img, d_soft
    for layout in (("splat", "pixel") if extras else ("splat",)):
        g = backward(field, out, d_img, d_soft=d_soft, layout=layout)
        for k in GRAD_KEYS:
            rec[f"grad_{layout}_{k}"] = np.asarray(getattr(g, k))
    if not extras:
        densify = False
    # one optimizer step on the splat-layout grads
    g = backward(field, out, d_img, d_soft=d_soft, layout="splat")
    extent = 2.5
    rate = 1.6e-4
    opt = FieldOptimizer(field, scene_extent=extent)
    if extras:
        opt.step(field, g, position_rate=rate)
        rec["adam_extent"], rec["adam_rate"] = extent, rate
        for k in PARAM_KEYS:
            rec[f"adam_{k}"] = getattr(field, k).copy()
    if densify and len(field):
        field = _field(params)
        stats = np.abs(np.random.default_rng(7).standard_normal(len(field))) * 3e-4
        opts = DensifyOptions(scene_extent=0.5, prune_opacity=0.2)
        rec["dens_stats"] = stats
        rec["dens_opts"] = np.array([opts.grad_threshold, opts.percent_dense, opts.scene_extent,
                                     opts.prune_opacity, opts.split_scale_shrink])
        s = field.densify_and_prune(stats, opts, np.random.default_rng(11))
        rec["dens_counts"] = np.array([s.cloned, s.split, s.pruned, s.n_added])
        rec["dens_keep"] = s.keep_mask
        for k in PARAM_KEYS:
            rec[f"dens_{k}"] = getattr(field, k).copy()
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **rec)
    print(f"{name}: N={len(params)} V={sp.n_visible} M={sp.n_instances} "
          f"{cam.width}x{cam.height} -> {os.path.getsize(path) / 1e6:.2f} MB")


def _small(cfg, n, w, h, view, seed=0):
    p = scenes.make_params(cfg, seed=seed, n=n)
    cam = scenes.camera(cfg, view=view, width=w, height=h)
    return p, cam


def _edge_params(pos, log_scale, logit, rgb_dc, deg=0, rots=None):
    n = len(pos)
    k = (deg + 1) ** 2
    sh = np.zeros((n, 3, k), np.float32)
    sh[:, :, 0] = (np.asarray(rgb_dc, np.float64) - 0.5) / 0.28209479177387814
    rot = np.zeros((n, 4), np.float32) if rots is None else np.asarray(rots, np.float32)
    if rots is None:
        rot[:, 0] = 1.0
    return scenes.HostParams(np.asarray(pos, np.float32), rot,
                             np.full((n, 3), log_scale, np.float32),
                             np.full(n, logit, np.float32), sh)


def expansion_case():
    """field.py:111-161,258-301: SpatialIndex, filter_new_points, median_nn_spacing, insert_points."""
    from splatstream.field import SparsePoint, SpatialIndex, filter_new_points, median_nn_spacing

    rng = np.random.default_rng(41)
    existing = scenes.make_params(2, seed=3, n=700)
    field = _field(existing)
    pts = rng.standard_normal((300, 3)) * 2.0
    pts[:40] = np.asarray(existing.positions[:40], np.float64) + rng.normal(0, 1e-3, (40, 3))  # near duplicates
    pts[40:45] = pts[45:50]  # exact duplicates among the candidates
    cols = rng.uniform(0.0, 1.0, (300, 3))
    cands = [SparsePoint(p, c) for p, c in zip(pts, cols)]
    sparse = np.asarray(existing.positions, np.float64)
    idx = SpatialIndex(sparse)
    queries = rng.standard_normal((200, 3)) * 3.0
    rec = dict(exp_existing_pos=np.asarray(existing.positions, np.float64), exp_cand_pos=pts, exp_cand_col=cols,
               exp_queries=queries, exp_min_dist=idx.min_distance(queries),
               exp_median_nn=median_nn_spacing(sparse))
    thr = 0.05
    kept = filter_new_points(idx, cands, thr)
    rec["exp_threshold"] = thr
    rec["exp_kept"] = np.array([any(k is c for k in kept) for c in cands])
    g0 = field.generation
    n_in = field.insert_points(kept, init_opacity=0.1)
    rec["exp_n_inserted"] = n_in
    rec["exp_generation_delta"] = field.generation - g0
    for k in PARAM_KEYS:
        rec[f"exp_after_{k}"] = getattr(field, k).copy()
    for k in PARAM_KEYS:
        rec[f"in_{k}"] = np.asarray(getattr(existing, k), np.float64)
    path = os.path.join(HERE, "expansion.npz")
    np.savez_compressed(path, **rec)
    print(f"expansion: existing=700 candidates=300 kept={len(kept)} -> {os.path.getsize(path) / 1e6:.2f} MB")


def main():
    # config-0 at full size (the reference's own CPU-runnable case)
    p = scenes.make_params(0, seed=0)
    run_case("c0_full", p, scenes.camera(0, view=0), bg=(0.0, 0.0, 0.0),
             weights=LossWeights(l1=1.0, ssim=0.2, load=0.0), extras=False)
    # small cases of each distribution, ragged image sizes, SH 0..3, paper loss weights
    p, cam = _small(0, 600, 64, 48, view=3)
    run_case("c0_small_bg", p, cam, bg=(0.1, 0.2, 0.3))
    p, cam = _small(1, 1500, 96, 80, view=1)
    run_case("c1_small", p, cam, bg=(0.0, 0.0, 0.0), extras=False)
    p, cam = _small(2, 3000, 160, 90, view=5)
    run_case("c2_small", p, cam, bg=(0.2, 0.1, 0.0), extras=False)
    for deg in (1, 2):
        p, cam = _small(1, 400, 50, 37, view=2 + deg)
        k = (deg + 1) ** 2
        p.sh = np.ascontiguousarray(p.sh[:, :, :k])
        run_case(f"sh{deg}_ragged", p, cam, bg=(0.3, 0.3, 0.3))
    # edge cases (test_rasterize.py:70-154 analogues)
    eye = np.eye(3)
    from paper_2503_13086_b200.camera import CameraFrame
    cam = CameraFrame(1, 20, 12, 15.0, 15.0, 10.0, 6.0, eye, np.zeros(3))
    run_case("edge_empty", _edge_params(np.zeros((0, 3)), 0.0, 0.0, np.zeros((0, 3))), cam,
             bg=(0.2, 0.4, 0.6), densify=False)
    cam = CameraFrame(1, 16, 16, 20.0, 20.0, 8.0, 8.0, eye, np.zeros(3))
    run_case("edge_behind", _edge_params([[0.0, 0.0, -5.0]], 0.0, 0.0, [[1.0, 0.0, 0.0]]), cam,
             bg=(0.0, 0.0, 0.0))
    cam = CameraFrame(1, 32, 32, 40.0, 40.0, 16.0, 16.0, eye, np.zeros(3))
    wall = [[0.0, 0.0, 4.0 + 0.1 * i] for i in range(8)]
    run_case("edge_wall", _edge_params(wall, np.log(2.0), 40.0, [[1.0, 1.0, 1.0]] * 8), cam,
             bg=(0.0, 0.0, 0.0))
    cam = CameraFrame(1, 33, 33, 40.0, 40.0, 16.0, 16.0, eye, np.zeros(3))
    run_case("edge_center", _edge_params([[0.0, 0.0, 5.0]], np.log(0.5), 0.0, [[1.0, 1.0, 1.0]]), cam,
             bg=(0.0, 0.0, 0.0))
    # needle-like (near-singular conic) splats + coincident duplicates (depth ties)
    rng = np.random.default_rng(5)
    n = 40
    pos = np.concatenate([rng.uniform(-0.5, 0.5, (n, 3)) + [0, 0, 3.0], np.tile([[0.1, -0.1, 3.5]], (4, 1))])
    p = _edge_params(pos, -2.0, 1.0, rng.uniform(0.1, 0.9, (n + 4, 3)))
    p.log_scales[:n, 0] = 0.5
    p.log_scales[:n, 1] = -7.0
    p.rotations = rng.standard_normal((n + 4, 4)).astype(np.float32)
    rot, tr = look_at([0.2, -0.1, 0.0], [0.0, 0.0, 3.0])
    cam = CameraFrame(1, 64, 48, 60.0, 60.0, 32.0, 24.0, rot, tr)
    run_case("edge_needles_ties", p, cam, bg=(0.05, 0.05, 0.05))
    expansion_case()


if __name__ == "__main__":
    main()
