"""Pin the CPU oracle (oracle/) to golden vectors made by the reference itself.

The fixtures come from tests/golden/make_golden.py, which runs the unmodified
reference package (splatstream) on seeded inputs.  Integer/index outputs must
match exactly; float64 outputs agree to ~1e-10 (only libm exp and summation
order differ between numpy/numba and the C restatement).
"""

import numpy as np
import pytest

from conftest import golden_camera, golden_names, golden_params, load_golden

NAMES = golden_names()


def _close(a, b, rtol=1e-9, atol=1e-12, what=""):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    if a.size:
        scale = max(np.abs(b).max(), 1e-300)
        err = np.abs(a - b).max()
        assert err <= atol + rtol * scale, f"{what}: max err {err:.3e} (scale {scale:.3e})"


@pytest.mark.parametrize("name", NAMES)
def test_projection_and_binning(oracle_lib, name):
    g = load_golden(name)
    sp = oracle_lib.project_field(golden_params(g), golden_camera(g))
    for k in ("gauss_index", "inst_splat", "tile_starts", "tile_ends", "sh_lo", "sh_hi"):
        np.testing.assert_array_equal(np.asarray(sp[k]), g[f"proj_{k}"], err_msg=k)
    for k in ("means2d", "conics", "depths", "radii", "colors", "opacities", "cam_points", "clamp_mul",
              "cov2d", "cov3d_cam", "sh_dirs", "sh_radii"):
        _close(sp[k], g[f"proj_{k}"], what=k)


@pytest.mark.parametrize("name", NAMES)
def test_forward(oracle_lib, name):
    g = load_golden(name)
    out = oracle_lib.render(golden_params(g), golden_camera(g), bg=g["bg"])
    for k in ("n_walk", "terminated", "hard_count"):
        np.testing.assert_array_equal(out[k], g[f"out_{k}"], err_msg=k)
    for k in ("image", "t_final", "soft_count"):
        _close(out[k], g[f"out_{k}"], rtol=0, atol=1e-11, what=k)


@pytest.mark.parametrize("name", [n for n in NAMES if "loss_total" in load_golden(n)])
def test_loss(oracle_lib, name):
    g = load_golden(name)
    out = oracle_lib.render(golden_params(g), golden_camera(g), bg=g["bg"])
    w = oracle_lib.LossWeights(*g["loss_weights"])
    br = oracle_lib.total_loss(g["out_image"], g["target"], g["out_soft_count"], g["out_hard_count"], w)
    for k in ("l1", "ssim", "load", "total"):
        assert br[k if k != "ssim" else "ssim_loss"] == pytest.approx(float(g[f"loss_{k}"]), rel=1e-10, abs=1e-13)
    _close(br["d_image"], g["loss_d_image"], rtol=1e-9, what="d_image")
    _close(br["d_soft"], g["loss_d_soft"], rtol=1e-9, what="d_soft")
    assert out["image"].shape == g["out_image"].shape


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("layout", ["splat", "pixel"])
def test_backward(oracle_lib, name, layout):
    g = load_golden(name)
    if f"grad_{layout}_positions" not in g:
        pytest.skip("layout not recorded for this case")
    P = golden_params(g)
    out = oracle_lib.render(P, golden_camera(g), bg=g["bg"])
    gr = oracle_lib.backward(P, out, g["bwd_d_image"], g["bwd_d_soft"], layout=layout)
    np.testing.assert_array_equal(gr["visible"], g[f"grad_{layout}_visible"])
    for k in ("positions", "rotations", "log_scales", "opacity_logits", "sh", "screen_norms"):
        _close(gr[k], g[f"grad_{layout}_{k}"], rtol=1e-8, atol=1e-15, what=k)


@pytest.mark.parametrize("name", [n for n in NAMES if "adam_positions" in load_golden(n)])
def test_adam_step(oracle_lib, name):
    g = load_golden(name)
    P = golden_params(g)
    # Adam normalises every element, so feed the reference's own gradients
    gr = {k: g[f"grad_splat_{k}"] for k in ("positions", "rotations", "log_scales", "opacity_logits", "sh")}
    opt = oracle_lib.Optimizer(P, scene_extent=float(g["adam_extent"]))
    opt.step(P, gr, position_rate=float(g["adam_rate"]))
    for k in ("positions", "rotations", "log_scales", "opacity_logits", "sh"):
        _close(getattr(P, k), g[f"adam_{k}"], rtol=1e-12, atol=1e-14, what=k)


@pytest.mark.parametrize("name", [n for n in NAMES if "dens_keep" in load_golden(n)])
def test_densify(oracle_lib, name):
    g = load_golden(name)
    o = g["dens_opts"]
    opts = oracle_lib.DensifyOptions(*o)
    new, cl, sp, pr, keep, n_added = oracle_lib.densify_and_prune(
        golden_params(g), g["dens_stats"], opts, np.random.default_rng(11))
    np.testing.assert_array_equal([cl, sp, pr, n_added], g["dens_counts"])
    np.testing.assert_array_equal(keep, g["dens_keep"])
    for k in ("positions", "rotations", "log_scales", "opacity_logits", "sh"):
        _close(getattr(new, k), g[f"dens_{k}"], rtol=1e-14, atol=1e-15, what=k)
