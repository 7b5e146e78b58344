"""Render-only path (view_psnr, pipeline.py:180-182): the same
outputs as the training render, bit for bit, without the backward's bucket
checkpoints; such a render cannot be differentiated."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg,n,w,h", [(1, 30000, 320, 240), (2, 60000, 480, 270)])
def test_render_only_matches_training_render(cfg, n, w, h):
    import torch

    from paper_2503_13086_b200 import GaussianField, scenes
    from paper_2503_13086_b200.errors import InvalidParameter
    from paper_2503_13086_b200.rasterize import backward, render

    f = GaussianField.from_host(scenes.make_params(cfg, seed=3, n=n))
    cam = scenes.camera(cfg, view=5, width=w, height=h)
    full = render(f, cam)
    lite = render(f, cam, for_backward=False)
    torch.cuda.synchronize()
    assert lite.ckpt.numel() == 0 and full.ckpt.numel() > 0
    for k in ("image", "t_final", "n_walk", "terminated", "hard_count", "soft_count", "flagged"):
        assert torch.equal(getattr(full, k), getattr(lite, k)), k
    assert int(full.flagged.sum()) >= 0
    with pytest.raises(InvalidParameter):
        backward(f, lite, torch.zeros_like(lite.image))
    # the training render still differentiates after a render-only one
    g = backward(f, full, torch.full_like(full.image, 1e-3))
    assert bool(torch.isfinite(g.flat).all())
    np.testing.assert_array_less(0.0, float(g.positions.abs().sum()))


@pytest.mark.parametrize("cfg,n,w,h", [(1, 30000, 320, 240), (2, 60000, 480, 270)])
def test_render_without_soft_counts(cfg, n, w, h, oracle_lib):
    """render(soft_count=False): every output but the soft count identical to
    the full render and to the oracle; total_loss without the load term gives
    the same scalars and d_image; the gradients agree to rounding (d_soft is
    zero either way when the load weight is 0; without a d_soft the two-slot
    backward runs, whose rounding of w . C_front differs)."""
    import torch

    from paper_2503_13086_b200 import GaussianField, scenes
    from paper_2503_13086_b200.errors import InvalidParameter
    from paper_2503_13086_b200.losses import LossWeights, total_loss
    from paper_2503_13086_b200.optim import FieldOptimizer
    from paper_2503_13086_b200.rasterize import render
    from paper_2503_13086_b200.train import TrainState, train_iteration
    from parity import GRAD_CLASSES, forward_report

    hp = scenes.make_params(cfg, seed=4, n=n)
    f = GaussianField.from_host(hp)
    cam = scenes.camera(cfg, view=6, width=w, height=h)
    full = render(f, cam)
    lite = render(f, cam, soft_count=False)
    torch.cuda.synchronize()
    assert lite.soft_count is None
    for k in ("image", "t_final", "n_walk", "terminated", "hard_count", "flagged"):
        assert torch.equal(getattr(full, k), getattr(lite, k)), k
    ref = oracle_lib.render(oracle_lib.Params(*(getattr(hp, k).astype(np.float64) for k in GRAD_CLASSES)), cam)
    r = forward_report(full, ref)
    assert r["image_max_abs"] <= 1e-4 and r["n_walk_mismatch"] == 0 and r["hard_count_mismatch"] == 0, r
    tgt = torch.rand((h, w, 3), device="cuda", generator=torch.Generator("cuda").manual_seed(2))
    bw = LossWeights(l1=1.0, ssim=0.2, load=0.0)
    a, b = total_loss(full.image, tgt, full, bw), total_loss(lite.image, tgt, lite, bw)
    assert (a.l1, a.ssim_loss, a.load, a.total) == (b.l1, b.ssim_loss, b.load, b.total)
    assert torch.equal(a.d_image, b.d_image) and b.d_soft is None and float(a.d_soft.abs().max()) == 0.0
    with pytest.raises(InvalidParameter):
        total_loss(lite.image, tgt, lite, LossWeights())
    # the training iteration itself runs without soft counts (load weight 0)
    st = TrainState(field=GaussianField.from_host(hp), optimizer=None, weights=bw, densify_enabled=False)
    st.optimizer = FieldOptimizer(st.field, 3.0)
    assert np.isfinite(train_iteration(st, cam, tgt, 1e-4).total)
    # d_soft all zero on a soft-count frame vs d_soft None on a frame without
    # soft counts: the same decisions and contributions (the gradients are
    # compared, not trajectories: Adam's per-element normalisation would
    # amplify any rounding difference on near-zero gradients)
    from paper_2503_13086_b200.rasterize import backward

    f2 = GaussianField.from_host(hp)
    o1 = render(f2, cam)
    o2 = render(f2, cam, soft_count=False)
    d = torch.randn(o2.image.shape, device="cuda", generator=torch.Generator("cuda").manual_seed(5)) * 1e-3
    g1 = backward(f2, o1, d, torch.zeros(o1.image.shape[:2], device="cuda"))
    g2 = backward(f2, o2, d, None)
    # a frame without soft counts takes no soft-count gradient
    with pytest.raises(InvalidParameter):
        backward(f2, o2, d, torch.zeros(o2.image.shape[:2], device="cuda"))
    for k in ("positions", "rotations", "log_scales", "opacity_logits", "sh", "screen_norms"):
        a1, a2 = getattr(g1, k).double(), getattr(g2, k).double()
        assert float((a1 - a2).norm() / a1.norm().clamp_min(1e-30)) <= 1e-5, k
    assert torch.equal(g1.visible, g2.visible)


def _same_backward(f, full, lite):
    """The checkpoints the backward seeds from are the same: identical gradients."""
    import torch

    from paper_2503_13086_b200.rasterize import backward

    gen = torch.Generator("cuda").manual_seed(9)
    d = torch.randn(full.image.shape, device="cuda", generator=gen) * 1e-3
    ga, gb = backward(f, full, d), backward(f, lite, d)
    torch.cuda.synchronize()
    for k in ("positions", "rotations", "log_scales", "opacity_logits", "sh", "screen_norms", "visible"):
        assert torch.equal(getattr(ga, k), getattr(gb, k)), k  # the real rows (not the class-region padding)


def _golden_cases():
    from conftest import golden_names

    return golden_names()


@pytest.mark.parametrize("name", _golden_cases())
def test_no_soft_render_equals_full_render_on_golden_cases(name):
    """Every reference fixture (edge cases: empty, behind-camera, opaque walls,
    near-singular conics with ties, ragged sizes): the render without soft
    counts (per-splat far cut + warp-block reach masks) equals the full render
    on every other output, bit for bit."""
    import torch

    from conftest import golden_camera, load_golden
    from paper_2503_13086_b200 import GaussianField
    from paper_2503_13086_b200.rasterize import render

    g = load_golden(name)
    f = GaussianField.from_arrays(*(g["in_" + k].astype(np.float32) for k in (
        "positions", "rotations", "log_scales", "opacity_logits", "sh")))
    cam = golden_camera(g)
    full = render(f, cam, bg=g["bg"])
    lite = render(f, cam, bg=g["bg"], soft_count=False)
    torch.cuda.synchronize()
    for k in ("image", "t_final", "n_walk", "terminated", "hard_count", "flagged"):
        assert torch.equal(getattr(full, k), getattr(lite, k)), k
    _same_backward(f, full, lite)


@pytest.mark.parametrize("case", ["deep_lists", "opaque_big", "low_opacity_deep", "config2_1080p"])
def test_no_soft_render_equals_full_render_stress(case):
    import torch

    from paper_2503_13086_b200 import GaussianField, scenes
    from paper_2503_13086_b200.camera import CameraFrame, look_at
    from paper_2503_13086_b200.rasterize import render

    if case == "config2_1080p":
        hp = scenes.make_params(2, seed=0)
        cam = scenes.camera(2, view=8)
    else:
        rng = np.random.default_rng({"deep_lists": 11, "opaque_big": 12, "low_opacity_deep": 13}[case])
        n = 6000
        hp = scenes.make_params(1, seed=5, n=n)
        hp.positions[:] = rng.uniform(-0.6, 0.6, (n, 3)).astype(np.float32)
        ls, lo = {"deep_lists": (-1.6, -3.0), "opaque_big": (-1.0, 4.0), "low_opacity_deep": (-1.3, -6.5)}[case]
        hp.log_scales[:] = rng.normal(ls, 0.3, (n, 3)).astype(np.float32)
        hp.opacity_logits[:] = rng.normal(lo, 1.0, n).astype(np.float32)
        rot, tr = look_at(np.array([0.3, -0.2, -3.0]), np.zeros(3))
        cam = CameraFrame(1, 96, 80, 90.0, 90.0, 48.0, 40.0, rot, tr)
    f = GaussianField.from_host(hp)
    full = render(f, cam)
    lite = render(f, cam, soft_count=False)
    torch.cuda.synchronize()
    for k in ("image", "t_final", "n_walk", "terminated", "hard_count", "flagged"):
        assert torch.equal(getattr(full, k), getattr(lite, k)), k
    _same_backward(f, full, lite)
