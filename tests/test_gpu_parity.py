"""CUDA path vs the reference: golden vectors (made by the reference itself) and
the float64 oracle at full BASELINE.json sizes.  Calls go through the same
C ABI (libssr.so) the Python operator API uses."""

import numpy as np
import pytest

from conftest import golden_camera, golden_names, load_golden
from parity import GRAD_CLASSES, forward_ok, forward_report, grads_ok, grads_report, projection_report, rel_l2

pytestmark = pytest.mark.gpu

NAMES = golden_names()


def _field(g, prefix="in_"):
    from paper_2503_13086_b200 import GaussianField

    return GaussianField.from_arrays(*(g[prefix + k].astype(np.float32) for k in (
        "positions", "rotations", "log_scales", "opacity_logits", "sh")))


def _ref(g, prefix):
    return {k[len(prefix):]: v for k, v in g.items() if k.startswith(prefix)}


@pytest.mark.parametrize("name", NAMES)
def test_projection_bit_exact(name):
    from paper_2503_13086_b200.rasterize import project_field

    g = load_golden(name)
    sp = project_field(_field(g), golden_camera(g))
    r = projection_report(sp, _ref(g, "proj_"))
    assert all(v for k, v in r.items() if k.endswith("_equal")), r
    if sp.n_visible:
        np.testing.assert_allclose(sp.means2d.cpu().numpy(), g["proj_means2d"], rtol=1e-12, atol=1e-9)
        np.testing.assert_allclose(sp.conics.cpu().numpy(), g["proj_conics"], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(sp.colors.cpu().numpy(), g["proj_colors"], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(sp.depths.cpu().numpy(), g["proj_depths"], rtol=1e-13)
        np.testing.assert_array_equal(sp.radii.cpu().numpy(), g["proj_radii"])
        np.testing.assert_array_equal(sp.sh_lo.cpu().numpy(), g["proj_sh_lo"])
        np.testing.assert_allclose(sp.cov3d_cam.cpu().numpy(), g["proj_cov3d_cam"], rtol=1e-9, atol=1e-14)


@pytest.mark.parametrize("name", NAMES)
def test_forward_parity(name):
    from paper_2503_13086_b200.rasterize import render

    g = load_golden(name)
    out = render(_field(g), golden_camera(g), bg=g["bg"])
    r = forward_report(out, _ref(g, "out_"))
    assert forward_ok(r), r


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("layout", ["splat", "pixel"])
def test_backward_parity(name, layout):
    from paper_2503_13086_b200.rasterize import backward, render

    g = load_golden(name)
    f = _field(g)
    out = render(f, golden_camera(g), bg=g["bg"])
    gr = backward(f, out, g["bwd_d_image"], g["bwd_d_soft"], layout=layout)
    r = grads_report(gr, _ref(g, "grad_splat_"))
    assert grads_ok(r), r


@pytest.mark.parametrize("name", [n for n in NAMES if "loss_total" in load_golden(n)])
def test_loss_parity(name):
    from paper_2503_13086_b200.losses import LossWeights, total_loss
    from paper_2503_13086_b200.rasterize import render

    g = load_golden(name)
    out = render(_field(g), golden_camera(g), bg=g["bg"])
    br = total_loss(g["out_image"].astype(np.float32), g["target"].astype(np.float32), out,
                    LossWeights(*g["loss_weights"]))
    assert br.l1 == pytest.approx(float(g["loss_l1"]), rel=1e-5)
    assert br.ssim_loss == pytest.approx(float(g["loss_ssim"]), rel=1e-4, abs=1e-6)
    assert br.load == pytest.approx(float(g["loss_load"]), rel=1e-4, abs=1e-6)
    assert br.total == pytest.approx(float(g["loss_total"]), rel=1e-4)
    # the reference d_image is a sum of an exact L1 sign term and the SSIM term
    assert rel_l2(br.d_image, g["loss_d_image"]) < 1e-4
    assert rel_l2(br.d_soft, g["loss_d_soft"]) < 1e-3


@pytest.mark.parametrize("name", [n for n in NAMES if "adam_positions" in load_golden(n)])
def test_adam_parity(name):
    from paper_2503_13086_b200.optim import FieldOptimizer
    from paper_2503_13086_b200.rasterize import FieldGrads

    g = load_golden(name)
    f = _field(g)
    grads = FieldGrads(*(g[f"grad_splat_{k}"] for k in GRAD_CLASSES), g["grad_splat_screen_norms"],
                       g["grad_splat_visible"])
    opt = FieldOptimizer(f, scene_extent=float(g["adam_extent"]))
    opt.step(f, grads, position_rate=float(g["adam_rate"]))
    for k in GRAD_CLASSES:
        got = getattr(f, k).cpu().numpy().astype(np.float64)
        want = g[f"adam_{k}"]
        # float32 storage: one step moves each value by <= lr; compare the step itself
        step_want = want - g[f"in_{k}"]
        step_got = got - g[f"in_{k}"]
        if step_got.size == 0:
            continue
        assert np.abs(step_got - step_want).max() <= 1e-6 * max(1.0, np.abs(g[f"in_{k}"]).max()), k


@pytest.mark.parametrize("name", [n for n in NAMES if "dens_keep" in load_golden(n)])
def test_densify_parity(name):
    from paper_2503_13086_b200.field import DensifyOptions

    g = load_golden(name)
    f = _field(g)
    s = f.densify_and_prune(g["dens_stats"], DensifyOptions(*g["dens_opts"]), np.random.default_rng(11))
    np.testing.assert_array_equal([s.cloned, s.split, s.pruned, s.n_added], g["dens_counts"])
    np.testing.assert_array_equal(s.keep_mask, g["dens_keep"])
    for k in GRAD_CLASSES:
        np.testing.assert_allclose(getattr(f, k).cpu().numpy(), g[f"dens_{k}"], rtol=1e-6, atol=1e-6, err_msg=k)


# ---------------------------------------------------------------- full-size configs vs the oracle
@pytest.mark.slow
@pytest.mark.parametrize("cfg", [0, 1, 2])
def test_full_config_vs_oracle(cfg, oracle_lib):
    from paper_2503_13086_b200 import GaussianField, scenes
    from paper_2503_13086_b200.rasterize import backward, render

    hp = scenes.make_params(cfg, seed=0)
    cam = scenes.camera(cfg, view=1)
    P = oracle_lib.Params(*(getattr(hp, k).astype(np.float64) for k in GRAD_CLASSES))
    ref_out = oracle_lib.render(P, cam)
    f = GaussianField.from_host(hp)
    out = render(f, cam)
    pr = projection_report(out.splats, ref_out["splats"])
    assert all(v for k, v in pr.items() if k.endswith("_equal")), pr
    fr = forward_report(out, ref_out)
    assert forward_ok(fr), fr
    rng = np.random.default_rng(3)
    d_img = (rng.standard_normal((cam.height, cam.width, 3)) * 1e-6).astype(np.float32)
    d_soft = (rng.standard_normal((cam.height, cam.width)) * 1e-7).astype(np.float32)
    ref_g = oracle_lib.backward(P, ref_out, d_img.astype(np.float64), d_soft.astype(np.float64))
    gr = backward(f, out, d_img, d_soft)
    r = grads_report(gr, ref_g)
    assert grads_ok(r), r
    # the training configuration's path: no soft-count gradient (load weight 0,
    # d_soft all zero), where the backward skips pairs below 1/255
    ref_g0 = oracle_lib.backward(P, ref_out, d_img.astype(np.float64), np.zeros((cam.height, cam.width)))
    r0 = grads_report(backward(f, out, d_img, np.zeros((cam.height, cam.width), np.float32)), ref_g0)
    assert grads_ok(r0), r0
    r1 = grads_report(backward(f, out, d_img, None), ref_g0)
    assert grads_ok(r1), r1


# ---------------------------------------------------------------- field expansion
def test_expansion_spatial_index_and_insert():
    """GPU grid k-NN vs the reference's cKDTree results (golden: expansion.npz)."""
    from paper_2503_13086_b200 import GaussianField, SparsePoint
    from paper_2503_13086_b200.spatial import SpatialIndex, filter_new_points, median_nn_spacing

    g = load_golden("expansion")
    sparse = g["exp_existing_pos"]
    idx = SpatialIndex(sparse)
    np.testing.assert_allclose(idx.min_distance(g["exp_queries"]).cpu().numpy(), g["exp_min_dist"], rtol=1e-12)
    assert median_nn_spacing(sparse) == pytest.approx(float(g["exp_median_nn"]), rel=1e-12)
    cands = [SparsePoint(p, c) for p, c in zip(g["exp_cand_pos"], g["exp_cand_col"])]
    kept = filter_new_points(idx, cands, float(g["exp_threshold"]))
    np.testing.assert_array_equal([any(k is c for k in kept) for c in cands], g["exp_kept"])
    f = _field(g)
    g0 = f.generation
    assert f.insert_points(kept, init_opacity=0.1) == int(g["exp_n_inserted"])
    assert f.generation - g0 == int(g["exp_generation_delta"])
    for k in GRAD_CLASSES:
        np.testing.assert_allclose(getattr(f, k).cpu().numpy(), g[f"exp_after_{k}"], rtol=2e-6, atol=2e-7,
                                   err_msg=k)


def test_spatial_index_edge_cases():
    from paper_2503_13086_b200.spatial import SpatialIndex, knn_distances

    assert np.isinf(SpatialIndex(np.empty((0, 3))).min_distance([[1.0, 2.0, 3.0]]).cpu().numpy()).all()
    pts = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0]])
    np.testing.assert_array_equal(SpatialIndex(pts).min_distance(pts).cpu().numpy(), 0.0)
    rng = np.random.default_rng(21)
    pool = np.concatenate([rng.standard_normal((3000, 3)) * 0.05, rng.uniform(-50, 50, (200, 3))])
    q = np.concatenate([rng.standard_normal((100, 3)), rng.uniform(-80, 80, (50, 3))])
    got = knn_distances(pool, q, 4).cpu().numpy()
    brute = np.sort(np.sqrt(((q[:, None, :] - pool[None, :, :]) ** 2).sum(-1)), axis=1)[:, :4]
    np.testing.assert_allclose(got, brute, rtol=1e-12)


def test_iteration_after_densify_odd_row_count():
    """Unaligned class offsets (N not a multiple of 4) after densify must not break any kernel."""
    import torch

    from paper_2503_13086_b200 import GaussianField, scenes
    from paper_2503_13086_b200.field import DensifyOptions
    from paper_2503_13086_b200.losses import LossWeights
    from paper_2503_13086_b200.optim import FieldOptimizer
    from paper_2503_13086_b200.train import TrainState, densify, train_iteration

    hp = scenes.make_params(1, seed=5, n=4001)
    f = GaussianField.from_host(hp)
    cam = scenes.camera(1, view=2, width=160, height=96)
    st = TrainState(field=f, optimizer=FieldOptimizer(f, 2.0), weights=LossWeights(),
                    densify=DensifyOptions(grad_threshold=1e-9), densify_interval=2)
    target = torch.full((96, 160, 3), 0.3, device="cuda")
    for _ in range(5):
        br = train_iteration(st, cam, target, 1e-4)
    torch.cuda.synchronize()
    assert len(f) != 4001 and np.isfinite(br.total)
    assert bool(torch.isfinite(f.flat).all())


@pytest.mark.parametrize("deg,n", [(3, 20001), (0, 3000)])
def test_fused_chain_adam_matches_backward_then_step(deg, n):
    """backward_and_step == backward() + FieldOptimizer.step() (including invisible rows)."""
    import torch

    from paper_2503_13086_b200 import GaussianField, scenes
    from paper_2503_13086_b200.losses import LossWeights
    from paper_2503_13086_b200.optim import FieldOptimizer
    from paper_2503_13086_b200.train import TrainState, train_iteration

    hp = scenes.make_params(1 if deg == 3 else 0, seed=9, n=n)
    cam = scenes.camera(1 if deg == 3 else 0, view=3, width=200, height=120)
    target = torch.rand((120, 200, 3), device="cuda", generator=torch.Generator("cuda").manual_seed(0))
    states = []
    for fused in (False, True):
        f = GaussianField.from_host(hp)
        st = TrainState(field=f, optimizer=FieldOptimizer(f, 3.0), weights=LossWeights(), densify_enabled=False)
        for it in range(3):
            train_iteration(st, cam, target, 1e-4, fused=fused)
        states.append(st)
    torch.cuda.synchronize()
    a, b = states
    # Adam normalises each element, so rounding-order differences of near-zero
    # gradients can move a handful of elements by up to ~a step size; bound both
    for name, step in (("positions", 3e-4 * 3), ("rotations", 1e-3), ("log_scales", 5e-3),
                       ("opacity_logits", 0.05), ("sh", 2.5e-3)):
        pa, pb = getattr(a.field, name).cpu().numpy(), getattr(b.field, name).cpu().numpy()
        bad = ~np.isclose(pb, pa, rtol=2e-5, atol=2e-6)
        assert bad.mean() < 1e-3, (name, bad.mean())
        assert np.abs(pb - pa).max() <= 3 * step, name
    np.testing.assert_allclose(b.stats.cpu().numpy(), a.stats.cpu().numpy(), rtol=1e-5, atol=1e-8)


@pytest.mark.gpu
def test_loss_accepts_8bit_target():
    """total_loss with a uint8 target == with the float target value/255 (io/images.py)."""
    import torch

    from paper_2503_13086_b200 import GaussianField, scenes
    from paper_2503_13086_b200.losses import LossWeights, total_loss
    from paper_2503_13086_b200.rasterize import render

    f = GaussianField.from_host(scenes.make_params(0, seed=2, n=3000))
    out = render(f, scenes.camera(0, view=1, width=72, height=56))
    t8 = torch.randint(0, 256, (56, 72, 3), dtype=torch.uint8, device="cuda")
    tf = t8.float() * torch.tensor(1.0 / 255.0, dtype=torch.float32, device="cuda")
    for w in (LossWeights(), LossWeights(l1=1.0, ssim=0.2, load=0.0)):
        a, b = total_loss(out.image, t8, out, w), total_loss(out.image, tf, out, w)
        assert a.total == pytest.approx(b.total, rel=1e-6)
        assert float((a.d_image - b.d_image).abs().max()) <= 1e-6 * float(b.d_image.abs().max()) + 1e-12


def test_insert_arrays_matches_insert_points_and_skips_nonfinite():
    from paper_2503_13086_b200 import SparsePoint

    g = load_golden("expansion")
    pos, col = g["exp_cand_pos"], g["exp_cand_col"]
    f1, f2 = _field(g), _field(g)
    n1 = f1.insert_points([SparsePoint(p, c) for p, c in zip(pos, col)])
    bad_pos = np.concatenate([pos, [[np.nan, 0.0, 0.0]]])
    bad_col = np.concatenate([col, [[0.5, 0.5, 0.5]]])
    n2 = f2.insert_arrays(bad_pos, bad_col)
    assert n1 == n2 == len(pos)
    assert f1.checksum() == f2.checksum() and f1.generation == f2.generation


def test_optimizer_growth_keeps_moments_and_cold_starts_new_rows():
    import torch

    from paper_2503_13086_b200 import GaussianField, scenes
    from paper_2503_13086_b200.field import CLASSES
    from paper_2503_13086_b200.optim import FieldOptimizer

    f = GaussianField.from_host(scenes.make_params(1, seed=4, n=777))
    opt = FieldOptimizer(f, 2.0)
    opt.m.copy_(torch.rand_like(opt.m))
    opt.v.copy_(torch.rand_like(opt.v))
    before = {k: [t.clone() for t in opt.moments(k)] for k in CLASSES}
    n_add = f.insert_arrays(np.random.default_rng(1).normal(size=(13, 3)), np.full((13, 3), 0.5))
    opt.sync(f, np.ones(777, dtype=bool), n_add)
    assert opt.n_rows == len(f) == 790
    for k in CLASSES:
        for old, new in zip(before[k], opt.moments(k)):
            assert bool((new[:777] == old).all()) and bool((new[777:] == 0).all()), k


@pytest.mark.parametrize("case", ["deep_lists", "opaque_big", "low_opacity_deep"])
def test_stress_cases_vs_oracle(case, oracle_lib):
    """Long tile lists (many 256-splat batches, dozens of 32-slot buckets and
    checkpoints), large opaque splats (early termination, huge rect merges) and
    very low opacities (walks through whole lists): GPU vs the float64 oracle."""
    from paper_2503_13086_b200 import GaussianField, scenes
    from paper_2503_13086_b200.camera import CameraFrame, look_at
    from paper_2503_13086_b200.rasterize import backward, render

    rng = np.random.default_rng({"deep_lists": 11, "opaque_big": 12, "low_opacity_deep": 13}[case])
    n = 6000
    hp = scenes.make_params(1, seed=5, n=n)
    hp.positions[:] = rng.uniform(-0.6, 0.6, (n, 3)).astype(np.float32)
    if case == "deep_lists":
        hp.log_scales[:] = rng.normal(-1.6, 0.3, (n, 3)).astype(np.float32)
        hp.opacity_logits[:] = rng.normal(-3.0, 1.0, n).astype(np.float32)
    elif case == "opaque_big":
        hp.log_scales[:] = rng.normal(-1.0, 0.3, (n, 3)).astype(np.float32)
        hp.opacity_logits[:] = rng.normal(4.0, 1.0, n).astype(np.float32)
    else:
        hp.log_scales[:] = rng.normal(-1.3, 0.2, (n, 3)).astype(np.float32)
        hp.opacity_logits[:] = np.full(n, -6.5, np.float32)
    rot, tr = look_at(np.array([0.3, -0.2, -3.0]), np.zeros(3))
    cam = CameraFrame(1, 96, 80, 90.0, 90.0, 48.0, 40.0, rot, tr)
    P = oracle_lib.Params(*(getattr(hp, k).astype(np.float64) for k in GRAD_CLASSES))
    ref = oracle_lib.render(P, cam)
    f = GaussianField.from_host(hp)
    out = render(f, cam)
    assert all(v for k, v in projection_report(out.splats, ref["splats"]).items() if k.endswith("_equal"))
    fr = forward_report(out, ref)
    assert forward_ok(fr), fr
    assert int(out.n_walk.max()) > 300, "case does not produce deep walks"
    d_img = (rng.standard_normal((80, 96, 3)) * 1e-3).astype(np.float32)
    for d_soft in (None, (rng.standard_normal((80, 96)) * 1e-4).astype(np.float32)):
        ds = np.zeros((80, 96)) if d_soft is None else d_soft.astype(np.float64)
        ref_g = oracle_lib.backward(P, ref, d_img.astype(np.float64), ds)
        for layout in ("splat", "pixel"):
            r = grads_report(backward(f, out, d_img, d_soft, layout=layout), ref_g)
            assert grads_ok(r), (layout, d_soft is None, r)


def test_instance_capacity_reuse_and_growth():
    """Renders through the capacity path (buffers sized from the field's last
    instance count, ssr_bin_tiles_capacity) equal renders of a fresh field,
    both when M fits the capacity and when it outgrows it (fallback)."""
    import torch

    from paper_2503_13086_b200 import GaussianField, scenes
    from paper_2503_13086_b200.rasterize import render

    hp = scenes.make_params(1, seed=3, n=6000)
    small = scenes.camera(1, view=2, width=64, height=48)
    big = scenes.camera(1, view=2, width=320, height=240)

    def fields_equal(a, b):
        for k in ("image", "t_final", "n_walk", "terminated", "hard_count", "soft_count"):
            assert torch.equal(getattr(a, k), getattr(b, k)), k
        assert torch.equal(a.splats.inst_gauss, b.splats.inst_gauss)
        assert torch.equal(a.splats.tile_ranges, b.splats.tile_ranges)

    f = GaussianField.from_host(hp)
    r_small = render(f, small)  # sets the capacity hint
    assert getattr(f, "_m_hint", 0) >= r_small.splats.n_instances
    r_big = render(f, big)  # M outgrows the capacity: exact-size fallback
    r_big2 = render(f, big)  # now within the (grown) capacity
    ref_big = render(GaussianField.from_host(hp), big)
    ref_small = render(GaussianField.from_host(hp), small)
    r_small2 = render(f, small)  # capacity larger than M
    torch.cuda.synchronize()
    assert r_big.splats.n_instances > r_small.splats.n_instances
    fields_equal(r_big, ref_big)
    fields_equal(r_big2, ref_big)
    fields_equal(r_small2, ref_small)


def test_loss_values_into_pinned_host_memory():
    """total_loss(values_out=pinned host tensor): the kernel writes the scalar
    terms straight into mapped host memory; same values as the device buffer."""
    import torch

    from paper_2503_13086_b200 import GaussianField, scenes
    from paper_2503_13086_b200.errors import InvalidParameter
    from paper_2503_13086_b200.losses import LossWeights, total_loss
    from paper_2503_13086_b200.rasterize import render

    f = GaussianField.from_host(scenes.make_params(0, seed=4, n=3000))
    out = render(f, scenes.camera(0, view=2, width=80, height=64))
    tgt = torch.rand((64, 80, 3), device="cuda", generator=torch.Generator("cuda").manual_seed(1))
    w = LossWeights()
    ref = total_loss(out.image, tgt, out, w)
    host = torch.zeros(5, dtype=torch.float64).pin_memory()
    br = total_loss(out.image, tgt, out, w, values_out=host)
    for name in ("l1", "ssim_loss", "load", "total", "hard_count_std"):
        assert getattr(br, name) == getattr(ref, name), name
    assert torch.equal(br.d_image, ref.d_image) and torch.equal(br.d_soft, ref.d_soft)
    with pytest.raises(InvalidParameter):
        total_loss(out.image, tgt, out, w, values_out=torch.zeros(5, dtype=torch.float64))


def test_render_invariants_and_stale_render_rejected():
    """test_rasterize.py:109-118 invariants (image in [0, 1], T in (0, 1], hard <= n_walk,
    soft <= n_walk) and :254-259 (a render of an older field generation is rejected)."""
    import torch

    from paper_2503_13086_b200 import GaussianField, scenes
    from paper_2503_13086_b200.errors import StaleFieldError
    from paper_2503_13086_b200.rasterize import backward, render

    f = GaussianField.from_host(scenes.make_params(1, seed=6, n=20000))
    out = render(f, scenes.camera(1, view=4, width=200, height=150))
    img, t = out.image, out.t_final
    assert float(img.min()) >= 0.0 and float(img.max()) <= 1.0
    assert float(t.min()) > 0.0 and float(t.max()) <= 1.0
    nw = out.n_walk.to(torch.int64)
    assert bool((out.hard_count.to(torch.int64) <= nw).all())
    assert bool((out.soft_count <= nw.to(torch.float64) + 1e-9).all())
    f.insert_arrays(np.array([[0.0, 0.0, 1.0]]), np.array([[0.5, 0.5, 0.5]]))
    with pytest.raises(StaleFieldError):
        backward(f, out, torch.zeros_like(out.image))


def test_iteration_is_bit_deterministic():
    """Same state, same view: render + loss + fused backward/Adam twice give bit-identical
    parameters, moments and loss terms (the reference's worker-count invariance)."""
    import torch

    from paper_2503_13086_b200 import GaussianField, scenes
    from paper_2503_13086_b200.losses import LossWeights
    from paper_2503_13086_b200.optim import FieldOptimizer
    from paper_2503_13086_b200.train import TrainState, train_iteration

    hp = scenes.make_params(1, seed=8, n=30000)
    cam = scenes.camera(1, view=5, width=240, height=160)
    target = torch.rand((160, 240, 3), device="cuda", generator=torch.Generator("cuda").manual_seed(3))
    runs = []
    for _ in range(2):
        f = GaussianField.from_host(hp)
        st = TrainState(field=f, optimizer=FieldOptimizer(f, 3.0), weights=LossWeights(), densify_enabled=False)
        totals = [train_iteration(st, cam, target, 1e-4).total for _ in range(3)]
        torch.cuda.synchronize()
        runs.append((f.flat.clone(), st.optimizer.m.clone(), st.optimizer.v.clone(), totals))
    a, b = runs
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]) and torch.equal(a[2], b[2])
    assert a[3] == b[3]


def test_gradient_matches_finite_differences():
    """test_rasterize.py:158-191 style: for every parameter class, the directional
    derivative of a linear image functional along a random direction matches central
    differences of the CUDA forward.  Pixels whose discrete decisions (blend set,
    termination, guard-band flag) differ between the +eps / -eps renders are left out
    of both sides (the functional is masked before the backward); eps = 1e-4 keeps the
    position curvature term below the bar; relative 2e-2 plus an fp32 noise floor."""
    import torch

    from paper_2503_13086_b200 import GaussianField, scenes
    from paper_2503_13086_b200.field import class_slices
    from paper_2503_13086_b200.rasterize import backward, render

    hp = scenes.make_params(0, seed=11, n=400)
    cam = scenes.camera(0, view=2, width=64, height=48)
    f = GaussianField.from_host(hp)
    n, k = len(f), f.n_sh_coeffs
    gen = torch.Generator("cuda").manual_seed(5)
    w = torch.randn((48, 64, 3), device="cuda", generator=gen)
    base = f.flat.clone()
    out0 = render(f, cam)
    eps = 1e-4
    names = ("positions", "rotations", "log_scales", "opacity_logits", "sh")
    for (off, width), name in zip(class_slices(n, k), names):
        d = torch.zeros_like(base)
        d[off: off + width * n] = torch.randn(width * n, device="cuda", generator=gen)
        imgs, same = [], (out0.flagged == 0)
        for sgn in (1.0, -1.0):
            f.flat.copy_(base + sgn * eps * d)
            o = render(f, cam)
            imgs.append(o.image.double())
            same &= (o.n_walk == out0.n_walk) & (o.hard_count == out0.hard_count) & (o.flagged == 0)
            # a changed (tile, depth) order -- two splats swapping depth -- is a jump too
            for t in range(out0.splats.tiles_x * out0.splats.tiles_y):
                a0, a1 = (int(v) for v in out0.splats.tile_ranges[t])
                b0, b1 = (int(v) for v in o.splats.tile_ranges[t])
                if a1 - a0 != b1 - b0 or not torch.equal(out0.splats.inst_gauss[a0:a1], o.splats.inst_gauss[b0:b1]):
                    ty, tx = divmod(t, out0.splats.tiles_x)
                    same[ty * 16:(ty + 1) * 16, tx * 16:(tx + 1) * 16] = False
        f.flat.copy_(base)
        assert float(same.float().mean()) > 0.3, name
        wm = w * same[..., None].float()
        fd = float(((imgs[0] - imgs[1]) * wm.double()).sum()) / (2 * eps)
        g = backward(f, render(f, cam), wm)
        analytic = float((getattr(g, name).reshape(-1).double() * d[off: off + width * n].double()).sum())
        assert abs(fd - analytic) <= 2e-2 * abs(analytic) + 1e-2, (name, fd, analytic)


@pytest.mark.parametrize("w,h", [(200, 120), (2048, 1280), (3840, 2176), (4096, 4096)])
def test_tile_sort_all_tile_id_widths(w, h):
    """The stable tile sort splits the tile id's bits over its passes (one pass
    up to 256 tiles, 7 + 6 bits at 1080p, up to 8 + 8 at 65536 tiles): its
    instance order and ranges equal a plain stable sort of the depth-ordered
    duplicates by tile id (projection.py:184-191) at every id width."""
    import torch

    from paper_2503_13086_b200 import GaussianField, scenes
    from paper_2503_13086_b200.rasterize.projection import project_field

    f = GaussianField.from_host(scenes.make_params(1, seed=31, n=40000))
    cam = scenes.camera(1, view=2, width=w, height=h)
    sp = project_field(f, cam)
    tx, ty = sp.tiles_x, sp.tiles_y
    b = sp.bufs
    order = b["depth_order"][: sp.n].long()
    tiles = b["tiles"][: sp.n].long()
    rect = b["rect"][: sp.n].view(-1, 4).long()
    vis = order[tiles[order] > 0]  # visible rows in depth order
    # duplicates in depth order, each row's tiles ty-outer / tx-inner
    r = rect[vis]
    wd, cnt = r[:, 2] - r[:, 0], tiles[vis]
    idx = torch.repeat_interleave(torch.arange(vis.numel(), device=vis.device), cnt)
    first = torch.cumsum(cnt, 0) - cnt
    local = torch.arange(idx.numel(), device=vis.device) - first[idx]
    row, col = local // wd[idx], local % wd[idx]
    keys = (r[idx, 1] + row) * tx + r[idx, 0] + col
    vals = vis[idx].int()
    sk, perm = torch.sort(keys, stable=True)
    assert keys.numel() == sp.n_instances and int(tx * ty) > 0
    assert torch.equal(sp.inst_gauss, vals[perm])
    n_tiles = tx * ty
    t_ids = torch.arange(n_tiles, device=sk.device)
    starts = torch.searchsorted(sk, t_ids, right=False)
    ends = torch.searchsorted(sk, t_ids, right=True)
    ranges = sp.tile_ranges.long()
    assert torch.equal(ranges[:, 0], starts) and torch.equal(ranges[:, 1], ends)


def test_tile_sort_rejects_more_than_65536_tiles():
    from paper_2503_13086_b200 import GaussianField, scenes
    from paper_2503_13086_b200.errors import InvalidParameter
    from paper_2503_13086_b200.rasterize.projection import project_field

    f = GaussianField.from_host(scenes.make_params(1, seed=31, n=2000))
    with pytest.raises(InvalidParameter):
        project_field(f, scenes.camera(1, view=2, width=4112, height=4096))  # 257 x 256 tiles
