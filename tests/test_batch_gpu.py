"""Multi-view batches and densify bookkeeping on the CUDA path vs the reference semantics.

* SemiGlobalBatch / backward(accumulate=True): the summed gradient of a view
  batch equals the sum over views of the float64 oracle's backward at fixed
  parameters (SURVEY 8e parity), including screen_norms and the per-row
  visible count that densify consumes (pipeline.py:201-202).
* The chain kernel's fused statistics (``stats=``) equal the oracle's
  screen_norms / visible summed over iterations.
* densify_and_prune(optimizer=) remaps the Adam moments exactly like the
  reference's FieldOptimizer.sync -> AdamBuffer.remap (optim.py:49-54,
  101-111): kept rows keep their moments in order, appended rows start at 0.
"""

import numpy as np
import pytest

from parity import GRAD_CLASSES, grads_ok, grads_report, rel_l2

pytestmark = pytest.mark.gpu


def _views(n_views, w=160, h=120):
    from paper_2503_13086_b200 import scenes

    return [scenes.camera(1, view=v, width=w, height=h) for v in range(n_views)]


@pytest.mark.parametrize("world", [1, 2])
def test_semi_global_batch_equals_sum_over_views(world, oracle_lib):
    import torch

    from paper_2503_13086_b200 import GaussianField, scenes
    from paper_2503_13086_b200.losses import LossWeights, total_loss
    from paper_2503_13086_b200.optim import FieldOptimizer
    from paper_2503_13086_b200.rasterize import FieldGrads, backward, render
    from paper_2503_13086_b200.train import SemiGlobalBatch, TrainState

    hp = scenes.make_params(1, seed=12, n=20000)
    cams = _views(4)
    gen = torch.Generator("cuda").manual_seed(4)
    targets = [torch.rand((120, 160, 3), device="cuda", generator=gen) for _ in cams]
    weights = LossWeights()  # paper objective: d_soft != 0 exercises the soft-count backward
    P = oracle_lib.Params(*(getattr(hp, k).astype(np.float64) for k in GRAD_CLASSES))
    n = len(hp)
    want = {k: 0.0 for k in GRAD_CLASSES}
    want_norms, want_vis = np.zeros(n), np.zeros(n)
    f0 = GaussianField.from_host(hp)
    for cam, tgt in zip(cams, targets):
        out = render(f0, cam)
        br = total_loss(out.image, tgt, out, weights)
        ref = oracle_lib.render(P, cam)
        g = oracle_lib.backward(P, ref, br.d_image.cpu().numpy().astype(np.float64),
                                br.d_soft.cpu().numpy().astype(np.float64))
        for k in GRAD_CLASSES:
            want[k] = want[k] + g[k]
        want_norms += g["screen_norms"]
        want_vis += g["visible"]
    want["screen_norms"], want["visible"] = want_norms, want_vis > 0

    # each "rank" sums its shard; the all-reduce is the sum of the shard buffers
    total = None
    f = GaussianField.from_host(hp)
    for rank in range(world):
        st = TrainState(field=f, optimizer=FieldOptimizer(f, 3.0), weights=weights, densify_enabled=False)
        flat_before = f.flat.clone()
        grads, losses = SemiGlobalBatch(st).step(cams, targets, [1e-4] * len(cams), rank=rank, world=world)
        assert len(losses) == len(cams) // world
        total = grads.flat.clone() if total is None else total + grads.flat
        f.flat.copy_(flat_before)  # every rank starts from the same replica
    gsum = FieldGrads(_flat=total, _n=n, _k=f.n_sh_coeffs)
    r = grads_report(gsum, want)
    assert grads_ok(r), r
    np.testing.assert_array_equal(gsum.visible_count.cpu().numpy(), want_vis)


def test_fused_grad_statistics_equal_oracle_sums(oracle_lib):
    """stats= of backward (the chain kernel's fused grad_accum / grad_count) vs
    the oracle's screen_norms / visible summed over three views."""
    import torch

    from paper_2503_13086_b200 import GaussianField, scenes
    from paper_2503_13086_b200.rasterize import backward, render

    hp = scenes.make_params(1, seed=13, n=15000)
    f = GaussianField.from_host(hp)
    n = len(f)
    P = oracle_lib.Params(*(getattr(hp, k).astype(np.float64) for k in GRAD_CLASSES))
    stats = torch.zeros(2 * n, dtype=torch.float32, device="cuda")
    acc, cnt = np.zeros(n), np.zeros(n)
    rng = np.random.default_rng(2)
    for cam in _views(3, 144, 96):
        out = render(f, cam)
        d_img = (rng.standard_normal((96, 144, 3)) * 1e-3).astype(np.float32)
        backward(f, out, d_img, None, stats=stats)
        ref = oracle_lib.render(P, cam)
        g = oracle_lib.backward(P, ref, d_img.astype(np.float64), np.zeros((96, 144)))
        acc += g["screen_norms"]
        cnt += g["visible"]
    s = stats.cpu().numpy()
    assert rel_l2(s[:n], acc) <= 1e-3
    np.testing.assert_array_equal(s[n:], cnt)


@pytest.mark.parametrize("seed", [0, 1])
def test_densify_moment_remap_matches_reference_sync(seed):
    """densify_and_prune(optimizer=) == densify_and_prune + the reference's
    sync (AdamBuffer.remap: moments[keep] then zeros for n_added rows)."""
    import torch

    from paper_2503_13086_b200 import GaussianField, scenes
    from paper_2503_13086_b200.field import CLASSES, DensifyOptions
    from paper_2503_13086_b200.optim import FieldOptimizer

    hp = scenes.make_params(1, seed=20 + seed, n=5003)
    hp.opacity_logits[::7] = -7.0  # prune candidates
    rng = np.random.default_rng(seed)
    stats = rng.uniform(0.0, 4e-4, len(hp)).astype(np.float32)  # ~half are hot
    opts = DensifyOptions(scene_extent=2.0, percent_dense=0.015)  # threshold ~ the median scale

    f = GaussianField.from_host(hp)
    opt = FieldOptimizer(f, 2.0)
    gen = torch.Generator("cuda").manual_seed(seed)
    opt.m.copy_(torch.randn(opt.m.shape, device="cuda", generator=gen))
    opt.v.copy_(torch.rand(opt.v.shape, device="cuda", generator=gen))
    opt.steps = {k: 7 + i for i, k in enumerate(CLASSES)}
    before = {k: [t.cpu().numpy().copy() for t in opt.moments(k)] for k in CLASSES}
    s = f.densify_and_prune(stats, opts, np.random.default_rng(99), optimizer=opt)
    assert s.cloned > 0 and s.split > 0 and s.pruned > 0, s
    assert opt.n_rows == len(f) == int(s.keep_mask.sum()) + s.n_added
    assert opt.steps == {k: 7 + i for i, k in enumerate(CLASSES)}  # step counters are not reset
    for k in CLASSES:
        for old, new in zip(before[k], opt.moments(k)):
            tail = old.shape[1:]
            want = np.concatenate([old[s.keep_mask], np.zeros((s.n_added,) + tail, old.dtype)])
            np.testing.assert_array_equal(new.cpu().numpy(), want, err_msg=k)
    # and the same parameters as densify followed by the host-side sync
    f2 = GaussianField.from_host(hp)
    s2 = f2.densify_and_prune(stats, opts, np.random.default_rng(99))
    assert (s2.cloned, s2.split, s2.pruned) == (s.cloned, s.split, s.pruned)
    assert torch.equal(f.flat, f2.flat)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_adam_range_chunks_equal_full_adam(world):
    """ssr_adam_range over a sharded step's chunks (each with only its chunk of
    the gradients, grads_offset = lo) + the tail == one full ssr_adam."""
    import torch

    from paper_2503_13086_b200 import GaussianField, _lib, scenes
    from paper_2503_13086_b200.optim import SH_REST_LR, FieldOptimizer
    from paper_2503_13086_b200.rasterize import FieldGrads
    from paper_2503_13086_b200.train import shard_layout

    hp = scenes.make_params(1, seed=31, n=10007)
    fa, fb = GaussianField.from_host(hp), GaussianField.from_host(hp)
    oa, ob = FieldOptimizer(fa, 2.0), FieldOptimizer(fb, 2.0)
    gen = torch.Generator("cuda").manual_seed(world)
    for o in (oa, ob):
        o.m.copy_(torch.randn(o.m.shape, device="cuda", generator=torch.Generator("cuda").manual_seed(1)))
        o.v.copy_(torch.rand(o.v.shape, device="cuda", generator=torch.Generator("cuda").manual_seed(2)))
    g = FieldGrads.zeros(len(fa), fa.sh_degree, fa.flat.device)
    g.flat.copy_(torch.randn(g.flat.shape, device="cuda", generator=gen))
    oa.step(fa, g, position_rate=1e-4)
    lr, bc1, bc2 = ob.advance(1e-4)
    p = fb.flat.numel()
    chunk, main = shard_layout(p, world)
    pieces = [(r * chunk, (r + 1) * chunk, g.flat[r * chunk:(r + 1) * chunk].clone(), r * chunk) for r in range(world)]
    pieces.append((main, p, g.flat, 0))
    for lo, hi, gt, goff in pieces:
        _lib.call("ssr_adam_range", len(fb), fb.sh_degree, fb.flat.data_ptr(), gt.data_ptr(), goff, ob.m.data_ptr(),
                  ob.v.data_ptr(), lo, hi, lr, SH_REST_LR, bc1, bc2, _lib.stream_ptr())
    torch.cuda.synchronize()
    assert torch.equal(fa.flat, fb.flat) and torch.equal(oa.m, ob.m) and torch.equal(oa.v, ob.v)


@pytest.mark.slow
def test_config4_batch_gradients_vs_oracle(oracle_lib):
    """Config 4 at full size (3M Gaussians, SH3, 1080p): a two-view semi-global
    batch's summed gradients vs the sum of the float64 oracle's per-view
    backwards (SURVEY 8e parity at the config's scale), with projections and
    renders of both views checked on the way."""
    import torch

    from paper_2503_13086_b200 import GaussianField, scenes
    from paper_2503_13086_b200.rasterize import FieldGrads, backward, render
    from parity import forward_ok, forward_report, projection_report

    hp = scenes.make_params(4, seed=0)
    f = GaussianField.from_host(hp)
    P = oracle_lib.Params(*(getattr(hp, k).astype(np.float64) for k in GRAD_CLASSES))
    rng = np.random.default_rng(7)
    grads = FieldGrads.zeros(len(f), f.sh_degree, f.flat.device)
    want = {k: 0.0 for k in GRAD_CLASSES}
    want_norms, want_vis = 0.0, 0.0
    for v in (5, 37):
        cam = scenes.camera(4, view=v)
        out = render(f, cam)
        ref = oracle_lib.render(P, cam)
        pr = projection_report(out.splats, ref["splats"])
        assert all(x for k, x in pr.items() if k.endswith("_equal")), pr
        fr = forward_report(out, ref)
        assert forward_ok(fr), fr
        d_img = (rng.standard_normal((cam.height, cam.width, 3)) * 1e-6).astype(np.float32)
        d_soft = (rng.standard_normal((cam.height, cam.width)) * 1e-7).astype(np.float32)
        backward(f, out, d_img, d_soft, grads=grads, accumulate=True)
        g = oracle_lib.backward(P, ref, d_img.astype(np.float64), d_soft.astype(np.float64))
        for k in GRAD_CLASSES:
            want[k] = want[k] + g[k]
        want_norms = want_norms + g["screen_norms"]
        want_vis = want_vis + g["visible"].astype(np.float64)
        del out, ref
    torch.cuda.synchronize()
    want["screen_norms"], want["visible"] = want_norms, want_vis > 0
    r = grads_report(grads, want)
    assert grads_ok(r), r
    np.testing.assert_array_equal(grads.visible_count.cpu().numpy(), want_vis)
