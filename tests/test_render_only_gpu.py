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
