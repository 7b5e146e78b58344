"""The fused loss (ssr_loss) at image sizes that exercise its tiling edges:
the 11×11 minimum, widths that are not a multiple of 4 (the adjoint maps' row
padding for the backward's TMA tile loads), partial 32×32 tiles on both axes,
and 8-bit targets — against the float64 oracle (oracle/oracle.py total_loss,
losses.py:55-173), on seeded random images, soft and hard counts.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("h,w", [(11, 11), (37, 100), (70, 65), (33, 97), (64, 64), (45, 129)])
@pytest.mark.parametrize("u8", [0, 1])
def test_loss_matches_oracle_at_edge_sizes(oracle_lib, h, w, u8):
    import torch

    from paper_2503_13086_b200 import _lib

    rng = np.random.default_rng(h * 1000 + w + u8)
    img = rng.random((h, w, 3), dtype=np.float32)
    tgt8 = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
    tgt = tgt8 if u8 else rng.random((h, w, 3), dtype=np.float32)
    soft = rng.random((h, w)) * 40.0
    hard = rng.integers(0, 30, (h, w), dtype=np.int32)
    wts = (0.47, 0.12, 0.41)
    dev = torch.device("cuda")
    t_img, t_tgt = torch.from_numpy(img).to(dev), torch.from_numpy(tgt).to(dev)
    t_soft, t_hard = torch.from_numpy(soft).to(dev), torch.from_numpy(hard).to(dev)
    d_img = torch.empty_like(t_img)
    d_soft = torch.empty((h, w), device=dev)
    out = torch.empty(5, dtype=torch.float64, device=dev)
    ws = torch.empty(_lib.query("ssr_loss_workspace", w, h), dtype=torch.uint8, device=dev)
    ws.fill_(0xFF)  # NaN bit patterns: the maps' zero borders must be written by the kernels
    _lib.call("ssr_loss", w, h, t_img.data_ptr(), t_tgt.data_ptr(), u8, t_soft.data_ptr(), t_hard.data_ptr(), *wts,
              d_img.data_ptr(), d_soft.data_ptr(), out.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_ptr())
    torch.cuda.synchronize()
    tgt64 = tgt8.astype(np.float64) / 255.0 if u8 else tgt.astype(np.float64)
    ref = oracle_lib.total_loss(img.astype(np.float64), tgt64, soft, hard, oracle_lib.LossWeights(*wts))
    o = out.cpu().numpy()
    assert o[0] == pytest.approx(ref["l1"], rel=1e-5)
    assert o[1] == pytest.approx(ref["ssim_loss"], rel=1e-4, abs=1e-6)
    assert o[2] == pytest.approx(ref["load"], rel=1e-6)
    assert o[3] == pytest.approx(ref["total"], rel=1e-4)
    gi, gs = d_img.cpu().numpy().astype(np.float64), d_soft.cpu().numpy().astype(np.float64)
    assert np.isfinite(gi).all()
    assert np.linalg.norm(gi - ref["d_image"]) <= 1e-4 * np.linalg.norm(ref["d_image"])
    assert np.linalg.norm(gs - ref["d_soft"]) <= 1e-5 * np.linalg.norm(ref["d_soft"])


def test_loss_rejects_misaligned_workspace():
    import torch

    from paper_2503_13086_b200 import _lib
    from paper_2503_13086_b200.errors import InvalidParameter

    h, w = 32, 40
    dev = torch.device("cuda")
    img = torch.rand(h, w, 3, device=dev)
    hard = torch.zeros(h, w, dtype=torch.int32, device=dev)
    need = _lib.query("ssr_loss_workspace", w, h)
    ws = torch.empty(need + 64, dtype=torch.uint8, device=dev)
    out = torch.empty(5, dtype=torch.float64, device=dev)
    with pytest.raises(InvalidParameter, match="16-byte aligned"):
        _lib.call("ssr_loss", w, h, img.data_ptr(), img.data_ptr(), 0, None, hard.data_ptr(), 1.0, 0.2, 0.0,
                  torch.empty_like(img).data_ptr(), None, out.data_ptr(), ws.data_ptr() + 4, need, _lib.stream_ptr())
