"""Small end-to-end run of every entry point: render, loss, both backward
layouts, chain, Adam, fused chain+Adam, densify, PLY pack/unpack on config-0/1
sized scenes (a quick crash / error check: python tools/e2e_small.py)."""
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_13086_b200 import GaussianField, scenes  # noqa: E402
from paper_2503_13086_b200.field import DensifyOptions  # noqa: E402
from paper_2503_13086_b200.losses import LossWeights, total_loss  # noqa: E402
from paper_2503_13086_b200.optim import FieldOptimizer  # noqa: E402
from paper_2503_13086_b200.ply import read_ply, write_ply  # noqa: E402
from paper_2503_13086_b200.rasterize import backward, render  # noqa: E402
from paper_2503_13086_b200.rasterize.backward import backward_and_step  # noqa: E402

for cfg, n, w, h in ((0, 3000, 96, 80), (1, 6000, 120, 100)):
    hp = scenes.make_params(cfg, seed=3, n=n)
    cam = scenes.camera(cfg, view=2, width=w, height=h)
    f = GaussianField.from_host(hp)
    opt = FieldOptimizer(f, scene_extent=3.0)
    tgt = torch.rand((h, w, 3), device="cuda")
    for layout in ("splat", "pixel"):
        out = render(f, cam)
        br = total_loss(out.image, tgt, out, LossWeights())
        g = backward(f, out, br.d_image, br.d_soft, layout=layout)
        opt.step(f, g, position_rate=1e-4)
    out = render(f, cam)
    br = total_loss(out.image, tgt, out, LossWeights(l1=1.0, ssim=0.2, load=0.0))
    backward_and_step(f, out, br.d_image, br.d_soft, opt, 1e-4)
    stats = torch.rand(len(f), device="cuda") * 1e-3
    f.densify_and_prune(stats, DensifyOptions(scene_extent=3.0), np.random.default_rng(0), optimizer=opt)
    with tempfile.TemporaryDirectory() as d:
        write_ply(f, os.path.join(d, "s.ply"))
        assert read_ply(os.path.join(d, "s.ply")).checksum() == f.checksum()
torch.cuda.synchronize()
print("sanitize run ok")
