"""One config-2 training iteration for ncu captures (no timing, no oracle).

  ncu --set full -k regex:k_backward_splat -c 1 -o prof python tools/profile_step.py
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2503_13086_b200 import GaussianField, scenes  # noqa: E402
from paper_2503_13086_b200.losses import LossWeights, total_loss  # noqa: E402
from paper_2503_13086_b200.optim import FieldOptimizer  # noqa: E402
from paper_2503_13086_b200.rasterize import backward, render  # noqa: E402

cfg = int(os.environ.get("SSR_CFG", "2"))
iters = int(os.environ.get("SSR_ITERS", "2"))
hp = scenes.make_params(cfg, seed=0)
cam = scenes.camera(cfg, view=8)
f = GaussianField.from_host(hp)
opt = FieldOptimizer(f, scene_extent=6.6)
target = torch.full((cam.height, cam.width, 3), 0.5, device="cuda")
for _ in range(iters):
    w = LossWeights() if os.environ.get("SSR_WEIGHTS") == "paper" else LossWeights(l1=1.0, ssim=0.2, load=0.0)
    out = render(f, cam, soft_count=w.load > 0)  # as train.train_iteration does
    br = total_loss(out.image, target, out, w)
    if os.environ.get("SSR_FUSED") == "1":
        from paper_2503_13086_b200.rasterize.backward import backward_and_step

        backward_and_step(f, out, br.d_image, br.d_soft, opt, 1.6e-4)
    else:
        g = backward(f, out, br.d_image, br.d_soft)
        opt.step(f, g, position_rate=1.6e-4)
torch.cuda.synchronize()
print("flagged", int(out.flagged.sum()), "P", int(out.n_walk.sum()), "M", out.splats.n_instances)
