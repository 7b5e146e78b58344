"""Two views of config 4 accumulated into one FieldGrads (the semi-global batch
path, backward(accumulate=True)) for ncu captures of the accumulate-mode chain.
  ncu --set full -k regex:k_chain -s 2 -c 3 -o prof python tools/profile_accum.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_13086_b200 import GaussianField, scenes  # noqa: E402
from paper_2503_13086_b200.losses import LossWeights, total_loss  # noqa: E402
from paper_2503_13086_b200.rasterize import FieldGrads, backward, render  # noqa: E402

cfg = int(os.environ.get("SSR_CFG", "4"))
f = GaussianField.from_host(scenes.make_params(cfg, seed=0))
g = FieldGrads.zeros(len(f), f.sh_degree, f.flat.device)
w = LossWeights(l1=1.0, ssim=0.2, load=0.0)
for v in (8, 9, 10):
    cam = scenes.camera(cfg, view=v)
    out = render(f, cam, soft_count=False)
    br = total_loss(out.image, torch.full((cam.height, cam.width, 3), 0.5, device="cuda"), out, w)
    backward(f, out, br.d_image, None, grads=g, accumulate=True)
torch.cuda.synchronize()
print("ok")
