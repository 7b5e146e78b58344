"""Guard-band sweep: flagged pixels and UNFLAGGED decision flips vs the fp64
oracle for several configs/views/bands (flips must be 0 for parity)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_2503_13086_b200 import GaussianField, scenes  # noqa: E402
from paper_2503_13086_b200.rasterize import render  # noqa: E402

CLS = ("positions", "rotations", "log_scales", "opacity_logits", "sh")
bands = [(1e-4, 2e-4), (3e-5, 1e-4), (1e-5, 5e-5), (3e-6, 2e-5), (1e-6, 1e-5), (0.0, 0.0)]
for cfg, views in ((1, (0, 1, 2)), (2, (1, 9, 17)), (0, (0, 5))):
    hp = scenes.make_params(cfg, seed=0)
    P = oracle.Params(*(getattr(hp, k).astype(np.float64) for k in CLS))
    f = GaussianField.from_host(hp)
    for v in views:
        cam = scenes.camera(cfg, view=v)
        ref = oracle.render(P, cam)
        for ba, bt in bands:
            out = render(f, cam, band=ba, band_t=bt)
            fl = out.flagged.cpu().numpy().astype(bool)
            flips = np.zeros_like(fl)
            for k in ("n_walk", "terminated", "hard_count"):
                flips |= getattr(out, k).cpu().numpy().astype(np.int64) != ref[k].astype(np.int64)
            img = np.abs(out.image.cpu().numpy() - ref["image"]).max()
            print(json.dumps({"cfg": cfg, "view": v, "band_a": ba, "band_t": bt, "flagged": int(fl.sum()),
                              "flips_unflagged": int((flips & ~fl).sum()), "flips_total": int(flips.sum()),
                              "img_max_abs": float(img)}), flush=True)
