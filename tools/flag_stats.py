"""Distribution of guard-band flagged pixels over tiles (config 2)."""
import os, sys
sys.path.insert(0, "/root/repo")
import torch, numpy as np
from paper_2503_13086_b200 import GaussianField, scenes
from paper_2503_13086_b200.rasterize import render
hp = scenes.make_params(2, seed=0)
f = GaussianField.from_host(hp)
for v in (8, 1):
    cam = scenes.camera(2, view=v)
    out = render(f, cam)
    ti = out.tile_info.view(-1, 4).cpu().numpy() if hasattr(out, "tile_info") else None

    if ti is not None:
        nf = ti[:, 1]; nx = ti[:, 0]
        print("view", v, "tiles", len(nf), "flagged tiles", (nf > 0).sum(), "flagged px", nf.sum())
        print("nflag hist", np.histogram(nf[nf > 0], bins=[1, 2, 4, 8, 16, 32, 64, 128, 257])[0])
        print("top tiles (nflag, maxwalk)", sorted(zip(nf.tolist(), nx.tolist()))[-10:])
        print("buckets of flagged tiles: sum", ((nx[nf > 0] + 31) // 32).sum(), "max", ((nx + 31) // 32).max())
