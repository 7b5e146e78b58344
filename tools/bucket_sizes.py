import sys, json, torch
sys.path.insert(0, '.')
from paper_2503_13086_b200 import GaussianField, scenes
from paper_2503_13086_b200.rasterize import render
for cfg in (2, 4):
    f = GaussianField.from_host(scenes.make_params(cfg, seed=0))
    out = render(f, scenes.camera(cfg, view=8), soft_count=False)
    nw = out.n_walk.to(torch.int64)
    h, w = nw.shape
    th, tw = (h + 15) // 16, (w + 15) // 16
    pad = torch.zeros(th * 16, tw * 16, dtype=torch.int64, device=nw.device)
    pad[:h, :w] = nw
    tiles = pad.view(th, 16, tw, 16).permute(0, 2, 1, 3).reshape(th * tw, 256)
    P = int(nw.sum())
    res = {"cfg": cfg, "P": P}
    for B in (32, 64, 128):
        live = int(((tiles + B - 1) // B).sum())
        nb = int(((tiles.max(dim=1).values + B - 1) // B).sum())
        evals = B * (live + 31 * nb)
        res[B] = {"live": live, "nb": nb, "pair_evals": evals, "eff": P / evals}
    print(json.dumps(res))
