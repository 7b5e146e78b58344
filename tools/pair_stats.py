"""Walked-pair classes of one render (sampled tiles), to size per-pair work:
  far      power < -25 (soft term S0 only)
  small    alpha < 2.5e-3 (soft deviation only)
  mid      2.5e-3 <= alpha < 1/255 (exact sigmoid, not blended)
  blend    alpha >= 1/255 (blended)
plus, per 16x2 warp of the forward, the fraction of (warp, slot) pairs where
every walked pixel of the warp is far.
  python tools/pair_stats.py [config] [n_tiles_sampled]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def stats(out, n_sample=300, seed=0):
    import torch

    sp = out.splats
    dev = sp.tile_ranges.device
    ranges = sp.tile_ranges.long().cpu()
    n_tiles = ranges.shape[0]
    nonempty = torch.nonzero(ranges[:, 1] > ranges[:, 0]).flatten()
    g = torch.Generator().manual_seed(seed)
    pick = nonempty[torch.randperm(len(nonempty), generator=g)[:n_sample]]
    mean = sp.bufs["mean"].view(-1, 2)
    co = sp.bufs["conic_opa"].view(-1, 4).double()
    nw_img = out.n_walk
    h, w = nw_img.shape
    tot = dict(far=0, small=0, mid=0, blend=0)
    warp_pairs = warp_far = 0
    ys, xs = torch.meshgrid(torch.arange(16, device=dev), torch.arange(16, device=dev), indexing="ij")
    for t in pick.tolist():
        s0, s1 = int(ranges[t, 0]), int(ranges[t, 1])
        tx, ty = t % sp.tiles_x, t // sp.tiles_x
        px = (tx * 16 + xs).flatten().double()
        py = (ty * 16 + ys).flatten().double()
        inside = (px < w) & (py < h)
        nwp = torch.zeros(256, dtype=torch.int64, device=dev)
        nwp[inside] = nw_img[py[inside].long(), px[inside].long()].long()
        gi = sp.inst_gauss[s0:s1].long()
        m = mean[gi]
        c = co[gi]
        dx = px[:, None] - m[None, :, 0]
        dy = py[:, None] - m[None, :, 1]
        power = -0.5 * (c[None, :, 0] * dx * dx + c[None, :, 2] * dy * dy) - c[None, :, 1] * dx * dy
        alpha = c[None, :, 3].abs() * torch.exp(power)
        k = torch.arange(s1 - s0, device=dev)[None, :]
        walked = k < nwp[:, None]
        far = walked & (power < -25.0)
        small = walked & ~far & (alpha < 2.5e-3)
        mid = walked & ~far & ~small & (alpha < 1.0 / 255.0)
        blend = walked & ~far & ~small & ~mid
        for name, msk in (("far", far), ("small", small), ("mid", mid), ("blend", blend)):
            tot[name] += int(msk.sum())
        # 16x2 warps: rows 2w, 2w+1
        wk = walked.view(8, 32, -1)
        fr = far.view(8, 32, -1) | ~wk
        any_walk = wk.any(dim=1)
        warp_pairs += int(any_walk.sum())
        warp_far += int((fr.all(dim=1) & any_walk).sum())
    n = sum(tot.values())
    return {"tiles_sampled": len(pick), "pairs": n, **{k: v / max(n, 1) for k, v in tot.items()},
            "warp_slot_pairs": warp_pairs, "warp_all_far": warp_far / max(warp_pairs, 1)}


if __name__ == "__main__":
    from paper_2503_13086_b200 import GaussianField, scenes
    from paper_2503_13086_b200.rasterize import render

    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    ns = int(sys.argv[2]) if len(sys.argv) > 2 else 300
    f = GaussianField.from_host(scenes.make_params(cfg, seed=0))
    print(json.dumps(stats(render(f, scenes.camera(cfg, view=8)), ns)))
