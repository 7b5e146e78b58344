"""Systolic-stream occupancy of the splat-parallel backward for one render:
live pixel-buckets (sum over pixels of ceil(n_walk / 32)) vs the stream steps
the backward runs (live + 31 per bucket).  Used to size the pipeline fill cost.
  python tools/bucket_stats.py [config]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def stats(out):
    import torch

    nw = out.n_walk.to(torch.int64)
    h, w = nw.shape
    th, tw = (h + 15) // 16, (w + 15) // 16
    pad = torch.zeros(th * 16, tw * 16, dtype=torch.int64, device=nw.device)
    pad[:h, :w] = nw
    tiles = pad.view(th, 16, tw, 16).permute(0, 2, 1, 3).reshape(th * tw, 256)
    live = ((tiles + 31) // 32).sum().item()
    nb = ((tiles.max(dim=1).values + 31) // 32).sum().item()
    return {"pairs": int(nw.sum().item()), "live_pixel_buckets": int(live), "buckets": int(nb),
            "stream_steps": int(live + 31 * nb), "overhead": (live + 31 * nb) / max(live, 1)}


if __name__ == "__main__":
    from paper_2503_13086_b200 import GaussianField, scenes
    from paper_2503_13086_b200.rasterize import render

    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    f = GaussianField.from_host(scenes.make_params(cfg, seed=0))
    print(json.dumps(stats(render(f, scenes.camera(cfg, view=8)))))
