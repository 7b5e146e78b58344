"""Work shape of the two float64 fix-ups on one render (config 2 by default):
the forward fix-up walks each flagged pixel by one warp (light chunks before the
first ambiguous slot, exact chunks after); the backward fix-up's items are the
(flagged tile, bucket) pairs, each walking the tile's flagged pixels that meet
the bucket.  Both kernels are latency-bound, so their time follows the longest
serial chain per warp, reported here.
  python tools/fix_items.py [config]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_13086_b200 import GaussianField, scenes  # noqa: E402
from paper_2503_13086_b200.rasterize import backward, render  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
f = GaussianField.from_host(scenes.make_params(cfg, seed=0))
out = render(f, scenes.camera(cfg, view=8), soft_count=False)
backward(f, out, torch.full_like(out.image, 1e-3))
torch.cuda.synchronize()
nw = out.n_walk.cpu().numpy()
h, w = nw.shape
tiles_x, tiles_y = (w + 15) // 16, (h + 15) // 16
n_tiles = tiles_x * tiles_y
fix = out.fix_list.cpu().numpy()
ti = out.tile_info.cpu().numpy()
count, n_ft = int(fix[0]), int(fix[1])
px_list = fix[4 + 2 * n_tiles:][:count]
kflag = fix[4 + 2 * n_tiles + w * h:][: w * h].reshape(h, w)
fwd_light, fwd_exact = [], []
tiles = {}
for e in px_list:
    t, p = int(e) >> 8, int(e) & 255
    x, y = (t % tiles_x) * 16 + (p & 15), (t // tiles_x) * 16 + (p >> 4)
    n, k = int(nw[y, x]), int(kflag[y, x])
    fwd_light.append(k // 32)
    fwd_exact.append((n + 31) // 32 - k // 32)
    tiles.setdefault(t, []).append((n, k))
walks = []
for t, pix in tiles.items():
    z, kmin = int(ti[t, 2]), int(ti[t, 3])
    for b in range(kmin >> 5, (z + 31) >> 5):
        kb = 32 * b
        walks.append(sum(1 for n, k in pix if n > kb and k < kb + 32))
q = lambda a: np.percentile(a, [50, 90, 99, 100]).tolist() if len(a) else []
walks = np.array(walks)
n_warps = 148 * 2 * 8
per_warp = np.zeros(n_warps, dtype=np.int64)
for i, v in enumerate(walks):
    per_warp[i % n_warps] += v
print(json.dumps({"flagged": count, "flagged_tiles": n_ft, "fwd_light_chunks_pct": q(fwd_light),
                  "fwd_exact_chunks_pct": q(fwd_exact), "bwd_items": int(walks.size), "bwd_walks_per_item_pct": q(walks),
                  "bwd_walks_total": int(walks.sum()), "bwd_walks_per_warp_max": int(per_warp.max()),
                  "flagged_per_tile_pct": q([len(v) for v in tiles.values()])}))
