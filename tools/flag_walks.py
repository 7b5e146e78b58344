"""Flagged (guard-band) pixels of one config-2 render: how far the fp32 walk got
before the first ambiguous decision (kflag) vs the whole walk (n_walk) -- the
fp64 fix-ups walk the light part [0, kflag) and the exact part [kflag, n_walk).
  python tools/flag_walks.py [config]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_13086_b200 import GaussianField, scenes  # noqa: E402
from paper_2503_13086_b200.rasterize import render  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
f = GaussianField.from_host(scenes.make_params(cfg, seed=0))
out = render(f, scenes.camera(cfg, view=8), soft_count=False)
torch.cuda.synchronize()
fl = out.flagged.cpu().numpy().astype(bool)
nw = out.n_walk.cpu().numpy()
h, w = nw.shape
fix = out.fix_list.cpu().numpy()
kflag = fix[4 + 2 * ((w + 15) // 16) * ((h + 15) // 16) + w * h:][: w * h].reshape(h, w)
k, n = kflag[fl], nw[fl]
q = lambda a: np.percentile(a, [50, 90, 99, 100]).tolist() if a.size else []
print(json.dumps({"flagged": int(fl.sum()), "kflag_pct": q(k), "n_walk_pct": q(n), "exact_part_pct": q(n - k),
                  "all_n_walk_pct": q(nw.ravel())}))
