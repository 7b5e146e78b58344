"""Full-size parity report (no asserts): CUDA path vs the float64 oracle for
configs 0-2, one JSON line per config with every parity metric, the number of
guard-band pixels and GPU timings.  Usage: python tools/parity_report.py [cfg ...]"""

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

from oracle import oracle  # noqa: E402
from parity import forward_report, grads_report, projection_report  # noqa: E402
from paper_2503_13086_b200 import GaussianField, scenes  # noqa: E402
from paper_2503_13086_b200.rasterize import backward, render  # noqa: E402

CLS = ("positions", "rotations", "log_scales", "opacity_logits", "sh")


def run(cfg, view=1, band=None):
    hp = scenes.make_params(cfg, seed=0)
    cam = scenes.camera(cfg, view=view)
    f = GaussianField.from_host(hp)
    kw = {} if band is None else {"band": band}
    out = render(f, cam, **kw)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        out = render(f, cam, **kw)
    torch.cuda.synchronize()
    t_fwd = (time.perf_counter() - t0) / 3
    P = oracle.Params(*(getattr(hp, k).astype(np.float64) for k in CLS))
    t0 = time.perf_counter()
    ref = oracle.render(P, cam)
    t_orc = time.perf_counter() - t0
    rep = {"cfg": cfg, "N": len(hp), "V": int(ref["splats"]["gauss_index"].size),
           "M": int(ref["splats"]["inst_splat"].size), "P_walked": int(ref["n_walk"].sum()),
           "tile_len_max": int((ref["splats"]["tile_ends"] - ref["splats"]["tile_starts"]).max()),
           "gpu_render_ms": t_fwd * 1e3, "oracle_render_s": t_orc}
    rep.update(projection_report(out.splats, ref["splats"]))
    rep.update(forward_report(out, ref))
    rng = np.random.default_rng(3)
    d_img = (rng.standard_normal((cam.height, cam.width, 3)) * 1e-6).astype(np.float32)
    d_soft = (rng.standard_normal((cam.height, cam.width)) * 1e-7).astype(np.float32)
    for layout in ("splat", "pixel"):
        g = backward(f, out, d_img, d_soft, layout=layout)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            g = backward(f, out, d_img, d_soft, layout=layout)
        torch.cuda.synchronize()
        rep[f"gpu_backward_{layout}_ms"] = (time.perf_counter() - t0) / 3 * 1e3
        if layout == "splat":
            t0 = time.perf_counter()
            rg = oracle.backward(P, ref, d_img.astype(np.float64), d_soft.astype(np.float64))
            rep["oracle_backward_s"] = time.perf_counter() - t0
        rep.update({f"{layout}_{k}": v for k, v in grads_report(g, rg).items()})
    # flipped decisions among pixels the guard band did NOT flag (should be 0)
    fl = out.flagged.cpu().numpy().astype(bool)
    nw = out.n_walk.cpu().numpy()
    rep["unflagged_nwalk_flips"] = int(((nw != ref["n_walk"]) & ~fl).sum())
    return rep


if __name__ == "__main__":
    cfgs = [int(a) for a in sys.argv[1:]] or [0, 1, 2]
    print("oracle threads:", oracle.num_threads(), flush=True)
    for c in cfgs:
        print(json.dumps(run(c)), flush=True)
