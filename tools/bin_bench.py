"""Device time of the stage-2 entry points (ssr_scan_tiles, ssr_bin_tiles) at a
config, warm, CUDA events on the launching stream; no host sync inside the
timed calls (M is read once up front).

  python tools/bin_bench.py [--config 2] [--view 8] [--reps 50]
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--view", type=int, default=8)
    ap.add_argument("--reps", type=int, default=50)
    a = ap.parse_args()
    import torch

    from paper_2503_13086_b200 import GaussianField, _lib, scenes
    from paper_2503_13086_b200.rasterize.projection import project_field

    f = GaussianField.from_host(scenes.make_params(a.config, seed=0))
    cam = scenes.camera(a.config, view=a.view)
    sp = project_field(f, cam)
    n, m = sp.n, sp.n_instances
    s = sp.struct()
    st = _lib.stream_ptr()
    dev = f.flat.device
    ws = torch.empty(_lib.query("ssr_scan_workspace", n), dtype=torch.uint8, device=dev)
    total = torch.empty(1, dtype=torch.int64, device=dev)
    n_tiles = sp.tiles_x * sp.tiles_y
    bws = torch.empty(_lib.query("ssr_bin_workspace", m, n_tiles), dtype=torch.uint8, device=dev)
    inst = torch.empty(m, dtype=torch.int32, device=dev)
    ranges = torch.empty(n_tiles, 2, dtype=torch.int32, device=dev)

    def scan():
        _lib.call("ssr_scan_tiles", n, s, ws.data_ptr(), ws.numel(), total.data_ptr(), st)

    def binning():
        _lib.call("ssr_bin_tiles", n, m, sp.tiles_x, sp.tiles_y, s, inst.data_ptr(), ranges.data_ptr(),
                  bws.data_ptr(), bws.numel(), st)

    out = {"config": a.config, "n": n, "m": m, "visible": sp.n_visible, "tiles": n_tiles}
    for name, fn in (("scan_tiles", scan), ("bin_tiles", binning)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        out[name + "_us"] = e0.elapsed_time(e1) / a.reps * 1e3
    assert int(total.item()) == m
    assert torch.equal(inst, sp.inst_gauss) and torch.equal(ranges, sp.tile_ranges)
    # HBM model: scan = tiles/depth reads + 3 radix passes over N (key+val R/W) + scans;
    # bin = duplicate writes + 2 passes over M (key+val R/W) + ranges read
    out["bin_algorithmic_MB"] = (8 * m + 2 * 16 * m + 4 * m) / 1e6
    out["scan_algorithmic_MB"] = (12 * n + 3 * 16 * n + 16 * n) / 1e6
    print(json.dumps(out))


if __name__ == "__main__":
    main()
