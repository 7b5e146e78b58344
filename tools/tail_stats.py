"""Work balance of the splat-parallel backward (k_backward_splat2) for one render.

A CTA per tile, warp w streams buckets w, w + 8, ...; a bucket's stream costs
n_live + 31 steps (n_live = pixels whose blend limit passes the bucket start).
A CTA holds its 8 warp slots until its slowest warp ends, so the warp-slot
efficiency of the current assignment is sum(bucket costs) / (8 * sum over CTAs
of the slowest warp).  The balanced variant cuts each tile's concatenated
live-pixel stream into 8 equal chunks (each chunk pays 31 fill steps per bucket
segment it touches).  The makespan simulation dispatches CTAs in the given
order onto 148 x 3 slots.
  python tools/tail_stats.py [config]"""
import heapq
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def makespan(durs, slots):
    h = [0.0] * slots
    heapq.heapify(h)
    for d in durs:
        t = heapq.heappop(h)
        heapq.heappush(h, t + d)
    return max(h)


def stats(out, slots=148 * 3):
    import numpy as np

    nw = out.n_walk.cpu().numpy().astype(np.int64)
    term = out.terminated.cpu().numpy().astype(np.int64) if hasattr(out, "terminated") else 0
    lim = nw - term
    h, w = lim.shape
    th, tw = (h + 15) // 16, (w + 15) // 16
    pad = np.zeros((th * 16, tw * 16), dtype=np.int64)
    pad[:h, :w] = lim
    tiles = pad.reshape(th, 16, tw, 16).transpose(0, 2, 1, 3).reshape(th * tw, 256)
    cur, bal, tot, seg_tot = [], [], 0, 0
    nbs = []
    for t in range(tiles.shape[0]):
        lt = tiles[t]
        mx = int(lt.max())
        nb = (mx + 63) // 64
        nbs.append(nb)
        if nb == 0:
            continue
        live = np.array([(lt > 64 * b).sum() for b in range(nb)], dtype=np.int64)
        cost = live + 31
        tot += int(cost.sum())
        warps = np.zeros(8)
        for b in range(nb):
            warps[b % 8] += cost[b]
        cur.append(warps.max())
        # balanced: 8 equal chunks of the concatenated live stream
        L = int(live.sum())
        edges = np.concatenate([[0], np.cumsum(live)])
        chunk = [0.0] * 8
        for wi in range(8):
            a0, a1 = L * wi // 8, L * (wi + 1) // 8
            nseg = int(((edges[1:] > a0) & (edges[:-1] < a1)).sum())
            seg_tot += nseg
            chunk[wi] = (a1 - a0) + 31 * nseg
        bal.append(max(chunk))
    cur, bal = np.array(cur), np.array(bal)
    nbs = np.array(nbs)
    order = np.argsort(-cur, kind="stable")
    return {
        "tiles": int(tiles.shape[0]), "buckets": int(nbs.sum()),
        "buckets_per_tile": {"mean": float(nbs.mean()), "p50": float(np.median(nbs)), "max": int(nbs.max()),
                             "le8": float((nbs <= 8).mean())},
        "stream_steps": tot,
        "warp_slot_eff_current": tot / (8 * cur.sum()),
        "warp_slot_eff_balanced": tot / (8 * bal.sum()),
        "balanced_segments": seg_tot,
        "makespan_current_order": makespan(cur, slots), "makespan_lpt": makespan(cur[order], slots),
        "makespan_balanced": makespan(bal, slots),
        "makespan_balanced_lpt": makespan(np.sort(bal)[::-1], slots),
        "ideal": cur.sum() / slots, "ideal_balanced": bal.sum() / slots, "ideal_warp": tot / (8 * slots),
    }


if __name__ == "__main__":
    from paper_2503_13086_b200 import GaussianField, scenes
    from paper_2503_13086_b200.rasterize import render

    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    f = GaussianField.from_host(scenes.make_params(cfg, seed=0))
    print(json.dumps(stats(render(f, scenes.camera(cfg, view=8)))))
