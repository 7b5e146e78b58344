"""GPU idle gaps inside training iterations (torch.profiler / CUPTI timeline).

Runs warm-up iterations of train_iteration on a config's field, then profiles a
few more and reports, per iteration, the wall span of the GPU timeline, the
busy time (union of kernel and memcpy intervals) and the largest idle gaps
with the activities either side of them.

  SSR_CFG=3 python tools/gap_profile.py [--iters 10] [--fused 1]
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--fused", type=int, default=1)
    ap.add_argument("--view", type=int, default=99)
    ap.add_argument("--trace-out", default="")
    ap.add_argument("--u8", action="store_true", help="8-bit target image (as the e2e bench uploads)")
    ap.add_argument("--paper-weights", action="store_true",
                    help="losses.py default weights (load-balance term on: soft-count gradients)")
    args = ap.parse_args()
    import numpy as np
    import torch
    from torch.profiler import ProfilerActivity, profile

    from paper_2503_13086_b200 import GaussianField, scenes
    from paper_2503_13086_b200.losses import LossWeights
    from paper_2503_13086_b200.optim import FieldOptimizer
    from paper_2503_13086_b200.rasterize import render
    from paper_2503_13086_b200.train import TrainState, train_iteration

    cfg = int(os.environ.get("SSR_CFG", "3"))
    n = 2_000_000 if cfg == 3 else None
    hp = scenes.make_params(cfg, seed=0, n=n) if n else scenes.make_params(cfg, seed=0)
    field = GaussianField.from_host(hp)
    cam = scenes.camera(cfg, view=args.view)
    tp = scenes.make_params(cfg, seed=1, n=n) if n else scenes.make_params(cfg, seed=1)
    target = render(GaussianField.from_host(tp), cam).image.clone()
    if args.u8:
        target = (target * 255.0).round().clamp(0, 255).to(torch.uint8)
    state = TrainState(field=field, optimizer=FieldOptimizer(field, scene_extent=6.6),
                       weights=LossWeights() if args.paper_weights else LossWeights(l1=1.0, ssim=0.2, load=0.0),
                       scene_extent=6.6,
                       rng=np.random.default_rng(7))
    state.densify_enabled = False
    for _ in range(args.warmup):
        train_iteration(state, cam, target, 1.6e-4, fused=bool(args.fused))
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        for _ in range(args.iters):
            train_iteration(state, cam, target, 1.6e-4, fused=bool(args.fused))
        torch.cuda.synchronize()
    if args.trace_out:
        prof.export_chrome_trace(args.trace_out)
    analyse(prof, args.iters)


def analyse(prof, iters):
    """Busy/idle split of a torch.profiler capture's device timeline (per iteration)."""
    import torch

    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    iv = sorted((e.time_range.start, e.time_range.end, e.name) for e in ev)
    # drop the first iteration (profiler start-up): analyse from the second preprocess on
    starts = [i for i, x in enumerate(iv) if "k_preprocess" in x[2]]
    if len(starts) > 1:
        iv = iv[starts[1]:]
        iters = len(starts) - 1
    if not iv:
        print(json.dumps({"error": "no device events"}))
        return None
    span = iv[-1][1] - iv[0][0]
    busy, gaps = 0.0, []
    cur_s, cur_e, cur_n = iv[0]
    for s, e, nm in iv[1:]:
        if s > cur_e:
            busy += cur_e - cur_s
            gaps.append((s - cur_e, cur_n, nm))
            cur_s, cur_e, cur_n = s, e, nm
        else:
            if e > cur_e:
                cur_e, cur_n = e, nm
    busy += cur_e - cur_s
    gaps.sort(reverse=True)
    by_pair = {}
    for g, a, b in gaps:
        k = (a[:60], b[:60])
        t = by_pair.setdefault(k, [0.0, 0])
        t[0] += g
        t[1] += 1
    top = sorted(by_pair.items(), key=lambda kv: -kv[1][0])[:15]
    summary = {"iters": iters, "span_us_per_iter": span / iters, "busy_us_per_iter": busy / iters,
               "idle_us_per_iter": (span - busy) / iters, "n_gaps": len(gaps),
               "gap_pairs": [{"after": a, "before": b, "total_us_per_iter": t / iters, "count": c}
                             for (a, b), (t, c) in top]}
    print(json.dumps(summary, indent=1))
    names = {}
    for s, e, nm in iv:
        t = names.setdefault(nm[:70], [0.0, 0])
        t[0] += e - s
        t[1] += 1
    for nm, (t, c) in sorted(names.items(), key=lambda kv: -kv[1][0])[:30]:
        print(f"{t / iters:9.1f} us/iter  x{c / iters:5.1f}  {nm}")
    # host-side synchronisation points (each one drains the device queue)
    syncs = {}
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            continue
        nm = e.name
        if any(k in nm for k in ("Synchronize", "_local_scalar_dense", "cudaMemcpy", "aten::item", "EventSync")):
            t = syncs.setdefault(nm, [0, 0.0])
            t[0] += 1
            t[1] += e.cpu_time_total
    for nm, (c, t) in sorted(syncs.items(), key=lambda kv: -kv[1][1]):
        print(f"host sync {nm}: x{c / iters:.1f}/iter, {t / iters:.1f} us/iter")
    return summary


if __name__ == "__main__":
    main()
