"""Seconds per new image in the progressive On-the-Fly loop (BASELINE config 3).

A field of shell-distributed Gaussians (configs 2-4 generator) is grown by
20,000 Gaussians per arriving image (sampled near the new view's frustum,
exact 3-NN scale init on the GPU), then the event runs its T_I = 200
iterations (render -> loss -> backward -> Adam, densify statistics, densify
every 100 global iterations) over a Local & Semi-Global plan: half of the
iterations on the newest image and its overlap neighbours, half uniform over
all registered images (stand-in for scheduler.build_plan, which is host-side
and out of scope; the per-iteration cost does not depend on which view is
drawn).  One event = expand + 2 renders (psnr before/after) + 200 iterations.

  python tools/progressive.py [--events E] [--start N0]
"""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--events", type=int, default=3)
    ap.add_argument("--warmup-events", type=int, default=1,
                    help="untimed events first (allocator, kNN grid and first-call warm-up)")
    ap.add_argument("--start", type=int, default=1_980_000, help="field size before the timed events")
    ap.add_argument("--t-i", type=int, default=200)
    ap.add_argument("--per-event", type=int, default=20_000)
    ap.add_argument("--trace", action="store_true")
    ap.add_argument("--fused", type=int, default=1, help="chain + Adam in one pass (backward_and_step)")
    ap.add_argument("--profile", action="store_true",
                    help="after the events, one more iteration inside cudaProfilerStart/Stop "
                         "(ncu --profile-from-start off captures just that iteration)")
    ap.add_argument("--gaps", action="store_true",
                    help="torch.profiler timeline of the last event's iterations: device busy vs idle")
    ap.add_argument("--paper-weights", action="store_true",
                    help="losses.py defaults (load 0.41) instead of BASELINE's L1 + 0.2 D-SSIM")
    return ap.parse_args(argv)


def main(argv=None):
    """Run the events; prints one JSON line per event and a summary line, returns the summary."""
    args = parse_args(argv)
    import torch

    from paper_2503_13086_b200 import GaussianField, SparsePoint, scenes
    from paper_2503_13086_b200.losses import LossWeights, psnr
    from paper_2503_13086_b200.optim import FieldOptimizer
    from paper_2503_13086_b200.train import TrainState, train_iteration

    cfg = 3
    rng = np.random.default_rng(0)
    hp = scenes.make_params(3, seed=0, n=args.start)
    field = GaussianField.from_host(hp)
    n_views = 100
    cams = [scenes.camera(3, view=v) for v in range(n_views)]
    # targets: renders of a second-seed field at full size (the images that arrive)
    from paper_2503_13086_b200.rasterize import render

    # the arriving images: renders of a perturbed copy of the field (colours and
    # positions jittered), so the event's optimisation is a realistic refinement
    tp = scenes.make_params(3, seed=0, n=args.start)
    jr = np.random.default_rng(1)
    tp.positions += jr.normal(0.0, 0.01, tp.positions.shape).astype(np.float32)
    tp.sh[:, :, 0] += jr.normal(0.0, 0.3, tp.sh[:, :, 0].shape).astype(np.float32)
    tfield = GaussianField.from_host(tp)
    n_ev = args.warmup_events + args.events
    first = n_views - n_ev  # the timed events are the last ones of the 100-image sequence
    targets = {v: render(tfield, cams[v]).image.clone() for v in range(max(0, first - 10), n_views)}
    del tfield
    torch.cuda.synchronize()
    extent = 1.1 * float(np.max(np.linalg.norm(np.stack([c.center for c in cams]) -
                                               np.mean(np.stack([c.center for c in cams]), axis=0), axis=1)))
    # Objective: BASELINE's L1 + 0.2 D-SSIM (configs 0-2).  With the paper's
    # load-balance weight (--paper-weights) the random synthetic field's
    # opacities collapse and the walks lengthen ~4x within one event (the
    # reference documents the same trade-off, pkg/README.md:79-88); pruning is
    # then disabled so the timing stays at the config's field size.
    from paper_2503_13086_b200.field import DensifyOptions

    weights = LossWeights() if args.paper_weights else LossWeights(l1=1.0, ssim=0.2, load=0.0)
    dens = DensifyOptions(prune_opacity=0.0) if args.paper_weights else DensifyOptions()
    state = TrainState(field=field, optimizer=FieldOptimizer(field, scene_extent=extent),
                       weights=weights, scene_extent=extent, rng=np.random.default_rng(7), densify=dens)
    state.global_iteration = 1  # densify lands inside the timed events, not on their first iteration
    per_event = []
    for e in range(n_ev):
        v = first + e
        cam = cams[v]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        before = psnr(render(state.field, cam).image, targets[v])
        t_psnr0 = time.perf_counter() - t0
        # expansion: candidates sampled near the new view's frustum (in front of the camera)
        fwd = cam.rotation[2]
        depth = rng.uniform(2.0, 9.0, args.per_event)
        spread = rng.normal(0.0, 1.0, (args.per_event, 3)) * (0.35 * depth)[:, None]
        pos = cam.center[None, :] + depth[:, None] * fwd[None, :] + spread
        cols = rng.uniform(0.0, 1.0, (args.per_event, 3))
        t1 = time.perf_counter()
        n_old = len(state.field)
        state.field.insert_arrays(pos, cols)
        keep = np.ones(n_old, dtype=bool)
        state.optimizer.sync(state.field, keep, len(state.field) - n_old)
        state.stats = torch.cat([state.stats[:n_old], torch.zeros(len(state.field) - n_old, device=state.stats.device),
                                 state.stats[n_old:], torch.zeros(len(state.field) - n_old, device=state.stats.device)])
        # Local & Semi-Global plan: interleave newest-neighbourhood and uniform samples
        local = [max(0, v - (k % 10)) for k in range(args.t_i // 2)]
        semi = list(rng.integers(0, v + 1, args.t_i // 2))
        plan = [x for pair in zip(local, semi) for x in pair]
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        from paper_2503_13086_b200 import _lib

        _lib.enable_timers(args.trace)
        prof = None
        if args.gaps and e == n_ev - 1:
            from torch.profiler import ProfilerActivity, profile

            prof = profile(activities=[ProfilerActivity.CUDA])
            prof.__enter__()
        for k, tv in enumerate(plan):
            tgt = targets.get(int(tv))
            if tgt is None:
                tgt = targets[v]
            rate = 1.6e-4 * np.exp(-k / 200.0)
            br = train_iteration(state, cams[int(tv)], tgt, rate, fused=bool(args.fused))
            if args.trace and k % 100 == 99:
                torch.cuda.synchronize()
                o = render(state.field, cams[int(tv)])
                print(json.dumps({"event": e, "it": k + 1, "ms_per_it": (time.perf_counter() - t2) / (k + 1) * 1e3,
                                  "P": int(o.n_walk.sum()), "M": o.splats.n_instances, "field": len(state.field),
                                  "flagged": int(o.flagged.sum()), "loss": br.total}), flush=True)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        if prof is not None:
            prof.__exit__(None, None, None)
            sys.path.insert(0, os.path.join(ROOT, "tools"))
            from gap_profile import analyse

            analyse(prof, len(plan))
        if args.trace:
            st_ms = _lib.timer_ms()
            _lib.enable_timers(False)
            print(json.dumps({"event": e, "stage_ms": {k2: round(v2, 3) for k2, v2 in st_ms.items()},
                              "device_ms_per_it": round(sum(v2 for k2, v2 in st_ms.items() if "workspace" not in k2), 3)}),
                  flush=True)
        after = psnr(render(state.field, cam).image, targets[v])
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if e < args.warmup_events:
            continue
        per_event.append(dict(image=v, seconds=dt, field=len(state.field), psnr_before=before, psnr_after=after,
                              expand_s=t2 - t1, iterations_s=t3 - t2, ms_per_iteration=(t3 - t2) / len(plan) * 1e3,
                              psnr_renders_s=t_psnr0 + (time.perf_counter() - t3)))
        print(json.dumps(per_event[-1]), flush=True)
    if args.profile:
        v = n_views - 1
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        from bucket_stats import stats

        o = render(state.field, cams[v])
        tl = o.splats.bufs["tiles"][: len(state.field)].long()
        big = tl[tl > 32]
        print(json.dumps({"bucket_stats": stats(o), "instances": int(tl.sum()), "visible": int((tl > 0).sum()),
                          "big_splats": int(big.numel()), "big_rows": int(big.sum()),
                          "max_tiles": int(tl.max())}), flush=True)
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        train_iteration(state, cams[v], targets[v], 1.6e-4, fused=bool(args.fused))
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    summary = {"metric": "seconds per new image (config 3, final field size)",
               "value": float(np.mean([p["seconds"] for p in per_event])), "unit": "s/image",
               "events": len(per_event), "field_final": len(state.field),
               "width": cams[0].width, "height": cams[0].height, "t_i": args.t_i,
               "ms_per_iteration": float(np.mean([p["ms_per_iteration"] for p in per_event]))}
    print(json.dumps(summary), flush=True)
    return summary


if __name__ == "__main__":
    main()
