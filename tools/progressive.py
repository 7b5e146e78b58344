"""Seconds per new image in the progressive On-the-Fly loop (BASELINE config 3).

Every event runs ``pipeline.phase2_step``, the device port of the
reference's phase2_step (pipeline.py:256-303):

* register the frame and upload its 8-bit target once;
* PSNR of the new view before training;
* field expansion: 20,000 candidates near the new view's frustum, the novelty
  filter on the GPU k-NN index (threshold 1e-12 admits all, as SURVEY 8d
  asks), and exact 3-NN scale init;
* the reference scheduler's plan and per-iteration position rates, replayed
  from tests/golden/c3_plan_trace.npz (tools/record_plan_trace.py records them
  from the reference's build_plan / lr_blended on the config-3 match graph);
* T_I = 200 iterations of render -> loss -> backward + Adam, with densify every
  100 global iterations;
* PSNR after.

The field starts at 2.0 M - 20 k x (events) Gaussians, so the last event
(image 99) ends at 2.0 M.  The targets are renders of a perturbed copy of the
field (colours and positions jittered), so training is a real refinement.
Seconds are wall clock per event and include every host synchronisation.

The reference's host scheduling calls do not run here: the reference package
is not on the GPU box.  Their recorded time on the builder host is reported
separately (``reference_scheduler_s``).

  python tools/progressive.py [--events E] [--warmup-events W] [--paper-weights]
"""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
TRACE = os.path.join(ROOT, "tests", "golden", "c3_plan_trace.npz")


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--events", type=int, default=5)
    ap.add_argument("--warmup-events", type=int, default=1,
                    help="untimed events first (allocator, kNN grid and first-call warm-up)")
    ap.add_argument("--final", type=int, default=2_000_000, help="field size after the last event")
    ap.add_argument("--per-event", type=int, default=20_000)
    ap.add_argument("--trace", action="store_true", help="per-stage device times of each event")
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

    from paper_2503_13086_b200 import GaussianField, _lib, scenes
    from paper_2503_13086_b200.field import DensifyOptions
    from paper_2503_13086_b200.losses import LossWeights
    from paper_2503_13086_b200.pipeline import DeviceSession, LoopConfig, TracePlanner, phase2_step
    from paper_2503_13086_b200.rasterize import render

    z = np.load(TRACE)
    planner = TracePlanner.from_npz(TRACE)
    n_views = int(z["last_event"]) + 1
    n_ev = args.warmup_events + args.events
    first = n_views - n_ev
    if first < int(z["first_event"]):
        raise SystemExit(f"the trace covers events {int(z['first_event'])}..{n_views - 1}")
    start = args.final - args.per_event * n_ev
    hp = scenes.make_params(3, seed=0, n=start)
    cams = [scenes.camera(3, view=v) for v in range(n_views)]
    tp = scenes.make_params(3, seed=0, n=args.final)
    jr = np.random.default_rng(1)
    tp.positions += jr.normal(0.0, 0.01, tp.positions.shape).astype(np.float32)
    tp.sh[:, :, 0] += jr.normal(0.0, 0.3, tp.sh[:, :, 0].shape).astype(np.float32)
    tfield = GaussianField.from_host(tp)
    # 8-bit targets, as the reference's image files are (io/images.py)
    pixels = [(render(tfield, c).image * 255.0).round().clamp(0, 255).to(torch.uint8) for c in cams]
    del tfield
    field = GaussianField.from_host(hp)
    weights = LossWeights() if args.paper_weights else LossWeights(l1=1.0, ssim=0.2, load=0.0)
    cfg = LoopConfig(t_i=int(z["t_i"]), n_m=int(z["n_m"]), loss_weights=weights, densify=DensifyOptions(),
                     densify_interval=100, novelty_threshold=1e-12)
    sess = DeviceSession(field, cfg, planner, rng=np.random.default_rng(7))
    for v in range(first):  # images that arrived before the timed window
        sess.register_frame(cams[v], pixels=pixels[v])
    sess.start_optimizer()
    # the sparse cloud: one point per Gaussian inserted so far
    sess.sparse_positions = field.positions.double().clone()
    # the global iteration count the reference schedule had reached (densify cadence)
    sess.state.global_iteration = int(z["global_iteration_before_first"]) + cfg.t_i * (first - int(z["first_event"]))
    rng = np.random.default_rng(0)
    per_event = []
    for e in range(n_ev):
        v = first + e
        cam = cams[v]
        fwd = cam.rotation[2]
        depth = rng.uniform(2.0, 9.0, args.per_event)
        spread = rng.normal(0.0, 1.0, (args.per_event, 3)) * (0.35 * depth)[:, None]
        pos = cam.center[None, :] + depth[:, None] * fwd[None, :] + spread
        cols = rng.uniform(0.0, 1.0, (args.per_event, 3))
        _lib.enable_timers(args.trace)
        prof = None
        if args.gaps and e == n_ev - 1:
            from torch.profiler import ProfilerActivity, profile

            prof = profile(activities=[ProfilerActivity.CUDA])
            prof.__enter__()
        rep = phase2_step(sess, cam, pos, cols, pixels=pixels[v], fused=bool(args.fused))
        if prof is not None:
            prof.__exit__(None, None, None)
            sys.path.insert(0, os.path.join(ROOT, "tools"))
            from gap_profile import analyse

            analyse(prof, cfg.t_i)
        if args.trace:
            st_ms = _lib.timer_ms()
            _lib.enable_timers(False)
            print(json.dumps({"event": e, "stage_ms": {k2: round(v2, 3) for k2, v2 in st_ms.items()}}), flush=True)
        if e < args.warmup_events:
            continue
        o = render(sess.field, cam)
        per_event.append(dict(image=v, seconds=rep.seconds, field_before=rep.field_before, field=rep.field_after,
                              inserted=rep.n_inserted, psnr_before=rep.psnr_before, psnr_after=rep.psnr_after,
                              loss_first=rep.loss_first, loss_last=rep.loss_last,
                              reference_scheduler_s=float(z[f"host_s_{v}"]),
                              walked_pairs=int(o.n_walk.sum()), instances=o.splats.n_instances))
        print(json.dumps(per_event[-1]), flush=True)
    if args.profile:
        v = n_views - 1
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        from bucket_stats import stats

        from paper_2503_13086_b200.train import train_iteration

        o = render(sess.field, cams[v])
        tl = o.splats.bufs["tiles"][: len(sess.field)].long()
        big = tl[tl > 32]
        print(json.dumps({"bucket_stats": stats(o), "instances": int(tl.sum()), "visible": int((tl > 0).sum()),
                          "big_splats": int(big.numel()), "big_rows": int(big.sum()),
                          "max_tiles": int(tl.max())}), flush=True)
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        train_iteration(sess.state, cams[v], sess.targets[v], 1.6e-4, fused=bool(args.fused))
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    secs = [p["seconds"] for p in per_event]
    sched = [p["reference_scheduler_s"] for p in per_event]
    summary = {"metric": "seconds per new image (config 3)", "value": float(np.mean(secs)), "unit": "s/image",
               "median": float(np.median(secs)),
               "worst": float(np.max(secs)), "worst_image": per_event[int(np.argmax(secs))]["image"],
               "events": len(per_event), "field_final": len(sess.field),
               "objective": "paper LossWeights() (0.47, 0.12, 0.41)" if args.paper_weights
               else "L1 + 0.2 D-SSIM (BASELINE)",
               "plan": "reference build_plan / lr_blended replayed (tests/golden/c3_plan_trace.npz)",
               "reference_scheduler_s_mean": float(np.mean(sched)),
               "value_with_reference_scheduler": float(np.mean(np.add(secs, sched))),
               "width": cams[0].width, "height": cams[0].height, "t_i": cfg.t_i,
               "ms_per_iteration": float(np.mean(secs) / cfg.t_i * 1e3)}
    print(json.dumps(summary), flush=True)
    return summary


if __name__ == "__main__":
    main()
