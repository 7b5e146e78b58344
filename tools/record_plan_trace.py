"""Record the reference scheduler's schedule for the config-3 progressive loop.

Run in the builder container only (imports the reference's scheduler.py and
overlap.py from /root/reference, read-only):

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tools/record_plan_trace.py

Config 3 has 100 images at 1297x840 on the spiral path of scenes.camera(3, v).
Match counts come from shared feature tracks, the way synthetic.py:159-177
builds them.  A seeded sparse cloud on the config's noisy r=3 shell is
projected into every view.  A point is a feature of
a view when it lands in front of the camera (z > 0.2), inside the image, and
on the side of the shell that faces the camera.
feature_count is the view's number of features.  A pair's raw match count is
the number of points both views see.

The loop is phase1_initialize with n0 = 2 (200 round-robin iterations), then
one phase2_step per arriving image 2..99.  SchedulerPlanner
(paper_2503_13086_b200/pipeline.py) makes exactly the reference's calls:

* register_image and set_matches;
* weights_for_new_image and build_plan per event;
* lr_blended before, and record_iteration after, every iteration.

Densify's split draws share the session generator with build_plan.  They
depend on the rasterizer, so a host-only recording cannot include them.  The
trace therefore uses a generator that only the planner draws from.  It stores
the generator state after each plan, and the replay hands that state to
densify.

Output ``tests/golden/c3_plan_trace.npz``, for the last events:

* entries_<id>: the 200 image ids trained by event <id>;
* rates_<id>: the position rate of each of those iterations;
* rng_<id>: the generator state after planning event <id>;
* host_s_<id>: this host's wall time for the reference's scheduling calls in
  event <id>.  The GPU replay does not run the reference code, so this time is
  reported next to the GPU seconds per image.

The script also prints the match graph's overlap between consecutive views.
"""

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import splatstream.overlap as overlap  # noqa: E402
import splatstream.scheduler as scheduler  # noqa: E402

from paper_2503_13086_b200 import scenes  # noqa: E402
from paper_2503_13086_b200.pipeline import SchedulerPlanner  # noqa: E402

N_VIEWS, N0, T_I, N_M, KEEP = 100, 2, 200, 10, 12


def tracks(cams, n_points=30_000, seed=3):
    """Feature counts and shared-track matrix of the views.  Features are
    points of the config's noisy r=3 shell; a view sees a point when it is in
    front of the camera (z > 0.2), inside the image and on the shell side
    facing the camera (an opaque surface: no feature through the shell)."""
    rng = np.random.default_rng([3, seed])
    d = rng.standard_normal((n_points, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    pts = d * 3.0 + rng.normal(0.0, 0.05, (n_points, 3))
    vis = np.zeros((len(cams), n_points), dtype=np.int64)
    for k, c in enumerate(cams):
        pc = pts @ c.rotation.T + c.translation
        z = pc[:, 2]
        with np.errstate(divide="ignore", invalid="ignore"):
            u = c.fx * pc[:, 0] / z + c.cx
            v = c.fy * pc[:, 1] / z + c.cy
        facing = ((c.center[None, :] - pts) * d).sum(axis=1) > 0
        vis[k] = (z > 0.2) & (u >= 0) & (u < c.width) & (v >= 0) & (v < c.height) & facing
    return vis.sum(axis=1), vis @ vis.T


def main(out=os.path.join(ROOT, "tests", "golden", "c3_plan_trace.npz")):
    cams = [scenes.camera(3, view=v) for v in range(N_VIEWS)]
    feats, shared = tracks(cams)
    overlap_next = [shared[i, i + 1] / min(feats[i], feats[i + 1]) for i in range(N_VIEWS - 1)]
    rng = np.random.default_rng(0)
    pl = SchedulerPlanner(scheduler, overlap, t_i=T_I, n_m=N_M, rng=rng)
    for i in range(N0):
        pl.register(i, int(feats[i]))
    for i in range(N0):
        for j in range(i + 1, N0):
            pl.set_matches(i, j, int(shared[i, j]))
    for k in range(T_I):  # phase 1: round-robin over the bootstrap pair
        pl.rate(k % N0)
        pl.record(k % N0)
    rec = {}
    first = N_VIEWS - KEEP
    for i in range(N0, N_VIEWS):
        t0 = time.perf_counter()
        pl.register(i, int(feats[i]), {j: int(shared[i, j]) for j in range(i)})
        entries = pl.plan(i)
        state_after = json.dumps(rng.bit_generator.state)
        rates = []
        for t in entries:
            rates.append(pl.rate(t))
            pl.record(t)
        dt = time.perf_counter() - t0
        if i >= first:
            rec[f"entries_{i}"] = np.array(entries, dtype=np.int32)
            rec[f"rates_{i}"] = np.array(rates)
            rec[f"rng_{i}"] = np.array(state_after)
            rec[f"host_s_{i}"] = np.float64(dt)
    rec.update(first_event=np.int64(first), last_event=np.int64(N_VIEWS - 1), t_i=np.int64(T_I), n_m=np.int64(N_M),
               n0=np.int64(N0), feature_counts=feats, overlap_next=np.array(overlap_next),
               global_iteration_before_first=np.int64(T_I * (first - N0 + 1)))
    np.savez_compressed(out, **rec)
    host = [float(rec[f"host_s_{i}"]) for i in range(first, N_VIEWS)]
    print(json.dumps({"out": out, "bytes": os.path.getsize(out), "events": N_VIEWS - first,
                      "features_mean": float(np.mean(feats)),
                      "overlap_next_mean": float(np.mean(overlap_next)),
                      "overlap_next_min": float(np.min(overlap_next)),
                      "reference_scheduler_host_s_per_event_mean": float(np.mean(host)),
                      "reference_scheduler_host_s_per_event_max": float(np.max(host)),
                      "distinct_targets_last_event": len(set(rec[f"entries_{N_VIEWS - 1}"].tolist()))}))


if __name__ == "__main__":
    main()
