"""Record the REFERENCE's own progressive loop (pipeline.py) on a small scene.

Run in the builder container only (needs /root/reference, read-only):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_pipeline_golden.py

Writes ``tests/golden/pipeline_small.npz``.  The reference runs
phase1_initialize and then ``phase2_step`` for every fly-in image of a
``synthetic.make_scene`` replay, unchanged.  This script only observes it:
wrappers around ``build_plan``, ``lr_blended``, ``_train_one_iteration`` and
``densify_and_prune`` log each event's plan, the rate of every iteration, the
generator state after planning, every loss and the densify counts.

The parameters and Adam moments are rounded to float32 before phase 2, which is
the GPU's storage.  So both implementations start every event from identical
values.  The fixture holds:

* the scene: cameras, 8-bit-exact float pixels, sparse points and match rows;
* the session state after phase 1 (field, moments, step counts, densify
  statistics, per-image iteration counts, sparse cloud, novelty state);
* per event: the plan, rates, losses, densify summaries, EventReport and the
  field after the event.

tests/test_pipeline_gpu.py replays the events through
paper_2503_13086_b200.pipeline (TracePlanner) and compares.
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import splatstream.pipeline as P  # noqa: E402
from splatstream.field import GaussianField  # noqa: E402
from splatstream.io.replay import ReplayStream  # noqa: E402
from splatstream.losses import LossWeights  # noqa: E402
from splatstream.pipeline import PhaseConfig, phase1_initialize, phase2_step  # noqa: E402
from splatstream.synthetic import make_scene, to_bundle  # noqa: E402

PARAM_KEYS = ("positions", "rotations", "log_scales", "opacity_logits", "sh")


def f32(a):
    return np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)


def save_state(rec, tag, state):
    """Everything the next event starts from."""
    for k in PARAM_KEYS:
        rec[f"{tag}_{k}"] = np.array(getattr(state.field, k))
    for name, buf in zip(PARAM_KEYS, state.optimizer.state.buffers()):
        rec[f"{tag}_m_{name}"], rec[f"{tag}_v_{name}"] = buf.m.copy(), buf.v.copy()
        rec[f"{tag}_step_{name}"] = np.int64(buf.step)
    rec[f"{tag}_grad_accum"], rec[f"{tag}_grad_count"] = state.grad_accum.copy(), state.grad_count.copy()
    rec[f"{tag}_sparse"] = state.sparse_positions.copy()
    rec[f"{tag}_global_iteration"] = np.int64(state.tstate.global_iteration)
    rec[f"{tag}_extent"] = np.float64(state.scene_extent)
    rec[f"{tag}_novelty"] = np.float64(state._novelty)
    rec[f"{tag}_events_since_refresh"] = np.int64(state._events_since_refresh)
    rec[f"{tag}_frames"] = np.array(list(state.frames))


def main(out=os.path.join(HERE, "pipeline_small.npz"), n_events=3):
    scene = make_scene(seed=4, n_views=3 + n_events, width=64, height=48, focal=60.0)
    # the pixels the GPU gets are float32; round the reference's too
    for fr in scene.frames.values():
        fr.pixels = f32(fr.pixels)
    cfg = PhaseConfig(n0=3, initial_iters=30, t_i=20, n_m=2, seed=5, densify_interval=25, sh_degree=1,
                      loss_weights=LossWeights(), novelty_threshold=0.0)
    bundle, _ = to_bundle(scene)
    stream = ReplayStream(bundle)
    frames, pts, matches = stream.initial(cfg.n0)
    # the bootstrap field before any training (phase1_initialize's insert_points)
    boot = GaussianField(sh_degree=cfg.sh_degree)
    usable = [p for p in pts if p.finite]
    boot.insert_points(usable, init_opacity=cfg.init_opacity)
    boot_rec = {f"boot_{k}": np.array(getattr(boot, k)) for k in PARAM_KEYS}
    boot_rec["boot_points_pos"] = np.array([p.position for p in pts]).reshape(-1, 3)
    boot_rec["boot_points_col"] = np.array([p.color for p in pts]).reshape(-1, 3)
    state = phase1_initialize(frames, pts, cfg, matches=matches)

    # float32 storage: round parameters and moments before phase 2
    for k in PARAM_KEYS:
        setattr(state.field, k, f32(getattr(state.field, k)))
    for buf in state.optimizer.state.buffers():
        buf.m, buf.v = f32(buf.m), f32(buf.v)
    state.grad_accum = f32(state.grad_accum)

    rec = dict(boot_rec)
    save_state(rec, "p1", state)
    rec["init_ids"] = np.array([f.image_id for f in frames])
    rec["init_matches"] = np.array([[i, j, c] for (i, j), c in sorted((matches or {}).items())],
                                   dtype=np.int64).reshape(-1, 3)
    rec["initial_iters"] = np.int64(cfg.initial_iters)

    # ---- observe phase 2
    log = {}
    orig_plan, orig_rate, orig_iter = P.build_plan, P.lr_blended, P._train_one_iteration
    orig_dens = GaussianField.densify_and_prune

    def build_plan(*a, **kw):
        log["rng_before_plan"] = json.dumps(state.rng.bit_generator.state)
        plan = orig_plan(*a, **kw)
        log["entries"] = list(plan.entries)
        log["rng_after_plan"] = json.dumps(state.rng.bit_generator.state)
        return plan

    def lr_blended(*a, **kw):
        r = orig_rate(*a, **kw)
        log.setdefault("rates", []).append(r)
        return r

    def one_iteration(st, c, tid):
        br = orig_iter(st, c, tid)
        log.setdefault("losses", []).append([br.l1, br.ssim_loss, br.load, br.total])
        return br

    def densify_and_prune(self, *a, **kw):
        s = orig_dens(self, *a, **kw)
        log.setdefault("densify", []).append([s.cloned, s.split, s.pruned, state.tstate.global_iteration])
        return s

    P.build_plan, P.lr_blended, P._train_one_iteration = build_plan, lr_blended, one_iteration
    GaussianField.densify_and_prune = densify_and_prune
    ev_ids = []
    for e, ev in enumerate(stream.events()):
        if e >= n_events:
            break
        log.clear()
        fr = ev.frame
        fr.pixels = f32(fr.pixels)
        report = phase2_step(state, fr, ev.points, ev.match_row, cfg)
        i = fr.image_id
        ev_ids.append(i)
        rec[f"ev{e}_id"] = np.int64(i)
        rec[f"ev{e}_points_pos"] = np.array([p.position for p in ev.points]).reshape(-1, 3)
        rec[f"ev{e}_points_col"] = np.array([p.color for p in ev.points]).reshape(-1, 3)
        rec[f"ev{e}_match_row"] = np.array(sorted((ev.match_row or {}).items()), dtype=np.int64).reshape(-1, 2)
        rec[f"ev{e}_entries"] = np.array(log["entries"])
        rec[f"ev{e}_rates"] = np.array(log["rates"])
        rec[f"ev{e}_losses"] = np.array(log["losses"])
        rec[f"ev{e}_densify"] = np.array(log.get("densify", []), dtype=np.int64).reshape(-1, 4)
        rec[f"ev{e}_rng_after_plan"] = np.array(log["rng_after_plan"])
        rec[f"ev{e}_rng_before_plan"] = np.array(log["rng_before_plan"])
        rec[f"ev{e}_report"] = np.array([report.n_candidates, report.n_inserted, report.field_before,
                                         report.field_after, report.psnr_before, report.psnr_after,
                                         report.loss_first, report.loss_last])
        save_state(rec, f"ev{e}_after", state)
        print(f"event {e}: image {i}, inserted {report.n_inserted}, field {report.field_before}->"
              f"{report.field_after}, loss {report.loss_first:.5f}->{report.loss_last:.5f}, "
              f"densify {log.get('densify')}")
    P.build_plan, P.lr_blended, P._train_one_iteration = orig_plan, orig_rate, orig_iter
    GaussianField.densify_and_prune = orig_dens
    rec["n_events"] = np.int64(len(ev_ids))

    # the scene: every frame that took part
    for i, fr in scene.frames.items():
        rec[f"frame{i}_R"], rec[f"frame{i}_t"] = fr.rotation, fr.translation
        rec[f"frame{i}_intr"] = np.array([fr.fx, fr.fy, fr.cx, fr.cy])
        rec[f"frame{i}_wh"] = np.array([fr.width, fr.height])
        rec[f"frame{i}_features"] = np.int64(fr.feature_count)
        rec[f"frame{i}_pixels"] = np.asarray(fr.pixels, np.float32)
    rec["cfg"] = np.array(json.dumps(dict(t_i=cfg.t_i, n_m=cfg.n_m, densify_interval=cfg.densify_interval,
                                          sh_degree=cfg.sh_degree, init_opacity=cfg.init_opacity,
                                          novelty_threshold=cfg.novelty_threshold,
                                          novelty_refresh=cfg.novelty_refresh,
                                          weights=[cfg.loss_weights.l1, cfg.loss_weights.ssim,
                                                   cfg.loss_weights.load])))
    np.savez_compressed(out, **rec)
    print("wrote", out, os.path.getsize(out), "bytes")


if __name__ == "__main__":
    main()
