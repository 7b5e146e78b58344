"""Device-tensor port of the On-the-Fly loop's per-image path (pipeline.py:99-303).

The reference's ``SessionState`` keeps ``grad_accum`` / ``grad_count`` as host
numpy arrays and ``frame.pixels`` as float64 host images, so its loop cannot
run unchanged over device tensors (``np.maximum`` on a CUDA tensor fails).
This module keeps the reference's call order with everything the hot path
touches resident on the GPU:

* ``DeviceSession``: the slice of SessionState the per-image path uses
  (field, optimizer, densify statistics as one device buffer, frames with
  their target images uploaded once, sparse point cloud, scene extent).
* ``train_one_iteration``: pipeline.py:185-206 (rate from the scheduler,
  render -> total_loss -> backward -> optimizer.step -> grad statistics ->
  record the iteration -> periodic densify).
* ``phase2_step``: pipeline.py:256-303 (register, PSNR before, expand the
  field, weights + plan, T_I iterations, PSNR after, EventReport).

The scheduler and overlap graph (scheduler.py, overlap.py) are host Python
and out of scope.  They enter through a *planner*:

* ``SchedulerPlanner`` drives the reference's own modules (pass
  ``splatstream.scheduler`` / ``splatstream.overlap``) with exactly the calls
  phase2_step makes: register_image / set_matches / TrainingState.register,
  weights_for_new_image + build_plan per event, lr_blended before and
  record_iteration after every iteration;
* ``TracePlanner`` replays plans and rates recorded from those modules
  (tools/record_plan_trace.py), so the GPU box, which has no reference
  package, runs the reference's schedule bit for bit.
"""

from __future__ import annotations

import json
import math
import time
from dataclasses import dataclass

import numpy as np
import torch

from .errors import InvalidParameter
from .field import DensifyOptions
from .losses import LossBreakdown, LossWeights, psnr
from .optim import FieldOptimizer
from .rasterize import render
from .train import TrainState, train_iteration


@dataclass
class EventReport:
    """What one fly-in event did (pipeline.py:83-96)."""

    image_id: int
    n_candidates: int
    n_inserted: int
    field_before: int
    field_after: int
    psnr_before: float
    psnr_after: float
    loss_first: float
    loss_last: float
    seconds: float


@dataclass
class LoopConfig:
    """The PhaseConfig fields the per-image path reads (pipeline.py:43-80);
    the reference's own PhaseConfig is accepted wherever this is."""

    t_i: int = 200
    n_m: int = 10
    loss_weights: LossWeights = None
    densify: DensifyOptions = None
    densify_interval: int = 100
    novelty_threshold: float = 0.0
    novelty_refresh: int = 25
    init_opacity: float = 0.1
    workers: int = 1

    def __post_init__(self):
        if self.loss_weights is None:
            self.loss_weights = LossWeights()
        if self.densify is None:
            self.densify = DensifyOptions()
        if self.t_i <= 0 or self.t_i % 2:
            raise InvalidParameter(f"t_i must be a positive even integer, got {self.t_i}")
        if self.densify_interval < 1:
            raise InvalidParameter("densify_interval must be >= 1")


# ---------------------------------------------------------------- planners
class SchedulerPlanner:
    """The reference scheduler behind the planner interface.

    ``scheduler`` / ``overlap`` are modules (or objects) providing the
    reference API: MatchMatrix, weights_for_new_image, TrainingState,
    build_plan, lr_blended, LrSchedule.  Each method is the call phase2_step /
    _train_one_iteration makes at that point (pipeline.py:133-141, 189, 203,
    269-280).
    """

    def __init__(self, scheduler, overlap, lr=None, t_i=200, n_m=10, rng=None, semiglobal=True,
                 image_weighting=True):
        self.sch, self.ovl = scheduler, overlap
        self.lr = lr if lr is not None else scheduler.LrSchedule()
        self.t_i, self.n_m = int(t_i), int(n_m)
        self.rng = rng if rng is not None else np.random.default_rng(0)
        self.semiglobal, self.image_weighting = semiglobal, image_weighting
        self.matrix = overlap.MatchMatrix()
        self.tstate = scheduler.TrainingState()

    def register(self, image_id, feature_count, match_row=None):
        self.matrix.register_image(image_id, feature_count)
        for other, raw in (match_row or {}).items():
            self.matrix.set_matches(image_id, other, raw)
        self.tstate.register(image_id)

    def set_matches(self, i, j, raw):
        self.matrix.set_matches(i, j, raw)

    def plan(self, new_id):
        if self.image_weighting:
            weights, _ = self.ovl.weights_for_new_image(self.matrix, new_id)
        else:
            weights = {i: 1.0 for i in self.matrix.image_ids}
        return list(self.sch.build_plan(weights, self.tstate, self.t_i, self.n_m, self.rng,
                                        semiglobal=self.semiglobal).entries)

    def rate(self, target_id) -> float:
        return float(self.sch.lr_blended(target_id, self.matrix, self.tstate, self.lr))

    def record(self, target_id):
        self.tstate.record_iteration(target_id)

    @property
    def global_iteration(self) -> int:
        return self.tstate.global_iteration


class TracePlanner:
    """Replays a recorded schedule: per event the plan entries and the rate of
    every iteration, per bootstrap iteration its target and rate.

    ``trace`` maps ``("event", new_id)`` -> (entries, rates) and optionally
    ``"bootstrap"`` -> (entries, rates); see tools/record_plan_trace.py.
    Every ``rate`` call must name the recorded target, so a loop that drifts
    from the reference's call order fails loudly instead of timing a
    different schedule.
    """

    def __init__(self, trace: dict):
        self.trace = trace
        self._entries, self._rates, self._k = [], [], 0
        self.global_iteration = 0

    @classmethod
    def from_npz(cls, path):
        z = np.load(path)
        trace = {}
        for key in z.files:
            if key.startswith("entries_"):
                tag = key[len("entries_"):]
                k = ("event", int(tag)) if tag != "bootstrap" else "bootstrap"
                trace[k] = (z[key].tolist(), z["rates_" + tag].tolist())
            elif key.startswith("rng_"):
                trace[("rng", int(key[len("rng_"):]))] = json.loads(str(z[key]))
        return cls(trace)

    def rng_state_after_plan(self, new_id):
        """The session generator's state right after the reference planned
        this event (build_plan draws from the same generator as densify's
        split offsets, pipeline.py:212 / scheduler.py:169), or None."""
        return self.trace.get(("rng", new_id))

    def register(self, image_id, feature_count, match_row=None):
        pass

    def set_matches(self, i, j, raw):
        pass

    def _load(self, key):
        if key not in self.trace:
            raise InvalidParameter(f"trace has no schedule for {key}")
        self._entries, self._rates = self.trace[key]
        self._k = 0
        return list(self._entries)

    def plan(self, new_id):
        return self._load(("event", new_id))

    def bootstrap(self):
        return self._load("bootstrap")

    def rate(self, target_id) -> float:
        if self._k >= len(self._entries) or self._entries[self._k] != target_id:
            raise InvalidParameter(f"iteration {self._k} trains {target_id}, the trace recorded "
                                   f"{self._entries[self._k] if self._k < len(self._entries) else 'nothing'}")
        return float(self._rates[self._k])

    def record(self, target_id):
        self._k += 1
        self.global_iteration += 1


# ---------------------------------------------------------------- session
class DeviceSession:
    """SessionState (pipeline.py:99-183) with device-resident statistics and targets."""

    def __init__(self, field, cfg, planner, rng=None, ablations=(), target_dtype=torch.float32):
        self.cfg = cfg
        self.planner = planner
        self.ablations = frozenset(ablations)
        self.frames = {}
        self.targets = {}
        self.target_dtype = target_dtype
        weights = cfg.loss_weights
        if "no_load" in self.ablations:
            weights = LossWeights(weights.l1, weights.ssim, 0.0)
        self.state = TrainState(field=field, optimizer=None, weights=weights,
                                layout="pixel" if "no_splat_parallel" in self.ablations else "splat",
                                densify=cfg.densify, densify_interval=cfg.densify_interval,
                                rng=rng if rng is not None else np.random.default_rng(0))
        self.sparse_positions = torch.zeros((0, 3), dtype=torch.float64, device=field.flat.device)
        self._novelty = float(cfg.novelty_threshold)
        self._events_since_refresh = 0
        self.events = []

    # the reference's attribute names
    field = property(lambda s: s.state.field)
    optimizer = property(lambda s: s.state.optimizer)
    scene_extent = property(lambda s: s.state.scene_extent)

    @property
    def grad_accum(self) -> torch.Tensor:
        return self.state.stats[: len(self.field)]

    @property
    def grad_count(self) -> torch.Tensor:
        return self.state.stats[len(self.field):]

    def start_optimizer(self):
        """FieldOptimizer over the current field (pipeline.py:245)."""
        self.state.optimizer = FieldOptimizer(self.field, scene_extent=self.scene_extent)

    def register_frame(self, frame, match_row=None, pixels=None):
        """pipeline.py:133-141; the frame's target image is uploaded once here."""
        if frame.image_id in self.frames:
            raise InvalidParameter(f"image {frame.image_id} is already registered")
        self.planner.register(frame.image_id, int(getattr(frame, "feature_count", 0)), match_row)
        self.frames[frame.image_id] = frame
        px = pixels if pixels is not None else getattr(frame, "pixels", None)
        if px is not None:
            t = torch.as_tensor(px)
            if tuple(t.shape) != (frame.height, frame.width, 3):
                raise InvalidParameter(f"pixels of image {frame.image_id} have shape {tuple(t.shape)}")
            dt = torch.uint8 if t.dtype == torch.uint8 else self.target_dtype
            self.targets[frame.image_id] = t.to(device=self.field.flat.device, dtype=dt).contiguous()
        self._update_extent()

    def _update_extent(self):
        """pipeline.py:143-148."""
        centers = np.stack([np.asarray(f.center, dtype=np.float64) for f in self.frames.values()])
        radius = np.linalg.norm(centers - centers.mean(axis=0), axis=1).max()
        self.state.scene_extent = max(1.1 * float(radius), 1e-6)
        if self.optimizer is not None:
            self.optimizer.scene_extent = self.state.scene_extent

    def novelty_threshold(self) -> float:
        """pipeline.py:150-158 (median spacing on the GPU k-NN index)."""
        from .spatial import median_nn_spacing

        if self.cfg.novelty_threshold > 0:
            return float(self.cfg.novelty_threshold)
        if self._events_since_refresh == 0 and self.sparse_positions.shape[0] >= 2:
            self._novelty = median_nn_spacing(self.sparse_positions)
        self._events_since_refresh = (self._events_since_refresh + 1) % self.cfg.novelty_refresh
        return self._novelty

    def expand_field(self, positions, colors) -> int:
        """pipeline.py:160-178 over (n, 3) position / colour arrays (host or
        device): novelty filter on the GPU index, insertion with exact 3-NN
        scales, optimizer moments and densify statistics grown in place."""
        from .spatial import SpatialIndex

        dev = self.field.flat.device
        pos = torch.as_tensor(np.asarray(positions) if not torch.is_tensor(positions) else positions)
        col = torch.as_tensor(np.asarray(colors) if not torch.is_tensor(colors) else colors)
        pos = pos.to(device=dev, dtype=torch.float64).reshape(-1, 3)
        col = col.to(device=dev, dtype=torch.float64).reshape(-1, 3)
        ok = torch.isfinite(pos).all(dim=1) & torch.isfinite(col).all(dim=1)
        pos, col = pos[ok], col[ok]
        threshold = self.novelty_threshold()
        if self.sparse_positions.shape[0] and threshold > 0 and pos.shape[0]:
            keep = SpatialIndex(self.sparse_positions).min_distance(pos) > threshold
            pos, col = pos[keep], col[keep]
        if pos.shape[0] == 0:
            return 0
        n_old = len(self.field)
        inserted = self.field.insert_arrays(pos, col, init_opacity=self.cfg.init_opacity)
        if self.optimizer is not None:
            self.optimizer.sync(self.field, np.ones(n_old, dtype=bool), inserted)
        self.state.grow_stats(inserted)
        self.sparse_positions = torch.cat([self.sparse_positions, pos])
        return inserted

    def view_psnr(self, frame) -> float:
        """pipeline.py:180-182."""
        out = render(self.field, frame, workers=self.cfg.workers, for_backward=False, soft_count=False)
        return psnr(out.image, self._target(frame.image_id))

    def _target(self, image_id):
        t = self.targets.get(image_id)
        if t is None:
            raise InvalidParameter(f"image {image_id} has no pixels to train against")
        return t if t.dtype != torch.uint8 else t.float() / 255.0


def phase1_initialize(session: DeviceSession, frames, positions, colors, matches=None, initial_iters: int = 0,
                      fused: bool = True) -> DeviceSession:
    """pipeline.py:219-253 on a DeviceSession: register the bootstrap frames and
    their pairwise matches, insert the sparse cloud, start the optimizer and
    train ``initial_iters`` round-robin iterations."""
    frames = list(frames)
    if not frames:
        raise InvalidParameter("expected at least one bootstrap frame")
    for f in frames:
        session.register_frame(f)
    for (i, j), raw in (matches or {}).items():
        session.planner.set_matches(i, j, raw)
    pos = torch.as_tensor(np.asarray(positions) if not torch.is_tensor(positions) else positions)
    col = torch.as_tensor(np.asarray(colors) if not torch.is_tensor(colors) else colors)
    if pos.numel() == 0:
        raise InvalidParameter("initial sparse cloud is empty")
    n = session.field.insert_arrays(pos, col, init_opacity=session.cfg.init_opacity)
    if n == 0:
        raise InvalidParameter("initial sparse cloud has no finite points")
    ok = torch.isfinite(pos.double().reshape(-1, 3)).all(dim=1) & torch.isfinite(col.double().reshape(-1, 3)).all(dim=1)
    session.sparse_positions = pos.double().reshape(-1, 3)[ok].to(session.field.flat.device)
    session.state.stats = torch.zeros(2 * len(session.field), dtype=torch.float32, device=session.field.flat.device)
    session.start_optimizer()
    order = [f.image_id for f in frames]
    for k in range(initial_iters):
        train_one_iteration(session, order[k % len(order)], fused=fused)
    return session


def train_one_iteration(session: DeviceSession, target_id, fused: bool = True) -> LossBreakdown:
    """pipeline.py:185-206: rate from the scheduler, then the hot path
    (train.train_iteration: render -> total_loss -> backward + Adam with the
    grad statistics accumulated in the chain kernel -> periodic densify), then
    the iteration is recorded with the scheduler."""
    frame = session.frames[target_id]
    target = session.targets.get(target_id)
    if target is None:
        raise InvalidParameter(f"image {target_id} has no pixels to train against")
    rate = session.planner.rate(target_id)
    br = train_iteration(session.state, frame, target, rate, fused=fused)
    session.planner.record(target_id)
    return br


def phase2_step(session: DeviceSession, new_frame, new_positions, new_colors, match_row=None,
                pixels=None, fused: bool = True) -> EventReport:
    """pipeline.py:256-303 for one fly-in image.  Wall-clock seconds include
    every host synchronisation the loop does (PSNRs, loss reads)."""
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    session.register_frame(new_frame, match_row, pixels=pixels)
    psnr_before = session.view_psnr(new_frame)
    field_before = len(session.field)
    inserted = 0
    if "no_field_update" not in session.ablations:
        inserted = session.expand_field(new_positions, new_colors)
    entries = session.planner.plan(new_frame.image_id)
    rng_state = getattr(session.planner, "rng_state_after_plan", lambda _i: None)(new_frame.image_id)
    if rng_state is not None:
        session.state.rng.bit_generator.state = rng_state
    loss_first = loss_last = math.nan
    first = last = None
    for k, target in enumerate(entries):
        br = train_one_iteration(session, target, fused=fused)
        if k == 0:
            first = br
        last = br
    if first is not None:
        loss_first, loss_last = first.total, last.total
    report = EventReport(image_id=new_frame.image_id, n_candidates=int(np.shape(new_positions)[0]),
                         n_inserted=inserted, field_before=field_before, field_after=len(session.field),
                         psnr_before=psnr_before, psnr_after=session.view_psnr(new_frame),
                         loss_first=loss_first, loss_last=loss_last, seconds=0.0)
    torch.cuda.synchronize()
    report.seconds = time.perf_counter() - t0
    session.events.append(report)
    return report
