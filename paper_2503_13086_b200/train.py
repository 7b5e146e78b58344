"""Device-tensor port of the reference training iteration.

``train_iteration`` keeps the call order of ``_train_one_iteration``
(pipeline.py:185-206): render -> total_loss -> backward -> optimizer.step ->
grad stats -> periodic densify (``_densify``, pipeline.py:209-216).  The grad
statistics (``grad_accum += screen_norms``, ``grad_count += visible``) are
accumulated inside the chain kernel instead of a separate pass.

``SemiGlobalBatch`` is the multi-view extension for the semi-global half of
an event: each rank owns a shard of the batch's views, sums its
per-view gradients into one flat FieldGrads buffer (59 params + screen norm +
visible count per Gaussian), one NCCL all-reduce sums the shards over
NVLink, and every replica applies the identical fused Adam step.
"""

from __future__ import annotations

from dataclasses import dataclass, field as dc_field

import numpy as np
import torch

from .field import DensifyOptions, GaussianField
from .losses import LossBreakdown, LossWeights, total_loss
from .optim import FieldOptimizer
from .rasterize import FieldGrads, backward, render
from .rasterize.backward import backward_and_step


@dataclass
class TrainState:
    """The slice of SessionState (pipeline.py:99-127) the hot path touches."""

    field: GaussianField
    optimizer: FieldOptimizer
    weights: LossWeights = dc_field(default_factory=LossWeights)
    layout: str = "splat"
    densify: DensifyOptions = dc_field(default_factory=DensifyOptions)
    densify_interval: int = 100
    densify_enabled: bool = True
    scene_extent: float = 1.0
    global_iteration: int = 0
    rng: np.random.Generator = dc_field(default_factory=lambda: np.random.default_rng(0))
    stats: torch.Tensor = None  # (2N,) grad_accum | grad_count

    def __post_init__(self):
        if self.stats is None:
            self.stats = torch.zeros(2 * len(self.field), dtype=torch.float32, device=self.field.flat.device)

    def grow_stats(self, n_added: int) -> None:
        """Zero statistics for rows appended by a field expansion (pipeline.py:173-174)."""
        if n_added <= 0:
            return
        n_old = self.stats.numel() // 2
        z = torch.zeros(int(n_added), dtype=self.stats.dtype, device=self.stats.device)
        self.stats = torch.cat([self.stats[:n_old], z, self.stats[n_old:], z])


def densify(state: TrainState) -> None:
    """pipeline.py:209-216 on device; moments remapped in the same kernel pass."""
    n = len(state.field)
    accum, count = state.stats[:n], state.stats[n:]
    grad_stats = accum / torch.clamp(count, min=1.0)
    opts = DensifyOptions(**{**state.densify.__dict__, "scene_extent": state.scene_extent})
    state.field.densify_and_prune(grad_stats, opts, state.rng, optimizer=state.optimizer)
    state.stats = torch.zeros(2 * len(state.field), dtype=torch.float32, device=state.field.flat.device)


def train_iteration(state: TrainState, cam, target, position_rate: float, bg=(0.0, 0.0, 0.0),
                    fused: bool = True) -> LossBreakdown:
    """One iteration of the hot path on one view (pipeline.py:185-206).

    ``fused=True`` (default) runs backward_and_step: the chain applies the
    dense Adam step in the same pass, without materialising FieldGrads (same
    math as the reference's backward + step calls; tests/test_gpu_parity.py
    checks the two agree).  ``fused=False`` goes through FieldGrads exactly like
    the reference's backward + step calls.
    """
    out = render(state.field, cam, bg=bg)
    br = total_loss(out.image, target, out, state.weights)
    if fused:
        backward_and_step(state.field, out, br.d_image, br.d_soft, state.optimizer, position_rate,
                          layout=state.layout, stats=state.stats)
    else:
        grads = backward(state.field, out, br.d_image, br.d_soft, layout=state.layout, stats=state.stats)
        state.optimizer.step(state.field, grads, position_rate=position_rate)
    state.global_iteration += 1
    if state.densify_enabled and state.global_iteration % state.densify_interval == 0:
        densify(state)
    return br


def shard_views(views, rank: int, world: int):
    """Contiguous, balanced split of a batch's views over ranks."""
    n = len(views)
    lo = (n * rank) // world
    hi = (n * (rank + 1)) // world
    return list(views[lo:hi])


def allreduce_grads(flat: torch.Tensor, group=None) -> torch.Tensor:
    """Sum the flat FieldGrads buffers of all ranks in place (one collective)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    return flat


class SemiGlobalBatch:
    """View-sharded multi-view step: sum_v grad(view v) at fixed parameters.

    Batch rule (documented deviation): gradients of the batch's
    views are summed; the position rate is the mean of the per-view rates.
    """

    def __init__(self, state: TrainState, group=None):
        self.state = state
        self.group = group

    def step(self, cams, targets, position_rates, rank: int = 0, world: int = 1, bg=(0.0, 0.0, 0.0)):
        st = self.state
        f = st.field
        idx = shard_views(list(range(len(cams))), rank, world)
        grads = FieldGrads.zeros(len(f), f.sh_degree, f.flat.device)
        losses = []
        for i in idx:
            out = render(f, cams[i], bg=bg)
            br = total_loss(out.image, targets[i], out, st.weights)
            backward(f, out, br.d_image, br.d_soft, layout=st.layout, grads=grads, accumulate=True)
            losses.append(br)
        allreduce_grads(grads.flat, self.group)
        n = len(f)
        st.stats[:n] += grads.screen_norms
        st.stats[n:] += grads.visible_count
        rate = float(np.mean(position_rates)) if len(position_rates) else 0.0
        st.optimizer.step(f, grads, position_rate=rate)
        st.global_iteration += 1
        return grads, losses
