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

from . import _lib
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
    # soft counts only when the objective reads them (load weight > 0)
    out = render(state.field, cam, bg=bg, soft_count=state.weights.load > 0)
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


def shard_layout(param_floats: int, world: int):
    """(chunk, main) of a sharded step: the first ``main = world * chunk``
    floats of the flat parameter buffer are split into equal, 16-byte aligned
    chunks (rank r owns [r * chunk, (r + 1) * chunk)); the short tail
    [main, param_floats) is reduced and stepped on every rank."""
    chunk = (param_floats // (4 * world)) * 4
    return chunk, world * chunk


def exchange_and_step(field, grads, optimizer, position_rate: float, mode: str = "allreduce", group=None,
                      adam_range=None, exchanger=None):
    """Combine the ranks' gradient sums and apply the identical Adam step.

    ``mode="allreduce"``: one all-reduce of the whole 61-float-per-row buffer,
    then every replica runs the full Adam.  ``mode="sharded"``: reduce-scatter
    of the parameter gradients, each rank runs Adam on its own 1/world chunk
    (ssr_adam_range), an all-gather of the updated parameters, plus one small
    all-reduce of the tail and the densify statistics.  Same bytes on the wire
    as the all-reduce, 1/world of the Adam traffic per rank; rank r's moments
    are current only inside its chunk (``gather_moments`` before a densify).

    ``mode="p2p"``: the sharded step fused into one kernel per rank over peer
    memory (``exchange_p2p``; ``exchanger`` keeps the peer mappings).

    ``adam_range(lo, hi, g, goff)`` overrides the CUDA Adam (host-logic tests).
    """
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    if world == 1 or mode == "allreduce":
        allreduce_grads(grads.flat, group)
        if adam_range is None:
            optimizer.step(field, grads, position_rate=position_rate)
        else:
            adam_range(0, field.flat.numel(), grads.flat, 0)
        return
    if mode == "p2p":
        if adam_range is not None:
            raise ValueError("mode='p2p' runs the fused CUDA kernel; adam_range applies to 'sharded'")
        exchange_p2p(field, grads, optimizer, position_rate, exchanger or PeerExchange(group))
        return
    if mode != "sharded":
        raise ValueError(f"unknown exchange mode {mode!r}")
    rank = dist.get_rank(group)
    p_floats = field.flat.numel()
    chunk, main = shard_layout(p_floats, world)
    g = grads.flat
    mine = torch.empty(chunk, dtype=g.dtype, device=g.device)
    dist.reduce_scatter_tensor(mine, g[:main], group=group)
    dist.all_reduce(g[main:], group=group)  # parameter tail + screen_norms + visible
    lo = rank * chunk
    if adam_range is None:
        optimizer.check(field)
        lr, bc1, bc2 = optimizer.advance(position_rate)
        from .optim import SH_REST_LR

        n, deg = len(field), field.sh_degree
        field.version += 1
        for a, b, gt, goff in ((lo, lo + chunk, mine, lo), (main, p_floats, g, 0)):
            _lib.call("ssr_adam_range", n, deg, field.flat.data_ptr(), gt.data_ptr(), goff, optimizer.m.data_ptr(),
                      optimizer.v.data_ptr(), a, b, lr, SH_REST_LR, bc1, bc2, _lib.stream_ptr())
    else:
        adam_range(lo, lo + chunk, mine, lo)
        adam_range(main, p_floats, g, 0)
    src = field.flat[lo:lo + chunk]
    if dist.get_backend(group) != "nccl":
        src = src.clone()  # in-place all-gather is an NCCL feature
    dist.all_gather_into_tensor(field.flat[:main], src, group=group)


def gather_moments(field, optimizer, group=None, mode: str = "sharded"):
    """Make every rank's Adam moments complete after sharded steps (before a
    densify remaps rows across chunk boundaries).  ``mode="p2p"``: the last
    rank also owns the tail past ``world * chunk`` (ssr_exchange_chunk)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    p_floats = field.flat.numel()
    chunk, main = shard_layout(p_floats, world)
    for buf in (optimizer.m, optimizer.v):
        src = buf[rank * chunk:(rank + 1) * chunk]
        if dist.get_backend(group) != "nccl":
            src = src.clone()
        dist.all_gather_into_tensor(buf[:main], src, group=group)
        if mode == "p2p" and main < p_floats:
            tail = buf[main:p_floats]
            if dist.get_backend(group) != "nccl":
                t = tail.clone()
                dist.broadcast(t, src=dist.get_global_rank(group, world - 1) if group is not None else world - 1,
                               group=group)
                tail.copy_(t)
            else:
                dist.broadcast(tail, src=dist.get_global_rank(group, world - 1) if group is not None else world - 1,
                               group=group)


class PeerExchange:
    """Every rank's FieldGrads and parameter buffers mapped into this process
    for ``ssr_exchange_adam``: each rank exports its buffers' CUDA IPC handles
    (``ssr_ipc_export``) and opens the others' on its own device with lazy
    peer access (``ssr_ipc_open``), so the kernel addresses them over NVLink /
    NVSwitch (or, ranks sharing one GPU, that GPU's memory).  The mapping is
    re-done when any rank's buffers move (a densify reallocates them)."""

    def __init__(self, group=None):
        self.group = group
        self._keys = None
        self._ptrs = None
        self._opened = []  # handles this process opened (closed on re-mapping)
        self._flag = None
        self._epoch = self._local_key = None

    def _gather(self, obj):
        import torch.distributed as dist

        out = [None] * dist.get_world_size(self.group)
        dist.all_gather_object(out, obj, group=self.group)
        return out

    def _close(self):
        for h in self._opened:
            _lib.call_rc("ssr_ipc_close", h)
        self._opened = []

    def _map(self, t, rank):
        """Every rank's address of its copy of the buffer ``t`` (this rank's:
        ``t.data_ptr()``).  A failure on any rank raises RuntimeError on every
        rank (each step is a collective), so the ranks never disagree about
        whether the mapping exists."""
        import ctypes

        h = (ctypes.c_uint8 * 64)()
        off = ctypes.c_int64(0)
        rc = _lib.call_rc("ssr_ipc_export", t.data_ptr(), h, ctypes.byref(off))
        mine = (True, (bytes(h), off.value)) if rc == 0 else (False, _lib.load().ssr_last_error().decode())
        shared = self._gather(mine)
        bad = [str(x) for ok, x in shared if not ok]
        if bad:
            raise RuntimeError(f"peer mapping unavailable: {bad[0]}")
        out, err = [], None
        for q, (_, (handle, offset)) in enumerate(shared):
            if q == rank:
                out.append(t.data_ptr())
                continue
            p = ctypes.c_void_p(0)
            hb = (ctypes.c_uint8 * 64).from_buffer_copy(handle)
            if _lib.call_rc("ssr_ipc_open", hb, offset, ctypes.byref(p)) != 0:
                err = _lib.load().ssr_last_error().decode()
                break
            self._opened.append(hb)
            out.append(int(p.value))
        errs = [x for x in self._gather(err) if x]
        if errs:
            raise RuntimeError(f"peer mapping unavailable: {errs[0]}")
        return out

    def pointers(self, grads_flat: torch.Tensor, params_flat: torch.Tensor, epoch=None):
        """(grads, params): per-rank device addresses, rank order.

        ``epoch``: a value every rank changes at the same step whenever its
        buffers may have moved (exchange_p2p passes the field's identity,
        generation and size); while it stays the same no collective runs here
        (the mapping is reused), and a buffer that moved anyway raises.  Without
        it, the ranks compare buffer addresses collectively on every call."""
        import torch.distributed as dist

        rank = dist.get_rank(self.group)
        key = (grads_flat.data_ptr(), grads_flat.numel(), params_flat.data_ptr(), params_flat.numel())
        if epoch is not None and self._ptrs is not None and epoch == self._epoch:
            if key != self._local_key:
                raise RuntimeError("exchange buffers moved without a new epoch")
            return self._ptrs
        keys = self._gather(key)
        if keys != self._keys:
            self._close()
            self._ptrs = self._keys = None
            self._ptrs = (self._map(grads_flat, rank), self._map(params_flat, rank))
            self._keys = keys
        self._epoch, self._local_key = epoch, key
        return self._ptrs

    def probe(self, grads_flat: torch.Tensor, params_flat: torch.Tensor):
        """(True, "") when every rank can map every rank's buffers, else
        (False, reason) on every rank (a collective)."""
        try:
            self.pointers(grads_flat, params_flat)
            return True, ""
        except RuntimeError as e:
            self._close()
            self._keys = self._ptrs = None
            return False, str(e)

    def barrier(self, device) -> None:
        """Stream-ordered barrier: a one-element NCCL all-reduce completes on a
        rank only once every rank's stream has reached it (gloo: host barrier
        after a device synchronise)."""
        import torch.distributed as dist

        if dist.get_backend(self.group) == "nccl":
            if self._flag is None or self._flag.device != device:
                self._flag = torch.zeros(1, dtype=torch.float32, device=device)
            dist.all_reduce(self._flag, group=self.group)
        else:
            torch.cuda.synchronize(device)
            dist.barrier(group=self.group)


def exchange_p2p(field, grads, optimizer, position_rate: float, exchanger: PeerExchange) -> None:
    """The sharded exchange as one fused kernel per rank over peer memory
    (``ssr_exchange_adam``): reduce-scatter, Adam on the rank's chunk and the
    all-gather of the new parameters in one pass, plus the summed densify
    statistics in every rank's ``grads``.  Moments as in ``mode="sharded"``
    (``gather_moments(mode="p2p")`` before a densify)."""
    import ctypes

    import torch.distributed as dist

    from .optim import SH_REST_LR

    group = exchanger.group
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    optimizer.check(field)
    # the field's generation moves with every reallocation (insert / densify),
    # identically on every rank: the mapping is re-checked only then
    gp, pp = exchanger.pointers(grads.flat, field.flat,
                                epoch=(id(field), getattr(field, "generation", 0), len(field), grads.flat.numel()))
    arr = ctypes.c_void_p * world
    dev = field.flat.device
    exchanger.barrier(dev)  # every rank's gradient sums are final
    lr, bc1, bc2 = optimizer.advance(position_rate)
    field.version += 1
    _lib.call("ssr_exchange_adam", len(field), field.sh_degree, world, rank, arr(*gp), arr(*pp), optimizer.m.data_ptr(),
              optimizer.v.data_ptr(), lr, SH_REST_LR, bc1, bc2, _lib.stream_ptr())
    exchanger.barrier(dev)  # every replica holds every rank's chunk


def densify_top_fraction(state: TrainState, fraction: float) -> None:
    """Config-4 rule (BASELINE: "densify/prune of 5% per 100 iterations"):
    the clone/split threshold is the (1 - fraction) quantile of the averaged
    screen-gradient statistic over rows seen at least once, so the hottest
    ``fraction`` of the field densifies; prune and size rules are the
    reference's (field.py:321-327, where the threshold is a fixed 2e-4)."""
    n = len(state.field)
    accum, count = state.stats[:n], state.stats[n:]
    grad_stats = accum / torch.clamp(count, min=1.0)
    seen = grad_stats[count > 0]
    thr = float(torch.quantile(seen.double(), 1.0 - fraction)) if seen.numel() else float("inf")
    opts = DensifyOptions(**{**state.densify.__dict__, "scene_extent": state.scene_extent, "grad_threshold": thr})
    state.field.densify_and_prune(grad_stats, opts, state.rng, optimizer=state.optimizer)
    state.stats = torch.zeros(2 * len(state.field), dtype=torch.float32, device=state.field.flat.device)


class SemiGlobalBatch:
    """View-sharded multi-view step: sum_v grad(view v) at fixed parameters.

    Batch rule (documented deviation): gradients of the batch's
    views are summed; the position rate is the mean of the per-view rates.
    Each rank renders and differentiates its contiguous shard of the views into
    one flat buffer (``backward(accumulate=True)``), the buffers are combined by
    ``exchange_and_step`` (all-reduce, or reduce-scatter -> sharded Adam ->
    all-gather), and ``densify_every`` batch steps the field densifies, either
    by the reference's fixed threshold or, with ``densify_fraction`` set, by the
    config-4 top-fraction rule.
    """

    def __init__(self, state: TrainState, group=None, mode: str = "allreduce", densify_every: int = 0,
                 densify_fraction: float | None = None):
        self.state = state
        self.group = group
        self.mode = mode
        self.densify_every = int(densify_every)
        self.densify_fraction = densify_fraction
        self._grads = None
        self._exchanger = PeerExchange(group) if mode == "p2p" else None

    def _buffer(self):
        f = self.state.field
        if self._grads is None or self._grads._n != len(f) or self._grads.flat.device != f.flat.device:
            self._grads = FieldGrads.zeros(len(f), f.sh_degree, f.flat.device)
        else:
            self._grads.flat.zero_()
        return self._grads

    def step(self, cams, targets, position_rates, rank: int = 0, world: int = 1, bg=(0.0, 0.0, 0.0)):
        st = self.state
        f = st.field
        idx = shard_views(list(range(len(cams))), rank, world)
        grads = self._buffer()
        losses = []
        for i in idx:
            out = render(f, cams[i], bg=bg, soft_count=st.weights.load > 0)
            br = total_loss(out.image, targets[i], out, st.weights)
            backward(f, out, br.d_image, br.d_soft, layout=st.layout, grads=grads, accumulate=True)
            losses.append(br)
        rate = float(np.mean(position_rates)) if len(position_rates) else 0.0
        exchange_and_step(f, grads, st.optimizer, rate, mode=self.mode, group=self.group, exchanger=self._exchanger)
        n = len(f)
        st.stats[:n] += grads.screen_norms
        st.stats[n:] += grads.visible_count
        st.global_iteration += 1
        if self.densify_every and st.global_iteration % self.densify_every == 0:
            if self.mode in ("sharded", "p2p") and world > 1:
                gather_moments(f, st.optimizer, self.group, mode=self.mode)
            if self.densify_fraction:
                densify_top_fraction(st, self.densify_fraction)
            else:
                densify(st)
        return grads, losses
