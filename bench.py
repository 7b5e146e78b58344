"""Benchmark: fwd+bwd raster iterations/s at 1M Gaussians 1080p (BASELINE config 2).

One step = one training iteration of the hot path per GPU on one view:
render (preprocess + tile sort + forward) -> fused loss (L1 + 0.2 D-SSIM) ->
backward (splat-parallel + chain) -> fused Adam (+ densify statistics),
i.e. pipeline.py:_train_one_iteration on device.  With N GPUs every rank
trains its own view each step and the ranks' gradients are combined before the
identical Adam step (train.exchange_and_step; weak scaling: value =
N * steps / time).

Extra blocks on the same JSON line (each its own workload, timed the same way):
  paper_objective      config 2 under the reference's default LossWeights() (load 0.41)
  no_splat_parallel    config 2 with the pixel-parallel backward (the paper's No_SPB ablation)
  small_configs        configs 0 and 1 at N=1 (launch- and latency-bound sizes)
  semi_global_batch    config 4: 3M Gaussians, a 64-view 1080p batch sharded 64/N per rank,
                       summed gradients exchanged once per batch (strong scaling)
  progressive          config 3 seconds per new image (reference plan replayed), both objectives
  cpu_baseline         the float64 C port of the reference on the host cores

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--config C]

--impl reference times the CPU reference path instead: the float64 C port of
the reference rasterizer (oracle/, OpenMP over every host core) on the same
workload and metric; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fwd+bwd raster iters/s at 1M Gaussians 1080p"
FLOP_FWD_PER_PAIR = 30.0  # forward ~30 flops per walked pair
FLOP_BWD_PER_PAIR = 80.0  # backward ~80 flops per walked pair (incl. reduction)


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--views", type=int, default=8)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--progressive-events", type=int, default=5,
                    help="also time the progressive loop (config 3, seconds per new image) over this many "
                         "events after one warm-up event; 0 skips it (single GPU only)")
    ap.add_argument("--fused", type=int, default=1,
                    help="1 (default): chain + Adam in one pass (backward_and_step); 0: backward() + optimizer.step()")
    ap.add_argument("--e2e-target", default="u8", choices=["u8", "f32"],
                    help="e2e upload of each step's target image: 8-bit like the reference's image files "
                         "(io/images.py; read natively by the loss kernels) or float32")
    ap.add_argument("--exchange", default="auto", choices=["auto", "allreduce", "sharded", "p2p"],
                    help="N > 1: how the ranks' gradient sums meet (train.exchange_and_step; p2p = the "
                         "fused ssr_exchange_adam kernel over peer memory; auto = p2p when every rank "
                         "can map every rank's buffers, else allreduce)")
    ap.add_argument("--batch-views", type=int, default=64, help="semi_global_batch: views per batch (config 4)")
    ap.add_argument("--batch-steps", type=int, default=2, help="semi_global_batch: timed batches (0 skips)")
    ap.add_argument("--extra-steps", type=int, default=10,
                    help="timed steps of the paper_objective / no_splat_parallel legs (0 skips them)")
    return ap.parse_args()


def _workload(cfg):
    from paper_2503_13086_b200 import scenes

    c = scenes.CONFIGS[cfg]
    return (f"config{cfg}: {c['n']:,} Gaussians SH{c['sh_degree']} {c['width']}x{c['height']}, "
            "one view per GPU per step: render + L1/D-SSIM loss + splat-parallel backward + Adam")


def _views(args):
    # spread the ring cameras of config 2 over the circle
    return [v * (64 // max(args.views, 1)) for v in range(args.views)]


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def _host_cores() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


class ClockSampler:
    """nvidia-smi equivalent via NVML, sampled during the timed region."""

    def __init__(self, dev_index=0, period=0.01):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.period, self._stop, self._t = period, threading.Event(), None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # pragma: no cover - NVML missing
            self.nv = None

    _BITS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
             0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting", 0x1: "gpu_idle"}

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self._BITS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_mhz_min": float(np.min(self.samples)),
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def _dist():
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        # SSR_DIST_BACKEND / SSR_FORCE_DEVICE0: functional checks of the N > 1 path
        # on a one-GPU box (gloo, every rank on cuda:0) -- never a measurement
        backend = os.environ.get("SSR_DIST_BACKEND") or ("nccl" if torch.cuda.is_available() else "gloo")
        dist.init_process_group(backend)
    if os.environ.get("SSR_FORCE_DEVICE0"):
        local = 0
    return rank, world, local


# ------------------------------------------------------------------ CPU reference arm
def _oracle_iteration(orc, P, opt, cam, target, weights):
    out = orc.render(P, cam)
    br = orc.total_loss(out["image"], target, out["soft_count"], out["hard_count"], weights)
    g = orc.backward(P, out, br["d_image"], br["d_soft"])
    opt.step(P, g, position_rate=1.6e-4)
    return br["total"]


class _CpuWorkload:
    """The GPU arm's workload for the C port: same field, same 8 ring views in
    the same order, targets rendered (untimed, lazily) from the second seed."""

    def __init__(self, cfg, views):
        from oracle import oracle as orc
        from paper_2503_13086_b200 import scenes

        orc.build()
        self.orc = orc
        hp = scenes.make_params(cfg, seed=0)
        self.P = orc.Params(*(getattr(hp, k).astype(np.float64) for k in (
            "positions", "rotations", "log_scales", "opacity_logits", "sh")))
        tp = scenes.make_params(cfg, seed=1)
        self.TP = orc.Params(*(getattr(tp, k).astype(np.float64) for k in (
            "positions", "rotations", "log_scales", "opacity_logits", "sh")))
        self.cams = [scenes.camera(cfg, view=v) for v in views]
        self.targets = {}
        self.opt = orc.Optimizer(self.P, scene_extent=6.6)
        self.w = orc.LossWeights(l1=1.0, ssim=0.2, load=0.0)

    def target(self, i):
        if i not in self.targets:
            self.targets[i] = self.orc.render(self.TP, self.cams[i])["image"]
        return self.targets[i]

    def iteration(self, k):
        i = k % len(self.cams)
        t = self.target(i)
        return _oracle_iteration(self.orc, self.P, self.opt, self.cams[i], t, self.w)


def cpu_baseline(cfg, views, budget_s=25.0, max_iters=3, single_thread=True):
    wl = _CpuWorkload(cfg, views)
    wl.orc.set_threads(_host_cores())
    wl.target(0)
    n, t0 = 0, time.perf_counter()
    while n < max_iters and (n < 1 or time.perf_counter() - t0 < budget_s / 2):
        wl.iteration(n)
        n += 1
    dt = time.perf_counter() - t0
    out = {"value": n / dt, "unit": "iters/s", "cores": wl.orc.num_threads(), "kind": "port",
           "cpu_model": _cpu_model(), "host_cores": _host_cores(),
           "sample": f"{n} full iteration(s) (render+loss+backward+Adam) of {_workload(cfg).split(',')[0]} on the "
                     f"GPU arm's ring views in its order, float64 C port of the reference (oracle/), OpenMP"}
    if single_thread:
        # workers=1: one iteration on one host thread
        wl.orc.set_threads(1)
        t1 = time.perf_counter()
        wl.iteration(n)
        out["single_thread"] = {"value": 1.0 / (time.perf_counter() - t1), "unit": "iters/s", "cores": 1,
                                "sample": "1 iteration, same workload, 1 OpenMP thread"}
        wl.orc.set_threads(_host_cores())
    return out


def run_reference(args):
    rank, world, _ = _dist()
    if rank != 0:
        return
    wl = _CpuWorkload(args.config, _views(args))
    # every host core: torchrun sets OMP_NUM_THREADS=1 for its workers, which
    # would understate the reference arm at N > 1
    wl.orc.set_threads(_host_cores())
    for i in range(len(wl.cams)):  # the targets are inputs: rendered before the timed region
        if i < max(args.steps, 1) + 1:
            wl.target(i)
    wl.iteration(0)  # one warm-up iteration is enough for the C port
    t0 = time.perf_counter()
    k = 0
    budget = 150.0
    while k < args.steps:
        wl.iteration(1 + k)
        k += 1
        if time.perf_counter() - t0 > budget:
            break
    dt = time.perf_counter() - t0
    val = k / dt
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "iters/s", "n_gpus": world,
            "steps": k, "steps_requested": args.steps, "warmup": args.warmup, "ms_per_step": dt / k * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (BASELINE config generator, seeded)",
            "config": {"workload": _workload(args.config), "views": len(wl.cams), "parallelism": "host threads"},
            "cpu_baseline": {"value": val, "unit": "iters/s", "cores": wl.orc.num_threads(), "kind": "port",
                             "cpu_model": _cpu_model(),
                             "sample": f"{k} iteration(s) cycling the GPU arm's {len(wl.cams)} views in its order, "
                                       f"float64 C port of the reference, {wl.orc.num_threads()} OpenMP threads"},
            "e2e": {"value": val, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm helpers
def _device_loop(fn, steps):
    """Device ms of `steps` calls of fn(k), CUDA events on the launching stream."""
    import torch

    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(steps):
        fn(k)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def small_configs(args, local, steps=20):
    """Configs 0 and 1 (BASELINE's CPU-reference case and the 200k/800x800
    case) at N=1: the same single-view iteration, device-timed."""
    import torch

    from paper_2503_13086_b200 import GaussianField, scenes
    from paper_2503_13086_b200.losses import LossWeights
    from paper_2503_13086_b200.optim import FieldOptimizer
    from paper_2503_13086_b200.rasterize import render
    from paper_2503_13086_b200.train import TrainState, train_iteration

    out = {}
    for cfg in (0, 1):
        cams = [scenes.camera(cfg, view=v) for v in range(8)]
        tf = GaussianField.from_host(scenes.make_params(cfg, seed=1))
        targets = [render(tf, c, for_backward=False).image.clone() for c in cams]
        del tf
        f = GaussianField.from_host(scenes.make_params(cfg, seed=0))
        st = TrainState(field=f, optimizer=FieldOptimizer(f, scene_extent=4.4 if cfg == 0 else 5.5),
                        weights=LossWeights(l1=1.0, ssim=0.2, load=0.0), densify_enabled=False)
        for k in range(8 + 3):
            train_iteration(st, cams[k % 8], targets[k % 8], 1.6e-4)
        ms = _device_loop(lambda k: train_iteration(st, cams[k % 8], targets[k % 8], 1.6e-4), steps)
        c = scenes.CONFIGS[cfg]
        out[f"config{cfg}"] = {"value": steps / (ms / 1e3), "unit": "iters/s", "ms_per_step": ms / steps,
                               "workload": f"{c['n']:,} Gaussians SH{c['sh_degree']} {c['width']}x{c['height']}, "
                                           "render + L1/D-SSIM + backward + Adam, 8 views cycled"}
        del st, f, targets
        torch.cuda.empty_cache()
    return out


def semi_global_batch(args, rank, world, local):
    """Config 4: 3M Gaussians, a fixed batch of views sharded over the ranks."""
    import torch
    import torch.distributed as dist

    from paper_2503_13086_b200 import GaussianField, _lib, scenes
    from paper_2503_13086_b200.losses import LossWeights
    from paper_2503_13086_b200.optim import FieldOptimizer
    from paper_2503_13086_b200.rasterize import render
    from paper_2503_13086_b200.train import SemiGlobalBatch, TrainState, shard_views

    cfg = 4
    nv = args.batch_views
    cams = [scenes.camera(cfg, view=v * (64 // max(1, min(nv, 64))) % 64 if nv <= 64 else v) for v in range(nv)]
    mine = shard_views(list(range(nv)), rank, world)
    tf = GaussianField.from_host(scenes.make_params(cfg, seed=1))
    targets = [None] * nv
    for i in mine:  # 8-bit targets, as the reference's image files (io/images.py)
        targets[i] = (render(tf, cams[i], for_backward=False).image * 255.0).round().clamp(0, 255).to(torch.uint8)
    del tf
    torch.cuda.empty_cache()
    field = GaussianField.from_host(scenes.make_params(cfg, seed=0))
    state = TrainState(field=field, optimizer=FieldOptimizer(field, scene_extent=6.6),
                       weights=LossWeights(l1=1.0, ssim=0.2, load=0.0), scene_extent=6.6)
    batch = SemiGlobalBatch(state, mode=args.exchange, densify_every=100, densify_fraction=0.05)
    rates = [1.6e-4] * nv
    batch.step(cams, targets, rates, rank=rank, world=world)  # warm-up batch
    if world > 1:
        dist.barrier()
    with ClockSampler(local) as clk:
        ms = _device_loop(lambda k: batch.step(cams, targets, rates, rank=rank, world=world), args.batch_steps)
    if world > 1:
        dist.barrier()
    _lib.enable_timers(True)
    batch.step(cams, targets, rates, rank=rank, world=world)
    stage_ms = _lib.timer_ms()
    _lib.enable_timers(False)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=field.flat.device)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    out = None
    if rank == 0:
        P = 0
        for i in mine[:2]:
            P += int(render(field, cams[i], for_backward=False).n_walk.sum())
        P /= max(1, min(2, len(mine)))
        bwd_ms = stage_ms.get("ssr_backward", 0.0)
        sm_count = torch.cuda.get_device_properties(field.flat.device).multi_processor_count
        fp32_peak = sm_count * 128 * 2 * 1965.0e6 / 1e12
        ach = FLOP_BWD_PER_PAIR * P / (bwd_ms / 1e3) / 1e12 if bwd_ms else None
        out = {"metric": "semi-global batches/s (64-view batch, config 4)", "value": args.batch_steps / (ms / 1e3),
               "unit": "batches/s", "views_per_s": nv * args.batch_steps / (ms / 1e3),
               "ms_per_batch": ms / args.batch_steps, "batches": args.batch_steps, "n_gpus": world,
               "views_per_batch": nv, "views_per_rank": len(mine), "scaling": "strong", "exchange": args.exchange,
               "n_gaussians": len(field), "width": cams[0].width, "height": cams[0].height,
               "densify": "every 100 batch steps: hottest 5% clone/split (train.densify_top_fraction)",
               "walked_pairs_per_view": P,
               "roofline": {"bound": "fp32", "kernel": "ssr_backward (per view)", "achieved": ach, "peak": fp32_peak,
                            "unit": "TFLOP/s", "frac": (ach / fp32_peak) if ach else None},
               "stage_ms_per_call": {k: round(v, 4) for k, v in stage_ms.items() if not k.endswith("workspace")},
               "clocks": clk.summary()}
    del state, batch, field, targets
    torch.cuda.empty_cache()
    return out


# ------------------------------------------------------------------ GPU arm
def main():
    args = _args()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    from paper_2503_13086_b200 import GaussianField, _lib, scenes
    from paper_2503_13086_b200.losses import LossWeights, total_loss
    from paper_2503_13086_b200.optim import FieldOptimizer
    from paper_2503_13086_b200.rasterize import backward, render
    from paper_2503_13086_b200.rasterize.backward import FieldGrads, backward_and_step
    from paper_2503_13086_b200.train import PeerExchange, TrainState, exchange_and_step

    rank, world, local = _dist()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg = args.config
    views = _views(args)
    hp = scenes.make_params(cfg, seed=0)
    tp = scenes.make_params(cfg, seed=1)
    cams = [scenes.camera(cfg, view=v) for v in views]
    tfield = GaussianField.from_host(tp)
    targets = [render(tfield, c, for_backward=False).image.clone() for c in cams]
    del tfield
    field = GaussianField.from_host(hp)
    state = TrainState(field=field, optimizer=FieldOptimizer(field, scene_extent=6.6),
                       weights=LossWeights(l1=1.0, ssim=0.2, load=0.0), scene_extent=6.6)
    rate = 1.6e-4
    n = len(field)

    grads_buf = [None]
    layout = ["splat"]
    exchanger = None
    exchange_note = None
    if world > 1 and args.exchange in ("auto", "p2p"):
        # the fused peer-memory exchange when every rank can map every rank's
        # buffers (decided collectively: all ranks take the same branch)
        grads_buf[0] = FieldGrads.zeros(n, field.sh_degree, dev)
        exchanger = PeerExchange()
        ok, why = exchanger.probe(grads_buf[0].flat, field.flat)
        if not ok:
            if args.exchange == "p2p":
                raise SystemExit(f"--exchange p2p: {why}")
            exchanger, exchange_note = None, f"p2p unavailable ({why}); all-reduce"
        args.exchange = "p2p" if exchanger is not None else "allreduce"
    elif args.exchange == "auto":
        args.exchange = "allreduce"

    def step(k, target=None, values_out=None):
        cam_i = (k * world + rank) % len(cams)
        cam = cams[cam_i]
        # soft counts only when the objective reads them (load weight > 0, losses.py:155-160)
        out = render(state.field, cam, soft_count=state.weights.load > 0)
        br = total_loss(out.image, targets[cam_i] if target is None else target, out, state.weights,
                        values_out=values_out)
        if world > 1:
            # one view per rank: the chain writes every row (accumulate=False), so
            # the buffer needs no zero fill; the flat buffer is the exchange unit
            if grads_buf[0] is None:
                grads_buf[0] = FieldGrads.zeros(n, field.sh_degree, dev)
            grads = grads_buf[0]
            backward(state.field, out, br.d_image, br.d_soft, grads=grads, accumulate=False, layout=layout[0])
            exchange_and_step(state.field, grads, state.optimizer, rate, mode=args.exchange, exchanger=exchanger)
            state.stats[:n] += grads.screen_norms
            state.stats[n:] += grads.visible_count
        elif args.fused:
            backward_and_step(state.field, out, br.d_image, br.d_soft, state.optimizer, rate, stats=state.stats,
                              layout=layout[0])
        else:
            grads = backward(state.field, out, br.d_image, br.d_soft, stats=state.stats, layout=layout[0])
            state.optimizer.step(state.field, grads, position_rate=rate)
        state.global_iteration += 1
        return br

    def barrier():
        if world > 1:
            dist.barrier()

    # the e2e loop below replays the warm-up from this same state (field,
    # moments, step counts, densify statistics), so both loops time the same
    # iterations on the same field
    opt = state.optimizer
    snap = (field.flat.clone(), opt.m.clone(), opt.v.clone(), dict(opt.steps), state.stats.clone(),
            state.global_iteration)

    def restore():
        field.flat.copy_(snap[0])
        opt.m.copy_(snap[1])
        opt.v.copy_(snap[2])
        opt.steps = dict(snap[3])
        state.stats.copy_(snap[4])
        state.global_iteration = snap[5]

    # prime the caching allocator with every view's buffer sizes (instance counts
    # differ per view), then the W warm-up steps proper
    def prime_and_warm():
        for k in range(len(cams) // world):
            step(k)
        for k in range(args.warmup):
            step(k)
        torch.cuda.synchronize()

    prime_and_warm()
    # ---------------- timed region (device time, CUDA events on the launching stream)
    barrier()
    with ClockSampler(local) as clk:
        ms = _device_loop(lambda k: step(args.warmup + k), args.steps)
    barrier()
    # per-ABI-call device times, from a separate (untimed) pass: the event pairs
    # around every call would otherwise perturb the timed region
    _lib.enable_timers(True)
    for k in range(min(args.steps, 5)):
        step(args.warmup + k)
    stage_ms = _lib.timer_ms()
    _lib.enable_timers(False)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    value = world * args.steps / (ms / 1e3)

    # ---------------- end to end through the public API with host buffers
    # Every step copies its target image from pinned host memory (H2D) and reads
    # its loss terms back (D2H).  The H2D of step k+1 runs on a copy stream
    # while step k computes (double-buffered, ordered by events); step k's
    # loss read is consumed on the host one step later.
    if args.e2e_target == "u8":
        pinned = [(t * 255.0).round().clamp(0, 255).to(torch.uint8).cpu().pin_memory() for t in targets]
    else:
        pinned = [t.cpu().pin_memory() for t in targets]
    dbuf = [torch.empty_like(pinned[0], device=dev) for _ in range(2)]
    host_vals = [torch.empty(5, dtype=torch.float64).pin_memory() for _ in range(2)]
    copy_stream = torch.cuda.Stream()
    main_stream = torch.cuda.current_stream()
    loaded = [torch.cuda.Event() for _ in range(2)]
    consumed = [torch.cuda.Event() for _ in range(2)]
    read_done = [torch.cuda.Event() for _ in range(2)]
    losses_seen = []

    # the same view sequence as the device-timed loop, so the two numbers
    # measure the same workload
    def view_of(k):
        return ((args.warmup + k) * world + rank) % len(cams)

    def prefetch(k):
        b = k % 2
        with torch.cuda.stream(copy_stream):
            copy_stream.wait_event(consumed[b])  # the step that last read this buffer is done with it
            dbuf[b].copy_(pinned[view_of(k)], non_blocking=True)
            loaded[b].record(copy_stream)

    # the e2e path's own kernels (8-bit-target loss, mapped loss output) load
    # lazily on first use: run it twice before restoring the snapshot
    for k in range(2):
        dbuf[0].copy_(pinned[view_of(k)])
        step(args.warmup + k, target=dbuf[0], values_out=host_vals[0])
    torch.cuda.synchronize()
    restore()
    prime_and_warm()
    barrier()
    torch.cuda.synchronize()
    for e in consumed:
        e.record(main_stream)
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    prof = None
    if os.environ.get("SSR_E2E_GAPS"):  # diagnostics: device-timeline gaps of the e2e loop (stderr)
        from torch.profiler import ProfilerActivity, profile

        prof = profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA])
        prof.__enter__()
    f0.record()
    prefetch(0)
    for k in range(args.steps):
        b = k % 2
        main_stream.wait_event(loaded[b])
        # the loss kernel writes the step's five loss terms (40 bytes) straight
        # into pinned host memory (mapped), so no copy sits in the stream
        step(args.warmup + k, target=dbuf[b], values_out=host_vals[b])
        consumed[b].record(main_stream)
        # the next step's upload is issued once this step is queued (after its
        # instance-count read): it overlaps the forward / backward instead of
        # the preprocess and the depth sort (+2% e2e)
        if k + 1 < args.steps:
            prefetch(k + 1)
        read_done[b].record(main_stream)
        if k > 0:
            read_done[1 - b].synchronize()
            losses_seen.append(float(host_vals[1 - b][3]))
    read_done[(args.steps - 1) % 2].synchronize()
    losses_seen.append(float(host_vals[(args.steps - 1) % 2][3]))
    f1.record()
    torch.cuda.synchronize()
    if prof is not None:
        prof.__exit__(None, None, None)
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import contextlib

        from gap_profile import analyse

        with contextlib.redirect_stdout(sys.stderr):
            analyse(prof, args.steps)
    barrier()
    assert len(losses_seen) == args.steps and all(np.isfinite(losses_seen))
    e2e_ms = torch.tensor([f0.elapsed_time(f1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_val = world * args.steps / (float(e2e_ms.item()) / 1e3)

    # ---------------- kernel launches of one step (CUPTI via torch.profiler)
    launches = None
    try:
        from torch.profiler import ProfilerActivity, profile

        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            step(0)
            torch.cuda.synchronize()
        names = [e.name for e in prof.events() if e.device_type.name == "CUDA" and "ssr" in e.name]
        launches = len(names) * args.steps
    except Exception:
        pass

    # ---------------- the same workload under other settings (paper objective, No_SPB ablation)
    extras = {}
    if args.extra_steps > 0:
        for name, weights, lay in (("paper_objective", LossWeights(), "splat"),
                                   ("no_splat_parallel", state.weights, "pixel")):
            restore()
            keep_w = state.weights
            state.weights, layout[0] = weights, lay
            for k in range(3):
                step(k)
            barrier()
            ms_x = _device_loop(lambda k: step(args.warmup + k), args.extra_steps)
            _lib.enable_timers(True)
            for k in range(3):
                step(args.warmup + k)
            st_x = _lib.timer_ms()
            _lib.enable_timers(False)
            ms_xt = torch.tensor([ms_x], dtype=torch.float64, device=dev)
            if world > 1:
                dist.all_reduce(ms_xt, op=dist.ReduceOp.MAX)
            extras[name] = {"value": world * args.extra_steps / (float(ms_xt.item()) / 1e3), "unit": "iters/s",
                            "steps": args.extra_steps, "ms_per_step": float(ms_xt.item()) / args.extra_steps,
                            "objective": "LossWeights() = (0.47, 0.12, 0.41) (losses.py:24-27)"
                            if name == "paper_objective" else "L1 + 0.2 D-SSIM",
                            "backward_layout": lay, "backward_ms": round(st_x.get("ssr_backward", 0.0), 4)}
            state.weights, layout[0] = keep_w, "splat"

    # ---------------- roofline of the dominant kernel
    roofline = roofline_hbm = None
    P_mean = M_mean = 0.0
    if rank == 0:
        P = M = 0
        for c in cams:
            o = render(state.field, c, for_backward=False)
            P += int(o.n_walk.sum().item())
            M += o.splats.n_instances
        P_mean, M_mean = P / len(cams), M / len(cams)
        sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
        peaks = {}
        try:
            peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        except Exception:
            pass
        sm_max = float(peaks.get("sm_max_mhz", 1965.0))
        fp32_peak = sm_count * 128 * 2 * sm_max * 1e6 / 1e12  # TFLOP/s (no measured fp32 peak exists)
        fwd_ms = stage_ms.get("ssr_forward", 0.0)
        bwd_ms = stage_ms.get("ssr_backward", 0.0)
        if bwd_ms >= fwd_ms:
            dom, flops, dms = ("ssr_backward (k_backward_splat2 + k_backward_fixup)",
                               FLOP_BWD_PER_PAIR * P_mean, bwd_ms)
        else:
            dom, flops, dms = "ssr_forward (k_forward + k_forward_fixup)", FLOP_FWD_PER_PAIR * P_mean, fwd_ms
        achieved = flops / (dms / 1e3) / 1e12
        traffic = None
        try:
            prof_sum = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
            traffic = prof_sum.get(dom.split(" ")[0])
        except Exception:
            pass
        roofline = {"bound": "fp32", "kernel": dom, "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
                    "frac": achieved / fp32_peak, "traffic": traffic,
                    "peak_source": f"nominal {sm_count} SMs x 128 FMA/clk x 2 x {sm_max:.0f} MHz "
                                   "(MEASURED_PEAKS.json has no fp32 figure)",
                    "work": f"{flops / 1e9:.2f} GFLOP per launch = "
                            f"{FLOP_BWD_PER_PAIR if 'backward' in dom else FLOP_FWD_PER_PAIR:.0f}"
                            f" flop x {P_mean / 1e6:.1f} M walked pairs"}
        # HBM roofline of the streaming optimizer pass against the measured copy
        # bandwidth: k_adam moves 7 x S bytes per row (p, g, m, v read; p, m, v
        # written); the fused chain+Adam 6 x S bytes per row plus the 36-byte
        # instance rows it merges
        s_bytes = 4 * (11 + 3 * (field.sh_degree + 1) ** 2)
        n_rows = len(state.field)
        kms = None
        if stage_ms.get("ssr_adam"):
            kname, kms = "ssr_adam (k_adam)", stage_ms["ssr_adam"]
            kbytes = 7.0 * s_bytes * n_rows
            work = f"7 x {s_bytes} B x {n_rows:,} rows"
        elif stage_ms.get("ssr_chain_adam"):
            kname, kms = ("ssr_chain_adam (k_merge_big + k_chain_geo + k_chain_sh, fused Adam)",
                          stage_ms["ssr_chain_adam"])
            kbytes = 6.0 * s_bytes * n_rows + 40.0 * M_mean  # 10-word tagged rows
            work = f"6 x {s_bytes} B x {n_rows:,} rows + 40 B x {M_mean:,.0f} instance rows"
        if kms:
            hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
            ach = kbytes / (kms / 1e3) / 1e9
            roofline_hbm = {"bound": "hbm", "kernel": kname, "achieved": ach, "peak": hbm_peak, "unit": "GB/s",
                            "frac": ach / hbm_peak, "peak_source": "measured" if "hbm_gbs" in peaks else "fallback",
                            "work": f"{kbytes / 1e9:.3f} GB per launch = {work}", "traffic": None}
            try:
                tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
                roofline_hbm["traffic"] = tr.get("ssr_adam") if "k_adam" in kname else (
                    (tr.get("ssr_chain_sh_fused") or 0) + (tr.get("ssr_chain_geo_fused") or 0) or None)
            except Exception:
                pass
    h2d = int(pinned[0].numel() * pinned[0].element_size())
    del state, targets, pinned, dbuf
    grads_buf[0] = None
    torch.cuda.empty_cache()

    # ---------------- config 4: the semi-global view batch (every rank takes part)
    batch_block = None
    if args.batch_steps > 0:
        try:
            batch_block = semi_global_batch(args, rank, world, local)
        except Exception as ex:  # pragma: no cover
            batch_block = {"error": f"{type(ex).__name__}: {ex}"}
    if rank != 0:
        return
    small = None
    if world == 1 and args.extra_steps > 0:
        try:
            small = small_configs(args, local)
        except Exception as ex:  # pragma: no cover
            small = {"error": f"{type(ex).__name__}: {ex}"}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(cfg, views)
        except Exception as ex:  # pragma: no cover
            cpu = {"value": None, "error": str(ex)}
    # ---------------- seconds per new image (BASELINE metric, second half): config 3
    progressive = None
    if world == 1 and args.progressive_events > 0:
        import contextlib
        import io

        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import progressive as prog

        progressive = {}
        for name, extra in (("bench_objective", []), ("paper_objective", ["--paper-weights"])):
            try:
                torch.cuda.empty_cache()
                with contextlib.redirect_stdout(io.StringIO()), ClockSampler(local, period=0.05) as pclk:
                    summ = prog.main(["--events", str(args.progressive_events), "--warmup-events", "1"] + extra)
                progressive[name] = {
                    "metric": "seconds per new image", "value": summ["value"], "unit": "s/image",
                    "higher_is_better": False, "median": summ["median"], "worst": summ["worst"],
                    "events": summ["events"],
                    "field_final": summ["field_final"], "objective": summ["objective"],
                    "value_with_reference_scheduler": summ["value_with_reference_scheduler"],
                    "clocks": pclk.summary(),
                    "config": "config 3: 1297x840, +20k Gaussians per image, T_I = 200, reference build_plan / "
                              "lr_blended replayed, expansion + 2 render-only PSNRs included, wall clock"}
            except Exception as ex:  # pragma: no cover
                progressive[name] = {"error": f"{type(ex).__name__}: {ex}"}
    line = {
        "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (BASELINE config generator, seeded; targets = "
                                                      "renders of a second seed's field)",
        "config": {"workload": _workload(cfg), "n_gaussians": n, "width": cams[0].width, "height": cams[0].height,
                   "views": len(cams), "parallelism": f"view-sharded dp{world} ({exchange_note or args.exchange})"
                   if world > 1
                   else "single GPU",
                   "l2": "inputs larger than L2 (field + Adam moments 708 MB, per-step working set > 1 GB)",
                   "walked_pairs_per_view": P_mean},
        "roofline": roofline,
        "roofline_hbm": roofline_hbm,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_val, "unit": "iters/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 40,
                "target": f"{args.e2e_target} image uploaded every step (copy stream, overlapped); loss terms "
                          "written by the loss kernel into pinned host memory"},
        "gpu_launches": launches,
        **extras,
        "semi_global_batch": batch_block,
        "small_configs": small,
        "progressive": progressive,
        "clocks": clk.summary(),
        "stage_ms": {k: round(v, 4) for k, v in stage_ms.items() if not k.endswith("workspace")},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
