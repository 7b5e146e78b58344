"""CPU-only tests: the C ABI library loads and exports every symbol include/ssr.h
declares, host-side logic (camera, scenes, FieldGrads packing, view sharding,
loss-weight validation), loud failure without a GPU, and the N>1 gradient
all-reduce path over gloo with world_size 2."""

import ctypes
import os
import re
import socket

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "ssr.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ssr_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    import ctypes

    from paper_2503_13086_b200 import _lib

    names = _header_functions()
    assert len(names) >= 15
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), f"libssr.so does not export {n}"
    # every header function is typed in the ctypes binding
    assert set(names) <= set(_lib.EXPORTS), set(names) - set(_lib.EXPORTS)


def test_library_query_functions_without_gpu():
    from paper_2503_13086_b200 import _lib

    lib = _lib.load()
    assert lib.ssr_version() == 1
    assert _lib.query("ssr_bin_workspace", 1000, 64) > 0
    assert _lib.query("ssr_scan_workspace", 1000) > 0
    assert _lib.query("ssr_loss_workspace", 64, 48) >= 9 * 64 * 48 * 4
    assert lib.ssr_ckpt_floats(3200, 10) == (100 + 10 + 1) * 256 * 4


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    from paper_2503_13086_b200 import _lib
    from paper_2503_13086_b200.errors import ExtensionMissing

    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(ExtensionMissing):
        _lib.load(str(tmp_path / "missing_libssr.so"))


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_gpu_means_no_fallback():
    from paper_2503_13086_b200 import GaussianField
    from paper_2503_13086_b200.errors import ExtensionMissing

    with pytest.raises(ExtensionMissing):
        GaussianField(sh_degree=0)


def test_camera_validation_and_look_at():
    from paper_2503_13086_b200.camera import CameraFrame, look_at
    from paper_2503_13086_b200.errors import InvalidParameter

    rot, tr = look_at([0.0, 0.0, -4.0], [0.0, 0.0, 0.0])
    cam = CameraFrame(1, 64, 48, 50.0, 50.0, 32.0, 24.0, rot, tr)
    np.testing.assert_allclose(cam.center, [0.0, 0.0, -4.0], atol=1e-12)
    with pytest.raises(InvalidParameter):
        CameraFrame(1, 64, 48, -1.0, 50.0, 32.0, 24.0, rot, tr)
    r3, t3 = look_at([0.3, -0.2, 0.1], [0.0, 0.0, 6.0])
    with pytest.raises(InvalidParameter):  # an fp32-rounded pose is not orthonormal to 1e-9
        CameraFrame(1, 64, 48, 50.0, 50.0, 32.0, 24.0, r3.astype(np.float32).astype(np.float64), t3)
    # straight-down view falls back to another up vector (camera.py:97-100)
    r2, _ = look_at([0.0, 5.0, 0.0], [0.0, 0.0, 0.0])
    np.testing.assert_allclose(r2 @ r2.T, np.eye(3), atol=1e-12)


def test_scene_generators_are_seeded_and_float32():
    from paper_2503_13086_b200 import scenes

    a = scenes.make_params(1, seed=3, n=500)
    b = scenes.make_params(1, seed=3, n=500)
    c = scenes.make_params(1, seed=4, n=500)
    for k in ("positions", "rotations", "log_scales", "opacity_logits", "sh"):
        assert getattr(a, k).dtype == np.float32
        np.testing.assert_array_equal(getattr(a, k), getattr(b, k))
    assert not np.array_equal(a.positions, c.positions)
    assert a.sh.shape == (500, 3, 16)
    p2 = scenes.make_params(2, seed=0, n=1000)
    r = np.linalg.norm(p2.positions, axis=1)
    assert np.mean(np.abs(r - 3.0) < 0.3) > 0.85  # shell + 10% background
    cam = scenes.camera(2, view=3)
    assert (cam.width, cam.height) == (1920, 1080)
    assert np.linalg.norm(cam.center) == pytest.approx(6.0)


def test_fieldgrads_packing_layout():
    from paper_2503_13086_b200.rasterize import FieldGrads

    n, k = 5, 4
    rng = np.random.default_rng(0)
    arrs = dict(positions=rng.standard_normal((n, 3)), rotations=rng.standard_normal((n, 4)),
                log_scales=rng.standard_normal((n, 3)), opacity_logits=rng.standard_normal(n),
                sh=rng.standard_normal((n, 3, k)))
    from paper_2503_13086_b200.field import class_slices, row_stride

    g = FieldGrads(**arrs, screen_norms=np.zeros(n), visible=np.zeros(n, bool))
    flat = g.flat_params(torch.device("cpu"))
    ns = row_stride(n)
    assert ns == 8 and flat.numel() == ns * (11 + 3 * k)  # class regions padded to a multiple of 4 rows
    sl = class_slices(n, k)
    assert [o for o, _ in sl] == [0, 3 * ns, 7 * ns, 10 * ns, 11 * ns]
    np.testing.assert_allclose(flat[: 3 * n].numpy(), arrs["positions"].ravel(), rtol=1e-6)
    np.testing.assert_allclose(flat[11 * ns: 11 * ns + 3 * k * n].numpy(), arrs["sh"].ravel(), rtol=1e-6)
    z = FieldGrads.zeros(n, 1, torch.device("cpu"))
    assert z.positions.shape == (n, 3) and z.sh.shape == (n, 3, 4)
    assert z.flat.numel() == ns * (11 + 12 + 2)
    z.visible_count[2] = 3.0
    assert bool(z.visible[2]) and not bool(z.visible[1])


def test_loss_weights_validation():
    from paper_2503_13086_b200.errors import InvalidParameter
    from paper_2503_13086_b200.losses import LossWeights

    LossWeights(1.0, 0.2, 0.0)
    with pytest.raises(InvalidParameter):
        LossWeights(-1.0, 0.2, 0.0)
    with pytest.raises(InvalidParameter):
        LossWeights(float("nan"), 0.2, 0.0)


def test_shard_views_balanced_and_complete():
    from paper_2503_13086_b200.train import shard_views

    for n_views in (1, 7, 64):
        for world in (1, 2, 4, 8):
            shards = [shard_views(list(range(n_views)), r, world) for r in range(world)]
            flat = [v for s in shards for v in s]
            assert flat == list(range(n_views))
            sizes = [len(s) for s in shards]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _allreduce_worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2503_13086_b200.rasterize import FieldGrads
    from paper_2503_13086_b200.train import allreduce_grads, shard_views

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, deg = 6, 1
    views = list(range(5))
    g = FieldGrads.zeros(n, deg, torch.device("cpu"))
    # each "view" contributes a deterministic gradient; ranks own disjoint views
    for v in shard_views(views, rank, world):
        g.flat.add_(torch.arange(g.flat.numel(), dtype=torch.float32) * (v + 1))
    allreduce_grads(g.flat)
    q.put((rank, g.flat.numpy().copy()))
    dist.destroy_process_group()


def test_view_sharded_allreduce_gloo_world2():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_allreduce_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    n_el = res[0].size
    want = np.arange(n_el, dtype=np.float32) * sum(v + 1 for v in range(5))
    np.testing.assert_allclose(res[0], want, rtol=1e-6)
    np.testing.assert_array_equal(res[0], res[1])


def test_check_camera_accepts_duck_typed_frames():
    """render/project_field read only the pose, intrinsics and size, so the
    reference's own CameraFrame (or any object with those attributes) is accepted."""
    from types import SimpleNamespace

    from paper_2503_13086_b200.camera import CameraFrame, look_at
    from paper_2503_13086_b200.errors import InvalidParameter
    from paper_2503_13086_b200.rasterize.projection import check_camera

    rot, tr = look_at(np.array([0.0, 0.0, -4.0]), np.zeros(3))
    ours = CameraFrame(1, 32, 24, 30.0, 30.0, 16.0, 12.0, rot, tr)
    check_camera(ours)
    duck = SimpleNamespace(rotation=rot, translation=tr, center=-(rot.T @ tr), fx=30.0, fy=30.0, cx=16.0, cy=12.0,
                           width=32, height=24, pixels=None)
    check_camera(duck)
    with pytest.raises(InvalidParameter, match="lacks"):
        check_camera(SimpleNamespace(rotation=rot, translation=tr))
    with pytest.raises(InvalidParameter):
        check_camera(SimpleNamespace(**{**duck.__dict__, "width": 0}))


def test_look_at_is_orthonormal_and_handles_poles():
    from paper_2503_13086_b200.camera import CameraFrame, look_at

    for eye in ([0.0, 0.0, -4.0], [3.0, -2.0, 1.0], [0.0, 5.0, 0.0], [0.0, -5.0, 0.0]):
        rot, tr = look_at(np.array(eye), np.zeros(3))
        assert np.abs(rot @ rot.T - np.eye(3)).max() < 1e-12
        # +z looks at the target: the origin maps onto the optical axis
        pc = rot @ np.zeros(3) + tr
        assert pc[2] > 0 and abs(pc[0]) < 1e-12 and abs(pc[1]) < 1e-12
        cam = CameraFrame(0, 8, 8, 4.0, 4.0, 4.0, 4.0, rot, tr)
        np.testing.assert_allclose(cam.center, eye, atol=1e-12)


# ---------------------------------------------------------------- sharded batch step over gloo
class _FlatField:
    def __init__(self, flat, n, deg):
        self.flat, self._n, self.sh_degree, self.version = flat, n, deg, 0

    def __len__(self):
        return self._n


def _cpu_adam(field, opt, rate, steps):
    """optim.py AdamBuffer.apply restated over the flat class-major layout:
    returns adam_range(lo, hi, g, goff) updating field.flat / opt.m / opt.v."""
    from paper_2503_13086_b200.field import class_slices
    from paper_2503_13086_b200.optim import (BETA1, BETA2, EPS, OPACITY_LR, ROTATION_LR, SCALE_LR, SH_DC_LR,
                                             SH_REST_LR)

    n, k = len(field), (field.sh_degree + 1) ** 2
    lrs = (rate * opt.scene_extent, ROTATION_LR, SCALE_LR, OPACITY_LR, SH_DC_LR)
    lr = torch.zeros_like(field.flat)
    real = torch.zeros_like(field.flat, dtype=torch.bool)
    for c, ((off, w), base) in enumerate(zip(class_slices(n, k), lrs)):
        lr[off: off + w * n] = base
        real[off: off + w * n] = True
        if c == 4:
            j = torch.arange(w * n)
            lr[off: off + w * n] = torch.where(j % k == 0, torch.tensor(SH_DC_LR), torch.tensor(SH_REST_LR))
    bc1, bc2 = 1.0 - BETA1 ** steps, 1.0 - BETA2 ** steps

    def adam_range(lo, hi, g, goff):
        sl = slice(lo, hi)
        gg = g[lo - goff: hi - goff]
        msk = real[sl]
        m = BETA1 * opt.m[sl] + (1.0 - BETA1) * gg
        v = BETA2 * opt.v[sl] + (1.0 - BETA2) * gg * gg
        p = field.flat[sl] - lr[sl] * (m / bc1) / (torch.sqrt(v / bc2) + EPS)
        field.flat[sl] = torch.where(msk, p, field.flat[sl])
        opt.m[sl] = torch.where(msk, m, opt.m[sl])
        opt.v[sl] = torch.where(msk, v, opt.v[sl])

    return adam_range


def _sharded_worker(rank, world, port, q):
    import types

    import torch.distributed as dist

    from paper_2503_13086_b200.field import flat_size
    from paper_2503_13086_b200.rasterize import FieldGrads
    from paper_2503_13086_b200.train import exchange_and_step, gather_moments, shard_layout

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, deg = 37, 1
    gen = torch.Generator().manual_seed(0)
    base = torch.randn(flat_size(n, 4), generator=gen)
    out = {}
    for mode in ("allreduce", "sharded"):
        fld = _FlatField(base.clone(), n, deg)
        opt = types.SimpleNamespace(m=torch.zeros_like(base), v=torch.zeros_like(base), scene_extent=2.0)
        g = FieldGrads.zeros(n, deg, torch.device("cpu"))
        g.flat.copy_(torch.randn(g.flat.shape, generator=torch.Generator().manual_seed(10 + rank)))
        exchange_and_step(fld, g, opt, 1e-3, mode=mode, adam_range=_cpu_adam(fld, opt, 1e-3, 1))
        if mode == "sharded":
            gather_moments(fld, opt)
        out[mode] = (fld.flat.clone(), opt.m.clone(), opt.v.clone(), g.flat[fld.flat.numel():].clone())
    q.put((rank, {k: [t.numpy() for t in v] for k, v in out.items()}, shard_layout(base.numel(), world)))
    dist.destroy_process_group()


def test_sharded_batch_step_matches_allreduce_gloo_world2():
    """reduce-scatter -> Adam on the owned chunk -> all-gather gives the same
    parameters and (after gather_moments) moments as all-reduce -> full Adam,
    and both equal one step on the summed gradients (host logic over gloo)."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r, d, layout = q.get(timeout=180)
        res[r] = d
    for p in procs:
        p.join(timeout=60)
    chunk, main = layout
    assert chunk % 4 == 0 and 0 < main <= res[0]["sharded"][0].size
    for r in (0, 1):
        for a, b in zip(res[r]["allreduce"], res[r]["sharded"]):
            np.testing.assert_allclose(b, a, rtol=1e-6, atol=1e-7)
    for i in range(4):
        np.testing.assert_array_equal(res[0]["sharded"][i], res[1]["sharded"][i])


def _moments_worker(rank, world, port, q):
    import types

    import torch.distributed as dist

    from paper_2503_13086_b200 import _lib
    from paper_2503_13086_b200.train import gather_moments

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    total = 4 * 37 + 3  # a tail past world * chunk
    truth = torch.arange(total, dtype=torch.float32)
    lo, hi = ctypes.c_int64(0), ctypes.c_int64(0)
    _lib.call("ssr_exchange_chunk", total, world, rank, ctypes.byref(lo), ctypes.byref(hi))
    # each rank's moments are current only in its ssr_exchange_chunk range
    m = torch.full((total,), -1.0)
    m[lo.value:hi.value] = truth[lo.value:hi.value]
    opt = types.SimpleNamespace(m=m, v=m.clone() * 2)
    fld = types.SimpleNamespace(flat=torch.zeros(total))
    gather_moments(fld, opt, mode="p2p")
    q.put((rank, (lo.value, hi.value), opt.m.numpy().copy(), opt.v.numpy().copy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_p2p_gather_moments_gloo(world):
    """After p2p exchange steps (ssr_exchange_adam: the last rank also owns the
    tail past world * chunk), gather_moments leaves every rank complete moments;
    the ranks' chunks (the C ABI's ssr_exchange_chunk) tile the buffer."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_moments_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r, b, m, v = q.get(timeout=180)
        res[r] = (b, m, v)
    for p in procs:
        p.join(timeout=60)
    total = 4 * 37 + 3
    bounds = [res[r][0] for r in range(world)]
    assert bounds[0][0] == 0 and bounds[-1][1] == total
    assert all(a[1] == b[0] and a[0] % 4 == 0 for a, b in zip(bounds, bounds[1:]))
    truth = np.arange(total, dtype=np.float32)
    for r in range(world):
        np.testing.assert_array_equal(res[r][1], truth)
        np.testing.assert_array_equal(res[r][2], 2 * truth)
