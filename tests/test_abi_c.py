"""The C ABI from C: tests/abi/ssr_render.c is built with gcc against
include/ssr.h and libssr.so (no Python, no torch) and drives the path the way
INTEGRATION.md section 2 tells a non-Python host to.

* CPU: the host-only entry points (sizes, chunking, error reporting).
* GPU: a whole render through caller-owned device buffers, bit-identical to
  the package's render() of the same field and camera; a backward + chain
  from C, bit-identical to backward(); and K whole training iterations from C
  (render, loss, backward, chain + Adam), bit-identical to train_iteration()."""

import ctypes
import os
import shutil
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2503_13086_b200")


def _build(tmp_path):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    if not os.path.exists(os.path.join(LIBDIR, "libssr.so")):
        pytest.skip("libssr.so not built")
    exe = str(tmp_path / "ssr_render")
    cmd = ["gcc", "-O2", "-std=c11", f"-I{ROOT}/include", "-I/usr/local/cuda/include",
           os.path.join(ROOT, "tests", "abi", "ssr_render.c"), "-o", exe, f"-L{LIBDIR}", "-lssr",
           "-L/usr/local/cuda/lib64", "-lcudart", "-lm", f"-Wl,-rpath,{LIBDIR}", "-Wl,-rpath,/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_host_query_entry_points(tmp_path):
    exe = _build(tmp_path)
    out = subprocess.run([exe, "--query"], check=True, capture_output=True, text=True).stdout
    vals = dict(line.split(" ", 1) for line in out.strip().splitlines())
    from paper_2503_13086_b200 import _lib

    lib = _lib.load()
    assert int(vals["version"]) == lib.ssr_version()
    assert int(vals["ckpt_floats"]) == lib.ssr_ckpt_floats(100000, 8160)
    assert int(vals["rows_floats"]) == lib.ssr_rows_floats(1000) == 4 + 10 * 1000 + 4
    assert vals["exchange_chunk"] == "744 1003"  # 1003 // 16 * 4 = 248 per rank; the last owns the tail
    rc, msg = vals["invalid"].split(" ", 1)
    assert int(rc) == 1 and "invalid argument" in msg


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,n,w,h", [(0, 3000, 96, 80), (1, 20000, 320, 240)])
def test_c_host_render_matches_python(tmp_path, cfg, n, w, h):
    import torch

    from paper_2503_13086_b200 import GaussianField, _lib, scenes
    from paper_2503_13086_b200.rasterize import render

    exe = _build(tmp_path)
    hp = scenes.make_params(cfg, seed=21, n=n)
    cam = scenes.camera(cfg, view=4, width=w, height=h)
    bg = np.array([0.1, 0.2, 0.3])
    f = GaussianField.from_host(hp)
    ref = render(f, cam, bg=bg, for_backward=False)
    torch.cuda.synchronize()
    src = tmp_path / "in.bin"
    with open(src, "wb") as fh:
        fh.write(np.int64(n).tobytes() + np.int32(f.sh_degree).tobytes() + bg.astype(np.float64).tobytes())
        fh.write(bytes(_lib.camera_struct(cam)))
        for k in ("positions", "rotations", "log_scales", "opacity_logits", "sh"):
            fh.write(np.ascontiguousarray(getattr(hp, k), dtype=np.float32).tobytes())
    dst = tmp_path / "out.bin"
    run = subprocess.run([exe, str(src), str(dst)], capture_output=True, text=True, timeout=120)
    assert run.returncode == 0, run.stderr
    raw = np.fromfile(dst, dtype=np.uint8)
    img = raw[: 12 * h * w].view(np.float32).reshape(h, w, 3)
    nw = raw[12 * h * w:].view(np.int32).reshape(h, w)
    assert np.array_equal(img, ref.image.cpu().numpy())
    assert np.array_equal(nw, ref.n_walk.cpu().numpy())
    assert ctypes.sizeof(_lib.SsrCamera) == 9 * 8 + 3 * 8 + 4 * 8 + 3 * 8 + 2 * 4


@pytest.mark.gpu
def test_c_host_backward_matches_python(tmp_path):
    import torch

    from paper_2503_13086_b200 import GaussianField, _lib, scenes
    from paper_2503_13086_b200.field import flat_size
    from paper_2503_13086_b200.rasterize import backward, render

    exe = _build(tmp_path)
    n, w, h = 20000, 320, 240
    hp = scenes.make_params(1, seed=22, n=n)
    cam = scenes.camera(1, view=6, width=w, height=h)
    bg = np.zeros(3)
    f = GaussianField.from_host(hp)
    out = render(f, cam, bg=bg, soft_count=False)
    g = backward(f, out, torch.full_like(out.image, 1e-3))
    torch.cuda.synchronize()
    src = tmp_path / "in.bin"
    with open(src, "wb") as fh:
        fh.write(np.int64(n).tobytes() + np.int32(f.sh_degree).tobytes() + bg.astype(np.float64).tobytes())
        fh.write(bytes(_lib.camera_struct(cam)))
        for k in ("positions", "rotations", "log_scales", "opacity_logits", "sh"):
            fh.write(np.ascontiguousarray(getattr(hp, k), dtype=np.float32).tobytes())
    dst = tmp_path / "out.bin"
    run = subprocess.run([exe, str(src), str(dst), "--grad"], capture_output=True, text=True, timeout=120)
    assert run.returncode == 0, run.stderr
    raw = np.fromfile(dst, dtype=np.uint8)
    img = raw[: 12 * h * w].view(np.float32).reshape(h, w, 3)
    flat = raw[16 * h * w:].view(np.float32)
    assert flat.size == flat_size(n, f.n_sh_coeffs, extra=2)
    assert np.array_equal(img, out.image.cpu().numpy())
    got = {k: getattr(type(g)(_flat=torch.from_numpy(flat.copy()), _n=n, _k=f.n_sh_coeffs), k).numpy()
           for k in ("positions", "rotations", "log_scales", "opacity_logits", "sh", "screen_norms")}
    for k, v in got.items():
        assert np.array_equal(v, getattr(g, k).cpu().numpy()), k


@pytest.mark.gpu
def test_c_host_training_matches_python(tmp_path):
    import torch

    from paper_2503_13086_b200 import GaussianField, _lib, scenes
    from paper_2503_13086_b200.losses import LossWeights
    from paper_2503_13086_b200.optim import (BETA1, BETA2, OPACITY_LR, ROTATION_LR, SCALE_LR, SH_DC_LR,
                                             SH_REST_LR, FieldOptimizer)
    from paper_2503_13086_b200.rasterize import render
    from paper_2503_13086_b200.train import TrainState, train_iteration

    exe = _build(tmp_path)
    n, w, h, iters, rate, extent = 20000, 320, 240, 4, 1.6e-4, 3.0
    hp = scenes.make_params(1, seed=23, n=n)
    cam = scenes.camera(1, view=5, width=w, height=h)
    tf = GaussianField.from_host(scenes.make_params(1, seed=24, n=n))
    tgt = (render(tf, cam, for_backward=False).image * 255.0).round().clamp(0, 255).to(torch.uint8)
    f = GaussianField.from_host(hp)
    st = TrainState(field=f, optimizer=FieldOptimizer(f, scene_extent=extent),
                    weights=LossWeights(l1=1.0, ssim=0.2, load=0.0), scene_extent=extent)
    st.densify_enabled = False
    for _ in range(iters):
        br = train_iteration(st, cam, tgt, rate)
    torch.cuda.synchronize()
    src = tmp_path / "in.bin"
    with open(src, "wb") as fh:
        fh.write(np.int64(n).tobytes() + np.int32(f.sh_degree).tobytes())
        fh.write(np.zeros(3).tobytes())
        fh.write(bytes(_lib.camera_struct(cam)))
        for k in ("positions", "rotations", "log_scales", "opacity_logits", "sh"):
            fh.write(np.ascontiguousarray(getattr(hp, k), dtype=np.float32).tobytes())
        fh.write(np.array([rate * extent, ROTATION_LR, SCALE_LR, OPACITY_LR, SH_DC_LR, SH_REST_LR, BETA1, BETA2,
                           1.0, 0.2], dtype=np.float64).tobytes())
        fh.write(np.int32(iters).tobytes())
        fh.write(tgt.cpu().numpy().tobytes())
    dst = tmp_path / "out.bin"
    run = subprocess.run([exe, str(src), str(dst), "--train"], capture_output=True, text=True, timeout=300)
    assert run.returncode == 0, run.stderr
    raw = np.fromfile(dst, dtype=np.uint8)
    flat = raw[: 4 * f.flat.numel()].view(np.float32)
    loss = raw[4 * f.flat.numel():].view(np.float64)
    assert np.array_equal(flat, f.flat.cpu().numpy())
    assert np.array_equal(loss[:4], np.array([br.l1, br.ssim_loss, br.load, br.total]))
