"""Seeded synthetic workloads for BASELINE.json configs 0-4.

The paper's datasets are not available offline, so every measurement and parity
case uses these generators (shapes and value distributions from BASELINE.json
``configs``).  Gaussian parameters are drawn in float64 and rounded to float32
(the GPU's storage); the CPU oracle receives those exact values upcast to
float64.  Cameras stay float64.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .camera import CameraFrame, look_at


@dataclass
class HostParams:
    """float32 SoA parameters in the reference layout (field.py:199-203)."""

    positions: np.ndarray  # (N, 3)
    rotations: np.ndarray  # (N, 4) unnormalized wxyz
    log_scales: np.ndarray  # (N, 3)
    opacity_logits: np.ndarray  # (N,)
    sh: np.ndarray  # (N, 3, K) channel-major

    def __len__(self):
        return self.positions.shape[0]

    @property
    def sh_degree(self) -> int:
        return int(round(np.sqrt(self.sh.shape[2]))) - 1

    def as_float64(self) -> "HostParams":
        return HostParams(*(a.astype(np.float64) for a in (
            self.positions, self.rotations, self.log_scales, self.opacity_logits, self.sh)))


CONFIGS = {
    0: dict(n=10_000, sh_degree=0, width=128, height=128),
    1: dict(n=200_000, sh_degree=3, width=800, height=800),
    2: dict(n=1_000_000, sh_degree=3, width=1920, height=1080),
    3: dict(n=2_000_000, sh_degree=3, width=1297, height=840),
    4: dict(n=3_000_000, sh_degree=3, width=1920, height=1080),
}


def _unit_quats(rng, n):
    q = rng.standard_normal((n, 4))
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def _sh(rng, n, degree, dc_std=0.3, rest_std=0.05):
    k = (degree + 1) ** 2
    sh = np.zeros((n, 3, k))
    sh[:, :, 0] = rng.normal(0.0, dc_std, (n, 3))
    if k > 1:
        sh[:, :, 1:] = rng.normal(0.0, rest_std, (n, 3, k - 1))
    return sh


def _means(cfg: int, rng, n):
    if cfg == 0:
        return rng.uniform(-1.0, 1.0, (n, 3))
    if cfg == 1:
        centers = rng.uniform(-1.5, 1.5, (20, 3))
        axes = np.stack([np.linalg.qr(rng.standard_normal((3, 3)))[0] for _ in range(20)])
        sig = rng.uniform(0.05, 0.45, (20, 3))
        lab = rng.integers(0, 20, n)
        local = rng.standard_normal((n, 3)) * sig[lab]
        pts = centers[lab] + np.einsum("nij,nj->ni", axes[lab], local)
        return np.clip(pts, -2.0, 2.0)
    # configs 2-4: noisy shell r=3 (sigma 0.05) plus 10% uniform background in [-10,10]^3
    n_bg = n // 10
    n_sh = n - n_bg
    d = rng.standard_normal((n_sh, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    shell = d * 3.0 + rng.normal(0.0, 0.05, (n_sh, 3))
    bg = rng.uniform(-10.0, 10.0, (n_bg, 3))
    pts = np.concatenate([shell, bg])
    return pts[rng.permutation(n)]


def make_params(cfg: int, seed: int = 0, n: int | None = None) -> HostParams:
    c = CONFIGS[cfg]
    n = c["n"] if n is None else int(n)
    rng = np.random.default_rng([cfg, seed])
    pos = _means(cfg, rng, n)
    ls_mu, ls_sd = (-4.5, 0.5) if cfg >= 2 else (-3.5, 0.3)
    log_scales = rng.normal(ls_mu, ls_sd, (n, 3))
    rot = _unit_quats(rng, n)
    logits = rng.normal(0.0, 1.0, n)
    sh = _sh(rng, n, c["sh_degree"])
    f32 = lambda a: np.ascontiguousarray(a, dtype=np.float32)
    return HostParams(f32(pos), f32(rot), f32(log_scales), f32(logits), f32(sh))


def camera(cfg: int, view: int = 0, width: int | None = None, height: int | None = None,
           image_id: int | None = None) -> CameraFrame:
    c = CONFIGS[cfg]
    w = c["width"] if width is None else int(width)
    h = c["height"] if height is None else int(height)
    f = w / (2.0 * np.tan(np.deg2rad(30.0)))  # fov 60 degrees
    if cfg == 0:
        ang = 2.0 * np.pi * view / 16.0
        eye = np.array([4.0 * np.sin(ang), 0.0, -4.0 * np.cos(ang)])
    elif cfg == 1:
        rng = np.random.default_rng([101, view])
        d = rng.standard_normal(3)
        eye = 5.0 * d / np.linalg.norm(d)
    elif cfg == 3:
        # spiral path, 0.11 turn per image: consecutive views share 60% of their
        # feature tracks (front-facing shell points, tools/record_plan_trace.py),
        # BASELINE config 3's "60% view overlap"
        ang = 2.0 * np.pi * view * 0.11
        eye = np.array([6.0 * np.cos(ang), -1.5 + 3.0 * view / 100.0, 6.0 * np.sin(ang)])
    else:
        ang = 2.0 * np.pi * view / 64.0
        eye = np.array([6.0 * np.cos(ang), 0.0, 6.0 * np.sin(ang)])
    rot, tr = look_at(eye, np.zeros(3))
    return CameraFrame(view if image_id is None else image_id, w, h, f, f, w / 2.0, h / 2.0, rot, tr)
