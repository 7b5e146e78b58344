"""Parity metrics between the CUDA path and an oracle / golden record.

Bars (BASELINE.json north_star): sort indices + tile ranges bit-exact; image
max-abs <= 1e-4; t_final / soft_count <= 1e-4; n_walk / terminated /
hard_count exact; per-parameter-class gradient rel-L2 <= 1e-3.
"""

from __future__ import annotations

import numpy as np

GRAD_CLASSES = ("positions", "rotations", "log_scales", "opacity_logits", "sh")
IMAGE_TOL = 1e-4
GRAD_RTOL = 1e-3


def np_(x):
    try:
        import torch

        if torch.is_tensor(x):
            return x.detach().cpu().numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(x)


def rel_l2(a, b) -> float:
    a = np_(a).astype(np.float64).ravel()
    b = np_(b).astype(np.float64).ravel()
    den = np.linalg.norm(b)
    num = np.linalg.norm(a - b)
    if den == 0.0:
        return 0.0 if num == 0.0 else float("inf")
    return float(num / den)


def max_abs(a, b) -> float:
    a = np_(a).astype(np.float64)
    b = np_(b).astype(np.float64)
    return float(np.abs(a - b).max()) if a.size else 0.0


def projection_report(sp, ref: dict) -> dict:
    """sp = GPU ProjectedSplats, ref = oracle/golden dict with reference keys."""
    r = {}
    for k in ("gauss_index", "inst_splat", "tile_starts", "tile_ends"):
        a, b = np_(getattr(sp, k)).astype(np.int64), np.asarray(ref[k]).astype(np.int64)
        r[f"{k}_equal"] = bool(a.shape == b.shape and np.array_equal(a, b))
        if not r[f"{k}_equal"]:
            r[f"{k}_shape"] = (a.shape, b.shape)
            if a.shape == b.shape:
                r[f"{k}_mismatches"] = int((a != b).sum())
    return r


def forward_report(out, ref: dict) -> dict:
    r = {"image_max_abs": max_abs(out.image, ref["image"]),
         "t_final_max_abs": max_abs(out.t_final, ref["t_final"]),
         "soft_max_abs": max_abs(out.soft_count, ref["soft_count"])}
    for k in ("n_walk", "terminated", "hard_count"):
        a, b = np_(getattr(out, k)).astype(np.int64), np.asarray(ref[k]).astype(np.int64)
        r[f"{k}_mismatch"] = int((a != b).sum())
    fl = np_(out.flagged)
    r["flagged_pixels"] = int(fl.sum())
    r["flagged_frac"] = float(fl.mean()) if fl.size else 0.0
    return r


def forward_ok(r: dict) -> bool:
    return (r["image_max_abs"] <= IMAGE_TOL and r["t_final_max_abs"] <= IMAGE_TOL and r["soft_max_abs"] <= IMAGE_TOL
            and r["n_walk_mismatch"] == 0 and r["terminated_mismatch"] == 0 and r["hard_count_mismatch"] == 0)


def grads_report(g, ref: dict) -> dict:
    r = {f"{k}_rel_l2": rel_l2(getattr(g, k), ref[k]) for k in GRAD_CLASSES}
    r["screen_norms_rel_l2"] = rel_l2(g.screen_norms, ref["screen_norms"])
    r["visible_equal"] = bool(np.array_equal(np_(g.visible).astype(bool), np.asarray(ref["visible"]).astype(bool)))
    return r


def grads_ok(r: dict, rtol=GRAD_RTOL) -> bool:
    """Every parameter class AND the densify statistics: screen_norms (rel-L2,
    backward.py:128) and the visible mask (exact) feed every densify decision."""
    return (all(r[f"{k}_rel_l2"] <= rtol for k in GRAD_CLASSES) and r["screen_norms_rel_l2"] <= rtol
            and r["visible_equal"])
