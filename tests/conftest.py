import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: full-size parity cases (config 1/2)")


def golden_names():
    """Rasterizer cases (the expansion and PLY fixtures are tested separately)."""
    names = (os.path.splitext(os.path.basename(p))[0] for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz")))
    other = ("expansion", "pipeline_small", "c3_plan_trace")  # tested by their own modules
    return sorted(n for n in names if n not in other and not n.startswith("ply_"))


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN_DIR, f"{name}.npz")))


def golden_camera(g):
    from paper_2503_13086_b200.camera import CameraFrame

    fx, fy, cx, cy = g["cam_intr"]
    w, h = (int(v) for v in g["cam_wh"])
    return CameraFrame(1, w, h, fx, fy, cx, cy, g["cam_R"], g["cam_t"])


def golden_params(g, prefix="in_"):
    from oracle.oracle import Params

    return Params(*(np.ascontiguousarray(g[prefix + k], np.float64) for k in (
        "positions", "rotations", "log_scales", "opacity_logits", "sh")))


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle import oracle

    oracle.build()
    return oracle
