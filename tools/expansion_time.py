"""Time the pieces of one progressive-loop field expansion at config 3
(2 M Gaussians + 20 k new points): python tools/expansion_time.py"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_13086_b200 import GaussianField, scenes  # noqa: E402
from paper_2503_13086_b200.optim import FieldOptimizer  # noqa: E402
from paper_2503_13086_b200.spatial import mean_knn_scale  # noqa: E402


def timed(label, fn, reps=3):
    out = None
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(f"{label:40s} {min(ts):8.2f} ms (min of {reps})", flush=True)
    return out


field = GaussianField.from_host(scenes.make_params(3, seed=0, n=2_000_000))
opt = FieldOptimizer(field, scene_extent=6.0)
rng = np.random.default_rng(0)
pos = rng.normal(0.0, 2.0, (20_000, 3))
cols = rng.uniform(0.0, 1.0, (20_000, 3))
newp = torch.as_tensor(pos, device="cuda")
timed("positions.double()", lambda: field.positions.double())
timed("mean_knn_scale (2M pool, 20k queries)", lambda: mean_knn_scale(field.positions.double(), newp))
timed("field._check_finite()", lambda: field._check_finite())
n0 = len(field)


def insert():
    field.insert_arrays(pos, cols)


timed("insert_arrays (total)", insert, reps=1)
keep = np.ones(n0, dtype=bool)
timed("optimizer.sync (grow moments)", lambda: opt.sync(field, keep, len(field) - n0), reps=1)


# steady state: three more events (expansion + moment growth each)
for ev in range(3):
    n0 = len(field)

    def one_event():
        field.insert_arrays(pos + 0.01 * (ev + 1), cols)
        opt.sync(field, np.ones(n0, dtype=bool), len(field) - n0)

    timed(f"event {ev}: insert_arrays + optimizer.sync", one_event, reps=1)
