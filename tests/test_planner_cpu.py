"""Host-side planner logic of the pipeline port (no GPU).

* SchedulerPlanner driven by the reference's own scheduler / overlap modules
  reproduces, call for call, the plans and per-iteration rates that the
  reference's phase2_step produced in tests/golden/pipeline_small.npz
  (skipped where the reference is absent, e.g. on the GPU box).
* TracePlanner replays a recorded schedule and rejects a loop that drifts
  from it.
* The config-3 trace (tests/golden/c3_plan_trace.npz) is complete and
  well formed.
"""

import json
import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN_DIR

REF_SRC = "/root/reference/pkg/src"


def _ref_modules():
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference package not present (GPU box)")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    import splatstream.overlap as overlap
    import splatstream.scheduler as scheduler

    return scheduler, overlap


def test_scheduler_planner_reproduces_reference_phase2_schedule():
    from paper_2503_13086_b200.pipeline import SchedulerPlanner

    scheduler, overlap = _ref_modules()
    g = dict(np.load(os.path.join(GOLDEN_DIR, "pipeline_small.npz")))
    c = json.loads(str(g["cfg"]))
    rng = np.random.default_rng()
    pl = SchedulerPlanner(scheduler, overlap, t_i=c["t_i"], n_m=c["n_m"], rng=rng)
    init = [int(i) for i in g["init_ids"]]
    for i in init:  # phase1_initialize: register, then the batch's matches (pipeline.py:233-236)
        pl.register(i, int(g[f"frame{i}_features"]))
    for i, j, cnt in g["init_matches"]:
        pl.set_matches(int(i), int(j), int(cnt))
    for k in range(int(g["initial_iters"])):  # round-robin bootstrap (pipeline.py:248-250)
        pl.record(init[k % len(init)])
    for e in range(int(g["n_events"])):
        i = int(g[f"ev{e}_id"])
        pl.register(i, int(g[f"frame{i}_features"]), dict(g[f"ev{e}_match_row"].tolist()))
        rng.bit_generator.state = json.loads(str(g[f"ev{e}_rng_before_plan"]))
        entries = pl.plan(i)
        assert entries == g[f"ev{e}_entries"].tolist()
        assert rng.bit_generator.state == json.loads(str(g[f"ev{e}_rng_after_plan"]))
        rates = []
        for t in entries:
            rates.append(pl.rate(t))
            pl.record(t)
        assert rates == g[f"ev{e}_rates"].tolist()  # bit-identical host arithmetic


def test_trace_planner_replays_and_rejects_drift():
    from paper_2503_13086_b200.errors import InvalidParameter
    from paper_2503_13086_b200.pipeline import TracePlanner

    tp = TracePlanner({("event", 7): ([3, 7, 3], [1e-4, 2e-4, 3e-4])})
    assert tp.plan(7) == [3, 7, 3]
    got = []
    for t in (3, 7, 3):
        got.append(tp.rate(t))
        tp.record(t)
    assert got == [1e-4, 2e-4, 3e-4] and tp.global_iteration == 3
    tp.plan(7)
    with pytest.raises(InvalidParameter):
        tp.rate(7)  # the trace's first entry trains image 3
    with pytest.raises(InvalidParameter):
        tp.plan(8)


def test_config3_trace_is_complete():
    from paper_2503_13086_b200.pipeline import TracePlanner

    path = os.path.join(GOLDEN_DIR, "c3_plan_trace.npz")
    z = np.load(path)
    tp = TracePlanner.from_npz(path)
    first, last = int(z["first_event"]), int(z["last_event"])
    assert last == 99 and first <= 90
    for i in range(first, last + 1):
        entries, rates = tp.trace[("event", i)]
        assert len(entries) == len(rates) == int(z["t_i"])
        assert all(0 <= e <= i for e in entries)
        assert all(1.6e-6 <= r <= 1.6e-4 for r in rates)
        assert ("rng", i) in tp.trace
