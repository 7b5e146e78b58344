import sys, time, json, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tools')
import torch
from paper_2503_13086_b200 import pipeline
T = {}
def wrap(obj, name):
    f = getattr(obj, name)
    def g(*a, **k):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize(); T[name] = T.get(name, 0.0) + time.perf_counter() - t0
        return r
    setattr(obj, name, g)
for n in ("expand_field", "view_psnr", "register_frame"):
    wrap(pipeline.DeviceSession, n)
orig = pipeline.train_one_iteration
it_times = []
def toi(s, tid, fused=True):
    t0 = time.perf_counter(); r = orig(s, tid, fused=fused); it_times.append(time.perf_counter() - t0); return r
pipeline.train_one_iteration = toi
import progressive
import contextlib, io
ev = []
orig_p2 = pipeline.phase2_step
def p2(*a, **k):
    T.clear(); it_times.clear()
    r = orig_p2(*a, **k)
    ev.append({"seconds": round(r.seconds, 3), **{k2: round(v, 4) for k2, v in T.items()},
               "iters": len(it_times), "iter_sum": round(sum(it_times), 3), "iter_max_ms": round(1e3 * max(it_times), 2),
               "slow_iters": sum(1 for x in it_times if x > 0.01)})
    return r
pipeline.phase2_step = p2
progressive.phase2_step = p2
with contextlib.redirect_stdout(io.StringIO()):
    progressive.main(["--events", "5", "--warmup-events", "1"])
for e in ev: print(json.dumps(e))
