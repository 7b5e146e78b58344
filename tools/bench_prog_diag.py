import sys, time, json
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
for n in ("expand_field", "view_psnr"):
    wrap(pipeline.DeviceSession, n)
orig = pipeline.train_one_iteration
it_times = []
def toi(s, tid, fused=True):
    t0 = time.perf_counter(); r = orig(s, tid, fused=fused); it_times.append(time.perf_counter() - t0); return r
pipeline.train_one_iteration = toi
orig_p2 = pipeline.phase2_step
def p2(*a, **k):
    T.clear(); it_times.clear()
    r = orig_p2(*a, **k)
    big = sorted(((round(1e3 * x, 1), i) for i, x in enumerate(it_times)), reverse=True)[:3]
    print(json.dumps({"seconds": round(r.seconds, 3), **{k2: round(v, 4) for k2, v in T.items()},
                      "iter_sum": round(sum(it_times), 3), "top_iters_ms": big}), file=sys.stderr, flush=True)
    return r
pipeline.phase2_step = p2
sys.argv = ["bench.py", "--steps", "20", "--warmup", "3", "--no-cpu-baseline"]
import bench
bench.main()
