"""Device time of ssr_exchange_adam with the W "peers" as buffers on one GPU
(the kernel sees only W pointers, so this times its whole data path, with
local HBM standing in for NVLink): every rank's call in turn = one full
exchange.  Reports the HBM bytes moved per exchange and the rate.

  python tools/exchange_bench.py [--n 3000000] [--deg 3] [--world 2 4 8] [--reps 10]
"""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=3_000_000)
    ap.add_argument("--deg", type=int, default=3)
    ap.add_argument("--world", type=int, nargs="+", default=[2, 4, 8])
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    import torch

    from paper_2503_13086_b200 import _lib
    from paper_2503_13086_b200.field import flat_size
    from paper_2503_13086_b200.optim import BETA1, BETA2, OPACITY_LR, ROTATION_LR, SCALE_LR, SH_DC_LR, SH_REST_LR

    k = (a.deg + 1) ** 2
    pf, gf = flat_size(a.n, k), flat_size(a.n, k, extra=2)
    d5 = ctypes.c_double * 5
    lr, bc1, bc2 = d5(1e-4, ROTATION_LR, SCALE_LR, OPACITY_LR, SH_DC_LR), d5(*[1 - BETA1] * 5), d5(*[1 - BETA2] * 5)
    st = _lib.stream_ptr()
    out = []
    for w in a.world:
        P = [torch.randn(pf, device="cuda") for _ in range(w)]
        G = [torch.randn(gf, device="cuda") * 1e-3 for _ in range(w)]
        M = [torch.zeros(pf, device="cuda") for _ in range(w)]
        V = [torch.zeros(pf, device="cuda") for _ in range(w)]
        arr = ctypes.c_void_p * w
        gp, pp = arr(*[g.data_ptr() for g in G]), arr(*[p.data_ptr() for p in P])

        def exchange():
            for r in range(w):
                _lib.call("ssr_exchange_adam", a.n, a.deg, w, r, gp, pp, M[r].data_ptr(), V[r].data_ptr(), lr,
                          SH_REST_LR, bc1, bc2, st)

        exchange()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            exchange()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        # per element of the parameter classes: W gradient reads, p / m / v read,
        # W parameter writes, m / v written; the statistics: W reads + W writes
        byts = 4 * (pf * (w + 3 + w + 2) + (gf - pf) * 2 * w)
        out.append({"world": w, "n": a.n, "ms_per_exchange": ms, "GB": byts / 1e9, "GBps": byts / ms / 1e6,
                    "per_rank_ms_if_concurrent": ms / w})
        del P, G, M, V
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
