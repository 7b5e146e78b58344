"""The fused sharded exchange (ssr_exchange_adam): every rank sums
its chunk's gradients over the ranks' buffers, runs Adam on it and stores the
new parameters into every replica; the densify statistics are summed into
every rank's gradient buffer.

Checked bit for bit against the sum of the ranks' gradients (rank order)
followed by the ordinary full Adam (ssr_adam):

* in one process, the "peers" being separate buffers on the one device (the
  kernel only sees W pointers, so this is its whole data path);
* with two processes sharing the GPU, the buffers mapped across processes by
  CUDA IPC through ``train.PeerExchange`` (the multi-GPU host path; the two
  kernels never wait on each other: host barriers order them).
"""

import ctypes
import os
import socket

import pytest

pytestmark = pytest.mark.gpu


def _problem(n, deg, world, seed=0):
    """Field parameters, per-rank gradient buffers (params + statistics), moments."""
    import torch

    from paper_2503_13086_b200.field import flat_size

    k = (deg + 1) ** 2
    g = torch.Generator().manual_seed(seed)
    p = torch.randn(flat_size(n, k), generator=g)
    grads = [torch.randn(flat_size(n, k, extra=2), generator=g) * 1e-2 for _ in range(world)]
    m = torch.randn(p.numel(), generator=g) * 1e-3
    v = torch.rand(p.numel(), generator=g) * 1e-5
    return p, grads, m, v


def _reference(n, deg, p, grads, m, v, steps=3, rate=1.6e-4):
    """Sum in rank order, then the full Adam (ssr_adam) on one replica."""
    import torch

    from paper_2503_13086_b200 import _lib
    from paper_2503_13086_b200.optim import SH_REST_LR

    dev = torch.device("cuda")
    acc = grads[0].to(dev).clone()
    for gq in grads[1:]:
        acc += gq.to(dev)
    P, M, V = p.to(dev).clone(), m.to(dev).clone(), v.to(dev).clone()
    lr, bc1, bc2 = _rates(steps, rate)
    _lib.call("ssr_adam", n, deg, P.data_ptr(), acc.data_ptr(), M.data_ptr(), V.data_ptr(), lr, SH_REST_LR, bc1, bc2,
              _lib.stream_ptr())
    torch.cuda.synchronize()
    return P.cpu(), M.cpu(), V.cpu(), acc[p.numel():].cpu()


def _rates(steps, rate):
    from paper_2503_13086_b200.optim import BETA1, BETA2, OPACITY_LR, ROTATION_LR, SCALE_LR, SH_DC_LR

    d5 = ctypes.c_double * 5
    lr = d5(rate * 2.5, ROTATION_LR, SCALE_LR, OPACITY_LR, SH_DC_LR)
    bc1 = d5(*[1.0 - BETA1 ** steps] * 5)
    bc2 = d5(*[1.0 - BETA2 ** steps] * 5)
    return lr, bc1, bc2


def _chunk(total, world, rank):
    from paper_2503_13086_b200 import _lib

    lo, hi = ctypes.c_int64(0), ctypes.c_int64(0)
    _lib.call("ssr_exchange_chunk", total, world, rank, ctypes.byref(lo), ctypes.byref(hi))
    return lo.value, hi.value


@pytest.mark.parametrize("world,n,deg", [(1, 1000, 3), (2, 4099, 3), (3, 1001, 1), (8, 777, 0), (8, 20000, 3)])
def test_exchange_adam_simulated_peers(world, n, deg):
    import torch

    from paper_2503_13086_b200 import _lib
    from paper_2503_13086_b200.field import row_stride
    from paper_2503_13086_b200.optim import SH_REST_LR

    p, grads, m, v = _problem(n, deg, world, seed=world * 7 + deg)
    P_ref, M_ref, V_ref, S_ref = _reference(n, deg, p, grads, m, v)
    dev = torch.device("cuda")
    P = [p.to(dev).clone() for _ in range(world)]
    G = [g.to(dev).clone() for g in grads]
    M = [m.to(dev).clone() for _ in range(world)]
    V = [v.to(dev).clone() for _ in range(world)]
    arr = ctypes.c_void_p * world
    gp, pp = arr(*[g.data_ptr() for g in G]), arr(*[x.data_ptr() for x in P])
    lr, bc1, bc2 = _rates(3, 1.6e-4)
    for r in range(world):  # in rank order; each call touches only its own chunk
        _lib.call("ssr_exchange_adam", n, deg, world, r, gp, pp, M[r].data_ptr(), V[r].data_ptr(), lr, SH_REST_LR,
                  bc1, bc2, _lib.stream_ptr())
    torch.cuda.synchronize()
    pf = p.numel()
    for q in range(world):
        assert torch.equal(P[q].cpu(), P_ref), q  # every replica: every chunk
        assert torch.equal(G[q][pf:].cpu(), S_ref), q  # summed statistics
    for r in range(world):
        lo, hi = _chunk(pf, world, r)
        assert torch.equal(M[r][lo:hi].cpu(), M_ref[lo:hi]) and torch.equal(V[r][lo:hi].cpu(), V_ref[lo:hi])
    # the chunks tile the buffer: 16-byte aligned, the last rank owns the tail
    bounds = [_chunk(pf, world, r) for r in range(world)]
    assert bounds[0][0] == 0 and bounds[-1][1] == pf
    assert all(a[1] == b[0] and a[0] % 4 == 0 for a, b in zip(bounds, bounds[1:]))
    s_bounds = [_chunk(2 * row_stride(n), world, r) for r in range(world)]
    assert s_bounds[-1][1] == 2 * row_stride(n)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class _FlatField:
    def __init__(self, flat, n, deg):
        self.flat, self._n, self.sh_degree, self.version, self.generation = flat, n, deg, 0, 0

    def __len__(self):
        return self._n


def _ipc_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        import types

        from paper_2503_13086_b200.rasterize import FieldGrads
        from paper_2503_13086_b200.train import PeerExchange, exchange_and_step, gather_moments

        n, deg = 3001, 3
        p, grads, m, v = _problem(n, deg, world, seed=5)
        P_ref, M_ref, V_ref, S_ref = _reference(n, deg, p, grads, m, v, steps=1)
        dev = torch.device("cuda", 0)
        fld = _FlatField(p.to(dev).clone(), n, deg)
        opt = types.SimpleNamespace(m=m.to(dev).clone(), v=v.to(dev).clone(), check=lambda f: None,
                                    advance=lambda rate: _rates(1, rate))
        g = FieldGrads(_flat=grads[rank].to(dev).clone(), _n=n, _k=(deg + 1) ** 2)
        ex = PeerExchange()
        results = []
        for it in range(3):  # step 2 reuses the mappings; step 3 follows reallocated buffers
            if it == 1:
                fld.flat.copy_(p.to(dev))
                opt.m.copy_(m.to(dev))
                opt.v.copy_(v.to(dev))
                g.flat.copy_(grads[rank].to(dev))
            if it == 2:  # as after a densify: new parameter and gradient buffers, a new generation
                fld.flat = p.to(dev).clone()
                fld.generation += 1
                opt.m.copy_(m.to(dev))
                opt.v.copy_(v.to(dev))
                g = FieldGrads(_flat=grads[rank].to(dev).clone(), _n=n, _k=(deg + 1) ** 2)
            exchange_and_step(fld, g, opt, 1.6e-4, mode="p2p", exchanger=ex)
            torch.cuda.synchronize()
            gather_moments(fld, opt, mode="p2p")
            results.append((torch.equal(fld.flat.cpu(), P_ref), torch.equal(opt.m.cpu(), M_ref),
                            torch.equal(opt.v.cpu(), V_ref), torch.equal(g.flat[p.numel():].cpu(), S_ref)))
        q.put((rank, results, None))
        dist.barrier()
        dist.destroy_process_group()
    except Exception:  # report instead of hanging the parent
        import traceback

        q.put((rank, None, traceback.format_exc()))
        raise


def test_exchange_p2p_two_processes_one_gpu_ipc():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = {}
    for _ in procs:
        r, out, err = q.get(timeout=300)
        assert err is None, err
        res[r] = out
    for pr in procs:
        pr.join(timeout=60)
    for r in (0, 1):
        for step in res[r]:
            assert all(step), (r, step)  # params, m, v (after gather_moments), statistics
