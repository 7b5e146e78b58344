"""The inst_rows workspace (include/ssr.h ssr_rows_floats): ssr_backward writes
gradient rows only for walked slots, tagged with a generation; rows left over
from earlier views carry stale tags and must read as zero in ssr_chain.

Each test compares against a backward run on a freshly zero-filled workspace
(the kernels are deterministic, so the results must be bit-identical).
"""

import pytest

pytestmark = pytest.mark.gpu


def _scene(cfg, n, w, h, seed=11):
    from paper_2503_13086_b200 import GaussianField, scenes

    f = GaussianField.from_host(scenes.make_params(cfg, seed=seed, n=n))
    cams = [scenes.camera(cfg, view=v, width=w, height=h) for v in (2, 7)]
    return f, cams


def _bmod():
    # the module (rasterize/__init__ re-exports the function under the same name)
    import importlib

    return importlib.import_module("paper_2503_13086_b200.rasterize.backward")


def _fresh(backward_fn):
    _bmod()._ROWS.clear()
    return backward_fn()


@pytest.mark.parametrize("layout", ["splat", "pixel"])
def test_stale_rows_of_another_view_read_as_zero(layout):
    import torch

    from paper_2503_13086_b200.rasterize import backward, render

    f, (ca, cb) = _scene(1, 30000, 320, 240)
    out_a, out_b = render(f, ca), render(f, cb)
    da = torch.full_like(out_a.image, 1e-3)
    db = torch.linspace(-1e-3, 1e-3, out_b.image.numel(), device="cuda").view_as(out_b.image)
    ref_b = _fresh(lambda: backward(f, out_b, db, layout=layout)).flat.clone()
    # view A writes rows B never walks (and vice versa) into the same workspace
    for _ in range(2):
        backward(f, out_a, da, layout=layout)
        g = backward(f, out_b, db, layout=layout)
        torch.cuda.synchronize()
        assert torch.equal(g.flat, ref_b)


def test_mixed_layouts_and_soft_gradient_share_the_workspace():
    import torch

    from paper_2503_13086_b200.rasterize import backward, render

    f, (ca, cb) = _scene(2, 60000, 480, 270, seed=5)
    out_a, out_b = render(f, ca), render(f, cb)
    da = torch.full_like(out_a.image, 2e-3)
    db = torch.full_like(out_b.image, -1e-3)
    sb = torch.full_like(out_b.t_final, 1e-4)  # soft-count gradient: the soft pair block
    ref = {lay: _fresh(lambda: backward(f, out_b, db, sb, layout=lay)).flat.clone() for lay in ("splat", "pixel")}
    for lay_a in ("pixel", "splat"):
        for lay_b in ("splat", "pixel"):
            backward(f, out_a, da, layout=lay_a)
            g = backward(f, out_b, db, sb, layout=lay_b)
            torch.cuda.synchronize()
            assert torch.equal(g.flat, ref[lay_b]), (lay_a, lay_b)


def test_two_backwards_before_one_chain_abi():
    """ABI contract: every ssr_backward starts a new generation, so a chain
    after two backwards sees only the second one's rows."""
    import torch

    from paper_2503_13086_b200 import _lib
    from paper_2503_13086_b200.field import class_slices
    from paper_2503_13086_b200.rasterize import backward, render
    from paper_2503_13086_b200.field import flat_size

    FieldGrads, rows_workspace = _bmod().FieldGrads, _bmod().rows_workspace

    f, (ca, cb) = _scene(1, 30000, 320, 240, seed=8)
    out_a, out_b = render(f, ca), render(f, cb)
    da = torch.full_like(out_a.image, 1e-3)
    db = torch.full_like(out_b.image, 5e-4)
    ref = _fresh(lambda: backward(f, out_b, db)).flat.clone()
    n, k = len(f), f.n_sh_coeffs
    st = _lib.stream_ptr()
    m = max(out_a.splats.n_instances, out_b.splats.n_instances)
    rows = rows_workspace(f.flat.device, m)
    for out, d in ((out_a, da), (out_b, db)):
        sp = out.splats
        _lib.call("ssr_backward", 0, sp.n_instances, sp.struct(), sp.inst_gauss.data_ptr(), sp.tile_ranges.data_ptr(),
                  out.frame_struct(), d.data_ptr(), None, rows.data_ptr(), st)
    grads = FieldGrads(_flat=torch.empty(flat_size(n, k, extra=2), dtype=torch.float32, device="cuda"), _n=n, _k=k)
    flat, sl = f.flat, class_slices(n, k)
    _lib.call("ssr_chain", _lib.camera_struct(cb), n, f.sh_degree, flat[sl[0][0]:].data_ptr(),
              flat[sl[1][0]:].data_ptr(), flat[sl[2][0]:].data_ptr(), flat[sl[4][0]:].data_ptr(), out_b.splats.struct(),
              rows.data_ptr(), grads.flat.data_ptr(), 0, None, None, st)
    torch.cuda.synchronize()
    assert torch.equal(grads.flat, ref)


def test_workspace_regrows_zero_filled():
    import torch

    from paper_2503_13086_b200.rasterize import backward, render

    bmod = _bmod()
    f_small, (cs, _) = _scene(0, 2000, 64, 64)
    f_big, (cb, _) = _scene(1, 30000, 320, 240)
    bmod._ROWS.clear()
    o_s = render(f_small, cs)
    backward(f_small, o_s, torch.full_like(o_s.image, 1e-3))
    cap0 = next(iter(bmod._ROWS.values())).numel()
    o_b = render(f_big, cb)
    d = torch.full_like(o_b.image, 1e-3)
    g = backward(f_big, o_b, d).flat.clone()
    assert next(iter(bmod._ROWS.values())).numel() > cap0
    ref = _fresh(lambda: backward(f_big, o_b, d)).flat
    torch.cuda.synchronize()
    assert torch.equal(g, ref)
