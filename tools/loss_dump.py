"""Dump total_loss outputs (scalars, d_image, d_soft) for a few seeded image
sizes, for bit-exact A/B of two library builds:
  SSR_LIB=... python tools/loss_dump.py OUT.npz"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_13086_b200 import _lib  # noqa: E402

res = {}
g = torch.Generator(device="cuda").manual_seed(3)
for (h, w) in [(1080, 1920), (840, 1297), (11, 11), (37, 100), (70, 65)]:
    img = torch.rand(h, w, 3, device="cuda", generator=g)
    for u8 in (0, 1):
        tgt = (torch.rand(h, w, 3, device="cuda", generator=g) * 255).to(torch.uint8) if u8 else \
            torch.rand(h, w, 3, device="cuda", generator=g)
        soft = torch.rand(h, w, device="cuda", generator=g, dtype=torch.float64) * 40
        hard = (torch.rand(h, w, device="cuda", generator=g) * 30).to(torch.int32)
        d_img = torch.empty_like(img)
        d_soft = torch.empty(h, w, device="cuda")
        out = torch.empty(5, device="cuda", dtype=torch.float64)
        ws = torch.empty(_lib.query("ssr_loss_workspace", w, h), dtype=torch.uint8, device="cuda")
        _lib.call("ssr_loss", w, h, img.data_ptr(), tgt.data_ptr(), u8, soft.data_ptr(), hard.data_ptr(), 0.47, 0.12,
                  0.41, d_img.data_ptr(), d_soft.data_ptr(), out.data_ptr(), ws.data_ptr(), ws.numel(),
                  _lib.stream_ptr())
        k = f"{h}x{w}_{u8}"
        res[k + "_out"] = out.cpu().numpy()
        res[k + "_dimg"] = d_img.cpu().numpy()
        res[k + "_dsoft"] = d_soft.cpu().numpy()
torch.cuda.synchronize()
np.savez(sys.argv[1], **res)
print("saved", len(res))
