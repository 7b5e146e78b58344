"""PLY snapshot fixtures written by the REFERENCE's io/ply.py:write_ply.

Run in the builder container only (needs /root/reference, read-only):

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_ply.py

For SH degrees 0..3 (and an empty field) a seeded random field whose values
are float32-representable (the GPU field stores float32) is handed to the
reference GaussianField and written with the reference writer.  The .ply
bytes and the parameters (.npz) are committed; tests/test_ply.py checks that
our read_ply recovers the parameters exactly and our write_ply reproduces the
reference's bytes.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from splatstream.field import GaussianField  # noqa: E402
from splatstream.io.ply import write_ply  # noqa: E402


def main():
    rng = np.random.default_rng(2503)
    for deg, n in ((0, 5), (1, 7), (2, 3), (3, 11), (3, 0)):
        k = (deg + 1) ** 2
        f32 = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)
        p = dict(positions=f32(rng.normal(size=(n, 3))), rotations=f32(rng.normal(size=(n, 4)) + 0.1),
                 log_scales=f32(rng.normal(size=(n, 3))), opacity_logits=f32(rng.normal(size=n)),
                 sh=f32(rng.normal(size=(n, 3, k))))
        fld = GaussianField(sh_degree=deg)
        if n:
            fld._append(**p)
        name = f"ply_deg{deg}_n{n}"
        write_ply(fld, os.path.join(HERE, name + ".ply"))
        np.savez(os.path.join(HERE, name + ".npz"), sh_degree=deg, **p)
        print("wrote", name)


if __name__ == "__main__":
    main()
