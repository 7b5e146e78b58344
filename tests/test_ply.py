"""PLY field snapshots (io/ply.py of the reference).

Fixtures ``tests/golden/ply_*.ply`` were written by the reference's own
write_ply (tests/golden/make_golden_ply.py).  CPU tests cover the header
grammar and every error path (they raise before any device work); GPU tests
check that our reader recovers the reference's parameters exactly, that our
writer reproduces the reference's bytes, and the bit-exact round trip of the
reference's own test (pkg/tests/test_io.py:207-247).
"""

import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN_DIR

PLY_CASES = sorted(os.path.splitext(os.path.basename(p))[0] for p in glob.glob(os.path.join(GOLDEN_DIR, "ply_*.ply")))


def _header_names(data: bytes):
    head = data[: data.find(b"end_header\n")].decode("ascii").splitlines()
    return [ln.split()[2] for ln in head if ln.startswith("property")], head


def test_fixtures_present():
    assert len(PLY_CASES) >= 5


@pytest.mark.parametrize("name", PLY_CASES)
def test_property_names_match_reference_header(name):
    from paper_2503_13086_b200.ply import _property_names

    data = open(os.path.join(GOLDEN_DIR, name + ".ply"), "rb").read()
    names, head = _header_names(data)
    deg = int(np.load(os.path.join(GOLDEN_DIR, name + ".npz"))["sh_degree"])
    assert names == _property_names((deg + 1) ** 2)
    assert head[:2] == ["ply", "format binary_little_endian 1.0"]


def _write(tmp_path, text, body=b""):
    p = tmp_path / "x.ply"
    p.write_bytes(text.encode("ascii") + body)
    return p


def test_error_paths(tmp_path):
    from paper_2503_13086_b200.errors import InvalidParameter
    from paper_2503_13086_b200.ply import _property_names, read_ply

    with pytest.raises(InvalidParameter, match="missing"):
        read_ply(tmp_path / "nope.ply")
    with pytest.raises(InvalidParameter, match="not a PLY"):
        read_ply(_write(tmp_path, "plx\nend_header\n"))
    good = "".join(f"property double {n}\n" for n in _property_names(1))
    with pytest.raises(InvalidParameter, match="unsupported element"):
        read_ply(_write(tmp_path, "ply\nformat binary_little_endian 1.0\nelement face 1\n" + good + "end_header\n"))
    with pytest.raises(InvalidParameter, match="expected double"):
        read_ply(_write(tmp_path, "ply\nformat binary_little_endian 1.0\nelement vertex 0\nproperty float x\n"
                                  "end_header\n"))
    with pytest.raises(InvalidParameter, match="unsupported format"):
        read_ply(_write(tmp_path, "ply\nformat ascii 1.0\nelement vertex 0\n" + good + "end_header\n"))
    with pytest.raises(InvalidParameter, match="no vertex element"):
        read_ply(_write(tmp_path, "ply\nformat binary_little_endian 1.0\n" + good + "end_header\n"))
    rest2 = good.replace("property double opacity\n", "property double f_rest_0\nproperty double f_rest_1\n"
                                                      "property double opacity\n")
    with pytest.raises(InvalidParameter, match="not divisible by 3"):
        read_ply(_write(tmp_path, "ply\nformat binary_little_endian 1.0\nelement vertex 0\n" + rest2 + "end_header\n"))
    rest6 = "".join(f"property double f_rest_{i}\n" for i in range(6))
    with pytest.raises(InvalidParameter, match="match no degree"):
        read_ply(_write(tmp_path, "ply\nformat binary_little_endian 1.0\nelement vertex 0\n" + good + rest6 +
                        "end_header\n"))
    with pytest.raises(InvalidParameter, match="unexpected property set"):
        read_ply(_write(tmp_path, "ply\nformat binary_little_endian 1.0\nelement vertex 0\n" +
                        good.replace("rot_3", "rot_9") + "end_header\n"))
    with pytest.raises(InvalidParameter, match="body"):
        read_ply(_write(tmp_path, "ply\nformat binary_little_endian 1.0\nelement vertex 1\n" + good + "end_header\n",
                        b"\0" * 8))


@pytest.mark.gpu
@pytest.mark.parametrize("name", PLY_CASES)
def test_reference_files_read_and_rewritten_bit_exact(name, tmp_path):
    from paper_2503_13086_b200 import GaussianField
    from paper_2503_13086_b200.ply import read_ply, write_ply

    src = os.path.join(GOLDEN_DIR, name + ".ply")
    g = np.load(os.path.join(GOLDEN_DIR, name + ".npz"))
    f = read_ply(src)
    assert f.sh_degree == int(g["sh_degree"]) and len(f) == g["positions"].shape[0]
    for k in ("positions", "rotations", "log_scales", "opacity_logits", "sh"):
        np.testing.assert_array_equal(getattr(f, k).cpu().numpy().astype(np.float64), g[k])
    out = tmp_path / "again.ply"
    write_ply(f, out)
    assert out.read_bytes() == open(src, "rb").read()
    if len(f):
        f2 = GaussianField.from_arrays(*(g[k].astype(np.float32) for k in (
            "positions", "rotations", "log_scales", "opacity_logits", "sh")))
        out2 = tmp_path / "fresh.ply"
        write_ply(f2, out2)
        assert out2.read_bytes() == open(src, "rb").read()


@pytest.mark.gpu
def test_round_trip_bit_exact(tmp_path):
    """pkg/tests/test_io.py:207-222: 40 random fields, every degree."""
    from paper_2503_13086_b200 import GaussianField
    from paper_2503_13086_b200.ply import read_ply, write_ply

    rng = np.random.default_rng(1)
    for case in range(40):
        deg = case % 4
        n, k = int(rng.integers(1, 30)), (deg + 1) ** 2
        f = GaussianField.from_arrays(rng.normal(size=(n, 3)), rng.normal(size=(n, 4)) + 0.1,
                                      rng.normal(size=(n, 3)), rng.normal(size=n), rng.normal(size=(n, 3, k)))
        p = tmp_path / f"f{case}.ply"
        write_ply(f, p)
        again = read_ply(p)
        assert again.sh_degree == f.sh_degree
        for name in ("positions", "rotations", "log_scales", "opacity_logits", "sh"):
            assert bool((getattr(again, name) == getattr(f, name)).all()), name
        assert again.checksum() == f.checksum()


@pytest.mark.gpu
def test_empty_degree0_and_truncated(tmp_path):
    from paper_2503_13086_b200 import GaussianField
    from paper_2503_13086_b200.errors import InvalidParameter
    from paper_2503_13086_b200.ply import read_ply, write_ply

    p = tmp_path / "empty.ply"
    write_ply(GaussianField(sh_degree=0), p)
    assert len(read_ply(p)) == 0
    assert "element vertex 0" in p.read_bytes().split(b"end_header")[0].decode()
    rng = np.random.default_rng(2)
    f = GaussianField.from_arrays(rng.normal(size=(3, 3)), rng.normal(size=(3, 4)), rng.normal(size=(3, 3)),
                                  rng.normal(size=3), rng.normal(size=(3, 3, 1)))
    write_ply(f, p)
    assert b"f_rest" not in p.read_bytes().split(b"end_header")[0]
    p.write_bytes(p.read_bytes()[:-8])
    with pytest.raises(InvalidParameter, match="body"):
        read_ply(p)
