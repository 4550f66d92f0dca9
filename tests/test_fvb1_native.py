"""Native FVB1 reader/writer (csrc/fvb_io.cpp) vs the reference format.

Host-only C code: runs on the CPU, against the committed golden dumps that the
reference itself wrote (tests/golden/make_golden.py).
"""

import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN, assert_bits_equal
from paper_2302_09005_b200 import fvb1, mesh
from paper_2302_09005_b200.errors import ContractViolationError

FILES = sorted(glob.glob(os.path.join(GOLDEN, "*.fvb")))


@pytest.mark.parametrize("path", FILES, ids=os.path.basename)
def test_native_read_matches_python_reader(path):
    ref = mesh.load_batch(path)
    got = fvb1.read(path)
    assert fvb1.header(path) == (ref.spec.dimensions, ref.spec.volumes_per_axis, ref.spec.unknowns, ref.n_patches)
    for name in ("QIn", "QOut", "cell_centre", "cell_size", "t", "dt", "max_eigenvalue"):
        assert_bits_equal(getattr(got, name), getattr(ref, name), name)


@pytest.mark.parametrize("path", FILES[:6], ids=os.path.basename)
def test_native_write_is_byte_identical(path, tmp_path):
    b = mesh.load_batch(path)
    out = str(tmp_path / "native.fvb")
    fvb1.write(b, out)
    with open(path, "rb") as f, open(out, "rb") as g:
        assert f.read() == g.read()


def test_round_trip_random_batch(tmp_path):
    rng = np.random.default_rng(3)
    b = mesh.make_patch_batch(mesh.PatchSpec(3, 5, 5), 7)
    for name in ("QIn", "QOut", "cell_centre", "cell_size", "t", "dt", "max_eigenvalue"):
        a = getattr(b, name)
        a[...] = rng.standard_normal(a.shape)
    b.QIn.reshape(-1)[::97] = -0.0
    b.QOut.reshape(-1)[::89] = np.nan
    out = str(tmp_path / "rt.fvb")
    fvb1.write(b, out)
    py = mesh.load_batch(out)
    nat = fvb1.read(out)
    for name in ("QIn", "QOut", "cell_centre", "cell_size", "t", "dt", "max_eigenvalue"):
        assert_bits_equal(getattr(nat, name), getattr(b, name), name)
        assert_bits_equal(getattr(py, name), getattr(b, name), name)


def test_errors(tmp_path):
    bad = tmp_path / "bad.fvb"
    bad.write_bytes(b"NOPE" + bytes(32))
    with pytest.raises(ContractViolationError):
        fvb1.read(str(bad))
    with pytest.raises(OSError):
        fvb1.header(str(tmp_path / "missing.fvb"))
    trunc = tmp_path / "trunc.fvb"
    data = open(FILES[0], "rb").read()
    trunc.write_bytes(data[: len(data) // 2])
    with pytest.raises(OSError):
        fvb1.read(str(trunc))
