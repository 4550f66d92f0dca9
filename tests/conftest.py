"""Shared fixtures.  GPU tests carry @pytest.mark.gpu and run on a B200 via gpurun."""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def manifest():
    with open(os.path.join(GOLDEN, "manifest.json")) as f:
        return json.load(f)


def load_golden(name_or_file):
    from paper_2302_09005_b200 import mesh

    fname = name_or_file if name_or_file.endswith(".fvb") else name_or_file + ".fvb"
    return mesh.load_batch(os.path.join(GOLDEN, fname))


def assert_bits_equal(a, b, what=""):
    """Bitwise equality of float64 arrays; NaN positions must coincide (payloads may differ)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    nan_a, nan_b = np.isnan(a), np.isnan(b)
    assert np.array_equal(nan_a, nan_b), f"{what}: NaN positions differ"
    same = (a.view(np.uint64) == b.view(np.uint64)) | nan_a
    if not np.all(same):
        idx = np.argwhere(~same)[:5]
        details = [(tuple(i), a[tuple(i)], b[tuple(i)]) for i in idx]
        raise AssertionError(f"{what}: {int((~same).sum())} elements differ bitwise, e.g. {details}")


def import_reference():
    """The reference package `fvbatch`, or None.

    Looked up in baseline/_ref (the offline pip install of /root/reference,
    git-ignored but shipped to the GPU box with the snapshot) and then in
    /root/reference/pkg/src (this container only).  Tests use it as the
    caller side of the drop-in and as a second checker; the product package
    never imports it."""
    import importlib

    for path in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(path, "fvbatch")):
            if path not in sys.path:
                sys.path.append(path)
            try:
                return importlib.import_module("fvbatch")
            except Exception:  # pragma: no cover - broken install
                return None
    return None
