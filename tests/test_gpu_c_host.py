"""The C-ABI boundary from a plain C host (examples/c_host_demo.c): gcc + libfvb200.so + cudart,
no Python or torch on the data path; bit-identical to the oracle."""

import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)


def test_c_host_demo_bit_identical():
    ex = os.path.join(ROOT, "examples")
    subprocess.run(["make", "-s", "-C", ex], check=True, capture_output=True, timeout=120)
    r = subprocess.run([os.path.join(ex, "c_host_demo")], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("bit-identical to the oracle") == 2, r.stdout
