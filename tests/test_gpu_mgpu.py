"""GPU tests of the C ABI's multi-GPU entry points (fvb_mgpu_*, include/fvb200.h): the step's
MAX all-reduce of the wave speed over NCCL, in both process models, on the one GPU a test box
has (a single-rank communicator; the exchange pattern across ranks is the driver's, tested
with gloo in test_multirank_gloo.py)."""

import ctypes

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2302_09005_b200 import _lib  # noqa: E402
from paper_2302_09005_b200.device import _stream_handle, _vp  # noqa: E402


def test_mgpu_single_process_model():
    L = _lib.load()
    devs = (ctypes.c_int * 1)(torch.cuda.current_device())
    assert L.fvb_mgpu_init(1, devs) == 0
    try:
        assert L.fvb_mgpu_init(1, devs) == 1            # already initialised: contract error
        buf = torch.tensor([3.25], dtype=torch.float64, device="cuda")
        st = _stream_handle(torch, None)
        assert L.fvb_mgpu_allreduce_max(0, _vp(buf), st) == 0
        assert L.fvb_mgpu_allreduce_max(1, _vp(buf), st) == 1   # no such rank
        bufs = (ctypes.c_void_p * 1)(buf.data_ptr())
        streams = (ctypes.c_void_p * 1)(st)
        assert L.fvb_mgpu_allreduce_max_all(bufs, streams) == 0
        torch.cuda.synchronize()
        assert float(buf.item()) == 3.25
    finally:
        assert L.fvb_mgpu_finalize() == 0


def test_mgpu_process_per_gpu_model():
    L = _lib.load()
    uid = (ctypes.c_uint8 * 128)()
    assert L.fvb_mgpu_unique_id(uid) == 0
    assert L.fvb_mgpu_init_rank(1, 1, uid) == 1          # rank out of range
    assert L.fvb_mgpu_init_rank(1, 0, uid) == 0
    try:
        buf = torch.tensor([float("inf")], dtype=torch.float64, device="cuda")
        assert L.fvb_mgpu_allreduce_max(0, _vp(buf), _stream_handle(torch, None)) == 0
        torch.cuda.synchronize()
        assert buf.item() == float("inf")
    finally:
        assert L.fvb_mgpu_finalize() == 0
