"""FVB1 batch files through the C ABI.

The native reader/writer (csrc/fvb_io.cpp) is byte-compatible with the
reference's fixture dumps (save_batch / load_batch, mesh.py:313-353), so golden
vectors can be produced and consumed by C code on either side of the GPU box.
Host-only: no device is touched.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import ContractViolationError
from .mesh import PatchBatch, PatchSpec, make_patch_batch

_ARRAYS = ("QIn", "QOut", "cell_centre", "cell_size", "t", "dt", "max_eigenvalue")


def _ptrs(batch: PatchBatch):
    out = []
    for name in _ARRAYS:
        a = getattr(batch, name)
        if not (a.dtype == np.float64 and a.flags.c_contiguous):
            raise ContractViolationError(f"{name} must be C-contiguous float64")
        out.append(ctypes.c_void_p(a.ctypes.data))
    return out


def _raise(rc: int, what: str, path: str) -> None:
    if rc == _lib.FVB_OK:
        return
    if rc == _lib.FVB_ERR_CONTRACT:
        raise ContractViolationError(f"{what}: not a valid FVB1 dump or size mismatch ({path})")
    raise OSError(f"{what}: I/O error on {path} (code {rc})")


def header(path: str) -> tuple[int, int, int, int]:
    """(dimensions, volumes_per_axis, unknowns, n_patches) of an FVB1 file."""
    h = (ctypes.c_int64 * 4)()
    _raise(_lib.load().fvb_fvb1_header(path.encode(), h), "fvb_fvb1_header", path)
    return tuple(int(v) for v in h)


def read(path: str, pinned: bool = False) -> PatchBatch:
    """Load an FVB1 file with the native reader."""
    d, p, s, n = header(path)
    batch = make_patch_batch(PatchSpec(d, p, s), n, pinned=pinned)
    h = (ctypes.c_int64 * 4)(d, p, s, n)
    _raise(_lib.load().fvb_fvb1_read(path.encode(), h, *_ptrs(batch)), "fvb_fvb1_read", path)
    return batch


def write(batch: PatchBatch, path: str) -> None:
    """Dump a batch as FVB1 with the native writer."""
    sp = batch.spec
    h = (ctypes.c_int64 * 4)(sp.dimensions, sp.volumes_per_axis, sp.unknowns, batch.n_patches)
    _raise(_lib.load().fvb_fvb1_write(path.encode(), h, *_ptrs(batch)), "fvb_fvb1_write", path)
