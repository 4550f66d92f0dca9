"""ctypes binding of libfvb200.so (the C ABI in include/fvb200.h).

The shared library is built in-tree (`paper_2302_09005_b200/libfvb200.so`,
see csrc/Makefile and `__graft_entry__.build()`).  There is no fallback: if
the library or a CUDA device is missing, every device entry point raises.
"""

from __future__ import annotations

import ctypes
import os

from .errors import ContractViolationError, DeviceError

HERE = os.path.dirname(os.path.abspath(__file__))
# FVB_LIB_PATH selects an alternative in-tree build (A/B measurements of kernel variants)
LIB_PATH = os.environ.get("FVB_LIB_PATH") or os.path.join(HERE, "libfvb200.so")

FVB_OK = 0
FVB_ERR_CONTRACT = 1
FVB_ERR_NONPHYSICAL = 2
FVB_ERR_CUDA = 3
FVB_ERR_IO = 4

KERNEL_AUTO = 0
KERNEL_GENERIC = 1
KERNEL_FUSED = 2

# Every symbol include/fvb200.h declares (checked by the CPU test suite).
EXPORTED = (
    "fvb_version", "fvb_strerror", "fvb_select_kernel", "fvb_update", "fvb_update_cfl", "fvb_status_words",
    "fvb_update_host_workspace", "fvb_update_host", "fvb_locate", "fvb_pack", "fvb_unpack",
    "fvb_reduce_dt", "fvb_set_dt", "fvb_patch_max_eig", "fvb_probe", "fvb_selftest_div",
    "fvb_halo_project", "fvb_halo_project_totals", "fvb_halo_project_window",
    "fvb_host_pin", "fvb_host_unpin", "fvb_update_to_haloed", "fvb_halo_shell", "fvb_totals_haloed",
    "fvb_mgpu_unique_id", "fvb_mgpu_init_rank", "fvb_mgpu_init", "fvb_mgpu_allreduce_max",
    "fvb_mgpu_allreduce_max_all", "fvb_mgpu_finalize", "fvb_totals_scratch_bytes", "fvb_totals",
    "fvb_fvb1_header", "fvb_fvb1_read", "fvb_fvb1_write", "fvb_time_next_update",
    "fvb_step_record",
)


class FvbSpec(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("p", ctypes.c_int32), ("unknowns", ctypes.c_int32),
                ("layout", ctypes.c_int32), ("n_patches", ctypes.c_int64), ("gamma", ctypes.c_double)]


class FvbBoxInfo(ctypes.Structure):
    _fields_ = [("trig_rho", ctypes.c_int64), ("trig_p", ctypes.c_int64),
                ("first_nonpos", ctypes.c_int64), ("first_badpl", ctypes.c_int64)]


_lib = None


def load():
    """Load and prototype libfvb200.so (raises ImportError when it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    vp, sp = ctypes.c_void_p, ctypes.POINTER(FvbSpec)
    i64, i32, dbl = ctypes.c_int64, ctypes.c_int, ctypes.c_double
    L.fvb_version.restype = i32
    L.fvb_version.argtypes = []
    L.fvb_strerror.restype = ctypes.c_char_p
    L.fvb_strerror.argtypes = [i32]
    L.fvb_select_kernel.restype = i32
    L.fvb_select_kernel.argtypes = [sp]
    L.fvb_update.restype = i32
    L.fvb_update.argtypes = [sp, vp, vp, vp, vp, vp, vp, i32, i32, vp]
    L.fvb_update_cfl.restype = i32
    L.fvb_update_cfl.argtypes = [sp, vp, vp, vp, vp, vp, vp, i32, ctypes.c_double, ctypes.c_double, vp, vp, i32, vp]
    L.fvb_status_words.restype = ctypes.c_size_t
    L.fvb_status_words.argtypes = [i64]
    L.fvb_update_host_workspace.restype = ctypes.c_size_t
    L.fvb_update_host_workspace.argtypes = [sp, i64]
    L.fvb_update_host.restype = i32
    L.fvb_update_host.argtypes = [sp, vp, vp, vp, vp, vp, vp, ctypes.c_size_t, i64, i32, vp]
    L.fvb_locate.restype = i32
    L.fvb_locate.argtypes = [sp, vp, vp, vp]
    L.fvb_pack.restype = i32
    L.fvb_pack.argtypes = [sp, vp, vp, i32, vp]
    L.fvb_unpack.restype = i32
    L.fvb_unpack.argtypes = [sp, vp, vp, i32, vp]
    L.fvb_reduce_dt.restype = i32
    L.fvb_reduce_dt.argtypes = [vp, i64, dbl, dbl, vp, vp, vp, i32, vp]
    L.fvb_set_dt.restype = i32
    L.fvb_set_dt.argtypes = [vp, dbl, dbl, vp, vp, i64, vp]
    L.fvb_patch_max_eig.restype = i32
    L.fvb_patch_max_eig.argtypes = [sp, vp, vp, vp, vp]
    L.fvb_probe.restype = i32
    L.fvb_probe.argtypes = [i32, dbl, vp, i64, vp, vp, vp, vp, vp]
    L.fvb_halo_project.restype = i32
    L.fvb_halo_project.argtypes = [sp, vp, vp, vp, i32, vp]
    L.fvb_halo_project_totals.restype = i32
    L.fvb_halo_project_totals.argtypes = [sp, vp, vp, vp, i32, vp, vp, vp]
    L.fvb_halo_project_window.restype = i32
    L.fvb_halo_project_window.argtypes = [sp, vp, vp, vp, vp, vp, i32, i32, vp, vp, vp]
    L.fvb_step_record.restype = i32
    L.fvb_step_record.argtypes = [vp, vp, vp, vp, i32, vp, vp, vp, vp, vp, vp]
    L.fvb_time_next_update.restype = i32
    L.fvb_time_next_update.argtypes = [vp, vp]
    L.fvb_update_to_haloed.restype = i32
    L.fvb_update_to_haloed.argtypes = [sp, vp, vp, vp, vp, vp, vp, i32, vp]
    L.fvb_halo_shell.restype = i32
    L.fvb_halo_shell.argtypes = [sp, vp, vp, i32, vp]
    L.fvb_totals_haloed.restype = i32
    L.fvb_totals_haloed.argtypes = [sp, vp, vp, vp, vp]
    L.fvb_host_pin.restype = i32
    L.fvb_host_pin.argtypes = [vp, ctypes.c_size_t]
    L.fvb_host_unpin.restype = i32
    L.fvb_host_unpin.argtypes = [vp]
    L.fvb_mgpu_unique_id.restype = i32
    L.fvb_mgpu_unique_id.argtypes = [vp]
    L.fvb_mgpu_init_rank.restype = i32
    L.fvb_mgpu_init_rank.argtypes = [i32, i32, vp]
    L.fvb_mgpu_init.restype = i32
    L.fvb_mgpu_init.argtypes = [i32, vp]
    L.fvb_mgpu_allreduce_max.restype = i32
    L.fvb_mgpu_allreduce_max.argtypes = [i32, vp, vp]
    L.fvb_mgpu_allreduce_max_all.restype = i32
    L.fvb_mgpu_allreduce_max_all.argtypes = [vp, vp]
    L.fvb_mgpu_finalize.restype = i32
    L.fvb_mgpu_finalize.argtypes = []
    L.fvb_totals_scratch_bytes.restype = ctypes.c_size_t
    L.fvb_totals_scratch_bytes.argtypes = [sp]
    L.fvb_totals.restype = i32
    L.fvb_totals.argtypes = [sp, vp, vp, vp, vp]
    cp, i64p = ctypes.c_char_p, ctypes.POINTER(ctypes.c_int64)
    L.fvb_fvb1_header.restype = i32
    L.fvb_fvb1_header.argtypes = [cp, i64p]
    L.fvb_fvb1_read.restype = i32
    L.fvb_fvb1_read.argtypes = [cp, i64p] + [vp] * 7
    L.fvb_fvb1_write.restype = i32
    L.fvb_fvb1_write.argtypes = [cp, i64p] + [vp] * 7
    L.fvb_selftest_div.restype = i32
    L.fvb_selftest_div.argtypes = [vp, vp, vp, vp, i64, vp]
    _lib = L
    return L


def spec(dim: int, p: int, n: int, gamma: float, layout: int = 0, unknowns: int | None = None) -> FvbSpec:
    """C-ABI spec; `unknowns` defaults to the Euler count d + 2 (only fvb_halo_project accepts others)."""
    return FvbSpec(dim, p, dim + 2 if unknowns is None else unknowns, layout, n, gamma)


def check(rc: int, what: str) -> None:
    """Map a C-ABI return code onto the reference's exception classes."""
    if rc == FVB_OK:
        return
    msg = load().fvb_strerror(rc).decode(errors="replace")
    if rc == FVB_ERR_CONTRACT:
        raise ContractViolationError(f"{what}: {msg}")
    raise DeviceError(f"{what}: {msg} (code {rc})")
