"""CPU oracle for the batched Rusanov patch update -- TEST INFRASTRUCTURE ONLY.

A plain-C restatement of the reference's default engine
(`fvbatch.kernel.vectorized`, /root/reference/pkg/src/fvbatch/kernel/vectorized.py)
compiled from `oracle/fvb_oracle.c` into `oracle/_build/libfvb_oracle.so`.

Only `tests/`, `__graft_entry__.smoke()` and the `cpu_baseline` /
`--impl reference` legs of `bench.py` may import this module, and only as the
checker or as the timed CPU baseline.  The product package
(`paper_2302_09005_b200`) never imports it.

Parity of this restatement is pinned bit-for-bit against golden vectors the
reference itself produced (tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libfvb_oracle.so")
_lib = None


class BoxInfo(ctypes.Structure):
    _fields_ = [("trig_rho", ctypes.c_int64), ("trig_p", ctypes.c_int64),
                ("first_nonpos", ctypes.c_int64), ("first_badpl", ctypes.c_int64)]


def build() -> str:
    """Compile the oracle with its Makefile (no-op when up to date)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        dp = ctypes.POINTER(ctypes.c_double)
        L.fvb_oracle_update.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_double,
                                        dp, dp, dp, dp, dp, ctypes.c_int]
        L.fvb_oracle_update.restype = ctypes.c_int
        L.fvb_oracle_locate.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_double,
                                        dp, ctypes.POINTER(BoxInfo), ctypes.c_int]
        L.fvb_oracle_locate.restype = ctypes.c_int
        L.fvb_oracle_first_error.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.POINTER(BoxInfo), ctypes.c_int,
            ctypes.c_int64, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int),
            ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int)]
        L.fvb_oracle_first_error.restype = ctypes.c_int
        _lib = L
    return _lib


def _dp(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def update(dim: int, p: int, gamma: float, qin: np.ndarray, cell_size: np.ndarray,
           dt: np.ndarray, nthreads: int = 0):
    """Return (qout, max_eig, status); status 0 ok, 2 non-physical state."""
    n = qin.shape[0]
    s = dim + 2
    qin = np.ascontiguousarray(qin, dtype=np.float64)
    cell_size = np.ascontiguousarray(cell_size, dtype=np.float64)
    dt = np.ascontiguousarray(dt, dtype=np.float64)
    qout = np.zeros((n, p ** dim * s))
    max_eig = np.zeros(n)
    st = lib().fvb_oracle_update(dim, p, n, gamma, _dp(qin), _dp(qout), _dp(cell_size), _dp(dt),
                                 _dp(max_eig), nthreads)
    return qout, max_eig, st


def locate(dim: int, p: int, gamma: float, qin: np.ndarray, nthreads: int = 0) -> np.ndarray:
    """Per-(patch, box) diagnostics as an int64 array (n, 2*dim+1, 4)."""
    n = qin.shape[0]
    qin = np.ascontiguousarray(qin, dtype=np.float64)
    info = (BoxInfo * (n * (2 * dim + 1)))()
    lib().fvb_oracle_locate(dim, p, n, gamma, _dp(qin), info, nthreads)
    arr = np.ctypeslib.as_array(ctypes.cast(info, ctypes.POINTER(ctypes.c_int64)),
                                shape=(n, 2 * dim + 1, 4)).copy()
    return arr


def first_error(dim: int, p: int, info: np.ndarray, ordering: int, nchunks: int):
    """(patch, box, lin, kind) of the first error the vectorized engine raises, or None."""
    n = info.shape[0]
    flat = np.ascontiguousarray(info, dtype=np.int64)
    ptr = flat.ctypes.data_as(ctypes.POINTER(BoxInfo))
    patch, lin = ctypes.c_int64(), ctypes.c_int64()
    box, kind = ctypes.c_int(), ctypes.c_int()
    hit = lib().fvb_oracle_first_error(dim, p, n, ptr, ordering, nchunks, ctypes.byref(patch),
                                       ctypes.byref(box), ctypes.byref(lin), ctypes.byref(kind))
    if not hit:
        return None
    return int(patch.value), int(box.value), int(lin.value), int(kind.value)


def box_ranges(dim: int, p: int):
    """Haloed (x, y, z) half-open ranges per box, vectorized._plan order (vectorized.py:42-53)."""
    inner = [(1, p + 1) if a < dim else (0, 1) for a in range(3)]
    boxes = [list(inner)]
    for n in range(dim):
        lo = list(inner); lo[n] = (0, 1)
        hi = list(inner); hi[n] = (p + 1, p + 2)
        boxes += [lo, hi]
    return boxes


def box_volume(dim: int, p: int, box: int, lin: int):
    """Haloed volume tuple (x, y[, z]) of a box-linear index (C order z, y, x)."""
    (x0, x1), (y0, y1), (z0, z1) = box_ranges(dim, p)[box]
    nx, ny = x1 - x0, y1 - y0
    z, rem = divmod(lin, nx * ny)
    y, x = divmod(rem, nx)
    vol = (x + x0, y + y0, z + z0)
    return vol[:dim]


# --- synthetic inputs -----------------------------------------

def synthetic_qin(dim: int, p: int, n: int, seed: int = 0, gamma: float = 1.4) -> np.ndarray:
    """Random admissible Euler states over ALL haloed volumes (corners included):
    rho ~ U[0.5,2], u_i ~ U[-1,1], p ~ U[0.5,2], E = p/(gamma-1) + 0.5 rho |u|^2."""
    rng = np.random.default_rng(seed)
    e = p + 2
    v = e ** dim
    rho = rng.uniform(0.5, 2.0, size=(n, v))
    vel = rng.uniform(-1.0, 1.0, size=(n, v, dim))
    pr = rng.uniform(0.5, 2.0, size=(n, v))
    q = np.empty((n, v, dim + 2))
    q[..., 0] = rho
    q[..., 1:1 + dim] = rho[..., None] * vel
    q[..., -1] = pr / (gamma - 1.0) + 0.5 * rho * np.sum(vel * vel, axis=-1)
    return q.reshape(n, v * (dim + 2))


def halo_project(dim: int, p: int, qout: np.ndarray, grid, periodic: bool, s: int | None = None) -> np.ndarray:
    """Restatement of mesh.halo_project (mesh.py:261-310) as index arithmetic (numpy):
    haloed QIn of every patch from the grid's interior QOut, per-axis wrap / clamp."""
    grid = tuple(int(g) for g in grid)
    n = int(np.prod(grid))
    s = dim + 2 if s is None else s
    e = p + 2
    qo = np.asarray(qout).reshape(n, p ** dim, s)
    qin = np.empty((n, e ** dim, s))
    h = np.indices((e,) * dim).reshape(dim, -1)[::-1]           # rows: haloed x, y[, z]
    for patch in range(n):
        c, rem = [], patch
        for a in range(dim):
            rem, ca = divmod(rem, grid[a])
            c.append(ca)
        src_patch = np.zeros(h.shape[1], dtype=np.int64)
        src_vol = np.zeros(h.shape[1], dtype=np.int64)
        for a in reversed(range(dim)):
            ext = grid[a] * p
            gi = c[a] * p + h[a] - 1
            gi = np.mod(gi, ext) if periodic else np.clip(gi, 0, ext - 1)
            src_patch = src_patch * grid[a] + gi // p
            src_vol = src_vol * p + gi % p
        qin[patch] = qo[src_patch, src_vol]
    return qin.reshape(n, -1)
