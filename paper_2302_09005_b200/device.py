"""Device-side plumbing: PyTorch owns the CUDA buffers and streams, libfvb200.so computes.

* `DeviceBatch`   a PatchBatch resident in HBM (AoS or packed SoA), with
                  `update()` (fvb_update), `locate()` (fvb_locate),
                  `max_eig_prepass()` and host round trips.
* `update_host`   the drop-in path used by `kernel.update_patch_batch`: host
                  numpy arrays in, host arrays out, through fvb_update_host's
                  chunked H2D / kernel / D2H pipeline.
* `probe`         the closure probe behind the PdeDefinition callbacks.

There is no CPU fallback anywhere: without a CUDA device these raise.
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import _lib
from .errors import ContractViolationError, DeviceError
from .mesh import PatchBatch, PatchSpec

LAYOUTS = {"aos": 0, "soa": 1}
KERNELS = {"auto": _lib.KERNEL_AUTO, "generic": _lib.KERNEL_GENERIC, "fused": _lib.KERNEL_FUSED}


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device visible: the B200 patch update has no CPU fallback")
    return torch


def _vp(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def _hp(a: np.ndarray) -> ctypes.c_void_p:
    return ctypes.c_void_p(a.ctypes.data)


def _stream_handle(torch, stream) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


MODES = {"exact": 0, "fast": 0x100}   # FVB_MODE_FAST (include/fvb200.h)


def kernel_id(kernel, mode: str = "exact") -> int:
    """C-ABI kernel selector; mode "fast" ORs in FVB_MODE_FAST (1e-12 relative parity)."""
    if mode not in MODES:
        raise ContractViolationError(f"unknown mode {mode!r} (expected 'exact' or 'fast')")
    if isinstance(kernel, int):
        return kernel | MODES[mode]
    try:
        return KERNELS[kernel] | MODES[mode]
    except KeyError:
        raise ContractViolationError(f"unknown kernel selector {kernel!r}") from None


def selected_kernel(dim: int, p: int, n: int, gamma: float, layout: str = "aos") -> str:
    """Name of the kernel FVB_KERNEL_AUTO resolves to for this shape."""
    k = _lib.load().fvb_select_kernel(ctypes.byref(_lib.spec(dim, p, n, gamma, LAYOUTS[layout])))
    return {1: "generic", 2: "fused"}.get(k, "invalid")


class DeviceBatch:
    """A batch of haloed patches resident in device memory.

    layout "aos" keeps the reference's PatchBatch order; "soa" stores the
    packed LayoutEnumerator(SOA) order produced by fvb_pack.
    """

    def __init__(self, spec: PatchSpec, n_patches: int, gamma: float, device=None, layout: str = "aos"):
        torch = _torch()
        if layout not in LAYOUTS:
            raise ContractViolationError(f"unknown layout {layout!r}")
        self.spec = spec
        self.n_patches = int(n_patches)
        self.gamma = float(gamma)
        self.layout = layout
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        d, s = spec.dimensions, spec.unknowns
        f64 = dict(dtype=torch.float64, device=self.device)
        self.QIn = torch.empty(self.n_patches * spec.haloed_volumes * s, **f64)
        self.QOut = torch.empty(self.n_patches * spec.interior_volumes * s, **f64)
        self.cell_size = torch.ones(self.n_patches * d, **f64)
        self.dt = torch.zeros(self.n_patches, **f64)
        self.max_eigenvalue = torch.zeros(self.n_patches, **f64)
        # status[0]: non-physical flag; status[1], status[2..]: redo list (include/fvb200.h)
        self.status = torch.zeros(int(_lib.load().fvb_status_words(self.n_patches)), dtype=torch.int32,
                                  device=self.device)

    # -- construction / transfer ---------------------------------------------------------------
    @classmethod
    def from_host(cls, batch: PatchBatch, gamma: float, device=None, layout: str = "aos") -> "DeviceBatch":
        torch = _torch()
        db = cls(batch.spec, batch.n_patches, gamma, device, layout)
        with torch.cuda.device(db.device):
            src = torch.from_numpy(np.ascontiguousarray(batch.QIn, dtype=np.float64).reshape(-1))
            if layout == "aos":
                db.QIn.copy_(src)
            else:
                tmp = src.to(db.device)
                db.pack_from(tmp, interior=False)
            db.cell_size.copy_(torch.from_numpy(np.ascontiguousarray(batch.cell_size, dtype=np.float64).reshape(-1)))
            db.dt.copy_(torch.from_numpy(np.ascontiguousarray(batch.dt, dtype=np.float64)))
        return db

    def fvb_spec(self) -> _lib.FvbSpec:
        return _lib.spec(self.spec.dimensions, self.spec.volumes_per_axis, self.n_patches, self.gamma,
                         LAYOUTS[self.layout])

    def pack_from(self, aos_qin, interior: bool = False, stream=None):
        """Fill QIn (or QOut if interior) from an AoS device tensor via fvb_pack."""
        torch = _torch()
        dst = self.QOut if interior else self.QIn
        _lib.check(_lib.load().fvb_pack(ctypes.byref(self.fvb_spec()), _vp(aos_qin), _vp(dst), int(interior),
                                        _stream_handle(torch, stream)), "fvb_pack")

    def qout_aos(self, stream=None):
        """QOut in the reference's AoS order (unpacked on the device for SoA batches)."""
        torch = _torch()
        if self.layout == "aos":
            return self.QOut
        out = torch.empty_like(self.QOut)
        _lib.check(_lib.load().fvb_unpack(ctypes.byref(self.fvb_spec()), _vp(self.QOut), _vp(out), 1,
                                          _stream_handle(torch, stream)), "fvb_unpack")
        return out

    # -- compute --------------------------------------------------------------------------------
    def update(self, kernel="auto", stream=None, zero_status: bool = True, mode: str = "exact") -> None:
        """One Rusanov step, asynchronous on `stream` (torch's current stream by default)."""
        torch = _torch()
        _lib.check(_lib.load().fvb_update(
            ctypes.byref(self.fvb_spec()), _vp(self.QIn), _vp(self.QOut), _vp(self.cell_size), _vp(self.dt),
            _vp(self.max_eigenvalue), _vp(self.status), kernel_id(kernel, mode), int(zero_status),
            _stream_handle(torch, stream)), "fvb_update")

    def update_cfl(self, cfl: float, dx: float, gmax, dt_scalar=None, kernel="auto", stream=None,
                   mode: str = "exact") -> None:
        """update() plus the CFL step control in the same launches (fvb_update_cfl): gmax <- max
        wave speed of the batch; with dt_scalar, dt = (cfl*dx)/gmax into dt_scalar and self.dt."""
        torch = _torch()
        _lib.check(_lib.load().fvb_update_cfl(
            ctypes.byref(self.fvb_spec()), _vp(self.QIn), _vp(self.QOut), _vp(self.cell_size), _vp(self.dt),
            _vp(self.max_eigenvalue), _vp(self.status), kernel_id(kernel, mode), float(cfl), float(dx), _vp(gmax),
            _vp(dt_scalar) if dt_scalar is not None else None, int(dt_scalar is not None),
            _stream_handle(torch, stream)), "fvb_update_cfl")

    def update_range(self, p0: int, p1: int, kernel="auto", stream=None, mode: str = "exact") -> None:
        """The update of patches [p0, p1) only (a contiguous sub-batch: same buffers, offset
        pointers; the status flag accumulates, the redo list empties itself).
        run_simulation_sharded updates its boundary layers first with it, so their exchange
        overlaps the update of the interior layers."""
        torch = _torch()
        if not (0 <= p0 < p1 <= self.n_patches):
            raise ContractViolationError(f"patch range [{p0}, {p1}) outside the batch of {self.n_patches}")
        d, s = self.spec.dimensions, self.spec.unknowns
        V, I = self.spec.haloed_volumes, self.spec.interior_volumes
        sub = _lib.spec(d, self.spec.volumes_per_axis, p1 - p0, self.gamma, LAYOUTS[self.layout])
        if self.layout != "aos":
            raise ContractViolationError("update_range: AoS batches only")
        _lib.check(_lib.load().fvb_update(
            ctypes.byref(sub), _vp(self.QIn[p0 * V * s:]), _vp(self.QOut[p0 * I * s:]),
            _vp(self.cell_size[p0 * d:]), _vp(self.dt[p0:]), _vp(self.max_eigenvalue[p0:]), _vp(self.status),
            kernel_id(kernel, mode), 0, _stream_handle(torch, stream)), "fvb_update")

    def max_eig_prepass(self, stream=None) -> None:
        """Per-patch wave speed of QIn without an update (first-step dt)."""
        torch = _torch()
        self.max_eigenvalue.zero_()
        _lib.check(_lib.load().fvb_patch_max_eig(ctypes.byref(self.fvb_spec()), _vp(self.QIn),
                                                 _vp(self.max_eigenvalue), _vp(self.status),
                                                 _stream_handle(torch, stream)), "fvb_patch_max_eig")

    def nonphysical(self) -> bool:
        return bool(int(self.status[0].item()) != 0)

    def locate(self, stream=None) -> np.ndarray:
        """Per-(patch, box) diagnostics (n, 2d+1, 4) int64 -- the error path."""
        torch = _torch()
        nbox = 2 * self.spec.dimensions + 1
        info = torch.empty(self.n_patches * nbox * 4, dtype=torch.int64, device=self.device)
        _lib.check(_lib.load().fvb_locate(ctypes.byref(self.fvb_spec()), _vp(self.QIn), _vp(info),
                                          _stream_handle(torch, stream)), "fvb_locate")
        return info.cpu().numpy().reshape(self.n_patches, nbox, 4)

    def halo_project(self, grid_shape, periodic: bool = True, stream=None) -> None:
        """QIn <- halo projection of QOut over the patch grid (mesh.py:261-310), on the device."""
        from .mesh import check_grid

        torch = _torch()
        shape = check_grid(self.spec.dimensions, self.n_patches, grid_shape)
        g = (ctypes.c_int32 * 3)(*(list(shape) + [1] * (3 - len(shape))))
        _lib.check(_lib.load().fvb_halo_project(ctypes.byref(self.fvb_spec()), _vp(self.QOut), _vp(self.QIn), g,
                                                int(bool(periodic)), _stream_handle(torch, stream)),
                   "fvb_halo_project")

    def halo_project_totals(self, grid_shape, periodic: bool, out, scratch, stream=None) -> None:
        """halo_project, then out[u] <- totals of QOut (totals_into), fused into one pass where supported."""
        from .mesh import check_grid

        torch = _torch()
        shape = check_grid(self.spec.dimensions, self.n_patches, grid_shape)
        g = (ctypes.c_int32 * 3)(*(list(shape) + [1] * (3 - len(shape))))
        _lib.check(_lib.load().fvb_halo_project_totals(ctypes.byref(self.fvb_spec()), _vp(self.QOut), _vp(self.QIn),
                                                       g, int(bool(periodic)), _vp(scratch), _vp(out),
                                                       _stream_handle(torch, stream)), "fvb_halo_project_totals")

    def halo_project_window(self, window_grid, lo_layers: int, ghost_lo, ghost_hi, periodic_mask: int,
                            totals_out=None, scratch=None, stream=None) -> None:
        """QIn of this shard from its own QOut and the ghost layers of a sharded grid
        (fvb_halo_project_window; driver.ShardedGrid assembles the arguments)."""
        torch = _torch()
        g = (ctypes.c_int32 * 3)(*(list(window_grid) + [1] * (3 - len(window_grid))))
        _lib.check(_lib.load().fvb_halo_project_window(
            ctypes.byref(self.fvb_spec()), _vp(ghost_lo) if ghost_lo is not None else None, _vp(self.QOut),
            _vp(ghost_hi) if ghost_hi is not None else None, _vp(self.QIn), g, int(lo_layers), int(periodic_mask),
            _vp(scratch) if scratch is not None else None, _vp(totals_out) if totals_out is not None else None,
            _stream_handle(torch, stream)), "fvb_halo_project_window")

    def totals_scratch(self):
        """Device scratch for totals_into (fvb_totals_scratch_bytes)."""
        torch = _torch()
        L = _lib.load()
        return torch.empty(L.fvb_totals_scratch_bytes(ctypes.byref(self.fvb_spec())) // 8, dtype=torch.float64,
                           device=self.device)

    def totals_into(self, out, scratch, stream=None) -> None:
        """out[u] <- sum of unknown u of QOut over all interior volumes; asynchronous, no host sync."""
        torch = _torch()
        _lib.check(_lib.load().fvb_totals(ctypes.byref(self.fvb_spec()), _vp(self.QOut), _vp(scratch), _vp(out),
                                          _stream_handle(torch, stream)), "fvb_totals")

    def totals(self, stream=None) -> np.ndarray:
        """Per-unknown sums of QOut over all interior volumes (conservation diagnostics)."""
        torch = _torch()
        out = torch.empty(self.spec.unknowns, dtype=torch.float64, device=self.device)
        self.totals_into(out, self.totals_scratch(), stream)
        return out.cpu().numpy()

    def to_host(self, batch: PatchBatch) -> None:
        """Copy QOut (AoS) and max_eigenvalue back into a host PatchBatch."""
        batch.QOut.reshape(-1)[...] = self.qout_aos().cpu().numpy()
        batch.max_eigenvalue[...] = self.max_eigenvalue.cpu().numpy()


# --- host-buffer path -----------------------------------------------------------------------------

_tls = threading.local()


def _workspace(torch, device, nbytes: int):
    """Per-thread, per-device workspace and stream (concurrent calls on disjoint batches are legal)."""
    cache = getattr(_tls, "cache", None)
    if cache is None:
        cache = _tls.cache = {}
    key = device.index
    ws, stream = cache.get(key, (None, None))
    if ws is None or ws.numel() < nbytes:
        ws = torch.empty(nbytes, dtype=torch.uint8, device=device)
    if stream is None:
        stream = torch.cuda.Stream(device=device)
    cache[key] = (ws, stream)
    return ws, stream


def _host_stage(torch, name: str, like: np.ndarray) -> np.ndarray:
    """Per-thread page-locked staging array for a small per-patch host array (cell_size, dt,
    max_eigenvalue): pageable sources would turn each chunk's tiny copies into synchronous,
    driver-staged transfers that stall the pipeline."""
    cache = getattr(_tls, "stage", None)
    if cache is None:
        cache = _tls.stage = {}
    buf = cache.get(name)
    if buf is None or buf.numel() < like.size:
        buf = torch.empty(max(like.size, 1024), dtype=torch.float64, pin_memory=True)
        cache[name] = buf
    return buf.numpy()[:like.size].reshape(like.shape)


def default_chunk(spec: PatchSpec, n: int, pipeline_chunks: int | None = None) -> int:
    """Host-pipeline chunk: at most 256 MB of device buffers per set, and about
    `pipeline_chunks` (default 32) chunks per call so the unoverlapped first H2D /
    last D2H (pipeline fill and drain) stay a small fraction of the transfer."""
    per_patch = (spec.haloed_volumes + spec.interior_volumes) * spec.unknowns * 8
    by_bytes = max(1, (256 << 20) // per_patch)
    k = int(pipeline_chunks or 32)
    by_pipeline = max(1, -(-n // k))
    floor = max(16, -(-(4 << 20) // per_patch))   # >= 4 MB per chunk: small batches are not worth pipelining
    return int(max(1, min(n, by_bytes, max(by_pipeline, min(n, floor)))))


# Page-locking of caller arrays (drop-in path).  Pageable host arrays make every H2D / D2H a
# driver-staged synchronous copy: the C3 drop-in call takes 131 ms from pageable numpy arrays
# against 19.6 ms from page-locked ones.  The first call on an array registers its memory
# (cudaHostRegister, ~25 ms per GB) and keeps it registered while the array lives, so a
# batch that is stepped repeatedly -- the reference's usage -- runs at pinned speed from the
# second call on.  Set `device.AUTO_PIN = False` to disable it.
AUTO_PIN = True
_PINNED: dict[int, int] = {}        # registered start address -> bytes
_PIN_LOCK = threading.Lock()


def _owner(a: np.ndarray):
    while isinstance(a.base, np.ndarray):
        a = a.base
    return a


def _ensure_pinned(arrays) -> None:
    if not AUTO_PIN:
        return
    import weakref

    L = _lib.load()
    for a in arrays:
        if a.nbytes < (1 << 20):          # small arrays: not worth a registration
            continue
        ptr = a.__array_interface__["data"][0]
        with _PIN_LOCK:
            if _PINNED.get(ptr, 0) >= a.nbytes:
                continue
            if L.fvb_host_pin(ctypes.c_void_p(ptr), ctypes.c_size_t(a.nbytes)) != _lib.FVB_OK:
                continue                     # already page-locked (torch pinned) or cannot pin: as is
            _PINNED[ptr] = a.nbytes

        def _release(p=ptr):
            with _PIN_LOCK:
                if _PINNED.pop(p, None) is not None:
                    try:
                        _lib.load().fvb_host_unpin(ctypes.c_void_p(p))
                    except Exception:  # pragma: no cover - interpreter shutdown
                        pass

        weakref.finalize(_owner(a), _release)


def update_host(batch: PatchBatch, gamma: float, device=None, kernel="auto", chunk_patches: int | None = None,
                mode: str = "exact"):
    """fvb_update_host on the batch's numpy arrays.  Returns the C-ABI code (0 or FVB_ERR_NONPHYSICAL)."""
    torch = _torch()
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    spec = batch.spec
    n = batch.n_patches
    chunk = int(chunk_patches or default_chunk(spec, n))
    fs = _lib.spec(spec.dimensions, spec.volumes_per_axis, n, gamma, 0)
    L = _lib.load()
    need = L.fvb_update_host_workspace(ctypes.byref(fs), chunk)
    arrays = []
    for name in ("QIn", "QOut", "cell_size", "dt", "max_eigenvalue"):
        a = getattr(batch, name)
        if a.dtype != np.float64 or not a.flags.c_contiguous:
            raise ContractViolationError(f"batch.{name} must be a C-contiguous float64 array")
        arrays.append(a)
    with torch.cuda.device(dev):
        _ensure_pinned(arrays[:2])                       # QIn, QOut: registered in place
        cs = _host_stage(torch, "cell_size", batch.cell_size)
        dts = _host_stage(torch, "dt", batch.dt)
        me = _host_stage(torch, "max_eigenvalue", batch.max_eigenvalue)
        np.copyto(cs, batch.cell_size)
        np.copyto(dts, batch.dt)
        ws, stream = _workspace(torch, dev, need)
        rc = L.fvb_update_host(ctypes.byref(fs), _hp(batch.QIn), _hp(batch.QOut), _hp(cs), _hp(dts), _hp(me),
                               _vp(ws), ctypes.c_size_t(ws.numel()), chunk, kernel_id(kernel, mode),
                               ctypes.c_void_p(stream.cuda_stream))
        np.copyto(batch.max_eigenvalue, me)   # fvb_update_host returns after its last D2H
    if rc not in (_lib.FVB_OK, _lib.FVB_ERR_NONPHYSICAL):
        _lib.check(rc, "fvb_update_host")
    return rc


def locate_host(batch: PatchBatch, gamma: float, device=None, chunk_patches: int | None = None) -> np.ndarray:
    """fvb_locate over a host batch, chunk by chunk (error path only)."""
    torch = _torch()
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    spec = batch.spec
    n = batch.n_patches
    d = spec.dimensions
    nbox = 2 * d + 1
    chunk = int(chunk_patches or default_chunk(spec, n))
    out = np.empty((n, nbox, 4), dtype=np.int64)
    L = _lib.load()
    with torch.cuda.device(dev):
        for p0 in range(0, n, chunk):
            p1 = min(n, p0 + chunk)
            q = torch.from_numpy(np.ascontiguousarray(batch.QIn[p0:p1]).reshape(-1)).to(dev)
            info = torch.empty((p1 - p0) * nbox * 4, dtype=torch.int64, device=dev)
            fs = _lib.spec(d, spec.volumes_per_axis, p1 - p0, gamma, 0)
            _lib.check(L.fvb_locate(ctypes.byref(fs), _vp(q), _vp(info),
                                    _stream_handle(torch, None)), "fvb_locate")
            out[p0:p1] = info.cpu().numpy().reshape(p1 - p0, nbox, 4)
    return out


def halo_project_host(batch: PatchBatch, grid_shape, periodic: bool, device=None) -> None:
    """mesh.halo_project on host arrays through the device kernel (AoS both ways)."""
    torch = _torch()
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    spec = batch.spec
    with torch.cuda.device(dev):
        qout = torch.from_numpy(np.ascontiguousarray(batch.QOut, dtype=np.float64).reshape(-1)).to(dev)
        qin = torch.empty(batch.n_patches * spec.haloed_volumes * spec.unknowns, dtype=torch.float64, device=dev)
        fs = _lib.spec(spec.dimensions, spec.volumes_per_axis, batch.n_patches, 1.4, 0, unknowns=spec.unknowns)
        g = (ctypes.c_int32 * 3)(*(list(grid_shape) + [1] * (3 - len(grid_shape))))
        _lib.check(_lib.load().fvb_halo_project(ctypes.byref(fs), _vp(qout), _vp(qin), g, int(bool(periodic)),
                                                _stream_handle(torch, None)), "fvb_halo_project")
        batch.QIn.reshape(-1)[...] = qin.cpu().numpy()


def probe(dim: int, gamma: float, states: np.ndarray):
    """(lam (n,d), flux (n,d,s), pressure (n,), bad (n,)) of AoS states, on the device."""
    torch = _torch()
    n = states.shape[0]
    s = dim + 2
    dev = torch.device("cuda", torch.cuda.current_device())
    q = torch.from_numpy(np.ascontiguousarray(states, dtype=np.float64).reshape(-1)).to(dev)
    lam = torch.empty(n * dim, dtype=torch.float64, device=dev)
    flux = torch.empty(n * dim * s, dtype=torch.float64, device=dev)
    pres = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    bad = torch.zeros(max(n, 1), dtype=torch.uint8, device=dev)
    _lib.check(_lib.load().fvb_probe(dim, gamma, _vp(q), n, _vp(lam), _vp(flux), _vp(pres), _vp(bad),
                                     _stream_handle(torch, None)), "fvb_probe")
    return (lam.cpu().numpy().reshape(n, dim), flux.cpu().numpy().reshape(n, dim, s),
            pres.cpu().numpy()[:n], bad.cpu().numpy()[:n])
