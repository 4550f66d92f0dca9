"""Multi-step / multi-GPU driver: the CFL step around the fused patch update.

SPEC.md:446-449 (run_simulation, no code in the reference) fixes the global
time step as dt = cflFactor * dx / max_patches maxEigenvalue, using the
previous step's per-patch maxima (a wave-speed pre-pass for the first step,
SPEC.md:467).  One process drives one GPU (torch.distributed, NCCL over
NVLink); patches are sharded contiguously across ranks, and the only
exchange of the step is one 8-byte MAX all-reduce of the wave speed.

Per step, entirely on the device and asynchronous on one stream:

    fvb_update            fused Rusanov update of the local shard
    fvb_reduce_dt(do_dt=0) local max of max_eigenvalue -> gmax (1 double)
    all_reduce(gmax, MAX)  NCCL, only when world_size > 1
    fvb_set_dt             dt = (cfl*dx)/gmax broadcast into the shard's dt[]

A multi-step run over a sharded grid (run_simulation_sharded) adds the halo
exchange: each rank owns whole layers of the patch grid along its slowest axis
and swaps one boundary layer of interior QOut with each neighbour (NCCL
send/recv over NVLink), then rebuilds its QIn from its own layers and the two
ghost layers (fvb_halo_project_window), bit-identical to the single-GPU
halo_project of the whole grid.
"""

from __future__ import annotations

import ctypes

from . import _lib
from .device import DeviceBatch, _stream_handle, _torch, _vp


def allreduce_max_(t, group=None):
    """In-place MAX all-reduce of the wave speed across ranks (the step's only exchange).

    NCCL over NVLink on the GPU ranks; any backend works (the CPU tests use gloo).
    A no-op for a single process."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t


def shard_bounds(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous patch range of a rank (preserves the global patch order)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


class CflStepper:
    """Device-resident step loop for one shard: update -> local max wave speed ->
    (NCCL MAX all-reduce) -> dt, every step enqueued without a host synchronisation.

    The redo list of the fused kernels empties itself (fvb_status_words), the max
    reduction rides on the update kernel (a running max its CTAs fold into; the last one
    writes gmax and dt_scalar) and the redo pass broadcasts dt (fvb_update_cfl), so a step
    is two kernels and no memset on one GPU for any batch size; on N GPUs the local max,
    the all-reduce and fvb_set_dt.
    graph=True captures that step once in a CUDA graph and replays it, which removes the
    per-launch host cost (ctypes + driver) from small-shard strong scaling."""

    def __init__(self, db: DeviceBatch, cfl: float = 0.4, dx: float | None = None, group=None,
                 kernel="auto", stream=None, mode: str = "exact", graph: bool = False, local: bool = False):
        torch = _torch()
        self.db = db
        self.cfl = float(cfl)
        self.dx = float(dx) if dx is not None else float(db.cell_size[0].item()) / db.spec.volumes_per_axis
        self.group = group
        self.kernel = kernel
        self.mode = mode
        self.stream = stream
        self.use_graph = bool(graph)
        self._graph = None
        self.gmax = torch.zeros(1, dtype=torch.float64, device=db.device)
        self.dt_scalar = torch.zeros(1, dtype=torch.float64, device=db.device)
        import torch.distributed as dist

        # local: this batch is the whole problem (run_simulation), even inside a multi-rank job
        self._dist = dist if (not local and dist.is_available() and dist.is_initialized()) else None

    def _multi(self) -> bool:
        return self._dist is not None and self._dist.get_world_size(self.group) > 1

    def reduce_dt(self, stream=None) -> None:
        torch = _torch()
        L = _lib.load()
        st = _stream_handle(torch, stream if stream is not None else self.stream)
        if not self._multi():
            _lib.check(L.fvb_reduce_dt(_vp(self.db.max_eigenvalue), self.db.n_patches, self.cfl, self.dx,
                                       _vp(self.gmax), _vp(self.dt_scalar), _vp(self.db.dt), 1, st), "fvb_reduce_dt")
            return
        _lib.check(L.fvb_reduce_dt(_vp(self.db.max_eigenvalue), self.db.n_patches, self.cfl, self.dx,
                                   _vp(self.gmax), None, None, 0, st), "fvb_reduce_dt")
        allreduce_max_(self.gmax, self.group)
        _lib.check(L.fvb_set_dt(_vp(self.gmax), self.cfl, self.dx, _vp(self.dt_scalar), _vp(self.db.dt),
                                self.db.n_patches, st), "fvb_set_dt")

    def prepass(self) -> None:
        """First-step dt from the initial wave speeds; clears the status words."""
        self.db.status.zero_()
        self.db.max_eig_prepass(stream=self.stream)
        self.reduce_dt()

    def _enqueue(self, stream, events=None) -> None:
        """One step: fvb_update_cfl (update + redo pass + local max, and on one GPU the dt in
        the same launches), then on N GPUs the all-reduce and fvb_set_dt.  events = (start,
        end) CUDA events recorded around the update launches only."""
        torch = _torch()
        st = stream   # None: torch's current stream (the capture stream inside a graph capture)
        rec = torch.cuda.current_stream() if st is None else st
        if events is not None:
            events[0].record(rec)
        if not self._multi():
            self.db.update_cfl(self.cfl, self.dx, self.gmax, self.dt_scalar, kernel=self.kernel, stream=st,
                               mode=self.mode)
            if events is not None:
                events[1].record(rec)
            return
        self.db.update_cfl(self.cfl, self.dx, self.gmax, None, kernel=self.kernel, stream=st, mode=self.mode)
        if events is not None:
            events[1].record(rec)
        allreduce_max_(self.gmax, self.group)
        _lib.check(_lib.load().fvb_set_dt(_vp(self.gmax), self.cfl, self.dx, _vp(self.dt_scalar), _vp(self.db.dt),
                                          self.db.n_patches, _stream_handle(torch, st)), "fvb_set_dt")

    def make_graph(self, steps: int, timing: bool = False):
        """Capture `steps` consecutive steps in one CUDA graph (replay with graph.replay()).
        With timing=True every step's update is bracketed by its own pair of (external)
        timing events, so the update kernels' durations can be read back after a replay:
        returns (graph, [(start, end), ...])."""
        torch = _torch()
        self._enqueue(self.stream)   # lazy library / NCCL setup outside the capture
        side = torch.cuda.Stream(device=self.db.device)
        side.wait_stream(self.stream if self.stream is not None else torch.cuda.current_stream())
        events = [(torch.cuda.Event(enable_timing=True, external=True),
                   torch.cuda.Event(enable_timing=True, external=True)) for _ in range(steps if timing else 0)]
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            for k in range(steps):
                if timing:
                    events[k][0].record()
                self._enqueue(None)
                if timing:
                    events[k][1].record()
        return g, events

    def step(self, events=None) -> None:
        """update -> local max -> (all-reduce) -> dt, enqueued on the stream (or replayed).
        events: (start, end) around the update launches (eager steps only)."""
        if not self.use_graph:
            self._enqueue(self.stream, events)
            return
        torch = _torch()
        if self._graph is None:
            self._enqueue(self.stream)   # one eager step: lazy library / NCCL setup before capture
            side = torch.cuda.Stream(device=self.db.device)
            side.wait_stream(self.stream if self.stream is not None else torch.cuda.current_stream())
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                self._enqueue(None)      # the capture stream is current inside the context
            self._graph = g
            return
        self._graph.replay()


def cfl_dt(db: DeviceBatch, cfl: float = 0.4, dx: float | None = None, group=None):
    """(global max wave speed, dt) from db.max_eigenvalue; synchronises."""
    s = CflStepper(db, cfl, dx, group)
    s.reduce_dt()
    return float(s.gmax.item()), float(s.dt_scalar.item())


# --- multi-step driver ----------------------------------------------------

CSV_HEADER = ("step", "t", "dt", "globalMaxEigenvalue", "totalMass", "totalMomentum", "totalEnergy")


class SimulationResult:
    """Per-step record of run_simulation: dt, global max wave speed and conserved totals."""

    def __init__(self, dim: int):
        self.dim = dim
        self.t, self.dt, self.max_eigenvalue, self.totals = [], [], [], []

    @property
    def steps(self) -> int:
        return len(self.dt)

    def rows(self):
        for k in range(len(self.totals)):
            tot = self.totals[k]
            yield (k, self.t[k], self.dt[k - 1] if k else 0.0, self.max_eigenvalue[k], float(tot[0]),
                   " ".join(repr(float(v)) for v in tot[1:1 + self.dim]), float(tot[-1]))

    def to_csv(self, path: str) -> None:
        with open(path, "w") as f:
            f.write(",".join(CSV_HEADER) + "\n")
            for r in self.rows():
                f.write(",".join(str(v) for v in r) + "\n")


def run_simulation(db: DeviceBatch, grid_shape, steps: int, cfl: float = 0.4, periodic: bool = True,
                   kernel="auto", dx: float | None = None, graph: bool | None = None,
                   direct: bool | None = None, diagnose: bool = True, mode: str = "exact") -> SimulationResult:
    """Device-resident time loop on one GPU.

    db.QOut holds the initial interior field of a logical uniform patch grid
    (patch index x-fastest).  Per step: dt = (cfl*dx)/max wave speed of the
    previous state (a pre-pass for the first step), the fused
    update of every patch, and the halo projection that rebuilds QIn from the
    new QOut (mesh.py:261-310).  Conserved totals are recorded per step.

    Every step is enqueued on the stream without a host synchronisation: dt,
    the global wave speed, the totals and the non-physical flag of each step
    land in device histories that are copied back once at the end (a
    NonPhysicalStateError then names the first failing step).

    graph=True captures one step (its ~12 kernel launches and copies) in a CUDA
    graph and replays it: the step writes its history entries through a device
    step counter, so every replay is the same graph.  Results are bit-identical
    to the eager loop (graph=False), which is also the fallback when capture is
    unavailable.

    mode: "exact" (bit-identical to the reference's update, the default) or "fast"
    (the 1e-12 parity bar; the shapes with a fast kernel run it).

    Errors: a non-physical state raises NonPhysicalStateError with the
    first failing step and -- with diagnose=True (the default, at the cost of one
    device copy of the initial field) -- its patch and haloed volume, found by
    replaying the run bit-identically up to that step and running the locator on its
    input; a step whose global maximum wave speed is <= 0 (dt = cfl*dx/0) raises
    TimeStepUnderflowError.

    Per step the device sees the update (fused kernel + redo pass), the dt reduction,
    the fused halo projection / totals and one fvb_step_record launch that writes the
    step's history entries and advances the device step counter (no PyTorch kernels).
    """
    import numpy as np

    torch = _torch()
    s = db.spec.unknowns
    dev = db.device
    f64 = dict(dtype=torch.float64, device=dev)
    tot_h = torch.empty((steps + 1, s), **f64)
    gmax_h = torch.empty(steps + 1, **f64)
    dt_h = torch.empty(steps + 1, **f64)      # dt_h[k] = the dt step k advances by
    flag_h = torch.zeros(steps + 1, dtype=torch.int32, device=dev)
    scratch = db.totals_scratch()

    init = db.QOut.clone() if diagnose and steps > 0 else None   # replayed on the error path only
    db.halo_project_totals(grid_shape, periodic, tot_h[0], scratch)
    db.status.zero_()
    stepper = CflStepper(db, cfl=cfl, dx=dx, kernel=kernel, local=True)
    stepper.prepass()
    gmax_h[0].copy_(stepper.gmax[0])
    dt_h[0].copy_(stepper.dt_scalar[0])
    k_t = torch.zeros(1, dtype=torch.int64, device=dev)    # device step counter (graph mode)
    from .device import MODES, kernel_id

    kernel_id("auto", mode)                                # validates the mode
    fast_flag = MODES[mode]                                # fvb_update_to_haloed flags (bit 0 unused here)
    tot_cur = torch.empty(s, **f64)

    # 2D AoS fast path: the update writes into the interior of the other haloed buffer,
    # then only its halo shell is filled (fvb_update_to_haloed / fvb_halo_shell)
    p = db.spec.volumes_per_axis
    direct_ok = db.spec.dimensions == 2 and db.layout == "aos" and 2 <= p <= 32 and kernel in ("auto", "fused")
    direct = direct_ok if direct is None else (bool(direct) and direct_ok)
    bufs = [db.QIn, torch.empty_like(db.QIn)] if direct else None
    gshape = (ctypes.c_int32 * 3)(*(list(grid_shape) + [1] * (3 - len(grid_shape))))

    def record():
        """flag_h[k] = status[0]; dt_h[k+1], gmax_h[k+1], tot_h[k+1]; k += 1 (one launch)."""
        _lib.check(_lib.load().fvb_step_record(
            _vp(k_t), _vp(stepper.dt_scalar), _vp(db.status), _vp(tot_cur), s, _vp(stepper.gmax), _vp(dt_h),
            _vp(flag_h), _vp(tot_h), _vp(gmax_h), _stream_handle(torch, None)), "fvb_step_record")

    def direct_step(k):
        L = _lib.load()
        fs = ctypes.byref(db.fvb_spec())
        st = _stream_handle(torch, None)
        src, dst = bufs[k % 2], bufs[(k + 1) % 2]
        _lib.check(L.fvb_update_to_haloed(fs, _vp(src), _vp(dst), _vp(db.cell_size), _vp(db.dt),
                                          _vp(db.max_eigenvalue), _vp(db.status), fast_flag, st),
                   "fvb_update_to_haloed")
        stepper.reduce_dt()
        _lib.check(L.fvb_halo_shell(fs, _vp(dst), gshape, int(bool(periodic)), st), "fvb_halo_shell")
        _lib.check(L.fvb_totals_haloed(fs, _vp(dst), _vp(scratch), _vp(tot_cur), st), "fvb_totals_haloed")
        record()

    def step_body():
        db.update(kernel=kernel, zero_status=False, mode=mode)   # status[0] accumulates; the redo list self-empties
        stepper.reduce_dt()                               # next step's dt from this step's wave speeds
        db.halo_project_totals(grid_shape, periodic, tot_cur, scratch)   # one pass over QOut
        record()

    g = None
    if graph is None:
        graph = steps >= 64
    if direct:
        for k in range(steps):
            direct_step(k)
        final = bufs[steps % 2]
        e = p + 2
        n = db.n_patches
        db.QOut.view(n, p, p, 4).copy_(final.view(n, e, e, 4)[:, 1:-1, 1:-1, :])
        if final is not db.QIn:
            db.QIn.copy_(final)
        graph = False
    elif graph and steps > 1:
        try:
            side = torch.cuda.Stream(device=dev)
            side.wait_stream(torch.cuda.current_stream(dev))
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side, capture_error_mode="thread_local"):
                step_body()
        except Exception:   # pragma: no cover - capture unavailable: eager loop
            g = None
            torch.cuda.synchronize(dev)
    if g is not None:
        for _ in range(steps):
            g.replay()
    elif not direct:
        for _ in range(steps):
            step_body()

    gm = gmax_h.cpu().numpy()
    kind, step = _first_failure(flag_h.cpu().numpy()[:steps], gm[:steps])
    if kind == "nonphysical" and init is not None:
        _raise_located(db, init, grid_shape, step, cfl, periodic, kernel, dx, mode)
    _raise_failure(kind, step, gm)
    res = SimulationResult(db.spec.dimensions)
    res.dt = [float(v) for v in dt_h.cpu().numpy()[:steps]]
    res.t = [0.0] + [float(v) for v in np.cumsum(res.dt)]
    res.max_eigenvalue = [float(v) for v in gmax_h.cpu().numpy()]
    res.totals = list(tot_h.cpu().numpy())
    return res


def _first_failure(flags, gmax_used):
    """(kind, step) of the first failing step, or (None, None).  Step k advances by the dt
    set from gmax_used[k] (an underflow there comes first), then its update raises the
    non-physical flag."""
    import numpy as np

    under = np.flatnonzero(gmax_used <= 0.0)
    bad = np.flatnonzero(flags)
    ku = int(under[0]) if under.size else None
    kb = int(bad[0]) if bad.size else None
    if ku is not None and (kb is None or ku <= kb):
        return "underflow", ku
    if kb is not None:
        return "nonphysical", kb
    return None, None


def _raise_failure(kind, step, gm) -> None:
    if kind == "underflow":
        from .errors import TimeStepUnderflowError
        raise TimeStepUnderflowError(f"dt underflow: global max eigenvalue {float(gm[step])!r} <= 0", step=step)
    if kind == "nonphysical":
        from .errors import NonPhysicalStateError
        raise NonPhysicalStateError("non-physical state during run_simulation", step=step)


def _raise_located(db, init, grid_shape, step, cfl, periodic, kernel, dx, mode="exact") -> None:
    """Replay the run (bit-identical, eager) from the saved initial field up to `step`, then
    locate the first inadmissible volume of that step's input (patch-wise order) and raise
    with step, patch and haloed volume."""
    from .errors import NonPhysicalStateError
    from .kernel import Ordering, box_volume, first_error

    db.QOut.copy_(init)
    if step > 0:
        run_simulation(db, grid_shape, step, cfl=cfl, periodic=periodic, kernel=kernel, dx=dx, graph=False,
                       diagnose=False, mode=mode)
    else:
        db.halo_project(grid_shape, periodic)
    hit = first_error(db.locate(), Ordering.PATCH_WISE, 1)
    if hit is None:  # pragma: no cover - the flag and the locator disagree
        raise NonPhysicalStateError("non-physical state during run_simulation", step=step)
    msg, patch, box, lin = hit
    d, p = db.spec.dimensions, db.spec.volumes_per_axis
    raise NonPhysicalStateError(msg, patch=patch, volume=box_volume(d, p, box, lin), step=step)


# --- sharded grid: ghost-layer exchange + windowed halo projection (multi-GPU run_simulation) ---------


def _neighbours(rank: int, world: int, periodic: bool):
    """(lower, upper) neighbour ranks along the sharded axis; None at a non-periodic edge."""
    lo = rank - 1 if rank > 0 else (world - 1 if periodic else None)
    hi = rank + 1 if rank < world - 1 else (0 if periodic else None)
    return lo, hi


def exchange_ghost_layers(own, layer_elems: int, ghost_lo, ghost_hi, rank: int, world: int, periodic: bool,
                          group=None) -> None:
    """Blocking form of exchange_ghost_layers_start (see there)."""
    for w in exchange_ghost_layers_start(own, layer_elems, ghost_lo, ghost_hi, rank, world, periodic, group):
        w.wait()


def exchange_ghost_layers_start(own, layer_elems: int, ghost_lo, ghost_hi, rank: int, world: int, periodic: bool,
                                group=None) -> list:
    """Fill ghost_lo with the lower neighbour's last layer and ghost_hi with the upper
    neighbour's first layer (flat tensors; `own` holds whole layers of layer_elems values).

    Point-to-point sends / receives (NCCL over NVLink on GPU ranks, any backend on CPU),
    issued in one fixed order on every rank -- [send last -> upper, send first -> lower,
    recv lower, recv upper] -- so that with two ranks, where the lower and upper
    neighbour are the same rank, the k-th message between a pair still lands in the
    right buffer.  A single periodic rank copies its own layers.  Returns the pending
    requests (wait on them before reading the ghosts)."""
    lo, hi = _neighbours(rank, world, periodic)
    first, last = own[:layer_elems], own[own.numel() - layer_elems:]
    if world == 1:
        if lo is not None:
            ghost_lo.copy_(last)
        if hi is not None:
            ghost_hi.copy_(first)
        return []
    import torch.distributed as dist

    # a backend without device point-to-point (gloo) moves device layers through host copies;
    # the returned waits then also copy the received layers to the device ghosts
    staged = own.is_cuda and dist.get_backend(group) != "nccl"
    send_last = last.cpu() if staged else last.contiguous()
    send_first = first.cpu() if staged else first.contiguous()
    recv_lo = torch_empty_like_host(ghost_lo) if (staged and lo is not None) else ghost_lo
    recv_hi = torch_empty_like_host(ghost_hi) if (staged and hi is not None) else ghost_hi
    ops = []
    if hi is not None:
        ops.append(dist.P2POp(dist.isend, send_last, hi, group))
    if lo is not None:
        ops.append(dist.P2POp(dist.isend, send_first, lo, group))
    if lo is not None:
        ops.append(dist.P2POp(dist.irecv, recv_lo, lo, group))
    if hi is not None:
        ops.append(dist.P2POp(dist.irecv, recv_hi, hi, group))
    works = dist.batch_isend_irecv(ops)   # the caller waits (after overlapping work, if any)
    if not staged:
        return works

    class _StagedWait:
        def wait(self_):
            for w in works:
                w.wait()
            if lo is not None:
                ghost_lo.copy_(recv_lo)
            if hi is not None:
                ghost_hi.copy_(recv_hi)

    return [_StagedWait()]


def torch_empty_like_host(t):
    """A host tensor shaped like device tensor t (the staging buffer of a gloo exchange)."""
    return _torch().empty(t.shape, dtype=t.dtype)


def shard_layout(grid_shape, rank: int, world: int, periodic: bool) -> dict:
    """Host-side geometry of one rank's shard (no device work): its layers [l0, l1) along
    the slowest axis, its patch range, whether it has a lower / upper ghost layer, the
    window grid the windowed halo projection sees and the per-axis wrap mask."""
    from .errors import ContractViolationError

    grid = tuple(int(g) for g in grid_shape)
    if grid[-1] < world:
        raise ContractViolationError(f"{world} ranks need at least {world} layers along the sharded "
                                     f"axis, grid {grid} has {grid[-1]}")
    layer = 1
    for g in grid[:-1]:
        layer *= g
    l0, l1 = shard_bounds(grid[-1], rank, world)
    lo, hi = _neighbours(rank, world, periodic)
    lo_layers, hi_layers = (1 if lo is not None else 0), (1 if hi is not None else 0)
    return {"layer": layer, "l0": l0, "l1": l1, "patch_lo": l0 * layer, "patch_hi": l1 * layer,
            "lower": lo, "upper": hi, "lo_layers": lo_layers,
            "window_grid": grid[:-1] + (lo_layers + (l1 - l0) + hi_layers,),
            # wrap along x / y (3D) or x (2D); the sharded axis wraps through the ghost layers
            "pmask": ((1 << (len(grid) - 1)) - 1) if periodic else 0}


class ShardedGrid:
    """One rank's shard of a logical uniform patch grid, split in whole layers along the
    slowest axis (z in 3D, y in 2D; patch index x-fastest as in halo_project).

    db is the rank's DeviceBatch (its own patches, global order); ghost_lo / ghost_hi
    hold the neighbours' boundary layers of interior QOut.  halo() exchanges them and
    rebuilds db.QIn exactly as halo_project of the whole grid would."""

    def __init__(self, spec, grid_shape, gamma: float, periodic: bool = True, rank: int | None = None,
                 world: int | None = None, group=None, device=None):
        import torch.distributed as dist

        torch = _torch()
        self.grid = tuple(int(g) for g in grid_shape)
        d = spec.dimensions
        if len(self.grid) != d:
            from .errors import ContractViolationError
            raise ContractViolationError(f"grid shape {self.grid} has {len(self.grid)} axes, expected {d}")
        on = dist.is_available() and dist.is_initialized()
        self.rank = rank if rank is not None else (dist.get_rank(group) if on else 0)
        self.world = world if world is not None else (dist.get_world_size(group) if on else 1)
        self.group, self.periodic = group, bool(periodic)
        lay = shard_layout(self.grid, self.rank, self.world, self.periodic)
        self.layer, self.l0, self.l1 = lay["layer"], lay["l0"], lay["l1"]
        self.patch_lo, self.patch_hi = lay["patch_lo"], lay["patch_hi"]
        self.db = DeviceBatch(spec, self.patch_hi - self.patch_lo, gamma, device)
        self.layer_elems = self.layer * spec.interior_volumes * spec.unknowns
        f64 = dict(dtype=torch.float64, device=self.db.device)
        self.ghost_lo = torch.empty(self.layer_elems, **f64) if lay["lower"] is not None else None
        self.ghost_hi = torch.empty(self.layer_elems, **f64) if lay["upper"] is not None else None
        self.lo_layers = lay["lo_layers"]
        self.window_grid = lay["window_grid"]
        self.pmask = lay["pmask"]

    def exchange(self) -> None:
        exchange_ghost_layers(self.db.QOut, self.layer_elems, self.ghost_lo, self.ghost_hi, self.rank, self.world,
                              self.periodic, self.group)

    def update_and_exchange(self, kernel="auto", mode: str = "exact") -> None:
        """The step's update with the ghost exchange overlapped: the two boundary layers are
        updated first and sent while the interior layers update (NCCL runs on its own stream,
        ordered after the boundary launches; the ghosts are awaited before the halo)."""
        own_layers = self.l1 - self.l0
        if self.world == 1 or own_layers < 3 or self.db.layout != "aos":
            self.db.update(kernel=kernel, zero_status=False, mode=mode)
            self.exchange()
            return
        L, n = self.layer, self.db.n_patches
        self.db.update_range(0, L, kernel, mode=mode)
        self.db.update_range(n - L, n, kernel, mode=mode)
        works = exchange_ghost_layers_start(self.db.QOut, self.layer_elems, self.ghost_lo, self.ghost_hi, self.rank,
                                            self.world, self.periodic, self.group)
        self.db.update_range(L, n - L, kernel, mode=mode)
        for w in works:
            w.wait()

    def halo_only(self, totals_out=None, scratch=None) -> None:
        """This shard's QIn from its own layers and the (already exchanged) ghosts."""
        self.db.halo_project_window(self.window_grid, self.lo_layers, self.ghost_lo, self.ghost_hi, self.pmask,
                                    totals_out, scratch)

    def halo(self, totals_out=None, scratch=None) -> None:
        """Ghost exchange, then this shard's QIn (and its local totals if totals_out is given)."""
        self.exchange()
        self.db.halo_project_window(self.window_grid, self.lo_layers, self.ghost_lo, self.ghost_hi, self.pmask,
                                    totals_out, scratch)


def run_simulation_sharded(sg: ShardedGrid, steps: int, cfl: float = 0.4, kernel="auto",
                           dx: float | None = None, mode: str = "exact") -> SimulationResult:
    """run_simulation over a grid sharded across ranks (one GPU each): the same step --
    dt from the global maximum wave speed (one MAX all-reduce), fused update of the own
    patches (the two boundary layers first, so their ghost-layer exchange overlaps the
    update of the interior layers), then the windowed halo projection.  Totals are
    summed over ranks in rank order.  With one rank it reproduces run_simulation bit for bit
    (the exchange is a local copy)."""
    import numpy as np
    import torch.distributed as dist

    torch = _torch()
    db = sg.db
    s = db.spec.unknowns
    f64 = dict(dtype=torch.float64, device=db.device)
    tot_h = torch.empty((steps + 1, s), **f64)
    gmax_h = torch.empty(steps + 1, **f64)
    dt_h = torch.empty(steps + 1, **f64)
    flag_h = torch.zeros(steps + 1, dtype=torch.int32, device=db.device)
    tot_cur = torch.empty(s, **f64)
    k_t = torch.zeros(1, dtype=torch.int64, device=db.device)
    scratch = db.totals_scratch()
    multi = sg.world > 1

    def halo_and_totals(out, exchanged=False):
        if exchanged:
            sg.halo_only(out, scratch)
        else:
            sg.halo(out, scratch)
        if multi:   # global totals: gather the shards' vectors, sum in rank order (deterministic)
            parts = [torch.empty(s, **f64) for _ in range(sg.world)]
            dist.all_gather(parts, out.contiguous(), group=sg.group)
            acc = parts[0].clone()
            for t in parts[1:]:
                acc += t
            out.copy_(acc)

    halo_and_totals(tot_h[0])
    db.status.zero_()
    stepper = CflStepper(db, cfl=cfl, dx=dx, kernel=kernel, group=sg.group)
    stepper.prepass()
    gmax_h[0].copy_(stepper.gmax[0])
    dt_h[0].copy_(stepper.dt_scalar[0])
    L = _lib.load()
    for _ in range(steps):
        sg.update_and_exchange(kernel, mode)  # boundary layers first, their exchange overlaps the rest
        stepper.reduce_dt()
        halo_and_totals(tot_cur, exchanged=True)
        _lib.check(L.fvb_step_record(_vp(k_t), _vp(stepper.dt_scalar), _vp(db.status), _vp(tot_cur), s,
                                     _vp(stepper.gmax), _vp(dt_h), _vp(flag_h), _vp(tot_h), _vp(gmax_h),
                                     _stream_handle(torch, None)), "fvb_step_record")

    flags = flag_h.clone()
    if multi:
        dist.all_reduce(flags, op=dist.ReduceOp.MAX, group=sg.group)
    gm = gmax_h.cpu().numpy()   # global after the all-reduce: the same on every rank
    _raise_failure(*_first_failure(flags.cpu().numpy()[:steps], gm[:steps]), gm)
    res = SimulationResult(db.spec.dimensions)
    res.dt = [float(v) for v in dt_h.cpu().numpy()[:steps]]
    res.t = [0.0] + [float(v) for v in np.cumsum(res.dt)]
    res.max_eigenvalue = [float(v) for v in gmax_h.cpu().numpy()]
    res.totals = [row for row in tot_h.cpu().numpy()]
    return res
