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
    """Device-resident step loop for one shard."""

    def __init__(self, db: DeviceBatch, cfl: float = 0.4, dx: float | None = None, group=None,
                 kernel="auto", stream=None):
        torch = _torch()
        self.db = db
        self.cfl = float(cfl)
        self.dx = float(dx) if dx is not None else float(db.cell_size[0].item()) / db.spec.volumes_per_axis
        self.group = group
        self.kernel = kernel
        self.stream = stream
        self.gmax = torch.zeros(1, dtype=torch.float64, device=db.device)
        self.dt_scalar = torch.zeros(1, dtype=torch.float64, device=db.device)
        import torch.distributed as dist

        self._dist = dist if (dist.is_available() and dist.is_initialized()) else None

    def reduce_dt(self) -> None:
        torch = _torch()
        L = _lib.load()
        st = _stream_handle(torch, self.stream)
        if self._dist is None or self._dist.get_world_size(self.group) == 1:
            _lib.check(L.fvb_reduce_dt(_vp(self.db.max_eigenvalue), self.db.n_patches, self.cfl, self.dx,
                                       _vp(self.gmax), _vp(self.dt_scalar), _vp(self.db.dt), 1, st), "fvb_reduce_dt")
            return
        _lib.check(L.fvb_reduce_dt(_vp(self.db.max_eigenvalue), self.db.n_patches, self.cfl, self.dx,
                                   _vp(self.gmax), None, None, 0, st), "fvb_reduce_dt")
        allreduce_max_(self.gmax, self.group)
        _lib.check(L.fvb_set_dt(_vp(self.gmax), self.cfl, self.dx, _vp(self.dt_scalar), _vp(self.db.dt),
                                self.db.n_patches, st), "fvb_set_dt")

    def prepass(self) -> None:
        """First-step dt from the initial wave speeds."""
        self.db.max_eig_prepass(stream=self.stream)
        self.reduce_dt()

    def step(self) -> None:
        """update -> local max -> (all-reduce) -> dt, all enqueued on the stream."""
        self.db.update(kernel=self.kernel, stream=self.stream)
        self.reduce_dt()


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
                   kernel="auto", dx: float | None = None) -> SimulationResult:
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
    """
    import numpy as np

    torch = _torch()
    s = db.spec.unknowns
    dev = db.device
    f64 = dict(dtype=torch.float64, device=dev)
    tot_h = torch.empty((steps + 1, s), **f64)
    gmax_h = torch.empty(steps + 1, **f64)
    dt_h = torch.empty(max(steps, 1), **f64)
    flag_h = torch.zeros(max(steps, 1), dtype=torch.int32, device=dev)
    scratch = db.totals_scratch()

    db.halo_project_totals(grid_shape, periodic, tot_h[0], scratch)
    db.status.zero_()
    stepper = CflStepper(db, cfl=cfl, dx=dx, kernel=kernel)
    stepper.prepass()
    gmax_h[0].copy_(stepper.gmax[0])
    for k in range(steps):
        dt_h[k].copy_(stepper.dt_scalar[0])   # the dt this step advances by
        db.status[1:2].zero_()                # redo count of this launch; status[0] accumulates
        db.update(kernel=kernel, zero_status=False)
        flag_h[k].copy_(db.status[0])
        stepper.reduce_dt()                   # next step's dt from this step's wave speeds
        db.halo_project_totals(grid_shape, periodic, tot_h[k + 1], scratch)   # one pass over QOut
        gmax_h[k + 1].copy_(stepper.gmax[0])

    flags = flag_h.cpu().numpy()[:steps]
    bad = np.flatnonzero(flags)
    if bad.size:
        from .errors import NonPhysicalStateError
        raise NonPhysicalStateError("non-physical state during run_simulation", step=int(bad[0]))
    res = SimulationResult(db.spec.dimensions)
    res.dt = [float(v) for v in dt_h.cpu().numpy()[:steps]]
    res.t = [0.0] + [float(v) for v in np.cumsum(res.dt)]
    res.max_eigenvalue = [float(v) for v in gmax_h.cpu().numpy()]
    res.totals = list(tot_h.cpu().numpy())
    return res
