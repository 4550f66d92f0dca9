"""GPU tests of the between-step path: device halo_project (mesh.py:261-310) and the
multi-step CFL driver -- conservation and constant-state properties."""

import json
import os

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, assert_bits_equal, load_golden

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2302_09005_b200 import device, driver, mesh, pde  # noqa: E402
from paper_2302_09005_b200.errors import ContractViolationError  # noqa: E402

with open(os.path.join(GOLDEN, "manifest.json")) as _f:
    HALO = json.load(_f)["halo_cases"]


@pytest.mark.parametrize("case", HALO, ids=lambda c: c["name"])
def test_halo_project_matches_reference(case):
    gold = load_golden(case["file"])
    b = gold.copy()
    b.QIn[...] = np.nan
    mesh.halo_project(b, case["grid"], case["periodic"])
    assert_bits_equal(b.QIn, gold.QIn, case["name"])
    db = device.DeviceBatch(gold.spec, gold.n_patches, 1.4, layout="soa")
    db.pack_from(torch.from_numpy(gold.QOut.reshape(-1).copy()).cuda(), interior=True)
    db.halo_project(case["grid"], case["periodic"])
    out = torch.empty_like(db.QIn)
    import ctypes
    from paper_2302_09005_b200 import _lib
    _lib.check(_lib.load().fvb_unpack(ctypes.byref(db.fvb_spec()), device._vp(db.QIn), device._vp(out), 0,
                                      device._stream_handle(torch, None)), "unpack")
    assert_bits_equal(out.cpu().numpy().reshape(gold.QIn.shape), gold.QIn, case["name"] + " soa")


HALO_GRIDS = [(3, 16, (4, 3, 2)), (2, 16, (8, 5)), (3, 4, (3, 3, 3)), (3, 5, (1, 2, 3)), (2, 3, (1, 1)),
              (2, 33, (2, 3)), (3, 2, (5, 1, 2)), (2, 17, (3, 7)), (3, 19, (2, 1, 2)), (2, 65, (2, 2)),
              (3, 32, (1, 2, 1))]


@pytest.mark.parametrize("dim,p,grid", HALO_GRIDS)
def test_halo_project_random_vs_oracle(dim, p, grid):
    n = int(np.prod(grid))
    b = mesh.make_patch_batch(mesh.PatchSpec(dim, p, dim + 2), n)
    b.QOut[...] = np.random.default_rng(n).standard_normal(b.QOut.shape)
    for periodic in (True, False):
        mesh.halo_project(b, grid, periodic)
        assert_bits_equal(b.QIn, oracle.halo_project(dim, p, b.QOut, grid, periodic), f"{grid} {periodic}")
    with pytest.raises(ContractViolationError):
        mesh.halo_project(b, grid[:-1], True)


@pytest.mark.parametrize("dim,p,s,grid", [(2, 4, 3, (2, 3)), (3, 1, 1, (2, 2, 2)), (3, 4, 1, (3, 1, 2)),
                                          (2, 16, 7, (4, 2)), (3, 5, 9, (2, 1, 2)), (2, 3, 1, (1, 1))])
def test_halo_project_any_unknown_count(dim, p, s, grid):
    """halo_project is data movement: any s (s != d + 2 used to overrun the buffers)."""
    n = int(np.prod(grid))
    b = mesh.make_patch_batch(mesh.PatchSpec(dim, p, s), n)
    b.QOut[...] = np.random.default_rng(s * 100 + n).standard_normal(b.QOut.shape)
    for periodic in (True, False):
        b.QIn[...] = np.nan
        mesh.halo_project(b, grid, periodic)
        assert_bits_equal(b.QIn, oracle.halo_project(dim, p, b.QOut, grid, periodic, s=s), f"s={s} {periodic}")


@pytest.mark.parametrize("dim,p,grid", [(3, 16, (4, 3, 2)), (3, 4, (3, 3, 3)), (3, 5, (1, 2, 3)), (2, 16, (8, 5)),
                                        (3, 32, (1, 2, 1))])
def test_halo_project_totals_fused(dim, p, grid):
    """fvb_halo_project_totals: QIn bit-identical to halo_project, totals equal to an exact
    (math.fsum) sum of QOut within fp64 summation error (the row-copy kernel sums in its own order)."""
    import math

    n = int(np.prod(grid))
    spec = mesh.PatchSpec(dim, p, dim + 2)
    b = mesh.make_patch_batch(spec, n)
    b.QOut[...] = np.random.default_rng(7 * n + p).uniform(0.5, 2.0, b.QOut.shape)
    for periodic in (True, False):
        db = device.DeviceBatch(spec, n, 1.4)
        db.QOut.copy_(torch.from_numpy(b.QOut.reshape(-1)))
        tot = torch.empty(dim + 2, dtype=torch.float64, device="cuda")
        db.halo_project_totals(grid, periodic, tot, db.totals_scratch())
        qin = db.QIn.cpu().numpy().reshape(b.QIn.shape)
        assert_bits_equal(qin, oracle.halo_project(dim, p, b.QOut, grid, periodic), f"{grid} {periodic}")
        q = b.QOut.reshape(-1, dim + 2)
        exact = np.array([math.fsum(q[:, u]) for u in range(dim + 2)])
        np.testing.assert_allclose(tot.cpu().numpy(), exact, rtol=1e-13, atol=0)
        np.testing.assert_allclose(db.totals(), exact, rtol=1e-13, atol=0)


def _db_with_field(dim, p, grid, qout):
    n = int(np.prod(grid))
    spec = mesh.PatchSpec(dim, p, dim + 2)
    b = mesh.make_patch_batch(spec, n)
    b.QOut[...] = qout
    db = device.DeviceBatch(spec, n, 1.4)
    db.QOut.copy_(torch.from_numpy(b.QOut.reshape(-1)))
    return db


def test_run_simulation_conserves_totals():
    """on a periodic grid the conserved totals drift <= 1e-12 relative per 100 steps."""
    dim, p, grid = 2, 16, (4, 4)
    n = int(np.prod(grid))
    q = oracle.synthetic_qin(dim, p, n, seed=4).reshape(n, (p + 2) ** dim, dim + 2)
    interior = q.reshape(n, p + 2, p + 2, dim + 2)[:, 1:-1, 1:-1, :].reshape(n, -1)
    db = _db_with_field(dim, p, grid, interior)
    res = driver.run_simulation(db, grid, steps=100, cfl=0.4, periodic=True)
    tot = np.asarray(res.totals)
    scale = np.abs(tot[0]).max()
    drift = np.abs(tot[-1] - tot[0]) / np.maximum(np.abs(tot[0]), scale * 1e-3)
    assert res.steps == 100 and all(dt > 0 for dt in res.dt)
    assert drift.max() <= 1e-12, drift


def test_run_simulation_constant_state_is_fixed_point():
    """SPEC.md run_simulation example: a constant state stays bitwise constant; dt stays constant."""
    dim, p, grid = 3, 16, (2, 2, 2)
    n = int(np.prod(grid))
    state = pde.euler_state(1.2, [0.3, -0.1, 0.2], 0.8)
    field = np.tile(state, (n, p ** dim))
    db = _db_with_field(dim, p, grid, field)
    res = driver.run_simulation(db, grid, steps=10, cfl=0.3, periodic=True)
    assert_bits_equal(db.QOut.cpu().numpy().reshape(n, -1), field, "constant field after 10 steps")
    assert len(set(res.dt)) == 1


def _moving_contact(g, p, t):
    """rho = 1 + 0.2 sin(2 pi (x - t)), u = (1, 0), p = 1 on [0,1]^2, periodic; cell-centre values."""
    n_ax = g * p
    xc = (np.arange(n_ax) + 0.5) / n_ax
    rho = 1.0 + 0.2 * np.sin(2.0 * np.pi * (xc - t))
    return np.broadcast_to(rho[None, :], (n_ax, n_ax))   # [y, x]


def _field_from_global(g, p, glob):
    """Global [y, x, u] field -> interior QOut rows of a g x g patch grid (patch index x-fastest)."""
    s = glob.shape[-1]
    return glob.reshape(g, p, g, p, s).transpose(0, 2, 1, 3, 4).reshape(g * g, p * p * s)


def test_run_simulation_convergence_order():
    """SPEC.md:562 (acceptance criterion 5): moving contact, L1 density error at 30 / 90 / 270
    volumes per axis decreases with observed order >= 0.7 (first-order Rusanov)."""
    p, gamma, t_end = 10, 1.4, 0.05
    errors = []
    for g in (3, 9, 27):
        n_ax = g * p
        rho = _moving_contact(g, p, 0.0)
        q = np.zeros((n_ax, n_ax, 4))
        q[..., 0] = rho
        q[..., 1] = rho * 1.0
        q[..., 3] = 1.0 / (gamma - 1.0) + 0.5 * rho * 1.0
        db = _db_with_field(2, p, (g, g), _field_from_global(g, p, q))
        db.cell_size.fill_(1.0 / g)
        dx = 1.0 / n_ax
        steps = int(np.ceil(t_end / (0.4 * dx / (1.0 + np.sqrt(gamma / 0.8)))))
        res = driver.run_simulation(db, (g, g), steps=steps, cfl=0.4, periodic=True)
        out = db.QOut.cpu().numpy().reshape(g, g, p, p, 4).transpose(0, 2, 1, 3, 4).reshape(n_ax, n_ax, 4)
        exact = _moving_contact(g, p, res.t[-1])
        errors.append(float(np.abs(out[..., 0] - exact).mean()))
    orders = [np.log(errors[k] / errors[k + 1]) / np.log(3.0) for k in range(2)]
    assert min(orders) >= 0.7, (errors, orders)


@pytest.mark.parametrize("dim,p,grid", [(3, 16, (3, 2, 5)), (3, 5, (2, 3, 4)), (2, 16, (4, 7)), (2, 17, (3, 3)),
                                        (3, 4, (2, 2, 1))])
@pytest.mark.parametrize("world", [1, 2, 3])
def test_sharded_halo_window_matches_global(dim, p, grid, world):
    """fvb_halo_project_window on each shard of a grid split in whole layers along its slowest
    axis, ghosts filled with the neighbours' boundary layers, equals the single-GPU halo
    projection of the whole grid bit for bit (periodic and zero-gradient); the shards' totals
    sum to the whole grid's."""
    import math

    n = int(np.prod(grid))
    spec = mesh.PatchSpec(dim, p, dim + 2)
    if grid[-1] < world:   # every rank must own a layer
        with pytest.raises(ContractViolationError):
            driver.ShardedGrid(spec, grid, 1.4, True, rank=0, world=world)
        return
    qout = np.random.default_rng(n + 31 * p + world).uniform(0.5, 2.0, (n, p ** dim * (dim + 2)))
    layer = n // grid[-1]
    le = layer * p ** dim * (dim + 2)
    for periodic in (True, False):
        ref = oracle.halo_project(dim, p, qout, grid, periodic).reshape(n, -1)
        tot_sum = np.zeros(dim + 2)
        for rank in range(world):
            sg = driver.ShardedGrid(spec, grid, 1.4, periodic, rank=rank, world=world)
            sg.db.QOut.copy_(torch.from_numpy(qout[sg.patch_lo:sg.patch_hi].reshape(-1).copy()))
            flat = qout.reshape(-1)
            if sg.ghost_lo is not None:   # the lower neighbour's last layer (wrapping)
                z = (sg.l0 - 1) % grid[-1]
                sg.ghost_lo.copy_(torch.from_numpy(flat[z * le:(z + 1) * le].copy()))
            if sg.ghost_hi is not None:
                z = sg.l1 % grid[-1]
                sg.ghost_hi.copy_(torch.from_numpy(flat[z * le:(z + 1) * le].copy()))
            tot = torch.empty(dim + 2, dtype=torch.float64, device="cuda")
            sg.db.halo_project_window(sg.window_grid, sg.lo_layers, sg.ghost_lo, sg.ghost_hi, sg.pmask, tot,
                                      sg.db.totals_scratch())
            got = sg.db.QIn.cpu().numpy().reshape(sg.db.n_patches, -1)
            assert_bits_equal(got, ref[sg.patch_lo:sg.patch_hi], f"rank {rank}/{world} periodic={periodic}")
            tot_sum += tot.cpu().numpy()
        exact = np.array([math.fsum(qout.reshape(-1, dim + 2)[:, u]) for u in range(dim + 2)])
        np.testing.assert_allclose(tot_sum, exact, rtol=1e-13)


@pytest.mark.parametrize("dim,p,grid", [(3, 16, (2, 2, 3)), (2, 16, (4, 5))])
@pytest.mark.parametrize("periodic", [True, False])
def test_run_simulation_sharded_single_rank_matches(dim, p, grid, periodic):
    """run_simulation_sharded with one rank (the exchange is a local copy) reproduces
    run_simulation bit for bit: QOut and the dt history (totals to summation-order rounding:
    2D run_simulation sums them in a separate pass)."""
    n = int(np.prod(grid))
    q = oracle.synthetic_qin(dim, p, n, seed=12).reshape(n, (p + 2) ** dim, dim + 2)
    sl = (slice(None),) + (slice(1, -1),) * dim + (slice(None),)
    interior = q.reshape((n,) + (p + 2,) * dim + (dim + 2,))[sl].reshape(n, -1)
    db = _db_with_field(dim, p, grid, interior)
    ref = driver.run_simulation(db, grid, steps=6, cfl=0.4, periodic=periodic)
    sg = driver.ShardedGrid(mesh.PatchSpec(dim, p, dim + 2), grid, 1.4, periodic, rank=0, world=1)
    sg.db.QOut.copy_(torch.from_numpy(interior.reshape(-1).copy()))
    res = driver.run_simulation_sharded(sg, steps=6, cfl=0.4)
    assert_bits_equal(sg.db.QOut.cpu().numpy(), db.QOut.cpu().numpy(), "QOut after 6 steps")
    assert res.dt == ref.dt
    np.testing.assert_allclose(np.asarray(res.totals), np.asarray(ref.totals), rtol=1e-13)


@pytest.mark.parametrize("dim,p,grid", [(3, 16, (2, 2, 3)), (2, 17, (3, 4)), (3, 4, (3, 3, 3))])
def test_run_simulation_graph_matches_eager(dim, p, grid):
    """run_simulation's CUDA-graph step replay gives the eager loop's field and histories bit for bit."""
    n = int(np.prod(grid))
    q = oracle.synthetic_qin(dim, p, n, seed=21).reshape(n, (p + 2) ** dim, dim + 2)
    sl = (slice(None),) + (slice(1, -1),) * dim + (slice(None),)
    interior = q.reshape((n,) + (p + 2,) * dim + (dim + 2,))[sl].reshape(n, -1)
    dbs, res = [], []
    for graph in (False, True):
        db = _db_with_field(dim, p, grid, interior)
        res.append(driver.run_simulation(db, grid, steps=7, cfl=0.4, periodic=True, graph=graph))
        dbs.append(db)
    assert_bits_equal(dbs[1].QOut.cpu().numpy(), dbs[0].QOut.cpu().numpy(), "QOut")
    assert res[1].dt == res[0].dt and res[1].max_eigenvalue == res[0].max_eigenvalue
    assert_bits_equal(np.asarray(res[1].totals), np.asarray(res[0].totals), "totals")


@pytest.mark.parametrize("p,grid,periodic", [(16, (4, 5), True), (16, (3, 3), False), (17, (3, 4), True),
                                             (5, (6, 2), False), (32, (2, 2), True), (3, (1, 1), True)])
def test_run_simulation_2d_direct_path_matches(p, grid, periodic):
    """2D run_simulation's fast path (update straight into the next haloed batch + halo shell)
    gives the classic path's field, QIn, dt history and wave speeds bit for bit."""
    dim = 2
    n = int(np.prod(grid))
    q = oracle.synthetic_qin(dim, p, n, seed=33 + p).reshape(n, p + 2, p + 2, dim + 2)
    interior = q[:, 1:-1, 1:-1, :].reshape(n, -1)
    out = {}
    for direct in (False, True):
        db = _db_with_field(dim, p, grid, interior)
        res = driver.run_simulation(db, grid, steps=5, cfl=0.4, periodic=periodic, direct=direct)
        out[direct] = (db.QOut.cpu().numpy(), db.QIn.cpu().numpy(), res)
    assert_bits_equal(out[True][0], out[False][0], "QOut")
    assert_bits_equal(out[True][1], out[False][1], "QIn (final halo)")
    assert out[True][2].dt == out[False][2].dt and out[True][2].max_eigenvalue == out[False][2].max_eigenvalue
    np.testing.assert_allclose(np.asarray(out[True][2].totals), np.asarray(out[False][2].totals), rtol=1e-13)


@pytest.mark.parametrize("dim,p,grid", [(3, 16, (2, 2, 5)), (2, 16, (3, 7)), (3, 4, (2, 3, 4))])
def test_update_range_split_matches_whole(dim, p, grid, monkeypatch):
    """ShardedGrid.update_and_exchange's split update (first layer, last layer, then the
    interior layers, the exchange started in between) equals one whole update bit for bit."""
    n = int(np.prod(grid))
    spec = mesh.PatchSpec(dim, p, dim + 2)
    qin = oracle.synthetic_qin(dim, p, n, seed=77)
    b = mesh.make_patch_batch(spec, n)
    b.QIn[...] = qin
    b.dt[...] = 0.4 / p / 3.4
    whole = device.DeviceBatch.from_host(b, 1.4)
    whole.update()
    calls = []
    monkeypatch.setattr(driver, "exchange_ghost_layers_start", lambda *a, **k: calls.append(1) or [])
    sg = driver.ShardedGrid(spec, grid, 1.4, True, rank=1, world=3)   # a middle rank: both ghosts
    lay = driver.shard_layout(grid, 1, 3, True)
    sg.db.QIn.copy_(whole.QIn.view(n, -1)[lay["patch_lo"]:lay["patch_hi"]].reshape(-1))
    sg.db.dt.copy_(whole.dt[lay["patch_lo"]:lay["patch_hi"]])
    sg.db.status.zero_()
    sg.update_and_exchange()
    torch.cuda.synchronize()
    assert calls == [1]
    lo, hi = lay["patch_lo"], lay["patch_hi"]
    assert_bits_equal(sg.db.QOut.cpu().numpy(), whole.QOut.view(n, -1)[lo:hi].reshape(-1).cpu().numpy(), "QOut")
    assert_bits_equal(sg.db.max_eigenvalue.cpu().numpy(), whole.max_eigenvalue[lo:hi].cpu().numpy(), "max_eig")


@pytest.mark.parametrize("dim,p,n,kernel,negzero,layout", [
    (3, 16, 300, "auto", False, "aos"), (3, 16, 40, "auto", True, "aos"), (2, 16, 2000, "auto", False, "aos"),
    (3, 4, 20000, "auto", False, "aos"), (3, 4, 20000, "auto", True, "aos"), (2, 16, 20000, "auto", True, "aos"),
    (3, 7, 30, "generic", False, "aos"), (2, 5, 64, "auto", True, "aos"), (2, 16, 3000, "auto", True, "soa"),
    (3, 16, 60, "auto", False, "soa")])
@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_update_cfl_tail_matches_host(dim, p, n, kernel, negzero, layout, mode):
    """fvb_update_cfl: QOut / max_eig as fvb_update, gmax = max(max_eig) and dt = (cfl*dx)/gmax
    (fvb_set_dt's rounding) in every dt slot -- via the fused kernel's running max and the redo
    pass's broadcast (empty list), the redo pass's last CTA (queued patches), or the reduce
    kernels (generic kernel); every fused kernel family (3D p=16 fast / half, small-patch, 2D
    warp AoS, 2D block SoA), above and below 16,384 patches."""
    b = mesh.make_patch_batch(mesh.PatchSpec(dim, p, dim + 2), n)
    q = oracle.synthetic_qin(dim, p, n, seed=n + p).reshape(n, -1, dim + 2)
    if negzero:
        q[::3, ::7, 1] = -0.0      # leaves the range gate: those patches go through the redo list
    b.QIn[...] = q.reshape(n, -1)
    b.dt[...] = 0.4 * (1.0 / p) / 3.4
    ref_q, ref_l, st = oracle.update(dim, p, 1.4, b.QIn, b.cell_size, b.dt)
    assert st == 0
    db = device.DeviceBatch.from_host(b, 1.4, layout=layout)
    gmax = torch.zeros(1, dtype=torch.float64, device="cuda")
    dts = torch.zeros(1, dtype=torch.float64, device="cuda")
    for _ in range(2):   # twice: the redo list, the CTA counters and the running max reset themselves
        db.dt.fill_(b.dt[0])
        db.update_cfl(0.4, 1.0 / p, gmax, dts, kernel=kernel, mode=mode)
        torch.cuda.synchronize()
        st_words = db.status.cpu().numpy()
        assert st_words[1] == 0 and np.all(st_words[-6:] == 0), st_words[-6:]   # list, counters, running max
        out = mesh.make_patch_batch(b.spec, n)
        db.to_host(out)
        # fast kernels (3D p = 16, 2D p = 2..32, 3D p = 2, 4..8): 1e-12 parity, not bitwise
        fast16 = mode == "fast" and kernel == "auto" and layout == "aos" and (p == 16 or dim == 2 or
                                                                              p in (2, 4, 5, 6, 7, 8))
        if not fast16:
            assert_bits_equal(out.QOut, ref_q, "QOut")
            assert_bits_equal(out.max_eigenvalue, ref_l, "max_eig")
        else:
            assert np.max(np.abs(out.max_eigenvalue - ref_l) / ref_l) < 1e-14
        g = float(np.max(out.max_eigenvalue))   # the tail reduces the launch's own maxima
        assert gmax.item() == g
        dt = (0.4 * (1.0 / p)) / g
        assert dts.item() == dt
        assert np.all(db.dt.cpu().numpy() == dt)


@pytest.mark.parametrize("mode", ["exact", "fast"])
@pytest.mark.parametrize("explicit_stream", [False, True])
def test_cfl_stepper_graph_equals_eager(mode, explicit_stream):
    """The captured step does the same work as the eager one -- also when the stepper was
    given an explicit stream (bench.py's usage; the capture must still record the launches)."""
    dim, p, n = 3, 16, 24
    b = mesh.make_patch_batch(mesh.PatchSpec(dim, p, dim + 2), n)
    b.QIn[...] = oracle.synthetic_qin(dim, p, n, seed=5)
    res = []
    for graph in (False, True):
        db = device.DeviceBatch.from_host(b, 1.4)
        db.QOut.fill_(-1.0)
        stream = torch.cuda.current_stream() if explicit_stream else None
        st = driver.CflStepper(db, cfl=0.4, mode=mode, graph=graph, stream=stream)
        st.prepass()
        dts = []
        for _ in range(4):   # the stepper re-reads the same QIn: every step is the same update
            st.step()
            dts.append(st.dt_scalar.item())
        res.append((db.QOut.cpu().numpy(), db.max_eigenvalue.cpu().numpy(), dts))
    assert not np.any(res[1][0] == -1.0), "the replayed graph did not write QOut"
    assert_bits_equal(res[0][0], res[1][0], "QOut")
    assert_bits_equal(res[0][1], res[1][1], "max_eig")
    assert res[0][2] == res[1][2]


def test_run_simulation_dt_underflow_raises():
    """a zero global wave speed with a nonzero field (here rho = 1, j = 0, E = 0,
    so p = c = 0) cannot set dt = cfl*dx/max -- run_simulation raises instead of stepping with
    an infinite dt."""
    from paper_2302_09005_b200.errors import TimeStepUnderflowError

    dim, p, grid = 2, 8, (2, 2)
    n = int(np.prod(grid))
    field = np.tile(np.array([1.0, 0.0, 0.0, 0.0]), (n, p ** dim))
    db = _db_with_field(dim, p, grid, field)
    with pytest.raises(TimeStepUnderflowError) as ei:
        driver.run_simulation(db, grid, steps=3, cfl=0.4, periodic=True)
    assert ei.value.step == 0
    assert "step=0" in str(ei.value)


@pytest.mark.parametrize("graph", [False, True])
def test_run_simulation_nonphysical_is_located(graph):
    """A non-physical volume aborts the run with the step, patch and haloed volume (SPEC.md:451,
    the reference's NonPhysicalStateError fields), found by replaying the run to that step."""
    from paper_2302_09005_b200.errors import NonPhysicalStateError

    dim, p, grid = 2, 16, (3, 3)
    n = int(np.prod(grid))
    state = pde.euler_state(1.0, [0.2, 0.1], 1.0)
    field = np.tile(state, (n, p ** dim)).reshape(n, p, p, 4)
    field[4, 7, 5, 0] = -1.0          # patch 4, interior cell (x=5, y=7): rho < 0
    db = _db_with_field(dim, p, grid, field.reshape(n, -1))
    with pytest.raises(NonPhysicalStateError) as ei:
        driver.run_simulation(db, grid, steps=70, cfl=0.4, periodic=True, graph=graph)
    assert (ei.value.step, ei.value.patch, ei.value.volume) == (0, 4, (6, 8)), str(ei.value)


@pytest.mark.parametrize("dim,p,grid,direct", [(3, 16, (2, 2, 2), None), (2, 16, (4, 3), True), (2, 16, (4, 3), False),
                                               (3, 4, (3, 2, 4), None)])
def test_run_simulation_fast_mode_within_bar(dim, p, grid, direct):
    """mode="fast" runs the fast kernels inside run_simulation (classic and 2D direct paths):
    after 12 steps the field, the dt history and the totals are within the north star's
    1e-12 relative of the exact (bit-identical-to-reference) run."""
    n = int(np.prod(grid))
    q = oracle.synthetic_qin(dim, p, n, seed=61).reshape(n, (p + 2) ** dim, dim + 2)
    inner = q.reshape((n,) + (p + 2,) * dim + (dim + 2,))[(slice(None),) + (slice(1, -1),) * dim].reshape(n, -1)
    res, fields = [], []
    for mode in ("exact", "fast"):
        db = _db_with_field(dim, p, grid, inner)
        res.append(driver.run_simulation(db, grid, steps=12, cfl=0.4, periodic=True, direct=direct, mode=mode))
        fields.append(db.QOut.cpu().numpy().reshape(-1, dim + 2))
    ex, fa = fields
    rel = np.max(np.abs(fa - ex), axis=0) / np.max(np.abs(ex), axis=0)
    assert np.all(rel <= 1e-12) and np.all(rel < 1e-13), rel
    assert np.max(np.abs(np.array(res[1].dt) / np.array(res[0].dt) - 1.0)) < 1e-13
    t0, t1 = np.asarray(res[0].totals), np.asarray(res[1].totals)
    assert np.all(np.abs(t1 - t0) <= 1e-12 * np.abs(t0).max(axis=0))


@pytest.mark.parametrize("dim,p,grid", [(3, 16, (2, 2, 2)), (2, 16, (4, 3)), (3, 4, (3, 2, 2))])
def test_run_simulation_fast_with_redone_patches(dim, p, grid):
    """mode="fast" steps where some patches leave the fast gate every step (a block at rest
    with a tiny pressure: c^2 below 2^-600) -- they are redone exactly inside the loop, the
    redo list empties itself between steps and the CFL tail then reduces max_eig afresh:
    the run stays within 1e-12 of the exact one, dt history included."""
    n = int(np.prod(grid))
    q = oracle.synthetic_qin(dim, p, n, seed=41).reshape((n,) + (p + 2,) * dim + (dim + 2,))
    inner = q[(slice(None),) + (slice(1, -1),) * dim].copy()
    blk = (slice(0, n, 3),) + (slice(1, 4),) * dim
    inner[blk + (slice(1, 1 + dim),)] = 0.0
    inner[blk + (slice(dim + 1, dim + 2),)] = 1e-190          # p ~ 4e-191: c^2 ~ 5e-191 < 2^-600
    inner = inner.reshape(n, -1)
    res, fields = [], []
    for mode in ("exact", "fast"):
        db = _db_with_field(dim, p, grid, inner)
        res.append(driver.run_simulation(db, grid, steps=6, cfl=0.4, periodic=True, mode=mode))
        fields.append(db.QOut.cpu().numpy().reshape(-1, dim + 2))
    ex, fa = fields
    rel = np.max(np.abs(fa - ex), axis=0) / np.max(np.abs(ex), axis=0)
    assert np.all(rel <= 1e-12), rel
    assert np.max(np.abs(np.array(res[1].dt) / np.array(res[0].dt) - 1.0)) < 1e-13
