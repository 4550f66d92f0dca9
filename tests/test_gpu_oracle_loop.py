"""Multi-step runs pinned to the oracle (VERDICT r1 'missing' 1 / 'next' 2b) and the full-size
BASELINE configs[3] (1,048,576 3D p=4 patches) bit for bit (VERDICT r1 'next' 2a).

The multi-step loop is composed from pinned pieces only -- oracle.update (the reference's
update, pinned to reference-written goldens), oracle.halo_project (mesh.py:261-310) and the
SPEC's time step (dt = cflFactor*dx / max_patches max_eigenvalue of the
previous step, a wave-speed pre-pass for the first) -- and driver.run_simulation (classic,
2D direct, CUDA graph replay) and run_simulation_sharded must reproduce its final field,
every dt and every global wave speed bit for bit.
"""

import numpy as np
import pytest

import oracle
from conftest import assert_bits_equal

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2302_09005_b200 import device, driver, mesh  # noqa: E402

CFL = 0.4


def oracle_loop(dim, p, grid, qout0, steps, periodic, cell=1.0, gamma=1.4):
    """(final QOut, dt history, global max wave speed history) of the SPEC loop, on the CPU."""
    n = int(np.prod(grid))
    dx = cell / p                                     # driver: cell_size[0] / p
    cs = np.full((n, dim), cell)
    qin = oracle.halo_project(dim, p, qout0, grid, periodic)
    _, lam0, st = oracle.update(dim, p, gamma, qin, cs, np.zeros(n))   # wave-speed pre-pass
    assert st == 0
    gmax = [float(np.max(lam0))]
    dts = []
    qout = qout0
    for _ in range(steps):
        dt = (CFL * dx) / gmax[-1]                    # SPEC.md:449 (fvb_set_dt: RN(RN(cfl*dx)/gmax))
        dts.append(dt)
        qout, lam, st = oracle.update(dim, p, gamma, qin, cs, np.full(n, dt))
        assert st == 0
        gmax.append(float(np.max(lam)))
        qin = oracle.halo_project(dim, p, qout, grid, periodic)
    return qout, qin, dts, gmax


def initial_field(dim, p, grid, seed):
    n = int(np.prod(grid))
    q = oracle.synthetic_qin(dim, p, n, seed=seed).reshape(n, *(p + 2,) * dim, dim + 2)
    sl = (slice(None),) + (slice(1, -1),) * dim
    return np.ascontiguousarray(q[sl]).reshape(n, -1)


CASES = [(2, 16, (4, 3), True), (2, 16, (3, 2), False), (2, 5, (2, 3), True), (3, 8, (2, 2, 2), True),
         (3, 8, (3, 1, 2), False), (3, 16, (2, 1, 2), True), (3, 4, (3, 2, 2), False)]


@pytest.mark.parametrize("dim,p,grid,periodic", CASES)
@pytest.mark.parametrize("mode", ["classic", "direct", "graph"])
def test_run_simulation_matches_oracle_loop(dim, p, grid, periodic, mode):
    if mode == "direct" and dim != 2:
        pytest.skip("the direct (update into the next haloed batch) path is 2D")
    steps = 10
    n = int(np.prod(grid))
    q0 = initial_field(dim, p, grid, seed=100 + p)
    ref_q, ref_qin, ref_dt, ref_g = oracle_loop(dim, p, grid, q0, steps, periodic)
    db = device.DeviceBatch(mesh.PatchSpec(dim, p, dim + 2), n, 1.4)
    db.QOut.copy_(torch.from_numpy(q0.reshape(-1)))
    res = driver.run_simulation(db, grid, steps=steps, cfl=CFL, periodic=periodic, direct=(mode == "direct"),
                                graph=(mode == "graph"))
    assert_bits_equal(db.QOut.cpu().numpy().reshape(n, -1), ref_q, f"{mode} final QOut")
    assert_bits_equal(db.QIn.cpu().numpy().reshape(n, -1), ref_qin, f"{mode} final QIn")
    assert_bits_equal(np.array(res.dt), np.array(ref_dt), f"{mode} dt history")
    assert_bits_equal(np.array(res.max_eigenvalue), np.array(ref_g), f"{mode} max eigenvalue history")


@pytest.mark.parametrize("dim,p,grid,periodic", [(3, 8, (2, 2, 2), True), (2, 16, (3, 2), False)])
def test_run_simulation_sharded_one_rank_matches_oracle_loop(dim, p, grid, periodic):
    steps = 6
    q0 = initial_field(dim, p, grid, seed=7)
    ref_q, _, ref_dt, ref_g = oracle_loop(dim, p, grid, q0, steps, periodic)
    sg = driver.ShardedGrid(mesh.PatchSpec(dim, p, dim + 2), grid, 1.4, periodic, rank=0, world=1)
    sg.db.QOut.copy_(torch.from_numpy(q0.reshape(-1)))
    res = driver.run_simulation_sharded(sg, steps=steps, cfl=CFL)
    assert_bits_equal(sg.db.QOut.cpu().numpy().reshape(q0.shape), ref_q, "sharded final QOut")
    assert_bits_equal(np.array(res.dt), np.array(ref_dt), "sharded dt history")
    assert_bits_equal(np.array(res.max_eigenvalue), np.array(ref_g), "sharded max eigenvalue history")


def test_full_size_c4_device_resident_vs_oracle():
    """BASELINE configs[3]: 1,048,576 3D p=4 patches in one device-resident launch (QIn 9.06 GB,
    element offsets beyond 2^32 bytes), distinct random data per patch, bit for bit."""
    dim, p, n = 3, 4, 1 << 20
    free, _ = torch.cuda.mem_get_info()
    spec = mesh.PatchSpec(dim, p, dim + 2)
    if free < 16 << 30:  # pragma: no cover
        pytest.skip("needs ~12 GB of device memory")
    db = device.DeviceBatch(spec, n, 1.4)
    qv = db.QIn.view(n, -1)
    chunk = 1 << 17
    host_qin = np.empty((n, spec.haloed_volumes * spec.unknowns))
    for lo in range(0, n, chunk):
        host_qin[lo:lo + chunk] = oracle.synthetic_qin(dim, p, chunk, seed=lo)
    qv.copy_(torch.from_numpy(host_qin))
    rng = np.random.default_rng(4)
    dt = rng.uniform(0.0, 0.4, size=n) * (1.0 / p) / 3.4
    db.dt.copy_(torch.from_numpy(dt))
    db.update()
    torch.cuda.synchronize()
    assert not db.nonphysical()
    ref_q, ref_l, st = oracle.update(dim, p, 1.4, host_qin, np.ones((n, dim)), dt)
    assert st == 0
    del host_qin
    out_q = db.QOut.cpu().numpy().reshape(n, -1)
    assert_bits_equal(out_q, ref_q, "C4 full size QOut")
    assert_bits_equal(db.max_eigenvalue.cpu().numpy(), ref_l, "C4 full size max_eig")
    # mode "fast" on the same batch (the small-patch kernel's boxed TMA staging, tensor-map
    # patch coordinates up to 2^20): within the north star's 1e-12 relative max-norm
    del out_q
    db.update(mode="fast")
    torch.cuda.synchronize()
    assert not db.nonphysical()
    out_q = db.QOut.cpu().numpy().reshape(-1, dim + 2)
    ref5 = ref_q.reshape(-1, dim + 2)
    err = float(np.max(np.max(np.abs(out_q - ref5), axis=0) / np.max(np.abs(ref5), axis=0)))
    assert err <= 1e-12 and err < 1e-14, err
    le = db.max_eigenvalue.cpu().numpy()
    assert float(np.max(np.abs(le - ref_l) / ref_l)) < 1e-14
