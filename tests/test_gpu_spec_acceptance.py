"""SPEC.md acceptance criteria in their own scenarios, on the B200 path.
Criteria 2 (variant equivalence), 3 / 6 (scalar oracle, eigenvalue reduction), 5 (convergence),
9 (concurrent batches) and 10 (benchmark integrity) are covered in test_gpu_parity.py,
test_gpu_driver.py and test_bench_cli.py; 7 (the enclave scheduler) is out of scope."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2302_09005_b200 import device, driver, mesh, pde  # noqa: E402


def _interior_field(dim, p, grid, fn):
    """Per-patch interior blocks (x fastest) of a field given as fn(x, y) on cell centres in [0, 1)^2."""
    gx, gy = grid
    nx, ny = gx * p, gy * p
    xs = (np.arange(nx) + 0.5) / nx
    ys = (np.arange(ny) + 0.5) / ny
    X, Y = np.meshgrid(xs, ys, indexing="xy")          # (ny, nx)
    q = fn(X, Y)                                       # (ny, nx, s)
    blocks = q.reshape(gy, p, gx, p, -1).transpose(0, 2, 1, 3, 4)
    return np.ascontiguousarray(blocks).reshape(gx * gy, -1)


def _run(dim, p, grid, field, steps, **kw):
    n = int(np.prod(grid))
    spec = mesh.PatchSpec(dim, p, dim + 2)
    db = device.DeviceBatch(spec, n, 1.4)
    db.QOut.copy_(torch.from_numpy(field.reshape(-1).copy()))
    db.cell_size.fill_(1.0 / grid[0])
    res = driver.run_simulation(db, grid, steps=steps, cfl=0.4, periodic=True, **kw)
    return db, res


def test_criterion_1_constant_state_preservation():
    """SPEC.md:558 #1: rho=1, u=0, p=1, gamma=1.4, d=2, p=17, periodic 3x3 grid, 10 steps:
    the final field is bitwise the initial one."""
    state = pde.euler_state(1.0, [0.0, 0.0], 1.0)
    field = _interior_field(2, 17, (3, 3), lambda X, Y: np.broadcast_to(state, X.shape + (4,)).copy())
    db, res = _run(2, 17, (3, 3), field, 10)
    assert np.array_equal(db.QOut.cpu().numpy().view(np.uint64), field.reshape(-1).view(np.uint64))
    assert res.steps == 10


def _gaussian(X, Y):
    rho = 1.0 + 0.5 * np.exp(-((X - 0.5) ** 2 + (Y - 0.5) ** 2) / 0.02)
    q = np.empty(X.shape + (4,))
    q[..., 0] = rho
    q[..., 1] = rho * 0.3
    q[..., 2] = rho * -0.2
    q[..., 3] = 1.0 / 0.4 + 0.5 * rho * (0.3 ** 2 + 0.2 ** 2)
    return q


def test_criterion_4_conservation():
    """SPEC.md:561 #4: periodic 4x4 grid, p=10, Gaussian density perturbation, CFL 0.4, 100 steps:
    mass, momentum and energy each drift <= 1e-12 relative."""
    field = _interior_field(2, 10, (4, 4), _gaussian)
    _, res = _run(2, 10, (4, 4), field, 100)
    tot = np.asarray(res.totals)
    drift = np.abs(tot[-1] - tot[0]) / np.abs(tot[0])
    assert drift.max() <= 1e-12, drift


def test_criterion_8_schedule_independence():
    """SPEC.md:565 #8: the conservation scenario gives bitwise identical final fields whatever the
    batch size N in {1, 4, 16} the patches are updated in (here: the update launched over
    consecutive sub-batches of N patches, DeviceBatch.update_range, each step)."""
    dim, p, grid, steps = 2, 10, (4, 4), 12
    n = int(np.prod(grid))
    field = _interior_field(dim, p, grid, _gaussian)
    ref, _ = _run(dim, p, grid, field, steps, graph=False)
    spec = mesh.PatchSpec(dim, p, dim + 2)
    for N in (1, 4, 16):
        db = device.DeviceBatch(spec, n, 1.4)
        db.QOut.copy_(torch.from_numpy(field.reshape(-1).copy()))
        db.cell_size.fill_(1.0 / grid[0])
        tot = torch.empty(dim + 2, dtype=torch.float64, device="cuda")
        scratch = db.totals_scratch()
        db.halo_project_totals(grid, True, tot, scratch)
        db.status.zero_()
        stepper = driver.CflStepper(db, cfl=0.4)
        stepper.prepass()
        for _ in range(steps):
            for p0 in range(0, n, N):
                db.update_range(p0, min(n, p0 + N))
            stepper.reduce_dt()
            db.halo_project_totals(grid, True, tot, scratch)
        assert not db.nonphysical()
        assert np.array_equal(db.QOut.cpu().numpy().view(np.uint64), ref.QOut.cpu().numpy().view(np.uint64)), N


@pytest.mark.parametrize("dim,p", [(2, 17), (3, 16), (3, 4), (2, 5)])
def test_criterion_6_eigenvalue_reduction(dim, p):
    """SPEC.md:563 #6: per-patch max_eigenvalue equals the brute-force max over the interior
    volumes' directional eigenvalues |j_n / rho| + sqrt(gamma p / rho) (numpy, pde.py:62-70
    operation order), exactly, on 100 random patches."""
    import oracle

    n, g = 100, 1.4
    spec = mesh.PatchSpec(dim, p, dim + 2)
    b = mesh.make_patch_batch(spec, n)
    b.QIn[...] = oracle.synthetic_qin(dim, p, n, seed=600 + p)
    b.dt[...] = 0.4 / p / 3.4
    db = device.DeviceBatch.from_host(b, g)
    db.update()
    lam = db.max_eigenvalue.cpu().numpy()
    e = p + 2
    q = b.QIn.reshape((n,) + (e,) * dim + (dim + 2,))
    q = q[(slice(None),) + (slice(1, -1),) * dim].reshape(n, -1, dim + 2)
    rho = q[..., 0]
    mom2 = q[..., 1] * q[..., 1]
    for a in range(2, dim + 1):
        mom2 = mom2 + q[..., a] * q[..., a]
    pr = (g - 1.0) * (q[..., -1] - (0.5 * mom2) / rho)
    c = np.sqrt((g * pr) / rho)
    brute = np.max(np.stack([np.abs(q[..., 1 + k] / rho) + c for k in range(dim)], axis=-1), axis=(1, 2))
    assert np.array_equal(lam.view(np.uint64), brute.view(np.uint64))
