"""Seeded randomized parity sweep (B200): shapes, layouts, kernels and value sets drawn at
random -- admissible states with +-0.0 and tiny momenta, huge / tiny scales, zero dt, varied
cell sizes, occasionally inadmissible volumes -- each checked against the CPU oracle: bit for
bit when the reference succeeds, and the non-physical flag when it raises."""

import numpy as np
import pytest

import oracle
from conftest import assert_bits_equal

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2302_09005_b200 import device, mesh  # noqa: E402

SHAPES_2D = list(range(2, 33)) + [40]
SHAPES_3D = [2, 3, 4, 4, 5, 6, 7, 8, 8, 9, 16, 16, 16, 17]   # fused shapes weighted up


def _case(seed):
    rng = np.random.default_rng(seed)
    dim = int(rng.choice([2, 3]))
    p = int(rng.choice(SHAPES_2D if dim == 2 else SHAPES_3D))
    cells = p ** dim
    n = int(rng.integers(1, max(2, min(400, 60000 // cells))))
    layout = "soa" if rng.random() < 0.25 else "aos"
    kernel = "generic" if rng.random() < 0.15 else "auto"
    gamma = float(rng.choice([1.4, 5.0 / 3.0]))
    s = dim + 2
    v = (p + 2) ** dim
    scale = 10.0 ** rng.uniform(-30, 30) if rng.random() < 0.2 else 1.0
    rho = rng.uniform(0.5, 2.0, (n, v)) * scale
    vel = rng.uniform(-1.0, 1.0, (n, v, dim))
    pr = rng.uniform(0.5, 2.0, (n, v)) * scale
    mode = rng.random()
    if mode < 0.3:                                   # fluid at rest in some components / patches
        vel[rng.random((n, v, dim)) < 0.4] = 0.0
    elif mode < 0.4:                                 # signed zeros
        vel[rng.random((n, v, dim)) < 0.3] = -0.0
    elif mode < 0.5:                                 # tiny momenta (outside the fast range)
        vel[rng.random((n, v, dim)) < 0.05] = 1e-70
    q = np.empty((n, v, s))
    q[..., 0] = rho
    q[..., 1:1 + dim] = rho[..., None] * vel
    q[..., -1] = pr / (gamma - 1.0) + 0.5 * rho * np.sum(vel * vel, axis=-1)
    if rng.random() < 0.1:                           # an inadmissible volume somewhere
        k = rng.integers(n)
        q[k, rng.integers(v), -1] = -1.0 * scale
    cs = rng.uniform(0.25, 4.0, n)
    c_max = np.sqrt(gamma * 4.0) + 1.0
    dt = rng.uniform(0.0, 0.4, n) * (cs / p) / c_max
    dt[rng.random(n) < 0.1] = 0.0
    return dim, p, n, layout, kernel, gamma, q.reshape(n, -1), cs, dt


@pytest.mark.parametrize("seed", range(128))
def test_fuzz_vs_oracle(seed):
    dim, p, n, layout, kernel, gamma, qin, cs, dt = _case(seed)
    if kernel == "auto" and layout == "soa" and device.selected_kernel(dim, p, n, gamma, "soa") != "fused":
        kernel = "auto"
    spec = mesh.PatchSpec(dim, p, dim + 2)
    b = mesh.make_patch_batch(spec, n)
    b.QIn[...] = qin
    b.cell_size[...] = cs[:, None]
    b.dt[...] = dt
    ref_q, ref_l, st = oracle.update(dim, p, gamma, b.QIn, b.cell_size, b.dt)
    db = device.DeviceBatch.from_host(b, gamma, layout=layout)
    db.update(kernel=kernel)
    out = mesh.make_patch_batch(spec, n)
    db.to_host(out)
    what = f"seed {seed}: {dim}D p={p} n={n} {layout} {kernel} gamma={gamma:.3f}"
    assert db.nonphysical() == (st != 0), what
    if st == 0:
        assert_bits_equal(out.QOut, ref_q, what)
        assert_bits_equal(out.max_eigenvalue, ref_l, what + " max_eig")


@pytest.mark.parametrize("seed", range(32))
def test_fuzz_drop_in_vs_oracle(seed):
    """The drop-in update_patch_batch on host arrays (chunked H2D / kernel / D2H pipeline with a
    random chunk size, random variant labels): bits when admissible; when not, the same
    NonPhysicalStateError patch and volume the reference's engine would raise first."""
    from paper_2302_09005_b200 import kernel as K
    from paper_2302_09005_b200 import pde
    from paper_2302_09005_b200.errors import NonPhysicalStateError

    dim, p, n, _, _, gamma, qin, cs, dt = _case(1000 + seed)
    rng = np.random.default_rng(seed)
    if rng.random() < 0.35:   # make some batches inadmissible on purpose
        q = qin.reshape(n, -1, dim + 2)
        k = rng.integers(n, size=int(rng.integers(1, 4)))
        q[k, rng.integers(q.shape[1], size=k.size), 0] = -1.0
    ordering = str(rng.choice(["patchwise", "batched"]))
    strategy = str(rng.choice(["seq", "par"]))
    variant = K.variant_from_labels(ordering, "aos", strategy, int(rng.integers(1, 9)))
    chunk = None if rng.random() < 0.5 else int(rng.integers(1, n + 1))
    spec = mesh.PatchSpec(dim, p, dim + 2)
    b = mesh.make_patch_batch(spec, n)
    b.QIn[...] = qin
    b.cell_size[...] = cs[:, None]
    b.dt[...] = dt
    euler = pde.make_euler_pde(dim, pde.EulerParameters(gamma))
    ref_q, ref_l, st = oracle.update(dim, p, gamma, b.QIn, b.cell_size, b.dt)
    what = f"seed {seed}: {dim}D p={p} n={n} {ordering}/{strategy} chunk={chunk}"
    if st == 0:
        K.update_patch_batch(b, euler, variant, chunk_patches=chunk)
        assert_bits_equal(b.QOut, ref_q, what)
        assert_bits_equal(b.max_eigenvalue, ref_l, what + " max_eig")
        return
    info = oracle.locate(dim, p, gamma, b.QIn)
    nch = K.host_chunks(variant, n) if ordering == "batched" else 1
    patch, box, lin, _ = oracle.first_error(dim, p, info, 0 if ordering == "patchwise" else 1, nch)
    with pytest.raises(NonPhysicalStateError) as ei:
        K.update_patch_batch(b, euler, variant, chunk_patches=chunk)
    assert ei.value.patch == patch, what
    assert tuple(ei.value.volume) == tuple(oracle.box_volume(dim, p, box, lin)), what


@pytest.mark.parametrize("seed", range(24))
def test_fuzz_halo_project_vs_oracle(seed):
    """halo_project on random grids / patch sizes / layouts (every kernel path: TMA, row kernels,
    thread-copy fallbacks, SoA) equals the oracle's np.pad restatement bit for bit."""
    rng = np.random.default_rng(500 + seed)
    dim = int(rng.choice([2, 3]))
    p = int(rng.choice([2, 3, 4, 5, 8, 16, 17, 33] if dim == 2 else [2, 3, 4, 5, 8, 16, 19]))
    grid = tuple(int(g) for g in rng.integers(1, 5 if dim == 3 else 7, size=dim))
    n = int(np.prod(grid))
    layout = "soa" if rng.random() < 0.3 else "aos"
    periodic = bool(rng.random() < 0.5)
    spec = mesh.PatchSpec(dim, p, dim + 2)
    qout = rng.standard_normal((n, p ** dim * (dim + 2)))
    ref = oracle.halo_project(dim, p, qout, grid, periodic)
    db = device.DeviceBatch(spec, n, 1.4, layout=layout)
    src = torch.from_numpy(qout.reshape(-1).copy()).cuda()
    if layout == "aos":
        db.QOut.copy_(src)
    else:
        db.pack_from(src, interior=True)
    db.halo_project(grid, periodic)
    if layout == "aos":
        got = db.QIn.cpu().numpy()
    else:
        import ctypes

        from paper_2302_09005_b200 import _lib
        out = torch.empty_like(db.QIn)
        _lib.check(_lib.load().fvb_unpack(ctypes.byref(db.fvb_spec()), device._vp(db.QIn), device._vp(out), 0,
                                          device._stream_handle(torch, None)), "unpack")
        got = out.cpu().numpy()
    assert_bits_equal(got.reshape(ref.shape), ref, f"seed {seed}: {dim}D p={p} grid={grid} {layout} periodic={periodic}")


FAST_SHAPES = [(3, 16), (2, 16), (3, 4)]


def _fast_case(seed):
    """The sweep's value sets on the shapes with a fast kernel (AoS, kernel auto)."""
    rng = np.random.default_rng(10_000 + seed)
    dim, p = FAST_SHAPES[seed % len(FAST_SHAPES)]
    gamma = float(rng.choice([1.4, 5.0 / 3.0]))
    v = (p + 2) ** dim
    n = int(rng.integers(1, max(2, min(300, 40000 // p ** dim))))
    scale = 10.0 ** rng.uniform(-30, 30) if rng.random() < 0.2 else 1.0
    rho = rng.uniform(0.5, 2.0, (n, v)) * scale
    vel = rng.uniform(-1.0, 1.0, (n, v, dim))
    pr = rng.uniform(0.5, 2.0, (n, v)) * scale
    m = rng.random()
    if m < 0.3:
        vel[rng.random((n, v, dim)) < 0.4] = 0.0
    elif m < 0.4:
        vel[rng.random((n, v, dim)) < 0.3] = -0.0
    elif m < 0.5:
        vel[rng.random((n, v, dim)) < 0.05] = 1e-70
    q = np.empty((n, v, dim + 2))
    q[..., 0] = rho
    q[..., 1:1 + dim] = rho[..., None] * vel
    q[..., -1] = pr / (gamma - 1.0) + 0.5 * rho * np.sum(vel * vel, axis=-1)
    if rng.random() < 0.1:
        q[rng.integers(n), rng.integers(v), -1] = -1.0 * scale
    cs = rng.uniform(0.25, 4.0, n)
    dt = rng.uniform(0.0, 0.4, n) * (cs / p) / (np.sqrt(gamma * 4.0) + 1.0)
    dt[rng.random(n) < 0.1] = 0.0
    return dim, p, n, gamma, q.reshape(n, -1), cs, dt


@pytest.mark.parametrize("seed", range(48))
def test_fuzz_fast_mode_vs_oracle(seed):
    """mode="fast" over random value sets: the non-physical flag as the reference, and -- when the
    reference succeeds -- QOut per patch and max_eigenvalue within 1e-12 relative (NaN / inf
    positions identical)."""
    dim, p, n, gamma, qin, cs, dt = _fast_case(seed)
    spec = mesh.PatchSpec(dim, p, dim + 2)
    b = mesh.make_patch_batch(spec, n)
    b.QIn[...] = qin
    b.cell_size[...] = cs[:, None]
    b.dt[...] = dt
    ref_q, ref_l, st = oracle.update(dim, p, gamma, b.QIn, b.cell_size, b.dt)
    db = device.DeviceBatch.from_host(b, gamma)
    db.update(mode="fast")
    out = mesh.make_patch_batch(spec, n)
    db.to_host(out)
    what = f"seed {seed}: {dim}D p={p} n={n} gamma={gamma:.3f}"
    assert db.nonphysical() == (st != 0), what
    if st != 0:
        return
    s = dim + 2
    fin = np.isfinite(ref_q)
    assert np.array_equal(np.isfinite(out.QOut), fin), what
    a, r = np.where(fin, out.QOut, 0.0), np.where(fin, ref_q, 0.0)
    for k in range(n):   # per patch: scales differ by up to 1e60 across a batch
        ak, rk = a[k].reshape(-1, s), r[k].reshape(-1, s)
        num = np.max(np.abs(ak - rk), axis=0)
        den = np.maximum(np.max(np.abs(rk), axis=0), np.finfo(np.float64).tiny)
        assert np.max(num / den) <= 1e-12, (what, k, np.max(num / den))
    lf = np.isfinite(ref_l)
    assert np.array_equal(np.isfinite(out.max_eigenvalue), lf), what
    rel = np.abs(out.max_eigenvalue[lf] - ref_l[lf]) / np.maximum(np.abs(ref_l[lf]), np.finfo(np.float64).tiny)
    assert rel.size == 0 or rel.max() <= 1e-12, (what, rel.max())
