"""GPU parity of mode="fast" (csrc/fvb_fast3d.cu) against the reference.

The north star's parity bar is a relative tolerance of 1e-12 in fp64
(BASELINE.json); SPEC.md:374 / :378 define it as the relative max-norm per
unknown.  Fast mode must meet that bar for QOut (it measures ~1e-16) and for
max_eigenvalue (a few ulp: the sound speed comes from the one-pass closure),
keep the reference's error semantics, and keep the exact invariants the
face-shared flux makes possible: a constant state and dt = 0 reproduce QIn's
interior bit for bit, and the update conserves the totals over a periodic grid
to rounding.
"""

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

from paper_2302_09005_b200 import device, mesh, pde  # noqa: E402
from paper_2302_09005_b200.errors import ContractViolationError, NonPhysicalStateError  # noqa: E402
from paper_2302_09005_b200.kernel import update_patch_batch, variant_from_labels  # noqa: E402

TOL = 1e-12   # BASELINE.json north_star: "within a relative tolerance of 1e-12 in fp64"
PW = variant_from_labels("patchwise", "aos", "seq")

with open(os.path.join(GOLDEN, "manifest.json")) as _f:
    MANIFEST = json.load(_f)


def rel_maxnorm(a, b, s):
    """max |a - b| / max |b| per unknown, the worst unknown."""
    a = np.asarray(a).reshape(-1, s)
    b = np.asarray(b).reshape(-1, s)
    num = np.max(np.abs(a - b), axis=0)
    den = np.maximum(np.max(np.abs(b), axis=0), np.finfo(np.float64).tiny)
    return float(np.max(num / den))


def assert_max_eig_close(got, ref, what="max_eig"):
    """Wave speeds within 1e-12 relative (and ~1e-15 by design); NaN where the reference has NaN."""
    got, ref = np.asarray(got, dtype=np.float64), np.asarray(ref, dtype=np.float64)
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(got), nan), what
    g, r = got[~nan], ref[~nan]
    inf = np.isinf(r)
    assert np.array_equal(g[inf], r[inf]), what
    g, r = g[~inf], r[~inf]
    if r.size:
        rel = np.max(np.abs(g - r) / np.maximum(np.abs(r), np.finfo(np.float64).tiny))
        assert rel <= TOL, (what, rel)
        assert rel < 1e-14, (what, "far above the few-ulp design accuracy", rel)


def _batch(n, seed, p=16, vary=True, dim=3):
    b = mesh.make_patch_batch(mesh.PatchSpec(dim, p, dim + 2), n)
    b.QIn[...] = oracle.synthetic_qin(dim, p, n, seed=seed)
    rng = np.random.default_rng(seed)
    if vary:
        b.cell_size[...] = rng.uniform(0.5, 2.0, size=n)[:, None]
        b.dt[...] = rng.uniform(0.0, 0.4, size=n) * (b.cell_size[:, 0] / p) / 3.4
    else:
        b.dt[...] = 0.4 * (1.0 / p) / 3.4
    return b


def _fast_device(b, kernel="auto"):
    db = device.DeviceBatch.from_host(b, 1.4)
    db.update(kernel=kernel, mode="fast")
    out = mesh.make_patch_batch(b.spec, b.n_patches)
    db.to_host(out)
    return db, out


@pytest.mark.parametrize("case", [c for c in MANIFEST["solution_cases"] if c["p"] == 16], ids=lambda c: c["name"])
def test_fast_golden(case):
    """Every reference-written p = 16 golden case, 3D (fvb_fast3d.cu) and 2D (the FAST warp kernel)."""
    gold = load_golden(case["file"])
    d = case["dim"]
    b = gold.copy()
    b.QOut[...] = 0.0
    b.max_eigenvalue[...] = 0.0
    update_patch_batch(b, pde.make_euler_pde(d, pde.EulerParameters(case["gamma"])), PW, mode="fast")
    fin = np.isfinite(gold.QOut)
    assert np.array_equal(np.isfinite(b.QOut), fin), case["name"]
    assert rel_maxnorm(np.where(fin, b.QOut, 0.0), np.where(fin, gold.QOut, 0.0), d + 2) <= TOL, case["name"]
    assert_max_eig_close(b.max_eigenvalue, gold.max_eigenvalue, case["name"] + " max_eig")


@pytest.mark.parametrize("n,seed", [(1, 3), (7, 4), (300, 5), (1000, 6)])
def test_fast_random_vs_oracle(n, seed):
    b = _batch(n, seed)
    ref_q, ref_l, st = oracle.update(3, 16, 1.4, b.QIn, b.cell_size, b.dt)
    assert st == 0
    db, out = _fast_device(b)
    assert not db.nonphysical()
    err = rel_maxnorm(out.QOut, ref_q, 5)
    assert err <= TOL, err
    assert err < 1e-14, f"fast mode drifted far above its ~1e-16 design accuracy: {err}"
    assert_max_eig_close(out.max_eigenvalue, ref_l)


def test_fast_full_size_c3():
    """BASELINE configs[2] at full size (4,096 patches)."""
    b = _batch(4096, 42, vary=False)
    ref_q, ref_l, st = oracle.update(3, 16, 1.4, b.QIn, b.cell_size, b.dt)
    assert st == 0
    b2 = b.copy()
    update_patch_batch(b2, pde.make_euler_pde(3), variant_from_labels("batched", "soa", "par"), mode="fast")
    assert rel_maxnorm(b2.QOut, ref_q, 5) <= TOL
    assert_max_eig_close(b2.max_eigenvalue, ref_l)


def test_fast_constant_state_and_dt0_bitwise():
    n = 64
    b = mesh.make_patch_batch(mesh.PatchSpec(3, 16, 5), n)
    q = b.qin_view()
    rng = np.random.default_rng(8)
    for k in range(n):   # one constant admissible state per patch
        q[k] = pde.euler_state(rng.uniform(0.5, 2), rng.uniform(-1, 1, 3), rng.uniform(0.5, 2))
    b.dt[...] = rng.uniform(0.0, 0.01, size=n)
    db, out = _fast_device(b)
    interior = b.qin_view()[:, 1:-1, 1:-1, 1:-1, :].reshape(n, -1)
    assert_bits_equal(out.QOut, interior, "constant state")
    # dt = 0 on random fields: QOut is QIn's interior exactly
    r = _batch(n, 9)
    r.dt[...] = 0.0
    _, out = _fast_device(r)
    assert_bits_equal(out.QOut, r.qin_view()[:, 1:-1, 1:-1, 1:-1, :].reshape(n, -1), "dt = 0")


def test_fast_conservation_periodic_grid():
    """Faces are shared: over a periodic grid the totals change only by rounding."""
    grid = (4, 4, 2)
    n = int(np.prod(grid))
    b = _batch(n, 12, vary=False)
    b.QOut[...] = b.qin_view()[:, 1:-1, 1:-1, 1:-1, :].reshape(n, -1)
    mesh.halo_project(b, grid, True)
    before = b.QOut.reshape(-1, 5).sum(axis=0)
    db, out = _fast_device(b)
    after = out.QOut.reshape(-1, 5).sum(axis=0)
    scale = np.abs(b.QOut.reshape(-1, 5)).sum(axis=0)
    assert np.all(np.abs(after - before) <= 1e-13 * scale), (after - before) / scale


@pytest.mark.parametrize("dt_value", [0.0, 1e-3])
def test_fast_signed_zero_and_rest(dt_value):
    """-0.0 / +0.0 momenta: -0.0 leaves the range gate (exact redo), +0.0 stays fast."""
    p, n = 16, 30
    rng = np.random.default_rng(77)
    v = (p + 2) ** 3
    q = oracle.synthetic_qin(3, p, n, seed=5).reshape(n, v, 5)
    q[::2, :, 1:4] = rng.choice([-0.0, 0.0, -0.5], size=(len(q[::2]), v, 3))
    b = mesh.make_patch_batch(mesh.PatchSpec(3, p, 5), n)
    b.QIn[...] = q.reshape(n, -1)
    b.dt[...] = dt_value
    ref_q, ref_l, st = oracle.update(3, p, 1.4, b.QIn, b.cell_size, b.dt)
    assert st == 0
    db, out = _fast_device(b)
    assert not db.nonphysical()
    assert rel_maxnorm(out.QOut, ref_q, 5) <= TOL
    assert_max_eig_close(out.max_eigenvalue, ref_l)


def test_fast_extreme_values_take_the_exact_path():
    p, n = 16, 12
    b = mesh.make_patch_batch(mesh.PatchSpec(3, p, 5), n)
    b.QIn[...] = oracle.synthetic_qin(3, p, n, seed=91)
    b.dt[...] = [5e-324, 1e-310, 0.0, 1e-3, 1e300, 2.2250738585072014e-308, 1e-320, 0.5, 3e-308, 1e-200,
                 7.0, 1e-5]
    b.cell_size[...] = np.array([1.0, 2.0, 1e-300, 1.0, 1e-10, 3.0, 1.0, 0.25, 1.0, 1e200, 1.0, 1.0])[:, None]
    q = b.qin_view()
    q[3, 5, 5, 5, :] = [1e-250, 0.0, 0.0, 0.0, 1.0]   # tiny density at rest: outside the fast range gate
    q[4, 9, 2, 7, 4] = 1e250       # huge energy
    ref_q, ref_l, st = oracle.update(3, p, 1.4, b.QIn, b.cell_size, b.dt)
    assert st == 0
    _, out = _fast_device(b)
    fin = np.isfinite(ref_q)
    assert np.array_equal(np.isfinite(out.QOut), fin)
    a = np.where(fin, out.QOut, 0.0)
    r = np.where(fin, ref_q, 0.0)
    for k in range(n):   # per patch: the extreme patches must not set the others' scale
        assert rel_maxnorm(a[k], r[k], 5) <= TOL, k
    assert_max_eig_close(out.max_eigenvalue, ref_l)


@pytest.mark.parametrize("case", MANIFEST["error_cases"], ids=lambda c: c["name"])
def test_fast_error_semantics(case):
    """Every reference-written error case (2D and 3D): the same exception text in mode "fast"."""
    gold = load_golden(case["file"])
    pd = pde.make_euler_pde(case["dim"], pde.EulerParameters(case["gamma"]))
    for exp in case["expect"]:
        b = gold.copy()
        v = variant_from_labels(exp["ordering"], "aos", exp["strategy"], worker_hint=exp["workers"])
        if not exp["raised"]:
            update_patch_batch(b, pd, v, mode="fast")
            continue
        with pytest.raises(NonPhysicalStateError) as ei:
            update_patch_batch(b, pd, v, mode="fast")
        assert str(ei.value) == exp["str"]


def test_fast_mode_other_shapes_fall_back_to_exact():
    """Shapes without a fast kernel (the generic kernel's: 3D p=3, p > 8 but 16, 2D p > 32)
    run the exact kernels in mode="fast" (bitwise)."""
    for dim, p, n in [(2, 40, 6), (3, 3, 30), (3, 9, 4), (3, 12, 2)]:
        b = mesh.make_patch_batch(mesh.PatchSpec(dim, p, dim + 2), n)
        b.QIn[...] = oracle.synthetic_qin(dim, p, n, seed=3)
        b.dt[...] = 0.4 * (1.0 / p) / 3.4
        ref_q, ref_l, _ = oracle.update(dim, p, 1.4, b.QIn, b.cell_size, b.dt)
        update_patch_batch(b, pde.make_euler_pde(dim), PW, mode="fast")
        assert_bits_equal(b.QOut, ref_q, f"{dim}D p={p}")
        assert_bits_equal(b.max_eigenvalue, ref_l, "max_eig")


FAST_ALL = [(2, p) for p in range(2, 33)] + [(3, p) for p in (2, 4, 5, 6, 7, 8)]


@pytest.mark.parametrize("dim,p", FAST_ALL, ids=lambda v: str(v))
def test_fast_every_shape_vs_oracle(dim, p):
    """mode="fast" on every shape with a fast kernel (2D p = 2..32: the FAST warp kernel;
    3D p = 2, 4..8: the FAST small-patch kernel): random batches within 1e-12 of the
    oracle, a constant state bitwise."""
    n = max(1, min(257, 30000 // p ** dim))
    b = _batch(n, 100 + 7 * p + dim, p=p, dim=dim)
    ref_q, ref_l, st = oracle.update(dim, p, 1.4, b.QIn, b.cell_size, b.dt)
    assert st == 0
    db, out = _fast_device(b)
    assert not db.nonphysical()
    err = rel_maxnorm(out.QOut, ref_q, dim + 2)
    assert err <= TOL and err < 1e-14, err
    assert_max_eig_close(out.max_eigenvalue, ref_l)
    c = mesh.make_patch_batch(mesh.PatchSpec(dim, p, dim + 2), 5)
    c.qin_view()[...] = pde.euler_state(1.3, [0.2, -0.4, 0.1][:dim], 0.9)
    c.dt[...] = 0.01
    _, outc = _fast_device(c)
    inner = (slice(None),) + (slice(1, -1),) * dim
    assert_bits_equal(outc.QOut, c.qin_view()[inner].reshape(5, -1), "constant state")


def test_unknown_mode_is_a_contract_violation():
    b = _batch(2, 1)
    with pytest.raises(ContractViolationError):
        update_patch_batch(b, pde.make_euler_pde(3), PW, mode="turbo")


# ---- 2D p = 16 (BASELINE configs[1]): the FAST warp kernel ----

@pytest.mark.parametrize("n,seed", [(1, 3), (2, 4), (7, 5), (300, 6), (5001, 7)])
def test_fast2d_random_vs_oracle(n, seed):
    b = _batch(n, seed, dim=2)
    ref_q, ref_l, st = oracle.update(2, 16, 1.4, b.QIn, b.cell_size, b.dt)
    assert st == 0
    db, out = _fast_device(b)
    assert not db.nonphysical()
    err = rel_maxnorm(out.QOut, ref_q, 4)
    assert err <= TOL and err < 1e-14, err
    assert_max_eig_close(out.max_eigenvalue, ref_l)


def test_fast2d_full_size_c2():
    """BASELINE configs[1] at full size (65,536 patches)."""
    b = _batch(65536, 21, vary=False, dim=2)
    ref_q, ref_l, st = oracle.update(2, 16, 1.4, b.QIn, b.cell_size, b.dt)
    assert st == 0
    b2 = b.copy()
    update_patch_batch(b2, pde.make_euler_pde(2), variant_from_labels("batched", "aos", "par"), mode="fast")
    assert rel_maxnorm(b2.QOut, ref_q, 4) <= TOL
    assert_max_eig_close(b2.max_eigenvalue, ref_l)


def test_fast2d_constant_state_dt0_and_conservation():
    n = 48
    b = mesh.make_patch_batch(mesh.PatchSpec(2, 16, 4), n)
    q = b.qin_view()
    rng = np.random.default_rng(18)
    for k in range(n):
        q[k] = pde.euler_state(rng.uniform(0.5, 2), rng.uniform(-1, 1, 2), rng.uniform(0.5, 2))
    b.dt[...] = rng.uniform(0.0, 0.01, size=n)
    _, out = _fast_device(b)
    assert_bits_equal(out.QOut, b.qin_view()[:, 1:-1, 1:-1, :].reshape(n, -1), "constant state")
    r = _batch(n, 19, dim=2)
    r.dt[...] = 0.0
    _, out = _fast_device(r)
    assert_bits_equal(out.QOut, r.qin_view()[:, 1:-1, 1:-1, :].reshape(n, -1), "dt = 0")
    grid = (4, 3)
    g = _batch(12, 20, vary=False, dim=2)
    g.QOut[...] = g.qin_view()[:, 1:-1, 1:-1, :].reshape(12, -1)
    mesh.halo_project(g, grid, True)
    before = g.QOut.reshape(-1, 4).sum(axis=0)
    _, out = _fast_device(g)
    after = out.QOut.reshape(-1, 4).sum(axis=0)
    scale = np.abs(g.QOut.reshape(-1, 4)).sum(axis=0)
    assert np.all(np.abs(after - before) <= 1e-13 * scale), (after - before) / scale


@pytest.mark.parametrize("case", [c for c in MANIFEST["error_cases"] if c["dim"] == 2], ids=lambda c: c["name"])
def test_fast2d_error_semantics(case):
    gold = load_golden(case["file"])
    pd = pde.make_euler_pde(2, pde.EulerParameters(case["gamma"]))
    for exp in case["expect"]:
        b = gold.copy()
        v = variant_from_labels(exp["ordering"], "aos", exp["strategy"], worker_hint=exp["workers"])
        if not exp["raised"]:
            update_patch_batch(b, pd, v, mode="fast")
            continue
        with pytest.raises(NonPhysicalStateError) as ei:
            update_patch_batch(b, pd, v, mode="fast")
        assert str(ei.value) == exp["str"]


# ---- 3D p = 4 (BASELINE configs[3]): the FAST small-patch kernel ----

@pytest.mark.parametrize("n,seed", [(1, 31), (5, 32), (333, 33), (20000, 34)])
def test_fast_small3d_random_vs_oracle(n, seed):
    b = _batch(n, seed, p=4)
    ref_q, ref_l, st = oracle.update(3, 4, 1.4, b.QIn, b.cell_size, b.dt)
    assert st == 0
    db, out = _fast_device(b)
    assert not db.nonphysical()
    err = rel_maxnorm(out.QOut, ref_q, 5)
    assert err <= TOL and err < 1e-14, err
    assert_max_eig_close(out.max_eigenvalue, ref_l)


def test_fast_small3d_constant_state_dt0_and_conservation():
    n = 40
    b = mesh.make_patch_batch(mesh.PatchSpec(3, 4, 5), n)
    q = b.qin_view()
    rng = np.random.default_rng(35)
    for k in range(n):
        q[k] = pde.euler_state(rng.uniform(0.5, 2), rng.uniform(-1, 1, 3), rng.uniform(0.5, 2))
    b.dt[...] = rng.uniform(0.0, 0.01, size=n)
    _, out = _fast_device(b)
    assert_bits_equal(out.QOut, b.qin_view()[:, 1:-1, 1:-1, 1:-1, :].reshape(n, -1), "constant state")
    r = _batch(n, 36, p=4)
    r.dt[...] = 0.0
    _, out = _fast_device(r)
    assert_bits_equal(out.QOut, r.qin_view()[:, 1:-1, 1:-1, 1:-1, :].reshape(n, -1), "dt = 0")
    grid = (3, 2, 4)
    g = _batch(24, 37, p=4, vary=False)
    g.QOut[...] = g.qin_view()[:, 1:-1, 1:-1, 1:-1, :].reshape(24, -1)
    mesh.halo_project(g, grid, True)
    before = g.QOut.reshape(-1, 5).sum(axis=0)
    _, out = _fast_device(g)
    after = out.QOut.reshape(-1, 5).sum(axis=0)
    scale = np.abs(g.QOut.reshape(-1, 5)).sum(axis=0)
    assert np.all(np.abs(after - before) <= 1e-13 * scale), (after - before) / scale


def test_fast_small3d_golden_and_errors():
    """The reference-written 3D p = 4 cases: solution within the bar, NaN corners untouched."""
    for case in [c for c in MANIFEST["solution_cases"] if c["p"] == 4 and c["dim"] == 3]:
        gold = load_golden(case["file"])
        b = gold.copy()
        b.QOut[...] = 0.0
        update_patch_batch(b, pde.make_euler_pde(3, pde.EulerParameters(case["gamma"])), PW, mode="fast")
        fin = np.isfinite(gold.QOut)
        assert np.array_equal(np.isfinite(b.QOut), fin), case["name"]
        assert rel_maxnorm(np.where(fin, b.QOut, 0.0), np.where(fin, gold.QOut, 0.0), 5) <= TOL, case["name"]
        assert_max_eig_close(b.max_eigenvalue, gold.max_eigenvalue, case["name"])


@pytest.mark.parametrize("dim,p", [(3, 16), (2, 16), (3, 4), (2, 7), (2, 2), (2, 17), (2, 32), (3, 2), (3, 5),
                                   (3, 6), (3, 7), (3, 8)])
def test_fast_gate_edges(dim, p):
    """The fast gate (c^2 = gamma p / rho positive, normal, finite; fvb_fast.cuh) at its lower
    edge: patches whose states have c^2 ~ 1e-289 stay on the fast path (within the 1e-12 bar,
    all intermediates still normal), patches with c^2 ~ 1e-296 go through the exact redo pass
    (bit for bit); both kinds mixed in one batch, every fast kernel family."""
    n = 12
    v = (p + 2) ** dim
    rng = np.random.default_rng(90 + p + dim)
    b = mesh.make_patch_batch(mesh.PatchSpec(dim, p, dim + 2), n)
    q = b.QIn.reshape(n, v, dim + 2)
    rho = rng.uniform(0.5, 2.0, (n, v))
    # pressure scale per patch: even patches c^2 ~ 1e-289 (fast), odd ones ~ 1e-296 (redo)
    pscale = np.where(np.arange(n) % 2 == 0, 1e-289, 1e-296)[:, None]
    pr = rng.uniform(0.5, 2.0, (n, v)) * pscale
    vel = rng.uniform(-1.0, 1.0, (n, v, dim)) * np.sqrt(pscale)[..., None]
    q[..., 0] = rho
    q[..., 1:1 + dim] = rho[..., None] * vel
    q[..., dim + 1] = pr / 0.4 + 0.5 * rho * np.sum(vel * vel, axis=-1)
    b.dt[...] = 0.4 * (1.0 / p) / (3.4 * np.sqrt(pscale[:, 0]))   # a CFL-sized step at that wave speed
    ref_q, ref_l, st = oracle.update(dim, p, 1.4, b.QIn, b.cell_size, b.dt)
    assert st == 0
    db, out = _fast_device(b)
    assert not db.nonphysical()
    s = dim + 2
    for k in range(n):
        if k % 2:   # redone exactly
            assert_bits_equal(out.QOut[k], ref_q[k], f"redo patch {k}")
            assert_bits_equal(out.max_eigenvalue[k:k + 1], ref_l[k:k + 1], f"redo patch {k} max_eig")
        else:
            err = rel_maxnorm(out.QOut[k], ref_q[k], s)
            assert err <= TOL and err < 1e-14, (k, err)
    assert_max_eig_close(out.max_eigenvalue, ref_l)


@pytest.mark.parametrize("dim,p", [(3, 16), (2, 16), (3, 4), (2, 5), (2, 31), (3, 7), (3, 8)])
def test_fast_negative_density_and_energy_flagged(dim, p):
    """A volume with rho < 0 AND E < 0 has p < 0 too, so c^2 = gamma p / rho > 0: the fast
    gate must still send its patch to the exact pass, which raises the non-physical flag as
    the reference does (rho <= 0, pde.py:36-38)."""
    n = 5
    b = _batch(n, 17, p=p, vary=False, dim=dim)
    v = (p + 2) ** dim
    q = b.QIn.reshape(n, v, dim + 2)
    e = p + 2
    centre = (e // 2) * (e * e if dim == 3 else e) + (e // 2) * e + e // 2 if dim == 3 else (e // 2) * e + e // 2
    q[2, centre, 0] = -1.0
    q[2, centre, dim + 1] = -3.0
    ref_q, ref_l, st = oracle.update(dim, p, 1.4, b.QIn, b.cell_size, b.dt)
    assert st != 0
    db, _ = _fast_device(b)
    assert db.nonphysical()


@pytest.mark.parametrize("dim,p", [(3, 16), (2, 16), (3, 4)])
def test_fast_gate_upper_edges(dim, p):
    """Large scales stay within the bar on the fast path: densities ~1e80 and ~1e100, sound
    speeds with c^2 ~ 1e190 (every flux product of both operation orders stays finite)."""
    n = 9
    v = (p + 2) ** dim
    rng = np.random.default_rng(70 + p + dim)
    b = mesh.make_patch_batch(mesh.PatchSpec(dim, p, dim + 2), n)
    q = b.QIn.reshape(n, v, dim + 2)
    kind = np.arange(n) % 3                      # 0: fast (rho ~ 1e80), 1: huge rho, 2: huge c^2
    rs = np.array([1e80, 1e100, 1.0])[kind][:, None]
    cs2 = np.array([1.0, 1.0, 1e190])[kind][:, None]
    rho = rng.uniform(0.5, 2.0, (n, v)) * rs
    pr = rng.uniform(0.5, 2.0, (n, v)) * rs * cs2
    vel = rng.uniform(-1.0, 1.0, (n, v, dim)) * np.sqrt(cs2)[..., None]
    q[..., 0] = rho
    q[..., 1:1 + dim] = rho[..., None] * vel
    q[..., dim + 1] = pr / 0.4 + 0.5 * rho * np.sum(vel * vel, axis=-1)
    b.dt[...] = 0.4 * (1.0 / p) / (3.4 * np.sqrt(cs2[:, 0]))
    ref_q, ref_l, st = oracle.update(dim, p, 1.4, b.QIn, b.cell_size, b.dt)
    assert st == 0
    db, out = _fast_device(b)
    assert not db.nonphysical()
    for k in range(n):
        err = rel_maxnorm(out.QOut[k], ref_q[k], dim + 2)
        assert err <= TOL and err < 1e-14, (k, kind[k], err)
    assert_max_eig_close(out.max_eigenvalue, ref_l)


@pytest.mark.parametrize("dim,p", [(3, 16), (2, 16), (3, 4)])
@pytest.mark.parametrize("mach", [30.0, 1e3, 1e5, 1e7])
def test_fast_high_mach_within_bar(mach, dim, p):
    """High-Mach flow: the pressure p = (gamma - 1)(E - |j|^2 / 2 rho) cancels catastrophically
    (E / p ~ mach^2), and fast mode forms it in another order (FMA) than the reference; beyond
    E / p = 2^30 the gate sends the patch to the exact pass, below it the update is within the
    bar."""
    n = 6
    v = (p + 2) ** dim
    rng = np.random.default_rng(int(mach) % 1000 + 7)
    b = mesh.make_patch_batch(mesh.PatchSpec(dim, p, dim + 2), n)
    q = b.QIn.reshape(n, v, dim + 2)
    rho = rng.uniform(0.5, 2.0, (n, v))
    pr = rng.uniform(0.5, 2.0, (n, v))
    vel = rng.uniform(0.5, 1.0, (n, v, dim)) * mach
    q[..., 0] = rho
    q[..., 1:1 + dim] = rho[..., None] * vel
    q[..., dim + 1] = pr / 0.4 + 0.5 * rho * np.sum(vel * vel, axis=-1)
    b.dt[...] = 0.4 * (1.0 / p) / (3.4 * 2.0 * mach)
    ref_q, ref_l, st = oracle.update(dim, p, 1.4, b.QIn, b.cell_size, b.dt)
    if st != 0:   # cancellation made some p negative in the reference: both must flag it
        db, _ = _fast_device(b)
        assert db.nonphysical()
        return
    db, out = _fast_device(b)
    assert not db.nonphysical()
    for k in range(n):
        err = rel_maxnorm(out.QOut[k], ref_q[k], dim + 2)
        assert err <= TOL, (k, err)
    rel = np.max(np.abs(out.max_eigenvalue - ref_l) / ref_l)
    assert rel <= TOL, rel


@pytest.mark.parametrize("dim,p,decades", [(3, 16, 6), (2, 16, 6), (3, 4, 6), (3, 16, 12)])
def test_fast_strong_contrasts_within_bar(dim, p, decades):
    """Density and pressure varying over +-`decades` decades from volume to volume inside a
    patch (shock-like jumps at every face), velocities up to a few sound speeds: every patch
    within the bar (relative max-norm per unknown) of the reference."""
    n = 6
    v = (p + 2) ** dim
    rng = np.random.default_rng(300 + decades + p + dim)
    b = mesh.make_patch_batch(mesh.PatchSpec(dim, p, dim + 2), n)
    q = b.QIn.reshape(n, v, dim + 2)
    rho = 10.0 ** rng.uniform(-decades, decades, (n, v))
    pr = 10.0 ** rng.uniform(-decades, decades, (n, v))
    c = np.sqrt(1.4 * pr / rho)
    vel = rng.uniform(-3.0, 3.0, (n, v, dim)) * c[..., None]
    q[..., 0] = rho
    q[..., 1:1 + dim] = rho[..., None] * vel
    q[..., dim + 1] = pr / 0.4 + 0.5 * rho * np.sum(vel * vel, axis=-1)
    cmax = np.max(4.0 * c, axis=1)
    b.dt[...] = 0.4 * (1.0 / p) / cmax
    ref_q, ref_l, st = oracle.update(dim, p, 1.4, b.QIn, b.cell_size, b.dt)
    db, out = _fast_device(b)
    assert db.nonphysical() == (st != 0)
    if st != 0:
        return
    for k in range(n):
        err = rel_maxnorm(out.QOut[k], ref_q[k], dim + 2)
        assert err <= TOL, (k, err)
    rel = np.max(np.abs(out.max_eigenvalue - ref_l) / ref_l)
    assert rel <= TOL, rel


@pytest.mark.parametrize("dim,p", [(3, 16), (2, 16), (3, 4), (2, 17), (3, 9)])
def test_exact_strong_contrasts_bitwise(dim, p):
    """The same 12-decade contrasts in mode "exact": bit for bit (range gates and the redo pass
    cover whatever the fast quotient paths cannot)."""
    n = 4
    v = (p + 2) ** dim
    rng = np.random.default_rng(500 + p + dim)
    b = mesh.make_patch_batch(mesh.PatchSpec(dim, p, dim + 2), n)
    q = b.QIn.reshape(n, v, dim + 2)
    rho = 10.0 ** rng.uniform(-12, 12, (n, v))
    pr = 10.0 ** rng.uniform(-12, 12, (n, v))
    c = np.sqrt(1.4 * pr / rho)
    vel = rng.uniform(-3.0, 3.0, (n, v, dim)) * c[..., None]
    q[..., 0] = rho
    q[..., 1:1 + dim] = rho[..., None] * vel
    q[..., dim + 1] = pr / 0.4 + 0.5 * rho * np.sum(vel * vel, axis=-1)
    b.dt[...] = 0.4 * (1.0 / p) / np.max(4.0 * c, axis=1)
    ref_q, ref_l, st = oracle.update(dim, p, 1.4, b.QIn, b.cell_size, b.dt)
    db = device.DeviceBatch.from_host(b, 1.4)
    db.update(mode="exact")
    assert db.nonphysical() == (st != 0)
    if st != 0:
        return
    out = mesh.make_patch_batch(b.spec, n)
    db.to_host(out)
    assert_bits_equal(out.QOut, ref_q, "QOut")
    assert_bits_equal(out.max_eigenvalue, ref_l, "max_eig")


@pytest.mark.parametrize("dim,p", [(3, 16), (2, 16), (3, 4)])
@pytest.mark.parametrize("where", ["face_halo", "corner"])
def test_fast_negative_state_in_halo(dim, p, where):
    """rho < 0 and E < 0 in a face-halo volume (read by the reference's face boxes: flagged) or
    in an edge / corner volume (never read: no flag, results unchanged)."""
    n = 3
    b = _batch(n, 23, p=p, vary=False, dim=dim)
    e = p + 2
    v = e ** dim
    q = b.QIn.reshape(n, v, dim + 2)
    mid = e // 2
    if dim == 3:
        vol = (mid * e + mid) * e + 0 if where == "face_halo" else (0 * e + 0) * e + 0   # x-face halo / corner
    else:
        vol = mid * e + 0 if where == "face_halo" else 0
    q[1, vol, 0] = -1.0
    q[1, vol, dim + 1] = -3.0
    ref_q, ref_l, st = oracle.update(dim, p, 1.4, b.QIn, b.cell_size, b.dt)
    db, out = _fast_device(b)
    assert db.nonphysical() == (st != 0), (where, st)
    if st == 0:
        err = rel_maxnorm(out.QOut, ref_q, dim + 2)
        assert err <= TOL, err


@pytest.mark.parametrize("mach", [1e5, 1e7])
def test_fast3d_high_mach_halo_volume(mach):
    """The 3D p=16 kernel tests E/p on its own volumes only (the halo warp skips it): a face-halo
    volume at extreme Mach next to an ordinary interior must still leave the patch within the
    bar -- its pressure's rounding enters only beside momentum / energy fluxes and a wave speed
    that are Mach-times larger."""
    dim, p, n = 3, 16, 4
    b = _batch(n, 29, p=p, vary=False, dim=dim)
    e = p + 2
    q = b.QIn.reshape(n, e ** dim, dim + 2)
    for vol in ((5 * e + 7) * e + 0, (9 * e + 0) * e + 4, (0 * e + 8) * e + 8):   # x-, y-, z-face halos
        rho, pr = 1.3, 0.9
        vel = np.array([mach, -0.5 * mach, 0.25 * mach])
        q[1, vol] = [rho, *(rho * vel), pr / 0.4 + 0.5 * rho * vel @ vel]
    b.dt[...] = 0.4 * (1.0 / p) / (3.4 * mach)
    ref_q, ref_l, st = oracle.update(dim, p, 1.4, b.QIn, b.cell_size, b.dt)
    db, out = _fast_device(b)
    assert db.nonphysical() == (st != 0)
    if st != 0:
        return
    for k in range(n):
        err = rel_maxnorm(out.QOut[k], ref_q[k], dim + 2)
        assert err <= TOL, (k, err)


@pytest.mark.parametrize("dim,p", [(3, 16), (2, 16), (3, 4), (2, 17), (3, 6), (3, 9)])
@pytest.mark.parametrize("scale", [1e-289, 1e-296, 1e100, 1e150])
def test_exact_extreme_scales_bitwise(dim, p, scale):
    """Mode "exact" at extreme pressure / density scales (the fast gate's edges and beyond, and
    huge densities): bit for bit with the reference, whichever internal path (fused fast
    quotients, range-gated slow paths, redo pass) each volume takes."""
    n = 4
    v = (p + 2) ** dim
    rng = np.random.default_rng(int(np.log10(scale)) % 97 + p)
    b = mesh.make_patch_batch(mesh.PatchSpec(dim, p, dim + 2), n)
    q = b.QIn.reshape(n, v, dim + 2)
    big = scale > 1.0
    rho = rng.uniform(0.5, 2.0, (n, v)) * (scale if big else 1.0)
    pr = rng.uniform(0.5, 2.0, (n, v)) * scale
    vel = rng.uniform(-1.0, 1.0, (n, v, dim)) * (1.0 if big else np.sqrt(scale))
    q[..., 0] = rho
    q[..., 1:1 + dim] = rho[..., None] * vel
    q[..., dim + 1] = pr / 0.4 + 0.5 * rho * np.sum(vel * vel, axis=-1)
    b.dt[...] = 0.4 * (1.0 / p) / (3.4 * (1.0 if big else np.sqrt(scale)))
    ref_q, ref_l, st = oracle.update(dim, p, 1.4, b.QIn, b.cell_size, b.dt)
    db = device.DeviceBatch.from_host(b, 1.4)
    db.update(mode="exact")
    assert db.nonphysical() == (st != 0)
    if st != 0:
        return
    out = mesh.make_patch_batch(b.spec, n)
    db.to_host(out)
    assert_bits_equal(out.QOut, ref_q, "QOut")
    assert_bits_equal(out.max_eigenvalue, ref_l, "max_eig")


@pytest.mark.parametrize("dim,p,chunk", [(3, 16, 3), (2, 16, 7), (3, 4, 5)])
def test_fast_host_pipeline_with_redone_patches(dim, p, chunk):
    """The drop-in host path (chunked H2D -> fast kernel -> redo pass -> D2H, per-chunk status
    words) with patches that leave the fast gate in several chunks: redone ones bit for bit,
    the rest within the bar."""
    n = 16
    v = (p + 2) ** dim
    rng = np.random.default_rng(61 + p + chunk)
    b = mesh.make_patch_batch(mesh.PatchSpec(dim, p, dim + 2), n)
    q = b.QIn.reshape(n, v, dim + 2)
    tiny = np.arange(n) % 3 == 1
    pscale = np.where(tiny, 1e-296, 1.0)[:, None]
    rho = rng.uniform(0.5, 2.0, (n, v))
    pr = rng.uniform(0.5, 2.0, (n, v)) * pscale
    vel = rng.uniform(-1.0, 1.0, (n, v, dim)) * np.sqrt(pscale)[..., None]
    q[..., 0] = rho
    q[..., 1:1 + dim] = rho[..., None] * vel
    q[..., dim + 1] = pr / 0.4 + 0.5 * rho * np.sum(vel * vel, axis=-1)
    b.dt[...] = 0.4 * (1.0 / p) / (3.4 * np.sqrt(pscale[:, 0]))
    ref_q, ref_l, st = oracle.update(dim, p, 1.4, b.QIn, b.cell_size, b.dt)
    assert st == 0
    update_patch_batch(b, pde.make_euler_pde(dim), PW, mode="fast", chunk_patches=chunk)
    for k in range(n):
        if tiny[k]:
            assert_bits_equal(b.QOut[k], ref_q[k], f"redo patch {k}")
        else:
            assert rel_maxnorm(b.QOut[k], ref_q[k], dim + 2) <= TOL, k
    assert_max_eig_close(b.max_eigenvalue, ref_l)
