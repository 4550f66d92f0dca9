"""CPU-only tests of the boundary: C-ABI exports, validation order, PDE binding,
error composition, data model, FVB1 fixtures, sharding.  No GPU compute here."""

import ctypes
import json
import os
import re

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, ROOT, load_golden
from paper_2302_09005_b200 import _lib, driver, itspace, mesh, pde
from paper_2302_09005_b200.errors import ContractViolationError, DeviceError, NonPhysicalStateError
from paper_2302_09005_b200.kernel import (Ordering, bind_euler, box_volume, first_error, host_chunks,
                                          update_patch_batch, variant_from_labels)


def _manifest():
    with open(os.path.join(GOLDEN, "manifest.json")) as f:
        return json.load(f)


def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "fvb200.h")).read()
    declared = set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\*?\s+\*?(fvb_[a-z_0-9]+)\s*\(", header, re.M))
    assert declared == set(_lib.EXPORTED), declared ^ set(_lib.EXPORTED)
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    L = _lib.load()
    assert L.fvb_version() >= 1
    assert L.fvb_status_words(10) == 28


def test_capi_contract_checks_without_gpu():
    """Argument validation happens before any CUDA call (safe on a CPU-only host)."""
    L = _lib.load()
    bad = _lib.FvbSpec(4, 16, 6, 0, 10, 1.4)
    assert L.fvb_update(ctypes.byref(bad), None, None, None, None, None, None, 0, 1, None) == _lib.FVB_ERR_CONTRACT
    wrong_s = _lib.FvbSpec(3, 16, 4, 0, 10, 1.4)
    assert L.fvb_update(ctypes.byref(wrong_s), None, None, None, None, None, None, 0, 1, None) == _lib.FVB_ERR_CONTRACT
    ok = _lib.spec(3, 16, 0, 1.4)
    assert L.fvb_update(ctypes.byref(ok), None, None, None, None, None, None, 0, 1, None) == _lib.FVB_OK  # N == 0
    assert L.fvb_select_kernel(ctypes.byref(_lib.spec(3, 16, 5, 1.4))) == _lib.KERNEL_FUSED
    assert L.fvb_select_kernel(ctypes.byref(_lib.spec(3, 4, 5, 1.4))) == _lib.KERNEL_FUSED
    assert L.fvb_select_kernel(ctypes.byref(_lib.spec(3, 4, 5, 1.4, 1))) == _lib.KERNEL_GENERIC
    assert L.fvb_select_kernel(ctypes.byref(_lib.spec(3, 6, 5, 1.4))) == _lib.KERNEL_FUSED     # p = 2..8
    assert L.fvb_select_kernel(ctypes.byref(_lib.spec(3, 5, 5, 1.4))) == _lib.KERNEL_FUSED     # odd p: cp.async
    assert L.fvb_select_kernel(ctypes.byref(_lib.spec(3, 3, 5, 1.4))) == _lib.KERNEL_GENERIC   # p = 3: generic
    assert L.fvb_select_kernel(ctypes.byref(_lib.spec(3, 9, 5, 1.4))) == _lib.KERNEL_GENERIC
    assert L.fvb_select_kernel(ctypes.byref(_lib.spec(3, 6, 5, 1.4, 1))) == _lib.KERNEL_GENERIC   # SoA
    assert L.fvb_select_kernel(ctypes.byref(_lib.spec(2, 16, 5, 1.4, 1))) == _lib.KERNEL_FUSED
    assert L.fvb_select_kernel(ctypes.byref(_lib.spec(2, 17, 5, 1.4))) == _lib.KERNEL_FUSED     # 2D p = 2..32
    assert L.fvb_select_kernel(ctypes.byref(_lib.spec(2, 33, 5, 1.4))) == _lib.KERNEL_GENERIC
    assert L.fvb_select_kernel(ctypes.byref(_lib.spec(2, 17, 5, 1.4, 1))) == _lib.KERNEL_GENERIC
    assert L.fvb_update_host_workspace(ctypes.byref(_lib.spec(3, 16, 8, 1.4)), 4) > 4 * 233280 * 2
    # entry points added for run_simulation / multi-GPU / host pinning: contract checks first
    C = _lib.FVB_ERR_CONTRACT
    g2 = (ctypes.c_int32 * 3)(2, 3, 1)
    assert L.fvb_update_to_haloed(ctypes.byref(_lib.spec(3, 16, 4, 1.4)), None, None, None, None, None, None, 0,
                                  None) == C                                      # 3D: no fast path
    assert L.fvb_update_to_haloed(ctypes.byref(_lib.spec(2, 33, 4, 1.4)), None, None, None, None, None, None, 0,
                                  None) == C                                      # p > 32
    assert L.fvb_update_to_haloed(ctypes.byref(_lib.spec(2, 16, 4, 1.4)), None, None, None, None, None, None, 0,
                                  None) == C                                      # null buffers
    assert L.fvb_halo_shell(ctypes.byref(_lib.spec(2, 16, 5, 1.4)), None, g2, 1, None) == C   # 2x3 != 5 patches
    assert L.fvb_halo_shell(ctypes.byref(_lib.spec(3, 16, 6, 1.4)), None, g2, 1, None) == C   # 3D
    assert L.fvb_totals_haloed(ctypes.byref(_lib.spec(2, 16, 0, 1.4)), None, None, None, None) == C
    assert L.fvb_halo_project_window(ctypes.byref(_lib.spec(2, 40, 4, 1.4)), None, None, None, None, g2, 0, 0,
                                     None, None, None) == C                       # p > 32
    assert L.fvb_halo_project_window(ctypes.byref(_lib.spec(2, 16, 5, 1.4)), None, None, None, None, g2, 0, 0,
                                     None, None, None) == C                       # not whole layers
    assert L.fvb_mgpu_init(0, None) == C
    assert L.fvb_mgpu_allreduce_max(0, None, None) == C
    assert L.fvb_host_pin(None, 0) == C


def test_validation_order_matches_reference():
    """kernel/__init__.py:123-140: N=0 no-op, unknowns, dt < 0, engine -- before any device work."""
    euler2 = pde.make_euler_pde(2)
    pw = variant_from_labels("patchwise", "aos", "seq")
    empty = mesh.PatchBatch(mesh.PatchSpec(2, 4, 4), 0, np.zeros((0, 144)), np.zeros((0, 64)),
                            np.zeros((0, 2)), np.zeros((0, 2)), np.zeros(0), np.zeros(0), np.zeros(0))
    update_patch_batch(empty, euler2, pw, engine="bogus")   # returns before the engine check
    b = mesh.make_patch_batch(mesh.PatchSpec(2, 4, 3), 2)
    with pytest.raises(ContractViolationError, match="unknowns"):
        update_patch_batch(b, euler2, pw)
    b = mesh.make_patch_batch(mesh.PatchSpec(2, 4, 4), 2)
    b.dt[1] = -1.0
    with pytest.raises(ContractViolationError, match="negative dt"):
        update_patch_batch(b, euler2, pw, engine="bogus")
    b.dt[1] = 0.0
    with pytest.raises(ContractViolationError, match="unknown engine"):
        update_patch_batch(b, euler2, pw, engine="bogus")


def test_no_cpu_fallback():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    b = mesh.make_patch_batch(mesh.PatchSpec(2, 4, 4), 2)
    with pytest.raises(DeviceError):
        update_patch_batch(b, pde.make_euler_pde(2), variant_from_labels("patchwise", "aos", "seq"))


def test_pde_binding():
    assert bind_euler(pde.make_euler_pde(3), 3) == 1.4
    assert bind_euler(pde.make_euler_pde(2, pde.EulerParameters(5.0 / 3.0)), 2) == 5.0 / 3.0
    with pytest.raises(ContractViolationError):
        bind_euler(pde.make_euler_pde(2), 3)
    custom = pde.PdeDefinition(unknowns=4, flux=lambda *a: None, max_abs_eigenvalue=lambda *a: None, name="burgers")
    with pytest.raises(ContractViolationError):
        bind_euler(custom, 2)
    ncp = pde.PdeDefinition(unknowns=4, flux=lambda *a: None, max_abs_eigenvalue=lambda *a: None,
                            nonconservative_product=lambda *a: None, name="euler2d")
    with pytest.raises(ContractViolationError):
        bind_euler(ncp, 2)
    anon = pde.PdeDefinition(unknowns=4, flux=lambda *a: None, max_abs_eigenvalue=lambda *a: None, name="euler2d")
    with pytest.raises(ContractViolationError):
        bind_euler(anon, 2)
    assert bind_euler(anon, 2, gamma=1.3) == 1.3


def test_pde_binding_accepts_reference_objects():
    import sys
    src = "/root/reference/pkg/src"
    if not os.path.isdir(src):
        pytest.skip("reference not present on this host")
    sys.path.insert(0, src)
    try:
        from fvbatch import pde as refpde
    finally:
        sys.path.remove(src)
    assert bind_euler(refpde.make_euler_pde(3, refpde.EulerParameters(1.3)), 3) == 1.3


@pytest.mark.parametrize("case", _manifest()["error_cases"], ids=lambda c: c["name"])
def test_error_composition_matches_reference(case):
    """The product's host-side error composition (kernel.first_error) over per-box diagnostics
    reproduces the reference's exception for every ordering / strategy; diagnostics from the oracle."""
    b = load_golden(case["file"])
    d, p = case["dim"], case["p"]
    info = oracle.locate(d, p, case["gamma"], b.QIn)
    for exp in case["expect"]:
        variant = variant_from_labels(exp["ordering"], "aos", exp["strategy"], exp["workers"])
        ordering = Ordering(exp["ordering"])
        hit = first_error(info, ordering, host_chunks(variant, b.n_patches) if ordering is Ordering.BATCHED else 1)
        if not exp["raised"]:
            assert hit is None
            continue
        msg, patch, box, lin = hit
        err = NonPhysicalStateError(msg, patch=patch, volume=box_volume(d, p, box, lin))
        assert str(err) == exp["str"]
        assert box_volume(d, p, box, lin) == oracle.box_volume(d, p, box, lin)


def test_layout_enumerator_known_answers():
    """SPEC.md:77-79, :87-89 examples and exhaustive bijection for small shapes."""
    assert mesh.make_patch_batch(mesh.PatchSpec(2, 4, 4), 1).QIn.shape == (1, 144)
    assert mesh.make_patch_batch(mesh.PatchSpec(2, 4, 4), 1).QOut.shape == (1, 64)
    assert mesh.make_patch_batch(mesh.PatchSpec(3, 1, 1), 1).QIn.shape == (1, 27)
    assert mesh.make_patch_batch(mesh.PatchSpec(2, 17, 4), 16).QIn.shape == (16, 19 * 19 * 4)
    aos = mesh.LayoutEnumerator(mesh.Layout.AOS, 1, 2, 2, 3)
    soa = mesh.LayoutEnumerator(mesh.Layout.SOA, 1, 2, 2, 3)
    assert aos.index(0, (0, 0), 0) == 0 and aos.index(0, (1, 0), 2) == 5 and soa.index(0, (1, 0), 2) == 9
    for kind in mesh.Layout:
        for d, ext, c, n in ((2, 3, 5, 3), (3, 2, 4, 2), (2, 4, 3, 1)):
            e = mesh.LayoutEnumerator(kind, n, d, ext, c)
            off = e.offset_tensor().reshape(-1)
            assert np.array_equal(np.sort(off), np.arange(e.total))
            assert e.index(n - 1, (ext - 1,) * d, c - 1) == off[-1]
    with pytest.raises(ContractViolationError):
        aos.index(0, (2, 0), 0)


def test_fvb1_roundtrip(tmp_path):
    b = load_golden("3d_p4_n8")
    f = tmp_path / "x.fvb"
    mesh.save_batch(b, str(f))
    c = mesh.load_batch(str(f))
    for name in ("QIn", "QOut", "cell_centre", "cell_size", "t", "dt", "max_eigenvalue"):
        assert np.array_equal(getattr(b, name), getattr(c, name))
    with open(f, "r+b") as fh:
        fh.write(b"XXXX")
    with pytest.raises(ContractViolationError):
        mesh.load_batch(str(f))


def test_variant_labels_and_workers(monkeypatch):
    v = variant_from_labels("batched", "aosoa", "par", 3)
    assert v.label == "batched-aosoa-par" and v.strategy.workers() == 3
    monkeypatch.setenv("FVBATCH_WORKERS", "5")
    assert itspace.PARALLEL.workers() == 5
    assert host_chunks(variant_from_labels("batched", "aos", "par"), 3) == 3
    assert host_chunks(variant_from_labels("batched", "aos", "seq"), 30) == 1
    with pytest.raises(ContractViolationError):
        variant_from_labels("diagonal", "aos", "seq")


def test_shard_bounds_cover_in_order():
    for n in (1, 7, 4096, 1 << 20):
        for w in (1, 2, 3, 8):
            spans = [driver.shard_bounds(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1


def test_shard_layout_covers_grid_with_ghosts():
    """driver.shard_layout: shards tile the grid in order; ghost layers exist exactly where a
    neighbour is (all sides when periodic, none at a non-periodic edge); the window grid is
    own layers plus ghosts; the wrap mask leaves the sharded axis to the ghosts."""
    import pytest

    from paper_2302_09005_b200 import driver
    from paper_2302_09005_b200.errors import ContractViolationError

    for grid in ((4, 3, 7), (5, 9)):
        for world in (1, 2, 3, 7):
            for periodic in (True, False):
                if grid[-1] < world:
                    with pytest.raises(ContractViolationError):
                        driver.shard_layout(grid, 0, world, periodic)
                    continue
                prev = 0
                for r in range(world):
                    lay = driver.shard_layout(grid, r, world, periodic)
                    assert lay["l0"] == prev and lay["l1"] > lay["l0"]
                    prev = lay["l1"]
                    has_lo = periodic or r > 0
                    has_hi = periodic or r < world - 1
                    assert (lay["lower"] is not None) == has_lo and (lay["upper"] is not None) == has_hi
                    assert lay["window_grid"][:-1] == grid[:-1]
                    assert lay["window_grid"][-1] == (lay["l1"] - lay["l0"]) + has_lo + has_hi
                    assert lay["pmask"] == (((1 << (len(grid) - 1)) - 1) if periodic else 0)
                    assert lay["patch_hi"] - lay["patch_lo"] == (lay["l1"] - lay["l0"]) * lay["layer"]
                assert prev == grid[-1]


def test_c_host_demo_compiles():
    """examples/c_host_demo.c builds against include/fvb200.h and links libfvb200.so with a
    plain C compiler (no Python / torch types on the boundary); it runs on the GPU box
    (tests/test_gpu_c_host.py)."""
    import shutil
    import subprocess

    import pytest

    if shutil.which("gcc") is None or shutil.which("make") is None:  # pragma: no cover
        pytest.skip("no C toolchain")
    ex = os.path.join(ROOT, "examples")
    r = subprocess.run(["make", "-s", "-B", "-C", ex], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert os.path.exists(os.path.join(ex, "c_host_demo"))
