"""Drop-in replacement of `fvbatch.kernel` (reference kernel/__init__.py:1-168).

`update_patch_batch(batch, pde, variant, temporaries=None, engine="vectorized")`
keeps the reference signature, validation order and exceptions
(kernel/__init__.py:114-140) and advances every patch by one forward-Euler
Rusanov step on the GPU (libfvb200.so, sm_100a).  Results are bit-identical
to the reference's vectorized and loop-body engines for every variant.

* The kernel variant (ordering / temporaries layout / host strategy) does not
  change the arithmetic -- all reference variants are bitwise identical --
  so the device ignores it for the update.  It is still honoured where the
  reference's behaviour depends on it: which NonPhysicalStateError is raised
  first when several patches are inadmissible (patch-wise: first patch in
  order; batched: first failing face box over each host patch chunk,
  vectorized.py:82-99, :234-288).
* `temporaries` are accepted and unused: the fused kernel keeps its
  eigenvalue / flux scratch on chip.
* The PDE must be compressible Euler (`make_euler_pde` of this package or of
  the reference); gamma is recovered from the callback closure.  Other PDEs
  cannot be evaluated on the device and raise ContractViolationError.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np

from ..errors import ContractViolationError, NonPhysicalStateError
from ..itspace import PARALLEL, SEQUENTIAL, ExecutionStrategy, StrategyKind, strategy_from_label, strategy_kind_of
from ..mesh import DEFAULT_AOSOA_BLOCK, Layout, LayoutEnumerator, PatchBatch, PatchSpec, layout_from_label
from ..pde import PdeDefinition, bound_gamma


class Ordering(Enum):
    PATCH_WISE = "patchwise"
    BATCHED = "batched"


def ordering_from_label(label: str) -> Ordering:
    for o in Ordering:
        if o.value == label:
            return o
    raise ContractViolationError(f"unknown ordering label {label!r}")


@dataclass(frozen=True)
class KernelVariant:
    """Loop ordering, temporaries layout and execution strategy (kernel/__init__.py:46-57)."""

    ordering: Ordering
    layout: Layout
    strategy: ExecutionStrategy

    @property
    def label(self) -> str:
        return f"{self.ordering.value}-{self.layout.value}-{self.strategy.label}"


def variant_from_labels(ordering: str, layout: str, strategy: str, worker_hint: int | None = None) -> KernelVariant:
    return KernelVariant(ordering=ordering_from_label(ordering), layout=layout_from_label(layout),
                         strategy=strategy_from_label(strategy, worker_hint))


@dataclass(frozen=True)
class KernelEnumerators:
    """Enumerators of the AoS solution arrays (kernel/__init__.py:69-74)."""

    qin: LayoutEnumerator
    qout: LayoutEnumerator


def solution_enumerators(spec: PatchSpec, n_patches: int) -> KernelEnumerators:
    return KernelEnumerators(
        qin=LayoutEnumerator(Layout.AOS, n_patches, spec.dimensions, spec.haloed_per_axis, spec.unknowns),
        qout=LayoutEnumerator(Layout.AOS, n_patches, spec.dimensions, spec.volumes_per_axis, spec.unknowns),
    )


@dataclass
class KernelTemporaries:
    """Shape descriptors of the reference's scratch (kernel/__init__.py:86-96).

    The device path keeps eigenvalues and fluxes on chip, so no host scratch
    is allocated: `eigenvalues` / `flux_values` stay None."""

    eigenvalues: np.ndarray | None
    flux_values: np.ndarray | None
    eig_enum: LayoutEnumerator
    flux_enum: LayoutEnumerator
    enums: KernelEnumerators


def allocate_temporaries(spec: PatchSpec, n_patches: int, layout: Layout,
                         block: int = DEFAULT_AOSOA_BLOCK) -> KernelTemporaries:
    d = spec.dimensions
    return KernelTemporaries(
        eigenvalues=None, flux_values=None,
        eig_enum=LayoutEnumerator(layout, n_patches, d, spec.haloed_per_axis, d, block),
        flux_enum=LayoutEnumerator(layout, n_patches, d, spec.haloed_per_axis, d * spec.unknowns, block),
        enums=solution_enumerators(spec, n_patches),
    )


ENGINES = ("vectorized", "loopbody")
_MSG_RHO = "non-positive density in pressure closure"   # pde.py:38
_MSG_P = "negative pressure in eigenvalue evaluation"   # pde.py:68


def bind_euler(pde, dimensions: int, gamma: float | None = None) -> float:
    """Map a PdeDefinition onto the device closure; returns gamma."""
    name = getattr(pde, "name", None)
    if name != f"euler{dimensions}d":
        raise ContractViolationError(
            f"the device path evaluates compressible Euler only; got PDE {name!r} for {dimensions}D patches")
    if getattr(pde, "has_ncp", False):
        raise ContractViolationError("the device path has no non-conservative product (Euler has none)")
    g = gamma if gamma is not None else bound_gamma(pde)
    if g is None:
        raise ContractViolationError("cannot recover gamma from the PDE callbacks; pass gamma= explicitly")
    if not g > 1.0:
        raise ContractViolationError(f"gamma must exceed 1, got {g}")
    return float(g)


def _chunk_bounds(n: int, chunks: int):
    """vectorized._patch_chunks (vectorized.py:234-243)."""
    base, extra = divmod(n, chunks)
    start = 0
    for i in range(chunks):
        size = base + (1 if i < extra else 0)
        yield start, start + size
        start += size


def box_volume(dim: int, p: int, box: int, lin: int) -> tuple:
    """Haloed (x, y[, z]) of a box-linear index; boxes in vectorized._plan order (vectorized.py:42-53)."""
    lo = [1 if a < dim else 0 for a in range(3)]
    hi = [p + 1 if a < dim else 1 for a in range(3)]
    if box > 0:
        n = (box - 1) // 2
        if (box - 1) % 2 == 0:
            lo[n], hi[n] = 0, 1
        else:
            lo[n], hi[n] = p + 1, p + 2
    nx, ny = hi[0] - lo[0], hi[1] - lo[1]
    z, rem = divmod(int(lin), nx * ny)
    y, x = divmod(rem, nx)
    return tuple(int(v) for v in (x + lo[0], y + lo[1], z + lo[2])[:dim])


def first_error(info: np.ndarray, ordering: Ordering, nchunks: int):
    """The (message, patch, box, lin) the reference raises first, from per-(patch, box) diagnostics.

    info[patch, box] = (trig_rho, trig_p, first_nonpos, first_badpl) (fvb_locate).
    patch-wise: patches in order, boxes in order (vectorized.py:277-288);
    batched: host chunks in order, then boxes over the whole chunk, where
    _locate_bad_state scans (patch, z, y, x) for !(rho>0) before !(p_like>=0)
    (vectorized.py:82-99, :253-275)."""
    n, nbox, _ = info.shape
    trig = (info[:, :, 0] != 0) | (info[:, :, 1] != 0)
    if not trig.any():
        return None
    if ordering is Ordering.PATCH_WISE:
        patch = int(np.argmax(trig.any(axis=1)))
        box = int(np.argmax(trig[patch]))
        r = info[patch, box]
        lin = r[2] if r[2] >= 0 else r[3]
        return (_MSG_RHO if r[0] else _MSG_P), patch, box, int(lin)
    for lo, hi in _chunk_bounds(n, max(1, min(nchunks, n))):
        blk = info[lo:hi]
        for box in range(nbox):
            col = blk[:, box]
            any_rho = bool((col[:, 0] != 0).any())
            if not (any_rho or (col[:, 1] != 0).any()):
                continue
            msg = _MSG_RHO if any_rho else _MSG_P
            np_hit = np.nonzero(col[:, 2] >= 0)[0]
            if np_hit.size:
                return msg, lo + int(np_hit[0]), box, int(col[np_hit[0], 2])
            bp_hit = np.nonzero(col[:, 3] >= 0)[0]
            return msg, lo + int(bp_hit[0]), box, int(col[bp_hit[0], 3])
    return None


def host_chunks(variant, n: int) -> int:
    """Number of host chunks the reference's vectorized engine would use (vectorized.py:250-256)."""
    kind = strategy_kind_of(variant.strategy)
    if kind is not StrategyKind.PARALLEL_UNORDERED:
        return 1
    return min(variant.strategy.workers(), n)


def raise_first_error(info: np.ndarray, variant, dim: int, p: int) -> None:
    ordering = ordering_from_label(getattr(variant.ordering, "value", variant.ordering))
    hit = first_error(info, ordering, host_chunks(variant, info.shape[0]) if ordering is Ordering.BATCHED else 1)
    if hit is None:  # pragma: no cover - the status word and the locator disagree
        raise NonPhysicalStateError("non-physical state (unlocated)")
    msg, patch, box, lin = hit
    raise NonPhysicalStateError(msg, patch=patch, volume=box_volume(dim, p, box, lin))


def update_patch_batch(batch: PatchBatch, pde: PdeDefinition, variant: KernelVariant,
                       temporaries: KernelTemporaries | None = None, engine: str = "vectorized", *,
                       device=None, kernel: str = "auto", gamma: float | None = None,
                       chunk_patches: int | None = None, mode: str = "exact") -> None:
    """Advance every patch of the batch by its own dt (kernel/__init__.py:114-140).

    QOut receives the updated interior solution and max_eigenvalue the
    per-patch directional maximum; QIn is read-only.  Extra keyword-only
    arguments select the CUDA device, the kernel ("auto" | "fused" |
    "generic"), an explicit gamma, the host pipeline chunk size and the
    arithmetic mode: "exact" (default; bit-identical to the reference) or
    "fast" (QOut and max_eigenvalue within 1e-12 relative per unknown -- the
    north star's parity bar; measured ~1e-16 -- with face-shared fluxes and one
    closure per volume: csrc/fvb_fast3d.cu for 3D p = 16, the FAST warp kernel
    of csrc/fvb_fused2d_warp.cu for 2D p = 2..32, the FAST small-patch kernel of
    csrc/fvb_small3d.cu for 3D p = 2, 4..8; AoS).  Shapes without a fast kernel
    run the exact one.
    """
    if batch.n_patches == 0:
        return
    if batch.spec.unknowns != pde.unknowns:
        raise ContractViolationError(
            f"batch carries {batch.spec.unknowns} unknowns, PDE defines {pde.unknowns}")
    if np.any(batch.dt < 0.0):
        raise ContractViolationError("negative dt in batch")
    if engine not in ENGINES:
        raise ContractViolationError(f"unknown engine {engine!r}")
    g = bind_euler(pde, batch.spec.dimensions, gamma)
    from .. import device as _device

    rc = _device.update_host(batch, g, device=device, kernel=kernel, chunk_patches=chunk_patches, mode=mode)
    if rc != 0:
        info = _device.locate_host(batch, g, device=device, chunk_patches=chunk_patches)
        raise_first_error(info, variant, batch.spec.dimensions, batch.spec.volumes_per_axis)


__all__ = [
    "Ordering", "KernelVariant", "KernelEnumerators", "KernelTemporaries", "allocate_temporaries",
    "solution_enumerators", "update_patch_batch", "variant_from_labels", "ordering_from_label",
    "SEQUENTIAL", "PARALLEL", "bind_euler", "first_error", "box_volume",
]
