"""paper_2302_09005_b200 -- B200-native batched Rusanov finite-volume patch update.

Drop-in for the hot path of the reference package `fvbatch`
(arXiv 2302.09005 clean-room re-implementation): `kernel.update_patch_batch`
advances a batch of haloed p^d compressible-Euler patches by one
forward-Euler Rusanov step on sm_100a, bit-identical to the reference.

Modules mirror the reference's layout: `errors`, `mesh`, `pde`, `itspace`,
`kernel`; `device` holds the PyTorch-owned device buffers and `driver` the
multi-step / multi-GPU CFL loop.  The compute lives in `libfvb200.so`
(csrc/, C ABI in include/fvb200.h).
"""

from . import errors, itspace, mesh, pde  # noqa: F401
from .errors import ContractViolationError, NonPhysicalStateError  # noqa: F401

__version__ = "0.1.0"
