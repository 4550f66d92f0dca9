"""Drop-in update_patch_batch on pinned vs pageable host batches (3D p=16, 4,096 patches)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
from paper_2302_09005_b200 import mesh, pde  # noqa: E402
from paper_2302_09005_b200.kernel import update_patch_batch, variant_from_labels  # noqa: E402

dim, p, n = 3, 16, 4096
spec = mesh.PatchSpec(dim, p, dim + 2)
tmpl = oracle.synthetic_qin(dim, p, 64, seed=3)
v = variant_from_labels("batched", "aos", "par")
for pinned in (True, False):
    b = mesh.make_patch_batch(spec, n, pinned=pinned)
    b.QIn[...] = np.tile(tmpl, (n // 64, 1))
    b.dt[...] = 0.4 / p / 3.4
    t0 = time.perf_counter()
    update_patch_batch(b, pde.make_euler_pde(dim), v)   # first call (registers pageable arrays)
    print(f"pinned={pinned}: first call {(time.perf_counter() - t0) * 1e3:.1f} ms")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        update_patch_batch(b, pde.make_euler_pde(dim), v)
    dt = (time.perf_counter() - t0) / 5
    print(f"pinned={pinned}: {dt * 1e3:.1f} ms per call, {n * p ** dim / dt / 1e9:.3f} Gcell/s")
