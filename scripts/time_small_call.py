"""Latency of the drop-in update_patch_batch on small batches (BASELINE configs[0]: 2D p=16, 16 patches)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402
from paper_2302_09005_b200 import mesh, pde  # noqa: E402
from paper_2302_09005_b200.kernel import update_patch_batch, variant_from_labels  # noqa: E402

v = variant_from_labels("patchwise", "aos", "seq")
for dim, p, n in ((2, 16, 16), (2, 16, 256), (3, 16, 16)):
    spec = mesh.PatchSpec(dim, p, dim + 2)
    b = mesh.make_patch_batch(spec, n)
    b.QIn[...] = oracle.synthetic_qin(dim, p, n, seed=1)
    b.dt[...] = 0.4 / p / 3.4
    for _ in range(5):
        update_patch_batch(b, pde.make_euler_pde(dim), v)
    t0 = time.perf_counter()
    k = 50
    for _ in range(k):
        update_patch_batch(b, pde.make_euler_pde(dim), v)
    us = (time.perf_counter() - t0) / k * 1e6
    t1 = time.perf_counter()
    oracle.update(dim, p, 1.4, b.QIn, b.cell_size, b.dt)
    cpu = (time.perf_counter() - t1) * 1e6
    print(f"{dim}D p={p} N={n}: {us:.0f} us per call (oracle port on the host: {cpu:.0f} us)")
