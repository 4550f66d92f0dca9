"""Device time of DeviceBatch.halo_project (run_simulation's other kernel) on the C3 grid (16^3 patches, p = 16)
and on the C2 grid (256^2 patches, p = 16); reports effective HBM bandwidth (QOut read + QIn write)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2302_09005_b200 import device, mesh  # noqa: E402

for dim, p, g in ((3, 16, (16, 16, 16)), (2, 16, (256, 256)), (3, 4, (32, 32, 32)), (3, 8, (16, 16, 32)),
                  (2, 17, (128, 128))):
    n = int(np.prod(g))
    db = device.DeviceBatch(mesh.PatchSpec(dim, p, dim + 2), n, 1.4)
    db.QOut.normal_()
    for _ in range(3):
        db.halo_project(g)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    reps = 20
    for _ in range(reps):
        db.halo_project(g)
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / reps * 1e3
    byts = (db.QOut.numel() + db.QIn.numel()) * 8
    print(f"{dim}D p={p} {g} halo_project: {us:.1f} us, {byts / us / 1e3:.0f} GB/s ({byts / 1e6:.0f} MB)")
