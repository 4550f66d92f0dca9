"""Diagnostic: per-role work / ring-wait / barrier shares of the 3D p=16 half kernel (needs a library
built with -DFVB3D_PROFILE_BARRIER, e.g. scripts/build_variant.sh pbar -DFVB3D_PROFILE_BARRIER=1)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
from paper_2302_09005_b200 import device, mesh  # noqa: E402

n, p = 4096, 16
spec = mesh.PatchSpec(3, p, 5)
b = mesh.make_patch_batch(spec, 64)
b.QIn[...] = oracle.synthetic_qin(3, p, 64, seed=1)
db = device.DeviceBatch(spec, n, 1.4)
db.QIn.view(n, -1).copy_(torch.from_numpy(np.tile(b.QIn, (n // 64, 1))))
db.dt.fill_(0.4 / p / 3.4)
extra = 2 * n + 64 + 8
db.status = torch.zeros(int(db.status.numel()) + extra * 2 + 64, dtype=torch.int32, device="cuda")
db.update(kernel="fused")
torch.cuda.synchronize()
acc = db.status[2 + 2 * n + 64: 2 + 2 * n + 64 + 12].cpu().numpy().view(np.uint64)
for name, o in (("interior warps", 0), ("halo warp", 3)):
    work, wait, tot = acc[o], acc[o + 1], acc[o + 2]
    print(f"{name}: work {work / tot * 100:.1f} %, ring wait {wait / tot * 100:.1f} %, "
          f"barrier + rest {(tot - work - wait) / tot * 100:.1f} % of their cycles")
