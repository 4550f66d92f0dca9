"""Diagnostic: per-role ring-wait / work / barrier shares of the fast 3D p=16 kernel and which role
arrives last at the per-plane barrier (needs a library built with -DFVB_FAST3D_PROFILE, e.g.
scripts/build_variant.sh fprof -DFVB_FAST3D_PROFILE=1)."""
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
db.status = torch.zeros(2 * n + 5 + 64 + 512, dtype=torch.int32, device="cuda")
for _ in range(3):   # warm launches; the counters of the last one are read
    db.status.zero_()
    db.update(mode="fast")
torch.cuda.synchronize()
acc = db.status[2 + 2 * n + 64: 2 + 2 * n + 64 + 192].cpu().numpy().view(np.uint64)
for name, o in (("interior warps", 0), ("halo warp", 3)):
    ring, work, bar = (float(v) for v in acc[o:o + 3])
    tot = ring + work + bar
    print(f"{name}: ring wait {ring / tot * 100:.1f} %, work {work / tot * 100:.1f} %, "
          f"barrier {bar / tot * 100:.1f} % of their loop cycles")
last_i, last_h = int(acc[6]), int(acc[7])
print(f"last to arrive at the plane barrier: interior warp {last_i}, halo warp {last_h} "
      f"({last_h / max(1, last_i + last_h) * 100:.1f} % halo)")
lat, nlat, lead, nlead = (float(v) for v in acc[11:15])
print(f"stalled ring waits: {nlat / max(1, nlead) * 100:.1f} % of planes, mean issue-to-arrival {lat / max(1, nlat):.0f} cyc; "
      f"mean issue-to-use lead {lead / max(1, nlead):.0f} cyc")
print("last arrivals by warp index:", [int(v) for v in acc[16:26]])
print("warps per sub-partition (interior, halo):", [(int(acc[32 + 2 * i]), int(acc[33 + 2 * i])) for i in range(4)])
print("last arrivals by sub-partition:", [int(v) for v in acc[40:44]])
print("warp index -> sub-partition counts:", [[int(v) for v in acc[44 + 4 * w: 48 + 4 * w]] for w in range(10)])
