"""Worst case of the exact redo pass: every patch queued (-0.0 momentum everywhere), C3 shape,
fused kernel + redo vs the generic kernel."""
import sys

import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
from paper_2302_09005_b200 import device, mesh  # noqa: E402

dim, p, n = 3, 16, 4096
spec = mesh.PatchSpec(dim, p, dim + 2)
db = device.DeviceBatch(spec, n, 1.4)
t = torch.from_numpy(oracle.synthetic_qin(dim, p, 16, seed=2)).cuda().view(16, -1, dim + 2)
t[..., 1:1 + dim] = -0.0
db.QIn.view(n, -1).copy_(t.reshape(16, -1)[torch.arange(n, device="cuda") % 16])
db.dt.fill_(0.4 / p / 3.4)
for k in ("fused", "generic"):
    for _ in range(2):
        db.update(kernel=k)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(5):
        db.update(kernel=k)
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / 5 * 1e3
    print(f"{k}: {us:.0f} us, {n * p ** dim / us / 1e3:.2f} Gcell/s, queued {int(db.status[1].item())}")
