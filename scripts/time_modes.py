"""Device-resident update time of exact vs fast mode (CUDA events, launch-only).

    python scripts/time_modes.py [--config c3|c4|c2] [--iters 20]
"""
import argparse
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
from paper_2302_09005_b200 import device, mesh  # noqa: E402

CFG = {"c3": (3, 16, 4096), "c4": (3, 4, 1 << 20), "c2": (2, 16, 65536)}
BYTES = {"c3": 389144, "c4": 8984, "c2": 18456}
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
dim, p, n = CFG[a.config]
spec = mesh.PatchSpec(dim, p, dim + 2)
db = device.DeviceBatch(spec, n, 1.4)
chunk = 4096 if dim == 3 and p == 16 else 65536
for lo in range(0, n, chunk):
    hi = min(n, lo + chunk)
    q = oracle.synthetic_qin(dim, p, hi - lo, seed=lo)
    db.QIn.view(n, -1)[lo:hi].copy_(torch.from_numpy(q))
db.dt.fill_(0.4 * (1.0 / p) / 3.4)
cells = n * p ** dim
for mode in ("exact", "fast", "exact", "fast"):
    for _ in range(3):
        db.update(mode=mode)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * a.iters)]
    for i in range(a.iters):
        ev[2 * i].record()
        db.update(mode=mode)
        ev[2 * i + 1].record()
    torch.cuda.synchronize()
    ts = np.array([ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(a.iters)])
    ms = float(np.median(ts))
    print(f"{a.config} {mode:5s}: median {ms * 1e3:8.1f} us  min {ts.min() * 1e3:8.1f}  "
          f"{cells / ms / 1e6:6.2f} Gcell/s  {BYTES[a.config] * n / ms / 1e6:7.1f} GB/s  "
          f"redo={int(db.status[1].item())}")
