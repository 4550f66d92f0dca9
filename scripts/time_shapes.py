"""Device time per update, both modes, for arbitrary shapes (generic-kernel shapes included):
    python scripts/time_shapes.py 3:9:20000 3:12:6000 2:40:20000 ..."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
from paper_2302_09005_b200 import device, mesh  # noqa: E402

for arg in sys.argv[1:] or ["3:9:20000", "3:12:6000", "2:40:20000", "3:3:200000"]:
    dim, p, n = (int(v) for v in arg.split(":"))
    db = device.DeviceBatch(mesh.PatchSpec(dim, p, dim + 2), n, 1.4)
    chunk = max(1, min(n, (64 << 20) // ((p + 2) ** dim * (dim + 2) * 8)))
    q = oracle.synthetic_qin(dim, p, chunk, seed=1)
    v = db.QIn.view(n, -1)
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        v[lo:hi].copy_(torch.from_numpy(q[: hi - lo]))
    db.dt.fill_(0.4 / p / 3.4)
    out = []
    for mode in ("exact", "fast"):
        for _ in range(3):
            db.update(mode=mode)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
        for a, b in ev:
            a.record()
            db.update(mode=mode)
            b.record()
        torch.cuda.synchronize()
        ms = float(np.median([a.elapsed_time(b) for a, b in ev]))
        out.append(f"{mode} {ms * 1e3:9.1f} us {n * p ** dim / ms / 1e6:6.2f} Gcell/s")
    print(f"{dim}D p={p:2d} n={n:7d} [{device.selected_kernel(dim, p, n, 1.4)}]: " + " | ".join(out), flush=True)
