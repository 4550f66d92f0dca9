"""Drop-in host path (fvb_update_host) time vs the pipeline chunk count, pinned numpy batch.

    python scripts/time_e2e_chunks.py [--config c3|c2|c4] [--reps 5]
"""
import argparse
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
from paper_2302_09005_b200 import device, mesh  # noqa: E402

CFG = {"c3": (3, 16, 4096), "c4": (3, 4, 1 << 20), "c2": (2, 16, 65536)}
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
dim, p, n = CFG[a.config]
spec = mesh.PatchSpec(dim, p, dim + 2)
b = mesh.make_patch_batch(spec, n, pinned=True)
q = oracle.synthetic_qin(dim, p, min(n, 4096), seed=1)
rep = (n + q.shape[0] - 1) // q.shape[0]
b.QIn.reshape(n, -1)[...] = np.tile(q, (rep, 1))[:n]
b.dt[...] = 0.4 / p / 3.4
cells = n * p ** dim
for k in (16, 32, 48, 64, 96, 128):
    chunk = device.default_chunk(spec, n, k)
    for _ in range(2):
        device.update_host(b, 1.4, mode="fast", chunk_patches=chunk)
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        t0 = time.perf_counter()
        device.update_host(b, 1.4, mode="fast", chunk_patches=chunk)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    t = float(np.median(ts))
    print(f"{a.config} chunks~{k:4d} (chunk {chunk:6d} patches): {t * 1e3:7.2f} ms  {cells / t / 1e9:.3f} Gcell/s")
