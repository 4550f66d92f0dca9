"""Tiny 2D fused-kernel smoke run (hang / parity triage): python scripts/try2d.py N"""
import sys
print("start", flush=True)
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle
from paper_2302_09005_b200 import device, mesh

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
spec = mesh.PatchSpec(2, 16, 4)
b = mesh.make_patch_batch(spec, n)
b.QIn[...] = oracle.synthetic_qin(2, 16, n, seed=5)
b.dt[...] = 0.4 / 16 / 3.4
print("imported", flush=True)
db = device.DeviceBatch.from_host(b, 1.4)
print("uploaded", flush=True)
db.update(kernel="fused")
torch.cuda.synchronize()
print("ran", flush=True)
db.to_host(b)
rq, rl, st = oracle.update(2, 16, 1.4, b.QIn, b.cell_size, b.dt)
dq = b.QOut.view(np.uint64) != rq.view(np.uint64)
print("QOut mismatches", int(dq.sum()), "of", dq.size, "max_eig equal", np.array_equal(b.max_eigenvalue, rl))
if dq.any():
    idx = np.argwhere(dq.reshape(n, 16, 16, 4))
    print(idx[:10])
