"""Experiment: the fused kernel reading QIn from / writing QOut to pinned HOST memory directly
(zero-copy over PCIe, TMA bulk copies on mapped host pointers) vs the chunked copy pipeline.

    python scripts/time_zerocopy.py [--config c3|c2|c4] [--mode fast]
"""
import argparse
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
from paper_2302_09005_b200 import _lib, device, mesh  # noqa: E402

CFG = {"c3": (3, 16, 4096), "c4": (3, 4, 1 << 20), "c2": (2, 16, 65536)}
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--mode", default="fast")
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
L = _lib.load()
db = device.DeviceBatch.from_host(b, 1.4)
ref = mesh.make_patch_batch(spec, n)
db.update(mode=a.mode)
db.to_host(ref)
fs = db.fvb_spec()
kid = device.kernel_id("auto", a.mode)
hq = ctypes.c_void_p(b.QIn.__array_interface__["data"][0])
ho = ctypes.c_void_p(b.QOut.__array_interface__["data"][0])
st = torch.cuda.current_stream().cuda_stream


def zc():
    rc = L.fvb_update(ctypes.byref(fs), hq, ho, device._vp(db.cell_size), device._vp(db.dt),
                      device._vp(db.max_eigenvalue), device._vp(db.status), kid, 1, ctypes.c_void_p(st))
    assert rc == 0, rc


b.QOut[...] = 0
zc()
torch.cuda.synchronize()
print("zero-copy QOut == device path:", bool(np.array_equal(b.QOut, ref.QOut)))
for name, fn in (("zero-copy fvb_update", zc),
                 ("copy pipeline update_host", lambda: device.update_host(b, 1.4, mode=a.mode))):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    t = float(np.median(ts))
    print(f"{a.config} {name}: {t * 1e3:.2f} ms, {cells / t / 1e9:.3f} Gcell/s")
