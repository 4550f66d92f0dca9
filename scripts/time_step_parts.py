"""Where a CFL step's time goes beyond its main kernel: events before the fused kernel (a),
after it (b, recorded inside the C ABI before the redo pass), after the whole fvb_update_cfl
call (c), and the next step's a.  Eager launches, device-resident batch.

    python scripts/time_step_parts.py [--config c3|c2|c4|small] [--steps 200] [--mode fast]
"""
import argparse
import ctypes
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
from paper_2302_09005_b200 import _lib, device, driver, mesh  # noqa: E402

CFG = {"c3": (3, 16, 4096), "c4": (3, 4, 1 << 20), "c2": (2, 16, 65536), "small": (3, 16, 512)}
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--steps", type=int, default=200)
ap.add_argument("--mode", default="fast")
a = ap.parse_args()
dim, p, n = CFG[a.config]
spec = mesh.PatchSpec(dim, p, dim + 2)
db = device.DeviceBatch(spec, n, 1.4)
q = oracle.synthetic_qin(dim, p, min(n, 4096), seed=1)
rep = (n + q.shape[0] - 1) // q.shape[0]
db.QIn.view(n, -1).copy_(torch.from_numpy(np.tile(q, (rep, 1))[:n]))
db.dt.fill_(0.4 / p / 3.4)
L = _lib.load()
st = driver.CflStepper(db, cfl=0.4, dx=1.0 / p, mode=a.mode)
st.prepass()
for _ in range(10):
    st.step()
torch.cuda.synchronize()
ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(a.steps)]
for e in ev:
    for x in e:
        x.record()
torch.cuda.synchronize()
for e in ev:
    L.fvb_time_next_update(ctypes.c_void_p(e[0].cuda_event), ctypes.c_void_p(e[1].cuda_event))
    st.step()
    e[2].record()
torch.cuda.synchronize()
k = [e[0].elapsed_time(e[1]) * 1e3 for e in ev]
r = [e[1].elapsed_time(e[2]) * 1e3 for e in ev]
g = [ev[i][2].elapsed_time(ev[i + 1][0]) * 1e3 for i in range(a.steps - 1)]
tot = ev[0][0].elapsed_time(ev[-1][2]) * 1e3 / a.steps
print(f"{a.config} {a.mode}: step {tot:.1f} us = kernel {statistics.median(k):.1f} + after-kernel "
      f"{statistics.median(r):.1f} + gap {statistics.median(g):.1f} (medians)")
