"""Host enqueue cost of one CFL step (fvb_update_cfl through ctypes) vs its device time:
if the host needs longer than the device, eager steps leave the GPU idle between launches.

    python scripts/time_enqueue.py [--config c3] [--steps 300]
"""
import argparse
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
from paper_2302_09005_b200 import device, driver, mesh  # noqa: E402

CFG = {"c3": (3, 16, 4096), "c4": (3, 4, 1 << 20), "c2": (2, 16, 65536), "small": (3, 16, 512)}
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--steps", type=int, default=300)
ap.add_argument("--mode", default="fast")
a = ap.parse_args()
dim, p, n = CFG[a.config]
spec = mesh.PatchSpec(dim, p, dim + 2)
db = device.DeviceBatch(spec, n, 1.4)
q = oracle.synthetic_qin(dim, p, min(n, 4096), seed=1)
rep = (n + q.shape[0] - 1) // q.shape[0]
db.QIn.view(n, -1).copy_(torch.from_numpy(np.tile(q, (rep, 1))[:n]))
db.dt.fill_(0.4 / p / 3.4)
for graph in (False, True):
    st = driver.CflStepper(db, cfl=0.4, dx=1.0 / p, mode=a.mode, graph=graph)
    st.prepass()
    for _ in range(5):
        st.step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(a.steps):
        st.step()
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    dev = e0.elapsed_time(e1) / a.steps * 1e3
    print(f"{a.config} {a.mode} graph={graph}: host enqueue {(t1 - t0) / a.steps * 1e6:7.1f} us/step, "
          f"device {dev:7.1f} us/step, wall {(t2 - t0) / a.steps * 1e6:7.1f} us/step")

# the step's parts: plain update (fused + redo pass) vs update_cfl (+ the CFL tail in the last CTA)
gmax = torch.zeros(1, dtype=torch.float64, device="cuda")
dts = torch.zeros(1, dtype=torch.float64, device="cuda")
for name, fn in (("update", lambda: db.update(mode=a.mode, zero_status=False)),
                 ("update_cfl", lambda: db.update_cfl(0.4, 1.0 / p, gmax, dts, mode=a.mode)),
                 ("update_cfl (no dt)", lambda: db.update_cfl(0.4, 1.0 / p, gmax, None, mode=a.mode))):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{a.config} {a.mode} {name}: device {e0.elapsed_time(e1) / a.steps * 1e3:7.1f} us/step")

# the same plain update with an event pair around every launch (as scripts/time_modes.py)
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for x, y in ev:
    x.record()
    db.update(mode=a.mode, zero_status=False)
    y.record()
e1.record()
torch.cuda.synchronize()
d = np.array([x.elapsed_time(y) for x, y in ev]) * 1e3
print(f"{a.config} {a.mode} update, events per launch: mean {d.mean():.1f} median {np.median(d):.1f} "
      f"min {d.min():.1f} max {d.max():.1f} us; loop {e0.elapsed_time(e1) / a.steps * 1e3:.1f} us/step; "
      f"redo count now {int(db.status[1].item())}")
