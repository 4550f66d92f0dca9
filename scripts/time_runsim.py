"""Wall time per step of driver.run_simulation on a 16^3 grid of 3D p=16 patches (4,096 patches).

    python scripts/time_runsim.py          # moving fluid with a random density perturbation
    python scripts/time_runsim.py --sod    # Sod shock tube along x: fluid at rest (exact +0 momentum)
    --eager                                # step by step instead of replaying the captured CUDA graph
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2302_09005_b200 import device, driver, mesh, pde  # noqa: E402

g, p = (16, 16, 16), 16
n = int(np.prod(g))
spec = mesh.PatchSpec(3, p, 5)
db = device.DeviceBatch(spec, n, 1.4)
q = db.QOut.view(n, p ** 3, 5)
if "--sod" in sys.argv:
    left = torch.tensor(pde.euler_state(1.0, [0.0, 0.0, 0.0], 1.0), dtype=torch.float64, device="cuda")
    right = torch.tensor(pde.euler_state(0.125, [0.0, 0.0, 0.0], 0.1), dtype=torch.float64, device="cuda")
    px = torch.arange(n, device="cuda") % g[0]               # patch x index (x fastest)
    q[...] = torch.where((px < g[0] // 2)[:, None, None], left, right)
else:
    state = torch.tensor(pde.euler_state(1.0, [0.2, 0.1, -0.1], 1.0), dtype=torch.float64, device="cuda")
    q[...] = state
    q[:, :, 0] += 0.1 * torch.rand(n, p ** 3, device="cuda", dtype=torch.float64)
db.cell_size.fill_(1.0 / 16)
driver.run_simulation(db, g, steps=2, graph="--eager" not in sys.argv)
torch.cuda.synchronize()
graph = "--eager" not in sys.argv
for steps in (10, 40, 200):
    t0 = time.perf_counter()
    res = driver.run_simulation(db, g, steps=steps, graph=graph)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"run_simulation {steps} steps: {dt / steps * 1e3:.3f} ms/step, {n * p**3 * steps / dt / 1e9:.2f} Gcell/s")
