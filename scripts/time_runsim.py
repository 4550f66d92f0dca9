"""Wall time per step of driver.run_simulation on a 16^3 grid of 3D p=16 patches (4,096 patches),
or with --2d on a 256^2 grid of 2D p=16 patches (65,536 patches, C2's batch).

    python scripts/time_runsim.py          # moving fluid with a random density perturbation
    python scripts/time_runsim.py --sod    # Sod shock tube along x: fluid at rest (exact +0 momentum)
    --eager                                # step by step instead of replaying the captured CUDA graph
    --fast                                 # mode="fast" (the 1e-12 parity bar)
    --classic                              # update + full halo projection (no direct path)
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2302_09005_b200 import device, driver, mesh, pde  # noqa: E402

dim = 2 if "--2d" in sys.argv else 3
g, p = ((256, 256) if dim == 2 else (16, 16, 16)), 16
n = int(np.prod(g))
spec = mesh.PatchSpec(dim, p, dim + 2)
db = device.DeviceBatch(spec, n, 1.4)
q = db.QOut.view(n, p ** dim, dim + 2)
vel0 = [0.0, 0.0, 0.0][:dim]
if "--sod" in sys.argv:
    left = torch.tensor(pde.euler_state(1.0, vel0, 1.0), dtype=torch.float64, device="cuda")
    right = torch.tensor(pde.euler_state(0.125, vel0, 0.1), dtype=torch.float64, device="cuda")
    px = torch.arange(n, device="cuda") % g[0]               # patch x index (x fastest)
    q[...] = torch.where((px < g[0] // 2)[:, None, None], left, right)
else:
    state = torch.tensor(pde.euler_state(1.0, [0.2, 0.1, -0.1][:dim], 1.0), dtype=torch.float64, device="cuda")
    q[...] = state
    q[:, :, 0] += 0.1 * torch.rand(n, p ** dim, device="cuda", dtype=torch.float64)
db.cell_size.fill_(1.0 / 16)
mode = "fast" if "--fast" in sys.argv else "exact"
direct = False if "--classic" in sys.argv else None
driver.run_simulation(db, g, steps=2, graph="--eager" not in sys.argv, mode=mode, direct=direct)
torch.cuda.synchronize()
graph = "--eager" not in sys.argv
for steps in (10, 40, 200):
    t0 = time.perf_counter()
    res = driver.run_simulation(db, g, steps=steps, graph=graph, mode=mode, direct=direct)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"run_simulation {dim}D {mode} {steps} steps: {dt / steps * 1e3:.3f} ms/step, "
          f"{n * p**dim * steps / dt / 1e9:.2f} Gcell/s")
