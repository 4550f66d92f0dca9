"""Device time of the 2D run_simulation fast-path pieces on C2's grid (256^2 patches, p=16)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
from paper_2302_09005_b200 import _lib, device, mesh  # noqa: E402
from paper_2302_09005_b200.device import _stream_handle, _vp  # noqa: E402

p, g = 16, (256, 256)
n = int(np.prod(g))
spec = mesh.PatchSpec(2, p, 4)
db = device.DeviceBatch(spec, n, 1.4)
t = torch.from_numpy(oracle.synthetic_qin(2, p, 64, seed=1)).cuda()
db.QIn.view(n, -1).copy_(t[torch.arange(n, device="cuda") % 64])
db.dt.fill_(0.4 / p / 3.4)
nxt = torch.empty_like(db.QIn)
L = _lib.load()
fs = ctypes.byref(db.fvb_spec())
st = _stream_handle(torch, None)
gs = (ctypes.c_int32 * 3)(g[0], g[1], 1)
scr = db.totals_scratch()
tot = torch.empty(4, dtype=torch.float64, device="cuda")
ops = {
    "update (classic)": lambda: db.update(),
    "update_to_haloed": lambda: L.fvb_update_to_haloed(fs, _vp(db.QIn), _vp(nxt), _vp(db.cell_size), _vp(db.dt),
                                                       _vp(db.max_eigenvalue), _vp(db.status), 1, st),
    "halo_shell": lambda: L.fvb_halo_shell(fs, _vp(nxt), gs, 1, st),
    "totals_haloed": lambda: L.fvb_totals_haloed(fs, _vp(nxt), _vp(scr), _vp(tot), st),
    "halo_project_totals (classic)": lambda: db.halo_project_totals(g, True, tot, scr),
}
for name, fn in ops.items():
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(20):
        fn()
    b.record()
    torch.cuda.synchronize()
    print(f"{name}: {a.elapsed_time(b) / 20 * 1e3:.1f} us")
