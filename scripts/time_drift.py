"""Per-launch time of the fast C3 update over a sustained run, with NVML clock / power / throttle
samples: does the kernel slow down as the board heats up?   python scripts/time_drift.py [seconds]"""
import sys
import time

import numpy as np
import pynvml
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
from paper_2302_09005_b200 import device, mesh  # noqa: E402

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 20.0
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
dim, p, n = 3, 16, 4096
db = device.DeviceBatch(mesh.PatchSpec(dim, p, 5), n, 1.4)
db.QIn.view(n, -1).copy_(torch.from_numpy(oracle.synthetic_qin(dim, p, n, seed=seed)))
db.dt.fill_(0.4 / p / 3.4)
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
t_end = time.time() + secs
while time.time() < t_end:
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(200)]
    for x, y in ev:
        x.record()
        db.update(mode="fast", zero_status=False)
        y.record()
    time.sleep(0.03)
    clk = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
    pw = pynvml.nvmlDeviceGetPowerUsage(h) / 1000
    thr = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
    tmp = pynvml.nvmlDeviceGetTemperature(h, pynvml.NVML_TEMPERATURE_GPU)
    torch.cuda.synchronize()
    d = np.array([x.elapsed_time(y) for x, y in ev]) * 1e3
    print(f"median {np.median(d):6.1f} us  min {d.min():6.1f}  sm {clk} MHz  {pw:6.0f} W  {tmp} C  throttle 0x{thr:x}",
          flush=True)
