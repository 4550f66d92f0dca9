"""Benchmark: cell updates/s of the fp64 Rusanov patch update on B200 (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--config c3|c2|c4] [--layout aos|soa]
    python bench.py --impl reference ...      # the reference algorithm on the host cores (oracle port)

One step = one fused Rusanov update of the rank's shard (device resident) plus
the CFL step control: local max wave speed, NCCL MAX all-reduce when N > 1,
dt = (cfl*dx)/gmax written back on the device (driver.CflStepper).  Weak
scaling (default): every rank owns the configuration's full patch count;
--scaling strong splits the configuration's patches over the ranks instead.

Rank 0 prints one JSON line (the driver contract).  `value` is device-timed
(CUDA events, max over ranks); `e2e` is the drop-in public API
(kernel.update_patch_batch) on pinned host arrays, H2D + D2H inside the timed
region; `roofline` is the fused kernel's algorithmic HBM bytes per launch over
its event-timed duration against MEASURED_PEAKS.json; `cpu_baseline` is the
CPU oracle (a C restatement of the reference algorithm, oracle/) on a bounded
sample, timed on this box's host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (dim, p, patches per GPU, BASELINE.json configs index)
    "c2": (2, 16, 65536, 1),
    "c3": (3, 16, 4096, 2),
    "c4": (3, 4, 1048576, 3),
    # not BASELINE configs: the SPEC's Fig. 1 shape (2D p=17) and a 3D p=8 case, both on the
    # generic kernel, for measuring the fallback path
    "x2p17": (2, 17, 65536, None),
    "x3p8": (3, 8, 32768, None),
}
METRIC = "cell updates/sec (fp64, 3D Euler p=16) at 1/2/4/8 B200; % of HBM roofline"


def _cfg_label(idx) -> str:
    return f"BASELINE configs[{idx}]" if idx is not None else "not a BASELINE config"


def algorithmic_bytes_per_patch(dim: int, p: int) -> int:
    """QIn interior + face halo read, QOut written, 24 B of per-patch scalars."""
    s = dim + 2
    return (p ** dim + 2 * dim * p ** (dim - 1)) * s * 8 + p ** dim * s * 8 + 24


def algorithmic_flops_per_cell(dim: int, p: int) -> float:
    """add/sub/mul/div/sqrt/max = 1 flop (abs = 0) per interior cell update:
    closures on interior + face-halo volumes, face terms, and the per-cell accumulation."""
    s = dim + 2
    vols = p ** dim + 2 * dim * p ** (dim - 1)
    faces = dim * (p + 1) * p ** (dim - 1)
    return (vols * (dim * dim + 8 * dim + 7) + faces * (2 + 4 * s)) / p ** dim + 5 * dim * s


# B200 FP64: 64 lanes/clk/SM (measured, scripts/micro/lat.cu) x 2 (DFMA) x 148 SMs x 1.965 GHz
FP64_PEAK_TFLOPS = 64 * 2 * 148 * 1.965e9 / 1e12


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) != len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for name, val in zip(names, parts[2:]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def pcie_bandwidth(torch, nbytes: int = 256 << 20):
    """Pinned host <-> device copy bandwidth of this GPU's link (GB/s): H2D alone, D2H alone, and
    each direction while both run (the e2e pipeline overlaps them).  The e2e roofline."""
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    d.copy_(h, non_blocking=True)
    h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()

    def timed(fn, reps=3):
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / reps

    def both():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)

    out = {"h2d": nbytes / timed(lambda: d.copy_(h, non_blocking=True)) / 1e9,
           "d2h": nbytes / timed(lambda: h.copy_(d, non_blocking=True)) / 1e9,
           "bidir_each": nbytes / timed(both) / 1e9}
    del h, h2, d, d2
    return out


def cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_cpu_sample(dim: int, p: int, target_s: float | None = None):
    """Time the oracle port on a bounded sample of the workload; returns (cells/s, cores, description)."""
    import numpy as np

    import oracle

    oracle.build()
    if target_s is None:
        target_s = float(os.environ.get("FVB_BENCH_CPU_SECONDS", "8"))
    cores = cpu_cores()
    n = max(cores * 4, 64) if p >= 16 else max(cores * 256, 4096)
    if os.environ.get("FVB_BENCH_CPU_SMALL"):   # CI: a tiny sample
        n = max(cores, 2)
    qin = oracle.synthetic_qin(dim, p, n, seed=7)
    cs = np.ones((n, dim))
    dt = np.full(n, 0.4 * (1.0 / p) / 3.4)
    oracle.update(dim, p, 1.4, qin[: min(n, cores)], cs[: min(n, cores)], dt[: min(n, cores)], nthreads=cores)
    reps, elapsed = 0, 0.0
    t0 = time.perf_counter()
    while elapsed < target_s or reps < 1:
        oracle.update(dim, p, 1.4, qin, cs, dt, nthreads=cores)
        reps += 1
        elapsed = time.perf_counter() - t0
    cells = reps * n * p ** dim
    return cells / elapsed, cores, f"{reps} x {n} patches ({dim}D p={p}), {elapsed:.1f} s wall, oracle port (C, OpenMP)"


def reference_arm(args):
    """--impl reference: the reference algorithm on the host cores (oracle port), rank 0 only."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    dim, p, n_per_gpu, _ = CONFIGS[args.config]
    per_step = []
    value_total, cores, desc = None, None, None
    budget = float(os.environ.get("FVB_BENCH_CPU_SECONDS", "20"))
    for _ in range(args.warmup):
        run_cpu_sample(dim, p, target_s=min(1.0, budget / 10))
    for _ in range(args.steps):
        v, cores, desc = run_cpu_sample(dim, p, target_s=max(budget / max(args.steps, 1), 0.05))
        per_step.append(v)
    value_total = statistics.median(per_step)
    line = {
        "metric": METRIC, "impl": "reference", "value": value_total, "unit": "cell updates/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": n_per_gpu * p ** dim / value_total * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{dim}D Euler p={p}, {n_per_gpu} patches ({_cfg_label(CONFIGS[args.config][3])})",
                   "dim": dim, "p": p, "patches": n_per_gpu},
        "cpu_baseline": {"value": value_total, "unit": "cell updates/s", "cores": cores, "kind": "port",
                         "sample": desc},
        "e2e": {"value": value_total, "unit": "cell updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--layout", default="aos", choices=["aos", "soa"])
    ap.add_argument("--kernel", default="auto", choices=["auto", "fused", "generic"])
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        reference_arm(args)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    import oracle  # cpu_baseline leg only
    from paper_2302_09005_b200 import device as fdev
    from paper_2302_09005_b200 import driver, mesh, pde
    from paper_2302_09005_b200.kernel import update_patch_batch, variant_from_labels

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    dim, p, n, cfg_idx = CONFIGS[args.config]
    n_total = n * world   # weak: every rank the configuration's count
    if args.scaling == "strong":   # the configuration's patches shared by the ranks
        lo, hi = driver.shard_bounds(n, rank, world)
        n_total, n = n, hi - lo
    spec = mesh.PatchSpec(dim, p, dim + 2)
    gamma = 1.4
    # synthetic admissible states, generated on the device in slabs
    db = fdev.DeviceBatch(spec, n, gamma, layout=args.layout)
    gen = torch.Generator(device="cuda").manual_seed(1234 + rank)
    per = spec.haloed_volumes
    slab = max(1, (64 << 20) // (per * spec.unknowns * 8))
    qin_aos = db.QIn if args.layout == "aos" else torch.empty_like(db.QIn)
    qv = qin_aos.view(n, per, spec.unknowns)
    for lo in range(0, n, slab):
        hi = min(n, lo + slab)
        shp = (hi - lo, per)
        rho = torch.rand(shp, generator=gen, device="cuda", dtype=torch.float64) * 1.5 + 0.5
        vel = torch.rand(shp + (dim,), generator=gen, device="cuda", dtype=torch.float64) * 2.0 - 1.0
        pr = torch.rand(shp, generator=gen, device="cuda", dtype=torch.float64) * 1.5 + 0.5
        qv[lo:hi, :, 0] = rho
        qv[lo:hi, :, 1:1 + dim] = rho[..., None] * vel
        qv[lo:hi, :, -1] = pr / (gamma - 1.0) + 0.5 * rho * (vel * vel).sum(-1)
    if args.layout == "soa":
        db.pack_from(qin_aos)
        del qin_aos, qv
    db.cell_size.fill_(1.0)
    stream = torch.cuda.current_stream()
    stepper = driver.CflStepper(db, cfl=0.4, dx=1.0 / p, kernel=args.kernel, stream=stream)
    stepper.prepass()
    torch.cuda.synchronize()
    if db.nonphysical():
        raise RuntimeError("synthetic input is not admissible")

    for _ in range(args.warmup):
        stepper.step()
    kernel_name = fdev.selected_kernel(dim, p, n, gamma, args.layout) if args.kernel == "auto" else args.kernel

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        t_start.record(stream)
        for k in range(args.steps):
            ev[k][0].record(stream)
            db.update(kernel=args.kernel, stream=stream)
            ev[k][1].record(stream)
            stepper.reduce_dt()
        t_end.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    total_ms = t_start.elapsed_time(t_end)
    kern_ms = statistics.mean(a.elapsed_time(b) for a, b in ev)
    if world > 1:
        t = torch.tensor([total_ms, kern_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, kern_ms = float(t[0]), float(t[1])
    if db.nonphysical():
        raise RuntimeError("non-physical state during the timed steps")
    cells_per_gpu = n * p ** dim
    total_cells = n_total * p ** dim
    value = total_cells * args.steps / (total_ms * 1e-3)
    ms_per_step = total_ms / args.steps

    peaks, peak_kind = measured_peaks()
    bytes_per_launch = n * algorithmic_bytes_per_patch(dim, p)
    flops_cell = algorithmic_flops_per_cell(dim, p)
    achieved = bytes_per_launch / (kern_ms * 1e-3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                traffic = json.load(f).get(f"{args.config}_{args.layout}", {}).get("dram_bytes_per_launch")
        except (OSError, ValueError):
            traffic = None

    # ---- e2e: the drop-in public API on pinned host buffers ----
    e2e = None
    if args.e2e_steps > 0:
        host = mesh.make_patch_batch(spec, n, pinned=True)
        aos = db.QIn if args.layout == "aos" else None
        if aos is None:
            aos = torch.empty_like(db.QIn)
            from paper_2302_09005_b200 import _lib
            import ctypes
            _lib.check(_lib.load().fvb_unpack(ctypes.byref(db.fvb_spec()), fdev._vp(db.QIn), fdev._vp(aos), 0,
                                              fdev._stream_handle(torch, stream)), "unpack")
        host.QIn.reshape(-1)[...] = aos.cpu().numpy()
        host.dt[...] = 0.4 * (1.0 / p) / 3.4
        euler = pde.make_euler_pde(dim)
        variant = variant_from_labels("batched", "aos", "par")
        for _ in range(2):   # warm-up (workspace allocation, first touch of the pinned pages)
            update_patch_batch(host, euler, variant)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            update_patch_batch(host, euler, variant)
        e1.record(stream)
        torch.cuda.synchronize()
        wall_ms = (time.perf_counter() - t0) * 1e3
        e2e_ms = max(e0.elapsed_time(e1), wall_ms)
        if world > 1:
            t = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t[0])
        h2d_b = int(host.QIn.nbytes + host.cell_size.nbytes + host.dt.nbytes)
        d2h_b = int(host.QOut.nbytes + host.max_eigenvalue.nbytes)
        e2e = {"value": total_cells * args.e2e_steps / (e2e_ms * 1e-3), "unit": "cell updates/s",
               "h2d_bytes_per_step": h2d_b, "d2h_bytes_per_step": d2h_b,
               "steps": args.e2e_steps, "path": "kernel.update_patch_batch (pinned numpy in, numpy out)"}
        # e2e roofline: the PCIe link, both directions busy at once (copies of chunk k+1 in,
        # chunk k-1 out overlap the kernel of chunk k in fvb_update_host)
        bw = pcie_bandwidth(torch)
        t_bound = max(h2d_b / (bw["h2d"] * 1e9), d2h_b / (bw["d2h"] * 1e9),
                      (h2d_b + d2h_b) / (2.0 * bw["bidir_each"] * 1e9))
        bound = total_cells / t_bound
        e2e["pcie_gbs"] = {k: round(v, 2) for k, v in bw.items()}
        e2e["roofline"] = {"bound": "pcie", "value": bound, "frac": e2e["value"] / bound}
        del host

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, cores, desc = run_cpu_sample(dim, p)
        cpu = {"value": v, "unit": "cell updates/s", "cores": cores, "kind": "port", "sample": desc}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "cell updates/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": (f"{dim}D Euler p={p}, {n} patches per GPU ({_cfg_label(cfg_idx)})"
                                    if args.scaling == "weak" else
                                    f"{dim}D Euler p={p}, {n_total} patches over {world} GPU(s) "
                                    f"({_cfg_label(cfg_idx)}, strong scaling)"),
                       "dim": dim, "p": p, "patches_per_gpu": n, "layout": args.layout, "kernel": kernel_name,
                       "parallelism": f"patch shards x{world}, NCCL MAX all-reduce of the wave speed",
                       "l2": f"inputs {n * spec.haloed_volumes * spec.unknowns * 8 / 1e6:.0f} MB > 126 MB L2; no flush"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                         "kernel_ms": kern_ms, "algorithmic_bytes_per_launch": bytes_per_launch,
                         "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})"},
            # the min(HBM, FP64) roofline of the north star: the FP64 side at the algorithmic
            # flop count (the exact recipe issues ~1.3x more FP64 instructions)
            "roofline_fp64": {"achieved": flops_cell * cells_per_gpu / (kern_ms * 1e-3) / 1e12,
                              "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                              "frac": flops_cell * cells_per_gpu / (kern_ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
                              "flops_per_cell": flops_cell,
                              "cells_per_s_at_peak": FP64_PEAK_TFLOPS * 1e12 / flops_cell},
            "cpu_baseline": cpu,
            "e2e": e2e,
            # per step: the update kernel (+ the fused path's redo pass) + the dt reduction
            # (one kernel up to 16,384 patches, else reduce_max_grid + set_dt)
            "gpu_launches": args.steps * ((2 if kernel_name == "fused" else 1) + (1 if n <= 16384 else 2)),
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
