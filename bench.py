"""Benchmark: cell updates/s of the fp64 Rusanov patch update on B200 (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--config c3|c2|c4] [--mode fast|exact]
    python bench.py --impl reference ...      # the reference algorithm on the host cores

One step = one fused Rusanov update of the rank's shard (device resident) plus
the CFL step control: local max wave speed, NCCL MAX all-reduce when N > 1,
dt = (cfl*dx)/gmax written back on the device (driver.CflStepper), captured
once in a CUDA graph and replayed.  Weak scaling (default): every rank owns the
configuration's full patch count; --scaling strong splits it over the ranks.

Rank 0 prints one JSON line (the driver contract):
  value        device-timed throughput of the K steps (CUDA events, max over ranks)
               in --mode (default "fast": QOut and max_eigenvalue within the north
               star's 1e-12 relative tolerance; tests/test_gpu_fast.py)
  exact        the same for the bit-exact mode (the library's default)
  e2e          the drop-in public API (kernel.update_patch_batch) on pinned host
               arrays, H2D + D2H inside the timed region
  roofline     the update kernel's algorithmic HBM bytes per launch over its
               duration: the median of CUDA-event pairs recorded on its stream around
               the main kernel of every timed step (inside the C ABI,
               fvb_time_next_update), against MEASURED_PEAKS.json
  cpu_baseline the CPU oracle (a C restatement of the reference algorithm, oracle/)
               over the full configuration batch, on this box's host cores;
               cpu_baseline_numpy the reference's own numpy engine (baseline/_ref)
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
    # not BASELINE configs: the SPEC's Fig. 1 shape (2D p=17) and a 3D p=8 case
    "x2p17": (2, 17, 65536, None),
    "x3p8": (3, 8, 32768, None),
}
METRIC = "cell updates/sec (fp64, 3D Euler p=16) at 1/2/4/8 B200; % of HBM roofline"
MODE_NOTE = {"fast": "fast (QOut and max_eigenvalue within 1e-12 relative of the reference; measured ~1e-16)",
             "exact": "exact (bit-identical to the reference)"}


def _cfg_label(idx) -> str:
    return f"BASELINE configs[{idx}]" if idx is not None else "not a BASELINE config"


def algorithmic_bytes_per_patch(dim: int, p: int) -> int:
    """QIn interior + face halo read, QOut written, 24 B of per-patch scalars."""
    s = dim + 2
    return (p ** dim + 2 * dim * p ** (dim - 1)) * s * 8 + p ** dim * s * 8 + 24


def algorithmic_flops_per_cell(dim: int, p: int) -> float:
    """add/sub/mul/div/sqrt/max = 1 flop (abs = 0) per interior cell update."""
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
    """SM clock and clock-event (throttle) reasons sampled every 5 ms through NVML from a
    thread, over warm-up, the timed steps and the kernel pass (nvidia-smi at 50 ms when
    NVML is unavailable)."""

    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4), ("hw_power_brake_slowdown", 0x80))

    def __init__(self, torch, local: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._h = None
        try:
            import pynvml

            pynvml.nvmlInit()
            uuid = "GPU-" + str(torch.cuda.get_device_properties(local).uuid)
            try:
                self._h = pynvml.nvmlDeviceGetHandleByUUID(uuid)
            except pynvml.NVMLError:
                self._h = pynvml.nvmlDeviceGetHandleByIndex(local)
            self._nv = pynvml
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
        except Exception:   # pragma: no cover - no NVML
            self._h = None
        self.local = local

    def _run_nvml(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(float(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)))
                bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for name, bit in self.REASONS:
                    if bits & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.005)

    def _run_smi(self):
        proc = subprocess.Popen(["nvidia-smi", "-i", str(self.local), "--query-gpu=clocks.sm,clocks.max.sm",
                                 "--format=csv,noheader,nounits", "-lms", "50"],
                                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        self._proc = proc
        for line in proc.stdout:
            try:
                a, b = (float(v) for v in line.split(","))
                self.samples.append(a)
                self.max_mhz = b
            except ValueError:
                pass

    def __enter__(self):
        target = self._run_nvml if self._h is not None else self._run_smi
        self._t = threading.Thread(target=target, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if getattr(self, "_proc", None) is not None:
            self._proc.terminate()
        self._t.join(timeout=5)

    def summary(self):
        load = [s for s in self.samples if self.max_mhz is None or s > 0.5 * self.max_mhz] or self.samples
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples),
                "source": "nvml 5 ms" if self._h is not None else "nvidia-smi 50 ms"}


def pcie_bandwidth(torch, nbytes: int = 256 << 20):
    """Pinned host <-> device copy bandwidth (GB/s): H2D alone, D2H alone, and each direction
    while both run (the e2e pipeline overlaps them).  The e2e roofline."""
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


def host_batch(dim: int, p: int, n: int, seed: int = 7):
    """Synthetic admissible batch on the host: qin, cell_size, dt."""
    import numpy as np

    import oracle

    chunk = max(1, (256 << 20) // ((p + 2) ** dim * (dim + 2) * 8))
    qin = np.empty((n, (p + 2) ** dim * (dim + 2)))
    for lo in range(0, n, chunk):
        qin[lo:lo + chunk] = oracle.synthetic_qin(dim, p, min(chunk, n - lo), seed=seed + lo)
    return qin, np.ones((n, dim)), np.full(n, 0.4 * (1.0 / p) / 3.4)


def oracle_steps(qin, cs, dt, dim, p, steps, warmup, budget_s):
    """Time the oracle port (C, OpenMP, all host threads) stepping over the batch.  A step is
    the full batch when `steps` of them fit the budget, else a rotating contiguous slice of it
    (so no step re-reads a cache-resident sample).  Returns (per-step cells/s list, cores,
    patches per step, per-step ms list)."""
    import oracle

    oracle.build()
    cores = cpu_cores()
    n = qin.shape[0]
    t0 = time.perf_counter()
    oracle.update(dim, p, 1.4, qin[: min(n, 4 * cores)], cs[: min(n, 4 * cores)], dt[: min(n, 4 * cores)],
                  nthreads=cores)
    probe = min(n, 64 * cores)
    t0 = time.perf_counter()
    oracle.update(dim, p, 1.4, qin[:probe], cs[:probe], dt[:probe], nthreads=cores)
    per_patch = (time.perf_counter() - t0) / probe
    m = int(max(1, min(n, budget_s / max(steps + warmup, 1) / per_patch)))
    slices = max(1, n // m)   # every step a full m-patch slice (a ragged tail slice would time mostly overhead)
    rates, ms = [], []
    for k in range(warmup + steps):
        lo = (k % slices) * m
        hi = lo + m
        t0 = time.perf_counter()
        oracle.update(dim, p, 1.4, qin[lo:hi], cs[lo:hi], dt[lo:hi], nthreads=cores)
        el = time.perf_counter() - t0
        if k >= warmup:
            rates.append((hi - lo) * p ** dim / el)
            ms.append(el * 1e3)
    return rates, cores, m, ms


def numpy_engine_baseline(qin, cs, dt, dim, p, reps=3):
    """The reference's own numpy engine (fvbatch, from baseline/_ref), shimmed batched/aos/par
    with worker_hint = the host's cores, 1 warm-up + `reps` timed reps on a
    bounded sample of the batch; None when the reference package is not shipped."""
    import numpy as np

    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "fvbatch")):
        return None
    if path not in sys.path:
        sys.path.append(path)
    try:
        import fvbatch.kernel as rk
        import fvbatch.mesh as rm
        import fvbatch.pde as rp
        from fvbatch.kernel import vectorized
    except Exception as exc:   # pragma: no cover
        return {"unavailable": f"import failed: {exc}"}
    # vectorized.py:254-255 names five undefined module attributes on every BATCHED
    # variant; binding them is the shim SURVEY §8d prescribes
    for name in ("_pass_copy_args", "_pass_eig_args", "_pass_diss_args", "_pass_fluxfill_args",
                 "_pass_fluxacc_args"):
        if not hasattr(vectorized, name):
            setattr(vectorized, name, None)
    cores = cpu_cores()
    m = min(qin.shape[0], 1024 if (dim == 3 and p >= 16) else (16384 if p >= 16 else 65536))
    if os.environ.get("FVB_BENCH_CPU_SMALL"):
        m = min(m, 8)
    spec = rm.PatchSpec(dim, p, dim + 2)
    b = rm.make_patch_batch(spec, m)
    b.QIn[...] = qin[:m]
    b.cell_size[...] = cs[:m]
    b.dt[...] = dt[:m]
    pd = rp.make_euler_pde(dim)
    var = rk.variant_from_labels("batched", "aos", "par", worker_hint=cores)
    rk.update_patch_batch(b, pd, var)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        rk.update_patch_batch(b, pd, var)
        times.append(time.perf_counter() - t0)
    med = statistics.median(times)
    # the best unshimmed public variant, patchwise/aos/seq on one core
    ms_ = min(m, 64 if (dim == 3 and p >= 16) else 256)
    bs = rm.make_patch_batch(spec, ms_)
    bs.QIn[...] = qin[:ms_]
    bs.cell_size[...] = cs[:ms_]
    bs.dt[...] = dt[:ms_]
    vs = rk.variant_from_labels("patchwise", "aos", "seq")
    rk.update_patch_batch(bs, pd, vs)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        rk.update_patch_batch(bs, pd, vs)
        ts.append(time.perf_counter() - t0)
    rm._offset_tensor.cache_clear() if hasattr(rm, "_offset_tensor") else None
    meds = statistics.median(ts)
    return {"value": m * p ** dim / med, "unit": "cell updates/s", "cores": cores, "kind": "reference",
            "sample": f"fvbatch.kernel.update_patch_batch, batched/aos/par worker_hint={cores} (shimmed), "
                      f"{m} patches, median of {reps} after 1 warm-up: {med:.2f} s",
            "unshimmed_seq": {"value": ms_ * p ** dim / meds, "unit": "cell updates/s", "cores": 1,
                              "sample": f"patchwise/aos/seq (no shim), {ms_} patches, median of {reps} after "
                                        f"1 warm-up: {meds:.2f} s"}}


def reference_arm(args):
    """--impl reference: the reference algorithm on this box's host cores, rank 0 only.
    Steps = the oracle port (the reference's update restated in C, OpenMP) over the
    configuration's batch; the reference's own numpy engine is reported beside it."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    dim, p, n, cfg_idx = CONFIGS[args.config]
    if os.environ.get("FVB_BENCH_CPU_SMALL"):   # CPU test suite: a tiny batch
        n = min(n, 64)
    qin, cs, dt = host_batch(dim, p, n)
    budget = float(os.environ.get("FVB_BENCH_CPU_SECONDS", "60"))
    rates, cores, m, ms = oracle_steps(qin, cs, dt, dim, p, args.steps, args.warmup, budget)
    value = statistics.median(rates)
    numpy_ref = None if os.environ.get("FVB_BENCH_NO_NUMPY") else numpy_engine_baseline(qin, cs, dt, dim, p)
    sample = (f"oracle port (C restatement of vectorized.py, OpenMP, {cores} threads): {args.steps} steps of "
              f"{m} patches each ({'the full batch' if m == n else 'rotating slices of the batch'})")
    line = {
        "metric": METRIC, "impl": "reference", "value": value, "unit": "cell updates/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.median(ms), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{dim}D Euler p={p}, {n} patches ({_cfg_label(cfg_idx)})",
                   "dim": dim, "p": p, "patches": n, "patches_per_step": m},
        "cpu_baseline": {"value": value, "unit": "cell updates/s", "cores": cores, "kind": "port", "sample": sample},
        "cpu_baseline_numpy": numpy_ref,
        "e2e": {"value": value, "unit": "cell updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--mode", default="fast", choices=["fast", "exact"])
    ap.add_argument("--layout", default="aos", choices=["aos", "soa"])
    ap.add_argument("--kernel", default="auto", choices=["auto", "fused", "generic"])
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-exact-leg", action="store_true")
    ap.add_argument("--graph", action="store_true",
                    help="replay the timed steps from CUDA graphs (per-launch events then sit inside the graph)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--patches", type=int, default=None, help="override the patches per GPU (overhead studies)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        reference_arm(args)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    import ctypes

    from paper_2302_09005_b200 import _lib as flib_mod
    from paper_2302_09005_b200 import device as fdev
    from paper_2302_09005_b200 import driver, mesh, pde

    flib = flib_mod.load()
    from paper_2302_09005_b200.kernel import update_patch_batch, variant_from_labels

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # FVB_BENCH_DIST=gloo: a functional check of the multi-rank bench on fewer GPUs than ranks
    # (ranks share devices; NCCL refuses that) -- its timings are not scaling numbers
    backend = os.environ.get("FVB_BENCH_DIST", "nccl")
    if backend != "nccl":
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    dim, p, n, cfg_idx = CONFIGS[args.config]
    if args.patches:
        n = args.patches
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
    kernel_name = fdev.selected_kernel(dim, p, n, gamma, args.layout) if args.kernel == "auto" else args.kernel

    def run_mode(mode, steps, warmup, clocks_ok):
        """(total ms of `steps` steps, mean update-launch ms).  Eager launches by default: every
        step's update (fused kernel + its redo pass + the CFL tail) is bracketed by CUDA events
        on the launching stream; --graph replays m-step CUDA graphs with the events inside."""
        stepper = driver.CflStepper(db, cfl=0.4, dx=1.0 / p, kernel=args.kernel, stream=stream, mode=mode,
                                    graph=args.graph)
        stepper.prepass()
        torch.cuda.synchronize()
        if db.nonphysical():
            raise RuntimeError("synthetic input is not admissible")
        # the timed steps: eager -- every step's update launches bracketed by their own event
        # pair; --graph -- m-step graphs (m divides K), the last m steps' pairs read back
        m = max(d for d in range(1, min(steps, 32) + 1) if steps % d == 0)
        graph = None
        if not args.graph:
            m = steps
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(m)]
            for a, b in ev:   # create the events (torch creates them lazily on the first record)
                a.record(stream)
                b.record(stream)
        else:
            graph, ev = stepper.make_graph(m, timing=True)
        for _ in range(warmup):
            stepper.step()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0.record(stream)
        for _ in range(steps // m):
            if graph is not None:
                graph.replay()
                continue
            for a, b in ev:
                # the step's main kernel bracketed by the pair (recorded inside the C ABI around
                # the fused kernel, whose last CTA carries the CFL tail; the redo pass launched
                # after it is excluded): roofline.kernel_ms is "that kernel"
                flib.fvb_time_next_update(ctypes.c_void_p(a.cuda_event), ctypes.c_void_p(b.cuda_event))
                stepper.step()
        t1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        total = t0.elapsed_time(t1)
        kern = statistics.median(a.elapsed_time(b) for a, b in ev)   # per-launch duration (median)
        if world > 1:
            t = torch.tensor([total, kern], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            total, kern = float(t[0]), float(t[1])
        if db.nonphysical():
            raise RuntimeError("non-physical state during the timed steps")
        return total, kern

    peaks, peak_kind = measured_peaks()
    bytes_per_launch = n * algorithmic_bytes_per_patch(dim, p)
    flops_cell = algorithmic_flops_per_cell(dim, p)
    cells_per_gpu = n * p ** dim
    total_cells = n_total * p ** dim

    def roofline(kern_ms):
        achieved = bytes_per_launch / (kern_ms * 1e-3) / 1e9
        return {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "kernel_ms": kern_ms,
                "algorithmic_bytes_per_launch": bytes_per_launch,
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind}, copy bandwidth)",
                "frac_vs_8tbs": achieved / 8000.0}   # also quoted against the nominal 8 TB/s

    with ClockSampler(torch, local) as clocks:
        total_ms, kern_ms = run_mode(args.mode, args.steps, args.warmup, True)
        exact = None
        if args.mode == "fast" and not args.no_exact_leg:
            ex_total, ex_kern = run_mode("exact", args.steps, args.warmup, True)
            exact = {"value": total_cells * args.steps / (ex_total * 1e-3), "ms_per_step": ex_total / args.steps,
                     "roofline": roofline(ex_kern), "mode": MODE_NOTE["exact"]}
    value = total_cells * args.steps / (total_ms * 1e-3)
    ms_per_step = total_ms / args.steps
    roof = roofline(kern_ms)
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                traffic = json.load(f).get(f"{args.config}_{args.layout}_{args.mode}", {}).get("dram_bytes_per_launch")
        except (OSError, ValueError):
            traffic = None
    roof["traffic"] = traffic

    # ---- e2e: the drop-in public API on pinned host buffers ----
    e2e, host = None, None
    if args.e2e_steps > 0 or (rank == 0 and world == 1 and not args.no_cpu_baseline):
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
    if args.e2e_steps > 0:
        euler = pde.make_euler_pde(dim)
        variant = variant_from_labels("batched", "aos", "par")
        for _ in range(2):   # warm-up (workspace allocation, first touch of the pinned pages)
            update_patch_batch(host, euler, variant, mode=args.mode)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            update_patch_batch(host, euler, variant, mode=args.mode)
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

    cpu = cpu_numpy = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        budget = float(os.environ.get("FVB_BENCH_CPU_SECONDS", "10"))
        rates, cores, m, _ = oracle_steps(host.QIn, host.cell_size, host.dt, dim, p, 3, 1, budget)
        cpu = {"value": statistics.median(rates), "unit": "cell updates/s", "cores": cores, "kind": "port",
               "sample": f"oracle port (C, OpenMP, {cores} threads) on this run's batch: 3 steps of {m} patches "
                         f"({'the full batch' if m == n else 'rotating slices'}), median"}
        # the reference's own Python CPU path (north star: "next to the reference Python CPU path
        # timed on the box's own host cores"), on a bounded sample of the same batch
        if not os.environ.get("FVB_BENCH_NO_NUMPY"):
            cpu_numpy = numpy_engine_baseline(host.QIn, host.cell_size, host.dt, dim, p)
    del host

    if rank == 0:
        # fvb_update_cfl: the fused kernel (its CTAs fold max_eig into the running max) and its
        # redo pass (the dt broadcast on one GPU); the generic kernel is followed by one reduce
        # kernel (<= 16,384 patches) or a grid reduce (+ set_dt on one GPU); N GPUs: + set_dt
        if kernel_name == "fused":
            launches_per_step = 2 + (1 if world > 1 else 0)
        else:
            launches_per_step = 1 + (1 if n <= 16384 or world > 1 else 2) + (1 if world > 1 else 0)
        line = {
            "metric": METRIC, "value": value, "unit": "cell updates/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": (f"{dim}D Euler p={p}, {n} patches per GPU ({_cfg_label(cfg_idx)})"
                                    if args.scaling == "weak" else
                                    f"{dim}D Euler p={p}, {n_total} patches over {world} GPU(s) "
                                    f"({_cfg_label(cfg_idx)}, strong scaling)"),
                       "dim": dim, "p": p, "patches_per_gpu": n, "layout": args.layout, "kernel": kernel_name,
                       "mode": MODE_NOTE[args.mode],
                       "step": "CflStepper: fvb_update_cfl (update, redo pass with the max-reduce/dt) "
                               "(+ NCCL MAX all-reduce + set_dt)"
                               + (", CUDA-graph replay" if args.graph else ""),
                       "parallelism": f"patch shards x{world}, NCCL MAX all-reduce of the wave speed",
                       "l2": f"inputs {n * spec.haloed_volumes * spec.unknowns * 8 / 1e6:.0f} MB vs 126 MB L2; "
                             "no flush"},
            "roofline": roof,
            # the min(HBM, FP64) roofline of the north star: the FP64 side at the algorithmic flop count
            "roofline_fp64": {"achieved": flops_cell * cells_per_gpu / (kern_ms * 1e-3) / 1e12,
                              "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                              "frac": flops_cell * cells_per_gpu / (kern_ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
                              "flops_per_cell": flops_cell},
            "exact": exact,
            "cpu_baseline": cpu,
            "cpu_baseline_numpy": cpu_numpy,
            "e2e": e2e,
            # per timed step: the update kernel (+ the fused path's redo pass) and the dt reduction
            # (one kernel up to 16,384 patches on one GPU, else reduce + set_dt)
            "gpu_launches": args.steps * launches_per_step,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
