"""Multi-GPU multi-step run over a sharded patch grid (driver.run_simulation_sharded),
one process per GPU:

    python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \\
        --master-port 29600 scripts/run_sharded.py --dim 3 --p 16 --grid 16,16,16 --steps 20 --check

Each rank owns whole z-layers (y-rows in 2D) of the grid and swaps one boundary layer with
each neighbour per step (NCCL send/recv).  --check gathers the final field on rank 0 and
compares it bit for bit with the single-GPU run_simulation of the whole grid there.
"""
import argparse
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_09005_b200 import device, driver, mesh, pde  # noqa: E402


def initial_field(dim, p, grid, seed=3):
    """Smooth density wave on a moving background: interior QOut of every patch (x fastest)."""
    n = int(np.prod(grid))
    e = [np.arange(g * p) for g in grid]
    coords = np.meshgrid(*e[::-1], indexing="ij")[::-1]          # x, y[, z] of every global volume
    rho = 1.0 + 0.2 * np.sin(2 * np.pi * coords[0] / (grid[0] * p))
    vel = [0.3, -0.2, 0.1][:dim]
    q = np.empty(rho.shape + (dim + 2,))
    q[..., 0] = rho
    for a in range(dim):
        q[..., 1 + a] = rho * vel[a]
    q[..., -1] = 1.0 / 0.4 + 0.5 * rho * sum(v * v for v in vel)
    # global volume array -> per-patch interior blocks, patch index x fastest
    blocks = q.reshape(*[x for g in grid[::-1] for x in (g, p)], dim + 2)
    axes = list(range(0, 2 * dim, 2)) + list(range(1, 2 * dim, 2)) + [2 * dim]
    return np.ascontiguousarray(blocks.transpose(axes)).reshape(n, -1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=3)
    ap.add_argument("--p", type=int, default=16)
    ap.add_argument("--grid", default="16,16,16")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--aperiodic", action="store_true")
    ap.add_argument("--check", action="store_true")
    a = ap.parse_args()
    grid = tuple(int(g) for g in a.grid.split(","))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    backend = os.environ.get("FVB_BENCH_DIST", "nccl")   # gloo: ranks may share a GPU (functional check)
    if backend != "nccl":
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    spec = mesh.PatchSpec(a.dim, a.p, a.dim + 2)
    field = initial_field(a.dim, a.p, grid)
    sg = driver.ShardedGrid(spec, grid, 1.4, periodic=not a.aperiodic)
    sg.db.QOut.copy_(torch.from_numpy(field[sg.patch_lo:sg.patch_hi].reshape(-1).copy()))
    sg.db.cell_size.fill_(1.0 / grid[0])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = driver.run_simulation_sharded(sg, a.steps)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    if sg.rank == 0:
        cells = int(np.prod(grid)) * a.p ** a.dim
        print(f"{sg.world} GPU(s), grid {grid} p={a.p}: {a.steps} steps in {wall:.3f} s, "
              f"{cells * a.steps / wall / 1e9:.2f} Gcell/s (wall, incl. the first-step pre-pass); "
              f"totals drift {abs(res.totals[-1][0] - res.totals[0][0]) / abs(res.totals[0][0]):.2e}")
    if a.check:
        if sg.world > 1:   # shards differ by at most one layer: pad, all-gather, trim
            sizes = [None] * sg.world
            dist.all_gather_object(sizes, sg.db.QOut.numel())
            pad = torch.zeros(max(sizes), dtype=torch.float64, device="cuda")
            pad[:sg.db.QOut.numel()] = sg.db.QOut
            buf = [torch.empty_like(pad) for _ in range(sg.world)]
            dist.all_gather(buf, pad)
            parts = [b[:sz] for b, sz in zip(buf, sizes)]
        else:
            parts = [sg.db.QOut]
        if sg.rank == 0:
            got = torch.cat(parts).cpu().numpy()
            n = int(np.prod(grid))
            db = device.DeviceBatch(spec, n, 1.4)
            db.QOut.copy_(torch.from_numpy(field.reshape(-1).copy()))
            db.cell_size.fill_(1.0 / grid[0])
            driver.run_simulation(db, grid, a.steps, periodic=not a.aperiodic)
            ref = db.QOut.cpu().numpy()
            ok = np.array_equal(got.view(np.uint64), ref.view(np.uint64))
            print("check vs single-GPU run_simulation:", "bit-identical" if ok else "MISMATCH")
            if not ok:
                sys.exit(1)
    if dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
