"""world_size-2 CPU test (gloo) of the multi-GPU step's host logic: contiguous patch
shards and the single MAX all-reduce of the wave speed (driver.allreduce_max_)."""

import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2302_09005_b200 import driver

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = driver.shard_bounds(n, rank, world)
    # per-patch wave speeds of this rank's shard (global patch id based, so the max is known)
    local = torch.tensor([float(max(range(lo, hi), key=lambda i: (i * 37) % 101) * 37 % 101)], dtype=torch.float64)
    driver.allreduce_max_(local)
    out[rank] = (lo, hi, float(local.item()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_cfl_exchange():
    n, world = 1001, 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), n, out), nprocs=world, join=True)
    spans = sorted((out[r][0], out[r][1]) for r in range(world))
    assert spans[0][0] == 0 and spans[-1][1] == n and spans[0][1] == spans[1][0]
    expect = float(max((i * 37) % 101 for i in range(n)))
    assert all(out[r][2] == expect for r in range(world))
