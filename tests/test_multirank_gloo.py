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


def _ghost_worker(rank, world, port, periodic, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2302_09005_b200 import driver

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n_layers, le = 7, 5                      # global layers of a sharded grid, values per layer
    l0, l1 = driver.shard_bounds(n_layers, rank, world)
    own = torch.cat([torch.full((le,), 100.0 * layer) + torch.arange(le) for layer in range(l0, l1)])
    lo, hi = driver._neighbours(rank, world, periodic)
    g_lo = torch.full((le,), -1.0) if lo is not None else None
    g_hi = torch.full((le,), -1.0) if hi is not None else None
    driver.exchange_ghost_layers(own, le, g_lo, g_hi, rank, world, periodic)
    out[rank] = (l0, l1, None if g_lo is None else g_lo.tolist(), None if g_hi is None else g_hi.tolist())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,periodic", [(2, True), (2, False), (3, True), (3, False)])
def test_ghost_layer_exchange(world, periodic):
    """driver.exchange_ghost_layers: each rank's lower ghost is the lower neighbour's last
    layer and its upper ghost the upper neighbour's first layer (wrapping when periodic;
    none at a non-periodic edge), including two ranks that are each other's both neighbours."""
    n_layers, le = 7, 5
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_ghost_worker, args=(world, _free_port(), periodic, out), nprocs=world, join=True)
    layer = lambda z: [100.0 * (z % n_layers) + i for i in range(le)]  # noqa: E731
    for r in range(world):
        l0, l1, g_lo, g_hi = out[r]
        if periodic or r > 0:
            assert g_lo == layer(l0 - 1), (r, g_lo)
        else:
            assert g_lo is None
        if periodic or r < world - 1:
            assert g_hi == layer(l1), (r, g_hi)
        else:
            assert g_hi is None
