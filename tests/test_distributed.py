"""N > 1 paths of bench.py on CPU (gloo, world_size 2): replicas — each rank runs the
whole step on its own GPU and ranks meet only at the barrier and the max-over-ranks
reduction of the device timings — and --shard, whose partial W are summed in place
over the ranks."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import bench
    r, w, lr = bench.dist_env()
    assert (r, w, lr) == (rank, world, rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dist.barrier()
    vals = bench.reduce_max([1.0 + rank, 10.0 - rank, 0.5 * rank], dist, "cpu")
    # --shard: each rank holds a partial W (its share of the pair work); the in-place sum
    # over ranks gives every rank the full W
    import numpy as np
    import torch
    rng = np.random.default_rng(5)
    full = rng.standard_normal((6, 8))
    parts = [np.where(rng.random((6, 8)) < 0.5, full, 0.0) for _ in range(world - 1)]
    parts.append(full - sum(parts))
    t = torch.from_numpy(parts[rank].copy())
    bench.allreduce_sum_(t, dist, "cpu")
    out[rank] = (vals, np.abs(t.numpy() - full).max())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gloo_max_over_ranks():
    world, port = 2, _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    for rank in range(world):
        vals, err = out[rank]
        assert vals == [2.0, 10.0, 0.5]
        assert err < 1e-14


def test_single_rank_passthrough():
    import bench
    assert bench.reduce_max([3.0, 4.0]) == [3.0, 4.0]
