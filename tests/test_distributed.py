"""N > 1 path of bench.py on CPU (gloo, world_size 2): replicas only — each rank
runs the whole step on its own GPU; ranks meet only at the barrier and the
max-over-ranks reduction of the device timings."""
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
    out[rank] = vals
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gloo_max_over_ranks():
    world, port = 2, _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    for rank in range(world):
        assert out[rank] == [2.0, 10.0, 0.5]


def test_single_rank_passthrough():
    import bench
    assert bench.reduce_max([3.0, 4.0]) == [3.0, 4.0]
