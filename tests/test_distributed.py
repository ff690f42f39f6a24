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


def _exchange_worker(rank, world, port, n, out):
    """the row-panel PCG's all-gather hook (screenbem.allgather_exchange) on gloo, with
    host buffers standing in for the device vectors"""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import numpy as np
    import torch
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2310_09204_b200 import screenbem as S
    full = np.arange(1.0, n + 1.0) * 0.5
    y = np.full(n, -1.0)  # only this rank's panel is filled, as after its row kernel
    lo, hi = S.row_ranges(n, world)[rank]
    y[lo:hi] = full[lo:hi]
    keep = {}

    def wrap(ptr, m):
        assert ptr == y.ctypes.data and m == n
        keep["t"] = torch.from_numpy(y)
        return keep["t"]
    ex = S.allgather_exchange(dist, rank, world, n, wrap=wrap)
    ex(0, y.ctypes.data, n, 0)
    first = np.abs(y - full).max()
    y[:] = -1.0
    y[lo:hi] = 2 * full[lo:hi]
    ex(0, y.ctypes.data, n, 0)  # reused staging buffers
    out[rank] = (first, np.abs(y - 2 * full).max())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world,n", [(2, 11), (3, 10), (2, 1)])
def test_row_panel_exchange_gloo(world, n):
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_exchange_worker, args=(world, port, n, out), nprocs=world, join=True)
    for rank in range(world):
        assert out[rank] == (0.0, 0.0)


def test_row_ranges():
    from paper_2310_09204_b200 import screenbem as S
    assert S.row_ranges(10, 3) == [(0, 4), (4, 8), (8, 10)]
    assert S.row_ranges(3969, 8)[-1] == (3479, 3969)
    assert S.row_ranges(2, 4) == [(0, 1), (1, 2), (2, 2), (2, 2)]
    assert S.row_ranges(0, 2) == [(0, 0), (0, 0)]
    for n, w in [(25281, 8), (7, 7), (100, 3)]:
        rr = S.row_ranges(n, w)
        assert rr[0][0] == 0 and rr[-1][1] == n and all(a[1] == b[0] for a, b in zip(rr, rr[1:]))


def test_single_rank_passthrough():
    import bench
    assert bench.reduce_max([3.0, 4.0]) == [3.0, 4.0]


def _agree_worker(rank, world, port, out):
    """the collective stop of the row-panel PCG (screenbem.allreduce_agree): ranks stop
    only when every rank's local flag says stop (a rank whose state differs in
    the last bits must not stop early and leave the others waiting in an all-gather)"""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2310_09204_b200 import screenbem as S
    agree = S.allreduce_agree(dist)
    res = [agree(1), agree(1 if rank == 0 else 0), agree(0 if rank == 0 else 1), agree(0)]
    out[rank] = res
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_row_panel_collective_stop_gloo():
    world, port = 2, _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_agree_worker, args=(world, port, out), nprocs=world, join=True)
    for rank in range(world):
        assert out[rank] == [1, 0, 0, 0]


@pytest.mark.timeout(600)
def test_bench_gpus_flag_launches_ranks():
    """`bench.py --gpus 2` with no launcher re-executes itself under torch.distributed.run
    with two ranks; the reference arm runs on rank 0 only (one JSON line) and reports
    n_gpus 2 (the driver's SCALE command for the reference arm)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--config", "1", "--steps", "1", "--warmup", "0", "--cpu-seconds", "1", "--no-cpu-phases"],
                       capture_output=True, text=True, timeout=550, cwd=root, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2


def test_bench_world_size_mismatch_fails():
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--gpus", "4"],
                       capture_output=True, text=True, timeout=120, cwd=root, env=env)
    assert r.returncode != 0 and "WORLD_SIZE=2" in r.stderr
