"""Sharded assembly of one W (multi-GPU assembly), checked on one GPU:
the world shards of AssemblyPlan.run(shard=(rank, world)) sum entrywise to the full W,
as the reference's per-worker partial matrices do (inc/assemble.hpp:91-133), and the
in-place device reduction through __cuda_array_interface__ (what bench.py --shard
hands to NCCL) reproduces the sum."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
S = pytest.importorskip("paper_2310_09204_b200.screenbem")


@pytest.fixture(scope="module")
def ctx():
    return S.Context(0)


@pytest.mark.parametrize("spec", ["config1", "bowtie:3"])
def test_shards_sum_to_full_W(ctx, spec):
    m = S.make_config(1).fine if spec == "config1" else S.make_builtin(spec)
    im = S.inflate(m)
    plan = S.AssemblyPlan(im, ctx=ctx)
    full = plan.run()
    Wf = full.download()
    scale = np.abs(Wf).max()
    for world in (2, 3, 5):
        parts = [plan.run(shard=(r, world)) for r in range(world)]
        Ws = sum(p.download() for p in parts)
        # the reference's own worker-reorder bound (tests/test_assemble.cpp:271-279)
        assert np.abs(Ws - Wf).max() <= 1e-13 * scale, (world, np.abs(Ws - Wf).max() / scale)
        assert np.array_equal(Ws, Ws.T)
        for k in ("identical", "edge", "vertex", "near_pairs", "tiles", "tiles_skipped"):
            assert sum(p.stats[k] for p in parts) == full.stats[k], k
        assert all(p.stats["far_pairs"] == -1 for p in parts)
        # every shard is non-trivial
        assert all(np.abs(p.download()).max() > 0 for p in parts)


def test_device_reduction_through_array_interface(ctx):
    torch = pytest.importorskip("torch")
    im = S.inflate(S.make_builtin("bowtie:3"))
    plan = S.AssemblyPlan(im, ctx=ctx)
    Wf = plan.run().download()
    a, b = plan.run(shard=(0, 2)), plan.run(shard=(1, 2))
    ta = torch.as_tensor(a, device="cuda:0")
    tb = torch.as_tensor(b, device="cuda:0")
    assert ta.shape[0] == a.n and ta.shape[1] >= a.n and ta.dtype == torch.float64
    ta += tb  # in place on W's own storage
    torch.cuda.synchronize()
    Wa = a.download()
    assert np.abs(Wa - Wf).max() <= 1e-13 * np.abs(Wf).max()
    assert np.array_equal(Wa, Wa.T)
    assert not ta[:, a.n:].any()  # padding columns stay zero


def test_bad_shard_is_a_validation_error(ctx):
    plan = S.AssemblyPlan(S.inflate(S.make_builtin("bowtie:1")), ctx=ctx)
    for shard in ((2, 2), (-1, 2), (0, 0)):
        with pytest.raises(S.ValidationError, match="shard"):
            plan.run(shard=shard)


def test_packed_upper_triangle_roundtrip_and_shard_sum():
    """The multi-GPU reduction sums only W's upper triangle (sbg_matrix_pack_upper /
    unpack_upper): the round trip gives W back bit for bit, and packed shard sums equal the
    full W within the reorder bound."""
    import torch
    ctx = S.Context(0)
    im = S.inflate(S.make_config(2).fine)
    n = im.n
    plan = S.AssemblyPlan(im, ctx=ctx)
    W = plan.run()
    Wh = W.download()
    packed = torch.empty(n * (n + 1) // 2, dtype=torch.float64, device="cuda:0")
    W.pack_upper(packed.data_ptr())
    ctx.synchronize()
    iu = np.triu_indices(n)
    assert np.array_equal(packed.cpu().numpy(), Wh[iu])
    W2 = S.GalerkinMatrix.from_host(np.zeros((n, n)), ctx)
    W2.unpack_upper(packed.data_ptr())
    assert np.array_equal(W2.download(), Wh)
    acc = torch.zeros_like(packed)
    for r in range(3):
        Ws = plan.run(shard=(r, 3))
        Ws.pack_upper(packed.data_ptr())
        ctx.synchronize()
        acc += packed
    W2.unpack_upper(acc.data_ptr())
    ctx.synchronize()
    Wsum = W2.download()
    assert np.abs(Wsum - Wh).max() <= 1e-13 * np.abs(Wh).max()
    assert np.array_equal(Wsum, Wsum.T)


def _shard_worker(rank, world, port, spec, out):
    """one rank of a sharded assembly: its share of the pair work on the (shared) GPU, the
    partial W reduced over the ranks with gloo through host memory (bench.allreduce_sum_)"""
    import os
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    import bench
    from paper_2310_09204_b200 import screenbem as S2
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ctx = S2.Context(0)
    m = S2.make_config(1).fine if spec == "config1" else S2.make_builtin(spec)
    plan = S2.AssemblyPlan(S2.inflate(m), ctx=ctx)
    W = plan.run(shard=(rank, world))
    t = torch.from_numpy(W.download())
    bench.allreduce_sum_(t, dist, "cpu")
    out[rank] = t.numpy()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("spec", ["config1", "bowtie:3"])
def test_two_process_sharded_assembly_gloo(ctx, spec):
    """Two processes (gloo, world size 2, both on this GPU) each assemble their shard and
    sum the partial W over the ranks: every rank ends with the single-process W within
    the reference's worker-reorder bound (tests/test_assemble.cpp:271-279)."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    m = S.make_config(1).fine if spec == "config1" else S.make_builtin(spec)
    Wf = S.AssemblyPlan(S.inflate(m), ctx=ctx).run().download()
    out = mp.Manager().dict()
    mp.spawn(_shard_worker, args=(2, port, spec, out), nprocs=2, join=True)
    for rank in range(2):
        Wr = out[rank]
        assert np.abs(Wr - Wf).max() <= 1e-13 * np.abs(Wf).max(), (rank, np.abs(Wr - Wf).max())
        assert np.array_equal(Wr, Wr.T)
