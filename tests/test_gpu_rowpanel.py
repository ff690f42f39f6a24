"""Row-panel PCG (W by row panels, one all-gather of W p per iteration) on one
GPU.  Ranks cannot be stood in for on one device (their collectives would wait on each
other), so the panels are checked two ways:
  * emulated exchange: one process owns panel r and its exchange hook computes the other
    panels' rows with the same row kernel on the same stream — the result must equal the
    single-GPU pcg bitwise when that runs the full-matrix form (matvec_form "full", n <= 8000:
    the same row kernel), and the default symmetric-form pcg (upper triangle only) or the
    column-sum form (larger n) to the PCG tolerances;
  * the real torch.distributed exchange (NCCL, world size 1) on the PCG's own stream.
The two-rank exchange logic itself is covered on CPU with gloo (tests/test_distributed.py).
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

S = pytest.importorskip("paper_2310_09204_b200.screenbem")


@pytest.fixture(scope="module")
def ctx():
    return S.Context(0)


@pytest.fixture
def full_form(ctx):
    """pcg with the full-matrix form (the row kernel the panels share) for this test"""
    ctx.matvec_form = "full"
    yield ctx
    ctx.matvec_form = "symmetric"


def system(ctx, cfg=1, kind=None, m=0, r=0):
    pair = S.make_config(cfg) if kind is None else S.make_panels(kind, m, r)
    fine, coarse = S.inflate(pair.fine), S.inflate(pair.coarse)
    W = S.assemble_W(fine, ctx=ctx)
    g = S.config_g(cfg) if kind is None else [0.0, 0.0, 1.0]
    L = S.assemble_rhs(fine, g, ctx=ctx)
    prec = S.build_preconditioner(W, S.partition_dofs(pair, fine), S.build_prolongation(pair, coarse, fine))
    return W, L, prec


def emulated(W, world, rank):
    """exchange hook of `rank`: the other ranks' rows computed here (same kernel, same stream)"""
    ranges = S.row_ranges(W.n, world)
    calls = []

    def exchange(d_p, d_y, n, stream):
        assert n == W.n and stream == W.ctx.stream
        for r, (lo, hi) in enumerate(ranges):
            if r != rank:
                S.matvec_rows_device(W, d_p, d_y, lo, hi)
        calls.append(1)
    return ranges[rank], exchange, calls


@pytest.mark.parametrize("cfg", [1, 2])
@pytest.mark.parametrize("world,rank", [(1, 0), (2, 0), (2, 1), (3, 2), (8, 5)])
def test_row_panels_equal_pcg_bitwise(full_form, cfg, world, rank):
    ctx = full_form
    W, L, prec = system(ctx, cfg)
    ref = S.pcg(W, prec, L, 1e-8)
    rows, ex, calls = emulated(W, world, rank)
    rep = S.pcg_rows(W, prec, L, rows, ex, 1e-8)
    assert rep.converged and rep.iterations == ref.iterations
    assert np.array_equal(rep.solution, ref.solution)
    assert np.array_equal(rep.residual_history, ref.residual_history)
    assert len(calls) >= rep.iterations  # one exchange per enqueued iteration


@pytest.mark.parametrize("world,rank", [(2, 1), (4, 3)])
def test_row_panels_match_symmetric_form_pcg(ctx, world, rank):
    # config 2 (n = 3969 >= 2048): pcg's default matvec reads the upper triangle only
    assert ctx.matvec_form == "symmetric"
    W, L, prec = system(ctx, 2)
    ref = S.pcg(W, prec, L, 1e-8)
    rows, ex, _ = emulated(W, world, rank)
    rep = S.pcg_rows(W, prec, L, rows, ex, 1e-8)
    assert rep.converged and abs(rep.iterations - ref.iterations) <= 1
    assert np.linalg.norm(rep.solution - ref.solution) / np.linalg.norm(ref.solution) < 1e-8


def test_row_panels_large_n_column_form_reference(ctx):
    # n = 9801 > 8000: pcg's matvec is the column-sum form, the panels use the row kernel
    W, L, prec = system(ctx, kind=0, m=100, r=10)
    assert W.n > 8000
    ref = S.pcg(W, prec, L, 1e-8)
    rows, ex, _ = emulated(W, 4, 1)
    rep = S.pcg_rows(W, prec, L, rows, ex, 1e-8)
    assert rep.converged and abs(rep.iterations - ref.iterations) <= 1
    assert np.linalg.norm(rep.solution - ref.solution) / np.linalg.norm(ref.solution) < 1e-8


def test_row_panels_unpreconditioned_and_edges(full_form):
    ctx = full_form
    W, L, prec = system(ctx, 1)
    ref = S.pcg(W, None, L, 1e-8)
    rows, ex, _ = emulated(W, 2, 1)
    rep = S.pcg_rows(W, None, L, rows, ex, 1e-8)
    assert rep.iterations == ref.iterations and np.array_equal(rep.solution, ref.solution)
    # zero RHS: converged at iteration 0 (tests/test_experiments.cpp:64-75)
    z = S.pcg_rows(W, prec, np.zeros(W.n), rows, ex, 1e-8)
    assert z.iterations == 0 and z.converged and not z.solution.any()
    # a failing exchange aborts the solve with its own exception
    def bad(*a):
        raise RuntimeError("link down")
    with pytest.raises(RuntimeError, match="link down"):
        S.pcg_rows(W, prec, L, rows, bad, 1e-8)
    with pytest.raises(S.ValidationError):
        S.pcg_rows(W, prec, L, (0, W.n + 1), ex, 1e-8)
    with pytest.raises(S.ValidationError):
        S.pcg_rows(W, prec, L[:-1], rows, ex, 1e-8)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_nccl_exchange_world1_on_pcg_stream(ctx):
    """the torch.distributed all-gather hook on the device, enqueued on the PCG stream"""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        ctx.matvec_form = "full"  # bitwise against the row kernel
        W, L, prec = system(ctx, 2)
        ref = S.pcg(W, prec, L, 1e-8)
        ex = S.allgather_exchange(dist, 0, 1, W.n, device="cuda:0")
        rep = S.pcg_rows(W, prec, L, S.row_ranges(W.n, 1)[0], ex, 1e-8)
        assert rep.iterations == ref.iterations and np.array_equal(rep.solution, ref.solution)
    finally:
        ctx.matvec_form = "symmetric"
        dist.destroy_process_group()
