"""Condition-number path on the device (reference
inc/schwarz.hpp:142-190) against the oracle's restatement (materialize by n applies,
Cholesky congruence L^T M L, dense symmetric eigensolve)."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
S = pytest.importorskip("paper_2310_09204_b200.screenbem")


@pytest.fixture(scope="module")
def ctx():
    return S.Context(0)


def omesh(m):
    return O.Mesh(m.vertices, m.facets)


def level(cfg):
    pair = S.make_config(cfg)
    fine, coarse = S.inflate(pair.fine, validate=False), S.inflate(pair.coarse)
    opair = O.LevelPair(omesh(pair.coarse), omesh(pair.fine), pair.parent)
    ofine, ocoarse = O.inflate(opair.fine, validate=False), O.inflate(opair.coarse)
    return pair, fine, coarse, opair, ofine, ocoarse


def bowtie_level():
    """proj/test_output.txt:31 golden: bow-tie, coarse = base, H/h = 16, 465 DOFs."""
    base = S.make_builtin("bowtie")
    pair = S.refine_uniform_times(base, 4)
    fine, coarse = S.inflate(pair.fine, validate=False), S.inflate(pair.coarse)
    opair = O.LevelPair(omesh(pair.coarse), omesh(pair.fine), pair.parent)
    ofine, ocoarse = O.inflate(opair.fine, validate=False), O.inflate(opair.coarse)
    return pair, fine, coarse, opair, ofine, ocoarse


@pytest.mark.parametrize("mode", ["inverse", "trsv", "factored"])
@pytest.mark.parametrize("which", ["cfg1", "bowtie"])
def test_materialize_matches_oracle(ctx, mode, which):
    pair, fine, coarse, opair, ofine, ocoarse = level(1) if which == "cfg1" else bowtie_level()
    W = S.assemble_W(fine, ctx=ctx)
    prec = S.build_preconditioner(W, S.partition_dofs(pair, fine), S.build_prolongation(pair, coarse, fine), mode=mode)
    M = S.materialize_preconditioner(prec)
    oprec = O.build_preconditioner(W.download(), O.partition_dofs(opair, ofine),
                                   O.build_prolongation(opair, ocoarse, ofine))
    Mo = O.materialize_preconditioner(oprec)
    assert np.abs(M - Mo).max() <= 1e-12 * np.abs(Mo).max()
    # columns are apply(e_j) of the device preconditioner itself
    for j in (0, fine.n // 2, fine.n - 1):
        e = np.zeros(fine.n)
        e[j] = 1.0
        assert np.abs(M[:, j] - prec.apply(e)).max() <= 1e-12 * np.abs(Mo).max()


@pytest.mark.parametrize("which", ["cfg1", "bowtie"])
def test_condition_numbers_match_dense_eigensolve(ctx, which):
    pair, fine, coarse, opair, ofine, ocoarse = level(1) if which == "cfg1" else bowtie_level()
    W = S.assemble_W(fine, ctx=ctx)
    prec = S.build_preconditioner(W, S.partition_dofs(pair, fine), S.build_prolongation(pair, coarse, fine))
    Wh = W.download()
    oprec = O.build_preconditioner(Wh, O.partition_dofs(opair, ofine), O.build_prolongation(opair, ocoarse, ofine))
    raw, raw_o = S.condition_number(W), O.condition_number(Wh)
    sp, sp_o = S.condition_number(W, prec), O.condition_number(Wh, oprec)
    for got, want in ((raw, raw_o), (sp, sp_o)):
        assert got.converged
        assert got.lambda_min == pytest.approx(want[0], rel=1e-9)
        assert got.lambda_max == pytest.approx(want[1], rel=1e-9)
        assert got.kappa == pytest.approx(want[2], rel=1e-9)
    # condition_number(W, M) with the materialized M (schwarz.hpp:174-183) agrees
    spm = S.condition_number(W, S.materialize_preconditioner(prec))
    assert spm.kappa == pytest.approx(sp_o[2], rel=1e-9)
    if which == "bowtie":  # proj/test_output.txt:31
        assert fine.n == 465
        assert round(sp.kappa, 2) == 6.93
        assert round(raw.kappa, 2) == 12.96


def test_condition_number_config2(ctx):
    """3969 DOFs: Lanczos extremes vs the dense eigensolve of the oracle."""
    pair, fine, coarse, opair, ofine, ocoarse = level(2)
    W = S.assemble_W(fine, ctx=ctx)
    prec = S.build_preconditioner(W, S.partition_dofs(pair, fine), S.build_prolongation(pair, coarse, fine))
    Wh = W.download()
    oprec = O.build_preconditioner(Wh, O.partition_dofs(opair, ofine), O.build_prolongation(opair, ocoarse, ofine))
    sp, sp_o = S.condition_number(W, prec), O.condition_number(Wh, oprec)
    raw, raw_o = S.condition_number(W), O.condition_number(Wh)
    assert sp.kappa == pytest.approx(sp_o[2], rel=1e-8)
    assert raw.kappa == pytest.approx(raw_o[2], rel=1e-8)
    assert sp.kappa < raw.kappa


def test_condition_number_errors(ctx):
    pair, fine, coarse, *_ = level(1)
    W = S.assemble_W(fine, ctx=ctx)
    with pytest.raises(S.ValidationError):
        S.condition_number(W, np.eye(fine.n + 1))
