"""Full-size parity on the BASELINE configs 3-5 (GPU, `-m gpu`).

Dense oracle assembly of a 12k-25k DOF matrix is out of reach for a CPU test, so
at full size parity goes through size-independent properties and sampled
restatements:
  * W is exactly symmetric and matches the oracle's restated rows
    (`assemble_W_rows`, the reference loop restricted to the sampled rows) per entry
    to 1e-10 |W| + 1e-13 max|W|;
  * the oracle's own Schwarz preconditioner and PCG, run on the GPU-assembled W
    (downloaded), reproduce the device PCG: iterations within +-1, solution within
    1e-8, and the device preconditioner apply matches to 1e-11;
  * DOF numbering / partition / prolongation at these sizes are covered bit-exactly
    on the CPU side (tests/test_host_parity.py).
"""
import os

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
S = pytest.importorskip("paper_2310_09204_b200.screenbem")
WORKERS = os.cpu_count() or 1


@pytest.fixture(scope="module")
def ctx():
    return S.Context(0)


def omesh(m):
    return O.Mesh(m.vertices, m.facets)


@pytest.mark.parametrize("cfg,ratio,rows", [
    (3, 0, [0, 1, 46, 47, 3000, 6720]),      # junction DOFs (q = 3) sit next to the shared edge
    (4, 0, [0, 3000, 6048, 6049, 12096]),    # 6048/6049: DOFs of the origin vertex (q = 8)
    (5, 40, [0, 12640, 25280]),              # corner rows: the farthest, most cancelling entries
])
def test_fullsize_W_symmetric_and_sampled_rows(ctx, cfg, ratio, rows):
    """Both far-field paths: the fast one (distance expansion + refined rsqrt) and the
    SURVEY Appendix B parity-gate path (exact_far: far pairs bitwise the oracle's)."""
    pair = S.make_config(cfg, ratio)
    im = S.inflate(pair.fine, validate=False)
    rows = np.array([r for r in rows if r < im.n], dtype=np.int32)
    oim = O.inflate(omesh(pair.fine), validate=False)
    Wo = O.assemble_W_rows(oim, rows, workers=WORKERS)
    scale = np.abs(Wo).max()
    for exact in (False, True):
        W = S.assemble_W(im, S.QuadratureConfig(exact_far=exact), ctx=ctx)
        assert W.symmetry_defect() == 0.0
        Wg = W.rows(rows)
        bad = np.abs(Wg - Wo) > 1e-10 * np.abs(Wo) + 1e-13 * scale
        assert not bad.any(), (exact, bad.sum(), np.abs(Wg - Wo).max() / scale)
        del W


@pytest.mark.parametrize("cfg,ratio", [(3, 0), (4, 0), (5, 40)])
def test_fullsize_pcg_matches_oracle_on_device_W(ctx, cfg, ratio):
    pair = S.make_config(cfg, ratio)
    fine, coarse = S.inflate(pair.fine, validate=False), S.inflate(pair.coarse)
    g = S.config_g(cfg)
    W = S.assemble_W(fine, ctx=ctx)
    L = S.assemble_rhs(fine, g, ctx=ctx)
    part, P = S.partition_dofs(pair, fine), S.build_prolongation(pair, coarse, fine)
    prec = S.build_preconditioner(W, part, P)
    rep = S.pcg(W, prec, L, 1e-8)
    assert rep.converged
    # oracle on the same matrix and right-hand side
    Wh = W.download()
    opair = O.LevelPair(omesh(pair.coarse), omesh(pair.fine), pair.parent)
    ofine, ocoarse = O.inflate(opair.fine, validate=False), O.inflate(opair.coarse)
    oprec = O.build_preconditioner(Wh, O.partition_dofs(opair, ofine), O.build_prolongation(opair, ocoarse, ofine))
    r = O.normal_draws(17, fine.n)
    z, zo = prec.apply(r), oprec.apply(r)
    assert np.abs(z - zo).max() <= 1e-11 * np.abs(zo).max()
    Lo = O.assemble_rhs(ofine, g)
    np.testing.assert_allclose(L, Lo, rtol=1e-12, atol=1e-15 * np.abs(Lo).max())
    orep = O.pcg(Wh, oprec, Lo, 1e-8)
    assert orep.converged
    assert abs(rep.iterations - orep.iterations) <= 1, (rep.iterations, orep.iterations)
    xerr = np.linalg.norm(rep.solution - orep.solution) / np.linalg.norm(orep.solution)
    assert xerr <= 1e-8, xerr


def test_config2_full_W_every_entry(ctx):
    """The bench workload (BASELINE configs[1]): all 15.75M entries of the device W against
    the oracle's full assemble_W (all host threads, ~15 s), per entry, with the worst
    entries reported both ways."""
    pair = S.make_config(2)
    im = S.inflate(pair.fine)
    Wg = S.assemble_W(im, ctx=ctx).download()
    Wo = O.assemble_W(O.inflate(omesh(pair.fine)), workers=WORKERS)
    scale = np.abs(Wo).max()
    err = np.abs(Wg - Wo)
    bad = err > 1e-10 * np.abs(Wo) + 1e-13 * scale
    rel = err / np.maximum(np.abs(Wo), 1e-300)
    assert not bad.any(), (bad.sum(), err.max() / scale, rel.max())
    assert err.max() / scale < 1e-12, err.max() / scale      # norm-relative: far below 1e-10
    assert np.array_equal(Wg, Wg.T)


def test_beyond_configs_size_independent_properties(ctx):
    """A flat 200x200 screen (80 000 triangles, 39 601 DOFs, 12.5 GB W) — larger than any
    BASELINE config: W exactly symmetric, PCG converges, and the returned solution's true
    residual ||b - W x|| (device matvec, independent of the PCG recurrences) is consistent
    with the stopping rule."""
    pair = S.make_panels(0, 200, 20)
    fine, coarse = S.inflate(pair.fine, validate=False), S.inflate(pair.coarse)
    W = S.assemble_W(fine, ctx=ctx)
    assert W.n == 39601 and W.symmetry_defect() == 0.0
    L = S.assemble_rhs(fine, [0.0, 0.0, 1.0], ctx=ctx)
    prec = S.build_preconditioner(W, S.partition_dofs(pair, fine), S.build_prolongation(pair, coarse, fine))
    rep = S.pcg(W, prec, L, 1e-8)
    assert rep.converged and rep.iterations < 40
    res = L - W.matvec(rep.solution)
    assert np.linalg.norm(res) <= 1e-6 * np.linalg.norm(L), np.linalg.norm(res) / np.linalg.norm(L)
