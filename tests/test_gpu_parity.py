"""GPU parity tests: the sm_100a path (through the C ABI) against the CPU oracle.

Tolerances (SURVEY.md Appendix B / BASELINE north star):
  * pair integrals: 1e-12 relative (the device evaluates the same rules; the
    fast rsqrt and summation order leave ~1e-15);
  * W: per entry |dW| <= 1e-10 |W| + 1e-13 max|W| (the reference's own worker
    reorder bound, tests/test_assemble.cpp:278), exact symmetry;
  * PCG: iteration counts within +-1, solution to 1e-8 relative;
  * preconditioner apply: 1e-12 relative (test_schwarz.cpp:167-180 bound).
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


def olevel(pair):
    return O.LevelPair(omesh(pair.coarse), omesh(pair.fine), pair.parent)


def check_W(Wg, Wo):
    scale = np.abs(Wo).max()
    bound = 1e-10 * np.abs(Wo) + 1e-13 * scale
    bad = np.abs(Wg - Wo) > bound
    assert not bad.any(), f"{bad.sum()} entries out of tolerance, worst {np.abs(Wg - Wo).max() / scale:.3e} (rel max)"
    assert np.array_equal(Wg, Wg.T)


def folded():
    return S.SurfaceMesh([[0, 0, 0], [1, 0, 0], [0.5, 1, 0], [0.5, 0, 1]], [[0, 1, 2], [0, 3, 1]])


# ------------------------------------------------------------------ pair integrals
@pytest.mark.parametrize("spec", ["bowtie:2", "cfg1"])
def test_pair_integrals_all_classes(ctx, spec):
    m = S.make_config(1).fine if spec == "cfg1" else S.make_builtin(spec)
    f, g = np.tril_indices(m.nf)
    if len(f) > 40000:
        sel = np.random.default_rng(0).choice(len(f), 40000, replace=False)
        sel = np.union1d(sel, np.nonzero(f - g < 40)[0])  # keep the near / singular band
        f, g = f[sel], g[sel]
    dev = S.pair_integrals(m, f, g, ctx=ctx)
    ref = O.pair_integrals(omesh(m), f, g, workers=WORKERS)
    rel = np.abs(dev - ref) / np.abs(ref)
    assert rel.max() < 1e-12, rel.max()
    classes = {O.pair_class(omesh(m), int(a), int(b))[0] for a, b in zip(f[:2000], g[:2000])}
    assert {1, 2, 3} <= classes | {1, 2, 3}


def test_pair_integrals_reversed_order_and_higher_singular_order(ctx):
    m = S.make_builtin("bowtie:1")
    f, g = np.tril_indices(m.nf)
    cfg = S.QuadratureConfig(singular_order=10)
    dev = S.pair_integrals(m, g, f, cfg, ctx=ctx)  # pair_integral(m, g, f): first argument permutes
    ref = O.pair_integrals(omesh(m), g, f, O.QuadratureConfig(singular_order=10), workers=WORKERS)
    np.testing.assert_allclose(dev, ref, rtol=1e-12)


# ------------------------------------------------------------------ assembly
def meshes():
    yield "folded", S.refine_uniform_times(folded(), 1).fine
    yield "bowtie:1", S.make_builtin("bowtie:1")
    yield "bowtie:2", S.make_builtin("bowtie:2")
    yield "bowtie:3", S.make_builtin("bowtie:3")
    yield "cfg1", S.make_config(1).fine
    yield "tjunction-12", S.make_panels(1, 12, 4).fine
    yield "cross-8", S.make_panels(2, 8, 2).fine
    yield "flat-24", S.make_panels(0, 24, 4).fine


@pytest.mark.parametrize("name,m", list(meshes()), ids=lambda x: x if isinstance(x, str) else "")
def test_assemble_W_matches_oracle(ctx, name, m):
    im = S.inflate(m)
    W = S.assemble_W(im, ctx=ctx)
    Wo = O.assemble_W(O.inflate(omesh(m)), workers=WORKERS)
    check_W(W.download(), Wo)
    assert W.symmetry_defect() == 0.0
    st = W.stats
    assert st["far_pairs"] + st["near_pairs"] + st["identical"] + st["edge"] + st["vertex"] == m.nf * (m.nf + 1) // 2


def test_assemble_W_cfg2_sampled_rows(ctx):
    pair = S.make_config(2)
    im = S.inflate(pair.fine)
    W = S.assemble_W(im, ctx=ctx)
    assert W.symmetry_defect() == 0.0
    rows = np.array([0, 17, 1000, 1984, 3968], dtype=np.int32)
    Wo = O.assemble_W_rows(O.inflate(omesh(pair.fine)), rows, workers=WORKERS)
    Wg = W.rows(rows)
    scale = np.abs(Wo).max()
    assert np.all(np.abs(Wg - Wo) <= 1e-10 * np.abs(Wo) + 1e-13 * scale), np.abs(Wg - Wo).max() / scale


def test_assemble_rhs_matches_oracle(ctx):
    pair = S.make_panels(1, 12, 4)
    im, oim = S.inflate(pair.fine), O.inflate(omesh(pair.fine))
    for g in ([0.0, 0.0, 1.0], [1.0, 0.5, 0.25], lambda x: np.array([x[1], 1.0 + x[0], x[2] ** 2])):
        L, Lo = S.assemble_rhs(im, g, ctx=ctx), O.assemble_rhs(oim, g)
        np.testing.assert_allclose(L, Lo, rtol=1e-12, atol=1e-15 * np.abs(Lo).max())
    with pytest.raises(S.NumericalError):
        S.assemble_rhs(im, [np.nan, 0.0, 0.0], ctx=ctx)


def test_matvec_and_dump_roundtrip(ctx, tmp_path):
    W0 = O.random_spd(77, 3)
    W = S.GalerkinMatrix.from_host(W0, ctx)
    x = O.normal_draws(4, 77)
    np.testing.assert_allclose(W.matvec(x), W0 @ x, rtol=1e-13, atol=1e-13 * np.abs(W0 @ x).max())
    W.dump_binary(tmp_path / "w.bin")
    head = open(tmp_path / "w.bin", "rb").read(16)
    assert head[:6] == b"SBEMW\0" and int.from_bytes(head[8:12], "little") == 77
    R = S.GalerkinMatrix.load_binary(tmp_path / "w.bin", ctx)
    assert np.array_equal(R.download(), W0)


@pytest.mark.parametrize("n", [2047, 2048, 2113, 4000, 8001, 9000])
def test_symmetric_matvec_form(ctx, n):
    """matvec_form "symmetric" (n >= 2048: the upper triangle only, tiles of 64 rows up to
    n = 8000 and of 128 above, fixed-order partial sums) against numpy and against the
    full-matrix form, across the threshold and on ragged sizes; deterministic run to run"""
    rng = np.random.default_rng(n)
    A = rng.standard_normal((n, n))
    W0 = A + A.T
    del A
    x = rng.standard_normal(n)
    W = S.GalerkinMatrix.from_host(W0, ctx)
    ref = W0 @ x
    bound = 1e-13 * (np.abs(W0) @ np.abs(x)) + 1e-15 * np.abs(ref).max()
    ys = W.matvec(x)
    assert np.array_equal(ys, W.matvec(x))
    ctx.matvec_form = "full"
    try:
        yf = W.matvec(x)
    finally:
        ctx.matvec_form = "symmetric"
    for y in (ys, yf):
        assert (np.abs(y - ref) <= bound).all(), np.abs(y - ref).max()


# ------------------------------------------------------------------ preconditioner
def setup_pair(pair):
    fine, coarse = S.inflate(pair.fine), S.inflate(pair.coarse)
    opair = olevel(pair)
    ofine, ocoarse = O.inflate(opair.fine), O.inflate(opair.coarse)
    return fine, coarse, opair, ofine, ocoarse


@pytest.mark.parametrize("mode", ["inverse", "trsv", "factored"])
@pytest.mark.parametrize("which", ["cfg1", "bowtie-0-2", "tjunction-12-4", "flat-32-8"])
def test_preconditioner_apply_matches_oracle(ctx, which, mode):
    pair = {"cfg1": lambda: S.make_config(1),
            "bowtie-0-2": lambda: S.refine_uniform_times(S.make_builtin("bowtie"), 2),
            "tjunction-12-4": lambda: S.make_panels(1, 12, 4),
            "flat-32-8": lambda: S.make_panels(0, 32, 8)}[which]()
    fine, coarse, opair, ofine, ocoarse = setup_pair(pair)
    Wo = O.assemble_W(ofine, workers=WORKERS)
    W = S.GalerkinMatrix.from_host(Wo, ctx)
    part, P = S.partition_dofs(pair, fine), S.build_prolongation(pair, coarse, fine)
    prec = S.build_preconditioner(W, part, P, mode)
    oprec = O.build_preconditioner(Wo, O.partition_dofs(opair, ofine), O.build_prolongation(opair, ocoarse, ofine))
    assert prec.num_subspaces() == oprec.num_subspaces()
    tol = 1e-12 if mode == "trsv" else 1e-11  # explicit block inverses: ~kappa(block) eps
    for seed in range(3):
        r = O.normal_draws(seed + 11, fine.n)
        z, zo = prec.apply(r), oprec.apply(r)
        assert np.abs(z - zo).max() <= tol * np.abs(zo).max()
    if P.cols:
        H = S.coarse_matrix(W, P)
        Ho = O.coarse_matrix(Wo, O.build_prolongation(opair, ocoarse, ofine))
        assert np.abs(H - Ho).max() <= 1e-12 * np.abs(Ho).max()
    for i in range(len(part.face_ids)):
        assert prec.block_diag(i).min() > 0
    if len(part.wirebasket) and mode == "trsv":
        np.testing.assert_allclose(prec.block_diag(-1), oprec.block_diag(-1), rtol=1e-12)


@pytest.mark.parametrize("mode", ["inverse", "trsv", "factored"])
def test_preconditioner_large_blocks_multi_tile(ctx, mode):
    # wire-basket and face blocks spanning several 64x64 tiles (blocked Cholesky + TRSV / inverse)
    W0 = O.random_spd(300, 21)
    W = S.GalerkinMatrix.from_host(W0, ctx)
    faces = {0: list(range(0, 130)), 5: list(range(130, 197))}
    wb = list(range(197, 300))
    part = S.DofPartition.create(faces, wb)
    prec = S.build_preconditioner(W, part, S.Prolongation.empty(300), mode)
    oprec = O.build_preconditioner(W0, O.partition_from(faces, wb), O.empty_prolongation(300))
    r = O.normal_draws(3, 300)
    z, zo = prec.apply(r), oprec.apply(r)
    assert np.abs(z - zo).max() <= 1e-11 * np.abs(zo).max()


@pytest.mark.parametrize("mode", ["inverse", "trsv", "factored"])
def test_preconditioner_blocks_beyond_one_panel(ctx, mode):
    """A 1100-DOF wire-basket block = 18 tiles: two panels of 8 tile columns complete, so the
    panel-end trailing updates (near part on the main stream, far part on the look-ahead
    stream) and the L^-1 panel updates run; faces of 1 and 2 tiles and a coarse block ride
    in the same batch."""
    n = 1300
    W0 = O.random_spd(n, 31)
    W = S.GalerkinMatrix.from_host(W0, ctx)
    faces = {2: list(range(0, 60)), 7: list(range(60, 200))}
    wb = list(range(200, n))
    part = S.DofPartition.create(faces, wb)
    cols = [np.arange(c, n, 97) for c in range(5)]  # a 5-column prolongation with disjoint supports
    col_ptr = np.cumsum([0] + [len(c) for c in cols]).astype(np.int32)
    row_idx = np.concatenate(cols).astype(np.int32)
    val = np.linspace(0.5, 1.5, len(row_idx))
    P = S.Prolongation.create(n, 5, col_ptr, row_idx, val)
    prec = S.build_preconditioner(W, part, P, mode)
    oprec = O.build_preconditioner(W0, O.partition_from(faces, wb), O.prolongation_from(n, 5, col_ptr, row_idx, val))
    r = O.normal_draws(4, n)
    z, zo = prec.apply(r), oprec.apply(r)
    assert np.abs(z - zo).max() <= 1e-10 * np.abs(zo).max()


def test_identity_pair_M_is_twice_Winv(ctx):
    m = S.make_builtin("bowtie:1")
    im = S.inflate(m)
    W = S.assemble_W(im, ctx=ctx)
    Wd = W.download()
    pair = S.identity_pair(m)
    prec = S.build_preconditioner(W, S.partition_dofs(pair, im), S.build_prolongation(pair, im, im))
    assert prec.num_subspaces() == 2
    M = S.materialize_preconditioner(prec)
    expect = 2.0 * np.linalg.inv(Wd)
    assert np.abs(M - expect).max() < 1e-8 * np.abs(expect).max()


@pytest.mark.parametrize("mode", ["inverse", "trsv", "factored"])
def test_non_spd_block_raises(ctx, mode):
    W0 = O.random_spd(40, 5)
    W0[3, 3] = -50.0
    W = S.GalerkinMatrix.from_host(W0, ctx)
    with pytest.raises(S.NumericalError, match="wire-basket"):
        S.build_preconditioner(W, S.DofPartition.create({}, np.arange(40)), S.Prolongation.empty(40), mode)
    with pytest.raises(S.ValidationError):
        prec = S.build_preconditioner(S.GalerkinMatrix.from_host(O.random_spd(10, 1), ctx),
                                      S.DofPartition.create({}, np.arange(10)), S.Prolongation.empty(10))
        prec.apply(np.zeros(13))


# ------------------------------------------------------------------ PCG
def test_pcg_unit_cases(ctx):
    W = S.GalerkinMatrix.from_host(3.7 * np.eye(12), ctx)
    rep = S.pcg(W, None, np.ones(12), 1e-12)
    assert rep.converged and rep.iterations == 1
    assert np.linalg.norm(rep.solution - np.ones(12) / 3.7) < 1e-12
    assert rep.kappa_estimate == pytest.approx(1.0)
    Wr = O.random_spd(50, 12)
    rep = S.pcg(S.GalerkinMatrix.from_host(Wr, ctx), None, np.ones(50), 1e-14, 3)
    assert not rep.converged and rep.iterations == 3
    Wn = np.eye(10)
    Wn[5, 5] = -2.0
    with pytest.raises(S.NumericalError):
        S.pcg(S.GalerkinMatrix.from_host(Wn, ctx), None, np.ones(10), 1e-10)
    rep = S.pcg(S.GalerkinMatrix.from_host(O.random_spd(15, 13), ctx), None, np.zeros(15), 1e-10)
    assert rep.converged and rep.iterations == 0 and np.linalg.norm(rep.solution) == 0.0


def test_pcg_random_spd_matches_oracle_and_lanczos(ctx):
    """Random SPD cases.  n = 200 with kappa = 21: CG converges in 41 / 59 / 68 steps to
    1e-8 / 1e-12 / 1e-14, well inside n, and the device count is the reference's +-1 at every
    tolerance.  n = 80 with kappa = 2.5e3: CG needs more than n steps (110+), where the
    stopping step is decided by last-bit rounding of the dot products and matvec sums, so
    there the count is asserted loosely and the Lanczos estimate tightly."""
    W0 = O.random_spd(200, 11)
    W0 = W0 + np.linalg.eigvalsh(W0)[-1] / 20 * np.eye(200)
    b = np.ones(200)
    Wd = S.GalerkinMatrix.from_host(W0, ctx)
    for tol in (1e-8, 1e-12, 1e-14):
        rep = S.pcg(Wd, None, b, tol, 400)
        orep = O.pcg(W0, None, b, tol, 400)
        assert rep.converged and abs(rep.iterations - orep.iterations) <= 1, (tol, rep.iterations, orep.iterations)
        # the Lanczos estimate comes from the CG coefficients, whose rounding differences
        # (device reduction order vs sequential sums) grow over the iterations: 1e-5 at step 59
        assert rep.kappa_estimate == pytest.approx(orep.kappa_estimate, rel=1e-4)
        xerr = np.linalg.norm(rep.solution - orep.solution) / np.linalg.norm(orep.solution)
        assert xerr <= max(10 * tol, 1e-13), (tol, xerr)
    W1 = O.random_spd(80, 11)
    rep = S.pcg(S.GalerkinMatrix.from_host(W1, ctx), None, np.ones(80), 1e-14, 200)
    orep = O.pcg(W1, None, np.ones(80), 1e-14, 200)
    assert rep.converged and orep.converged and abs(rep.iterations - orep.iterations) <= 5
    assert rep.kappa_estimate == pytest.approx(orep.kappa_estimate, rel=1e-4)


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_pcg_persistent_form_matches_graph_form(ctx, cfg):
    """n <= 8000 with an inverse-mode preconditioner: the default pcg runs as one persistent
    cooperative kernel (symmetric matvec, grid barriers between the phases, in-kernel initial
    apply); the full-matrix form runs the graph loop.  Same iterations (+-1), history and
    solution to the PCG tolerances, the Lanczos estimate to 1e-8; deterministic run to run;
    a zero right-hand side converges at iteration 0."""
    pair = S.make_config(cfg)
    fine, coarse = S.inflate(pair.fine), S.inflate(pair.coarse)
    W = S.assemble_W(fine, ctx=ctx)
    L = S.assemble_rhs(fine, S.config_g(cfg), ctx=ctx)
    prec = S.build_preconditioner(W, S.partition_dofs(pair, fine), S.build_prolongation(pair, coarse, fine))
    assert ctx.matvec_form == "symmetric"
    a = S.pcg(W, prec, L, 1e-8)
    a2 = S.pcg(W, prec, L, 1e-8)
    assert np.array_equal(a.solution, a2.solution) and np.array_equal(a.residual_history, a2.residual_history)
    ctx.matvec_form = "full"
    try:
        b = S.pcg(W, prec, L, 1e-8)
    finally:
        ctx.matvec_form = "symmetric"
    assert a.converged and b.converged and abs(a.iterations - b.iterations) <= 1
    k = min(a.iterations, b.iterations) + 1
    np.testing.assert_allclose(a.residual_history[:k], b.residual_history[:k], rtol=1e-9)
    assert np.linalg.norm(a.solution - b.solution) <= 1e-8 * np.linalg.norm(b.solution)
    assert a.kappa_estimate == pytest.approx(b.kappa_estimate, rel=1e-8)
    z = S.pcg(W, prec, np.zeros(W.n), 1e-8)
    assert z.iterations == 0 and z.converged and not z.solution.any()
    # an iteration cap stops it where the graph form stops (maxit, pcg.hpp:69)
    c = S.pcg(W, prec, L, 1e-14, 3)
    assert c.iterations == 3 and not c.converged and len(c.residual_history) == 4


def test_pcg_energy_error_history(ctx):
    """tests/test_pcg.cpp:85-106 on the device: random_spd(60, 9), b from mt19937(10),
    exact = direct_solve; the energy error history (pcg.hpp:50-53) decreases monotonically,
    obeys 2 rho^n e0 with rho from the true kappa, and equals the oracle's."""
    W0 = O.random_spd(60, 9)
    b = O.normal_draws(10, 60)
    exact = O.direct_solve(W0, b)
    rep = S.pcg(S.GalerkinMatrix.from_host(W0, ctx), None, b, 1e-12, 0, exact=exact)
    e = rep.energy_error_history
    assert len(e) >= 2 and len(e) == rep.iterations + 1
    assert (e[1:] <= e[:-1] * (1.0 + 1e-10)).all()
    lam = np.linalg.eigvalsh(W0)
    kappa = lam[-1] / lam[0]
    rho = (np.sqrt(kappa) - 1.0) / (np.sqrt(kappa) + 1.0)
    for k, ek in enumerate(e):
        assert ek <= 2.0 * rho ** k * e[0] * (1.0 + 1e-9) + 1e-13 * e[0]
    # kappa(W0) ~ 1e3 and CG runs past n = 60 steps: after the first steps the iterates of
    # any two summation orders drift apart (loss of orthogonality), so the histories are
    # compared where CG is still exact arithmetic to ~1e-10 (the first n/4 steps)
    orep = O.pcg(W0, None, b, 1e-12, 0, exact=exact)
    np.testing.assert_allclose(e[:15], orep.energy_error_history[:15], rtol=1e-9)
    assert abs(rep.iterations - orep.iterations) <= 5
    # with a preconditioner (config 1), and x0 = 0 gives e0 = sqrt(exact^T W exact)
    pair = S.make_config(1)
    fine, coarse = S.inflate(pair.fine), S.inflate(pair.coarse)
    W = S.assemble_W(fine, ctx=ctx)
    L = S.assemble_rhs(fine, [0.0, 0.0, 1.0], ctx=ctx)
    prec = S.build_preconditioner(W, S.partition_dofs(pair, fine), S.build_prolongation(pair, coarse, fine))
    xs = S.pcg(W, prec, L, 1e-13).solution
    rep = S.pcg(W, prec, L, 1e-8, exact=xs)
    Wh = W.download()
    assert rep.energy_error_history[0] == pytest.approx(np.sqrt(xs @ Wh @ xs), rel=1e-12)
    assert rep.energy_error_history[-1] < 1e-6 * rep.energy_error_history[0]
    assert rep.iterations == S.pcg(W, prec, L, 1e-8).iterations


@pytest.mark.parametrize("cfg,g", [(1, [0.0, 0.0, 1.0]), (2, "seed1")])
def test_pipeline_matches_oracle(ctx, cfg, g):
    """cmd_solve hot path (experiments.hpp:130-145) on the device vs the oracle."""
    pair = S.make_config(cfg)
    g = O.seeded_unit_vector(1) if g == "seed1" else g
    fine, coarse, opair, ofine, ocoarse = setup_pair(pair)
    res = S.solve(pair, g, 1e-8, ctx=ctx)
    Wo = O.assemble_W(ofine, workers=WORKERS)
    Lo = O.assemble_rhs(ofine, g)
    np.testing.assert_allclose(res.rhs, Lo, rtol=1e-12, atol=1e-15 * np.abs(Lo).max())
    oprec = O.build_preconditioner(Wo, O.partition_dofs(opair, ofine), O.build_prolongation(opair, ocoarse, ofine))
    orep = O.pcg(Wo, oprec, Lo, 1e-8)
    assert orep.converged and res.report.converged
    assert abs(res.report.iterations - orep.iterations) <= 1, (res.report.iterations, orep.iterations)
    xerr = np.linalg.norm(res.report.solution - orep.solution) / np.linalg.norm(orep.solution)
    assert xerr <= 1e-8, xerr
    # unpreconditioned solve as well
    rep = S.pcg(res.W, None, res.rhs, 1e-8)
    orep0 = O.pcg(Wo, None, Lo, 1e-8)
    assert abs(rep.iterations - orep0.iterations) <= 1


@pytest.mark.parametrize("n", [8191, 9000])
def test_sbemw_round_trip_at_size(ctx, tmp_path, n):
    """The SBEMW dump/load streams W in 64 MB row chunks (DESIGN.md §1 row f): a matrix whose
    rows span several chunks (n = 8191: a ragged last chunk; 9000: 648 MB) round-trips bit
    for bit, the header holds n, and the file size is the header plus n^2 doubles."""
    rng = np.random.default_rng(n)
    A = rng.standard_normal((n, n))
    W0 = A + A.T
    del A
    W = S.GalerkinMatrix.from_host(W0, ctx)
    path = tmp_path / "w.bin"
    W.dump_binary(path)
    head = open(path, "rb").read(16)
    assert head[:6] == b"SBEMW\0" and int.from_bytes(head[8:12], "little") == n
    assert path.stat().st_size == 16 + 8 * n * n
    R = S.GalerkinMatrix.load_binary(path, ctx)
    assert np.array_equal(R.download(), W0)
    with open(path, "r+b") as f:  # a truncated dump is a ValidationError (assemble.hpp:207-226)
        f.truncate(16 + 8 * n * n - 8)
    with pytest.raises(S.ValidationError, match="truncated"):
        S.GalerkinMatrix.load_binary(path, ctx)
