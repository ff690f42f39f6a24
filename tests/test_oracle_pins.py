"""Pins the CPU oracle (oracle/sbo.hpp) to the reference's own known-answer
tests and recorded numbers before anything is checked against it.

Each test names the reference test it ports (proj/tests/*.cpp) and keeps its
tolerance.  The 2-D (plus/threefold) variants of those tests are replaced by
3-D bow-tie ones: the 2-D segment path is out of scope.
"""
import numpy as np
import pytest

from oracle import oracle as O

CFG = O.QuadratureConfig()


def folded_two_triangle_screen():
    """tests/test_assemble.cpp:14-22"""
    return O.Mesh([[0, 0, 0], [1, 0, 0], [0.5, 1, 0], [0.5, 0, 1]], [[0, 1, 2], [0, 3, 1]])


def bowtie_patch():
    """tests/test_assemble.cpp:26-57: ten facets of bowtie:1"""
    full = O.make_builtin_bowtie(1)
    fac = []
    for b in (0, 2):
        fac += [full.facets[4 * b + 0], full.facets[4 * b + 2]]
    for b in (1, 3):
        fac += [full.facets[4 * b + 0], full.facets[4 * b + 1]]
    fac += [full.facets[3], full.facets[2 * 4 + 3]]
    remap, verts, out = {}, [], []
    for f in fac:
        row = []
        for v in f:
            if int(v) not in remap:
                remap[int(v)] = len(verts)
                verts.append(full.vertices[v])
            row.append(remap[int(v)])
        out.append(row)
    return O.Mesh(np.array(verts), np.array(out))


def flat_square(k):
    """tests/test_assemble.cpp:288-292: unit square {0,1,2},{0,2,3} refined k times"""
    m = O.Mesh([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0]], [[0, 1, 2], [0, 2, 3]])
    return O.refine_uniform_times(m, k).fine


def all_pairs(nf):
    f, g = np.tril_indices(nf)
    return f.astype(np.int32), g.astype(np.int32)


def oracle_assemble(im, rel_tol=1e-9):
    """Brute-force basis assembly with the adaptive integrator
    (tests/test_assemble.cpp:59-82)."""
    nf, n = im.base.nf, im.n
    f, g = all_pairs(nf)
    Iv = O.quad_oracle_pair_integrals(im.base, f, g, rel_tol)
    I = np.zeros((nf, nf))
    I[f, g] = Iv
    I[g, f] = Iv
    curls = np.array([[im.basis_curl(d, o) for o in range(2 * nf)] for d in range(n)])  # n x 2nf x 3
    C = curls.reshape(n, nf, 2, 3).sum(axis=2)  # per-facet side-summed curls
    return np.einsum("afc,fg,bgc->ab", C, I, C)


# ------------------------------------------------------------------ rules
def test_rules_shapes_and_weights():
    for n in (4, 6, 10):
        x, w = O.gauss_legendre(n)
        assert np.all(np.diff(x) > 0) and abs(w.sum() - 1.0) < 1e-14
    for order in (4, 6):
        u, v, w = O.triangle_rule(order)
        assert len(w) == order * order and abs(w.sum() - 0.5) < 1e-14
    sizes = {3: 60000, 2: 50000, 1: 20000}
    for cls, npts in sizes.items():
        assert O.sauter_rule(10, cls).shape == (npts, 5)


# ------------------------------------------------------------------ curls (test_assemble.cpp:86-132)
def test_curl_kat_right_triangle():
    m = O.Mesh([[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[0, 1, 2]])
    im = O.inflate(m)
    coeff = np.zeros(im.n_gvertices)
    coeff[im.gv_index(0, im.ofacet_branch[0][0])] = 1.0
    side0 = 0 if im.normals[0][2] > 0 else 1
    c = im.field_curl(coeff, side0)
    assert np.linalg.norm(c - np.array([1.0, -1.0, 0.0])) < 1e-14


def test_constant_trace_has_zero_curl():
    im = O.inflate(O.make_builtin_bowtie(0))
    coeff = np.ones(im.n_gvertices)
    for o in range(2 * im.base.nf):
        assert np.linalg.norm(im.field_curl(coeff, o)) < 1e-13


def test_flipping_side_negates_curl():
    im = O.inflate(O.make_builtin_bowtie(1))
    v = O.normal_draws(3, im.n)
    coeff = np.zeros(im.n_gvertices)
    for d, (vert, j) in enumerate(im.jump_dofs):  # expand (jump.hpp:45-57)
        coeff[im.gv_index(vert, j)] += v[d]
        coeff[im.gv_index(vert, im.q[vert] - 1)] -= v[d]
    for f in range(im.base.nf):
        sym = coeff.copy()
        for k in range(3):
            vtx = im.base.facets[f][k]
            sym[im.gv_index(vtx, im.ofacet_branch[2 * f + 1][k])] = sym[im.gv_index(vtx, im.ofacet_branch[2 * f][k])]
        c0, c1 = im.field_curl(sym, 2 * f), im.field_curl(sym, 2 * f + 1)
        assert np.linalg.norm(c0 + c1) < 1e-12 * (1 + np.linalg.norm(c0))


# ------------------------------------------------------------------ quadrature (test_assemble.cpp:134-198)
def test_closed_form_triangle_potential_vs_gauss():
    tri = np.array([[0, 0, 0], [1.2, 0.1, 0], [0.3, 0.9, 0]], dtype=float)
    u, v, w = O.triangle_rule(16)
    area = 0.5 * np.linalg.norm(np.cross(tri[1] - tri[0], tri[2] - tri[0]))
    rng = np.random.default_rng(5)
    for trial in range(20):
        x = rng.uniform(-2, 2, 3)
        x[2] += 2.5 if trial % 2 else -2.5
        y = tri[0] + u[:, None] * (tri[1] - tri[0]) + v[:, None] * (tri[2] - tri[0])
        gauss = 2.0 * area * np.sum(w / np.linalg.norm(x - y, axis=1))
        closed = O.triangle_inverse_distance_integral(tri, x)
        assert closed == pytest.approx(gauss, rel=1e-10)


def test_production_pair_integrals_match_adaptive_oracle():
    m = O.refine_uniform_times(folded_two_triangle_screen(), 1).fine
    f, g = all_pairs(m.nf)
    prod = O.pair_integrals(m, f, g)
    ref = O.quad_oracle_pair_integrals(m, f, g, 1e-9)
    np.testing.assert_allclose(prod, ref, rtol=1e-6)
    classes = {O.pair_class(m, int(a), int(b))[0] for a, b in zip(f, g)}
    assert classes == {0, 1, 2, 3}


# ------------------------------------------------------------------ W properties (test_assemble.cpp:200-280)
def test_W_exactly_symmetric_and_spd():
    im = O.inflate(O.make_builtin_bowtie(1))
    W = O.assemble_W(im)
    assert np.max(np.abs(W - W.T)) == 0.0
    assert np.linalg.eigvalsh(W).min() > 0


@pytest.mark.parametrize("which", ["folded", "bowtie_patch"])
def test_W_entries_match_bruteforce_oracle(which):
    m = O.refine_uniform_times(folded_two_triangle_screen(), 1).fine if which == "folded" else bowtie_patch()
    im = O.inflate(m)
    assert im.n > 0
    W = O.assemble_W(im)
    Wo = oracle_assemble(im)
    rel = np.abs(W - Wo) / np.maximum(np.abs(Wo), 1e-300)
    assert rel.max() <= 1e-6, rel.max()  # recorded worst 1.31e-09 (proj/test_output.txt:32)


def test_single_trace_rows_annihilate():
    """tests/test_assemble.cpp:215-244 on a 3-D geometry: the form against the
    single-valued hat at v vanishes."""
    im = O.inflate(O.make_builtin_bowtie(1))
    nf = im.base.nf
    f, g = all_pairs(nf)
    Iv = O.pair_integrals(im.base, f, g)
    I = np.zeros((nf, nf))
    I[f, g] = Iv
    I[g, f] = Iv
    basis = np.array([[im.basis_curl(d, o) for o in range(2 * nf)] for d in range(im.n)])
    for v in range(im.base.nv):
        coeff = np.zeros(im.n_gvertices)
        for j in range(im.q[v]):
            coeff[im.gv_index(v, j)] = 1.0
        cs = np.array([im.field_curl(coeff, o) for o in range(2 * nf)])
        terms = np.einsum("tc,duc,tu->dtu", cs, basis, I[np.arange(2 * nf) // 2][:, np.arange(2 * nf) // 2])
        entry = terms.sum(axis=(1, 2))
        scale = np.abs(terms).sum()
        assert np.abs(entry).max() <= 1e-6 * max(scale, 1e-30)


def test_raising_singular_order_moves_W_little():
    im = O.inflate(O.make_builtin_bowtie(1))
    W1 = O.assemble_W(im)
    W2 = O.assemble_W(im, O.QuadratureConfig(singular_order=10))
    assert np.abs(W1 - W2).max() < 1e-8 * np.abs(W1).max()


def test_bit_stable_at_fixed_workers_and_reorder_bound():
    im = O.inflate(O.make_builtin_bowtie(2))
    Wa = O.assemble_W(im, workers=3)
    Wb = O.assemble_W(im, workers=3)
    assert np.abs(Wa - Wb).max() == 0.0
    W1 = O.assemble_W(im, workers=1)
    assert np.abs(W1 - Wa).max() < 1e-13 * np.abs(W1).max()


# ------------------------------------------------------------------ RHS (test_assemble.cpp:282-325)
def test_rhs_tangential_field_is_zero():
    im = O.inflate(flat_square(2))
    L = O.assemble_rhs(im, lambda x: np.array([x[1], 1.0, 0.0]))
    assert np.abs(L).max() < 1e-14


def test_rhs_flat_screen_twice_hat_integral():
    fine = flat_square(2)
    im = O.inflate(fine)
    L = O.assemble_rhs(im, [0.0, 0.0, 1.0])
    for d, (v, j) in enumerate(im.jump_dofs):
        hat = 0.0
        for f in range(fine.nf):
            if v in fine.facets[f]:
                a, b, c = fine.vertices[fine.facets[f]]
                hat += 0.5 * np.linalg.norm(np.cross(b - a, c - a)) / 3.0
        assert abs(L[d]) == pytest.approx(2.0 * hat, rel=1e-12)


def test_rhs_non_finite_rejected():
    im = O.inflate(O.make_builtin_bowtie(1))
    with pytest.raises(O.NumericalError):
        O.assemble_rhs(im, [np.nan, 0.0, 0.0])


# ------------------------------------------------------------------ partition (test_schwarz.cpp:48-87)
def setup(coarse_refines, fine_offset):
    cm = O.make_builtin_bowtie(coarse_refines)
    pair = O.refine_uniform_times(cm, fine_offset)
    imc, imf = O.inflate(pair.coarse), O.inflate(pair.fine)
    P = O.build_prolongation(pair, imc, imf)
    W = O.assemble_W(imf, workers=O.default_workers())
    part = O.partition_dofs(pair, imf)
    return pair, imc, imf, P, W, part


def test_partition_identity_pair_all_wirebasket():
    m = O.make_builtin_bowtie(1)
    im = O.inflate(m)
    part = O.partition_dofs(O.identity_pair(m), im)
    assert len(part.face_sets) == 0 and len(part.wirebasket) == im.n


def test_partition_bowtie_median_in_wirebasket():
    pair, imc, imf, P, W, part = setup(0, 1)
    assert len(part.wirebasket) > 0 and len(part.face_sets) == 0
    for d in part.wirebasket:
        p = pair.fine.vertices[imf.jump_dofs[d][0]]
        assert np.linalg.norm(p[:2]) < 1e-12
    pair2, _, imf2, _, _, part2 = setup(0, 2)
    assert len(part2.face_sets) == 4
    for d in part2.wirebasket:
        assert np.linalg.norm(pair2.fine.vertices[imf2.jump_dofs[d][0]][:2]) < 1e-12


def test_partition_disjoint_and_complete():
    pair, imc, imf, P, W, part = setup(1, 2)
    seen = list(part.wirebasket) + [d for s in part.face_sets.values() for d in s]
    assert len(seen) == len(set(seen)) == imf.n


# ------------------------------------------------------------------ preconditioner (test_schwarz.cpp:89-188)
def test_identity_pair_M_is_twice_Winv():
    m = O.make_builtin_bowtie(1)
    im = O.inflate(m)
    W = O.assemble_W(im)
    prec = O.build_preconditioner(W, O.partition_dofs(O.identity_pair(m), im),
                                  O.build_prolongation(O.identity_pair(m), im, im))
    assert prec.num_subspaces() == 2
    M = O.materialize_preconditioner(prec)
    expect = 2.0 * np.linalg.inv(W)
    assert np.abs(M - expect).max() < 1e-8 * np.abs(expect).max()


def test_coarse_galerkin_equals_direct_coarse_assembly():
    pair, imc, imf, P, W, part = setup(1, 1)
    assert imc.n > 0
    WH = P.dense().T @ W @ P.dense()
    Wc = O.assemble_W(imc)
    assert np.abs(WH - Wc).max() <= 1e-8 * np.abs(Wc).max()
    assert np.abs(O.coarse_matrix(W, P) - Wc).max() <= 1e-8 * np.abs(Wc).max()


def test_blocks_factor_with_positive_pivots_and_apply_symmetric():
    pair, imc, imf, P, W, part = setup(0, 2)
    prec = O.build_preconditioner(W, part, P)
    for i in range(len(part.face_ids)):
        assert prec.block_diag(i).min() > 0
    assert prec.block_diag(-1).min() > 0
    draws = O.normal_draws(5, 10 * imf.n).reshape(10, imf.n)
    for t in range(5):
        a, b = draws[2 * t], draws[2 * t + 1]
        assert a @ prec.apply(b) == pytest.approx(b @ prec.apply(a), rel=1e-12)


def test_materialized_matches_apply_and_length_mismatch():
    pair, imc, imf, P, W, part = setup(0, 1)
    assert imf.n <= 200
    prec = O.build_preconditioner(W, part, P)
    M = O.materialize_preconditioner(prec)
    r = O.normal_draws(9, imf.n)
    direct = prec.apply(r)
    assert np.abs(M @ r - direct).max() <= 1e-12 * np.abs(direct).max()
    with pytest.raises(O.ValidationError):
        prec.apply(np.zeros(imf.n + 3))


def kappa_prec(W, prec):
    """condition_number(W, prec) (schwarz.hpp:174-190), oracle restatement."""
    return O.condition_number(W, prec)


def test_single_subspace_exact_inverse_kappa_one():
    im = O.inflate(O.make_builtin_bowtie(1))
    W = O.assemble_W(im)
    prec = O.build_preconditioner(W, O.partition_from({}, np.arange(im.n)), O.empty_prolongation(im.n))
    assert prec.num_subspaces() == 1
    assert kappa_prec(W, prec)[2] == pytest.approx(1.0, rel=1e-10)


def test_lambda_max_bounded_and_prec_beats_raw():
    pair, imc, imf, P, W, part = setup(0, 2)
    prec = O.build_preconditioner(W, part, P)
    lmin, lmax, kap = kappa_prec(W, prec)
    assert lmax <= prec.num_subspaces() * (1 + 1e-10)
    ev = np.linalg.eigvalsh(W)
    assert kap <= ev[-1] / ev[0]


def test_identity_pair_lambda_min_at_least_one():
    m = O.make_builtin_bowtie(1)
    im = O.inflate(m)
    W = O.assemble_W(im)
    prec = O.build_preconditioner(W, O.partition_dofs(O.identity_pair(m), im),
                                  O.build_prolongation(O.identity_pair(m), im, im))
    assert kappa_prec(W, prec)[0] >= 1.0 - 1e-10


def test_recorded_bowtie_condition_numbers():
    """Golden: proj/test_output.txt:31 (acceptance.cpp:175-221) — bow-tie,
    coarse = base, H/h = 16: 465 DOFs, kappa_prec 6.93, kappa_unprec 12.96."""
    base = O.make_bowtie_base()
    pair = O.refine_uniform_times(base, 4)
    imc, imf = O.inflate(pair.coarse), O.inflate(pair.fine, validate=False)
    assert imf.n == 465
    W = O.assemble_W(imf, workers=O.default_workers())
    prec = O.build_preconditioner(W, O.partition_dofs(pair, imf), O.build_prolongation(pair, imc, imf))
    _, _, kp = kappa_prec(W, prec)
    assert round(kp, 2) == 6.93
    assert round(O.condition_number(W)[2], 2) == 12.96


# ------------------------------------------------------------------ PCG (test_pcg.cpp:24-151)
def test_direct_solve_cases():
    W = O.random_spd(20, 1)
    assert np.linalg.norm(O.direct_solve(W, np.zeros(20))) == 0.0
    W = O.random_spd(20, 2)
    e1 = np.eye(20)[0]
    assert np.linalg.norm(O.direct_solve(W, W @ e1) - e1) < 1e-10
    W = O.random_spd(10, 5)
    W[0, 0] = -100.0
    with pytest.raises(O.NumericalError):
        O.direct_solve(W, np.ones(10))


def test_pcg_scaled_identity_one_iteration():
    W = 3.7 * np.eye(12)
    rep = O.pcg(W, None, np.ones(12), 1e-12)
    assert rep.converged and rep.iterations == 1
    assert np.linalg.norm(rep.solution - np.ones(12) / 3.7) < 1e-12
    assert rep.kappa_estimate == pytest.approx(1.0)


def test_pcg_matches_direct_in_energy_norm():
    W = O.random_spd(40, 7)
    b = O.normal_draws(8, 40)
    tol = 1e-9
    rep = O.pcg(W, None, b, tol)
    assert rep.converged
    xd = O.direct_solve(W, b)
    e = rep.solution - xd
    assert np.sqrt(e @ W @ e) <= 10 * tol * np.sqrt(xd @ W @ xd)


def test_pcg_energy_monotone_and_kappa_bound():
    W = O.random_spd(60, 9)
    b = O.normal_draws(10, 60)
    exact = O.direct_solve(W, b)
    rep = O.pcg(W, None, b, 1e-12, 0, exact)
    eh = rep.energy_error_history
    assert len(eh) >= 2
    assert np.all(eh[1:] <= eh[:-1] * (1 + 1e-10))
    ev = np.linalg.eigvalsh(W)
    kap = ev[-1] / ev[0]
    rho = (np.sqrt(kap) - 1) / (np.sqrt(kap) + 1)
    bound = 2.0 * rho ** np.arange(len(eh)) * eh[0]
    assert np.all(eh <= bound * (1 + 1e-9) + 1e-13 * eh[0])


def test_lanczos_estimate_from_below():
    W = O.random_spd(80, 11)
    rep = O.pcg(W, None, np.ones(80), 1e-14, 200)
    ev = np.linalg.eigvalsh(W)
    kap = ev[-1] / ev[0]
    assert kap * 0.5 <= rep.kappa_estimate <= kap * 1.05


def test_pcg_maxit_nonspd_zero_rhs_history():
    rep = O.pcg(O.random_spd(50, 12), None, np.ones(50), 1e-14, 3)
    assert not rep.converged and rep.iterations == 3
    W = np.eye(10)
    W[5, 5] = -2.0
    with pytest.raises(O.NumericalError):
        O.pcg(W, None, np.ones(10), 1e-10)
    rep = O.pcg(O.random_spd(15, 13), None, np.zeros(15), 1e-10)
    assert rep.converged and rep.iterations == 0 and np.linalg.norm(rep.solution) == 0.0
    rep = O.pcg(O.random_spd(30, 14), None, np.ones(30), 1e-10)
    assert rep.converged and np.all(rep.residual_history[:-1] > 0)
