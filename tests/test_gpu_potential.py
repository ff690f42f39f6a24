"""The device double-layer potential (csrc/cuda/potential.cu, reference inc/potential.hpp:15-138,
3-D) against the CPU restatement (oracle.eval_DL):
  * exact_far: every facet in the reference's operation order and the facets summed in order
    — bitwise the oracle's, on grids that include points near the screen (deep subdivision);
  * default (far facets in the constant-normal form with a refined rsqrt): within
    1e-12 (|U|_max + 1) of the oracle;
  * the evaluation grid (potential.hpp:15-25) point for point, the reference's properties
    (tests/test_potential.cpp) on the device, and the edge cases (on-screen points, no points,
    a mesh without jump DOFs, far orders 1-8)."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

S = pytest.importorskip("paper_2310_09204_b200.screenbem")


@pytest.fixture(scope="module")
def ctx():
    return S.Context(0)


def both(pair_or_mesh):
    """(product InflatedMesh, oracle InflatedMesh, product mesh, oracle mesh) of one mesh"""
    m = pair_or_mesh.fine if hasattr(pair_or_mesh, "fine") else pair_or_mesh
    om = O.Mesh(m.vertices, m.facets)
    return S.inflate(m), O.inflate(om), m, om


def near_points(m, rng, k, scale):
    """k points at distance ~scale * h from random facet barycentres (both sides)"""
    v, f = np.asarray(m.vertices), np.asarray(m.facets)
    pick = rng.integers(0, len(f), k)
    tri = v[f[pick]]
    cen = tri.mean(axis=1)
    n = np.cross(tri[:, 1] - tri[:, 0], tri[:, 2] - tri[:, 0])
    n /= np.linalg.norm(n, axis=1)[:, None]
    h = np.linalg.norm(tri[:, 1] - tri[:, 0], axis=1)
    sgn = np.where(rng.random(k) < 0.5, -1.0, 1.0)
    return cen + (sgn * scale * h)[:, None] * n


CASES = [("bowtie2", lambda: S.make_builtin("bowtie:2")), ("flat", lambda: S.make_panels(0, 12, 3)),
         ("tjunction", lambda: S.make_panels(1, 6, 3)), ("cross", lambda: S.make_panels(2, 8, 4))]


@pytest.mark.parametrize("name,make", CASES)
def test_eval_dl_exact_far_is_bitwise_the_oracle(ctx, name, make):
    im, oim, m, om = both(make())
    rng = np.random.default_rng(7)
    v = rng.standard_normal(im.n)
    pts = np.concatenate([O.make_cartesian_grid(om, -1.5, 1.5, 6, 6, 0.05), near_points(m, rng, 12, 1e-3),
                          near_points(m, rng, 12, 0.3), [[7.0, -3.0, 2.0]]])
    ref = O.eval_DL(v, oim, pts)
    got = S.eval_DL(v, im, pts, S.QuadratureConfig(exact_far=True), ctx=ctx)
    assert np.array_equal(got, ref), np.abs(got - ref).max()


@pytest.mark.parametrize("name,make", CASES)
def test_eval_dl_fast_form_matches_the_oracle(ctx, name, make):
    im, oim, m, om = both(make())
    rng = np.random.default_rng(11)
    v = rng.standard_normal(im.n)
    pts = np.concatenate([O.make_cartesian_grid(om, -2, 2, 9, 9, 0.02), near_points(m, rng, 20, 1e-3),
                          near_points(m, rng, 20, 0.05), near_points(m, rng, 20, 2.0)])
    ref = O.eval_DL(v, oim, pts)
    got = S.eval_DL(v, im, pts, ctx=ctx)
    err = np.abs(got - ref)
    assert err.max() <= 1e-12 * (np.abs(ref).max() + 1.0), (err.max(), np.abs(ref).max())


@pytest.mark.parametrize("far_order", [1, 2, 5, 8])
def test_eval_dl_far_orders(ctx, far_order):
    im, oim, m, om = both(S.make_panels(1, 4, 2))
    rng = np.random.default_rng(far_order)
    v = rng.standard_normal(im.n)
    pts = np.concatenate([near_points(m, rng, 8, 1e-2), near_points(m, rng, 8, 1.0)])
    cfg = S.QuadratureConfig(far_order=far_order)
    ref = O.eval_DL(v, oim, pts, O.QuadratureConfig(far_order=far_order))
    assert np.array_equal(S.eval_DL(v, im, pts, S.QuadratureConfig(far_order=far_order, exact_far=True), ctx=ctx),
                          ref)
    got = S.eval_DL(v, im, pts, cfg, ctx=ctx)
    assert np.abs(got - ref).max() <= 1e-12 * (np.abs(ref).max() + 1.0)


def test_cartesian_grid_matches_the_oracle(ctx):
    for mk in (lambda: S.make_panels(0, 8, 2).fine, lambda: S.make_builtin("bowtie:1"),
               lambda: S.make_panels(2, 4, 2).fine):
        m = mk()
        om = O.Mesh(m.vertices, m.facets)
        for (lo, hi, nx, ny, eps) in ((-2, 2, 7, 7, 0.05), (-1, 1, 10, 6, 1e-3), (-1.5, 0.5, 3, 11, 0.3)):
            got = S.make_cartesian_grid(m, lo, hi, nx, ny, eps, ctx=ctx).points
            ref = O.make_cartesian_grid(om, lo, hi, nx, ny, eps)
            assert np.array_equal(got, ref)
    assert len(S.make_cartesian_grid(m, -1, 1, 0, 5, 0.1, ctx=ctx)) == 0


def test_eval_dl_reference_properties_on_device(ctx):
    """tests/test_potential.cpp:108-239 (3-D) through the product path"""
    # zero density: exactly zero
    im, oim, m, om = both(S.make_builtin("bowtie:2"))
    g = S.make_cartesian_grid(m, -2, 2, 7, 7, 0.05, ctx=ctx)
    assert np.abs(S.eval_DL(np.zeros(im.n), im, g, ctx=ctx)).max() == 0.0
    # linearity
    rng = np.random.default_rng(3)
    a, b = rng.standard_normal(im.n), rng.standard_normal(im.n)
    ua, ub, uab = (S.eval_DL(x, im, g, ctx=ctx) for x in (a, b, 2.0 * a - 0.5 * b))
    assert np.abs(uab - (2.0 * ua - 0.5 * ub)).max() < 1e-12 * (1.0 + np.abs(ua).max())
    # jump relation at barycentres of a flat panel with interior DOFs: U(x0 + eps n) - U(x0 - eps n)
    # = [phi](x0) to 1% (2 eps = 2e-3 h, the subdivision resolves the facet)
    im, oim, m, om = both(S.make_panels(0, 8, 2))
    v = rng.standard_normal(im.n)
    verts, facets = np.asarray(m.vertices), np.asarray(m.facets)
    coeff = np.zeros(oim.n_gvertices)
    for d, (vx, j) in enumerate(oim.jump_dofs):
        coeff[oim.gv_first[vx] + j] += v[d]
        coeff[oim.gv_first[vx] + oim.q[vx] - 1] -= v[d]
    h = np.linalg.norm(verts[facets[:, 1]] - verts[facets[:, 0]], axis=1).max()
    checked = 0
    for f in rng.permutation(len(facets))[:40]:
        vals = [[coeff[oim.gv_first[facets[f][k]] + oim.ofacet_branch[o][k]] for k in range(3)] for o in (2 * f, 2 * f + 1)]
        jump = np.mean(vals[1]) - np.mean(vals[0])
        if abs(jump) < 0.1:
            continue
        x0, n0 = verts[facets[f]].mean(axis=0), oim.normals[2 * f]
        up, um = S.eval_DL(v, im, [x0 + 1e-3 * h * n0, x0 - 1e-3 * h * n0], ctx=ctx)
        assert up - um == pytest.approx(jump, rel=0.01)
        checked += 1
    assert checked >= 5
    # far-field decay along a ray
    im, oim, m, om = both(S.make_builtin("bowtie:1"))
    v = rng.standard_normal(im.n)
    d = np.array([1.0, 2.0, 0.5]) / np.linalg.norm([1.0, 2.0, 0.5])
    prev = 1e300
    for r in (10.0, 20.0, 40.0):
        bound = abs(S.eval_DL(v, im, [r * d], ctx=ctx)[0]) * r
        assert bound < 10.0 * abs(v.sum() + 1.0) and bound < prev * 2.5
        prev = bound


def test_eval_dl_edges(ctx):
    im, oim, m, om = both(S.make_builtin("bowtie:1"))
    v = np.ones(im.n)
    # a point on the screen (a facet barycentre) is rejected (potential.hpp:119-120)
    on = np.asarray(m.vertices)[list(m.facets[3])].mean(axis=0)
    with pytest.raises(S.ValidationError, match="on the screen"):
        S.eval_DL(v, im, [[5.0, 5.0, 5.0], on], ctx=ctx)
    # no points; wrong density length
    assert len(S.eval_DL(v, im, np.zeros((0, 3)), ctx=ctx)) == 0
    with pytest.raises(S.ValidationError):
        S.eval_DL(v[:-1], im, [[5.0, 5.0, 5.0]], ctx=ctx)
    # a screen without interior vertices has no jump DOFs: the field is zero
    im0, _, m0, _ = both(S.make_panels(0, 1, 1))
    assert im0.n == 0
    assert np.array_equal(S.eval_DL(np.zeros(0), im0, [[0.3, 0.2, 0.5]], ctx=ctx), [0.0])
    # deterministic run to run, single points and many
    pts = np.random.default_rng(1).standard_normal((3000, 3)) * 2.0 + [0.0, 0.0, 0.01]
    pts = pts[O.distance_to(om, pts) > 1e-6]
    a = S.eval_DL(v, im, pts, ctx=ctx)
    assert np.array_equal(a, S.eval_DL(v, im, pts, ctx=ctx))
    assert np.array_equal(a[:7], [S.eval_DL(v, im, p[None], ctx=ctx)[0] for p in pts[:7]]) or \
        np.abs(a[:7] - [S.eval_DL(v, im, p[None], ctx=ctx)[0] for p in pts[:7]]).max() <= 1e-15 * np.abs(a).max()
