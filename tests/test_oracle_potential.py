"""The oracle's double-layer potential (oracle/sbo.hpp: eval_DL, restating
inc/potential.hpp:31-138, 3-D) pinned by the reference's own test cases
(tests/test_potential.cpp:108-239, their 3-D geometries): zero density, single-trace
annihilation, linearity, the jump relation at facet barycentres, far-field decay,
harmonicity, on-screen rejection; and the evaluation grid (potential.hpp:15-25)."""
import numpy as np
import pytest

from oracle import oracle as O


def expand(im, v):
    """jump.hpp:45-57 on the oracle's exported numbering"""
    coeff = np.zeros(im.n_gvertices)
    for d, (vx, j) in enumerate(im.jump_dofs):
        coeff[im.gv_first[vx] + j] += v[d]
        coeff[im.gv_first[vx] + im.q[vx] - 1] -= v[d]
    return coeff


def trace_eval(im, m, coeff, o, u, w):
    """TraceField::eval (jump.hpp:25-29) on oriented facet o"""
    f = o // 2
    vals = [coeff[im.gv_first[m.facets[f][k]] + im.ofacet_branch[o][k]] for k in range(3)]
    return (1.0 - u - w) * vals[0] + u * vals[1] + w * vals[2]


def density(im, seed):
    return O.normal_draws(seed, im.n)


def doctest_approx(a, b, eps):
    """doctest's Approx(b).epsilon(eps) == a: |a - b| < eps (1 + max(|a|, |b|))"""
    return abs(a - b) < eps * (1.0 + max(abs(a), abs(b)))


def test_zero_density_gives_zero_field():
    m = O.make_builtin_bowtie(2)
    im = O.inflate(m)
    g = O.make_cartesian_grid(m, -2, 2, 7, 7, 0.05)
    assert len(g) > 0
    assert np.abs(O.eval_DL(np.zeros(im.n), im, g)).max() == 0.0


def test_single_trace_density_is_annihilated():
    # test_potential.cpp:121-137: the same nodal values on every branch have zero jump
    # coordinates, and eval_DL of them vanishes
    m = O.make_builtin_bowtie(1)
    im = O.inflate(m)
    coeff = np.zeros(im.n_gvertices)
    for vx in range(len(m.vertices)):
        for j in range(im.q[vx]):
            coeff[im.gv_first[vx] + j] = np.cos(0.7 * vx)
    coords = O.jump_coordinates(im, coeff)
    assert np.abs(coords).max() < 1e-14
    assert abs(O.eval_DL(coords, im, [[0.4, 0.4, 0.9]])[0]) < 1e-8


def test_linearity_in_the_density():
    # test_potential.cpp:139-149 (on a 3-D T-junction instead of the 2-D threefold arm)
    pair = O.make_panels(1, 6, 3)
    im = O.inflate(pair.fine)
    g = O.make_cartesian_grid(pair.fine, -2, 2, 5, 5, 0.07)
    a, b = density(im, 3), density(im, 4)
    ua, ub, uab = O.eval_DL(a, im, g), O.eval_DL(b, im, g), O.eval_DL(2.0 * a - 0.5 * b, im, g)
    assert np.abs(uab - (2.0 * ua - 0.5 * ub)).max() < 1e-12 * (1.0 + np.abs(ua).max())


def test_jump_relation_at_facet_barycentres():
    # test_potential.cpp:151-174 (the 3-D geometry): U(x0 + eps n) - U(x0 - eps n) equals the
    # density's jump at the barycentre to 1%
    m = O.make_builtin_bowtie(1)
    im = O.inflate(m)
    v = density(im, 18)
    coeff = expand(im, v)
    verts = np.asarray(m.vertices)
    h = max(np.linalg.norm(verts[t[a]] - verts[t[b]]) for t in m.facets for a in range(3) for b in range(a + 1, 3))
    eps = 1e-3 * h
    rng = np.random.default_rng(23)
    for f in rng.integers(0, len(m.facets), 10):
        x0 = verts[m.facets[f]].mean(axis=0)
        n0 = im.normals[2 * f]
        jump = trace_eval(im, m, coeff, 2 * f + 1, 1 / 3, 1 / 3) - trace_eval(im, m, coeff, 2 * f, 1 / 3, 1 / 3)
        up, um = O.eval_DL(v, im, [x0 + eps * n0, x0 - eps * n0])
        assert doctest_approx(up - um, jump, 0.01), (f, up - um, jump)


def test_far_field_decay_along_a_ray():
    # test_potential.cpp:176-189
    m = O.make_builtin_bowtie(1)
    im = O.inflate(m)
    v = density(im, 5)
    d = np.array([1.0, 2.0, 0.5]) / np.linalg.norm([1.0, 2.0, 0.5])
    prev = 1e300
    for r in (10.0, 20.0, 40.0):
        bound = abs(O.eval_DL(v, im, [r * d])[0]) * r
        assert bound < 10.0 * abs(v.sum() + 1.0)
        assert bound < prev * 2.5
        prev = bound


def test_harmonicity_probe():
    # test_potential.cpp:191-207 in 3-D: the 7-point Laplacian is O(spacing^2)
    pair = O.make_panels(1, 6, 3)
    im = O.inflate(pair.fine)
    v = density(im, 8)
    c = np.array([0.8, 0.9, 0.3])
    prev = 0.0
    for sp in (0.02, 0.01):
        pts = [c] + [c + s * sp * e for e in np.eye(3) for s in (1, -1)]
        u = O.eval_DL(v, im, pts)
        lap = (u[1:].sum() - 6 * u[0]) / sp ** 2
        assert abs(lap) < 1.0
        if prev:
            assert abs(lap) < prev
        prev = abs(lap)


def test_on_screen_point_is_rejected():
    # test_potential.cpp:233-239
    m = O.make_builtin_bowtie(0)
    im = O.inflate(m)
    on = np.asarray(m.vertices)[list(m.facets[0])].mean(axis=0)
    with pytest.raises(O.ValidationError, match="on the screen"):
        O.eval_DL(np.zeros(im.n), im, [on])


def test_cartesian_grid_masks_points_near_the_screen():
    # potential.hpp:15-25: cell centres, x-major; a flat screen in z = 0 masks the points over it
    pair = O.make_panels(0, 4, 1)
    g = O.make_cartesian_grid(pair.fine, -2, 2, 8, 8, 0.05)
    full = np.array([[-2 + 4 * (i + 0.5) / 8, -2 + 4 * (j + 0.5) / 8, 0.0] for i in range(8) for j in range(8)])
    d = O.distance_to(pair.fine, full)
    assert np.array_equal(g, full[d > 0.05])
    assert len(g) < len(full)
