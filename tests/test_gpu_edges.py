"""Edge cases of the device path (GPU, `-m gpu`): empty DOF spaces, quadrature
configuration, reproducibility of the atomic scatter, and input errors mapped to the
reference's exception types (inc/common.hpp:16-26)."""
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


def check_W(Wg, Wo):
    scale = np.abs(Wo).max()
    bad = np.abs(Wg - Wo) > 1e-10 * np.abs(Wo) + 1e-13 * scale
    assert not bad.any(), (bad.sum(), np.abs(Wg - Wo).max() / scale)
    assert np.array_equal(Wg, Wg.T)


def test_no_interior_dofs(ctx):
    """A single triangle (and a two-triangle square) has only boundary vertices: n = 0."""
    for m in (S.SurfaceMesh([[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[0, 1, 2]]),
              S.SurfaceMesh([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0]], [[0, 1, 2], [0, 2, 3]])):
        im = S.inflate(m)
        assert im.n == 0
        W = S.assemble_W(im, ctx=ctx)
        assert W.n == 0 and W.download().shape == (0, 0)
        assert S.assemble_rhs(im, [0.0, 0.0, 1.0], ctx=ctx).shape == (0,)
        rep = S.pcg(W, None, np.zeros(0), 1e-8)
        assert rep.converged and rep.iterations == 0


def test_repeated_assembly_within_reorder_bound(ctx):
    """fp64 atomics reorder the scatter: two assemblies agree to the reference's own
    worker-reorder bound (tests/test_assemble.cpp:271-279), symmetry stays exact."""
    im = S.inflate(S.make_builtin("bowtie:3"))
    Wa = S.assemble_W(im, ctx=ctx).download()
    Wb = S.assemble_W(im, ctx=ctx).download()
    assert np.abs(Wa - Wb).max() <= 1e-13 * np.abs(Wa).max()
    assert np.array_equal(Wa, Wa.T) and np.array_equal(Wb, Wb.T)


def test_singular_order_and_threshold_configurations(ctx):
    """QuadratureConfig (quadrature.hpp:12-16) other than the default: singular order 10
    moves W by < 1e-8 max|W| (tests/test_assemble.cpp:260-269) and matches the oracle at
    the same setting; a near threshold of 3 (more near-field recursion) matches too."""
    m = S.make_builtin("bowtie:2")
    im = S.inflate(m)
    oim = O.inflate(O.Mesh(m.vertices, m.facets))
    W8 = S.assemble_W(im, ctx=ctx).download()
    W10 = S.assemble_W(im, S.QuadratureConfig(singular_order=10), ctx=ctx).download()
    assert np.abs(W8 - W10).max() < 1e-8 * np.abs(W8).max()
    check_W(W10, O.assemble_W(oim, O.QuadratureConfig(singular_order=10), workers=WORKERS))
    W3 = S.assemble_W(im, S.QuadratureConfig(near_threshold=3.0), ctx=ctx).download()
    check_W(W3, O.assemble_W(oim, O.QuadratureConfig(near_threshold=3.0), workers=WORKERS))


@pytest.mark.parametrize("far_order", [1, 2, 3, 5, 6])
def test_far_order_configurations_match_oracle(ctx, far_order):
    """far_order sets both the far rule (far_order^2 points) and the near-leaf rule
    ((far_order+2)^2, quadrature.hpp:105-112): the padded device rules reproduce the
    oracle's W and RHS at every order."""
    m = S.make_builtin("bowtie:2")
    im = S.inflate(m)
    oim = O.inflate(O.Mesh(m.vertices, m.facets))
    cfg, ocfg = S.QuadratureConfig(far_order=far_order), O.QuadratureConfig(far_order=far_order)
    check_W(S.assemble_W(im, cfg, ctx=ctx).download(), O.assemble_W(oim, ocfg, workers=WORKERS))
    L, Lo = S.assemble_rhs(im, [0.3, -0.2, 1.0], cfg, ctx=ctx), O.assemble_rhs(oim, [0.3, -0.2, 1.0], ocfg)
    np.testing.assert_allclose(L, Lo, rtol=1e-12, atol=1e-15 * np.abs(Lo).max())


def test_far_order_out_of_range_is_a_validation_error(ctx):
    im = S.inflate(S.make_builtin("bowtie:1"))
    with pytest.raises(S.ValidationError, match="far_order"):
        S.assemble_W(im, S.QuadratureConfig(far_order=9), ctx=ctx)


def test_malformed_meshes_raise_validation_error(ctx):
    with pytest.raises(S.ValidationError):
        S.inflate(S.SurfaceMesh([[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[0, 1, 3]]))
    with pytest.raises(S.ValidationError):
        S.inflate(S.SurfaceMesh([[0, 0, 0], [1, 0, 0], [np.nan, 1, 0]], [[0, 1, 2]]))
    with pytest.raises(S.ValidationError):
        S.inflate(S.SurfaceMesh([[0, 0, 0], [1, 0, 0], [2, 0, 0]], [[0, 1, 2]]))  # degenerate facet


def test_exact_far_switch_is_bitwise_on_far_pairs(ctx):
    """with exact_far the depth-0 far pair integrals are bitwise the
    CPU restatement's (one thread per pair, i-major order, IEEE sqrt/division, no FMA);
    the W it assembles matches the oracle per entry and the fast path to the reorder bound."""
    m = S.make_config(1).fine
    om = O.Mesh(m.vertices, m.facets)
    f, g = np.tril_indices(m.nf, -1)
    sel = np.random.default_rng(3).choice(len(f), 1500, replace=False)
    f, g = f[sel].astype(np.int32), g[sel].astype(np.int32)
    dev = S.pair_integrals(m, f, g, S.QuadratureConfig(exact_far=True), ctx=ctx)
    far = np.zeros(len(f), dtype=bool)
    ref = np.zeros(len(f))
    for k in range(len(f)):
        v, st = O.pair_integrals(om, f[k:k + 1], g[k:k + 1], workers=1, stats=True)
        ref[k] = v[0]
        far[k] = st[0] == 1 and st[1] == 0 and st[2] == 0
    assert far.sum() > 1000
    assert np.array_equal(dev[far], ref[far]), np.abs(dev[far] - ref[far]).max()
    assert (np.abs(dev[~far] - ref[~far]) <= 1e-12 * np.abs(ref[~far])).all()
    im = S.inflate(m)
    oim = O.inflate(om)
    We = S.assemble_W(im, S.QuadratureConfig(exact_far=True), ctx=ctx).download()
    Wf = S.assemble_W(im, ctx=ctx).download()
    check_W(We, O.assemble_W(oim, workers=WORKERS))
    assert np.abs(We - Wf).max() <= 1e-13 * np.abs(We).max()


def test_download_into_pinned_buffer(ctx):
    """download(out=) into page-locked memory (one pitched DMA, ld > n here) equals the
    staged download into pageable memory bit for bit."""
    im = S.inflate(S.make_config(1).fine)
    W = S.assemble_W(im, ctx=ctx)
    assert W.n == 225  # ld = 256: the pitched copy drops the padding columns
    ref = W.download()
    buf = S.pinned_empty((W.n, W.n))
    out = W.download(out=buf)
    assert out is buf and np.array_equal(buf, ref)
    big = S.assemble_W(S.inflate(S.make_builtin("bowtie:3")), ctx=ctx)
    b2 = S.pinned_empty((big.n, big.n))
    assert np.array_equal(big.download(out=b2), big.download())


@pytest.mark.parametrize("spec", ["config1", "bowtie:3"])
def test_recursion_counts_equal_the_oracle(ctx, spec):
    """The device near-field classification makes every leaf/split decision of the
    reference recursion (quadrature.hpp:231-249): its near-leaf count equals the oracle's
    exactly, and the depth-0 far pairs plus near and singular pairs cover all pairs."""
    m = S.make_config(1).fine if spec == "config1" else S.make_builtin(spec)
    im = S.inflate(m)
    W = S.assemble_W(im, ctx=ctx)
    _, st = O.assemble_W(O.inflate(O.Mesh(m.vertices, m.facets)), workers=WORKERS, stats=True)
    far_leaves, near_leaves, _ = (int(v) for v in st)
    s = W.stats
    assert s["near_leaves"] == near_leaves
    assert s["far_pairs"] == far_leaves
    assert s["far_pairs"] + s["near_pairs"] + s["identical"] + s["edge"] + s["vertex"] == m.nf * (m.nf + 1) // 2


def test_config2_work_counts_match_the_survey_probe(ctx):
    """SURVEY §8a probe counts for config 2 (a8, a9): 400 082 near-subdivided pairs,
    1.87e7 near leaves, 8 192 / 12 160 / 35 973 identical / edge / vertex pairs."""
    s = S.assemble_W(S.inflate(S.make_config(2).fine), ctx=ctx).stats
    assert (s["identical"], s["edge"], s["vertex"], s["near_pairs"]) == (8192, 12160, 35973, 400082)
    assert round(s["near_leaves"] / 1e5) == 187


def test_jittered_nonplanar_mesh_matches_oracle(ctx):
    """A seeded random perturbation of config 1 (in-plane jitter and a non-planar z
    displacement): irregular triangles, curved screen, no congruent pairs — the device W and
    RHS match the oracle per entry, and the recursion counts match exactly."""
    m = S.make_config(1).fine
    v = np.array(m.vertices, dtype=float)
    rng = np.random.default_rng(2024)
    h = 1.0 / 16
    v[:, :2] += rng.uniform(-0.2 * h, 0.2 * h, size=(len(v), 2))
    v[:, 2] = 0.15 * np.sin(2.0 * v[:, 0]) * np.cos(3.0 * v[:, 1]) + rng.uniform(-0.05 * h, 0.05 * h, len(v))
    mj = S.SurfaceMesh(v, np.array(m.facets))
    im = S.inflate(mj)
    om = O.Mesh(v, np.array(m.facets))
    oim = O.inflate(om)
    W = S.assemble_W(im, ctx=ctx)
    Wo, st = O.assemble_W(oim, workers=WORKERS, stats=True)
    check_W(W.download(), Wo)
    assert W.stats["near_leaves"] == int(st[1]) and W.stats["far_pairs"] == int(st[0])
    g = [0.3, -0.2, 1.0]
    L, Lo = S.assemble_rhs(im, g, ctx=ctx), O.assemble_rhs(oim, g)
    np.testing.assert_allclose(L, Lo, rtol=1e-12, atol=1e-15 * np.abs(Lo).max())


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_assemble_W_into_host_buffer(cfg):
    """assemble_W(im, out=buf) (C ABI sbg_assemble_w_host): the host copy equals the device W
    bit for bit — page-locked buffers get the copy overlapped with the near field plus the
    band patch (config 4's junction numbering takes the wide-band fallback), pageable ones
    the ordinary download."""
    ctx = S.Context(0)
    im = S.inflate(S.make_config(cfg).fine, validate=False)
    n = im.n
    for pinned in (True, False):
        buf = S.pinned_empty((n, n)) if pinned else np.full((n, n), np.nan)
        W = S.assemble_W(im, ctx=ctx, out=buf)
        Wd = W.download()
        assert np.array_equal(buf, Wd), (cfg, pinned, np.abs(buf - Wd).max())
        assert np.array_equal(Wd, Wd.T)
    with pytest.raises(S.ValidationError):
        S.assemble_W(im, ctx=ctx, out=np.zeros((n, n - 1)))


@pytest.mark.parametrize("axis,offset", [(2, 0.0), (2, 0.3), (1, -0.7), (0, 1.1)])
def test_coordinate_plane_screens_match_oracle(ctx, axis, offset):
    """Far tiles and near leaves whose facets all lie in one coordinate plane skip the
    evaluation's zero coordinate (assemble.cu far_flat / flat_axes): config 1 moved into the
    planes z = 0, z = 0.3, y = -0.7 and x = 1.1 (the permuted axis orders of the flat path)
    matches the oracle per entry, and the four placements agree with each other to the
    reorder bound (the same screen up to a rigid motion)."""
    m = S.make_config(1).fine
    v0 = np.array(m.vertices, dtype=float)
    # in-plane coordinates (u, w) -> the two axes other than `axis`; the flat coordinate = offset
    others = [a for a in range(3) if a != axis]
    v = np.empty_like(v0)
    v[:, others[0]], v[:, others[1]], v[:, axis] = v0[:, 0], v0[:, 1], offset
    f = np.array(m.facets)
    Wg = S.assemble_W(S.inflate(S.SurfaceMesh(v, f)), ctx=ctx).download()
    Wo = O.assemble_W(O.inflate(O.Mesh(v, f)), workers=WORKERS)
    check_W(Wg, Wo)
    Wz = S.assemble_W(S.inflate(S.SurfaceMesh(v0, f)), ctx=ctx).download()
    assert np.abs(Wg - Wz).max() <= 1e-13 * np.abs(Wz).max()


def test_solve_on_an_invalid_mesh_raises_the_validation_error(ctx):
    """S.solve validates the fine mesh beside the inflation and the assembly (screenbem.solve):
    an invalid fine mesh still raises the reference's ValidationError with validate_mesh's
    message, whatever the invalid data produced meanwhile (inflate.hpp validates first)."""
    pair = S.make_config(1)
    v = np.array(pair.fine.vertices, dtype=float)
    f = np.array(pair.fine.facets)
    f_dup = np.vstack([f, f[:1]])  # a duplicate facet
    for fine in (S.SurfaceMesh(v, f_dup),):
        with pytest.raises(S.ValidationError) as want:
            S.validate_mesh(fine)
        try:
            bad = S.MeshLevelPair(pair.coarse, fine, np.append(pair.parent, pair.parent[0]))
        except S.ValidationError:
            continue  # rejected when the level pair is made: nothing reaches solve
        with pytest.raises(S.ValidationError) as got:
            S.solve(bad, [0.0, 0.0, 1.0], ctx=ctx)
        assert str(got.value) == str(want.value)
    # vertex ids out of range are caught before the inflation (the cheap checks)
    with pytest.raises(S.ValidationError):
        fine = S.SurfaceMesh(v, np.vstack([f, [[0, 1, len(v) + 5]]]))
        S.solve(S.MeshLevelPair(pair.coarse, fine, np.append(pair.parent, pair.parent[0])), [0.0, 0.0, 1.0],
                ctx=ctx)
