"""CPU tests of the product's host layer and C ABI (no GPU needed).

* libscreenbem_b200.so loads and exports every function include/screenbem_b200.h declares;
* the BASELINE config generators give the sizes of SURVEY.md §8 (nf, nv, DOFs, q
  histogram, face/wire-basket/coarse sizes);
* DOF numbering, partition and prolongation are identical, bit for bit, to the
  oracle's restatement of inflate.hpp / schwarz.hpp / jump.hpp.
"""
import os
import re

import numpy as np
import pytest

from oracle import oracle as O
from paper_2310_09204_b200 import screenbem as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "screenbem_b200.h")).read()
    declared = set(re.findall(r"\b(sbg_[a-z0-9_]+)\s*\(", header))
    assert len(declared) > 40
    lib = S.lib()
    missing = [name for name in declared if not hasattr(lib, name)]
    assert not missing, missing
    assert declared == set(S.SIGNATURES), declared ^ set(S.SIGNATURES)


def to_oracle(m: S.SurfaceMesh) -> O.Mesh:
    return O.Mesh(m.vertices, m.facets)


def oracle_level(pair: S.MeshLevelPair) -> O.LevelPair:
    return O.LevelPair(to_oracle(pair.coarse), to_oracle(pair.fine), pair.parent)


def q_hist(q):
    vals, cnt = np.unique(q[q >= 1], return_counts=True)
    return {int(v): int(c) for v, c in zip(vals, cnt)}


# SURVEY.md §8 config table and a16/a17 (exact probe numbers)
CONFIGS = [
    (1, 0, 512, 289, 225, {1: 64, 2: 225}, (8, 21), 57, 1),
    (2, 0, 8192, 4225, 3969, {1: 256, 2: 3969}, (32, 105), 609, 9),
    (3, 0, 13824, 7105, 6721, {1: 431, 2: 6627, 3: 47}, (96, 55), 1441, 33),
    (4, 0, 24576, 12481, 12097, {1: 762, 2: 11532, 4: 186, 8: 1}, (384, 21), 4033, 169),
    (5, 8, 51200, 25921, 25281, {1: 640, 2: 25281}, (800, 21), 8481, 361),
    (5, 16, 51200, 25921, 25281, {1: 640, 2: 25281}, (200, 105), 4281, 81),
    (5, 20, 51200, 25921, 25281, {1: 640, 2: 25281}, (128, 171), 3393, 49),
    (5, 40, 51200, 25921, 25281, {1: 640, 2: 25281}, (32, 741), 1569, 9),
]


@pytest.mark.parametrize("cfg,ratio,nf,nv,n,qh,faces,nwb,nc", CONFIGS)
def test_config_sizes_match_survey(cfg, ratio, nf, nv, n, qh, faces, nwb, nc):
    pair = S.make_config(cfg, ratio)
    assert pair.fine.nf == nf and pair.fine.nv == nv
    fine = S.inflate(pair.fine, validate=cfg <= 4)
    assert fine.n == n
    assert q_hist(fine.q) == qh
    part = S.partition_dofs(pair, fine)
    sizes = {len(d) for d in part.face_sets.values()}
    assert (len(part.face_sets), sizes) == (faces[0], {faces[1]})
    assert len(part.wirebasket) == nwb
    coarse = S.inflate(pair.coarse)
    assert coarse.n == nc
    P = S.build_prolongation(pair, coarse, fine)
    assert (P.rows, P.cols) == (n, nc)


def small_levels():
    yield "bowtie-0-2", S.refine_uniform_times(S.make_builtin("bowtie"), 2)
    yield "bowtie-1-2", S.refine_uniform_times(S.make_builtin("bowtie:1"), 2)
    yield "cfg1", S.make_config(1)
    yield "flat-12-3", S.make_panels(0, 12, 3)
    yield "tjunction-12-4", S.make_panels(1, 12, 4)
    yield "cross-8-2", S.make_panels(2, 8, 2)
    yield "cross-8-4", S.make_panels(2, 8, 4)


@pytest.mark.parametrize("name,pair", list(small_levels()), ids=lambda x: x if isinstance(x, str) else "")
def test_inflation_partition_prolongation_bitwise(name, pair):
    opair = oracle_level(pair)
    for pm, om in ((pair.fine, opair.fine), (pair.coarse, opair.coarse)):
        a, b = S.inflate(pm), O.inflate(om)
        assert a.n == b.n and a.n_gvertices == b.n_gvertices
        for attr in ("q", "gv_first", "dof_first", "ofacet_branch", "jump_dofs"):
            np.testing.assert_array_equal(getattr(a, attr), getattr(b, attr), err_msg=attr)
        np.testing.assert_array_equal(a.normals, b.normals)
    fa, fo = S.inflate(pair.fine), O.inflate(opair.fine)
    ca, co = S.inflate(pair.coarse), O.inflate(opair.coarse)
    pa, po = S.partition_dofs(pair, fa), O.partition_dofs(opair, fo)
    np.testing.assert_array_equal(pa.face_ids, po.face_ids)
    np.testing.assert_array_equal(pa.face_ptr, po.face_ptr)
    np.testing.assert_array_equal(pa.face_dofs, po.face_dofs)
    np.testing.assert_array_equal(pa.wirebasket, po.wirebasket)
    Ra, Ro = S.build_prolongation(pair, ca, fa), O.build_prolongation(opair, co, fo)
    assert (Ra.rows, Ra.cols) == (Ro.rows, Ro.cols)
    np.testing.assert_array_equal(Ra.col_ptr, Ro.col_ptr)
    np.testing.assert_array_equal(Ra.row_idx, Ro.row_idx)
    np.testing.assert_array_equal(Ra.val, Ro.val)  # bitwise


def test_dyadic_panels_equal_uniform_refinement_up_to_permutation():
    pair = S.make_panels(0, 8, 4)
    ref = S.refine_uniform_times(pair.coarse, 2)

    def tri_set(m):
        return {tuple(sorted(tuple(np.round(m.vertices[v], 12)) for v in f)) for f in m.facets}

    assert tri_set(pair.fine) == tri_set(ref.fine)
    # parents agree geometrically: each fine facet's parent contains its centroid
    cen = pair.fine.vertices[pair.fine.facets].mean(axis=1)
    pcen = {tuple(np.round(c, 12)): p for c, p in zip(ref.fine.vertices[ref.fine.facets].mean(axis=1), ref.parent)}
    for c, p in zip(cen, pair.parent):
        cref = pcen[tuple(np.round(c, 12))]
        assert set(map(tuple, pair.coarse.vertices[pair.coarse.facets[p]])) == \
            set(map(tuple, ref.coarse.vertices[ref.coarse.facets[cref]]))


def test_builtins_and_refinement_match_oracle():
    for k in range(3):
        a = S.make_builtin(f"bowtie:{k}")
        b = O.make_builtin_bowtie(k)
        np.testing.assert_array_equal(a.vertices, b.vertices)
        np.testing.assert_array_equal(a.facets, b.facets)
    with pytest.raises(S.ValidationError):
        S.make_builtin("plus:2")  # 2-D geometries are outside the 3-D GPU path
    with pytest.raises(S.ValidationError):
        S.make_builtin("nosuch")


@pytest.mark.parametrize("case", ["duplicate", "degenerate", "overlap", "pierce", "range"])
def test_validate_mesh_rejects_like_oracle(case):
    v = [[0, 0, 0], [1, 0, 0], [0, 1, 0], [1, 1, 0], [0.25, 0.25, -0.5], [0.25, 0.25, 0.5]]
    f = {
        "duplicate": [[0, 1, 2], [2, 1, 0]],
        "degenerate": [[0, 1, 1]] if False else [[0, 1, 2], [0, 1, 3]] if False else [[0, 1, 2], [0, 3, 3]],
        "overlap": [[0, 1, 2], [0, 1, 3]],
        "pierce": [[0, 1, 2], [4, 5, 3]],
        "range": [[0, 1, 9]],
    }[case]
    with pytest.raises(S.ValidationError):
        S.validate_mesh(S.SurfaceMesh(v, f))
    with pytest.raises(O.ValidationError):
        O.validate_mesh(O.Mesh(v, f))


def test_point_contact_rejected():
    # two triangles touching only at a vertex (inflate.hpp:129-151)
    v = [[0, 0, 0], [1, 0, 0], [0, 1, 0], [-1, 0, 0.5], [0, -1, 0.5]]
    f = [[0, 1, 2], [0, 3, 4]]
    with pytest.raises(S.ValidationError, match="point contact"):
        S.inflate(S.SurfaceMesh(v, f))
    with pytest.raises(O.ValidationError, match="point contact"):
        O.inflate(O.Mesh(v, f))


def test_broken_nesting_rejected():
    pair = S.make_panels(0, 4, 2)
    bad = pair.parent.copy()
    bad[0] = (bad[0] + 3) % pair.coarse.nf
    lvl = S.MeshLevelPair(pair.coarse, pair.fine, bad)
    with pytest.raises(S.ValidationError):
        S.build_prolongation(lvl, S.inflate(pair.coarse), S.inflate(pair.fine))


def test_null_handles_are_validation_errors():
    """Every C-ABI entry point that takes a handle or an output pointer rejects NULL with
    status 2 (SBG_EVALIDATION, the reference's ValidationError) instead of crashing
    (ADVICE r01).  Runs without a GPU: the checks come before any device work."""
    import ctypes as C
    raw = C.CDLL(S.lib()._name)
    allowed_ok = {"sbg_device_free", "sbg_host_free"}  # freeing NULL is a no-op
    optional_ptrs = {"sbg_device_name"}  # name buffer and SM count are optional outputs
    checked, bad = 0, []
    for name, (res, args) in S.SIGNATURES.items():
        if res is not C.c_int or not args or name in optional_ptrs or name in ("sbg_matrix_n",
                                                                               "sbg_prec_num_subspaces"):
            continue
        if not any(a in (C.c_void_p,) or (isinstance(a, type) and issubclass(a, C._Pointer)) for a in args):
            continue  # no handle / output pointer (e.g. sbg_device_name, sbg_make_config's ints come first)
        fn = getattr(raw, name)
        fn.restype = C.c_int
        fn.argtypes = [C.c_void_p if (a is not C.c_int and a is not C.c_double and a is not C.c_longlong) else a
                       for a in args]
        call = [None if t is C.c_void_p else 0 for t in fn.argtypes]
        rc = fn(*call)
        if rc != (0 if name in allowed_ok else 2):
            bad.append((name, rc, S.lib().sbg_last_error()))
        checked += 1
    assert not bad, bad
    assert checked > 50, checked
    for name in ("sbg_ctx_destroy", "sbg_matrix_destroy", "sbg_prec_destroy", "sbg_mesh_destroy"):
        getattr(raw, name)(None)
    assert S.lib().sbg_prec_num_subspaces(None) == -1 and S.lib().sbg_matrix_n(None) == -1
