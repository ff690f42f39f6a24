"""ctypes front-end of the C++ ORACLE (oracle/sbo.hpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
bench CPU-baseline leg, as the checker.  The product package never imports it.
Names follow the reference API (proj/include/screenbem/*.hpp) so parity tests
read like the reference's doctest suites.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libsbo_oracle.so")
_lib = None

i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")


class ValidationError(RuntimeError):
    """reference: inc/common.hpp:17-20"""


class NumericalError(RuntimeError):
    """reference: inc/common.hpp:23-26"""


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB_PATH):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        vp = C.c_void_p
        sig = {
            "orc_last_error": (C.c_char_p, []),
            "orc_mesh_new": (vp, [C.c_int, f64p, C.c_int, i32p]),
            "orc_mesh_free": (None, [vp]),
            "orc_mesh_sizes": (C.c_int, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
            "orc_mesh_export": (C.c_int, [vp, f64p, i32p]),
            "orc_validate_mesh": (C.c_int, [vp]),
            "orc_bowtie_base": (vp, []),
            "orc_level_new": (vp, [vp, vp, i32p]),
            "orc_refine_uniform_times": (vp, [vp, C.c_int]),
            "orc_level_free": (None, [vp]),
            "orc_level_fine": (vp, [vp]),
            "orc_level_coarse": (vp, [vp]),
            "orc_level_parent": (C.c_int, [vp, i32p]),
            "orc_gauss_legendre": (C.c_int, [C.c_int, f64p, f64p]),
            "orc_triangle_rule": (C.c_int, [C.c_int, f64p, f64p, f64p]),
            "orc_sauter_rule": (C.c_longlong, [C.c_int, C.c_int, C.c_void_p]),
            "orc_pair_integrals": (C.c_int, [vp, i32p, i32p, C.c_longlong, C.c_int, C.c_int, C.c_double,
                                             C.c_int, f64p, i64p]),
            "orc_quad_oracle_pair_integrals": (C.c_int, [vp, i32p, i32p, C.c_longlong, C.c_double, C.c_int,
                                                         f64p]),
            "orc_pair_class": (C.c_int, [vp, C.c_int, C.c_int, i32p, i32p]),
            "orc_triangle_inverse_distance_integral": (C.c_double, [f64p, f64p]),
            "orc_inflate": (vp, [vp, C.c_int, C.POINTER(C.c_int)]),
            "orc_im_free": (None, [vp]),
            "orc_im_sizes": (C.c_int, [vp, i32p]),
            "orc_im_export": (C.c_int, [vp, i32p, i32p, i32p, i32p, i32p, f64p]),
            "orc_basis_curl": (C.c_int, [vp, C.c_int, C.c_int, f64p]),
            "orc_field_curl": (C.c_int, [vp, f64p, C.c_int, f64p]),
            "orc_assemble_W": (C.c_int, [vp, C.c_int, C.c_int, C.c_double, C.c_int, C.c_longlong,
                                         C.c_longlong, f64p, i64p]),
            "orc_assemble_W_rows": (C.c_int, [vp, C.c_int, C.c_int, C.c_double, i32p, C.c_int, C.c_int, f64p]),
            "orc_sampler_new": (vp, [vp, C.c_int, C.c_int, C.c_double, C.c_int, C.POINTER(C.c_int)]),
            "orc_sampler_free": (None, [vp]),
            "orc_sampler_fixed": (C.c_int, [vp, C.POINTER(C.c_double)]),
            "orc_sampler_run": (C.c_int, [vp, i64p, C.c_longlong, C.POINTER(C.c_double)]),
            "orc_rhs_points": (C.c_int, [vp, C.c_int, f64p]),
            "orc_assemble_rhs": (C.c_int, [vp, C.c_int, f64p, f64p]),
            "orc_build_prolongation": (vp, [vp, vp, vp, C.POINTER(C.c_int)]),
            "orc_empty_prolongation": (vp, [C.c_int]),
            "orc_identity_prolongation": (vp, [C.c_int]),
            "orc_prolongation_from": (vp, [C.c_int, C.c_int, i32p, i32p, f64p]),
            "orc_prolongation_free": (None, [vp]),
            "orc_prolongation_sizes": (C.c_int, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
            "orc_prolongation_export": (C.c_int, [vp, i32p, i32p, f64p]),
            "orc_partition": (vp, [vp, vp, C.POINTER(C.c_int)]),
            "orc_partition_from": (vp, [C.c_int, i32p, i32p, i32p, C.c_int, i32p]),
            "orc_partition_free": (None, [vp]),
            "orc_partition_sizes": (C.c_int, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
            "orc_partition_export": (C.c_int, [vp, i32p, i32p, i32p, i32p]),
            "orc_build_preconditioner": (vp, [f64p, C.c_int, vp, vp, C.POINTER(C.c_int)]),
            "orc_prec_free": (None, [vp]),
            "orc_prec_num_subspaces": (C.c_int, [vp]),
            "orc_apply_preconditioner": (C.c_int, [vp, f64p, C.c_int, f64p]),
            "orc_coarse_matrix": (C.c_int, [f64p, C.c_int, vp, f64p]),
            "orc_prec_block_diag": (C.c_int, [vp, C.c_int, C.c_void_p, C.POINTER(C.c_int)]),
            "orc_pcg": (C.c_int, [f64p, C.c_int, vp, f64p, C.c_double, C.c_int, C.c_void_p, f64p,
                                  C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_double), f64p,
                                  C.c_void_p, f64p, f64p, C.c_int, C.POINTER(C.c_int)]),
            "orc_direct_solve": (C.c_int, [f64p, C.c_int, f64p, f64p]),
            "orc_matvec": (C.c_int, [f64p, C.c_int, f64p, f64p, C.c_int]),
            "orc_lanczos_kappa": (C.c_double, [f64p, f64p, C.c_int]),
            "orc_random_spd": (C.c_int, [C.c_int, C.c_uint, f64p]),
            "orc_normal_draws": (C.c_int, [C.c_uint, C.c_int, f64p]),
            "orc_eval_dl": (C.c_int, [vp, f64p, f64p, C.c_longlong, C.c_int, C.c_int, f64p]),
            "orc_distance_to": (C.c_int, [vp, f64p, C.c_longlong, f64p]),
            "orc_make_cartesian_grid": (C.c_int, [vp, C.c_double, C.c_double, C.c_int, C.c_int, C.c_double, f64p,
                                                  C.POINTER(C.c_int)]),
            "orc_jump_coordinates": (C.c_int, [vp, f64p, f64p]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(rc: int):
    if rc == 0:
        return
    msg = lib().orc_last_error().decode()
    if rc == 2:
        raise ValidationError(msg)
    if rc == 3:
        raise NumericalError(msg)
    raise RuntimeError(msg)


def default_workers() -> int:
    return max(1, os.cpu_count() or 1)


# --------------------------------------------------------------------------- meshes
class Mesh:
    """SurfaceMesh (reference: inc/mesh.hpp:19-83), 3-D triangles."""

    def __init__(self, vertices, facets, _handle=None):
        self.vertices = np.ascontiguousarray(vertices, dtype=np.float64).reshape(-1, 3)
        self.facets = np.ascontiguousarray(facets, dtype=np.int32).reshape(-1, 3)
        self.h = _handle or lib().orc_mesh_new(len(self.vertices), self.vertices.reshape(-1),
                                               len(self.facets), self.facets.reshape(-1))

    @classmethod
    def _from_handle(cls, h):
        nv, nf = C.c_int(), C.c_int()
        lib().orc_mesh_sizes(h, C.byref(nv), C.byref(nf))
        v = np.zeros(3 * nv.value)
        f = np.zeros(3 * nf.value, dtype=np.int32)
        lib().orc_mesh_export(h, v, f)
        return cls(v, f, _handle=h)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.orc_mesh_free(self.h)
            self.h = None

    @property
    def nf(self):
        return len(self.facets)

    @property
    def nv(self):
        return len(self.vertices)


def validate_mesh(m: Mesh):
    _check(lib().orc_validate_mesh(m.h))


def make_bowtie_base() -> Mesh:
    return Mesh._from_handle(lib().orc_bowtie_base())


class LevelPair:
    """MeshLevelPair (reference: inc/mesh.hpp:86-92)."""

    def __init__(self, coarse: Mesh, fine: Mesh, parent, _handle=None):
        self.coarse, self.fine = coarse, fine
        self.parent = np.ascontiguousarray(parent, dtype=np.int32)
        self.h = _handle or lib().orc_level_new(coarse.h, fine.h, self.parent)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.orc_level_free(self.h)
            self.h = None


def refine_uniform_times(m: Mesh, k: int) -> LevelPair:
    """reference: inc/mesh.hpp:388-405"""
    h = lib().orc_refine_uniform_times(m.h, k)
    fine = Mesh._from_handle(lib().orc_level_fine(h))
    coarse = Mesh._from_handle(lib().orc_level_coarse(h))
    parent = np.zeros(fine.nf, dtype=np.int32)
    lib().orc_level_parent(h, parent)
    return LevelPair(coarse, fine, parent, _handle=h)


def make_builtin_bowtie(refinements: int = 0) -> Mesh:
    """make_builtin("bowtie:k") (reference: inc/mesh.hpp:530-531)"""
    return refine_uniform_times(make_bowtie_base(), refinements).fine


def identity_pair(m: Mesh) -> LevelPair:
    """H = h pair (reference: tests/test_schwarz.cpp:35-44)"""
    return LevelPair(m, m, np.arange(m.nf, dtype=np.int32))


# --------------------------------------------------------------------------- rules
def gauss_legendre(n: int):
    x, w = np.zeros(n), np.zeros(n)
    lib().orc_gauss_legendre(n, x, w)
    return x, w


def triangle_rule(order: int):
    u, v, w = np.zeros(order * order), np.zeros(order * order), np.zeros(order * order)
    lib().orc_triangle_rule(order, u, v, w)
    return u, v, w


def sauter_rule(order: int, cls: int) -> np.ndarray:
    n = lib().orc_sauter_rule(order, cls, None)
    out = np.zeros(5 * n)
    lib().orc_sauter_rule(order, cls, out.ctypes.data_as(C.c_void_p))
    return out.reshape(n, 5)


@dataclass
class QuadratureConfig:
    """reference: inc/quadrature.hpp:12-16"""
    far_order: int = 4
    singular_order: int = 8
    near_threshold: float = 2.0


def pair_integrals(m: Mesh, f, g, cfg: QuadratureConfig = QuadratureConfig(), workers: int = 0,
                   stats: bool = False):
    """pair_integral(m, f, g, eng) for arrays of pairs (reference: inc/quadrature.hpp:268-334)."""
    f = np.ascontiguousarray(f, dtype=np.int32)
    g = np.ascontiguousarray(g, dtype=np.int32)
    out = np.zeros(len(f))
    st = np.zeros(3, dtype=np.int64)
    _check(lib().orc_pair_integrals(m.h, f, g, len(f), cfg.far_order, cfg.singular_order, cfg.near_threshold,
                                    workers or default_workers(), out, st))
    return (out, st) if stats else out


def quad_oracle_pair_integrals(m: Mesh, f, g, rel_tol=1e-9, workers: int = 0):
    """reference: inc/quad_oracle.hpp:128-141"""
    f = np.ascontiguousarray(f, dtype=np.int32)
    g = np.ascontiguousarray(g, dtype=np.int32)
    out = np.zeros(len(f))
    _check(lib().orc_quad_oracle_pair_integrals(m.h, f, g, len(f), rel_tol, workers or default_workers(), out))
    return out


def pair_class(m: Mesh, f: int, g: int):
    pf, pg = np.zeros(3, dtype=np.int32), np.zeros(3, dtype=np.int32)
    s = lib().orc_pair_class(m.h, f, g, pf, pg)
    return s, pf, pg


def triangle_inverse_distance_integral(tri, x) -> float:
    return lib().orc_triangle_inverse_distance_integral(np.ascontiguousarray(tri, dtype=np.float64).reshape(-1),
                                                        np.ascontiguousarray(x, dtype=np.float64))


# --------------------------------------------------------------------------- inflation
class InflatedMesh:
    """reference: inc/inflate.hpp:48-76"""

    def __init__(self, mesh: Mesh, validate: bool = True):
        st = C.c_int()
        h = lib().orc_inflate(mesh.h, 1 if validate else 0, C.byref(st))
        _check(st.value)
        self.h, self.base = h, mesh
        sizes = np.zeros(4, dtype=np.int32)
        lib().orc_im_sizes(h, sizes)
        self.n, self.n_gvertices, nv, nf = (int(x) for x in sizes)
        self.q = np.zeros(nv, dtype=np.int32)
        self.gv_first = np.zeros(nv, dtype=np.int32)
        self.dof_first = np.zeros(nv, dtype=np.int32)
        self.ofacet_branch = np.zeros(6 * nf, dtype=np.int32)
        self.jump_dofs = np.zeros(2 * self.n, dtype=np.int32)
        self.normals = np.zeros(6 * nf)
        lib().orc_im_export(h, self.q, self.gv_first, self.dof_first, self.ofacet_branch, self.jump_dofs,
                            self.normals)
        self.ofacet_branch = self.ofacet_branch.reshape(-1, 3)
        self.jump_dofs = self.jump_dofs.reshape(-1, 2)
        self.normals = self.normals.reshape(-1, 3)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.orc_im_free(self.h)
            self.h = None

    def num_jump_dofs(self):
        return self.n

    def gv_index(self, v, b):
        return int(self.gv_first[v]) + b

    def basis_curl(self, d: int, o: int):
        out = np.zeros(3)
        _check(lib().orc_basis_curl(self.h, d, o, out))
        return out

    def field_curl(self, coeff, o: int):
        out = np.zeros(3)
        _check(lib().orc_field_curl(self.h, np.ascontiguousarray(coeff, dtype=np.float64), o, out))
        return out


def inflate(mesh: Mesh, validate: bool = True) -> InflatedMesh:
    return InflatedMesh(mesh, validate)


def assemble_W(im: InflatedMesh, cfg: QuadratureConfig = QuadratureConfig(), workers: int = 1,
               pair_range=None, stats: bool = False):
    """reference: inc/assemble.hpp:72-139 (row-major dense result)"""
    n = im.n
    W = np.zeros(n * n)
    lo, hi = pair_range if pair_range else (0, -1)
    st = np.zeros(3, dtype=np.int64)
    _check(lib().orc_assemble_W(im.h, cfg.far_order, cfg.singular_order, cfg.near_threshold, workers, lo, hi,
                                W, st))
    W = W.reshape(n, n)
    return (W, st) if stats else W


class AssemblySampler:
    """Timing model of the reference assemble_W (oracle/sbo.hpp AssemblySampler) for the
    CPU baseline: fixed() times the per-call work (per-worker dense partials allocated and
    zeroed, worker-ordered sum, mirror), run(idx) the pair loop over a sorted sample of
    pair indices split across workers as run_partitioned splits the full range.  Holds
    `workers` resident n x n partials (8 n^2 bytes each)."""

    def __init__(self, im: InflatedMesh, workers: int, cfg: QuadratureConfig = QuadratureConfig()):
        st = C.c_int()
        self.h = lib().orc_sampler_new(im.h, cfg.far_order, cfg.singular_order, cfg.near_threshold, workers,
                                       C.byref(st))
        _check(st.value)
        self.workers = workers

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.orc_sampler_free(self.h)
            self.h = None

    def fixed(self) -> float:
        t = C.c_double()
        _check(lib().orc_sampler_fixed(self.h, C.byref(t)))
        return t.value

    def run(self, idx) -> float:
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        t = C.c_double()
        _check(lib().orc_sampler_run(self.h, idx, len(idx), C.byref(t)))
        return t.value


def systematic_pair_sample(nf: int, k: int, seed: int = 0):
    """k pair indices spread evenly over the reference's pair order (f <= g ranked as
    f(f+1)/2 + g, inc/assemble.hpp:97-103) with one seeded random offset: every region of
    the pair space — near-heavy early rows, far-heavy late rows — in proportion."""
    total = nf * (nf + 1) // 2
    k = max(1, min(int(k), total))
    u = np.random.default_rng(seed).random()
    idx = np.floor((np.arange(k) + u) * (total / k)).astype(np.int64)
    return np.minimum(idx, total - 1)


def assemble_W_rows(im: InflatedMesh, rows, cfg: QuadratureConfig = QuadratureConfig(), workers: int = 0):
    rows = np.ascontiguousarray(rows, dtype=np.int32)
    out = np.zeros(len(rows) * im.n)
    _check(lib().orc_assemble_W_rows(im.h, cfg.far_order, cfg.singular_order, cfg.near_threshold, rows,
                                     len(rows), workers or default_workers(), out))
    return out.reshape(len(rows), im.n)


def rhs_points(im: InflatedMesh, cfg: QuadratureConfig = QuadratureConfig()):
    npt = cfg.far_order ** 2
    pts = np.zeros(im.base.nf * npt * 3)
    lib().orc_rhs_points(im.h, cfg.far_order, pts)
    return pts.reshape(-1, 3)


def assemble_rhs(im: InflatedMesh, g, cfg: QuadratureConfig = QuadratureConfig()):
    """reference: inc/assemble.hpp:143-184; g is a callable of a point or a constant 3-vector."""
    pts = rhs_points(im, cfg)
    if callable(g):
        gv = np.array([g(p) for p in pts], dtype=np.float64).reshape(-1)
    else:
        gv = np.tile(np.asarray(g, dtype=np.float64), len(pts))
    L = np.zeros(im.n)
    _check(lib().orc_assemble_rhs(im.h, cfg.far_order, np.ascontiguousarray(gv), L))
    return L


# --------------------------------------------------------------------------- potential.hpp (3-D)
def distance_to(m: Mesh, points) -> np.ndarray:
    """reference: inc/mesh.hpp:121-133 (SurfaceMesh::distance_to), per point"""
    pts = np.ascontiguousarray(np.asarray(points, dtype=np.float64).reshape(-1, 3))
    out = np.zeros(len(pts))
    _check(lib().orc_distance_to(m.h, pts.reshape(-1), len(pts), out))
    return out


def make_cartesian_grid(m: Mesh, lo: float, hi: float, nx: int, ny: int, mask_eps: float) -> np.ndarray:
    """reference: inc/potential.hpp:15-25 (z = 0 grid, points within mask_eps of the screen dropped)"""
    out = np.zeros(3 * max(nx * ny, 1))
    cnt = C.c_int()
    _check(lib().orc_make_cartesian_grid(m.h, lo, hi, nx, ny, mask_eps, out, C.byref(cnt)))
    return out[:3 * cnt.value].reshape(-1, 3)


def eval_DL(v, im: InflatedMesh, points, cfg: QuadratureConfig = QuadratureConfig(), workers: int = 0):
    """reference: inc/potential.hpp:104-138 (3-D): the double-layer potential of jump vector v at
    the points (n x 3); ValidationError for a point on the screen"""
    vv = np.ascontiguousarray(np.asarray(v, dtype=np.float64))
    if len(vv) != im.n:
        raise ValidationError("jump vector length does not match the DOF count")
    pts = np.ascontiguousarray(np.asarray(points, dtype=np.float64).reshape(-1, 3))
    out = np.zeros(len(pts))
    _check(lib().orc_eval_dl(im.h, vv, pts.reshape(-1), len(pts), cfg.far_order, workers or default_workers(), out))
    return out


def jump_coordinates(im: InflatedMesh, coeff) -> np.ndarray:
    """reference: inc/jump.hpp:61-74 (trace field by gvertex coefficient -> jump coordinates)"""
    c = np.ascontiguousarray(np.asarray(coeff, dtype=np.float64))
    out = np.zeros(im.n)
    _check(lib().orc_jump_coordinates(im.h, c, out))
    return out


# --------------------------------------------------------------------------- prolongation / partition
class Prolongation:
    """reference: inc/jump.hpp:87-89 (CSC export)"""

    def __init__(self, h):
        self.h = h
        r, c, z = C.c_int(), C.c_int(), C.c_int()
        lib().orc_prolongation_sizes(h, C.byref(r), C.byref(c), C.byref(z))
        self.rows, self.cols = r.value, c.value
        self.col_ptr = np.zeros(c.value + 1, dtype=np.int32)
        self.row_idx = np.zeros(z.value, dtype=np.int32)
        self.val = np.zeros(z.value)
        lib().orc_prolongation_export(h, self.col_ptr, self.row_idx, self.val)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.orc_prolongation_free(self.h)
            self.h = None

    def dense(self):
        R = np.zeros((self.rows, self.cols))
        for c in range(self.cols):
            for p in range(self.col_ptr[c], self.col_ptr[c + 1]):
                R[self.row_idx[p], c] = self.val[p]
        return R


def build_prolongation(pair: LevelPair, coarse: InflatedMesh, fine: InflatedMesh) -> Prolongation:
    st = C.c_int()
    h = lib().orc_build_prolongation(pair.h, coarse.h, fine.h, C.byref(st))
    _check(st.value)
    return Prolongation(h)


def empty_prolongation(rows: int) -> Prolongation:
    return Prolongation(lib().orc_empty_prolongation(rows))


def prolongation_from(rows: int, cols: int, col_ptr, row_idx, val) -> Prolongation:
    """a given sparse R in CSC form (jump.hpp:87-89 layout)"""
    return Prolongation(lib().orc_prolongation_from(rows, cols, np.ascontiguousarray(col_ptr, dtype=np.int32),
                                                    np.ascontiguousarray(row_idx, dtype=np.int32),
                                                    np.ascontiguousarray(val, dtype=np.float64)))


def identity_prolongation(n: int) -> Prolongation:
    return Prolongation(lib().orc_identity_prolongation(n))


class DofPartition:
    """reference: inc/schwarz.hpp:14-17 (face_sets in std::map order)"""

    def __init__(self, h):
        self.h = h
        nf, nd, nw = C.c_int(), C.c_int(), C.c_int()
        lib().orc_partition_sizes(h, C.byref(nf), C.byref(nd), C.byref(nw))
        self.face_ids = np.zeros(nf.value, dtype=np.int32)
        self.face_ptr = np.zeros(nf.value + 1, dtype=np.int32)
        self.face_dofs = np.zeros(nd.value, dtype=np.int32)
        self.wirebasket = np.zeros(nw.value, dtype=np.int32)
        lib().orc_partition_export(h, self.face_ids, self.face_ptr, self.face_dofs, self.wirebasket)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.orc_partition_free(self.h)
            self.h = None

    @property
    def face_sets(self):
        return {int(f): self.face_dofs[self.face_ptr[i]:self.face_ptr[i + 1]].copy()
                for i, f in enumerate(self.face_ids)}


def partition_dofs(pair: LevelPair, fine: InflatedMesh) -> DofPartition:
    st = C.c_int()
    h = lib().orc_partition(pair.h, fine.h, C.byref(st))
    _check(st.value)
    return DofPartition(h)


def partition_from(face_sets: dict, wirebasket) -> DofPartition:
    ids = np.array(sorted(face_sets), dtype=np.int32)
    ptr = np.zeros(len(ids) + 1, dtype=np.int32)
    dofs = []
    for i, f in enumerate(ids):
        dofs.extend(face_sets[int(f)])
        ptr[i + 1] = len(dofs)
    wb = np.ascontiguousarray(wirebasket, dtype=np.int32)
    return DofPartition(lib().orc_partition_from(len(ids), ids, ptr, np.array(dofs, dtype=np.int32), len(wb), wb))


# --------------------------------------------------------------------------- Schwarz / PCG
class SchwarzPreconditioner:
    """reference: inc/schwarz.hpp:55-73, build at :100-118, apply at :121-140"""

    def __init__(self, W, part: DofPartition, P: Prolongation):
        W = np.ascontiguousarray(W, dtype=np.float64)
        self.n = W.shape[0]
        st = C.c_int()
        self.h = lib().orc_build_preconditioner(W.reshape(-1), self.n, part.h, P.h, C.byref(st))
        _check(st.value)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.orc_prec_free(self.h)
            self.h = None

    def num_subspaces(self):
        return lib().orc_prec_num_subspaces(self.h)

    def apply(self, r):
        r = np.ascontiguousarray(r, dtype=np.float64)
        z = np.zeros(len(r))
        _check(lib().orc_apply_preconditioner(self.h, r, len(r), z))
        return z

    def block_diag(self, which: int):
        n = C.c_int()
        lib().orc_prec_block_diag(self.h, which, None, C.byref(n))
        d = np.zeros(n.value)
        lib().orc_prec_block_diag(self.h, which, d.ctypes.data_as(C.c_void_p), C.byref(n))
        return d


def build_preconditioner(W, part, P) -> SchwarzPreconditioner:
    return SchwarzPreconditioner(W, part, P)


def apply_preconditioner(prec: SchwarzPreconditioner, r):
    return prec.apply(r)


def materialize_preconditioner(prec: SchwarzPreconditioner):
    """reference: inc/schwarz.hpp:142-148"""
    M = np.zeros((prec.n, prec.n))
    for j in range(prec.n):
        e = np.zeros(prec.n)
        e[j] = 1.0
        M[:, j] = prec.apply(e)
    return M


def spectrum_of(S):
    """reference: inc/schwarz.hpp:156-166 (Eigen SelfAdjointEigenSolver -> LAPACK syevd via numpy)"""
    S = np.asarray(S, dtype=np.float64)
    if S.size == 0:
        raise ValidationError("spectrum of an empty matrix")
    ev = np.linalg.eigvalsh(S)
    return ev[0], ev[-1], ev[-1] / ev[0]


def condition_number(W, M=None):
    """reference: inc/schwarz.hpp:168-190: kappa(W) from 0.5 (W + W^T); with a
    preconditioner (SchwarzPreconditioner or materialized M) the spectrum of the
    Cholesky congruence L^T M L.  Returns (lambda_min, lambda_max, kappa)."""
    W = np.asarray(W, dtype=np.float64)
    if M is None:
        return spectrum_of(0.5 * (W + W.T))
    if isinstance(M, SchwarzPreconditioner):
        M = materialize_preconditioner(M)
    try:
        L = np.linalg.cholesky(W)
    except np.linalg.LinAlgError as e:
        raise NumericalError("Cholesky factorization failed: matrix not positive definite") from e
    S = L.T @ M @ L
    return spectrum_of(0.5 * (S + S.T))


def coarse_matrix(W, P: Prolongation):
    W = np.ascontiguousarray(W, dtype=np.float64)
    H = np.zeros(P.cols * P.cols)
    lib().orc_coarse_matrix(W.reshape(-1), W.shape[0], P.h, H)
    return H.reshape(P.cols, P.cols)


@dataclass
class PcgReport:
    """reference: inc/pcg.hpp:9-16"""
    solution: np.ndarray
    iterations: int
    converged: bool
    residual_history: np.ndarray
    energy_error_history: np.ndarray
    kappa_estimate: float
    alphas: np.ndarray = field(default_factory=lambda: np.zeros(0))
    betas: np.ndarray = field(default_factory=lambda: np.zeros(0))


def pcg(W, prec, rhs, tol=1e-8, maxit=0, exact=None) -> PcgReport:
    """reference: inc/pcg.hpp:33-116"""
    W = np.ascontiguousarray(W, dtype=np.float64)
    n = W.shape[0]
    rhs = np.ascontiguousarray(rhs, dtype=np.float64)
    cap = (maxit if maxit > 0 else max(10 * n, 100)) + 2
    x = np.zeros(n)
    it, conv, kap, hl = C.c_int(), C.c_int(), C.c_double(), C.c_int()
    hist, en, al, be = np.zeros(cap), np.zeros(cap), np.zeros(cap), np.zeros(cap)
    ex = None
    if exact is not None:
        ex = np.ascontiguousarray(exact, dtype=np.float64)
    _check(lib().orc_pcg(W.reshape(-1), n, prec.h if prec is not None else None, rhs, tol, maxit,
                         ex.ctypes.data_as(C.c_void_p) if ex is not None else None, x, C.byref(it), C.byref(conv),
                         C.byref(kap), hist, en.ctypes.data_as(C.c_void_p), al, be, cap, C.byref(hl)))
    k = it.value
    nb = k  # betas has one entry per completed iteration
    return PcgReport(x, k, bool(conv.value), hist[:hl.value].copy(),
                     en[:hl.value].copy() if ex is not None else np.zeros(0), kap.value, al[:k].copy(),
                     be[:nb].copy())


def matvec(W, x, reps: int = 1):
    """y = W x as in the PCG loop (pcg.hpp:70), dense row-major, single thread."""
    W = np.ascontiguousarray(W, dtype=np.float64)
    y = np.zeros(W.shape[0])
    _check(lib().orc_matvec(W.reshape(-1), W.shape[0], np.ascontiguousarray(x, dtype=np.float64), y, reps))
    return y


def direct_solve(W, rhs):
    W = np.ascontiguousarray(W, dtype=np.float64)
    x = np.zeros(W.shape[0])
    _check(lib().orc_direct_solve(W.reshape(-1), W.shape[0], np.ascontiguousarray(rhs, dtype=np.float64), x))
    return x


def lanczos_kappa(alphas, betas) -> float:
    a = np.ascontiguousarray(alphas, dtype=np.float64)
    b = np.ascontiguousarray(betas, dtype=np.float64)
    if len(b) < len(a):
        b = np.concatenate([b, np.zeros(len(a) - len(b))])
    return lib().orc_lanczos_kappa(a, b, len(a))


def random_spd(n: int, seed: int):
    """tests/test_pcg.cpp:12-20 with std::mt19937 + std::normal_distribution"""
    W = np.zeros(n * n)
    lib().orc_random_spd(n, seed, W)
    return W.reshape(n, n)


def normal_draws(seed: int, count: int):
    out = np.zeros(count)
    lib().orc_normal_draws(seed, count, out)
    return out


def seeded_unit_vector(seed: int):
    """g from std::mt19937(seed), 3 normal draws, normalised (SURVEY.md §8d cfg 2/4)."""
    v = normal_draws(seed, 3)
    return v / np.sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2])


# --------------------------------------------------------------------------- BASELINE configs
# The oracle's own restatement of the SURVEY.md Appendix A panel generator, so the CPU
# baseline and the reference arm of bench.py never load the product library.  The
# geometry follows the reference's flat-square fixture (tests/test_inflate.cpp:14-15:
# cell (i,j) -> {p00,p10,p11},{p00,p11,p01}); coincident vertices of different panels
# are merged by position quantised to 1e-9 (conformity, inc/mesh.hpp:191-234); the
# parent map is Appendix A's.  tests/test_host_parity.py checks it bit for bit against
# the product's make_config.
def _llround(x: float) -> int:
    import math
    return int(math.copysign(math.floor(abs(x) + 0.5), x))


def _panel_mesh(panels, L: float, m: int):
    verts, facets, ids = [], [], {}
    for o, a, b in panels:
        local = np.zeros((m + 1, m + 1), dtype=np.int64)  # [j][i]
        for j in range(m + 1):
            sj = (L * j) / m
            for i in range(m + 1):
                si = (L * i) / m
                p = ((o[0] + si * a[0]) + sj * b[0], (o[1] + si * a[1]) + sj * b[1],
                     (o[2] + si * a[2]) + sj * b[2])
                k = (_llround(p[0] * 1e9), _llround(p[1] * 1e9), _llround(p[2] * 1e9))
                vid = ids.get(k)
                if vid is None:
                    vid = ids[k] = len(verts)
                    verts.append(p)
                local[j, i] = vid
        for j in range(m):
            for i in range(m):
                p00, p10, p11, p01 = local[j, i], local[j, i + 1], local[j + 1, i + 1], local[j + 1, i]
                facets.append((p00, p10, p11))
                facets.append((p00, p11, p01))
    return Mesh(np.array(verts, dtype=np.float64), np.array(facets, dtype=np.int32))


def make_panels(kind: int, m: int, r: int) -> LevelPair:
    """kind 0: flat unit square; 1: T-junction of three unit squares about the z-axis
    (azimuth 0, 120, 240 degrees); 2: triple cross of [-1,1]^2 in the coordinate planes."""
    import math
    if r < 1 or m % r:
        raise ValidationError("panel refinement ratio must divide the cell count")
    L = 1.0
    if kind == 0:
        P = [((0.0, 0.0, 0.0), (1.0, 0.0, 0.0), (0.0, 1.0, 0.0))]
    elif kind == 1:
        P = []
        for k in range(3):
            th = 2.0 * math.pi * k / 3.0
            P.append(((0.0, 0.0, 0.0), (math.cos(th), math.sin(th), 0.0), (0.0, 0.0, 1.0)))
    elif kind == 2:
        if m % 2:
            raise ValidationError("triple cross needs an even cell count")
        L = 2.0
        P = [((-1.0, -1.0, 0.0), (1.0, 0.0, 0.0), (0.0, 1.0, 0.0)),
             ((0.0, -1.0, -1.0), (0.0, 1.0, 0.0), (0.0, 0.0, 1.0)),
             ((-1.0, 0.0, -1.0), (1.0, 0.0, 0.0), (0.0, 0.0, 1.0))]
    else:
        raise ValidationError(f"unknown panel geometry kind {kind}")
    mc = m // r
    fine, coarse = _panel_mesh(P, L, m), _panel_mesh(P, L, mc)
    parent = np.zeros(fine.nf, dtype=np.int32)
    for p in range(len(P)):
        for j in range(m):
            for i in range(m):
                I, J, a, b = i // r, j // r, i % r, j % r
                cbase = p * 2 * mc * mc + 2 * (J * mc + I)
                fbase = p * 2 * m * m + 2 * (j * m + i)
                parent[fbase] = cbase + (0 if b <= a else 1)
                parent[fbase + 1] = cbase + (1 if a <= b else 0)
    return LevelPair(coarse, fine, parent)


CONFIG_DEFAULT_RATIO = {1: 8, 2: 16, 3: 12, 4: 8, 5: 8}


def make_config(cfg: int, ratio: int = 0) -> LevelPair:
    """BASELINE.json configs[cfg-1]."""
    kind, m = {1: (0, 16), 2: (0, 64), 3: (1, 48), 4: (2, 64), 5: (0, 160)}[cfg]
    return make_panels(kind, m, ratio if ratio > 0 else CONFIG_DEFAULT_RATIO[cfg])


def config_g(cfg: int):
    """Neumann field g of a BASELINE config (seeded unit vectors for cfg 2/4)."""
    if cfg in (2, 4):
        return seeded_unit_vector(1 if cfg == 2 else 7)
    if cfg == 3:
        return np.array([1.0, 0.5, 0.25])
    if cfg in (1, 5):
        return np.array([0.0, 0.0, 1.0])
    raise ValidationError(f"unknown BASELINE config {cfg}")
