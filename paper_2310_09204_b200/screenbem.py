"""Host-side mirror of the reference's screenbem API over the sm_100a C ABI.

Names, argument meaning and error classes follow proj/include/screenbem/*.hpp
(ValidationError -> exit 2, NumericalError -> exit 3); every call goes through
libscreenbem_b200.so (include/screenbem_b200.h).  There is no CPU fallback:
the device entry points raise CudaError when no B200 is usable, and importing
this module fails loudly if the shared library has not been built.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SBG_LIB_PATH: an alternative build of the same library (A/B measurements of kernel variants)
LIB_PATH = os.environ.get("SBG_LIB_PATH") or os.path.join(_HERE, "_lib", "libscreenbem_b200.so")


class ValidationError(RuntimeError):
    """reference: inc/common.hpp:17-20 (CLI exit code 2)"""


class NumericalError(RuntimeError):
    """reference: inc/common.hpp:23-26 (CLI exit code 3)"""


class CudaError(RuntimeError):
    """No usable sm_100a device or a CUDA runtime failure."""


i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
vp = C.c_void_p


class QuadCfgC(C.Structure):
    _fields_ = [("far_order", C.c_int), ("singular_order", C.c_int), ("near_threshold", C.c_double),
                ("exact_far", C.c_int)]


class PcgReportC(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("kappa_estimate", C.c_double),
                ("history_len", C.c_int)]


class AssemblyStatsC(C.Structure):
    _fields_ = [(n, C.c_longlong) for n in ("far_pairs", "near_pairs", "identical", "edge", "vertex",
                                             "near_leaves", "tiles", "tiles_skipped", "h2d_bytes")]


# signature table: name -> (restype, argtypes); also the exported-symbol contract
SIGNATURES = {
    "sbg_last_error": (C.c_char_p, []),
    "sbg_version": (C.c_char_p, []),
    "sbg_ctx_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
    "sbg_ctx_destroy": (None, [vp]),
    "sbg_ctx_synchronize": (C.c_int, [vp]),
    "sbg_ctx_set_matvec_form": (C.c_int, [vp, C.c_int]),
    "sbg_ctx_get_matvec_form": (C.c_int, [vp, C.POINTER(C.c_int)]),
    "sbg_device_name": (C.c_int, [C.c_int, C.c_char_p, C.c_int, C.POINTER(C.c_int)]),
    "sbg_timers_enable": (C.c_int, [vp, C.c_int]),
    "sbg_timers_reset": (C.c_int, [vp]),
    "sbg_timer_get": (C.c_int, [vp, C.c_char_p, C.POINTER(C.c_double), C.POINTER(C.c_longlong)]),
    "sbg_timer_begin": (C.c_int, [vp, C.c_char_p]),
    "sbg_timer_end": (C.c_int, [vp]),
    "sbg_launch_count": (C.c_longlong, []),
    "sbg_assembly_plan_create": (C.c_int, [vp, vp, C.POINTER(QuadCfgC), C.POINTER(vp)]),
    "sbg_assembly_run": (C.c_int, [vp, C.POINTER(vp), C.POINTER(AssemblyStatsC)]),
    "sbg_assembly_run_shard": (C.c_int, [vp, C.POINTER(vp), C.c_int, C.c_int, C.POINTER(AssemblyStatsC)]),
    "sbg_matrix_device_view": (C.c_int, [vp, C.POINTER(vp), C.POINTER(C.c_int), C.POINTER(C.c_longlong)]),
    "sbg_matrix_pack_upper": (C.c_int, [vp, vp]),
    "sbg_matrix_unpack_upper": (C.c_int, [vp, vp]),
    "sbg_assembly_plan_destroy": (None, [vp]),
    "sbg_mesh_create": (C.c_int, [C.c_int, f64p, C.c_int, i32p, C.POINTER(vp)]),
    "sbg_mesh_destroy": (None, [vp]),
    "sbg_mesh_sizes": (C.c_int, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "sbg_mesh_export": (C.c_int, [vp, f64p, i32p]),
    "sbg_validate_mesh": (C.c_int, [vp]),
    "sbg_make_builtin": (C.c_int, [C.c_char_p, C.POINTER(vp)]),
    "sbg_refine_uniform_times": (C.c_int, [vp, C.c_int, C.POINTER(vp)]),
    "sbg_level_create": (C.c_int, [vp, vp, i32p, C.POINTER(vp)]),
    "sbg_make_config": (C.c_int, [C.c_int, C.c_int, C.POINTER(vp)]),
    "sbg_make_panels": (C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(vp)]),
    "sbg_level_mesh": (C.c_int, [vp, C.c_int, C.POINTER(vp)]),
    "sbg_level_parent": (C.c_int, [vp, i32p]),
    "sbg_level_sizes": (C.c_int, [vp, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "sbg_level_destroy": (None, [vp]),
    "sbg_inflate": (C.c_int, [vp, C.c_int, C.POINTER(vp)]),
    "sbg_inflated_destroy": (None, [vp]),
    "sbg_inflated_sizes": (C.c_int, [vp] + [C.POINTER(C.c_int)] * 4),
    "sbg_inflated_export": (C.c_int, [vp, i32p, i32p, i32p, i32p, i32p, f64p]),
    "sbg_assemble_w": (C.c_int, [vp, vp, C.POINTER(QuadCfgC), C.c_int, C.POINTER(vp), C.POINTER(AssemblyStatsC)]),
    "sbg_assemble_w_host": (C.c_int, [vp, vp, C.POINTER(QuadCfgC), C.c_int, vp, C.POINTER(vp),
                                      C.POINTER(AssemblyStatsC)]),
    "sbg_matrix_create": (C.c_int, [vp, C.c_int, C.c_void_p, C.POINTER(vp)]),
    "sbg_matrix_n": (C.c_int, [vp]),
    "sbg_matrix_download": (C.c_int, [vp, f64p]),
    "sbg_matrix_download_rows": (C.c_int, [vp, i32p, C.c_int, f64p]),
    "sbg_matrix_symmetry_defect": (C.c_int, [vp, C.POINTER(C.c_double)]),
    "sbg_matvec": (C.c_int, [vp, vp, f64p, f64p]),
    "sbg_matrix_destroy": (None, [vp]),
    "sbg_matrix_dump_binary": (C.c_int, [vp, C.c_char_p]),
    "sbg_matrix_load_binary": (C.c_int, [vp, C.c_char_p, C.POINTER(vp)]),
    "sbg_pair_integrals": (C.c_int, [vp, vp, C.POINTER(QuadCfgC), i32p, i32p, C.c_longlong, f64p]),
    "sbg_rhs_points": (C.c_int, [vp, C.POINTER(QuadCfgC), f64p]),
    "sbg_assemble_rhs": (C.c_int, [vp, vp, C.POINTER(QuadCfgC), f64p, C.c_int, f64p]),
    "sbg_eval_dl": (C.c_int, [vp, vp, C.c_void_p, C.c_void_p, C.c_longlong, C.POINTER(QuadCfgC), C.c_void_p]),
    "sbg_make_cartesian_grid": (C.c_int, [vp, vp, C.c_double, C.c_double, C.c_int, C.c_int, C.c_double, C.c_void_p,
                                          C.POINTER(C.c_int)]),
    "sbg_partition_dofs": (C.c_int, [vp, vp, C.POINTER(vp)]),
    "sbg_partition_create": (C.c_int, [C.c_int, i32p, i32p, i32p, C.c_int, i32p, C.POINTER(vp)]),
    "sbg_partition_sizes": (C.c_int, [vp] + [C.POINTER(C.c_int)] * 3),
    "sbg_partition_export": (C.c_int, [vp, i32p, i32p, i32p, i32p]),
    "sbg_partition_destroy": (None, [vp]),
    "sbg_build_prolongation": (C.c_int, [vp, vp, vp, C.POINTER(vp)]),
    "sbg_prolong_create": (C.c_int, [C.c_int, C.c_int, i32p, i32p, f64p, C.POINTER(vp)]),
    "sbg_prolong_sizes": (C.c_int, [vp] + [C.POINTER(C.c_int)] * 3),
    "sbg_prolong_export": (C.c_int, [vp, i32p, i32p, f64p]),
    "sbg_prolong_destroy": (None, [vp]),
    "sbg_build_preconditioner": (C.c_int, [vp, vp, vp, vp, C.POINTER(vp)]),
    "sbg_build_preconditioner_mode": (C.c_int, [vp, vp, vp, vp, C.c_int, C.POINTER(vp)]),
    "sbg_apply_preconditioner": (C.c_int, [vp, vp, f64p, C.c_int, f64p]),
    "sbg_prec_num_subspaces": (C.c_int, [vp]),
    "sbg_prec_block_diag": (C.c_int, [vp, vp, C.c_int, C.c_void_p, C.POINTER(C.c_int)]),
    "sbg_coarse_matrix": (C.c_int, [vp, vp, vp, f64p]),
    "sbg_prec_factor_bytes": (C.c_double, [vp]),
    "sbg_materialize_preconditioner": (C.c_int, [vp, vp, C.POINTER(vp)]),
    "sbg_prec_from_dense": (C.c_int, [vp, vp, C.POINTER(vp)]),
    "sbg_condition_number": (C.c_int, [vp, vp, vp, C.c_double, C.c_int, C.c_void_p]),
    "sbg_prec_destroy": (None, [vp]),
    "sbg_pcg": (C.c_int, [vp, vp, vp, f64p, C.c_int, C.c_double, C.c_int, f64p, f64p, f64p, f64p, C.c_int,
                          C.POINTER(PcgReportC)]),
    "sbg_pcg_exact": (C.c_int, [vp, vp, vp, f64p, C.c_int, C.c_double, C.c_int, f64p, f64p, f64p, f64p, f64p, f64p,
                                C.c_int, C.POINTER(PcgReportC)]),
    "sbg_pcg_rows": (C.c_int, [vp, vp, vp, vp, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int,
                               vp, vp, vp, f64p, f64p, f64p, C.c_int, C.POINTER(PcgReportC)]),
    "sbg_pcg_rows_agree": (C.c_int, [vp, vp, vp, vp, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int,
                                     vp, vp, vp, vp, f64p, f64p, f64p, C.c_int, C.POINTER(PcgReportC)]),
    "sbg_matvec_rows_device": (C.c_int, [vp, vp, vp, vp, C.c_int, C.c_int]),
    "sbg_ctx_stream": (C.c_int, [vp, C.POINTER(vp)]),
    "sbg_device_alloc": (C.c_int, [vp, C.c_longlong, C.POINTER(vp)]),
    "sbg_device_free": (C.c_int, [vp]),
    "sbg_host_alloc": (C.c_int, [C.c_longlong, C.POINTER(vp)]),
    "sbg_host_free": (C.c_int, [vp]),
    "sbg_memcpy_h2d": (C.c_int, [vp, vp, vp, C.c_longlong]),
    "sbg_memcpy_d2h": (C.c_int, [vp, vp, vp, C.c_longlong]),
    "sbg_pcg_device": (C.c_int, [vp, vp, vp, vp, C.c_double, C.c_int, vp, C.POINTER(PcgReportC)]),
    "sbg_matvec_device": (C.c_int, [vp, vp, vp, vp, C.c_int]),
    "sbg_matvec_bytes": (C.c_int, [vp, vp, C.POINTER(C.c_double)]),
    "sbg_apply_preconditioner_device": (C.c_int, [vp, vp, vp, vp, C.c_int]),
    "sbg_l2_flush": (C.c_int, [vp]),
    "sbg_pool_stats": (C.c_int, [vp, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)]),
    "sbg_fp64_peak": (C.c_int, [vp, C.POINTER(C.c_double)]),
    "sbg_config_g": (C.c_int, [C.c_int, f64p]),
}

_lib = None


def lib():
    """Load libscreenbem_b200.so; raises if it is missing (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(rc: int):
    if rc == 0:
        return
    msg = lib().sbg_last_error().decode()
    if rc == 2:
        raise ValidationError(msg)
    if rc == 3:
        raise NumericalError(msg)
    if rc == 4:
        raise CudaError(msg)
    raise RuntimeError(msg)


class _Handle:
    _destroy = None

    def __init__(self, h):
        self.h = h

    def __del__(self):
        h = getattr(self, "h", None)
        if h and _lib is not None and self._destroy:
            getattr(_lib, self._destroy)(h)
            self.h = None


# --------------------------------------------------------------------------- context
class Context(_Handle):
    """One CUDA stream on one B200; all device objects live on a context."""
    _destroy = "sbg_ctx_destroy"

    def __init__(self, device: int = 0):
        h = vp()
        _check(lib().sbg_ctx_create(device, C.byref(h)))
        super().__init__(h)
        self.device = device

    def synchronize(self):
        _check(lib().sbg_ctx_synchronize(self.h))

    @property
    def matvec_form(self) -> str:
        """"symmetric" (default: W x from the upper triangle, n >= 2048) or "full" (every entry;
        the row kernel sbg_pcg_rows shares, so pcg_rows then equals pcg bitwise)"""
        f = C.c_int()
        _check(lib().sbg_ctx_get_matvec_form(self.h, C.byref(f)))
        return ("symmetric", "full")[f.value]

    @matvec_form.setter
    def matvec_form(self, form: str):
        if form not in ("symmetric", "full"):
            raise ValidationError("matvec_form: 'symmetric' or 'full'")
        _check(lib().sbg_ctx_set_matvec_form(self.h, 0 if form == "symmetric" else 1))

    @property
    def stream(self) -> int:
        """The context's cudaStream_t (address), e.g. for torch.cuda.ExternalStream."""
        p = vp()
        _check(lib().sbg_ctx_stream(self.h, C.byref(p)))
        return p.value or 0

    def timers(self, on: bool = True):
        _check(lib().sbg_timers_enable(self.h, 1 if on else 0))

    def reset_timers(self):
        _check(lib().sbg_timers_reset(self.h))

    def timer(self, name: str):
        ms, cnt = C.c_double(), C.c_longlong()
        _check(lib().sbg_timer_get(self.h, name.encode(), C.byref(ms), C.byref(cnt)))
        return ms.value, cnt.value

    def l2_flush(self):
        _check(lib().sbg_l2_flush(self.h))

    def pool_stats(self):
        """(reserved, used) bytes of the device memory pool"""
        r, u = C.c_longlong(), C.c_longlong()
        _check(lib().sbg_pool_stats(self.h, C.byref(r), C.byref(u)))
        return r.value, u.value

    def begin(self, name: str):
        _check(lib().sbg_timer_begin(self.h, name.encode()))

    def end(self):
        _check(lib().sbg_timer_end(self.h))


def fp64_peak_tflops(ctx: "Context" = None) -> float:
    """Measured DFMA throughput of the device (TFLOP/s)."""
    ctx = ctx or default_context()
    t = C.c_double()
    _check(lib().sbg_fp64_peak(ctx.h, C.byref(t)))
    return t.value


def config_g(cfg: int):
    """Neumann field g of a BASELINE config (seeded std::mt19937 draws for cfg 2 and 4)."""
    g = np.zeros(3)
    _check(lib().sbg_config_g(cfg, g))
    return g


def launch_count() -> int:
    """Kernels launched by libscreenbem_b200 so far (all contexts)."""
    return lib().sbg_launch_count()


class _PinnedBlock:
    """Owner of one sbg_host_alloc block (freed when the last array view goes away)."""

    def __init__(self, nbytes):
        self.p = vp()
        _check(lib().sbg_host_alloc(max(int(nbytes), 1), C.byref(self.p)))

    def __del__(self):
        if getattr(self, "p", None) and _lib is not None:
            _lib.sbg_host_free(self.p)
            self.p = None


def pinned_empty(shape, dtype=np.float64):
    """Uninitialised numpy array in page-locked host memory: GalerkinMatrix.download(out=)
    into it is a single DMA, without the staging copy a pageable destination needs."""
    dtype = np.dtype(dtype)
    count = int(np.prod(shape)) if np.ndim(shape) else int(shape)
    blk = _PinnedBlock(count * dtype.itemsize)
    raw = (C.c_char * max(count * dtype.itemsize, 1)).from_address(blk.p.value)
    raw._owner = blk  # keep the block alive as long as any view of it
    return np.frombuffer(raw, dtype=dtype, count=count).reshape(shape)


_default_ctx = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(int(os.environ.get("LOCAL_RANK", "0")) if os.environ.get("SBG_USE_LOCAL_RANK") else 0)
    return _default_ctx


def device_name(device: int = 0):
    buf = C.create_string_buffer(256)
    sms = C.c_int()
    _check(lib().sbg_device_name(device, buf, 256, C.byref(sms)))
    return buf.value.decode(), sms.value


# --------------------------------------------------------------------------- meshes
class SurfaceMesh(_Handle):
    """reference: inc/mesh.hpp:19-83 (3-D triangles)"""
    _destroy = "sbg_mesh_destroy"

    def __init__(self, vertices, facets, _handle=None):
        if _handle is None:
            v = np.ascontiguousarray(vertices, dtype=np.float64).reshape(-1)
            f = np.ascontiguousarray(facets, dtype=np.int32).reshape(-1)
            h = vp()
            _check(lib().sbg_mesh_create(len(v) // 3, v, len(f) // 3, f, C.byref(h)))
            _handle = h
        super().__init__(_handle)
        nv, nf = C.c_int(), C.c_int()
        _check(lib().sbg_mesh_sizes(self.h, C.byref(nv), C.byref(nf)))
        self.vertices = np.zeros((nv.value, 3))
        self.facets = np.zeros((nf.value, 3), dtype=np.int32)
        _check(lib().sbg_mesh_export(self.h, self.vertices.reshape(-1), self.facets.reshape(-1)))

    @property
    def nf(self):
        return len(self.facets)

    @property
    def nv(self):
        return len(self.vertices)

    def num_facets(self):
        return self.nf

    def num_vertices(self):
        return self.nv


def validate_mesh(m: SurfaceMesh):
    """reference: inc/mesh.hpp:238-272"""
    _check(lib().sbg_validate_mesh(m.h))


def make_builtin(spec: str) -> SurfaceMesh:
    """reference: inc/mesh.hpp:516-537 (3-D builtin "bowtie[:k]")"""
    h = vp()
    _check(lib().sbg_make_builtin(spec.encode(), C.byref(h)))
    return SurfaceMesh(None, None, _handle=h)


class MeshLevelPair(_Handle):
    """reference: inc/mesh.hpp:86-92"""
    _destroy = "sbg_level_destroy"

    def __init__(self, coarse: SurfaceMesh = None, fine: SurfaceMesh = None, parent=None, _handle=None):
        if _handle is None:
            h = vp()
            _check(lib().sbg_level_create(coarse.h, fine.h, np.ascontiguousarray(parent, dtype=np.int32),
                                          C.byref(h)))
            _handle = h
        super().__init__(_handle)
        hc, hf = vp(), vp()
        _check(lib().sbg_level_mesh(self.h, 0, C.byref(hc)))
        _check(lib().sbg_level_mesh(self.h, 1, C.byref(hf)))
        self.coarse = SurfaceMesh(None, None, _handle=hc)
        self.fine = SurfaceMesh(None, None, _handle=hf)
        self.parent = np.zeros(self.fine.nf, dtype=np.int32)
        _check(lib().sbg_level_parent(self.h, self.parent))
        H, hh = C.c_double(), C.c_double()
        _check(lib().sbg_level_sizes(self.h, C.byref(H), C.byref(hh)))
        self.H, self.h_fine = H.value, hh.value


def refine_uniform_times(m: SurfaceMesh, k: int) -> MeshLevelPair:
    """reference: inc/mesh.hpp:388-405"""
    h = vp()
    _check(lib().sbg_refine_uniform_times(m.h, k, C.byref(h)))
    return MeshLevelPair(_handle=h)


def make_config(cfg: int, ratio: int = 0) -> MeshLevelPair:
    """BASELINE.json configs 1-5 with their nested coarse mesh."""
    h = vp()
    _check(lib().sbg_make_config(cfg, ratio, C.byref(h)))
    return MeshLevelPair(_handle=h)


def make_panels(kind: int, m: int, r: int) -> MeshLevelPair:
    """Panel geometries: 0 flat unit square, 1 T-junction, 2 triple cross; m cells, ratio r."""
    h = vp()
    _check(lib().sbg_make_panels(kind, m, r, C.byref(h)))
    return MeshLevelPair(_handle=h)


def identity_pair(m: SurfaceMesh) -> MeshLevelPair:
    """H = h pair (tests/test_schwarz.cpp:35-44)"""
    return MeshLevelPair(m, m, np.arange(m.nf, dtype=np.int32))


# --------------------------------------------------------------------------- inflation
class InflatedMesh(_Handle):
    """reference: inc/inflate.hpp:48-76"""
    _destroy = "sbg_inflated_destroy"

    def __init__(self, mesh: SurfaceMesh, validate: bool = True):
        h = vp()
        _check(lib().sbg_inflate(mesh.h, 1 if validate else 0, C.byref(h)))
        super().__init__(h)
        self.base = mesh
        n, ng, nv, nf = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        _check(lib().sbg_inflated_sizes(h, C.byref(n), C.byref(ng), C.byref(nv), C.byref(nf)))
        self.n, self.n_gvertices = n.value, ng.value
        self.q = np.zeros(nv.value, dtype=np.int32)
        self.gv_first = np.zeros(nv.value, dtype=np.int32)
        self.dof_first = np.zeros(nv.value, dtype=np.int32)
        self.ofacet_branch = np.zeros(6 * nf.value, dtype=np.int32)
        self.jump_dofs = np.zeros(2 * self.n, dtype=np.int32)
        self.normals = np.zeros(6 * nf.value)
        _check(lib().sbg_inflated_export(h, self.q, self.gv_first, self.dof_first, self.ofacet_branch,
                                         self.jump_dofs, self.normals))
        self.ofacet_branch = self.ofacet_branch.reshape(-1, 3)
        self.jump_dofs = self.jump_dofs.reshape(-1, 2)
        self.normals = self.normals.reshape(-1, 3)

    def num_jump_dofs(self):
        return self.n


def inflate(mesh: SurfaceMesh, validate: bool = True) -> InflatedMesh:
    return InflatedMesh(mesh, validate)


# --------------------------------------------------------------------------- quadrature / assembly
@dataclass
class QuadratureConfig:
    """reference: inc/quadrature.hpp:12-16"""
    far_order: int = 4
    singular_order: int = 8
    near_threshold: float = 2.0
    exact_far: bool = False  # far pairs bitwise like the CPU restatement

    def c(self):
        return QuadCfgC(self.far_order, self.singular_order, self.near_threshold, 1 if self.exact_far else 0)


class GalerkinMatrix(_Handle):
    """Dense symmetric W resident in HBM (reference: inc/assemble.hpp:12)."""
    _destroy = "sbg_matrix_destroy"

    def __init__(self, h, ctx: Context, stats=None):
        super().__init__(h)
        self.ctx = ctx
        self.n = lib().sbg_matrix_n(h)
        self.stats = stats

    @classmethod
    def from_host(cls, W, ctx: Context = None):
        ctx = ctx or default_context()
        W = np.ascontiguousarray(W, dtype=np.float64)
        h = vp()
        _check(lib().sbg_matrix_create(ctx.h, W.shape[0], W.ctypes.data_as(C.c_void_p), C.byref(h)))
        return cls(h, ctx)

    def download(self, out=None):
        """Row-major host copy (n x n); `out` may supply a C-contiguous float64 buffer."""
        if out is None:
            out = np.empty((self.n, self.n))
        elif out.shape != (self.n, self.n) or out.dtype != np.float64 or not out.flags.c_contiguous:
            raise ValidationError("download: out must be a C-contiguous float64 (n, n) array")
        _check(lib().sbg_matrix_download(self.h, out.reshape(-1)))
        return out

    @property
    def __cuda_array_interface__(self):
        """The device storage, row-major (n, ld) float64 with zero padding columns: lets
        torch / NCCL reduce the shards of a sharded assembly in place (AssemblyPlan.run)."""
        p, ld, cnt = vp(), C.c_int(), C.c_longlong()
        _check(lib().sbg_matrix_device_view(self.h, C.byref(p), C.byref(ld), C.byref(cnt)))
        return {"shape": (self.n, ld.value), "typestr": "<f8", "data": (p.value or 0, False), "version": 3,
                "strides": None, "stream": None}

    def pack_upper(self, d_packed: int):
        """the upper triangle into the device vector at d_packed (n (n + 1) / 2 doubles)"""
        _check(lib().sbg_matrix_pack_upper(self.h, d_packed))

    def unpack_upper(self, d_packed: int):
        """W (both triangles) from a packed upper triangle at d_packed"""
        _check(lib().sbg_matrix_unpack_upper(self.h, d_packed))

    def rows(self, rows):
        rows = np.ascontiguousarray(rows, dtype=np.int32)
        out = np.zeros(len(rows) * self.n)
        _check(lib().sbg_matrix_download_rows(self.h, rows, len(rows), out))
        return out.reshape(len(rows), self.n)

    def symmetry_defect(self):
        d = C.c_double()
        _check(lib().sbg_matrix_symmetry_defect(self.h, C.byref(d)))
        return d.value

    def matvec(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(self.n)
        _check(lib().sbg_matvec(self.ctx.h, self.h, x, y))
        return y

    def dump_binary(self, path):
        """dump_matrix_binary (inc/assemble.hpp:191-205)"""
        _check(lib().sbg_matrix_dump_binary(self.h, str(path).encode()))

    @classmethod
    def load_binary(cls, path, ctx: Context = None):
        """load_matrix_binary (inc/assemble.hpp:207-226)"""
        ctx = ctx or default_context()
        h = vp()
        _check(lib().sbg_matrix_load_binary(ctx.h, str(path).encode(), C.byref(h)))
        return cls(h, ctx)


def assemble_W(im: InflatedMesh, cfg: QuadratureConfig = None, workers: int = 1, ctx: Context = None, out=None):
    """reference: inc/assemble.hpp:72-139.  `workers` is accepted and ignored.  `out` (an n x n
    C-contiguous float64 array): also fill it with W — the reference returns W by value on the
    host; a page-locked `out` (pinned_empty) gets the copy overlapped with the near field."""
    ctx = ctx or default_context()
    cfg = cfg or QuadratureConfig()
    c = cfg.c()
    st = AssemblyStatsC()
    h = vp()
    if out is None:
        _check(lib().sbg_assemble_w(ctx.h, im.h, C.byref(c), workers, C.byref(h), C.byref(st)))
    else:
        n = im.n
        if not (isinstance(out, np.ndarray) and out.dtype == np.float64 and out.flags.c_contiguous
                and out.size == n * n):
            raise ValidationError("assemble_W: out must be a C-contiguous float64 array of n*n entries")
        _check(lib().sbg_assemble_w_host(ctx.h, im.h, C.byref(c), workers, out.ctypes.data, C.byref(h),
                                         C.byref(st)))
    stats = {n: getattr(st, n) for n, _ in AssemblyStatsC._fields_}
    return GalerkinMatrix(h, ctx, stats)


class AssemblyPlan(_Handle):
    """Mesh-derived device data of assemble_W, built once (host preparation);
    run() is the device-only assembly into a resident GalerkinMatrix."""
    _destroy = "sbg_assembly_plan_destroy"

    def __init__(self, im: InflatedMesh, cfg: QuadratureConfig = None, ctx: Context = None):
        self.ctx = ctx or default_context()
        cfg = cfg or QuadratureConfig()
        c = cfg.c()
        h = vp()
        _check(lib().sbg_assembly_plan_create(self.ctx.h, im.h, C.byref(c), C.byref(h)))
        super().__init__(h)
        self.n, self.nf = im.n, im.base.nf
        self._W = None

    def run(self, W: GalerkinMatrix = None, shard=None) -> GalerkinMatrix:
        """shard=(rank, world): only that share of the pair work, into a zeroed W; the
        world shards sum entrywise to the full W (reference: the per-worker partial
        matrices of inc/assemble.hpp:91-133, here one per process / GPU)."""
        st = AssemblyStatsC()
        hw = vp(W.h.value if W is not None else None)
        rank, world = shard if shard is not None else (0, 1)
        _check(lib().sbg_assembly_run_shard(self.h, C.byref(hw), int(rank), int(world), C.byref(st)))
        stats = {n: getattr(st, n) for n, _ in AssemblyStatsC._fields_}
        if W is None:
            W = GalerkinMatrix(hw, self.ctx, stats)
        else:
            W.stats = stats
        return W


def pair_integrals(m: SurfaceMesh, f, g, cfg: QuadratureConfig = None, ctx: Context = None):
    """pair_integral(m, f, g, eng) on the device (reference: inc/quadrature.hpp:268-334)."""
    ctx = ctx or default_context()
    cfg = cfg or QuadratureConfig()
    f = np.ascontiguousarray(f, dtype=np.int32)
    g = np.ascontiguousarray(g, dtype=np.int32)
    out = np.zeros(len(f))
    c = cfg.c()
    _check(lib().sbg_pair_integrals(ctx.h, m.h, C.byref(c), f, g, len(f), out))
    return out


def rhs_points(im: InflatedMesh, cfg: QuadratureConfig = None):
    cfg = cfg or QuadratureConfig()
    pts = np.zeros(im.base.nf * cfg.far_order ** 2 * 3)
    c = cfg.c()
    _check(lib().sbg_rhs_points(im.h, C.byref(c), pts))
    return pts.reshape(-1, 3)


def assemble_rhs(im: InflatedMesh, g, cfg: QuadratureConfig = None, ctx: Context = None):
    """reference: inc/assemble.hpp:143-184; g is a callable of a point or a constant 3-vector."""
    ctx = ctx or default_context()
    cfg = cfg or QuadratureConfig()
    c = cfg.c()
    if callable(g):
        gv = np.ascontiguousarray(np.array([g(p) for p in rhs_points(im, cfg)], dtype=np.float64).reshape(-1))
        field_flag = 1
    else:
        gv = np.ascontiguousarray(np.asarray(g, dtype=np.float64).reshape(3))
        field_flag = 0
    L = np.zeros(im.n)
    _check(lib().sbg_assemble_rhs(ctx.h, im.h, C.byref(c), gv, field_flag, L))
    return L


# --------------------------------------------------------------------------- potential (3-D)
@dataclass
class EvaluationGrid:
    """reference: inc/potential.hpp:11-13 — off-screen evaluation points (n x 3)"""
    points: np.ndarray

    def __post_init__(self):
        self.points = np.ascontiguousarray(np.asarray(self.points, dtype=np.float64).reshape(-1, 3))

    def __len__(self):
        return len(self.points)


def make_cartesian_grid(mesh: SurfaceMesh, lo: float, hi: float, nx: int, ny: int, mask_eps: float,
                        ctx: Context = None) -> EvaluationGrid:
    """reference: inc/potential.hpp:15-25 — cell centres of [lo, hi]^2 in the z = 0 plane (x-major),
    points within mask_eps of the mesh dropped (the distances on the device)"""
    ctx = ctx or default_context()
    out = np.zeros(3 * max(nx * ny, 1))
    cnt = C.c_int()
    _check(lib().sbg_make_cartesian_grid(ctx.h, mesh.h, lo, hi, nx, ny, mask_eps, out.ctypes.data, C.byref(cnt)))
    return EvaluationGrid(out[:3 * cnt.value].reshape(-1, 3))


def eval_DL(v, im: InflatedMesh, grid, cfg: QuadratureConfig = None, ctx: Context = None) -> np.ndarray:
    """reference: inc/potential.hpp:104-138 (3-D) — the double-layer potential of jump vector v at
    the grid's points; ValidationError for a point on the screen.  cfg.exact_far: bitwise the
    CPU restatement (every facet in the reference's operation order)."""
    ctx = ctx or default_context()
    cfg = cfg or QuadratureConfig()
    vv = np.ascontiguousarray(np.asarray(v, dtype=np.float64).reshape(-1))
    if len(vv) != im.n:
        raise ValidationError("jump vector length does not match the DOF count")
    pts = grid.points if isinstance(grid, EvaluationGrid) else EvaluationGrid(grid).points
    out = np.zeros(len(pts))
    c = cfg.c()
    _check(lib().sbg_eval_dl(ctx.h, im.h, vv.ctypes.data, pts.ctypes.data, len(pts), C.byref(c), out.ctypes.data))
    return out


def grid_error(computed, exact) -> float:
    """reference: inc/potential.hpp:188-195 — discrete l2 distance of two grid samplings"""
    a, b = np.asarray(computed, dtype=np.float64), np.asarray(exact, dtype=np.float64)
    if a.shape != b.shape:
        raise ValidationError("grid error: length mismatch")
    return 0.0 if a.size == 0 else float(np.sqrt(np.mean((a - b) ** 2)))


# --------------------------------------------------------------------------- partition / prolongation
class DofPartition(_Handle):
    """reference: inc/schwarz.hpp:14-17"""
    _destroy = "sbg_partition_destroy"

    def __init__(self, h):
        super().__init__(h)
        nf, nd, nw = C.c_int(), C.c_int(), C.c_int()
        _check(lib().sbg_partition_sizes(h, C.byref(nf), C.byref(nd), C.byref(nw)))
        self.face_ids = np.zeros(nf.value, dtype=np.int32)
        self.face_ptr = np.zeros(nf.value + 1, dtype=np.int32)
        self.face_dofs = np.zeros(nd.value, dtype=np.int32)
        self.wirebasket = np.zeros(nw.value, dtype=np.int32)
        _check(lib().sbg_partition_export(h, self.face_ids, self.face_ptr, self.face_dofs, self.wirebasket))

    @property
    def face_sets(self):
        return {int(f): self.face_dofs[self.face_ptr[i]:self.face_ptr[i + 1]].copy()
                for i, f in enumerate(self.face_ids)}

    @classmethod
    def create(cls, face_sets: dict, wirebasket):
        ids = np.array(sorted(face_sets), dtype=np.int32)
        ptr = np.zeros(len(ids) + 1, dtype=np.int32)
        dofs = []
        for i, f in enumerate(ids):
            dofs.extend(face_sets[int(f)])
            ptr[i + 1] = len(dofs)
        wb = np.ascontiguousarray(wirebasket, dtype=np.int32)
        h = vp()
        _check(lib().sbg_partition_create(len(ids), ids, ptr, np.array(dofs + [0], dtype=np.int32), len(wb),
                                          wb if len(wb) else np.zeros(1, dtype=np.int32), C.byref(h)))
        return cls(h)


def partition_dofs(pair: MeshLevelPair, fine: InflatedMesh) -> DofPartition:
    """reference: inc/schwarz.hpp:19-51"""
    h = vp()
    _check(lib().sbg_partition_dofs(pair.h, fine.h, C.byref(h)))
    return DofPartition(h)


class Prolongation(_Handle):
    """reference: inc/jump.hpp:87-89 (CSC, ascending rows per column)"""
    _destroy = "sbg_prolong_destroy"

    def __init__(self, h):
        super().__init__(h)
        r, c, z = C.c_int(), C.c_int(), C.c_int()
        _check(lib().sbg_prolong_sizes(h, C.byref(r), C.byref(c), C.byref(z)))
        self.rows, self.cols = r.value, c.value
        self.col_ptr = np.zeros(c.value + 1, dtype=np.int32)
        self.row_idx = np.zeros(max(z.value, 1), dtype=np.int32)
        self.val = np.zeros(max(z.value, 1))
        _check(lib().sbg_prolong_export(h, self.col_ptr, self.row_idx, self.val))
        self.row_idx, self.val = self.row_idx[:z.value], self.val[:z.value]

    @classmethod
    def create(cls, rows, cols, col_ptr, row_idx, val):
        h = vp()
        _check(lib().sbg_prolong_create(rows, cols, np.ascontiguousarray(col_ptr, dtype=np.int32),
                                        np.ascontiguousarray(list(row_idx) + [0], dtype=np.int32),
                                        np.ascontiguousarray(list(val) + [0.0], dtype=np.float64), C.byref(h)))
        return cls(h)

    @classmethod
    def empty(cls, rows):
        return cls.create(rows, 0, [0], [], [])

    def dense(self):
        R = np.zeros((self.rows, self.cols))
        for c in range(self.cols):
            for p in range(self.col_ptr[c], self.col_ptr[c + 1]):
                R[self.row_idx[p], c] = self.val[p]
        return R


def build_prolongation(pair: MeshLevelPair, coarse: InflatedMesh, fine: InflatedMesh) -> Prolongation:
    """reference: inc/jump.hpp:118-185"""
    h = vp()
    _check(lib().sbg_build_prolongation(pair.h, coarse.h, fine.h, C.byref(h)))
    return Prolongation(h)


# --------------------------------------------------------------------------- Schwarz / PCG
class SchwarzPreconditioner(_Handle):
    """reference: inc/schwarz.hpp:55-73 (factors resident in HBM)"""
    _destroy = "sbg_prec_destroy"

    def __init__(self, h, ctx: Context, n: int):
        super().__init__(h)
        self.ctx, self.n = ctx, n

    def num_subspaces(self):
        return lib().sbg_prec_num_subspaces(self.h)

    def apply(self, r):
        r = np.ascontiguousarray(r, dtype=np.float64)
        z = np.zeros(len(r))
        _check(lib().sbg_apply_preconditioner(self.ctx.h, self.h, r, len(r), z))
        return z

    def block_diag(self, which: int):
        n = C.c_int()
        _check(lib().sbg_prec_block_diag(self.ctx.h, self.h, which, None, C.byref(n)))
        d = np.zeros(n.value)
        _check(lib().sbg_prec_block_diag(self.ctx.h, self.h, which, d.ctypes.data_as(C.c_void_p), C.byref(n)))
        return d

    def factor_bytes(self):
        return lib().sbg_prec_factor_bytes(self.h)


def build_preconditioner(W: GalerkinMatrix, part: DofPartition, P: Prolongation,
                         mode: str = "inverse") -> SchwarzPreconditioner:
    """reference: inc/schwarz.hpp:100-118.  mode "inverse" (default) forms the block
    inverses L^-T L^-1 once and applies one batched GEMV (for a largest block above 2048
    DOFs it keeps X = L^-1 and applies X^T (X r), two triangular GEMVs over the same bytes);
    "factored" forces that form; "trsv" applies the blocked triangular solves with L as
    llt.solve does (schwarz.hpp:130)."""
    modes = {"trsv": 0, "inverse": 1, "factored": 2}
    if mode not in modes:
        raise ValidationError(f"unknown preconditioner mode {mode!r}")
    h = vp()
    _check(lib().sbg_build_preconditioner_mode(W.ctx.h, W.h, part.h, P.h if P is not None else None, modes[mode],
                                               C.byref(h)))
    return SchwarzPreconditioner(h, W.ctx, W.n)


def apply_preconditioner(prec: SchwarzPreconditioner, r):
    """reference: inc/schwarz.hpp:121-140"""
    return prec.apply(r)


def materialize_preconditioner(prec: SchwarzPreconditioner, device: bool = False):
    """reference: inc/schwarz.hpp:142-148.  M (columns apply(e_j)) is built on the
    device from the block inverses and the coarse term; device=True keeps it in HBM
    (a GalerkinMatrix handle), else a host (n, n) array."""
    h = vp()
    _check(lib().sbg_materialize_preconditioner(prec.ctx.h, prec.h, C.byref(h)))
    M = GalerkinMatrix(h, prec.ctx)
    return M if device else M.download()


class _Spectrum(C.Structure):
    _fields_ = [("lambda_min", C.c_double), ("lambda_max", C.c_double), ("kappa", C.c_double),
                ("iterations", C.c_int), ("converged", C.c_int)]


@dataclass
class SpectrumResult:
    """reference: inc/schwarz.hpp:150-154 (+ the Lanczos step count)"""
    lambda_min: float
    lambda_max: float
    kappa: float
    iterations: int = 0
    converged: bool = True


def condition_number(W: GalerkinMatrix, M=None, tol: float = 1e-10, maxit: int = 0) -> SpectrumResult:
    """reference: inc/schwarz.hpp:166-190.  condition_number(W) when M is None;
    condition_number(W, prec) for a SchwarzPreconditioner; condition_number(W, M) for a
    materialized M (host array or device GalerkinMatrix).  Extreme eigenvalues by
    Lanczos on the device (W inner product, full reorthogonalisation, stopped when both
    extreme Ritz residuals are <= tol |theta|) instead of the dense eigensolve."""
    keep = None
    if M is None:
        ph = None
    elif isinstance(M, SchwarzPreconditioner):
        ph = M.h
    else:
        Md = M if isinstance(M, GalerkinMatrix) else GalerkinMatrix.from_host(M, W.ctx)
        if Md.n != W.n:
            raise ValidationError("condition_number: preconditioner size mismatch")
        h = vp()
        _check(lib().sbg_prec_from_dense(W.ctx.h, Md.h, C.byref(h)))
        keep = SchwarzPreconditioner(h, W.ctx, W.n)
        ph = keep.h
    out = _Spectrum()
    _check(lib().sbg_condition_number(W.ctx.h, W.h, ph, tol, maxit, C.byref(out)))
    return SpectrumResult(out.lambda_min, out.lambda_max, out.kappa, out.iterations, bool(out.converged))


def coarse_matrix(W: GalerkinMatrix, P: Prolongation):
    H = np.zeros(P.cols * P.cols)
    _check(lib().sbg_coarse_matrix(W.ctx.h, W.h, P.h, H))
    return H.reshape(P.cols, P.cols)


@dataclass
class PcgReport:
    """reference: inc/pcg.hpp:9-16"""
    solution: np.ndarray
    iterations: int
    converged: bool
    residual_history: np.ndarray
    kappa_estimate: float
    alphas: np.ndarray = field(default_factory=lambda: np.zeros(0))
    betas: np.ndarray = field(default_factory=lambda: np.zeros(0))
    energy_error_history: np.ndarray = field(default_factory=lambda: np.zeros(0))


def pcg(W: GalerkinMatrix, prec, rhs, tol: float = 1e-8, maxit: int = 0, exact=None) -> PcgReport:
    """reference: inc/pcg.hpp:33-116.  `exact` (optional) fills energy_error_history with
    sqrt(e^T W e), e = x_k - exact, for k = 0..iterations (pcg.hpp:50-53, 59, 82)."""
    rhs = np.ascontiguousarray(rhs, dtype=np.float64)
    n = len(rhs)
    cap = (maxit if maxit > 0 else max(10 * n, 100)) + 2
    x = np.zeros(max(n, 1))
    hist, al, be = np.zeros(cap), np.zeros(cap), np.zeros(cap)
    rep = PcgReportC()
    energy = np.zeros(0)
    if exact is None:
        _check(lib().sbg_pcg(W.ctx.h, W.h, prec.h if prec is not None else None,
                             rhs if n else np.zeros(1), n, tol, maxit, x, hist, al, be, cap, C.byref(rep)))
    else:
        ex = np.ascontiguousarray(exact, dtype=np.float64)
        if len(ex) != n:
            raise ValidationError("pcg: exact solution length mismatch")
        en = np.zeros(cap)
        _check(lib().sbg_pcg_exact(W.ctx.h, W.h, prec.h if prec is not None else None,
                                   rhs if n else np.zeros(1), n, tol, maxit, ex if n else np.zeros(1), x, hist, en,
                                   al, be, cap, C.byref(rep)))
        energy = en[:rep.history_len].copy()
    k = rep.iterations
    return PcgReport(x[:n], k, bool(rep.converged), hist[:rep.history_len].copy(), rep.kappa_estimate,
                     al[:k].copy(), be[:k].copy(), energy)


# --------------------------------------------------------------------------- row-panel PCG
# exchange hook of sbg_pcg_rows: (user, d_p, d_y, n, stream) -> 0 | error
EXCHANGE_FN = C.CFUNCTYPE(C.c_int, vp, vp, vp, C.c_int, vp)
# agreement hook of sbg_pcg_rows_agree: (user, local_stop, *global_stop) -> 0 | error
AGREE_FN = C.CFUNCTYPE(C.c_int, vp, C.c_int, C.POINTER(C.c_int))


def row_ranges(n: int, world: int):
    """Row panels of the multi-GPU PCG: rank r owns rows
    [r*k, min(n, (r+1)*k)) with k = ceil(n / world) — equal panels, so the all-gather
    of W p moves k doubles per rank (the last panel is padded)."""
    if world < 1:
        raise ValidationError("world size must be positive")
    k = -(-n // world) if n else 0
    return [(min(n, r * k), min(n, (r + 1) * k)) for r in range(world)]


class DeviceVector:
    """A float64 device vector given by address and length (`__cuda_array_interface__`),
    so torch / NCCL can read and write PCG buffers in place."""

    def __init__(self, ptr: int, n: int):
        self.ptr, self.n = int(ptr or 0), int(n)

    @property
    def __cuda_array_interface__(self):
        return {"shape": (self.n,), "typestr": "<f8", "data": (self.ptr, False), "version": 3, "strides": None,
                "stream": None}


def allgather_exchange(dist, rank: int, world: int, n: int, device=None, wrap=None, host_staging=False):
    """The exchange of the row-panel PCG over torch.distributed: every rank contributes its
    panel of y = W p (row_ranges) and receives the others', in place in y.  On the GPU the
    collective is enqueued on the PCG's own stream (torch's current stream is switched to
    it), so no host synchronisation happens per iteration; NCCL moves the panels over
    NVLink.  `wrap(ptr, n)` maps a buffer address to a tensor (default: the device vector
    through __cuda_array_interface__; tests pass a host-memory wrapper to run it on gloo).
    host_staging: gather through host memory (gloo functional runs, ranks sharing a GPU).
    Returns f(d_p, d_y, n, stream) for pcg_rows."""
    import torch
    ranges = row_ranges(n, world)
    k = ranges[0][1] - ranges[0][0] if n else 0
    if wrap is None:
        def wrap(ptr, m):
            return torch.as_tensor(DeviceVector(ptr, m), device=device)
    state = {}

    def exchange(d_p, d_y, m, stream):
        if m != n:
            raise ValidationError("row exchange: length mismatch")
        y = wrap(d_y, n)
        lo, hi = ranges[rank]
        ctxm = torch.cuda.stream(torch.cuda.ExternalStream(stream, device=y.device)) if y.is_cuda else _nullctx()
        with ctxm:
            if "mine" not in state:  # staging allocated once, on the PCG stream
                sd = "cpu" if host_staging else y.device
                state["mine"] = torch.zeros(k, dtype=torch.float64, device=sd)
                state["all"] = [torch.zeros(k, dtype=torch.float64, device=sd) for _ in range(world)]
            mine, parts = state["mine"], state["all"]
            mine[:hi - lo].copy_(y[lo:hi])
            dist.all_gather(parts, mine)
            for r, (a, b) in enumerate(ranges):
                if r != rank and b > a:
                    y[a:b].copy_(parts[r][:b - a])
        return 0
    return exchange


def allreduce_agree(dist, device=None):
    """The collective stop of the row-panel PCG: every rank passes its local stop flag
    (converged or out of iterations) at each batch boundary and all ranks get the minimum,
    so they stop together and enqueue the same all-gathers (include/screenbem_b200.h,
    sbg_pcg_rows_agree).  `device` is where the flag is reduced (the NCCL device; None =
    host, gloo).  Returns f(local_stop) -> global_stop for pcg_rows."""
    import torch

    def agree(local_stop: int) -> int:
        t = torch.tensor([int(local_stop)], dtype=torch.int32, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return int(t.item())
    return agree


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def pcg_rows(W: GalerkinMatrix, prec, rhs, rows, exchange, tol: float = 1e-8, maxit: int = 0,
             agree=None) -> PcgReport:
    """Row-panel PCG (sbg_pcg_rows / sbg_pcg_rows_agree): the reference's pcg
    (inc/pcg.hpp:33-116) with this rank computing rows `rows = (lo, hi)` of each matvec
    and `exchange(d_p, d_y, n, stream)` filling in the rest (allgather_exchange for one
    GPU per rank).  `agree(local_stop) -> global_stop` (allreduce_agree) makes the stop
    decision collective; without it every rank must hold bitwise-identical W and rhs.
    The result equals pcg's (same kernels per row, same replicated reductions)."""
    rhs = np.ascontiguousarray(rhs, dtype=np.float64)
    n = len(rhs)
    cap = (maxit if maxit > 0 else max(10 * n, 100)) + 2
    x = np.zeros(max(n, 1))
    hist, al, be = np.zeros(cap), np.zeros(cap), np.zeros(cap)
    rep = PcgReportC()
    err = []

    def hook(user, d_p, d_y, m, stream):
        try:
            exchange(d_p, d_y, m, stream)
            return 0
        except BaseException as e:  # surfaced after the C call returns
            err.append(e)
            return 1
    def ahook(user, local_stop, out):
        try:
            out[0] = int(agree(int(local_stop)))
            return 0
        except BaseException as e:
            err.append(e)
            return 1
    cb = EXCHANGE_FN(hook)
    ab = AGREE_FN(ahook) if agree is not None else None
    rb = (rhs if n else np.zeros(1))
    code = lib().sbg_pcg_rows_agree(W.ctx.h, W.h, prec.h if prec is not None else None, rb.ctypes.data, n, 0, tol,
                                    maxit, int(rows[0]), int(rows[1]), C.cast(cb, vp),
                                    C.cast(ab, vp) if ab is not None else None, None, x.ctypes.data, hist, al, be,
                                    cap, C.byref(rep))
    if err:
        raise err[0]
    _check(code)
    k = rep.iterations
    return PcgReport(x[:n], k, bool(rep.converged), hist[:rep.history_len].copy(), rep.kappa_estimate,
                     al[:k].copy(), be[:k].copy())


def matvec_rows_device(W: GalerkinMatrix, d_x: int, d_y: int, lo: int, hi: int) -> None:
    """d_y[lo:hi] = W[lo:hi, :] d_x on device buffers, enqueued on the context stream."""
    _check(lib().sbg_matvec_rows_device(W.ctx.h, W.h, d_x, d_y, lo, hi))


# --------------------------------------------------------------------------- pipeline
@dataclass
class SolveResult:
    """cmd_solve outputs (reference: inc/experiments.hpp:111-196) without the file IO."""
    dofs: int
    report: PcgReport
    W: GalerkinMatrix
    rhs: np.ndarray
    prec: "SchwarzPreconditioner" = None


def solve(pair: MeshLevelPair, g, tol: float = 1e-8, cfg: QuadratureConfig = None, precondition: bool = True,
          ctx: Context = None) -> SolveResult:
    """The cmd_solve hot path (experiments.hpp:130-145): inflate -> assemble_W ->
    assemble_rhs -> partition/prolongation -> build_preconditioner -> pcg.  The coarse
    level's host setup (inflate, partition_dofs, build_prolongation) runs on a host thread
    while this thread drives the device assembly (the C calls release the GIL), so it is
    off the critical path; results are identical to the sequential order."""
    ctx = ctx or default_context()
    fine = inflate(pair.fine)
    setup, err = {}, []

    def coarse_setup():
        try:
            coarse = inflate(pair.coarse)
            setup["P"] = build_prolongation(pair, coarse, fine)
            setup["part"] = partition_dofs(pair, fine)
        except BaseException as e:  # re-raised on the calling thread
            err.append(e)
    th = None
    if precondition:
        import threading
        th = threading.Thread(target=coarse_setup, daemon=True)
        th.start()
    try:
        W = assemble_W(fine, cfg, ctx=ctx)
        L = assemble_rhs(fine, g, cfg, ctx=ctx)
    finally:
        if th is not None:
            th.join()
    if err:
        raise err[0]
    prec = build_preconditioner(W, setup["part"], setup["P"]) if precondition else None
    rep = pcg(W, prec, L, tol)
    if not rep.converged:
        raise NumericalError("solver did not converge")
    return SolveResult(fine.n, rep, W, L, prec)
