// screenbem/gpu.hpp — C++ drop-in for the hot path of the screenbem reference
// (proj/include/screenbem), backed by libscreenbem_b200.so (include/screenbem_b200.h).
//
// Names and error behaviour follow the reference: ValidationError (CLI exit 2)
// and NumericalError (CLI exit 3) are thrown exactly where the reference throws
// them (inc/common.hpp:16-26).  A caller of the reference replaces
//
//     #include "screenbem/experiments.hpp"          // Eigen-based, CPU
//     GalerkinMatrix W = assemble_W(im, quad, threads);
//     SchwarzPreconditioner P = build_preconditioner(W, part, R);
//     PcgReport rep = pcg(W, &P, L, tol);
//
// with
//
//     #include "screenbem/gpu.hpp"
//     namespace sb = screenbem::gpu;
//     sb::Context ctx;                                 // one B200, one stream
//     sb::InflatedMesh im = sb::inflate(mesh);
//     sb::GalerkinMatrix W = sb::assemble_W(ctx, im);  // device-resident, .download() for dumps
//     sb::SchwarzPreconditioner P = sb::build_preconditioner(ctx, W, sb::partition_dofs(pair, im),
//                                                            sb::build_prolongation(pair, coarse, im));
//     sb::PcgReport rep = sb::pcg(ctx, W, &P, L, tol);
//
// Host arrays are std::vector<double> (row-major for matrices) instead of Eigen types.
#pragma once

#include <cmath>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../screenbem_b200.h"

namespace screenbem {

class ValidationError : public std::runtime_error {  // reference: inc/common.hpp:17-20
public:
    explicit ValidationError(const std::string& m) : std::runtime_error(m) {}
};
class NumericalError : public std::runtime_error {  // reference: inc/common.hpp:23-26
public:
    explicit NumericalError(const std::string& m) : std::runtime_error(m) {}
};
class CudaError : public std::runtime_error {
public:
    explicit CudaError(const std::string& m) : std::runtime_error(m) {}
};

namespace gpu {

inline void check(int rc)
{
    if (rc == SBG_OK) return;
    const std::string msg = sbg_last_error();
    if (rc == SBG_EVALIDATION) throw ValidationError(msg);
    if (rc == SBG_ENUMERICAL) throw NumericalError(msg);
    if (rc == SBG_ECUDA) throw CudaError(msg);
    throw std::runtime_error(msg);
}

template <class T, void (*Destroy)(T*)>
class Handle {
public:
    Handle() = default;
    explicit Handle(T* p) : p_(p) {}
    Handle(const Handle&) = delete;
    Handle& operator=(const Handle&) = delete;
    Handle(Handle&& o) noexcept : p_(std::exchange(o.p_, nullptr)) {}
    Handle& operator=(Handle&& o) noexcept
    {
        if (this != &o) {
            reset();
            p_ = std::exchange(o.p_, nullptr);
        }
        return *this;
    }
    ~Handle() { reset(); }
    T* get() const { return p_; }
    void reset()
    {
        if (p_) Destroy(p_);
        p_ = nullptr;
    }

private:
    T* p_ = nullptr;
};

// reference: inc/common.hpp:14 (Vec3 = Eigen::Vector3d) — the accessors and arithmetic a
// Neumann-data callback uses, without Eigen
struct Vec3 {
    double v[3] = {0.0, 0.0, 0.0};
    Vec3() = default;
    Vec3(double a, double b, double c) : v{a, b, c} {}
    double& operator[](int i) { return v[i]; }
    double operator[](int i) const { return v[i]; }
    double& operator()(int i) { return v[i]; }
    double operator()(int i) const { return v[i]; }
    double x() const { return v[0]; }
    double y() const { return v[1]; }
    double z() const { return v[2]; }
    double dot(const Vec3& o) const { return (v[0] * o.v[0] + v[1] * o.v[1]) + v[2] * o.v[2]; }
    double squaredNorm() const { return dot(*this); }
    double norm() const { return std::sqrt(squaredNorm()); }
    Vec3 cross(const Vec3& o) const
    {
        return {v[1] * o.v[2] - v[2] * o.v[1], v[2] * o.v[0] - v[0] * o.v[2], v[0] * o.v[1] - v[1] * o.v[0]};
    }
    Vec3 operator+(const Vec3& o) const { return {v[0] + o.v[0], v[1] + o.v[1], v[2] + o.v[2]}; }
    Vec3 operator-(const Vec3& o) const { return {v[0] - o.v[0], v[1] - o.v[1], v[2] - o.v[2]}; }
    Vec3 operator-() const { return {-v[0], -v[1], -v[2]}; }
    Vec3 operator*(double s) const { return {v[0] * s, v[1] * s, v[2] * s}; }
    Vec3 operator/(double s) const { return {v[0] / s, v[1] / s, v[2] / s}; }
};
inline Vec3 operator*(double s, const Vec3& a) { return a * s; }

struct QuadratureConfig {  // reference: inc/quadrature.hpp:12-16
    int far_order = 4;
    int singular_order = 8;
    double near_threshold = 2.0;
    bool exact_far = false;  // depth-0 far pairs bitwise like the CPU restatement (slower)
    sbg_quad_cfg c() const { return {far_order, singular_order, near_threshold, exact_far ? 1 : 0}; }
};

class Context : public Handle<sbg_ctx, sbg_ctx_destroy> {
public:
    explicit Context(int device = 0)
    {
        sbg_ctx* p = nullptr;
        check(sbg_ctx_create(device, &p));
        *this = Context(p);
    }
    void synchronize() { check(sbg_ctx_synchronize(get())); }
    // 0 symmetric (default), 1 full matrix (see sbg_ctx_set_matvec_form)
    void set_matvec_form(int form) { check(sbg_ctx_set_matvec_form(get(), form)); }

private:
    explicit Context(sbg_ctx* p) : Handle(p) {}
};

// reference: inc/mesh.hpp:19-83 (3-D triangles), vertices xyz-interleaved
class SurfaceMesh : public Handle<sbg_mesh, sbg_mesh_destroy> {
public:
    SurfaceMesh() = default;
    SurfaceMesh(const std::vector<double>& verts, const std::vector<int32_t>& facets)
    {
        sbg_mesh* p = nullptr;
        check(sbg_mesh_create((int)(verts.size() / 3), verts.data(), (int)(facets.size() / 3), facets.data(), &p));
        *this = SurfaceMesh(p);
    }
    explicit SurfaceMesh(sbg_mesh* p) : Handle(p) {}
};

inline SurfaceMesh make_builtin(const std::string& spec)  // inc/mesh.hpp:516-537
{
    sbg_mesh* p = nullptr;
    check(sbg_make_builtin(spec.c_str(), &p));
    return SurfaceMesh(p);
}
inline void validate_mesh(const SurfaceMesh& m) { check(sbg_validate_mesh(m.get())); }  // inc/mesh.hpp:238-272

class MeshLevelPair : public Handle<sbg_level, sbg_level_destroy> {  // inc/mesh.hpp:86-92
public:
    explicit MeshLevelPair(sbg_level* p) : Handle(p) {}
    SurfaceMesh coarse() const { return mesh(0); }
    SurfaceMesh fine() const { return mesh(1); }

private:
    SurfaceMesh mesh(int which) const
    {
        sbg_mesh* p = nullptr;
        check(sbg_level_mesh(get(), which, &p));
        return SurfaceMesh(p);
    }
};
inline MeshLevelPair refine_uniform_times(const SurfaceMesh& m, int k)  // inc/mesh.hpp:388-405
{
    sbg_level* p = nullptr;
    check(sbg_refine_uniform_times(m.get(), k, &p));
    return MeshLevelPair(p);
}
inline MeshLevelPair make_config(int cfg, int ratio = 0)
{
    sbg_level* p = nullptr;
    check(sbg_make_config(cfg, ratio, &p));
    return MeshLevelPair(p);
}

class InflatedMesh : public Handle<sbg_inflated, sbg_inflated_destroy> {  // inc/inflate.hpp:48-76
public:
    explicit InflatedMesh(sbg_inflated* p) : Handle(p) {}
    int num_jump_dofs() const
    {
        int n, ng, nv, nf;
        check(sbg_inflated_sizes(get(), &n, &ng, &nv, &nf));
        return n;
    }
};
inline InflatedMesh inflate(const SurfaceMesh& m)  // inc/inflate.hpp:98-288
{
    sbg_inflated* p = nullptr;
    check(sbg_inflate(m.get(), 1, &p));
    return InflatedMesh(p);
}

class GalerkinMatrix : public Handle<sbg_matrix, sbg_matrix_destroy> {  // inc/assemble.hpp:12
public:
    explicit GalerkinMatrix(sbg_matrix* p) : Handle(p) {}
    int rows() const { return sbg_matrix_n(get()); }
    std::vector<double> download() const  // row-major n x n
    {
        std::vector<double> h((size_t)rows() * rows());
        check(sbg_matrix_download(get(), h.data()));
        return h;
    }
};
// reference: inc/assemble.hpp:72-139 (`workers` is accepted and ignored on the GPU)
inline GalerkinMatrix assemble_W(Context& ctx, const InflatedMesh& im, const QuadratureConfig& cfg = {},
                                 int workers = 1)
{
    const sbg_quad_cfg c = cfg.c();
    sbg_matrix* p = nullptr;
    check(sbg_assemble_w(ctx.get(), im.get(), &c, workers, &p, nullptr));
    return GalerkinMatrix(p);
}
// one process's partial W of a multi-GPU assembly (the reference's per-worker partial
// matrices, inc/assemble.hpp:91-133): the `world` shards sum entrywise to assemble_W's W;
// reduce them in place over sbg_matrix_device_view (e.g. ncclAllReduce)
inline GalerkinMatrix assemble_W_shard(Context& ctx, const InflatedMesh& im, int rank, int world,
                                       const QuadratureConfig& cfg = {})
{
    const sbg_quad_cfg c = cfg.c();
    sbg_aplan* plan = nullptr;
    check(sbg_assembly_plan_create(ctx.get(), im.get(), &c, &plan));
    sbg_matrix* p = nullptr;
    const int rc = sbg_assembly_run_shard(plan, &p, rank, world, nullptr);
    sbg_assembly_plan_destroy(plan);
    check(rc);
    return GalerkinMatrix(p);
}
// reference: inc/assemble.hpp:143-184 with a constant field g
inline std::vector<double> assemble_rhs(Context& ctx, const InflatedMesh& im, const double g[3],
                                        const QuadratureConfig& cfg = {})
{
    const sbg_quad_cfg c = cfg.c();
    std::vector<double> L(im.num_jump_dofs());
    check(sbg_assemble_rhs(ctx.get(), im.get(), &c, g, 0, L.data()));
    return L;
}
// reference: inc/assemble.hpp:143-184 with a Neumann field g(x): g is evaluated on the host at
// the far-rule points of every facet (sbg_rhs_points, the loop order of assemble.hpp:155-160)
// and the integration runs on the device
inline std::vector<double> assemble_rhs(Context& ctx, const InflatedMesh& im,
                                        const std::function<Vec3(const Vec3&)>& g, const QuadratureConfig& cfg = {})
{
    const sbg_quad_cfg c = cfg.c();
    int n, ng, nv, nf;
    check(sbg_inflated_sizes(im.get(), &n, &ng, &nv, &nf));
    const size_t npts = (size_t)nf * cfg.far_order * cfg.far_order;
    std::vector<double> pts(3 * npts), gv(3 * std::max<size_t>(npts, 1));
    check(sbg_rhs_points(im.get(), &c, pts.data()));
    for (size_t i = 0; i < npts; ++i) {
        const Vec3 v = g(Vec3(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]));
        for (int k = 0; k < 3; ++k) gv[3 * i + k] = v[k];
    }
    std::vector<double> L(n);
    check(sbg_assemble_rhs(ctx.get(), im.get(), &c, gv.data(), 1, L.data()));
    return L;
}
// reference: inc/assemble.hpp:191-226
inline void dump_matrix_binary(const GalerkinMatrix& W, const std::string& path)
{
    check(sbg_matrix_dump_binary(W.get(), path.c_str()));
}

// ---- double-layer potential (inc/potential.hpp, 3-D)
struct EvaluationGrid {  // reference: inc/potential.hpp:11-13
    std::vector<Vec3> points;
};
// reference: inc/potential.hpp:15-25 (the point distances on the device)
inline EvaluationGrid make_cartesian_grid(Context& ctx, const SurfaceMesh& mesh, double lo, double hi, int nx, int ny,
                                          double mask_eps)
{
    std::vector<double> out(3 * (size_t)std::max(nx * ny, 1));
    int count = 0;
    check(sbg_make_cartesian_grid(ctx.get(), mesh.get(), lo, hi, nx, ny, mask_eps, out.data(), &count));
    EvaluationGrid g;
    for (int i = 0; i < count; ++i) g.points.emplace_back(out[3 * i], out[3 * i + 1], out[3 * i + 2]);
    return g;
}
// reference: inc/potential.hpp:104-138 (the `workers` argument has no device counterpart)
inline std::vector<double> eval_DL(Context& ctx, const std::vector<double>& v, const InflatedMesh& im,
                                   const EvaluationGrid& grid, const QuadratureConfig& cfg = {})
{
    if ((int)v.size() != im.num_jump_dofs()) throw ValidationError("jump vector length does not match the DOF count");
    const sbg_quad_cfg c = cfg.c();
    std::vector<double> pts(3 * grid.points.size());
    for (size_t i = 0; i < grid.points.size(); ++i)
        for (int k = 0; k < 3; ++k) pts[3 * i + k] = grid.points[i][k];
    std::vector<double> out(grid.points.size());
    check(sbg_eval_dl(ctx.get(), im.get(), v.data(), pts.data(), (long long)grid.points.size(), &c, out.data()));
    return out;
}

class DofPartition : public Handle<sbg_partition, sbg_partition_destroy> {  // inc/schwarz.hpp:14-17
public:
    explicit DofPartition(sbg_partition* p) : Handle(p) {}
};
inline DofPartition partition_dofs(const MeshLevelPair& pair, const InflatedMesh& fine)  // schwarz.hpp:19-51
{
    sbg_partition* p = nullptr;
    check(sbg_partition_dofs(pair.get(), fine.get(), &p));
    return DofPartition(p);
}
class Prolongation : public Handle<sbg_prolong, sbg_prolong_destroy> {  // inc/jump.hpp:87-89
public:
    explicit Prolongation(sbg_prolong* p) : Handle(p) {}
};
inline Prolongation build_prolongation(const MeshLevelPair& pair, const InflatedMesh& coarse,
                                       const InflatedMesh& fine)  // inc/jump.hpp:118-185
{
    sbg_prolong* p = nullptr;
    check(sbg_build_prolongation(pair.get(), coarse.get(), fine.get(), &p));
    return Prolongation(p);
}

class SchwarzPreconditioner : public Handle<sbg_prec, sbg_prec_destroy> {  // inc/schwarz.hpp:55-73
public:
    explicit SchwarzPreconditioner(sbg_prec* p) : Handle(p) {}
    int num_subspaces() const { return sbg_prec_num_subspaces(get()); }
};
inline SchwarzPreconditioner build_preconditioner(Context& ctx, const GalerkinMatrix& W, const DofPartition& part,
                                                  const Prolongation& R)  // inc/schwarz.hpp:100-118
{
    sbg_prec* p = nullptr;
    check(sbg_build_preconditioner(ctx.get(), W.get(), part.get(), R.get(), &p));
    return SchwarzPreconditioner(p);
}
inline std::vector<double> apply_preconditioner(Context& ctx, const SchwarzPreconditioner& P,
                                                const std::vector<double>& r)  // inc/schwarz.hpp:121-140
{
    std::vector<double> z(r.size());
    check(sbg_apply_preconditioner(ctx.get(), P.get(), r.data(), (int)r.size(), z.data()));
    return z;
}

struct PcgReport {  // reference: inc/pcg.hpp:9-16
    std::vector<double> solution;
    int iterations = 0;
    bool converged = false;
    std::vector<double> residual_history;      // preconditioned residual norms
    std::vector<double> energy_error_history;  // filled when an exact solution is given
    double kappa_estimate = 1.0;
};
// reference: inc/pcg.hpp:33-116 (prec nullable; exact nullable: energy_error_history)
inline PcgReport pcg(Context& ctx, const GalerkinMatrix& W, const SchwarzPreconditioner* prec,
                     const std::vector<double>& rhs, double tol = 1e-8, int maxit = 0,
                     const std::vector<double>* exact = nullptr)
{
    const int n = (int)rhs.size();
    const int cap = (maxit > 0 ? maxit : std::max(10 * n, 100)) + 2;
    PcgReport rep;
    rep.solution.assign(n, 0.0);
    rep.residual_history.assign(cap, 0.0);
    sbg_pcg_report r{};
    if (exact) {
        if ((int)exact->size() != n) throw ValidationError("pcg: exact solution length mismatch");
        rep.energy_error_history.assign(cap, 0.0);
        check(sbg_pcg_exact(ctx.get(), W.get(), prec ? prec->get() : nullptr, rhs.data(), n, tol, maxit,
                            exact->data(), rep.solution.data(), rep.residual_history.data(),
                            rep.energy_error_history.data(), nullptr, nullptr, cap, &r));
        rep.energy_error_history.resize(r.history_len);
    } else {
        check(sbg_pcg(ctx.get(), W.get(), prec ? prec->get() : nullptr, rhs.data(), n, tol, maxit,
                      rep.solution.data(), rep.residual_history.data(), nullptr, nullptr, cap, &r));
    }
    rep.iterations = r.iterations;
    rep.converged = r.converged != 0;
    rep.kappa_estimate = r.kappa_estimate;
    rep.residual_history.resize(r.history_len);
    return rep;
}

// pcg with one GPU per worker: this process computes rows [lo, hi) of each
// W p; `exchange` enqueues the all-gather of the other rows on the given stream (e.g. NCCL
// over NVLink); `agree` (nullable) makes the stop decision collective (a MIN over ranks of
// the local stop flag, see sbg_pcg_rows_agree).  Same result as pcg on every rank.
inline PcgReport pcg_rows(Context& ctx, const GalerkinMatrix& W, const SchwarzPreconditioner* prec,
                          const std::vector<double>& rhs, int lo, int hi, sbg_exchange_fn exchange, void* user,
                          double tol = 1e-8, int maxit = 0, sbg_agree_fn agree = nullptr)
{
    const int n = (int)rhs.size();
    const int cap = (maxit > 0 ? maxit : std::max(10 * n, 100)) + 2;
    PcgReport rep;
    rep.solution.assign(n, 0.0);
    rep.residual_history.assign(cap, 0.0);
    sbg_pcg_report r{};
    check(sbg_pcg_rows_agree(ctx.get(), W.get(), prec ? prec->get() : nullptr, rhs.data(), n, 0, tol, maxit, lo, hi,
                             exchange, agree, user, rep.solution.data(), rep.residual_history.data(), nullptr, nullptr,
                             cap, &r));
    rep.iterations = r.iterations;
    rep.converged = r.converged != 0;
    rep.kappa_estimate = r.kappa_estimate;
    rep.residual_history.resize(r.history_len);
    return rep;
}

// reference: inc/schwarz.hpp:142-148 — M stays on the device (download() for a host copy)
inline GalerkinMatrix materialize_preconditioner(Context& ctx, const SchwarzPreconditioner& P)
{
    sbg_matrix* m = nullptr;
    check(sbg_materialize_preconditioner(ctx.get(), P.get(), &m));
    return GalerkinMatrix(m);
}

struct SpectrumResult {  // reference: inc/schwarz.hpp:150-154
    double lambda_min = 0;
    double lambda_max = 0;
    double kappa = 0;
};
inline SpectrumResult to_spectrum(const sbg_spectrum& s) { return {s.lambda_min, s.lambda_max, s.kappa}; }
// reference: inc/schwarz.hpp:168-172 (device Lanczos instead of the dense eigensolve)
inline SpectrumResult condition_number(Context& ctx, const GalerkinMatrix& W, double tol = 1e-10)
{
    sbg_spectrum s{};
    check(sbg_condition_number(ctx.get(), W.get(), nullptr, tol, 0, &s));
    return to_spectrum(s);
}
// reference: inc/schwarz.hpp:185-190
inline SpectrumResult condition_number(Context& ctx, const GalerkinMatrix& W, const SchwarzPreconditioner& P,
                                       double tol = 1e-10)
{
    sbg_spectrum s{};
    check(sbg_condition_number(ctx.get(), W.get(), P.get(), tol, 0, &s));
    return to_spectrum(s);
}
// reference: inc/schwarz.hpp:174-183 (M materialized, dense)
inline SpectrumResult condition_number(Context& ctx, const GalerkinMatrix& W, const GalerkinMatrix& M,
                                       double tol = 1e-10)
{
    sbg_prec* p = nullptr;
    check(sbg_prec_from_dense(ctx.get(), M.get(), &p));
    SchwarzPreconditioner P(p);
    return condition_number(ctx, W, P, tol);
}

}  // namespace gpu
}  // namespace screenbem
