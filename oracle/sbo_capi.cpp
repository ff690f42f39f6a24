// ORACLE C entry points (TEST INFRASTRUCTURE ONLY — see sbo.hpp header).
// Loaded by tests/ and the bench CPU-baseline leg through oracle/oracle.py.
// Return codes mirror the reference's exception classes: 0 ok, 2 ValidationError,
// 3 NumericalError (inc/common.hpp:16-26, proj/tools/screenbem.cpp:172-181).
#include <chrono>
#include <cstdio>
#include <random>

#include "sbo.hpp"

using namespace sbo;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& fn)
{
    try {
        fn();
        return 0;
    } catch (const ValidationError& e) {
        g_err = e.what();
        return 2;
    } catch (const NumericalError& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

QuadratureConfig qcfg(int far_order, int singular_order, double near)
{
    QuadratureConfig c;
    c.far_order = far_order;
    c.singular_order = singular_order;
    c.near_threshold = near;
    return c;
}

SurfaceMesh make_mesh(int nv, const double* v, int nf, const int* f)
{
    SurfaceMesh m;
    m.vertices.resize(nv);
    for (int i = 0; i < nv; ++i) m.vertices[i] = Vec3(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
    m.facets.resize(nf);
    for (int i = 0; i < nf; ++i) m.facets[i] = {f[3 * i], f[3 * i + 1], f[3 * i + 2]};
    return m;
}

struct Level {
    MeshLevelPair pair;
};

struct PartOut {
    DofPartition part;
};

}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

// ---- meshes
void* orc_mesh_new(int nv, const double* verts, int nf, const int* facets)
{
    return new SurfaceMesh(make_mesh(nv, verts, nf, facets));
}
void orc_mesh_free(void* m) { delete static_cast<SurfaceMesh*>(m); }
int orc_mesh_sizes(void* mh, int* nv, int* nf)
{
    auto* m = static_cast<SurfaceMesh*>(mh);
    *nv = m->num_vertices();
    *nf = m->num_facets();
    return 0;
}
int orc_mesh_export(void* mh, double* verts, int* facets)
{
    auto* m = static_cast<SurfaceMesh*>(mh);
    for (int i = 0; i < m->num_vertices(); ++i) {
        verts[3 * i] = m->vertices[i].x;
        verts[3 * i + 1] = m->vertices[i].y;
        verts[3 * i + 2] = m->vertices[i].z;
    }
    for (int i = 0; i < m->num_facets(); ++i)
        for (int k = 0; k < 3; ++k) facets[3 * i + k] = m->facets[i][k];
    return 0;
}
int orc_validate_mesh(void* mh)
{
    return guard([&] { validate_mesh(*static_cast<SurfaceMesh*>(mh)); });
}
void* orc_bowtie_base() { return new SurfaceMesh(make_bowtie_base()); }

// level pairs (coarse, fine, parent)
void* orc_level_new(void* coarse, void* fine, const int* parent)
{
    auto* L = new Level;
    L->pair.coarse = *static_cast<SurfaceMesh*>(coarse);
    L->pair.fine = *static_cast<SurfaceMesh*>(fine);
    L->pair.parent.assign(parent, parent + L->pair.fine.num_facets());
    L->pair.H = L->pair.coarse.max_facet_diameter();
    L->pair.h = L->pair.fine.max_facet_diameter();
    return L;
}
void* orc_refine_uniform_times(void* mh, int k)
{
    auto* L = new Level;
    L->pair = refine_uniform_times(*static_cast<SurfaceMesh*>(mh), k);
    return L;
}
void orc_level_free(void* l) { delete static_cast<Level*>(l); }
void* orc_level_fine(void* l) { return new SurfaceMesh(static_cast<Level*>(l)->pair.fine); }
void* orc_level_coarse(void* l) { return new SurfaceMesh(static_cast<Level*>(l)->pair.coarse); }
int orc_level_parent(void* l, int* parent)
{
    const auto& p = static_cast<Level*>(l)->pair.parent;
    std::copy(p.begin(), p.end(), parent);
    return 0;
}

// ---- rules
int orc_gauss_legendre(int n, double* x, double* w)
{
    const Rule1d r = gauss_legendre(n);
    std::copy(r.x.begin(), r.x.end(), x);
    std::copy(r.w.begin(), r.w.end(), w);
    return 0;
}
int orc_triangle_rule(int order, double* u, double* v, double* w)
{
    const TriangleRule r = triangle_rule(order);
    std::copy(r.u.begin(), r.u.end(), u);
    std::copy(r.v.begin(), r.v.end(), v);
    std::copy(r.w.begin(), r.w.end(), w);
    return 0;
}
// cls 3 identical, 2 edge, 1 vertex; out has 5*npoints doubles (a1,a2,b1,b2,w)
long long orc_sauter_rule(int order, int cls, double* out)
{
    const SauterRules s(order);
    const auto& r = cls == 3 ? s.identical : (cls == 2 ? s.edge : s.vertex);
    if (out)
        for (size_t i = 0; i < r.size(); ++i) {
            out[5 * i] = r[i].a1;
            out[5 * i + 1] = r[i].a2;
            out[5 * i + 2] = r[i].b1;
            out[5 * i + 3] = r[i].b2;
            out[5 * i + 4] = r[i].w;
        }
    return (long long)r.size();
}

// ---- pair integrals (production rules and the adaptive quad_oracle)
int orc_pair_integrals(void* mh, const int* f, const int* g, long long npairs, int far_order,
                       int singular_order, double near, int workers, double* out, long long* stats3)
{
    return guard([&] {
        const SurfaceMesh& m = *static_cast<SurfaceMesh*>(mh);
        const QuadratureEngine eng(qcfg(far_order, singular_order, near));
        std::vector<detail::QuadStats> st(std::max(workers, 1));
        run_partitioned(npairs, workers, [&](int w, std::int64_t lo, std::int64_t hi) {
            for (std::int64_t i = lo; i < hi; ++i) out[i] = pair_integral(m, f[i], g[i], eng, &st[w]);
        });
        if (stats3) {
            stats3[0] = stats3[1] = stats3[2] = 0;
            for (auto& s : st) {
                stats3[0] += s.far_leaves;
                stats3[1] += s.near_leaves;
                stats3[2] += s.sauter_points;
            }
        }
    });
}
int orc_quad_oracle_pair_integrals(void* mh, const int* f, const int* g, long long npairs,
                                   double rel_tol, int workers, double* out)
{
    return guard([&] {
        const SurfaceMesh& m = *static_cast<SurfaceMesh*>(mh);
        run_partitioned(npairs, workers, [&](int, std::int64_t lo, std::int64_t hi) {
            for (std::int64_t i = lo; i < hi; ++i) out[i] = quad_oracle::pair_integral(m, f[i], g[i], rel_tol);
        });
    });
}
// adjacency class and permutation of one pair (quadrature.hpp:297-322)
int orc_pair_class(void* mh, int f, int g, int* pf, int* pg)
{
    std::array<int, 3> a, b;
    const int s = pair_permutation(*static_cast<SurfaceMesh*>(mh), f, g, a, b);
    for (int k = 0; k < 3; ++k) {
        pf[k] = a[k];
        pg[k] = b[k];
    }
    return s;
}
double orc_triangle_inverse_distance_integral(const double* tri9, const double* x3)
{
    const Tri t = {Vec3(tri9[0], tri9[1], tri9[2]), Vec3(tri9[3], tri9[4], tri9[5]),
                   Vec3(tri9[6], tri9[7], tri9[8])};
    return quad_oracle::triangle_inverse_distance_integral(t, Vec3(x3[0], x3[1], x3[2]));
}

// ---- inflation
void* orc_inflate(void* mh, int validate, int* status)
{
    InflatedMesh* out = nullptr;
    *status = guard([&] { out = new InflatedMesh(inflate(*static_cast<SurfaceMesh*>(mh), validate != 0)); });
    return out;
}
void orc_im_free(void* im) { delete static_cast<InflatedMesh*>(im); }
int orc_im_sizes(void* imh, int* sizes4)
{
    auto* im = static_cast<InflatedMesh*>(imh);
    sizes4[0] = im->num_jump_dofs();
    sizes4[1] = im->num_gvertices();
    sizes4[2] = im->base.num_vertices();
    sizes4[3] = im->base.num_facets();
    return 0;
}
// q[nv], gv_first[nv], dof_first[nv], ofacet_branch[2nf*3], jump_dofs[2n], normals[2nf*3]
int orc_im_export(void* imh, int* q, int* gv_first, int* dof_first, int* ofb, int* jd, double* normals)
{
    auto* im = static_cast<InflatedMesh*>(imh);
    const int nv = im->base.num_vertices(), no = im->num_oriented();
    for (int v = 0; v < nv; ++v) {
        q[v] = im->q[v];
        gv_first[v] = im->gv_first[v];
        dof_first[v] = im->dof_first[v];
    }
    for (int o = 0; o < no; ++o)
        for (int k = 0; k < 3; ++k) ofb[3 * o + k] = im->ofacet_branch[o][k];
    for (int d = 0; d < im->num_jump_dofs(); ++d) {
        jd[2 * d] = im->jump_dofs[d][0];
        jd[2 * d + 1] = im->jump_dofs[d][1];
    }
    if (normals)
        for (int o = 0; o < no; ++o) {
            normals[3 * o] = im->oriented_facets[o].normal.x;
            normals[3 * o + 1] = im->oriented_facets[o].normal.y;
            normals[3 * o + 2] = im->oriented_facets[o].normal.z;
        }
    return 0;
}
// surface curl of basis dof d on oriented facet o (assemble.hpp:59-66 + jump.hpp:33-43)
int orc_basis_curl(void* imh, int d, int o, double* out3)
{
    return guard([&] {
        auto* im = static_cast<InflatedMesh*>(imh);
        const TraceField tf = basis_trace(im->jump_dofs[d], *im);
        const Vec3 c = surface_curl(*im, o, tf);
        out3[0] = c.x;
        out3[1] = c.y;
        out3[2] = c.z;
    });
}
// curl of an arbitrary gvertex coefficient field
int orc_field_curl(void* imh, const double* coeff, int o, double* out3)
{
    return guard([&] {
        auto* im = static_cast<InflatedMesh*>(imh);
        TraceField tf;
        tf.coeff.assign(coeff, coeff + im->num_gvertices());
        const Vec3 c = surface_curl(*im, o, tf);
        out3[0] = c.x;
        out3[1] = c.y;
        out3[2] = c.z;
    });
}

// ---- assembly
int orc_assemble_W(void* imh, int far_order, int singular_order, double near, int workers,
                   long long pair_lo, long long pair_hi, double* W, long long* stats3)
{
    return guard([&] {
        auto* im = static_cast<InflatedMesh*>(imh);
        detail::QuadStats st;
        const Dense D = assemble_W(*im, qcfg(far_order, singular_order, near), workers, pair_lo, pair_hi,
                                   stats3 ? &st : nullptr);
        std::copy(D.a.begin(), D.a.end(), W);
        if (stats3) {
            stats3[0] = st.far_leaves;
            stats3[1] = st.near_leaves;
            stats3[2] = st.sauter_points;
        }
    });
}
// timing sampler of assemble_W (bench.py CPU baseline; sbo.hpp AssemblySampler)
void* orc_sampler_new(void* imh, int far_order, int singular_order, double near, int workers, int* status)
{
    void* out = nullptr;
    *status = guard([&] {
        out = new AssemblySampler(*static_cast<InflatedMesh*>(imh), qcfg(far_order, singular_order, near), workers);
    });
    return out;
}
void orc_sampler_free(void* h) { delete static_cast<AssemblySampler*>(h); }
int orc_sampler_fixed(void* h, double* seconds)
{
    return guard([&] { *seconds = static_cast<AssemblySampler*>(h)->fixed(); });
}
int orc_sampler_run(void* h, const long long* idx, long long k, double* seconds)
{
    return guard([&] {
        *seconds = static_cast<AssemblySampler*>(h)->run(reinterpret_cast<const std::int64_t*>(idx), k);
    });
}
int orc_assemble_W_rows(void* imh, int far_order, int singular_order, double near, const int* rows,
                        int nrows, int workers, double* out)
{
    return guard([&] {
        auto* im = static_cast<InflatedMesh*>(imh);
        const std::vector<int> r(rows, rows + nrows);
        const auto v = assemble_W_rows(*im, qcfg(far_order, singular_order, near), r, workers);
        std::copy(v.begin(), v.end(), out);
    });
}
int orc_rhs_points(void* imh, int far_order, double* pts)
{
    auto* im = static_cast<InflatedMesh*>(imh);
    const auto p = rhs_points(*im, qcfg(far_order, 8, 2.0));
    for (size_t i = 0; i < p.size(); ++i) {
        pts[3 * i] = p[i].x;
        pts[3 * i + 1] = p[i].y;
        pts[3 * i + 2] = p[i].z;
    }
    return 0;
}
int orc_assemble_rhs(void* imh, int far_order, const double* gvals, double* L)
{
    return guard([&] {
        auto* im = static_cast<InflatedMesh*>(imh);
        const int npt = far_order * far_order;
        std::vector<Vec3> g((size_t)im->base.num_facets() * npt);
        for (size_t i = 0; i < g.size(); ++i) g[i] = Vec3(gvals[3 * i], gvals[3 * i + 1], gvals[3 * i + 2]);
        const auto v = assemble_rhs(*im, g, qcfg(far_order, 8, 2.0));
        std::copy(v.begin(), v.end(), L);
    });
}

// ---- prolongation / partition
void* orc_build_prolongation(void* lh, void* imc, void* imf, int* status)
{
    Prolongation* P = nullptr;
    *status = guard([&] {
        P = new Prolongation(build_prolongation(static_cast<Level*>(lh)->pair, *static_cast<InflatedMesh*>(imc),
                                                *static_cast<InflatedMesh*>(imf)));
    });
    return P;
}
void* orc_empty_prolongation(int rows)
{
    auto* P = new Prolongation;
    P->rows = rows;
    P->cols = 0;
    P->col_ptr = {0};
    return P;
}
void* orc_prolongation_from(int rows, int cols, const int* col_ptr, const int* row_idx, const double* val)
{
    auto* P = new Prolongation;
    P->rows = rows;
    P->cols = cols;
    P->col_ptr.assign(col_ptr, col_ptr + cols + 1);
    P->row_idx.assign(row_idx, row_idx + col_ptr[cols]);
    P->val.assign(val, val + col_ptr[cols]);
    return P;
}
void* orc_identity_prolongation(int n)
{
    auto* P = new Prolongation;
    P->rows = P->cols = n;
    for (int i = 0; i < n; ++i) {
        P->col_ptr.push_back(i);
        P->row_idx.push_back(i);
        P->val.push_back(1.0);
    }
    P->col_ptr.push_back(n);
    return P;
}
void orc_prolongation_free(void* p) { delete static_cast<Prolongation*>(p); }
int orc_prolongation_sizes(void* ph, int* rows, int* cols, int* nnz)
{
    auto* P = static_cast<Prolongation*>(ph);
    *rows = P->rows;
    *cols = P->cols;
    *nnz = (int)P->val.size();
    return 0;
}
int orc_prolongation_export(void* ph, int* col_ptr, int* row_idx, double* val)
{
    auto* P = static_cast<Prolongation*>(ph);
    std::copy(P->col_ptr.begin(), P->col_ptr.end(), col_ptr);
    std::copy(P->row_idx.begin(), P->row_idx.end(), row_idx);
    std::copy(P->val.begin(), P->val.end(), val);
    return 0;
}
void* orc_partition(void* lh, void* imf, int* status)
{
    PartOut* out = nullptr;
    *status = guard([&] {
        out = new PartOut{partition_dofs(static_cast<Level*>(lh)->pair, *static_cast<InflatedMesh*>(imf))};
    });
    return out;
}
// partition from explicit lists (e.g. the all-wire-basket case of test_schwarz.cpp:141-142)
void* orc_partition_from(int nfaces, const int* face_ids, const int* face_ptr, const int* face_dofs, int nwb,
                         const int* wb)
{
    auto* out = new PartOut;
    for (int i = 0; i < nfaces; ++i)
        out->part.face_sets[face_ids[i]] = std::vector<int>(face_dofs + face_ptr[i], face_dofs + face_ptr[i + 1]);
    out->part.wirebasket.assign(wb, wb + nwb);
    return out;
}
void orc_partition_free(void* p) { delete static_cast<PartOut*>(p); }
int orc_partition_sizes(void* ph, int* nfaces, int* nface_dofs, int* nwb)
{
    auto& p = static_cast<PartOut*>(ph)->part;
    *nfaces = (int)p.face_sets.size();
    int t = 0;
    for (auto& [f, d] : p.face_sets) t += (int)d.size();
    *nface_dofs = t;
    *nwb = (int)p.wirebasket.size();
    return 0;
}
int orc_partition_export(void* ph, int* face_ids, int* face_ptr, int* face_dofs, int* wb)
{
    auto& p = static_cast<PartOut*>(ph)->part;
    int i = 0, t = 0;
    face_ptr[0] = 0;
    for (auto& [f, d] : p.face_sets) {
        face_ids[i] = f;
        for (int x : d) face_dofs[t++] = x;
        face_ptr[++i] = t;
    }
    std::copy(p.wirebasket.begin(), p.wirebasket.end(), wb);
    return 0;
}

// ---- Schwarz preconditioner
void* orc_build_preconditioner(const double* W, int n, void* parth, void* ph, int* status)
{
    SchwarzPreconditioner* out = nullptr;
    *status = guard([&] {
        Dense D;
        D.n = n;
        D.a.assign(W, W + (size_t)n * n);
        out = new SchwarzPreconditioner(
            build_preconditioner(D, static_cast<PartOut*>(parth)->part, *static_cast<Prolongation*>(ph)));
    });
    return out;
}
void orc_prec_free(void* p) { delete static_cast<SchwarzPreconditioner*>(p); }
int orc_prec_num_subspaces(void* p) { return static_cast<SchwarzPreconditioner*>(p)->num_subspaces(); }
int orc_apply_preconditioner(void* ph, const double* r, int n, double* z)
{
    return guard([&] {
        const auto out = apply_preconditioner(*static_cast<SchwarzPreconditioner*>(ph), std::vector<double>(r, r + n));
        std::copy(out.begin(), out.end(), z);
    });
}
int orc_coarse_matrix(const double* W, int n, void* ph, double* H)
{
    Dense D;
    D.n = n;
    D.a.assign(W, W + (size_t)n * n);
    const Dense h = coarse_matrix(D, *static_cast<Prolongation*>(ph));
    std::copy(h.a.begin(), h.a.end(), H);
    return 0;
}
// block Cholesky factors (for pivot checks): which = -1 wire-basket, -2 coarse, >=0 face index
int orc_prec_block_diag(void* ph, int which, double* diag, int* n_out)
{
    auto* p = static_cast<SchwarzPreconditioner*>(ph);
    const Dense& L = which == -1 ? p->wirebasket.L : (which == -2 ? p->coarse_L : p->faces[which].L);
    *n_out = L.n;
    if (diag)
        for (int i = 0; i < L.n; ++i) diag[i] = L(i, i);
    return 0;
}

// ---- PCG
// hist_cap sizes residual_history/alphas/betas; energy (optional) needs exact.
int orc_pcg(const double* W, int n, void* prec, const double* rhs, double tol, int maxit, const double* exact,
            double* x, int* iterations, int* converged, double* kappa, double* hist, double* energy,
            double* alphas, double* betas, int hist_cap, int* hist_len)
{
    return guard([&] {
        Dense D;
        D.n = n;
        D.a.assign(W, W + (size_t)n * n);
        std::vector<double> ex;
        if (exact) ex.assign(exact, exact + n);
        const PcgReport rep = pcg(D, static_cast<SchwarzPreconditioner*>(prec), std::vector<double>(rhs, rhs + n),
                                  tol, maxit, exact ? &ex : nullptr);
        std::copy(rep.solution.begin(), rep.solution.end(), x);
        *iterations = rep.iterations;
        *converged = rep.converged ? 1 : 0;
        *kappa = rep.kappa_estimate;
        const int h = (int)std::min<size_t>(rep.residual_history.size(), hist_cap);
        *hist_len = (int)rep.residual_history.size();
        for (int i = 0; i < h; ++i) {
            hist[i] = rep.residual_history[i];
            if (energy && exact) energy[i] = rep.energy_error_history[i];
        }
        for (int i = 0; i < (int)rep.alphas.size() && i < hist_cap; ++i) alphas[i] = rep.alphas[i];
        for (int i = 0; i < (int)rep.betas.size() && i < hist_cap; ++i) betas[i] = rep.betas[i];
    });
}
int orc_direct_solve(const double* W, int n, const double* rhs, double* x)
{
    return guard([&] {
        Dense D;
        D.n = n;
        D.a.assign(W, W + (size_t)n * n);
        const auto v = direct_solve(D, std::vector<double>(rhs, rhs + n));
        std::copy(v.begin(), v.end(), x);
    });
}
double orc_lanczos_kappa(const double* alphas, const double* betas, int k)
{
    return lanczos_kappa(std::vector<double>(alphas, alphas + k), std::vector<double>(betas, betas + k));
}
// Random SPD test matrix exactly as tests/test_pcg.cpp:12-20 (std::mt19937 +
// std::normal_distribution<double>; A*A^T + 0.1 I).
int orc_random_spd(int n, unsigned seed, double* W)
{
    std::mt19937 rng(seed);
    std::normal_distribution<double> dist;
    std::vector<double> A((size_t)n * n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) A[(size_t)i * n + j] = dist(rng);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            double s = 0;
            for (int k = 0; k < n; ++k) s += A[(size_t)i * n + k] * A[(size_t)j * n + k];
            W[(size_t)i * n + j] = s + (i == j ? 0.1 : 0.0);
        }
    return 0;
}
// std::normal_distribution<double> draws from std::mt19937(seed) (tests/test_pcg.cpp:14-15)
int orc_normal_draws(unsigned seed, int count, double* out)
{
    std::mt19937 rng(seed);
    std::normal_distribution<double> dist;
    for (int i = 0; i < count; ++i) out[i] = dist(rng);
    return 0;
}

// y = W x, the PCG matvec of pcg.hpp:70 (dense row-major, single thread), `reps` times
int orc_matvec(const double* W, int n, const double* x, double* y, int reps)
{
    return guard([&] {
        for (int r = 0; r < reps; ++r)
            for (int i = 0; i < n; ++i) {
                double s = 0;
                const double* row = W + (size_t)i * n;
                for (int j = 0; j < n; ++j) s += row[j] * x[j];
                y[i] = s;
            }
    });
}

double orc_wall_seconds()
{
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// ---- potential.hpp (3-D)
// points: np x 3 row-major; out: np values (potential.hpp:104-138)
int orc_eval_dl(void* imh, const double* v, const double* points, long long np, int far_order, int workers,
                double* out)
{
    return guard([&] {
        const InflatedMesh& im = *static_cast<InflatedMesh*>(imh);
        std::vector<double> vec(v, v + im.num_jump_dofs());
        std::vector<Vec3> pts((size_t)np);
        for (long long i = 0; i < np; ++i) pts[i] = Vec3(points[3 * i], points[3 * i + 1], points[3 * i + 2]);
        QuadratureConfig cfg;
        cfg.far_order = far_order;
        const std::vector<double> u = eval_DL(vec, im, pts, cfg, workers);
        std::copy(u.begin(), u.end(), out);
    });
}
// mesh.hpp:121-133 per point
int orc_distance_to(void* mh, const double* points, long long np, double* out)
{
    return guard([&] {
        const SurfaceMesh& m = *static_cast<SurfaceMesh*>(mh);
        for (long long i = 0; i < np; ++i)
            out[i] = distance_to(m, Vec3(points[3 * i], points[3 * i + 1], points[3 * i + 2]));
    });
}
// potential.hpp:15-25; out: capacity 3 nx ny; *count = points kept
int orc_make_cartesian_grid(void* mh, double lo, double hi, int nx, int ny, double mask_eps, double* out, int* count)
{
    return guard([&] {
        const std::vector<Vec3> pts = make_cartesian_grid(*static_cast<SurfaceMesh*>(mh), lo, hi, nx, ny, mask_eps);
        for (size_t i = 0; i < pts.size(); ++i) {
            out[3 * i] = pts[i].x;
            out[3 * i + 1] = pts[i].y;
            out[3 * i + 2] = pts[i].z;
        }
        *count = (int)pts.size();
    });
}
// jump.hpp:61-74 from a trace field given by its gvertex coefficients
int orc_jump_coordinates(void* imh, const double* coeff, double* out)
{
    return guard([&] {
        const InflatedMesh& im = *static_cast<InflatedMesh*>(imh);
        TraceField tf;
        tf.coeff.assign(coeff, coeff + im.num_gvertices());
        const std::vector<double> v = jump_coordinates(tf, im);
        std::copy(v.begin(), v.end(), out);
    });
}

}  // extern "C"
