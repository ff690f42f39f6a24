// C ABI (include/screenbem_b200.h) over the host layer and the device modules.
#include <cstring>
#include <memory>
#include <random>
#include <fstream>

#include "../../include/screenbem_b200.h"
#include "cuda/kernels.cuh"

using namespace sbg;

struct sbg_ctx {
    Ctx c;
};
struct sbg_mesh {
    SurfaceMesh m;
};
struct sbg_level {
    MeshLevelPair p;
};
struct sbg_inflated {
    InflatedMesh im;
};
struct sbg_matrix {
    DMatrix M;
};
struct sbg_partition {
    DofPartition p;
};
struct sbg_prolong {
    Prolongation R;
};
struct sbg_prec {
    Prec* P = nullptr;
    ~sbg_prec() { prec_destroy(P); }
};
struct sbg_aplan {
    AssemblyPlan* P = nullptr;
    Ctx* ctx = nullptr;
    ~sbg_aplan() { assembly_plan_destroy(P); }
};
namespace {
struct UserScope {
    std::string name;
    std::unique_ptr<TimedScope> ts;
};
thread_local std::vector<std::unique_ptr<UserScope>> g_user_scopes;
}  // namespace

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& fn)
{
    try {
        fn();
        return SBG_OK;
    } catch (const ValidationError& e) {
        g_err = e.what();
        return SBG_EVALIDATION;
    } catch (const NumericalError& e) {
        g_err = e.what();
        return SBG_ENUMERICAL;
    } catch (const CudaError& e) {
        g_err = e.what();
        return SBG_ECUDA;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SBG_EINTERNAL;
    }
}

// entry points run on the device of the context they are given (whatever the calling
// thread's current device is)
void bind_device(int dev)
{
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess || cur != dev) SBG_CUDA(cudaSetDevice(dev));
}
void bind_device(const Ctx* c)
{
    if (c) bind_device(c->device);
}

void need(const void* p, const char* what)
{
    if (!p) throw ValidationError(std::string("null argument: ") + what);
}
// every entry point validates its handles before touching them: a NULL handle is a
// validation error (status 2), never a crash
void bind_ctx(const sbg_ctx* ctx)
{
    need(ctx, "ctx");
    bind_device(&ctx->c);
}
void bind_mat(const sbg_matrix* W)
{
    need(W, "W");
    bind_device(W->M.ctx);
}

// The GEMV kernels read x with 16-byte vector loads over the padded row length W.ld
// (W's padding columns are zero).  A caller's d_x holds exactly n doubles with no
// alignment promise, so it is copied into a context scratch vector of ld entries whose
// tail is zeroed: no read past the caller's buffer, no NaN * 0 from garbage padding.
const double* padded_x(Ctx* c, const DMatrix& M, const double* d_x)
{
    need(d_x, "d_x");
    double* xp = scratch(c, kScratchMatvecX, (size_t)std::max(M.ld, 1));
    if (M.n) SBG_CUDA(cudaMemcpyAsync(xp, d_x, (size_t)M.n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    if (M.ld > M.n) SBG_CUDA(cudaMemsetAsync(xp + M.n, 0, (size_t)(M.ld - M.n) * sizeof(double), c->stream));
    return xp;
}

QuadCfg qcfg(const sbg_quad_cfg* c)
{
    QuadCfg q;
    if (c) {
        q.far_order = c->far_order;
        q.singular_order = c->singular_order;
        q.near_threshold = c->near_threshold;
        q.exact_far = c->exact_far != 0;
    }
    if (q.far_order < 1 || q.singular_order < 1) throw ValidationError("quadrature orders must be positive");
    return q;
}

SurfaceMesh make_mesh(int nv, const double* v, int nf, const int32_t* f)
{
    if (nv < 0 || nf < 0) throw ValidationError("negative count in mesh");
    SurfaceMesh m;
    m.vertices.resize(nv);
    for (int i = 0; i < nv; ++i) m.vertices[i] = Vec3(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
    m.facets.resize(nf);
    for (int i = 0; i < nf; ++i) m.facets[i] = {f[3 * i], f[3 * i + 1], f[3 * i + 2]};
    return m;
}
}  // namespace

extern "C" {

const char* sbg_last_error(void) { return g_err.c_str(); }
const char* sbg_version(void) { return "screenbem_b200 0.1 (sm_100a)"; }

// ---------------------------------------------------------------- context
int sbg_ctx_create(int device, sbg_ctx** out)
{
    return guard([&] {
        need(out, "out");
        int count = 0;
        SBG_CUDA(cudaGetDeviceCount(&count));
        if (device < 0 || device >= count) throw CudaError("no CUDA device " + std::to_string(device));
        cudaDeviceProp prop;
        SBG_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10) throw CudaError("sm_100a (B200) device required, found sm_" + std::to_string(prop.major) +
                                              std::to_string(prop.minor));
        SBG_CUDA(cudaSetDevice(device));
        auto* c = new sbg_ctx;
        c->c.device = device;
        c->c.sm_count = prop.multiProcessorCount;
        device_pool_init(device);
        // a blocking stream: the pool's legacy-stream allocations order against it (common.cuh)
        // highest priority: when the look-ahead's auxiliary stream (lowest priority) has
        // blocks pending too, the main stream's critical-path blocks are scheduled first
        int least = 0, greatest = 0;
        SBG_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        SBG_CUDA(cudaStreamCreateWithPriority(&c->c.stream, cudaStreamDefault, greatest));
        *out = c;
    });
}
void sbg_ctx_destroy(sbg_ctx* ctx) { delete ctx; }
int sbg_ctx_synchronize(sbg_ctx* ctx)
{
    return guard([&] {
        bind_ctx(ctx);
        SBG_CUDA(cudaStreamSynchronize(ctx->c.stream));
    });
}
int sbg_ctx_set_matvec_form(sbg_ctx* ctx, int form)
{
    return guard([&] {
        bind_ctx(ctx);
        if (form != 0 && form != 1) throw ValidationError("matvec form: 0 (symmetric) or 1 (full matrix)");
        ctx->c.matvec_form = form;
    });
}
int sbg_ctx_get_matvec_form(sbg_ctx* ctx, int* form)
{
    return guard([&] {
        bind_ctx(ctx);
        need(form, "form");
        *form = ctx->c.matvec_form;
    });
}
int sbg_device_name(int device, char* buf, int cap, int* sm_count)
{
    return guard([&] {
        cudaDeviceProp prop;
        SBG_CUDA(cudaGetDeviceProperties(&prop, device));
        if (buf && cap > 0) {
            std::strncpy(buf, prop.name, cap - 1);
            buf[cap - 1] = 0;
        }
        if (sm_count) *sm_count = prop.multiProcessorCount;
    });
}
int sbg_timers_enable(sbg_ctx* ctx, int on)
{
    return guard([&] {
        need(ctx, "ctx");
        ctx->c.timers.enabled = on != 0;
    });
}
int sbg_timers_reset(sbg_ctx* ctx)
{
    return guard([&] {
        need(ctx, "ctx");
        ctx->c.timers.reset();
    });
}
int sbg_timer_get(sbg_ctx* ctx, const char* name, double* total_ms, long long* count)
{
    return guard([&] {
        bind_ctx(ctx);
        ctx->c.timers.collect();
        *total_ms = 0;
        *count = 0;
        for (auto& t : ctx->c.timers.totals)
            if (t.first == name) {
                *total_ms = t.second.first;
                *count = t.second.second;
            }
    });
}

int sbg_timer_begin(sbg_ctx* ctx, const char* name)
{
    return guard([&] {
        bind_ctx(ctx);
        auto u = std::make_unique<UserScope>();
        u->name = name;
        u->ts = std::make_unique<TimedScope>(&ctx->c, u->name.c_str());
        g_user_scopes.push_back(std::move(u));
    });
}
int sbg_timer_end(sbg_ctx* ctx)
{
    return guard([&] {
        bind_ctx(ctx);
        (void)ctx;
        if (g_user_scopes.empty()) throw ValidationError("sbg_timer_end without sbg_timer_begin");
        g_user_scopes.back()->ts.reset();
        g_user_scopes.pop_back();
    });
}
long long sbg_launch_count(void) { return launch_count(); }

// ---------------------------------------------------------------- meshes
int sbg_mesh_create(int nv, const double* verts, int nf, const int32_t* facets, sbg_mesh** out)
{
    return guard([&] {
        need(out, "out");
        auto* m = new sbg_mesh;
        m->m = make_mesh(nv, verts, nf, facets);
        *out = m;
    });
}
void sbg_mesh_destroy(sbg_mesh* m) { delete m; }
int sbg_mesh_sizes(const sbg_mesh* m, int* nv, int* nf)
{
    return guard([&] {
        need(m, "m");
        *nv = m->m.num_vertices();
        *nf = m->m.num_facets();
    });
}
int sbg_mesh_export(const sbg_mesh* m, double* verts, int32_t* facets)
{
    return guard([&] {
        need(m, "m");
        for (int i = 0; i < m->m.num_vertices(); ++i) {
            verts[3 * i] = m->m.vertices[i].x;
            verts[3 * i + 1] = m->m.vertices[i].y;
            verts[3 * i + 2] = m->m.vertices[i].z;
        }
        for (int i = 0; i < m->m.num_facets(); ++i)
            for (int k = 0; k < 3; ++k) facets[3 * i + k] = m->m.facets[i][k];
    });
}
int sbg_validate_mesh(const sbg_mesh* m)
{
    return guard([&] {
        need(m, "m");
        validate_mesh(m->m);
    });
}
int sbg_make_builtin(const char* spec, sbg_mesh** out)
{
    return guard([&] {
        need(out, "out");
        auto* m = new sbg_mesh;
        try {
            m->m = make_builtin(spec);
        } catch (...) {
            delete m;
            throw;
        }
        *out = m;
    });
}
int sbg_refine_uniform_times(const sbg_mesh* m, int k, sbg_level** out)
{
    return guard([&] {
        need(m, "m");
        need(out, "out");
        auto* l = new sbg_level;
        l->p = refine_uniform_times(m->m, k);
        *out = l;
    });
}
int sbg_level_create(const sbg_mesh* coarse, const sbg_mesh* fine, const int32_t* parent, sbg_level** out)
{
    return guard([&] {
        need(coarse, "coarse");
        need(fine, "fine");
        need(out, "out");
        auto* l = new sbg_level;
        l->p.coarse = coarse->m;
        l->p.fine = fine->m;
        l->p.parent.assign(parent, parent + fine->m.num_facets());
        l->p.H = l->p.coarse.max_facet_diameter();
        l->p.h = l->p.fine.max_facet_diameter();
        *out = l;
    });
}
int sbg_make_config(int cfg, int ratio, sbg_level** out)
{
    return guard([&] {
        need(out, "out");
        auto* l = new sbg_level;
        try {
            l->p = make_config(cfg, ratio);
        } catch (...) {
            delete l;
            throw;
        }
        *out = l;
    });
}
int sbg_make_panels(int kind, int m, int r, sbg_level** out)
{
    return guard([&] {
        need(out, "out");
        auto* l = new sbg_level;
        try {
            l->p = make_panels(kind, m, r);
        } catch (...) {
            delete l;
            throw;
        }
        *out = l;
    });
}
int sbg_config_g(int cfg, double* g)
{
    return guard([&] {
        if (cfg == 2 || cfg == 4) {
            std::mt19937 rng(cfg == 2 ? 1u : 7u);
            std::normal_distribution<double> dist;
            double v[3];
            for (double& x : v) x = dist(rng);
            const double nrm = std::sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]);
            for (int k = 0; k < 3; ++k) g[k] = v[k] / nrm;
        } else if (cfg == 3) {
            g[0] = 1.0;
            g[1] = 0.5;
            g[2] = 0.25;
        } else if (cfg == 1 || cfg == 5) {
            g[0] = 0.0;
            g[1] = 0.0;
            g[2] = 1.0;
        } else {
            throw ValidationError("unknown BASELINE config " + std::to_string(cfg));
        }
    });
}
int sbg_level_mesh(const sbg_level* l, int fine, sbg_mesh** out)
{
    return guard([&] {
        need(l, "l");
        need(out, "out");
        auto* m = new sbg_mesh;
        m->m = fine ? l->p.fine : l->p.coarse;
        *out = m;
    });
}
int sbg_level_parent(const sbg_level* l, int32_t* parent)
{
    return guard([&] {
        need(l, "l");
        std::copy(l->p.parent.begin(), l->p.parent.end(), parent);
    });
}
int sbg_level_sizes(const sbg_level* l, double* H, double* h)
{
    return guard([&] {
        need(l, "l");
        *H = l->p.H;
        *h = l->p.h;
    });
}
void sbg_level_destroy(sbg_level* l) { delete l; }

// ---------------------------------------------------------------- inflation
int sbg_inflate(const sbg_mesh* m, int validate, sbg_inflated** out)
{
    return guard([&] {
        need(m, "m");
        need(out, "out");
        auto* im = new sbg_inflated;
        try {
            im->im = inflate(m->m, validate != 0);
        } catch (...) {
            delete im;
            throw;
        }
        *out = im;
    });
}
void sbg_inflated_destroy(sbg_inflated* im) { delete im; }
int sbg_inflated_sizes(const sbg_inflated* im, int* n, int* ng, int* nv, int* nf)
{
    return guard([&] {
        need(im, "im");
        *n = im->im.num_jump_dofs();
        *ng = im->im.num_gvertices();
        *nv = im->im.base.num_vertices();
        *nf = im->im.base.num_facets();
    });
}
int sbg_inflated_export(const sbg_inflated* imh, int32_t* q, int32_t* gv_first, int32_t* dof_first, int32_t* ofb,
                        int32_t* jd, double* normals)
{
    return guard([&] {
        need(imh, "imh");
        const InflatedMesh& im = imh->im;
        const int nv = im.base.num_vertices(), no = 2 * im.base.num_facets();
        for (int v = 0; v < nv; ++v) {
            if (q) q[v] = im.q[v];
            if (gv_first) gv_first[v] = im.gv_first[v];
            if (dof_first) dof_first[v] = im.dof_first[v];
        }
        for (int o = 0; o < no; ++o)
            for (int k = 0; k < 3; ++k) {
                if (ofb) ofb[3 * o + k] = im.ofacet_branch[o][k];
                if (normals) normals[3 * o + k] = k == 0 ? im.onormal[o].x : (k == 1 ? im.onormal[o].y : im.onormal[o].z);
            }
        if (jd)
            for (int d = 0; d < im.num_jump_dofs(); ++d) {
                jd[2 * d] = im.jump_dofs[d][0];
                jd[2 * d + 1] = im.jump_dofs[d][1];
            }
    });
}

// ---------------------------------------------------------------- matrices
int sbg_assemble_w(sbg_ctx* ctx, const sbg_inflated* im, const sbg_quad_cfg* cfg, int workers, sbg_matrix** out,
                   sbg_assembly_stats* stats)
{
    return sbg_assemble_w_host(ctx, im, cfg, workers, nullptr, out, stats);
}
int sbg_assemble_w_host(sbg_ctx* ctx, const sbg_inflated* im, const sbg_quad_cfg* cfg, int workers, double* host_w,
                        sbg_matrix** out, sbg_assembly_stats* stats)
{
    (void)workers;  // the reference's std::thread count; the GPU path ignores it
    return guard([&] {
        need(ctx, "ctx");
        need(im, "im");
        need(out, "out");
        bind_device(&ctx->c);
        auto* W = new sbg_matrix;
        try {
            AssemblyStats st;
            // a page-locked destination gets the copy overlapped with the near field; any other
            // destination is filled by the ordinary download afterwards
            bool pinned = false;
            if (host_w) {
                cudaPointerAttributes pa{};
                pinned = cudaPointerGetAttributes(&pa, host_w) == cudaSuccess && pa.type == cudaMemoryTypeHost;
                (void)cudaGetLastError();
            }
            assemble_W(&ctx->c, im->im, qcfg(cfg), W->M, &st, pinned ? host_w : nullptr);
            if (host_w && !pinned) matrix_download(W->M, host_w);
            if (stats) {
                stats->far_pairs = st.far_pairs;
                stats->near_pairs = st.near_pairs;
                stats->identical = st.identical;
                stats->edge = st.edge;
                stats->vertex = st.vertex;
                stats->near_leaves = st.near_leaves;
                stats->tiles = st.tiles;
                stats->tiles_skipped = st.tiles_skipped;
                stats->h2d_bytes = st.h2d_bytes;
            }
        } catch (...) {
            delete W;
            throw;
        }
        *out = W;
    });
}
int sbg_assembly_plan_create(sbg_ctx* ctx, const sbg_inflated* im, const sbg_quad_cfg* cfg, sbg_aplan** out)
{
    return guard([&] {
        need(im, "im");
        need(out, "out");
        bind_ctx(ctx);
        auto* p = new sbg_aplan;
        p->ctx = &ctx->c;
        try {
            p->P = assembly_plan_create(&ctx->c, im->im, qcfg(cfg));
        } catch (...) {
            delete p;
            throw;
        }
        *out = p;
    });
}
int sbg_assembly_run(sbg_aplan* plan, sbg_matrix** W, sbg_assembly_stats* stats)
{
    return sbg_assembly_run_shard(plan, W, 0, 1, stats);
}
int sbg_assembly_run_shard(sbg_aplan* plan, sbg_matrix** W, int rank, int world, sbg_assembly_stats* stats)
{
    return guard([&] {
        bind_device(plan ? plan->ctx : nullptr);
        need(plan, "plan");
        if (world < 1 || rank < 0 || rank >= world) throw ValidationError("shard: need 0 <= rank < world");
        need(W, "W");
        const bool fresh = *W == nullptr;
        if (fresh) *W = new sbg_matrix;
        try {
            AssemblyStats st;
            assembly_run(plan->P, (*W)->M, &st, rank, world);
            SBG_CUDA(cudaStreamSynchronize(plan->ctx->stream));
            if (stats) {
                stats->far_pairs = st.far_pairs;
                stats->near_pairs = st.near_pairs;
                stats->identical = st.identical;
                stats->edge = st.edge;
                stats->vertex = st.vertex;
                stats->near_leaves = st.near_leaves;
                stats->tiles = st.tiles;
                stats->tiles_skipped = st.tiles_skipped;
                stats->h2d_bytes = st.h2d_bytes;
            }
        } catch (...) {
            if (fresh) {
                delete *W;
                *W = nullptr;
            }
            throw;
        }
    });
}
void sbg_assembly_plan_destroy(sbg_aplan* plan) { delete plan; }
int sbg_matrix_create(sbg_ctx* ctx, int n, const double* host, sbg_matrix** out)
{
    return guard([&] {
        need(out, "out");
        bind_ctx(ctx);
        need(ctx, "ctx");
        if (n < 0) throw ValidationError("negative matrix size");
        auto* W = new sbg_matrix;
        try {
            matrix_alloc(&ctx->c, n, W->M);
            if (host) matrix_upload(W->M, host);
            SBG_CUDA(cudaStreamSynchronize(ctx->c.stream));
        } catch (...) {
            delete W;
            throw;
        }
        *out = W;
    });
}
int sbg_matrix_n(const sbg_matrix* W) { return W ? W->M.n : -1; }
int sbg_matrix_device_view(const sbg_matrix* W, void** data, int* ld, long long* count)
{
    return guard([&] {
        bind_mat(W);
        need(W, "W");
        if (data) *data = W->M.a.p;
        if (ld) *ld = W->M.ld;
        if (count) *count = (long long)W->M.a.n;
    });
}
int sbg_matrix_pack_upper(const sbg_matrix* W, double* d_packed)
{
    return guard([&] {
        bind_mat(W);
        need(d_packed, "d_packed");
        matrix_pack_upper(W->M, d_packed);
    });
}
int sbg_matrix_unpack_upper(sbg_matrix* W, const double* d_packed)
{
    return guard([&] {
        bind_mat(W);
        need(d_packed, "d_packed");
        matrix_unpack_upper(W->M, d_packed);
    });
}
int sbg_matrix_download(const sbg_matrix* W, double* host)
{
    return guard([&] {
        bind_mat(W);
        matrix_download(W->M, host);
    });
}
int sbg_matrix_download_rows(const sbg_matrix* W, const int32_t* rows, int nrows, double* host)
{
    return guard([&] {
        bind_mat(W);
        matrix_download_rows(W->M, rows, nrows, host);
    });
}
int sbg_matrix_symmetry_defect(const sbg_matrix* W, double* m)
{
    return guard([&] {
        bind_mat(W);
        *m = matrix_symmetry_defect(W->M);
    });
}
int sbg_matvec(sbg_ctx* ctx, const sbg_matrix* W, const double* x, double* y)
{
    return guard([&] {
        need(W, "W");
        bind_ctx(ctx);
        const int n = W->M.n;
        cudaStream_t s = ctx->c.stream;
        DBuf<double> dx(W->M.ld), dy(W->M.ld);
        SBG_CUDA(cudaMemsetAsync(dx.p, 0, dx.n * sizeof(double), s));
        SBG_CUDA(cudaMemcpyAsync(dx.p, x, n * sizeof(double), cudaMemcpyHostToDevice, s));
        GemvPlan plan;
        gemv_plan(&ctx->c, n, W->M.ld, plan);
        gemv(&ctx->c, W->M, plan, dx.p, dy.p);
        SBG_CUDA(cudaMemcpyAsync(y, dy.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
        SBG_CUDA(cudaStreamSynchronize(s));
    });
}
void sbg_matrix_destroy(sbg_matrix* W) { delete W; }

// reference: inc/assemble.hpp:191-205 (16-byte header, row-major doubles)
int sbg_matrix_dump_binary(const sbg_matrix* W, const char* path)
{
    return guard([&] {
        bind_mat(W);
        std::ofstream os(path, std::ios::binary);
        if (!os) throw ValidationError(std::string("cannot open matrix dump file: ") + path);
        char header[16] = {};
        std::memcpy(header, "SBEMW\0", 6);
        const uint32_t n = (uint32_t)W->M.n;
        std::memcpy(header + 8, &n, 4);
        os.write(header, 16);
        std::vector<double> rows;
        const int chunk = std::max(1, (int)((64u << 20) / (8 * std::max(1, W->M.n))));
        for (int r0 = 0; r0 < W->M.n; r0 += chunk) {
            const int r1 = std::min(W->M.n, r0 + chunk);
            std::vector<int> idx(r1 - r0);
            for (int i = r0; i < r1; ++i) idx[i - r0] = i;
            rows.resize((size_t)(r1 - r0) * W->M.n);
            matrix_download_rows(W->M, idx.data(), (int)idx.size(), rows.data());
            os.write(reinterpret_cast<const char*>(rows.data()), (std::streamsize)(rows.size() * 8));
        }
    });
}
// reference: inc/assemble.hpp:207-226
int sbg_matrix_load_binary(sbg_ctx* ctx, const char* path, sbg_matrix** out)
{
    return guard([&] {
        need(out, "out");
        bind_ctx(ctx);
        std::ifstream is(path, std::ios::binary);
        if (!is) throw ValidationError(std::string("cannot open matrix dump file: ") + path);
        char header[16] = {};
        is.read(header, 16);
        if (std::memcmp(header, "SBEMW\0", 6) != 0) throw ValidationError(std::string("bad magic in matrix dump: ") + path);
        uint32_t n = 0;
        std::memcpy(&n, header + 8, 4);
        std::vector<double> h((size_t)n * n);
        is.read(reinterpret_cast<char*>(h.data()), (std::streamsize)(h.size() * 8));
        if (!is) throw ValidationError(std::string("truncated matrix dump: ") + path);
        auto* W = new sbg_matrix;
        try {
            matrix_alloc(&ctx->c, (int)n, W->M);
            matrix_upload(W->M, h.data());
        } catch (...) {
            delete W;
            throw;
        }
        *out = W;
    });
}

int sbg_pair_integrals(sbg_ctx* ctx, const sbg_mesh* m, const sbg_quad_cfg* cfg, const int32_t* f, const int32_t* g,
                       long long np, double* out)
{
    return guard([&] {
        need(m, "m");
        bind_ctx(ctx);
        pair_integrals(&ctx->c, m->m, qcfg(cfg), f, g, np, out);
        for (long long i = 0; i < np; ++i)
            if (!std::isfinite(out[i])) throw NumericalError("quadrature produced a non-finite pair integral");
    });
}

int sbg_rhs_points(const sbg_inflated* im, const sbg_quad_cfg* cfg, double* pts)
{
    return guard([&] {
        need(im, "im");
        const auto p = rhs_points(im->im, qcfg(cfg));
        std::copy(p.begin(), p.end(), pts);
    });
}
int sbg_assemble_rhs(sbg_ctx* ctx, const sbg_inflated* im, const sbg_quad_cfg* cfg, const double* g, int g_is_field,
                     double* L)
{
    return guard([&] {
        need(im, "im");
        bind_ctx(ctx);
        assemble_rhs(&ctx->c, im->im, qcfg(cfg), g, g_is_field != 0, L);
    });
}

// ---------------------------------------------------------------- potential (3-D)
// reference: inc/potential.hpp:104-138
int sbg_eval_dl(sbg_ctx* ctx, const sbg_inflated* im, const double* v, const double* points, long long np,
                const sbg_quad_cfg* cfg, double* out)
{
    return guard([&] {
        need(im, "im");
        bind_ctx(ctx);
        if (np > 0) {
            need(points, "points");
            need(out, "out");
        }
        if (im->im.num_jump_dofs() > 0) need(v, "v");
        eval_dl(&ctx->c, im->im, v, points, np, qcfg(cfg), out);
    });
}
// reference: inc/potential.hpp:15-25
int sbg_make_cartesian_grid(sbg_ctx* ctx, const sbg_mesh* mesh, double lo, double hi, int nx, int ny,
                            double mask_eps, double* out, int* count)
{
    return guard([&] {
        need(mesh, "mesh");
        need(count, "count");
        bind_ctx(ctx);
        const std::vector<double> pts = make_cartesian_grid(&ctx->c, mesh->m, lo, hi, nx, ny, mask_eps);
        if (!pts.empty()) need(out, "out");
        std::copy(pts.begin(), pts.end(), out);
        *count = (int)(pts.size() / 3);
    });
}

// ---------------------------------------------------------------- partition / prolongation
int sbg_partition_dofs(const sbg_level* pair, const sbg_inflated* fine, sbg_partition** out)
{
    return guard([&] {
        need(pair, "pair");
        need(fine, "fine");
        need(out, "out");
        auto* p = new sbg_partition;
        try {
            p->p = partition_dofs(pair->p, fine->im);
        } catch (...) {
            delete p;
            throw;
        }
        *out = p;
    });
}
int sbg_partition_create(int nfaces, const int32_t* face_ids, const int32_t* face_ptr, const int32_t* face_dofs,
                         int nwb, const int32_t* wb, sbg_partition** out)
{
    return guard([&] {
        need(out, "out");
        auto* p = new sbg_partition;
        p->p.face_ids.assign(face_ids, face_ids + nfaces);
        p->p.face_ptr.assign(face_ptr, face_ptr + nfaces + 1);
        p->p.face_dofs.assign(face_dofs, face_dofs + (nfaces ? face_ptr[nfaces] : 0));
        p->p.wirebasket.assign(wb, wb + nwb);
        *out = p;
    });
}
int sbg_partition_sizes(const sbg_partition* p, int* nfaces, int* nface_dofs, int* nwb)
{
    return guard([&] {
        need(p, "p");
        *nfaces = (int)p->p.face_ids.size();
        *nface_dofs = (int)p->p.face_dofs.size();
        *nwb = (int)p->p.wirebasket.size();
    });
}
int sbg_partition_export(const sbg_partition* p, int32_t* ids, int32_t* ptr, int32_t* dofs, int32_t* wb)
{
    return guard([&] {
        need(p, "p");
        std::copy(p->p.face_ids.begin(), p->p.face_ids.end(), ids);
        std::copy(p->p.face_ptr.begin(), p->p.face_ptr.end(), ptr);
        std::copy(p->p.face_dofs.begin(), p->p.face_dofs.end(), dofs);
        std::copy(p->p.wirebasket.begin(), p->p.wirebasket.end(), wb);
    });
}
void sbg_partition_destroy(sbg_partition* p) { delete p; }
int sbg_build_prolongation(const sbg_level* pair, const sbg_inflated* coarse, const sbg_inflated* fine,
                           sbg_prolong** out)
{
    return guard([&] {
        need(pair, "pair");
        need(coarse, "coarse");
        need(fine, "fine");
        need(out, "out");
        auto* p = new sbg_prolong;
        try {
            p->R = build_prolongation(pair->p, coarse->im, fine->im);
        } catch (...) {
            delete p;
            throw;
        }
        *out = p;
    });
}
int sbg_prolong_create(int rows, int cols, const int32_t* col_ptr, const int32_t* row_idx, const double* val,
                       sbg_prolong** out)
{
    return guard([&] {
        need(out, "out");
        auto* p = new sbg_prolong;
        p->R.rows = rows;
        p->R.cols = cols;
        p->R.col_ptr.assign(col_ptr, col_ptr + cols + 1);
        const int nnz = col_ptr[cols];
        p->R.row_idx.assign(row_idx, row_idx + nnz);
        p->R.val.assign(val, val + nnz);
        *out = p;
    });
}
int sbg_prolong_sizes(const sbg_prolong* p, int* rows, int* cols, int* nnz)
{
    return guard([&] {
        need(p, "p");
        *rows = p->R.rows;
        *cols = p->R.cols;
        *nnz = (int)p->R.val.size();
    });
}
int sbg_prolong_export(const sbg_prolong* p, int32_t* col_ptr, int32_t* row_idx, double* val)
{
    return guard([&] {
        need(p, "p");
        std::copy(p->R.col_ptr.begin(), p->R.col_ptr.end(), col_ptr);
        std::copy(p->R.row_idx.begin(), p->R.row_idx.end(), row_idx);
        std::copy(p->R.val.begin(), p->R.val.end(), val);
    });
}
void sbg_prolong_destroy(sbg_prolong* p) { delete p; }

// ---------------------------------------------------------------- Schwarz
int sbg_build_preconditioner(sbg_ctx* ctx, const sbg_matrix* W, const sbg_partition* part, const sbg_prolong* R,
                             sbg_prec** out)
{
    return guard([&] {
        need(W, "W");
        need(part, "part");
        need(out, "out");
        bind_ctx(ctx);
        Prolongation none;
        none.rows = W->M.n;
        auto* p = new sbg_prec;
        try {
            p->P = prec_build(&ctx->c, W->M, part->p, R ? R->R : none, kPrecInverse);
        } catch (...) {
            delete p;
            throw;
        }
        *out = p;
    });
}
int sbg_build_preconditioner_mode(sbg_ctx* ctx, const sbg_matrix* W, const sbg_partition* part, const sbg_prolong* R,
                                  int mode, sbg_prec** out)
{
    return guard([&] {
        need(W, "W");
        need(part, "part");
        need(out, "out");
        bind_ctx(ctx);
        if (mode != kPrecTrsv && mode != kPrecInverse && mode != kPrecFactored)
            throw ValidationError("unknown preconditioner apply mode");
        Prolongation none;
        none.rows = W->M.n;
        auto* p = new sbg_prec;
        try {
            p->P = prec_build(&ctx->c, W->M, part->p, R ? R->R : none, mode);
        } catch (...) {
            delete p;
            throw;
        }
        *out = p;
    });
}
int sbg_apply_preconditioner(sbg_ctx* ctx, sbg_prec* p, const double* r, int n, double* z)
{
    return guard([&] {
        need(p, "p");
        bind_ctx(ctx);
        if (n != prec_n(p->P)) throw ValidationError("preconditioner length mismatch");
        cudaStream_t s = ctx->c.stream;
        DBuf<double> dr(std::max(n, 1)), dz(std::max(n, 1));
        SBG_CUDA(cudaMemcpyAsync(dr.p, r, n * sizeof(double), cudaMemcpyHostToDevice, s));
        prec_apply(&ctx->c, p->P, dr.p, dz.p, nullptr);
        SBG_CUDA(cudaMemcpyAsync(z, dz.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
        SBG_CUDA(cudaStreamSynchronize(s));
    });
}
int sbg_prec_num_subspaces(const sbg_prec* p) { return p ? prec_num_subspaces(p->P) : -1; }
int sbg_prec_block_diag(sbg_ctx* ctx, sbg_prec* p, int which, double* diag, int* n_out)
{
    return guard([&] {
        need(p, "p");
        bind_ctx(ctx);
        std::vector<double> d;
        prec_block_diag(&ctx->c, p->P, which, d);
        *n_out = (int)d.size();
        if (diag) std::copy(d.begin(), d.end(), diag);
    });
}
int sbg_coarse_matrix(sbg_ctx* ctx, const sbg_matrix* W, const sbg_prolong* R, double* H)
{
    return guard([&] {
        need(W, "W");
        need(R, "R");
        bind_ctx(ctx);
        std::vector<double> h;
        coarse_galerkin(&ctx->c, W->M, R->R, h);
        std::copy(h.begin(), h.end(), H);
    });
}
double sbg_prec_factor_bytes(const sbg_prec* p) { return p ? prec_factor_bytes(p->P) : -1.0; }

// ---------------------------------------------------------------- condition numbers
int sbg_materialize_preconditioner(sbg_ctx* ctx, sbg_prec* p, sbg_matrix** out)
{
    return guard([&] {
        bind_ctx(ctx);
        need(out, "out");
        need(p, "preconditioner");
        auto* m = new sbg_matrix;
        try {
            prec_materialize(&ctx->c, p->P, m->M);
        } catch (...) {
            delete m;
            throw;
        }
        *out = m;
    });
}
int sbg_prec_from_dense(sbg_ctx* ctx, const sbg_matrix* M, sbg_prec** out)
{
    return guard([&] {
        bind_ctx(ctx);
        need(out, "out");
        need(M, "matrix");
        auto* p = new sbg_prec;
        try {
            p->P = prec_from_dense(&ctx->c, M->M);
        } catch (...) {
            delete p;
            throw;
        }
        *out = p;
    });
}
int sbg_condition_number(sbg_ctx* ctx, const sbg_matrix* W, sbg_prec* p, double tol, int maxit, sbg_spectrum* out)
{
    return guard([&] {
        bind_ctx(ctx);
        need(out, "out");
        need(W, "matrix");
        const Spectrum sp = spectrum(&ctx->c, W->M, p ? p->P : nullptr, tol, maxit);
        out->lambda_min = sp.lambda_min;
        out->lambda_max = sp.lambda_max;
        out->kappa = sp.kappa;
        out->iterations = sp.iterations;
        out->converged = sp.converged ? 1 : 0;
    });
}
void sbg_prec_destroy(sbg_prec* p) { delete p; }

// ---------------------------------------------------------------- PCG
static void fill_report(const PcgResult& r, double* history, double* alphas, double* betas, int cap,
                        sbg_pcg_report* rep)
{
    if (rep) {
        rep->iterations = r.iterations;
        rep->converged = r.converged ? 1 : 0;
        rep->kappa_estimate = r.kappa;
        rep->history_len = (int)r.history.size();
    }
    for (int i = 0; i < cap; ++i) {
        if (history && i < (int)r.history.size()) history[i] = r.history[i];
        if (alphas && i < (int)r.alphas.size()) alphas[i] = r.alphas[i];
        if (betas && i < (int)r.betas.size()) betas[i] = r.betas[i];
    }
}
int sbg_pcg(sbg_ctx* ctx, const sbg_matrix* W, sbg_prec* prec, const double* rhs, int n, double tol, int maxit,
            double* x, double* history, double* alphas, double* betas, int hist_cap, sbg_pcg_report* rep)
{
    return guard([&] {
        need(W, "W");
        bind_ctx(ctx);
        if (n != W->M.n) throw ValidationError("pcg: right-hand side length mismatch");
        PcgResult r;
        pcg_run(&ctx->c, W->M, prec ? prec->P : nullptr, rhs, x, false, tol, maxit, r);
        fill_report(r, history, alphas, betas, hist_cap, rep);
    });
}

int sbg_pcg_exact(sbg_ctx* ctx, const sbg_matrix* W, sbg_prec* prec, const double* rhs, int n, double tol, int maxit,
                  const double* exact, double* x, double* history, double* energy, double* alphas, double* betas,
                  int hist_cap, sbg_pcg_report* rep)
{
    return guard([&] {
        bind_ctx(ctx);
        need(W, "W");
        need(exact, "exact");
        if (n != W->M.n) throw ValidationError("pcg: right-hand side length mismatch");
        PcgResult r;
        pcg_run(&ctx->c, W->M, prec ? prec->P : nullptr, rhs, x, false, tol, maxit, r, nullptr, exact);
        fill_report(r, history, alphas, betas, hist_cap, rep);
        for (int i = 0; energy && i < hist_cap && i < (int)r.energy.size(); ++i) energy[i] = r.energy[i];
    });
}
int sbg_pcg_rows(sbg_ctx* ctx, const sbg_matrix* W, sbg_prec* prec, const double* rhs, int n, int on_device,
                 double tol, int maxit, int row_lo, int row_hi, sbg_exchange_fn exchange, void* user, double* x,
                 double* history, double* alphas, double* betas, int hist_cap, sbg_pcg_report* rep)
{
    return sbg_pcg_rows_agree(ctx, W, prec, rhs, n, on_device, tol, maxit, row_lo, row_hi, exchange, nullptr, user, x,
                              history, alphas, betas, hist_cap, rep);
}
int sbg_pcg_rows_agree(sbg_ctx* ctx, const sbg_matrix* W, sbg_prec* prec, const double* rhs, int n, int on_device,
                       double tol, int maxit, int row_lo, int row_hi, sbg_exchange_fn exchange, sbg_agree_fn agree,
                       void* user, double* x, double* history, double* alphas, double* betas, int hist_cap,
                       sbg_pcg_report* rep)
{
    return guard([&] {
        bind_ctx(ctx);
        need(W, "W");
        if (n != W->M.n) throw ValidationError("pcg: right-hand side length mismatch");
        if (!exchange) throw ValidationError("pcg: row panel needs an exchange");
        RowPanel rows;
        rows.lo = row_lo;
        rows.hi = row_hi;
        rows.exchange = exchange;
        rows.agree = agree;
        rows.user = user;
        PcgResult r;
        pcg_run(&ctx->c, W->M, prec ? prec->P : nullptr, rhs, x, on_device != 0, tol, maxit, r, &rows);
        fill_report(r, history, alphas, betas, hist_cap, rep);
    });
}
int sbg_matvec_rows_device(sbg_ctx* ctx, const sbg_matrix* W, const double* d_x, double* d_y, int row_lo, int row_hi)
{
    return guard([&] {
        bind_ctx(ctx);
        need(W, "W");
        gemv_rows_range(&ctx->c, W->M, padded_x(&ctx->c, W->M, d_x), d_y, row_lo, row_hi);
    });
}
int sbg_ctx_stream(sbg_ctx* ctx, void** stream)
{
    return guard([&] {
        need(ctx, "ctx");
        need(stream, "stream");
        *stream = (void*)ctx->c.stream;
    });
}

// ---------------------------------------------------------------- device-resident helpers
int sbg_device_alloc(sbg_ctx* ctx, long long bytes, void** dptr)
{
    return guard([&] {
        bind_ctx(ctx);
        SBG_CUDA(cudaSetDevice(ctx->c.device));
        *dptr = device_alloc((size_t)bytes);
        SBG_CUDA(cudaMemsetAsync(*dptr, 0, (size_t)bytes, ctx->c.stream));
        SBG_CUDA(cudaStreamSynchronize(ctx->c.stream));
    });
}
int sbg_device_free(void* dptr)
{
    return guard([&] { device_free(dptr); });
}
int sbg_host_alloc(long long bytes, void** hptr)
{
    return guard([&] {
        need(hptr, "hptr");
        *hptr = nullptr;
        if (bytes > 0) SBG_CUDA(cudaHostAlloc(hptr, (size_t)bytes, cudaHostAllocDefault));
    });
}
int sbg_host_free(void* hptr)
{
    return guard([&] {
        if (hptr) SBG_CUDA(cudaFreeHost(hptr));
    });
}
int sbg_memcpy_h2d(sbg_ctx* ctx, void* dst, const void* src, long long bytes)
{
    return guard([&] {
        bind_ctx(ctx);
        SBG_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyHostToDevice, ctx->c.stream));
        SBG_CUDA(cudaStreamSynchronize(ctx->c.stream));
    });
}
int sbg_memcpy_d2h(sbg_ctx* ctx, void* dst, const void* src, long long bytes)
{
    return guard([&] {
        bind_ctx(ctx);
        SBG_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToHost, ctx->c.stream));
        SBG_CUDA(cudaStreamSynchronize(ctx->c.stream));
    });
}
int sbg_pcg_device(sbg_ctx* ctx, const sbg_matrix* W, sbg_prec* prec, const double* d_rhs, double tol, int maxit,
                   double* d_x, sbg_pcg_report* rep)
{
    return guard([&] {
        need(W, "W");
        bind_ctx(ctx);
        PcgResult r;
        pcg_run(&ctx->c, W->M, prec ? prec->P : nullptr, d_rhs, d_x, true, tol, maxit, r);
        fill_report(r, nullptr, nullptr, nullptr, 0, rep);
    });
}
int sbg_matvec_device(sbg_ctx* ctx, const sbg_matrix* W, const double* d_x, double* d_y, int reps)
{
    return guard([&] {
        need(W, "W");
        bind_ctx(ctx);
        GemvPlan plan;
        gemv_plan(&ctx->c, W->M.n, W->M.ld, plan);
        const double* xp = padded_x(&ctx->c, W->M, d_x);
        for (int i = 0; i < reps; ++i) gemv(&ctx->c, W->M, plan, xp, d_y);
        SBG_CUDA(cudaStreamSynchronize(ctx->c.stream));
    });
}
int sbg_matvec_bytes(sbg_ctx* ctx, const sbg_matrix* W, double* bytes)
{
    return guard([&] {
        need(W, "W");
        need(bytes, "bytes");
        bind_ctx(ctx);
        GemvPlan plan;
        gemv_plan(&ctx->c, W->M.n, W->M.ld, plan);
        *bytes = gemv_bytes(plan);
    });
}
int sbg_apply_preconditioner_device(sbg_ctx* ctx, sbg_prec* p, const double* d_r, double* d_z, int reps)
{
    return guard([&] {
        need(p, "p");
        bind_ctx(ctx);
        for (int i = 0; i < reps; ++i) prec_apply(&ctx->c, p->P, d_r, d_z, nullptr);
        SBG_CUDA(cudaStreamSynchronize(ctx->c.stream));
    });
}
int sbg_fp64_peak(sbg_ctx* ctx, double* tflops)
{
    return guard([&] {
        bind_ctx(ctx);
        *tflops = fp64_peak_tflops(&ctx->c);
    });
}
// L2 flush between timed launches: write 256 MiB (> the 126 MB L2), then read another
// 256 MiB, so the next timed kernel starts with a cold L2 holding only clean lines (a
// write-only flush leaves ~126 MB of dirty lines whose write-back lands inside the
// next timed kernel)
// device memory pool statistics (bytes): reserved by the pool, in use by allocations
int sbg_pool_stats(sbg_ctx* ctx, long long* reserved, long long* used)
{
    return guard([&] {
        bind_ctx(ctx);
        cudaMemPool_t pool;
        SBG_CUDA(cudaDeviceGetDefaultMemPool(&pool, ctx->c.device));
        unsigned long long r = 0, u = 0;
        SBG_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &r));
        SBG_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &u));
        *reserved = (long long)r;
        *used = (long long)u;
    });
}
int sbg_l2_flush(sbg_ctx* ctx)
{
    return guard([&] {
        bind_ctx(ctx);
        l2_flush(&ctx->c);
    });
}

}  // extern "C"
