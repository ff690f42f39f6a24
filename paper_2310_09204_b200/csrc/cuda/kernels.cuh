// Internal interfaces between the C-ABI layer and the device modules.
#pragma once

#include "common.cuh"

namespace sbg {

// ---------------------------------------------------------------- device math helpers
// No-FMA arithmetic in the oracle's operation order (oracle/sbo.hpp Vec3 ops);
// used wherever a decision (near/far, which facet to split) must be bitwise
// identical to the CPU restatement of quadrature.hpp:186-249.
struct D3 {
    double x, y, z;
};
__device__ __forceinline__ D3 d3_sub(D3 a, D3 b) { return {__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y), __dsub_rn(a.z, b.z)}; }
__device__ __forceinline__ D3 d3_add(D3 a, D3 b) { return {__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y), __dadd_rn(a.z, b.z)}; }
__device__ __forceinline__ D3 d3_scale(double s, D3 a) { return {__dmul_rn(s, a.x), __dmul_rn(s, a.y), __dmul_rn(s, a.z)}; }
__device__ __forceinline__ double d3_sqnorm(D3 a)
{
    return __dadd_rn(__dadd_rn(__dmul_rn(a.x, a.x), __dmul_rn(a.y, a.y)), __dmul_rn(a.z, a.z));
}
__device__ __forceinline__ double d3_norm(D3 a) { return __dsqrt_rn(d3_sqnorm(a)); }
__device__ __forceinline__ D3 d3_cross(D3 a, D3 b)
{
    return {__dsub_rn(__dmul_rn(a.y, b.z), __dmul_rn(a.z, b.y)), __dsub_rn(__dmul_rn(a.z, b.x), __dmul_rn(a.x, b.z)),
            __dsub_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x))};
}

// 1/sqrt(r2) to ~1 ulp: MUFU.RSQ64H seed + one third-order Newton step.
__device__ __forceinline__ double rsqrt_fast(double r2)
{
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
    const double h = r2 * y;
    const double e = fma(-h, y, 1.0);          // 1 - r2 y^2
    const double c = fma(0.375, e, 0.5);
    return fma(y, e * c, y);                    // y (1 + e/2 + 3e^2/8)
}

// acc + w / |x - y| from r2s = |x - y|^2 / w^2 (the rule weight folded into the squared
// distance, w > 0): rsqrt seed and one 3rd-order Newton step, y (1 + e (1/2 + 3e/8)) with
// e = 1 - r2s y^2 — five FP64 instructions after the seed, the weight multiply included.
// e comes from the seed's square: y has a zero low word (<= 21 significant bits), so y * y is
// exact, and the square reads one register where r2s * y would read two — on sm_100a the FP64
// pipe is bound by its register operands (profiles/r02b_micro_operand.md): config 5 far tiles
// 202.1 -> 197.7 ms, near leaves 103.6 -> 100.1 ms for the same instruction count
__device__ __forceinline__ double rsqrt_acc(double r2s, double acc)
{
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2s));
    const double e = fma(-r2s, y * y, 1.0);
    const double c = fma(0.375, e, 0.5);
    return fma(y, fma(e, c, 1.0), acc);
}
// the same step accumulated with the factor 8/3: y (8/3 + e (4/3 + e)) — the polynomial's
// constants enter as immediates of a DADD and a DFMA (0.375 above lives in a register: one
// operand read more per evaluation); the caller multiplies its sum by kRsqrtAccScale once
#ifndef RSQRT_ACC_SCALED
#define RSQRT_ACC_SCALED 3
#endif
#if RSQRT_ACC_SCALED
constexpr double kRsqrtAccScale = 0.375;
__device__ __forceinline__ double rsqrt_acc_s(double r2s, double acc)
{
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2s));
#if RSQRT_ACC_SCALED == 3
    // 8/3 + 4e/3 + e^2 = (e + 2/3)^2 + 20/9 with d = e + 2/3 = 5/3 - r2s y^2 formed by the
    // residual's own FMA: four FP64 instructions after the seed (d carries an absolute error
    // of 2^-54, i.e. 2^-55 relative in the polynomial: below its own rounding)
    const double d = fma(-r2s, y * y, 5.0 / 3.0);
    return fma(y, fma(d, d, 20.0 / 9.0), acc);
#elif RSQRT_ACC_SCALED == 2
    // 8/3 + 4e/3 + e^2 = (e + 2/3)^2 + 20/9: the square reads one register
    const double e = fma(-r2s, y * y, 1.0);
    const double d = e + 2.0 / 3.0;
    return fma(y, fma(d, d, 20.0 / 9.0), acc);
#else
    const double e = fma(-r2s, y * y, 1.0);
    const double c = e + 4.0 / 3.0;
    return fma(y, fma(e, c, 8.0 / 3.0), acc);
#endif
}
#else
constexpr double kRsqrtAccScale = 1.0;
__device__ __forceinline__ double rsqrt_acc_s(double r2s, double acc) { return rsqrt_acc(r2s, acc); }
#endif
// a padded (zero-weight) rule point: s = 0 and this constant term make r2s huge, so its
// contribution (~1e-150) vanishes below the rounding of any accumulated sum
constexpr double kPadR2 = 1e300;

double fp64_peak_tflops(Ctx* ctx);
void add_launches(long long k);  // launch bookkeeping for graph-replayed kernels
bool pcg_graph_enabled();        // PCG loop as one graph with a device-side while node (SBG_PCG_GRAPH=0: off)
void l2_flush(Ctx* ctx);  // write 256 MiB then read 256 MiB: cold, clean L2
// grow-only device scratch buffer `slot` of at least `count` doubles, cached on the
// context (large per-call temporaries: no pool growth or fragmentation between calls)
enum { kScratchInverse = 0, kScratchCoarseWR = 1, kScratchCoarsePart = 2, kScratchMatvecX = 3, kScratchSlots = 4 };
double* scratch(Ctx* ctx, int slot, size_t count);
cudaStream_t aux_stream(Ctx* ctx, int which = 0);  // the context's second (0) / third (1) stream

// ---------------------------------------------------------------- matrices
void matrix_alloc(Ctx* ctx, int n, DMatrix& M);
// W's upper triangle <-> a contiguous n (n + 1) / 2 vector (enqueued, no synchronisation)
void matrix_pack_upper(const DMatrix& M, double* d_packed);
void matrix_unpack_upper(DMatrix& M, const double* d_packed);
void matrix_upload(DMatrix& M, const double* host);
void matrix_download(const DMatrix& M, double* host);
void matrix_download_rows(const DMatrix& M, const int* rows, int nrows, double* host);
double matrix_symmetry_defect(const DMatrix& M);

// ---------------------------------------------------------------- dense fp64 GEMV (y = W x, W symmetric)
struct GemvPlan {
    int n = 0, ld = 0, strips = 0, chunks = 0, rows_per_chunk = 0;
    bool rows = false;  // row-per-warp form: the result lands in part directly (chunks = 1)
    DBuf<double> part;  // chunks x ld partial column sums
    // symmetric form: only the upper triangle is read, in tiles of H rows x C columns; each
    // tile adds its row sums (W x) and column sums (W^T x) to per-tile partials that one
    // fixed-order reduction combines (deterministic) — half the bytes of the full forms
    bool sym = false;
    int H = 0, C = 0, nstrips = 0, ntiles = 0;
    DBuf<int2> tiles;      // (strip, global column chunk) per tile, strip-major
    DBuf<int> tbase;       // first tile of each strip (nstrips + 1)
    DBuf<double> rowpart;  // ntiles x H row sums
    DBuf<double> colpart;  // nstrips x ld column sums (only columns right of the strip's block)
};
// form: 0 = the symmetric form where it pays (Ctx::matvec_form default), 1 = full-matrix forms
void gemv_plan(Ctx* ctx, int n, int ld, GemvPlan& plan);
double gemv_bytes(const GemvPlan& plan);  // algorithmic DRAM bytes of one matvec
// y[0:n] = W x ; x,y device vectors of length >= ld (padding zero)
void gemv(Ctx* ctx, const DMatrix& W, GemvPlan& plan, const double* x, double* y);

// ---------------------------------------------------------------- Schwarz preconditioner
struct Prec;
// kPrecInverse stores W_bb^-1 and applies one GEMV per block; when the largest block is big
// (n_b > 2048: the L^-T L^-1 product costs more than it saves) it stores X = L^-1 instead
// and applies z = X^T (X r) as two triangular GEMVs over the same bytes (kPrecFactored
// forces that form)
enum { kPrecTrsv = 0, kPrecInverse = 1, kPrecFactored = 2 };
Prec* prec_build(Ctx* ctx, const DMatrix& W, const DofPartition& part, const Prolongation& R, int mode);
int prec_mode(const Prec* p);
unsigned long long prec_uid(const Prec* p);  // unique per preconditioner object
void prec_destroy(Prec* p);
int prec_n(const Prec* p);
int prec_num_subspaces(const Prec* p);
// z = M r on device vectors (length n)
void prec_apply(Ctx* ctx, Prec* p, const double* r, double* z, const int* done_flag);
// the PCG-fused apply (precond.cu): update x, r, apply, r.z and the iteration's scalars
struct PcgDev;
struct PcgFused {
    PcgDev* st;
    double *x, *r, *rn;
    const double *p, *Wp;
    double *z, *partials, *hist, *alphas, *betas;
    const int* done;
    cudaGraphConditionalHandle gate;  // graph body: the while node's handle, set by the last kernel
    bool has_gate;
};
bool prec_apply_pcg(Ctx* ctx, Prec* p, const PcgFused& f);
struct PrecView;
bool prec_view(const Prec* p, PrecView& v);  // inverse mode with compact inverses only
void prec_block_diag(Ctx* ctx, Prec* p, int which, std::vector<double>& diag);
double prec_factor_bytes(const Prec* p);  // sum n_b^2 * 8 (roofline bookkeeping)
void prec_materialize(Ctx* ctx, Prec* p, DMatrix& M);  // schwarz.hpp:142-148
Prec* prec_from_dense(Ctx* ctx, const DMatrix& M);     // a dense SPD M as the preconditioner
// coarse Galerkin matrix R^T W R (n_c x n_c, row-major) — exposed for parity tests
void coarse_galerkin(Ctx* ctx, const DMatrix& W, const Prolongation& R, std::vector<double>& H);

// ---------------------------------------------------------------- PCG
struct PcgResult {
    int iterations = 0;
    bool converged = false;
    double kappa = 1.0;
    std::vector<double> history, alphas, betas;
    std::vector<double> energy;  // energy_error_history when an exact solution is given
};
// Row-panel PCG: this rank computes rows [lo, hi) of y = W p; `exchange`
// enqueues on `stream` the collective that fills the other ranks' rows of y (an
// all-gather).  Every other step of the iteration is replicated on each rank.
typedef int (*ExchangeFn)(void* user, const double* d_p, double* d_y, int n, void* stream);
// Collective stopping decision: given this rank's local "stop" (converged or maxit),
// return in *global_stop whether EVERY rank stops (a min over ranks), so all ranks
// enqueue the same number of exchanges even when their states differ in the last bits.
typedef int (*AgreeFn)(void* user, int local_stop, int* global_stop);
struct RowPanel {
    int lo = 0, hi = 0;
    ExchangeFn exchange = nullptr;
    AgreeFn agree = nullptr;
    void* user = nullptr;
};
// rhs/x: device vectors when on_device, else host; rows: null = the whole matvec here
void pcg_run(Ctx* ctx, const DMatrix& W, Prec* prec, const double* rhs, double* x, bool on_device, double tol,
             int maxit, PcgResult& out, const RowPanel* rows = nullptr, const double* exact = nullptr);
// y[lo:hi] = W[lo:hi, :] x on device vectors, enqueued on the context stream (no sync)
void gemv_rows_range(Ctx* ctx, const DMatrix& W, const double* x, double* y, int lo, int hi);
double lanczos_kappa(const std::vector<double>& alphas, const std::vector<double>& betas);
void lanczos_extremes(const std::vector<double>& alphas, const std::vector<double>& betas, double& lmin, double& lmax);
struct Spectrum {
    double lambda_min = 0, lambda_max = 0, kappa = 0;
    int iterations = 0;
    bool converged = false;
};
// schwarz.hpp:150-190 (condition_number) by Lanczos on the device (see linalg.cu)
Spectrum spectrum(Ctx* ctx, const DMatrix& W, Prec* prec, double tol, int maxit);

// ---------------------------------------------------------------- assembly
struct QuadCfg {
    int far_order = 4;
    int singular_order = 8;
    double near_threshold = 2.0;
    // SURVEY Appendix B switch: depth-0 far pairs evaluated bitwise like the oracle (one
    // thread per pair, i-major 16x16 order, IEEE sqrt and division, no FMA) instead of the
    // distance expansion with the refined rsqrt
    bool exact_far = false;
};
struct AssemblyStats {
    long long far_pairs = 0, near_pairs = 0, identical = 0, edge = 0, vertex = 0;
    long long near_leaves = 0, tiles = 0, tiles_skipped = 0;
    long long h2d_bytes = 0;  // bytes uploaded by the plan build
};
struct AssemblyPlan;
// defer: leave the curl-dependent half (plan_finish) to the first assembly_run, which builds
// it on the host while the near-field kernels run (the one-shot assemble_W)
AssemblyPlan* assembly_plan_create(Ctx* ctx, const InflatedMesh& im, const QuadCfg& cfg, bool defer = false);
void assembly_plan_destroy(AssemblyPlan* p);
// (rank, world): one shard of the work (world 1 = the whole assembly), see assemble.cu
// host_dst: also copy W to this page-locked n x n row-major buffer, overlapped with the near field
void assembly_run(AssemblyPlan* p, DMatrix& W, AssemblyStats* stats, int rank = 0, int world = 1,
                  double* host_dst = nullptr);
void assemble_W(Ctx* ctx, const InflatedMesh& im, const QuadCfg& cfg, DMatrix& W, AssemblyStats* stats,
                double* host_dst = nullptr);
void pair_integrals(Ctx* ctx, const SurfaceMesh& m, const QuadCfg& cfg, const int* f, const int* g, long long np,
                    double* out);
std::vector<double> rhs_points(const InflatedMesh& im, const QuadCfg& cfg);
// potential.hpp:104-138 (3-D): double-layer potential of jump vector v at np points (host
// arrays, points np x 3) into out; potential.hpp:15-25: the z = 0 evaluation grid (potential.cu)
void eval_dl(Ctx* ctx, const InflatedMesh& im, const double* v, const double* points, long long np,
             const QuadCfg& cfg, double* out);
std::vector<double> make_cartesian_grid(Ctx* ctx, const SurfaceMesh& m, double lo, double hi, int nx, int ny,
                                        double mask_eps);
void assemble_rhs(Ctx* ctx, const InflatedMesh& im, const QuadCfg& cfg, const double* g, bool g_is_field,
                  double* L_host);

}  // namespace sbg
