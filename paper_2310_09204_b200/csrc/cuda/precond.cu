// Two-level additive Schwarz preconditioner on the device.
// reference: inc/schwarz.hpp:55-140 (blocks, factor_block, build, apply).
//
// All blocks — faces (map order), the wire-basket and the coarse matrix — form
// one batch of dense SPD matrices stored as padded 64x64 tiles (identity on the
// padded diagonal, so every tile is full).  Build: batched panel-blocked tiled
// Cholesky — per tile column k ONE launch (k_panel_step) in which every CTA of the
// column applies the in-panel updates left-looking, factors and inverts the diagonal
// tile in shared memory (D_k = L_kk^-1) and forms its L_ik = A_ik D_k^T, plus one
// trailing update A_ij -= sum_panel A_iq A_jq^T per completed panel of 8 tile columns
// — with every tile GEMM on the FP64 tensor cores (DMMA, mma.sync.m8n8k4.f64).
// Apply, two modes:
//   * kPrecTrsv: blocked forward/backward triangular solves with L (the
//     reference's llt.solve, schwarz.hpp:130), one launch per tile step;
//   * kPrecInverse (default): the factor is turned into W_bb^-1 = L^-T L^-1 once
//     (blocked triangular inverse + L^-T L^-1 product, both DMMA), and every
//     apply is one batched dense GEMV over all blocks — the same HBM bytes as
//     two triangular solves with L, without their sequential tile chain.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>

#include "kernels.cuh"
#include "pcg_dev.cuh"
#include "prec_dev.cuh"

namespace sbg {

namespace {
constexpr int TB = 64;   // tile size
constexpr int TLD = 68;  // padded shared-memory leading dimension (conflict-free DMMA fragments)
constexpr int GEMV_ROWS = 8;  // one row per warp
// tile columns per panel of the blocked factorisation / inversion (SBG_PANEL overrides,
// for measurements)
int panel_width()
{
    static const int w = [] {
        const char* e = std::getenv("SBG_PANEL");
        const int v = e ? std::atoi(e) : 8;
        return v >= 1 && v <= 64 ? v : 8;
    }();
    return w;
}
enum { K_UPDATE = 1, K_XSTEP = 2, K_LAUUM = 3, K_XUPD = 4 };
struct GTask {
    int b, i, j, pad;
};
}  // namespace

namespace {
struct PrecSchedule;
}

struct Prec {
    Ctx* ctx = nullptr;
    int n = 0, nfaces = 0, nwb = 0, nc = 0, mode = kPrecInverse;
    bool factored = false;  // inverse mode storing X = L^-1 (Mc: X below the diagonal, X^T above)
    int nblocks = 0, coarse_block = -1, Tmax = 0, maxnb = 0;
    std::vector<int> h_nb, h_T, h_loc, h_Doff, h_ldm;
    std::vector<long long> h_Poff, h_Moff;
    DBuf<int> d_nb, d_T, d_loc, d_Doff, d_ldm;
    DBuf<long long> d_Poff, d_Moff;
    DBuf<double> Lp, Xp, D, Mc, loc, locy, loct;  // loct: X r of the factored apply
    DBuf<int> pos;  // dof -> loc index (face/WB), -1 if none
    DBuf<int> d_bptr, d_bdofs;  // face/WB block dof lists (CSR), for materialisation
    int ngather = 0;
    // R in CSC (restriction, ascending rows) and CSR (prolongation, ascending cols)
    DBuf<int> Rc_ptr, Rc_row, Rr_ptr, Rr_col;
    DBuf<double> Rc_val, Rr_val;
    std::shared_ptr<PrecSchedule> sched;  // task lists of build and apply (shared, cached per shape)
    unsigned long long uid = next_uid();
    static unsigned long long next_uid()
    {
        static std::atomic<unsigned long long> c{1};
        return c.fetch_add(1);
    }
    double apply_bytes = 0;
};

namespace {

// ---------------------------------------------------------------- DMMA helper
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// ---------------------------------------------------------------- gather / coarse Galerkin
// padded block b <- W[dofs, dofs] (full square) with identity on the padding; tasks
// (block, first row) of 8 rows, one warp per row (the big WB block gets enough CTAs)
__global__ void __launch_bounds__(256) k_gather_blocks(const double* __restrict__ W, int ld,
                                                       const int* __restrict__ bptr, const int* __restrict__ bdofs,
                                                       const int* __restrict__ Tv, const long long* __restrict__ Poff,
                                                       const int2* __restrict__ tasks, double* __restrict__ Lp)
{
    const int2 t = tasks[blockIdx.x];
    const int b = t.x, i = t.y + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    const int p0 = bptr[b], nb = bptr[b + 1] - p0;
    const int np = Tv[b] * TB;
    if (i >= np) return;
    double* dst = Lp + Poff[b] + (size_t)i * np;
    if (i < nb) {
        const double* wi = W + (size_t)bdofs[p0 + i] * ld;
        const int* cols = bdofs + p0;
#pragma unroll 4
        for (int j = lane; j < np; j += 32) dst[j] = j < nb ? wi[cols[j]] : 0.0;
    } else {
        for (int j = lane; j < np; j += 32) dst[j] = (i == j) ? 1.0 : 0.0;
    }
}

// WRt[c][i] = (W R)[i][c] = sum_{q in col c} R(r_q, c) W[r_q][i]  (W symmetric).
// Pass 1: task (column chunk of <= kQC support rows, 2048-wide i range): the chunk's rows
// of W are streamed coalesced and accumulated in registers (8 per thread) into a
// partial row; pass 2 sums a column's chunk partials in ascending order
// (deterministic).  Every row of W is read once per coarse column containing it
// (<= 3 for P1 prolongations), with thousands of CTAs whatever H/h is.
constexpr int kQC = 64, kIR = 1024;
__global__ void __launch_bounds__(256) k_coarse_WR_chunks(const double* __restrict__ W, int ld, int n,
                                                          const int4* __restrict__ chunks,
                                                          const int* __restrict__ crow,
                                                          const double* __restrict__ cval, double* __restrict__ part)
{
    const int4 ch = chunks[blockIdx.x];  // (column, q begin, q end, chunk index)
    const int i0 = blockIdx.y * kIR + threadIdx.x;
    double acc[kIR / 256];
#pragma unroll
    for (int k = 0; k < kIR / 256; ++k) acc[k] = 0.0;
    for (int q = ch.y; q < ch.z; ++q) {
        const double v = cval[q];
        const double* row = W + (size_t)crow[q] * ld;
#pragma unroll
        for (int k = 0; k < kIR / 256; ++k) {
            const int i = i0 + 256 * k;
            if (i < n) acc[k] = fma(v, __ldg(row + i), acc[k]);
        }
    }
    double* out = part + (size_t)ch.w * n;
#pragma unroll
    for (int k = 0; k < kIR / 256; ++k) {
        const int i = i0 + 256 * k;
        if (i < n) out[i] = acc[k];
    }
}

__global__ void k_coarse_WR_reduce(const double* __restrict__ part, const int* __restrict__ cfirst, int n,
                                   double* __restrict__ WRt)
{
    const int c = blockIdx.y;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s = 0.0;
    for (int k = cfirst[c]; k < cfirst[c + 1]; ++k) s += part[(size_t)k * n + i];
    WRt[(size_t)c * n + i] = s;
}

// H[a][b] = sum_{q in col b} R(r_q, b) WRt[a][r_q] (= (R^T W R)[b][a]) into a padded block
// (ldh) with identity padding; one warp per entry b of row a
__global__ void __launch_bounds__(256) k_coarse_Ht(const double* __restrict__ WRt, int n,
                                                   const int* __restrict__ cptr, const int* __restrict__ crow,
                                                   const double* __restrict__ cval, int nc, int ldh,
                                                   double* __restrict__ H)
{
    const int a = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const double* wa = WRt + (size_t)a * n;
    for (int b = warp; b < ldh; b += blockDim.x >> 5) {
        double s = 0.0;
        if (a < nc && b < nc) {
            for (int q = cptr[b] + lane; q < cptr[b + 1]; q += 32) s += cval[q] * wa[crow[q]];
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        } else {
            s = (a == b) ? 1.0 : 0.0;
        }
        if (lane == 0) H[(size_t)a * ldh + b] = s;
    }
}

// ---------------------------------------------------------------- tile GEMMs on DMMA
// 64x64 output tile per CTA (4 warps x 32x32), K streamed in half tiles of 32 through a
// two-stage cp.async pipeline.  Operands are staged as plain row copies in either
// layout — [m][k] (a row-major tile whose rows are output rows) or [k][m] (a tile whose
// rows are k) — and the DMMA fragments are read from whichever layout, so no operand is
// ever transposed on the way into shared memory.  Row strides 36 ([m][k]) and 68
// ([k][m]) keep both fragment reads bank-conflict free.
constexpr int HS_MK = 36, HS_KM = 68;          // half-tile row strides (doubles)
constexpr int HBUF = TB * HS_MK;               // >= 32 * HS_KM, doubles per staged half tile
constexpr size_t GEMM_SMEM = 4 * HBUF * sizeof(double);

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem)
{
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait()
{
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// half h (k in [32h, 32h+32)) of a 64x64 row-major tile: KM = false -> [m][k] copy of the
// columns, KM = true -> [k][m] copy of the rows
template <bool KM>
__device__ __forceinline__ void stage_half(double* __restrict__ dst, const double* __restrict__ src, size_t ld, int h)
{
    if (!KM) {
        for (int e = threadIdx.x; e < TB * 16; e += blockDim.x) {
            const int r = e >> 4, c = (e & 15) * 2;
            cp_async16(dst + r * HS_MK + c, src + (size_t)r * ld + 32 * h + c);
        }
    } else {
        for (int e = threadIdx.x; e < 32 * 32; e += blockDim.x) {
            const int r = e >> 5, c = (e & 31) * 2;
            cp_async16(dst + r * HS_KM + c, src + (size_t)(32 * h + r) * ld + c);
        }
    }
}

// acc[m][n] += sum_k A[m][k] B'[k][n] over one half tile; AK: A staged [k][m]; BK: B staged
// [k][n] (else [n][k], i.e. the product with the staged tile transposed)
template <bool AK, bool BK>
__device__ __forceinline__ void mma_half(const double* __restrict__ As, const double* __restrict__ Bs,
                                         double (&acc)[4][4][2])
{
    if (threadIdx.x >= 128) return;  // the 64x64 tile is 4 warps' work (wider CTAs: extra warps idle)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gid = lane >> 2, tig = lane & 3;
    const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
#pragma unroll
    for (int kk = 0; kk < 32; kk += 4) {
        double af[4], bf[4];
#pragma unroll
        for (int x = 0; x < 4; ++x)
            af[x] = AK ? As[(kk + tig) * HS_KM + wm + 8 * x + gid] : As[(wm + 8 * x + gid) * HS_MK + kk + tig];
#pragma unroll
        for (int y = 0; y < 4; ++y)
            bf[y] = BK ? Bs[(kk + tig) * HS_KM + wn + 8 * y + gid] : Bs[(wn + 8 * y + gid) * HS_MK + kk + tig];
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) dmma(acc[x][y][0], acc[x][y][1], af[x], bf[y]);
    }
}

// acc += sum_{q < nq} op(A_q) op(B_q), tiles given by the callables (pointer, ld)
template <bool AK, bool BK, class FA, class FB>
__device__ __forceinline__ void gemm_pipeline(double* sm, int nq, FA tileA, FB tileB, size_t lda, size_t ldb,
                                              double (&acc)[4][4][2])
{
    const int steps = 2 * nq;
    if (steps == 0) return;
    stage_half<AK>(sm, tileA(0), lda, 0);
    stage_half<BK>(sm + HBUF, tileB(0), ldb, 0);
    cp_commit();
    for (int st = 0; st < steps; ++st) {
        double* cur = sm + (st & 1) * 2 * HBUF;
        if (st + 1 < steps) {
            double* nxt = sm + ((st + 1) & 1) * 2 * HBUF;
            const int q = (st + 1) >> 1, h = (st + 1) & 1;
            stage_half<AK>(nxt, tileA(q), lda, h);
            stage_half<BK>(nxt + HBUF, tileB(q), ldb, h);
            cp_commit();
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        mma_half<AK, BK>(cur, cur + HBUF, acc);
        __syncthreads();
    }
}

// visit the accumulator elements: f(row, col, value)
template <class F>
__device__ __forceinline__ void for_acc(const double (&acc)[4][4][2], F f)
{
    if (threadIdx.x >= 128) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gid = lane >> 2, tig = lane & 3;
    const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y)
#pragma unroll
            for (int h = 0; h < 2; ++h) f(wm + 8 * x + gid, wn + 8 * y + 2 * tig + h, acc[x][y][h]);
}

#include "tile_factor.cuh"

// One step k of the panel-blocked Cholesky (panel [p0, p0 + kPanel)), all blocks and all
// tile rows i >= k of column k in one launch, task (block, i):
//   diag  A(k,k) - sum_{q=p0}^{k-1} L(k,q) L(k,q)^T   (left-looking inside the panel,
//         recomputed by every CTA of the column: no potrf launch and no inter-CTA wait)
//   own   A(i,k) - sum_{q=p0}^{k-1} L(i,q) L(k,q)^T   (i > k)
// then the diagonal tile is factored and inverted in shared memory (tile_ldl_inverse),
// CTA (b, k) stores L_kk (into Ld: the diagonal tile is still being read by the other
// CTAs of the step) and D_k = L_kk^-1, and CTA (b, i > k) forms L(i,k) = own D_k^T on DMMA
// with D_k taken straight from shared memory.  The previous panels' contributions came in
// through the panel-end trailing updates (K_UPDATE, K = the whole panel).
constexpr size_t STEP_SMEM = GEMM_SMEM + (size_t)TB * AS * sizeof(double) + TB * sizeof(double);
constexpr int kStepThreads = kFactorThreads;  // 8 warps: 4x4 blocks of the tile factor; the GEMMs use warps 0-3
__global__ void __launch_bounds__(kStepThreads) k_panel_step(int k, int p0, const GTask* __restrict__ tasks,
                                                    const int* __restrict__ Tv, const long long* __restrict__ Poff,
                                                    const int* __restrict__ Doff, double* __restrict__ Lp,
                                                    double* __restrict__ D, double* __restrict__ Ld,
                                                    int* __restrict__ fail)
{
    extern __shared__ __align__(16) double sm[];
    double* stg = sm;  // 4 half-tile staging buffers (GEMM pipeline, then the trsm operands)
    double* a = sm + 4 * HBUF;
    double* sq = a + TB * AS;
    __shared__ FactorBufs fb;
    const GTask t = tasks[blockIdx.x];
    const int b = t.b, i = t.i;
    const size_t ld = (size_t)Tv[b] * TB;
    double* L = Lp + Poff[b];
    auto tile = [&](int ti, int tj) { return L + (size_t)ti * TB * ld + (size_t)tj * TB; };
    const int nq = k - p0;
    double acc[4][4][2];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int z = 0; z < 4; ++z) acc[x][z][0] = acc[x][z][1] = 0.0;
    gemm_pipeline<false, false>(
        stg, nq, [&](int q) { return (const double*)tile(k, p0 + q); },
        [&](int q) { return (const double*)tile(k, p0 + q); }, ld, ld, acc);
    {
        const double* Akk = tile(k, k);
        for_acc(acc, [&](int r, int c, double v) { a[r * AS + c] = (c <= r) ? Akk[(size_t)r * ld + c] - v : 0.0; });
    }
    if (i != k) {
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int z = 0; z < 4; ++z) acc[x][z][0] = acc[x][z][1] = 0.0;
        gemm_pipeline<false, false>(
            stg, nq, [&](int q) { return (const double*)tile(i, p0 + q); },
            [&](int q) { return (const double*)tile(k, p0 + q); }, ld, ld, acc);
        const double* Aik = tile(i, k);
        // the updated A(i,k) as the trsm's A operand: [m][k] half tiles in stg[0], stg[HBUF]
        for_acc(acc, [&](int r, int c, double v) {
            stg[(c >> 5) * HBUF + r * HS_MK + (c & 31)] = Aik[(size_t)r * ld + c] - v;
        });
    }
    __syncthreads();
    double x[4][4];
    const bool ok = tile_ldl_inverse(a, fb, x);
    if (threadIdx.x < TB) sq[threadIdx.x] = sqrt(a[threadIdx.x * AS + threadIdx.x]);
    __syncthreads();
    const int r0 = blk_r0(), c0 = blk_c0();
    if (i == k) {
        double* Lkk = Ld + Doff[b] + (size_t)k * TB * TB;
        double* Dk = D + Doff[b] + (size_t)k * TB * TB;
        for (int e = threadIdx.x; e < TB * TB; e += blockDim.x) {
            const int r = e / TB, c = e % TB;
            Lkk[e] = c < r ? a[r * AS + c] / sq[c] : (c == r ? sq[r] : 0.0);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const int r = r0 + u, c = c0 + v;
                Dk[r * TB + c] = c <= r ? x[u][v] / sq[r] : 0.0;
            }
        if (threadIdx.x == 0 && !ok) atomicExch(&fail[b], 1);
        return;
    }
    // D_k = L_kk^-1 as the trsm's B operand ([n][k] half tiles: row n of D_k)
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int r = r0 + u, c = c0 + v;
            stg[(2 + (c >> 5)) * HBUF + r * HS_MK + (c & 31)] = c <= r ? x[u][v] / sq[r] : 0.0;
        }
    __syncthreads();
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int z = 0; z < 4; ++z) acc[x][z][0] = acc[x][z][1] = 0.0;
    mma_half<false, false>(stg, stg + 2 * HBUF, acc);
    mma_half<false, false>(stg + HBUF, stg + 3 * HBUF, acc);
    double* C = tile(i, k);
    for_acc(acc, [&](int r, int c, double v) { C[(size_t)r * ld + c] = v; });
}

// diagonal tiles L_kk from Ld into the factor (after the factorisation)
__global__ void k_put_diag(const int* __restrict__ Tv, const long long* __restrict__ Poff,
                           const int* __restrict__ Doff, const double* __restrict__ Ld, double* __restrict__ Lp)
{
    const int b = blockIdx.y, k = blockIdx.x;
    const int T = Tv[b];
    if (k >= T) return;
    const size_t ld = (size_t)T * TB;
    double* dst = Lp + Poff[b] + (size_t)k * TB * ld + (size_t)k * TB;
    const double* src = Ld + Doff[b] + (size_t)k * TB * TB;
    for (int e = threadIdx.x; e < TB * TB; e += blockDim.x) dst[(size_t)(e / TB) * ld + (e % TB)] = src[e];
}

// KIND K_UPDATE: L(i,j) -= sum_{q=k0}^{k1-1} L(i,q) L(j,q)^T   (task.i, task.j, K range in task.pad)
//      K_XSTEP : X(i,j) = -D_i (S(i,j) + sum_{q=k0}^{i-1} L(i,q) X(q,j)), X(i,i) = D_i  (step k = i;
//                S = the earlier panels' part, accumulated in X; left-looking inside the panel)
//      K_XUPD  : X(i',j) += sum_{q=k0}^{k1-1} L(i',q) X(q,j)          (K range in task.pad)
//                (right-looking blocked L^-1: X(i,j) = -D_i sum_{q=j}^{i-1} L(i,q) X(q,j))
//      K_LAUUM : M(i,j) = sum_{q=i}^{T-1} X(q,i)^T X(q,j)   (written over L)
template <int KIND>
__global__ void __launch_bounds__(128) k_tile_gemm(int k, const GTask* __restrict__ tasks, const int* __restrict__ Tv,
                                                   const long long* __restrict__ Poff, const int* __restrict__ Doff,
                                                   double* __restrict__ Lp, double* __restrict__ Xp,
                                                   const double* __restrict__ D)
{
    extern __shared__ __align__(16) double sm[];
    const GTask t = tasks[blockIdx.x];
    const int T = Tv[t.b];
    const size_t ld = (size_t)T * TB;
    double* L = Lp + Poff[t.b];
    double* X = Xp ? Xp + Poff[t.b] : nullptr;
    const double* Db = D + Doff[t.b];
    auto tile = [&](double* base, int ti, int tj) { return base + (size_t)ti * TB * ld + (size_t)tj * TB; };
    double acc[4][4][2];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;

    if (KIND == K_UPDATE) {  // K range [k0, k1) packed in t.pad (panel-blocked trailing update)
        const int k0 = t.pad >> 16, k1 = t.pad & 0xffff;
        gemm_pipeline<false, false>(
            sm, k1 - k0, [&](int q) { return (const double*)tile(L, t.i, k0 + q); },
            [&](int q) { return (const double*)tile(L, t.j, k0 + q); }, ld, ld, acc);
        double* C = tile(L, t.i, t.j);
        for_acc(acc, [&](int r, int c, double v) { C[(size_t)r * ld + c] -= v; });
    } else if (KIND == K_XSTEP) {  // in-panel K range [k0, t.i) packed in t.pad
        double* C = tile(X, t.i, t.j);
        const double* Di = Db + (size_t)t.i * TB * TB;
        if (t.i == t.j) {
            for (int e = threadIdx.x; e < TB * TB; e += blockDim.x) C[(size_t)(e / TB) * ld + (e % TB)] = Di[e];
            return;
        }
        const int k0 = t.pad >> 16, k1 = t.pad & 0xffff;
        gemm_pipeline<false, true>(
            sm, k1 - k0, [&](int q) { return (const double*)tile(L, t.i, k0 + q); },
            [&](int q) { return (const double*)tile(X, k0 + q, t.j); }, ld, ld, acc);
        // D_i as the A operand ([m][k] halves, cp.async) and S + acc as the B operand ([k][n])
        stage_half<false>(sm, Di, (size_t)TB, 0);
        stage_half<false>(sm + HBUF, Di, (size_t)TB, 1);
        cp_commit();
        for_acc(acc, [&](int r, int c, double v) {
            sm[(2 + (r >> 5)) * HBUF + (r & 31) * HS_KM + c] = C[(size_t)r * ld + c] + v;
        });
        cp_wait<0>();
        __syncthreads();
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
        mma_half<false, true>(sm, sm + 2 * HBUF, acc);
        mma_half<false, true>(sm + HBUF, sm + 3 * HBUF, acc);
        for_acc(acc, [&](int r, int c, double v) { C[(size_t)r * ld + c] = -v; });
    } else if (KIND == K_XUPD) {  // K range [k0, k1) packed in t.pad
        const int k0 = t.pad >> 16, k1 = t.pad & 0xffff;
        gemm_pipeline<false, true>(
            sm, k1 - k0, [&](int q) { return (const double*)tile(L, t.i, k0 + q); },
            [&](int q) { return (const double*)tile(X, k0 + q, t.j); }, ld, ld, acc);
        double* C = tile(X, t.i, t.j);
        for_acc(acc, [&](int r, int c, double v) { C[(size_t)r * ld + c] += v; });
    } else {  // K_LAUUM
        gemm_pipeline<true, true>(
            sm, T - t.i, [&](int q) { return (const double*)tile(X, t.i + q, t.i); },
            [&](int q) { return (const double*)tile(X, t.i + q, t.j); }, ld, ld, acc);
        double* C = tile(L, t.i, t.j);
        for_acc(acc, [&](int r, int c, double v) { C[(size_t)r * ld + c] = v; });
    }
}

// compact inverse: Mc_b[r][c] = M[max(r,c)][min(r,c)] over the valid n_b x n_b part,
// rows padded with zeros to ldm_b (a multiple of 4) so every row is 32-byte aligned.
// Tasks (block, tile row, tile col) of 32 x 32 output tiles; strictly-upper tiles read
// the mirrored lower tile coalesced and transpose it through shared memory.
__global__ void __launch_bounds__(256) k_compact_inverse(const double* __restrict__ Lp,
                                                         const long long* __restrict__ Poff,
                                                         const int* __restrict__ Tv, const int* __restrict__ nbv,
                                                         const int* __restrict__ ldmv,
                                                         const long long* __restrict__ Moff,
                                                         const int4* __restrict__ tasks, double* __restrict__ Mc)
{
    __shared__ double t[32][33];
    const int4 tk = tasks[blockIdx.x];
    const int b = tk.x, ti = tk.y, tj = tk.z;
    const int nb = nbv[b], ldm = ldmv[b];
    const size_t ld = (size_t)Tv[b] * TB;
    const double* M = Lp + Poff[b];
    double* out = Mc + Moff[b];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    if (ti >= tj) {
        for (int yy = ty; yy < 32; yy += 8) {
            const int r = ti * 32 + yy, c = tj * 32 + tx;
            if (r < nb && c < ldm) out[(size_t)r * ldm + c] = c >= nb ? 0.0 : (r >= c ? M[r * ld + c] : M[c * ld + r]);
        }
    } else {
        for (int yy = ty; yy < 32; yy += 8) {
            const int rr = tj * 32 + yy, cc = ti * 32 + tx;
            t[yy][tx] = (rr < nb && cc < nb) ? M[rr * ld + cc] : 0.0;
        }
        __syncthreads();
        for (int yy = ty; yy < 32; yy += 8) {
            const int r = ti * 32 + yy, c = tj * 32 + tx;
            if (r < nb && c < ldm) out[(size_t)r * ldm + c] = c >= nb ? 0.0 : t[tx][yy];
        }
    }
}

// ---------------------------------------------------------------- apply
// gather r into the block-local vector (faces/WB) and restrict to the coarse space:
// blocks [0, dof_blocks) gather one dof per thread, block dof_blocks + c restricts
// coarse column c (its support is ~n / nc DOFs: thousands at H/h = 40, so a whole
// CTA with four independent loads per thread, then a fixed-order reduction)
__global__ void __launch_bounds__(256) k_prec_gather(const double* __restrict__ r, int n, const int* __restrict__ pos,
                                                     double* __restrict__ loc, const int* __restrict__ cptr,
                                                     const int* __restrict__ crow, const double* __restrict__ cval,
                                                     int nc, double* __restrict__ loc_c, int dof_blocks, const int* done)
{
    pdl_wait();
    if (done && *done) return;
    if ((int)blockIdx.x < dof_blocks) {
        const int d = blockIdx.x * blockDim.x + threadIdx.x;
        if (d < n && pos[d] >= 0) loc[pos[d]] = r[d];
        return;
    }
    __shared__ double red[8];
    const int c = (int)blockIdx.x - dof_blocks;
    if (c >= nc) return;
    const int q0 = cptr[c], q1 = cptr[c + 1];
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int q = q0 + threadIdx.x;
    for (; q + 3 * 256 < q1; q += 4 * 256) {
        const int i0 = crow[q], i1 = crow[q + 256], i2 = crow[q + 512], i3 = crow[q + 768];
        s0 += cval[q] * r[i0];
        s1 += cval[q + 256] * r[i1];
        s2 += cval[q + 512] * r[i2];
        s3 += cval[q + 768] * r[i3];
    }
    for (; q < q1; q += 256) s0 += cval[q] * r[crow[q]];
    double s = (s0 + s1) + (s2 + s3);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += red[w];
        loc_c[c] = t;
    }
}

// y_b = M_b x_b: one row per warp, 8 rows per CTA; 128-bit streaming loads of M
// (8 in flight per lane), x_b through the L1 (it is re-read by every row of the block)
__global__ void __launch_bounds__(256) k_block_gemv(const int2* __restrict__ tasks, const int* __restrict__ nbv,
                                                    const int* __restrict__ ldmv, const int* __restrict__ locv,
                                                    const long long* __restrict__ Moff, const double* __restrict__ Mc,
                                                    const double* __restrict__ loc, double* __restrict__ locy,
                                                    const int* done)
{
    pdl_wait();
    if (done && *done) return;
    block_gemv_body(tasks[blockIdx.x], nbv, ldmv, locv, Moff, Mc, loc, locy);
}

// The factored apply's two passes over Mc (X below the diagonal, X^T above, X's diagonal on
// it): UPPER = false: t = X x over columns c <= r; UPPER = true: z = X^T t over columns c >= r.
// Same layout and loads as k_block_gemv; the band edges are masked per element.
template <bool UPPER>
__global__ void __launch_bounds__(256) k_block_gemv_tri(const int2* __restrict__ tasks, const int* __restrict__ nbv,
                                                        const int* __restrict__ ldmv, const int* __restrict__ locv,
                                                        const long long* __restrict__ Moff,
                                                        const double* __restrict__ Mc, const double* __restrict__ xin,
                                                        double* __restrict__ yout, const int* done)
{
    pdl_wait();
    if (done && *done) return;
    // the lower pass takes the rows longest-first (its rows grow with r), so the last wave
    // holds the shortest rows instead of the longest
    const int2 t = tasks[UPPER ? blockIdx.x : gridDim.x - 1 - blockIdx.x];
    const int b = t.x, nb = nbv[b], ldm = ldmv[b];
    const int r = t.y + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (r >= nb) return;
    const double2* x2 = reinterpret_cast<const double2*>(xin + locv[b]);
    const double2* row = reinterpret_cast<const double2*>(Mc + Moff[b] + (size_t)r * ldm);
    const int c2lo = UPPER ? (r >> 1) : 0, c2hi = UPPER ? (ldm >> 1) : (r >> 1) + 1;
    auto term = [&](int c2, const double2& a, const double2& xv) {
        const int c = 2 * c2;
        const double ax = (UPPER ? c >= r : c <= r) ? a.x : 0.0;
        const double ay = (UPPER ? c + 1 >= r : c + 1 <= r) ? a.y : 0.0;
        return fma(ax, xv.x, ay * xv.y);
    };
    double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int c2 = c2lo + lane;
    for (; c2 + 7 * 32 < c2hi; c2 += 8 * 32) {
        double2 a[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) a[u] = __ldcs(row + c2 + 32 * u);
#pragma unroll
        for (int u = 0; u < 8; ++u) s[u] += term(c2 + 32 * u, a[u], __ldg(x2 + c2 + 32 * u));
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const int cc = c2 + 32 * u;
        if (cc < c2hi) s[u] += term(cc, __ldcs(row + cc), __ldg(x2 + cc));
    }
    double v = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) yout[locv[b] + r] = v;
}

// full block inverses M_b = X_b^T X_b from the factored storage, for materialize / block_diag:
// M[r][c] = sum_{q >= max(r,c)} X[q][r] X[q][c] (X[q][r] = Mc[q][r] below the diagonal)
__global__ void k_factored_to_full(const int* __restrict__ nbv, const int* __restrict__ ldmv,
                                   const long long* __restrict__ Moff, const double* __restrict__ Mc,
                                   double* __restrict__ Mfull, int b)
{
    const int nb = nbv[b], ldm = ldmv[b];
    const double* X = Mc + Moff[b];
    double* M = Mfull + Moff[b];
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < (long long)nb * ldm;
         e += (long long)gridDim.x * blockDim.x) {
        const int r = (int)(e / ldm), c = (int)(e % ldm);
        double acc = 0.0;
        if (c < nb)
            for (int q = max(r, c); q < nb; ++q) acc = fma(X[(size_t)q * ldm + r], X[(size_t)q * ldm + c], acc);
        M[e] = acc;
    }
}

// 4 threads per row: partial dot of a 64-wide tile row
__device__ __forceinline__ double tile_row_dot(const double* __restrict__ T, size_t ld, int r, int kc,
                                               const double* v, int part)
{
    double s = 0.0;
    for (int c = part; c < kc; c += 4) s += T[(size_t)r * ld + c] * v[c];
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    return s;
}

// Forward step k (padded tiles): tasks (b, i >= k): v_i = loc_i - L(i,k-1) y_{k-1}; i == k: y_k = D_k v_k
__global__ void __launch_bounds__(256) k_trsv_fwd(int k, const int2* __restrict__ tasks, const int* __restrict__ Tv,
                                                  const int* __restrict__ locv, const long long* __restrict__ Poff,
                                                  const int* __restrict__ Doff, const double* __restrict__ Lp,
                                                  const double* __restrict__ D, double* __restrict__ loc,
                                                  const int* done)
{
    if (done && *done) return;
    __shared__ double yprev[TB], v[TB];
    const int2 t = tasks[blockIdx.x];
    const int b = t.x, i = t.y;
    const size_t ld = (size_t)Tv[b] * TB;
    double* lb = loc + locv[b];
    const int row = threadIdx.x >> 2, part = threadIdx.x & 3;
    if (threadIdx.x < TB) v[threadIdx.x] = lb[i * TB + threadIdx.x];
    if (k >= 1) {
        if (threadIdx.x < TB) yprev[threadIdx.x] = lb[(k - 1) * TB + threadIdx.x];
        __syncthreads();
        const double* T = Lp + Poff[b] + (size_t)i * TB * ld + (size_t)(k - 1) * TB;
        const double s = tile_row_dot(T, ld, row, TB, yprev, part);
        __syncthreads();
        if (part == 0) v[row] -= s;
    }
    __syncthreads();
    if (i == k) {
        const double* Dk = D + Doff[b] + (size_t)k * TB * TB;
        const double s = tile_row_dot(Dk, TB, row, row + 1, v, part);
        __syncthreads();
        if (part == 0) lb[i * TB + row] = s;
    } else if (threadIdx.x < TB) {
        lb[i * TB + threadIdx.x] = v[threadIdx.x];
    }
}

// Backward step with block-local k = T_b - 1 - s: tasks (b, i <= k):
//   v_i = loc_i - L(k+1,i)^T z_{k+1} (k+1 < T_b); i == k: z_k = D_k^T v_k
__global__ void __launch_bounds__(256) k_trsv_bwd(int s, const int2* __restrict__ tasks, const int* __restrict__ Tv,
                                                  const int* __restrict__ locv, const long long* __restrict__ Poff,
                                                  const int* __restrict__ Doff, const double* __restrict__ Lp,
                                                  const double* __restrict__ D, double* __restrict__ loc,
                                                  const int* done)
{
    if (done && *done) return;
    __shared__ double znext[TB], v[TB], red[4][TB];
    const int2 t = tasks[blockIdx.x];
    const int b = t.x, i = t.y, T = Tv[b];
    const size_t ld = (size_t)T * TB;
    const int k = T - 1 - s;
    double* lb = loc + locv[b];
    const int col = threadIdx.x & 63, grp = threadIdx.x >> 6;
    if (threadIdx.x < TB) v[threadIdx.x] = lb[i * TB + threadIdx.x];
    if (k + 1 < T) {
        if (threadIdx.x < TB) znext[threadIdx.x] = lb[(k + 1) * TB + threadIdx.x];
        __syncthreads();
        const double* Tt = Lp + Poff[b] + (size_t)(k + 1) * TB * ld + (size_t)i * TB;  // tile (k+1, i)
        double acc = 0.0;
        for (int r = grp; r < TB; r += 4) acc += Tt[(size_t)r * ld + col] * znext[r];
        red[grp][col] = acc;
        __syncthreads();
        if (threadIdx.x < TB) v[threadIdx.x] -= (red[0][threadIdx.x] + red[1][threadIdx.x]) +
                                                (red[2][threadIdx.x] + red[3][threadIdx.x]);
    }
    __syncthreads();
    if (i == k) {
        const double* Dk = D + Doff[b] + (size_t)k * TB * TB;
        double acc = 0.0;
        for (int r = col + grp; r < TB; r += 4) acc += Dk[(size_t)r * TB + col] * v[r];
        red[grp][col] = acc;
        __syncthreads();
        if (threadIdx.x < TB)
            lb[i * TB + threadIdx.x] = (red[0][threadIdx.x] + red[1][threadIdx.x]) +
                                       (red[2][threadIdx.x] + red[3][threadIdx.x]);
    } else if (threadIdx.x < TB) {
        lb[i * TB + threadIdx.x] = v[threadIdx.x];
    }
}

// z[d] = z_block[d] + (R y_c)[d]  (schwarz.hpp:126-138: faces/WB, then coarse)
__global__ void k_prec_scatter(const double* __restrict__ locy, const int* __restrict__ pos, int n,
                               const int* __restrict__ rptr, const int* __restrict__ rcol,
                               const double* __restrict__ rval, const double* __restrict__ y_c,
                               double* __restrict__ z, const int* done)
{
    pdl_wait();
    if (done && *done) return;
    const int d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= n) return;
    double out = pos[d] >= 0 ? locy[pos[d]] : 0.0;
    if (rptr) {
        double y = 0.0;
        for (int q = rptr[d]; q < rptr[d + 1]; ++q) y += rval[q] * y_c[rcol[q]];
        out += y;
    }
    z[d] = out;
}

// ---------------------------------------------------------------- PCG-fused apply
// The preconditioner apply inside a PCG iteration, fused with its neighbours
// (pcg.hpp:74-79): k_prec_gather_upd does the iteration's update — x += alpha p, the new
// residual r - alpha Wp into rn — while gathering it into the block-local vector, and the
// coarse restriction CTAs form R^T (r - alpha Wp) from the untouched r; k_block_gemv is
// unchanged; k_prec_scatter_rz forms z and r.z in one pass (copying rn back to r) and its
// last block finishes the iteration's scalars (beta, history, stopping test).
__global__ void __launch_bounds__(256) k_prec_gather_upd(const PcgDev* st, double* __restrict__ x,
                                                         const double* __restrict__ r, double* __restrict__ rn,
                                                         const double* __restrict__ p, const double* __restrict__ Wp,
                                                         int n, const int* __restrict__ pos, double* __restrict__ loc,
                                                         const int* __restrict__ cptr, const int* __restrict__ crow,
                                                         const double* __restrict__ cval, int nc,
                                                         double* __restrict__ loc_c, int dof_blocks)
{
    __shared__ double red[8];
    pdl_wait();
    if (st->done) return;
    prec_gather_upd_body(blockIdx.x, st->alpha, x, r, rn, p, Wp, n, pos, loc, cptr, crow, cval, nc, loc_c, dof_blocks,
                         red);
}

__global__ void __launch_bounds__(256) k_prec_scatter_rz(PcgDev* st, const double* __restrict__ locy,
                                                         const int* __restrict__ pos, int n,
                                                         const int* __restrict__ rptr, const int* __restrict__ rcol,
                                                         const double* __restrict__ rval,
                                                         const double* __restrict__ y_c, double* __restrict__ z,
                                                         double* __restrict__ r, const double* __restrict__ rn,
                                                         double* partials, double* hist, double* alphas, double* betas,
                                                         cudaGraphConditionalHandle gate, int has_gate)
{
    pdl_wait();
    if (st->done) {  // (an earlier kernel of this iteration stopped it: end the loop)
        if (has_gate && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(gate, 0u);
        return;
    }
    __shared__ double sh[32];
    double v = prec_scatter_body(blockIdx.x, locy, pos, n, rptr, rcol, rval, y_c, z, r, rn);
    v = block_sum(v, sh);
    if (last_block(v, partials, &st->counter) && threadIdx.x == 0) {
        const double rz_new = sum_partials(partials, gridDim.x);
        st->counter = 0;
        pcg_finish_rz(st, rz_new, hist, alphas, betas);
        if (has_gate) cudaGraphSetConditional(gate, st->done ? 0u : 1u);  // the while node's test
    }
}

// H = R^T W R (schwarz.hpp:110-116 with the sparse R) into a padded ldh x ldh block
// sync: wait for the kernels on the host (the build enqueues them and goes on)
void coarse_galerkin_device(Ctx* ctx, const DMatrix& W, const std::vector<int>& col_ptr,
                            const std::vector<int>& row_idx, const int* cptr, const int* crow, const double* cval,
                            int nc, int ldh, double* H, bool sync = true)
{
    const int n = W.n;
    cudaStream_t s = ctx->stream;
    std::vector<int4> chunks;
    std::vector<int> cfirst{0};
    for (int c = 0; c < nc; ++c) {
        for (int q = col_ptr[c]; q < col_ptr[c + 1]; q += kQC)
            chunks.push_back(make_int4(c, q, std::min(q + kQC, col_ptr[c + 1]), (int)chunks.size()));
        cfirst.push_back((int)chunks.size());
    }
    // launch order by first support row: the (<= 3) chunks of different coarse columns that
    // stream the same rows of W run back to back, so the re-reads hit L2 instead of HBM
    // (the partial index .w keeps the column order of the reduction: deterministic)
    std::stable_sort(chunks.begin(), chunks.end(),
                     [&](const int4& a, const int4& b) { return row_idx[a.y] < row_idx[b.y]; });
    double* WRt = scratch(ctx, kScratchCoarseWR, (size_t)n * std::max(nc, 1));
    if (!chunks.empty()) {
        DBuf<int4> d_chunks;
        DBuf<int> d_cfirst;
        d_chunks.upload(chunks, s);
        d_cfirst.upload(cfirst, s);
        double* part = scratch(ctx, kScratchCoarsePart, chunks.size() * (size_t)n);
        k_coarse_WR_chunks<<<dim3((unsigned)chunks.size(), (n + kIR - 1) / kIR), 256, 0, s>>>(W.a.p, W.ld, n,
                                                                                         d_chunks.p, crow, cval,
                                                                                         part);
        count_launch();
        k_coarse_WR_reduce<<<dim3((n + 255) / 256, nc), 256, 0, s>>>(part, d_cfirst.p, n, WRt);
        count_launch();
        SBG_LAUNCH_CHECK();
        if (sync) SBG_CUDA(cudaStreamSynchronize(s));  // (the task lists' frees are stream-ordered)
    } else {
        SBG_CUDA(cudaMemsetAsync(WRt, 0, (size_t)n * std::max(nc, 1) * sizeof(double), s));
    }
    k_coarse_Ht<<<ldh, 256, 0, s>>>(WRt, n, cptr, crow, cval, nc, ldh, H);
    count_launch();
    SBG_LAUNCH_CHECK();
    if (sync) SBG_CUDA(cudaStreamSynchronize(s));
}

// far = a look-ahead far update: its CTAs reserve FAR_SMEM of shared memory, so at most one
// sits on an SM and a critical-path CTA (STEP_SMEM or GEMM_SMEM) always fits beside it
constexpr size_t FAR_SMEM = 227 * 1024 - STEP_SMEM - 4096;
template <int KIND>
void launch_gemm(Ctx* ctx, Prec* P, int k, const GTask* dev_tasks, int count, double* Lp, double* Xp,
                 cudaStream_t st = nullptr, bool far = false)
{
    if (count <= 0) return;
    const size_t smem = far ? std::max(GEMM_SMEM, FAR_SMEM) : GEMM_SMEM;
    set_max_dynamic_smem(k_tile_gemm<KIND>, smem);
    k_tile_gemm<KIND><<<count, 128, smem, st ? st : ctx->stream>>>(k, dev_tasks, P->d_T.p, P->d_Poff.p, P->d_Doff.p,
                                                                  Lp, Xp, P->D.p);
    count_launch();
    SBG_LAUNCH_CHECK();
}

// Panel look-ahead on two streams.  At a panel end the trailing update is split into the
// next panel's tiles ("near", on the main stream, ahead of the next panel's steps) and all
// tiles beyond it ("far", on the context's auxiliary stream), so the far update — the bulk
// of the flops — runs beside the next panel's chain of latency-bound steps.  Ordering:
// a far update waits for its panel's last step; the next near update waits for the
// previous far update (both read-modify-write the tiles of the panel after next).
struct Lookahead {
    Ctx* ctx;
    cudaStream_t main, aux;
    cudaEvent_t done_steps = nullptr, far_done = nullptr;
    bool far_pending = false;
    explicit Lookahead(Ctx* c) : ctx(c), main(c->stream), aux(aux_stream(c))
    {
        SBG_CUDA(cudaEventCreateWithFlags(&done_steps, cudaEventDisableTiming));
        SBG_CUDA(cudaEventCreateWithFlags(&far_done, cudaEventDisableTiming));
    }
    ~Lookahead()
    {
        cudaEventDestroy(done_steps);
        cudaEventDestroy(far_done);
    }
    // at a panel end: enqueue_far(aux) after the steps so far; near(main) after the previous far
    template <class Near, class Far>
    void panel_end(Near near, Far far)
    {
        SBG_CUDA(cudaEventRecord(done_steps, main));
        if (far_pending) SBG_CUDA(cudaStreamWaitEvent(main, far_done, 0));
        near(main);
        SBG_CUDA(cudaStreamWaitEvent(aux, done_steps, 0));
        far(aux);
        SBG_CUDA(cudaEventRecord(far_done, aux));
        far_pending = true;
    }
    void join()
    {
        if (far_pending) SBG_CUDA(cudaStreamWaitEvent(main, far_done, 0));
        far_pending = false;
    }
};

// per-step task lists, built on the host once and uploaded in one copy
struct StepTasks {
    std::vector<GTask> all;
    std::vector<int> off{0};
    void close() { off.push_back((int)all.size()); }
    int count(int st) const { return off[st + 1] - off[st]; }
};

// Every task list of the build and the apply depends only on the block sizes, so it
// is generated once per partition shape and cached on the context (rebuilding the
// preconditioner after a re-assembly — the common pattern — does no host work).
struct PrecSchedule {
    std::vector<int> key;  // ngather, then n_b of every block
    std::vector<int2> gather;                // (block, first row), 8 rows each
    StepTasks pt, upd, upd_far, xd, xu;  // panel steps, trailing updates (near / far), L^-1 steps
    std::vector<GTask> la;
    std::vector<int4> ct;                    // compact-inverse 32x32 output tiles
    std::vector<int2> gemv, fw, bw;
    std::vector<int> fw_off{0}, bw_off{0};
    DBuf<int2> d_gather, d_gemv, d_fw, d_bw;
    DBuf<GTask> d_pt, d_upd, d_upd_far, d_xd, d_xu, d_la;
    DBuf<int4> d_ct;
};

std::shared_ptr<PrecSchedule> prec_schedule(Ctx* ctx, const Prec* P)
{
    const int kPanel = panel_width();
    std::vector<int> key{P->ngather, kPanel};
    key.insert(key.end(), P->h_nb.begin(), P->h_nb.end());
    if (auto* c = static_cast<std::shared_ptr<PrecSchedule>*>(ctx->prec_sched.get()))
        if (*c && (*c)->key == key) return *c;
    auto S = std::make_shared<PrecSchedule>();
    S->key = key;
    const int nb = P->nblocks;
    for (int b = 0; b < P->ngather; ++b)
        for (int r = 0; r < P->h_T[b] * TB; r += 8) S->gather.push_back({b, r});
    // Cholesky: panel-blocked, left-looking inside a panel (k_panel_step: every tile of
    // column k, diagonal included, in one launch) and one right-looking trailing update
    // with K = the whole panel when a panel completes (see prec_build)
    for (int k = 0; k < P->Tmax; ++k) {
        const int p0 = k - k % kPanel;
        for (int b = 0; b < nb; ++b) {
            const int T = P->h_T[b];
            if (T <= k) continue;
            for (int i = k; i < T; ++i) S->pt.all.push_back({b, i, k, 0});
            const int p1 = std::min(p0 + kPanel, T);
            if (k + 1 == p1)  // near: the next panel's columns; far: the columns beyond
                for (int j = p1; j < T; ++j)
                    for (int i = j; i < T; ++i)
                        (j < p1 + kPanel ? S->upd : S->upd_far).all.push_back({b, i, j, (p0 << 16) | p1});
        }
        S->pt.close();
        S->upd.close();
        S->upd_far.close();
    }
    // blocked L^-1 (left-looking inside a panel, one trailing update per panel), then L^-T L^-1
    for (int k = 0; k < P->Tmax; ++k) {
        const int p0 = k - k % kPanel;
        for (int b = 0; b < nb; ++b) {
            const int T = P->h_T[b];
            if (T <= k) continue;
            // row k of X in one launch: the in-panel rows q in [max(p0, j), k) left-looking
            for (int j = 0; j <= k; ++j) S->xd.all.push_back({b, k, j, (std::max(p0, j) << 16) | k});
            const int p1 = std::min(p0 + kPanel, T);
            if (k + 1 == p1)  // panel complete: rows below take K = the panel rows at once
                for (int i = p1; i < T; ++i)
                    for (int j = 0; j < p1; ++j) S->xu.all.push_back({b, i, j, (std::max(p0, j) << 16) | p1});
        }
        S->xd.close();
        S->xu.close();
    }
    for (int b = 0; b < nb; ++b)
        for (int i = 0; i < P->h_T[b]; ++i)
            for (int j = 0; j <= i; ++j) S->la.push_back({b, i, j, 0});
    for (int b = 0; b < nb; ++b) {
        const int tr = (P->h_nb[b] + 31) / 32, tc = (P->h_ldm[b] + 31) / 32;
        for (int ti = 0; ti < tr; ++ti)
            for (int tj = 0; tj < tc; ++tj) S->ct.push_back(make_int4(b, ti, tj, 0));
    }
    for (int b = 0; b < nb; ++b)
        for (int r = 0; r < P->h_nb[b]; r += GEMV_ROWS) S->gemv.push_back({b, r});
    for (int k = 0; k < P->Tmax; ++k) {
        for (int b = 0; b < nb; ++b)
            for (int i = k; i < P->h_T[b]; ++i) S->fw.push_back({b, i});
        S->fw_off.push_back((int)S->fw.size());
    }
    for (int st = 0; st < P->Tmax; ++st) {
        for (int b = 0; b < nb; ++b) {
            const int kk = P->h_T[b] - 1 - st;
            for (int i = 0; i <= kk; ++i) S->bw.push_back({b, i});
        }
        S->bw_off.push_back((int)S->bw.size());
    }
    cudaStream_t s = ctx->stream;
    S->d_gather.upload(S->gather, s);
    S->d_pt.upload(S->pt.all, s);
    S->d_upd.upload(S->upd.all, s);
    S->d_upd_far.upload(S->upd_far.all, s);
    S->d_xd.upload(S->xd.all, s);
    S->d_xu.upload(S->xu.all, s);
    S->d_la.upload(S->la, s);
    S->d_ct.upload(S->ct, s);
    S->d_gemv.upload(S->gemv, s);
    S->d_fw.upload(S->fw, s);
    S->d_bw.upload(S->bw, s);
    SBG_CUDA(cudaStreamSynchronize(s));
    ctx->prec_sched = std::make_shared<std::shared_ptr<PrecSchedule>>(S);
    return S;
}

// W_bb^-1 = L^-T L^-1 for every block from the tiled factor in Lwork (overwritten):
// X = L^-1 by panels (K_XSTEP per row of tiles, K_XUPD at panel ends), then M = X^T X over Lwork, then
// the compact row-major inverses (row stride ldm_b) into Mc.
// X = L^-1 scratch (zeroed, enqueued on the main stream)
double* inverse_scratch(Ctx* ctx, size_t n)
{
    double* Xp = scratch(ctx, kScratchInverse, std::max<size_t>(n, 1));
    TimedScope t0(ctx, "inv_alloc");
    SBG_CUDA(cudaMemsetAsync(Xp, 0, std::max<size_t>(n, 1) * sizeof(double), ctx->stream));
    return Xp;
}
// row k of X = L^-1 (K_XSTEP) and, at a panel end, its update of the rows below (K_XUPD):
// needs rows < k of X and the tiles L(k, q <= k), final once factorisation step k is done
void enqueue_inverse_row(Ctx* ctx, Prec* P, const PrecSchedule& S, int k, double* Lp, double* Xp, cudaStream_t st)
{
    launch_gemm<K_XSTEP>(ctx, P, k, S.d_xd.p + S.xd.off[k], S.xd.count(k), Lp, Xp, st);
    launch_gemm<K_XUPD>(ctx, P, k, S.d_xu.p + S.xu.off[k], S.xu.count(k), Lp, Xp, st);
}

// lower_done: X = L^-1 was already formed into the inverse scratch beside the factorisation
// (prec_build), so only the product / compaction remain
void form_inverses(Ctx* ctx, Prec* P, DBuf<double>& Lwork, DBuf<double>& Mc, bool factored = false,
                   bool lower_done = false)
{
    cudaStream_t s = ctx->stream;
    const PrecSchedule& S = *P->sched;
    struct {
        double* p;
    } Xp{lower_done ? scratch(ctx, kScratchInverse, std::max<size_t>(Lwork.n, 1)) : inverse_scratch(ctx, Lwork.n)};
    if (!lower_done) {
        TimedScope t1(ctx, "inv_lower");
        for (int k = 0; k < P->Tmax; ++k) enqueue_inverse_row(ctx, P, S, k, Lwork.p, Xp.p, s);
    }
    if (!factored) {
        TimedScope t2(ctx, "inv_lauum");
        launch_gemm<K_LAUUM>(ctx, P, 0, S.d_la.p, (int)S.la.size(), Lwork.p, Xp.p);
    }
    const long long Msize = P->h_Moff.empty() ? 0 : P->h_Moff.back() + (long long)P->h_nb.back() * P->h_ldm.back();
    Mc.alloc(std::max<long long>(Msize, 1));
    if (!S.ct.empty()) {
        // the symmetric completion of a lower triangle: of M = X^T X (over Lwork), or of X
        // itself for the factored storage (X below the diagonal, X^T above)
        k_compact_inverse<<<(int)S.ct.size(), 256, 0, s>>>(factored ? Xp.p : Lwork.p, P->d_Poff.p, P->d_T.p,
                                                           P->d_nb.p, P->d_ldm.p, P->d_Moff.p, S.d_ct.p, Mc.p);
        count_launch();
    }
    SBG_LAUNCH_CHECK();
    SBG_CUDA(cudaStreamSynchronize(s));
}

}  // namespace

// reference: inc/schwarz.hpp:100-118
Prec* prec_build(Ctx* ctx, const DMatrix& W, const DofPartition& part, const Prolongation& R, int mode)
{
    cudaStream_t s = ctx->stream;
    const int n = W.n;
    if (R.cols > 0 && R.rows != n) throw ValidationError("prolongation row count does not match the matrix");
    TimedScope tbuild(ctx, "build_preconditioner");
    auto* P = new Prec;
    try {
        P->ctx = ctx;
        P->n = n;
        P->mode = mode;
        P->nfaces = (int)part.face_ids.size();
        P->nwb = (int)part.wirebasket.size();
        P->nc = R.cols;
        // block dof lists: faces in map order, then WB (empty blocks skipped as in factor_block)
        std::vector<int> bptr{0}, bdofs, kinds;  // kinds: 0 face, 1 wb, 2 coarse
        for (int f = 0; f < P->nfaces; ++f) {
            const int a = part.face_ptr[f], e = part.face_ptr[f + 1];
            if (e == a) continue;
            bdofs.insert(bdofs.end(), part.face_dofs.begin() + a, part.face_dofs.begin() + e);
            bptr.push_back((int)bdofs.size());
            kinds.push_back(0);
        }
        if (P->nwb > 0) {
            bdofs.insert(bdofs.end(), part.wirebasket.begin(), part.wirebasket.end());
            bptr.push_back((int)bdofs.size());
            kinds.push_back(1);
        }
        for (int d : bdofs)
            if (d < 0 || d >= n) throw ValidationError("partition DOF out of range");
        const int ngather = (int)kinds.size();
        if (P->nc > 0) {
            kinds.push_back(2);
            P->coarse_block = ngather;
        }
        P->nblocks = (int)kinds.size();
        long long Poff = 0, Moff = 0;
        int Doff = 0, loc = 0;
        for (int b = 0; b < P->nblocks; ++b) {
            const int nb = b < ngather ? bptr[b + 1] - bptr[b] : P->nc;
            const int T = (nb + TB - 1) / TB;
            P->h_nb.push_back(nb);
            P->h_T.push_back(T);
            P->h_loc.push_back(loc);
            P->h_Poff.push_back(Poff);
            P->h_Doff.push_back(Doff);
            P->h_Moff.push_back(Moff);
            const int ldm = (nb + 3) / 4 * 4;
            P->h_ldm.push_back(ldm);
            Poff += (long long)T * TB * T * TB;
            Moff += (long long)nb * ldm;
            if ((long long)Doff + (long long)T * TB * TB > 0x7fffffffLL) throw ValidationError("preconditioner too large");
            Doff += T * TB * TB;
            loc += T * TB;
            P->Tmax = std::max(P->Tmax, T);
            P->maxnb = std::max(P->maxnb, ldm);
            P->apply_bytes += (double)nb * nb * 8.0;
        }
        P->d_nb.upload(P->h_nb, s);
        P->d_T.upload(P->h_T, s);
        P->d_loc.upload(P->h_loc, s);
        P->d_Poff.upload(P->h_Poff, s);
        P->d_Doff.upload(P->h_Doff, s);
        P->d_Moff.upload(P->h_Moff, s);
        P->d_ldm.upload(P->h_ldm, s);
        P->Lp.alloc(std::max<long long>(Poff, 1));
        P->D.alloc(std::max(Doff, 1));
        P->loc.alloc(std::max(loc, 1));
        P->locy.alloc(std::max(loc, 1));
        SBG_CUDA(cudaMemsetAsync(P->loc.p, 0, P->loc.n * sizeof(double), s));
        SBG_CUDA(cudaMemsetAsync(P->locy.p, 0, P->locy.n * sizeof(double), s));
        std::vector<int> pos(n, -1);
        for (int b = 0; b < ngather; ++b)
            for (int q = bptr[b]; q < bptr[b + 1]; ++q) pos[bdofs[q]] = P->h_loc[b] + (q - bptr[b]);
        P->pos.upload(pos, s);
        P->ngather = ngather;
        P->d_bptr.upload(bptr, s);
        P->d_bdofs.upload(bdofs, s);
        P->sched = prec_schedule(ctx, P);
        const PrecSchedule& S = *P->sched;
        if (ngather > 0) {  // factor_block's submatrix (schwarz.hpp:77-83)
            k_gather_blocks<<<(int)S.gather.size(), 256, 0, s>>>(W.a.p, W.ld, P->d_bptr.p, P->d_bdofs.p, P->d_T.p,
                                                                 P->d_Poff.p, S.d_gather.p, P->Lp.p);
            count_launch();
            SBG_LAUNCH_CHECK();
        }
        if (P->nc > 0) {  // R^T W R with the sparse R (schwarz.hpp:110-116)
            P->Rc_ptr.upload(R.col_ptr, s);
            P->Rc_row.upload(R.row_idx, s);
            P->Rc_val.upload(R.val, s);
            std::vector<int> rptr(n + 1, 0), rcol(R.val.size());
            std::vector<double> rval(R.val.size());
            for (int c = 0; c < R.cols; ++c)
                for (int q = R.col_ptr[c]; q < R.col_ptr[c + 1]; ++q) rptr[R.row_idx[q] + 1]++;
            for (int i = 0; i < n; ++i) rptr[i + 1] += rptr[i];
            std::vector<int> fill(rptr.begin(), rptr.end() - 1);
            for (int c = 0; c < R.cols; ++c)
                for (int q = R.col_ptr[c]; q < R.col_ptr[c + 1]; ++q) {
                    const int r = R.row_idx[q];
                    rcol[fill[r]] = c;
                    rval[fill[r]] = R.val[q];
                    fill[r]++;
                }
            P->Rr_ptr.upload(rptr, s);
            P->Rr_col.upload(rcol, s);
            P->Rr_val.upload(rval, s);
            TimedScope ts(ctx, "coarse_galerkin");
            const int ldh = P->h_T[P->coarse_block] * TB;
            coarse_galerkin_device(ctx, W, R.col_ptr, R.row_idx, P->Rc_ptr.p, P->Rc_row.p, P->Rc_val.p, P->nc, ldh,
                                   P->Lp.p + P->h_Poff[P->coarse_block], /*sync=*/false);
        }
        // ---- batched tiled Cholesky: per step k, potrf of tile (k,k), trsm of column k, trailing update
        DBuf<int> fail(std::max(P->nblocks, 1));
        SBG_CUDA(cudaMemsetAsync(fail.p, 0, fail.n * sizeof(int), s));
        // the inverse modes form X = L^-1 row by row on a third stream right behind the
        // factorisation (row k needs only factorisation step k and the rows above), so the
        // two latency-bound chains of Tmax steps run side by side instead of one after the other
        const bool need_inv = mode == kPrecInverse || mode == kPrecFactored;
        double* Xp = need_inv ? inverse_scratch(ctx, P->Lp.n) : nullptr;
        cudaStream_t xs = need_inv ? aux_stream(ctx, 1) : nullptr;
        cudaEvent_t step_ev = nullptr, x_ev = nullptr;
        if (need_inv) {
            SBG_CUDA(cudaEventCreateWithFlags(&step_ev, cudaEventDisableTiming));
            SBG_CUDA(cudaEventCreateWithFlags(&x_ev, cudaEventDisableTiming));
        }
        {
            TimedScope ts(ctx, "cholesky");
            set_max_dynamic_smem(k_panel_step, STEP_SMEM);
            DBuf<double> Ld(std::max(P->D.n, (size_t)1));
            Lookahead la(ctx);
            for (int k = 0; k < P->Tmax; ++k) {
                const int cnt = S.pt.count(k);
                if (cnt) {
                    k_panel_step<<<cnt, kStepThreads, STEP_SMEM, s>>>(k, k - k % panel_width(), S.d_pt.p + S.pt.off[k],
                                                                      P->d_T.p, P->d_Poff.p, P->d_Doff.p, P->Lp.p,
                                                                      P->D.p, Ld.p, fail.p);
                    count_launch();
                    SBG_LAUNCH_CHECK();
                }
                if (need_inv) {
                    SBG_CUDA(cudaEventRecord(step_ev, s));
                    SBG_CUDA(cudaStreamWaitEvent(xs, step_ev, 0));
                    enqueue_inverse_row(ctx, P, S, k, P->Lp.p, Xp, xs);
                }
                if (S.upd.count(k) + S.upd_far.count(k) > 0)
                    la.panel_end(
                        [&](cudaStream_t st) {
                            launch_gemm<K_UPDATE>(ctx, P, k, S.d_upd.p + S.upd.off[k], S.upd.count(k), P->Lp.p,
                                                  nullptr, st);
                        },
                        [&](cudaStream_t st) {
                            launch_gemm<K_UPDATE>(ctx, P, k, S.d_upd_far.p + S.upd_far.off[k], S.upd_far.count(k),
                                                  P->Lp.p, nullptr, st, true);
                        });
            }
            la.join();
            k_put_diag<<<dim3(P->Tmax, P->nblocks), 256, 0, s>>>(P->d_T.p, P->d_Poff.p, P->d_Doff.p, Ld.p, P->Lp.p);
            count_launch();
            SBG_LAUNCH_CHECK();
            SBG_CUDA(cudaStreamSynchronize(s));
        }
        if (need_inv) {  // the L^-1 chain's tail (its rows only read off-diagonal L tiles and D)
            TimedScope ts(ctx, "inv_lower");
            SBG_CUDA(cudaEventRecord(x_ev, xs));
            SBG_CUDA(cudaStreamWaitEvent(s, x_ev, 0));
            SBG_CUDA(cudaEventSynchronize(x_ev));
            cudaEventDestroy(step_ev);
            cudaEventDestroy(x_ev);
        }
        std::vector<int> hfail(fail.n);
        SBG_CUDA(cudaMemcpy(hfail.data(), fail.p, hfail.size() * sizeof(int), cudaMemcpyDeviceToHost));
        for (int b = 0; b < P->nblocks; ++b)
            if (hfail[b]) {
                if (kinds[b] == 2) throw NumericalError("coarse matrix factorization failed");
                throw NumericalError(std::string("block factorization failed (") +
                                     (kinds[b] == 0 ? "face" : "wire-basket") +
                                     "): partition inconsistent with the assembled matrix");
            }
        if (mode == kPrecInverse || mode == kPrecFactored) {
            // the factored storage when the L^-T L^-1 product would cost more than the second
            // GEMV pass of every apply saves (largest block > 2048 DOFs: config 5 H/h 8-20, 4)
            static const int force = [] {
                const char* e = std::getenv("SBG_PREC_FACTORED");
                return e ? std::atoi(e) : -1;
            }();
            P->factored = mode == kPrecFactored || (force < 0 ? P->maxnb > 2048 : force > 0);
            P->mode = kPrecInverse;
            if (P->factored) P->loct.alloc(P->loc.n);
            {
                TimedScope ts(ctx, "block_inverse");
                form_inverses(ctx, P, P->Lp, P->Mc, P->factored, true);
            }
            P->Lp.release();
            P->D.release();
        }
    } catch (...) {
        delete P;
        throw;
    }
    return P;
}

void prec_destroy(Prec* p) { delete p; }
int prec_n(const Prec* p) { return p->n; }
int prec_mode(const Prec* p) { return p->mode; }
unsigned long long prec_uid(const Prec* p) { return p->uid; }
int prec_num_subspaces(const Prec* p)  // schwarz.hpp:66-72
{
    return p->nfaces + (p->nwb > 0 ? 1 : 0) + (p->nc > 0 ? 1 : 0);
}
double prec_factor_bytes(const Prec* p) { return p->apply_bytes; }

// reference: inc/schwarz.hpp:121-140
// y_b = W_bb^-1 x_b for every block (loc -> locy): one GEMV over the stored inverses, or the
// factored storage's two triangular passes t = X x (loc -> loct), y = X^T t (loct -> locy)
static void enqueue_block_inverse(Ctx* ctx, Prec* P, const int* done)
{
    cudaStream_t s = ctx->stream;
    const dim3 grid((unsigned)P->sched->gemv.size()), block(256);
    if (!P->factored) {
        launch_pdl(k_block_gemv, grid, block, 0, s, P->sched->d_gemv.p, P->d_nb.p, P->d_ldm.p, P->d_loc.p,
                   P->d_Moff.p, P->Mc.p, P->loc.p, P->locy.p, done);
        count_launch();
        return;
    }
    launch_pdl(k_block_gemv_tri<false>, grid, block, 0, s, (const int2*)P->sched->d_gemv.p, (const int*)P->d_nb.p,
               (const int*)P->d_ldm.p, (const int*)P->d_loc.p, (const long long*)P->d_Moff.p, (const double*)P->Mc.p,
               (const double*)P->loc.p, P->loct.p, done);
    count_launch();
    launch_pdl(k_block_gemv_tri<true>, grid, block, 0, s, (const int2*)P->sched->d_gemv.p, (const int*)P->d_nb.p,
               (const int*)P->d_ldm.p, (const int*)P->d_loc.p, (const long long*)P->d_Moff.p, (const double*)P->Mc.p,
               (const double*)P->loct.p, P->locy.p, done);
    count_launch();
}

void prec_apply(Ctx* ctx, Prec* P, const double* r, double* z, const int* done)
{
    TimedScope ts(ctx, "precond_apply");
    cudaStream_t s = ctx->stream;
    const int n = P->n;
    if (n == 0) return;
    const int cb = P->coarse_block;
    double* loc_c = cb >= 0 ? P->loc.p + P->h_loc[cb] : nullptr;
    const int dof_blocks = (n + 255) / 256;
    launch_pdl(k_prec_gather, dim3(dof_blocks + P->nc), dim3(256), 0, s, r, n, P->pos.p, P->loc.p, P->Rc_ptr.p,
               P->Rc_row.p, P->Rc_val.p, P->nc, loc_c, dof_blocks, done);
    count_launch();
    const double* yloc;
    if (P->mode == kPrecInverse) {
        enqueue_block_inverse(ctx, P, done);
        yloc = P->locy.p;
    } else {
        for (int k = 0; k < P->Tmax; ++k) {
            const int cnt = P->sched->fw_off[k + 1] - P->sched->fw_off[k];
            if (cnt) {
                k_trsv_fwd<<<cnt, 256, 0, s>>>(k, P->sched->d_fw.p + P->sched->fw_off[k], P->d_T.p, P->d_loc.p, P->d_Poff.p,
                                               P->d_Doff.p, P->Lp.p, P->D.p, P->loc.p, done);
                count_launch();
            }
        }
        for (int st = 0; st < P->Tmax; ++st) {
            const int cnt = P->sched->bw_off[st + 1] - P->sched->bw_off[st];
            if (cnt) {
                k_trsv_bwd<<<cnt, 256, 0, s>>>(st, P->sched->d_bw.p + P->sched->bw_off[st], P->d_T.p, P->d_loc.p,
                                               P->d_Poff.p, P->d_Doff.p, P->Lp.p, P->D.p, P->loc.p, done);
                count_launch();
            }
        }
        yloc = P->loc.p;
    }
    launch_pdl(k_prec_scatter, dim3((n + 255) / 256), dim3(256), 0, s, (const double*)yloc, (const int*)P->pos.p, n,
               (const int*)(P->nc > 0 ? P->Rr_ptr.p : nullptr), (const int*)P->Rr_col.p, (const double*)P->Rr_val.p,
               (const double*)(cb >= 0 ? yloc + P->h_loc[cb] : nullptr), z, done);
    count_launch();
    SBG_LAUNCH_CHECK();
}

// The PCG-fused apply (inverse mode; see k_prec_gather_upd): the iteration's update, the
// apply and r.z in three launches.  Returns false for the TRSV mode (not fused).
bool prec_apply_pcg(Ctx* ctx, Prec* P, const PcgFused& f)
{
    if (P->mode != kPrecInverse || P->n == 0) return false;
    TimedScope ts(ctx, "precond_apply");
    cudaStream_t s = ctx->stream;
    const int n = P->n;
    const int cb = P->coarse_block;
    double* loc_c = cb >= 0 ? P->loc.p + P->h_loc[cb] : nullptr;
    const int dof_blocks = (n + 255) / 256;
    launch_pdl(k_prec_gather_upd, dim3(dof_blocks + P->nc), dim3(256), 0, s, (const PcgDev*)f.st, f.x,
               (const double*)f.r, f.rn, f.p, f.Wp, n, (const int*)P->pos.p, P->loc.p, (const int*)P->Rc_ptr.p,
               (const int*)P->Rc_row.p, (const double*)P->Rc_val.p, P->nc, loc_c, dof_blocks);
    count_launch();
    enqueue_block_inverse(ctx, P, f.done);
    launch_pdl(k_prec_scatter_rz, dim3(dof_blocks), dim3(256), 0, s, f.st, (const double*)P->locy.p,
               (const int*)P->pos.p, n, (const int*)(P->nc > 0 ? P->Rr_ptr.p : nullptr), (const int*)P->Rr_col.p,
               (const double*)P->Rr_val.p, (const double*)(cb >= 0 ? P->locy.p + P->h_loc[cb] : nullptr), f.z, f.r,
               (const double*)f.rn, f.partials, f.hist, f.alphas, f.betas, f.gate, f.has_gate ? 1 : 0);
    count_launch();
    SBG_LAUNCH_CHECK();
    return true;
}

// device pointers of an inverse-mode preconditioner with compact block inverses (not the
// factored or TRSV forms), for the persistent PCG kernel (linalg.cu)
bool prec_view(const Prec* P, PrecView& V)
{
    if (P->mode != kPrecInverse || P->factored || P->n == 0) return false;
    const int cb = P->coarse_block;
    V.n = P->n;
    V.nc = P->nc;
    V.dof_blocks = (P->n + 255) / 256;
    V.ntasks = (int)P->sched->gemv.size();
    V.pos = P->pos.p;
    V.loc = P->loc.p;
    V.locy = P->locy.p;
    V.Rc_ptr = P->Rc_ptr.p;
    V.Rc_row = P->Rc_row.p;
    V.Rc_val = P->Rc_val.p;
    V.loc_c = cb >= 0 ? P->loc.p + P->h_loc[cb] : nullptr;
    V.Rr_ptr = P->nc > 0 ? P->Rr_ptr.p : nullptr;
    V.Rr_col = P->Rr_col.p;
    V.Rr_val = P->Rr_val.p;
    V.y_c = cb >= 0 ? P->locy.p + P->h_loc[cb] : nullptr;
    V.tasks = P->sched->d_gemv.p;
    V.nbv = P->d_nb.p;
    V.ldmv = P->d_ldm.p;
    V.locv = P->d_loc.p;
    V.Moff = P->d_Moff.p;
    V.Mc = P->Mc.p;
    return true;
}

// diagonal of the block's Cholesky factor (TRSV mode) or of its inverse (inverse mode)
void prec_block_diag(Ctx* ctx, Prec* P, int which, std::vector<double>& diag)
{
    int b = -1;
    if (which >= 0)
        b = which;
    else if (which == -1)
        b = P->nwb > 0 ? (P->coarse_block >= 0 ? P->coarse_block - 1 : P->nblocks - 1) : -1;
    else if (which == -2)
        b = P->coarse_block;
    diag.clear();
    if (b < 0 || b >= P->nblocks) return;
    const int nb = P->h_nb[b];
    if (P->mode == kPrecInverse) {
        const int ldm = P->h_ldm[b];
        std::vector<double> h((size_t)nb * ldm);
        SBG_CUDA(cudaMemcpy(h.data(), P->Mc.p + P->h_Moff[b], h.size() * sizeof(double), cudaMemcpyDeviceToHost));
        for (int i = 0; i < nb; ++i) {
            if (!P->factored) {
                diag.push_back(h[(size_t)i * ldm + i]);
                continue;
            }
            double d = 0.0;  // (X^T X)_ii = sum_{q >= i} X_qi^2, row i above the diagonal holds X_qi
            for (int c = i; c < nb; ++c) d += h[(size_t)i * ldm + c] * h[(size_t)i * ldm + c];
            diag.push_back(d);
        }
    } else {
        const size_t ld = (size_t)P->h_T[b] * TB;
        std::vector<double> h(ld * ld);
        SBG_CUDA(cudaMemcpy(h.data(), P->Lp.p + P->h_Poff[b], h.size() * sizeof(double), cudaMemcpyDeviceToHost));
        for (int i = 0; i < nb; ++i) diag.push_back(h[(size_t)i * ld + i]);
    }
    (void)ctx;
}

namespace {
// M[d_r][d_c] = (W_bb^-1)[r][c] for the face / WB blocks (their DOF sets are disjoint)
__global__ void k_mat_blocks(const int* __restrict__ bptr, const int* __restrict__ bdofs,
                             const int* __restrict__ nbv, const int* __restrict__ ldmv,
                             const long long* __restrict__ Moff, const double* __restrict__ Mc, double* __restrict__ M,
                             int ld)
{
    const int b = blockIdx.x, p0 = bptr[b], nb = nbv[b], ldm = ldmv[b];
    const double* Mb = Mc + Moff[b];
    for (int r = blockIdx.y; r < nb; r += gridDim.y) {
        double* row = M + (size_t)bdofs[p0 + r] * ld;
        for (int c = threadIdx.x; c < nb; c += blockDim.x) row[bdofs[p0 + c]] = Mb[(size_t)r * ldm + c];
    }
}

// M[i][j] += sum_a R(i,a) sum_c H^-1[a][c] R(j,c)  (the coarse term of apply(e_j), schwarz.hpp:132-138)
__global__ void k_mat_coarse(int n, const int* __restrict__ rptr, const int* __restrict__ rcol,
                             const double* __restrict__ rval, const double* __restrict__ Hinv, int ldh,
                             double* __restrict__ M, int ld)
{
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
        const int q0 = rptr[i], q1 = rptr[i + 1];
        if (q0 == q1) continue;
        double* row = M + (size_t)i * ld;
        for (int j = threadIdx.x; j < n; j += blockDim.x) {
            double z = 0.0;
            for (int q = q0; q < q1; ++q) {
                const double* Ha = Hinv + (size_t)rcol[q] * ldh;
                double y = 0.0;
                for (int q2 = rptr[j]; q2 < rptr[j + 1]; ++q2) y += Ha[rcol[q2]] * rval[q2];
                z += rval[q] * y;
            }
            row[j] += z;
        }
    }
}
}  // namespace

// reference: inc/schwarz.hpp:142-148 (materialize_preconditioner).  The columns of M
// are apply(e_j); M is assembled from the block inverses (formed from a copy of the
// factor in TRSV mode) and the coarse term instead of n applies.
void prec_materialize(Ctx* ctx, Prec* P, DMatrix& M)
{
    cudaStream_t s = ctx->stream;
    const int n = P->n;
    matrix_alloc(ctx, n, M);
    if (n == 0) return;
    DBuf<double> work, Mtmp;
    const DBuf<double>* Mc = &P->Mc;
    if (P->mode != kPrecInverse) {
        work.alloc(P->Lp.n);
        SBG_CUDA(cudaMemcpyAsync(work.p, P->Lp.p, P->Lp.n * sizeof(double), cudaMemcpyDeviceToDevice, s));
        form_inverses(ctx, P, work, Mtmp);
        Mc = &Mtmp;
    } else if (P->factored) {  // full inverses X^T X from the factored storage
        Mtmp.alloc(P->Mc.n);
        for (int b = 0; b < P->nblocks; ++b) {
            k_factored_to_full<<<4 * ctx->sm_count, 256, 0, s>>>(P->d_nb.p, P->d_ldm.p, P->d_Moff.p, P->Mc.p, Mtmp.p, b);
            count_launch();
        }
        Mc = &Mtmp;
    }
    if (P->ngather > 0) {
        k_mat_blocks<<<dim3(P->ngather, 64), 128, 0, s>>>(P->d_bptr.p, P->d_bdofs.p, P->d_nb.p, P->d_ldm.p,
                                                          P->d_Moff.p, Mc->p, M.a.p, M.ld);
        count_launch();
    }
    if (P->coarse_block >= 0) {
        const int cb = P->coarse_block;
        k_mat_coarse<<<std::min(n, 16 * ctx->sm_count), 256, 0, s>>>(
            n, P->Rr_ptr.p, P->Rr_col.p, P->Rr_val.p, Mc->p + P->h_Moff[cb], P->h_ldm[cb], M.a.p, M.ld);
        count_launch();
    }
    SBG_LAUNCH_CHECK();
    SBG_CUDA(cudaStreamSynchronize(s));
}

// A dense SPD matrix used as the preconditioner M (condition_number(W, M),
// schwarz.hpp:174-183): one inverse-mode block over all DOFs holding M itself.
Prec* prec_from_dense(Ctx* ctx, const DMatrix& Mdense)
{
    cudaStream_t s = ctx->stream;
    auto* P = new Prec;
    try {
        const int n = Mdense.n;
        P->ctx = ctx;
        P->n = n;
        P->mode = kPrecInverse;
        P->nblocks = n > 0 ? 1 : 0;
        P->ngather = P->nblocks;
        if (n > 0) {
            const int T = (n + TB - 1) / TB, ldm = (n + 3) / 4 * 4;
            P->h_nb = {n};
            P->h_T = {T};
            P->h_loc = {0};
            P->h_Poff = {0};
            P->h_Doff = {0};
            P->h_Moff = {0};
            P->h_ldm = {ldm};
            P->Tmax = T;
            P->maxnb = ldm;
            P->apply_bytes = (double)n * n * 8.0;
            P->d_nb.upload(P->h_nb, s);
            P->d_T.upload(P->h_T, s);
            P->d_loc.upload(P->h_loc, s);
            P->d_Moff.upload(P->h_Moff, s);
            P->d_ldm.upload(P->h_ldm, s);
            P->loc.alloc((size_t)T * TB);
            P->locy.alloc((size_t)T * TB);
            SBG_CUDA(cudaMemsetAsync(P->loc.p, 0, P->loc.n * sizeof(double), s));
            SBG_CUDA(cudaMemsetAsync(P->locy.p, 0, P->locy.n * sizeof(double), s));
            std::vector<int> pos(n), bptr{0, n};
            for (int d = 0; d < n; ++d) pos[d] = d;
            P->pos.upload(pos, s);
            P->d_bptr.upload(bptr, s);
            P->d_bdofs.upload(pos, s);
            P->Mc.alloc((size_t)n * ldm);
            SBG_CUDA(cudaMemsetAsync(P->Mc.p, 0, P->Mc.n * sizeof(double), s));
            SBG_CUDA(cudaMemcpy2DAsync(P->Mc.p, ldm * sizeof(double), Mdense.a.p, Mdense.ld * sizeof(double),
                                       n * sizeof(double), n, cudaMemcpyDeviceToDevice, s));
            auto S = std::make_shared<PrecSchedule>();  // apply-only schedule (not cached)
            for (int r = 0; r < n; r += GEMV_ROWS) S->gemv.push_back({0, r});
            S->d_gemv.upload(S->gemv, s);
            P->sched = S;
            SBG_CUDA(cudaStreamSynchronize(s));
        }
    } catch (...) {
        delete P;
        throw;
    }
    return P;
}

void coarse_galerkin(Ctx* ctx, const DMatrix& W, const Prolongation& R, std::vector<double>& H)
{
    cudaStream_t s = ctx->stream;
    const int nc = R.cols;
    H.assign((size_t)nc * nc, 0.0);
    if (nc == 0) return;
    DBuf<int> cp, cr;
    DBuf<double> cv, dH((size_t)nc * nc);
    cp.upload(R.col_ptr, s);
    cr.upload(R.row_idx, s);
    cv.upload(R.val, s);
    coarse_galerkin_device(ctx, W, R.col_ptr, R.row_idx, cp.p, cr.p, cv.p, nc, nc, dH.p);
    SBG_CUDA(cudaMemcpyAsync(H.data(), dH.p, H.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    SBG_CUDA(cudaStreamSynchronize(s));
}

}  // namespace sbg
