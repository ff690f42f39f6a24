// Dense fp64 GEMV (HBM-streaming) and the device-resident PCG loop.
// reference: inc/pcg.hpp:33-116 (the loop), :70 (W*p — the dominant cost).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>

#include <random>

#include "kernels.cuh"
#include "pcg_dev.cuh"
#include "prec_dev.cuh"

namespace sbg {

namespace {

constexpr int kGemvThreads = 256;
constexpr int kGemvCols = 2 * kGemvThreads;  // each thread owns 2 adjacent columns (one 128-bit load per row)
constexpr int kUnroll = 8;

// Column-sum formulation of y = W x for symmetric W (y_j = sum_i W(i,j) x_i):
// every warp streams contiguous 512-byte row segments with 128-bit
// evict-first loads; x is staged in shared memory and read as a broadcast.
// Grid: (column strips of 512, row chunks); partial sums per row chunk are
// reduced in a fixed order by the second pass (deterministic).
__global__ void __launch_bounds__(kGemvThreads) k_gemv_partial(const double* __restrict__ W, int ld, int n,
                                                               const double* __restrict__ x, int rows_per_chunk,
                                                               double* __restrict__ part, const int* done)
{
    pdl_wait();
    if (done && *done) return;
    extern __shared__ double sx[];
    const int r0 = blockIdx.y * rows_per_chunk;
    const int rows = min(n, r0 + rows_per_chunk) - r0;
    for (int i = threadIdx.x; i < rows; i += blockDim.x) sx[i] = x[r0 + i];
    __syncthreads();
    const int c = blockIdx.x * kGemvCols + 2 * threadIdx.x;
    if (c >= ld) return;
    const double* base = W + (size_t)r0 * ld + c;
    double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
    int i = 0;
    for (; i + kUnroll <= rows; i += kUnroll) {
        double2 w[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) w[u] = __ldcs(reinterpret_cast<const double2*>(base + (size_t)(i + u) * ld));
#pragma unroll
        for (int u = 0; u < kUnroll; u += 2) {
            a0 = fma(w[u].x, sx[i + u], a0);
            a1 = fma(w[u].y, sx[i + u], a1);
            b0 = fma(w[u + 1].x, sx[i + u + 1], b0);
            b1 = fma(w[u + 1].y, sx[i + u + 1], b1);
        }
    }
    for (; i < rows; ++i) {
        const double2 w = __ldcs(reinterpret_cast<const double2*>(base + (size_t)i * ld));
        a0 = fma(w.x, sx[i], a0);
        a1 = fma(w.y, sx[i], a1);
    }
    double2 out;
    out.x = a0 + b0;
    out.y = a1 + b1;
    *reinterpret_cast<double2*>(part + (size_t)blockIdx.y * ld + c) = out;
}

__global__ void k_gemv_reduce(const double* __restrict__ part, int chunks, int ld, int n, double* __restrict__ y)
{
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    double s = 0.0;
    for (int c = 0; c < chunks; ++c) s += part[(size_t)c * ld + j];
    y[j] = s;
}

// init: p = z, rz = r.z, r0, history[0] (pcg.hpp:53-67)
__global__ void k_pcg_init(PcgDev* st, const double* __restrict__ r, const double* __restrict__ z,
                           double* __restrict__ p, int n, double* partials, double* hist)
{
    __shared__ double sh[32];
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    double v = 0.0;
    if (j < n) {
        v = r[j] * z[j];
        p[j] = z[j];
    }
    v = block_sum(v, sh);
    if (last_block(v, partials, &st->counter) && threadIdx.x == 0) {
        const double rz = sum_partials(partials, gridDim.x);
        st->counter = 0;
        st->rz = rz;
        if (rz < 0) {
            st->error = 2;
            st->done = 1;
            return;
        }
        st->r0 = sqrt(fmax(rz, 0.0));
        hist[0] = st->r0;
        if (st->r0 == 0.0) {
            st->converged = 1;
            st->done = 1;
        }
        if (st->maxit <= 0) st->done = 1;
    }
}

// Wp = sum of GEMV partials; alpha = rz / p.Wp (pcg.hpp:70-73)
__global__ void k_pcg_alpha(PcgDev* st, const double* __restrict__ part, int chunks, int ld, int n,
                            const double* __restrict__ p, double* __restrict__ Wp, double* partials)
{
    pdl_wait();
    if (st->done) return;
    __shared__ double sh[32];
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    double v = 0.0;
    if (j < n) {
        double s = 0.0;
        for (int c = 0; c < chunks; ++c) s += part[(size_t)c * ld + j];
        Wp[j] = s;
        v = p[j] * s;
    }
    v = block_sum(v, sh);
    if (last_block(v, partials, &st->counter) && threadIdx.x == 0) {
        const double pwp = sum_partials(partials, gridDim.x);
        st->counter = 0;
        st->pwp = pwp;
        if (pwp <= 0) {
            st->error = 1;
            st->done = 1;
            return;
        }
        st->alpha = st->rz / pwp;
    }
}

// x += alpha p ; r -= alpha Wp (pcg.hpp:74-75)
__global__ void k_pcg_update(const PcgDev* st, double* __restrict__ x, double* __restrict__ r,
                             const double* __restrict__ p, const double* __restrict__ Wp, int n)
{
    pdl_wait();
    if (st->done) return;
    const double a = st->alpha;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n) {
        x[j] += a * p[j];
        r[j] -= a * Wp[j];
    }
}

// rz_new = r.z ; history, stopping test, beta (pcg.hpp:76-93)
__global__ void k_pcg_rz(PcgDev* st, const double* __restrict__ r, const double* __restrict__ z, int n,
                         double* partials, double* hist, double* alphas, double* betas)
{
    pdl_wait();
    if (st->done) return;
    __shared__ double sh[32];
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    double v = (j < n) ? r[j] * z[j] : 0.0;
    v = block_sum(v, sh);
    if (last_block(v, partials, &st->counter) && threadIdx.x == 0) {
        const double rz_new = sum_partials(partials, gridDim.x);
        st->counter = 0;
        pcg_finish_rz(st, rz_new, hist, alphas, betas);
    }
}

// e = x - exact, the error of the energy history (pcg.hpp:50-53); `gated`: skip once done
__global__ void k_pcg_err(const PcgDev* st, const double* __restrict__ x, const double* __restrict__ exact,
                          double* __restrict__ e, int n, int gated)
{
    pdl_wait();
    if (gated && st->done) return;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n) e[j] = x[j] - exact[j];
}

// energy[st->it + off] = sqrt(max(0, e . W e)) from the GEMV partials of W e (pcg.hpp:50-53, 59, 82)
__global__ void k_pcg_energy(PcgDev* st, const double* __restrict__ part, int chunks, int ld, int n,
                             const double* __restrict__ e, double* partials, double* energy, int off, int gated)
{
    pdl_wait();
    if (gated && st->done) return;
    __shared__ double sh[32];
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    double v = 0.0;
    if (j < n) {
        double s = 0.0;
        for (int c = 0; c < chunks; ++c) s += part[(size_t)c * ld + j];
        v = e[j] * s;
    }
    v = block_sum(v, sh);
    if (last_block(v, partials, &st->counter) && threadIdx.x == 0) {
        const double ewe = sum_partials(partials, gridDim.x);
        st->counter = 0;
        energy[st->it + off] = sqrt(fmax(0.0, ewe));
    }
}

// device-side loop control of the graph form: the while node runs its body while the
// handle is non-zero
__global__ void k_pcg_gate(const PcgDev* st, cudaGraphConditionalHandle h)
{
    pdl_wait();
    if (threadIdx.x == 0) cudaGraphSetConditional(h, st->done ? 0u : 1u);
}

// p = z + beta p (pcg.hpp:93)
__global__ void k_pcg_p(const PcgDev* st, double* __restrict__ p, const double* __restrict__ z, int n)
{
    pdl_wait();
    if (st->done) return;
    const double b = st->beta;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n) p[j] = z[j] + b * p[j];
}

// Row-per-warp form for matrices up to a few hundred MB: y_i = W_i . x with U
// 128-bit loads in flight per lane and a warp reduction — one launch, no partials.
// The row's last partial round issues its loads together (a row is ~8 dependent
// memory rounds at n = 3969; a segment-at-a-time tail added up to 7 more).  U = 8:
// 16 was slower (fewer resident CTAs), 4/6/10/12 no better.
constexpr int kRowsPerCta = 8;
constexpr int kSymvMinN = 2048;
// row . x for one warp (the row's lanes), U 128-bit loads in flight per lane; KEEP: default
// caching (W held in L2 by the PCG's access-policy window) instead of evict-first
template <int U, bool KEEP>
__device__ __forceinline__ double warp_row_dot(const double* __restrict__ Wrow, int ld, const double* __restrict__ x)
{
    const int lane = threadIdx.x & 31;
    const double2* w = reinterpret_cast<const double2*>(Wrow);
    const double2* x2 = reinterpret_cast<const double2*>(x);
    const int half = ld >> 1;  // the padding of W and x is zero
    auto ld2 = [&](const double2* q) { return KEEP ? __ldg(q) : __ldcs(q); };
    double s[U];
#pragma unroll
    for (int u = 0; u < U; ++u) s[u] = 0.0;
    int c = lane;
    for (; c + (U - 1) * 32 < half; c += U * 32) {
        double2 a[U];
#pragma unroll
        for (int u = 0; u < U; ++u) a[u] = ld2(w + c + 32 * u);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const double2 xv = __ldg(x2 + c + 32 * u);
            s[u] = fma(a[u].x, xv.x, fma(a[u].y, xv.y, s[u]));
        }
    }
    double2 a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) a[u] = c + 32 * u < half ? ld2(w + c + 32 * u) : make_double2(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < U; ++u)
        if (c + 32 * u < half) {
            const double2 xv = __ldg(x2 + c + 32 * u);
            s[u] = fma(a[u].x, xv.x, fma(a[u].y, xv.y, s[u]));
        }
    double v = 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) v += s[u];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Wp = W p with alpha = rz / p.Wp fused in (the rows form inside PCG, pcg.hpp:70-73): each
// warp's row also contributes p_row (W p)_row to the block's partial, and the last block
// finishes the reduction in the fixed block order (deterministic)
template <bool KEEP>
__global__ void __launch_bounds__(256) k_gemv_rows_alpha(PcgDev* st, const double* __restrict__ W, int ld, int n,
                                                         const double* __restrict__ p, double* __restrict__ Wp,
                                                         double* partials)
{
    pdl_wait();
    if (st->done) return;
    __shared__ double sh[32];
    const int row = blockIdx.x * kRowsPerCta + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    double v = 0.0;
    if (row < n) {
        const double y = warp_row_dot<8, KEEP>(W + (size_t)row * ld, ld, p);
        if (lane == 0) {
            Wp[row] = y;
            v = p[row] * y;
        }
    }
    v = block_sum(v, sh);
    if (last_block(v, partials, &st->counter)) {
        const double pwp = sum_partials_block(partials, gridDim.x, sh);
        if (threadIdx.x != 0) return;
        st->counter = 0;
        st->pwp = pwp;
        if (pwp <= 0) {
            st->error = 1;
            st->done = 1;
            return;
        }
        st->alpha = st->rz / pwp;
    }
}

// alpha from a complete W p (the row-panel PCG after its exchange) with exactly the
// reduction tree of k_gemv_rows_alpha (8 rows per block, lane 0 of each warp), so the
// row-panel PCG stays bitwise equal to pcg; Wp <- y
__global__ void __launch_bounds__(256) k_pcg_alpha8(PcgDev* st, const double* __restrict__ y, int n,
                                                    const double* __restrict__ p, double* __restrict__ Wp,
                                                    double* partials)
{
    pdl_wait();
    if (st->done) return;
    __shared__ double sh[32];
    const int row = blockIdx.x * kRowsPerCta + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    double v = 0.0;
    if (row < n && lane == 0) {
        const double yv = y[row];
        Wp[row] = yv;
        v = p[row] * yv;
    }
    v = block_sum(v, sh);
    if (last_block(v, partials, &st->counter)) {
        const double pwp = sum_partials_block(partials, gridDim.x, sh);
        if (threadIdx.x != 0) return;
        st->counter = 0;
        st->pwp = pwp;
        if (pwp <= 0) {
            st->error = 1;
            st->done = 1;
            return;
        }
        st->alpha = st->rz / pwp;
    }
}

template <int U>
__global__ void __launch_bounds__(256) k_gemv_rows(const double* __restrict__ W, int ld, int n,
                                                   const double* __restrict__ x, double* __restrict__ y,
                                                   const int* done)
{
    pdl_wait();
    if (done && *done) return;
    const int row = blockIdx.x * kRowsPerCta + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (row >= n) return;
    const double2* w = reinterpret_cast<const double2*>(W + (size_t)row * ld);
    const double2* x2 = reinterpret_cast<const double2*>(x);
    const int half = ld >> 1;  // the padding of W and x is zero
    double s[U];
#pragma unroll
    for (int u = 0; u < U; ++u) s[u] = 0.0;
    int c = lane;
    for (; c + (U - 1) * 32 < half; c += U * 32) {
        double2 a[U];
#pragma unroll
        for (int u = 0; u < U; ++u) a[u] = __ldcs(w + c + 32 * u);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const double2 xv = __ldg(x2 + c + 32 * u);
            s[u] = fma(a[u].x, xv.x, fma(a[u].y, xv.y, s[u]));
        }
    }
    // remainder: up to U - 1 more 512-byte segments, loads issued together
    double2 a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) a[u] = c + 32 * u < half ? __ldcs(w + c + 32 * u) : make_double2(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < U; ++u)
        if (c + 32 * u < half) {
            const double2 xv = __ldg(x2 + c + 32 * u);
            s[u] = fma(a[u].x, xv.x, fma(a[u].y, xv.y, s[u]));
        }
    double v = 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) v += s[u];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) y[row] = v;
}
// ---------------------------------------------------------------- symmetric form
// W symmetric: y = W x from the upper triangle alone (half the bytes of the full forms).
// Tile (I, J) covers rows [I H, I H + H) and columns [J C, J C + C) right of column I H; its
// row sums W_IJ x_J go to rowpart[tile], and, right of the strip's own diagonal block, its
// column sums W_IJ^T x_I go to colpart[I][cols].  A warp owns rows warp, warp + 8, ...; a
// lane owns the column pairs 2 lane + 64 k, loads them with 128-bit evict-first loads (two
// rows per pass: 2 C / 64 loads in flight) and keeps the column sums in registers until the
// 8 warps combine them in shared memory in a fixed order.
// PF (inside PCG): the vector is p = z + beta p_old formed on the fly (pcg.hpp:93; p itself is
// rewritten by k_symv_alpha once every tile has read p_old), so no separate p-update launch
template <int H, int C, bool KEEP, bool PF>
__device__ __forceinline__ void symv_tile_body(int tile, const double* __restrict__ W, int ld, int n,
                                               const double* __restrict__ x, const int2* __restrict__ tiles,
                                               double* __restrict__ rowpart, double* __restrict__ colpart,
                                               const double* __restrict__ z, double beta, double (*red)[C])
{
    static_assert(C % 64 == 0 && H % 16 == 0 && C % H == 0, "tile shape");
    constexpr int KC = C / 64, RW = H / 8;
    const int2 t = tiles[tile];
    const int r0 = t.x * H, c0 = t.y * C;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    auto xv = [&](int i) { return PF ? fma(beta, __ldg(x + i), __ldg(z + i)) : __ldg(x + i); };
    double2 xj[KC], ca[KC];
    bool in[KC], off[KC];
#pragma unroll
    for (int k = 0; k < KC; ++k) {
        const int c = c0 + 2 * lane + 64 * k;
        in[k] = c >= r0 && c < ld;
        off[k] = c >= r0 + H && c < ld;
        xj[k] = in[k] ? make_double2(xv(c), xv(c + 1)) : make_double2(0.0, 0.0);
        ca[k] = make_double2(0.0, 0.0);
    }
    const double* wbase = W + c0 + 2 * lane;
    constexpr int RP = 4;  // rows per pass: RP * KC 128-bit loads in flight per lane
    static_assert(RW % RP == 0, "rows per warp");
#pragma unroll 1
    for (int j = 0; j < RW; j += RP) {
        double2 a[RP][KC];
        double xr[RP];
#pragma unroll
        for (int u = 0; u < RP; ++u) {
            const int r = r0 + warp + 8 * (j + u);
            const bool v = r < n;
#pragma unroll
            for (int k = 0; k < KC; ++k) {
                const double2* q = reinterpret_cast<const double2*>(wbase + (size_t)r * ld + 64 * k);
                a[u][k] = v && in[k] ? (KEEP ? __ldg(q) : __ldcs(q)) : make_double2(0.0, 0.0);
            }
            xr[u] = v ? xv(r) : 0.0;
        }
        double sr[RP];
#pragma unroll
        for (int u = 0; u < RP; ++u) {
            double s0 = 0.0, s1 = 0.0;
#pragma unroll
            for (int k = 0; k < KC; ++k) {
                s0 = fma(a[u][k].x, xj[k].x, s0);
                s1 = fma(a[u][k].y, xj[k].y, s1);
                if (off[k]) {
                    ca[k].x = fma(a[u][k].x, xr[u], ca[k].x);
                    ca[k].y = fma(a[u][k].y, xr[u], ca[k].y);
                }
            }
            sr[u] = s0 + s1;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int u = 0; u < RP; ++u) sr[u] += __shfl_xor_sync(0xffffffffu, sr[u], o);
        if (lane == 0)
#pragma unroll
            for (int u = 0; u < RP; ++u) {
                const int r = r0 + warp + 8 * (j + u);
                if (r < n) rowpart[(size_t)tile * H + (r - r0)] = sr[u];
            }
    }
#pragma unroll
    for (int k = 0; k < KC; ++k) {
        red[warp][2 * lane + 64 * k] = ca[k].x;
        red[warp][2 * lane + 64 * k + 1] = ca[k].y;
    }
    __syncthreads();
    for (int cc = threadIdx.x; cc < C; cc += blockDim.x) {
        const int c = c0 + cc;
        if (c < r0 + H || c >= ld) continue;
        double v = red[0][cc];
#pragma unroll
        for (int w = 1; w < 8; ++w) v += red[w][cc];
        colpart[(size_t)t.x * ld + c] = v;
    }
}

template <int H, int C, bool KEEP, bool PF>
__global__ void __launch_bounds__(256, 2) k_symv_tiles(const double* __restrict__ W, int ld, int n,
                                                      const double* __restrict__ x, const int2* __restrict__ tiles,
                                                      double* __restrict__ rowpart, double* __restrict__ colpart,
                                                      const int* done, const double* __restrict__ z,
                                                      const PcgDev* st)
{
    __shared__ double red[8][C];
    pdl_wait();
    if (done && *done) return;
    symv_tile_body<H, C, KEEP, PF>(blockIdx.x, W, ld, n, x, tiles, rowpart, colpart, z, PF ? st->beta : 0.0, red);
}

// (W x)_i for the 32 entries i = 32 blockIdx.x + lane of a 256-thread block: group g (warp g)
// sums the strip's row partials k = g, g + 8, ... and the column partials of the strips
// q = g, g + 8, ... above it; warp 0 adds the 8 group sums in group order (deterministic).
// Returns the entry in warp 0 (0 elsewhere).
__device__ __forceinline__ double symv_entry_block(int vb, int n, int H, int ld, const int* __restrict__ tbase,
                                                   const double* __restrict__ rowpart,
                                                   const double* __restrict__ colpart, double (*sh)[33])
{
    const int g = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i = vb * 32 + lane;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    if (i < n) {
        const int I = i / H, ri = i - I * H;
        const int k1 = tbase[I + 1];
        for (int k = tbase[I] + g; k < k1; k += 8) s0 += rowpart[(size_t)k * H + ri];
        const double* cp = colpart + i;
        int q = g;
        for (; q + 24 < I; q += 32) {  // four loads in flight per thread
            s0 += cp[(size_t)q * ld];
            s1 += cp[(size_t)(q + 8) * ld];
            s2 += cp[(size_t)(q + 16) * ld];
            s3 += cp[(size_t)(q + 24) * ld];
        }
        for (; q < I; q += 8) s0 += cp[(size_t)q * ld];
    }
    sh[g][lane] = (s0 + s1) + (s2 + s3);
    __syncthreads();
    double y = 0.0;
    if (g == 0) {
#pragma unroll
        for (int w = 0; w < 8; ++w) y += sh[w][lane];
    }
    return y;
}

__global__ void __launch_bounds__(256) k_symv_reduce(int n, int H, int ld, const int* __restrict__ tbase,
                                                     const double* __restrict__ rowpart,
                                                     const double* __restrict__ colpart, double* __restrict__ y,
                                                     const int* done)
{
    __shared__ double sh[8][33];
    pdl_wait();
    if (done && *done) return;
    const double v = symv_entry_block(blockIdx.x, n, H, ld, tbase, rowpart, colpart, sh);
    const int i = blockIdx.x * 32 + threadIdx.x;
    if (threadIdx.x < 32 && i < n) y[i] = v;
}

// Wp from the symmetric form's partials, p = z + beta p (the tiles formed the same values on
// the fly), alpha = rz / p.Wp (pcg.hpp:70-73, 93)
__global__ void __launch_bounds__(256) k_symv_alpha(PcgDev* st, int n, int H, int ld, const int* __restrict__ tbase,
                                                    const double* __restrict__ rowpart,
                                                    const double* __restrict__ colpart, double* __restrict__ p,
                                                    const double* __restrict__ z, double* __restrict__ Wp,
                                                    double* partials)
{
    __shared__ double sh[8][33];
    __shared__ double red[32];
    pdl_wait();
    if (st->done) return;
    const double y = symv_entry_block(blockIdx.x, n, H, ld, tbase, rowpart, colpart, sh);
    const int i = blockIdx.x * 32 + threadIdx.x;
    double v = 0.0;
    if (threadIdx.x < 32 && i < n) {
        const double pn = fma(st->beta, p[i], z[i]);
        p[i] = pn;
        Wp[i] = y;
        v = pn * y;
    }
    v = block_sum(v, red);
    if (last_block(v, partials, &st->counter)) {
        const double pwp = sum_partials_block(partials, gridDim.x, red);
        if (threadIdx.x != 0) return;
        st->counter = 0;
        st->pwp = pwp;
        if (pwp <= 0) {
            st->error = 1;
            st->done = 1;
            return;
        }
        st->alpha = st->rz / pwp;
    }
}

// ---------------------------------------------------------------- persistent PCG
// The whole PCG loop (pcg.hpp:69-93) as one cooperative kernel for systems whose symmetric W,
// block inverses and vectors stay in L2 (n <= kPersistMaxN): every CTA runs the iterations,
// with a grid barrier between the phases — (1) the symmetric-form tiles of W p (p = z + beta p
// formed on the fly), (2) Wp, p and p.Wp, (3) the update and gather of the fused apply,
// (4) the block-inverse GEMV, (5) the scatter and r.z — instead of five launches per iteration.
// Every CTA sums the same per-CTA partials in the same order, so alpha, beta and the stopping
// decision are computed identically everywhere without a further barrier (deterministic).
constexpr int kPersistMaxN = 8000;
constexpr int kHistPre = 256;  // history entries returned with the state (more: a second copy)

// grid barrier among the co-resident CTAs of a cooperative launch: the k-th barrier waits
// for k * gridDim.x arrivals on a counter zeroed before the launch
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned& target)
{
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(bar, 1u);
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
        } while (v < target);
        __threadfence();
    }
    __syncthreads();
}

struct PcgPersistArgs {
    PcgDev* st;
    const double* W;
    int ld, n;
    double *x, *r, *rn, *p, *Wp, *z;
    const int2* tiles;
    int ntiles;
    const int* tbase;
    double *rowpart, *colpart;
    PrecView V;
    double *hist, *alphas, *betas;
    double* part;  // 2 x gridDim.x per-CTA partial sums
    unsigned* bar;
    unsigned long long* trace;  // SBG_PCG_TRACE: CTA 0's phase timestamps (globaltimer, ns), 8 per iteration
};

__device__ __forceinline__ void trace_mark(unsigned long long* trace, int it, int k)
{
    if (trace && blockIdx.x == 0 && threadIdx.x == 0 && it < 64) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        trace[8 * it + k] = t;
    }
}

// the fixed-order sum of the per-CTA partials, in every thread of every CTA
__device__ __forceinline__ double grid_total(const double* part, int count, double* sred, double* bcast)
{
    const double t = sum_partials_block(part, count, sred);
    if (threadIdx.x == 0) *bcast = t;
    __syncthreads();
    const double v = *bcast;
    __syncthreads();
    return v;
}

__global__ void __launch_bounds__(256, 2) k_pcg_persistent(PcgPersistArgs A)
{
    __shared__ double red[8][256];
    __shared__ double sh33[8][33];
    __shared__ double sred[32];
    __shared__ double bcast;
    unsigned target = 0;
    PcgDev* st = A.st;
    const PrecView& V = A.V;
    const int G = gridDim.x, nvb = (A.n + 31) / 32;
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    // loop state, identical in every CTA
    double rz = 0.0, beta = 0.0, alpha = 0.0, r0 = 0.0;
    const double tol = st->tol;
    int it = st->it, done = st->done, converged = st->converged, error = st->error;
    const int maxit = st->maxit;
    {
        // initial apply z = M r and r.z (pcg.hpp:45-67; k_pcg_init): the fused phases with
        // alpha = 0 (x, p and Wp are zero: rn = r, x unchanged); p = z + 0 p forms in phase (1)
        for (int vb = blockIdx.x; vb < V.dof_blocks + V.nc; vb += G) {
            prec_gather_upd_body(vb, 0.0, A.x, A.r, A.rn, A.p, A.Wp, A.n, V.pos, V.loc, V.Rc_ptr, V.Rc_row, V.Rc_val,
                                 V.nc, V.loc_c, V.dof_blocks, &red[0][0]);
            __syncthreads();
        }
        grid_barrier(A.bar, target);
        for (int t = blockIdx.x; t < V.ntasks; t += G)
            block_gemv_body<true>(V.tasks[t], V.nbv, V.ldmv, V.locv, V.Moff, V.Mc, V.loc, V.locy);
        grid_barrier(A.bar, target);
        double acc = 0.0;
        for (int vb = blockIdx.x; vb < V.dof_blocks; vb += G) {
            double v = prec_scatter_body(vb, V.locy, V.pos, A.n, V.Rr_ptr, V.Rr_col, V.Rr_val, V.y_c, A.z, A.r, A.rn);
            v = block_sum(v, sred);
            if (threadIdx.x == 0) acc += v;
            __syncthreads();
        }
        if (threadIdx.x == 0) A.part[G + blockIdx.x] = acc;
        grid_barrier(A.bar, target);
        rz = grid_total(A.part + G, G, sred, &bcast);
        beta = 0.0;
        if (rz < 0) {
            error = 2;
            done = 1;
        } else {
            const double rr = sqrt(fmax(rz, 0.0));
            if (lead) {
                st->r0 = rr;
                A.hist[0] = rr;
            }
            r0 = rr;
            if (rr == 0.0) {
                converged = 1;
                done = 1;
            }
            if (maxit <= 0) done = 1;
        }
    }
    while (!done) {
        trace_mark(A.trace, it, 0);
        // (1) W p from the upper triangle
        for (int t = blockIdx.x; t < A.ntiles; t += G) {
            symv_tile_body<64, 256, true, true>(t, A.W, A.ld, A.n, A.p, A.tiles, A.rowpart, A.colpart, A.z, beta, red);
            __syncthreads();
        }
        trace_mark(A.trace, it, 1);
        grid_barrier(A.bar, target);
        trace_mark(A.trace, it, 2);
        // (2) Wp, p = z + beta p, p.Wp
        double acc = 0.0;
        for (int vb = blockIdx.x; vb < nvb; vb += G) {
            const double y = symv_entry_block(vb, A.n, 64, A.ld, A.tbase, A.rowpart, A.colpart, sh33);
            const int i = vb * 32 + threadIdx.x;
            double v = 0.0;
            if (threadIdx.x < 32 && i < A.n) {
                const double pn = fma(beta, A.p[i], A.z[i]);
                A.p[i] = pn;
                A.Wp[i] = y;
                v = pn * y;
            }
            v = block_sum(v, sred);
            if (threadIdx.x == 0) acc += v;
            __syncthreads();
        }
        if (threadIdx.x == 0) A.part[blockIdx.x] = acc;
        grid_barrier(A.bar, target);
        const double pwp = grid_total(A.part, G, sred, &bcast);
        if (pwp <= 0) {  // W not positive definite (pcg.hpp:72)
            error = 1;
            done = 1;
            break;
        }
        alpha = rz / pwp;
        trace_mark(A.trace, it, 3);
        // (3) x += alpha p, r - alpha Wp gathered into the blocks, coarse restriction
        for (int vb = blockIdx.x; vb < V.dof_blocks + V.nc; vb += G) {
            prec_gather_upd_body(vb, alpha, A.x, A.r, A.rn, A.p, A.Wp, A.n, V.pos, V.loc, V.Rc_ptr, V.Rc_row, V.Rc_val,
                                 V.nc, V.loc_c, V.dof_blocks, &red[0][0]);
            __syncthreads();
        }
        grid_barrier(A.bar, target);
        trace_mark(A.trace, it, 4);
        // (4) block inverses (schwarz.hpp:121-140)
        for (int t = blockIdx.x; t < V.ntasks; t += G)
            block_gemv_body<true>(V.tasks[t], V.nbv, V.ldmv, V.locv, V.Moff, V.Mc, V.loc, V.locy);
        grid_barrier(A.bar, target);
        trace_mark(A.trace, it, 5);
        // (5) z, r, r.z
        acc = 0.0;
        for (int vb = blockIdx.x; vb < V.dof_blocks; vb += G) {
            double v = prec_scatter_body(vb, V.locy, V.pos, A.n, V.Rr_ptr, V.Rr_col, V.Rr_val, V.y_c, A.z, A.r, A.rn);
            v = block_sum(v, sred);
            if (threadIdx.x == 0) acc += v;
            __syncthreads();
        }
        if (threadIdx.x == 0) A.part[G + blockIdx.x] = acc;
        grid_barrier(A.bar, target);
        const double rz_new = grid_total(A.part + G, G, sred, &bcast);
        trace_mark(A.trace, it, 6);
        // history, beta, stopping test (pcg_finish_rz, pcg.hpp:76-93)
        if (rz_new < 0) {
            error = 2;
            done = 1;
            break;
        }
        if (lead) A.alphas[it] = alpha;
        ++it;
        const double res = sqrt(fmax(rz_new, 0.0));
        beta = rz_new / rz;
        if (lead) {
            A.hist[it] = res;
            A.betas[it - 1] = beta;
        }
        rz = rz_new;
        if (res <= tol * r0) {
            converged = 1;
            done = 1;
        } else if (it >= maxit) {
            done = 1;
        }
    }
    if (lead) {
        st->it = it;
        st->rz = rz;
        st->alpha = alpha;
        st->beta = beta;
        st->done = done;
        st->converged = converged;
        st->error = error;
    }
}

template <typename... A>
void launch_gemv_rows(bool pdl, cudaStream_t s, int n, A... args)
{
    const dim3 grid((n + kRowsPerCta - 1) / kRowsPerCta), block(256);
    if (pdl)
        launch_pdl(k_gemv_rows<8>, grid, block, 0, s, args...);
    else
        k_gemv_rows<8><<<grid, block, 0, s>>>(args...);
}
}  // namespace

// smallest n that takes the symmetric form (below it the one-launch row form wins on latency)
static int symv_min_n()
{
    static const int v = [] {
        const char* e = getenv("SBG_SYMV_MIN_N");
        return e ? atoi(e) : kSymvMinN;
    }();
    return v;
}

static void symv_plan(Ctx* ctx, int n, int ld, GemvPlan& plan)
{
    plan.sym = true;
    plan.H = n <= 8000 ? 64 : 128;
    plan.C = 256;  // 512 columns per tile needs more than the 128 registers of 2 CTAs/SM
    plan.nstrips = (n + plan.H - 1) / plan.H;
    const int nchunks = (ld + plan.C - 1) / plan.C;
    std::vector<int2> tiles;
    std::vector<int> tbase(plan.nstrips + 1, 0);
    for (int I = 0; I < plan.nstrips; ++I) {
        tbase[I] = (int)tiles.size();
        for (int J = I * plan.H / plan.C; J < nchunks; ++J) tiles.push_back(make_int2(I, J));
    }
    tbase[plan.nstrips] = (int)tiles.size();
    plan.ntiles = (int)tiles.size();
    plan.tiles.alloc(tiles.size());
    plan.tbase.alloc(tbase.size());
    plan.rowpart.alloc((size_t)plan.ntiles * plan.H);
    plan.colpart.alloc((size_t)plan.nstrips * ld);
    // pageable sources: the copies are staged before the calls return
    SBG_CUDA(cudaMemcpyAsync(plan.tiles.p, tiles.data(), tiles.size() * sizeof(int2), cudaMemcpyHostToDevice,
                             ctx->stream));
    SBG_CUDA(cudaMemcpyAsync(plan.tbase.p, tbase.data(), tbase.size() * sizeof(int), cudaMemcpyHostToDevice,
                             ctx->stream));
    SBG_CUDA(cudaStreamSynchronize(ctx->stream));
}

// keep: default-cached loads (W held in L2 by the PCG's access-policy window)
// z, st (PCG): the vector is z + st->beta x (x = p), see k_symv_tiles
static void symv_tiles_launch(Ctx* ctx, const DMatrix& W, const GemvPlan& plan, const double* x, const int* done,
                              bool keep = false, const double* z = nullptr, const PcgDev* st = nullptr)
{
    const dim3 grid(plan.ntiles), block(256);
    auto go = [&](auto kern) {
        launch_pdl(kern, grid, block, 0, ctx->stream, (const double*)W.a.p, W.ld, W.n, x, (const int2*)plan.tiles.p,
                   plan.rowpart.p, plan.colpart.p, done, z, st);
    };
    const bool pf = z != nullptr;
    if (plan.H == 64) {
        if (pf) keep ? go(k_symv_tiles<64, 256, true, true>) : go(k_symv_tiles<64, 256, false, true>);
        else keep ? go(k_symv_tiles<64, 256, true, false>) : go(k_symv_tiles<64, 256, false, false>);
    } else {
        if (pf) keep ? go(k_symv_tiles<128, 256, true, true>) : go(k_symv_tiles<128, 256, false, true>);
        else keep ? go(k_symv_tiles<128, 256, true, false>) : go(k_symv_tiles<128, 256, false, false>);
    }
    ::sbg::count_launch();
    SBG_LAUNCH_CHECK();
}

static void symv_reduce_launch(Ctx* ctx, const DMatrix& W, const GemvPlan& plan, double* y, const int* done)
{
    launch_pdl(k_symv_reduce, dim3((W.n + 31) / 32), dim3(256), 0, ctx->stream, W.n, plan.H, W.ld,
               (const int*)plan.tbase.p, (const double*)plan.rowpart.p, (const double*)plan.colpart.p, y, done);
    ::sbg::count_launch();
    SBG_LAUNCH_CHECK();
}

// algorithmic DRAM bytes of one matvec with this plan: the matrix entries it reads, x, y and
// (symmetric form) its partial sums written and read back once
double gemv_bytes(const GemvPlan& plan)
{
    const double n = plan.n, ld = plan.ld, e = sizeof(double);
    if (!plan.sym) return e * n * n + 2 * e * n;  // (the zero padding of each row is not counted)
    double w = 0.0, colp = 0.0;
    for (int I = 0; I < plan.nstrips; ++I) {
        const double rows = std::min(plan.H, plan.n - I * plan.H);
        w += rows * (n - (double)I * plan.H);
        colp += std::max(0.0, ld - (double)(I + 1) * plan.H);
    }
    const double rowp = (double)plan.ntiles * plan.H;
    return e * w + 2 * e * n + 2 * e * (rowp + colp);
}

void gemv_plan(Ctx* ctx, int n, int ld, GemvPlan& plan)
{
    plan.n = n;
    plan.ld = ld;
    if (ctx->matvec_form == 0 && n >= symv_min_n()) {
        symv_plan(ctx, n, ld, plan);
        return;
    }
    // measured crossover (B200, L2 flushed): rows form faster at n = 3969 (27.3 vs 35.9 us)
    // and n = 6721 (67.2 vs 68.6 us), even at 12097 (182 us both), column-sum form faster at
    // 25281 (731 vs 805 us)
    constexpr int kGemvRowsMaxN = 8000;
    if (n <= kGemvRowsMaxN) {
        plan.rows = true;
        plan.strips = 1;
        plan.chunks = 1;
        plan.rows_per_chunk = n;
        plan.part.alloc((size_t)ld);
        SBG_CUDA(cudaMemsetAsync(plan.part.p, 0, (size_t)ld * sizeof(double), ctx->stream));
        return;
    }
    plan.strips = std::max(1, (ld + kGemvCols - 1) / kGemvCols);
    const int target = 4 * ctx->sm_count;
    int chunks = std::max(1, (target + plan.strips - 1) / plan.strips);
    chunks = std::min(chunks, std::max(1, n / 32));
    // x of a row chunk is staged in shared memory: keep it within the 48 KB default
    constexpr int kMaxChunkRows = (48 << 10) / (int)sizeof(double) - 8;
    chunks = std::max(chunks, (n + kMaxChunkRows - 1) / kMaxChunkRows);
    plan.rows_per_chunk = std::max(8, ((n + chunks - 1) / chunks + 7) / 8 * 8);
    plan.chunks = std::max(1, (n + plan.rows_per_chunk - 1) / plan.rows_per_chunk);
    plan.part.alloc((size_t)plan.chunks * ld);
}

static void gemv_partial_launch(Ctx* ctx, const DMatrix& W, GemvPlan& plan, const double* x, const int* done)
{
    if (plan.rows) {
        launch_gemv_rows(true, ctx->stream, W.n, (const double*)W.a.p, W.ld, W.n, x, plan.part.p, done);
        ::sbg::count_launch();
        SBG_LAUNCH_CHECK();
        return;
    }
    const size_t smem = (size_t)plan.rows_per_chunk * sizeof(double);
    launch_pdl(k_gemv_partial, dim3(plan.strips, plan.chunks), dim3(kGemvThreads), smem, ctx->stream, W.a.p, W.ld, W.n,
               x, plan.rows_per_chunk, plan.part.p, done);
    ::sbg::count_launch();
    SBG_LAUNCH_CHECK();
}

// "gemv_f64" times the whole matvec (partials + their reduction); inside PCG the
// reduction is fused into k_pcg_alpha and the scope covers the partial pass
void gemv_rows_range(Ctx* ctx, const DMatrix& W, const double* x, double* y, int lo, int hi)
{
    if (lo < 0 || hi > W.n || lo > hi) throw ValidationError("matvec rows: range outside the matrix");
    if (hi == lo) return;
    launch_gemv_rows(false, ctx->stream, hi - lo, (const double*)W.a.p + (size_t)lo * W.ld, W.ld, hi - lo, x, y + lo,
                     (const int*)nullptr);
    ::sbg::count_launch();
    SBG_LAUNCH_CHECK();
}

void gemv(Ctx* ctx, const DMatrix& W, GemvPlan& plan, const double* x, double* y)
{
    if (W.n == 0) return;
    TimedScope ts(ctx, "gemv_f64");
    if (plan.sym) {
        symv_tiles_launch(ctx, W, plan, x, nullptr);
        symv_reduce_launch(ctx, W, plan, y, nullptr);
        return;
    }
    if (plan.rows) {
        launch_gemv_rows(false, ctx->stream, W.n, (const double*)W.a.p, W.ld, W.n, x, y, (const int*)nullptr);
        ::sbg::count_launch();
        SBG_LAUNCH_CHECK();
        return;
    }
    gemv_partial_launch(ctx, W, plan, x, nullptr);
    k_gemv_reduce<<<(W.n + 255) / 256, 256, 0, ctx->stream>>>(plan.part.p, plan.chunks, W.ld, W.n, y); ::sbg::count_launch();
    SBG_LAUNCH_CHECK();
}

// Symmetric tridiagonal extreme eigenvalues by Sturm bisection (replaces the
// dense eigensolve on the Lanczos matrix, pcg.hpp:96-113).  The CG coefficients
// give the Lanczos matrix T: T_jj = 1/a_j + b_{j-1}/a_{j-1}, T_j,j+1 = sqrt(b_j)/a_j.
void lanczos_extremes(const std::vector<double>& alphas, const std::vector<double>& betas, double& lmin, double& lmax)
{
    const int k = (int)alphas.size();
    if (k == 0) {
        lmin = lmax = 0.0;
        return;
    }
    std::vector<double> d(k), e(k > 1 ? k - 1 : 0);
    for (int i = 0; i < k; ++i) {
        d[i] = 1.0 / alphas[i];
        if (i > 0) d[i] += betas[i - 1] / alphas[i - 1];
        if (i + 1 < k) e[i] = std::sqrt(std::max(betas[i], 0.0)) / alphas[i];
    }
    double lo = 1e300, hi = -1e300;
    for (int i = 0; i < k; ++i) {
        const double rad = (i > 0 ? std::abs(e[i - 1]) : 0.0) + (i + 1 < k ? std::abs(e[i]) : 0.0);
        lo = std::min(lo, d[i] - rad);
        hi = std::max(hi, d[i] + rad);
    }
    auto count_below = [&](double x) {
        int c = 0;
        double q = 1.0;
        for (int i = 0; i < k; ++i) {
            q = d[i] - x - (i == 0 ? 0.0 : e[i - 1] * e[i - 1] / q);
            if (q == 0.0) q = -1e-300;
            if (q < 0) ++c;
        }
        return c;
    };
    auto kth = [&](int idx) {
        double a = lo, b = hi;
        for (int it = 0; it < 200; ++it) {
            const double mid = 0.5 * (a + b);
            if (mid <= a || mid >= b) break;
            if (count_below(mid) > idx)
                b = mid;
            else
                a = mid;
        }
        return 0.5 * (a + b);
    };
    lmin = kth(0);
    lmax = kth(k - 1);
}

double lanczos_kappa(const std::vector<double>& alphas, const std::vector<double>& betas)
{
    if (alphas.empty()) return 1.0;
    double lmin, lmax;
    lanczos_extremes(alphas, betas, lmin, lmax);
    const double kappa = lmin > 0 ? lmax / lmin : 1.0;
    return kappa < 1.0 ? 1.0 : kappa;
}

// Device workspace of one PCG size, cached on the context (no allocation or
// pinned-memory registration per solve).
struct PcgWork {
    int ld = 0, cap = 0, form = 0;
    DBuf<double> buf, partials, hist, alphas, betas, xbuf;  // xbuf: row-panel exchange buffer (ld)
    DBuf<double> ebuf, energy;  // energy history: e and exact (2 ld), per-iteration values (cap)
    DBuf<PcgDev> st;
    GemvPlan plan;
    GemvPlan splan;             // symmetric-form plan of the persistent kernel (any n)
    DBuf<double> ppart;         // its per-CTA partials
    DBuf<unsigned> bar;         // its grid-barrier counter
    DBuf<unsigned long long> trace;  // SBG_PCG_TRACE phase timestamps
    PcgDev* hs = nullptr;
    PcgDev* hs0 = nullptr;  // page-locked initial state record
    double* hh = nullptr;  // page-locked: the first kHistPre history, alpha and beta entries
    double* hx = nullptr;  // page-locked right-hand side / solution staging (ld)
    // the whole iteration loop as one graph (a device-side while node), per (W, prec)
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    const void* gW = nullptr;
    unsigned long long gP = 0;  // preconditioner uid (addresses are reused after a free)
    int kernels_per_iter = 0;
    bool body_gate = true;  // a gate kernel ends each iteration (else its last kernel sets the handle)
    void drop_graph()
    {
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
        exec = nullptr;
        graph = nullptr;
        gW = nullptr;
        gP = 0;
    }
    ~PcgWork()
    {
        drop_graph();
        if (hs) cudaFreeHost(hs);
        if (hh) cudaFreeHost(hh);
        if (hs0) cudaFreeHost(hs0);
        if (hx) cudaFreeHost(hx);
    }
};

static PcgWork& pcg_work(Ctx* ctx, const DMatrix& W, int maxit)
{
    auto* w = static_cast<PcgWork*>(ctx->pcg_ws.get());
    if (!w || w->ld != W.ld || w->plan.n != W.n || w->cap < maxit + 2 || w->form != ctx->matvec_form) {
        auto fresh = std::make_shared<PcgWork>();
        fresh->ld = W.ld;
        fresh->form = ctx->matvec_form;
        fresh->cap = std::max(maxit + 2, 128);
        fresh->buf.alloc(6 * (size_t)W.ld);
        fresh->partials.alloc(std::max((W.n + kRowsPerCta - 1) / kRowsPerCta, 1));  // one per block: the 8-row blocks of the rows form are the most
        fresh->hist.alloc(fresh->cap);
        fresh->alphas.alloc(fresh->cap);
        fresh->betas.alloc(fresh->cap);
        fresh->st.alloc(1);
        fresh->xbuf.alloc((size_t)W.ld);
        SBG_CUDA(cudaMemsetAsync(fresh->xbuf.p, 0, (size_t)W.ld * sizeof(double), ctx->stream));
        gemv_plan(ctx, W.n, W.ld, fresh->plan);
        SBG_CUDA(cudaMallocHost(&fresh->hs, sizeof(PcgDev)));
        SBG_CUDA(cudaMallocHost(&fresh->hh, 3 * kHistPre * sizeof(double)));
        SBG_CUDA(cudaMallocHost(&fresh->hs0, sizeof(PcgDev)));
        SBG_CUDA(cudaMallocHost(&fresh->hx, (size_t)W.ld * sizeof(double)));
        ctx->pcg_ws = fresh;
        w = fresh.get();
    }
    return *w;
}

// L2 residency of W across the PCG iterations.  B200's 126 MB L2 can hold most of a
// matrix of up to ~100 MB (config 2: 126 MB, config 3: 361 MB, partly): W is read once per
// iteration, so an access-policy window marking it persisting keeps the part that fits in
// the persisting carve-out on chip from one iteration to the next instead of streaming it
// from HBM every time (hitRatio = carve-out / window when W is larger).  Matrices far larger
// than L2 (config 5: 5.1 GB) gain nothing and get no window.  SBG_L2_PERSIST=0 disables it.
static bool l2_window(Ctx* ctx, const DMatrix& W, bool sym, cudaAccessPolicyWindow& win)
{
    static const bool enabled = [] {
        const char* e = getenv("SBG_L2_PERSIST");
        return !(e && e[0] == '0');
    }();
    if (!enabled || W.n == 0) return false;
    int maxwin = 0, maxpersist = 0;
    SBG_CUDA(cudaDeviceGetAttribute(&maxwin, cudaDevAttrMaxAccessPolicyWindowSize, ctx->device));
    SBG_CUDA(cudaDeviceGetAttribute(&maxpersist, cudaDevAttrMaxPersistingL2CacheSize, ctx->device));
    size_t bytes = (size_t)W.n * W.ld * sizeof(double);
    // the symmetric form touches only the upper triangle (and its strips' diagonal blocks)
    const size_t touched = sym ? bytes / 2 + (size_t)W.n * 64 * sizeof(double) : bytes;
    if (maxwin <= 0 || maxpersist <= 0 || touched > 4 * (size_t)maxpersist) return false;
    static bool limit_set = false;
    if (!limit_set) {
        SBG_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)maxpersist));
        limit_set = true;
    }
    win.base_ptr = W.a.p;
    win.num_bytes = std::min(bytes, (size_t)maxwin);
    win.hitRatio = (float)std::min(1.0, (double)maxpersist / (double)std::min(touched, win.num_bytes));
    win.hitProp = cudaAccessPropertyPersisting;
    win.missProp = cudaAccessPropertyStreaming;
    return true;
}

// SBG_PCG_PERSIST=0 disables the persistent form (the graph form then runs every size)
static bool pcg_persist_enabled()
{
    static const bool on = [] {
        const char* e = getenv("SBG_PCG_PERSIST");
        return !(e && e[0] == '0');
    }();
    return on;
}

// co-resident CTAs of k_pcg_persistent on this device (0: no cooperative launch)
static int persist_grid(Ctx* ctx)
{
    static int grid = -1;
    if (grid < 0) {
        int coop = 0, per_sm = 0;
        SBG_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, ctx->device));
        SBG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pcg_persistent, 256, 0));
        grid = coop ? std::min(per_sm, 2) * ctx->sm_count : 0;
        if (const char* e = getenv("SBG_PCG_PERSIST_GRID"))  // (tuning)
            grid = std::max(1, std::min(grid, atoi(e)));
    }
    return grid;
}

// reference: inc/pcg.hpp:33-116.  All vectors and scalars stay on the device;
// the host enqueues iterations in growing batches and reads back one small
// state record per batch (iterations past convergence are no-op launches).
void pcg_run(Ctx* ctx, const DMatrix& W, Prec* prec, const double* rhs, double* x_out, bool on_device, double tol,
             int maxit, PcgResult& out, const RowPanel* rows, const double* exact)
{
    const int n = W.n;
    if (exact && rows) throw ValidationError("pcg: the energy history is not offered by the row-panel form");
    if (tol <= 0) throw ValidationError("pcg: tolerance must be positive");
    if (rows && (rows->lo < 0 || rows->hi > n || rows->lo > rows->hi || !rows->exchange))
        throw ValidationError("pcg: row panel outside the matrix or no exchange");
    if (prec && prec_n(prec) != n) throw ValidationError("preconditioner length mismatch");
    if (maxit <= 0) maxit = std::max(10 * n, 100);
    if (n == 0) {  // empty system: converged at iteration 0 (pcg.hpp:41-49 with r0 = 0)
        out = PcgResult{};
        out.converged = true;
        out.history.assign(1, 0.0);
        if (exact) out.energy.assign(1, 0.0);
        return;
    }
    TimedScope tpcg(ctx, "pcg");
    static const bool htrace = getenv("SBG_PCG_TRACE") != nullptr;
    const auto ht0 = std::chrono::steady_clock::now();
    auto hmark = [&](const char* what) {
        if (htrace)
            fprintf(stderr, " %s=%.1f", what,
                    std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - ht0).count());
    };
    if (htrace) fprintf(stderr, "[pcg host]");
    cudaStream_t s = ctx->stream;
    PcgWork& w = pcg_work(ctx, W, maxit);
    const size_t len = (size_t)W.ld;
    SBG_CUDA(cudaMemsetAsync(w.buf.p, 0, w.buf.n * sizeof(double), s));
    double* x = w.buf.p;
    double* r = x + len;
    double* zbuf = r + len;
    double* p = zbuf + len;
    double* Wp = p + len;
    double* rn = Wp + len;  // the fused apply's new residual (copied back into r)
    double* z = prec ? zbuf : r;  // no preconditioner: z = r (pcg.hpp:45-47)
    cudaAccessPolicyWindow keep_win{};
    bool keep_W = !rows && pcg_graph_enabled() && l2_window(ctx, W, w.plan.sym, keep_win);  // W held in L2 (graph form)
    // host vectors and the state record go through page-locked staging (no driver staging copies)
    if (on_device) {
        SBG_CUDA(cudaMemcpyAsync(r, rhs, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    } else {
        std::copy(rhs, rhs + n, w.hx);
        SBG_CUDA(cudaMemcpyAsync(r, w.hx, n * sizeof(double), cudaMemcpyHostToDevice, s));
    }
    const int nb = (n + 255) / 256;
    PcgDev h{};
    h.tol = tol;
    h.maxit = maxit;
    *w.hs0 = h;
    SBG_CUDA(cudaMemcpyAsync(w.st.p, w.hs0, sizeof(h), cudaMemcpyHostToDevice, s));
    const int* done = &w.st.p->done;
    // energy error history (pcg.hpp:50-53, 59, 82): e = x - exact, sqrt(e.We) after every
    // iteration's update and for x0 = 0 — one extra matvec per iteration, as in the reference
    double* e_err = nullptr;
    const double* d_exact = nullptr;
    if (exact) {
        if ((size_t)w.ebuf.n < 3 * len) w.ebuf.alloc(3 * len);
        if ((size_t)w.energy.n < (size_t)w.cap) w.energy.alloc(w.cap);
        e_err = w.ebuf.p;
        SBG_CUDA(cudaMemsetAsync(w.ebuf.p, 0, 3 * len * sizeof(double), s));
        SBG_CUDA(cudaMemcpyAsync(w.ebuf.p + len, exact, n * sizeof(double),
                                 on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
        d_exact = w.ebuf.p + len;
    }
    auto enqueue_energy = [&](int off, int gated) {
        launch_pdl(k_pcg_err, dim3(nb), dim3(256), 0, s, (const PcgDev*)w.st.p, (const double*)x, d_exact, e_err, n,
                   gated);
        count_launch();
        const double* We = w.plan.part.p;
        int chunks = w.plan.chunks;
        if (w.plan.sym) {  // W e into the third slice of ebuf
            symv_tiles_launch(ctx, W, w.plan, e_err, gated ? done : nullptr);
            symv_reduce_launch(ctx, W, w.plan, w.ebuf.p + 2 * len, gated ? done : nullptr);
            We = w.ebuf.p + 2 * len;
            chunks = 1;
        } else {
            gemv_partial_launch(ctx, W, w.plan, e_err, gated ? done : nullptr);
        }
        launch_pdl(k_pcg_energy, dim3(nb), dim3(256), 0, s, w.st.p, We, chunks, W.ld, n, (const double*)e_err,
                   w.partials.p, w.energy.p, off, gated);
        count_launch();
        SBG_LAUNCH_CHECK();
    };
    // persistent form (systems that stay in L2): the whole solve in one cooperative launch
    PrecView pv;
    const bool persist = n > 0 && n <= kPersistMaxN && !rows && !exact && prec && ctx->matvec_form == 0 &&
                         pcg_persist_enabled() && prec_view(prec, pv) && persist_grid(ctx) > 0;
    if (exact) enqueue_energy(0, 0);
    if (persist) {
        const int G = persist_grid(ctx);
        if (!w.splan.sym) symv_plan(ctx, n, W.ld, w.splan);
        if ((int)w.ppart.n < 2 * G) w.ppart.alloc(2 * (size_t)G);
        if (!w.bar.n) w.bar.alloc(1);
        SBG_CUDA(cudaMemsetAsync(w.bar.p, 0, sizeof(unsigned), s));
        static const bool tracing = getenv("SBG_PCG_TRACE") != nullptr;
        if (tracing && !w.trace.n) w.trace.alloc(8 * 64);
        PcgPersistArgs A{w.st.p, W.a.p, W.ld, n, x, r, rn, p, Wp, z, w.splan.tiles.p, w.splan.ntiles,
                         w.splan.tbase.p, w.splan.rowpart.p, w.splan.colpart.p, pv, w.hist.p, w.alphas.p, w.betas.p,
                         w.ppart.p, w.bar.p, tracing ? w.trace.p : nullptr};
        // (no access-policy window: the upper triangle, the inverses and the vectors of these
        // sizes stay in L2 anyway — measured equal or faster without one)
        void* args[] = {&A};
        hmark("pre_launch");
        SBG_CUDA(cudaLaunchCooperativeKernel((const void*)k_pcg_persistent, dim3(G), dim3(256), args, 0, s));
        hmark("launched");
        count_launch();
        SBG_LAUNCH_CHECK();
        if (tracing) {  // phase durations of the first iterations (us): tiles, barrier, alpha, gather+barrier, gemv+barrier, scatter+barrier+sum, next
            std::vector<unsigned long long> tr(8 * 64);
            SBG_CUDA(cudaMemcpyAsync(tr.data(), w.trace.p, tr.size() * 8, cudaMemcpyDeviceToHost, s));
            SBG_CUDA(cudaStreamSynchronize(s));
            for (int i = 1; i < 4; ++i) {
                fprintf(stderr, "[pcg trace] it %d:", i);
                for (int k = 1; k <= 6; ++k) fprintf(stderr, " %.2f", (tr[8 * i + k] - tr[8 * i + k - 1]) * 1e-3);
                fprintf(stderr, " | iter %.2f us\n", (tr[8 * (i + 1)] - tr[8 * i]) * 1e-3);
            }
        }
    }
    if (n > 0 && !persist) {
        if (prec) prec_apply(ctx, prec, r, z, nullptr);
        k_pcg_init<<<nb, 256, 0, s>>>(w.st.p, r, z, p, n, w.partials.p, w.hist.p);
        count_launch();
        SBG_LAUNCH_CHECK();
    } else if (!persist) {
        h.converged = 1;
        h.done = 1;
        SBG_CUDA(cudaMemcpyAsync(w.st.p, &h, sizeof(h), cudaMemcpyHostToDevice, s));
    }
    // one PCG iteration (pcg.hpp:69-93) on the context stream
    // gate (graph body only): the while node's handle; when the iteration's last kernel sets it
    // (the fused preconditioner path) no separate gate kernel follows — returns whether it did
    auto enqueue_iteration = [&](const cudaGraphConditionalHandle* gate) -> bool {
        bool gated = false;
        if (rows) {
            // row panel: this rank's rows of W p into the exchange buffer, then the
            // caller's all-gather fills the rest (issued even past convergence, so every
            // rank enqueues the same collectives; the kernels around it are no-ops then)
            {
                TimedScope ts(ctx, "gemv_f64");
                if (rows->hi > rows->lo)
                    launch_gemv_rows(true, s, rows->hi - rows->lo, (const double*)W.a.p + (size_t)rows->lo * W.ld, W.ld,
                                     rows->hi - rows->lo, (const double*)p, w.xbuf.p + rows->lo, done);
                count_launch();
                SBG_LAUNCH_CHECK();
            }
            {
                TimedScope ts(ctx, "pcg_exchange");
                if (rows->exchange(rows->user, p, w.xbuf.p, n, (void*)s) != 0)
                    throw std::runtime_error("pcg: the row-panel exchange failed");
            }
            if (w.plan.rows)  // the reduction tree of the single-GPU rows form (bitwise the same alpha)
                launch_pdl(k_pcg_alpha8, dim3((n + kRowsPerCta - 1) / kRowsPerCta), dim3(256), 0, s, w.st.p,
                           (const double*)w.xbuf.p, n, (const double*)p, Wp, w.partials.p);
            else
                launch_pdl(k_pcg_alpha, dim3(nb), dim3(256), 0, s, w.st.p, (const double*)w.xbuf.p, 1, W.ld, n, p,
                           Wp, w.partials.p);
        } else if (w.plan.sym) {  // symmetric form: upper-triangle tiles, then W p and alpha
            {
                TimedScope ts(ctx, "gemv_f64");
                symv_tiles_launch(ctx, W, w.plan, p, done, keep_W, z, w.st.p);
            }
            launch_pdl(k_symv_alpha, dim3((n + 31) / 32), dim3(256), 0, s, w.st.p, n, w.plan.H, W.ld,
                       (const int*)w.plan.tbase.p, (const double*)w.plan.rowpart.p, (const double*)w.plan.colpart.p, p,
                       (const double*)z, Wp, w.partials.p);
        } else if (w.plan.rows) {  // rows form: W p and alpha in one launch
            TimedScope ts(ctx, "gemv_f64");
            const dim3 grid((n + kRowsPerCta - 1) / kRowsPerCta);
            if (keep_W)
                launch_pdl(k_gemv_rows_alpha<true>, grid, dim3(256), 0, s, w.st.p, (const double*)W.a.p, W.ld, n,
                           (const double*)p, Wp, w.partials.p);
            else
                launch_pdl(k_gemv_rows_alpha<false>, grid, dim3(256), 0, s, w.st.p, (const double*)W.a.p, W.ld, n,
                           (const double*)p, Wp, w.partials.p);
        } else {
            {
                TimedScope ts(ctx, "gemv_f64");
                gemv_partial_launch(ctx, W, w.plan, p, done);
            }
            launch_pdl(k_pcg_alpha, dim3(nb), dim3(256), 0, s, w.st.p, w.plan.part.p, w.plan.chunks, W.ld, n, p, Wp,
                       w.partials.p);
        }
        count_launch();
        // x += alpha p, r -= alpha Wp, z = M r, r.z and beta: fused into the preconditioner's
        // three launches when it allows (inverse mode), else one kernel per step
        const PcgFused fu{w.st.p, x, r, rn, p, Wp, z, w.partials.p, w.hist.p, w.alphas.p, w.betas.p, done,
                          gate ? *gate : cudaGraphConditionalHandle{}, gate != nullptr};
        if (!exact && prec && prec_apply_pcg(ctx, prec, fu)) {
            gated = gate != nullptr;
        } else {
            launch_pdl(k_pcg_update, dim3(nb), dim3(256), 0, s, w.st.p, x, r, p, Wp, n);
            count_launch();
            if (exact) enqueue_energy(1, 1);
            if (prec) prec_apply(ctx, prec, r, z, done);
            launch_pdl(k_pcg_rz, dim3(nb), dim3(256), 0, s, w.st.p, r, z, n, w.partials.p, w.hist.p, w.alphas.p,
                       w.betas.p);
            count_launch();
        }
        if (!(w.plan.sym && !rows)) {  // (the symmetric form forms p inside the next matvec)
            launch_pdl(k_pcg_p, dim3(nb), dim3(256), 0, s, w.st.p, p, z, n);
            count_launch();
        }
        SBG_LAUNCH_CHECK();
        return gated;
    };
    // the exchange is a host call; the energy history (test path) runs host-driven too
    const bool graph = !persist && n > 0 && pcg_graph_enabled() && !rows && !exact;
    keep_W = keep_W && graph;
    if (graph) {
        // graph form: [gate] -> while(handle) { iteration ; gate } — the loop runs on the device
        // with no host round trips and no launches past convergence
        if (!w.exec || w.gW != W.a.p || w.gP != (prec ? prec_uid(prec) : 0)) {
            const bool timers = ctx->timers.enabled;
            ctx->timers.enabled = false;  // no timer events inside the captured body
            const long long launches0 = launch_count();
            long long captured = 0;
            cudaGraph_t ng = nullptr;
            try {
                SBG_CUDA(cudaGraphCreate(&ng, 0));
                cudaGraphConditionalHandle handle;
                SBG_CUDA(cudaGraphConditionalHandleCreate(&handle, ng, 0, 0));
                SBG_CUDA(cudaStreamBeginCaptureToGraph(s, ng, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
                k_pcg_gate<<<1, 32, 0, s>>>(w.st.p, handle);
                cudaGraph_t g_out = nullptr;
                SBG_CUDA(cudaStreamEndCapture(s, &g_out));
                size_t nroots = 0;
                SBG_CUDA(cudaGraphGetNodes(ng, nullptr, &nroots));
                std::vector<cudaGraphNode_t> nodes(nroots);
                SBG_CUDA(cudaGraphGetNodes(ng, nodes.data(), &nroots));
                cudaGraphNodeParams cp = {};
                cp.type = cudaGraphNodeTypeConditional;
                cp.conditional.handle = handle;
                cp.conditional.type = cudaGraphCondTypeWhile;
                cp.conditional.size = 1;
                cudaGraphNode_t cond;
                SBG_CUDA(cudaGraphAddNode(&cond, ng, nodes.data(), nroots, &cp));
                cudaGraph_t body = cp.conditional.phGraph_out[0];
                SBG_CUDA(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
                w.body_gate = !enqueue_iteration(&handle);
                if (w.body_gate) k_pcg_gate<<<1, 32, 0, s>>>(w.st.p, handle);
                SBG_CUDA(cudaStreamEndCapture(s, &g_out));
                cudaAccessPolicyWindow win{};
                if (l2_window(ctx, W, w.plan.sym, win)) {  // W persisting in L2 for every kernel of the body
                    size_t nb = 0;
                    SBG_CUDA(cudaGraphGetNodes(body, nullptr, &nb));
                    std::vector<cudaGraphNode_t> bn(nb);
                    SBG_CUDA(cudaGraphGetNodes(body, bn.data(), &nb));
                    cudaKernelNodeAttrValue v{};
                    v.accessPolicyWindow = win;
                    for (cudaGraphNode_t nd : bn) {
                        cudaGraphNodeType t;
                        SBG_CUDA(cudaGraphNodeGetType(nd, &t));
                        if (t == cudaGraphNodeTypeKernel)
                            SBG_CUDA(cudaGraphKernelNodeSetAttribute(nd, cudaKernelNodeAttributeAccessPolicyWindow, &v));
                    }
                }
                // same topology (a new preconditioner of the same kind): update the
                // instantiated graph in place instead of instantiating again
                bool updated = false;
                if (w.exec) {
                    cudaGraphExecUpdateResultInfo info;
                    if (cudaGraphExecUpdate(w.exec, ng, &info) == cudaSuccess) {
                        updated = true;
                    } else {
                        (void)cudaGetLastError();
                    }
                }
                if (!updated) {
                    w.drop_graph();
                    SBG_CUDA(cudaGraphInstantiate(&w.exec, ng, 0));
                }
                if (w.graph) cudaGraphDestroy(w.graph);
                w.graph = ng;
                ng = nullptr;
            } catch (...) {
                ctx->timers.enabled = timers;
                cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
                if (cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
                    cudaGraph_t junk = nullptr;  // leave capture mode before anything else touches the stream
                    cudaStreamEndCapture(s, &junk);
                    if (junk && junk != ng) cudaGraphDestroy(junk);
                }
                (void)cudaGetLastError();
                if (ng) cudaGraphDestroy(ng);
                w.drop_graph();
                throw;
            }
            ctx->timers.enabled = timers;
            captured = launch_count() - launches0;  // one iteration's kernels (recorded, not run)
            add_launches(-captured);
            w.kernels_per_iter = (int)captured;
            w.gW = W.a.p;
            w.gP = prec ? prec_uid(prec) : 0;
        }
        SBG_CUDA(cudaGraphLaunch(w.exec, s));
    }
    // the device-looped forms (graph, persistent) come back in one round trip: the state, the
    // first kHistPre history / alpha / beta entries (page-locked staging) and x
    const bool device_loop = graph || persist;
    const int pre = std::min(kHistPre, w.cap);
    if (device_loop) {
        SBG_CUDA(cudaMemcpyAsync(w.hs, w.st.p, sizeof(PcgDev), cudaMemcpyDeviceToHost, s));
        SBG_CUDA(cudaMemcpyAsync(w.hh, w.hist.p, pre * sizeof(double), cudaMemcpyDeviceToHost, s));
        SBG_CUDA(cudaMemcpyAsync(w.hh + kHistPre, w.alphas.p, pre * sizeof(double), cudaMemcpyDeviceToHost, s));
        SBG_CUDA(cudaMemcpyAsync(w.hh + 2 * kHistPre, w.betas.p, pre * sizeof(double), cudaMemcpyDeviceToHost, s));
        SBG_CUDA(cudaMemcpyAsync(on_device ? x_out : w.hx, x, n * sizeof(double),
                                 on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
        hmark("copies_enqueued");
        SBG_CUDA(cudaStreamSynchronize(s));
        hmark("synced");
        if (!on_device) std::copy(w.hx, w.hx + n, x_out);
        if (graph) add_launches((long long)w.kernels_per_iter * w.hs->it + 1 + (w.body_gate ? w.hs->it : 0));  // + gates
    }
    int batch = 4, enqueued = device_loop ? maxit : 0;
    while (!device_loop) {
        SBG_CUDA(cudaMemcpyAsync(w.hs, w.st.p, sizeof(PcgDev), cudaMemcpyDeviceToHost, s));
        SBG_CUDA(cudaStreamSynchronize(s));
        int stop = (w.hs->done || enqueued >= maxit) ? 1 : 0;
        if (rows && rows->agree) {  // every rank takes the same decision (kernels.cuh: AgreeFn)
            int all = stop;
            if (rows->agree(rows->user, stop, &all) != 0) throw std::runtime_error("pcg: the row-panel agreement failed");
            stop = all;
        }
        if (stop) break;
        const int todo = std::min(batch, maxit - enqueued);
        for (int t = 0; t < todo; ++t) enqueue_iteration(nullptr);
        enqueued += todo;
        batch = std::min(batch * 2, 64);
    }
    if (keep_W) SBG_CUDA(cudaCtxResetPersistingL2Cache());  // give L2 back to what follows
    const PcgDev fin = *w.hs;
    if (fin.error == 1) throw NumericalError("pcg: matrix is not positive definite");
    if (fin.error == 2) throw NumericalError("pcg: preconditioner is not positive definite");
    out.iterations = fin.it;
    out.converged = fin.converged != 0;
    out.history.assign(fin.it + 1, 0.0);
    out.alphas.assign(fin.it, 0.0);
    out.betas.assign(fin.it, 0.0);
    if (device_loop && fin.it + 1 <= pre) {  // everything already on the host
        std::copy(w.hh, w.hh + fin.it + 1, out.history.begin());
        std::copy(w.hh + kHistPre, w.hh + kHistPre + fin.it, out.alphas.begin());
        std::copy(w.hh + 2 * kHistPre, w.hh + 2 * kHistPre + fin.it, out.betas.begin());
        out.kappa = lanczos_kappa(out.alphas, out.betas);
        hmark("done");
        if (htrace) fprintf(stderr, "\n");
        return;
    }
    if (n > 0) {
        SBG_CUDA(cudaMemcpyAsync(out.history.data(), w.hist.p, (fin.it + 1) * sizeof(double), cudaMemcpyDeviceToHost, s));
        if (fin.it) {
            SBG_CUDA(cudaMemcpyAsync(out.alphas.data(), w.alphas.p, fin.it * sizeof(double), cudaMemcpyDeviceToHost, s));
            SBG_CUDA(cudaMemcpyAsync(out.betas.data(), w.betas.p, fin.it * sizeof(double), cudaMemcpyDeviceToHost, s));
        }
        if (exact) {
            out.energy.assign(fin.it + 1, 0.0);
            SBG_CUDA(cudaMemcpyAsync(out.energy.data(), w.energy.p, (fin.it + 1) * sizeof(double),
                                     cudaMemcpyDeviceToHost, s));
        }
        SBG_CUDA(cudaMemcpyAsync(x_out, x, n * sizeof(double), on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
    } else {
        out.history.assign(1, 0.0);
    }
    SBG_CUDA(cudaStreamSynchronize(s));
    out.kappa = lanczos_kappa(out.alphas, out.betas);
}

}  // namespace sbg
