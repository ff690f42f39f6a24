// 64x64 diagonal-tile factorisation + inverse in shared memory (precond.cu k_panel_step;
// also built standalone by tools/micro_factor.cu for timing).  Include inside namespace
// sbg::{anonymous} after TB is defined.
#pragma once

// ---------------------------------------------------------------- Cholesky: fused panel step
// Factor the 64x64 SPD tile a[] (lower part valid, row stride AS) and form its inverse:
// right-looking elimination in LDL^T form — multipliers m_rj = a_rj / a_jj, Schur update
// a_rc -= m_rj a_cj for j < c <= r — fused with the same eliminations applied to [L | I],
// whose rows Y_r = L_rr (L^-1)_r obey Y_r = e_r - sum_{j<r} m_rj Y_j (the multipliers are
// L_rj / L_jj).  256 threads, each owning a 4x4 register block of the tile: element (r,c)
// holds a_rc until column c is eliminated and Y_rc from then on, so every step is the same
// rank-1 update x -= m_r o_c of the whole block, with o = column j of a (c > j) or row j of
// Y (c <= j).  Column j (zero above the diagonal, the pivot kept apart) and row j of Y are
// published at the end of step j-1 into double-buffered shared vectors: ONE barrier per
// column.  On exit a[r][c] (r >= c) holds the eliminated columns (a[j][j] = pivot p_j,
// L_jj = sqrt(p_j), L_rc = a_rc / L_cc) and x[][] the thread's 4x4 block of Y; returns
// false (all threads) if a pivot is not positive and finite.
constexpr int AS = TB + 1;  // row stride of the tile in shared memory
constexpr int kFactorThreads = 256;
struct FactorBufs {
    double col[2][TB], yrow[2][TB], piv[2], inv[2];
};
// 4x4 block of thread t: column block t >> 4 (so a column's 16 owners are one half warp,
// and only that warp takes the publishing branch), row block t & 15
__device__ __forceinline__ int blk_r0() { return (threadIdx.x & 15) * 4; }
__device__ __forceinline__ int blk_c0() { return (threadIdx.x >> 4) * 4; }
// 1/p by MUFU.RCP64H and two Newton steps (within an ulp or two; no IEEE-division slow path)
__device__ __forceinline__ double rcp_fast(double p)
{
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(p));
    double e = fma(-p, y, 1.0);
    y = fma(y, e, y);
    e = fma(-p, y, 1.0);
    return fma(y, e, y);
}
template <bool FAST = false>
__device__ bool tile_ldl_inverse(double* __restrict__ a, FactorBufs& fb, double (&x)[4][4])
{
    const int r0 = blk_r0(), c0 = blk_c0();
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) x[u][v] = a[(r0 + u) * AS + c0 + v];
    // publish column 0 (pivot apart, rows <= 0 zero) and row 0 of Y for step 0
    auto publish = [&](int jn, int buf) {
        if (c0 <= jn && jn < c0 + 4) {
#pragma unroll
            for (int v = 0; v < 4; ++v)
                if (c0 + v == jn) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int r = r0 + u;
                        fb.col[buf][r] = r > jn ? x[u][v] : 0.0;
                        if (r >= jn) a[r * AS + jn] = x[u][v];
                        if (r == jn) {
                            fb.piv[buf] = x[u][v];
                            fb.inv[buf] = FAST ? rcp_fast(x[u][v]) : 1.0 / x[u][v];
                        }
                        x[u][v] = r == jn ? 1.0 : 0.0;  // element (r, jn) becomes Y_{r,jn}: delta
                    }
                }
        }
        if (r0 <= jn && jn < r0 + 4) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (r0 + u == jn)
#pragma unroll
                    for (int v = 0; v < 4; ++v) fb.yrow[buf][c0 + v] = x[u][v];
        }
    };
    publish(0, 0);
    __syncthreads();
    bool ok = true;
    for (int j = 0; j < TB; ++j) {
        const int cur = j & 1;
        const double p = fb.piv[cur];
        ok = ok && p > 0.0 && isfinite(p);
        if (r0 + 3 > j) {  // some row r > j of this block is still active (m_r = 0 otherwise)
            const double inv = fb.inv[cur];
            double m[4], o[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) m[u] = fb.col[cur][r0 + u] * inv;
#pragma unroll
            for (int v = 0; v < 4; ++v) o[v] = c0 + v > j ? fb.col[cur][c0 + v] : fb.yrow[cur][c0 + v];
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) x[u][v] = fma(-m[u], o[v], x[u][v]);
        }
        if (j + 1 < TB) publish(j + 1, cur ^ 1);
        __syncthreads();
    }
    return ok;
}

