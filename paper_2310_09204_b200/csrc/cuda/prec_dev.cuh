// Device bodies of the PCG-fused preconditioner apply (inverse mode), shared by its kernels
// (precond.cu: k_prec_gather_upd, k_block_gemv, k_prec_scatter_rz — one virtual block per
// CTA) and the persistent PCG kernel (linalg.cu: every CTA loops over the virtual blocks).
// reference: inc/schwarz.hpp:121-140 (apply), inc/pcg.hpp:74-79 (the update around it).
#pragma once

#include "common.cuh"

namespace sbg {

// device pointers of an inverse-mode preconditioner (prec_view, precond.cu)
struct PrecView {
    int n = 0, nc = 0, dof_blocks = 0, ntasks = 0;
    const int* pos = nullptr;  // dof -> block-local index, -1 if none
    double* loc = nullptr;     // block-local gathered residual
    double* locy = nullptr;    // block-local result
    const int *Rc_ptr = nullptr, *Rc_row = nullptr;  // R by coarse column (restriction)
    const double* Rc_val = nullptr;
    double* loc_c = nullptr;  // coarse block's slice of loc (nullptr: no coarse space)
    const int *Rr_ptr = nullptr, *Rr_col = nullptr;  // R by fine row (prolongation)
    const double* Rr_val = nullptr;
    const double* y_c = nullptr;  // coarse block's slice of locy
    const int2* tasks = nullptr;  // (block, first row) per 8-row GEMV task
    const int *nbv = nullptr, *ldmv = nullptr, *locv = nullptr;
    const long long* Moff = nullptr;
    const double* Mc = nullptr;  // compact block inverses
};

// virtual block vb < dof_blocks: x += a p, rn = r - a Wp gathered into loc; vb >= dof_blocks:
// coarse column c = vb - dof_blocks of R^T (r - a Wp) (red: 8 doubles of shared memory)
__device__ __forceinline__ void prec_gather_upd_body(int vb, double a, double* __restrict__ x,
                                                     const double* __restrict__ r, double* __restrict__ rn,
                                                     const double* __restrict__ p, const double* __restrict__ Wp,
                                                     int n, const int* __restrict__ pos, double* __restrict__ loc,
                                                     const int* __restrict__ cptr, const int* __restrict__ crow,
                                                     const double* __restrict__ cval, int nc,
                                                     double* __restrict__ loc_c, int dof_blocks, double* red)
{
    if (vb < dof_blocks) {
        const int d = vb * blockDim.x + threadIdx.x;
        if (d < n) {
            const double rv = r[d] - a * Wp[d];
            rn[d] = rv;
            x[d] += a * p[d];
            if (pos[d] >= 0) loc[pos[d]] = rv;
        }
        return;
    }
    const int c = vb - dof_blocks;
    if (c >= nc) return;
    const int q0 = cptr[c], q1 = cptr[c + 1];
    double s0 = 0.0, s1 = 0.0;
    int q = q0 + threadIdx.x;
    for (; q + 256 < q1; q += 2 * 256) {
        const int i0 = crow[q], i1 = crow[q + 256];
        s0 += cval[q] * (r[i0] - a * Wp[i0]);
        s1 += cval[q + 256] * (r[i1] - a * Wp[i1]);
    }
    for (; q < q1; q += 256) s0 += cval[q] * (r[crow[q]] - a * Wp[crow[q]]);
    double v = s0 + s1;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += red[w];
        loc_c[c] = t;
    }
}

// one 8-row task of the batched block-inverse GEMV: locy = M_b loc (warp per row, 8 x 128-bit
// loads in flight per lane on long rows, one predicated chunk on short ones); KEEP: default
// caching (the persistent PCG re-reads the inverses every iteration from L2) instead of
// evict-first
template <bool KEEP = false>
__device__ __forceinline__ void block_gemv_body(int2 t, const int* __restrict__ nbv, const int* __restrict__ ldmv,
                                                const int* __restrict__ locv, const long long* __restrict__ Moff,
                                                const double* __restrict__ Mc, const double* __restrict__ loc,
                                                double* __restrict__ locy)
{
    const int b = t.x, nb = nbv[b], ldm = ldmv[b];
    const int r = t.y + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (r >= nb) return;
    const double2* x2 = reinterpret_cast<const double2*>(loc + locv[b]);  // loc rows are 64-padded (zeros)
    const double2* row = reinterpret_cast<const double2*>(Mc + Moff[b] + (size_t)r * ldm);
    const int half = ldm >> 1;
    auto ldm2 = [](const double2* q) { return KEEP ? __ldg(q) : __ldcs(q); };
    double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (half > 8 * 32) {  // long rows (WB): 8 x 128-bit loads in flight per lane, serial tail
        int c = lane;
        for (; c + 7 * 32 < half; c += 8 * 32) {
            double2 a[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) a[u] = ldm2(row + c + 32 * u);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const double2 xv = __ldg(x2 + c + 32 * u);
                s[u] = fma(a[u].x, xv.x, fma(a[u].y, xv.y, s[u]));
            }
        }
        for (; c < half; c += 32) {
            const double2 a = ldm2(row + c);
            const double2 xv = __ldg(x2 + c);
            s[0] = fma(a.x, xv.x, fma(a.y, xv.y, s[0]));
        }
    } else {  // short rows (faces): one predicated chunk, every load issued before the FMAs
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int c = lane + 32 * u;
            if (c < half) {
                const double2 a = ldm2(row + c);
                const double2 xv = __ldg(x2 + c);
                s[u] = fma(a.x, xv.x, fma(a.y, xv.y, s[u]));
            }
        }
    }
    double v = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) locy[locv[b] + r] = v;
}

// virtual block vb: z = scatter of the block results + coarse prolongation, r = rn; returns
// this thread's r.z term (0 past n)
__device__ __forceinline__ double prec_scatter_body(int vb, const double* __restrict__ locy,
                                                    const int* __restrict__ pos, int n, const int* __restrict__ rptr,
                                                    const int* __restrict__ rcol, const double* __restrict__ rval,
                                                    const double* __restrict__ y_c, double* __restrict__ z,
                                                    double* __restrict__ r, const double* __restrict__ rn)
{
    const int d = vb * blockDim.x + threadIdx.x;
    if (d >= n) return 0.0;
    double out = pos[d] >= 0 ? locy[pos[d]] : 0.0;
    if (rptr) {
        double y = 0.0;
        for (int q = rptr[d]; q < rptr[d + 1]; ++q) y += rval[q] * y_c[rcol[q]];
        out += y;
    }
    z[d] = out;
    const double rv = rn[d];
    r[d] = rv;
    return rv * out;
}

}  // namespace sbg
