// Device-side PCG state and the deterministic reductions shared by the PCG kernels
// (linalg.cu) and the PCG-fused preconditioner apply (precond.cu).
#pragma once

#include "common.cuh"

namespace sbg {

__device__ __forceinline__ double block_sum(double v, double* sh)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    v = 0.0;
    if (warp == 0) {
        v = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    }
    return v;  // valid in thread 0
}

// ---------------------------------------------------------------- PCG state
struct PcgDev {
    double rz, alpha, beta, r0, tol, pwp;
    int it, maxit, done, converged, error;
    unsigned counter;
};

// Returns true in every thread of the last block to finish (threadfence reduction).
__device__ __forceinline__ bool last_block(double v_thread0, double* partials, unsigned* counter)
{
    __shared__ bool is_last;
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = v_thread0;
        __threadfence();
        const unsigned t = atomicAdd(counter, 1u);
        is_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    return is_last;
}

__device__ __forceinline__ double sum_partials(const double* partials, int count)
{
    double s = 0.0;
    for (int b = 0; b < count; ++b) s += ((volatile const double*)partials)[b];
    return s;
}


// Deterministic parallel sum of `count` block partials by every thread of the calling
// block (the last block of a grid-wide reduction): thread t adds partials t, t + blockDim,
// ... in order, then the block's fixed shuffle tree.  For grids with hundreds of blocks (the
// 8-row blocks of the rows-form GEMV) a serial sum by one thread would cost hundreds of
// dependent L2 round trips.  Result valid in thread 0.
__device__ __forceinline__ double sum_partials_block(const double* partials, int count, double* sh)
{
    double s = 0.0;
    for (int b = threadIdx.x; b < count; b += blockDim.x) s += ((volatile const double*)partials)[b];
    return block_sum(s, sh);
}

// rz_new = r.z reduced: history, alpha/beta bookkeeping, stopping test (pcg.hpp:76-93);
// called by thread 0 of the last block
__device__ __forceinline__ void pcg_finish_rz(PcgDev* st, double rz_new, double* hist, double* alphas, double* betas)
{
    if (rz_new < 0) {
        st->error = 2;
        st->done = 1;
        return;
    }
    const int it = st->it;
    alphas[it] = st->alpha;
    st->it = it + 1;
    const double res = sqrt(fmax(rz_new, 0.0));
    hist[it + 1] = res;
    const double beta = rz_new / st->rz;
    betas[it] = beta;
    st->beta = beta;
    st->rz = rz_new;
    if (res <= st->tol * st->r0) {
        st->converged = 1;
        st->done = 1;
    } else if (st->it >= st->maxit) {
        st->done = 1;
    }
}

}  // namespace sbg
