// Timing of the 64x64 diagonal-tile factor + inverse of the preconditioner build
// (tile_factor.cuh, used by k_panel_step) on one CTA per SM, and a check of L and
// D = L^-1 against a host Cholesky.  Not part of the library.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro_factor tools/micro_factor.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

namespace sbg {
namespace {
constexpr int TB = 64;
#include "../paper_2310_09204_b200/csrc/cuda/tile_factor.cuh"
}  // namespace
}  // namespace sbg
using namespace sbg;

template <int V>
__global__ void __launch_bounds__(256) k_factor(const double* __restrict__ A, double* __restrict__ Lout,
                                                double* __restrict__ Dout, long long* __restrict__ cyc, int reps)
{
    __shared__ double a[TB * AS];
    __shared__ double sq[TB];
    __shared__ FactorBufs fb;
    long long total = 0;
    double x[4][4];
    for (int rep = 0; rep < reps; ++rep) {
        for (int e = threadIdx.x; e < TB * TB; e += blockDim.x) a[(e / TB) * AS + e % TB] = A[e];
        __syncthreads();
        const long long t0 = clock64();
        tile_ldl_inverse<V == 1>(a, fb, x);
        if (threadIdx.x < TB) sq[threadIdx.x] = sqrt(a[threadIdx.x * AS + threadIdx.x]);
        __syncthreads();
        total += clock64() - t0;
    }
    if (threadIdx.x == 0) cyc[blockIdx.x] = total / reps;
    if (blockIdx.x != 0) return;
    const int r0 = blk_r0(), c0 = blk_c0();
    for (int e = threadIdx.x; e < TB * TB; e += blockDim.x) {
        const int r = e / TB, c = e % TB;
        Lout[e] = c < r ? a[r * AS + c] / sq[c] : (c == r ? sq[r] : 0.0);
    }
    for (int u = 0; u < 4; ++u)
        for (int v = 0; v < 4; ++v) {
            const int r = r0 + u, c = c0 + v;
            Dout[r * TB + c] = c <= r ? x[u][v] / sq[r] : 0.0;
        }
}

template <int V>
void run(const char* name, const double* dA, const std::vector<double>& Lh, const std::vector<double>& Dh)
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *dL, *dD;
    long long* dc;
    cudaMalloc(&dL, TB * TB * 8);
    cudaMalloc(&dD, TB * TB * 8);
    cudaMalloc(&dc, sms * 8);
    k_factor<V><<<sms, 256>>>(dA, dL, dD, dc, 2);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int reps = 50;
    cudaEventRecord(a);
    k_factor<V><<<sms, 256>>>(dA, dL, dD, dc, reps);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    std::vector<long long> c(sms);
    std::vector<double> L(TB * TB), D(TB * TB);
    cudaMemcpy(c.data(), dc, sms * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(L.data(), dL, TB * TB * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(D.data(), dD, TB * TB * 8, cudaMemcpyDeviceToHost);
    double el = 0, ed = 0, ml = 0, md = 0;
    for (int e = 0; e < TB * TB; ++e) {
        el = fmax(el, fabs(L[e] - Lh[e]));
        ed = fmax(ed, fabs(D[e] - Dh[e]));
        ml = fmax(ml, fabs(Lh[e]));
        md = fmax(md, fabs(Dh[e]));
    }
    printf("%-28s %8lld cycles per tile (%.2f us at 1.965 GHz); wall %.2f us per tile; |dL| %.2e |dD| %.2e (rel)\n",
           name, c[0], c[0] / 1965.0, ms * 1e3 / reps, el / ml, ed / md);
    cudaFree(dL);
    cudaFree(dD);
    cudaFree(dc);
}

// latency probes (one warp): dependent DFMA chain, MUFU.RCP64H + DFMA, shared store -> barrier -> load
__global__ void k_lat(double* out, long long* cyc, double v)
{
    __shared__ double buf[256];
    double x = v + threadIdx.x;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) x = fma(x, 0.999, 1e-3);
    long long t1 = clock64();
    double y = x;
#pragma unroll 1
    for (int i = 0; i < 256; ++i) {
        double r;
        asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y));
        y = fma(r, 1e-9, 2.0);
    }
    long long t2 = clock64();
    double z = y;
#pragma unroll 1
    for (int i = 0; i < 256; ++i) {
        buf[threadIdx.x] = z;
        __syncthreads();
        z = buf[(threadIdx.x + 1) & 255] * 0.5 + 1.0;
    }
    long long t3 = clock64();
    double w = z;
#pragma unroll 1
    for (int i = 0; i < 256; ++i) {
        buf[threadIdx.x & 31] = w;
        __syncwarp();
        w = buf[(threadIdx.x + 1) & 31] * 0.5 + 1.0;
        __syncwarp();
    }
    long long t4 = clock64();
    double q = w;
#pragma unroll 1
    for (int i = 0; i < 256; ++i) q = __shfl_sync(0xffffffffu, q, (threadIdx.x + 1) & 31) * 0.5 + 1.0;
    long long t5 = clock64();
    if (threadIdx.x == 0) {
        cyc[0] = (t1 - t0) / 1024;
        cyc[1] = (t2 - t1) / 256;
        cyc[2] = (t3 - t2) / 256;
        cyc[3] = (t4 - t3) / 256;
        cyc[4] = (t5 - t4) / 256;
    }
    if (q == 1.2345) out[0] = q;
}

int main()
{
    {
        double* d;
        long long* c;
        cudaMalloc(&d, 64);
        cudaMalloc(&c, 64);
        for (int threads : {32, 256}) {
            k_lat<<<1, threads>>>(d, c, 0.5);
            long long h[5];
            cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
            printf("latency (%d threads): DFMA %lld, RCP64H+DFMA %lld, STS+bar+LDS+DFMA(mul,add) %lld, "
                   "STS+syncwarp+LDS+2 %lld, SHFL(f64)+2 %lld cycles\n",
                   threads, h[0], h[1], h[2], h[3], h[4]);
        }
    }
    // SPD test tile: a well-conditioned kernel matrix like a W diagonal block
    std::vector<double> A(TB * TB), L(TB * TB, 0.0), D(TB * TB, 0.0);
    for (int r = 0; r < TB; ++r)
        for (int c = 0; c < TB; ++c) A[r * TB + c] = 1.0 / (1.0 + 0.3 * std::abs(r - c)) + (r == c ? 2.0 : 0.0);
    for (int j = 0; j < TB; ++j) {  // host Cholesky
        double s = A[j * TB + j];
        for (int q = 0; q < j; ++q) s -= L[j * TB + q] * L[j * TB + q];
        L[j * TB + j] = std::sqrt(s);
        for (int r = j + 1; r < TB; ++r) {
            double t = A[r * TB + j];
            for (int q = 0; q < j; ++q) t -= L[r * TB + q] * L[j * TB + q];
            L[r * TB + j] = t / L[j * TB + j];
        }
    }
    for (int c = 0; c < TB; ++c)  // D = L^-1 by forward substitution per column
        for (int r = c; r < TB; ++r) {
            double t = r == c ? 1.0 : 0.0;
            for (int q = c; q < r; ++q) t -= L[r * TB + q] * D[q * TB + c];
            D[r * TB + c] = t / L[r * TB + r];
        }
    double* dA;
    cudaMalloc(&dA, TB * TB * 8);
    cudaMemcpy(dA, A.data(), TB * TB * 8, cudaMemcpyHostToDevice);
    run<0>("tile_ldl_inverse", dA, L, D);
    run<1>("tile_ldl_inverse fast rcp", dA, L, D);
    return 0;
}
