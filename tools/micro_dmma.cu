// Does the FP64 tensor path (DMMA, mma.sync m8n8k4 f64) run beside the FP64 vector pipe
// (DFMA) on sm_100a?  Three loops with the same structure: DFMA chains only, DMMA chains
// only, and both interleaved in the same warps.  If the mixed loop takes max(t_dfma, t_dmma)
// rather than their sum, r^2 = |x|^2 + |y|^2 - 2 x.y can move to DMMA and free the vector
// pipe for the 1/r refinement.  Also measures the accuracy of rsqrt.approx.ftz.f64.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro_dmma tools/micro_dmma.cu
#include <cmath>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int MODE>  // 0 dfma, 1 dmma, 2 both
__global__ void k_loop(double* out, int reps)
{
    const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    double f[16], m0[8], m1[8];
#pragma unroll
    for (int k = 0; k < 16; ++k) f[k] = k * 1e-3;
#pragma unroll
    for (int k = 0; k < 8; ++k) m0[k] = m1[k] = k * 1e-3;
    for (int r = 0; r < reps; ++r) {
        if (MODE != 1) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int k = 0; k < 16; ++k) f[k] = fma(f[k], b, a);
        }
        if (MODE != 0) {
#pragma unroll
            for (int k = 0; k < 8; ++k) dmma(m0[k], m1[k], a, b);
        }
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) s += f[k];
#pragma unroll
    for (int k = 0; k < 8; ++k) s += m0[k] + m1[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_rsqrt_err(double* err, int n)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    // inputs spread over [1e-6, 1e6]
    const double x = exp(-13.8 + 27.6 * ((double)i + 0.5) / n);
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double ex = 1.0 / sqrt(x);
    err[3 * i] = fabs(y - ex) / ex;
    // 2nd order (Newton) and 3rd order refinement
    const double e = fma(-x * y, y, 1.0);
    const double y2 = fma(0.5 * y, e, y);
    const double y3 = fma(y, e * fma(0.375, e, 0.5), y);
    err[3 * i + 1] = fabs(y2 - ex) / ex;
    err[3 * i + 2] = fabs(y3 - ex) / ex;
}

int main()
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int blocks = sms * 4, threads = 256, reps = 4096;
    double* out;
    cudaMalloc(&out, (size_t)blocks * threads * sizeof(double));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](auto kern, const char* name, double dfma_per_rep, double dmma_per_rep) {
        kern<<<blocks, threads>>>(out, reps);
        cudaEventRecord(e0);
        for (int i = 0; i < 5; ++i) kern<<<blocks, threads>>>(out, reps);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double s = ms * 1e-3 / 5;
        const double warps = (double)blocks * threads / 32;
        const double fma_v = warps * reps * dfma_per_rep * 32;    // vector FMAs
        const double fma_t = warps * reps * dmma_per_rep * 256;   // tensor FMAs
        std::printf("%-6s %8.3f ms  vector %6.2f TF  tensor %6.2f TF  total %6.2f TF\n", name, ms / 5,
                    2 * fma_v / s / 1e12, 2 * fma_t / s / 1e12, 2 * (fma_v + fma_t) / s / 1e12);
    };
    run(k_loop<0>, "dfma", 64, 0);
    run(k_loop<1>, "dmma", 0, 8);
    run(k_loop<2>, "both", 64, 8);
    std::printf("SMs %d, clock %d MHz\n", sms, clk / 1000);
    const int n = 1 << 22;
    double* err;
    cudaMalloc(&err, (size_t)3 * n * sizeof(double));
    k_rsqrt_err<<<(n + 255) / 256, 256>>>(err, n);
    double* h = new double[(size_t)3 * n];
    cudaMemcpy(h, err, (size_t)3 * n * sizeof(double), cudaMemcpyDeviceToHost);
    double mx[3] = {0, 0, 0};
    for (int i = 0; i < n; ++i)
        for (int k = 0; k < 3; ++k) mx[k] = fmax(mx[k], h[3 * i + k]);
    std::printf("rsqrt.approx.ftz.f64 max rel err %.3e (2^%.1f); 2nd order %.3e; 3rd order %.3e\n", mx[0],
                std::log2(mx[0]), mx[1], mx[2]);
    return 0;
}
