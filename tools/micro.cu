// Microbenchmarks that shape the quadrature kernels (not part of the library):
//   1. accuracy of rsqrt.approx.f64 (MUFU.RSQ64H seed) and of the 3rd-order refined rsqrt
//   2. DFMA throughput, DMMA (mma.sync m8n8k4 f64) throughput, and both interleaved
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro tools/micro.cu
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

__device__ __forceinline__ double rsq_seed(double x)
{
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    return y;
}
__device__ __forceinline__ double rsq3(double r2)
{
    const double y = rsq_seed(r2);
    const double h = r2 * y;
    const double e = fma(-h, y, 1.0);
    const double c = fma(0.375, e, 0.5);
    return fma(y, e * c, y);
}
__device__ __forceinline__ double rsq2(double r2)
{
    const double y = rsq_seed(r2);
    const double h = r2 * y;
    const double e = fma(-h, y, 1.0);
    return fma(0.5 * y, e, y);
}

__global__ void k_acc(int n, double* out)
{
    double m0 = 0, m3 = 0, m2 = 0;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const double x = 1e-6 + (double)k * 7.3e-4 + 1e-9 * (k % 977);
        const double ref = 1.0 / sqrt(x);
        m0 = fmax(m0, fabs(rsq_seed(x) - ref) / ref);
        m3 = fmax(m3, fabs(rsq3(x) - ref) / ref);
        m2 = fmax(m2, fabs(rsq2(x) - ref) / ref);
    }
    atomicMax((unsigned long long*)&out[0], __double_as_longlong(m0));
    atomicMax((unsigned long long*)&out[1], __double_as_longlong(m3));
    atomicMax((unsigned long long*)&out[2], __double_as_longlong(m2));
}

__global__ void k_dfma(double* out, int iters)
{
    double a[8];
    for (int q = 0; q < 8; ++q) a[q] = threadIdx.x * 1e-9 + q;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int q = 0; q < 8; ++q) a[q] = fma(a[q], 0.999999999, 1e-12);
    double s = 0;
    for (int q = 0; q < 8; ++q) s += a[q];
    if (s == 1.2345) out[0] = s;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void k_dmma(double* out, int iters)
{
    double c[8][2];
    for (int q = 0; q < 8; ++q) c[q][0] = c[q][1] = 0;
    const double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int q = 0; q < 8; ++q) dmma(c[q][0], c[q][1], a, b);
    double s = 0;
    for (int q = 0; q < 8; ++q) s += c[q][0] + c[q][1];
    if (s == 1.2345) out[0] = s;
}

// DMMA and DFMA chains interleaved in the same warp
__global__ void k_mixed(double* out, int iters)
{
    double c[4][2], a8[8];
    for (int q = 0; q < 4; ++q) c[q][0] = c[q][1] = 0;
    for (int q = 0; q < 8; ++q) a8[q] = threadIdx.x * 1e-9 + q;
    const double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int q = 0; q < 4; ++q) dmma(c[q][0], c[q][1], a, b);
#pragma unroll
        for (int q = 0; q < 8; ++q) a8[q] = fma(a8[q], 0.999999999, 1e-12);
#pragma unroll
        for (int q = 0; q < 8; ++q) a8[q] = fma(a8[q], 0.999999999, 1e-12);
    }
    double s = 0;
    for (int q = 0; q < 4; ++q) s += c[q][0] + c[q][1];
    for (int q = 0; q < 8; ++q) s += a8[q];
    if (s == 1.2345) out[0] = s;
}

template <class K>
double time_kernel(K kern, int blocks, int threads, int iters, double* out)
{
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    kern<<<blocks, threads>>>(out, 64);
    cudaEventRecord(a);
    kern<<<blocks, threads>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms * 1e-3;
}

int main1()
{
    double* d;
    cudaMalloc(&d, 64);
    cudaMemset(d, 0, 64);
    k_acc<<<148 * 4, 256>>>(1 << 24, d);
    double h[3];
    cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("rsqrt.approx.f64 max rel err %.3e ; 3rd-order refined %.3e ; 2nd-order refined %.3e (eps 1.1e-16)\n", h[0],
           h[1], h[2]);
    int sms = 148;
    const int blocks = sms * 8, threads = 256, iters = 4096;
    const double t1 = time_kernel(k_dfma, blocks, threads, iters, d);
    const double fl1 = 2.0 * 8 * (double)iters * blocks * threads;
    printf("DFMA: %.2f TFLOP/s\n", fl1 / t1 / 1e12);
    const double t2 = time_kernel(k_dmma, blocks, threads, iters, d);
    const double fl2 = 2.0 * 256 * 8 * (double)iters * blocks * (threads / 32);
    printf("DMMA m8n8k4: %.2f TFLOP/s\n", fl2 / t2 / 1e12);
    const double t3 = time_kernel(k_mixed, blocks, threads, iters, d);
    const double fl3 = 2.0 * 256 * 4 * (double)iters * blocks * (threads / 32) + 2.0 * 16 * (double)iters * blocks * threads;
    printf("mixed 4 DMMA + 16 DFMA per iter: %.2f TFLOP/s total (%.3f ms; DFMA-only equiv %.3f ms, DMMA-only equiv %.3f ms)\n",
           fl3 / t3 / 1e12, t3 * 1e3, 2.0 * 16 * (double)iters * blocks * threads / (fl1 / t1) * 1e3,
           2.0 * 256 * 4 * (double)iters * blocks * (threads / 32) / (fl2 / t2) * 1e3);
    return 0;
}

// ---- MUFU.RSQ64H throughput and alternative seeds (appended experiments)
__global__ void k_mufu64(double* out, int iters)
{
    double a[8];
    for (int q = 0; q < 8; ++q) a[q] = 1.0 + threadIdx.x * 1e-6 + q;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int q = 0; q < 8; ++q) a[q] = rsq_seed(a[q]) + 1.0;
    double s = 0;
    for (int q = 0; q < 8; ++q) s += a[q];
    if (s == 1.2345) out[0] = s;
}
__global__ void k_mufu32cvt(double* out, int iters)
{
    double a[8];
    for (int q = 0; q < 8; ++q) a[q] = 1.0 + threadIdx.x * 1e-6 + q;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int q = 0; q < 8; ++q) a[q] = (double)rsqrtf((float)a[q]) + 1.0;
    double s = 0;
    for (int q = 0; q < 8; ++q) s += a[q];
    if (s == 1.2345) out[0] = s;
}
// full evaluation as in the far kernel: 4 FP64 for r2 + refined rsqrt + accumulate
__global__ void k_eval(double* out, int iters)
{
    double acc[8], x[8];
    for (int q = 0; q < 8; ++q) {
        acc[q] = 0;
        x[q] = 1.0 + threadIdx.x * 1e-6 + q;
    }
    const double y = 0.3, w = 0.7;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const double r2 = fma(x[q], y, fma(x[q], y, fma(x[q], y, x[q] + 2.0)));
            acc[q] = fma(w, rsq3(r2), acc[q]);
        }
    double s = 0;
    for (int q = 0; q < 8; ++q) s += acc[q];
    if (s == 1.2345) out[0] = s;
}
int main2()
{
    double* d;
    cudaMalloc(&d, 64);
    const int blocks = 148 * 8, threads = 256, iters = 2048;
    const double n = 8.0 * iters * blocks * threads;
    double t = time_kernel(k_mufu64, blocks, threads, iters, d);
    printf("MUFU.RSQ64H (+DADD): %.2f /clk/SM at 1.965 GHz\n", n / t / 148 / 1.965e9);
    t = time_kernel(k_mufu32cvt, blocks, threads, iters, d);
    printf("F2F+MUFU.RSQ+F2F (+DADD): %.2f /clk/SM\n", n / t / 148 / 1.965e9);
    t = time_kernel(k_eval, blocks, threads, iters, d);
    printf("full eval (10 FP64 + MUFU): %.2f evals/clk/SM (FP64 bound would be 6.4)\n", n / t / 148 / 1.965e9);
    return 0;
}
int main()
{
    main1();
    main2();
    return 0;
}
