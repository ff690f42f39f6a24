// Ceiling of the quadrature evaluation pattern (not part of the library): P x points in
// registers as (-2x, |x|^2), y points (y, |y|^2) streamed from shared memory, one
// accumulator per x point, refined rsqrt (MUFU.RSQ64H + 3rd-order step).  10 FP64
// instructions per evaluation, so 6.4 evaluations/clk/SM is the FP64-pipe bound.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro_eval tools/micro_eval.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double rsqrt_fast(double r2)
{
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
    const double h = r2 * y;
    const double e = fma(-h, y, 1.0);
    const double c = fma(0.375, e, 0.5);
    return fma(y, e * c, y);
}

// 1/r = y0 (15/8 - 5/4 q + 3/8 q^2), q = r2 y0^2 (the same 3rd-order step as rsqrt_fast),
// with the y weight folded into r2 (r2' = r2 / w^2, so rsqrt(r2') = w / r): the final
// multiply by y0 merges with the accumulation -> 4 + 5 = 9 FP64 instructions per evaluation
__device__ __forceinline__ double rsqrt_poly_acc(double r2, double acc)
{
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
    const double q = (r2 * y) * y;
    const double p = fma(fma(q, 0.375, -1.25), q, 1.875);
    return fma(y, p, acc);
}

// the library's form (kernels.cuh rsqrt_acc): y (1 + e (1/2 + 3e/8)) accumulated, 5 FP64 after the seed
__device__ __forceinline__ double rsqrt_acc(double r2s, double acc)
{
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2s));
    const double h = r2s * y;
    const double e = fma(-h, y, 1.0);
    const double c = fma(0.375, e, 0.5);
    return fma(y, fma(e, c, 1.0), acc);
}

template <int P, int UNROLL, int MODE = 0>
__global__ void k_eval(double* out, int reps)
{
    __shared__ double4 Y[16];
    if (threadIdx.x < 16) {
        const double v = 0.1 * threadIdx.x;
        Y[threadIdx.x] = make_double4(v, 0.5 - v, 0.25 * v, 3.0 + v * v);
    }
    __syncthreads();
    double mx[P], my[P], mz[P], x2[P], a[P];
#pragma unroll
    for (int r = 0; r < P; ++r) {
        const double x = 1.0 + 1e-3 * (threadIdx.x + r);
        mx[r] = -2.0 * x;
        my[r] = -1.0 * x;
        mz[r] = -0.5 * x;
        x2[r] = x * x * 1.3125;
        a[r] = 0.0;
    }
    for (int it = 0; it < reps; ++it) {
#pragma unroll UNROLL
        for (int j = 0; j < 16; ++j) {
            const double4 y = Y[j];
            const double wj = 0.01 * (j + 1);
#pragma unroll
            for (int r = 0; r < P; ++r) {
                if (MODE == 0) {
                    const double r2 = fma(mx[r], y.x, fma(my[r], y.y, fma(mz[r], y.z, x2[r] + y.w)));
                    a[r] = fma(wj, rsqrt_fast(r2), a[r]);
                } else if (MODE == 2) {  // timing probe: the MUFU replaced by an INT-pipe seed
                    const double r2 = fma(mx[r], y.x, fma(my[r], y.y, fma(mz[r], y.z, x2[r] + y.w)));
                    const double y0 = __hiloint2double(0x5fe6eb50 - (__double2hiint(r2) >> 1), 0);
                    const double hh = r2 * y0;
                    const double e = fma(-hh, y0, 1.0);
                    const double c = fma(0.375, e, 0.5);
                    a[r] = fma(wj, fma(y0, e * c, y0), a[r]);
                } else if (MODE == 3) {  // library form, 3-D: 9 FP64 per evaluation
                    const double r2 = fma(mx[r], y.x, fma(my[r], y.y, fma(mz[r], y.z, fma(x2[r], wj, y.w))));
                    a[r] = rsqrt_acc(r2, a[r]);
                } else if (MODE == 4) {  // library form, flat (one coordinate plane): 8 FP64
                    const double r2 = fma(mx[r], y.x, fma(my[r], y.y, fma(x2[r], wj, y.w)));
                    a[r] = rsqrt_acc(r2, a[r]);
                } else {  // y = (y / w^2, |y|^2 / w^2), wj = 1 / w^2
                    const double r2 = fma(mx[r], y.x, fma(my[r], y.y, fma(mz[r], y.z, fma(x2[r], wj, y.w))));
                    a[r] = rsqrt_poly_acc(r2, a[r]);
                }
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int r = 0; r < P; ++r) s += a[r];
    if (s == 1.2345) out[0] = s;
}

template <int P, int UNROLL, int MODE = 0>
void run(int threads, int ctas_per_sm, double* d, double clk_ghz)
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * ctas_per_sm * 4;
    const int reps = 256;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_eval<P, UNROLL, MODE><<<blocks, threads>>>(d, 4);
    cudaEventRecord(a);
    k_eval<P, UNROLL, MODE><<<blocks, threads>>>(d, reps);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k_eval<P, UNROLL, MODE>);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_eval<P, UNROLL, MODE>, threads, 0);
    const double evals = (double)blocks * threads * reps * 16 * P;
    const double per_clk_sm = evals / (ms * 1e-3) / sms / (clk_ghz * 1e9);
    printf("mode=%d P=%d unroll=%d threads=%d regs=%d resident CTAs/SM=%d : %.2f evals/clk/SM = %.1f%% of the 6.4 FP64 bound"
           " (%.1f TFLOP/s at 20 flop/eval)\n",
           MODE, P, UNROLL, threads, fa.numRegs, occ, per_clk_sm, 100.0 * per_clk_sm / 6.4, evals * 20 / (ms * 1e-3) / 1e12);
}

__global__ void k_mufu(double* out, int reps)
{
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = 1.0 + 1e-3 * (threadIdx.x + k);
    for (int it = 0; it < reps; ++it)
#pragma unroll
        for (int k = 0; k < 8; ++k) asm volatile("rsqrt.approx.ftz.f64 %0, %0;" : "+d"(x[k]));
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 1.2345) out[0] = s;
}

void mufu_rate(double ghz)
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* d;
    cudaMalloc(&d, 64);
    const int blocks = sms * 8, reps = 4096;
    k_mufu<<<blocks, 256>>>(d, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k_mufu<<<blocks, 256>>>(d, reps);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("MUFU.RSQ64H: %.2f per clk per SM\n", (double)blocks * 256 * reps * 8 / (ms * 1e-3) / sms / (ghz * 1e9));
}

__global__ void k_poly_err(double* err, int n)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double x = exp(-13.8 + 27.6 * ((double)i + 0.5) / n);
    const double ex = 1.0 / sqrt(x);
    err[2 * i] = fabs(rsqrt_fast(x) - ex) / ex;
    err[2 * i + 1] = fabs(rsqrt_poly_acc(x, 0.0) - ex) / ex;
}

void poly_error()
{
    const int n = 1 << 22;
    double* e;
    cudaMalloc(&e, (size_t)2 * n * sizeof(double));
    k_poly_err<<<(n + 255) / 256, 256>>>(e, n);
    double* h = new double[(size_t)2 * n];
    cudaMemcpy(h, e, (size_t)2 * n * sizeof(double), cudaMemcpyDeviceToHost);
    double m0 = 0, m1 = 0, s0 = 0, s1 = 0;
    for (int i = 0; i < n; ++i) {
        m0 = fmax(m0, h[2 * i]);
        m1 = fmax(m1, h[2 * i + 1]);
        s0 += h[2 * i];
        s1 += h[2 * i + 1];
    }
    printf("1/r relative error over [1e-6, 1e6]: rsqrt_fast max %.3e mean %.3e; poly max %.3e mean %.3e\n", m0, s0 / n,
           m1, s1 / n);
    cudaFree(e);
    delete[] h;
}

int main()
{
    double* d;
    cudaMalloc(&d, 64);
    int khz = 0;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    const double ghz = khz * 1e-6;
    printf("SM clock attribute %.3f GHz\n", ghz);
    run<2, 4>(256, 4, d, ghz);
    run<3, 4>(256, 3, d, ghz);
    run<4, 2>(256, 3, d, ghz);
    run<4, 4>(256, 3, d, ghz);
    run<4, 2>(128, 6, d, ghz);
    run<6, 2>(256, 2, d, ghz);
    run<8, 1>(256, 2, d, ghz);
    run<8, 2>(256, 2, d, ghz);
    run<4, 2, 1>(256, 3, d, ghz);
    run<4, 4, 1>(256, 3, d, ghz);
    run<4, 2, 1>(128, 6, d, ghz);
    run<6, 2, 1>(256, 2, d, ghz);
    run<8, 2, 1>(256, 2, d, ghz);
    run<4, 2, 2>(256, 3, d, ghz);
    run<4, 2, 3>(256, 3, d, ghz);
    run<4, 2, 4>(256, 3, d, ghz);
    run<4, 4, 4>(256, 3, d, ghz);
    run<4, 2, 4>(256, 4, d, ghz);
    run<6, 2, 4>(256, 2, d, ghz);
    run<8, 2, 4>(256, 2, d, ghz);
    run<4, 2, 4>(128, 8, d, ghz);
    // near-leaf shapes (2 CTAs of 256 per SM): 4 points unroll 3/9, 3 points unroll 3/6/12
    run<4, 3, 4>(256, 2, d, ghz);
    run<4, 9, 4>(256, 2, d, ghz);
    run<3, 3, 4>(256, 2, d, ghz);
    run<3, 6, 4>(256, 2, d, ghz);
    run<3, 12, 4>(256, 2, d, ghz);
    run<6, 3, 4>(256, 2, d, ghz);
    run<8, 2, 2>(256, 2, d, ghz);
    mufu_rate(ghz);
    poly_error();
    return 0;
}
