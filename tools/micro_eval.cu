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

template <int P, int UNROLL>
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
                const double r2 = fma(mx[r], y.x, fma(my[r], y.y, fma(mz[r], y.z, x2[r] + y.w)));
                a[r] = fma(wj, rsqrt_fast(r2), a[r]);
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int r = 0; r < P; ++r) s += a[r];
    if (s == 1.2345) out[0] = s;
}

template <int P, int UNROLL>
void run(int threads, int ctas_per_sm, double* d, double clk_ghz)
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * ctas_per_sm * 4;
    const int reps = 256;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_eval<P, UNROLL><<<blocks, threads>>>(d, 4);
    cudaEventRecord(a);
    k_eval<P, UNROLL><<<blocks, threads>>>(d, reps);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k_eval<P, UNROLL>);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_eval<P, UNROLL>, threads, 0);
    const double evals = (double)blocks * threads * reps * 16 * P;
    const double per_clk_sm = evals / (ms * 1e-3) / sms / (clk_ghz * 1e9);
    printf("P=%d unroll=%d threads=%d regs=%d resident CTAs/SM=%d : %.2f evals/clk/SM = %.1f%% of the 6.4 FP64 bound"
           " (%.1f TFLOP/s at 20 flop/eval)\n",
           P, UNROLL, threads, fa.numRegs, occ, per_clk_sm, 100.0 * per_clk_sm / 6.4, evals * 20 / (ms * 1e-3) / 1e12);
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
    return 0;
}
