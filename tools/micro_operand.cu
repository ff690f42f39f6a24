// Register-operand bandwidth of the FP64 pipe on sm_100a (not part of the library): the same
// DFMA count per thread with 1, 2 or 3 distinct 64-bit REGISTER operands per instruction (the
// others immediates or operands the previous instruction of the warp already read in the same
// slot).  The quadrature evaluation (kernels.cuh rsqrt_acc + the distance expansion) reads
// 18 64-bit registers in its 8 DFMA/DMUL; if the pipe takes one 64-bit operand per cycle and
// SM sub-partition, that evaluation cannot go faster than 18 cycles per warp, i.e. 89% of the
// 16 cycles its 8 instructions take at the DFMA-only rate.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro_operand tools/micro_operand.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 8;  // independent chains per thread

// MODE 1: a = fma(a, K1, K2) (one register operand, two immediates)
// MODE 2: a_i = fma(a_i, b, c): b, c shared by all chains (reuse across consecutive instructions)
// MODE 3: a_i = fma(b_i, c_i, a_i): three distinct registers per instruction, nothing shared
// MODE 4: a_i = fma(b_i, c, a_i): two distinct registers + one shared
// MODE 5: a_i = fma(b_i, b_i, a_i): two distinct registers, one of them in two slots
// MODE 6: a_i = fma(b_i, K, a_i): two distinct registers + an immediate
template <int MODE>
__global__ void __launch_bounds__(256) k_dfma(double* out, const double* in, int reps)
{
    double a[CH], b[CH], c[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) {
        a[i] = in[threadIdx.x + i];
        b[i] = in[threadIdx.x + 64 + i];
        c[i] = in[threadIdx.x + 128 + i];
    }
    for (int it = 0; it < reps; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
#pragma unroll
            for (int i = 0; i < CH; ++i) {
                if (MODE == 1) a[i] = fma(a[i], 0.999999, 1e-7);
                else if (MODE == 2) a[i] = fma(a[i], b[0], c[0]);
                else if (MODE == 3) a[i] = fma(b[i], c[i], a[i]);
                else if (MODE == 4) a[i] = fma(b[i], c[0], a[i]);
                else if (MODE == 5) a[i] = fma(b[i], b[i], a[i]);
                else a[i] = fma(b[i], 0.999999, a[i]);
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) s += a[i] + b[i] + c[i];
    if (s == 1.2345) out[0] = s;
}

template <int MODE>
void run(const char* what, double* d, const double* in, double clk_ghz, int ctas)
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * ctas, threads = 256, reps = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_dfma<MODE><<<blocks, threads>>>(d, in, 16);
    cudaEventRecord(e0);
    k_dfma<MODE><<<blocks, threads>>>(d, in, reps);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double inst = (double)blocks * threads * reps * 8 * CH;
    const double per_clk_sm = inst / (ms * 1e-3) / sms / (clk_ghz * 1e9);
    printf("mode %d (%s), %d CTAs/SM: %.1f DFMA/clk/SM = %.1f%% of 64, %.1f TFLOP/s\n", MODE, what, ctas, per_clk_sm,
           100.0 * per_clk_sm / 64.0, 2 * inst / (ms * 1e-3) / 1e12);
}

int main()
{
    int khz = 0;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    const double ghz = khz * 1e-6;
    double *d, *in;
    cudaMalloc(&d, 8);
    cudaMalloc(&in, 8 * 512);
    double h[512];
    for (int i = 0; i < 512; ++i) h[i] = 1.0 + 1e-6 * i;
    cudaMemcpy(in, h, sizeof h, cudaMemcpyHostToDevice);
    printf("SM clock %.3f GHz (attribute)\n", ghz);
    for (int ctas : {2, 4}) {
        run<1>("1 register + 2 immediates", d, in, ghz, ctas);
        run<2>("1 register + 2 shared registers", d, in, ghz, ctas);
        run<4>("2 registers + 1 shared register", d, in, ghz, ctas);
        run<6>("2 registers + 1 immediate", d, in, ghz, ctas);
        run<5>("2 registers, one in two slots", d, in, ghz, ctas);
        run<3>("3 distinct registers", d, in, ghz, ctas);
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("CUDA error: %s\n", cudaGetErrorString(e));
        return 1;
    }
    return 0;
}
