// Shared device-side infrastructure for the sm_100a screenbem path.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "../host/host.hpp"

namespace sbg {

#define SBG_CUDA(call)                                                                              \
    do {                                                                                            \
        cudaError_t _e = (call);                                                                    \
        if (_e != cudaSuccess)                                                                      \
            throw ::sbg::CudaError(std::string(#call) + ": " + cudaGetErrorString(_e) + " (" __FILE__ \
                                   ":" + std::to_string(__LINE__) + ")");                           \
    } while (0)

#define SBG_LAUNCH_CHECK() SBG_CUDA(cudaGetLastError())

constexpr int kNumSMs = 148;  // B200 (2 dies x 74); queried at runtime as well

// Number of kernels this library has launched (bench evidence: gpu_launches).
void count_launch();
long long launch_count();

// Device buffer owned by the host object (RAII, stream-ordered free not needed:
// objects are destroyed after a context synchronize).
// Device memory comes from the device's stream-ordered pool, allocated and freed
// on the legacy default stream: every context stream is a blocking stream, so a
// free is ordered after all work already queued on them and an allocation before
// all work queued after it.  The pool keeps freed memory (release threshold
// = max), so steady-state allocations make no driver calls (a plain cudaMalloc /
// cudaFree pair costs ~2-4 ms on the B200 boxes and synchronises the device).
void* device_alloc(size_t bytes);
void device_free(void* p);
// frees a block of known size: blocks of >= 64 MB are parked in a process-wide exact-size
// cache (capped) and handed to the next allocation of the same size, so repeated solves of
// one size (a new W, a new preconditioner while the old one is alive) do not make the
// stream-ordered pool map gigabytes again on the host thread (context.cu)
void device_free_sized(void* p, size_t bytes);
void device_cache_release();  // frees every parked block
void device_pool_init(int device);

template <class T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    explicit DBuf(size_t count) { alloc(count); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DBuf& operator=(DBuf&& o) noexcept
    {
        if (this != &o) {
            release();
            p = o.p;
            n = o.n;
            o.p = nullptr;
            o.n = 0;
        }
        return *this;
    }
    ~DBuf() { release(); }
    void alloc(size_t count)
    {
        release();
        if (count) p = static_cast<T*>(device_alloc(count * sizeof(T)));
        n = count;
    }
    void release()
    {
        if (p) device_free_sized(p, n * sizeof(T));
        p = nullptr;
        n = 0;
    }
    void upload(const T* h, size_t count, cudaStream_t s)
    {
        if (count > n) alloc(count);
        if (count) SBG_CUDA(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
    }
    void upload(const std::vector<T>& h, cudaStream_t s) { upload(h.data(), h.size(), s); }
};

// Named CUDA-event timers on the context stream (bench / roofline evidence).
struct Timers {
    struct Pending {
        std::string name;
        cudaEvent_t a, b;
    };
    bool enabled = false;
    std::vector<Pending> pending;
    std::vector<cudaEvent_t> pool;
    std::vector<std::pair<std::string, std::pair<double, long long>>> totals;
    cudaEvent_t get();
    void collect();  // synchronizes on the pending events
    void reset();
    void add(const std::string& name, double ms);  // host-side interval
    ~Timers();
};

struct Ctx {
    int device = 0;
    int sm_count = kNumSMs;
    cudaStream_t stream = nullptr;
    cudaStream_t aux = nullptr;  // second stream for look-ahead overlap (aux_stream(), created on first use)
    cudaStream_t aux2 = nullptr; // third stream: the L^-1 chain beside the factorisation (aux_stream(ctx, 1))
    Timers timers;
    // matrix-vector form of gemv / pcg: 0 = symmetric (reads the upper triangle only, for
    // n >= kSymvMinN), 1 = full-matrix forms (the row kernel the row-panel PCG shares)
    int matvec_form = 0;
    std::shared_ptr<void> pcg_ws;  // cached PCG workspace (linalg.cu)
    std::shared_ptr<void> dl_ws;   // cached pinned download ring (context.cu)
    std::shared_ptr<void> near_ws; // cached near-field frontier buffers (assemble.cu)
    std::shared_ptr<void> flush_ws; // L2 flush buffers (context.cu)
    std::shared_ptr<void> prec_sched; // last preconditioner task schedule (precond.cu)
    std::shared_ptr<void> diag_ws;    // host-copy diagonal patch buffers (assemble.cu)
    std::shared_ptr<void> scratch_ws; // grow-only scratch buffers (context.cu: scratch())
    std::shared_ptr<void> sauter_ws;  // device Sauter rules per singular order (assemble.cu)
    std::shared_ptr<void> stage_ws;   // page-locked staging arena of the plan uploads (assemble.cu)
    ~Ctx();
};

// RAII wall-clock scope for host-side work (recorded only when timing is on).
struct HostScope {
    Ctx* ctx;
    const char* name;
    double t0;
    HostScope(Ctx* c, const char* n);
    ~HostScope();
};

// RAII scope that records a named interval on the context stream when timing is on.
struct TimedScope {
    Ctx* ctx;
    const char* name;
    cudaEvent_t a = nullptr;
    TimedScope(Ctx* c, const char* n);
    ~TimedScope();
};

// Programmatic dependent launch: the next kernel of a dependent chain (the PCG iteration)
// is launched while the previous one drains; it waits in pdl_wait() until its predecessor
// has completed and flushed, so only launch latency and grid tails overlap.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SBG_CUDA(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
}

// Opt a kernel into more than 48 KB of dynamic shared memory, once per (kernel, device).
void set_max_dynamic_smem(const void* kernel, size_t bytes);
template <typename... KArgs>
void set_max_dynamic_smem(void (*kernel)(KArgs...), size_t bytes)
{
    set_max_dynamic_smem(reinterpret_cast<const void*>(kernel), bytes);
}

// Dense symmetric fp64 matrix resident in HBM (GalerkinMatrix, assemble.hpp:12).
// Row-major with a leading dimension padded to 32 doubles (256-byte rows) so
// every row starts 16-byte aligned for 128-bit streaming loads; the padding
// is kept at zero.
struct DMatrix {
    Ctx* ctx = nullptr;
    int n = 0;
    int ld = 0;
    DBuf<double> a;
    static int padded_ld(int n) { return ((n + 31) / 32) * 32; }
};

}  // namespace sbg
