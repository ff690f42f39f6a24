// Context, timers and dense-matrix utilities.
#include <cstdlib>
#include "common.cuh"
#include <atomic>
#include <chrono>
#include <cstring>
#include <sys/mman.h>
#include <condition_variable>
#include <list>
#include <mutex>
#include <set>
#include <tuple>
#include <thread>
#include <vector>

#include "kernels.cuh"

namespace sbg {

namespace {
std::atomic<long long> g_launches{0};
}
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void add_launches(long long k) { g_launches.fetch_add(k, std::memory_order_relaxed); }
bool pcg_graph_enabled()
{
    static const bool on = [] {
        const char* e = getenv("SBG_PCG_GRAPH");
        return !(e && e[0] == '0');
    }();
    return on;
}

void device_pool_init(int device)
{
    cudaMemPool_t pool;
    SBG_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    unsigned long long keep = ~0ull;
    SBG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
}

namespace {
constexpr size_t kCacheMin = size_t(64) << 20;   // smaller blocks come from the pool quickly
constexpr size_t kCacheCap = size_t(16) << 30;   // bytes parked at most (oldest freed first)
struct BlockCache {
    std::mutex mu;
    struct Block {
        void* p;
        size_t bytes;
        int device;
    };
    std::list<Block> blocks;  // oldest first
    size_t total = 0;
    cudaEvent_t mark = nullptr;
};
BlockCache& block_cache()
{
    static BlockCache* c = new BlockCache;  // never destroyed: no CUDA calls during static teardown
    return *c;
}
}  // namespace

void* device_alloc(size_t bytes)
{
    if (bytes >= kCacheMin) {
        int dev = 0;
        SBG_CUDA(cudaGetDevice(&dev));
        BlockCache& C = block_cache();
        std::lock_guard<std::mutex> lk(C.mu);
        for (auto it = C.blocks.begin(); it != C.blocks.end(); ++it)
            if (it->bytes == bytes && it->device == dev) {
                void* p = it->p;
                C.total -= bytes;
                C.blocks.erase(it);
                return p;
            }
    }
    void* p = nullptr;
    SBG_CUDA(cudaMallocAsync(&p, bytes, 0));
    return p;
}

void device_free(void* p)
{
    if (p) cudaFreeAsync(p, 0);
}

// A parked block may still be read by work in flight on a context stream.  The context
// streams are blocking streams: an event recorded on the legacy stream at park time begins
// only after all their earlier work, and any work issued to them later (by the block's next
// owner) waits for it — so the next owner is ordered after every earlier use.
void device_free_sized(void* p, size_t bytes)
{
    if (!p) return;
    if (bytes < kCacheMin) {
        cudaFreeAsync(p, 0);
        return;
    }
    int dev = 0;
    BlockCache& C = block_cache();
    std::lock_guard<std::mutex> lk(C.mu);
    if (cudaGetDevice(&dev) != cudaSuccess ||
        (!C.mark && cudaEventCreateWithFlags(&C.mark, cudaEventDisableTiming) != cudaSuccess) ||
        cudaEventRecord(C.mark, 0) != cudaSuccess) {
        cudaFreeAsync(p, 0);
        return;
    }
    C.blocks.push_back({p, bytes, dev});
    C.total += bytes;
    while (C.total > kCacheCap && !C.blocks.empty()) {
        const BlockCache::Block b = C.blocks.front();
        C.blocks.pop_front();
        C.total -= b.bytes;
        int cur = 0;
        cudaGetDevice(&cur);
        if (b.device != cur) cudaSetDevice(b.device);
        cudaFreeAsync(b.p, 0);
        if (b.device != cur) cudaSetDevice(cur);
    }
}

void device_cache_release()
{
    BlockCache& C = block_cache();
    std::lock_guard<std::mutex> lk(C.mu);
    int cur = 0;
    cudaGetDevice(&cur);
    for (const auto& b : C.blocks) {
        if (b.device != cur) cudaSetDevice(b.device);
        cudaFreeAsync(b.p, 0);
        if (b.device != cur) cudaSetDevice(cur);
    }
    C.blocks.clear();
    C.total = 0;
}
long long launch_count() { return g_launches.load(); }

cudaEvent_t Timers::get()
{
    if (!pool.empty()) {
        cudaEvent_t e = pool.back();
        pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    SBG_CUDA(cudaEventCreate(&e));
    return e;
}

void Timers::collect()
{
    for (auto& p : pending) {
        SBG_CUDA(cudaEventSynchronize(p.b));
        float ms = 0;
        SBG_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
        bool found = false;
        for (auto& t : totals)
            if (t.first == p.name) {
                t.second.first += ms;
                t.second.second += 1;
                found = true;
            }
        if (!found) totals.push_back({p.name, {ms, 1}});
        pool.push_back(p.a);
        pool.push_back(p.b);
    }
    pending.clear();
}

void Timers::reset()
{
    collect();
    totals.clear();
}

void Timers::add(const std::string& name, double ms)
{
    for (auto& t : totals)
        if (t.first == name) {
            t.second.first += ms;
            t.second.second += 1;
            return;
        }
    totals.push_back({name, {ms, 1}});
}

static double now_ms()
{
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

HostScope::HostScope(Ctx* c, const char* n) : ctx(c), name(n), t0(now_ms()) {}

HostScope::~HostScope()
{
    if (ctx && ctx->timers.enabled) ctx->timers.add(name, now_ms() - t0);
}

Timers::~Timers()
{
    for (auto& p : pending) {
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    for (auto e : pool) cudaEventDestroy(e);
}

Ctx::~Ctx()
{
    // the cached workspaces first (their large buffers go to the block cache), then the cache
    pcg_ws.reset();
    dl_ws.reset();
    near_ws.reset();
    flush_ws.reset();
    prec_sched.reset();
    scratch_ws.reset();
    sauter_ws.reset();
    stage_ws.reset();
    device_cache_release();
    if (aux) {
        cudaStreamSynchronize(aux);
        cudaStreamDestroy(aux);
    }
    if (stream) {
        cudaStreamSynchronize(stream);
        cudaStreamDestroy(stream);
    }
}

// a blocking stream too, so the stream-ordered pool's legacy-stream allocations order
// against it (common.cuh)
cudaStream_t aux_stream(Ctx* ctx, int which)
{
    cudaStream_t& st = which == 0 ? ctx->aux : ctx->aux2;
    if (!st) {
        int least = 0, greatest = 0;
        SBG_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        SBG_CUDA(cudaStreamCreateWithPriority(&st, cudaStreamDefault, least));
    }
    return st;
}

TimedScope::TimedScope(Ctx* c, const char* n) : ctx(c), name(n)
{
    if (ctx && ctx->timers.enabled) {
        a = ctx->timers.get();
        SBG_CUDA(cudaEventRecord(a, ctx->stream));
    }
}

TimedScope::~TimedScope()
{
    if (a) {
        cudaEvent_t b = ctx->timers.get();
        cudaEventRecord(b, ctx->stream);
        ctx->timers.pending.push_back({name, a, b});
    }
}

// ---------------------------------------------------------------- matrix utilities
namespace {

__global__ void k_pack_rows(const double* __restrict__ src, int n, double* __restrict__ dst, int ld)
{
    // src row-major n x n -> dst row-major n x ld
    const size_t i = blockIdx.y;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
        dst[i * ld + j] = src[i * (size_t)n + j];
}

__global__ void k_unpack_rows(const double* __restrict__ src, int ld, int n, double* __restrict__ dst)
{
    const size_t i = blockIdx.y;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
        dst[i * (size_t)n + j] = src[i * ld + j];
}

__global__ void k_gather_rows(const double* __restrict__ src, int ld, int n, const int* __restrict__ rows,
                              double* __restrict__ dst)
{
    const size_t r = blockIdx.y;
    const size_t i = rows[r];
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
        dst[r * n + j] = src[i * ld + j];
}

// the upper triangle (j >= i) of a symmetric W as one contiguous vector: row i at
// i n - i (i - 1) / 2, columns i..n-1 (half the bytes of a multi-GPU reduction of W)
__device__ __forceinline__ size_t upper_off(size_t i, size_t n) { return i * n - i * (i - 1) / 2; }
__global__ void k_pack_upper(const double* __restrict__ W, int ld, int n, double* __restrict__ out)
{
    const size_t i = blockIdx.y;
    double* row = out + upper_off(i, n) - i;
    for (int j = (int)i + blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
        row[j] = W[i * ld + j];
}
// W(i, j) = W(j, i) = packed(i, j) for j >= i
__global__ void k_unpack_upper(const double* __restrict__ in, int ld, int n, double* __restrict__ W)
{
    const size_t i = blockIdx.y;
    const double* row = in + upper_off(i, n) - i;
    for (int j = (int)i + blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const double v = row[j];
        W[i * ld + j] = v;
        W[(size_t)j * ld + i] = v;
    }
}

// max |W(i,j) - W(j,i)| over the upper triangle, per-block maxima
__global__ void k_symmetry_defect(const double* __restrict__ a, int ld, int n, double* __restrict__ out)
{
    __shared__ double red[256];
    double m = 0;
    const int i = blockIdx.y;
    for (int j = i + 1 + blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
        m = fmax(m, fabs(a[(size_t)i * ld + j] - a[(size_t)j * ld + i]));
    red[threadIdx.x] = m;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
        __syncthreads();
    }
    if (threadIdx.x == 0) out[(size_t)i * gridDim.x + blockIdx.x] = red[0];
}

}  // namespace

void set_max_dynamic_smem(const void* kernel, size_t bytes)
{
    static std::mutex mu;
    static std::set<std::tuple<const void*, int, size_t>> done;
    int dev = 0;
    SBG_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    if (done.count({kernel, dev, bytes})) return;
    SBG_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    done.insert({kernel, dev, bytes});
}

void matrix_alloc(Ctx* ctx, int n, DMatrix& M)
{
    M.ctx = ctx;
    M.n = n;
    M.ld = DMatrix::padded_ld(n);
    M.a.alloc((size_t)n * M.ld);
    if (M.a.n) SBG_CUDA(cudaMemsetAsync(M.a.p, 0, M.a.n * sizeof(double), ctx->stream));
}

void matrix_upload(DMatrix& M, const double* host)
{
    Ctx* ctx = M.ctx;
    const size_t rows_per = std::max<size_t>(1, (64u << 20) / (sizeof(double) * std::max(1, M.n)));
    DBuf<double> stage(std::min<size_t>(rows_per, M.n) * M.n);
    for (int r0 = 0; r0 < M.n; r0 += (int)rows_per) {
        const int r1 = std::min<int>(M.n, r0 + (int)rows_per);
        SBG_CUDA(cudaMemcpyAsync(stage.p, host + (size_t)r0 * M.n, (size_t)(r1 - r0) * M.n * sizeof(double),
                                 cudaMemcpyHostToDevice, ctx->stream));
        dim3 grid((M.n + 255) / 256 < 64 ? (M.n + 255) / 256 : 64, r1 - r0);
        k_pack_rows<<<grid, 256, 0, ctx->stream>>>(stage.p, M.n, M.a.p + (size_t)r0 * M.ld, M.ld); ::sbg::count_launch();
        SBG_LAUNCH_CHECK();
    }
    SBG_CUDA(cudaStreamSynchronize(ctx->stream));
}

namespace {
// Pinned staging ring for full-matrix downloads: the padded rows are packed on
// the device, DMA'd into pinned slots, and copied out by host threads while the
// next slots are in flight (a pageable D2H of a 5 GB matrix runs at a few GB/s).
struct DownloadRing {
    static constexpr int kSlots = 8;
    static constexpr size_t kSlotBytes = 32u << 20;
    double* pinned[kSlots] = {};
    DBuf<double> dev[kSlots];
    cudaEvent_t done[kSlots] = {};
    DownloadRing()
    {
        for (int k = 0; k < kSlots; ++k) {
            SBG_CUDA(cudaHostAlloc((void**)&pinned[k], kSlotBytes, cudaHostAllocDefault));
            dev[k].alloc(kSlotBytes / sizeof(double));
            // blocking sync: the waiting host thread sleeps instead of spinning on a core
            // the copy threads need
            SBG_CUDA(cudaEventCreateWithFlags(&done[k], cudaEventDisableTiming | cudaEventBlockingSync));
        }
    }
    ~DownloadRing()
    {
        for (int k = 0; k < kSlots; ++k) {
            if (pinned[k]) cudaFreeHost(pinned[k]);
            if (done[k]) cudaEventDestroy(done[k]);
        }
    }
};
}  // namespace

// Full download of the unpadded row-major matrix.  The device packs up to kSlots
// chunks ahead into pinned slots; copy threads move disjoint slices of each chunk
// into the destination (the first touch of a fresh destination costs page faults:
// ~2 GB/s per thread with 4 KB pages, ~47 GB/s over 16 threads with huge pages on
// the B200 hosts), and a slot is refilled once every thread is done with it.
namespace {
__global__ void k_l2_read(const double4* __restrict__ src, size_t n, double* __restrict__ sink)
{
    double s = 0.0;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const double4 v = src[i];
        s += v.x + v.y + v.z + v.w;
    }
    if (s == 1.2345e-300) sink[0] = s;  // never true for the zero-filled buffer; keeps the loads
}
}  // namespace

double* scratch(Ctx* ctx, int slot, size_t count)
{
    struct Scratch {
        DBuf<double> b[kScratchSlots];
    };
    if (!ctx->scratch_ws) ctx->scratch_ws = std::make_shared<Scratch>();
    DBuf<double>& b = static_cast<Scratch*>(ctx->scratch_ws.get())->b[slot];
    if (b.n < count) b.alloc(count + count / 8);
    return b.p;
}

void l2_flush(Ctx* ctx)
{
    const size_t bytes = 256u << 20;
    if (!ctx->flush_ws) {
        auto bufs = std::make_shared<DBuf<double>>(2 * bytes / sizeof(double));
        SBG_CUDA(cudaMemsetAsync(bufs->p, 0, 2 * bytes, ctx->stream));
        ctx->flush_ws = bufs;
    }
    auto* b = static_cast<DBuf<double>*>(ctx->flush_ws.get());
    SBG_CUDA(cudaMemsetAsync(b->p, 0, bytes, ctx->stream));
    k_l2_read<<<4 * ctx->sm_count, 256, 0, ctx->stream>>>(reinterpret_cast<const double4*>(b->p + bytes / 8),
                                                          bytes / sizeof(double4), b->p);
    SBG_LAUNCH_CHECK();  // not counted in launch_count(): measurement scaffolding, not the hot path
}

void matrix_download(const DMatrix& M, double* host)
{
    Ctx* ctx = M.ctx;
    if (M.n == 0) return;
    if (!ctx->dl_ws) ctx->dl_ws = std::make_shared<DownloadRing>();
    auto& R = *static_cast<DownloadRing*>(ctx->dl_ws.get());
    const size_t row_bytes = sizeof(double) * (size_t)M.n;
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, host) == cudaSuccess && pa.type == cudaMemoryTypeHost) {
        // page-locked destination (sbg_host_alloc / cudaHostRegister): one pitched DMA straight into it
        SBG_CUDA(cudaMemcpy2DAsync(host, row_bytes, M.a.p, sizeof(double) * (size_t)M.ld, row_bytes, M.n,
                                   cudaMemcpyDeviceToHost, ctx->stream));
        SBG_CUDA(cudaStreamSynchronize(ctx->stream));
        return;
    }
    (void)cudaGetLastError();  // a pageable pointer is not an error
    if (row_bytes > DownloadRing::kSlotBytes) {  // n > 4M: row by row through pageable copies
        for (int r = 0; r < M.n; ++r)
            SBG_CUDA(cudaMemcpyAsync(host + (size_t)r * M.n, M.a.p + (size_t)r * M.ld, row_bytes,
                                     cudaMemcpyDeviceToHost, ctx->stream));
        SBG_CUDA(cudaStreamSynchronize(ctx->stream));
        return;
    }
    const int rows_per = (int)(DownloadRing::kSlotBytes / row_bytes);
    const int nchunks = (M.n + rows_per - 1) / rows_per;
    const unsigned hw = std::thread::hardware_concurrency() ? std::thread::hardware_concurrency() : 1u;
    const int nthreads = (int)std::max(1u, std::min(16u, hw));  // including the calling thread
    {
        // fresh destinations: ask for transparent huge pages (advisory only)
        const uintptr_t a = reinterpret_cast<uintptr_t>(host), e = a + (size_t)M.n * row_bytes;
        const uintptr_t huge = 2u << 20, lo = (a + huge - 1) & ~(huge - 1), hi = e & ~(huge - 1);
        if (hi > lo + 16 * huge) madvise(reinterpret_cast<void*>(lo), hi - lo, MADV_HUGEPAGE);
    }
    auto enqueue = [&](int i) {
        const int slot = i % DownloadRing::kSlots;
        const int r0 = i * rows_per, r1 = std::min(M.n, r0 + rows_per);
        dim3 grid((M.n + 255) / 256 < 64 ? (M.n + 255) / 256 : 64, r1 - r0);
        k_unpack_rows<<<grid, 256, 0, ctx->stream>>>(M.a.p + (size_t)r0 * M.ld, M.ld, M.n, R.dev[slot].p);
        ::sbg::count_launch();
        SBG_LAUNCH_CHECK();
        SBG_CUDA(cudaMemcpyAsync(R.pinned[slot], R.dev[slot].p, (size_t)(r1 - r0) * row_bytes, cudaMemcpyDeviceToHost,
                                 ctx->stream));
        SBG_CUDA(cudaEventRecord(R.done[slot], ctx->stream));
    };
    auto copy_slice = [&](int i, int t) {
        const int r0 = i * rows_per, r1 = std::min(M.n, r0 + rows_per);
        const size_t total = (size_t)(r1 - r0) * M.n;
        const size_t lo = total * t / nthreads, hi = total * (t + 1) / nthreads;
        std::memcpy(host + (size_t)r0 * M.n + lo, R.pinned[i % DownloadRing::kSlots] + lo, (hi - lo) * sizeof(double));
    };
    // Copy threads run through the chunks independently (no per-chunk barrier); the
    // calling thread refills a slot once every thread has copied its chunk out.
    std::mutex mu;
    std::condition_variable cv_posted, cv_done;
    int posted = 0;
    bool failed = false;
    std::vector<int> finished(nchunks, 0);
    auto worker = [&](int t) {
        for (int i = 0; i < nchunks; ++i) {
            {
                std::unique_lock<std::mutex> lk(mu);
                cv_posted.wait(lk, [&] { return failed || posted > i; });
                if (failed) return;
            }
            if (cudaEventSynchronize(R.done[i % DownloadRing::kSlots]) != cudaSuccess) {
                std::lock_guard<std::mutex> lk(mu);
                failed = true;
                cv_done.notify_all();
                cv_posted.notify_all();
                return;
            }
            copy_slice(i, t);
            std::lock_guard<std::mutex> lk(mu);
            if (++finished[i] == nthreads) cv_done.notify_all();
        }
    };
    std::vector<std::thread> pool;
    auto shutdown = [&](bool fail) {
        if (fail) {
            std::lock_guard<std::mutex> lk(mu);
            failed = true;
        }
        cv_posted.notify_all();
        for (auto& th : pool) th.join();
    };
    try {
        for (int i = 0; i < std::min(nchunks, DownloadRing::kSlots); ++i) enqueue(i);
        posted = std::min(nchunks, DownloadRing::kSlots);
        for (int t = 0; t < nthreads; ++t) pool.emplace_back(worker, t);
        for (int i = DownloadRing::kSlots; i < nchunks; ++i) {
            {
                std::unique_lock<std::mutex> lk(mu);
                cv_done.wait(lk, [&] { return failed || finished[i - DownloadRing::kSlots] == nthreads; });
                if (failed) break;
            }
            enqueue(i);
            {
                std::lock_guard<std::mutex> lk(mu);
                posted = i + 1;
            }
            cv_posted.notify_all();
        }
    } catch (...) {
        shutdown(true);
        throw;
    }
    shutdown(false);
    if (failed) throw CudaError("matrix download: event synchronisation failed");
}

void matrix_download_rows(const DMatrix& M, const int* rows, int nrows, double* host)
{
    Ctx* ctx = M.ctx;
    for (int r : std::vector<int>(rows, rows + nrows))
        if (r < 0 || r >= M.n) throw ValidationError("row index out of range");
    DBuf<int> d_rows(nrows);
    d_rows.upload(rows, nrows, ctx->stream);
    DBuf<double> out((size_t)nrows * M.n);
    dim3 grid((M.n + 255) / 256 < 64 ? (M.n + 255) / 256 : 64, nrows);
    k_gather_rows<<<grid, 256, 0, ctx->stream>>>(M.a.p, M.ld, M.n, d_rows.p, out.p); ::sbg::count_launch();
    SBG_LAUNCH_CHECK();
    SBG_CUDA(cudaMemcpyAsync(host, out.p, (size_t)nrows * M.n * sizeof(double), cudaMemcpyDeviceToHost,
                             ctx->stream));
    SBG_CUDA(cudaStreamSynchronize(ctx->stream));
}

void matrix_pack_upper(const DMatrix& M, double* d_packed)
{
    if (M.n == 0) return;
    k_pack_upper<<<dim3(8, M.n), 256, 0, M.ctx->stream>>>(M.a.p, M.ld, M.n, d_packed);
    ::sbg::count_launch();
    SBG_LAUNCH_CHECK();
}
void matrix_unpack_upper(DMatrix& M, const double* d_packed)
{
    if (M.n == 0) return;
    k_unpack_upper<<<dim3(8, M.n), 256, 0, M.ctx->stream>>>(d_packed, M.ld, M.n, M.a.p);
    ::sbg::count_launch();
    SBG_LAUNCH_CHECK();
}

double matrix_symmetry_defect(const DMatrix& M)
{
    Ctx* ctx = M.ctx;
    if (M.n < 2) return 0.0;
    const int gx = 8;
    DBuf<double> part((size_t)M.n * gx);
    k_symmetry_defect<<<dim3(gx, M.n), 256, 0, ctx->stream>>>(M.a.p, M.ld, M.n, part.p); ::sbg::count_launch();
    SBG_LAUNCH_CHECK();
    std::vector<double> h(part.n);
    SBG_CUDA(cudaMemcpyAsync(h.data(), part.p, h.size() * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    SBG_CUDA(cudaStreamSynchronize(ctx->stream));
    double m = 0;
    for (double v : h) m = std::max(m, v);
    return m;
}

}  // namespace sbg

// ---------------------------------------------------------------- FP64 peak probe
namespace sbg {
namespace {
__global__ void k_dfma_peak(double* out, int iters)
{
    double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-9, a2 = a0 + 2e-9, a3 = a0 + 3e-9;
    double a4 = a0 + 4e-9, a5 = a0 + 5e-9, a6 = a0 + 6e-9, a7 = a0 + 7e-9;
    const double b = 0.999999999, c = 1e-12;
    for (int i = 0; i < iters; ++i) {
        a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
        a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
    const double s = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
    if (s == 12345.678) out[0] = s;
}
}  // namespace

// measured DFMA throughput (TFLOP/s, 2 flop per FMA) over a ~50 ms launch
double fp64_peak_tflops(Ctx* ctx)
{
    DBuf<double> out(1);
    const int blocks = ctx->sm_count * 8, threads = 256, iters = 1 << 14;
    cudaEvent_t a, b;
    SBG_CUDA(cudaEventCreate(&a));
    SBG_CUDA(cudaEventCreate(&b));
    k_dfma_peak<<<blocks, threads, 0, ctx->stream>>>(out.p, 1024);  // warm-up
    count_launch();
    SBG_CUDA(cudaEventRecord(a, ctx->stream));
    k_dfma_peak<<<blocks, threads, 0, ctx->stream>>>(out.p, iters);
    count_launch();
    SBG_CUDA(cudaEventRecord(b, ctx->stream));
    SBG_CUDA(cudaEventSynchronize(b));
    float ms = 0;
    SBG_CUDA(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    const double flops = 2.0 * 8.0 * (double)iters * blocks * threads;
    return flops / (ms * 1e-3) / 1e12;
}
}  // namespace sbg
