// Two-level additive Schwarz preconditioner on the device.
// reference: inc/schwarz.hpp:55-140 (blocks, factor_block, build, apply).
//
// All blocks — faces (map order), the wire-basket and the coarse matrix — form
// one batch of dense SPD matrices, factored by a batched right-looking tiled
// Cholesky (64x64 tiles): potrf of the diagonal tile (+ its inverse D_k), a
// "trsm" GEMM A_ik <- A_ik D_k^T and the trailing update A_ij -= A_ik A_jk^T,
// both on the FP64 tensor cores (DMMA, mma.sync.m8n8k4.f64).  The apply runs
// the blocked forward/backward triangular solves of every block in lock-step
// (one launch per tile step), using the inverted diagonal tiles so each step
// is a pair of tile GEMVs.
#include <algorithm>
#include <cmath>

#include "kernels.cuh"

namespace sbg {

namespace {
constexpr int TB = 64;     // tile size
constexpr int TLD = 68;    // padded shared-memory leading dimension (conflict-free DMMA fragments)
}  // namespace

struct Prec {
    Ctx* ctx = nullptr;
    int n = 0, nfaces = 0, nwb = 0, nc = 0;
    int nblocks = 0, coarse_block = -1, Tmax = 0;
    std::vector<int> h_nb, h_T, h_loc, h_Loff, h_Doff;
    DBuf<int> d_nb, d_loc, d_Loff, d_Doff, d_T;
    DBuf<double> L, D, loc;
    DBuf<int> pos;  // dof -> loc index (face/WB), -1 if none
    // R in CSC (restriction, ascending rows) and CSR (prolongation, ascending cols)
    DBuf<int> Rc_ptr, Rc_row, Rr_ptr, Rr_col;
    DBuf<double> Rc_val, Rr_val;
    // trsv tasks (block, tile row) per step
    DBuf<int2> fwd_tasks, bwd_tasks;
    std::vector<int> fwd_off, bwd_off;
    double factor_bytes = 0;
};

namespace {

// ---------------------------------------------------------------- DMMA helper
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// ---------------------------------------------------------------- gather
__global__ void k_gather_blocks(const double* __restrict__ W, int ld, const int* __restrict__ bdofs_ptr,
                                const int* __restrict__ bdofs, const int* __restrict__ Loff, double* __restrict__ L)
{
    const int b = blockIdx.x;
    const int p0 = bdofs_ptr[b], nb = bdofs_ptr[b + 1] - p0;
    double* Lb = L + Loff[b];
    for (int i = blockIdx.y; i < nb; i += gridDim.y) {
        const size_t wi = (size_t)bdofs[p0 + i] * ld;
        for (int j = threadIdx.x; j <= i; j += blockDim.x) Lb[(size_t)i * nb + j] = W[wi + bdofs[p0 + j]];
    }
}

// WR[i][c] = sum_{r in col c} W[i][r] R(r,c), rows ascending (deterministic)
__global__ void k_coarse_WR(const double* __restrict__ W, int ld, int n, const int* __restrict__ cptr,
                            const int* __restrict__ crow, const double* __restrict__ cval, int nc,
                            double* __restrict__ WR)
{
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
        const double* Wi = W + (size_t)i * ld;
        for (int c = threadIdx.x; c < nc; c += blockDim.x) {
            double s = 0.0;
            for (int q = cptr[c]; q < cptr[c + 1]; ++q) s += Wi[crow[q]] * cval[q];
            WR[(size_t)i * nc + c] = s;
        }
    }
}

// H[a][b] = sum_{r in col a} R(r,a) WR[r][b]  (lower triangle used)
__global__ void k_coarse_H(const double* __restrict__ WR, const int* __restrict__ cptr, const int* __restrict__ crow,
                           const double* __restrict__ cval, int nc, double* __restrict__ H)
{
    const int a = blockIdx.x;
    for (int b = threadIdx.x; b < nc; b += blockDim.x) {
        double s = 0.0;
        for (int q = cptr[a]; q < cptr[a + 1]; ++q) s += cval[q] * WR[(size_t)crow[q] * nc + b];
        H[(size_t)a * nc + b] = s;
    }
}

// ---------------------------------------------------------------- Cholesky: diagonal tile
// Factor tile (k,k) of each listed block in shared memory, write L_kk and its
// inverse D_k (lower triangular, stored as a full 64x64 slot).
__global__ void __launch_bounds__(256) k_potrf(int k, const int* __restrict__ blocks, const int* __restrict__ nbv,
                                               const int* __restrict__ Loff, const int* __restrict__ Doff,
                                               double* __restrict__ L, double* __restrict__ D, int* __restrict__ fail)
{
    extern __shared__ double sm[];
    double* a = sm;             // TB x (TB+1)
    double* x = sm + TB * (TB + 1);
    const int b = blocks[blockIdx.x];
    const int nb = nbv[b];
    const int r0 = k * TB;
    const int tn = min(TB, nb - r0);
    double* Lt = L + Loff[b] + (size_t)r0 * nb + r0;
    for (int e = threadIdx.x; e < tn * tn; e += blockDim.x) {
        const int i = e / tn, j = e % tn;
        a[i * (TB + 1) + j] = (j <= i) ? Lt[(size_t)i * nb + j] : 0.0;
    }
    __syncthreads();
    __shared__ int bad;
    if (threadIdx.x == 0) bad = 0;
    for (int j = 0; j < tn; ++j) {
        if (threadIdx.x == 0) {
            const double d = a[j * (TB + 1) + j];
            if (!(d > 0.0) || !isfinite(d)) bad = 1;
            a[j * (TB + 1) + j] = sqrt(d);
        }
        __syncthreads();
        const double djj = a[j * (TB + 1) + j];
        for (int i = j + 1 + threadIdx.x; i < tn; i += blockDim.x) a[i * (TB + 1) + j] /= djj;
        __syncthreads();
        const int m = tn - j - 1;
        for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
            const int i = j + 1 + e / m, l = j + 1 + e % m;
            if (l <= i) a[i * (TB + 1) + l] -= a[i * (TB + 1) + j] * a[l * (TB + 1) + j];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0 && bad) atomicExch(&fail[b], 1);
    for (int e = threadIdx.x; e < tn * tn; e += blockDim.x) {
        const int i = e / tn, j = e % tn;
        if (j <= i) Lt[(size_t)i * nb + j] = a[i * (TB + 1) + j];
    }
    // inverse of the lower-triangular tile, one column per thread
    double* Dt = D + Doff[b] + (size_t)k * TB * TB;
    const int c = threadIdx.x;
    if (c < TB) {
        for (int i = 0; i < TB; ++i) x[i * (TB + 1) + c] = 0.0;
        if (c < tn) {
            x[c * (TB + 1) + c] = 1.0 / a[c * (TB + 1) + c];
            for (int i = c + 1; i < tn; ++i) {
                double s = 0.0;
                for (int l = c; l < i; ++l) s += a[i * (TB + 1) + l] * x[l * (TB + 1) + c];
                x[i * (TB + 1) + c] = -s / a[i * (TB + 1) + i];
            }
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < TB * TB; e += blockDim.x) Dt[e] = x[(e / TB) * (TB + 1) + (e % TB)];
}

// ---------------------------------------------------------------- Cholesky: tile GEMMs on DMMA
// task.x = block, task.y = tile row i, task.z = tile col j; mode 0: C(i,k) = C(i,k) D_k^T
// (trsm through the inverted diagonal tile), mode 1: C(i,j) -= L(i,k) L(j,k)^T.
__global__ void __launch_bounds__(128) k_tile_gemm(int k, int mode, const int4* __restrict__ tasks,
                                                   const int* __restrict__ nbv, const int* __restrict__ Loff,
                                                   const int* __restrict__ Doff, double* __restrict__ L,
                                                   const double* __restrict__ D)
{
    extern __shared__ double sm[];
    double* As = sm;             // TB x TLD
    double* Bs = sm + TB * TLD;  // TB x TLD
    const int4 t = tasks[blockIdx.x];
    const int b = t.x, ti = t.y, tj = t.z;
    const int nb = nbv[b];
    double* Lb = L + Loff[b];
    const int mi = min(TB, nb - ti * TB), mj = min(TB, nb - tj * TB), mk = min(TB, nb - k * TB);
    const double* A = Lb + (size_t)ti * TB * nb + (size_t)k * TB;  // tile (i,k)
    for (int e = threadIdx.x; e < TB * TB; e += blockDim.x) {
        const int r = e / TB, c = e % TB;
        As[r * TLD + c] = (r < mi && c < mk) ? A[(size_t)r * nb + c] : 0.0;
    }
    if (mode == 0) {
        const double* Dk = D + Doff[b] + (size_t)k * TB * TB;
        for (int e = threadIdx.x; e < TB * TB; e += blockDim.x) Bs[(e / TB) * TLD + (e % TB)] = Dk[e];
    } else {
        const double* B = Lb + (size_t)tj * TB * nb + (size_t)k * TB;  // tile (j,k)
        for (int e = threadIdx.x; e < TB * TB; e += blockDim.x) {
            const int r = e / TB, c = e % TB;
            Bs[r * TLD + c] = (r < mj && c < mk) ? B[(size_t)r * nb + c] : 0.0;
        }
    }
    __syncthreads();
    // each warp: 32x32 output = 4x4 DMMA tiles of 8x8; C = A * B^T
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gid = lane >> 2, tig = lane & 3;
    const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
    double acc[4][4][2];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
#pragma unroll 4
    for (int kk = 0; kk < TB; kk += 4) {
        double af[4], bf[4];
#pragma unroll
        for (int x = 0; x < 4; ++x) af[x] = As[(wm + 8 * x + gid) * TLD + kk + tig];
#pragma unroll
        for (int y = 0; y < 4; ++y) bf[y] = Bs[(wn + 8 * y + gid) * TLD + kk + tig];
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) dmma(acc[x][y][0], acc[x][y][1], af[x], bf[y]);
    }
    double* C = Lb + (size_t)ti * TB * nb + (size_t)tj * TB;
    if (mode == 0) __syncthreads();  // C aliases A (already staged in smem)
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int r = wm + 8 * x + gid, c = wn + 8 * y + 2 * tig + h;
                if (r < mi && c < mj) {
                    double* dst = C + (size_t)r * nb + c;
                    if (mode == 0)
                        *dst = acc[x][y][h];
                    else
                        *dst -= acc[x][y][h];
                }
            }
}

// ---------------------------------------------------------------- apply
// gather r into the block-local vector and restrict to the coarse space
__global__ void k_prec_gather(const double* __restrict__ r, int n, const int* __restrict__ pos,
                              double* __restrict__ loc, const int* done)
{
    if (done && *done) return;
    const int d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d < n && pos[d] >= 0) loc[pos[d]] = r[d];
}

__global__ void k_prec_restrict(const double* __restrict__ r, const int* __restrict__ cptr,
                                const int* __restrict__ crow, const double* __restrict__ cval, int nc,
                                double* __restrict__ loc_c, const int* done)
{
    if (done && *done) return;
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nc) return;
    double s = 0.0;
    for (int q = cptr[c]; q < cptr[c + 1]; ++q) s += cval[q] * r[crow[q]];
    loc_c[c] = s;
}

// y[0:m] (smem) = sum_c T[r][c] v[c] over an m x kc tile (row-major, ld) — 4 threads per row
__device__ __forceinline__ double tile_row_dot(const double* __restrict__ T, size_t ld, int r, int kc,
                                               const double* v, int part, bool active)
{
    double s = 0.0;
    if (active)
        for (int c = part; c < kc; c += 4) s += T[(size_t)r * ld + c] * v[c];
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    return s;
}

// Forward step k: for each task (b, i) with i >= k:
//   v_i = loc_i - L(i,k-1) y_{k-1}   (k >= 1),  and if i == k: y_k = D_k v_k
__global__ void __launch_bounds__(256) k_trsv_fwd(int k, const int2* __restrict__ tasks, const int* __restrict__ nbv,
                                                  const int* __restrict__ locv, const int* __restrict__ Loff,
                                                  const int* __restrict__ Doff, const double* __restrict__ L,
                                                  const double* __restrict__ D, double* __restrict__ loc,
                                                  const int* done)
{
    if (done && *done) return;
    __shared__ double yprev[TB], v[TB];
    const int2 t = tasks[blockIdx.x];
    const int b = t.x, i = t.y, nb = nbv[b];
    double* lb = loc + locv[b];
    const int mi = min(TB, nb - i * TB);
    const int row = threadIdx.x >> 2, part = threadIdx.x & 3;
    if (threadIdx.x < TB) v[threadIdx.x] = threadIdx.x < mi ? lb[i * TB + threadIdx.x] : 0.0;
    if (k >= 1) {
        const int kc = TB;  // column tile k-1 is always full
        if (threadIdx.x < TB) yprev[threadIdx.x] = lb[(k - 1) * TB + threadIdx.x];
        __syncthreads();
        const double* T = L + Loff[b] + (size_t)i * TB * nb + (size_t)(k - 1) * TB;
        const double s = tile_row_dot(T, nb, row, kc, yprev, part, row < mi);
        __syncthreads();
        if (row < mi && part == 0) v[row] -= s;
    }
    __syncthreads();
    if (i == k) {
        const double* Dk = D + Doff[b] + (size_t)k * TB * TB;
        const double s = tile_row_dot(Dk, TB, row, row + 1, v, part, row < mi);
        __syncthreads();
        if (row < mi && part == 0) lb[i * TB + row] = s;
    } else if (threadIdx.x < mi) {
        lb[i * TB + threadIdx.x] = v[threadIdx.x];
    }
}

// Backward step with block-local k = T_b - 1 - s: tasks (b, i) with i <= k:
//   v_i = loc_i - L(k+1,i)^T z_{k+1}   (k+1 < T_b),  and if i == k: z_k = D_k^T v_k
__global__ void __launch_bounds__(256) k_trsv_bwd(int s, const int2* __restrict__ tasks, const int* __restrict__ nbv,
                                                  const int* __restrict__ Tv, const int* __restrict__ locv,
                                                  const int* __restrict__ Loff, const int* __restrict__ Doff,
                                                  const double* __restrict__ L, const double* __restrict__ D,
                                                  double* __restrict__ loc, const int* done)
{
    if (done && *done) return;
    __shared__ double znext[TB], v[TB], red[4][TB];
    const int2 t = tasks[blockIdx.x];
    const int b = t.x, i = t.y, nb = nbv[b], T = Tv[b];
    const int k = T - 1 - s;
    double* lb = loc + locv[b];
    const int mi = min(TB, nb - i * TB);
    const int col = threadIdx.x & 63, grp = threadIdx.x >> 6;  // 4 row groups x 64 columns
    if (threadIdx.x < TB) v[threadIdx.x] = threadIdx.x < mi ? lb[i * TB + threadIdx.x] : 0.0;
    if (k + 1 < T) {
        const int mk1 = min(TB, nb - (k + 1) * TB);
        if (threadIdx.x < TB) znext[threadIdx.x] = threadIdx.x < mk1 ? lb[(k + 1) * TB + threadIdx.x] : 0.0;
        __syncthreads();
        const double* Tt = L + Loff[b] + (size_t)(k + 1) * TB * nb + (size_t)i * TB;  // tile (k+1, i)
        double acc = 0.0;
        if (col < mi)
            for (int r = grp; r < mk1; r += 4) acc += Tt[(size_t)r * nb + col] * znext[r];
        red[grp][col] = acc;
        __syncthreads();
        if (threadIdx.x < mi) v[threadIdx.x] -= (red[0][threadIdx.x] + red[1][threadIdx.x]) +
                                                (red[2][threadIdx.x] + red[3][threadIdx.x]);
    }
    __syncthreads();
    if (i == k) {
        const double* Dk = D + Doff[b] + (size_t)k * TB * TB;
        double acc = 0.0;
        if (col < mi)
            for (int r = col + grp; r < mi; r += 4)
                if (r >= col) acc += Dk[(size_t)r * TB + col] * v[r];
        red[grp][col] = acc;
        __syncthreads();
        if (threadIdx.x < mi)
            lb[i * TB + threadIdx.x] = (red[0][threadIdx.x] + red[1][threadIdx.x]) +
                                       (red[2][threadIdx.x] + red[3][threadIdx.x]);
    } else if (threadIdx.x < mi) {
        lb[i * TB + threadIdx.x] = v[threadIdx.x];
    }
}

// z[d] = z_block[d] + (R y_c)[d]  (schwarz.hpp:126-138: faces/WB then coarse)
__global__ void k_prec_scatter(const double* __restrict__ loc, const int* __restrict__ pos, int n,
                               const int* __restrict__ rptr, const int* __restrict__ rcol,
                               const double* __restrict__ rval, const double* __restrict__ loc_c,
                               double* __restrict__ z, const int* done)
{
    if (done && *done) return;
    const int d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= n) return;
    double out = pos[d] >= 0 ? loc[pos[d]] : 0.0;
    if (rptr) {
        double y = 0.0;
        for (int q = rptr[d]; q < rptr[d + 1]; ++q) y += rval[q] * loc_c[rcol[q]];
        out += y;
    }
    z[d] = out;
}

}  // namespace

// reference: inc/schwarz.hpp:100-118
Prec* prec_build(Ctx* ctx, const DMatrix& W, const DofPartition& part, const Prolongation& R)
{
    cudaStream_t s = ctx->stream;
    const int n = W.n;
    if (R.cols > 0 && R.rows != n) throw ValidationError("prolongation row count does not match the matrix");
    auto* P = new Prec;
    try {
        P->ctx = ctx;
        P->n = n;
        P->nfaces = (int)part.face_ids.size();
        P->nwb = (int)part.wirebasket.size();
        P->nc = R.cols;
        // block dof lists: faces in map order, then WB (skipping empty blocks as factor_block does)
        std::vector<int> bptr{0}, bdofs;
        std::vector<int> kinds;  // 0 face, 1 wb, 2 coarse
        for (int f = 0; f < P->nfaces; ++f) {
            const int a = part.face_ptr[f], e = part.face_ptr[f + 1];
            if (e == a) continue;
            bdofs.insert(bdofs.end(), part.face_dofs.begin() + a, part.face_dofs.begin() + e);
            bptr.push_back((int)bdofs.size());
            kinds.push_back(0);
        }
        if (P->nwb > 0) {
            bdofs.insert(bdofs.end(), part.wirebasket.begin(), part.wirebasket.end());
            bptr.push_back((int)bdofs.size());
            kinds.push_back(1);
        }
        for (int d : bdofs)
            if (d < 0 || d >= n) throw ValidationError("partition DOF out of range");
        const int ngather = (int)kinds.size();
        if (P->nc > 0) {
            kinds.push_back(2);
            P->coarse_block = ngather;
        }
        P->nblocks = (int)kinds.size();
        size_t Loff = 0, Doff = 0, loc = 0;
        for (int b = 0; b < P->nblocks; ++b) {
            const int nb = b < ngather ? bptr[b + 1] - bptr[b] : P->nc;
            const int T = (nb + TB - 1) / TB;
            P->h_nb.push_back(nb);
            P->h_T.push_back(T);
            P->h_loc.push_back((int)loc);
            P->h_Loff.push_back((int)Loff);
            P->h_Doff.push_back((int)Doff);
            if (Loff + (size_t)nb * nb > 0x7fffffffULL || Doff + (size_t)T * TB * TB > 0x7fffffffULL)
                throw ValidationError("preconditioner blocks exceed the 2^31 element index range");
            Loff += (size_t)nb * nb;
            Doff += (size_t)T * TB * TB;
            loc += (size_t)T * TB;
            P->Tmax = std::max(P->Tmax, T);
            P->factor_bytes += (double)nb * nb * 8.0;
        }
        P->d_nb.upload(P->h_nb, s);
        P->d_T.upload(P->h_T, s);
        P->d_loc.upload(P->h_loc, s);
        P->d_Loff.upload(P->h_Loff, s);
        P->d_Doff.upload(P->h_Doff, s);
        P->L.alloc(std::max<size_t>(Loff, 1));
        P->D.alloc(std::max<size_t>(Doff, 1));
        P->loc.alloc(std::max<size_t>(loc, 1));
        SBG_CUDA(cudaMemsetAsync(P->loc.p, 0, P->loc.n * sizeof(double), s));
        std::vector<int> pos(n, -1);
        for (int b = 0; b < ngather; ++b)
            for (int q = bptr[b]; q < bptr[b + 1]; ++q) pos[bdofs[q]] = P->h_loc[b] + (q - bptr[b]);
        P->pos.upload(pos, s);
        // gather face/WB blocks from W (factor_block's submatrix, schwarz.hpp:77-83)
        if (ngather > 0) {
            DBuf<int> d_bptr, d_bdofs;
            d_bptr.upload(bptr, s);
            d_bdofs.upload(bdofs, s);
            k_gather_blocks<<<dim3(ngather, 64), 128, 0, s>>>(W.a.p, W.ld, d_bptr.p, d_bdofs.p, P->d_Loff.p, P->L.p); ::sbg::count_launch();
            SBG_LAUNCH_CHECK();
            SBG_CUDA(cudaStreamSynchronize(s));
        }
        // coarse space: R in CSC and CSR, H = R^T W R into the coarse block
        if (P->nc > 0) {
            P->Rc_ptr.upload(R.col_ptr, s);
            P->Rc_row.upload(R.row_idx, s);
            P->Rc_val.upload(R.val, s);
            std::vector<int> rptr(n + 1, 0), rcol(R.val.size());
            std::vector<double> rval(R.val.size());
            for (int c = 0; c < R.cols; ++c)
                for (int q = R.col_ptr[c]; q < R.col_ptr[c + 1]; ++q) rptr[R.row_idx[q] + 1]++;
            for (int i = 0; i < n; ++i) rptr[i + 1] += rptr[i];
            std::vector<int> fill(rptr.begin(), rptr.end() - 1);
            for (int c = 0; c < R.cols; ++c)
                for (int q = R.col_ptr[c]; q < R.col_ptr[c + 1]; ++q) {
                    const int r = R.row_idx[q];
                    rcol[fill[r]] = c;
                    rval[fill[r]] = R.val[q];
                    fill[r]++;
                }
            P->Rr_ptr.upload(rptr, s);
            P->Rr_col.upload(rcol, s);
            P->Rr_val.upload(rval, s);
            DBuf<double> WR((size_t)n * P->nc);
            TimedScope ts(ctx, "coarse_galerkin");
            k_coarse_WR<<<std::min(n, 8 * ctx->sm_count), 128, 0, s>>>(W.a.p, W.ld, n, P->Rc_ptr.p, P->Rc_row.p,
                                                                      P->Rc_val.p, P->nc, WR.p); ::sbg::count_launch();
            k_coarse_H<<<P->nc, 128, 0, s>>>(WR.p, P->Rc_ptr.p, P->Rc_row.p, P->Rc_val.p, P->nc,
                                             P->L.p + P->h_Loff[P->coarse_block]); ::sbg::count_launch();
            SBG_LAUNCH_CHECK();
            SBG_CUDA(cudaStreamSynchronize(s));
        }
        // batched tiled Cholesky
        DBuf<int> fail(std::max(P->nblocks, 1));
        SBG_CUDA(cudaMemsetAsync(fail.p, 0, fail.n * sizeof(int), s));
        {
            TimedScope ts(ctx, "cholesky");
            std::vector<int> pot;
            std::vector<int4> trsm, upd;
            DBuf<int> d_pot;
            DBuf<int4> d_trsm, d_upd;
            const size_t smem_potrf = 2 * TB * (TB + 1) * sizeof(double);
            const size_t smem_gemm = 2 * TB * TLD * sizeof(double);
            SBG_CUDA(cudaFuncSetAttribute(k_potrf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_potrf));
            SBG_CUDA(cudaFuncSetAttribute(k_tile_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_gemm));
            for (int k = 0; k < P->Tmax; ++k) {
                pot.clear();
                trsm.clear();
                upd.clear();
                for (int b = 0; b < P->nblocks; ++b) {
                    const int T = P->h_T[b];
                    if (T <= k) continue;
                    pot.push_back(b);
                    for (int i = k + 1; i < T; ++i) trsm.push_back({b, i, k, 0});
                    for (int j = k + 1; j < T; ++j)
                        for (int i = j; i < T; ++i) upd.push_back({b, i, j, 0});
                }
                d_pot.upload(pot, s);
                k_potrf<<<(int)pot.size(), 256, smem_potrf, s>>>(k, d_pot.p, P->d_nb.p, P->d_Loff.p, P->d_Doff.p,
                                                                 P->L.p, P->D.p, fail.p); ::sbg::count_launch();
                SBG_LAUNCH_CHECK();
                if (!trsm.empty()) {
                    d_trsm.upload(trsm, s);
                    k_tile_gemm<<<(int)trsm.size(), 128, smem_gemm, s>>>(k, 0, d_trsm.p, P->d_nb.p, P->d_Loff.p,
                                                                          P->d_Doff.p, P->L.p, P->D.p); ::sbg::count_launch();
                    SBG_LAUNCH_CHECK();
                }
                if (!upd.empty()) {
                    d_upd.upload(upd, s);
                    k_tile_gemm<<<(int)upd.size(), 128, smem_gemm, s>>>(k, 1, d_upd.p, P->d_nb.p, P->d_Loff.p,
                                                                         P->d_Doff.p, P->L.p, P->D.p); ::sbg::count_launch();
                    SBG_LAUNCH_CHECK();
                }
                // host task vectors are reused next step: wait for the async uploads
                SBG_CUDA(cudaStreamSynchronize(s));
            }
        }
        std::vector<int> hfail(fail.n);
        SBG_CUDA(cudaMemcpy(hfail.data(), fail.p, hfail.size() * sizeof(int), cudaMemcpyDeviceToHost));
        for (int b = 0; b < P->nblocks; ++b)
            if (hfail[b]) {
                if (kinds[b] == 2) throw NumericalError("coarse matrix factorization failed");
                throw NumericalError(std::string("block factorization failed (") +
                                     (kinds[b] == 0 ? "face" : "wire-basket") +
                                     "): partition inconsistent with the assembled matrix");
            }
        // trsv task lists
        std::vector<int2> fw, bw;
        P->fwd_off.assign(1, 0);
        P->bwd_off.assign(1, 0);
        for (int k = 0; k < P->Tmax; ++k) {
            for (int b = 0; b < P->nblocks; ++b)
                for (int i = k; i < P->h_T[b]; ++i) fw.push_back({b, i});
            P->fwd_off.push_back((int)fw.size());
        }
        for (int st = 0; st < P->Tmax; ++st) {
            for (int b = 0; b < P->nblocks; ++b) {
                const int kk = P->h_T[b] - 1 - st;
                for (int i = 0; i <= kk; ++i) bw.push_back({b, i});
            }
            P->bwd_off.push_back((int)bw.size());
        }
        P->fwd_tasks.upload(fw, s);
        P->bwd_tasks.upload(bw, s);
        SBG_CUDA(cudaStreamSynchronize(s));
    } catch (...) {
        delete P;
        throw;
    }
    return P;
}

void prec_destroy(Prec* p) { delete p; }
int prec_n(const Prec* p) { return p->n; }
int prec_num_subspaces(const Prec* p)  // schwarz.hpp:66-72
{
    return p->nfaces + (p->nwb > 0 ? 1 : 0) + (p->nc > 0 ? 1 : 0);
}
double prec_factor_bytes(const Prec* p) { return p->factor_bytes; }

// reference: inc/schwarz.hpp:121-140
void prec_apply(Ctx* ctx, Prec* P, const double* r, double* z, const int* done)
{
    TimedScope ts(ctx, "precond_apply");
    cudaStream_t s = ctx->stream;
    const int n = P->n;
    if (n == 0) return;
    const int nb = (n + 255) / 256;
    double* loc_c = P->coarse_block >= 0 ? P->loc.p + P->h_loc[P->coarse_block] : nullptr;
    k_prec_gather<<<nb, 256, 0, s>>>(r, n, P->pos.p, P->loc.p, done); ::sbg::count_launch();
    if (P->nc > 0)
        k_prec_restrict<<<(P->nc + 127) / 128, 128, 0, s>>>(r, P->Rc_ptr.p, P->Rc_row.p, P->Rc_val.p, P->nc, loc_c,
                                                            done); ::sbg::count_launch();
    for (int k = 0; k < P->Tmax; ++k) {
        const int cnt = P->fwd_off[k + 1] - P->fwd_off[k];
        if (cnt)
            k_trsv_fwd<<<cnt, 256, 0, s>>>(k, P->fwd_tasks.p + P->fwd_off[k], P->d_nb.p, P->d_loc.p, P->d_Loff.p,
                                           P->d_Doff.p, P->L.p, P->D.p, P->loc.p, done); ::sbg::count_launch();
    }
    for (int st = 0; st < P->Tmax; ++st) {
        const int cnt = P->bwd_off[st + 1] - P->bwd_off[st];
        if (cnt)
            k_trsv_bwd<<<cnt, 256, 0, s>>>(st, P->bwd_tasks.p + P->bwd_off[st], P->d_nb.p, P->d_T.p, P->d_loc.p,
                                           P->d_Loff.p, P->d_Doff.p, P->L.p, P->D.p, P->loc.p, done); ::sbg::count_launch();
    }
    k_prec_scatter<<<nb, 256, 0, s>>>(P->loc.p, P->pos.p, n, P->nc > 0 ? P->Rr_ptr.p : nullptr, P->Rr_col.p,
                                      P->Rr_val.p, loc_c, z, done); ::sbg::count_launch();
    SBG_LAUNCH_CHECK();
}

void prec_block_diag(Ctx* ctx, Prec* P, int which, std::vector<double>& diag)
{
    int b = -1;
    if (which >= 0) {
        // face index counted over non-empty faces
        b = which;
    } else if (which == -1) {
        b = P->nwb > 0 ? (P->coarse_block >= 0 ? P->coarse_block - 1 : P->nblocks - 1) : -1;
    } else if (which == -2) {
        b = P->coarse_block;
    }
    diag.clear();
    if (b < 0 || b >= P->nblocks) return;
    const int nb = P->h_nb[b];
    std::vector<double> h((size_t)nb * nb);
    SBG_CUDA(cudaMemcpy(h.data(), P->L.p + P->h_Loff[b], h.size() * sizeof(double), cudaMemcpyDeviceToHost));
    for (int i = 0; i < nb; ++i) diag.push_back(h[(size_t)i * nb + i]);
    (void)ctx;
}

void coarse_galerkin(Ctx* ctx, const DMatrix& W, const Prolongation& R, std::vector<double>& H)
{
    cudaStream_t s = ctx->stream;
    const int n = W.n, nc = R.cols;
    H.assign((size_t)nc * nc, 0.0);
    if (nc == 0) return;
    DBuf<int> cp, cr;
    DBuf<double> cv, WR((size_t)n * nc), dH((size_t)nc * nc);
    cp.upload(R.col_ptr, s);
    cr.upload(R.row_idx, s);
    cv.upload(R.val, s);
    k_coarse_WR<<<std::min(n, 8 * ctx->sm_count), 128, 0, s>>>(W.a.p, W.ld, n, cp.p, cr.p, cv.p, nc, WR.p); ::sbg::count_launch();
    k_coarse_H<<<nc, 128, 0, s>>>(WR.p, cp.p, cr.p, cv.p, nc, dH.p); ::sbg::count_launch();
    SBG_LAUNCH_CHECK();
    SBG_CUDA(cudaMemcpyAsync(H.data(), dH.p, H.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    SBG_CUDA(cudaStreamSynchronize(s));
}

}  // namespace sbg
