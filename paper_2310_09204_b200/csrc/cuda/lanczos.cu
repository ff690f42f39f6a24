// Extreme eigenvalues for condition_number (reference: inc/schwarz.hpp:150-190)
// without the dense eigensolve.
//
// Lanczos on A = M W in the W inner product <x, y> = x^T W y (A is self-adjoint
// there; M = I gives the spectrum of W itself, M = the Schwarz preconditioner or a
// dense M gives that of the congruence L^T M L).  The basis Q and U = W Q stay in
// HBM and every new vector is reorthogonalised twice against all of them, so
// clustered extreme eigenvalues (cfg 1 has two at a relative gap of 1e-5) resolve
// instead of being averaged the way CG's own Lanczos matrix does once the solve
// has converged.  The iteration stops when both extreme Ritz pairs have residual
// beta_j |s_last| <= tol * |theta| (so |lambda - theta| <= tol |theta|), or when the
// Krylov space is exhausted.
#include <algorithm>
#include <cmath>
#include <random>

#include "kernels.cuh"

namespace sbg {

namespace {

// out[j] = U_j . w  (U column-major with stride ld; one block per column, fixed order)
__global__ void k_basis_dots(const double* __restrict__ U, size_t ld, int m, const double* __restrict__ w, int n,
                             double* __restrict__ out)
{
    __shared__ double red[256];
    const int j = blockIdx.x;
    const double* u = U + (size_t)j * ld;
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s = fma(u[i], w[i], s);
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[j] = red[0];
}

// w -= Q c  (m columns)
__global__ void k_basis_sub(double* __restrict__ w, const double* __restrict__ Q, size_t ld, int m,
                            const double* __restrict__ c, int n)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s = 0.0;
    for (int j = 0; j < m; ++j) s = fma(Q[(size_t)j * ld + i], c[j], s);
    w[i] -= s;
}

// w = a w - alpha q - beta qprev
__global__ void k_three_term(double* __restrict__ w, const double* __restrict__ q, const double* __restrict__ qp,
                             double alpha, double beta, int n)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double v = w[i] - alpha * q[i];
    if (qp) v -= beta * qp[i];
    w[i] = v;
}

// dst = src * s
__global__ void k_scale_to(double* __restrict__ dst, const double* __restrict__ src, double s, int n)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[i] * s;
}

// a . b with a fixed-order block reduction (partials then one block)
__global__ void k_dot_partial(const double* __restrict__ a, const double* __restrict__ b, int n,
                              double* __restrict__ part)
{
    __shared__ double red[256];
    double s = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) s = fma(a[i], b[i], s);
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void k_sum(const double* __restrict__ part, int m, double* __restrict__ out)
{
    __shared__ double red[256];
    double s = 0.0;
    for (int i = threadIdx.x; i < m; i += blockDim.x) s += part[i];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = red[0];
}

// Ritz value theta of the symmetric tridiagonal (d, e) and |s_last| of its unit
// eigenvector, by inverse iteration on T - theta I (tridiagonal LU, no pivoting
// needed away from exact singularity: the shift is nudged by a relative 1e-15)
double last_component(const std::vector<double>& d, const std::vector<double>& e, double theta)
{
    const int k = (int)d.size();
    if (k == 1) return 1.0;
    const double shift = theta * (1.0 + 1e-15) + 1e-300;
    std::vector<double> x(k, 1.0), c(k), dd(k), y(k);
    for (int it = 0; it < 3; ++it) {
        // solve (T - shift) y = x with the Thomas algorithm
        dd[0] = d[0] - shift;
        y[0] = x[0];
        for (int i = 1; i < k; ++i) {
            const double piv = dd[i - 1] != 0.0 ? dd[i - 1] : 1e-300;
            c[i] = e[i - 1] / piv;
            dd[i] = d[i] - shift - c[i] * e[i - 1];
            y[i] = x[i] - c[i] * y[i - 1];
        }
        x[k - 1] = y[k - 1] / (dd[k - 1] != 0.0 ? dd[k - 1] : 1e-300);
        for (int i = k - 2; i >= 0; --i) x[i] = (y[i] - e[i] * x[i + 1]) / (dd[i] != 0.0 ? dd[i] : 1e-300);
        double nrm = 0.0;
        for (double v : x) nrm += v * v;
        nrm = std::sqrt(nrm);
        for (double& v : x) v /= nrm;
    }
    return std::abs(x[k - 1]);
}

}  // namespace

Spectrum spectrum(Ctx* ctx, const DMatrix& W, Prec* prec, double tol, int maxit)
{
    const int n = W.n;
    if (n == 0) throw ValidationError("spectrum of an empty matrix");
    if (prec && prec_n(prec) != n) throw ValidationError("preconditioner length mismatch");
    if (!(tol > 0)) throw ValidationError("condition_number: tolerance must be positive");
    const int mmax = std::min(n, maxit > 0 ? maxit : std::min(n, 1500));
    TimedScope tsc(ctx, "lanczos");
    cudaStream_t s = ctx->stream;
    const size_t ld = (size_t)W.ld;
    // basis Q, U = W Q (column j contiguous), work vectors, reductions
    DBuf<double> Q((size_t)(mmax + 1) * ld), U((size_t)(mmax + 1) * ld), w(ld), z(ld), coef(mmax + 1);
    const int nb = (n + 255) / 256, pblocks = std::min(nb, 256);
    DBuf<double> part(pblocks), scal(2);
    SBG_CUDA(cudaMemsetAsync(w.p, 0, ld * sizeof(double), s));
    SBG_CUDA(cudaMemsetAsync(z.p, 0, ld * sizeof(double), s));
    GemvPlan plan;
    gemv_plan(ctx, n, W.ld, plan);
    auto dot = [&](const double* a, const double* b) {
        k_dot_partial<<<pblocks, 256, 0, s>>>(a, b, n, part.p);
        k_sum<<<1, 256, 0, s>>>(part.p, pblocks, scal.p);
        count_launch();
        count_launch();
        double h = 0.0;
        SBG_CUDA(cudaMemcpyAsync(&h, scal.p, sizeof(double), cudaMemcpyDeviceToHost, s));
        SBG_CUDA(cudaStreamSynchronize(s));
        return h;
    };
    auto reorth = [&](int m) {  // w -= Q (U^T w), twice
        for (int pass = 0; pass < 2; ++pass) {
            k_basis_dots<<<m, 256, 0, s>>>(U.p, ld, m, w.p, n, coef.p);
            k_basis_sub<<<nb, 256, 0, s>>>(w.p, Q.p, ld, m, coef.p, n);
            count_launch();
            count_launch();
        }
    };
    // q_0 = b / |b|_W from a seeded normal b
    {
        std::mt19937 gen(2310);
        std::normal_distribution<double> nd(0.0, 1.0);
        std::vector<double> b(n);
        for (double& v : b) v = nd(gen);
        SBG_CUDA(cudaMemcpyAsync(w.p, b.data(), n * sizeof(double), cudaMemcpyHostToDevice, s));
    }
    gemv(ctx, W, plan, w.p, z.p);
    double bb = dot(w.p, z.p);
    if (!(bb > 0)) throw NumericalError("condition_number: matrix is not positive definite");
    double beta = std::sqrt(bb);
    k_scale_to<<<nb, 256, 0, s>>>(Q.p, w.p, 1.0 / beta, n);
    k_scale_to<<<nb, 256, 0, s>>>(U.p, z.p, 1.0 / beta, n);
    count_launch();
    count_launch();
    std::vector<double> d, e;
    Spectrum sp;
    double prev_beta = 0.0;
    for (int j = 0; j < mmax; ++j) {
        double* qj = Q.p + (size_t)j * ld;
        double* uj = U.p + (size_t)j * ld;
        // w = A q_j = M (W q_j) = M u_j
        if (prec)
            prec_apply(ctx, prec, uj, w.p, nullptr);
        else
            SBG_CUDA(cudaMemcpyAsync(w.p, uj, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
        const double alpha = dot(w.p, uj);  // <A q_j, q_j>_W
        k_three_term<<<nb, 256, 0, s>>>(w.p, qj, j > 0 ? qj - ld : nullptr, alpha, prev_beta, n);
        count_launch();
        reorth(j + 1);
        gemv(ctx, W, plan, w.p, z.p);
        bb = dot(w.p, z.p);
        d.push_back(alpha);
        sp.iterations = j + 1;
        const bool exhausted = !(bb > 0) || j + 1 == n;
        beta = exhausted ? 0.0 : std::sqrt(bb);
        // convergence of both extreme Ritz pairs: residual beta |s_last| <= tol |theta|
        if (exhausted || (j + 1) % 8 == 0 || j + 1 == mmax) {
            double lmin, lmax;
            // the CG-coefficient form is not used here: (d, e) is the Lanczos matrix itself
            std::vector<double> dd = d, ee = e;
            {
                const int k = (int)dd.size();
                double lo = 1e300, hi = -1e300;
                for (int i = 0; i < k; ++i) {
                    const double rad = (i > 0 ? std::abs(ee[i - 1]) : 0.0) + (i + 1 < k ? std::abs(ee[i]) : 0.0);
                    lo = std::min(lo, dd[i] - rad);
                    hi = std::max(hi, dd[i] + rad);
                }
                auto count_below = [&](double x) {
                    int c = 0;
                    double q = 1.0;
                    for (int i = 0; i < k; ++i) {
                        q = dd[i] - x - (i == 0 ? 0.0 : ee[i - 1] * ee[i - 1] / q);
                        if (q == 0.0) q = -1e-300;
                        if (q < 0) ++c;
                    }
                    return c;
                };
                auto kth = [&](int idx) {
                    double a = lo, b = hi;
                    for (int it = 0; it < 200; ++it) {
                        const double mid = 0.5 * (a + b);
                        if (mid <= a || mid >= b) break;
                        if (count_below(mid) > idx)
                            b = mid;
                        else
                            a = mid;
                    }
                    return 0.5 * (a + b);
                };
                lmin = kth(0);
                lmax = kth(k - 1);
            }
            sp.lambda_min = lmin;
            sp.lambda_max = lmax;
            const double rmin = beta * last_component(dd, ee, lmin), rmax = beta * last_component(dd, ee, lmax);
            if (exhausted || (rmin <= tol * std::abs(lmin) && rmax <= tol * std::abs(lmax))) {
                sp.converged = true;
                break;
            }
        }
        if (exhausted) break;
        e.push_back(beta);
        prev_beta = beta;
        k_scale_to<<<nb, 256, 0, s>>>(Q.p + (size_t)(j + 1) * ld, w.p, 1.0 / beta, n);
        k_scale_to<<<nb, 256, 0, s>>>(U.p + (size_t)(j + 1) * ld, z.p, 1.0 / beta, n);
        count_launch();
        count_launch();
    }
    SBG_LAUNCH_CHECK();
    SBG_CUDA(cudaStreamSynchronize(s));
    if (!(sp.lambda_min > 0)) throw NumericalError("condition_number: operator is not positive definite");
    sp.kappa = sp.lambda_max / sp.lambda_min;
    return sp;
}

}  // namespace sbg
