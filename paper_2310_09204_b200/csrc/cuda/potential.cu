// Double-layer potential of a jump density at points off the screen (3-D), on the device.
// reference: inc/potential.hpp:15-25 (make_cartesian_grid), :31-97 (facet_dipole_integral, the
// 3-D branch), :104-138 (eval_DL); inc/mesh.hpp:95-133 (point distances, distance_to).
//
// One thread per evaluation point; the facets stream through shared memory in index order, so
// a point's sum runs over the facets in the reference's order.  Per (point, facet):
//   * the reference's subdivision test dist < diam decides near / far, in its operation order
//     with IEEE non-fused arithmetic (a bounding-sphere test first skips the exact distance for
//     facets certainly farther than their diameter);
//   * a far facet (the depth-0 leaf) takes the rule triangle_rule(far_order + 2) in the form
//     (2A / 4 pi) n.(c0 - x) sum_j w_j [phi](y_j) / |y_j - x|^3 — n.(y - x) is the same for every
//     point y of the flat facet — with the y points and w_j [phi](y_j) staged per facet and
//     1/|r|^3 from a refined rsqrt;
//   * a near facet is subdivided exactly as the reference recurses (children in its order,
//     midpoints 0.5 (a + b)), depth first with per-depth state, and every leaf is integrated
//     in the reference's operation order (IEEE sqrt and division), so the near contributions
//     are bitwise the CPU restatement's; exact_far evaluates the far facets that way too (and
//     keeps one facet range per point), making the whole potential bitwise the oracle's.
#include <algorithm>
#include <cmath>
#include <vector>

#include "kernels.cuh"

namespace sbg {

namespace {

constexpr int DL_THREADS = 128;  // points per CTA
constexpr int DL_CHUNK = 16;     // facets staged per pass
constexpr int DL_MAXDEPTH = 24;  // potential.hpp:45
constexpr int DL_REC = 16;       // per-facet record: c0 c1 c2 (9), n0 (3), dv (3), pad

// ---- the reference's arithmetic, non-fused (the oracle is built with -ffp-contract=off)
struct R3 {
    double x, y, z;
};
__device__ __forceinline__ R3 r3(const double* p) { return {p[0], p[1], p[2]}; }
__device__ __forceinline__ R3 sub(R3 a, R3 b) { return {__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y), __dsub_rn(a.z, b.z)}; }
__device__ __forceinline__ R3 add(R3 a, R3 b) { return {__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y), __dadd_rn(a.z, b.z)}; }
__device__ __forceinline__ R3 scl(double s, R3 a) { return {__dmul_rn(s, a.x), __dmul_rn(s, a.y), __dmul_rn(s, a.z)}; }
__device__ __forceinline__ double dot3(R3 a, R3 b)
{
    return __dadd_rn(__dadd_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)), __dmul_rn(a.z, b.z));
}
__device__ __forceinline__ double sqn(R3 a) { return dot3(a, a); }
__device__ __forceinline__ R3 crs(R3 a, R3 b)
{
    return {__dsub_rn(__dmul_rn(a.y, b.z), __dmul_rn(a.z, b.y)), __dsub_rn(__dmul_rn(a.z, b.x), __dmul_rn(a.x, b.z)),
            __dsub_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x))};
}

// mesh.hpp:95-100
__device__ double pt_seg_dist(R3 x, R3 a, R3 b)
{
    const R3 d = sub(b, a);
    const double t = fmin(fmax(__ddiv_rn(dot3(sub(x, a), d), sqn(d)), 0.0), 1.0);
    return __dsqrt_rn(sqn(sub(x, add(a, scl(t, d)))));
}
// mesh.hpp:102-116
__device__ double pt_tri_dist(R3 x, R3 a, R3 b, R3 c)
{
    const R3 ab = sub(b, a), ac = sub(c, a);
    const R3 n = crs(ab, ac);
    const double nn = sqn(n);
    const R3 ax = sub(x, a);
    const double u = __ddiv_rn(dot3(crs(ax, ac), n), nn);
    const double v = __ddiv_rn(dot3(crs(ab, ax), n), nn);
    if (u >= 0 && v >= 0 && __dadd_rn(u, v) <= 1.0) return __ddiv_rn(fabs(dot3(ax, n)), __dsqrt_rn(nn));
    return fmin(fmin(pt_seg_dist(x, a, b), pt_seg_dist(x, b, c)), pt_seg_dist(x, a, c));
}
// potential.hpp:36-39 (sqrt is monotone and correctly rounded: one sqrt of the largest)
__device__ __forceinline__ double tri_diam3(R3 a, R3 b, R3 c)
{
    return __dsqrt_rn(fmax(fmax(sqn(sub(a, b)), sqn(sub(a, c))), sqn(sub(b, c))));
}

// potential.hpp:84-94: one leaf in the reference's order
__device__ double dl_leaf(const double* C, const double* D, R3 n0, R3 x, const double* ru, const double* rv,
                          const double* rw, int nr)
{
    const R3 c0 = r3(C), c1 = r3(C + 3), c2 = r3(C + 6);
    const R3 e1 = sub(c1, c0), e2 = sub(c2, c0);
    const double area = __dmul_rn(0.5, __dsqrt_rn(sqn(crs(e1, e2))));
    const double four_pi = 4.0 * M_PI;
    double acc = 0.0;
    for (int i = 0; i < nr; ++i) {
        const double u = ru[i], v = rv[i];
        const R3 y = add(add(c0, scl(u, e1)), scl(v, e2));
        const double val = __dadd_rn(__dadd_rn(__dmul_rn(__dsub_rn(__dsub_rn(1.0, u), v), D[0]), __dmul_rn(u, D[1])),
                                     __dmul_rn(v, D[2]));
        const R3 r = sub(y, x);
        const double rn = __dsqrt_rn(sqn(r));
        const double num = __dmul_rn(__dmul_rn(__dmul_rn(rw[i], 2.0), area), dot3(n0, r));
        const double den = __dmul_rn(__dmul_rn(__dmul_rn(four_pi, rn), rn), rn);
        acc = __dadd_rn(acc, __dmul_rn(__ddiv_rn(num, den), val));
    }
    return acc;
}

// child k of a subdivided node (potential.hpp:55-68, children in the reference's order)
__device__ __forceinline__ void dl_child(const double* C, const double* D, int k, double* Cc, double* Dc)
{
    const R3 c0 = r3(C), c1 = r3(C + 3), c2 = r3(C + 6);
    const R3 m01 = scl(0.5, add(c0, c1)), m12 = scl(0.5, add(c1, c2)), m02 = scl(0.5, add(c0, c2));
    const double d01 = __dmul_rn(0.5, __dadd_rn(D[0], D[1])), d12 = __dmul_rn(0.5, __dadd_rn(D[1], D[2])),
                 d02 = __dmul_rn(0.5, __dadd_rn(D[0], D[2]));
    R3 a, b, c;
    double da, db, dc;
    if (k == 0) {
        a = c0, b = m01, c = m02, da = D[0], db = d01, dc = d02;
    } else if (k == 1) {
        a = m01, b = c1, c = m12, da = d01, db = D[1], dc = d12;
    } else if (k == 2) {
        a = m02, b = m12, c = c2, da = d02, db = d12, dc = D[2];
    } else {
        a = m01, b = m12, c = m02, da = d01, db = d12, dc = d02;
    }
    Cc[0] = a.x, Cc[1] = a.y, Cc[2] = a.z, Cc[3] = b.x, Cc[4] = b.y, Cc[5] = b.z, Cc[6] = c.x, Cc[7] = c.y,
    Cc[8] = c.z;
    Dc[0] = da, Dc[1] = db, Dc[2] = dc;
}

// the recursion of facet_dipole_integral from its root (depth 0 already classified as split),
// depth first with per-depth state: a node's children are summed acc = ((0 + S0) + S1) + ...,
// exactly the reference's association
__device__ double dl_facet_near(const double* root_C, const double* root_D, R3 n0, R3 x, const double* ru,
                                const double* rv, const double* rw, int nr)
{
    double C[DL_MAXDEPTH + 1][9], D[DL_MAXDEPTH + 1][3], acc[DL_MAXDEPTH + 1];
    int idx[DL_MAXDEPTH + 1];
    for (int i = 0; i < 9; ++i) C[0][i] = root_C[i];
    for (int i = 0; i < 3; ++i) D[0][i] = root_D[i];
    acc[0] = 0.0;
    idx[0] = 0;
    dl_child(C[0], D[0], 0, C[1], D[1]);
    int d = 1;
    double ret = 0.0;
    bool back = false;
    while (true) {
        if (!back) {
            const R3 a = r3(C[d]), b = r3(C[d] + 3), c = r3(C[d] + 6);
            if (pt_tri_dist(x, a, b, c) < tri_diam3(a, b, c) && d < DL_MAXDEPTH) {
                acc[d] = 0.0;
                idx[d] = 0;
                dl_child(C[d], D[d], 0, C[d + 1], D[d + 1]);
                ++d;
                continue;
            }
            ret = dl_leaf(C[d], D[d], n0, x, ru, rv, rw, nr);
            back = true;
        }
        --d;  // hand ret to the parent
        acc[d] = __dadd_rn(acc[d], ret);
        if (++idx[d] < 4) {
            dl_child(C[d], D[d], idx[d], C[d + 1], D[d + 1]);
            ++d;
            back = false;
            continue;
        }
        ret = acc[d];
        if (d == 0) return ret;
    }
}

__device__ __forceinline__ double rsqrt_refined(double r2)
{
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
    const double e = fma(-r2, y * y, 1.0);  // the seed's square is exact (kernels.cuh rsqrt_acc)
    return fma(y, e * fma(0.375, e, 0.5), y);
}

// per staged facet: record (c0 c1 c2 n0 dv) + derived (cen, rad, diam, k = 2A / 4 pi)
struct DlFacet {
    double C[9], n[3], dv[3], cen[3], rad, diam, k;
};

// DL_P points per thread (points base + k DL_THREADS): every staged y point serves DL_P points,
// two rule points per pass — 2 DL_P independent accumulation chains per thread
constexpr int DL_P_FAST = 4;  // (exact_far: 1 — its IEEE division and sqrt chains gain nothing from more)

template <bool EXACT, int DL_P>
__global__ void __launch_bounds__(DL_THREADS) k_dl_eval(const double* __restrict__ pts, long long np,
                                                       const double* __restrict__ frec, int nf, int per_split,
                                                       const double* __restrict__ rule, int nr,
                                                       double* __restrict__ part)
{
    extern __shared__ __align__(16) unsigned char dl_smem[];
    DlFacet* F = reinterpret_cast<DlFacet*>(dl_smem);
    double* ru = reinterpret_cast<double*>(F + DL_CHUNK);
    double* rv = ru + nr;
    double* rw = rv + nr;
    double4* Y = reinterpret_cast<double4*>(rw + nr + (nr & 1));  // DL_CHUNK x nr: (y, w_j [phi](y_j))
    for (int i = threadIdx.x; i < 3 * nr; i += blockDim.x) ru[i] = rule[i];
    const long long base = (long long)blockIdx.x * DL_THREADS * DL_P + threadIdx.x;
    R3 x[DL_P];
    bool act[DL_P];
    double acc[DL_P];
#pragma unroll
    for (int k = 0; k < DL_P; ++k) {
        const long long p = base + (long long)k * DL_THREADS;
        act[k] = p < np;
        // an inactive slot sits far away (its sums are computed and dropped)
        x[k] = act[k] ? R3{pts[3 * p], pts[3 * p + 1], pts[3 * p + 2]} : R3{1e3, 1e3, 1e3};
        acc[k] = 0.0;
    }
    const int f0 = blockIdx.y * per_split, f1 = min(nf, f0 + per_split);
    for (int fc = f0; fc < f1; fc += DL_CHUNK) {
        const int cnt = min(DL_CHUNK, f1 - fc);
        __syncthreads();  // previous chunk consumed (and the rule staged)
        for (int e = threadIdx.x; e < cnt; e += blockDim.x) {
            DlFacet& G = F[e];
            const double* r = frec + (size_t)(fc + e) * DL_REC;
            for (int i = 0; i < 9; ++i) G.C[i] = r[i];
            for (int i = 0; i < 3; ++i) G.n[i] = r[9 + i], G.dv[i] = r[12 + i];
            const R3 a = r3(G.C), b = r3(G.C + 3), c = r3(G.C + 6);
            G.diam = tri_diam3(a, b, c);
            const double cx = (a.x + b.x + c.x) / 3.0, cy = (a.y + b.y + c.y) / 3.0, cz = (a.z + b.z + c.z) / 3.0;
            G.cen[0] = cx, G.cen[1] = cy, G.cen[2] = cz;
            auto d2 = [&](R3 v) { return (v.x - cx) * (v.x - cx) + (v.y - cy) * (v.y - cy) + (v.z - cz) * (v.z - cz); };
            G.rad = sqrt(fmax(fmax(d2(a), d2(b)), d2(c))) * (1.0 + 1e-12);
            G.k = sqrt(sqn(crs(sub(b, a), sub(c, a)))) * (0.5 * 2.0 / (4.0 * M_PI));
        }
        __syncthreads();
        if (!EXACT) {
            for (int e = threadIdx.x; e < cnt * nr; e += blockDim.x) {
                const int f = e / nr, j = e - f * nr;
                const DlFacet& G = F[f];
                const double u = ru[j], v = rv[j];
                const double y0 = G.C[0] + u * (G.C[3] - G.C[0]) + v * (G.C[6] - G.C[0]);
                const double y1 = G.C[1] + u * (G.C[4] - G.C[1]) + v * (G.C[7] - G.C[1]);
                const double y2 = G.C[2] + u * (G.C[5] - G.C[2]) + v * (G.C[8] - G.C[2]);
                const double val = (1.0 - u - v) * G.dv[0] + u * G.dv[1] + v * G.dv[2];
                Y[f * nr + j] = make_double4(y0, y1, y2, rw[j] * val);
            }
            __syncthreads();
        }
        for (int f = 0; f < cnt; ++f) {
            const DlFacet& G = F[f];
            const R3 n0 = {G.n[0], G.n[1], G.n[2]};
            // the reference's test dist < diam (depth 0); skipped when the bounding sphere puts
            // the facet certainly farther than its diameter
            bool near[DL_P];
#pragma unroll
            for (int k = 0; k < DL_P; ++k) {
                const double dcx = x[k].x - G.cen[0], dcy = x[k].y - G.cen[1], dcz = x[k].z - G.cen[2];
                const double dc = sqrt(dcx * dcx + dcy * dcy + dcz * dcz);
                near[k] = false;
                if (act[k] && dc - G.rad - G.diam <= 1e-12 * (dc + G.rad + G.diam))
                    near[k] = pt_tri_dist(x[k], r3(G.C), r3(G.C + 3), r3(G.C + 6)) < G.diam;
            }
            if (EXACT) {
#pragma unroll
                for (int k = 0; k < DL_P; ++k)
                    if (act[k]) {
                        const double val = near[k] ? dl_facet_near(G.C, G.dv, n0, x[k], ru, rv, rw, nr)
                                                   : dl_leaf(G.C, G.dv, n0, x[k], ru, rv, rw, nr);
                        acc[k] = __dadd_rn(acc[k], val);
                    }
                continue;
            }
            // far form: (2A / 4 pi) n.(c0 - x) sum_j w_j [phi](y_j) / |y_j - x|^3
            double s0[DL_P], s1[DL_P];
#pragma unroll
            for (int k = 0; k < DL_P; ++k) s0[k] = s1[k] = 0.0;
            const double4* Yf = Y + f * nr;
            int j = 0;
            for (; j + 1 < nr; j += 2) {
                const double4 ya = Yf[j], yb = Yf[j + 1];
#pragma unroll
                for (int k = 0; k < DL_P; ++k) {
                    const double ax = ya.x - x[k].x, ay = ya.y - x[k].y, az = ya.z - x[k].z;
                    const double bx = yb.x - x[k].x, by = yb.y - x[k].y, bz = yb.z - x[k].z;
                    const double ia = rsqrt_refined(fma(ax, ax, fma(ay, ay, az * az)));
                    const double ib = rsqrt_refined(fma(bx, bx, fma(by, by, bz * bz)));
                    s0[k] = fma(ya.w, ia * ia * ia, s0[k]);
                    s1[k] = fma(yb.w, ib * ib * ib, s1[k]);
                }
            }
            if (j < nr) {
                const double4 ya = Yf[j];
#pragma unroll
                for (int k = 0; k < DL_P; ++k) {
                    const double ax = ya.x - x[k].x, ay = ya.y - x[k].y, az = ya.z - x[k].z;
                    const double ia = rsqrt_refined(fma(ax, ax, fma(ay, ay, az * az)));
                    s0[k] = fma(ya.w, ia * ia * ia, s0[k]);
                }
            }
#pragma unroll
            for (int k = 0; k < DL_P; ++k) {
                const double nd = G.n[0] * (G.C[0] - x[k].x) + G.n[1] * (G.C[1] - x[k].y) + G.n[2] * (G.C[2] - x[k].z);
                // (rare) a subdivided facet's value replaces the far form's, which is dropped
                acc[k] += near[k] ? dl_facet_near(G.C, G.dv, n0, x[k], ru, rv, rw, nr) : G.k * nd * (s0[k] + s1[k]);
            }
        }
    }
#pragma unroll
    for (int k = 0; k < DL_P; ++k)
        if (act[k]) part[(size_t)blockIdx.y * np + base + (long long)k * DL_THREADS] = acc[k];
}

__global__ void k_dl_reduce(const double* __restrict__ part, long long np, int splits, double* __restrict__ out)
{
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= np) return;
    double s = 0.0;
    for (int k = 0; k < splits; ++k) s += part[(size_t)k * np + p];
    out[p] = s;
}

// per point: 1 if some facet lies within thr (the reference's distance_to(x) <= thr, exact
// distances where the bounding sphere cannot decide)
__global__ void __launch_bounds__(DL_THREADS) k_dl_within(const double* __restrict__ pts, long long np,
                                                         const double* __restrict__ frec, int nf, double thr,
                                                         int* __restrict__ flag)
{
    __shared__ double S[DL_CHUNK][13];  // 9 corners, centroid, radius
    const long long p = (long long)blockIdx.x * DL_THREADS + threadIdx.x;
    const bool active = p < np;
    const R3 x = active ? R3{pts[3 * p], pts[3 * p + 1], pts[3 * p + 2]} : R3{0.0, 0.0, 0.0};
    int hit = 0;
    for (int fc = 0; fc < nf; fc += DL_CHUNK) {
        const int cnt = min(DL_CHUNK, nf - fc);
        __syncthreads();
        for (int e = threadIdx.x; e < cnt; e += blockDim.x) {
            const double* r = frec + (size_t)(fc + e) * DL_REC;
            for (int i = 0; i < 9; ++i) S[e][i] = r[i];
            const double cx = (r[0] + r[3] + r[6]) / 3.0, cy = (r[1] + r[4] + r[7]) / 3.0,
                         cz = (r[2] + r[5] + r[8]) / 3.0;
            double m = 0.0;
            for (int k = 0; k < 3; ++k) {
                const double dx = r[3 * k] - cx, dy = r[3 * k + 1] - cy, dz = r[3 * k + 2] - cz;
                m = fmax(m, dx * dx + dy * dy + dz * dz);
            }
            S[e][9] = cx, S[e][10] = cy, S[e][11] = cz, S[e][12] = sqrt(m) * (1.0 + 1e-12);
        }
        __syncthreads();
        if (active && !hit)
            for (int f = 0; f < cnt; ++f) {
                const double dx = x.x - S[f][9], dy = x.y - S[f][10], dz = x.z - S[f][11];
                const double dc = sqrt(dx * dx + dy * dy + dz * dz);
                if (dc - S[f][12] - thr > 1e-12 * (dc + S[f][12] + thr)) continue;
                if (pt_tri_dist(x, r3(S[f]), r3(S[f] + 3), r3(S[f] + 6)) <= thr) {
                    hit = 1;
                    break;
                }
            }
    }
    if (active) flag[p] = hit;
}

// per-facet records: corners, the side-0 normal, the side-0 minus side-1 trace values of the
// jump density at the corners (potential.hpp:109, 123-125; jump.hpp:45-57 expand)
std::vector<double> facet_records(const InflatedMesh& im, const double* v)
{
    const SurfaceMesh& m = im.base;
    std::vector<double> coeff(im.num_gvertices(), 0.0);
    if (v)
        for (int d = 0; d < im.num_jump_dofs(); ++d) {
            const auto& jd = im.jump_dofs[d];
            coeff[im.gv_index(jd[0], jd[1])] += v[d];
            coeff[im.gv_index(jd[0], im.q[jd[0]] - 1)] -= v[d];
        }
    std::vector<double> rec((size_t)m.num_facets() * DL_REC, 0.0);
    for (int f = 0; f < m.num_facets(); ++f) {
        double* r = rec.data() + (size_t)f * DL_REC;
        for (int k = 0; k < 3; ++k) {
            const Vec3& p = m.vertices[m.facets[f][k]];
            r[3 * k] = p.x, r[3 * k + 1] = p.y, r[3 * k + 2] = p.z;
            const int vk = m.facets[f][k];
            r[12 + k] = coeff[im.gv_index(vk, im.ofacet_branch[2 * f][k])] -
                        coeff[im.gv_index(vk, im.ofacet_branch[2 * f + 1][k])];
        }
        const Vec3& n = im.onormal[2 * f];
        r[9] = n.x, r[10] = n.y, r[11] = n.z;
    }
    return rec;
}

std::vector<double> mesh_records(const SurfaceMesh& m)
{
    std::vector<double> rec((size_t)m.num_facets() * DL_REC, 0.0);
    for (int f = 0; f < m.num_facets(); ++f)
        for (int k = 0; k < 3; ++k) {
            const Vec3& p = m.vertices[m.facets[f][k]];
            double* r = rec.data() + (size_t)f * DL_REC;
            r[3 * k] = p.x, r[3 * k + 1] = p.y, r[3 * k + 2] = p.z;
        }
    return rec;
}

// flag[p] = 1 if some facet lies within thr of point p
void points_within(Ctx* ctx, const DBuf<double>& d_rec, int nf, const DBuf<double>& d_pts, long long np, double thr,
                   std::vector<int>& flag)
{
    cudaStream_t s = ctx->stream;
    flag.assign((size_t)np, 0);
    if (np == 0 || nf == 0) return;
    DBuf<int> d_flag((size_t)np);
    k_dl_within<<<(unsigned)((np + DL_THREADS - 1) / DL_THREADS), DL_THREADS, 0, s>>>(d_pts.p, np, d_rec.p, nf, thr,
                                                                                      d_flag.p);
    count_launch();
    SBG_LAUNCH_CHECK();
    SBG_CUDA(cudaMemcpyAsync(flag.data(), d_flag.p, np * sizeof(int), cudaMemcpyDeviceToHost, s));
    SBG_CUDA(cudaStreamSynchronize(s));
}

}  // namespace

// reference: inc/potential.hpp:104-138 (3-D)
void eval_dl(Ctx* ctx, const InflatedMesh& im, const double* v, const double* points, long long np,
             const QuadCfg& cfg, double* out)
{
    if (np < 0) throw ValidationError("eval_DL: negative point count");
    if (cfg.far_order < 1) throw ValidationError("eval_DL: far order must be positive");
    if (np == 0) return;
    const SurfaceMesh& m = im.base;
    const int nf = m.num_facets();
    TimedScope ts(ctx, "eval_dl");
    cudaStream_t s = ctx->stream;
    const std::vector<double> rec = facet_records(im, v);
    const TriangleRule tri = triangle_rule(cfg.far_order + 2);  // potential.hpp:110
    const int nr = (int)tri.w.size();
    std::vector<double> rule(3 * (size_t)nr);
    for (int i = 0; i < nr; ++i) rule[i] = tri.u[i], rule[nr + i] = tri.v[i], rule[2 * nr + i] = tri.w[i];
    DBuf<double> d_rec(std::max<size_t>(rec.size(), 1)), d_pts(3 * (size_t)np), d_rule(rule.size());
    SBG_CUDA(cudaMemcpyAsync(d_rec.p, rec.data(), rec.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    SBG_CUDA(cudaMemcpyAsync(d_pts.p, points, 3 * (size_t)np * sizeof(double), cudaMemcpyHostToDevice, s));
    SBG_CUDA(cudaMemcpyAsync(d_rule.p, rule.data(), rule.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    // potential.hpp:112, 119-120: no point within half a millionth of the largest facet
    const double mask = 0.5 * m.max_facet_diameter() * 1e-6;
    std::vector<int> flag;
    points_within(ctx, d_rec, nf, d_pts, np, mask, flag);
    for (long long p = 0; p < np; ++p)
        if (flag[p]) throw ValidationError("evaluation point lies on the screen");
    if (nf == 0) {
        std::fill(out, out + np, 0.0);
        return;
    }
    // facet ranges per point block (partial sums reduced in range order); exact_far keeps one
    // range, so the sum runs over all facets in order like the reference's
    const int P = cfg.exact_far ? 1 : DL_P_FAST;
    const long long pblocks = (np + DL_THREADS * P - 1) / (DL_THREADS * P);
    int splits = 1;
    if (!cfg.exact_far) {
        const long long want = (2LL * ctx->sm_count * 4 + pblocks - 1) / pblocks;
        splits = (int)std::max<long long>(1, std::min<long long>(want, (nf + DL_CHUNK - 1) / DL_CHUNK));
    }
    int per = (nf + splits - 1) / splits;
    per = (per + DL_CHUNK - 1) / DL_CHUNK * DL_CHUNK;
    splits = (nf + per - 1) / per;
    DBuf<double> d_part((size_t)splits * np), d_out((size_t)np);
    const size_t smem = DL_CHUNK * sizeof(DlFacet) + (3 * (size_t)nr + 1) * sizeof(double) +
                        (cfg.exact_far ? 0 : (size_t)DL_CHUNK * nr * sizeof(double4)) + 16;
    const dim3 grid((unsigned)pblocks, (unsigned)splits);
    if (cfg.exact_far) {
        set_max_dynamic_smem(k_dl_eval<true, 1>, smem);
        k_dl_eval<true, 1><<<grid, DL_THREADS, smem, s>>>(d_pts.p, np, d_rec.p, nf, per, d_rule.p, nr, d_part.p);
    } else {
        set_max_dynamic_smem(k_dl_eval<false, DL_P_FAST>, smem);
        k_dl_eval<false, DL_P_FAST><<<grid, DL_THREADS, smem, s>>>(d_pts.p, np, d_rec.p, nf, per, d_rule.p, nr,
                                                                   d_part.p);
    }
    count_launch();
    SBG_LAUNCH_CHECK();
    const double* res = d_part.p;
    if (splits > 1) {
        k_dl_reduce<<<(unsigned)((np + 255) / 256), 256, 0, s>>>(d_part.p, np, splits, d_out.p);
        count_launch();
        SBG_LAUNCH_CHECK();
        res = d_out.p;
    }
    SBG_CUDA(cudaMemcpyAsync(out, res, np * sizeof(double), cudaMemcpyDeviceToHost, s));
    SBG_CUDA(cudaStreamSynchronize(s));
}

// reference: inc/potential.hpp:15-25 and mesh.hpp:121-133 (distance_to(p) > mask_eps keeps p)
std::vector<double> make_cartesian_grid(Ctx* ctx, const SurfaceMesh& m, double lo, double hi, int nx, int ny,
                                        double mask_eps)
{
    if (nx < 0 || ny < 0) throw ValidationError("cartesian grid: negative size");
    std::vector<double> cand;
    cand.reserve(3 * (size_t)nx * ny);
    for (int i = 0; i < nx; ++i)
        for (int j = 0; j < ny; ++j) {
            cand.push_back(lo + (hi - lo) * (i + 0.5) / nx);
            cand.push_back(lo + (hi - lo) * (j + 0.5) / ny);
            cand.push_back(0.0);
        }
    const long long np = (long long)nx * ny;
    if (np == 0) return {};
    if (m.num_facets() == 0) return cand;  // distance_to = 1e300
    const std::vector<double> rec = mesh_records(m);
    cudaStream_t s = ctx->stream;
    DBuf<double> d_rec(rec.size()), d_pts(cand.size());
    SBG_CUDA(cudaMemcpyAsync(d_rec.p, rec.data(), rec.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    SBG_CUDA(cudaMemcpyAsync(d_pts.p, cand.data(), cand.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    std::vector<int> flag;
    points_within(ctx, d_rec, m.num_facets(), d_pts, np, mask_eps, flag);
    std::vector<double> kept;
    for (long long p = 0; p < np; ++p)
        if (!flag[p]) kept.insert(kept.end(), cand.begin() + 3 * p, cand.begin() + 3 * p + 3);
    return kept;
}

}  // namespace sbg
