// Dense Galerkin assembly of the hypersingular form on the device.
// reference: inc/assemble.hpp:72-139 (assemble_W), :143-184 (assemble_rhs),
//            inc/quadrature.hpp:186-334 (pair classification and rules).
//
// Work split (each class in its own warp-uniform batch):
//   * far pairs  (depth-0 leaves, 16x16 rule): tiles of 64x64 facets of a
//     Morton-ordered facet permutation.  Lanes own one facet (its 16 points in
//     registers), loop over the 64 facets of the other block, and write the
//     pair integrals into a shared-memory tile that is contracted with the
//     blocks' side-merged curl lists and flushed into W with fp64 RED.
//   * near pairs (split4 recursion to depth 5, 36x36 leaves): one warp per
//     pair walks the recursion in the reference's child order (no-FMA
//     classification, bitwise identical decisions) and evaluates leaves two at
//     a time on the two half-warps (9x9 register blocks per lane).
//   * coincident / edge / vertex pairs (Sauter rules, 60000/50000/20000
//     points): one lane per pair, rule points broadcast from shared memory,
//     point range split over CTAs, fixed-order reduction.
//   Near and singular pair integrals are scattered per pair; W is accumulated
//   in its upper triangle and mirrored at the end (assemble.hpp:136-137).
#include <algorithm>
#include <array>
#include <cstring>
#include <optional>
#include <cmath>
#include <future>
#include <thread>
#include <numeric>
#include <stdexcept>
#include <string>
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "kernels.cuh"

#include <map>
#include <memory>
#include <mutex>

namespace sbg {

namespace {

constexpr int BS = 64;          // facets per block
constexpr int FAR_THREADS = 256;
constexpr int NF = 16;          // far rule points at the default far_order 4
constexpr int NN = 36;          // near rule points at the default ((far_order + 2)^2)
constexpr int MAX_FAR_ORDER = 8;
constexpr int NF_MAX = 64;      // far rule capacity, padded to a multiple of 4 (far_order <= 8)
constexpr int NN_MAX = 112;     // near rule capacity, padded to a multiple of 16
constexpr int SAUTER_THREADS = 128;
constexpr int SAUTER_STAGE = 1024;  // rule points staged per smem pass

// rule sizes for a far_order (quadrature.hpp:105-112: far rule of far_order, near
// rule of far_order + 2), and the padded sizes the kernels are instantiated for
struct RuleDims {
    int far_order = 4, nf = NF, nfp = NF, nn = NN, nnp = NN;
};
RuleDims rule_dims(int far_order)
{
    if (far_order < 1 || far_order > MAX_FAR_ORDER)
        throw ValidationError("far_order must be in [1, " + std::to_string(MAX_FAR_ORDER) + "] on the GPU path");
    RuleDims r;
    r.far_order = far_order;
    r.nf = far_order * far_order;
    r.nfp = (r.nf + 3) / 4 * 4;
    r.nn = (far_order + 2) * (far_order + 2);
    r.nnp = far_order == 4 ? NN : (r.nn + 15) / 16 * 16;  // the default keeps its exact-fit kernel
    return r;
}

// rules padded with zero-weight points at the centroid (their terms add exact zeros)
__constant__ double c_far_u[NF_MAX], c_far_v[NF_MAX], c_far_w[NF_MAX];
__constant__ double c_near_u[NN_MAX], c_near_v[NN_MAX], c_near_w[NN_MAX];
// 1 / w^2 per rule point (0 for the zero-weight padding): the y points are staged scaled by
// it, so rsqrt of the scaled squared distance is already w_j / |x - y| (rsqrt_acc)
__constant__ double c_far_s[NF_MAX], c_near_s[NN_MAX];
// composed split4 maps: for every child path of depth <= 5 (index (4^d-1)/3 + base-4 digits),
// the barycentric weights (x32, exact dyadics) of the leaf vertices on the root vertices
constexpr int NPATH = 1365;
__constant__ unsigned char c_paths[NPATH * 9];
// the same near rule and path tables in global memory: read through L1 (__ldg) where the lanes
// of a warp index them divergently (the constant cache serialises distinct addresses)
__device__ double g_near_u[NN_MAX], g_near_v[NN_MAX], g_near_s[NN_MAX], g_near_w[NN_MAX];
__device__ unsigned char g_paths[NPATH * 9];
#ifndef NEAR_GLOBAL_TABLES
#define NEAR_GLOBAL_TABLES 1
#endif
#if NEAR_GLOBAL_TABLES
#define NEAR_TAB(name, i) __ldg(&g_##name[i])
#else
#define NEAR_TAB(name, i) c_##name[i]
#endif

// ---------------------------------------------------------------- facet geometry
struct GeoPtrs {
    const double* v;     // 9 per facet: t0,t1,t2 in stored order
    const double* c;     // centroid (3)
    const double* rad;   // max centroid-vertex distance
    const double* diam;  // max edge length
    const double* area;
    const int* vid;      // 3 vertex ids
};

// per-facet classification data, no-FMA in the oracle's operation order
// (quadrature.hpp:186-206)
__global__ void k_facet_geometry(const double* __restrict__ X, const int* __restrict__ F, int nf, double* gv,
                                 double* gc, double* grad, double* gdiam, double* garea, int* gvid)
{
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= nf) return;
    D3 t[3];
    for (int k = 0; k < 3; ++k) {
        const int v = F[3 * f + k];
        gvid[3 * f + k] = v;
        t[k] = {X[3 * v], X[3 * v + 1], X[3 * v + 2]};
        gv[9 * f + 3 * k] = t[k].x;
        gv[9 * f + 3 * k + 1] = t[k].y;
        gv[9 * f + 3 * k + 2] = t[k].z;
    }
    const D3 s = d3_add(d3_add(t[0], t[1]), t[2]);
    const D3 c = {__ddiv_rn(s.x, 3.0), __ddiv_rn(s.y, 3.0), __ddiv_rn(s.z, 3.0)};
    double r = 0.0;
    for (int k = 0; k < 3; ++k) r = fmax(r, d3_norm(d3_sub(t[k], c)));
    const double d = fmax(fmax(d3_norm(d3_sub(t[0], t[1])), d3_norm(d3_sub(t[1], t[2]))), d3_norm(d3_sub(t[0], t[2])));
    gc[3 * f] = c.x;
    gc[3 * f + 1] = c.y;
    gc[3 * f + 2] = c.z;
    grad[f] = r;
    gdiam[f] = d;
    garea[f] = __dmul_rn(0.5, d3_norm(d3_cross(d3_sub(t[1], t[0]), d3_sub(t[2], t[0]))));
}

// dist_estimate(t, s) >= thr * max(diam_t, diam_s)  (quadrature.hpp:186-196, 234-236)
__device__ __forceinline__ bool far_test(D3 ct, double rt, double dt, D3 cs, double rs, double ds, double thr)
{
    const double dist = fmax(0.0, __dsub_rn(__dsub_rn(d3_norm(d3_sub(ct, cs)), rt), rs));
    return dist >= __dmul_rn(thr, fmax(dt, ds));
}

__device__ __forceinline__ int shared_count(const int* a, const int* b)
{
    int s = 0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            if (a[i] == b[j]) {
                ++s;
                break;
            }
    return s;
}

// ---------------------------------------------------------------- far tiles
struct BlockPtrs {
    const int* facets;    // nblk * BS original facet ids (-1 padding)
    const int* dof_ptr;   // nblk + 1 into dofs
    const int* dofs;      // per-block sorted dof ids
    const int* ent_ptr;   // per block-local dof: start into ents (global index), size total_dofs + 1
    const double4* ents;  // (ux, uy, uz, facet_local)
};

struct TileInfo {
    int fb, gb, certain_far, pad;
};

// flush of one contracted W entry into W's upper triangle (W(j,i) = W(i,j) after the mirror)
__device__ __forceinline__ void flush_entry(double* __restrict__ W, int ld, bool diag, int da, int db, double s)
{
    if (s == 0.0) return;
    if (diag) {
        atomicAdd(W + (size_t)da * ld + db, s);
    } else if (da < db) {
        atomicAdd(W + (size_t)da * ld + db, s);
    } else if (da > db) {
        atomicAdd(W + (size_t)db * ld + da, s);
    } else {
        atomicAdd(W + (size_t)da * ld + da, 2.0 * s);
    }
}

// contraction of the I tile with the curl lists, flushed to W's upper triangle.  stage:
// shared memory no longer needed by the caller (stage_bytes of it): both blocks' curl-list
// entries are staged there once (u vectors + the I-tile row / column offsets as integers)
// instead of being re-read from global memory inside the double loop; blocks whose entries do
// not fit take the global path.
__device__ void tile_contract_flush(const double* __restrict__ It, int fb, int gb, bool diag, const BlockPtrs& B,
                                    double* __restrict__ W, int ld, unsigned char* stage, size_t stage_bytes)
{
    const int fa0 = B.dof_ptr[fb], na = B.dof_ptr[fb + 1] - fa0;
    const int gb0 = B.dof_ptr[gb], nbd = B.dof_ptr[gb + 1] - gb0;
    const int ef0 = B.ent_ptr[fa0], nef = B.ent_ptr[fa0 + na] - ef0;
    const int eg0 = B.ent_ptr[gb0], neg = B.ent_ptr[gb0 + nbd] - eg0;
    const size_t need = (size_t)(nef + neg) * (sizeof(double) * 3 + sizeof(int));
    if (stage && need <= stage_bytes) {
        double* uf = reinterpret_cast<double*>(stage);  // nef x 3
        double* ug = uf + 3 * nef;                       // neg x 3
        int* of = reinterpret_cast<int*>(ug + 3 * neg);  // nef: I-tile row offset f_local (BS + 1)
        int* og = of + nef;                              // neg: I-tile column g_local
        for (int i = threadIdx.x; i < nef + neg; i += blockDim.x) {
            const bool isf = i < nef;
            const double4 e = B.ents[isf ? ef0 + i : eg0 + (i - nef)];
            double* u = isf ? uf + 3 * i : ug + 3 * (i - nef);
            u[0] = e.x, u[1] = e.y, u[2] = e.z;
            if (isf) of[i] = (int)e.w * (BS + 1);
            else og[i - nef] = (int)e.w;
        }
        __syncthreads();
        for (int e = threadIdx.x; e < na * nbd; e += blockDim.x) {
            const int a = e / nbd, b = e % nbd;
            const int da = B.dofs[fa0 + a], db = B.dofs[gb0 + b];
            if (diag && da > db) continue;
            const int p0 = B.ent_ptr[fa0 + a] - ef0, p1 = B.ent_ptr[fa0 + a + 1] - ef0;
            const int q0 = B.ent_ptr[gb0 + b] - eg0, q1 = B.ent_ptr[gb0 + b + 1] - eg0;
            double s = 0.0;
            for (int p = p0; p < p1; ++p) {
                const double ax = uf[3 * p], ay = uf[3 * p + 1], az = uf[3 * p + 2];
                const double* Irow = It + of[p];
                for (int q = q0; q < q1; ++q)
                    s = fma(Irow[og[q]], fma(ax, ug[3 * q], fma(ay, ug[3 * q + 1], az * ug[3 * q + 2])), s);
            }
            flush_entry(W, ld, diag, da, db, s);
        }
        return;
    }
    for (int e = threadIdx.x; e < na * nbd; e += blockDim.x) {
        const int a = e / nbd, b = e % nbd;
        const int da = B.dofs[fa0 + a], db = B.dofs[gb0 + b];
        if (diag && da > db) continue;
        double s = 0.0;
        for (int p = B.ent_ptr[fa0 + a]; p < B.ent_ptr[fa0 + a + 1]; ++p) {
            const double4 ea = B.ents[p];
            const double* Irow = It + (int)ea.w * (BS + 1);
            for (int q = B.ent_ptr[gb0 + b]; q < B.ent_ptr[gb0 + b + 1]; ++q) {
                const double4 eb = B.ents[q];
                s = fma(Irow[(int)eb.w], fma(ea.x, eb.x, fma(ea.y, eb.y, ea.z * eb.z)), s);
            }
        }
        flush_entry(W, ld, diag, da, db, s);
    }
}

// Two-stage contraction of the I tile (the default far path): W(a,b) = sum_k sum_{p in a}
// u_pk V_k(f_p, b)... computed as V_k(a, g) = sum_{p in E_a} u_pk I(f_p, g) (stage A, into
// shared memory, 32 DOFs of the f block at a time) and W(a,b) += sum_{q in E_b} V_k(a, g_q)
// u_qk (stage B, register accumulators kept over the three components k), ~2.3x fewer
// FP64 operations and no per-(p,q) dot products against the direct double loop; W(a,b)
// is the same sum up to the association of its terms.  Needs nbd <= 64 DOFs in the g block
// and 32 x 64 doubles of dead shared memory (vbuf); returns false (nothing done) otherwise.
constexpr int CT_CH = 32;  // f-block DOFs per stage-A round
__device__ bool tile_contract_flush_2stage(const double* __restrict__ It, int fb, int gb, bool diag,
                                           const BlockPtrs& B, double* __restrict__ W, int ld,
                                           double* __restrict__ vbuf, size_t vbuf_bytes)
{
    const int fa0 = B.dof_ptr[fb], na = B.dof_ptr[fb + 1] - fa0;
    const int gb0 = B.dof_ptr[gb], nbd = B.dof_ptr[gb + 1] - gb0;
    if (nbd > BS || vbuf_bytes < (size_t)CT_CH * BS * sizeof(double)) return false;
    const int t = threadIdx.x;
    const int col = t & (BS - 1), row0 = t >> 6;  // 256 threads: 4 rows x 64 columns per sweep
    constexpr int RPT = CT_CH / 4;                // rows of a round per thread
    for (int a0 = 0; a0 < na; a0 += CT_CH) {
        const int ca = min(CT_CH, na - a0);
        double acc[RPT];
#pragma unroll
        for (int i = 0; i < RPT; ++i) acc[i] = 0.0;
        // E_b of this thread's column b (its g-block entries)
        const int q0 = col < nbd ? B.ent_ptr[gb0 + col] : 0, q1 = col < nbd ? B.ent_ptr[gb0 + col + 1] : 0;
#pragma unroll 1
        for (int k = 0; k < 3; ++k) {
            // stage A: vbuf[al][g] = sum_{p in E_(a0+al)} u_pk I(f_p, g), g = col
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                const int al = row0 + 4 * i;
                double v = 0.0;
                if (al < ca) {
                    const int p0 = B.ent_ptr[fa0 + a0 + al], p1 = B.ent_ptr[fa0 + a0 + al + 1];
                    for (int p = p0; p < p1; ++p) {
                        const double4 e = B.ents[p];  // uniform over the 64 threads of the row
                        const double u = k == 0 ? e.x : (k == 1 ? e.y : e.z);
                        v = fma(u, It[(int)e.w * (BS + 1) + col], v);
                    }
                }
                vbuf[al * BS + col] = v;
            }
            __syncthreads();
            // stage B: acc[i] += sum_{q in E_b} vbuf[al][g_q] u_qk, b = col
            for (int q = q0; q < q1; ++q) {
                const double4 e = B.ents[q];
                const double u = k == 0 ? e.x : (k == 1 ? e.y : e.z);
                const double* vc = vbuf + (int)e.w;
#pragma unroll
                for (int i = 0; i < RPT; ++i) acc[i] = fma(vc[(row0 + 4 * i) * BS], u, acc[i]);
            }
            __syncthreads();
        }
        if (col < nbd) {
            const int db = B.dofs[gb0 + col];
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                const int al = row0 + 4 * i;
                if (al >= ca) continue;
                const int da = B.dofs[fa0 + a0 + al];
                if (diag && da > db) continue;
                flush_entry(W, ld, diag, da, db, acc[i]);
            }
        }
    }
    return true;
}

// Far pairs with the distance expansion |x-y|^2 = |x|^2 + |y|^2 - 2 x.y in
// tile-local coordinates (origin o = first vertex of the tile's first f-facet):
// per evaluation DADD + 3 DFMA instead of 3 DADD + DMUL + 2 DFMA.  Each lane keeps
// 4 of its facet's 16 rule points in registers per pass (3 CTAs of 256 per SM).  Far pairs
// satisfy dist >= 2 diam, so (|x|^2+|y|^2)/|x-y|^2 stays O(10) inside a tile and
// ~1 between distant tiles: the rounding stays at the 1e-15 level.
#ifndef FAR_PASS_PTS
#define FAR_PASS_PTS 8  // rule points of f per pass where the padded rule allows (else 4)
#endif
#ifndef FAR_CTAS
#define FAR_CTAS 2
#endif
constexpr int FAR_PASS = 4;  // the pass width every padded rule admits (nfp is a multiple of 4)
// the far kernel's pass width for a rule of NFP (padded) points: FAR_PASS_PTS (8: the default
// rule's 16 points in two passes, 2 CTAs/SM with 128 registers) when it divides NFP
template <int NFP>
constexpr int far_pass_for() { return NFP % FAR_PASS_PTS == 0 ? FAR_PASS_PTS : FAR_PASS; }
#ifndef FAR_FLAT_UNROLL
#define FAR_FLAT_UNROLL 16  // the whole default rule (A/B: 2 -> 16 took config 5 from 213 to 205 ms)
#endif
#ifndef FAR_GEN_UNROLL
#define FAR_GEN_UNROLL 2
#endif
template <int PW = FAR_PASS>
struct XPts {
    double m2x[PW], m2y[PW], m2z[PW], x2[PW];  // -2x, -2y, -2z, |x|^2
};

// coordinate order (P.x, P.y, P.z): the identity, or a flat tile's two in-plane axes first and
// its flat axis last (far_flat_axis)
template <int PW>
__device__ __forceinline__ void far_xpoints(const double* t, const double* o, int pass, XPts<PW>& X,
                                            int3 P = make_int3(0, 1, 2))
{
    const double e1x = t[3 + P.x] - t[P.x], e1y = t[3 + P.y] - t[P.y], e1z = t[3 + P.z] - t[P.z];
    const double e2x = t[6 + P.x] - t[P.x], e2y = t[6 + P.y] - t[P.y], e2z = t[6 + P.z] - t[P.z];
    const double bx = t[P.x] - o[P.x], by = t[P.y] - o[P.y], bz = t[P.z] - o[P.z];
#pragma unroll
    for (int q = 0; q < PW; ++q) {
        const int i = PW * pass + q;
        const double x = fma(c_far_v[i], e2x, fma(c_far_u[i], e1x, bx));
        const double y = fma(c_far_v[i], e2y, fma(c_far_u[i], e1y, by));
        const double z = fma(c_far_v[i], e2z, fma(c_far_u[i], e1z, bz));
        X.m2x[q] = -2.0 * x;
        X.m2y[q] = -2.0 * y;
        X.m2z[q] = -2.0 * z;
        X.x2[q] = fma(x, x, fma(y, y, z * z));
    }
}

// the staged y point of rule point j, scaled by s_j = 1/w_j^2: (s y, s |y|^2), so that
// s_j |x - y|^2 = s_j |x|^2 + s |y|^2 - 2 x.(s y) costs the same four instructions
__device__ __forceinline__ double4 scaled_ypoint(double y0, double y1, double y2, double sj)
{
    if (sj == 0.0) return make_double4(0.0, 0.0, 0.0, kPadR2);
    return make_double4(sj * y0, sj * y1, sj * y2, sj * fma(y0, y0, fma(y1, y1, y2 * y2)));
}

__device__ __forceinline__ double4 far_ypoint(const double* s, const double* o, int j, int3 P = make_int3(0, 1, 2))
{
    const double y0 = fma(c_far_v[j], s[6 + P.x] - s[P.x], fma(c_far_u[j], s[3 + P.x] - s[P.x], s[P.x] - o[P.x]));
    const double y1 = fma(c_far_v[j], s[6 + P.y] - s[P.y], fma(c_far_u[j], s[3 + P.y] - s[P.y], s[P.y] - o[P.y]));
    const double y2 = fma(c_far_v[j], s[6 + P.z] - s[P.z], fma(c_far_u[j], s[3 + P.z] - s[P.z], s[P.z] - o[P.z]));
    return scaled_ypoint(y0, y1, y2, c_far_s[j]);
}

// sum_{q in pass} w_{4 pass + q} sum_j w_j / |x_q - y_j|  (16 y-points x 4 x-points); one
// accumulator per x point, so the four evaluations per y point are independent chains;
// w_j is folded into the staged y point (far_ypoint, rsqrt_acc): 9 FP64 instructions and one
// MUFU per evaluation.  FLAT: every point of the tile has a zero last coordinate (a tile lying
// in one coordinate plane, far_flat_axis), whose product term -2 x_z y_z = -0 adds nothing:
// it is left out, 8 FP64 instructions per evaluation, the same value
template <int NFP, bool FLAT = false, int UNROLL = 2, int PW = FAR_PASS>
__device__ __forceinline__ double far_pass_sum(const XPts<PW>& X, const double4* __restrict__ Y, int pass)
{
    double a[PW];
#pragma unroll
    for (int q = 0; q < PW; ++q) a[q] = 0.0;
#pragma unroll UNROLL
    for (int j = 0; j < NFP; ++j) {
        const double4 y = Y[j];
        const double sj = c_far_s[j];
#pragma unroll
        for (int q = 0; q < PW; ++q) {
            const double r2 = FLAT ? fma(X.m2x[q], y.x, fma(X.m2y[q], y.y, fma(X.x2[q], sj, y.w)))
                                   : fma(X.m2x[q], y.x, fma(X.m2y[q], y.y, fma(X.m2z[q], y.z, fma(X.x2[q], sj, y.w))));
            a[q] = rsqrt_acc_s(r2, a[q]);
        }
    }
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < PW; ++q) acc = fma(c_far_w[PW * pass + q], a[q], acc);
    return acc * kRsqrtAccScale;
}

// SURVEY Appendix B switch: the oracle's triangle_pair_rule (quadrature.hpp:208-220) in its
// exact operation order — affine points, |x-y| by IEEE sqrt, 1/(4 pi r) by IEEE division,
// (w_i w_j) k summed i-major, then (acc 4) A_t A_s — so the depth-0 far integral is
// bitwise the CPU restatement's (t = the facet with the larger index)
__device__ __forceinline__ D3 affine_exact(const double* t, double u, double v)
{
    return {__dadd_rn(__dadd_rn(t[0], __dmul_rn(u, __dsub_rn(t[3], t[0]))), __dmul_rn(v, __dsub_rn(t[6], t[0]))),
            __dadd_rn(__dadd_rn(t[1], __dmul_rn(u, __dsub_rn(t[4], t[1]))), __dmul_rn(v, __dsub_rn(t[7], t[1]))),
            __dadd_rn(__dadd_rn(t[2], __dmul_rn(u, __dsub_rn(t[5], t[2]))), __dmul_rn(v, __dsub_rn(t[8], t[2])))};
}
__device__ double far_pair_exact(const double* t, const double* s, double area_t, double area_s, int nr)
{
    const double four_pi = 4.0 * M_PI;
    double acc = 0.0;
    for (int i = 0; i < nr; ++i) {
        const D3 x = affine_exact(t, c_far_u[i], c_far_v[i]);
        const double wi = c_far_w[i];
        for (int j = 0; j < nr; ++j) {
            const D3 y = affine_exact(s, c_far_u[j], c_far_v[j]);
            const double r = d3_norm(d3_sub(x, y));
            const double k = __ddiv_rn(1.0, __dmul_rn(four_pi, r));
            acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(wi, c_far_w[j]), k));
        }
    }
    return __dmul_rn(__dmul_rn(__dmul_rn(acc, 4.0), area_t), area_s);
}

constexpr size_t far_smem_bytes(int nfp)
{
    return (size_t)BS * (BS + 1) * 8 + (size_t)BS * nfp * 32 + (size_t)BS * 6 * 8 + (size_t)BS * 4 * 4;
}

// NFP: far rule size padded to a multiple of FAR_PASS (16 at the default far_order 4)
template <int NFP, bool EXACT>
__global__ void __launch_bounds__(FAR_THREADS, FAR_CTAS)
    k_far_tiles(const TileInfo* __restrict__ tiles, int tstride, GeoPtrs G, BlockPtrs B, double thr,
                double* __restrict__ W, int ld, double inv_pi, int nr)
{
    extern __shared__ __align__(16) unsigned char far_smem[];
    double4* Ys = reinterpret_cast<double4*>(far_smem);                 // BS x NFP y-points (y, |y|^2)
    double* It = reinterpret_cast<double*>(Ys + (EXACT ? 0 : BS * NFP)); // BS x (BS+1)
    double* gcr = It + BS * (BS + 1);                                   // cx, cy, cz, rad, diam, area
    int* gid = reinterpret_cast<int*>(gcr + BS * 6);
    int* gvid = gid + BS;
    __shared__ double o[3];
    __shared__ int nzax;  // bit a: some vertex of the tile differs from o in coordinate a
    const TileInfo T = tiles[(size_t)blockIdx.x * tstride];  // tstride > 1: one shard of the tile list
    const bool diag = T.fb == T.gb;
    if (threadIdx.x < 3) o[threadIdx.x] = G.v[9 * B.facets[T.fb * BS] + threadIdx.x];
    if (threadIdx.x == 0) nzax = 0;
    for (int e = threadIdx.x; e < BS; e += blockDim.x) {
        const int g = B.facets[T.gb * BS + e];
        gid[e] = g;
        if (g >= 0) {
            gcr[e * 6] = G.c[3 * g];
            gcr[e * 6 + 1] = G.c[3 * g + 1];
            gcr[e * 6 + 2] = G.c[3 * g + 2];
            gcr[e * 6 + 3] = G.rad[g];
            gcr[e * 6 + 4] = G.diam[g];
            gcr[e * 6 + 5] = G.area[g];
            for (int k = 0; k < 3; ++k) gvid[e * 3 + k] = G.vid[3 * g + k];
        }
    }
    for (int e = threadIdx.x; e < BS * (BS + 1); e += blockDim.x) It[e] = 0.0;
    __syncthreads();
    // a tile whose 128 facets all lie in one coordinate plane (a flat screen panel: every
    // config-5 tile, most of configs 3-4) has that coordinate equal to o's at every vertex, so
    // it is exactly zero in tile-local coordinates: it goes last and the evaluation skips it
    int3 P = make_int3(0, 1, 2);
    bool flat = false;
    if (!EXACT) {
        if (threadIdx.x < 2 * BS) {
            const int h = threadIdx.x < BS ? B.facets[T.fb * BS + threadIdx.x] : gid[threadIdx.x - BS];
            int m = 0;
            if (h >= 0)
                for (int k = 0; k < 9; ++k)
                    if (G.v[9 * h + k] != o[k % 3]) m |= 1 << (k % 3);
            if (m) atomicOr(&nzax, m);
        }
        __syncthreads();
        const int nz = nzax;
        flat = (nz & 7) != 7;
        if (!(nz & 4) || nz == 7) P = make_int3(0, 1, 2);
        else if (!(nz & 2)) P = make_int3(0, 2, 1);
        else P = make_int3(1, 2, 0);
        for (int e = threadIdx.x; e < BS * NFP; e += blockDim.x) {
            const int g = gid[e / NFP];
            Ys[e] = g >= 0 ? far_ypoint(G.v + 9 * g, o, e % NFP, P) : make_double4(0, 0, 0, 1);
        }
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int fl = (warp & 1) * 32 + lane;
    const int f = B.facets[T.fb * BS + fl];
    if (f >= 0) {
        // classification: far mask over this warp's 16 g-facets (bit m <-> gl = warp/2 + 4m)
        unsigned mask = 0;
        {
            const D3 cf = {G.c[3 * f], G.c[3 * f + 1], G.c[3 * f + 2]};
            const double rf = G.rad[f], df = G.diam[f];
            const int fv[3] = {G.vid[3 * f], G.vid[3 * f + 1], G.vid[3 * f + 2]};
            for (int m = 0, gl = warp >> 1; gl < BS; gl += FAR_THREADS / 64, ++m) {
                const int g = gid[gl];
                if (g < 0 || (diag && gl >= fl)) continue;
                bool far = true;
                if (!T.certain_far) {
                    if (shared_count(fv, gvid + 3 * gl) > 0) {
                        far = false;
                    } else {
                        const D3 cg = {gcr[gl * 6], gcr[gl * 6 + 1], gcr[gl * 6 + 2]};
                        far = (f > g) ? far_test(cf, rf, df, cg, gcr[gl * 6 + 3], gcr[gl * 6 + 4], thr)
                                      : far_test(cg, gcr[gl * 6 + 3], gcr[gl * 6 + 4], cf, rf, df, thr);
                    }
                }
                if (far) mask |= 1u << m;
            }
        }
        if (EXACT) {
            for (int m = 0, gl = warp >> 1; gl < BS; gl += FAR_THREADS / 64, ++m) {
                if (!(mask >> m & 1)) continue;
                const int g = gid[gl];
                const int tt = f > g ? f : g, ss = f > g ? g : f;
                It[fl * (BS + 1) + gl] = far_pair_exact(G.v + 9 * tt, G.v + 9 * ss, G.area[tt], G.area[ss], nr);
            }
        }
        const double sf = G.area[f] * inv_pi;
        constexpr int PW = far_pass_for<NFP>();
        for (int pass = 0; !EXACT && pass < NFP / PW; ++pass) {
            XPts<PW> X;
            far_xpoints(G.v + 9 * f, o, pass, X, P);
            if (flat) {
                for (int m = 0, gl = warp >> 1; gl < BS; gl += FAR_THREADS / 64, ++m) {
                    if (!(mask >> m & 1)) continue;
                    It[fl * (BS + 1) + gl] += far_pass_sum<NFP, true, FAR_FLAT_UNROLL, PW>(X, Ys + gl * NFP, pass) * sf * gcr[gl * 6 + 5];
                }
            } else {
                for (int m = 0, gl = warp >> 1; gl < BS; gl += FAR_THREADS / 64, ++m) {
                    if (!(mask >> m & 1)) continue;
                    It[fl * (BS + 1) + gl] += far_pass_sum<NFP, false, FAR_GEN_UNROLL, PW>(X, Ys + gl * NFP, pass) * sf * gcr[gl * 6 + 5];
                }
            }
        }
    }
    __syncthreads();
    if (diag) {  // mirror the strictly-lower half computed above
        for (int e = threadIdx.x; e < BS * BS; e += blockDim.x) {
            const int i = e / BS, j = e % BS;
            if (j > i) It[i * (BS + 1) + j] = It[j * (BS + 1) + i];
        }
        __syncthreads();
    }
    // the staged y points are dead: their shared memory takes the contraction's buffers
    if (!EXACT && tile_contract_flush_2stage(It, T.fb, T.gb, diag, B, W, ld, reinterpret_cast<double*>(Ys),
                                             (size_t)BS * NFP * sizeof(double4)))
        return;
    tile_contract_flush(It, T.fb, T.gb, diag, B, W, ld, EXACT ? nullptr : reinterpret_cast<unsigned char*>(Ys),
                        EXACT ? 0 : (size_t)BS * NFP * sizeof(double4));
}

// Warp-aggregated append to a global list: every lane of the (converged) warp calls it;
// lane i wants n_i slots; one atomicAdd per warp instead of one per record (the near field
// appends tens of millions of records to two counters).  Returns lane i's first slot.
__device__ __forceinline__ unsigned long long warp_append(unsigned long long* counter, unsigned n)
{
    const int lane = threadIdx.x & 31;
    unsigned incl = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    const unsigned total = __shfl_sync(0xffffffffu, incl, 31);
    unsigned long long base = 0;
    if (lane == 31 && total) base = atomicAdd(counter, (unsigned long long)total);
    base = __shfl_sync(0xffffffffu, base, 31);
    return base + (incl - n);
}

// near-list builder: pairs of non-certainly-far tiles that are disjoint but not far
// (BS * BS is a multiple of the block size, so every warp runs the same trip count)
__global__ void k_classify_near(const TileInfo* __restrict__ tiles, int tstride, GeoPtrs G,
                                const int* __restrict__ bfacets, double thr, int2* __restrict__ near_list,
                                unsigned long long cap, unsigned long long* __restrict__ count)
{
    const TileInfo T = tiles[(size_t)blockIdx.x * tstride];
    const bool diag = T.fb == T.gb;
    for (int e = threadIdx.x; e < BS * BS; e += blockDim.x) {
        const int fl = e / BS, gl = e % BS;
        bool near = !(diag && gl >= fl);
        int t = 0, s = 0;
        if (near) {
            const int f = bfacets[T.fb * BS + fl], g = bfacets[T.gb * BS + gl];
            near = f >= 0 && g >= 0 && shared_count(G.vid + 3 * f, G.vid + 3 * g) == 0;
            if (near) {
                t = max(f, g);
                s = min(f, g);
                const D3 ct = {G.c[3 * t], G.c[3 * t + 1], G.c[3 * t + 2]};
                const D3 cs = {G.c[3 * s], G.c[3 * s + 1], G.c[3 * s + 2]};
                near = !far_test(ct, G.rad[t], G.diam[t], cs, G.rad[s], G.diam[s], thr);
            }
        }
        const unsigned long long k = warp_append(count, near ? 1u : 0u);
        if (near && k < cap) near_list[k] = make_int2(t, s);
    }
}

// ---------------------------------------------------------------- near pairs (recursion)
// The split4 recursion of triangle_pair_disjoint (quadrature.hpp:231-249) is
// run level-synchronously: the frontier of recursion nodes at depth L is a list
// of (local pair index, path code) records; one thread per node replays its
// path from the pair's triangles, classifies it with no-FMA arithmetic (bitwise
// the oracle's decision: leaf iff dist >= thr * diam or depth >= 5, split the
// larger triangle, t on ties) and appends either a leaf record or its four
// children.  Leaves of each level are then evaluated two per warp (one per
// half-warp, a 9x9 block of the 36x36 rule per lane) and accumulated into the
// pair's integral.  Path code: bits 0-2 depth, then per level 3 bits
// (split side | child << 1).
__device__ __forceinline__ double tri_diam(const double* t)
{
    const D3 a = {t[0], t[1], t[2]}, b = {t[3], t[4], t[5]}, c = {t[6], t[7], t[8]};
    // sqrt is monotone and correctly rounded: sqrt(max) == max(sqrt), one sqrt instead of three
    return __dsqrt_rn(fmax(fmax(d3_sqnorm(d3_sub(a, b)), d3_sqnorm(d3_sub(b, c))), d3_sqnorm(d3_sub(a, c))));
}
__device__ __forceinline__ void tri_centroid_rad(const double* t, D3& c, double& r)
{
    const D3 a = {t[0], t[1], t[2]}, b = {t[3], t[4], t[5]}, d = {t[6], t[7], t[8]};
    const D3 s = d3_add(d3_add(a, b), d);
    c = {__ddiv_rn(s.x, 3.0), __ddiv_rn(s.y, 3.0), __ddiv_rn(s.z, 3.0)};
    r = __dsqrt_rn(fmax(fmax(d3_sqnorm(d3_sub(a, c)), d3_sqnorm(d3_sub(b, c))), d3_sqnorm(d3_sub(d, c))));
}
__device__ __forceinline__ double tri_area(const double* t)
{
    const D3 a = {t[0], t[1], t[2]}, b = {t[3], t[4], t[5]}, c = {t[6], t[7], t[8]};
    return __dmul_rn(0.5, d3_norm(d3_cross(d3_sub(b, a), d3_sub(c, a))));
}
// child k of split4 (quadrature.hpp:222-229): {v0,m01,m02},{m01,v1,m12},{m02,m12,v2},{m01,m12,m02}
__device__ __forceinline__ void split4_child_inplace(double* t, int k)
{
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const double v0 = t[c], v1 = t[3 + c], v2 = t[6 + c];
        const double m01 = __dmul_rn(0.5, __dadd_rn(v0, v1));
        const double m12 = __dmul_rn(0.5, __dadd_rn(v1, v2));
        const double m02 = __dmul_rn(0.5, __dadd_rn(v0, v2));
        t[c] = k == 0 ? v0 : (k == 2 ? m02 : m01);
        t[3 + c] = k == 0 ? m01 : (k == 1 ? v1 : m12);
        t[6 + c] = k == 0 ? m02 : (k == 1 ? m12 : (k == 2 ? v2 : m02));
    }
}
// triangles of the node (pair root triangles replayed along the path)
__device__ __forceinline__ void node_triangles(const double* __restrict__ GV, int2 pr, unsigned code, double* t,
                                               double* s)
{
#pragma unroll
    for (int c = 0; c < 9; ++c) {
        t[c] = __ldg(GV + 9 * pr.x + c);
        s[c] = __ldg(GV + 9 * pr.y + c);
    }
    const int depth = code & 7;
    for (int lv = 0; lv < depth; ++lv) {
        const unsigned e = (code >> (3 + 3 * lv)) & 7;
        if (e & 1)
            split4_child_inplace(t, (int)(e >> 1));
        else
            split4_child_inplace(s, (int)(e >> 1));
    }
}

struct NearNode {
    int pair;       // index into the near-pair list
    unsigned code;  // path code
};

// classify every node of level `depth`: leaves go to `leaves`, split nodes append 4 children to `next`
// The node count comes from the device (the previous level's append counter), so all six
// levels are enqueued back to back with a fixed grid-stride launch and no host round trip;
// an append past a buffer's capacity raises *overflow (the host regrows and reruns) and the
// level's true population is recorded in level_pop[depth] for the regrowth.
__global__ void k_near_level(const NearNode* __restrict__ nodes, const unsigned long long* __restrict__ nnodes_dev,
                             long long cap_nodes, int depth, const int2* __restrict__ pairs,
                             const double* __restrict__ GV, double thr, NearNode* __restrict__ leaves,
                             unsigned long long* __restrict__ nleaves, long long cap_leaves,
                             NearNode* __restrict__ next, unsigned long long* __restrict__ nnext, long long cap_next,
                             unsigned long long* __restrict__ overflow, unsigned long long* __restrict__ level_pop)
{
    const long long nn_all = (long long)*nnodes_dev;
    const long long nn = min(nn_all, cap_nodes);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        level_pop[depth] = (unsigned long long)nn_all;
        if (nn_all > cap_nodes) atomicOr(overflow, 1ull);
    }
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < nn; k += (long long)gridDim.x * blockDim.x) {
        const NearNode nd = nodes[k];
        bool leaf = depth >= 5;
        int split_t = 0;
        if (!leaf) {
            double t[9], s[9];
            node_triangles(GV, pairs[nd.pair], nd.code, t, s);
            const double dt = tri_diam(t), ds = tri_diam(s);
            D3 ct, cs;
            double rt, rs;
            tri_centroid_rad(t, ct, rt);
            tri_centroid_rad(s, cs, rs);
            const double dist = fmax(0.0, __dsub_rn(__dsub_rn(d3_norm(d3_sub(ct, cs)), rt), rs));
            leaf = dist >= __dmul_rn(thr, fmax(dt, ds));
            split_t = dt >= ds ? 1 : 0;
        }
        if (leaf) {
            const unsigned long long ql = atomicAdd(nleaves, 1ull);
            if ((long long)ql < cap_leaves)
                leaves[ql] = nd;
            else
                atomicOr(overflow, 1ull);
        } else {
            const unsigned long long qn = atomicAdd(nnext, 4ull);
            const unsigned base = (nd.code & ~7u) | (unsigned)(depth + 1);
            if ((long long)qn + 4 > cap_next) atomicOr(overflow, 1ull);
            for (int c = 0; c < 4; ++c)
                if ((long long)qn + c < cap_next)
                    next[qn + c] = {nd.pair, base | ((unsigned)(split_t | (c << 1)) << (3 + 3 * depth))};
        }
    }
}

// leaf vertices from the root triangle and the composed barycentric map of a path
template <bool GLOBAL_TAB = false>
__device__ __forceinline__ void path_triangle(const double* __restrict__ root, int path, double* out)
{
    const unsigned char* B = (GLOBAL_TAB ? g_paths : c_paths) + 9 * path;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        const double w0 = (GLOBAL_TAB ? __ldg(B + 3 * r) : B[3 * r]) * (1.0 / 32),
                     w1 = (GLOBAL_TAB ? __ldg(B + 3 * r + 1) : B[3 * r + 1]) * (1.0 / 32),
                     w2 = (GLOBAL_TAB ? __ldg(B + 3 * r + 2) : B[3 * r + 2]) * (1.0 / 32);
#pragma unroll
        for (int c = 0; c < 3; ++c) out[3 * r + c] = fma(w2, root[6 + c], fma(w1, root[3 + c], w0 * root[c]));
    }
}

// Leaves: eight per warp, four lanes per leaf.  Leaf triangles come from the
// composed split4 maps (exact dyadic weights; the classification pass already
// reproduced the reference's recursion bit for bit), and their areas are the
// root areas / 4^depth.  Distances use the expansion |x-y|^2 = |x|^2 + |y|^2 -
// 2 x.y in leaf-local coordinates (origin t0).  The leaf's 36 y points (y,
// |y|^2) are staged in shared memory; lane xg of the leaf owns the x points
// x groups of four points (three passes, below) held in registers as (-2x,
// |x|^2), with one accumulator per x point: an evaluation is 3 FMA + 1 ADD for
// r^2, MUFU.RSQ64H + 4 FP64 for the refined 1/r and 1 FMA, and the four
// evaluations per loaded y point are independent chains (tools/micro_eval.cu:
// this 4-point block is the fastest register blocking of the pattern).
// coordinate a of vertex k (0-2) of a triangle held in registers, for a runtime axis a
__device__ __forceinline__ double vcoord(const double* v, int k, int a)
{
    return a == 0 ? v[3 * k] : (a == 1 ? v[3 * k + 1] : v[3 * k + 2]);
}
// the axis in which every vertex of both triangles has one and the same coordinate (z first),
// or -1; the axis order puts it last (identity when there is none)
__device__ __forceinline__ int3 flat_axes(const double* t, const double* s, bool& flat)
{
    int fa = -1;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double c = t[a];
        if (t[3 + a] == c && t[6 + a] == c && s[a] == c && s[3 + a] == c && s[6 + a] == c) fa = a;
    }
    flat = fa >= 0;
    return fa == 1 ? make_int3(0, 2, 1) : (fa == 0 ? make_int3(1, 2, 0) : make_int3(0, 1, 2));
}

constexpr int NEAR_LEAF_THREADS = 256;
#ifndef NEAR_LEAF_CTAS
#define NEAR_LEAF_CTAS 2  // resident CTAs per SM (launch bounds and the persistent grid)
#endif
#ifndef NEAR_FLAT_UNROLL
#define NEAR_FLAT_UNROLL 36
#endif
constexpr int kNearFlatUnroll = NEAR_FLAT_UNROLL;  // the flat leaf loop's unroll (A/B builds)
#ifndef NEAR_GEN_UNROLL
#define NEAR_GEN_UNROLL 3
#endif
constexpr int kNearGenUnroll = NEAR_GEN_UNROLL;  // the 3-D leaf loop's unroll
constexpr int NEAR_XP = 4;  // x points per pass (register block)
#ifndef NEAR_LEAF_XP
#define NEAR_LEAF_XP 3
#endif
// the default-rule leaf kernel: 4 x points per pass (groups xg, xg + 4, then group 8 split by
// y over the 4 lanes) or 3 (groups xg, xg + 4, xg + 8: three uniform passes of 36 y points)
constexpr int NLX = NEAR_LEAF_XP;
static_assert(NLX == 3 || NLX == 4, "near-leaf x block: 3 or 4 points");
constexpr int NEAR_LEAF_WARPS = NEAR_LEAF_THREADS / 32;
// one leaf's staged y points: npts double4 plus 16 bytes, so the eight leaves of a warp,
// read together by one LDS.128, start in eight different 16-byte bank groups (a plain
// 36 x 32-byte stride is a multiple of 128 bytes: an 8-way bank conflict on every load)
__host__ __device__ constexpr size_t leaf_stage_bytes(int npts) { return (size_t)npts * sizeof(double4) + 16; }
constexpr size_t NEAR_LEAF_SMEM = (size_t)NEAR_LEAF_WARPS * 8 * leaf_stage_bytes(NN);
__global__ void __launch_bounds__(NEAR_LEAF_THREADS, NEAR_LEAF_CTAS) k_near_leaves(const NearNode* __restrict__ leaves,
                                                                       const unsigned long long* __restrict__ nleaves_dev,
                                                                       long long cap, const int2* __restrict__ pairs,
                                                                       const double* __restrict__ GV,
                                                                       const double* __restrict__ GA, double inv_pi,
                                                                       double* __restrict__ out)
{
    extern __shared__ __align__(16) unsigned char near_smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int h = lane >> 2, xg = lane & 3;
    double4* Ys = reinterpret_cast<double4*>(near_smem + ((size_t)wib * 8 + h) * leaf_stage_bytes(NN));
    const long long nl = min((long long)*nleaves_dev, cap);
    const long long warps = (long long)gridDim.x * NEAR_LEAF_WARPS;
    for (long long w = (long long)blockIdx.x * NEAR_LEAF_WARPS + wib; 8 * w < nl; w += warps) {
        const long long q = 8 * w + h;
        const bool active = q < nl;
        double acc = 0.0, scale = 0.0;
        double f1x = 0, f1y = 0, f1z = 0, f2x = 0, f2y = 0, f2z = 0;
        int pair = 0;
        bool flat = false;
        __syncwarp();  // the previous iteration's reads of Ys are done
        if (active) {
            const NearNode nd = leaves[q];
            pair = nd.pair;
            const int2 pr = pairs[nd.pair];
            const int depth = nd.code & 7;
            int it = 0, is = 0, dt = 0, ds = 0;
            for (int lv = 0; lv < depth; ++lv) {
                const unsigned e = (nd.code >> (3 + 3 * lv)) & 7;
                if (e & 1) {
                    it = 4 * it + (int)(e >> 1);
                    ++dt;
                } else {
                    is = 4 * is + (int)(e >> 1);
                    ++ds;
                }
            }
            double t[9], s[9];
            path_triangle<NEAR_GLOBAL_TABLES>(GV + 9 * pr.x, ((1 << 2 * dt) - 1) / 3 + it, t);
            path_triangle<NEAR_GLOBAL_TABLES>(GV + 9 * pr.y, ((1 << 2 * ds) - 1) / 3 + is, s);
            scale = __ldg(GA + pr.x) * __ldg(GA + pr.y) * ldexp(inv_pi, -2 * (dt + ds));
            // a leaf pair in one coordinate plane: that axis goes last, all its leaf-local
            // coordinates are exact zeros and the evaluation leaves its term out (far_pass_sum)
            const int3 P = flat_axes(t, s, flat);
            const double e1x = vcoord(s, 1, P.x) - vcoord(s, 0, P.x), e1y = vcoord(s, 1, P.y) - vcoord(s, 0, P.y),
                         e1z = vcoord(s, 1, P.z) - vcoord(s, 0, P.z);
            const double e2x = vcoord(s, 2, P.x) - vcoord(s, 0, P.x), e2y = vcoord(s, 2, P.y) - vcoord(s, 0, P.y),
                         e2z = vcoord(s, 2, P.z) - vcoord(s, 0, P.z);
            const double bx = vcoord(s, 0, P.x) - vcoord(t, 0, P.x), by = vcoord(s, 0, P.y) - vcoord(t, 0, P.y),
                         bz = vcoord(s, 0, P.z) - vcoord(t, 0, P.z);
            if (flat) {  // the same values with the zero coordinate left out
                for (int j = xg; j < NN; j += 4) {
                    const double yx = fma(NEAR_TAB(near_v, j), e2x, fma(NEAR_TAB(near_u, j), e1x, bx));
                    const double yy = fma(NEAR_TAB(near_v, j), e2y, fma(NEAR_TAB(near_u, j), e1y, by));
                    const double sj = NEAR_TAB(near_s, j);
                    Ys[j] = sj == 0.0 ? make_double4(0.0, 0.0, 0.0, kPadR2)
                                      : make_double4(sj * yx, sj * yy, 0.0, sj * fma(yx, yx, yy * yy));
                }
            } else {
                for (int j = xg; j < NN; j += 4) {
                    const double yx = fma(NEAR_TAB(near_v, j), e2x, fma(NEAR_TAB(near_u, j), e1x, bx));
                    const double yy = fma(NEAR_TAB(near_v, j), e2y, fma(NEAR_TAB(near_u, j), e1y, by));
                    const double yz = fma(NEAR_TAB(near_v, j), e2z, fma(NEAR_TAB(near_u, j), e1z, bz));
                    Ys[j] = scaled_ypoint(yx, yy, yz, NEAR_TAB(near_s, j));
                }
            }
            f1x = vcoord(t, 1, P.x) - vcoord(t, 0, P.x), f1y = vcoord(t, 1, P.y) - vcoord(t, 0, P.y),
            f1z = vcoord(t, 1, P.z) - vcoord(t, 0, P.z);
            f2x = vcoord(t, 2, P.x) - vcoord(t, 0, P.x), f2y = vcoord(t, 2, P.y) - vcoord(t, 0, P.y),
            f2z = vcoord(t, 2, P.z) - vcoord(t, 0, P.z);
        }
        __syncwarp();
        flat = __all_sync(0xffffffffu, flat || !active);
        if (active) {
            // x groups of 4 consecutive points: lane xg takes groups xg and xg + 4 against all
            // 36 y points, and group 8 against y in [9 xg, 9 xg + 9)
#pragma unroll 1
            for (int pass = 0; pass < 3; ++pass) {
                const int g = (NLX == 3 || pass < 2) ? xg + 4 * pass : 8;
                const int j0 = (NLX == 3 || pass < 2) ? 0 : 9 * xg, j1 = (NLX == 3 || pass < 2) ? NN : 9 * xg + 9;
                double mx[NLX], my[NLX], mz[NLX], x2[NLX], a[NLX];
#pragma unroll
                for (int r = 0; r < NLX; ++r) {
                    const int i = NLX * g + r;
                    const double xx = fma(NEAR_TAB(near_v, i), f2x, NEAR_TAB(near_u, i) * f1x);
                    const double xy = fma(NEAR_TAB(near_v, i), f2y, NEAR_TAB(near_u, i) * f1y);
                    if (flat) {
                        x2[r] = fma(xx, xx, xy * xy);
                        mz[r] = 0.0;
                    } else {
                        const double xz = fma(NEAR_TAB(near_v, i), f2z, NEAR_TAB(near_u, i) * f1z);
                        x2[r] = fma(xx, xx, fma(xy, xy, xz * xz));
                        mz[r] = -2.0 * xz;
                    }
                    mx[r] = -2.0 * xx;
                    my[r] = -2.0 * xy;
                    a[r] = 0.0;
                }
                if (flat) {
#pragma unroll kNearFlatUnroll
                    for (int j = j0; j < j1; ++j) {
                        const double4 y = Ys[j];
                        const double sj = c_near_s[j];
#pragma unroll
                        for (int r = 0; r < NLX; ++r) {
                            const double r2 = fma(mx[r], y.x, fma(my[r], y.y, fma(x2[r], sj, y.w)));
                            a[r] = rsqrt_acc_s(r2, a[r]);
                        }
                    }
                } else {
#pragma unroll kNearGenUnroll
                    for (int j = j0; j < j1; ++j) {
                        const double4 y = Ys[j];
                        const double sj = c_near_s[j];
#pragma unroll
                        for (int r = 0; r < NLX; ++r) {
                            const double r2 = fma(mx[r], y.x, fma(my[r], y.y, fma(mz[r], y.z, fma(x2[r], sj, y.w))));
                            a[r] = rsqrt_acc_s(r2, a[r]);
                        }
                    }
                }
#pragma unroll
                for (int r = 0; r < NLX; ++r) acc = fma(NEAR_TAB(near_w, NLX * g + r), a[r], acc);
            }
        }
        for (int o = 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (active && xg == 0) atomicAdd(out + pair, acc * (scale * kRsqrtAccScale));
    }
}

// Near leaves for a non-default far_order: the same layout as k_near_leaves with the
// near rule padded to NNP (a multiple of 16) by zero-weight points, so lane xg takes
// the x groups xg, xg + 4, ... against all NNP y points; 4 warps per CTA keep the
// staged y points within shared memory for the larger rules.
constexpr int NEAR_G_THREADS = 128;
template <int NNP>
__global__ void __launch_bounds__(NEAR_G_THREADS) k_near_leaves_g(const NearNode* __restrict__ leaves,
                                                                  const unsigned long long* __restrict__ nleaves_dev,
                                                                  long long cap, const int2* __restrict__ pairs,
                                                                  const double* __restrict__ GV,
                                                                  const double* __restrict__ GA, double inv_pi,
                                                                  double* __restrict__ out)
{
    extern __shared__ __align__(16) unsigned char near_g_smem[];
    constexpr int WARPS = NEAR_G_THREADS / 32;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int h = lane >> 2, xg = lane & 3;
    double4* Ys = reinterpret_cast<double4*>(near_g_smem + ((size_t)wib * 8 + h) * leaf_stage_bytes(NNP));
    const long long nl = min((long long)*nleaves_dev, cap);
    const long long warps = (long long)gridDim.x * WARPS;
    for (long long w = (long long)blockIdx.x * WARPS + wib; 8 * w < nl; w += warps) {
        const long long q = 8 * w + h;
        const bool active = q < nl;
        double acc = 0.0, scale = 0.0;
        double f1x = 0, f1y = 0, f1z = 0, f2x = 0, f2y = 0, f2z = 0;
        int pair = 0;
        __syncwarp();
        if (active) {
            const NearNode nd = leaves[q];
            pair = nd.pair;
            const int2 pr = pairs[nd.pair];
            const int depth = nd.code & 7;
            int it = 0, is = 0, dt = 0, ds = 0;
            for (int lv = 0; lv < depth; ++lv) {
                const unsigned e = (nd.code >> (3 + 3 * lv)) & 7;
                if (e & 1) {
                    it = 4 * it + (int)(e >> 1);
                    ++dt;
                } else {
                    is = 4 * is + (int)(e >> 1);
                    ++ds;
                }
            }
            double t[9], s[9];
            path_triangle(GV + 9 * pr.x, ((1 << 2 * dt) - 1) / 3 + it, t);
            path_triangle(GV + 9 * pr.y, ((1 << 2 * ds) - 1) / 3 + is, s);
            scale = __ldg(GA + pr.x) * __ldg(GA + pr.y) * ldexp(inv_pi, -2 * (dt + ds));
            const double e1x = s[3] - s[0], e1y = s[4] - s[1], e1z = s[5] - s[2];
            const double e2x = s[6] - s[0], e2y = s[7] - s[1], e2z = s[8] - s[2];
            const double bx = s[0] - t[0], by = s[1] - t[1], bz = s[2] - t[2];
            for (int j = xg; j < NNP; j += 4) {
                const double yx = fma(c_near_v[j], e2x, fma(c_near_u[j], e1x, bx));
                const double yy = fma(c_near_v[j], e2y, fma(c_near_u[j], e1y, by));
                const double yz = fma(c_near_v[j], e2z, fma(c_near_u[j], e1z, bz));
                Ys[j] = scaled_ypoint(yx, yy, yz, c_near_s[j]);
            }
            f1x = t[3] - t[0], f1y = t[4] - t[1], f1z = t[5] - t[2];
            f2x = t[6] - t[0], f2y = t[7] - t[1], f2z = t[8] - t[2];
        }
        __syncwarp();
        if (active) {
#pragma unroll 1
            for (int g = xg; g < NNP / NEAR_XP; g += 4) {
                double mx[NEAR_XP], my[NEAR_XP], mz[NEAR_XP], x2[NEAR_XP], a[NEAR_XP];
#pragma unroll
                for (int r = 0; r < NEAR_XP; ++r) {
                    const int i = NEAR_XP * g + r;
                    const double xx = fma(c_near_v[i], f2x, c_near_u[i] * f1x);
                    const double xy = fma(c_near_v[i], f2y, c_near_u[i] * f1y);
                    const double xz = fma(c_near_v[i], f2z, c_near_u[i] * f1z);
                    x2[r] = fma(xx, xx, fma(xy, xy, xz * xz));
                    mx[r] = -2.0 * xx;
                    my[r] = -2.0 * xy;
                    mz[r] = -2.0 * xz;
                    a[r] = 0.0;
                }
#pragma unroll 2
                for (int j = 0; j < NNP; ++j) {
                    const double4 y = Ys[j];
                    const double sj = c_near_s[j];
#pragma unroll
                    for (int r = 0; r < NEAR_XP; ++r) {
                        const double r2 = fma(mx[r], y.x, fma(my[r], y.y, fma(mz[r], y.z, fma(x2[r], sj, y.w))));
                        a[r] = rsqrt_acc_s(r2, a[r]);
                    }
                }
#pragma unroll
                for (int r = 0; r < NEAR_XP; ++r) acc = fma(c_near_w[NEAR_XP * g + r], a[r], acc);
            }
        }
        for (int o = 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (active && xg == 0) atomicAdd(out + pair, acc * (scale * kRsqrtAccScale));
    }
}

template <int NNP>
void launch_near_leaves_g(Ctx* ctx, const NearNode* leaves, const unsigned long long* cnt, long long ncur,
                          const int2* pairs, const double* GV, const double* GA, double* out)
{
    const size_t smem = (size_t)(NEAR_G_THREADS / 32) * 8 * leaf_stage_bytes(NNP);
    set_max_dynamic_smem(k_near_leaves_g<NNP>, smem);
    const long long warps = (ncur + 7) / 8;
    const int grid = (int)std::min<long long>((warps + NEAR_G_THREADS / 32 - 1) / (NEAR_G_THREADS / 32),
                                              4LL * ctx->sm_count);
    k_near_leaves_g<NNP><<<grid, NEAR_G_THREADS, smem, ctx->stream>>>(leaves, cnt, ncur, pairs, GV, GA, 1.0 / M_PI, out);
}

// ---------------------------------------------------------------- Sauter (singular) pairs
// pairs: 6 ints per pair = permuted vertex ids of t then s (quadrature.hpp:297-322).
// The permutation puts the shared vertices first, so t0 = s0 in every class (d0 = 0).
// Identical (s = t): x - y = c1 e1 + c2 e2 with c = (a1-b1, a2-b2), so |x - y|^2 is the
// quadratic form of the triangle's Gram matrix: 3 FMA per point from the rule table's
// monomials (c1^2, 2 c1 c2, c2^2).  Edge (t1 = s1 too): x - y = c1 e1 + a2 e2t - b2 e2s,
// a 3x3 Gram form, 6 FMA from (c1^2, a2^2, b2^2, 2 c1 a2, -2 c1 b2, -2 a2 b2).  The Gram
// forms are positive definite on the rule's domain (the two triangles lie on either side
// of the shared edge); their rounding grows with the triangles' aspect, ~1e-15 relative on
// the configs.  Vertex: x - y = a1 e1t + a2 e2t - b1 e1s - b2 e2s by 4 FMA per coordinate
// (four vectors in 3-D: the Gram form would be singular).  Rule tables (upload_sauter):
// SAUTER_STRIDE doubles per point, the weight last.
template <int CLS>
struct SauterStride {
    static constexpr int value = CLS == 3 ? 4 : (CLS == 2 ? 8 : 5);  // 4, 8: 32-byte rows (LDS.128)
};

// FLAT (vertex class): the four edge vectors have a zero last component (the pair lies in a
// coordinate plane, axes ordered so that one is last): dz = 0 is left out, 10 FMA per point
template <int CLS, bool FLAT = false>
__device__ __forceinline__ double sauter_r2(const double* a, const double (&g)[12])
{
    if (CLS == 3) return fma(a[0], g[0], fma(a[1], g[1], a[2] * g[2]));
    if (CLS == 2)
        return fma(a[0], g[0], fma(a[1], g[1], fma(a[2], g[2], fma(a[3], g[3], fma(a[4], g[4], a[5] * g[5])))));
    const double dx = fma(-a[3], g[9], fma(-a[2], g[6], fma(a[1], g[3], a[0] * g[0])));
    const double dy = fma(-a[3], g[10], fma(-a[2], g[7], fma(a[1], g[4], a[0] * g[1])));
    if (FLAT) return fma(dx, dx, dy * dy);
    const double dz = fma(-a[3], g[11], fma(-a[2], g[8], fma(a[1], g[5], a[0] * g[2])));
    return fma(dx, dx, fma(dy, dy, dz * dz));
}

#ifndef SAUTER_UNROLL
#define SAUTER_UNROLL 2
#endif
constexpr int kSauterUnroll = SAUTER_UNROLL;  // 4-point steps per unrolled iteration (A/B builds)
// one stage of rule points, four independent evaluations per step
template <int CLS, bool FLAT, int ST>
__device__ __forceinline__ void sauter_stage(const double* __restrict__ R, int cnt, const double (&g)[12],
                                             double& acc0, double& acc1, double& acc2, double& acc3)
{
    int i = 0;
#pragma unroll kSauterUnroll
    for (; i + 4 <= cnt; i += 4) {
        double r2[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) r2[u] = sauter_r2<CLS, FLAT>(R + ST * (i + u), g);
        // the table's coefficients carry 1 / w^2 in r^2: rsqrt of it is w / r (rsqrt_acc)
        acc0 = rsqrt_acc_s(r2[0], acc0);
        acc1 = rsqrt_acc_s(r2[1], acc1);
        acc2 = rsqrt_acc_s(r2[2], acc2);
        acc3 = rsqrt_acc_s(r2[3], acc3);
    }
    for (; i < cnt; ++i) acc0 = rsqrt_acc_s(sauter_r2<CLS, FLAT>(R + ST * i, g), acc0);
}

template <int CLS>
__global__ void __launch_bounds__(SAUTER_THREADS)
    k_sauter_partial(const int* __restrict__ pv, int npairs, const double* __restrict__ X,
                     const double* __restrict__ rule, int npts, int chunk, double* __restrict__ part)
{
    constexpr int ST = SauterStride<CLS>::value;
    constexpr int STAGE = SAUTER_STAGE * 5 / ST;  // points per shared-memory pass
    __shared__ __align__(16) double R[SAUTER_STAGE * 5];
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    const bool active = p < npairs;
    double g[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};  // vertex: e1t, e2t, e1s, e2s; else Gram entries
    bool flat = false;
    if (active) {
        const int* q = pv + 6 * p;
        const double* t0 = X + 3 * q[0];
        const double* t1 = X + 3 * q[1];
        const double* t2 = X + 3 * q[2];
        const double* s0 = X + 3 * q[3];
        const double* s1 = X + 3 * q[4];
        const double* s2 = X + 3 * q[5];
        double e[12];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            e[c] = t1[c] - t0[c];
            e[3 + c] = t2[c] - t0[c];
            e[6 + c] = s1[c] - s0[c];
            e[9 + c] = s2[c] - s0[c];
        }
        auto dot = [&](int u, int v) { return fma(e[u], e[v], fma(e[u + 1], e[v + 1], e[u + 2] * e[v + 2])); };
        if (CLS == 3) {
            g[0] = dot(0, 0);
            g[1] = dot(0, 3);
            g[2] = dot(3, 3);
        } else if (CLS == 2) {
            g[0] = dot(0, 0);
            g[1] = dot(3, 3);
            g[2] = dot(9, 9);
            g[3] = dot(0, 3);
            g[4] = dot(0, 9);
            g[5] = dot(3, 9);
        } else {
            // a pair in a coordinate plane: that axis last, its components all exact zeros
            int fa = -1;
#pragma unroll
            for (int c = 0; c < 3; ++c)
                if (e[c] == 0.0 && e[3 + c] == 0.0 && e[6 + c] == 0.0 && e[9 + c] == 0.0) fa = c;
            flat = fa >= 0;
            const int px = fa == 0 ? 1 : 0, py = fa == 2 || fa < 0 ? 1 : 2, pz = fa < 0 ? 2 : fa;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const double v[3] = {e[3 * k], e[3 * k + 1], e[3 * k + 2]};
                g[3 * k] = px == 0 ? v[0] : v[1];
                g[3 * k + 1] = py == 1 ? v[1] : v[2];
                g[3 * k + 2] = pz == 0 ? v[0] : (pz == 1 ? v[1] : v[2]);
            }
        }
    }
    if (CLS == 1) flat = __syncthreads_and(flat || !active);  // CTA-uniform loop form
    const int q0 = blockIdx.y * chunk, q1 = min(npts, q0 + chunk);
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
    for (int base = q0; base < q1; base += STAGE) {
        const int cnt = min(STAGE, q1 - base);
        __syncthreads();
        for (int k = threadIdx.x; k < cnt * ST; k += blockDim.x) R[k] = rule[(size_t)base * ST + k];
        __syncthreads();
        if (active) {
            if (CLS == 1 && flat)
                sauter_stage<CLS, true, ST>(R, cnt, g, acc0, acc1, acc2, acc3);
            else
                sauter_stage<CLS, false, ST>(R, cnt, g, acc0, acc1, acc2, acc3);
        }
    }
    // (rsqrt_acc_s accumulates with the factor 8/3)
    if (active) part[(size_t)blockIdx.y * npairs + p] = ((acc0 + acc1) + (acc2 + acc3)) * kRsqrtAccScale;
}

// launch of one class: chunk count chosen (sauter_chunking) so the grid fills whole waves
void launch_sauter_partial(Ctx* ctx, int cls, const int* pv, int np, const double* X, const double* rule, int npts,
                           int chunk, int nchunks, double* part)
{
    const dim3 grid((np + SAUTER_THREADS - 1) / SAUTER_THREADS, nchunks);
    cudaStream_t s = ctx->stream;
    switch (cls) {
    case 1: k_sauter_partial<1><<<grid, SAUTER_THREADS, 0, s>>>(pv, np, X, rule, npts, chunk, part); break;
    case 2: k_sauter_partial<2><<<grid, SAUTER_THREADS, 0, s>>>(pv, np, X, rule, npts, chunk, part); break;
    case 3: k_sauter_partial<3><<<grid, SAUTER_THREADS, 0, s>>>(pv, np, X, rule, npts, chunk, part); break;
    default: throw std::logic_error("Sauter class out of range");
    }
    count_launch();
}

// (chunk, nchunks) for np pairs of a class: chunks of >= ~600 rule points, and among
// those the count whose grid (pair blocks x chunks) best fills whole waves of resident CTAs
void sauter_chunking(Ctx* ctx, int cls, int np, int npts, int& chunk, int& nchunks)
{
    int per_sm = 1;
    const void* fn = cls == 1 ? (const void*)k_sauter_partial<1>
                              : (cls == 2 ? (const void*)k_sauter_partial<2> : (const void*)k_sauter_partial<3>);
    SBG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, SAUTER_THREADS, 0));
    const long long slots = (long long)std::max(per_sm, 1) * ctx->sm_count;
    const long long pblocks = (np + SAUTER_THREADS - 1) / SAUTER_THREADS;
    const int cmax = std::max(1, npts / 600);
    double best = -1.0;
    int best_c = 1;
    for (int c = 1; c <= cmax; ++c) {
        const int ch = (npts + c - 1) / c, cc = (npts + ch - 1) / ch;
        const double waves = (double)(pblocks * cc) / (double)slots;
        const double eff = waves / std::ceil(waves);  // busy fraction of the launched waves
        // prefer fuller waves; among equally full, more waves (smaller tail per wave)
        const double score = eff + 1e-3 * std::min(waves, 8.0);
        if (score > best + 1e-12) {
            best = score;
            best_c = cc;
        }
    }
    chunk = (npts + best_c - 1) / best_c;
    nchunks = (npts + chunk - 1) / chunk;
}

// I = (sum of chunk partials) * 4 A_t A_s / (4 pi)   (quadrature.hpp:254-261)
__global__ void k_sauter_finish(const double* __restrict__ part, int npairs, int nchunks, const int* __restrict__ pv,
                                const double* __restrict__ X, double* __restrict__ out)
{
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= npairs) return;
    double acc = 0.0;
    for (int c = 0; c < nchunks; ++c) acc += part[(size_t)c * npairs + p];
    double t[9], s[9];
    for (int k = 0; k < 3; ++k)
        for (int c = 0; c < 3; ++c) {
            t[3 * k + c] = X[3 * pv[6 * p + k] + c];
            s[3 * k + c] = X[3 * pv[6 * p + 3 + k] + c];
        }
    const double scale = 4.0 * tri_area(t) * tri_area(s);
    out[p] = acc * scale / (4.0 * M_PI);
}

// ---------------------------------------------------------------- per-pair scatter (near + singular)
// pairs [0, nsing) are the singular pairs, then min(*nnear, near_cap) near pairs (device count)
// band (optional): max |da - db| over the entries written, for the host copy's band patch
// offs: marks |i - j| (<= kOffsMax) of every entry written (the host copy's diagonal patch)
constexpr int kOffsMax = 4095;
// pairs [lo, nsing + near count) — or [lo, nsing) when nnear is null (the singular pairs alone)
__global__ void k_local_scatter(const int2* __restrict__ pairs, const double* __restrict__ I, long long nsing,
                                const unsigned long long* __restrict__ nnear, long long near_cap,
                                const int* __restrict__ uptr, const int* __restrict__ udof,
                                const double* __restrict__ uval, double* __restrict__ W, int ld, int* __restrict__ band,
                                long long lo = 0, int* __restrict__ offs = nullptr)
{
    const long long k = lo + (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nsing + (nnear ? min((long long)*nnear, near_cap) : 0LL)) return;
    const int f = pairs[k].x, g = pairs[k].y;
    const double val = I[k];
    for (int p = uptr[f]; p < uptr[f + 1]; ++p) {
        const int da = udof[p];
        const double ax = uval[3 * p], ay = uval[3 * p + 1], az = uval[3 * p + 2];
        for (int q = uptr[g]; q < uptr[g + 1]; ++q) {
            const int db = udof[q];
            const double v = val * fma(ax, uval[3 * q], fma(ay, uval[3 * q + 1], az * uval[3 * q + 2]));
            if (band) atomicMax(band, abs(da - db));
            if (offs && abs(da - db) <= kOffsMax) offs[abs(da - db)] = 1;  // the entry's diagonal
            if (f == g) {
                if (da <= db) atomicAdd(W + (size_t)da * ld + db, v);
            } else if (da < db) {
                atomicAdd(W + (size_t)da * ld + db, v);
            } else if (da > db) {
                atomicAdd(W + (size_t)db * ld + da, v);
            } else {
                atomicAdd(W + (size_t)da * ld + da, 2.0 * v);
            }
        }
    }
}

// W(j,i) = W(i,j), j > i  (assemble.hpp:136-137), 32x32 tiles through smem
// also flags a non-finite entry of the upper triangle, where every pair integral lands
// (the reference throws NumericalError on a non-finite pair integral, assemble.hpp:106-107)
__global__ void k_mirror(double* __restrict__ W, int n, int ld, int* __restrict__ bad)
{
    __shared__ double tile[32][33];
    const int bi = blockIdx.y, bj = blockIdx.x;  // source tile (bi, bj), bi <= bj
    if (bi > bj) return;
    const int tx = threadIdx.x, ty = threadIdx.y;
    bool finite = true;
    for (int r = ty; r < 32; r += blockDim.y) {
        const int i = bi * 32 + r, j = bj * 32 + tx;
        const double v = (i < n && j < n) ? W[(size_t)i * ld + j] : 0.0;
        finite &= isfinite(v);
        tile[r][tx] = v;
    }
    if (__any_sync(0xffffffffu, !finite) && tx == 0) *bad = 1;
    __syncthreads();
    for (int r = ty; r < 32; r += blockDim.y) {
        const int i = bj * 32 + r, j = bi * 32 + tx;  // destination (lower) element (i, j) = source (j, i)
        if (i < n && j < n && i > j) W[(size_t)i * ld + j] = tile[tx][r];
    }
}

// entries W(i, i + d_k) of the listed diagonals (d_k may be negative), row-major by i
__global__ void k_pack_diagonals(const double* __restrict__ W, int n, int ld, const int* __restrict__ d, int nd,
                                 double* __restrict__ out)
{
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)n * nd) return;
    const int i = (int)(e / nd), j = i + d[e % nd];
    out[e] = (j >= 0 && j < n) ? W[(size_t)i * ld + j] : 0.0;
}

// the mirror restricted to the tiles that meet the band |i - j| <= *K (K measured on the
// device by the scatter): after a scatter only those entries changed
__global__ void k_mirror_band(double* __restrict__ W, int n, int ld, const int* __restrict__ Kdev, int* __restrict__ bad)
{
    __shared__ double tile[32][33];
    const int bi = blockIdx.y, bj = blockIdx.x;
    if (bi > bj || (bj - bi - 1) * 32 > *Kdev) return;  // every |i - j| in the tile exceeds K
    const int tx = threadIdx.x, ty = threadIdx.y;
    bool finite = true;
    for (int r = ty; r < 32; r += blockDim.y) {
        const int i = bi * 32 + r, j = bj * 32 + tx;
        const double v = (i < n && j < n) ? W[(size_t)i * ld + j] : 0.0;
        finite &= isfinite(v);
        tile[r][tx] = v;
    }
    if (__any_sync(0xffffffffu, !finite) && tx == 0) *bad = 1;
    __syncthreads();
    for (int r = ty; r < 32; r += blockDim.y) {
        const int i = bj * 32 + r, j = bi * 32 + tx;
        if (i < n && j < n && i > j) W[(size_t)i * ld + j] = tile[tx][r];
    }
}

// ---------------------------------------------------------------- RHS (assemble.hpp:143-184)
__global__ void k_rhs(int nf, int nr, const double* __restrict__ GV, const double* __restrict__ onormal,
                      const double* __restrict__ g, int g_is_field, const int* __restrict__ sptr,
                      const int* __restrict__ sdof, const double* __restrict__ ssgn, double* __restrict__ L)
{
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nf * nr) return;
    const int f = e / nr, i = e % nr;
    const double* t = GV + 9 * f;
    const double meas = tri_area(t);
    const double u = c_far_u[i], v = c_far_v[i], w = c_far_w[i] * 2.0 * meas;
    const double* gy = g_is_field ? g + 3 * (size_t)e : g;
    for (int s = 0; s < 2; ++s) {
        const int o = 2 * f + s;
        const double dn = (gy[0] * onormal[3 * o] + gy[1] * onormal[3 * o + 1]) + gy[2] * onormal[3 * o + 2];
        for (int k = 0; k < 3; ++k) {
            const double lambda = (k == 0) ? (1.0 - u - v) : ((k == 1) ? u : v);
            const int slot = 3 * o + k;
            for (int q = sptr[slot]; q < sptr[slot + 1]; ++q) atomicAdd(L + sdof[q], w * dn * lambda * ssgn[q]);
        }
    }
}

// ---------------------------------------------------------------- host helpers
std::uint64_t spread3(std::uint64_t x)
{
    x &= 0x1fffff;
    x = (x | x << 32) & 0x1f00000000ffffULL;
    x = (x | x << 16) & 0x1f0000ff0000ffULL;
    x = (x | x << 8) & 0x100f00f00f00f00fULL;
    x = (x | x << 4) & 0x10c30c30c30c30c3ULL;
    x = (x | x << 2) & 0x1249249249249249ULL;
    return x;
}

RuleDims upload_rules(Ctx* ctx, const QuadCfg& cfg)
{
    const RuleDims R = rule_dims(cfg.far_order);
    // the rules of quadrature.hpp:105-112, padded with zero-weight centroid points
    static std::mutex mu;
    static std::map<int, std::shared_ptr<const std::vector<double>>> cache;  // far_order -> u,v,w far | u,v,w near
    std::shared_ptr<const std::vector<double>> rules;
    {
        std::lock_guard<std::mutex> lock(mu);
        auto& slot = cache[R.far_order];
        if (!slot) {
            auto buf = std::make_shared<std::vector<double>>(4 * NF_MAX + 4 * NN_MAX, 0.0);
            const TriangleRule far = triangle_rule(R.far_order), nr = triangle_rule(R.far_order + 2);
            for (int i = 0; i < NF_MAX; ++i) {
                const bool real = i < R.nf;
                (*buf)[i] = real ? far.u[i] : 1.0 / 3.0;
                (*buf)[NF_MAX + i] = real ? far.v[i] : 1.0 / 3.0;
                (*buf)[2 * NF_MAX + i] = real ? far.w[i] : 0.0;
            }
            double* nb = buf->data() + 3 * NF_MAX;
            for (int i = 0; i < NN_MAX; ++i) {
                const bool real = i < R.nn;
                nb[i] = real ? nr.u[i] : 1.0 / 3.0;
                nb[NN_MAX + i] = real ? nr.v[i] : 1.0 / 3.0;
                nb[2 * NN_MAX + i] = real ? nr.w[i] : 0.0;
            }
            // 1 / w^2 (0 for padding); the collapsed Gauss rules have positive weights only
            double* fs = buf->data() + 3 * NF_MAX + 3 * NN_MAX;
            double* ns = fs + NF_MAX;
            for (int i = 0; i < NF_MAX; ++i) {
                const double w = (*buf)[2 * NF_MAX + i];
                if (i < R.nf && !(w > 0.0)) throw std::logic_error("far rule: non-positive weight");
                fs[i] = i < R.nf ? 1.0 / (w * w) : 0.0;
            }
            for (int i = 0; i < NN_MAX; ++i) {
                const double w = nb[2 * NN_MAX + i];
                if (i < R.nn && !(w > 0.0)) throw std::logic_error("near rule: non-positive weight");
                ns[i] = i < R.nn ? 1.0 / (w * w) : 0.0;
            }
            slot = buf;
        }
        rules = slot;
    }
    cudaStream_t s = ctx->stream;
    const double* rb = rules->data();
    SBG_CUDA(cudaMemcpyToSymbolAsync(c_far_u, rb, NF_MAX * sizeof(double), 0, cudaMemcpyHostToDevice, s));
    SBG_CUDA(cudaMemcpyToSymbolAsync(c_far_v, rb + NF_MAX, NF_MAX * sizeof(double), 0, cudaMemcpyHostToDevice, s));
    SBG_CUDA(cudaMemcpyToSymbolAsync(c_far_w, rb + 2 * NF_MAX, NF_MAX * sizeof(double), 0, cudaMemcpyHostToDevice, s));
    rb += 3 * NF_MAX;
    SBG_CUDA(cudaMemcpyToSymbolAsync(c_near_u, rb, NN_MAX * sizeof(double), 0, cudaMemcpyHostToDevice, s));
    SBG_CUDA(cudaMemcpyToSymbolAsync(c_near_v, rb + NN_MAX, NN_MAX * sizeof(double), 0, cudaMemcpyHostToDevice, s));
    SBG_CUDA(cudaMemcpyToSymbolAsync(c_near_w, rb + 2 * NN_MAX, NN_MAX * sizeof(double), 0, cudaMemcpyHostToDevice, s));
    rb += 3 * NN_MAX;
    SBG_CUDA(cudaMemcpyToSymbolAsync(c_far_s, rb, NF_MAX * sizeof(double), 0, cudaMemcpyHostToDevice, s));
    SBG_CUDA(cudaMemcpyToSymbolAsync(c_near_s, rb + NF_MAX, NN_MAX * sizeof(double), 0, cudaMemcpyHostToDevice, s));
    SBG_CUDA(cudaMemcpyToSymbolAsync(g_near_u, rb - 3 * NN_MAX, NN_MAX * sizeof(double), 0, cudaMemcpyHostToDevice, s));
    SBG_CUDA(cudaMemcpyToSymbolAsync(g_near_v, rb - 2 * NN_MAX, NN_MAX * sizeof(double), 0, cudaMemcpyHostToDevice, s));
    SBG_CUDA(cudaMemcpyToSymbolAsync(g_near_w, rb - NN_MAX, NN_MAX * sizeof(double), 0, cudaMemcpyHostToDevice, s));
    SBG_CUDA(cudaMemcpyToSymbolAsync(g_near_s, rb + NF_MAX, NN_MAX * sizeof(double), 0, cudaMemcpyHostToDevice, s));
    // composed split4 maps (quadrature.hpp:222-229 child order), weights x32
    static const std::vector<unsigned char> paths = [] {
        std::vector<unsigned char> paths(NPATH * 9);
        int idx = 0;
        for (int d = 0; d <= 5; ++d) {
            int count = 1;
            for (int l = 0; l < d; ++l) count *= 4;
            for (int code = 0; code < count; ++code, ++idx) {
                int B[3][3] = {{32, 0, 0}, {0, 32, 0}, {0, 0, 32}};
                for (int l = 0; l < d; ++l) {
                    int digit = code;
                    for (int r = 0; r < d - 1 - l; ++r) digit /= 4;
                    digit %= 4;
                    int m01[3], m12[3], m02[3];
                    for (int c = 0; c < 3; ++c) {
                        m01[c] = (B[0][c] + B[1][c]) / 2;
                        m12[c] = (B[1][c] + B[2][c]) / 2;
                        m02[c] = (B[0][c] + B[2][c]) / 2;
                    }
                    int nb[3][3];
                    for (int c = 0; c < 3; ++c) {
                        const int v0 = B[0][c], v1 = B[1][c], v2 = B[2][c];
                        const int rows[4][3] = {{v0, m01[c], m02[c]}, {m01[c], v1, m12[c]}, {m02[c], m12[c], v2},
                                                {m01[c], m12[c], m02[c]}};
                        for (int r = 0; r < 3; ++r) nb[r][c] = rows[digit][r];
                    }
                    for (int r = 0; r < 3; ++r)
                        for (int c = 0; c < 3; ++c) B[r][c] = nb[r][c];
                }
                for (int r = 0; r < 3; ++r)
                    for (int c = 0; c < 3; ++c) paths[9 * idx + 3 * r + c] = (unsigned char)B[r][c];
            }
        }
        return paths;
    }();
    SBG_CUDA(cudaMemcpyToSymbolAsync(c_paths, paths.data(), paths.size(), 0, cudaMemcpyHostToDevice, s));
    SBG_CUDA(cudaMemcpyToSymbolAsync(g_paths, paths.data(), paths.size(), 0, cudaMemcpyHostToDevice, s));
    return R;
}

struct DeviceGeometry {
    DBuf<double> X, v, c, rad, diam, area;
    DBuf<int> F, vid;
    GeoPtrs ptrs() const { return {v.p, c.p, rad.p, diam.p, area.p, vid.p}; }
};

// Plan uploads through a page-locked staging arena (cached on the context, grow-only):
// a host memcpy into the arena and an asynchronous DMA, instead of a pageable
// cudaMemcpyAsync per array (each stages and synchronises inside the driver).  The
// arena is reused only after a stream synchronisation (the plan build ends with one).
struct StageArena {
    char* p = nullptr;
    size_t cap = 0;
    ~StageArena()
    {
        if (p) cudaFreeHost(p);
    }
};
struct Stager {
    Ctx* ctx;
    StageArena* A;
    size_t off = 0;
    explicit Stager(Ctx* c) : ctx(c)
    {
        if (!c->stage_ws) c->stage_ws = std::make_shared<StageArena>();
        A = static_cast<StageArena*>(c->stage_ws.get());
    }
    template <typename T>
    void upload(DBuf<T>& b, const T* h, size_t count)
    {
        if (count > b.n) b.alloc(count);
        raw(b.p, h, count * sizeof(T));
    }
    void raw(void* dst, const void* h, size_t bytes)
    {
        if (!bytes) return;
        if (off + bytes > A->cap) {  // arena full: wait for its copies, then reuse or grow it
            SBG_CUDA(cudaStreamSynchronize(ctx->stream));
            off = 0;
            if (bytes > A->cap) {
                if (A->p) SBG_CUDA(cudaFreeHost(A->p));
                A->p = nullptr;
                A->cap = 0;
                const size_t cap = std::max(bytes, (size_t)64 << 20);
                SBG_CUDA(cudaHostAlloc((void**)&A->p, cap, cudaHostAllocDefault));
                A->cap = cap;
            }
        }
        std::memcpy(A->p + off, h, bytes);
        SBG_CUDA(cudaMemcpyAsync(dst, A->p + off, bytes, cudaMemcpyHostToDevice, ctx->stream));
        off = (off + bytes + 255) & ~(size_t)255;
    }
    template <typename T>
    void upload(DBuf<T>& b, const std::vector<T>& v)
    {
        upload(b, v.data(), v.size());
    }
};

void upload_geometry(Ctx* ctx, const SurfaceMesh& m, DeviceGeometry& G, Stager* st)
{
    cudaStream_t s = ctx->stream;
    const int nf = m.num_facets(), nv = m.num_vertices();
    std::vector<double> X(3 * (size_t)nv);
    for (int i = 0; i < nv; ++i) {
        X[3 * i] = m.vertices[i].x;
        X[3 * i + 1] = m.vertices[i].y;
        X[3 * i + 2] = m.vertices[i].z;
    }
    std::vector<int> F(3 * (size_t)nf);
    for (int f = 0; f < nf; ++f)
        for (int k = 0; k < 3; ++k) F[3 * f + k] = m.facets[f][k];
    if (st) {
        st->upload(G.X, X);
        st->upload(G.F, F);
    } else {
        G.X.upload(X, s);
        G.F.upload(F, s);
    }
    G.v.alloc(9 * (size_t)nf);
    G.c.alloc(3 * (size_t)nf);
    G.rad.alloc(nf);
    G.diam.alloc(nf);
    G.area.alloc(nf);
    G.vid.alloc(3 * (size_t)nf);
    if (nf)
        k_facet_geometry<<<(nf + 127) / 128, 128, 0, s>>>(G.X.p, G.F.p, nf, G.v.p, G.c.p, G.rad.p, G.diam.p, G.area.p,
                                                          G.vid.p); ::sbg::count_launch();
    SBG_LAUNCH_CHECK();
}

// singular pairs grouped by class, t = larger facet index, permuted vertex ids
struct SingularLists {
    std::vector<int> pv[4];        // by shared count (1..3)
    std::vector<int2> pairs[4];    // (t, s)
};

// vertex-adjacent (f, g <= f) pairs with the permutation of pair_integral
// (quadrature.hpp:297-322): t = facet f (the larger index), shared vertices first in f's
// order, the rest ascending.
// returns the lists of consecutive facet ranges (built on up to 8 threads); their
// concatenation in range order is the single-pass list of every class
std::vector<SingularLists> singular_pairs(const SurfaceMesh& m)
{
    const int nf = m.num_facets(), nv = m.num_vertices();
    std::vector<int> sptr(nv + 1, 0), sfac(3 * (size_t)nf);  // vertex -> facets (CSR, ascending)
    for (int f = 0; f < nf; ++f)
        for (int k = 0; k < 3; ++k) ++sptr[m.facets[f][k] + 1];
    for (int v = 0; v < nv; ++v) sptr[v + 1] += sptr[v];
    {
        std::vector<int> fill(sptr.begin(), sptr.end() - 1);
        for (int f = 0; f < nf; ++f)
            for (int k = 0; k < 3; ++k) sfac[fill[m.facets[f][k]]++] = f;
    }
    auto range = [&](int f0, int f1, SingularLists& L) {
        // reserve for a regular triangulation: 1 identical, 1.5 edge, 4.5 vertex pairs per facet
        const size_t nfr = (size_t)(f1 - f0);
        const size_t est[4] = {0, 5 * nfr, 2 * nfr, nfr + 16};
        for (int c = 1; c <= 3; ++c) {
            L.pairs[c].reserve(est[c]);
            L.pv[c].reserve(6 * est[c]);
        }
        std::vector<int> nb;
        for (int f = f0; f < f1; ++f) {
            nb.clear();
            for (int k = 0; k < 3; ++k) {
                const int v = m.facets[f][k];
                for (int p = sptr[v]; p < sptr[v + 1] && sfac[p] <= f; ++p) nb.push_back(sfac[p]);
            }
            std::sort(nb.begin(), nb.end());
            nb.erase(std::unique(nb.begin(), nb.end()), nb.end());
            for (int g : nb) {
                int pf[3] = {-1, -1, -1}, pg[3] = {-1, -1, -1}, shared = 0;
                for (int i = 0; i < 3; ++i)
                    for (int j = 0; j < 3; ++j)
                        if (m.facets[f][i] == m.facets[g][j]) {
                            pf[shared] = i;
                            pg[shared] = j;
                            ++shared;
                            break;
                        }
                auto fill = [](int* p, int have) {
                    for (int k = 0; k < 3; ++k) {
                        bool used = false;
                        for (int q = 0; q < have; ++q) used |= (p[q] == k);
                        if (!used) p[have++] = k;
                    }
                };
                fill(pf, shared);
                fill(pg, shared);
                for (int k = 0; k < 3; ++k) L.pv[shared].push_back(m.facets[f][pf[k]]);
                for (int k = 0; k < 3; ++k) L.pv[shared].push_back(m.facets[g][pg[k]]);
                L.pairs[shared].push_back(make_int2(f, g));
            }
        }
    };
    // runs beside the plan's main thread (assembly_plan_create); facet ranges on a few
    // threads, each class list concatenated in range order (= the single-pass lists)
    const int nt = std::max(1, std::min(8, nf / 1024));
    std::vector<SingularLists> parts(nt);
    std::vector<std::thread> th;
    for (int t = 1; t < nt; ++t)
        th.emplace_back(range, (int)((long long)nf * t / nt), (int)((long long)nf * (t + 1) / nt), std::ref(parts[t]));
    range(0, (int)((long long)nf / nt), parts[0]);
    for (auto& t : th) t.join();
    return parts;  // (no concatenation: the plan uploads the parts at their offsets)
}

struct SauterRulesDev {
    DBuf<double> r[4];
    int npts[4] = {0, 0, 0, 0};
};

void upload_sauter(Ctx* ctx, const QuadCfg& cfg, SauterRulesDev& R)
{
    // the rules depend only on the order: build them once per process
    struct Rules {
        SauterRule id, ed, vx;
    };
    static std::mutex mu;
    static std::map<int, std::shared_ptr<const Rules>> cache;
    std::shared_ptr<const Rules> rules;
    {
        std::lock_guard<std::mutex> lock(mu);
        auto& slot = cache[cfg.singular_order];
        if (!slot) {
            auto r = std::make_shared<Rules>();
            sauter_rules(cfg.singular_order + 2, r->id, r->ed, r->vx);
            slot = r;
        }
        rules = slot;
    }
    const SauterRule &id = rules->id, &ed = rules->ed, &vx = rules->vx;
    // Gram-form monomials (k_sauter_partial): identical (c1^2, 2 c1 c2, c2^2, w) with
    // c = (a1 - b1, a2 - b2); edge (c1^2, a2^2, b2^2, 2 c1 a2, -2 c1 b2, -2 a2 b2, 0, w)
    std::vector<double> idp((size_t)id.size() * 4), edp((size_t)ed.size() * 8, 0.0);
    for (int i = 0; i < id.size(); ++i) {
        const double* a = id.pts.data() + 5 * i;
        const double c1 = a[0] - a[2], c2 = a[1] - a[3];
        double* o = idp.data() + 4 * i;
        const double sw = 1.0 / (a[4] * a[4]);  // the weight folded into r^2 (rsqrt_acc)
        o[0] = c1 * c1 * sw;
        o[1] = 2.0 * c1 * c2 * sw;
        o[2] = c2 * c2 * sw;
        o[3] = a[4];
    }
    for (int i = 0; i < ed.size(); ++i) {
        const double* a = ed.pts.data() + 5 * i;
        const double c1 = a[0] - a[2], c2 = a[1], c3 = a[3];
        double* o = edp.data() + 8 * i;
        const double sw = 1.0 / (a[4] * a[4]);
        o[0] = c1 * c1 * sw;
        o[1] = c2 * c2 * sw;
        o[2] = c3 * c3 * sw;
        o[3] = 2.0 * c1 * c2 * sw;
        o[4] = -2.0 * c1 * c3 * sw;
        o[5] = -2.0 * c2 * c3 * sw;
        o[7] = a[4];  // o[6] = 0: padding to 32-byte rows
    }
    // vertex class: the four coefficients scaled by 1 / w (r^2 then carries 1 / w^2)
    std::vector<double> vxp(vx.pts);
    for (int i = 0; i < vx.size(); ++i) {
        double* o = vxp.data() + 5 * i;
        const double iw = 1.0 / o[4];
        for (int k = 0; k < 4; ++k) o[k] *= iw;
    }
    for (const SauterRule* r : {&id, &ed, &vx})
        for (int i = 0; i < r->size(); ++i)
            if (!(r->pts[5 * i + 4] > 0.0)) throw std::logic_error("Sauter rule weight not positive: cannot fold");
    R.r[3].upload(idp, ctx->stream);
    R.npts[3] = id.size();
    R.r[2].upload(edp, ctx->stream);
    R.npts[2] = ed.size();
    R.r[1].upload(vxp, ctx->stream);
    R.npts[1] = vx.size();
}

// device copies of the Sauter rules, cached on the context per singular order (a fresh
// plan — every reference-style assemble_W call — does not upload the 5 MB of rules again)
std::shared_ptr<const SauterRulesDev> device_sauter(Ctx* ctx, const QuadCfg& cfg)
{
    using Cache = std::map<int, std::shared_ptr<SauterRulesDev>>;
    if (!ctx->sauter_ws) ctx->sauter_ws = std::make_shared<Cache>();
    auto& cache = *static_cast<Cache*>(ctx->sauter_ws.get());
    auto& slot = cache[cfg.singular_order];
    if (!slot) {
        auto R = std::make_shared<SauterRulesDev>();
        upload_sauter(ctx, cfg, *R);
        slot = R;
    }
    return slot;
}

void run_sauter(Ctx* ctx, const DBuf<double>& X, const std::vector<int>& pv, const SauterRulesDev& R, int cls,
                double* out_dev)
{
    const int np = (int)(pv.size() / 6);
    if (np == 0) return;
    cudaStream_t s = ctx->stream;
    DBuf<int> d_pv;
    d_pv.upload(pv, s);
    const int npts = R.npts[cls];
    int chunk = 0, nchunks = 0;
    sauter_chunking(ctx, cls, np, npts, chunk, nchunks);
    DBuf<double> part((size_t)nchunks * np);
    {
        TimedScope ts(ctx, "sauter");
        launch_sauter_partial(ctx, cls, d_pv.p, np, X.p, R.r[cls].p, npts, chunk, nchunks, part.p);
        k_sauter_finish<<<(np + 127) / 128, 128, 0, s>>>(part.p, np, nchunks, d_pv.p, X.p, out_dev); ::sbg::count_launch();
        SBG_LAUNCH_CHECK();
    }
    SBG_CUDA(cudaStreamSynchronize(s));
}

struct NearWork {
    DBuf<NearNode> buf[2], leaves;  // frontier (by level parity) and the leaf list
    // [0], [1] frontier counts by level parity, [2] leaves, [3] overflow, [4..9] level populations
    DBuf<unsigned long long> cnt;
    unsigned long long* hcnt = nullptr;  // page-locked copy, read after the assembly's final synchronisation
    ~NearWork()
    {
        if (hcnt) cudaFreeHost(hcnt);
    }
};
constexpr int kNearCnt = 10;
// the page-locked counter block: [0, kNearCnt) the near-field counters, then the near-list
// count and the mirror's non-finite flag of the assembly (read after its one synchronisation)
unsigned long long* near_host_counters(NearWork& NW)
{
    if (!NW.hcnt) SBG_CUDA(cudaMallocHost(&NW.hcnt, (kNearCnt + 3) * sizeof(unsigned long long)));
    return NW.hcnt;
}

// frontier buffers are cached on the context, so a fresh plan (every assemble_W
// call through the reference-style API) reuses the previous call's capacity
NearWork& near_work(Ctx* ctx)
{
    if (!ctx->near_ws) ctx->near_ws = std::make_shared<NearWork>();
    return *static_cast<NearWork*>(ctx->near_ws.get());
}

// owner rank of a near pair in a sharded assembly: by pair identity (every rank builds
// the near list itself, in its own atomic order), hashed so ranks get similar mixes
__device__ __forceinline__ int near_owner(int2 p, int world)
{
    const unsigned h = ((unsigned)p.x * 2654435761u) ^ ((unsigned)p.y * 2246822519u);
    return (int)((h ^ (h >> 15)) % (unsigned)world);
}

// root nodes of the near pairs (world > 1: only those this rank owns; cnt[0] zeroed)
__global__ void k_near_init(const unsigned long long* __restrict__ np_dev, long long cap, NearNode* __restrict__ nodes,
                            double* __restrict__ out, unsigned long long* __restrict__ cnt,
                            const int2* __restrict__ pairs, int rank, int world)
{
    const long long np = min((long long)*np_dev, cap);
    const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (world == 1) {
        if (k < np) {
            nodes[k] = {(int)k, 0u};
            out[k] = 0.0;
        }
        if (k == 0) cnt[0] = (unsigned long long)np;
        return;
    }
    if (k < np) {
        out[k] = 0.0;
        if (near_owner(pairs[k], world) == rank) nodes[atomicAdd(cnt, 1ull)] = {(int)k, 0u};
    }
}

// near-pair integrals for the device list pairs[0:*np_dev] (capacity cap), enqueued with
// no host synchronisation: the six recursion levels (fixed grid-stride launches reading
// their populations from the device) and one launch over all leaves.  The counters land in
// NW.hcnt (page-locked) for near_results() after the caller's synchronisation; capacities
// come from the previous runs on this context (or generous first guesses), and an overflow
// is reported there so the caller can regrow (near_regrow) and run again.
// (rank, world): only the near pairs this rank owns are integrated (the others' out = 0).
void run_near_leaves(Ctx* ctx, const RuleDims& R, const double* GV, const double* GA, const int2* pairs, double* out,
                     NearWork& NW);
void run_near(Ctx* ctx, const RuleDims& R, const double* GV, const double* GA, const int2* pairs,
              const unsigned long long* np_dev, long long cap, double thr, double* out, NearWork& NW, int rank = 0,
              int world = 1, bool leaves_now = true)
{
    if (cap <= 0) return;
    cudaStream_t s = ctx->stream;
    TimedScope ts(ctx, "near");
    if (!NW.cnt.n) NW.cnt.alloc(kNearCnt);
    near_host_counters(NW);
    set_max_dynamic_smem(k_near_leaves, NEAR_LEAF_SMEM);
    if ((long long)NW.buf[0].n < cap) {
        const long long f = std::max<long long>(16 * cap, NW.buf[0].n);
        NW.buf[0].alloc(f);
        NW.buf[1].alloc(f);
    }
    if ((long long)NW.leaves.n < 16 * cap) NW.leaves.alloc(64 * cap);
    const long long F = (long long)NW.buf[0].n, Lcap = (long long)NW.leaves.n;
    SBG_CUDA(cudaMemsetAsync(NW.cnt.p, 0, kNearCnt * sizeof(unsigned long long), s));
    k_near_init<<<(int)((cap + 255) / 256), 256, 0, s>>>(np_dev, cap, NW.buf[0].p, out, NW.cnt.p, pairs, rank, world);
    count_launch();
    SBG_LAUNCH_CHECK();
    {
        TimedScope tc(ctx, "near_classify");
        const int grid = 16 * ctx->sm_count;
        for (int depth = 0; depth <= 5; ++depth) {
            const int cur = depth & 1, nxt = cur ^ 1;
            if (depth > 0) SBG_CUDA(cudaMemsetAsync(NW.cnt.p + nxt, 0, sizeof(unsigned long long), s));
            k_near_level<<<grid, 128, 0, s>>>(NW.buf[cur].p, NW.cnt.p + cur, F, depth, pairs, GV, thr, NW.leaves.p,
                                              NW.cnt.p + 2, Lcap, NW.buf[nxt].p, NW.cnt.p + nxt, depth < 5 ? F : 0,
                                              NW.cnt.p + 3, NW.cnt.p + 4);
            count_launch();
            SBG_LAUNCH_CHECK();
        }
    }
    SBG_CUDA(cudaMemcpyAsync(NW.hcnt, NW.cnt.p, kNearCnt * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    if (leaves_now) run_near_leaves(ctx, R, GV, GA, pairs, out, NW);
}

// the leaf launch of run_near (separate when the assembly puts the far tiles in between)
void run_near_leaves(Ctx* ctx, const RuleDims& R, const double* GV, const double* GA, const int2* pairs, double* out,
                     NearWork& NW)
{
    if (!NW.leaves.n) return;
    cudaStream_t s = ctx->stream;
    const long long Lcap = (long long)NW.leaves.n;
    {
        TimedScope tl_scope(ctx, "near_leaves");
        const int lgrid = NEAR_LEAF_CTAS * ctx->sm_count;  // persistent: the leaf count is read on the device
        if (R.nnp == NN) {
            k_near_leaves<<<lgrid, NEAR_LEAF_THREADS, NEAR_LEAF_SMEM, s>>>(NW.leaves.p, NW.cnt.p + 2, Lcap, pairs, GV,
                                                                           GA, 1.0 / M_PI, out);
        } else {
            switch (R.nnp) {
#define SBG_NEAR_G(N) \
    case N: launch_near_leaves_g<N>(ctx, NW.leaves.p, NW.cnt.p + 2, Lcap, pairs, GV, GA, out); break;
                SBG_NEAR_G(16) SBG_NEAR_G(32) SBG_NEAR_G(48) SBG_NEAR_G(64) SBG_NEAR_G(96) SBG_NEAR_G(112)
#undef SBG_NEAR_G
            default: throw std::logic_error("near rule size not instantiated");
            }
        }
        count_launch();
        SBG_LAUNCH_CHECK();
    }
}

// after the stream has synchronised: leaves, pairs this rank integrated, overflow
struct NearResult {
    long long leaves = 0, owned = 0;
    bool overflow = false;
};
NearResult near_results(const NearWork& NW)
{
    NearResult r;
    if (!NW.hcnt) return r;
    r.leaves = (long long)NW.hcnt[2];
    r.owned = (long long)NW.hcnt[4];
    r.overflow = NW.hcnt[3] != 0;
    return r;
}
// grow the frontier and leaf buffers after an overflowed run: to the populations it saw
// (+25%) and at least twice the old size — a level cut short by a full buffer hides the
// true populations of the levels below it, so a run can reveal one more level at a time
void near_regrow(NearWork& NW)
{
    unsigned long long lvl = 0;
    for (int d = 0; d <= 5; ++d) lvl = std::max(lvl, NW.hcnt[4 + d]);
    const long long f = std::max<long long>((long long)(lvl * 5 / 4) + 1024, 2 * (long long)NW.buf[0].n);
    NW.buf[0].alloc(f);
    NW.buf[1].alloc(f);
    const long long l = std::max<long long>((long long)(NW.hcnt[2] * 5 / 4) + 1024, 2 * (long long)NW.leaves.n);
    NW.leaves.alloc(l);
}

}  // namespace

template <int NFP, bool EXACT>
void launch_far_tiles_n(Ctx* ctx, const TileInfo* tiles, long long ntiles, int tstride, const GeoPtrs& G,
                        const BlockPtrs& BP, double thr, DMatrix& W, int nr)
{
    constexpr size_t smem = far_smem_bytes(EXACT ? 0 : NFP);
    set_max_dynamic_smem(k_far_tiles<NFP, EXACT>, smem);
    k_far_tiles<NFP, EXACT><<<(int)ntiles, FAR_THREADS, smem, ctx->stream>>>(tiles, tstride, G, BP, thr, W.a.p,
                                                                            W.ld, 1.0 / M_PI, nr);
}

// ntiles launches: tile k of the launch is tiles[k * tstride]
void launch_far_tiles(Ctx* ctx, const RuleDims& R, const TileInfo* tiles, long long ntiles, int tstride,
                      const GeoPtrs& G, const BlockPtrs& BP, double thr, DMatrix& W, bool exact)
{
    if (ntiles <= 0) return;
    if (exact) {  // one instantiation: the rule size is a runtime loop bound there
        launch_far_tiles_n<4, true>(ctx, tiles, ntiles, tstride, G, BP, thr, W, R.nf);
        count_launch();
        return;
    }
    switch (R.nfp) {
#define SBG_FAR_TILES(N) \
    case N: launch_far_tiles_n<N, false>(ctx, tiles, ntiles, tstride, G, BP, thr, W, R.nf); break;
        SBG_FAR_TILES(4) SBG_FAR_TILES(12) SBG_FAR_TILES(16) SBG_FAR_TILES(28) SBG_FAR_TILES(36) SBG_FAR_TILES(52)
        SBG_FAR_TILES(64)
#undef SBG_FAR_TILES
    default: throw std::logic_error("far rule size not instantiated");
    }
    count_launch();
}

// ---------------------------------------------------------------- assembly plan
// Host-side preparation of one mesh (facet blocks, curl lists, tile list,
// singular lists, rules), uploaded once; assembly_run only launches kernels.
struct AssemblyPlan {
    Ctx* ctx = nullptr;
    QuadCfg cfg;
    RuleDims dims;
    int nf = 0, n = 0;
    DeviceGeometry G;
    DBuf<int> uptr, udof;
    DBuf<double> uval;
    DBuf<int> bfac, dof_ptr, dofs, ent_ptr;
    DBuf<double4> ents;
    DBuf<TileInfo> tiles, cand;
    long long ntiles = 0, ncand = 0;
    // local pairs: singular classes (vertex, edge, identical) then the near list
    long long nsing = 0, cls_off[4] = {0, 0, 0, 0}, cls_cnt[4] = {0, 0, 0, 0};
    DBuf<int> pv[4];
    DBuf<double> spart[4];
    int schunks[4] = {0, 0, 0, 0}, schunk[4] = {0, 0, 0, 0};
    std::shared_ptr<const SauterRulesDev> SR;
    long long near_cap = 0;
    long long h2d_bytes = 0;  // host-to-device bytes of the plan build (e2e bookkeeping)
    DBuf<int2> loc_pairs;
    DBuf<double> loc_I;
    DBuf<unsigned long long> near_cnt;
    DBuf<int> bad;  // non-finite flag of the mirror pass
    DBuf<int> band;  // max |i - j| of the near [0] and singular [1] entries (the host copy's band patches)
    // deferred curl-dependent half (plan_finish)
    std::unique_ptr<Stager> st;
    std::future<FacetCurls> curl_fut;
    std::vector<int> bfac_h;
    bool pending = false;
};
void plan_finish(AssemblyPlan* P);

// The curl-dependent half of a plan: curl lists (helper thread) and the per-block DOF
// lists of the far-tile contraction, uploaded through the plan's staging arena.
void plan_finish(AssemblyPlan* P)
{
    if (!P->pending) return;
    P->pending = false;
    Ctx* ctx = P->ctx;
    Stager& st = *P->st;
    const std::vector<int>& bfac = P->bfac_h;
    const int nblk = (int)(bfac.size() / BS);
    std::optional<HostScope> hs_wait(std::in_place, ctx, "plan_curl_wait");
    const FacetCurls U = P->curl_fut.get();
    hs_wait.reset();
    {
        HostScope hsu(ctx, "plan_upload_curls");
        st.upload(P->uptr, U.ptr);
        st.upload(P->udof, U.dof);
        st.upload(P->uval, U.u);
    }
    struct BlockLists {
        std::vector<int> dofs, ent_ptr, ndofs;
        std::vector<double4> ents;
    };
    auto build_blocks = [&](int b0, int b1, BlockLists& out) {
        struct DE {
            int dof, l, p;
        };
        std::vector<DE> dl;
        for (int b = b0; b < b1; ++b) {
            dl.clear();
            for (int l = 0; l < BS; ++l) {
                const int f = bfac[b * BS + l];
                if (f < 0) continue;
                for (int p = U.ptr[f]; p < U.ptr[f + 1]; ++p) dl.push_back({U.dof[p], l, p});
            }
            std::sort(dl.begin(), dl.end(),
                      [](const DE& x, const DE& y) { return x.dof != y.dof ? x.dof < y.dof : x.l < y.l; });
            int nd = 0;
            for (size_t i = 0; i < dl.size(); ++i) {
                if (i == 0 || dl[i].dof != dl[i - 1].dof) {
                    out.dofs.push_back(dl[i].dof);
                    out.ent_ptr.push_back((int)out.ents.size());
                    ++nd;
                }
                const int p = dl[i].p;
                out.ents.push_back(make_double4(U.u[3 * p], U.u[3 * p + 1], U.u[3 * p + 2], (double)dl[i].l));
            }
            out.ndofs.push_back(nd);
        }
    };
    const int nth = std::max(1, std::min(4, nblk / 32));
    std::vector<BlockLists> parts(nth);
    {
        HostScope hsb(ctx, "plan_blocks");
        std::vector<std::thread> th;
        for (int t = 1; t < nth; ++t)
            th.emplace_back(build_blocks, (int)((long long)nblk * t / nth), (int)((long long)nblk * (t + 1) / nth),
                            std::ref(parts[t]));
        build_blocks(0, (int)((long long)nblk / nth), parts[0]);
        for (auto& t : th) t.join();
    }
    std::vector<int> dof_ptr{0}, dofs, ent_ptr;
    std::vector<double4> ents;
    dof_ptr.reserve((size_t)nblk + 1);
    for (const auto& q : parts) {
        const int ebase = (int)ents.size();
        for (int c : q.ent_ptr) ent_ptr.push_back(ebase + c);
        for (int nd : q.ndofs) dof_ptr.push_back(dof_ptr.back() + nd);
        dofs.insert(dofs.end(), q.dofs.begin(), q.dofs.end());
        ents.insert(ents.end(), q.ents.begin(), q.ents.end());
    }
    ent_ptr.push_back((int)ents.size());
    st.upload(P->dof_ptr, dof_ptr);
    st.upload(P->dofs, dofs);
    st.upload(P->ent_ptr, ent_ptr);
    st.upload(P->ents, ents);
    // host-to-device bytes of this plan (e2e bookkeeping; rules are cached per context)
    auto bytes = [](const auto& b) { return (long long)(b.n * sizeof(*b.p)); };
    P->h2d_bytes = bytes(P->G.X) + bytes(P->G.F) + bytes(P->uptr) + bytes(P->udof) + bytes(P->uval) +
                   bytes(P->bfac) + bytes(P->dof_ptr) + bytes(P->dofs) + bytes(P->ent_ptr) + bytes(P->ents) +
                   bytes(P->tiles) + bytes(P->cand) + P->nsing * (long long)sizeof(int2);
    for (int cls = 1; cls <= 3; ++cls) P->h2d_bytes += bytes(P->pv[cls]);
}

AssemblyPlan* assembly_plan_create(Ctx* ctx, const InflatedMesh& im, const QuadCfg& cfg, bool defer)
{
    HostScope hs_all(ctx, "plan_total");
    auto* P = new AssemblyPlan;
    try {
        cudaStream_t s = ctx->stream;
        const SurfaceMesh& m = im.base;
        const int nf = m.num_facets();
        P->ctx = ctx;
        P->cfg = cfg;
        P->nf = nf;
        P->n = im.num_jump_dofs();
        if (nf == 0 || P->n == 0) return P;
        // host preparation that depends only on the mesh runs beside the main thread:
        // the singular lists (vertex adjacency) and the curl lists
        auto sing_fut = std::async(std::launch::async, [&m] {
            return singular_pairs(m);
        });
        auto curl_fut = std::async(std::launch::async, [&im] { return facet_curls(im); });
        P->st = std::make_unique<Stager>(ctx);
        Stager& st = *P->st;
        P->dims = upload_rules(ctx, cfg);
        upload_geometry(ctx, m, P->G, &st);
        HostScope hs1(ctx, "plan_curls");
        std::optional<HostScope> hs_morton(std::in_place, ctx, "plan_morton");
        // ---- Morton-ordered facet blocks
        std::vector<Vec3> cen(nf);
        double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
        double rmax = 0, dmax = 0;
        for (int f = 0; f < nf; ++f) {
            cen[f] = m.facet_centroid(f);
            const double xyz[3] = {cen[f].x, cen[f].y, cen[f].z};
            for (int d = 0; d < 3; ++d) {
                lo[d] = std::min(lo[d], xyz[d]);
                hi[d] = std::max(hi[d], xyz[d]);
            }
            for (int k = 0; k < 3; ++k) rmax = std::max(rmax, norm(m.vertices[m.facets[f][k]] - cen[f]));
            dmax = std::max(dmax, m.facet_diameter(f));
        }
        const double span = std::max({hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2], 1e-300});
        std::vector<std::uint64_t> key(nf);
        for (int f = 0; f < nf; ++f) {
            const double xyz[3] = {cen[f].x, cen[f].y, cen[f].z};
            std::uint64_t q[3];
            for (int d = 0; d < 3; ++d) q[d] = (std::uint64_t)((xyz[d] - lo[d]) / span * 2097151.0);
            key[f] = spread3(q[0]) | (spread3(q[1]) << 1) | (spread3(q[2]) << 2);
        }
        std::vector<int> perm(nf);
        std::iota(perm.begin(), perm.end(), 0);
        std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) { return key[a] < key[b]; });
        hs_morton.reset();
        const int nblk = (nf + BS - 1) / BS;
        std::vector<int> bfac((size_t)nblk * BS, -1);
        for (int k = 0; k < nf; ++k) bfac[k] = perm[k];
        std::vector<double> bcx(nblk), bcy(nblk), bcz(nblk), brad(nblk);
        for (int b = 0; b < nblk; ++b) {  // block centres and radii (the tile classification)
            Vec3 cs;
            int cnt = 0;
            for (int l = 0; l < BS; ++l) {
                const int f = bfac[b * BS + l];
                if (f < 0) continue;
                cs = cs + cen[f];
                ++cnt;
            }
            const Vec3 cc = cs / (double)cnt;
            double R = 0;
            for (int l = 0; l < BS; ++l) {
                const int f = bfac[b * BS + l];
                if (f >= 0) R = std::max(R, norm(cen[f] - cc));
            }
            bcx[b] = cc.x;
            bcy[b] = cc.y;
            bcz[b] = cc.z;
            brad[b] = R;
        }
        // the curl-dependent half (curl lists, per-block DOF lists) waits for the helper
        // thread; a deferred plan (one-shot assemble_W) runs it after the near-field launches
        P->curl_fut = std::move(curl_fut);
        P->bfac_h = bfac;
        P->pending = true;
        HostScope hs2(ctx, "plan_tiles");
        // ---- tiles (fb >= gb); certainly-far tiles skip per-pair classification
        const double thr = cfg.near_threshold;
        const double margin = 1e-9 * std::max(1.0, dmax);
        // launch order: full-cost tiles first (certain-far, off-diagonal), then the tiles with
        // per-pair tests and near pairs skipped, diagonal (half) tiles last, so the grid's
        // last wave holds the cheapest tiles (stable: fb-major within each class).  Generated
        // on host threads by fb ranges of equal pair counts into per-range class buckets,
        // concatenated in range order: the stable sort's order, and the candidate list's.
        const int nth = (int)std::min<long long>(8, std::max<long long>(1, (long long)nblk * nblk / 20000));
        std::vector<int> fb_cut(nth + 1, nblk);
        fb_cut[0] = 0;
        for (int t = 1; t < nth; ++t)  // fb^2 / 2 pairs below fb: equal-work cuts
            fb_cut[t] = std::min(nblk, (int)std::lround(nblk * std::sqrt((double)t / nth)));
        std::vector<std::array<std::vector<TileInfo>, 4>> part(nth);  // classes 0-2, candidates
        auto gen = [&](int t) {
            auto& B = part[t];
            for (int fb = fb_cut[t]; fb < fb_cut[t + 1]; ++fb)
                for (int gb = 0; gb <= fb; ++gb) {
                    const double dx = bcx[fb] - bcx[gb], dy = bcy[fb] - bcy[gb], dz = bcz[fb] - bcz[gb];
                    // any pair: dist_estimate >= D - R_f - R_g - 2 rmax >= thr * dmax (and no shared vertex)
                    const double lower = std::sqrt(dx * dx + dy * dy + dz * dz) - brad[fb] - brad[gb] - 2.0 * rmax;
                    const bool certain =
                        fb != gb && lower > margin && lower >= std::max(0.0, thr) * dmax * (1.0 + 1e-9) + margin;
                    B[fb == gb ? 2 : (certain ? 0 : 1)].push_back({fb, gb, certain ? 1 : 0, 0});
                    if (!certain) B[3].push_back({fb, gb, 0, 0});
                }
        };
        {
            std::vector<std::thread> th;
            for (int t = 1; t < nth; ++t) th.emplace_back(gen, t);
            gen(0);
            for (auto& x : th) x.join();
        }
        std::vector<TileInfo> tiles, cand;
        tiles.reserve((size_t)nblk * (nblk + 1) / 2);
        for (int r = 0; r < 3; ++r)
            for (int t = 0; t < nth; ++t) tiles.insert(tiles.end(), part[t][r].begin(), part[t][r].end());
        for (int t = 0; t < nth; ++t) cand.insert(cand.end(), part[t][3].begin(), part[t][3].end());
        st.upload(P->bfac, bfac);
        st.upload(P->tiles, tiles);
        st.upload(P->cand, cand);
        P->ntiles = (long long)tiles.size();
        P->ncand = (long long)cand.size();
        HostScope hs3(ctx, "plan_singular");
        // ---- singular lists (host adjacency, deterministic order) and Sauter workspaces
        std::optional<HostScope> hs_sw(std::in_place, ctx, "plan_singular_wait");
        const std::vector<SingularLists> SP = sing_fut.get();
        hs_sw.reset();
        P->SR = device_sauter(ctx, cfg);
        P->near_cap = std::max<long long>(1024, 64LL * nf);
        long long off = 0;
        for (int cls = 1; cls <= 3; ++cls) {
            P->cls_off[cls] = off;
            P->cls_cnt[cls] = 0;
            for (const auto& q : SP) P->cls_cnt[cls] += (long long)q.pairs[cls].size();
            off += P->cls_cnt[cls];
        }
        P->nsing = off;
        P->loc_pairs.alloc(P->nsing + P->near_cap);
        P->loc_I.alloc(P->nsing + P->near_cap);
        for (int cls = 1; cls <= 3; ++cls) {
            const long long np = P->cls_cnt[cls];
            if (!np) continue;
            if ((long long)P->pv[cls].n < 6 * np) P->pv[cls].alloc(6 * np);
            long long o = 0;
            for (const auto& q : SP) {  // the facet ranges' lists at their offsets (range order)
                const long long k = (long long)q.pairs[cls].size();
                st.raw(P->loc_pairs.p + P->cls_off[cls] + o, q.pairs[cls].data(), k * sizeof(int2));
                st.raw(P->pv[cls].p + 6 * o, q.pv[cls].data(), 6 * k * sizeof(int));
                o += k;
            }
            sauter_chunking(ctx, cls, (int)np, P->SR->npts[cls], P->schunk[cls], P->schunks[cls]);
            P->spart[cls].alloc((size_t)P->schunks[cls] * np);
        }
        P->near_cnt.alloc(1);
        P->bad.alloc(1);
        if (!defer) plan_finish(P);
        HostScope hs_sync(ctx, "plan_sync");
        SBG_CUDA(cudaStreamSynchronize(s));
    } catch (...) {
        cudaStreamSynchronize(ctx->stream);  // staged copies may still read the arena
        delete P;
        throw;
    }
    return P;
}

void assembly_plan_destroy(AssemblyPlan* P) { delete P; }

// reference: inc/assemble.hpp:72-139 (device kernels only; the plan holds the mesh data)
// Shard (rank, world) of world > 1 computes only its share of the work into a
// zeroed W: far tiles k with k % world == rank, the near pairs it owns
// (near_owner), and a contiguous 1/world range of each singular class.  The shards' W sum to the
// full W (up to fp64 atomic reordering); DESIGN.md §5.3.
namespace {
// SBG_TRACE_ASM=1: host-side timeline of one assembly (stderr), for diagnosing host stalls
struct HostTrace {
    bool on = std::getenv("SBG_TRACE_ASM") != nullptr;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    std::string line;
    void mark(const char* what)
    {
        if (!on) return;
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        char b[64];
        std::snprintf(b, sizeof b, " %s=%.1f", what, ms);
        line += b;
    }
    ~HostTrace()
    {
        if (on) std::fprintf(stderr, "[asm trace]%s\n", line.c_str());
    }
};
}  // namespace

// the host copy's diagonal patch (cached on the context: one-shot assemble_W plans are rebuilt
// every call): the singular entries' diagonals |i - j| (marks, kOffsMax + 1), the offset list,
// and the packed diagonals on the device and in page-locked memory
struct DiagPatchWork {
    DBuf<int> offs, dlist;
    DBuf<double> dpack;
    int* hoffs = nullptr;
    double* hpack = nullptr;
    size_t hpack_n = 0;
    ~DiagPatchWork()
    {
        if (hoffs) cudaFreeHost(hoffs);
        if (hpack) cudaFreeHost(hpack);
    }
};
DiagPatchWork& diag_work(Ctx* ctx)
{
    if (!ctx->diag_ws) {
        auto w = std::make_shared<DiagPatchWork>();
        w->offs.alloc(kOffsMax + 1);
        SBG_CUDA(cudaMallocHost(&w->hoffs, (kOffsMax + 1) * sizeof(int)));
        ctx->diag_ws = w;
    }
    return *static_cast<DiagPatchWork*>(ctx->diag_ws.get());
}

void assembly_run(AssemblyPlan* P, DMatrix& W, AssemblyStats* stats, int rank, int world, double* host_dst)
{
    HostTrace tr;
    if (world < 1 || rank < 0 || rank >= world) throw ValidationError("shard: need 0 <= rank < world");
    Ctx* ctx = P->ctx;
    cudaStream_t s = ctx->stream;
    TimedScope total(ctx, "assemble_W");
    if (tr.on) {
        cudaMemPool_t pool;
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetDefaultMemPool(&pool, dev);
        unsigned long long res = 0, used = 0;
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &res);
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
        char b[96];
        std::snprintf(b, sizeof b, " pool_res=%.2fG pool_used=%.2fG", res / 1e9, used / 1e9);
        tr.line += b;
    }
    if (W.n != P->n || !W.a.p) matrix_alloc(ctx, P->n, W);
    else SBG_CUDA(cudaMemsetAsync(W.a.p, 0, W.a.n * sizeof(double), s));
    tr.mark("alloc");
    if (P->nf == 0 || P->n == 0) return;
    const RuleDims R = upload_rules(ctx, P->cfg);
    tr.mark("rules");
    const double thr = P->cfg.near_threshold;
    auto share = [&](long long cnt) { return cnt > rank ? (cnt - rank + world - 1) / world : 0LL; };
    // far tiles are strided over the ranks; every rank classifies all candidate tiles (cheap)
    // and integrates the near pairs it owns (near_owner), which balances the near work
    const long long my_tiles = share(P->ntiles), my_cand = P->ncand;
    long long sing_lo[4] = {0, 0, 0, 0}, sing_cnt[4] = {0, 0, 0, 0};
    for (int cls = 1; cls <= 3; ++cls) {
        sing_lo[cls] = P->cls_cnt[cls] * rank / world;
        sing_cnt[cls] = P->cls_cnt[cls] * (rank + 1) / world - sing_lo[cls];
    }
    // Everything is enqueued without a host round trip; one synchronisation at the end reads
    // the near-list count, the near-field counters and the mirror's non-finite flag.  A
    // near list or near frontier that outgrew its buffers (first run of a mesh size on this
    // context) is regrown to the measured size and the assembly runs again.
    NearWork& NW = near_work(ctx);
    tr.mark("nearwork");
    unsigned long long* hnear = near_host_counters(NW) + kNearCnt;
    NearResult nr;
    // host_dst (page-locked, n x n row-major): W is also copied to the host, overlapped with
    // the near field — the far tiles run first and are mirrored, the copy of the whole W then
    // streams out on the auxiliary stream while the near leaves, the Sauter classes and their
    // scatter run, and afterwards only the band |i - j| <= K of entries the near/singular pairs
    // touched (K measured on the device) is copied again, straight from the device rows into
    // the host rows with one pitched DMA (row i's band starts (n + 1) elements after row i-1's)
    const bool to_host = host_dst != nullptr && world == 1;
    cudaStream_t cs = to_host ? aux_stream(ctx) : nullptr;
    cudaEvent_t ev_far = nullptr, ev_copy = nullptr;
    if (to_host) {
        SBG_CUDA(cudaEventCreateWithFlags(&ev_far, cudaEventDisableTiming));
        SBG_CUDA(cudaEventCreateWithFlags(&ev_copy, cudaEventDisableTiming));
    }
    struct EvGuard {
        cudaEvent_t a, b;
        ~EvGuard()
        {
            if (a) cudaEventDestroy(a);
            if (b) cudaEventDestroy(b);
        }
    } evg{ev_far, ev_copy};
    if (to_host && P->band.n < 2) P->band.alloc(2);
    DiagPatchWork* DW = to_host ? &diag_work(ctx) : nullptr;
    auto enqueue_far = [&]() {
        {
            TimedScope ts(ctx, "far_tiles");
            BlockPtrs BP{P->bfac.p, P->dof_ptr.p, P->dofs.p, P->ent_ptr.p, P->ents.p};
            launch_far_tiles(ctx, R, P->tiles.p + rank, my_tiles, world, P->G.ptrs(), BP, thr, W, P->cfg.exact_far);
            SBG_LAUNCH_CHECK();
        }
    };
    auto enqueue_mirror = [&]() {
        TimedScope ts(ctx, "mirror");
        const int nt = (P->n + 31) / 32;
        k_mirror<<<dim3(nt, nt), dim3(32, 8), 0, s>>>(W.a.p, P->n, W.ld, P->bad.p);
        count_launch();
        SBG_LAUNCH_CHECK();
    };
    // the rows' band |i - j| <= K of W into host_dst on stream st: the diagonal band of the
    // interior rows, and the fixed 2K + 1-column window at the matrix edge for the first and
    // last K rows (a few more final entries copied is harmless) — three pitched DMAs; a band
    // wider than n/4 (junction numberings) copies the whole W
    const int nW = P->n;
    auto band_wide = [&](int K) { return !(nW > 2 * K + 1 && (size_t)(2 * K + 1) * 4 < (size_t)nW); };
    auto band_copy = [&](cudaStream_t st, int K) {
        const size_t es = sizeof(double);
        const int n = nW;
        K = std::min(K, n - 1);
        if (!band_wide(K)) {
            const size_t w = es * (2 * (size_t)K + 1);
            SBG_CUDA(cudaMemcpy2DAsync(host_dst + (size_t)K * (n + 1) - K, es * ((size_t)n + 1),
                                       W.a.p + (size_t)K * (W.ld + 1) - K, es * ((size_t)W.ld + 1), w, n - 2 * K,
                                       cudaMemcpyDeviceToHost, st));
            if (K > 0) {
                SBG_CUDA(cudaMemcpy2DAsync(host_dst, es * n, W.a.p, es * W.ld, w, K, cudaMemcpyDeviceToHost, st));
                const size_t c0 = (size_t)n - (2 * (size_t)K + 1), r0 = (size_t)n - K;
                SBG_CUDA(cudaMemcpy2DAsync(host_dst + r0 * n + c0, es * n, W.a.p + r0 * W.ld + c0, es * W.ld, w, K,
                                           cudaMemcpyDeviceToHost, st));
            }
        } else {
            SBG_CUDA(cudaMemcpy2DAsync(host_dst, es * n, W.a.p, es * W.ld, es * n, n, cudaMemcpyDeviceToHost, st));
        }
    };
    auto enqueue_mirror_band = [&](const int* Kdev) {
        TimedScope ts(ctx, "mirror");
        const int nt = (P->n + 31) / 32;
        k_mirror_band<<<dim3(nt, nt), dim3(32, 8), 0, s>>>(W.a.p, P->n, W.ld, Kdev, P->bad.p);
        count_launch();
        SBG_LAUNCH_CHECK();
    };
    // to_host: the band the near pairs touched is copied on the second stream while the Sauter
    // classes run (its width is read from the device mid-assembly); only the narrower band
    // of the singular pairs is copied after the end
    int* hband = reinterpret_cast<int*>(hnear + 1) + 1;  // [0] near band, [1] singular band (hcnt has a spare word)
    bool near_patched = false;
    cudaEvent_t ev_near = nullptr, ev_patch = nullptr;
    if (to_host) {
        SBG_CUDA(cudaEventCreateWithFlags(&ev_near, cudaEventDisableTiming));
        SBG_CUDA(cudaEventCreateWithFlags(&ev_patch, cudaEventDisableTiming));
    }
    EvGuard evg2{ev_near, ev_patch};
    for (int attempt = 0;; ++attempt) {
        std::fill(NW.hcnt, NW.hcnt + kNearCnt + 3, 0ull);  // the previous run has synchronised
        if (attempt) SBG_CUDA(cudaMemsetAsync(W.a.p, 0, W.a.n * sizeof(double), s));
        SBG_CUDA(cudaMemsetAsync(P->near_cnt.p, 0, sizeof(unsigned long long), s));
        SBG_CUDA(cudaMemsetAsync(P->bad.p, 0, sizeof(int), s));
        if (to_host) SBG_CUDA(cudaMemsetAsync(P->band.p, 0, 2 * sizeof(int), s));
        tr.mark("memsets");
        if (my_cand) {  // near list: classification of the non-certainly-far tiles
            TimedScope ts(ctx, "classify");
            k_classify_near<<<(int)my_cand, 256, 0, s>>>(P->cand.p, 1, P->G.ptrs(), P->bfac.p, thr,
                                                         P->loc_pairs.p + P->nsing, P->near_cap, P->near_cnt.p);
            count_launch();
            SBG_LAUNCH_CHECK();
        }
        tr.mark("classify");
        run_near(ctx, R, P->G.v.p, P->G.area.p, P->loc_pairs.p + P->nsing, P->near_cnt.p, P->near_cap, thr,
                 P->loc_I.p + P->nsing, NW, rank, world, /*leaves_now=*/!to_host);
        tr.mark("near");
        // a deferred plan builds its curl-dependent half while the near field runs
        plan_finish(P);
        tr.mark("plan_finish");
        if (to_host) {
            enqueue_far();
            enqueue_mirror();
            SBG_CUDA(cudaEventRecord(ev_far, s));
            SBG_CUDA(cudaStreamWaitEvent(cs, ev_far, 0));
            cudaEvent_t ta = nullptr;
            if (ctx->timers.enabled) {  // "w_copy": the overlapped copy on the second stream
                ta = ctx->timers.get();
                SBG_CUDA(cudaEventRecord(ta, cs));
            }
            SBG_CUDA(cudaMemcpy2DAsync(host_dst, sizeof(double) * (size_t)P->n, W.a.p, sizeof(double) * (size_t)W.ld,
                                       sizeof(double) * (size_t)P->n, P->n, cudaMemcpyDeviceToHost, cs));
            if (ta) {
                cudaEvent_t tb = ctx->timers.get();
                SBG_CUDA(cudaEventRecord(tb, cs));
                ctx->timers.pending.push_back({"w_copy", ta, tb});
            }
            SBG_CUDA(cudaEventRecord(ev_copy, cs));
            tr.mark("far_copy");
            run_near_leaves(ctx, R, P->G.v.p, P->G.area.p, P->loc_pairs.p + P->nsing, P->loc_I.p + P->nsing, NW);
            tr.mark("leaves");
            if (P->near_cap > 0) {  // the near pairs' scatter (band[0]) and its band's mirror now
                TimedScope ts(ctx, "local_scatter");
                k_local_scatter<<<(int)((P->near_cap + 127) / 128), 128, 0, s>>>(
                    P->loc_pairs.p, P->loc_I.p, P->nsing, P->near_cnt.p, P->near_cap, P->uptr.p, P->udof.p, P->uval.p,
                    W.a.p, W.ld, P->band.p, P->nsing);
                count_launch();
                SBG_LAUNCH_CHECK();
            }
            enqueue_mirror_band(P->band.p);
            SBG_CUDA(cudaMemcpyAsync(hband, P->band.p, sizeof(int), cudaMemcpyDeviceToHost, s));
            SBG_CUDA(cudaEventRecord(ev_near, s));
        }
        // singular pairs (Sauter rules); a shard zeroes the integrals it does not own
        if (world > 1 && P->nsing) SBG_CUDA(cudaMemsetAsync(P->loc_I.p, 0, P->nsing * sizeof(double), s));
        for (int cls = 1; cls <= 3; ++cls) {
            const long long np = sing_cnt[cls];
            if (!np) continue;
            TimedScope ts(ctx, "sauter");
            const int* pv = P->pv[cls].p + 6 * sing_lo[cls];
            launch_sauter_partial(ctx, cls, pv, (int)np, P->G.X.p, P->SR->r[cls].p, P->SR->npts[cls], P->schunk[cls],
                                  P->schunks[cls], P->spart[cls].p);
            k_sauter_finish<<<(int)((np + 127) / 128), 128, 0, s>>>(P->spart[cls].p, (int)np, P->schunks[cls], pv,
                                                                     P->G.X.p,
                                                                     P->loc_I.p + P->cls_off[cls] + sing_lo[cls]);
            count_launch();
            SBG_LAUNCH_CHECK();
        }
        if (!to_host) enqueue_far();
        if (to_host) {  // the singular pairs' scatter (band[1]) and its band's mirror
            if (P->nsing > 0) {
                TimedScope ts(ctx, "local_scatter");
                SBG_CUDA(cudaMemsetAsync(DW->offs.p, 0, DW->offs.n * sizeof(int), s));
                k_local_scatter<<<(int)((P->nsing + 127) / 128), 128, 0, s>>>(
                    P->loc_pairs.p, P->loc_I.p, P->nsing, nullptr, 0, P->uptr.p, P->udof.p, P->uval.p, W.a.p, W.ld,
                    P->band.p + 1, 0, DW->offs.p);
                count_launch();
                SBG_LAUNCH_CHECK();
            }
            enqueue_mirror_band(P->band.p + 1);
        } else {  // per-pair scatter of singular + near integrals (near count read on the device)
            if (P->nsing + P->near_cap > 0) {
                TimedScope ts(ctx, "local_scatter");
                const long long nmax = P->nsing + P->near_cap;
                k_local_scatter<<<(int)((nmax + 127) / 128), 128, 0, s>>>(P->loc_pairs.p, P->loc_I.p, P->nsing,
                                                                          P->near_cnt.p, P->near_cap, P->uptr.p,
                                                                          P->udof.p, P->uval.p, W.a.p, W.ld, nullptr);
                count_launch();
                SBG_LAUNCH_CHECK();
            }
            enqueue_mirror();
        }
        SBG_CUDA(cudaMemcpyAsync(hnear, P->near_cnt.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
        SBG_CUDA(cudaMemcpyAsync(hnear + 1, P->bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        if (to_host) {
            SBG_CUDA(cudaMemcpyAsync(hband + 1, P->band.p + 1, sizeof(int), cudaMemcpyDeviceToHost, s));
            if (P->nsing > 0)
                SBG_CUDA(cudaMemcpyAsync(DW->hoffs, DW->offs.p, DW->offs.n * sizeof(int), cudaMemcpyDeviceToHost, s));
            else
                std::fill(DW->hoffs, DW->hoffs + DW->offs.n, 0);
            // the near band's copy beside the Sauter classes, once its width has landed
            SBG_CUDA(cudaEventSynchronize(ev_near));
            near_patched = !band_wide(hband[0]);
            if (near_patched) {
                SBG_CUDA(cudaStreamWaitEvent(cs, ev_near, 0));
                band_copy(cs, hband[0]);
            }
            SBG_CUDA(cudaEventRecord(ev_patch, cs));
        }
        tr.mark("enqueued");
        SBG_CUDA(cudaStreamSynchronize(s));
        tr.mark("sync");
        nr = near_results(NW);
        const bool list_over = (long long)hnear[0] > P->near_cap;
        if (!list_over && !nr.overflow) break;
        if (attempt >= 6) throw std::logic_error("near field: buffers still too small after regrowth");
        if (nr.overflow) near_regrow(NW);
        if (list_over) {  // near list overflow: grow (keeping the singular pairs) and redo
            P->near_cap = (long long)hnear[0] + 1024;
            DBuf<int2> np2(P->nsing + P->near_cap);
            DBuf<double> ni2(P->nsing + P->near_cap);
            if (P->nsing)
                SBG_CUDA(cudaMemcpyAsync(np2.p, P->loc_pairs.p, P->nsing * sizeof(int2), cudaMemcpyDeviceToDevice, s));
            P->loc_pairs = std::move(np2);
            P->loc_I = std::move(ni2);
        }
    }
    if (to_host) {
        // the last patch, after the whole-W copy and the near band's patch have landed: the
        // singular pairs' band (or, when the near band was too wide to patch, the larger band)
        TimedScope ts(ctx, "band_patch");
        SBG_CUDA(cudaStreamWaitEvent(s, ev_copy, 0));
        SBG_CUDA(cudaStreamWaitEvent(s, ev_patch, 0));
        // the singular entries lie on a few diagonals (a regular grid numbering: |i - j| in a
        // handful of short runs): when those diagonals are fewer than a quarter of the band,
        // they are packed on the device, copied in one piece and unpacked on host threads
        std::vector<int> dl;
        if (near_patched && hband[1] <= kOffsMax) {
            const int* mk = DW->hoffs;
            for (int d = 0; d <= hband[1]; ++d)
                if (mk[d]) {
                    dl.push_back(d);
                    if (d) dl.push_back(-d);
                }
        }
        const int nd = (int)dl.size();
        if (near_patched && hband[1] <= kOffsMax && (size_t)nd * 4 <= 2 * (size_t)hband[1] + 1) {
            const size_t cnt = (size_t)nW * std::max(nd, 1);
            if (DW->dlist.n < (size_t)std::max(nd, 1)) DW->dlist.alloc(std::max(nd, 1));
            if (DW->dpack.n < cnt) DW->dpack.alloc(cnt);
            if (DW->hpack_n < cnt) {
                if (DW->hpack) SBG_CUDA(cudaFreeHost(DW->hpack));
                DW->hpack = nullptr;
                DW->hpack_n = 0;
                SBG_CUDA(cudaMallocHost(&DW->hpack, cnt * sizeof(double)));
                DW->hpack_n = cnt;
            }
            if (nd) {  // dl is read by the copy engine before the synchronisation below
                SBG_CUDA(cudaMemcpyAsync(DW->dlist.p, dl.data(), nd * sizeof(int), cudaMemcpyHostToDevice, s));
                k_pack_diagonals<<<(unsigned)((cnt + 255) / 256), 256, 0, s>>>(W.a.p, nW, W.ld, DW->dlist.p, nd,
                                                                               DW->dpack.p);
                count_launch();
                SBG_LAUNCH_CHECK();
                SBG_CUDA(cudaMemcpyAsync(DW->hpack, DW->dpack.p, cnt * sizeof(double), cudaMemcpyDeviceToHost, s));
            }
            SBG_CUDA(cudaStreamSynchronize(s));  // (also: the W copy and the near band patch have landed)
            const double* hp = DW->hpack;
            const int nth = nd ? std::max(1, std::min(16, nW / 2048)) : 0;
            auto unpack = [&](int t) {
                for (int i = (int)((long long)nW * t / nth); i < (int)((long long)nW * (t + 1) / nth); ++i)
                    for (int k = 0; k < nd; ++k) {
                        const int j = i + dl[k];
                        if (j >= 0 && j < nW) host_dst[(size_t)i * nW + j] = hp[(size_t)i * nd + k];
                    }
            };
            std::vector<std::thread> th;
            for (int t = 1; t < nth; ++t) th.emplace_back(unpack, t);
            if (nth) unpack(0);
            for (auto& x : th) x.join();
        } else {
            band_copy(s, near_patched ? hband[1] : std::max(hband[0], hband[1]));
        }
        tr.mark("band_enq");
        SBG_CUDA(cudaStreamSynchronize(s));
        tr.mark("band_sync");
    }
    if (*reinterpret_cast<const int*>(hnear + 1)) throw NumericalError("quadrature produced a non-finite pair integral");
    const unsigned long long nnear = hnear[0];
    const long long leaves = nr.leaves, near_owned = nr.owned;
    const long long nloc = P->nsing + (long long)nnear;
    if (stats) {
        stats->identical = sing_cnt[3];
        stats->edge = sing_cnt[2];
        stats->vertex = sing_cnt[1];
        stats->near_pairs = world == 1 ? (long long)nnear : near_owned;
        stats->near_leaves = leaves;
        // per shard the far count is not separated from the tiles' own classification
        stats->far_pairs = world == 1 ? (long long)P->nf * (P->nf + 1) / 2 - nloc : -1;
        stats->tiles = my_tiles;
        stats->tiles_skipped = my_tiles - share(P->ncand);  // sums to the total over the ranks
        stats->h2d_bytes = P->h2d_bytes;
    }
}

void assemble_W(Ctx* ctx, const InflatedMesh& im, const QuadCfg& cfg, DMatrix& W, AssemblyStats* stats,
                double* host_dst)
{
    AssemblyPlan* P = assembly_plan_create(ctx, im, cfg, /*defer=*/true);
    try {
        assembly_run(P, W, stats, 0, 1, host_dst);
        SBG_CUDA(cudaStreamSynchronize(ctx->stream));
    } catch (...) {
        delete P;
        throw;
    }
    delete P;
}

namespace {
__global__ void k_far_pair_list_exact(GeoPtrs G, const int2* __restrict__ pairs, long long np,
                                      double* __restrict__ out, int nr)
{
    const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= np) return;
    const int f = pairs[k].x, g = pairs[k].y;  // f = t (the larger index, host-ordered)
    out[k] = far_pair_exact(G.v + 9 * f, G.v + 9 * g, G.area[f], G.area[g], nr);
}

template <int NFP>
__global__ void k_far_pair_list(GeoPtrs G, const int2* __restrict__ pairs, long long np, double* __restrict__ out,
                                double inv_pi)
{
    const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= np) return;
    const int f = pairs[k].x, g = pairs[k].y;
    const double* t = G.v + 9 * f;
    const double* sv = G.v + 9 * g;
    double4 Y[NFP];
    for (int j = 0; j < NFP; ++j) Y[j] = far_ypoint(sv, t, j);
    double acc = 0.0;
    for (int pass = 0; pass < NFP / FAR_PASS; ++pass) {
        XPts<> X;
        far_xpoints(t, t, pass, X);
        acc += far_pass_sum<NFP>(X, Y, pass) * (G.area[f] * inv_pi) * G.area[g];
    }
    out[k] = acc;
}
void far_pair_list(Ctx* ctx, const RuleDims& R, const GeoPtrs& G, const int2* pairs, long long np, double* out,
                   bool exact)
{
    const int grid = (int)((np + 127) / 128);
    cudaStream_t s = ctx->stream;
    if (exact) {
        k_far_pair_list_exact<<<grid, 128, 0, s>>>(G, pairs, np, out, R.nf);
        ::sbg::count_launch();
        SBG_LAUNCH_CHECK();
        return;
    }
    switch (R.nfp) {
#define SBG_FAR_LIST(N) \
    case N: k_far_pair_list<N><<<grid, 128, 0, s>>>(G, pairs, np, out, 1.0 / M_PI); break;
        SBG_FAR_LIST(4) SBG_FAR_LIST(12) SBG_FAR_LIST(16) SBG_FAR_LIST(28) SBG_FAR_LIST(36) SBG_FAR_LIST(52)
        SBG_FAR_LIST(64)
#undef SBG_FAR_LIST
    default: throw std::logic_error("far rule size not instantiated");
    }
    ::sbg::count_launch();
    SBG_LAUNCH_CHECK();
}

}  // namespace

// Device quadrature on an explicit pair list (parity harness): each pair is
// classified on the host exactly as pair_integral does and routed to the same
// kernels the assembly uses.
void pair_integrals(Ctx* ctx, const SurfaceMesh& m, const QuadCfg& cfg, const int* f, const int* g, long long np,
                    double* out)
{
    cudaStream_t s = ctx->stream;
    const RuleDims R = upload_rules(ctx, cfg);
    DeviceGeometry G;
    upload_geometry(ctx, m, G, nullptr);
    const SauterRulesDev& SR = *device_sauter(ctx, cfg);
    std::vector<double> hgc(3 * (size_t)m.num_facets()), hrad(m.num_facets()), hdiam(m.num_facets());
    SBG_CUDA(cudaMemcpyAsync(hgc.data(), G.c.p, hgc.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    SBG_CUDA(cudaMemcpyAsync(hrad.data(), G.rad.p, hrad.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    SBG_CUDA(cudaMemcpyAsync(hdiam.data(), G.diam.p, hdiam.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    SBG_CUDA(cudaStreamSynchronize(s));
    std::vector<int> pv[4];
    std::vector<long long> idx[5];  // 1..3 singular, 0 near, 4 far
    std::vector<int2> nearp, farp;
    for (long long k = 0; k < np; ++k) {
        const int a = f[k], b = g[k];
        if (a < 0 || b < 0 || a >= m.num_facets() || b >= m.num_facets()) throw ValidationError("facet index out of range");
        const int t = std::max(a, b), sf = std::min(a, b);
        int pf[3] = {-1, -1, -1}, pg[3] = {-1, -1, -1}, shared = 0;
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j)
                if (m.facets[a][i] == m.facets[b][j]) {
                    pf[shared] = i;
                    pg[shared] = j;
                    ++shared;
                    break;
                }
        if (shared > 0) {
            // pair_integral(m, f, g) permutes in the order of its first argument
            auto fill = [](int* p, int have) {
                for (int q = 0; q < 3; ++q) {
                    bool used = false;
                    for (int r = 0; r < have; ++r) used |= (p[r] == q);
                    if (!used) p[have++] = q;
                }
            };
            fill(pf, shared);
            fill(pg, shared);
            for (int q = 0; q < 3; ++q) pv[shared].push_back(m.facets[a][pf[q]]);
            for (int q = 0; q < 3; ++q) pv[shared].push_back(m.facets[b][pg[q]]);
            idx[shared].push_back(k);
            continue;
        }
        // classification as in the device kernels (host copy of the device geometry)
        auto nrm = [](double x, double y, double z) { return std::sqrt((x * x + y * y) + z * z); };
        const double* ct = &hgc[3 * t];
        const double* cs = &hgc[3 * sf];
        const double dist = std::max(0.0, (nrm(ct[0] - cs[0], ct[1] - cs[1], ct[2] - cs[2]) - hrad[t]) - hrad[sf]);
        if (dist >= cfg.near_threshold * std::max(hdiam[t], hdiam[sf])) {
            farp.push_back(make_int2(a, b));
            idx[4].push_back(k);
        } else {
            nearp.push_back(make_int2(t, sf));
            idx[0].push_back(k);
        }
    }
    std::vector<double> tmp;
    auto fetch = [&](const double* d, const std::vector<long long>& ids) {
        tmp.resize(ids.size());
        SBG_CUDA(cudaMemcpyAsync(tmp.data(), d, ids.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
        SBG_CUDA(cudaStreamSynchronize(s));
        for (size_t i = 0; i < ids.size(); ++i) out[ids[i]] = tmp[i];
    };
    for (int cls = 1; cls <= 3; ++cls)
        if (!idx[cls].empty()) {
            DBuf<double> o(idx[cls].size());
            run_sauter(ctx, G.X, pv[cls], SR, cls, o.p);
            fetch(o.p, idx[cls]);
        }
    if (!nearp.empty()) {
        DBuf<int2> d_p;
        d_p.upload(nearp, s);
        DBuf<double> o(nearp.size());
        DBuf<unsigned long long> cnt(1);
        const unsigned long long hn = nearp.size();
        SBG_CUDA(cudaMemcpyAsync(cnt.p, &hn, sizeof(hn), cudaMemcpyHostToDevice, s));
        NearWork NW;
        for (int attempt = 0;; ++attempt) {
            run_near(ctx, R, G.v.p, G.area.p, d_p.p, cnt.p, (long long)nearp.size(), cfg.near_threshold, o.p, NW);
            SBG_CUDA(cudaStreamSynchronize(s));
            if (!near_results(NW).overflow) break;
            if (attempt >= 6) throw std::logic_error("near field: buffers still too small after regrowth");
            near_regrow(NW);
        }
        fetch(o.p, idx[0]);
    }
    if (!farp.empty()) {
        // far pairs through the tile kernel's evaluation: a dedicated 1-facet
        // block layout so each pair is its own (fb, gb) tile is wasteful; use the
        // same device functions on a pair list instead.
        DBuf<int2> d_p;
        d_p.upload(farp, s);
        DBuf<double> o(farp.size());
        far_pair_list(ctx, R, G.ptrs(), d_p.p, (long long)farp.size(), o.p, cfg.exact_far);
        fetch(o.p, idx[4]);
    }
}

std::vector<double> rhs_points(const InflatedMesh& im, const QuadCfg& cfg)
{
    const SurfaceMesh& m = im.base;
    const TriangleRule r = triangle_rule(cfg.far_order);
    std::vector<double> pts;
    pts.reserve((size_t)m.num_facets() * r.w.size() * 3);
    for (int f = 0; f < m.num_facets(); ++f) {
        const auto& t = m.facets[f];
        for (size_t i = 0; i < r.w.size(); ++i) {
            Vec3 y = m.vertices[t[0]] + r.u[i] * (m.vertices[t[1]] - m.vertices[t[0]]);
            y = y + r.v[i] * (m.vertices[t[2]] - m.vertices[t[0]]);
            pts.insert(pts.end(), {y.x, y.y, y.z});
        }
    }
    return pts;
}

// reference: inc/assemble.hpp:143-184
void assemble_rhs(Ctx* ctx, const InflatedMesh& im, const QuadCfg& cfg, const double* g, bool g_is_field,
                  double* L_host)
{
    cudaStream_t s = ctx->stream;
    const SurfaceMesh& m = im.base;
    const int nf = m.num_facets(), n = im.num_jump_dofs();
    const RuleDims R = rule_dims(cfg.far_order);
    const size_t ng = g_is_field ? (size_t)nf * R.nf * 3 : 3;
    for (size_t i = 0; i < ng; ++i)
        if (!std::isfinite(g[i])) throw NumericalError("g returned a non-finite value");
    upload_rules(ctx, cfg);
    DeviceGeometry G;
    upload_geometry(ctx, m, G, nullptr);
    // scatter terms per (oriented facet, slot) (assemble.hpp:34-53)
    std::vector<int> sptr{0}, sdof;
    std::vector<double> ssgn, onorm(6 * (size_t)nf);
    for (int o = 0; o < 2 * nf; ++o) {
        onorm[3 * o] = im.onormal[o].x;
        onorm[3 * o + 1] = im.onormal[o].y;
        onorm[3 * o + 2] = im.onormal[o].z;
        for (int k = 0; k < 3; ++k) {
            const int v = m.facets[o / 2][k], b = im.ofacet_branch[o][k], q = im.q[v];
            if (q >= 2) {
                if (b < q - 1) {
                    sdof.push_back(im.dof_index(v, b));
                    ssgn.push_back(1.0);
                } else {
                    for (int j = 0; j + 1 < q; ++j) {
                        sdof.push_back(im.dof_index(v, j));
                        ssgn.push_back(-1.0);
                    }
                }
            }
            sptr.push_back((int)sdof.size());
        }
    }
    DBuf<int> d_sptr, d_sdof;
    DBuf<double> d_ssgn, d_on, d_g, d_L(std::max(n, 1));
    d_sptr.upload(sptr, s);
    d_sdof.upload(sdof, s);
    d_ssgn.upload(ssgn, s);
    d_on.upload(onorm, s);
    d_g.upload(g, ng, s);
    SBG_CUDA(cudaMemsetAsync(d_L.p, 0, d_L.n * sizeof(double), s));
    if (nf)
        k_rhs<<<(nf * R.nf + 127) / 128, 128, 0, s>>>(nf, R.nf, G.v.p, d_on.p, d_g.p, g_is_field ? 1 : 0, d_sptr.p, d_sdof.p,
                                                    d_ssgn.p, d_L.p); ::sbg::count_launch();
    SBG_LAUNCH_CHECK();
    if (n) SBG_CUDA(cudaMemcpyAsync(L_host, d_L.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    SBG_CUDA(cudaStreamSynchronize(s));
}

}  // namespace sbg
