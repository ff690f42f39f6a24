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
#include <cmath>
#include <numeric>

#include "kernels.cuh"

namespace sbg {

namespace {

constexpr int BS = 64;          // facets per block
constexpr int FAR_THREADS = 256;
constexpr int NF = 16;          // far rule points (far_order 4)
constexpr int NN = 36;          // near rule points (far_order + 2 = 6)
constexpr int SAUTER_THREADS = 128;
constexpr int SAUTER_STAGE = 1024;  // rule points staged per smem pass
constexpr int NEAR_WARPS = 8;

__constant__ double c_far_u[NF], c_far_v[NF], c_far_w[NF];
__constant__ double c_near_u[NN], c_near_v[NN], c_near_w[NN];

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

// ---------------------------------------------------------------- far rule
struct FarPts {
    double x[NF], y[NF], z[NF];
};

__device__ __forceinline__ void far_points(const double* t, FarPts& P)
{
    const double e1x = t[3] - t[0], e1y = t[4] - t[1], e1z = t[5] - t[2];
    const double e2x = t[6] - t[0], e2y = t[7] - t[1], e2z = t[8] - t[2];
#pragma unroll
    for (int i = 0; i < NF; ++i) {
        P.x[i] = fma(c_far_v[i], e2x, fma(c_far_u[i], e1x, t[0]));
        P.y[i] = fma(c_far_v[i], e2y, fma(c_far_u[i], e1y, t[1]));
        P.z[i] = fma(c_far_v[i], e2z, fma(c_far_u[i], e1z, t[2]));
    }
}

// sum_ij w_i w_j / |x_i - y_j| for the 16x16 tensor rule (triangle_pair_rule,
// quadrature.hpp:208-220, without the 4 A A' / (4 pi) factor)
__device__ __forceinline__ double far_sum(const FarPts& P, const double* s)
{
    const double e1x = s[3] - s[0], e1y = s[4] - s[1], e1z = s[5] - s[2];
    const double e2x = s[6] - s[0], e2y = s[7] - s[1], e2z = s[8] - s[2];
    double acc = 0.0;
#pragma unroll 1
    for (int j = 0; j < NF; ++j) {
        const double u = c_far_u[j], v = c_far_v[j];
        const double yx = fma(v, e2x, fma(u, e1x, s[0]));
        const double yy = fma(v, e2y, fma(u, e1y, s[1]));
        const double yz = fma(v, e2z, fma(u, e1z, s[2]));
        double in0 = 0.0, in1 = 0.0;
#pragma unroll
        for (int i = 0; i < NF; i += 2) {
            const double ax = P.x[i] - yx, ay = P.y[i] - yy, az = P.z[i] - yz;
            const double bx = P.x[i + 1] - yx, by = P.y[i + 1] - yy, bz = P.z[i + 1] - yz;
            const double ra = fma(ax, ax, fma(ay, ay, az * az));
            const double rb = fma(bx, bx, fma(by, by, bz * bz));
            in0 = fma(c_far_w[i], rsqrt_fast(ra), in0);
            in1 = fma(c_far_w[i + 1], rsqrt_fast(rb), in1);
        }
        acc = fma(c_far_w[j], in0 + in1, acc);
    }
    return acc;
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

// contraction of the I tile with the curl lists, flushed to W's upper triangle
__device__ void tile_contract_flush(const double* __restrict__ It, int fb, int gb, bool diag, const BlockPtrs& B,
                                    double* __restrict__ W, int ld)
{
    const int fa0 = B.dof_ptr[fb], na = B.dof_ptr[fb + 1] - fa0;
    const int gb0 = B.dof_ptr[gb], nbd = B.dof_ptr[gb + 1] - gb0;
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
        if (s == 0.0) continue;
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
}

__global__ void __launch_bounds__(FAR_THREADS, 1)
    k_far_tiles(const TileInfo* __restrict__ tiles, GeoPtrs G, BlockPtrs B, double thr, double* __restrict__ W,
                int ld, double inv_pi)
{
    __shared__ double It[BS * (BS + 1)];
    __shared__ double gv[BS * 9];
    __shared__ double gcr[BS * 5];  // cx, cy, cz, rad, diam
    __shared__ double garea[BS];
    __shared__ int gid[BS], gvid[BS * 3];
    const TileInfo T = tiles[blockIdx.x];
    const bool diag = T.fb == T.gb;
    for (int e = threadIdx.x; e < BS; e += blockDim.x) {
        const int g = B.facets[T.gb * BS + e];
        gid[e] = g;
        if (g >= 0) {
            for (int k = 0; k < 9; ++k) gv[e * 9 + k] = G.v[9 * g + k];
            gcr[e * 5] = G.c[3 * g];
            gcr[e * 5 + 1] = G.c[3 * g + 1];
            gcr[e * 5 + 2] = G.c[3 * g + 2];
            gcr[e * 5 + 3] = G.rad[g];
            gcr[e * 5 + 4] = G.diam[g];
            garea[e] = G.area[g];
            for (int k = 0; k < 3; ++k) gvid[e * 3 + k] = G.vid[3 * g + k];
        }
    }
    for (int e = threadIdx.x; e < BS * (BS + 1); e += blockDim.x) It[e] = 0.0;
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int fl = (warp & 1) * 32 + lane;
    const int f = B.facets[T.fb * BS + fl];
    if (f >= 0) {
        double t[9];
        for (int k = 0; k < 9; ++k) t[k] = G.v[9 * f + k];
        const D3 cf = {G.c[3 * f], G.c[3 * f + 1], G.c[3 * f + 2]};
        const double rf = G.rad[f], df = G.diam[f], af = G.area[f];
        int fv[3] = {G.vid[3 * f], G.vid[3 * f + 1], G.vid[3 * f + 2]};
        FarPts P;
        far_points(t, P);
        for (int gl = warp >> 1; gl < BS; gl += FAR_THREADS / 64) {
            const int g = gid[gl];
            if (g < 0 || (diag && gl >= fl)) continue;
            bool far = true;
            if (!T.certain_far) {
                if (shared_count(fv, gvid + 3 * gl) > 0) {
                    far = false;
                } else {
                    const D3 cg = {gcr[gl * 5], gcr[gl * 5 + 1], gcr[gl * 5 + 2]};
                    far = (f > g) ? far_test(cf, rf, df, cg, gcr[gl * 5 + 3], gcr[gl * 5 + 4], thr)
                                  : far_test(cg, gcr[gl * 5 + 3], gcr[gl * 5 + 4], cf, rf, df, thr);
                }
            }
            if (!far) continue;
            const double acc = far_sum(P, gv + 9 * gl);
            It[fl * (BS + 1) + gl] = acc * af * garea[gl] * inv_pi;
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
    tile_contract_flush(It, T.fb, T.gb, diag, B, W, ld);
}

// near-list builder: pairs of non-certainly-far tiles that are disjoint but not far
__global__ void k_classify_near(const TileInfo* __restrict__ tiles, GeoPtrs G, const int* __restrict__ bfacets,
                                double thr, int2* __restrict__ near_list, unsigned long long cap,
                                unsigned long long* __restrict__ count)
{
    const TileInfo T = tiles[blockIdx.x];
    const bool diag = T.fb == T.gb;
    for (int e = threadIdx.x; e < BS * BS; e += blockDim.x) {
        const int fl = e / BS, gl = e % BS;
        if (diag && gl >= fl) continue;
        const int f = bfacets[T.fb * BS + fl], g = bfacets[T.gb * BS + gl];
        if (f < 0 || g < 0) continue;
        if (shared_count(G.vid + 3 * f, G.vid + 3 * g) > 0) continue;
        const int t = max(f, g), s = min(f, g);
        const D3 ct = {G.c[3 * t], G.c[3 * t + 1], G.c[3 * t + 2]};
        const D3 cs = {G.c[3 * s], G.c[3 * s + 1], G.c[3 * s + 2]};
        if (far_test(ct, G.rad[t], G.diam[t], cs, G.rad[s], G.diam[s], thr)) continue;
        const unsigned long long k = atomicAdd(count, 1ull);
        if (k < cap) near_list[k] = make_int2(t, s);
    }
}

// ---------------------------------------------------------------- near pairs (recursion)
struct NearFrame {
    double t[9], s[9], kids[36];
    int split_t, next, expanded, pad;
};

__device__ __forceinline__ double tri_diam(const double* t)
{
    const D3 a = {t[0], t[1], t[2]}, b = {t[3], t[4], t[5]}, c = {t[6], t[7], t[8]};
    return fmax(fmax(d3_norm(d3_sub(a, b)), d3_norm(d3_sub(b, c))), d3_norm(d3_sub(a, c)));
}
__device__ __forceinline__ void tri_centroid_rad(const double* t, D3& c, double& r)
{
    const D3 a = {t[0], t[1], t[2]}, b = {t[3], t[4], t[5]}, d = {t[6], t[7], t[8]};
    const D3 s = d3_add(d3_add(a, b), d);
    c = {__ddiv_rn(s.x, 3.0), __ddiv_rn(s.y, 3.0), __ddiv_rn(s.z, 3.0)};
    r = fmax(fmax(fmax(0.0, d3_norm(d3_sub(a, c))), d3_norm(d3_sub(b, c))), d3_norm(d3_sub(d, c)));
}
__device__ __forceinline__ double tri_area(const double* t)
{
    const D3 a = {t[0], t[1], t[2]}, b = {t[3], t[4], t[5]}, c = {t[6], t[7], t[8]};
    return __dmul_rn(0.5, d3_norm(d3_cross(d3_sub(b, a), d3_sub(c, a))));
}
// split4 children {v0,m01,m02},{m01,v1,m12},{m02,m12,v2},{m01,m12,m02} (quadrature.hpp:222-229)
__device__ __forceinline__ void split4(const double* t, double* kids)
{
    double m01[3], m12[3], m02[3];
    for (int c = 0; c < 3; ++c) {
        m01[c] = __dmul_rn(0.5, __dadd_rn(t[c], t[3 + c]));
        m12[c] = __dmul_rn(0.5, __dadd_rn(t[3 + c], t[6 + c]));
        m02[c] = __dmul_rn(0.5, __dadd_rn(t[c], t[6 + c]));
    }
    for (int c = 0; c < 3; ++c) {
        kids[0 * 9 + 0 + c] = t[c];
        kids[0 * 9 + 3 + c] = m01[c];
        kids[0 * 9 + 6 + c] = m02[c];
        kids[1 * 9 + 0 + c] = m01[c];
        kids[1 * 9 + 3 + c] = t[3 + c];
        kids[1 * 9 + 6 + c] = m12[c];
        kids[2 * 9 + 0 + c] = m02[c];
        kids[2 * 9 + 3 + c] = m12[c];
        kids[2 * 9 + 6 + c] = t[6 + c];
        kids[3 * 9 + 0 + c] = m01[c];
        kids[3 * 9 + 3 + c] = m12[c];
        kids[3 * 9 + 6 + c] = m02[c];
    }
}

// Evaluate the 36x36 rule on up to two leaves: half-warp h takes leaf h; each
// lane owns a 9x9 block (i in [9*ia, 9*ia+9), j in [9*jb, 9*jb+9)).
__device__ __forceinline__ double near_leaf_eval(const double* leaf /* 2 x 19 */, int nleaves, int lane)
{
    const int h = lane >> 4;
    if (h >= nleaves) return 0.0;
    const double* L = leaf + 19 * h;
    const double* t = L;
    const double* s = L + 9;
    const double scale = L[18];
    const int l16 = lane & 15, ia = l16 >> 2, jb = l16 & 3;
    const double e1x = s[3] - s[0], e1y = s[4] - s[1], e1z = s[5] - s[2];
    const double e2x = s[6] - s[0], e2y = s[7] - s[1], e2z = s[8] - s[2];
    double yx[9], yy[9], yz[9], wj[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) {
        const int j = 9 * jb + q;
        const double u = c_near_u[j], v = c_near_v[j];
        yx[q] = fma(v, e2x, fma(u, e1x, s[0]));
        yy[q] = fma(v, e2y, fma(u, e1y, s[1]));
        yz[q] = fma(v, e2z, fma(u, e1z, s[2]));
        wj[q] = c_near_w[j];
    }
    const double f1x = t[3] - t[0], f1y = t[4] - t[1], f1z = t[5] - t[2];
    const double f2x = t[6] - t[0], f2y = t[7] - t[1], f2z = t[8] - t[2];
    double acc = 0.0;
#pragma unroll 1
    for (int p = 0; p < 9; ++p) {
        const int i = 9 * ia + p;
        const double u = c_near_u[i], v = c_near_v[i];
        const double xx = fma(v, f2x, fma(u, f1x, t[0]));
        const double xy = fma(v, f2y, fma(u, f1y, t[1]));
        const double xz = fma(v, f2z, fma(u, f1z, t[2]));
        double in = 0.0;
#pragma unroll
        for (int q = 0; q < 9; ++q) {
            const double dx = xx - yx[q], dy = xy - yy[q], dz = xz - yz[q];
            in = fma(wj[q], rsqrt_fast(fma(dx, dx, fma(dy, dy, dz * dz))), in);
        }
        acc = fma(c_near_w[i], in, acc);
    }
    return acc * scale;
}

// One warp per near pair (dynamic scheduling).  The recursion of
// triangle_pair_disjoint (quadrature.hpp:231-249) is walked iteratively with a
// per-warp frame stack in shared memory; all lanes take the same branches.
__global__ void __launch_bounds__(NEAR_WARPS * 32)
    k_near_pairs(const int2* __restrict__ pairs, long long npairs, const double* __restrict__ GV, double thr,
                 double* __restrict__ out, unsigned long long* __restrict__ next, double inv_pi,
                 unsigned long long* __restrict__ leaf_count)
{
    __shared__ NearFrame frames[NEAR_WARPS][6];
    __shared__ double leafbuf[NEAR_WARPS][2 * 19];
    __shared__ long long cur[NEAR_WARPS];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    NearFrame* F = frames[warp];
    double* LB = leafbuf[warp];
    unsigned long long leaves_total = 0;
    while (true) {
        if (lane == 0) cur[warp] = (long long)atomicAdd(next, 1ull);
        __syncwarp();
        const long long pi = cur[warp];
        if (pi >= npairs) break;
        const int2 pr = pairs[pi];  // (t, s) = (larger index, smaller index)
        if (lane == 0) {
            for (int k = 0; k < 9; ++k) {
                F[0].t[k] = GV[9 * pr.x + k];
                F[0].s[k] = GV[9 * pr.y + k];
            }
            F[0].expanded = 0;
        }
        __syncwarp();
        int depth = 0, nleaf = 0;
        double acc = 0.0;
        while (depth >= 0) {
            NearFrame& fr = F[depth];
            if (!fr.expanded) {
                const double dt = tri_diam(fr.t), ds = tri_diam(fr.s);
                D3 ct, cs;
                double rt, rs;
                tri_centroid_rad(fr.t, ct, rt);
                tri_centroid_rad(fr.s, cs, rs);
                const double dist = fmax(0.0, __dsub_rn(__dsub_rn(d3_norm(d3_sub(ct, cs)), rt), rs));
                const bool leaf = dist >= __dmul_rn(thr, fmax(dt, ds)) || depth >= 5;
                if (leaf) {
                    const double sc = __dmul_rn(tri_area(fr.t), tri_area(fr.s));
                    if (lane == 0) {
                        for (int k = 0; k < 9; ++k) {
                            LB[19 * nleaf + k] = fr.t[k];
                            LB[19 * nleaf + 9 + k] = fr.s[k];
                        }
                        LB[19 * nleaf + 18] = sc;
                    }
                    __syncwarp();
                    ++nleaf;
                    ++leaves_total;
                    if (nleaf == 2) {
                        acc += near_leaf_eval(LB, 2, lane);
                        nleaf = 0;
                        __syncwarp();
                    }
                    --depth;
                    continue;
                }
                const int split_t = dt >= ds ? 1 : 0;
                if (lane == 0) {
                    split4(split_t ? fr.t : fr.s, fr.kids);
                    fr.split_t = split_t;
                    fr.next = 0;
                    fr.expanded = 1;
                }
                __syncwarp();
            }
            if (fr.next == 4) {
                --depth;
                continue;
            }
            const int k = fr.next;
            __syncwarp();
            if (lane == 0) {
                fr.next = k + 1;
                NearFrame& ch = F[depth + 1];
                for (int q = 0; q < 9; ++q) {
                    ch.t[q] = fr.split_t ? fr.kids[9 * k + q] : fr.t[q];
                    ch.s[q] = fr.split_t ? fr.s[q] : fr.kids[9 * k + q];
                }
                ch.expanded = 0;
            }
            __syncwarp();
            ++depth;
        }
        if (nleaf) acc += near_leaf_eval(LB, nleaf, lane);
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) out[pi] = acc * inv_pi;
        __syncwarp();
    }
    if (leaf_count && lane == 0) atomicAdd(leaf_count, leaves_total);
}

// ---------------------------------------------------------------- Sauter (singular) pairs
// pairs: 6 ints per pair = permuted vertex ids of t then s (quadrature.hpp:297-322)
__global__ void __launch_bounds__(SAUTER_THREADS)
    k_sauter_partial(const int* __restrict__ pv, int npairs, const double* __restrict__ X,
                     const double* __restrict__ rule, int npts, int chunk, double* __restrict__ part)
{
    __shared__ double R[SAUTER_STAGE * 5];
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    const bool active = p < npairs;
    double d0x = 0, d0y = 0, d0z = 0, e1x = 0, e1y = 0, e1z = 0, e2x = 0, e2y = 0, e2z = 0;
    double g1x = 0, g1y = 0, g1z = 0, g2x = 0, g2y = 0, g2z = 0;
    if (active) {
        const int* q = pv + 6 * p;
        const double* t0 = X + 3 * q[0];
        const double* t1 = X + 3 * q[1];
        const double* t2 = X + 3 * q[2];
        const double* s0 = X + 3 * q[3];
        const double* s1 = X + 3 * q[4];
        const double* s2 = X + 3 * q[5];
        d0x = t0[0] - s0[0];
        d0y = t0[1] - s0[1];
        d0z = t0[2] - s0[2];
        e1x = t1[0] - t0[0];
        e1y = t1[1] - t0[1];
        e1z = t1[2] - t0[2];
        e2x = t2[0] - t0[0];
        e2y = t2[1] - t0[1];
        e2z = t2[2] - t0[2];
        g1x = s1[0] - s0[0];
        g1y = s1[1] - s0[1];
        g1z = s1[2] - s0[2];
        g2x = s2[0] - s0[0];
        g2y = s2[1] - s0[1];
        g2z = s2[2] - s0[2];
    }
    const int q0 = blockIdx.y * chunk, q1 = min(npts, q0 + chunk);
    double acc0 = 0.0, acc1 = 0.0;
    for (int base = q0; base < q1; base += SAUTER_STAGE) {
        const int cnt = min(SAUTER_STAGE, q1 - base);
        __syncthreads();
        for (int e = threadIdx.x; e < cnt * 5; e += blockDim.x) R[e] = rule[(size_t)base * 5 + e];
        __syncthreads();
        if (active) {
            int i = 0;
            for (; i + 2 <= cnt; i += 2) {
                const double* a = R + 5 * i;
                const double* b = a + 5;
                // x - y = (t0 - s0) + a1 e1t + a2 e2t - b1 e1s - b2 e2s
                const double ax = fma(-a[3], g2x, fma(-a[2], g1x, fma(a[1], e2x, fma(a[0], e1x, d0x))));
                const double ay = fma(-a[3], g2y, fma(-a[2], g1y, fma(a[1], e2y, fma(a[0], e1y, d0y))));
                const double az = fma(-a[3], g2z, fma(-a[2], g1z, fma(a[1], e2z, fma(a[0], e1z, d0z))));
                const double bx = fma(-b[3], g2x, fma(-b[2], g1x, fma(b[1], e2x, fma(b[0], e1x, d0x))));
                const double by = fma(-b[3], g2y, fma(-b[2], g1y, fma(b[1], e2y, fma(b[0], e1y, d0y))));
                const double bz = fma(-b[3], g2z, fma(-b[2], g1z, fma(b[1], e2z, fma(b[0], e1z, d0z))));
                acc0 = fma(a[4], rsqrt_fast(fma(ax, ax, fma(ay, ay, az * az))), acc0);
                acc1 = fma(b[4], rsqrt_fast(fma(bx, bx, fma(by, by, bz * bz))), acc1);
            }
            for (; i < cnt; ++i) {
                const double* a = R + 5 * i;
                const double ax = fma(-a[3], g2x, fma(-a[2], g1x, fma(a[1], e2x, fma(a[0], e1x, d0x))));
                const double ay = fma(-a[3], g2y, fma(-a[2], g1y, fma(a[1], e2y, fma(a[0], e1y, d0y))));
                const double az = fma(-a[3], g2z, fma(-a[2], g1z, fma(a[1], e2z, fma(a[0], e1z, d0z))));
                acc0 = fma(a[4], rsqrt_fast(fma(ax, ax, fma(ay, ay, az * az))), acc0);
            }
        }
    }
    if (active) part[(size_t)blockIdx.y * npairs + p] = acc0 + acc1;
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
__global__ void k_local_scatter(const int2* __restrict__ pairs, const double* __restrict__ I, long long np,
                                const int* __restrict__ uptr, const int* __restrict__ udof,
                                const double* __restrict__ uval, double* __restrict__ W, int ld)
{
    const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= np) return;
    const int f = pairs[k].x, g = pairs[k].y;
    const double val = I[k];
    for (int p = uptr[f]; p < uptr[f + 1]; ++p) {
        const int da = udof[p];
        const double ax = uval[3 * p], ay = uval[3 * p + 1], az = uval[3 * p + 2];
        for (int q = uptr[g]; q < uptr[g + 1]; ++q) {
            const int db = udof[q];
            const double v = val * fma(ax, uval[3 * q], fma(ay, uval[3 * q + 1], az * uval[3 * q + 2]));
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
__global__ void k_mirror(double* __restrict__ W, int n, int ld)
{
    __shared__ double tile[32][33];
    const int bi = blockIdx.y, bj = blockIdx.x;  // source tile (bi, bj), bi <= bj
    if (bi > bj) return;
    const int tx = threadIdx.x, ty = threadIdx.y;
    for (int r = ty; r < 32; r += blockDim.y) {
        const int i = bi * 32 + r, j = bj * 32 + tx;
        tile[r][tx] = (i < n && j < n) ? W[(size_t)i * ld + j] : 0.0;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += blockDim.y) {
        const int i = bj * 32 + r, j = bi * 32 + tx;  // destination (lower) element (i, j) = source (j, i)
        if (i < n && j < n && i > j) W[(size_t)i * ld + j] = tile[tx][r];
    }
}

// ---------------------------------------------------------------- RHS (assemble.hpp:143-184)
__global__ void k_rhs(int nf, const double* __restrict__ GV, const double* __restrict__ onormal,
                      const double* __restrict__ g, int g_is_field, const int* __restrict__ sptr,
                      const int* __restrict__ sdof, const double* __restrict__ ssgn, double* __restrict__ L)
{
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nf * NF) return;
    const int f = e / NF, i = e % NF;
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

void upload_rules(Ctx* ctx, const QuadCfg& cfg)
{
    if (cfg.far_order != 4)
        throw ValidationError("the GPU assembly path is specialised for far_order 4 (the reference default)");
    const TriangleRule far = triangle_rule(4), nr = triangle_rule(6);
    cudaStream_t s = ctx->stream;
    SBG_CUDA(cudaMemcpyToSymbolAsync(c_far_u, far.u.data(), NF * sizeof(double), 0, cudaMemcpyHostToDevice, s));
    SBG_CUDA(cudaMemcpyToSymbolAsync(c_far_v, far.v.data(), NF * sizeof(double), 0, cudaMemcpyHostToDevice, s));
    SBG_CUDA(cudaMemcpyToSymbolAsync(c_far_w, far.w.data(), NF * sizeof(double), 0, cudaMemcpyHostToDevice, s));
    SBG_CUDA(cudaMemcpyToSymbolAsync(c_near_u, nr.u.data(), NN * sizeof(double), 0, cudaMemcpyHostToDevice, s));
    SBG_CUDA(cudaMemcpyToSymbolAsync(c_near_v, nr.v.data(), NN * sizeof(double), 0, cudaMemcpyHostToDevice, s));
    SBG_CUDA(cudaMemcpyToSymbolAsync(c_near_w, nr.w.data(), NN * sizeof(double), 0, cudaMemcpyHostToDevice, s));
}

struct DeviceGeometry {
    DBuf<double> X, v, c, rad, diam, area;
    DBuf<int> F, vid;
    GeoPtrs ptrs() const { return {v.p, c.p, rad.p, diam.p, area.p, vid.p}; }
};

void upload_geometry(Ctx* ctx, const SurfaceMesh& m, DeviceGeometry& G)
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
    G.X.upload(X, s);
    G.F.upload(F, s);
    G.v.alloc(9 * (size_t)nf);
    G.c.alloc(3 * (size_t)nf);
    G.rad.alloc(nf);
    G.diam.alloc(nf);
    G.area.alloc(nf);
    G.vid.alloc(3 * (size_t)nf);
    if (nf)
        k_facet_geometry<<<(nf + 127) / 128, 128, 0, s>>>(G.X.p, G.F.p, nf, G.v.p, G.c.p, G.rad.p, G.diam.p, G.area.p,
                                                          G.vid.p);
    SBG_LAUNCH_CHECK();
}

// singular pairs grouped by class, t = larger facet index, permuted vertex ids
struct SingularLists {
    std::vector<int> pv[4];        // by shared count (1..3)
    std::vector<int2> pairs[4];    // (t, s)
};

void singular_pairs(const SurfaceMesh& m, SingularLists& S)
{
    const int nf = m.num_facets(), nv = m.num_vertices();
    std::vector<std::vector<int>> star(nv);
    for (int f = 0; f < nf; ++f)
        for (int k = 0; k < 3; ++k) star[m.facets[f][k]].push_back(f);
    std::vector<int> nb;
    for (int f = 0; f < nf; ++f) {
        nb.clear();
        for (int k = 0; k < 3; ++k)
            for (int g : star[m.facets[f][k]])
                if (g <= f) nb.push_back(g);
        std::sort(nb.begin(), nb.end());
        nb.erase(std::unique(nb.begin(), nb.end()), nb.end());
        for (int g : nb) {
            // permutation of pair_integral (quadrature.hpp:297-322): t = facet f (larger index)
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
            for (int k = 0; k < 3; ++k) S.pv[shared].push_back(m.facets[f][pf[k]]);
            for (int k = 0; k < 3; ++k) S.pv[shared].push_back(m.facets[g][pg[k]]);
            S.pairs[shared].push_back(make_int2(f, g));
        }
    }
}

struct SauterRulesDev {
    DBuf<double> r[4];
    int npts[4] = {0, 0, 0, 0};
};

void upload_sauter(Ctx* ctx, const QuadCfg& cfg, SauterRulesDev& R)
{
    SauterRule id, ed, vx;
    sauter_rules(cfg.singular_order + 2, id, ed, vx);
    R.r[3].upload(id.pts, ctx->stream);
    R.npts[3] = id.size();
    R.r[2].upload(ed.pts, ctx->stream);
    R.npts[2] = ed.size();
    R.r[1].upload(vx.pts, ctx->stream);
    R.npts[1] = vx.size();
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
    const int pblocks = (np + SAUTER_THREADS - 1) / SAUTER_THREADS;
    // enough CTAs for ~4 waves; chunks of rule points in multiples of the stage size
    int nchunks = std::max(1, std::min((4 * ctx->sm_count + pblocks - 1) / pblocks, (npts + 999) / 1000));
    const int chunk = (npts + nchunks - 1) / nchunks;
    nchunks = (npts + chunk - 1) / chunk;
    DBuf<double> part((size_t)nchunks * np);
    {
        TimedScope ts(ctx, "sauter");
        k_sauter_partial<<<dim3(pblocks, nchunks), SAUTER_THREADS, 0, s>>>(d_pv.p, np, X.p, R.r[cls].p, npts, chunk,
                                                                          part.p);
        k_sauter_finish<<<(np + 127) / 128, 128, 0, s>>>(part.p, np, nchunks, d_pv.p, X.p, out_dev);
        SBG_LAUNCH_CHECK();
    }
    SBG_CUDA(cudaStreamSynchronize(s));
}

void run_near(Ctx* ctx, const DBuf<double>& GV, const int2* pairs, long long np, double thr, double* out_dev,
              long long* leaves)
{
    if (np == 0) return;
    cudaStream_t s = ctx->stream;
    DBuf<unsigned long long> ctr(2);
    SBG_CUDA(cudaMemsetAsync(ctr.p, 0, 2 * sizeof(unsigned long long), s));
    const int grid = std::min<long long>((np + NEAR_WARPS - 1) / NEAR_WARPS, 4LL * ctx->sm_count);
    {
        TimedScope ts(ctx, "near");
        k_near_pairs<<<grid, NEAR_WARPS * 32, 0, s>>>(pairs, np, GV.p, thr, out_dev, ctr.p, 1.0 / M_PI, ctr.p + 1);
        SBG_LAUNCH_CHECK();
    }
    if (leaves) {
        unsigned long long h = 0;
        SBG_CUDA(cudaMemcpyAsync(&h, ctr.p + 1, sizeof(h), cudaMemcpyDeviceToHost, s));
        SBG_CUDA(cudaStreamSynchronize(s));
        *leaves = (long long)h;
    }
}

}  // namespace

// reference: inc/assemble.hpp:72-139
void assemble_W(Ctx* ctx, const InflatedMesh& im, const QuadCfg& cfg, DMatrix& W, AssemblyStats* stats)
{
    cudaStream_t s = ctx->stream;
    const SurfaceMesh& m = im.base;
    const int nf = m.num_facets(), n = im.num_jump_dofs();
    matrix_alloc(ctx, n, W);
    if (nf == 0 || n == 0) return;
    upload_rules(ctx, cfg);
    DeviceGeometry G;
    upload_geometry(ctx, m, G);
    const double thr = cfg.near_threshold;

    // curl lists (per facet CSR) for the per-pair scatter
    const FacetCurls U = facet_curls(im);
    DBuf<int> d_uptr, d_udof;
    DBuf<double> d_uval;
    d_uptr.upload(U.ptr, s);
    d_udof.upload(U.dof, s);
    d_uval.upload(U.u, s);

    // ---- Morton-ordered facet blocks
    std::vector<int> perm(nf);
    {
        double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
        std::vector<Vec3> c(nf);
        for (int f = 0; f < nf; ++f) {
            c[f] = m.facet_centroid(f);
            const double xyz[3] = {c[f].x, c[f].y, c[f].z};
            for (int d = 0; d < 3; ++d) {
                lo[d] = std::min(lo[d], xyz[d]);
                hi[d] = std::max(hi[d], xyz[d]);
            }
        }
        const double span = std::max({hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2], 1e-300});
        std::vector<std::uint64_t> key(nf);
        for (int f = 0; f < nf; ++f) {
            const double xyz[3] = {c[f].x, c[f].y, c[f].z};
            std::uint64_t q[3];
            for (int d = 0; d < 3; ++d) q[d] = (std::uint64_t)((xyz[d] - lo[d]) / span * 2097151.0);
            key[f] = spread3(q[0]) | (spread3(q[1]) << 1) | (spread3(q[2]) << 2);
        }
        std::iota(perm.begin(), perm.end(), 0);
        std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) { return key[a] < key[b]; });
    }
    const int nblk = (nf + BS - 1) / BS;
    std::vector<int> bfac((size_t)nblk * BS, -1);
    for (int k = 0; k < nf; ++k) bfac[k] = perm[k];
    // per-block dof lists and per-dof entry lists (facet_local, U)
    std::vector<int> dof_ptr{0}, dofs, ent_ptr;
    std::vector<double4> ents;
    std::vector<double> bcx(nblk), bcy(nblk), bcz(nblk), brad(nblk);
    double rmax = 0, dmax = 0;
    for (int f = 0; f < nf; ++f) {
        rmax = std::max(rmax, [&] {
            const Vec3 cc = m.facet_centroid(f);
            double r = 0;
            for (int k = 0; k < 3; ++k) r = std::max(r, norm(m.vertices[m.facets[f][k]] - cc));
            return r;
        }());
        dmax = std::max(dmax, m.facet_diameter(f));
    }
    int max_dofs = 0;
    struct DE {
        int dof, l, p;
    };
    std::vector<DE> dl;
    for (int b = 0; b < nblk; ++b) {
        dl.clear();
        Vec3 cs;
        int cnt = 0;
        for (int l = 0; l < BS; ++l) {
            const int f = bfac[b * BS + l];
            if (f < 0) continue;
            cs = cs + m.facet_centroid(f);
            ++cnt;
            for (int p = U.ptr[f]; p < U.ptr[f + 1]; ++p) dl.push_back({U.dof[p], l, p});
        }
        const Vec3 cc = cs / (double)cnt;
        double R = 0;
        for (int l = 0; l < BS; ++l) {
            const int f = bfac[b * BS + l];
            if (f >= 0) R = std::max(R, norm(m.facet_centroid(f) - cc));
        }
        bcx[b] = cc.x;
        bcy[b] = cc.y;
        bcz[b] = cc.z;
        brad[b] = R;
        std::sort(dl.begin(), dl.end(), [](const DE& x, const DE& y) { return x.dof != y.dof ? x.dof < y.dof : x.l < y.l; });
        int nd = 0;
        for (size_t i = 0; i < dl.size(); ++i) {
            if (i == 0 || dl[i].dof != dl[i - 1].dof) {
                dofs.push_back(dl[i].dof);
                ent_ptr.push_back((int)ents.size());
                ++nd;
            }
            const int p = dl[i].p;
            ents.push_back(make_double4(U.u[3 * p], U.u[3 * p + 1], U.u[3 * p + 2], (double)dl[i].l));
        }
        dof_ptr.push_back((int)dofs.size());
        max_dofs = std::max(max_dofs, nd);
    }
    ent_ptr.push_back((int)ents.size());
    // ---- tiles (fb >= gb); certainly-far tiles skip per-pair classification
    std::vector<TileInfo> tiles, cand;
    tiles.reserve((size_t)nblk * (nblk + 1) / 2);
    const double margin = 1e-9 * std::max(1.0, dmax);
    for (int fb = 0; fb < nblk; ++fb)
        for (int gb = 0; gb <= fb; ++gb) {
            const double dx = bcx[fb] - bcx[gb], dy = bcy[fb] - bcy[gb], dz = bcz[fb] - bcz[gb];
            const double D = std::sqrt(dx * dx + dy * dy + dz * dz);
            // any pair: dist_estimate >= D - R_f - R_g - 2 rmax >= thr * dmax (and no shared vertex)
            const double lower = D - brad[fb] - brad[gb] - 2.0 * rmax;
            const bool certain = fb != gb && lower > margin && lower >= std::max(0.0, thr) * dmax * (1.0 + 1e-9) + margin;
            tiles.push_back({fb, gb, certain ? 1 : 0, 0});
            if (!certain) cand.push_back({fb, gb, 0, 0});
        }
    DBuf<int> d_bfac, d_dof_ptr, d_dofs, d_ent_ptr;
    DBuf<double4> d_ents;
    d_bfac.upload(bfac, s);
    d_dof_ptr.upload(dof_ptr, s);
    d_dofs.upload(dofs, s);
    d_ent_ptr.upload(ent_ptr, s);
    d_ents.upload(ents, s);
    BlockPtrs BP{d_bfac.p, d_dof_ptr.p, d_dofs.p, d_ent_ptr.p, d_ents.p};
    // dof_ptr indexes ent_ptr by global block-dof position: ent_ptr has one entry per block-dof + 1
    DBuf<TileInfo> d_tiles, d_cand;
    d_tiles.upload(tiles, s);
    d_cand.upload(cand, s);

    // ---- near list
    unsigned long long cap = std::max<unsigned long long>(1024, 64ULL * nf);
    DBuf<int2> d_near;
    DBuf<unsigned long long> d_cnt(1);
    unsigned long long nnear = 0;
    for (int attempt = 0; attempt < 2; ++attempt) {
        d_near.alloc(cap);
        SBG_CUDA(cudaMemsetAsync(d_cnt.p, 0, sizeof(unsigned long long), s));
        if (!cand.empty()) {
            TimedScope ts(ctx, "classify");
            k_classify_near<<<(int)cand.size(), 256, 0, s>>>(d_cand.p, G.ptrs(), d_bfac.p, thr, d_near.p, cap, d_cnt.p);
            SBG_LAUNCH_CHECK();
        }
        SBG_CUDA(cudaMemcpyAsync(&nnear, d_cnt.p, sizeof(nnear), cudaMemcpyDeviceToHost, s));
        SBG_CUDA(cudaStreamSynchronize(s));
        if (nnear <= cap) break;
        cap = nnear;
    }

    // ---- singular lists (host adjacency, deterministic order)
    SingularLists S;
    singular_pairs(m, S);
    SauterRulesDev SR;
    upload_sauter(ctx, cfg, SR);

    // local pairs: [vertex | edge | identical | near] with their integrals
    const long long nloc_sing = (long long)S.pairs[1].size() + S.pairs[2].size() + S.pairs[3].size();
    const long long nloc = nloc_sing + (long long)nnear;
    DBuf<int2> d_loc_pairs(std::max<long long>(nloc, 1));
    DBuf<double> d_loc_I(std::max<long long>(nloc, 1));
    long long off = 0;
    for (int cls = 1; cls <= 3; ++cls) {
        const long long np = (long long)S.pairs[cls].size();
        if (!np) continue;
        SBG_CUDA(cudaMemcpyAsync(d_loc_pairs.p + off, S.pairs[cls].data(), np * sizeof(int2), cudaMemcpyHostToDevice, s));
        run_sauter(ctx, G.X, S.pv[cls], SR, cls, d_loc_I.p + off);
        off += np;
    }
    if (nnear) {
        SBG_CUDA(cudaMemcpyAsync(d_loc_pairs.p + off, d_near.p, nnear * sizeof(int2), cudaMemcpyDeviceToDevice, s));
        long long leaves = 0;
        run_near(ctx, G.v, d_loc_pairs.p + off, (long long)nnear, thr, d_loc_I.p + off, stats ? &leaves : nullptr);
        if (stats) stats->near_leaves = leaves;
    }
    // ---- far tiles
    {
        TimedScope ts(ctx, "far_tiles");
        k_far_tiles<<<(int)tiles.size(), FAR_THREADS, 0, s>>>(d_tiles.p, G.ptrs(), BP, thr, W.a.p, W.ld, 1.0 / M_PI);
        SBG_LAUNCH_CHECK();
    }
    // ---- per-pair scatter of near + singular integrals
    if (nloc) {
        TimedScope ts(ctx, "local_scatter");
        k_local_scatter<<<(int)((nloc + 127) / 128), 128, 0, s>>>(d_loc_pairs.p, d_loc_I.p, nloc, d_uptr.p, d_udof.p,
                                                                  d_uval.p, W.a.p, W.ld);
        SBG_LAUNCH_CHECK();
    }
    {
        TimedScope ts(ctx, "mirror");
        const int nt = (n + 31) / 32;
        k_mirror<<<dim3(nt, nt), dim3(32, 8), 0, s>>>(W.a.p, n, W.ld);
        SBG_LAUNCH_CHECK();
    }
    SBG_CUDA(cudaStreamSynchronize(s));
    (void)max_dofs;
    if (stats) {
        stats->identical = (long long)S.pairs[3].size();
        stats->edge = (long long)S.pairs[2].size();
        stats->vertex = (long long)S.pairs[1].size();
        stats->near_pairs = (long long)nnear;
        stats->far_pairs = (long long)nf * (nf + 1) / 2 - nloc;
        stats->tiles = (long long)tiles.size();
        stats->tiles_skipped = (long long)(tiles.size() - cand.size());
    }
}

namespace {
__global__ void k_far_pair_list(GeoPtrs G, const int2* __restrict__ pairs, long long np, double* __restrict__ out,
                                double inv_pi)
{
    const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= np) return;
    const int f = pairs[k].x, g = pairs[k].y;
    double t[9];
    for (int q = 0; q < 9; ++q) t[q] = G.v[9 * f + q];
    FarPts P;
    far_points(t, P);
    out[k] = far_sum(P, G.v + 9 * g) * G.area[f] * G.area[g] * inv_pi;
}
void far_pair_list(Ctx* ctx, const GeoPtrs& G, const int2* pairs, long long np, double* out)
{
    k_far_pair_list<<<(int)((np + 127) / 128), 128, 0, ctx->stream>>>(G, pairs, np, out, 1.0 / M_PI);
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
    upload_rules(ctx, cfg);
    DeviceGeometry G;
    upload_geometry(ctx, m, G);
    SauterRulesDev SR;
    upload_sauter(ctx, cfg, SR);
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
        run_near(ctx, G.v, d_p.p, (long long)nearp.size(), cfg.near_threshold, o.p, nullptr);
        fetch(o.p, idx[0]);
    }
    if (!farp.empty()) {
        // far pairs through the tile kernel's evaluation: a dedicated 1-facet
        // block layout so each pair is its own (fb, gb) tile is wasteful; use the
        // same device functions on a pair list instead.
        DBuf<int2> d_p;
        d_p.upload(farp, s);
        DBuf<double> o(farp.size());
        far_pair_list(ctx, G.ptrs(), d_p.p, (long long)farp.size(), o.p);
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
    const size_t ng = g_is_field ? (size_t)nf * NF * 3 : 3;
    for (size_t i = 0; i < ng; ++i)
        if (!std::isfinite(g[i])) throw NumericalError("g returned a non-finite value");
    upload_rules(ctx, cfg);
    DeviceGeometry G;
    upload_geometry(ctx, m, G);
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
        k_rhs<<<(nf * NF + 127) / 128, 128, 0, s>>>(nf, G.v.p, d_on.p, d_g.p, g_is_field ? 1 : 0, d_sptr.p, d_sdof.p,
                                                    d_ssgn.p, d_L.p);
    SBG_LAUNCH_CHECK();
    if (n) SBG_CUDA(cudaMemcpyAsync(L_host, d_L.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    SBG_CUDA(cudaStreamSynchronize(s));
}

}  // namespace sbg
