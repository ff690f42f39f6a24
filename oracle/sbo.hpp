// ============================================================================
// screenbem ORACLE — CPU restatement of the reference hot path.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py may load this code, and only
// as the checker (never as the thing measured as the product or shipped).
//
// The reference (`/root/reference/proj/include/screenbem/*.hpp`) cannot be
// compiled here: Eigen 3 is absent.  This file restates each
// reference function without Eigen, keeping the reference's loop order and
// expression order so results are reproducible; every function cites the
// reference file:line it follows.  Eigen's own rounding (e.g. the summation
// order inside Vector3d::norm) is parity-unpinned; this oracle fixes
// |v|^2 = (x*x + y*y) + z*z, a.b = (ax*bx + ay*by) + az*bz and those orders are
// the bitwise contract the GPU classification code mirrors.
//
// Parity pins (tests/test_oracle_*.py): curl KAT, RHS KATs, production pair
// integrals vs the adaptive quad_oracle (1e-6), W entries vs the brute-force
// basis assembly (1e-6), singular-order stability (1e-8), worker-reorder
// bound (1e-13 max|W|), Schwarz/PCG properties and the recorded bow-tie
// condition numbers of proj/test_output.txt:31 (kappa_prec 6.93,
// kappa_unprec 12.96 at 465 DOFs).
//
// Compiled like the reference: -O3, C++20, no -march (proj/CMakeLists.txt:8-10,24),
// plus -ffp-contract=off so no FMA contraction can appear.
// ============================================================================
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <functional>
#include <map>
#include <numeric>
#include <set>
#include <stdexcept>
#include <string>
#include <thread>
#include <chrono>
#include <vector>

namespace sbo {

// ---------------------------------------------------------------- common.hpp
// reference: inc/common.hpp:16-26
struct ValidationError : std::runtime_error {
    explicit ValidationError(const std::string& m) : std::runtime_error(m) {}
};
struct NumericalError : std::runtime_error {
    explicit NumericalError(const std::string& m) : std::runtime_error(m) {}
};

// reference: inc/common.hpp:31-59 (contiguous chunks, worker-ordered merge)
inline void run_partitioned(std::int64_t n, int workers,
                            const std::function<void(int, std::int64_t, std::int64_t)>& body)
{
    if (workers < 1) workers = 1;
    if (n <= 0) return;
    if (workers == 1 || n < 2 * workers) {
        body(0, 0, n);
        return;
    }
    std::vector<std::thread> pool;
    std::vector<std::exception_ptr> errors(workers);
    const std::int64_t chunk = (n + workers - 1) / workers;
    for (int w = 0; w < workers; ++w) {
        const std::int64_t b = std::min<std::int64_t>(w * chunk, n);
        const std::int64_t e = std::min<std::int64_t>(b + chunk, n);
        if (b >= e) break;
        pool.emplace_back([=, &body, &errors] {
            try {
                body(w, b, e);
            } catch (...) {
                errors[w] = std::current_exception();
            }
        });
    }
    for (auto& t : pool) t.join();
    for (auto& err : errors)
        if (err) std::rethrow_exception(err);
}

// ---------------------------------------------------------------- Vec3
struct Vec3 {
    double x = 0, y = 0, z = 0;
    Vec3() = default;
    Vec3(double a, double b, double c) : x(a), y(b), z(c) {}
    double operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
};
inline Vec3 operator+(const Vec3& a, const Vec3& b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline Vec3 operator-(const Vec3& a, const Vec3& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline Vec3 operator-(const Vec3& a) { return {-a.x, -a.y, -a.z}; }
inline Vec3 operator*(double s, const Vec3& a) { return {s * a.x, s * a.y, s * a.z}; }
inline Vec3 operator/(const Vec3& a, double s) { return {a.x / s, a.y / s, a.z / s}; }
inline double dot(const Vec3& a, const Vec3& b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
inline double sqnorm(const Vec3& a) { return (a.x * a.x + a.y * a.y) + a.z * a.z; }
inline double norm(const Vec3& a) { return std::sqrt(sqnorm(a)); }
inline Vec3 cross(const Vec3& a, const Vec3& b)
{
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
inline Vec3 normalized(const Vec3& a)
{
    const double z = sqnorm(a);
    if (z > 0) return a / std::sqrt(z);
    return a;
}
using Tri = std::array<Vec3, 3>;

// ---------------------------------------------------------------- mesh.hpp
// reference: inc/mesh.hpp:19-92 (3-D triangles only: the 2-D segment paths are
// out of scope, SURVEY.md §2.1 "Pair quadrature")
struct SurfaceMesh {
    int dim = 3;
    std::vector<Vec3> vertices;
    std::vector<std::array<int, 3>> facets;

    int num_vertices() const { return (int)vertices.size(); }
    int num_facets() const { return (int)facets.size(); }
    Vec3 facet_centroid(int f) const
    {
        Vec3 c;
        for (int k = 0; k < 3; ++k) c = c + vertices[facets[f][k]];
        return c / 3.0;
    }
    double facet_diameter(int f) const
    {
        double d = 0;
        for (int a = 0; a < 3; ++a)
            for (int b = a + 1; b < 3; ++b)
                d = std::max(d, norm(vertices[facets[f][a]] - vertices[facets[f][b]]));
        return d;
    }
    double facet_measure(int f) const  // mesh.hpp:45-50
    {
        const auto& t = facets[f];
        return 0.5 * norm(cross(vertices[t[1]] - vertices[t[0]], vertices[t[2]] - vertices[t[0]]));
    }
    Vec3 facet_normal(int f) const  // mesh.hpp:54-62
    {
        const auto& t = facets[f];
        return normalized(cross(vertices[t[1]] - vertices[t[0]], vertices[t[2]] - vertices[t[0]]));
    }
    double max_facet_diameter() const
    {
        double h = 0;
        for (int f = 0; f < num_facets(); ++f) h = std::max(h, facet_diameter(f));
        return h;
    }
    double diameter() const  // mesh.hpp:71-79
    {
        Vec3 lo(1e300, 1e300, 1e300), hi(-1e300, -1e300, -1e300);
        for (const auto& p : vertices) {
            lo = {std::min(lo.x, p.x), std::min(lo.y, p.y), std::min(lo.z, p.z)};
            hi = {std::max(hi.x, p.x), std::max(hi.y, p.y), std::max(hi.z, p.z)};
        }
        return norm(hi - lo);
    }
};

struct MeshLevelPair {  // mesh.hpp:86-92
    SurfaceMesh coarse, fine;
    std::vector<int> parent;
    double H = 0, h = 0;
};

namespace detail {
inline double point_segment_distance(const Vec3& x, const Vec3& a, const Vec3& b)  // mesh.hpp:96-101
{
    const Vec3 d = b - a;
    const double t = std::clamp(dot(x - a, d) / sqnorm(d), 0.0, 1.0);
    return norm(x - (a + t * d));
}
inline double point_triangle_distance(const Vec3& x, const Vec3& a, const Vec3& b, const Vec3& c)
{  // mesh.hpp:103-117
    const Vec3 ab = b - a, ac = c - a;
    const Vec3 n = cross(ab, ac);
    const double nn = sqnorm(n);
    const Vec3 ax = x - a;
    const double u = dot(cross(ax, ac), n) / nn;
    const double v = dot(cross(ab, ax), n) / nn;
    if (u >= 0 && v >= 0 && u + v <= 1.0) return std::abs(dot(ax, n)) / std::sqrt(nn);
    return std::min({point_segment_distance(x, a, b), point_segment_distance(x, b, c),
                     point_segment_distance(x, a, c)});
}
inline bool segment_hits_triangle(const Vec3& a, const Vec3& b, const Vec3& t0, const Vec3& t1,
                                  const Vec3& t2, double eps)  // mesh.hpp:183-194
{
    const Vec3 n = cross(t1 - t0, t2 - t0);
    const double da = dot(n, a - t0), db = dot(n, b - t0);
    if ((da > eps && db > eps) || (da < -eps && db < -eps)) return false;
    if (std::abs(da - db) < 1e-300) return false;
    const double s = da / (da - db);
    if (s < -eps || s > 1 + eps) return false;
    const Vec3 p = a + s * (b - a);
    return point_triangle_distance(p, t0, t1, t2) < eps;
}
inline bool triangles_conforming(const SurfaceMesh& m, int f, int g, double eps)  // mesh.hpp:196-234
{
    const auto& a = m.facets[f];
    const auto& b = m.facets[g];
    std::set<int> sa(a.begin(), a.end()), sb(b.begin(), b.end());
    std::vector<int> shared;
    std::set_intersection(sa.begin(), sa.end(), sb.begin(), sb.end(), std::back_inserter(shared));
    const Vec3 A0 = m.vertices[a[0]], A1 = m.vertices[a[1]], A2 = m.vertices[a[2]];
    const Vec3 B0 = m.vertices[b[0]], B1 = m.vertices[b[1]], B2 = m.vertices[b[2]];
    for (int v : a)
        if (!sb.count(v) && point_triangle_distance(m.vertices[v], B0, B1, B2) < eps) return false;
    for (int v : b)
        if (!sa.count(v) && point_triangle_distance(m.vertices[v], A0, A1, A2) < eps) return false;
    const int eidx[3][2] = {{0, 1}, {1, 2}, {2, 0}};
    for (const auto& e : eidx) {
        const int u = a[e[0]], v = a[e[1]];
        if (sb.count(u) || sb.count(v)) continue;
        if (segment_hits_triangle(m.vertices[u], m.vertices[v], B0, B1, B2, eps)) return false;
    }
    for (const auto& e : eidx) {
        const int u = b[e[0]], v = b[e[1]];
        if (sa.count(u) || sa.count(v)) continue;
        if (segment_hits_triangle(m.vertices[u], m.vertices[v], A0, A1, A2, eps)) return false;
    }
    if (shared.size() >= 1) {
        const Vec3 n1 = normalized(cross(A1 - A0, A2 - A0));
        const Vec3 n2 = normalized(cross(B1 - B0, B2 - B0));
        if (std::abs(std::abs(dot(n1, n2)) - 1.0) < 1e-12 && std::abs(dot(n1, B0 - A0)) < eps) {
            const Vec3 ca = ((A0 + A1) + A2) / 3.0, cb = ((B0 + B1) + B2) / 3.0;
            if (point_triangle_distance(ca, B0, B1, B2) < eps ||
                point_triangle_distance(cb, A0, A1, A2) < eps)
                return false;
        }
    }
    return true;
}
}  // namespace detail

// reference: inc/mesh.hpp:238-272 (O(nf^2) pair loop, bounding-sphere reject)
inline void validate_mesh(const SurfaceMesh& m)
{
    if (m.dim != 3) throw ValidationError("oracle restates the 3-D path only");
    const int nv = m.num_vertices();
    for (const auto& p : m.vertices)
        if (!std::isfinite(p.x) || !std::isfinite(p.y) || !std::isfinite(p.z))
            throw ValidationError("non-finite vertex coordinate");
    const double eps = 1e-12 * std::max(m.diameter(), 1e-300);
    std::set<std::array<int, 3>> seen;
    for (int f = 0; f < m.num_facets(); ++f) {
        std::array<int, 3> t = m.facets[f];
        for (int k = 0; k < 3; ++k)
            if (t[k] < 0 || t[k] >= nv) throw ValidationError("facet vertex id out of range");
        std::array<int, 3> key = t;
        std::sort(key.begin(), key.end());
        if (!seen.insert(key).second) throw ValidationError("duplicate facet");
        const double scale = eps * std::max(m.facet_diameter(f), eps);
        if (m.facet_measure(f) < scale) throw ValidationError("degenerate facet " + std::to_string(f));
    }
    for (int f = 0; f < m.num_facets(); ++f)
        for (int g = f + 1; g < m.num_facets(); ++g) {
            const double rr = 0.5 * (m.facet_diameter(f) + m.facet_diameter(g)) + eps;
            if (norm(m.facet_centroid(f) - m.facet_centroid(g)) > rr) continue;
            if (!detail::triangles_conforming(m, f, g, eps))
                throw ValidationError("non-conforming facet pair " + std::to_string(f) + "," +
                                      std::to_string(g));
        }
}

// reference: inc/mesh.hpp:322-337
inline SurfaceMesh make_bowtie_base()
{
    const double mlen = std::sqrt(3.0) / 2.0;
    SurfaceMesh m;
    m.vertices = {Vec3(0, 0, 0),     Vec3(0, 0, mlen), Vec3(0.5, 0, mlen),
                  Vec3(-0.5, 0, mlen), Vec3(0, 0.5, mlen), Vec3(0, -0.5, mlen)};
    m.facets = {{0, 2, 1}, {0, 1, 3}, {0, 4, 1}, {0, 1, 5}};
    return m;
}

// reference: inc/mesh.hpp:342-386 (3-D branch)
inline MeshLevelPair refine_uniform(const SurfaceMesh& mesh)
{
    MeshLevelPair pair;
    pair.coarse = mesh;
    SurfaceMesh& fine = pair.fine;
    fine.vertices = mesh.vertices;
    std::map<std::array<int, 2>, int> edge_mid;
    auto midpoint = [&](int a, int b) {
        std::array<int, 2> key = {std::min(a, b), std::max(a, b)};
        auto it = edge_mid.find(key);
        if (it != edge_mid.end()) return it->second;
        fine.vertices.push_back(0.5 * (mesh.vertices[a] + mesh.vertices[b]));
        const int id = fine.num_vertices() - 1;
        edge_mid.emplace(key, id);
        return id;
    };
    for (int f = 0; f < mesh.num_facets(); ++f) {
        const auto& t = mesh.facets[f];
        const int m01 = midpoint(t[0], t[1]);
        const int m12 = midpoint(t[1], t[2]);
        const int m02 = midpoint(t[0], t[2]);
        fine.facets.push_back({t[0], m01, m02});
        fine.facets.push_back({m01, t[1], m12});
        fine.facets.push_back({m02, m12, t[2]});
        fine.facets.push_back({m01, m12, m02});
        for (int k = 0; k < 4; ++k) pair.parent.push_back(f);
    }
    pair.H = pair.coarse.max_facet_diameter();
    pair.h = fine.max_facet_diameter();
    return pair;
}

// reference: inc/mesh.hpp:388-405
inline MeshLevelPair refine_uniform_times(const SurfaceMesh& mesh, int k)
{
    MeshLevelPair pair;
    pair.coarse = mesh;
    pair.fine = mesh;
    pair.parent.resize(mesh.num_facets());
    for (int f = 0; f < mesh.num_facets(); ++f) pair.parent[f] = f;
    for (int i = 0; i < k; ++i) {
        MeshLevelPair step = refine_uniform(pair.fine);
        std::vector<int> parent(step.fine.num_facets());
        for (int f = 0; f < step.fine.num_facets(); ++f) parent[f] = pair.parent[step.parent[f]];
        pair.fine = std::move(step.fine);
        pair.parent = std::move(parent);
    }
    pair.H = pair.coarse.max_facet_diameter();
    pair.h = pair.fine.max_facet_diameter();
    return pair;
}

// ---------------------------------------------------------------- gauss.hpp
struct Rule1d {
    std::vector<double> x, w;
};
// reference: inc/gauss.hpp:16-52
inline Rule1d gauss_legendre(int n)
{
    Rule1d r;
    r.x.resize(n);
    r.w.resize(n);
    for (int i = 0; i < (n + 1) / 2; ++i) {
        double t = std::cos(M_PI * (i + 0.75) / (n + 0.5));
        double p0 = 0, p1 = 0;
        for (int it = 0; it < 100; ++it) {
            p0 = 1.0;
            p1 = 0.0;
            for (int k = 0; k < n; ++k) {
                const double p2 = p1;
                p1 = p0;
                p0 = ((2.0 * k + 1.0) * t * p1 - k * p2) / (k + 1.0);
            }
            const double dp = n * (t * p0 - p1) / (t * t - 1.0);
            const double dt = p0 / dp;
            t -= dt;
            if (std::abs(dt) < 1e-15) break;
        }
        p0 = 1.0;
        p1 = 0.0;
        for (int k = 0; k < n; ++k) {
            const double p2 = p1;
            p1 = p0;
            p0 = ((2.0 * k + 1.0) * t * p1 - k * p2) / (k + 1.0);
        }
        const double dp = n * (t * p0 - p1) / (t * t - 1.0);
        const double w = 2.0 / ((1.0 - t * t) * dp * dp);
        r.x[i] = 0.5 * (1.0 - t);
        r.w[i] = 0.5 * w;
        r.x[n - 1 - i] = 0.5 * (1.0 + t);
        r.w[n - 1 - i] = 0.5 * w;
    }
    return r;
}

struct TriangleRule {
    std::vector<double> u, v, w;
    int size() const { return (int)w.size(); }
};
// reference: inc/gauss.hpp:56-76
inline TriangleRule triangle_rule(int order)
{
    const Rule1d g = gauss_legendre(order);
    TriangleRule r;
    for (int i = 0; i < order; ++i)
        for (int j = 0; j < order; ++j) {
            r.u.push_back(g.x[i]);
            r.v.push_back(g.x[j] * (1.0 - g.x[i]));
            r.w.push_back(g.w[i] * g.w[j] * (1.0 - g.x[i]));
        }
    return r;
}

// ---------------------------------------------------------------- quadrature.hpp
struct QuadratureConfig {  // quadrature.hpp:12-16
    int far_order = 4;
    int singular_order = 8;
    double near_threshold = 2.0;
};
struct PairRulePoint {  // quadrature.hpp:28-30
    double a1, a2, b1, b2, w;
};
// reference: inc/quadrature.hpp:35-92 (point order: i0,i1,i2,i3 then subdomain)
struct SauterRules {
    std::vector<PairRulePoint> identical, edge, vertex;
    explicit SauterRules(int order)
    {
        const Rule1d g = gauss_legendre(order);
        auto push = [](std::vector<PairRulePoint>& out, double x1, double x2, double y1, double y2,
                       double w) { out.push_back({x1 - x2, x2, y1 - y2, y2, w}); };
        for (int i0 = 0; i0 < order; ++i0)
            for (int i1 = 0; i1 < order; ++i1)
                for (int i2 = 0; i2 < order; ++i2)
                    for (int i3 = 0; i3 < order; ++i3) {
                        const double xi = g.x[i0], e1 = g.x[i1], e2 = g.x[i2], e3 = g.x[i3];
                        const double wp = g.w[i0] * g.w[i1] * g.w[i2] * g.w[i3];
                        const double xi3 = xi * xi * xi;
                        {
                            const double w = wp * xi3 * e1 * e1 * e2;
                            push(identical, xi, xi * (1 - e1 + e1 * e2), xi * (1 - e1 * e2 * e3),
                                 xi * (1 - e1), w);
                            push(identical, xi * (1 - e1 * e2 * e3), xi * (1 - e1), xi,
                                 xi * (1 - e1 + e1 * e2), w);
                            push(identical, xi, xi * e1 * (1 - e2 + e2 * e3), xi * (1 - e1 * e2),
                                 xi * e1 * (1 - e2), w);
                            push(identical, xi * (1 - e1 * e2), xi * e1 * (1 - e2), xi,
                                 xi * e1 * (1 - e2 + e2 * e3), w);
                            push(identical, xi * (1 - e1 * e2 * e3), xi * e1 * (1 - e2 * e3), xi,
                                 xi * e1 * (1 - e2), w);
                            push(identical, xi, xi * e1 * (1 - e2), xi * (1 - e1 * e2 * e3),
                                 xi * e1 * (1 - e2 * e3), w);
                        }
                        {
                            const double w1 = wp * xi3 * e1 * e1;
                            const double w2 = wp * xi3 * e1 * e1 * e2;
                            push(edge, xi, xi * e1 * e3, xi * (1 - e1 * e2), xi * e1 * (1 - e2), w1);
                            push(edge, xi, xi * e1, xi * (1 - e1 * e2 * e3), xi * e1 * e2 * (1 - e3),
                                 w2);
                            push(edge, xi * (1 - e1 * e2), xi * e1 * (1 - e2), xi, xi * e1 * e2 * e3,
                                 w2);
                            push(edge, xi * (1 - e1 * e2 * e3), xi * e1 * e2 * (1 - e3), xi, xi * e1,
                                 w2);
                            push(edge, xi * (1 - e1 * e2 * e3), xi * e1 * (1 - e2 * e3), xi,
                                 xi * e1 * e2, w2);
                        }
                        {
                            const double w = wp * xi3 * e2;
                            push(vertex, xi, xi * e1, xi * e2, xi * e2 * e3, w);
                            push(vertex, xi * e2, xi * e2 * e3, xi, xi * e1, w);
                        }
                    }
    }
};

// reference: inc/quadrature.hpp:95-114 (2-D segment rules dropped)
struct QuadratureEngine {
    QuadratureConfig cfg;
    SauterRules sauter;
    TriangleRule tri_far, tri_near;
    explicit QuadratureEngine(const QuadratureConfig& c)
        : cfg(c), sauter(c.singular_order + 2), tri_far(triangle_rule(c.far_order)),
          tri_near(triangle_rule(c.far_order + 2))
    {
    }
};

namespace detail {
// reference: inc/quadrature.hpp:19-23 (dim 3)
inline double kernel3(double r) { return 1.0 / (4.0 * M_PI * r); }

// reference: inc/quadrature.hpp:186-196
inline double triangle_pair_distance_estimate(const Tri& t, const Tri& s)
{
    const Vec3 ct = ((t[0] + t[1]) + t[2]) / 3.0, cs = ((s[0] + s[1]) + s[2]) / 3.0;
    double rt = 0, rs = 0;
    for (int k = 0; k < 3; ++k) {
        rt = std::max(rt, norm(t[k] - ct));
        rs = std::max(rs, norm(s[k] - cs));
    }
    return std::max(0.0, norm(ct - cs) - rt - rs);
}
// reference: inc/quadrature.hpp:198-201
inline double triangle_diameter(const Tri& t)
{
    return std::max({norm(t[0] - t[1]), norm(t[1] - t[2]), norm(t[0] - t[2])});
}
// reference: inc/quadrature.hpp:203-206
inline double triangle_area(const Tri& t) { return 0.5 * norm(cross(t[1] - t[0], t[2] - t[0])); }

// affine map t0 + u (t1 - t0) + v (t2 - t0), per component in that order
inline Vec3 affine(const Tri& t, double u, double v)
{
    return {(t[0].x + u * (t[1].x - t[0].x)) + v * (t[2].x - t[0].x),
            (t[0].y + u * (t[1].y - t[0].y)) + v * (t[2].y - t[0].y),
            (t[0].z + u * (t[1].z - t[0].z)) + v * (t[2].z - t[0].z)};
}

// reference: inc/quadrature.hpp:208-220
inline double triangle_pair_rule(const Tri& t, const Tri& s, const TriangleRule& r)
{
    double acc = 0;
    for (int i = 0; i < r.size(); ++i) {
        const Vec3 x = affine(t, r.u[i], r.v[i]);
        for (int j = 0; j < r.size(); ++j) {
            const Vec3 y = affine(s, r.u[j], r.v[j]);
            acc += r.w[i] * r.w[j] * kernel3(norm(x - y));
        }
    }
    return acc * 4.0 * triangle_area(t) * triangle_area(s);
}

// reference: inc/quadrature.hpp:222-229 (child order)
inline void split4(const Tri& t, Tri out[4])
{
    const Vec3 m01 = 0.5 * (t[0] + t[1]), m12 = 0.5 * (t[1] + t[2]), m02 = 0.5 * (t[0] + t[2]);
    out[0] = {t[0], m01, m02};
    out[1] = {m01, t[1], m12};
    out[2] = {m02, m12, t[2]};
    out[3] = {m01, m12, m02};
}

// Work counters for the probe / roofline bookkeeping (not part of the reference).
struct QuadStats {
    std::int64_t far_leaves = 0, near_leaves = 0, sauter_points = 0;
};

// reference: inc/quadrature.hpp:231-249
inline double triangle_pair_disjoint(const Tri& t, const Tri& s, const QuadratureEngine& eng,
                                     int depth, QuadStats* st = nullptr)
{
    const double diam = std::max(triangle_diameter(t), triangle_diameter(s));
    const double dist = triangle_pair_distance_estimate(t, s);
    if (dist >= eng.cfg.near_threshold * diam || depth >= 5) {
        if (st) (depth == 0 ? st->far_leaves : st->near_leaves)++;
        return triangle_pair_rule(t, s, depth == 0 ? eng.tri_far : eng.tri_near);
    }
    Tri kids[4];
    double acc = 0;
    if (triangle_diameter(t) >= triangle_diameter(s)) {
        split4(t, kids);
        for (int k = 0; k < 4; ++k) acc += triangle_pair_disjoint(kids[k], s, eng, depth + 1, st);
    } else {
        split4(s, kids);
        for (int k = 0; k < 4; ++k) acc += triangle_pair_disjoint(t, kids[k], eng, depth + 1, st);
    }
    return acc;
}

// reference: inc/quadrature.hpp:251-262
inline double triangle_pair_sauter(const Tri& t, const Tri& s, const std::vector<PairRulePoint>& rule)
{
    const double scale = 4.0 * triangle_area(t) * triangle_area(s);
    double acc = 0;
    for (const auto& p : rule) {
        const Vec3 x = affine(t, p.a1, p.a2);
        const Vec3 y = affine(s, p.b1, p.b2);
        acc += p.w / norm(x - y);
    }
    return acc * scale / (4.0 * M_PI);
}
}  // namespace detail

// Adjacency class of a facet pair: number of shared vertices (0..3), plus the
// permuted vertex slots (reference: inc/quadrature.hpp:297-322).
inline int pair_permutation(const SurfaceMesh& m, int f, int g, std::array<int, 3>& pf,
                            std::array<int, 3>& pg)
{
    pf = {-1, -1, -1};
    pg = {-1, -1, -1};
    int shared = 0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            if (m.facets[f][i] == m.facets[g][j]) {
                pf[shared] = i;
                pg[shared] = j;
                ++shared;
                break;
            }
    auto fill_rest = [](std::array<int, 3>& p, int have) {
        for (int k = 0; k < 3; ++k) {
            bool used = false;
            for (int q = 0; q < have; ++q) used |= (p[q] == k);
            if (!used) p[have++] = k;
        }
    };
    fill_rest(pf, shared);
    fill_rest(pg, shared);
    return shared;
}

// reference: inc/quadrature.hpp:268-334 (3-D dispatch)
inline double pair_integral(const SurfaceMesh& m, int f, int g, const QuadratureEngine& eng,
                            detail::QuadStats* st = nullptr)
{
    std::array<int, 3> pf, pg;
    const int shared = pair_permutation(m, f, g, pf, pg);
    Tri t, s;
    for (int k = 0; k < 3; ++k) {
        t[k] = m.vertices[m.facets[f][pf[k]]];
        s[k] = m.vertices[m.facets[g][pg[k]]];
    }
    switch (shared) {
        case 3:
            if (st) st->sauter_points += (std::int64_t)eng.sauter.identical.size();
            return detail::triangle_pair_sauter(t, s, eng.sauter.identical);
        case 2:
            if (st) st->sauter_points += (std::int64_t)eng.sauter.edge.size();
            return detail::triangle_pair_sauter(t, s, eng.sauter.edge);
        case 1:
            if (st) st->sauter_points += (std::int64_t)eng.sauter.vertex.size();
            return detail::triangle_pair_sauter(t, s, eng.sauter.vertex);
        default:
            return detail::triangle_pair_disjoint(t, s, eng, 0, st);
    }
}

// ---------------------------------------------------------------- quad_oracle.hpp
// Brute-force adaptive pair integral (reference: inc/quad_oracle.hpp:15-141), 3-D.
namespace quad_oracle {
inline double triangle_inverse_distance_integral(const Tri& tri, const Vec3& x)  // :15-42
{
    const Vec3 n = normalized(cross(tri[1] - tri[0], tri[2] - tri[0]));
    const double h = dot(x - tri[0], n);
    const Vec3 rho = x - h * n;
    const double scale = detail::triangle_diameter(tri);
    double acc = 0;
    for (int i = 0; i < 3; ++i) {
        const Vec3 a = tri[i], b = tri[(i + 1) % 3];
        const Vec3 s = normalized(b - a);
        const Vec3 mm = cross(s, n);
        const double t = dot(a - rho, mm);
        const double lm = dot(a - rho, s);
        const double lp = dot(b - rho, s);
        const double r0sq = t * t + h * h;
        const double rm = std::sqrt(lm * lm + r0sq);
        const double rp = std::sqrt(lp * lp + r0sq);
        if (r0sq > 1e-28 * scale * scale) {
            acc += t * std::log((rp + lp) / (rm + lm));
            acc -= std::abs(h) * (std::atan2(t * lp, r0sq + std::abs(h) * rp) -
                                  std::atan2(t * lm, r0sq + std::abs(h) * rm));
        }
    }
    return acc;
}
inline double inner_kernel_integral(const SurfaceMesh& m, int g, const Vec3& x)  // :64-73
{
    const Tri tri = {m.vertices[m.facets[g][0]], m.vertices[m.facets[g][1]], m.vertices[m.facets[g][2]]};
    return triangle_inverse_distance_integral(tri, x) / (4.0 * M_PI);
}
inline double outer_rule_tri(const SurfaceMesh& m, int g, const Tri& t)  // :76-85
{
    static const TriangleRule r = triangle_rule(3);
    double acc = 0;
    for (int i = 0; i < r.size(); ++i) acc += r.w[i] * inner_kernel_integral(m, g, detail::affine(t, r.u[i], r.v[i]));
    return acc * 2.0 * detail::triangle_area(t);
}
inline double adapt_tri(const SurfaceMesh& m, int g, const Tri& t, double coarse, double tol, int depth)
{  // :96-111
    Tri kids[4];
    detail::split4(t, kids);
    double fine = 0;
    std::array<double, 4> kv;
    for (int k = 0; k < 4; ++k) {
        kv[k] = outer_rule_tri(m, g, kids[k]);
        fine += kv[k];
    }
    if (std::abs(fine - coarse) <= tol || depth >= 26) return fine;
    double acc = 0;
    for (int k = 0; k < 4; ++k) acc += adapt_tri(m, g, kids[k], kv[k], 0.5 * tol, depth + 1);
    return acc;
}
inline double pair_integral(const SurfaceMesh& m, int f, int g, double rel_tol = 1e-9)  // :128-141
{
    const Tri t = {m.vertices[m.facets[f][0]], m.vertices[m.facets[f][1]], m.vertices[m.facets[f][2]]};
    const double rough = outer_rule_tri(m, g, t);
    const double tol = rel_tol * std::max(std::abs(rough), 1e-12);
    return adapt_tri(m, g, t, rough, tol, 0);
}
}  // namespace quad_oracle

// ---------------------------------------------------------------- inflate.hpp
struct OrientedFacet {  // inflate.hpp:19-23
    int facet = -1, side = 0;
    Vec3 normal;
};
struct EdgeFan {  // inflate.hpp:27-39
    std::array<int, 2> edge = {-1, -1};
    std::vector<std::array<int, 2>> pairs;
};
struct GeneralizedVertex {  // inflate.hpp:42-46
    int vertex = -1, branch = -1;
    std::vector<int> alpha;
};
struct InflatedMesh {  // inflate.hpp:48-76
    SurfaceMesh base;
    std::vector<OrientedFacet> oriented_facets;
    std::vector<EdgeFan> fans;
    std::vector<GeneralizedVertex> gvertices;
    std::vector<int> q;
    std::vector<std::array<int, 2>> jump_dofs;
    std::vector<int> gv_first, dof_first;
    std::vector<std::array<int, 3>> ofacet_branch;
    std::vector<std::vector<int>> vertex_fans;

    int num_oriented() const { return (int)oriented_facets.size(); }
    int num_gvertices() const { return (int)gvertices.size(); }
    int num_jump_dofs() const { return (int)jump_dofs.size(); }
    int gv_index(int v, int b) const { return gv_first[v] + b; }
    int dof_index(int v, int b) const
    {
        if (q[v] < 2 || b >= q[v] - 1) return -1;
        return dof_first[v] + b;
    }
    int branch_at(int o, int k) const { return ofacet_branch[o][k]; }
};

namespace detail {
struct DisjointSet {  // inflate.hpp:80-89
    std::vector<int> parent;
    explicit DisjointSet(int n) : parent(n) { std::iota(parent.begin(), parent.end(), 0); }
    int find(int a)
    {
        while (parent[a] != a) a = parent[a] = parent[parent[a]];
        return a;
    }
    void unite(int a, int b) { parent[find(a)] = find(b); }
};
struct FanSlot {
    int local;
    double angle;
};
}  // namespace detail

// reference: inc/inflate.hpp:98-288 (3-D)
inline InflatedMesh inflate(const SurfaceMesh& mesh, bool validate = true)
{
    if (validate) validate_mesh(mesh);
    InflatedMesh im;
    im.base = mesh;
    const int nf = mesh.num_facets(), nv = mesh.num_vertices();
    im.oriented_facets.resize(2 * nf);
    for (int f = 0; f < nf; ++f) {
        const Vec3 n = mesh.facet_normal(f);
        im.oriented_facets[2 * f + 0] = {f, 0, n};
        im.oriented_facets[2 * f + 1] = {f, 1, -n};
    }
    std::map<std::array<int, 2>, std::vector<int>> edge_facets;
    for (int f = 0; f < nf; ++f) {
        const auto& t = mesh.facets[f];
        for (int k = 0; k < 3; ++k) {
            const int a = t[k], b = t[(k + 1) % 3];
            edge_facets[{std::min(a, b), std::max(a, b)}].push_back(f);
        }
    }
    {  // point-contact check, inflate.hpp:129-151 (O(V*E) as in the reference)
        std::vector<std::vector<int>> vstar(nv);
        for (int f = 0; f < nf; ++f)
            for (int k = 0; k < 3; ++k) vstar[mesh.facets[f][k]].push_back(f);
        for (int v = 0; v < nv; ++v) {
            const auto& star = vstar[v];
            if (star.size() < 2) continue;
            std::map<int, int> local;
            for (int i = 0; i < (int)star.size(); ++i) local[star[i]] = i;
            detail::DisjointSet ds((int)star.size());
            for (const auto& [edge, fl] : edge_facets) {
                if (edge[0] != v && edge[1] != v) continue;
                for (size_t i = 1; i < fl.size(); ++i) ds.unite(local[fl[0]], local[fl[i]]);
            }
            const int root = ds.find(0);
            for (int i = 1; i < (int)star.size(); ++i)
                if (ds.find(i) != root)
                    throw ValidationError("point contact at vertex " + std::to_string(v) +
                                          " (unsupported geometry)");
        }
    }
    im.vertex_fans.resize(nv);
    for (const auto& [edge, facets] : edge_facets) {  // inflate.hpp:155-228
        EdgeFan fan;
        fan.edge = edge;
        const Vec3 origin = mesh.vertices[edge[0]];
        const Vec3 e_dir = normalized(mesh.vertices[edge[1]] - mesh.vertices[edge[0]]);
        auto in_plane_dir = [&](int f) {
            const auto& t = mesh.facets[f];
            int opp = -1;
            for (int k = 0; k < 3; ++k)
                if (t[k] != edge[0] && t[k] != edge[1]) opp = t[k];
            Vec3 d = mesh.vertices[opp] - origin;
            d = d - dot(d, e_dir) * e_dir;
            return normalized(d);
        };
        const Vec3 ref = in_plane_dir(facets[0]);
        const Vec3 up = cross(e_dir, ref);
        std::vector<detail::FanSlot> slots;
        for (int i = 0; i < (int)facets.size(); ++i) {
            const Vec3 d = in_plane_dir(facets[i]);
            slots.push_back({i, std::atan2(dot(d, up), dot(d, ref))});
        }
        std::sort(slots.begin(), slots.end(),
                  [](const detail::FanSlot& a, const detail::FanSlot& b) { return a.angle < b.angle; });
        const int k = (int)slots.size();
        for (int i = 0; i + 1 < k; ++i)
            if (slots[i + 1].angle - slots[i].angle < 1e-9)
                throw ValidationError("coplanar facets overlap at an edge fan (angular tie)");
        if (k > 1 && slots[0].angle + 2.0 * M_PI - slots[k - 1].angle < 1e-9)
            throw ValidationError("coplanar facets overlap at an edge fan (angular tie)");
        auto ccw_side = [&](int f) {
            const Vec3 d = in_plane_dir(f);
            const Vec3 tangent = cross(e_dir, d);
            return (dot(im.oriented_facets[2 * f].normal, tangent) > 0) ? 0 : 1;
        };
        for (int i = 0; i < k; ++i) {
            const int fa = facets[slots[i].local];
            const int fb = facets[slots[(i + 1) % k].local];
            fan.pairs.push_back({2 * fa + (1 - ccw_side(fa)), 2 * fb + ccw_side(fb)});
        }
        const int fan_id = (int)im.fans.size();
        im.fans.push_back(std::move(fan));
        im.vertex_fans[edge[0]].push_back(fan_id);
        im.vertex_fans[edge[1]].push_back(fan_id);
    }
    std::vector<std::vector<int>> vstar_of(nv);  // inflate.hpp:232-279
    for (int f = 0; f < nf; ++f)
        for (int k = 0; k < 3; ++k) {
            vstar_of[mesh.facets[f][k]].push_back(2 * f);
            vstar_of[mesh.facets[f][k]].push_back(2 * f + 1);
        }
    im.q.assign(nv, 0);
    im.gv_first.assign(nv, -1);
    im.dof_first.assign(nv, -1);
    im.ofacet_branch.assign(2 * nf, {-1, -1, -1});
    for (int v = 0; v < nv; ++v) {
        const auto& star = vstar_of[v];
        if (star.empty()) throw ValidationError("isolated vertex " + std::to_string(v));
        std::map<int, int> local;
        for (int i = 0; i < (int)star.size(); ++i) local[star[i]] = i;
        detail::DisjointSet ds((int)star.size());
        for (int fan_id : im.vertex_fans[v])
            for (const auto& p : im.fans[fan_id].pairs) ds.unite(local[p[0]], local[p[1]]);
        std::map<int, std::vector<int>> comp;
        for (int i = 0; i < (int)star.size(); ++i) comp[ds.find(i)].push_back(star[i]);
        std::vector<std::vector<int>> branches;
        for (auto& [root, members] : comp) {
            std::sort(members.begin(), members.end());
            branches.push_back(std::move(members));
        }
        std::sort(branches.begin(), branches.end(),
                  [](const auto& a, const auto& b) { return a.front() < b.front(); });
        im.gv_first[v] = im.num_gvertices();
        im.q[v] = (int)branches.size();
        for (int j = 0; j < im.q[v]; ++j) {
            GeneralizedVertex gv;
            gv.vertex = v;
            gv.branch = j;
            gv.alpha = branches[j];
            for (int o : gv.alpha) {
                const int f = o / 2;
                for (int k = 0; k < 3; ++k)
                    if (mesh.facets[f][k] == v) im.ofacet_branch[o][k] = j;
            }
            im.gvertices.push_back(std::move(gv));
        }
    }
    for (int v = 0; v < nv; ++v) {  // inflate.hpp:281-285
        if (im.q[v] < 2) continue;
        im.dof_first[v] = im.num_jump_dofs();
        for (int j = 0; j + 1 < im.q[v]; ++j) im.jump_dofs.push_back({v, j});
    }
    return im;
}

// ---------------------------------------------------------------- jump.hpp
struct TraceField {  // jump.hpp:14-30
    std::vector<double> coeff;
    double at(const InflatedMesh& im, int o, int k) const
    {
        const int f = o / 2;
        const int v = im.base.facets[f][k];
        return coeff[im.gv_index(v, im.branch_at(o, k))];
    }
    double eval(const InflatedMesh& im, int o, double u, double v) const
    {
        return (1.0 - u - v) * at(im, o, 0) + u * at(im, o, 1) + v * at(im, o, 2);
    }
};
inline TraceField basis_trace(const std::array<int, 2>& dof, const InflatedMesh& im)  // jump.hpp:33-43
{
    const int v = dof[0], j = dof[1];
    if (v < 0 || v >= im.base.num_vertices() || im.q[v] < 2 || j < 0 || j >= im.q[v] - 1)
        throw ValidationError("not a jump degree of freedom");
    TraceField tf;
    tf.coeff.assign(im.num_gvertices(), 0.0);
    tf.coeff[im.gv_index(v, j)] = 1.0;
    tf.coeff[im.gv_index(v, im.q[v] - 1)] = -1.0;
    return tf;
}
inline TraceField expand(const std::vector<double>& vec, const InflatedMesh& im)  // jump.hpp:45-57
{
    if ((int)vec.size() != im.num_jump_dofs())
        throw ValidationError("jump vector length does not match the DOF count");
    TraceField tf;
    tf.coeff.assign(im.num_gvertices(), 0.0);
    for (int d = 0; d < im.num_jump_dofs(); ++d) {
        const auto [v, j] = im.jump_dofs[d];
        tf.coeff[im.gv_index(v, j)] += vec[d];
        tf.coeff[im.gv_index(v, im.q[v] - 1)] -= vec[d];
    }
    return tf;
}
inline std::vector<double> jump_coordinates(const TraceField& tf, const InflatedMesh& im)  // jump.hpp:61-74
{
    std::vector<double> v(im.num_jump_dofs(), 0.0);
    for (int i = 0; i < im.base.num_vertices(); ++i) {
        double mean = 0;
        for (int j = 0; j < im.q[i]; ++j) mean += tf.coeff[im.gv_index(i, j)];
        mean /= im.q[i];
        for (int j = 0; j + 1 < im.q[i]; ++j) {
            const int d = im.dof_index(i, j);
            if (d >= 0) v[d] = tf.coeff[im.gv_index(i, j)] - mean;
        }
    }
    return v;
}

// Sparse coarse->fine map in column-major triplet form (jump.hpp:87-89).
struct Prolongation {
    int rows = 0, cols = 0;
    std::vector<int> col_ptr, row_idx;  // CSC, rows ascending within a column
    std::vector<double> val;
};

namespace detail {
// reference: inc/jump.hpp:94-111 (3-D)
inline void barycentric(const SurfaceMesh& m, int f, const Vec3& x, double& u, double& v)
{
    const auto& t = m.facets[f];
    const Vec3 e1 = m.vertices[t[1]] - m.vertices[t[0]];
    const Vec3 e2 = m.vertices[t[2]] - m.vertices[t[0]];
    const Vec3 r = x - m.vertices[t[0]];
    const double a11 = sqnorm(e1), a12 = dot(e1, e2), a22 = sqnorm(e2);
    const double b1 = dot(r, e1), b2 = dot(r, e2);
    const double det = a11 * a22 - a12 * a12;
    u = (a22 * b1 - a12 * b2) / det;
    v = (a11 * b2 - a12 * b1) / det;
}
}  // namespace detail

// reference: inc/jump.hpp:118-185 (O(n_c * n_gv * |alpha|), as in the reference)
inline Prolongation build_prolongation(const MeshLevelPair& pair, const InflatedMesh& coarse,
                                       const InflatedMesh& fine)
{
    const int n_fine = fine.num_jump_dofs(), n_coarse = coarse.num_jump_dofs();
    std::vector<int> oparent(fine.num_oriented(), -1);
    for (int f = 0; f < pair.fine.num_facets(); ++f) {
        const int cf = pair.parent[f];
        if (cf < 0 || cf >= pair.coarse.num_facets())
            throw ValidationError("orphan fine facet " + std::to_string(f) + " (broken nesting)");
        for (int k = 0; k < 3; ++k) {
            double u, v;
            detail::barycentric(pair.coarse, cf, pair.fine.vertices[pair.fine.facets[f][k]], u, v);
            if (u < -1e-9 || v < -1e-9 || u + v > 1 + 1e-9)
                throw ValidationError("fine facet " + std::to_string(f) +
                                      " escapes its parent (broken nesting)");
        }
        for (int s = 0; s < 2; ++s) {
            const double d = dot(fine.oriented_facets[2 * f + s].normal, coarse.oriented_facets[2 * cf].normal);
            if (std::abs(d) < 0.5)
                throw ValidationError("fine facet " + std::to_string(f) + " normal mismatch (broken nesting)");
            oparent[2 * f + s] = 2 * cf + (d > 0 ? 0 : 1);
        }
    }
    Prolongation P;
    P.rows = n_fine;
    P.cols = n_coarse;
    P.col_ptr.push_back(0);
    for (int cd = 0; cd < n_coarse; ++cd) {
        const TraceField cf_field = basis_trace(coarse.jump_dofs[cd], coarse);
        TraceField restricted;
        restricted.coeff.assign(fine.num_gvertices(), 0.0);
        for (int g = 0; g < fine.num_gvertices(); ++g) {
            const auto& gv = fine.gvertices[g];
            const Vec3 x = fine.base.vertices[gv.vertex];
            double value = 0;
            bool first = true;
            for (int o : gv.alpha) {
                const int po = oparent[o];
                double u, v;
                detail::barycentric(pair.coarse, po / 2, x, u, v);
                const double val = cf_field.eval(coarse, po, u, v);
                if (first) {
                    value = val;
                    first = false;
                } else if (std::abs(val - value) > 1e-8 * (1.0 + std::abs(value))) {
                    throw ValidationError("inconsistent coarse branch values across a fine sector "
                                          "(branch structure not refinement-invariant)");
                }
            }
            restricted.coeff[g] = value;
        }
        const std::vector<double> col = jump_coordinates(restricted, fine);
        for (int r = 0; r < n_fine; ++r)
            if (col[r] != 0.0) {
                P.row_idx.push_back(r);
                P.val.push_back(col[r]);
            }
        P.col_ptr.push_back((int)P.row_idx.size());
    }
    return P;
}

// ---------------------------------------------------------------- assemble.hpp
// Dense matrices are row-major n x n (W is symmetric, so layout is moot).
struct Dense {
    int n = 0;
    std::vector<double> a;
    double& operator()(int i, int j) { return a[(size_t)i * n + j]; }
    double operator()(int i, int j) const { return a[(size_t)i * n + j]; }
};

namespace detail {
// reference: inc/assemble.hpp:18-29 (3-D)
inline Vec3 shape_gradient(const SurfaceMesh& m, int f, int k)
{
    const auto& t = m.facets[f];
    const Vec3 n = m.facet_normal(f);
    const Vec3 e = m.vertices[t[(k + 2) % 3]] - m.vertices[t[(k + 1) % 3]];
    return cross(n, e) / (2.0 * m.facet_measure(f));
}
struct Scatter {  // assemble.hpp:34-36
    std::vector<std::pair<int, double>> terms;
};
inline std::vector<Scatter> build_scatter(const InflatedMesh& im)  // assemble.hpp:38-53
{
    std::vector<Scatter> sc(im.num_gvertices());
    for (int g = 0; g < im.num_gvertices(); ++g) {
        const auto& gv = im.gvertices[g];
        const int q = im.q[gv.vertex];
        if (q < 2) continue;
        if (gv.branch < q - 1) {
            sc[g].terms.emplace_back(im.dof_index(gv.vertex, gv.branch), 1.0);
        } else {
            for (int j = 0; j + 1 < q; ++j) sc[g].terms.emplace_back(im.dof_index(gv.vertex, j), -1.0);
        }
    }
    return sc;
}
}  // namespace detail

// reference: inc/assemble.hpp:59-66
inline Vec3 surface_curl(const InflatedMesh& im, int o, const TraceField& tr)
{
    const int f = o / 2;
    Vec3 grad;
    for (int k = 0; k < 3; ++k) grad = grad + tr.at(im, o, k) * detail::shape_gradient(im.base, f, k);
    return cross(im.oriented_facets[o].normal, grad);
}

// reference: inc/assemble.hpp:72-139.  `pair_lo/pair_hi` restrict the pair
// index range (bounded CPU-baseline samples); the default is the full range.
namespace detail {
// Per-pair unrank + integral + scatter of the reference loop body
// (inc/assemble.hpp:97-128), shared by assemble_W and the timing sampler.
struct PairScatter {
    const InflatedMesh& im;
    const QuadratureEngine eng;
    const std::vector<Scatter> scatter;
    std::vector<std::array<Vec3, 3>> slot_curl;
    PairScatter(const InflatedMesh& m, const QuadratureConfig& cfg)
        : im(m), eng(cfg), scatter(build_scatter(m)), slot_curl(m.num_oriented())
    {
        for (int o = 0; o < im.num_oriented(); ++o) {
            const int f = o / 2;
            for (int k = 0; k < 3; ++k)
                slot_curl[o][k] = cross(im.oriented_facets[o].normal, shape_gradient(im.base, f, k));
        }
    }
    // reference: assemble.hpp:98-103 (unrank the (f <= g) pair index)
    static void unrank(std::int64_t idx, int& ff, int& g)
    {
        const int f = (int)((std::sqrt(8.0 * idx + 1.0) - 1.0) / 2.0);
        ff = f;
        while ((std::int64_t)(ff + 1) * (ff + 2) / 2 <= idx) ++ff;
        while ((std::int64_t)ff * (ff + 1) / 2 > idx) --ff;
        g = (int)(idx - (std::int64_t)ff * (ff + 1) / 2);
    }
    void operator()(std::int64_t idx, Dense& W, QuadStats* stats) const
    {
        const SurfaceMesh& m = im.base;
        int ff, g;
        unrank(idx, ff, g);
        const double I = pair_integral(m, ff, g, eng, stats);
        if (!std::isfinite(I)) throw NumericalError("quadrature produced a non-finite pair integral");
        for (int sa = 0; sa < 2; ++sa)
            for (int sb = 0; sb < 2; ++sb) {
                const int oa = 2 * ff + sa, ob = 2 * g + sb;
                for (int ka = 0; ka < 3; ++ka) {
                    const int ga = im.gv_index(m.facets[ff][ka], im.branch_at(oa, ka));
                    if (scatter[ga].terms.empty()) continue;
                    for (int kb = 0; kb < 3; ++kb) {
                        const int gb = im.gv_index(m.facets[g][kb], im.branch_at(ob, kb));
                        if (scatter[gb].terms.empty()) continue;
                        const double c = dot(slot_curl[oa][ka], slot_curl[ob][kb]) * I;
                        for (const auto& [da, wa] : scatter[ga].terms)
                            for (const auto& [db, wb] : scatter[gb].terms) {
                                const double v = c * wa * wb;
                                W(da, db) += v;
                                if (ff != g) W(db, da) += v;
                            }
                    }
                }
            }
    }
};
}  // namespace detail

// reference: inc/assemble.hpp:72-139 (per-worker dense partials over contiguous pair
// ranges, worker-ordered sum, mirror of the upper triangle)
inline Dense assemble_W(const InflatedMesh& im, const QuadratureConfig& cfg, int workers = 1,
                        std::int64_t pair_lo = 0, std::int64_t pair_hi = -1,
                        detail::QuadStats* stats = nullptr)
{
    const int n = im.num_jump_dofs();
    const int nf = im.base.num_facets();
    const detail::PairScatter body(im, cfg);
    const std::int64_t npairs = (std::int64_t)nf * (nf + 1) / 2;
    if (pair_hi < 0 || pair_hi > npairs) pair_hi = npairs;
    if (pair_lo < 0) pair_lo = 0;
    std::vector<Dense> partial(std::max(workers, 1));
    std::vector<detail::QuadStats> wstats(std::max(workers, 1));
    run_partitioned(pair_hi - pair_lo, workers, [&](int w, std::int64_t lo, std::int64_t hi) {
        Dense& W = partial[w];
        W.n = n;
        W.a.assign((size_t)n * n, 0.0);
        for (std::int64_t idx = pair_lo + lo; idx < pair_lo + hi; ++idx) body(idx, W, stats ? &wstats[w] : nullptr);
    });
    Dense W = std::move(partial[0]);
    if (W.a.empty()) {
        W.n = n;
        W.a.assign((size_t)n * n, 0.0);
    }
    for (int w = 1; w < (int)partial.size(); ++w)
        if (!partial[w].a.empty())
            for (size_t i = 0; i < W.a.size(); ++i) W.a[i] += partial[w].a[i];
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j) W(j, i) = W(i, j);
    if (stats)
        for (const auto& s : wstats) {
            stats->far_leaves += s.far_leaves;
            stats->near_leaves += s.near_leaves;
            stats->sauter_points += s.sauter_points;
        }
    return W;
}

// Timing sampler of assemble_W for the CPU baseline (bench.py): the reference's cost
// split into its per-call part and its per-pair part, so a bounded, unbiased sample of
// the pair space gives the full call's time without running it for minutes.
//   fixed():  the per-call work of assemble.hpp:91-137 with no pairs — `workers` dense
//             n x n partials allocated and zeroed in their worker threads, the
//             worker-ordered sum and the mirror;
//   run(idx): the loop body of assemble.hpp:97-128 over a sorted list of pair indices,
//             split into contiguous chunks per worker exactly as run_partitioned splits
//             the full range (common.hpp:31-59), each worker scattering into its own
//             resident dense partial.
// Full-call estimate: fixed + (npairs / k) * run(k sampled pairs).
struct AssemblySampler {
    const InflatedMesh& im;
    detail::PairScatter body;
    int workers;
    std::vector<Dense> partial;
    AssemblySampler(const InflatedMesh& m, const QuadratureConfig& cfg, int w)
        : im(m), body(m, cfg), workers(std::max(w, 1)), partial(workers)
    {
    }
    // the resident partials of run(), allocated on first use outside the timed region
    // (fixed() runs before them, so at most `workers` n x n matrices exist at a time)
    void prepare()
    {
        const int n = im.num_jump_dofs();
        if (!partial[0].a.empty()) return;
        run_partitioned(2 * workers, workers, [&](int k, std::int64_t, std::int64_t) {
            partial[k].n = n;
            partial[k].a.assign((size_t)n * n, 0.0);
        });
    }
    static double now()
    {
        return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
    }
    double fixed() const
    {
        const int n = im.num_jump_dofs();
        const double t0 = now();
        std::vector<Dense> p(workers);
        run_partitioned(2 * workers, workers, [&](int k, std::int64_t, std::int64_t) {
            p[k].n = n;
            p[k].a.assign((size_t)n * n, 0.0);
        });
        Dense W = std::move(p[0]);
        for (int k = 1; k < workers; ++k)
            if (!p[k].a.empty())
                for (size_t i = 0; i < W.a.size(); ++i) W.a[i] += p[k].a[i];
        for (int i = 0; i < n; ++i)
            for (int j = i + 1; j < n; ++j) W(j, i) = W(i, j);
        volatile double sink = W.a.empty() ? 0.0 : W.a[W.a.size() / 2];
        (void)sink;
        return now() - t0;
    }
    double run(const std::int64_t* idx, std::int64_t k)
    {
        prepare();
        const double t0 = now();
        run_partitioned(k, workers, [&](int w, std::int64_t lo, std::int64_t hi) {
            for (std::int64_t i = lo; i < hi; ++i) body(idx[i], partial[w], nullptr);
        });
        return now() - t0;
    }
};

// Selected rows of assemble_W (same per-entry summation order restricted to
// the requested rows; rows-only evaluation of the reference loop at
// assemble.hpp:97-128, used to pin full-size GPU matrices on sampled rows).
// Entries are the upper-triangle values the mirror (assemble.hpp:136-137)
// would leave: row r, column c takes W(min(r,c), max(r,c)).
inline std::vector<double> assemble_W_rows(const InflatedMesh& im, const QuadratureConfig& cfg,
                                           const std::vector<int>& rows, int workers = 1)
{
    const SurfaceMesh& m = im.base;
    const int n = im.num_jump_dofs();
    const int nf = m.num_facets();
    const QuadratureEngine eng(cfg);
    const auto scatter = detail::build_scatter(im);
    std::vector<std::array<Vec3, 3>> slot_curl(im.num_oriented());
    for (int o = 0; o < im.num_oriented(); ++o)
        for (int k = 0; k < 3; ++k)
            slot_curl[o][k] = cross(im.oriented_facets[o].normal, detail::shape_gradient(m, o / 2, k));
    // facets whose scatter touches each requested row
    std::vector<char> touch(nf, 0);
    std::vector<int> rowpos(n, -1);
    for (size_t i = 0; i < rows.size(); ++i) rowpos[rows[i]] = (int)i;
    for (int f = 0; f < nf; ++f)
        for (int s = 0; s < 2; ++s)
            for (int k = 0; k < 3; ++k)
                for (const auto& [d, w] : scatter[im.gv_index(m.facets[f][k], im.branch_at(2 * f + s, k))].terms)
                    if (rowpos[d] >= 0) touch[f] = 1;
    std::vector<int> tf;
    for (int f = 0; f < nf; ++f)
        if (touch[f]) tf.push_back(f);
    // pair list (ff >= g, ascending reference index) with at least one touching facet
    std::vector<std::int64_t> pairs;
    for (int ff = 0; ff < nf; ++ff)
        for (int g = 0; g <= ff; ++g)
            if (touch[ff] || touch[g]) pairs.push_back((std::int64_t)ff * (ff + 1) / 2 + g);
    std::vector<double> Ival(pairs.size());
    run_partitioned((std::int64_t)pairs.size(), workers, [&](int, std::int64_t lo, std::int64_t hi) {
        for (std::int64_t p = lo; p < hi; ++p) {
            const std::int64_t idx = pairs[p];
            int ff = (int)((std::sqrt(8.0 * idx + 1.0) - 1.0) / 2.0);
            while ((std::int64_t)(ff + 1) * (ff + 2) / 2 <= idx) ++ff;
            while ((std::int64_t)ff * (ff + 1) / 2 > idx) --ff;
            const int g = (int)(idx - (std::int64_t)ff * (ff + 1) / 2);
            Ival[p] = pair_integral(m, ff, g, eng);
        }
    });
    // accumulate exactly as the single-worker reference loop into the full
    // matrix restricted to entries (i,j) with i or j in rows
    std::vector<double> full(rows.size() * (size_t)n, 0.0);   // W(row, j)
    std::vector<double> fullT(rows.size() * (size_t)n, 0.0);  // W(j, row)
    for (size_t p = 0; p < pairs.size(); ++p) {
        const std::int64_t idx = pairs[p];
        int ff = (int)((std::sqrt(8.0 * idx + 1.0) - 1.0) / 2.0);
        while ((std::int64_t)(ff + 1) * (ff + 2) / 2 <= idx) ++ff;
        while ((std::int64_t)ff * (ff + 1) / 2 > idx) --ff;
        const int g = (int)(idx - (std::int64_t)ff * (ff + 1) / 2);
        const double I = Ival[p];
        for (int sa = 0; sa < 2; ++sa)
            for (int sb = 0; sb < 2; ++sb) {
                const int oa = 2 * ff + sa, ob = 2 * g + sb;
                for (int ka = 0; ka < 3; ++ka) {
                    const int ga = im.gv_index(m.facets[ff][ka], im.branch_at(oa, ka));
                    if (scatter[ga].terms.empty()) continue;
                    for (int kb = 0; kb < 3; ++kb) {
                        const int gb = im.gv_index(m.facets[g][kb], im.branch_at(ob, kb));
                        if (scatter[gb].terms.empty()) continue;
                        const double c = dot(slot_curl[oa][ka], slot_curl[ob][kb]) * I;
                        for (const auto& [da, wa] : scatter[ga].terms)
                            for (const auto& [db, wb] : scatter[gb].terms) {
                                const double v = c * wa * wb;
                                if (rowpos[da] >= 0) full[rowpos[da] * (size_t)n + db] += v;
                                if (rowpos[db] >= 0) fullT[rowpos[db] * (size_t)n + da] += v;
                                if (ff != g) {
                                    if (rowpos[db] >= 0) full[rowpos[db] * (size_t)n + da] += v;
                                    if (rowpos[da] >= 0) fullT[rowpos[da] * (size_t)n + db] += v;
                                }
                            }
                    }
                }
            }
    }
    std::vector<double> out(rows.size() * (size_t)n);
    for (size_t i = 0; i < rows.size(); ++i)
        for (int c = 0; c < n; ++c)
            out[i * n + c] = (c >= rows[i]) ? full[i * (size_t)n + c] : fullT[i * (size_t)n + c];
    return out;
}

// reference: inc/assemble.hpp:143-184 (3-D); g is given by its values at the
// nf*16 far-rule points (point i of facet f at index f*npt+i), which is what
// the std::function of the reference evaluates.
inline std::vector<Vec3> rhs_points(const InflatedMesh& im, const QuadratureConfig& cfg)
{
    const SurfaceMesh& m = im.base;
    const TriangleRule r = triangle_rule(cfg.far_order);
    std::vector<Vec3> pts;
    for (int f = 0; f < m.num_facets(); ++f) {
        const auto& t = m.facets[f];
        for (int i = 0; i < r.size(); ++i) {
            Vec3 y = m.vertices[t[0]] + r.u[i] * (m.vertices[t[1]] - m.vertices[t[0]]);
            y = y + r.v[i] * (m.vertices[t[2]] - m.vertices[t[0]]);
            pts.push_back(y);
        }
    }
    return pts;
}
inline std::vector<double> assemble_rhs(const InflatedMesh& im, const std::vector<Vec3>& gvals,
                                        const QuadratureConfig& cfg)
{
    const SurfaceMesh& m = im.base;
    const TriangleRule r = triangle_rule(cfg.far_order);
    const auto scatter = detail::build_scatter(im);
    std::vector<double> L(im.num_jump_dofs(), 0.0);
    for (int f = 0; f < m.num_facets(); ++f) {
        const double meas = m.facet_measure(f);
        const auto& t = m.facets[f];
        for (int i = 0; i < r.size(); ++i) {
            const double u = r.u[i], v = r.v[i], w = r.w[i] * 2.0 * meas;
            const Vec3 gy = gvals[(size_t)f * r.size() + i];
            if (!std::isfinite(gy.x) || !std::isfinite(gy.y) || !std::isfinite(gy.z))
                throw NumericalError("g returned a non-finite value");
            for (int s = 0; s < 2; ++s) {
                const int o = 2 * f + s;
                const double dn = dot(gy, im.oriented_facets[o].normal);
                for (int k = 0; k < 3; ++k) {
                    const double lambda = (k == 0) ? (1.0 - u - v) : ((k == 1) ? u : v);
                    const int gv = im.gv_index(t[k], im.branch_at(o, k));
                    for (const auto& [d, sgn] : scatter[gv].terms) L[d] += w * dn * lambda * sgn;
                }
            }
        }
    }
    return L;
}

// ---------------------------------------------------------------- schwarz.hpp
struct DofPartition {  // schwarz.hpp:14-17
    std::map<int, std::vector<int>> face_sets;
    std::vector<int> wirebasket;
};
// reference: inc/schwarz.hpp:19-51
inline DofPartition partition_dofs(const MeshLevelPair& pair, const InflatedMesh& fine)
{
    DofPartition part;
    std::vector<std::set<int>> vertex_parents(pair.fine.num_vertices());
    for (int f = 0; f < pair.fine.num_facets(); ++f) {
        if (pair.parent[f] < 0 || pair.parent[f] >= pair.coarse.num_facets())
            throw ValidationError("fine facet has no coarse parent (nesting violation)");
        for (int k = 0; k < 3; ++k) vertex_parents[pair.fine.facets[f][k]].insert(pair.parent[f]);
    }
    for (int d = 0; d < fine.num_jump_dofs(); ++d) {
        const int v = fine.jump_dofs[d][0];
        const auto& parents = vertex_parents[v];
        if (parents.empty()) throw ValidationError("fine vertex not locatable on the coarse geometry");
        bool interior = false;
        int face = -1;
        if (parents.size() == 1) {
            face = *parents.begin();
            double u, w;
            detail::barycentric(pair.coarse, face, pair.fine.vertices[v], u, w);
            const double tol = 1e-9;
            interior = (u > tol && u + w < 1.0 - tol && w > tol);
        }
        if (interior)
            part.face_sets[face].push_back(d);
        else
            part.wirebasket.push_back(d);
    }
    return part;
}

// Dense Cholesky W = L L^T (lower, row-major), unblocked right-looking.  Eigen's
// blocked LLT (schwarz.hpp:91) rounds differently; parity is to tolerance.
inline bool cholesky(Dense& A)
{
    const int n = A.n;
    for (int j = 0; j < n; ++j) {
        double d = A(j, j);
        for (int k = 0; k < j; ++k) d -= A(j, k) * A(j, k);
        if (!(d > 0) || !std::isfinite(d)) return false;
        d = std::sqrt(d);
        A(j, j) = d;
        for (int i = j + 1; i < n; ++i) {
            double s = A(i, j);
            for (int k = 0; k < j; ++k) s -= A(i, k) * A(j, k);
            A(i, j) = s / d;
        }
    }
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j) A(i, j) = 0.0;
    return true;
}
inline void llt_solve(const Dense& L, std::vector<double>& b)
{
    const int n = L.n;
    for (int i = 0; i < n; ++i) {
        double s = b[i];
        for (int k = 0; k < i; ++k) s -= L(i, k) * b[k];
        b[i] = s / L(i, i);
    }
    for (int i = n - 1; i >= 0; --i) {
        double s = b[i];
        for (int k = i + 1; k < n; ++k) s -= L(k, i) * b[k];
        b[i] = s / L(i, i);
    }
}

struct SchwarzPreconditioner {  // schwarz.hpp:55-73
    struct Block {
        std::vector<int> dofs;
        Dense L;
    };
    std::vector<Block> faces;
    Block wirebasket;
    Prolongation R;
    Dense coarse_L;
    int n = 0;
    int num_subspaces() const
    {
        int c = (int)faces.size();
        if (!wirebasket.dofs.empty()) ++c;
        if (R.cols > 0) ++c;
        return c;
    }
};

namespace detail {
inline SchwarzPreconditioner::Block factor_block(const Dense& W, std::vector<int> idx, const char* what)
{  // schwarz.hpp:77-96
    SchwarzPreconditioner::Block b;
    b.dofs = std::move(idx);
    if (b.dofs.empty()) return b;
    b.L.n = (int)b.dofs.size();
    b.L.a.resize((size_t)b.L.n * b.L.n);
    for (int i = 0; i < b.L.n; ++i)
        for (int j = 0; j < b.L.n; ++j) b.L(i, j) = W(b.dofs[i], b.dofs[j]);
    if (!cholesky(b.L))
        throw NumericalError(std::string("block factorization failed (") + what +
                             "): partition inconsistent with the assembled matrix");
    return b;
}
}  // namespace detail

// Coarse Galerkin matrix R^T W R (schwarz.hpp:110-112 computes it with a
// densified R; here with the sparse columns, same value to rounding).
inline Dense coarse_matrix(const Dense& W, const Prolongation& R)
{
    const int nc = R.cols, n = W.n;
    Dense WR;  // n x nc
    WR.n = 0;
    std::vector<double> wr((size_t)n * nc, 0.0);
    for (int c = 0; c < nc; ++c)
        for (int p = R.col_ptr[c]; p < R.col_ptr[c + 1]; ++p) {
            const int r = R.row_idx[p];
            const double v = R.val[p];
            for (int i = 0; i < n; ++i) wr[(size_t)i * nc + c] += W(i, r) * v;
        }
    Dense H;
    H.n = nc;
    H.a.assign((size_t)nc * nc, 0.0);
    for (int a = 0; a < nc; ++a)
        for (int p = R.col_ptr[a]; p < R.col_ptr[a + 1]; ++p) {
            const int r = R.row_idx[p];
            const double v = R.val[p];
            for (int b = 0; b < nc; ++b) H(a, b) += v * wr[(size_t)r * nc + b];
        }
    return H;
}

// reference: inc/schwarz.hpp:100-118
inline SchwarzPreconditioner build_preconditioner(const Dense& W, const DofPartition& part,
                                                  const Prolongation& P)
{
    SchwarzPreconditioner prec;
    prec.n = W.n;
    for (const auto& [face, dofs] : part.face_sets) prec.faces.push_back(detail::factor_block(W, dofs, "face"));
    prec.wirebasket = detail::factor_block(W, part.wirebasket, "wire-basket");
    prec.R = P;
    if (prec.R.cols > 0) {
        prec.coarse_L = coarse_matrix(W, prec.R);
        if (!cholesky(prec.coarse_L)) throw NumericalError("coarse matrix factorization failed");
    }
    return prec;
}

// reference: inc/schwarz.hpp:121-140 (faces in map order, WB, then coarse)
inline std::vector<double> apply_preconditioner(const SchwarzPreconditioner& prec,
                                                const std::vector<double>& r)
{
    if ((int)r.size() != prec.n) throw ValidationError("preconditioner length mismatch");
    std::vector<double> out(prec.n, 0.0);
    auto add_block = [&](const SchwarzPreconditioner::Block& b) {
        if (b.dofs.empty()) return;
        std::vector<double> local(b.dofs.size());
        for (size_t i = 0; i < b.dofs.size(); ++i) local[i] = r[b.dofs[i]];
        llt_solve(b.L, local);
        for (size_t i = 0; i < b.dofs.size(); ++i) out[b.dofs[i]] += local[i];
    };
    for (const auto& b : prec.faces) add_block(b);
    add_block(prec.wirebasket);
    if (prec.R.cols > 0) {
        std::vector<double> rc(prec.R.cols, 0.0);
        for (int c = 0; c < prec.R.cols; ++c) {
            double s = 0;
            for (int p = prec.R.col_ptr[c]; p < prec.R.col_ptr[c + 1]; ++p) s += prec.R.val[p] * r[prec.R.row_idx[p]];
            rc[c] = s;
        }
        llt_solve(prec.coarse_L, rc);
        std::vector<double> y(prec.n, 0.0);
        for (int c = 0; c < prec.R.cols; ++c)
            for (int p = prec.R.col_ptr[c]; p < prec.R.col_ptr[c + 1]; ++p)
                y[prec.R.row_idx[p]] += prec.R.val[p] * rc[c];
        for (int i = 0; i < prec.n; ++i) out[i] += y[i];
    }
    return out;
}

// ---------------------------------------------------------------- pcg.hpp
// Extreme eigenvalues of a symmetric tridiagonal matrix by Sturm bisection
// (replaces Eigen::SelfAdjointEigenSolver on the Lanczos T, pcg.hpp:109).
inline int sturm_count(const std::vector<double>& d, const std::vector<double>& e, double x)
{
    int cnt = 0;
    double q = 1.0;
    for (size_t i = 0; i < d.size(); ++i) {
        const double e2 = (i == 0) ? 0.0 : e[i - 1] * e[i - 1];
        q = d[i] - x - ((i == 0) ? 0.0 : e2 / q);
        if (q == 0.0) q = -1e-300;
        if (q < 0) ++cnt;
    }
    return cnt;
}
inline void tridiag_extremes(const std::vector<double>& d, const std::vector<double>& e, double& lmin,
                             double& lmax)
{
    const int k = (int)d.size();
    double lo = 1e300, hi = -1e300;
    for (int i = 0; i < k; ++i) {
        const double r = (i > 0 ? std::abs(e[i - 1]) : 0.0) + (i + 1 < k ? std::abs(e[i]) : 0.0);
        lo = std::min(lo, d[i] - r);
        hi = std::max(hi, d[i] + r);
    }
    auto kth = [&](int idx) {  // idx-th smallest eigenvalue (0-based)
        double a = lo, b = hi;
        for (int it = 0; it < 200; ++it) {
            const double mid = 0.5 * (a + b);
            if (mid <= a || mid >= b) break;
            if (sturm_count(d, e, mid) > idx)
                b = mid;
            else
                a = mid;
        }
        return 0.5 * (a + b);
    };
    lmin = kth(0);
    lmax = kth(k - 1);
}

struct PcgReport {  // pcg.hpp:9-16
    std::vector<double> solution;
    int iterations = 0;
    bool converged = false;
    std::vector<double> residual_history, energy_error_history, alphas, betas;
    double kappa_estimate = 1.0;
};

inline std::vector<double> matvec(const Dense& W, const std::vector<double>& p)
{
    std::vector<double> y(W.n, 0.0);
    for (int i = 0; i < W.n; ++i) {
        double s = 0;
        const double* row = &W.a[(size_t)i * W.n];
        for (int j = 0; j < W.n; ++j) s += row[j] * p[j];
        y[i] = s;
    }
    return y;
}
inline double vdot(const std::vector<double>& a, const std::vector<double>& b)
{
    double s = 0;
    for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
    return s;
}

// Lanczos kappa from the CG coefficients (reference: inc/pcg.hpp:96-114)
inline double lanczos_kappa(const std::vector<double>& alphas, const std::vector<double>& betas)
{
    const int k = (int)alphas.size();
    double kappa = 1.0;
    if (k > 0) {
        std::vector<double> d(k), e(k > 1 ? k - 1 : 0);
        for (int i = 0; i < k; ++i) {
            d[i] = 1.0 / alphas[i];
            if (i > 0) d[i] += betas[i - 1] / alphas[i - 1];
            if (i + 1 < k) e[i] = std::sqrt(std::max(betas[i], 0.0)) / alphas[i];
        }
        double lmin, lmax;
        tridiag_extremes(d, e, lmin, lmax);
        kappa = (lmin > 0) ? lmax / lmin : 1.0;
    }
    if (kappa < 1.0) kappa = 1.0;
    return kappa;
}

// reference: inc/pcg.hpp:33-116
inline PcgReport pcg(const Dense& W, const SchwarzPreconditioner* prec, const std::vector<double>& rhs,
                     double tol = 1e-8, int maxit = 0, const std::vector<double>* exact = nullptr)
{
    const int n = W.n;
    if ((int)rhs.size() != n) throw ValidationError("pcg: right-hand side length mismatch");
    if (tol <= 0) throw ValidationError("pcg: tolerance must be positive");
    if (maxit <= 0) maxit = std::max(10 * n, 100);
    PcgReport rep;
    rep.solution.assign(n, 0.0);
    auto precond = [&](const std::vector<double>& r) { return prec ? apply_preconditioner(*prec, r) : r; };
    auto energy_error = [&](const std::vector<double>& x) {
        std::vector<double> e(n);
        for (int i = 0; i < n; ++i) e[i] = x[i] - (*exact)[i];
        return std::sqrt(std::max(0.0, vdot(e, matvec(W, e))));
    };
    std::vector<double> r = rhs;
    std::vector<double> z = precond(r);
    double rz = vdot(r, z);
    if (rz < 0) throw NumericalError("pcg: preconditioner is not positive definite");
    const double r0 = std::sqrt(std::max(rz, 0.0));
    rep.residual_history.push_back(r0);
    if (exact) rep.energy_error_history.push_back(energy_error(rep.solution));
    std::vector<double> p = z;
    if (r0 == 0.0) {
        rep.converged = true;
        return rep;
    }
    for (int it = 0; it < maxit; ++it) {
        const std::vector<double> Wp = matvec(W, p);
        const double pWp = vdot(p, Wp);
        if (pWp <= 0) throw NumericalError("pcg: matrix is not positive definite");
        const double alpha = rz / pWp;
        for (int i = 0; i < n; ++i) rep.solution[i] += alpha * p[i];
        for (int i = 0; i < n; ++i) r[i] -= alpha * Wp[i];
        z = precond(r);
        const double rz_new = vdot(r, z);
        if (rz_new < 0) throw NumericalError("pcg: preconditioner is not positive definite");
        rep.alphas.push_back(alpha);
        rep.iterations = it + 1;
        rep.residual_history.push_back(std::sqrt(std::max(rz_new, 0.0)));
        if (exact) rep.energy_error_history.push_back(energy_error(rep.solution));
        if (rep.residual_history.back() <= tol * r0) {
            rep.converged = true;
            rep.betas.push_back(rz_new / rz);
            rz = rz_new;
            break;
        }
        const double beta = rz_new / rz;
        rep.betas.push_back(beta);
        rz = rz_new;
        for (int i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    }
    rep.kappa_estimate = lanczos_kappa(rep.alphas, rep.betas);
    return rep;
}

// reference: inc/pcg.hpp:18-28
inline std::vector<double> direct_solve(const Dense& W, const std::vector<double>& rhs)
{
    Dense L = W;
    if (!cholesky(L)) throw NumericalError("direct solve: Cholesky factorization failed");
    std::vector<double> x = rhs;
    llt_solve(L, x);
    const std::vector<double> Wx = matvec(W, x);
    double res = 0, bn = 0;
    for (int i = 0; i < W.n; ++i) {
        res += (Wx[i] - rhs[i]) * (Wx[i] - rhs[i]);
        bn += rhs[i] * rhs[i];
    }
    res = std::sqrt(res);
    bn = std::sqrt(bn);
    if (res > 1e-10 * std::max(bn, 1e-300) && bn > 0)
        throw NumericalError("direct solve: residual exceeds tolerance");
    return x;
}

// ---------------------------------------------------------------- potential.hpp (3-D)
// reference: inc/mesh.hpp:121-133 (SurfaceMesh::distance_to: min over facets, from 1e300)
inline double distance_to(const SurfaceMesh& m, const Vec3& x)
{
    double d = 1e300;
    for (int f = 0; f < m.num_facets(); ++f) {
        const auto& t = m.facets[f];
        d = std::min(d, detail::point_triangle_distance(x, m.vertices[t[0]], m.vertices[t[1]], m.vertices[t[2]]));
    }
    return d;
}

// reference: inc/potential.hpp:15-25 (grid in the z = 0 plane, points within mask_eps dropped)
inline std::vector<Vec3> make_cartesian_grid(const SurfaceMesh& mesh, double lo, double hi, int nx, int ny,
                                             double mask_eps)
{
    std::vector<Vec3> pts;
    for (int i = 0; i < nx; ++i)
        for (int j = 0; j < ny; ++j) {
            const Vec3 p(lo + (hi - lo) * (i + 0.5) / nx, lo + (hi - lo) * (j + 0.5) / ny, 0.0);
            if (distance_to(mesh, p) > mask_eps) pts.push_back(p);
        }
    return pts;
}

namespace detail {
// reference: inc/potential.hpp:31-97 (the 3-D branch): the dipole kernel n0.(y-x)/(4 pi |y-x|^3)
// times the side-0/side-1 value difference over one facet, split4 subdivision in barycentric
// space (children in the reference's order) while the point is closer than the diameter
inline double facet_dipole_integral(const Vec3& n0, const Vec3& x, const std::array<double, 3>& dvals,
                                    const TriangleRule& tri, const std::array<Vec3, 3>& corner, int depth)
{
    double diam = 0;
    for (int a = 0; a < 3; ++a)
        for (int b = a + 1; b < 3; ++b) diam = std::max(diam, norm(corner[a] - corner[b]));
    const double dist = point_triangle_distance(x, corner[0], corner[1], corner[2]);
    if (dist < diam && depth < 24) {
        const Vec3 m01 = 0.5 * (corner[0] + corner[1]);
        const Vec3 m12 = 0.5 * (corner[1] + corner[2]);
        const Vec3 m02 = 0.5 * (corner[0] + corner[2]);
        const double d01 = 0.5 * (dvals[0] + dvals[1]);
        const double d12 = 0.5 * (dvals[1] + dvals[2]);
        const double d02 = 0.5 * (dvals[0] + dvals[2]);
        double acc = 0;
        acc += facet_dipole_integral(n0, x, {dvals[0], d01, d02}, tri, {corner[0], m01, m02}, depth + 1);
        acc += facet_dipole_integral(n0, x, {d01, dvals[1], d12}, tri, {m01, corner[1], m12}, depth + 1);
        acc += facet_dipole_integral(n0, x, {d02, d12, dvals[2]}, tri, {m02, m12, corner[2]}, depth + 1);
        acc += facet_dipole_integral(n0, x, {d01, d12, d02}, tri, {m01, m12, m02}, depth + 1);
        return acc;
    }
    const double area = 0.5 * norm(cross(corner[1] - corner[0], corner[2] - corner[0]));
    double acc = 0;
    for (int i = 0; i < tri.size(); ++i) {
        const Vec3 y = corner[0] + tri.u[i] * (corner[1] - corner[0]) + tri.v[i] * (corner[2] - corner[0]);
        const double val = (1.0 - tri.u[i] - tri.v[i]) * dvals[0] + tri.u[i] * dvals[1] + tri.v[i] * dvals[2];
        const Vec3 r = y - x;
        const double rn = norm(r);
        acc += tri.w[i] * 2.0 * area * dot(n0, r) / (4.0 * M_PI * rn * rn * rn) * val;
    }
    return acc;
}
}  // namespace detail

// reference: inc/potential.hpp:104-138: U(x) = sum_t int n_t.(y-x)/(4 pi |x-y|^3) [phi](y), the
// two copies of each facet combined (side-0 minus side-1 trace), rule triangle_rule(far+2)
inline std::vector<double> eval_DL(const std::vector<double>& v, const InflatedMesh& im,
                                   const std::vector<Vec3>& points, const QuadratureConfig& cfg, int workers = 1)
{
    const SurfaceMesh& m = im.base;
    const TraceField tf = expand(v, im);
    const TriangleRule tri = triangle_rule(cfg.far_order + 2);
    const double mask = 0.5 * m.max_facet_diameter() * 1e-6;
    std::vector<double> out(points.size(), 0.0);
    run_partitioned((std::int64_t)points.size(), workers, [&](int, std::int64_t lo, std::int64_t hi) {
        for (std::int64_t p = lo; p < hi; ++p) {
            const Vec3& x = points[p];
            if (distance_to(m, x) <= mask) throw ValidationError("evaluation point lies on the screen");
            double acc = 0;
            for (int f = 0; f < m.num_facets(); ++f) {
                std::array<double, 3> dv = {0, 0, 0};
                for (int k = 0; k < 3; ++k) dv[k] = tf.at(im, 2 * f, k) - tf.at(im, 2 * f + 1, k);
                const std::array<Vec3, 3> corner = {m.vertices[m.facets[f][0]], m.vertices[m.facets[f][1]],
                                                    m.vertices[m.facets[f][2]]};
                acc += detail::facet_dipole_integral(im.oriented_facets[2 * f].normal, x, dv, tri, corner, 0);
            }
            out[p] = acc;
        }
    });
    return out;
}

}  // namespace sbo
