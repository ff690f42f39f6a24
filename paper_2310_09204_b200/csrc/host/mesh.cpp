// Meshes, validation, refinement and the BASELINE config generators.
// reference: proj/include/screenbem/mesh.hpp
#include <algorithm>
#include <cstdint>
#include <set>
#include <thread>
#include <unordered_map>

#include "host.hpp"

namespace sbg {

double SurfaceMesh::facet_measure(int f) const  // mesh.hpp:45-50
{
    const auto& t = facets[f];
    return 0.5 * norm(cross(vertices[t[1]] - vertices[t[0]], vertices[t[2]] - vertices[t[0]]));
}
Vec3 SurfaceMesh::facet_normal(int f) const  // mesh.hpp:54-62
{
    const auto& t = facets[f];
    return normalized(cross(vertices[t[1]] - vertices[t[0]], vertices[t[2]] - vertices[t[0]]));
}
double SurfaceMesh::facet_diameter(int f) const  // mesh.hpp:36-43
{
    double d = 0;
    for (int a = 0; a < 3; ++a)
        for (int b = a + 1; b < 3; ++b) d = std::max(d, norm(vertices[facets[f][a]] - vertices[facets[f][b]]));
    return d;
}
Vec3 SurfaceMesh::facet_centroid(int f) const
{
    Vec3 c;
    for (int k = 0; k < 3; ++k) c = c + vertices[facets[f][k]];
    return c / 3.0;
}
double SurfaceMesh::max_facet_diameter() const
{
    double h = 0;
    for (int f = 0; f < num_facets(); ++f) h = std::max(h, facet_diameter(f));
    return h;
}
double SurfaceMesh::diameter() const
{
    Vec3 lo(1e300, 1e300, 1e300), hi(-1e300, -1e300, -1e300);
    for (const auto& p : vertices) {
        lo = {std::min(lo.x, p.x), std::min(lo.y, p.y), std::min(lo.z, p.z)};
        hi = {std::max(hi.x, p.x), std::max(hi.y, p.y), std::max(hi.z, p.z)};
    }
    return norm(hi - lo);
}

namespace {

double point_segment_distance(const Vec3& x, const Vec3& a, const Vec3& b)  // mesh.hpp:96-101
{
    const Vec3 d = b - a;
    const double t = std::clamp(dot(x - a, d) / sqnorm(d), 0.0, 1.0);
    return norm(x - (a + t * d));
}
double point_triangle_distance(const Vec3& x, const Vec3& a, const Vec3& b, const Vec3& c)  // :103-117
{
    const Vec3 ab = b - a, ac = c - a, n = cross(ab, ac);
    const double nn = sqnorm(n);
    const Vec3 ax = x - a;
    const double u = dot(cross(ax, ac), n) / nn, v = dot(cross(ab, ax), n) / nn;
    if (u >= 0 && v >= 0 && u + v <= 1.0) return std::abs(dot(ax, n)) / std::sqrt(nn);
    return std::min({point_segment_distance(x, a, b), point_segment_distance(x, b, c), point_segment_distance(x, a, c)});
}
bool segment_hits_triangle(const Vec3& a, const Vec3& b, const Vec3& t0, const Vec3& t1, const Vec3& t2,
                           double eps)  // :183-194
{
    const Vec3 n = cross(t1 - t0, t2 - t0);
    const double da = dot(n, a - t0), db = dot(n, b - t0);
    if ((da > eps && db > eps) || (da < -eps && db < -eps)) return false;
    if (std::abs(da - db) < 1e-300) return false;
    const double s = da / (da - db);
    if (s < -eps || s > 1 + eps) return false;
    return point_triangle_distance(a + s * (b - a), t0, t1, t2) < eps;
}
bool conforming(const SurfaceMesh& m, int f, int g, double eps)  // :196-234
{
    const auto& a = m.facets[f];
    const auto& b = m.facets[g];
    auto in = [](const std::array<int, 3>& t, int v) { return t[0] == v || t[1] == v || t[2] == v; };
    int nshared = 0;
    for (int v : a) nshared += in(b, v) ? 1 : 0;
    const Vec3 A0 = m.vertices[a[0]], A1 = m.vertices[a[1]], A2 = m.vertices[a[2]];
    const Vec3 B0 = m.vertices[b[0]], B1 = m.vertices[b[1]], B2 = m.vertices[b[2]];
    for (int v : a)
        if (!in(b, v) && point_triangle_distance(m.vertices[v], B0, B1, B2) < eps) return false;
    for (int v : b)
        if (!in(a, v) && point_triangle_distance(m.vertices[v], A0, A1, A2) < eps) return false;
    static const int eidx[3][2] = {{0, 1}, {1, 2}, {2, 0}};
    for (const auto& e : eidx) {
        const int u = a[e[0]], v = a[e[1]];
        if (in(b, u) || in(b, v)) continue;
        if (segment_hits_triangle(m.vertices[u], m.vertices[v], B0, B1, B2, eps)) return false;
    }
    for (const auto& e : eidx) {
        const int u = b[e[0]], v = b[e[1]];
        if (in(a, u) || in(a, v)) continue;
        if (segment_hits_triangle(m.vertices[u], m.vertices[v], A0, A1, A2, eps)) return false;
    }
    if (nshared >= 1) {
        const Vec3 n1 = normalized(cross(A1 - A0, A2 - A0)), n2 = normalized(cross(B1 - B0, B2 - B0));
        if (std::abs(std::abs(dot(n1, n2)) - 1.0) < 1e-12 && std::abs(dot(n1, B0 - A0)) < eps) {
            const Vec3 ca = ((A0 + A1) + A2) / 3.0, cb = ((B0 + B1) + B2) / 3.0;
            if (point_triangle_distance(ca, B0, B1, B2) < eps || point_triangle_distance(cb, A0, A1, A2) < eps)
                return false;
        }
    }
    return true;
}

struct CellKey {
    std::int64_t x, y, z;
    bool operator==(const CellKey& o) const { return x == o.x && y == o.y && z == o.z; }
};
struct CellHash {
    size_t operator()(const CellKey& k) const
    {
        return (size_t)(k.x * 73856093LL ^ k.y * 19349663LL ^ k.z * 83492791LL);
    }
};

}  // namespace

// reference: inc/mesh.hpp:238-272.  Same checks and the same bounding-sphere
// predicate; candidate pairs come from a uniform grid of facet centroids with
// cell size >= the largest reject radius, so exactly the pairs the reference's
// O(nf^2) loop tests are tested.  The per-facet checks and the conformity test run on
// host threads over facet ranges; the error raised is the one the reference's
// sequential loops reach first (smallest facet, then smallest partner; per facet the
// order id range, duplicate, degenerate).
void validate_mesh(const SurfaceMesh& m)
{
    const int nv = m.num_vertices(), nf = m.num_facets();
    for (const auto& p : m.vertices)
        if (!std::isfinite(p.x) || !std::isfinite(p.y) || !std::isfinite(p.z))
            throw ValidationError("non-finite vertex coordinate");
    const double eps = 1e-12 * std::max(m.diameter(), 1e-300);
    // first facet with an id out of range: the facets before it are checked for duplicates
    // (second occurrence of a sorted vertex triple) and degeneracy
    int f_range = nf;
    for (int f = 0; f < nf && f_range == nf; ++f)
        for (int k = 0; k < 3; ++k)
            if (m.facets[f][k] < 0 || m.facets[f][k] >= nv) {
                f_range = f;
                break;
            }
    std::vector<std::pair<std::array<int, 3>, int>> keys(f_range);
    for (int f = 0; f < f_range; ++f) {
        std::array<int, 3> key = m.facets[f];
        std::sort(key.begin(), key.end());
        keys[f] = {key, f};
    }
    std::sort(keys.begin(), keys.end());
    int f_dup = nf;
    for (size_t i = 1; i < keys.size(); ++i)
        if (keys[i].first == keys[i - 1].first) f_dup = std::min(f_dup, keys[i].second);
    const int nthreads = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    auto parallel = [&](int count, const auto& body) {  // body(lo, hi, slot) over contiguous ranges
        const int nt = std::max(1, std::min(nthreads, count / 2048));
        std::vector<std::thread> pool;
        for (int t = 1; t < nt; ++t)
            pool.emplace_back([&, t] { body((int)((long long)count * t / nt), (int)((long long)count * (t + 1) / nt), t); });
        body(0, (int)((long long)count / nt), 0);
        for (auto& th : pool) th.join();
        return nt;
    };
    // degenerate facets before the first id/duplicate error (at that facet its own error wins)
    std::vector<int> deg(nthreads, nf);
    const int f_chk = std::min(f_range, f_dup);
    parallel(f_chk, [&](int lo, int hi, int slot) {
        for (int f = lo; f < hi; ++f) {
            const double scale = eps * std::max(m.facet_diameter(f), eps);
            if (m.facet_measure(f) < scale) {
                deg[slot] = f;
                return;
            }
        }
    });
    const int f_deg = *std::min_element(deg.begin(), deg.end());
    if (f_deg < f_chk) throw ValidationError("degenerate facet " + std::to_string(f_deg));
    if (f_chk < nf) throw ValidationError(f_range == f_chk ? "facet vertex id out of range" : "duplicate facet");
    if (nf == 0) return;
    std::vector<Vec3> cen(nf);
    std::vector<double> dia(nf);
    double dmax = 0;
    for (int f = 0; f < nf; ++f) {
        cen[f] = m.facet_centroid(f);
        dia[f] = m.facet_diameter(f);
        dmax = std::max(dmax, dia[f]);
    }
    const double cell = (dmax + eps) * (1.0 + 1e-9) + 1e-300;
    auto key_of = [&](const Vec3& c) {
        return CellKey{(std::int64_t)std::floor(c.x / cell), (std::int64_t)std::floor(c.y / cell),
                       (std::int64_t)std::floor(c.z / cell)};
    };
    std::unordered_map<CellKey, std::vector<int>, CellHash> grid;
    grid.reserve((size_t)nf);
    for (int f = 0; f < nf; ++f) grid[key_of(cen[f])].push_back(f);
    // first non-conforming pair per thread range (facets ascending, partners ascending)
    std::vector<std::pair<int, int>> bad(nthreads, {nf, nf});
    parallel(nf, [&](int lo, int hi, int slot) {
        std::vector<int> cand;
        for (int f = lo; f < hi; ++f) {
            const CellKey k = key_of(cen[f]);
            cand.clear();
            for (int dx = -1; dx <= 1; ++dx)
                for (int dy = -1; dy <= 1; ++dy)
                    for (int dz = -1; dz <= 1; ++dz) {
                        auto it = grid.find(CellKey{k.x + dx, k.y + dy, k.z + dz});
                        if (it == grid.end()) continue;
                        for (int g : it->second)
                            if (g > f) cand.push_back(g);
                    }
            std::sort(cand.begin(), cand.end());
            for (int g : cand) {
                const double rr = 0.5 * (dia[f] + dia[g]) + eps;
                if (norm(cen[f] - cen[g]) > rr) continue;
                if (!conforming(m, f, g, eps)) {
                    bad[slot] = {f, g};
                    return;
                }
            }
        }
    });
    const auto first = *std::min_element(bad.begin(), bad.end());
    if (first.first < nf)
        throw ValidationError("non-conforming facet pair " + std::to_string(first.first) + "," +
                              std::to_string(first.second));
}

SurfaceMesh make_bowtie_base()  // mesh.hpp:322-337
{
    const double mlen = std::sqrt(3.0) / 2.0;
    SurfaceMesh m;
    m.vertices = {Vec3(0, 0, 0), Vec3(0, 0, mlen), Vec3(0.5, 0, mlen), Vec3(-0.5, 0, mlen), Vec3(0, 0.5, mlen),
                  Vec3(0, -0.5, mlen)};
    m.facets = {{0, 2, 1}, {0, 1, 3}, {0, 4, 1}, {0, 1, 5}};
    return m;
}

MeshLevelPair refine_uniform(const SurfaceMesh& mesh)  // mesh.hpp:342-386
{
    MeshLevelPair pair;
    pair.coarse = mesh;
    SurfaceMesh& fine = pair.fine;
    fine.vertices = mesh.vertices;
    std::map<std::array<int, 2>, int> edge_mid;
    auto midpoint = [&](int a, int b) {
        const std::array<int, 2> key = {std::min(a, b), std::max(a, b)};
        auto it = edge_mid.find(key);
        if (it != edge_mid.end()) return it->second;
        fine.vertices.push_back(0.5 * (mesh.vertices[a] + mesh.vertices[b]));
        const int id = fine.num_vertices() - 1;
        edge_mid.emplace(key, id);
        return id;
    };
    for (int f = 0; f < mesh.num_facets(); ++f) {
        const auto& t = mesh.facets[f];
        const int m01 = midpoint(t[0], t[1]), m12 = midpoint(t[1], t[2]), m02 = midpoint(t[0], t[2]);
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

MeshLevelPair refine_uniform_times(const SurfaceMesh& mesh, int k)  // mesh.hpp:388-405
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

SurfaceMesh make_builtin(const std::string& spec)  // mesh.hpp:516-537
{
    std::string name = spec;
    int param = -1;
    if (const auto pos = spec.find(':'); pos != std::string::npos) {
        name = spec.substr(0, pos);
        try {
            param = std::stoi(spec.substr(pos + 1));
        } catch (const std::exception&) {
            throw ValidationError("bad builtin parameter in '" + spec + "'");
        }
    }
    if (name == "plus" || name == "threefold")
        throw ValidationError("2-D builtin '" + name + "' is outside the 3-D GPU path");
    if (name != "bowtie") throw ValidationError("unknown builtin geometry '" + name + "'");
    SurfaceMesh m = refine_uniform_times(make_bowtie_base(), param < 0 ? 0 : param).fine;
    validate_mesh(m);
    return m;
}

// ---------------------------------------------------------------- configs
namespace {
struct Panel {
    Vec3 o, a, b;
};

struct QKey {
    std::int64_t x, y, z;
    bool operator<(const QKey& r) const { return x != r.x ? x < r.x : (y != r.y ? y < r.y : z < r.z); }
};

// Panels of m x m cells of size L/m; vertex (i,j) = o + (L i/m) a + (L j/m) b,
// cell (i,j) -> {p00,p10,p11},{p00,p11,p01} (the
// diagonal and vertex order of tests/test_inflate.cpp:14-15).  Coincident
// vertices of different panels are merged by quantised position.
SurfaceMesh panel_mesh(const std::vector<Panel>& panels, double L, int m)
{
    SurfaceMesh out;
    std::map<QKey, int> ids;
    for (const auto& P : panels) {
        std::vector<int> local((size_t)(m + 1) * (m + 1));
        for (int j = 0; j <= m; ++j)
            for (int i = 0; i <= m; ++i) {
                const double si = (L * i) / m, sj = (L * j) / m;
                const Vec3 p((P.o.x + si * P.a.x) + sj * P.b.x, (P.o.y + si * P.a.y) + sj * P.b.y,
                             (P.o.z + si * P.a.z) + sj * P.b.z);
                const QKey k{std::llround(p.x * 1e9), std::llround(p.y * 1e9), std::llround(p.z * 1e9)};
                auto it = ids.find(k);
                int id;
                if (it == ids.end()) {
                    id = out.num_vertices();
                    out.vertices.push_back(p);
                    ids.emplace(k, id);
                } else {
                    id = it->second;
                }
                local[(size_t)j * (m + 1) + i] = id;
            }
        auto V = [&](int i, int j) { return local[(size_t)j * (m + 1) + i]; };
        for (int j = 0; j < m; ++j)
            for (int i = 0; i < m; ++i) {
                out.facets.push_back({V(i, j), V(i + 1, j), V(i + 1, j + 1)});
                out.facets.push_back({V(i, j), V(i + 1, j + 1), V(i, j + 1)});
            }
    }
    return out;
}

MeshLevelPair panel_pair(const std::vector<Panel>& panels, double L, int m, int r)
{
    if (r < 1 || m % r != 0) throw ValidationError("panel refinement ratio must divide the cell count");
    const int mc = m / r;
    MeshLevelPair pair;
    pair.fine = panel_mesh(panels, L, m);
    pair.coarse = panel_mesh(panels, L, mc);
    pair.parent.resize(pair.fine.num_facets());
    for (int P = 0; P < (int)panels.size(); ++P)
        for (int j = 0; j < m; ++j)
            for (int i = 0; i < m; ++i) {
                const int I = i / r, J = j / r, a = i % r, b = j % r;
                const int cbase = P * 2 * mc * mc + 2 * (J * mc + I);
                const int fbase = P * 2 * m * m + 2 * (j * m + i);
                pair.parent[fbase + 0] = cbase + ((b <= a) ? 0 : 1);  // fine lower triangle
                pair.parent[fbase + 1] = cbase + ((a <= b) ? 1 : 0);  // fine upper triangle
            }
    pair.H = pair.coarse.max_facet_diameter();
    pair.h = pair.fine.max_facet_diameter();
    return pair;
}
}  // namespace

// kind 0: flat unit square; 1: T-junction of three unit squares about the
// z-axis; 2: triple cross of [-1,1]^2 squares in the coordinate planes.
MeshLevelPair make_panels(int kind, int m, int r)
{
    std::vector<Panel> P;
    double L = 1.0;
    if (kind == 0) {
        P.push_back({Vec3(0, 0, 0), Vec3(1, 0, 0), Vec3(0, 1, 0)});
    } else if (kind == 1) {
        for (int k = 0; k < 3; ++k) {
            const double th = 2.0 * M_PI * k / 3.0;
            P.push_back({Vec3(0, 0, 0), Vec3(std::cos(th), std::sin(th), 0), Vec3(0, 0, 1)});
        }
    } else if (kind == 2) {
        L = 2.0;
        P.push_back({Vec3(-1, -1, 0), Vec3(1, 0, 0), Vec3(0, 1, 0)});
        P.push_back({Vec3(0, -1, -1), Vec3(0, 1, 0), Vec3(0, 0, 1)});
        P.push_back({Vec3(-1, 0, -1), Vec3(1, 0, 0), Vec3(0, 0, 1)});
        if (m % 2 != 0) throw ValidationError("triple cross needs an even cell count (axes on grid lines)");
    } else {
        throw ValidationError("unknown panel geometry kind " + std::to_string(kind));
    }
    return panel_pair(P, L, m, r);
}

// BASELINE.json configs
MeshLevelPair make_config(int cfg, int ratio)
{
    switch (cfg) {
        case 1: return make_panels(0, 16, ratio > 0 ? ratio : 8);
        case 2: return make_panels(0, 64, ratio > 0 ? ratio : 16);
        case 3: return make_panels(1, 48, ratio > 0 ? ratio : 12);
        case 4: return make_panels(2, 64, ratio > 0 ? ratio : 8);
        case 5: return make_panels(0, 160, ratio > 0 ? ratio : 8);
        default: throw ValidationError("unknown BASELINE config " + std::to_string(cfg));
    }
}

}  // namespace sbg
