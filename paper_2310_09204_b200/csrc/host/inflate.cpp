// Inflation / DOF numbering, prolongation, partition, facet curl lists and
// quadrature rules.  reference: inflate.hpp, jump.hpp, schwarz.hpp:19-51,
// assemble.hpp:18-53, gauss.hpp, quadrature.hpp:35-92.
#include <algorithm>
#include <numeric>
#include <unordered_map>

#include <cstdlib>
#include <thread>

#include "host.hpp"

namespace sbg {

namespace {
struct DSU {
    std::vector<int> p;
    DSU() = default;
    explicit DSU(int n) : p(n) { std::iota(p.begin(), p.end(), 0); }
    void reset(int n)
    {
        p.resize(n);
        std::iota(p.begin(), p.end(), 0);
    }
    int find(int a)
    {
        while (p[a] != a) a = p[a] = p[p[a]];
        return a;
    }
    void unite(int a, int b) { p[find(a)] = find(b); }
};
}  // namespace

// contiguous ranges of [0, count) on up to 16 host threads (the calling thread included);
// body(lo, hi, slot)
template <class F>
static int parallel_ranges(int count, int min_chunk, const F& body)
{
    const unsigned hw = std::thread::hardware_concurrency() ? std::thread::hardware_concurrency() : 1u;
    const int nt = std::max(1, std::min({(int)std::min(16u, hw), count / std::max(min_chunk, 1), 64}));
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t)
        pool.emplace_back([&, t] { body((int)((long long)count * t / nt), (int)((long long)count * (t + 1) / nt), t); });
    body(0, (int)((long long)count / nt), 0);
    for (auto& th : pool) th.join();
    return nt;
}

// reference: inc/inflate.hpp:98-288.  The edge->facets map is a sorted edge
// list (same lexicographic order as the reference's std::map), and the
// point-contact test visits only the edges incident to each vertex (the
// reference scans every edge for every vertex, O(V*E)); outputs are identical.
// validate_mesh runs on a helper thread beside the inflation (after a sequential check of
// the vertex ids, the one thing the inflation itself relies on); the per-vertex and per-edge
// phases run on host threads.  Errors are raised in the reference's order: validation first,
// then the first point contact, the first angular tie, the first isolated vertex.
InflatedMesh inflate(const SurfaceMesh& mesh, bool validate)
{
    const int nf = mesh.num_facets(), nv = mesh.num_vertices();
    std::thread vthread;
    std::exception_ptr verr;
    if (validate) {
        bool ids_ok = true;
        for (int f = 0; f < nf && ids_ok; ++f)
            for (int k = 0; k < 3; ++k)
                if (mesh.facets[f][k] < 0 || mesh.facets[f][k] >= nv) ids_ok = false;
        if (!ids_ok) validate_mesh(mesh);  // throws the reference's first error
        vthread = std::thread([&] {
            try {
                validate_mesh(mesh);
            } catch (...) {
                verr = std::current_exception();
            }
        });
    }
    struct Joiner {
        std::thread& t;
        ~Joiner()
        {
            if (t.joinable()) t.join();
        }
    } joiner{vthread};
    auto raise_validation = [&] {
        if (vthread.joinable()) vthread.join();
        if (verr) std::rethrow_exception(verr);
    };
    InflatedMesh im;
    im.base = mesh;
    im.onormal.resize(2 * nf);
    for (int f = 0; f < nf; ++f) {
        const Vec3 n = mesh.facet_normal(f);
        im.onormal[2 * f] = n;
        im.onormal[2 * f + 1] = -n;
    }
    // edges: (min, max, facet) sorted
    struct E {
        int a, b, f;
    };
    std::vector<E> el;
    el.reserve(3 * (size_t)nf);
    for (int f = 0; f < nf; ++f) {
        const auto& t = mesh.facets[f];
        for (int k = 0; k < 3; ++k) {
            const int a = t[k], b = t[(k + 1) % 3];
            el.push_back({std::min(a, b), std::max(a, b), f});
        }
    }
    std::sort(el.begin(), el.end(), [](const E& x, const E& y) {
        return x.a != y.a ? x.a < y.a : (x.b != y.b ? x.b < y.b : x.f < y.f);
    });
    std::vector<int> eptr;  // group starts
    for (size_t i = 0; i < el.size(); ++i)
        if (i == 0 || el[i].a != el[i - 1].a || el[i].b != el[i - 1].b) eptr.push_back((int)i);
    const int ne = (int)eptr.size();
    eptr.push_back((int)el.size());
    // vertex -> incident edges / facets as CSR lists (ascending)
    std::vector<int> ve_ptr(nv + 1, 0), vs_ptr(nv + 1, 0);
    for (int e = 0; e < ne; ++e) {
        ++ve_ptr[el[eptr[e]].a + 1];
        ++ve_ptr[el[eptr[e]].b + 1];
    }
    for (int f = 0; f < nf; ++f)
        for (int k = 0; k < 3; ++k) ++vs_ptr[mesh.facets[f][k] + 1];
    for (int v = 0; v < nv; ++v) {
        ve_ptr[v + 1] += ve_ptr[v];
        vs_ptr[v + 1] += vs_ptr[v];
    }
    std::vector<int> vedges(ve_ptr[nv]), vstar(vs_ptr[nv]);
    {
        std::vector<int> fill(ve_ptr.begin(), ve_ptr.end() - 1);
        for (int e = 0; e < ne; ++e) {
            vedges[fill[el[eptr[e]].a]++] = e;
            vedges[fill[el[eptr[e]].b]++] = e;
        }
        fill.assign(vs_ptr.begin(), vs_ptr.end() - 1);
        for (int f = 0; f < nf; ++f)
            for (int k = 0; k < 3; ++k) vstar[fill[mesh.facets[f][k]]++] = f;
    }
    constexpr int kSlots = 64;
    auto first_of = [](const std::vector<int>& v) { return *std::min_element(v.begin(), v.end()); };

    // point-contact check (inflate.hpp:129-151): the first vertex whose star splits
    std::vector<int> contact(kSlots, nv);
    parallel_ranges(nv, 1024, [&](int lo, int hi, int slot) {
        DSU ds;
        for (int v = lo; v < hi; ++v) {
            const int* star = vstar.data() + vs_ptr[v];
            const int ns = vs_ptr[v + 1] - vs_ptr[v];
            if (ns < 2) continue;
            auto local = [&](int f) { return (int)(std::lower_bound(star, star + ns, f) - star); };
            ds.reset(ns);
            for (int q = ve_ptr[v]; q < ve_ptr[v + 1]; ++q) {
                const int e = vedges[q];
                for (int i = eptr[e] + 1; i < eptr[e + 1]; ++i) ds.unite(local(el[eptr[e]].f), local(el[i].f));
            }
            const int root = ds.find(0);
            for (int i = 1; i < ns; ++i)
                if (ds.find(i) != root) {
                    contact[slot] = v;
                    return;
                }
        }
    });
    {
        const int v = first_of(contact);
        if (v < nv) {
            raise_validation();
            throw ValidationError("point contact at vertex " + std::to_string(v) + " (unsupported geometry)");
        }
    }

    // fans (inflate.hpp:155-228): edge e's k facets give k pairs at fan_pairs[eptr[e]...]
    std::vector<std::array<int, 2>> fan_pairs(el.size());
    const std::vector<int>& fan_ptr = eptr;
    std::vector<int> tie(kSlots, ne);
    parallel_ranges(ne, 2048, [&](int lo, int hi, int slot) {
        std::vector<std::pair<double, int>> slots;  // (angle, local)
        for (int e = lo; e < hi; ++e) {
            const int ea = el[eptr[e]].a, eb = el[eptr[e]].b;
            const Vec3 origin = mesh.vertices[ea];
            const Vec3 e_dir = normalized(mesh.vertices[eb] - mesh.vertices[ea]);
            auto in_plane_dir = [&](int f) {
                const auto& t = mesh.facets[f];
                int opp = -1;
                for (int k = 0; k < 3; ++k)
                    if (t[k] != ea && t[k] != eb) opp = t[k];
                Vec3 d = mesh.vertices[opp] - origin;
                d = d - dot(d, e_dir) * e_dir;
                return normalized(d);
            };
            const int k = eptr[e + 1] - eptr[e];
            const Vec3 ref = in_plane_dir(el[eptr[e]].f);
            const Vec3 up = cross(e_dir, ref);
            slots.clear();
            for (int i = 0; i < k; ++i) {
                const Vec3 d = in_plane_dir(el[eptr[e] + i].f);
                slots.push_back({std::atan2(dot(d, up), dot(d, ref)), i});
            }
            std::sort(slots.begin(), slots.end(),
                      [](const auto& x, const auto& y) { return x.first < y.first; });
            bool bad = false;
            for (int i = 0; i + 1 < k; ++i)
                if (slots[i + 1].first - slots[i].first < 1e-9) bad = true;
            if (k > 1 && slots[0].first + 2.0 * M_PI - slots[k - 1].first < 1e-9) bad = true;
            if (bad) {
                tie[slot] = e;
                return;
            }
            auto ccw_side = [&](int f) {
                const Vec3 tangent = cross(e_dir, in_plane_dir(f));
                return dot(im.onormal[2 * f], tangent) > 0 ? 0 : 1;
            };
            for (int i = 0; i < k; ++i) {
                const int fa = el[eptr[e] + slots[i].second].f;
                const int fb = el[eptr[e] + slots[(i + 1) % k].second].f;
                fan_pairs[eptr[e] + i] = {2 * fa + (1 - ccw_side(fa)), 2 * fb + ccw_side(fb)};
            }
        }
    });
    if (first_of(tie) < ne) {
        raise_validation();
        throw ValidationError("coplanar facets overlap at an edge fan (angular tie)");
    }

    // branches (inflate.hpp:232-279): per vertex the branch of every oriented facet of its
    // star (bid, at 2 vs_ptr[v] + i) and the branch count, then the numbering in vertex order
    std::vector<int> bidv(2 * (size_t)vs_ptr[nv]), nbv(nv, 0);
    std::vector<int> isolated(kSlots, nv);
    parallel_ranges(nv, 1024, [&](int lo, int hi, int slot) {
        DSU ds;
        std::vector<int> star, broot;
        for (int v = lo; v < hi; ++v) {
            const int ns = vs_ptr[v + 1] - vs_ptr[v];
            if (ns == 0) {
                isolated[slot] = v;
                return;
            }
            star.clear();  // oriented facets, ascending
            for (int q = vs_ptr[v]; q < vs_ptr[v + 1]; ++q) {
                star.push_back(2 * vstar[q]);
                star.push_back(2 * vstar[q] + 1);
            }
            const int m = (int)star.size();
            auto local = [&](int o) { return (int)(std::lower_bound(star.begin(), star.end(), o) - star.begin()); };
            ds.reset(m);
            for (int q = ve_ptr[v]; q < ve_ptr[v + 1]; ++q) {
                const int e = vedges[q];
                for (int p = fan_ptr[e]; p < fan_ptr[e + 1]; ++p)
                    ds.unite(local(fan_pairs[p][0]), local(fan_pairs[p][1]));
            }
            // branches ordered by their smallest oriented facet = order of first appearance
            broot.assign(m, -1);
            int nb = 0;
            int* bid = bidv.data() + 2 * (size_t)vs_ptr[v];
            for (int i = 0; i < m; ++i) {
                const int r = ds.find(i);
                if (broot[r] < 0) broot[r] = nb++;
                bid[i] = broot[r];
            }
            nbv[v] = nb;
        }
    });
    if (first_of(isolated) < nv) {
        raise_validation();
        throw ValidationError("isolated vertex " + std::to_string(first_of(isolated)));
    }
    im.q = nbv;
    im.gv_first.assign(nv, -1);
    im.dof_first.assign(nv, -1);
    im.ofacet_branch.assign(2 * nf, {-1, -1, -1});
    int ngv = 0;
    for (int v = 0; v < nv; ++v) {
        im.gv_first[v] = ngv;
        ngv += nbv[v];
    }
    im.gv_vertex.resize(ngv);
    im.gv_branch.resize(ngv);
    im.gv_alpha_ptr.assign(ngv + 1, 0);
    // a vertex's sectors hold all 2 ns oriented facets of its star, split among its branches
    for (int v = 0; v < nv; ++v)
        for (int j = 0; j < nbv[v]; ++j) {
            const int* bid = bidv.data() + 2 * (size_t)vs_ptr[v];
            int cnt = 0;
            for (int i = 0; i < 2 * (vs_ptr[v + 1] - vs_ptr[v]); ++i) cnt += bid[i] == j;
            im.gv_alpha_ptr[im.gv_first[v] + j + 1] = cnt;
        }
    for (int g = 0; g < ngv; ++g) im.gv_alpha_ptr[g + 1] += im.gv_alpha_ptr[g];
    im.gv_alpha.resize(im.gv_alpha_ptr[ngv]);
    parallel_ranges(nv, 1024, [&](int lo, int hi, int) {
        for (int v = lo; v < hi; ++v) {
            const int* bid = bidv.data() + 2 * (size_t)vs_ptr[v];
            const int m = 2 * (vs_ptr[v + 1] - vs_ptr[v]);
            for (int j = 0; j < nbv[v]; ++j) {
                const int g = im.gv_first[v] + j;
                im.gv_vertex[g] = v;
                im.gv_branch[g] = j;
                int w = im.gv_alpha_ptr[g];
                for (int i = 0; i < m; ++i) {
                    if (bid[i] != j) continue;
                    const int o = 2 * vstar[vs_ptr[v] + i / 2] + (i & 1);
                    im.gv_alpha[w++] = o;
                    const int f = o / 2;
                    for (int k = 0; k < 3; ++k)
                        if (mesh.facets[f][k] == v) im.ofacet_branch[o][k] = j;
                }
            }
        }
    });
    for (int v = 0; v < nv; ++v) {  // inflate.hpp:281-285
        if (im.q[v] < 2) continue;
        im.dof_first[v] = im.num_jump_dofs();
        for (int j = 0; j + 1 < im.q[v]; ++j) im.jump_dofs.push_back({v, j});
    }
    raise_validation();
    return im;
}

namespace {
// reference: inc/jump.hpp:94-111
void barycentric(const SurfaceMesh& m, int f, const Vec3& x, double& u, double& v)
{
    const auto& t = m.facets[f];
    const Vec3 e1 = m.vertices[t[1]] - m.vertices[t[0]], e2 = m.vertices[t[2]] - m.vertices[t[0]];
    const Vec3 r = x - m.vertices[t[0]];
    const double a11 = sqnorm(e1), a12 = dot(e1, e2), a22 = sqnorm(e2);
    const double b1 = dot(r, e1), b2 = dot(r, e2);
    const double det = a11 * a22 - a12 * a12;
    u = (a22 * b1 - a12 * b2) / det;
    v = (a11 * b2 - a12 * b1) / det;
}
}  // namespace

// reference: inc/jump.hpp:118-185.  The reference evaluates every coarse basis
// at every fine generalized vertex, O(n_c * n_gv * |alpha|).  A coarse basis at
// coarse vertex V is non-zero on a fine sector only if V is a vertex of a
// sector member's parent facet, so only those (fine vertex, coarse DOF)
// combinations are evaluated — with the same arithmetic, giving the same R.
Prolongation build_prolongation(const MeshLevelPair& pair, const InflatedMesh& coarse, const InflatedMesh& fine)
{
    const int nff = pair.fine.num_facets();
    std::vector<int> oparent(2 * (size_t)nff, -1);
    for (int f = 0; f < nff; ++f) {
        const int cf = pair.parent[f];
        if (cf < 0 || cf >= pair.coarse.num_facets())
            throw ValidationError("orphan fine facet " + std::to_string(f) + " (broken nesting)");
        for (int k = 0; k < 3; ++k) {
            double u, v;
            barycentric(pair.coarse, cf, pair.fine.vertices[pair.fine.facets[f][k]], u, v);
            if (u < -1e-9 || v < -1e-9 || u + v > 1 + 1e-9)
                throw ValidationError("fine facet " + std::to_string(f) + " escapes its parent (broken nesting)");
        }
        for (int s = 0; s < 2; ++s) {
            const double d = dot(fine.onormal[2 * f + s], coarse.onormal[2 * cf]);
            if (std::abs(d) < 0.5)
                throw ValidationError("fine facet " + std::to_string(f) + " normal mismatch (broken nesting)");
            oparent[2 * f + s] = 2 * cf + (d > 0 ? 0 : 1);
        }
    }
    struct Trip {
        int col, row;
        double v;
    };
    std::vector<Trip> trip;
    const int nv = fine.base.num_vertices();
    std::vector<double> vals;
    for (int i = 0; i < nv; ++i) {
        const int qi = fine.q[i];
        // candidate coarse DOFs: at vertices of the parents of the star of i
        std::vector<int> cand;
        for (int j = 0; j < qi; ++j) {
            const int g = fine.gv_index(i, j);
            for (int p = fine.gv_alpha_ptr[g]; p < fine.gv_alpha_ptr[g + 1]; ++p) {
                const int cf = oparent[fine.gv_alpha[p]] / 2;
                for (int k = 0; k < 3; ++k) {
                    const int V = pair.coarse.facets[cf][k];
                    for (int J = 0; J + 1 < coarse.q[V]; ++J) cand.push_back(coarse.dof_index(V, J));
                }
            }
        }
        std::sort(cand.begin(), cand.end());
        cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
        const Vec3 x = fine.base.vertices[i];
        for (int cd : cand) {
            const int V = coarse.jump_dofs[cd][0], J = coarse.jump_dofs[cd][1];
            const int gplus = coarse.gv_index(V, J), gminus = coarse.gv_index(V, coarse.q[V] - 1);
            vals.assign(qi, 0.0);
            for (int j = 0; j < qi; ++j) {
                const int g = fine.gv_index(i, j);
                double value = 0;
                bool first = true;
                for (int p = fine.gv_alpha_ptr[g]; p < fine.gv_alpha_ptr[g + 1]; ++p) {
                    const int po = oparent[fine.gv_alpha[p]];
                    double u, v;
                    barycentric(pair.coarse, po / 2, x, u, v);
                    double at[3];
                    for (int k = 0; k < 3; ++k) {
                        const int gv = coarse.gv_index(pair.coarse.facets[po / 2][k], coarse.ofacet_branch[po][k]);
                        at[k] = gv == gplus ? 1.0 : (gv == gminus ? -1.0 : 0.0);
                    }
                    const double val = (1.0 - u - v) * at[0] + u * at[1] + v * at[2];  // jump.hpp:25-29
                    if (first) {
                        value = val;
                        first = false;
                    } else if (std::abs(val - value) > 1e-8 * (1.0 + std::abs(value))) {
                        throw ValidationError("inconsistent coarse branch values across a fine sector "
                                              "(branch structure not refinement-invariant)");
                    }
                }
                vals[j] = value;
            }
            if (qi < 2) continue;
            double mean = 0;  // jump.hpp:61-74
            for (int j = 0; j < qi; ++j) mean += vals[j];
            mean /= qi;
            for (int j = 0; j + 1 < qi; ++j) {
                const double c = vals[j] - mean;
                if (c != 0.0) trip.push_back({cd, fine.dof_index(i, j), c});
            }
        }
    }
    std::sort(trip.begin(), trip.end(), [](const Trip& a, const Trip& b) { return a.col != b.col ? a.col < b.col : a.row < b.row; });
    Prolongation P;
    P.rows = fine.num_jump_dofs();
    P.cols = coarse.num_jump_dofs();
    P.col_ptr.assign(P.cols + 1, 0);
    for (const auto& t : trip) {
        P.col_ptr[t.col + 1]++;
        P.row_idx.push_back(t.row);
        P.val.push_back(t.v);
    }
    for (int c = 0; c < P.cols; ++c) P.col_ptr[c + 1] += P.col_ptr[c];
    return P;
}

// reference: inc/schwarz.hpp:19-51
DofPartition partition_dofs(const MeshLevelPair& pair, const InflatedMesh& fine)
{
    const int nv = pair.fine.num_vertices();
    std::vector<std::vector<int>> parents(nv);
    for (int f = 0; f < pair.fine.num_facets(); ++f) {
        if (pair.parent[f] < 0 || pair.parent[f] >= pair.coarse.num_facets())
            throw ValidationError("fine facet has no coarse parent (nesting violation)");
        for (int k = 0; k < 3; ++k) parents[pair.fine.facets[f][k]].push_back(pair.parent[f]);
    }
    for (auto& p : parents) {
        std::sort(p.begin(), p.end());
        p.erase(std::unique(p.begin(), p.end()), p.end());
    }
    std::map<int, std::vector<int>> faces;
    DofPartition part;
    for (int d = 0; d < fine.num_jump_dofs(); ++d) {
        const int v = fine.jump_dofs[d][0];
        const auto& ps = parents[v];
        if (ps.empty()) throw ValidationError("fine vertex not locatable on the coarse geometry");
        bool interior = false;
        int face = -1;
        if (ps.size() == 1) {
            face = ps[0];
            double u, w;
            barycentric(pair.coarse, face, pair.fine.vertices[v], u, w);
            const double tol = 1e-9;
            interior = (u > tol && u + w < 1.0 - tol && w > tol);
        }
        if (interior)
            faces[face].push_back(d);
        else
            part.wirebasket.push_back(d);
    }
    for (auto& [f, ds] : faces) {
        part.face_ids.push_back(f);
        part.face_dofs.insert(part.face_dofs.end(), ds.begin(), ds.end());
        part.face_ptr.push_back((int)part.face_dofs.size());
    }
    return part;
}

// reference: inc/assemble.hpp:18-29 (shape gradient), :34-53 (scatter), :83-89 (slot curls)
// facets [f0, f1): ptr holds the running entry counts relative to the range start
static void facet_curls_range(const InflatedMesh& im, int f0, int f1, FacetCurls& out)
{
    const SurfaceMesh& m = im.base;
    out.ptr.clear();
    out.ptr.reserve((size_t)(f1 - f0));
    out.dof.reserve((size_t)(f1 - f0) * 3);
    out.u.reserve((size_t)(f1 - f0) * 9);
    std::vector<std::pair<int, Vec3>> acc;
    for (int f = f0; f < f1; ++f) {
        acc.clear();
        const auto& t = m.facets[f];
        const Vec3 n = m.facet_normal(f);
        const double two_area = 2.0 * m.facet_measure(f);
        // n x e_k / (2A) is the same for both sides (computed once; same values)
        Vec3 g[3];
        for (int k = 0; k < 3; ++k) g[k] = cross(n, m.vertices[t[(k + 2) % 3]] - m.vertices[t[(k + 1) % 3]]) / two_area;
        for (int s = 0; s < 2; ++s) {
            const int o = 2 * f + s;
            for (int k = 0; k < 3; ++k) {
                const int v = t[k], b = im.ofacet_branch[o][k], q = im.q[v];
                if (q < 2) continue;
                const Vec3 curl = cross(im.onormal[o], g[k]);
                auto add = [&](int d, double w) {
                    for (auto& [dd, u] : acc)
                        if (dd == d) {
                            u = u + w * curl;
                            return;
                        }
                    acc.push_back({d, w * curl});
                };
                if (b < q - 1)
                    add(im.dof_index(v, b), 1.0);
                else
                    for (int j = 0; j + 1 < q; ++j) add(im.dof_index(v, j), -1.0);
            }
        }
        std::sort(acc.begin(), acc.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
        for (const auto& [d, u] : acc) {
            out.dof.push_back(d);
            out.u.push_back(u.x);
            out.u.push_back(u.y);
            out.u.push_back(u.z);
        }
        out.ptr.push_back((int)out.dof.size());
        out.kmax = std::max(out.kmax, (int)acc.size());
    }
}

// Facets are independent: large meshes split into contiguous ranges on a few threads,
// concatenated in facet order (the same lists as one pass).
FacetCurls facet_curls(const InflatedMesh& im)
{
    const int nf = im.base.num_facets();
    int want = std::thread::hardware_concurrency() >= 8 ? 4 : 1;
    if (const char* e = std::getenv("SBG_CURL_THREADS")) want = std::max(1, std::atoi(e));
    const int nt = std::min(want, std::max(1, nf / 2048));
    std::vector<FacetCurls> parts(std::max(nt, 1));
    if (nt <= 1) {
        facet_curls_range(im, 0, nf, parts[0]);
    } else {
        std::vector<std::thread> th;
        for (int i = 1; i < nt; ++i)
            th.emplace_back([&, i] { facet_curls_range(im, (int)((long long)nf * i / nt), (int)((long long)nf * (i + 1) / nt), parts[i]); });
        facet_curls_range(im, 0, (int)((long long)nf / nt), parts[0]);
        for (auto& t : th) t.join();
    }
    FacetCurls out;
    size_t ne = 0;
    for (const auto& p : parts) ne += p.dof.size();
    out.ptr.reserve((size_t)nf + 1);
    out.dof.reserve(ne);
    out.u.reserve(3 * ne);
    for (const auto& p : parts) {
        const int base = (int)out.dof.size();
        for (int c : p.ptr) out.ptr.push_back(base + c);
        out.dof.insert(out.dof.end(), p.dof.begin(), p.dof.end());
        out.u.insert(out.u.end(), p.u.begin(), p.u.end());
        out.kmax = std::max(out.kmax, p.kmax);
    }
    return out;
}

// reference: inc/gauss.hpp:16-52 (identical arithmetic; built with -ffp-contract=off)
Rule1d gauss_legendre(int n)
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

TriangleRule triangle_rule(int order)  // gauss.hpp:56-76
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

// reference: inc/quadrature.hpp:35-92 (same subdomain maps and point order)
void sauter_rules(int order, SauterRule& identical, SauterRule& edge, SauterRule& vertex)
{
    const Rule1d g = gauss_legendre(order);
    identical.pts.clear();
    edge.pts.clear();
    vertex.pts.clear();
    auto push = [](SauterRule& out, double x1, double x2, double y1, double y2, double w) {
        out.pts.insert(out.pts.end(), {x1 - x2, x2, y1 - y2, y2, w});
    };
    for (int i0 = 0; i0 < order; ++i0)
        for (int i1 = 0; i1 < order; ++i1)
            for (int i2 = 0; i2 < order; ++i2)
                for (int i3 = 0; i3 < order; ++i3) {
                    const double xi = g.x[i0], e1 = g.x[i1], e2 = g.x[i2], e3 = g.x[i3];
                    const double wp = g.w[i0] * g.w[i1] * g.w[i2] * g.w[i3];
                    const double xi3 = xi * xi * xi;
                    {
                        const double w = wp * xi3 * e1 * e1 * e2;
                        push(identical, xi, xi * (1 - e1 + e1 * e2), xi * (1 - e1 * e2 * e3), xi * (1 - e1), w);
                        push(identical, xi * (1 - e1 * e2 * e3), xi * (1 - e1), xi, xi * (1 - e1 + e1 * e2), w);
                        push(identical, xi, xi * e1 * (1 - e2 + e2 * e3), xi * (1 - e1 * e2), xi * e1 * (1 - e2), w);
                        push(identical, xi * (1 - e1 * e2), xi * e1 * (1 - e2), xi, xi * e1 * (1 - e2 + e2 * e3), w);
                        push(identical, xi * (1 - e1 * e2 * e3), xi * e1 * (1 - e2 * e3), xi, xi * e1 * (1 - e2), w);
                        push(identical, xi, xi * e1 * (1 - e2), xi * (1 - e1 * e2 * e3), xi * e1 * (1 - e2 * e3), w);
                    }
                    {
                        const double w1 = wp * xi3 * e1 * e1;
                        const double w2 = wp * xi3 * e1 * e1 * e2;
                        push(edge, xi, xi * e1 * e3, xi * (1 - e1 * e2), xi * e1 * (1 - e2), w1);
                        push(edge, xi, xi * e1, xi * (1 - e1 * e2 * e3), xi * e1 * e2 * (1 - e3), w2);
                        push(edge, xi * (1 - e1 * e2), xi * e1 * (1 - e2), xi, xi * e1 * e2 * e3, w2);
                        push(edge, xi * (1 - e1 * e2 * e3), xi * e1 * e2 * (1 - e3), xi, xi * e1, w2);
                        push(edge, xi * (1 - e1 * e2 * e3), xi * e1 * (1 - e2 * e3), xi, xi * e1 * e2, w2);
                    }
                    {
                        const double w = wp * xi3 * e2;
                        push(vertex, xi, xi * e1, xi * e2, xi * e2 * e3, w);
                        push(vertex, xi * e2, xi * e2 * e3, xi, xi * e1, w);
                    }
                }
}

}  // namespace sbg
