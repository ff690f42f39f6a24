// Host layer of the B200 screenbem path: meshes, config generators, inflation /
// DOF numbering, partition and prolongation.  Semantics follow the reference
// (proj/include/screenbem/{mesh,inflate,jump,schwarz}.hpp); the algorithms are
// re-done for scale (hash/grid based instead of the reference's O(nf^2) and
// O(V*E) loops) with identical outputs: DOF numbering, partition and R are
// parity-checked against the oracle bit for bit (tests/test_host_parity.py).
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

namespace sbg {

struct ValidationError : std::runtime_error {  // reference: inc/common.hpp:17-20
    explicit ValidationError(const std::string& m) : std::runtime_error(m) {}
};
struct NumericalError : std::runtime_error {  // reference: inc/common.hpp:23-26
    explicit NumericalError(const std::string& m) : std::runtime_error(m) {}
};
struct CudaError : std::runtime_error {
    explicit CudaError(const std::string& m) : std::runtime_error(m) {}
};

struct Vec3 {
    double x = 0, y = 0, z = 0;
    Vec3() = default;
    Vec3(double a, double b, double c) : x(a), y(b), z(c) {}
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
    return z > 0 ? a / std::sqrt(z) : a;
}

// reference: inc/mesh.hpp:19-83 (3-D triangles; the GPU path rejects dim 2)
struct SurfaceMesh {
    std::vector<Vec3> vertices;
    std::vector<std::array<int, 3>> facets;
    int num_vertices() const { return (int)vertices.size(); }
    int num_facets() const { return (int)facets.size(); }
    double facet_measure(int f) const;
    Vec3 facet_normal(int f) const;
    double facet_diameter(int f) const;
    Vec3 facet_centroid(int f) const;
    double max_facet_diameter() const;
    double diameter() const;
};

// reference: inc/mesh.hpp:86-92
struct MeshLevelPair {
    SurfaceMesh coarse, fine;
    std::vector<int> parent;
    double H = 0, h = 0;
};

void validate_mesh(const SurfaceMesh& m);                      // mesh.hpp:238-272 (grid-accelerated)
SurfaceMesh make_bowtie_base();                                // mesh.hpp:322-337
MeshLevelPair refine_uniform(const SurfaceMesh& m);            // mesh.hpp:342-386
MeshLevelPair refine_uniform_times(const SurfaceMesh& m, int k);  // mesh.hpp:388-405
SurfaceMesh make_builtin(const std::string& spec);             // mesh.hpp:516-537 (3-D builtins)

// BASELINE.json configs 1-5: panel generator with an
// explicit parent map for integer ratio r (non-dyadic r allowed).
MeshLevelPair make_config(int cfg, int ratio);
MeshLevelPair make_panels(int kind, int m, int r);  // 0 flat, 1 T-junction, 2 triple cross

// reference: inc/inflate.hpp:48-76
struct InflatedMesh {
    SurfaceMesh base;
    std::vector<Vec3> onormal;                   // oriented facet normals (2 per facet)
    std::vector<int> q, gv_first, dof_first;     // per vertex
    std::vector<std::array<int, 3>> ofacet_branch;
    std::vector<std::array<int, 2>> jump_dofs;
    std::vector<int> gv_vertex, gv_branch;       // per gvertex
    std::vector<int> gv_alpha_ptr, gv_alpha;     // sectors (oriented facet ids, ascending)
    int num_gvertices() const { return (int)gv_vertex.size(); }
    int num_jump_dofs() const { return (int)jump_dofs.size(); }
    int gv_index(int v, int b) const { return gv_first[v] + b; }
    int dof_index(int v, int b) const { return (q[v] < 2 || b >= q[v] - 1) ? -1 : dof_first[v] + b; }
};

InflatedMesh inflate(const SurfaceMesh& mesh, bool validate = true);  // inflate.hpp:98-288

// reference: inc/jump.hpp:87-89, CSC with ascending rows per column
struct Prolongation {
    int rows = 0, cols = 0;
    std::vector<int> col_ptr{0}, row_idx;
    std::vector<double> val;
};
Prolongation build_prolongation(const MeshLevelPair& pair, const InflatedMesh& coarse,
                                const InflatedMesh& fine);  // jump.hpp:118-185

// reference: inc/schwarz.hpp:14-17 (face_sets in ascending coarse-facet order)
struct DofPartition {
    std::vector<int> face_ids, face_ptr{0}, face_dofs, wirebasket;
};
DofPartition partition_dofs(const MeshLevelPair& pair, const InflatedMesh& fine);  // schwarz.hpp:19-51

// Per-facet side-merged curl coefficients of the jump basis: for facet f and
// jump DOF d, U[f,d] = sum_{side s, slot k, scatter term (d,w)} w * curl(2f+s, k)
// (reference: assemble.hpp:34-53 scatter, :83-89 slot curls).  Then
// W(a,b) = sum_{f,g} I(f,g) U[f,a].U[g,b] reproduces the loop at :109-127.
struct FacetCurls {
    int kmax = 0;                       // max entries per facet
    std::vector<int> ptr{0}, dof;       // CSR over facets, dofs ascending
    std::vector<double> u;              // 3 per entry
};
FacetCurls facet_curls(const InflatedMesh& im);

// Quadrature rules (reference: gauss.hpp:16-76, quadrature.hpp:35-92), host-built
// and uploaded so the device uses the very same nodes and weights.
struct Rule1d {
    std::vector<double> x, w;
};
Rule1d gauss_legendre(int n);
struct TriangleRule {
    std::vector<double> u, v, w;
};
TriangleRule triangle_rule(int order);
struct SauterRule {  // AoS a1,a2,b1,b2,w per point
    std::vector<double> pts;
    int size() const { return (int)(pts.size() / 5); }
};
void sauter_rules(int order, SauterRule& identical, SauterRule& edge, SauterRule& vertex);

}  // namespace sbg
