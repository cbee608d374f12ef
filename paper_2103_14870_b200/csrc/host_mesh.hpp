// host_mesh.hpp — host-side setup for the B200 hot path: mesh build, rest quantities, the fixed
// system pattern (node-block CSR), node->tet incidence with CSR slot positions, and the non-local
// neighbour table. Runs once per Simulation; everything here is uploaded and stays HBM-resident.
//
// Floating point: compiled with -ffp-contract=off; the rest quantities follow the operation order
// of mesh.cpp:72-100 (Eigen det / 3x3 inverse / norm readings in DESIGN.md §3) so that B^-1, V,
// centroids, rest lengths and the table weights are bit-identical to the CPU oracle's.
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace gfb {

struct FormatError : std::runtime_error { using std::runtime_error::runtime_error; };
struct GeometryError : std::runtime_error { using std::runtime_error::runtime_error; };
struct SolveError : std::runtime_error { using std::runtime_error::runtime_error; };
struct CudaError : std::runtime_error { using std::runtime_error::runtime_error; };

// Tet local edge order 01,02,03,12,13,23 (mesh.hpp:41-42)
constexpr int kLocalEdge[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};

// TetMesh (mesh.hpp:15-43), flat arrays.
struct HostMesh {
  int32_t nn = 0, nt = 0, ne = 0;
  std::vector<double> X;            // 3*nn rest positions
  std::vector<int32_t> tets;        // 4*nt
  std::vector<int32_t> edges;       // 2*ne canonical (min,max), lexicographically sorted
  std::vector<int32_t> tet_edges;   // 6*nt in local edge order
  std::vector<int32_t> et_ptr, et_ids;  // edge -> incident tets, ascending tet id
  std::vector<double> vol;          // nt
  std::vector<double> binv;         // 9*nt row-major rest shape inverse
  std::vector<double> centroid;     // 3*nt
  std::vector<double> rest_len;     // ne
  double mean_face_area() const;
};

HostMesh mesh_from_arrays(std::vector<double> X, std::vector<int32_t> tets);
HostMesh mesh_box(const double size[3], const int32_t cells[3], const double origin[3], double jitter,
                  uint64_t seed);
HostMesh mesh_tetgen(const std::string& node_text, const std::string& ele_text);

// Fixed system pattern at node-block granularity. Row i lists the (sorted, unique) nodes sharing a tet
// with node i, itself included; the scalar CSR of make_system_pattern is its 3x3 expansion.
struct NodePattern {
  std::vector<int32_t> row_ptr;  // nn+1 (block offsets)
  std::vector<int32_t> cols;     // nb   (column node ids, ascending per row)
  std::vector<int32_t> diag;     // nn   (block index of the diagonal block)
  int32_t max_degree = 0;
  int64_t scalar_nnz() const { return 9 * (int64_t)cols.size(); }
  uint64_t structure_hash(int32_t nn) const;                  // == FixedPatternSparse::structure_hash
  void scalar_csr(int32_t nn, int32_t* row_ptr, int32_t* cols_out) const;
};
NodePattern make_node_pattern(const HostMesh& m);

// node -> (tet, packed column positions of the tet's 4 nodes within this node's block row)
struct NodeTets {
  std::vector<int32_t> ptr;    // nn+1
  std::vector<int32_t> tet;    // 4*nt, ascending tet id per node
  std::vector<uint32_t> slot;  // byte k = column position (in the node's row) of the tet's local node k
  int32_t max_valence = 0;
};
NodeTets make_node_tets(const HostMesh& m, const NodePattern& p);

// NonlocalTable (fracture.hpp:27-30) in CSR form, entries bit-identical to build_nonlocal_table.
struct NonlocalTable {
  std::vector<int64_t> ptr;
  std::vector<int32_t> ids;
  std::vector<double> w;
};
NonlocalTable make_nonlocal_table(const HostMesh& m, double r_d);

}  // namespace gfb
