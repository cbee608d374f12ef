// host_viz.hpp — render-side consumer of the GPU step's newly-broken edge lists.
//
// Replaces grafem::VizMesh (viz.hpp:17-82, viz.cpp:20-412): a render-only companion of the computational
// mesh. When edges break, the render mesh's edges, faces and tets split at their rest midpoints / centroids
// into per-corner pieces ("children"); a child follows the mean displacement of the computational nodes in
// its current bound group. The computational mesh and state are never touched. Host C++: it runs once per
// exported frame on the state the caller read back, and apply_splits consumes the ascending newly-broken list
// gf_sim_dynamic_step / gf_sim_damage_pass return. Output (vertex order, triangle order, OBJ bytes) follows
// the reference's deterministic rules: face ids in order of first appearance over (tet, local face),
// children in creation order, surface vertices = referenced original nodes ascending, then children.
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <unordered_map>
#include <vector>

#include "host_mesh.hpp"

namespace gfb {

class RenderMesh {
 public:
  enum Kind : int32_t { kEdge = 0, kFace = 1, kTet = 2 };

  struct Child {
    Kind kind;
    int32_t entity;                 // edge / face / tet id
    int32_t rep;                    // smallest node of the bound group at creation
    std::array<double, 3> rest;     // entity rest midpoint / centroid
    std::vector<int32_t> parents;   // bound group at creation (entity node order)
  };

  struct Surface {
    std::vector<double> xyz;                   // 3 per vertex
    std::vector<std::array<int32_t, 3>> tris;  // 0-based
    int64_t n_original = 0;                    // leading vertices bound 1:1 to nodes
  };

  explicit RenderMesh(HostMesh mesh);

  // VizMesh::apply_splits (viz.cpp:183-195): children required by this step's newly broken edges; idempotent
  void apply_splits(const int32_t* newly_broken, int64_t n, const uint8_t* zeta);
  // VizMesh::child_position (viz.cpp:197-203)
  std::array<double, 3> child_position(int64_t c, const double* u, const uint8_t* zeta) const;
  // VizMesh::build_surface (viz.cpp:222-317): exterior surface + open fracture surfaces
  Surface build_surface(const double* u, const uint8_t* zeta) const;
  // VizMesh::export_frame (viz.cpp:319-331): Wavefront OBJ, "v %.17g %.17g %.17g", 1-based "f"
  void export_frame(const std::string& path, const double* u, const uint8_t* zeta) const;
  // VizMesh::fragment_volumes (viz.cpp:333-412): volumes of the four corner fragments of one tet
  std::array<double, 4> fragment_volumes(int32_t tet, const double* u, const uint8_t* zeta) const;

  const std::vector<Child>& children() const { return children_; }
  const HostMesh& mesh() const { return m_; }
  int32_t face_count() const { return (int32_t)face_nodes_.size(); }

 private:
  // nodes of an entity in the reference's order: edge (min, max), face ascending, tet local order
  int nodes_of(Kind k, int32_t entity, int32_t out[4]) const;
  // the bound group of `node` inside the entity: its component over the entity's intact edges
  int group(Kind k, int32_t entity, int32_t node, const uint8_t* zeta, int32_t out[4]) const;
  int32_t group_rep(Kind k, int32_t entity, int32_t node, const uint8_t* zeta) const;
  std::array<double, 3> rest_point(Kind k, int32_t entity) const;
  std::array<double, 3> moved_point(Kind k, int32_t entity, int32_t side_node, const double* u,
                                    const uint8_t* zeta) const;
  void ensure_children(Kind k, int32_t entity, const uint8_t* zeta);
  int64_t handle(Kind k, int32_t entity, int32_t side_node, const uint8_t* zeta) const;
  int32_t face_edge(int32_t f, int32_t a, int32_t b) const;
  void edge_faces_in_tet(int32_t t, int32_t a, int32_t b, int32_t out[2]) const;
  static uint64_t key(Kind k, int32_t entity, int32_t rep) {
    return ((uint64_t)k << 62) | ((uint64_t)(uint32_t)entity << 31) | (uint64_t)(uint32_t)rep;
  }

  HostMesh m_;
  std::vector<std::array<int32_t, 3>> face_nodes_;  // ascending triple
  std::vector<std::array<int32_t, 3>> face_edges_;  // edges (0,1), (0,2), (1,2) of the triple
  std::vector<std::array<int32_t, 4>> tet_faces_;   // face id of local face k (opposite local node k)
  std::vector<int32_t> ef_ptr_, ef_ids_;            // edge -> faces, ascending face id
  std::vector<std::array<int32_t, 3>> boundary_;    // outward boundary triangles, ascending face id
  std::vector<int32_t> boundary_face_;              // parallel: face id
  std::unordered_map<uint64_t, int32_t> child_of_;
  std::vector<Child> children_;
};

}  // namespace gfb
