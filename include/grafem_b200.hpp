// grafem_b200.hpp — header-only C++ facade over the C ABI (grafem_b200.h) with the shape of the reference's
// grafem::Simulation API (/root/reference/proj/include/grafem/solver.hpp:60-118): same class and method
// names, same exception types (types.hpp:17-29), AoS std::array<double,3> node vectors like the reference's
// Eigen::Vector3d (solver.cpp:62-72 dof order). A reference caller switches by replacing
//   #include "grafem/solver.hpp"     ->  #include "grafem_b200.hpp"
//   grafem::Simulation sim(...)      ->  grafem_b200::Simulation sim(...)
// and linking libgrafem_b200.so.
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "grafem_b200.h"

namespace grafem_b200 {

struct FormatError : std::runtime_error { using std::runtime_error::runtime_error; };
struct GeometryError : std::runtime_error { using std::runtime_error::runtime_error; };
struct SolveError : std::runtime_error { using std::runtime_error::runtime_error; };
struct CudaError : std::runtime_error { using std::runtime_error::runtime_error; };

inline void check(int rc) {
  if (rc == GF_OK) return;
  const std::string msg = gf_last_error();
  switch (rc) {
    case GF_FORMAT_ERROR: throw FormatError(msg);
    case GF_GEOMETRY_ERROR: throw GeometryError(msg);
    case GF_SOLVE_ERROR: throw SolveError(msg);
    case GF_CUDA_ERROR: throw CudaError(msg);
    default: throw std::runtime_error(msg);
  }
}

using Vec3 = std::array<double, 3>;

// TetMesh (mesh.hpp:15-43)
class TetMesh {
 public:
  static TetMesh make_mesh(const std::vector<Vec3>& nodes, const std::vector<std::array<int, 4>>& tets) {
    gf_mesh* m = nullptr;
    check(gf_mesh_create(nodes.empty() ? nullptr : nodes[0].data(), (int32_t)nodes.size(),
                         tets.empty() ? nullptr : tets[0].data(), (int32_t)tets.size(), &m));
    return TetMesh(m);
  }
  static TetMesh make_box_mesh(const Vec3& size, const std::array<int, 3>& cells, const Vec3& origin = {0, 0, 0},
                               double jitter = 0.0, uint64_t seed = 0) {
    gf_mesh* m = nullptr;
    const int32_t c[3] = {cells[0], cells[1], cells[2]};
    check(gf_mesh_make_box(size.data(), c, origin.data(), jitter, seed, &m));
    return TetMesh(m);
  }
  static TetMesh load_tetgen(const std::string& node_text, const std::string& ele_text) {
    gf_mesh* m = nullptr;
    check(gf_mesh_load_tetgen(node_text.c_str(), ele_text.c_str(), &m));
    return TetMesh(m);
  }
  int num_nodes() const { return counts()[0]; }
  int num_tets() const { return counts()[1]; }
  int num_edges() const { return counts()[2]; }
  int num_dofs() const { return 3 * num_nodes(); }
  std::vector<Vec3> rest_positions() const {
    std::vector<Vec3> x(num_nodes());
    gf_mesh_get(m_.get(), x[0].data(), nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
    return x;
  }
  const gf_mesh* raw() const { return m_.get(); }

 private:
  explicit TetMesh(gf_mesh* m) : m_(m, gf_mesh_destroy) {}
  std::array<int, 3> counts() const {
    int32_t n, t, e;
    gf_mesh_counts(m_.get(), &n, &t, &e);
    return {n, t, e};
  }
  std::shared_ptr<gf_mesh> m_;
};

// MaterialParams::from_youngs (material.hpp:14-31); energy model 0 stable_neo_hookean, 1 stvk
inline gf_material material_from_youngs(double E, double nu, double rho, double sigma_thres, double r_d = 0.0,
                                        int model = 0) {
  gf_material p;
  check(gf_material_from_youngs(E, nu, rho, sigma_thres, r_d, model, &p));
  return p;
}
inline gf_solver_config default_solver_config() {
  gf_solver_config c;
  gf_solver_config_default(&c);
  return c;
}

// SimState (fem.hpp:15-28) host copy
struct SimState {
  std::vector<Vec3> displacements, velocities;
  std::vector<uint8_t> edge_damage;
  std::vector<double> element_chi;
  double time = 0.0;
  int broken_edge_count() const {
    int n = 0;
    for (auto z : edge_damage) n += z;
    return n;
  }
};

class VizMesh;

// Simulation (solver.hpp:60-118)
class Simulation {
 public:
  Simulation(const TetMesh& mesh, const gf_material& material, const gf_solver_config& config,
             const std::vector<gf_boundary_condition>& bcs = {}, const std::vector<gf_collider>& colliders = {})
      : mesh_(mesh) {
    gf_sim* s = nullptr;
    check(gf_sim_create(mesh.raw(), &material, &config, bcs.data(), (int32_t)bcs.size(), colliders.data(),
                        (int32_t)colliders.size(), &s));
    s_.reset(s);
  }
  gf_step_stats dynamic_step() {  // solver.hpp:71
    gf_step_stats st;
    check(gf_sim_dynamic_step(s_.get(), &st));
    return st;
  }
  gf_step_stats quasi_static_step(double t_load) {  // solver.hpp:76
    gf_step_stats st;
    check(gf_sim_quasi_static_step(s_.get(), t_load, &st));
    return st;
  }
  double newton_tolerance() const { return gf_sim_newton_tolerance(s_.get()); }  // solver.hpp:96
  std::vector<int> damage_pass() {  // solver.hpp:67
    std::vector<int32_t> ids(mesh_.num_edges());
    int64_t n = 0;
    check(gf_sim_damage_pass(s_.get(), ids.data(), (int64_t)ids.size(), &n));
    return std::vector<int>(ids.begin(), ids.begin() + n);
  }
  SimState state() const {  // solver.hpp:79 (copy; see set_state for the mutable path of solver.hpp:80)
    SimState st;
    st.displacements.resize(mesh_.num_nodes());
    st.velocities.resize(mesh_.num_nodes());
    st.edge_damage.resize(mesh_.num_edges());
    st.element_chi.resize(mesh_.num_tets());
    check(gf_sim_get_state(s_.get(), st.displacements[0].data(), st.velocities[0].data(), st.edge_damage.data(),
                           st.element_chi.data(), &st.time));
    return st;
  }
  void set_state(const SimState& st) {
    check(gf_sim_set_state(s_.get(), st.displacements[0].data(), st.velocities[0].data(), st.edge_damage.data(),
                           st.element_chi.data(), &st.time));
  }
  std::uint64_t pattern_hash() const { return gf_sim_pattern_hash(s_.get()); }
  int dof_count() const { return gf_sim_dof_count(s_.get()); }
  double last_collider_load() const { return gf_sim_last_collider_load(s_.get()); }
  double broken_fraction() const {
    int64_t n = 0;
    check(gf_sim_broken_edge_count(s_.get(), &n));
    return mesh_.num_edges() ? (double)n / mesh_.num_edges() : 0.0;
  }
  double reaction_load(const std::vector<int>& nodes, const Vec3& axis) const {
    double out = 0.0;
    check(gf_sim_reaction_load(s_.get(), nodes.data(), (int32_t)nodes.size(), axis.data(), &out));
    return out;
  }
  std::vector<double> mass() const {
    std::vector<double> m(3 * (size_t)mesh_.num_nodes());
    check(gf_sim_mass(s_.get(), m.data()));
    return m;
  }
  const TetMesh& mesh() const { return mesh_; }
  VizMesh& viz();  // solver.hpp:83 (defined after VizMesh)

 private:
  struct Del {
    void operator()(gf_sim* s) const { gf_sim_destroy(s); }
  };
  TetMesh mesh_;
  std::unique_ptr<gf_sim, Del> s_;
  std::unique_ptr<VizMesh> viz_;
};

// VizMesh (viz.hpp:17-82): render-only companion mesh, host code; consumes damage_pass() / the state
class VizMesh {
 public:
  enum class EntityKind : int { edge = 0, face = 1, tet = 2 };
  struct Child {
    EntityKind kind;
    int entity, rep;
    Vec3 rest_pos;
    std::vector<int> parents_at_creation;
  };
  struct Surface {
    std::vector<Vec3> vertices;
    std::vector<std::array<int, 3>> triangles;
    int original_vertex_count = 0;
  };
  explicit VizMesh(const TetMesh& mesh) {
    gf_viz* v = nullptr;
    check(gf_viz_create(mesh.raw(), &v));
    v_.reset(v);
  }
  explicit VizMesh(gf_viz* borrowed) : v_(borrowed) {}  // a simulation's own companion (gf_sim_viz)
  void apply_splits(const std::vector<int>& newly_broken_edges, const SimState& state) {  // viz.cpp:183
    check(gf_viz_apply_splits(v_.get(), newly_broken_edges.data(), (int64_t)newly_broken_edges.size(),
                              state.edge_damage.data()));
  }
  std::vector<Child> children() const {  // viz.hpp:62 (copy)
    std::vector<Child> out((size_t)gf_viz_child_count(v_.get()));
    for (size_t c = 0; c < out.size(); ++c) {
      int32_t k = 0, e = 0, r = 0, p[4], n = 0;
      check(gf_viz_child(v_.get(), (int64_t)c, &k, &e, &r, out[c].rest_pos.data(), p, &n));
      out[c].kind = (EntityKind)k;
      out[c].entity = e;
      out[c].rep = r;
      out[c].parents_at_creation.assign(p, p + n);
    }
    return out;
  }
  Vec3 child_position(int child, const SimState& state) const {  // viz.cpp:197
    Vec3 p;
    check(gf_viz_child_position(v_.get(), child, state.displacements[0].data(), state.edge_damage.data(), p.data()));
    return p;
  }
  Surface build_surface(const SimState& state) const {  // viz.cpp:222
    int64_t nv = 0, nt = 0, no = 0;
    check(gf_viz_build_surface(v_.get(), state.displacements[0].data(), state.edge_damage.data(), &nv, &nt, &no));
    Surface s;
    s.vertices.resize(nv);
    s.triangles.resize(nt);
    check(gf_viz_surface(v_.get(), nv ? s.vertices[0].data() : nullptr, nt ? s.triangles[0].data() : nullptr));
    s.original_vertex_count = (int)no;
    return s;
  }
  void export_frame(const std::string& path, const SimState& state) const {  // viz.cpp:319
    check(gf_viz_export_frame(v_.get(), path.c_str(), state.displacements[0].data(), state.edge_damage.data()));
  }
  std::array<double, 4> fragment_volumes(int tet, const SimState& state) const {  // viz.cpp:333
    std::array<double, 4> v;
    check(gf_viz_fragment_volumes(v_.get(), tet, state.displacements[0].data(), state.edge_damage.data(), v.data()));
    return v;
  }

 private:
  struct Del {
    void operator()(gf_viz* v) const { gf_viz_destroy(v); }
  };
  std::unique_ptr<gf_viz, Del> v_;
};

inline VizMesh& Simulation::viz() {
  if (!viz_) {
    gf_viz* v = nullptr;
    check(gf_sim_viz(s_.get(), &v));
    viz_.reset(new VizMesh(v));
  }
  return *viz_;
}

}  // namespace grafem_b200
