// grafem_b200.hpp — header-only C++ facade over the C ABI (grafem_b200.h) with the shape of the reference's
// grafem API (/root/reference/proj/include/grafem): the value types MaterialParams / EnergyModel (material.hpp:10-31),
// SolverConfig, BoundaryCondition, StepStats (solver.hpp:15-55), Schedule3 and Collider (collision.hpp:10-34),
// TetMesh / SimState, the Simulation class (solver.hpp:60-118) with the same method names and accessors, and the
// same exception types (types.hpp:17-29). Vec3 is a 3-double value with Eigen::Vector3d's constructor and
// Zero()/UnitX()/UnitZ() spellings; node vectors are AoS in dof order 3 node + axis (solver.cpp:62-72). A reference
// caller switches by replacing
//   #include "grafem/solver.hpp"     ->  #include "grafem_b200.hpp"
//   namespace grafem                 ->  namespace grafem_b200
// and linking libgrafem_b200.so. The one semantic difference: state() returns a copy of the
// device-resident SimState; the reference's mutable state() reference becomes set_state(SimState).
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

// Eigen::Vector3d stand-in: Vec3(x, y, z), Vec3::Zero(), UnitX/Y/Z(), x()/y()/z(); contiguous (24 bytes)
struct Vec3 : std::array<double, 3> {
  Vec3() : std::array<double, 3>{{0.0, 0.0, 0.0}} {}
  Vec3(double x, double y, double z) : std::array<double, 3>{{x, y, z}} {}
  static Vec3 Zero() { return Vec3(); }
  static Vec3 UnitX() { return Vec3(1.0, 0.0, 0.0); }
  static Vec3 UnitY() { return Vec3(0.0, 1.0, 0.0); }
  static Vec3 UnitZ() { return Vec3(0.0, 0.0, 1.0); }
  double x() const { return (*this)[0]; }
  double y() const { return (*this)[1]; }
  double z() const { return (*this)[2]; }
};
static_assert(sizeof(Vec3) == 3 * sizeof(double), "Vec3 must stay a packed triple (AoS node vectors)");

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

// free-function construction, as mesh.hpp:55-61 and primitives.hpp:12-13 declare it
inline TetMesh make_mesh(const std::vector<Vec3>& nodes, const std::vector<std::array<int, 4>>& tets) {
  return TetMesh::make_mesh(nodes, tets);
}
inline TetMesh make_box_mesh(const Vec3& size, const std::array<int, 3>& cells, const Vec3& origin = Vec3::Zero()) {
  return TetMesh::make_box_mesh(size, cells, origin);
}
inline TetMesh load_tetgen(const std::string& node_text, const std::string& ele_text) {
  return TetMesh::load_tetgen(node_text, ele_text);
}

// EnergyModel / MaterialParams (material.hpp:10-31)
enum class EnergyModel : int { stable_neo_hookean = 0, stvk = 1 };

struct MaterialParams {
  double youngs = 1e6, poisson = 0.3, density = 1000.0;
  double mu = 0.0, lambda = 0.0;
  double sigma_thres = 1e5, r_d = 0.0;
  double damp_mass_coeff = 0.0, damp_stiff_coeff = 0.0;
  EnergyModel energy_model = EnergyModel::stable_neo_hookean;
  // MaterialParams::from_youngs (material.cpp:17-30): Lame parameters derived, ranges validated (FormatError)
  static MaterialParams from_youngs(double youngs, double poisson, double density, double sigma_thres,
                                    double r_d = 0.0, EnergyModel model = EnergyModel::stable_neo_hookean) {
    gf_material g;
    check(gf_material_from_youngs(youngs, poisson, density, sigma_thres, r_d, (int32_t)model, &g));
    return from_raw(g);
  }
  static MaterialParams from_raw(const gf_material& g) {
    MaterialParams p;
    p.youngs = g.youngs;
    p.poisson = g.poisson;
    p.density = g.density;
    p.mu = g.mu;
    p.lambda = g.lambda;
    p.sigma_thres = g.sigma_thres;
    p.r_d = g.r_d;
    p.damp_mass_coeff = g.damp_mass_coeff;
    p.damp_stiff_coeff = g.damp_stiff_coeff;
    p.energy_model = (EnergyModel)g.energy_model;
    return p;
  }
  gf_material raw() const {
    gf_material g{};
    g.youngs = youngs;
    g.poisson = poisson;
    g.density = density;
    g.mu = mu;
    g.lambda = lambda;
    g.sigma_thres = sigma_thres;
    g.r_d = r_d;
    g.damp_mass_coeff = damp_mass_coeff;
    g.damp_stiff_coeff = damp_stiff_coeff;
    g.energy_model = (int32_t)energy_model;
    return g;
  }
};

// SolverConfig (solver.hpp:15-31), the reference's defaults
struct SolverConfig {
  double dt = 1e-3;
  double newton_tol = 0.0;
  int newton_max_iters = 40;
  double cg_tol = 1e-8;
  int cg_max_iters = 4000;
  double ls_backtrack = 0.5;
  double ls_sufficient_decrease = 1e-4;
  int ls_max_halvings = 40;
  Vec3 gravity = Vec3::Zero();
  bool dynamic_full_newton = false;
  int collision_substeps = 1;
  gf_solver_config raw() const {
    gf_solver_config c;
    gf_solver_config_default(&c);
    c.dt = dt;
    c.newton_tol = newton_tol;
    c.newton_max_iters = newton_max_iters;
    c.cg_tol = cg_tol;
    c.cg_max_iters = cg_max_iters;
    c.ls_backtrack = ls_backtrack;
    c.ls_sufficient_decrease = ls_sufficient_decrease;
    c.ls_max_halvings = ls_max_halvings;
    for (int a = 0; a < 3; ++a) c.gravity[a] = gravity[a];
    c.dynamic_full_newton = dynamic_full_newton ? 1 : 0;
    c.collision_substeps = collision_substeps;
    return c;
  }
};

// Schedule3 (collision.hpp:10-18): piecewise-linear keyframes (evaluated on the device side of the library)
struct Schedule3 {
  std::vector<double> times;
  std::vector<Vec3> values;
  bool empty() const { return times.empty(); }
  static Schedule3 constant(const Vec3& v) { return Schedule3{{0.0}, {v}}; }
};

// BoundaryCondition (solver.hpp:35-47)
struct BoundaryCondition {
  enum class Kind { translate, rotate };
  Kind kind = Kind::translate;
  std::string name;
  std::vector<int> nodes;
  Schedule3 translation;
  Vec3 axis_point = Vec3::Zero();
  Vec3 axis_dir = Vec3::UnitX();
  Schedule3 angle;
};

// Collider (collision.hpp:20-34)
struct Collider {
  enum class Kind { sphere, halfspace };
  Kind kind = Kind::sphere;
  Schedule3 center;
  double radius = 0.0;
  Vec3 point = Vec3::Zero();
  Vec3 normal = Vec3::UnitZ();
  double stiffness = 1e6, restitution = 0.0, friction = 0.0;
};

// StepStats (solver.hpp:49-55)
struct StepStats {
  int newton_iterations = 0, cg_iterations = 0, newly_broken = 0;
  double residual = 0.0, load = 0.0;
};

// the C-struct forms (kept for C-ABI callers of the earlier facade)
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
      : mesh_(mesh), material_(MaterialParams::from_raw(material)) {
    gf_sim* s = nullptr;
    check(gf_sim_create(mesh.raw(), &material, &config, bcs.data(), (int32_t)bcs.size(), colliders.data(),
                        (int32_t)colliders.size(), &s));
    s_.reset(s);
    config_.dt = config.dt;
    config_.newton_tol = config.newton_tol;
    config_.newton_max_iters = config.newton_max_iters;
    config_.cg_tol = config.cg_tol;
    config_.cg_max_iters = config.cg_max_iters;
    config_.ls_backtrack = config.ls_backtrack;
    config_.ls_sufficient_decrease = config.ls_sufficient_decrease;
    config_.ls_max_halvings = config.ls_max_halvings;
    config_.gravity = Vec3(config.gravity[0], config.gravity[1], config.gravity[2]);
    config_.dynamic_full_newton = config.dynamic_full_newton != 0;
    config_.collision_substeps = config.collision_substeps;
  }
  // Simulation(TetMesh, MaterialParams, SolverConfig, vector<BoundaryCondition>, vector<Collider>) (solver.hpp:62-63)
  Simulation(const TetMesh& mesh, const MaterialParams& material, const SolverConfig& config,
             const std::vector<BoundaryCondition>& bcs = {}, const std::vector<Collider>& colliders = {})
      : mesh_(mesh), material_(material), config_(config), colliders_(colliders) {
    const gf_material m = material.raw();
    const gf_solver_config c = config.raw();
    std::vector<gf_boundary_condition> b(bcs.size());
    std::vector<std::vector<int32_t>> nodes(bcs.size());
    std::vector<std::vector<double>> kv(bcs.size() + colliders.size());
    for (size_t i = 0; i < bcs.size(); ++i) {
      const Schedule3& sc = bcs[i].kind == BoundaryCondition::Kind::translate ? bcs[i].translation : bcs[i].angle;
      nodes[i].assign(bcs[i].nodes.begin(), bcs[i].nodes.end());
      for (const Vec3& v : sc.values) kv[i].insert(kv[i].end(), v.begin(), v.end());
      b[i] = gf_boundary_condition{};
      b[i].kind = bcs[i].kind == BoundaryCondition::Kind::translate ? 0 : 1;
      b[i].n_nodes = (int32_t)nodes[i].size();
      b[i].nodes = nodes[i].data();
      b[i].n_keys = (int32_t)sc.times.size();
      b[i].key_times = sc.times.data();
      b[i].key_values = kv[i].data();
      for (int a = 0; a < 3; ++a) {
        b[i].axis_point[a] = bcs[i].axis_point[a];
        b[i].axis_dir[a] = bcs[i].axis_dir[a];
      }
    }
    std::vector<gf_collider> k(colliders.size());
    for (size_t i = 0; i < colliders.size(); ++i) {
      const Collider& q = colliders[i];
      std::vector<double>& v = kv[bcs.size() + i];
      for (const Vec3& x : q.center.values) v.insert(v.end(), x.begin(), x.end());
      k[i] = gf_collider{};
      k[i].kind = q.kind == Collider::Kind::sphere ? 0 : 1;
      k[i].n_keys = (int32_t)q.center.times.size();
      k[i].key_times = q.center.times.data();
      k[i].key_values = v.data();
      k[i].radius = q.radius;
      for (int a = 0; a < 3; ++a) {
        k[i].point[a] = q.point[a];
        k[i].normal[a] = q.normal[a];
      }
      k[i].stiffness = q.stiffness;
      k[i].restitution = q.restitution;
      k[i].friction = q.friction;
    }
    gf_sim* s = nullptr;
    check(gf_sim_create(mesh.raw(), &m, &c, b.data(), (int32_t)b.size(), k.data(), (int32_t)k.size(), &s));
    s_.reset(s);
  }
  StepStats dynamic_step() {  // solver.hpp:71
    gf_step_stats st;
    check(gf_sim_dynamic_step(s_.get(), &st));
    return to_stats(st);
  }
  StepStats quasi_static_step(double t_load) {  // solver.hpp:76
    gf_step_stats st;
    check(gf_sim_quasi_static_step(s_.get(), t_load, &st));
    return to_stats(st);
  }
  const MaterialParams& material() const { return material_; }  // solver.hpp:81
  const SolverConfig& config() const { return config_; }         // solver.hpp:82
  const std::vector<Collider>& colliders() const { return colliders_; }
  // run_scenario's per-step row + damage-log values as device reductions (scenario.cpp:640-672)
  gf_step_metrics step_metrics() {
    gf_step_metrics m;
    check(gf_sim_step_metrics(s_.get(), &m));
    return m;
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
  static StepStats to_stats(const gf_step_stats& g) {
    StepStats s;
    s.newton_iterations = g.newton_iterations;
    s.cg_iterations = g.cg_iterations;
    s.newly_broken = g.newly_broken;
    s.residual = g.residual;
    s.load = g.load;
    return s;
  }
  TetMesh mesh_;
  MaterialParams material_;
  SolverConfig config_;
  std::vector<Collider> colliders_;
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
