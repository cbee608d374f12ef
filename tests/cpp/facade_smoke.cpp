// Compiles the header-only C++ facade against libgrafem_b200.so and exercises it the way a reference caller
// (grafem::Simulation user) would. Without a GPU, Simulation construction must throw CudaError (no fallback).
#include <cstdio>

#include "grafem_b200.hpp"

int main() {
  using namespace grafem_b200;
  const TetMesh mesh = TetMesh::make_box_mesh({0.08, 0.08, 0.32}, {8, 8, 32});
  if (mesh.num_tets() != 12288 || mesh.num_nodes() != 2673 || mesh.num_edges() != 16112) return 2;
  {  // render-side consumer (host only): split the mesh at one broken edge and rebuild its surface
    VizMesh viz(mesh);
    SimState st;
    st.displacements.assign(mesh.num_nodes(), Vec3{0.0, 0.0, 0.0});
    st.velocities = st.displacements;
    st.edge_damage.assign(mesh.num_edges(), 0);
    st.element_chi.assign(mesh.num_tets(), 1.0);
    const auto intact = viz.build_surface(st);
    st.edge_damage[0] = 1;
    viz.apply_splits({0}, st);
    const auto split = viz.build_surface(st);
    if (viz.children().empty() || split.triangles.size() <= intact.triangles.size()) return 4;
  }
  const gf_material mat = material_from_youngs(1e7, 0.3, 1000.0, 4.47e5);
  gf_solver_config cfg = default_solver_config();
  std::vector<int32_t> fixed;
  const auto X = mesh.rest_positions();
  for (int i = 0; i < mesh.num_nodes(); ++i)
    if (X[i][2] <= 1e-9) fixed.push_back(i);
  const double times[2] = {0.0, 1.0}, values[6] = {0, 0, 0, 0, 0, 0};
  gf_boundary_condition bc{};
  bc.kind = 0;
  bc.n_nodes = (int32_t)fixed.size();
  bc.nodes = fixed.data();
  bc.n_keys = 2;
  bc.key_times = times;
  bc.key_values = values;
  try {
    Simulation sim(mesh, mat, cfg, {bc});
    VizMesh& viz = sim.viz();  // solver.hpp:83: fed by every damage pass from here on
    for (int s = 0; s < 3; ++s) sim.dynamic_step();
    const SimState st = sim.state();
    viz.export_frame("/tmp/grafem_b200_facade.obj", st);
    std::printf("gpu: time=%g broken=%d hash=%llu\n", st.time, st.broken_edge_count(),
                (unsigned long long)sim.pattern_hash());
    return st.time > 0.0 ? 0 : 3;
  } catch (const CudaError& e) {
    std::printf("no gpu: %s\n", e.what());
    return 10;
  }
}
