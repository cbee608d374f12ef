// A reference-style call site (the grafem namespace's value types, solver.hpp:15-118 / collision.hpp:10-34 /
// material.hpp:14-31) compiled against the B200 facade with only the include and namespace changed. Without a GPU,
// Simulation construction must throw CudaError (no CPU fallback).
#include <cstdio>

#include "grafem_b200.hpp"

namespace grafem = grafem_b200;  // the one line a reference caller changes besides the include

int main() {
  using grafem::Vec3;
  const grafem::TetMesh mesh = grafem::make_box_mesh(Vec3(0.08, 0.08, 0.32), {8, 8, 32});
  const auto material = grafem::MaterialParams::from_youngs(1e7, 0.3, 1000.0, 4.47e5, 0.0,
                                                           grafem::EnergyModel::stable_neo_hookean);
  if (!(material.mu > 0.0 && material.lambda > 0.0)) return 2;
  grafem::SolverConfig config;
  config.dt = 1e-3;
  config.gravity = Vec3(0.0, -9.81, 0.0);
  grafem::BoundaryCondition ends;
  ends.name = "ends";
  const auto X = mesh.rest_positions();
  for (int i = 0; i < mesh.num_nodes(); ++i)
    if (X[i][2] <= 1e-9 || X[i][2] >= 0.32 - 1e-9) ends.nodes.push_back(i);
  ends.translation = grafem::Schedule3::constant(Vec3::Zero());
  grafem::Collider floor;
  floor.kind = grafem::Collider::Kind::halfspace;
  floor.point = Vec3(0.0, -0.05, 0.0);
  floor.normal = Vec3::UnitY();
  floor.stiffness = 1e9;
  try {
    grafem::Simulation sim(mesh, material, config, {ends}, {floor});
    if (sim.material().youngs != 1e7 || sim.config().dt != 1e-3) return 5;
    grafem::StepStats st;
    for (int s = 0; s < 3; ++s) st = sim.dynamic_step();
    const gf_step_metrics m = sim.step_metrics();
    std::printf("gpu: cg=%d broken=%lld E=%g K=%g\n", st.cg_iterations, (long long)m.broken_edges, m.strain_energy,
                m.kinetic_energy);
    return st.cg_iterations > 0 ? 0 : 3;
  } catch (const grafem::CudaError& e) {
    std::printf("no gpu: %s\n", e.what());
    return 10;
  }
}
