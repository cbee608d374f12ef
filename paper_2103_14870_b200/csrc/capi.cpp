// capi.cpp — extern "C" boundary (include/grafem_b200.h). Exceptions -> status codes + thread-local
// message, mirroring the reference's FormatError / GeometryError / SolveError (types.hpp:17-29).
#include <cuda_runtime.h>

#include <cstring>
#include <memory>
#include <string>

#include "../../include/grafem_b200.h"
#include "host_mesh.hpp"
#include "host_viz.hpp"
#include "sim.hpp"

using namespace gfb;

struct gf_mesh {
  HostMesh m;
};
struct gf_viz {
  std::unique_ptr<RenderMesh> own;  // null for the simulation's own companion (borrowed: gf_sim_viz)
  RenderMesh* r;
  RenderMesh::Surface surf;
};
struct gf_sim {
  std::unique_ptr<Simulation> s;
  std::unique_ptr<gf_viz> viz;
};

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return GF_OK;
  } catch (const FormatError& e) {
    g_err = e.what();
    return GF_FORMAT_ERROR;
  } catch (const GeometryError& e) {
    g_err = e.what();
    return GF_GEOMETRY_ERROR;
  } catch (const SolveError& e) {
    g_err = e.what();
    return GF_SOLVE_ERROR;
  } catch (const CudaError& e) {
    g_err = e.what();
    return GF_CUDA_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return GF_INTERNAL_ERROR;
  }
}
}  // namespace

extern "C" {

const char* gf_last_error(void) { return g_err.c_str(); }
const char* gf_version(void) { return "grafem-b200 0.1.0 (sm_100a)"; }

int gf_mesh_create(const double* nodes_xyz, int32_t n_nodes, const int32_t* tets, int32_t n_tets, gf_mesh** out) {
  return guard([&] {
    *out = new gf_mesh{mesh_from_arrays(std::vector<double>(nodes_xyz, nodes_xyz + 3 * (size_t)n_nodes),
                                        std::vector<int32_t>(tets, tets + 4 * (size_t)n_tets))};
  });
}
int gf_mesh_make_box(const double size[3], const int32_t cells[3], const double origin[3], double jitter,
                     uint64_t seed, gf_mesh** out) {
  return guard([&] { *out = new gf_mesh{mesh_box(size, cells, origin, jitter, seed)}; });
}
int gf_mesh_load_tetgen(const char* node_text, const char* ele_text, gf_mesh** out) {
  return guard([&] { *out = new gf_mesh{mesh_tetgen(node_text, ele_text)}; });
}
void gf_mesh_destroy(gf_mesh* m) { delete m; }
void gf_mesh_counts(const gf_mesh* m, int32_t* nodes, int32_t* tets, int32_t* edges) {
  if (nodes) *nodes = m->m.nn;
  if (tets) *tets = m->m.nt;
  if (edges) *edges = m->m.ne;
}
void gf_mesh_get(const gf_mesh* mh, double* rest_xyz, int32_t* tets, int32_t* edges, int32_t* tet_edges,
                 double* volumes, double* binv9, double* centroids, double* rest_lengths) {
  const HostMesh& m = mh->m;
  auto cp = [](void* dst, const void* src, size_t bytes) {
    if (dst) std::memcpy(dst, src, bytes);
  };
  cp(rest_xyz, m.X.data(), 8 * m.X.size());
  cp(tets, m.tets.data(), 4 * m.tets.size());
  cp(edges, m.edges.data(), 4 * m.edges.size());
  cp(tet_edges, m.tet_edges.data(), 4 * m.tet_edges.size());
  cp(volumes, m.vol.data(), 8 * m.vol.size());
  cp(binv9, m.binv.data(), 8 * m.binv.size());
  cp(centroids, m.centroid.data(), 8 * m.centroid.size());
  cp(rest_lengths, m.rest_len.data(), 8 * m.rest_len.size());
}
double gf_mesh_mean_face_area(const gf_mesh* m) { return m->m.mean_face_area(); }
int64_t gf_mesh_pattern_nnz(const gf_mesh* m) {
  int64_t nnz = 0;
  guard([&] { nnz = make_node_pattern(m->m).scalar_nnz(); });
  return nnz;
}
uint64_t gf_mesh_pattern(const gf_mesh* m, int32_t* row_ptr, int32_t* cols) {
  uint64_t h = 0;
  guard([&] {
    const NodePattern p = make_node_pattern(m->m);
    p.scalar_csr(m->m.nn, row_ptr, cols);
    h = p.structure_hash(m->m.nn);
  });
  return h;
}
int64_t gf_mesh_nonlocal_table(const gf_mesh* m, double r_d, int32_t* ptr, int32_t* ids, double* w) {
  int64_t n = -1;
  guard([&] {
    const NonlocalTable t = make_nonlocal_table(m->m, r_d);
    n = (int64_t)t.ids.size();
    if (ptr)
      for (size_t i = 0; i < t.ptr.size(); ++i) ptr[i] = (int32_t)t.ptr[i];
    if (ids) std::memcpy(ids, t.ids.data(), 4 * t.ids.size());
    if (w) std::memcpy(w, t.w.data(), 8 * t.w.size());
  });
  return n;
}

int gf_material_from_youngs(double youngs, double poisson, double density, double sigma_thres, double r_d,
                            int32_t energy_model, gf_material* out) {
  return guard([&] {
    gf_material p;
    std::memset(&p, 0, sizeof p);
    p.youngs = youngs;
    p.poisson = poisson;
    p.density = density;
    p.sigma_thres = sigma_thres;
    p.r_d = r_d;
    p.energy_model = energy_model;
    p.mu = youngs / (2.0 * (1.0 + poisson));  // derive_lame (material.cpp:32-35)
    p.lambda = youngs * poisson / ((1.0 + poisson) * (1.0 - 2.0 * poisson));
    if (!(p.youngs > 0.0)) throw FormatError("youngs modulus must be positive");  // validate (material.cpp:37-43)
    if (!(p.poisson >= 0.0 && p.poisson < 0.5)) throw FormatError("poisson ratio must be in [0, 0.5)");
    if (!(p.density > 0.0)) throw FormatError("density must be positive");
    if (!(p.sigma_thres > 0.0)) throw FormatError("sigma_thres must be positive");
    if (!(p.r_d >= 0.0)) throw FormatError("r_d must be non-negative");
    if (energy_model != 0 && energy_model != 1) throw FormatError("unknown energy model");
    *out = p;
  });
}
void gf_solver_config_default(gf_solver_config* c) {
  std::memset(c, 0, sizeof *c);
  c->dt = 1e-3;
  c->newton_tol = 0.0;
  c->newton_max_iters = 40;
  c->cg_tol = 1e-8;
  c->cg_max_iters = 4000;
  c->ls_backtrack = 0.5;
  c->ls_sufficient_decrease = 1e-4;
  c->ls_max_halvings = 40;
  c->collision_substeps = 1;
}

int gf_sim_create(const gf_mesh* mesh, const gf_material* material, const gf_solver_config* config,
                  const gf_boundary_condition* bcs, int32_t n_bcs, const gf_collider* colliders, int32_t n_colliders,
                  gf_sim** out) {
  return guard([&] {
    auto h = std::make_unique<gf_sim>();
    h->s = std::make_unique<Simulation>(mesh->m, *material, *config, bcs, n_bcs, colliders, n_colliders);
    *out = h.release();
  });
}
void gf_sim_destroy(gf_sim* s) { delete s; }
int gf_sim_dynamic_step(gf_sim* s, gf_step_stats* stats) {
  return guard([&] {
    const gf_step_stats r = s->s->dynamic_step();
    if (stats) *stats = r;
  });
}
int gf_sim_quasi_static_step(gf_sim* s, double t_load, gf_step_stats* stats) {
  return guard([&] {
    const gf_step_stats r = s->s->quasi_static_step(t_load);
    if (stats) *stats = r;
  });
}
double gf_sim_newton_tolerance(const gf_sim* s) { return s->s->newton_tolerance(); }
int32_t gf_sim_nonlocal_layout(const gf_sim* s) { return s->s->nonlocal_layout(); }
int gf_sim_damage_pass(gf_sim* s, int32_t* ids, int64_t cap, int64_t* n) {
  return guard([&] {
    const auto v = s->s->damage_pass();
    if (n) *n = (int64_t)v.size();
    if (ids)
      for (int64_t i = 0; i < std::min<int64_t>(cap, (int64_t)v.size()); ++i) ids[i] = v[i];
  });
}
int gf_sim_get_state(gf_sim* s, double* u, double* v, uint8_t* zeta, double* chi, double* time) {
  return guard([&] { s->s->get_state(u, v, zeta, chi, time); });
}
int gf_sim_set_state(gf_sim* s, const double* u, const double* v, const uint8_t* zeta, const double* chi,
                     const double* time) {
  return guard([&] { s->s->set_state(u, v, zeta, chi, time); });
}
int gf_sim_set_state_async(gf_sim* s, const double* u, const double* v) {
  return guard([&] { s->s->set_state(u, v, nullptr, nullptr, nullptr, true); });
}
int gf_sim_set_external_forces(gf_sim* s, const double* f3n) {
  return guard([&] { s->s->set_external_forces(f3n); });
}
uint64_t gf_sim_pattern_hash(const gf_sim* s) { return s->s->pattern_hash(); }
int32_t gf_sim_dof_count(const gf_sim* s) { return s->s->dof_count(); }
int gf_sim_broken_edge_count(gf_sim* s, int64_t* n) {
  return guard([&] { *n = s->s->broken_edge_count(); });
}
double gf_sim_last_collider_load(const gf_sim* s) { return s->s->last_collider_load(); }
int gf_sim_mass(const gf_sim* s, double* m3n) {
  return guard([&] { s->s->mass(m3n); });
}
int gf_sim_reaction_load(gf_sim* s, const int32_t* nodes, int32_t n_nodes, const double axis[3], double* out) {
  return guard([&] { *out = s->s->reaction_load(nodes, n_nodes, axis); });
}
int gf_sim_energies(gf_sim* s, double* strain, double* kinetic) {
  return guard([&] { s->s->energies(strain, kinetic); });
}
int gf_sim_eval_forces(gf_sim* s, double* f3n) {
  return guard([&] { s->s->eval_forces(f3n); });
}
int gf_sim_eval_stiffness(gf_sim* s, double* vals) {
  return guard([&] { s->s->eval_stiffness(vals); });
}
int gf_sim_eval_cauchy(gf_sim* s, double* sigma6) {
  return guard([&] { s->s->eval_cauchy(sigma6); });
}
int gf_sim_eval_screening(gf_sim* s, double* screening, double* sigma_f6, uint8_t* degenerate) {
  return guard([&] { s->s->eval_screening(screening, sigma_f6, degenerate); });
}
int gf_sim_last_system(gf_sim* s, double* vals, double* rhs) {
  return guard([&] { s->s->last_system(vals, rhs); });
}
int gf_sim_spmv(gf_sim* s, const double* x, double* y) {
  return guard([&] { s->s->spmv(x, y); });
}
int gf_sim_solve_system(gf_sim* s, const double* vals, const double* b, const double* x0, double tol,
                        int32_t max_iters, double* x, gf_cg_result* res) {
  return guard([&] { s->s->solve_system(vals, b, x0, tol, max_iters, x, res); });
}
int gf_cg_solve_csr(int32_t n, const int32_t* row_ptr, const int32_t* cols, const double* vals, const double* b,
                    double* x, double tol, int32_t max_iters, gf_cg_result* res) {
  return guard([&] { cg_solve_csr(n, row_ptr, cols, vals, b, x, tol, max_iters, res); });
}
void* gf_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaMallocHost(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}
void gf_host_free(void* p) {
  if (p) cudaFreeHost(p);
}
int gf_sim_set_profiling(gf_sim* s, int32_t enable) {
  return guard([&] { s->s->set_profiling(enable < 0 || enable > 2 ? 1 : enable); });
}
int gf_sim_kernel_times(gf_sim* s, gf_kernel_time* out, int32_t cap, int32_t* n) {
  return guard([&] {
    const auto v = s->s->kernel_times();
    if (n) *n = (int32_t)v.size();
    for (int32_t i = 0; i < std::min<int32_t>(cap, (int32_t)v.size()); ++i) out[i] = v[i];
  });
}
int gf_sim_reset_kernel_times(gf_sim* s) {
  return guard([&] { s->s->reset_kernel_times(); });
}
int gf_sim_synchronize(gf_sim* s) {
  return guard([&] { s->s->synchronize(); });
}
int gf_sim_timer_record(gf_sim* s, int32_t slot) {
  return guard([&] { s->s->timer_record(slot); });
}
int gf_sim_timer_elapsed(gf_sim* s, int32_t a, int32_t b, double* ms) {
  return guard([&] { *ms = s->s->timer_elapsed(a, b); });
}
int gf_sim_cg_trace(gf_sim* s, uint64_t* out) {
  return guard([&] { s->s->cg_trace(reinterpret_cast<unsigned long long*>(out)); });
}
int gf_sim_edge_forces(gf_sim* s, double* coeff6, uint8_t* ok) {
  return guard([&] { s->s->edge_forces(coeff6, ok); });
}
int gf_sim_assembly_energy(gf_sim* s, double* energy) {
  return guard([&] { *energy = s->s->assembly_energy(); });
}
int32_t gf_sim_element_form(const gf_sim* s) { return s->s->edge_form() ? 1 : 0; }
int gf_sim_step_metrics(gf_sim* s, gf_step_metrics* out) {
  return guard([&] { *out = s->s->step_metrics(); });
}
int gf_sim_info_get(const gf_sim* s, gf_sim_info* out) {
  return guard([&] { *out = s->s->info(); });
}
int gf_measure_bandwidth(int32_t kind, int64_t bytes, int32_t reps, double* gbps) {
  return guard([&] { *gbps = measure_bandwidth(kind, bytes, reps); });
}
int gf_set_device(int32_t device) {
  return guard([&] {
    const cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) {
      cudaGetLastError();
      throw CudaError(std::string("cudaSetDevice: ") + cudaGetErrorString(e));
    }
  });
}
int gf_device_info(int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor, char* name, int32_t name_cap) {
  return guard([&] {
    int dev = 0;
    cudaDeviceProp prop;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaGetDeviceProperties(&prop, dev) != cudaSuccess) {
      cudaGetLastError();
      throw CudaError("no CUDA device");
    }
    if (sm_count) *sm_count = prop.multiProcessorCount;
    if (cc_major) *cc_major = prop.major;
    if (cc_minor) *cc_minor = prop.minor;
    if (name && name_cap > 0) {
      std::strncpy(name, prop.name, name_cap - 1);
      name[name_cap - 1] = 0;
    }
  });
}

// ---------------------------------------------------------------- render-side consumer (host_viz.hpp)
int gf_viz_create(const gf_mesh* mesh, gf_viz** out) {
  return guard([&] {
    auto own = std::make_unique<RenderMesh>(mesh->m);
    RenderMesh* r = own.get();
    *out = new gf_viz{std::move(own), r, {}};
  });
}
void gf_viz_destroy(gf_viz* v) {
  if (v && v->own) delete v;  // the simulation's own companion is released with the simulation
}
int gf_sim_viz(gf_sim* s, gf_viz** out) {
  return guard([&] {
    if (!s->viz) s->viz.reset(new gf_viz{nullptr, &s->s->viz(), {}});
    *out = s->viz.get();
  });
}
int gf_viz_apply_splits(gf_viz* v, const int32_t* newly_broken, int64_t n, const uint8_t* edge_damage) {
  return guard([&] { v->r->apply_splits(newly_broken, n, edge_damage); });
}
int64_t gf_viz_child_count(const gf_viz* v) { return (int64_t)v->r->children().size(); }
int gf_viz_child(const gf_viz* v, int64_t c, int32_t* kind, int32_t* entity, int32_t* rep, double rest_pos[3],
                 int32_t parents[4], int32_t* n_parents) {
  return guard([&] {
    if (c < 0 || c >= (int64_t)v->r->children().size()) throw FormatError("child index out of range");
    const RenderMesh::Child& ch = v->r->children()[c];
    if (kind) *kind = ch.kind;
    if (entity) *entity = ch.entity;
    if (rep) *rep = ch.rep;
    if (rest_pos)
      for (int a = 0; a < 3; ++a) rest_pos[a] = ch.rest[a];
    if (parents)
      for (size_t k = 0; k < ch.parents.size(); ++k) parents[k] = ch.parents[k];
    if (n_parents) *n_parents = (int32_t)ch.parents.size();
  });
}
int gf_viz_child_position(const gf_viz* v, int64_t c, const double* displacements, const uint8_t* edge_damage,
                          double out[3]) {
  return guard([&] {
    const auto p = v->r->child_position(c, displacements, edge_damage);
    for (int a = 0; a < 3; ++a) out[a] = p[a];
  });
}
int gf_viz_build_surface(gf_viz* v, const double* displacements, const uint8_t* edge_damage, int64_t* n_vertices,
                         int64_t* n_triangles, int64_t* n_original) {
  return guard([&] {
    v->surf = v->r->build_surface(displacements, edge_damage);
    if (n_vertices) *n_vertices = (int64_t)v->surf.xyz.size() / 3;
    if (n_triangles) *n_triangles = (int64_t)v->surf.tris.size();
    if (n_original) *n_original = v->surf.n_original;
  });
}
int gf_viz_surface(const gf_viz* v, double* vertices, int32_t* triangles) {
  return guard([&] {
    if (vertices) std::memcpy(vertices, v->surf.xyz.data(), 8 * v->surf.xyz.size());
    if (triangles) std::memcpy(triangles, v->surf.tris.data(), 12 * v->surf.tris.size());
  });
}
int gf_viz_export_frame(const gf_viz* v, const char* path, const double* displacements, const uint8_t* edge_damage) {
  return guard([&] { v->r->export_frame(path, displacements, edge_damage); });
}
int gf_viz_fragment_volumes(const gf_viz* v, int32_t tet, const double* displacements, const uint8_t* edge_damage,
                            double out[4]) {
  return guard([&] {
    const auto vol = v->r->fragment_volumes(tet, displacements, edge_damage);
    for (int k = 0; k < 4; ++k) out[k] = vol[k];
  });
}

}  // extern "C"
