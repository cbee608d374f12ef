/*
 * oracle.h — C ABI of the CPU ORACLE (test infrastructure only).
 *
 * This library is a plain-C++ restatement of the reference grafem CPU hot path
 * (/root/reference/proj/src/{mesh,primitives,material,fem,fracture,sparse,solver,collision}.cpp).
 * It exists ONLY as the parity checker and the CPU baseline: tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it. The product
 * (paper_2103_14870_b200, libgrafem_b200.so) never links or calls it.
 *
 * Matrices crossing this ABI are row-major double[9] (a[3*r+c]); vectors are AoS
 * double[3*n]; per-tet six-vectors are AoS double[6*T].
 */
#ifndef GRAFEM_ORACLE_H
#define GRAFEM_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_OK = 0, OR_FORMAT_ERROR = 1, OR_GEOMETRY_ERROR = 2, OR_SOLVE_ERROR = 3, OR_INTERNAL_ERROR = 5 };

/* Same layout as gf_material / gf_solver_config / gf_boundary_condition / gf_collider
 * in include/grafem_b200.h so one ctypes definition serves both libraries. */
typedef struct {
  double youngs, poisson, density, mu, lambda, sigma_thres, r_d, damp_mass_coeff, damp_stiff_coeff;
  int32_t energy_model; /* 0 stable_neo_hookean, 1 stvk */
  int32_t _pad;
} or_material;

typedef struct {
  double dt, newton_tol;
  int32_t newton_max_iters;
  int32_t cg_max_iters;
  double cg_tol, ls_backtrack, ls_sufficient_decrease;
  int32_t ls_max_halvings;
  int32_t dynamic_full_newton;
  double gravity[3];
  int32_t collision_substeps;
  int32_t _pad;
} or_solver_config;

typedef struct {
  int32_t kind; /* 0 translate, 1 rotate */
  int32_t n_nodes;
  const int32_t* nodes;
  int32_t n_keys;
  int32_t _pad;
  const double* key_times;  /* n_keys */
  const double* key_values; /* 3*n_keys (rotate: x holds the angle) */
  double axis_point[3];
  double axis_dir[3];
} or_boundary_condition;

typedef struct {
  int32_t kind; /* 0 sphere, 1 halfspace */
  int32_t n_keys;
  const double* key_times;
  const double* key_values; /* sphere centre schedule */
  double radius;
  double point[3];
  double normal[3];
  double stiffness, restitution, friction;
} or_collider;

typedef struct {
  int32_t newton_iterations, cg_iterations, newly_broken, _pad;
  double residual, load;
} or_step_stats;

typedef struct {
  int32_t iterations, converged, negative_curvature, _pad;
  double relative_residual;
} or_cg_result;

typedef struct or_mesh or_mesh;
typedef struct or_sim or_sim;

const char* or_last_error(void);
int or_num_threads(void);
void or_set_num_threads(int n);

/* ---- mesh (mesh.cpp:34-109, primitives.cpp:13-79) ---- */
int or_mesh_create(const double* nodes, int32_t n_nodes, const int32_t* tets, int32_t n_tets, or_mesh** out);
int or_mesh_make_box(const double size[3], const int32_t cells[3], const double origin[3],
                     double jitter, uint64_t seed, or_mesh** out);
int or_mesh_load_tetgen(const char* node_text, const char* ele_text, or_mesh** out);
void or_mesh_destroy(or_mesh* m);
void or_mesh_counts(const or_mesh* m, int32_t* nodes, int32_t* tets, int32_t* edges);
void or_mesh_get(const or_mesh* m, double* rest_xyz, int32_t* tets, int32_t* edges, int32_t* tet_edges,
                 double* volumes, double* binv9, double* centroids, double* rest_lengths);
int64_t or_mesh_edge_tets(const or_mesh* m, int32_t* ptr, int32_t* ids);
double or_mesh_mean_face_area(const or_mesh* m);

/* ---- material point functions (material.cpp:17-135) ---- */
int or_material_from_youngs(double E, double nu, double rho, double sigma_thres, double r_d, int32_t model,
                            or_material* out);
double or_energy_density(const double F[9], const or_material* p);
void or_pk1(const double F[9], const or_material* p, double P[9]);
void or_pk1_differential(const double F[9], const double dF[9], const or_material* p, double out[9]);
int or_cauchy_sixvector(const double F[9], const or_material* p, double out[6]); /* returns pk1_fallback */

/* ---- fem (fem.cpp) : state arrays are AoS u[3N], chi[T] ---- */
void or_deformation_gradient(const or_mesh* m, const double* u, int32_t tet, double F[9]);
void or_element_internal_force(const or_mesh* m, const double* u, const double* chi, const or_material* p,
                               int32_t tet, double f[12]);
/* edge_decomposed_forces (fem.cpp:57-94): returns ok (1/0); coeff[6], residual */
int or_edge_decomposed_forces(const or_mesh* m, const double* u, const or_material* p, int32_t tet, double coeff[6],
                              double* residual);
void or_element_stiffness(const or_mesh* m, const double* u, const double* chi, const or_material* p,
                          int32_t tet, double k[144]);
void or_assemble_forces(const or_mesh* m, const double* u, const double* chi, const or_material* p, double* f);
int64_t or_pattern_nnz(const or_mesh* m);
uint64_t or_pattern(const or_mesh* m, int32_t* row_ptr, int32_t* cols); /* returns structure_hash */
void or_assemble_stiffness(const or_mesh* m, const double* u, const double* chi, const or_material* p,
                           double* vals);
void or_lumped_mass(const or_mesh* m, const or_material* p, double* mass3n);
double or_total_strain_energy(const or_mesh* m, const double* u, const double* chi, const or_material* p);

/* ---- fracture (fracture.cpp) ---- */
int or_build_T(const or_mesh* m, const double* u, int32_t tet, double T[36]);
int64_t or_nonlocal_table(const or_mesh* m, double r_d, int32_t brute_force, int32_t* ptr, int32_t* ids,
                          double* w);
void or_per_tet_cauchy(const or_mesh* m, const double* u, const or_material* p, double* sigma6);
void or_nonlocal_screen(const or_mesh* m, const double* u, const double* sigma6, double r_d,
                        double* screening, double* sigma_f6, uint8_t* degenerate);
int32_t or_update_damage(uint8_t* zeta, int32_t n_edges, const double* screening, double sigma_thres,
                         int32_t* newly);
void or_compute_chi(const or_mesh* m, const uint8_t* zeta, const double* sigma_f6, const or_material* p,
                    double* chi);
int32_t or_fragment_components(const or_mesh* m, const uint8_t* zeta, int32_t tet, int32_t labels[4]);

/* ---- sparse (sparse.cpp) on a caller-owned scalar CSR ---- */
void or_spmv_csr(int32_t n, const int32_t* row_ptr, const int32_t* cols, const double* vals, const double* x,
                 double* y);
void or_cg_solve_csr(int32_t n, const int32_t* row_ptr, const int32_t* cols, const double* vals,
                     const double* b, double* x, double tol, int32_t max_iters, or_cg_result* res);
void or_project_dirichlet_csr(int32_t n, const int32_t* row_ptr, const int32_t* cols, double* vals,
                              const int32_t* dofs, int32_t n_dofs, const double* values, double* rhs);

/* ---- simulation (solver.cpp) ---- */
/* collision.cpp:8-111 (Schedule3::eval/rate, Collider::validate, detect_and_respond); counts = {contact_count,
   deep_penetrations} */
void or_schedule_eval(int32_t n_keys, const double* times, const double* values, double t, double val[3],
                      double rate[3]);
int or_collider_validate(const or_collider* c);
int or_detect_and_respond(const or_mesh* mesh, const double* u, const double* v, const double* mass3n,
                          const or_collider* cols, int32_t n_cols, double t, double dt, double* force3n,
                          double* per_collider, int32_t counts[2], double* max_depth);

int or_sim_create(const or_mesh* mesh, const or_material* mat, const or_solver_config* cfg,
                  const or_boundary_condition* bcs, int32_t n_bcs, const or_collider* cols, int32_t n_cols,
                  or_sim** out);
void or_sim_destroy(or_sim* s);
void or_solver_config_default(or_solver_config* c);
int or_sim_dynamic_step(or_sim* s, or_step_stats* stats);
int or_sim_damage_pass(or_sim* s, int32_t* ids, int64_t cap, int64_t* n);
void or_sim_get_state(const or_sim* s, double* u, double* v, uint8_t* zeta, double* chi, double* time);
void or_sim_set_state(or_sim* s, const double* u, const double* v, const uint8_t* zeta, const double* chi,
                      const double* time);
void or_sim_set_external_forces(or_sim* s, const double* f3n);
uint64_t or_sim_pattern_hash(const or_sim* s);
double or_sim_last_collider_load(const or_sim* s);
void or_sim_mass(const or_sim* s, double* m3n);
/* system matrix A and rhs of the last dynamic_step (after projection), for parity of the assembly */
void or_sim_last_system(const or_sim* s, double* vals, double* rhs);
/* per-phase wall times (seconds) accumulated over dynamic_step calls: damage, assembly, solve, other */
void or_sim_phase_times(const or_sim* s, double t[4]);
int or_sim_quasi_static_step(or_sim* s, double t_load, or_step_stats* stats); /* solver.cpp:138-217 */
double or_sim_newton_tolerance(const or_sim* s);

#ifdef __cplusplus
}
#endif
#endif
