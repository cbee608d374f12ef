/*
 * grafem_b200.h — C ABI of the B200-native grafem hot path (libgrafem_b200.so).
 *
 * Drop-in boundary for the reference's C++ simulator API (namespace grafem, /root/reference/proj).
 * The reference has no FFI layer of its own (bindings/module.cpp:1-2 is an empty pybind module), so
 * each entry point below names the C++ interface it replaces (file:line, paths under proj/).
 * A header-only C++ facade with the reference's class/exception shape is in grafem_b200.hpp.
 *
 * Conventions
 *  - Plain pointers and sizes only. Host arrays are AoS: node vectors double[3*N] (x,y,z per node,
 *    dof = 3*node+axis as in solver.cpp:62-72), per-tet six-vectors double[6*T], matrices row-major.
 *  - Every call that can fail returns GF_OK (0) or an error code; gf_last_error() returns a
 *    thread-local message. The error codes map to the reference's exception types
 *    (types.hpp:17-29): FormatError, GeometryError, SolveError.
 *  - A gf_sim owns one CUDA stream on the current device; calls are synchronous with respect to the
 *    host (state queries return consistent data), single-writer, not thread-safe.
 *  - No CPU fallback: if no sm_100 device is present gf_sim_create fails with GF_CUDA_ERROR.
 */
#ifndef GRAFEM_B200_H
#define GRAFEM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  GF_OK = 0,
  GF_FORMAT_ERROR = 1,   /* grafem::FormatError   (types.hpp:17) */
  GF_GEOMETRY_ERROR = 2, /* grafem::GeometryError (types.hpp:22) */
  GF_SOLVE_ERROR = 3,    /* grafem::SolveError    (types.hpp:27) */
  GF_CUDA_ERROR = 4,     /* device unavailable / CUDA runtime failure */
  GF_INTERNAL_ERROR = 5
};

/* grafem::MaterialParams (material.hpp:14-31). energy_model: 0 stable_neo_hookean, 1 stvk */
typedef struct {
  double youngs, poisson, density, mu, lambda, sigma_thres, r_d, damp_mass_coeff, damp_stiff_coeff;
  int32_t energy_model;
  int32_t _pad;
} gf_material;

/* grafem::SolverConfig (solver.hpp:15-31) */
typedef struct {
  double dt, newton_tol;
  int32_t newton_max_iters;
  int32_t cg_max_iters;
  double cg_tol, ls_backtrack, ls_sufficient_decrease;
  int32_t ls_max_halvings;
  int32_t dynamic_full_newton; /* must be 0: the full-Newton dynamic variant is outside the ported path */
  double gravity[3];
  int32_t collision_substeps;
  int32_t _pad;
} gf_solver_config;

/* grafem::BoundaryCondition (solver.hpp:35-47) with its Schedule3 (collision.hpp:10-18).
 * kind 0 translate (key_values = u(t)), 1 rotate (key_values[3k] = angle at key k). */
typedef struct {
  int32_t kind;
  int32_t n_nodes;
  const int32_t* nodes;
  int32_t n_keys;
  int32_t _pad;
  const double* key_times;
  const double* key_values;
  double axis_point[3];
  double axis_dir[3];
} gf_boundary_condition;

/* grafem::Collider (collision.hpp:20-34). kind 0 sphere (centre schedule in key_*), 1 halfspace */
typedef struct {
  int32_t kind;
  int32_t n_keys;
  const double* key_times;
  const double* key_values;
  double radius;
  double point[3];
  double normal[3];
  double stiffness, restitution, friction;
} gf_collider;

/* grafem::StepStats (solver.hpp:49-55) */
typedef struct {
  int32_t newton_iterations, cg_iterations, newly_broken, _pad;
  double residual, load;
} gf_step_stats;

/* grafem::CgResult (sparse.hpp:64-69) */
typedef struct {
  int32_t iterations, converged, negative_curvature, _pad;
  double relative_residual;
} gf_cg_result;

/* per-kernel device timing (CUDA events on the simulation stream), for bench/roofline */
typedef struct {
  char name[32];
  int64_t launches;
  double total_ms;
  double bytes; /* algorithmic bytes summed over launches */
} gf_kernel_time;

typedef struct gf_mesh gf_mesh;
typedef struct gf_sim gf_sim;
typedef struct gf_viz gf_viz;

const char* gf_last_error(void);
const char* gf_version(void);

/* ---------------------------------------------------------------- mesh (host setup) */
/* make_mesh (mesh.hpp:55-56, mesh.cpp:102-109): validates indices / orientation */
int gf_mesh_create(const double* nodes_xyz, int32_t n_nodes, const int32_t* tets, int32_t n_tets, gf_mesh** out);
/* make_box_mesh (primitives.hpp:12-13, primitives.cpp:71-79); jitter = amplitude in cell units applied
 * to interior nodes with the splitmix64 generator of DESIGN.md (0 = the reference's box exactly) */
int gf_mesh_make_box(const double size[3], const int32_t cells[3], const double origin[3], double jitter,
                     uint64_t seed, gf_mesh** out);
/* load_tetgen (mesh.hpp:59-61, mesh.cpp:157-221) */
int gf_mesh_load_tetgen(const char* node_text, const char* ele_text, gf_mesh** out);
void gf_mesh_destroy(gf_mesh* m);
void gf_mesh_counts(const gf_mesh* m, int32_t* nodes, int32_t* tets, int32_t* edges);
/* TetMesh fields (mesh.hpp:15-43); any pointer may be NULL. binv9 row-major per tet. */
void gf_mesh_get(const gf_mesh* m, double* rest_xyz, int32_t* tets, int32_t* edges, int32_t* tet_edges,
                 double* volumes, double* binv9, double* centroids, double* rest_lengths);
double gf_mesh_mean_face_area(const gf_mesh* m); /* TetMesh::mean_face_area (mesh.cpp:18-32) */
/* make_system_pattern + finalize (fem.cpp:140-149, sparse.cpp:13-25); returns structure_hash (sparse.cpp:71) */
int64_t gf_mesh_pattern_nnz(const gf_mesh* m);
uint64_t gf_mesh_pattern(const gf_mesh* m, int32_t* row_ptr, int32_t* cols);
/* build_nonlocal_table (fracture.cpp:32-54), grid-binned, identical entries; returns the entry count */
int64_t gf_mesh_nonlocal_table(const gf_mesh* m, double r_d, int32_t* ptr, int32_t* ids, double* w);

/* ---------------------------------------------------------------- parameters */
/* MaterialParams::from_youngs (material.cpp:17-30) */
int gf_material_from_youngs(double youngs, double poisson, double density, double sigma_thres, double r_d,
                            int32_t energy_model, gf_material* out);
void gf_solver_config_default(gf_solver_config* out); /* SolverConfig defaults (solver.hpp:15-31) */

/* ---------------------------------------------------------------- simulation */
/* Simulation::Simulation (solver.hpp:62-63, solver.cpp:31-60); the mesh is copied */
int gf_sim_create(const gf_mesh* mesh, const gf_material* material, const gf_solver_config* config,
                  const gf_boundary_condition* bcs, int32_t n_bcs, const gf_collider* colliders,
                  int32_t n_colliders, gf_sim** out);
void gf_sim_destroy(gf_sim* s);
/* Simulation::dynamic_step (solver.hpp:71, solver.cpp:219-333) */
int gf_sim_dynamic_step(gf_sim* s, gf_step_stats* stats);
/* Simulation::quasi_static_step (solver.hpp:76, solver.cpp:138-217): Newton + energy line search to the load
 * time t_load, load-increment halving (<= 10) on failure, then a damage pass; GF_SOLVE_ERROR like SolveError */
int gf_sim_quasi_static_step(gf_sim* s, double t_load, gf_step_stats* stats);
/* Simulation::newton_tolerance (solver.hpp:92, solver.cpp:57-59) */
double gf_sim_newton_tolerance(const gf_sim* s);
/* device layout of the non-local table: 0 local screening (r_d = 0), 1 general sliced-ELL
 * table, 2 structured per-tet template, 3 structured cell template (the default for shift-invariant numbering,
 * e.g. make_box_mesh); GF_NL_LAYOUT=general in the environment forces 1, GF_NL_LAYOUT=tet forces 2. Runtime
 * utility, no reference counterpart. */
int32_t gf_sim_nonlocal_layout(const gf_sim* s);
/* Simulation::damage_pass (solver.hpp:67, solver.cpp:90-103): ascending newly-broken edge ids */
int gf_sim_damage_pass(gf_sim* s, int32_t* ids, int64_t cap, int64_t* n);
/* Simulation::state() const / mutable (solver.hpp:79-80): SimState fields (fem.hpp:15-28); NULL skips */
int gf_sim_get_state(gf_sim* s, double* displacements, double* velocities, uint8_t* edge_damage,
                     double* element_chi, double* time);
int gf_sim_set_state(gf_sim* s, const double* displacements, const double* velocities,
                     const uint8_t* edge_damage, const double* element_chi, const double* time);
/* stream-ordered variant of gf_sim_set_state for pinned host buffers (gf_host_alloc): returns once the copies
 * are enqueued; the buffers must stay unchanged until the next synchronous call on the simulation (the next
 * step reads the new state). Runtime utility for zero-stall pipelines, no reference counterpart. */
int gf_sim_set_state_async(gf_sim* s, const double* displacements, const double* velocities);
/* external nodal load f_ext (3N, constant until reset; NULL clears). SPEC.md:397 hook; not in the
 * reference's solver.cpp:229-249, which only has gravity and colliders */
int gf_sim_set_external_forces(gf_sim* s, const double* f3n);
uint64_t gf_sim_pattern_hash(const gf_sim* s);                 /* solver.hpp:85 */
int32_t gf_sim_dof_count(const gf_sim* s);                     /* solver.hpp:86 */
int gf_sim_broken_edge_count(gf_sim* s, int64_t* n);           /* SimState::broken_edge_count (fem.cpp:16) */
double gf_sim_last_collider_load(const gf_sim* s);             /* solver.hpp:87 */
int gf_sim_mass(const gf_sim* s, double* mass3n);              /* Simulation::mass (solver.hpp:82) */
/* Simulation::reaction_load (solver.cpp:335-340) */
int gf_sim_reaction_load(gf_sim* s, const int32_t* nodes, int32_t n_nodes, const double axis[3], double* out);
/* total_strain_energy (fem.cpp:190-199) + kinetic_energy (fem.cpp:201-206) of the current state (device reductions) */
int gf_sim_energies(gf_sim* s, double* strain, double* kinetic);
/* the run loop's per-step row and damage-log statistics (run_scenario make_row / log_damage, scenario.cpp:640-672)
 * of the current state, computed on the device and read back as one record */
typedef struct {
  double strain_energy, kinetic_energy; /* total_strain_energy (fem.cpp:190-199), kinetic_energy (fem.cpp:201-206) */
  double chi_min, chi_mean;             /* log_damage's chi_min / chi_mean */
  int64_t broken_edges;                 /* SimState::broken_edge_count */
  double time;
} gf_step_metrics;
int gf_sim_step_metrics(gf_sim* s, gf_step_metrics* out);

/* ---------------------------------------------------------------- parity / microbench hooks */
int gf_sim_eval_forces(gf_sim* s, double* f3n);      /* assemble_forces (fem.cpp:96-108) */
int gf_sim_eval_stiffness(gf_sim* s, double* vals);  /* assemble_stiffness (fem.cpp:151-169), scalar-CSR order */
int gf_sim_eval_cauchy(gf_sim* s, double* sigma6);   /* per_tet_cauchy (solver.cpp:79-88) */
/* nonlocal_screen (fracture.cpp:56-91) on the current state: screening[E], sigma_f[6T], degenerate[T] */
int gf_sim_eval_screening(gf_sim* s, double* screening, double* sigma_f6, uint8_t* degenerate);
/* projected system matrix A (scalar-CSR order) and rhs of the last dynamic_step (solver.cpp:279-295) */
int gf_sim_last_system(gf_sim* s, double* vals, double* rhs);
/* y = A x with the current system matrix (FixedPatternSparse::multiply, sparse.cpp:49-60) */
int gf_sim_spmv(gf_sim* s, const double* x, double* y);
/* edge_decomposed_forces (fem.cpp:57-94) of every tet on the current state, from the edge-length element kernel:
 * coeff6[6 t + k] = magnitude of local edge k's force (f_i = sum_k c_k s_ik dir_k, s = +1 where the edge leaves node
 * i; rest volume, no chi -- the reference's convention), ok[t] = 0 on a current edge shorter than 1e-14 or a
 * degenerate (det C <= 0) element. */
int gf_sim_edge_forces(gf_sim* s, double* coeff6, uint8_t* ok);
/* element form of the assembly: 0 = F-based closed-form rows, 1 = edge-length form (GF_ELEMENT=edge at create) */
int32_t gf_sim_element_form(const gf_sim* s);
/* total_strain_energy (fem.cpp:190-199) of the state the last system assembly evaluated (the step-start state of the
 * last dynamic_step / Newton iterate), the fused by-product of the force pass (either element form) */
int gf_sim_assembly_energy(gf_sim* s, double* energy);
/* cg_solve (sparse.cpp:129-188) with the PRODUCTION solver (the persistent PCG on the symmetric SELL-32 matrix) on a
 * caller-provided matrix with this simulation's pattern: vals in the scalar-CSR order of gf_sim_eval_stiffness,
 * symmetric (the upper blocks are used); x0 NULL = zero guess. Replaces the simulation's current system. */
int gf_sim_solve_system(gf_sim* s, const double* vals, const double* b, const double* x0, double tol,
                        int32_t max_iters, double* x, gf_cg_result* res);
/* cg_solve (sparse.cpp:129-188) on a caller-provided scalar CSR, on the device */
int gf_cg_solve_csr(int32_t n, const int32_t* row_ptr, const int32_t* cols, const double* vals, const double* b,
                    double* x, double tol, int32_t max_iters, gf_cg_result* res);

/* ---------------------------------------------------------------- runtime utilities */
void* gf_host_alloc(size_t bytes); /* pinned host memory for zero-stall state transfers */
void gf_host_free(void* p);
/* per-kernel timing: 0 off, 1 CUDA events around every kernel, 2 events around the PCG solve only (launch counts
 * and algorithmic bytes for every kernel) */
int gf_sim_set_profiling(gf_sim* s, int32_t enable);
int gf_sim_kernel_times(gf_sim* s, gf_kernel_time* out, int32_t cap, int32_t* n);
int gf_sim_reset_kernel_times(gf_sim* s);
int gf_sim_synchronize(gf_sim* s);
/* CUDA events on the simulation's stream (device-side timing of whole steps): record slot 0..7, then read
 * the elapsed milliseconds between two recorded slots (synchronizes) */
int gf_sim_timer_record(gf_sim* s, int32_t slot);
int gf_sim_timer_elapsed(gf_sim* s, int32_t slot_a, int32_t slot_b, double* ms);
/* diagnostics: %globaltimer stamps of the last PCG solve (5000 words): CTA 0's 8 phase points per iteration
 * (< 200) at [8 it + point], per-CTA phase ends of iterations 10 and 20 at [2000 + cta], [3000 + cta], [4000 + cta]
 * (only when GF_CG_TRACE is set in the environment at gf_sim_create; tools/cg_trace.py, tools/cg_spread.py) */
int gf_sim_cg_trace(gf_sim* s, uint64_t* out);
/* ---------------------------------------------------------------- render-side consumer (host)
 * grafem::VizMesh (viz.hpp:17-82): render-only companion mesh that splits at broken edges. Host code, no GPU.
 * State arguments are the caller's read-back SimState pieces: displacements (3N, interleaved) and edge_damage
 * (E labels, canonical edge order) as returned by gf_sim_get_state. */
/* VizMesh::VizMesh (viz.cpp:20-66); keeps its own copy of the mesh */
int gf_viz_create(const gf_mesh* mesh, gf_viz** out);
void gf_viz_destroy(gf_viz* v);
/* Simulation::viz (solver.hpp:83-84): the simulation's own companion, created on first call (splitting at the
 * edges already broken) and from then on fed by every damage pass with newly broken edges (solver.cpp:94).
 * Borrowed: owned and released by the simulation (gf_viz_destroy ignores it). */
int gf_sim_viz(gf_sim* s, gf_viz** out);
/* VizMesh::apply_splits (viz.cpp:183-195): the step's newly broken edges (e.g. the ascending list of
 * gf_sim_damage_pass); GF_GEOMETRY_ERROR on an unknown edge id */
int gf_viz_apply_splits(gf_viz* v, const int32_t* newly_broken, int64_t n, const uint8_t* edge_damage);
/* VizMesh::children (viz.hpp:62): count, and child c's kind (0 edge, 1 face, 2 tet), entity, rep, rest
 * position and parents_at_creation (<= 4) */
int64_t gf_viz_child_count(const gf_viz* v);
int gf_viz_child(const gf_viz* v, int64_t c, int32_t* kind, int32_t* entity, int32_t* rep, double rest_pos[3],
                 int32_t parents[4], int32_t* n_parents);
/* VizMesh::child_position (viz.cpp:197-203) */
int gf_viz_child_position(const gf_viz* v, int64_t c, const double* displacements, const uint8_t* edge_damage,
                          double out[3]);
/* VizMesh::build_surface (viz.cpp:222-317): builds and keeps the surface; returns its sizes. Then
 * gf_viz_surface copies it out: vertices (3 per vertex) and 0-based triangles (3 per triangle). */
int gf_viz_build_surface(gf_viz* v, const double* displacements, const uint8_t* edge_damage, int64_t* n_vertices,
                         int64_t* n_triangles, int64_t* n_original);
int gf_viz_surface(const gf_viz* v, double* vertices, int32_t* triangles);
/* VizMesh::export_frame (viz.cpp:319-331): Wavefront OBJ; GF_FORMAT_ERROR when the file cannot be written */
int gf_viz_export_frame(const gf_viz* v, const char* path, const double* displacements, const uint8_t* edge_damage);
/* VizMesh::fragment_volumes (viz.cpp:333-412) */
int gf_viz_fragment_volumes(const gf_viz* v, int32_t tet, const double* displacements, const uint8_t* edge_damage,
                            double out[4]);

/* storage sizes and setup time of one simulation (roofline byte models). Runtime utility, no
 * reference counterpart: the reference's setup is Simulation::Simulation (solver.cpp:31-60). */
typedef struct {
  int64_t nodes, tets, edges;
  int64_t node_blocks;        /* 3x3 blocks of the full pattern (scalar nonzeros / 9) */
  int64_t upper_blocks;       /* blocks stored by the symmetric format: (node_blocks + nodes) / 2 */
  int64_t upper_block_slots;  /* stored block slots incl. SELL-32 padding (32 per slice slot) */
  int64_t spmv_slots;         /* 4-byte SpMV slot words incl. padding (32 per slice slot) */
  int64_t nl_entries;         /* non-local table entries S (T when r_d = 0) */
  int64_t nl_slots;           /* device table slots x 32 lanes (template or sliced-ELL, padding included); 0 local */
  int32_t nl_layout;          /* as gf_sim_nonlocal_layout */
  int32_t pcg_dynamic_units;  /* PCG slices handed out by ticket: 0 = solver state on chip for the whole solve */
  double setup_s[4];          /* wall seconds: [0] pattern + incidence + assembly lists + SELL layout,
                                 [1] non-local table (grid-binned build), [2] device layout + uploads, [3] ctor total */
  int32_t pcg_solver;         /* production PCG instance: 0 k_pcg_sell (two barriers), 1 k_pcg_pipe (grid), 2 k_pcg_pipe
                                 (one cluster), 3 k_pcg_onchip (matrix in TMEM + shared memory), 4 k_pcg_sell large-matrix,
                                 5 k_pcg_onchip in one cluster, 6 k_pcg_big (large matrices: round-robin static
                                 slices, one partial per CTA, x += alpha p deferred into the next SpMV phase) */
  int32_t _pad0;
  int64_t oc_slot_blocks[7];  /* k_pcg_onchip: upper off-diagonal blocks per slot (column offset oc_offsets[b]) */
  int32_t oc_offsets[7];      /* k_pcg_onchip: the pattern's positive column offsets (0 when not used) */
  int32_t _pad1;
} gf_sim_info;
int gf_sim_info_get(const gf_sim* s, gf_sim_info* out);
/* measured device bandwidth in GB/s on the current device: kind 0 = reads of an L2-resident buffer of `bytes`
 * (16-byte ld.global.cg from every SM, L1 bypassed, `reps` passes after one warm pass); kind 1 = HBM copy of
 * `bytes` (read + write bytes counted, like MEASURED_PEAKS.json). Roofline denominators for bench.py. */
int gf_measure_bandwidth(int32_t kind, int64_t bytes, int32_t reps, double* gbps);

/* select the CUDA device for subsequently created simulations (one process per GPU) */
int gf_set_device(int32_t device);
int gf_device_info(int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor, char* name, int32_t name_cap);

#ifdef __cplusplus
}
#endif
#endif
