// sim.hpp — B200 Simulation: the reference's grafem::Simulation (solver.hpp:60-118) with all per-step
// state HBM-resident and every hot phase on the GPU (damage.cu, assemble.cu, cg.cu, misc.cu).
#pragma once

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../../include/grafem_b200.h"
#include "dev_types.cuh"
#include "host_mesh.hpp"
#include "host_viz.hpp"

namespace gfb {

struct Schedule {  // Schedule3 (collision.hpp:10-18)
  std::vector<double> t;
  std::vector<double> v;  // 3 per key
  void eval(double time, double out[3]) const;
  void rate(double time, double out[3]) const;
};

struct HostBc {
  int kind = 0;
  std::vector<int32_t> nodes;
  Schedule sched;
  double axis_point[3] = {0, 0, 0}, axis_dir[3] = {1, 0, 0};
  void displacement_params(double time, double d[3], double R[9]) const;
};

struct HostCollider {
  int kind = 0;
  Schedule center;
  double radius = 0, point[3] = {0, 0, 0}, normal[3] = {0, 0, 1}, stiffness = 1e6, restitution = 0, friction = 0;
};

class Simulation {
 public:
  Simulation(const HostMesh& mesh, const gf_material& mat, const gf_solver_config& cfg,
             const gf_boundary_condition* bcs, int32_t n_bcs, const gf_collider* cols, int32_t n_cols);
  ~Simulation();
  Simulation(const Simulation&) = delete;
  Simulation& operator=(const Simulation&) = delete;

  gf_step_stats dynamic_step();
  gf_step_stats quasi_static_step(double t_load);
  double newton_tolerance() const { return newton_tol_; }
  int32_t nonlocal_layout() const { return mat_.r_d <= 0.0 ? 0 : d_.nl_tpl == 2 ? 3 : d_.nl_tpl ? 2 : 1; }
  std::vector<int32_t> damage_pass();
  // Simulation::viz (solver.hpp:83-84): the render companion, created on first use (catching up on the edges
  // already broken); from then on every damage pass with newly broken edges feeds it (solver.cpp:94)
  RenderMesh& viz();
  void get_state(double* u, double* v, uint8_t* zeta, double* chi, double* time);
  void set_state(const double* u, const double* v, const uint8_t* zeta, const double* chi, const double* time,
                 bool async = false);
  void set_external_forces(const double* f3n);
  gf_sim_info info() const;
  uint64_t pattern_hash() const { return hash_; }
  int32_t dof_count() const { return 3 * mesh_.nn; }
  int64_t broken_edge_count();
  double last_collider_load() const { return last_load_; }
  void mass(double* m3n) const;
  double reaction_load(const int32_t* nodes, int32_t n, const double axis[3]);
  void energies(double* strain, double* kinetic);
  gf_step_metrics step_metrics();

  void eval_forces(double* f3n);
  void eval_stiffness(double* vals);
  void eval_cauchy(double* sigma6);
  void eval_screening(double* screening, double* sigma_f6, uint8_t* degenerate);
  void last_system(double* vals, double* rhs);
  void spmv(const double* x, double* y);
  void edge_forces(double* coeff6, uint8_t* ok);
  double assembly_energy();
  bool edge_form() const { return edge_form_; }
  void solve_system(const double* vals, const double* b, const double* x0, double tol, int32_t max_iters, double* x,
                    gf_cg_result* res);

  // 0 off; 1 CUDA events around every kernel; 2 events around the PCG solve only (the dominant kernel), launch
  // counts and algorithmic bytes for all -- per-kernel events cost ~3 % of the step at c3
  void set_profiling(int level) { profiling_ = level; }
  std::vector<gf_kernel_time> kernel_times();
  void reset_kernel_times() { ktimes_.clear(); }
  void synchronize();
  void timer_record(int slot);
  void cg_trace(unsigned long long* out);
  double timer_elapsed(int a, int b);

 private:
  template <class F>
  void launch(const char* name, double bytes, F&& f);
  void flush_events();
  void* dalloc(size_t bytes);
  void upload_bc_step(double t, double dt);
  void run_damage(bool relabel, bool keep_values, bool chi);
  void bsr_to_csr(const std::vector<double>& bval, double* vals) const;
  double run_cg(int max_iters);
  template <class Acc>
  void solve_ladder(bool ok, int32_t* iters, Acc&& account);
  double device_dot(const double* a, const double* b, int64_t n);
  double device_strain_energy();
  void device_metrics(double out[5]);
  void apply_boundary_displacements(double t);
  bool newton_solve(gf_step_stats& st);
  void launch_cg();
  void assemble(const StepCoeffs& c, int mode, const char* name, double bytes, bool energy_in_integrate = false);
  void fill_step_params(double t, double dt);
  void enqueue_step(double dt);
  void enqueue_prologue(double dt);
  gf_step_stats dynamic_step_full_newton();
  bool launch_step_graph(double dt);
  void check_edge_fallback();
  template <class Up>
  bool build_template_layout(const NonlocalTable& tb, Up&& up);
  template <class Up>
  bool build_cell_layout(const NonlocalTable& tb, int G, Up&& up);

  static constexpr bool kEdgeFormDefault = false;
  bool edge_form_ = false;
  HostMesh mesh_;
  NodePattern pat_;
  std::vector<int32_t> sell_ptr_;
  int64_t sell_slots_ = 0;
  int32_t zero_base_ = 0;
  std::vector<int32_t> usp_, uslot_;
  size_t bval_doubles_ = 0;
  gf_material mat_;
  gf_solver_config cfg_;
  MatDev md_{};
  std::vector<HostBc> bcs_;
  std::vector<HostCollider> cols_;
  std::vector<double> mass_;  // per node
  std::vector<double> fuser_;
  uint64_t hash_ = 0;
  int64_t nl_entries_ = 0;
  int64_t nl_tpl_slots_ = 0;
  int64_t nl_ell_slots_ = 0;
  double setup_s_[4] = {0, 0, 0, 0};
  double time_ = 0.0, last_load_ = 0.0;
  double newton_tol_ = 0.0, quasi_time_ = 0.0;
  double* d_usave_ = nullptr;    // line-search base displacements (quasi-static only, allocated on first use)
  double* d_ubackup_ = nullptr;  // last converged load increment
  double* h_partials_ = nullptr; // pinned, 8 doubles: reduction results read back
  int32_t n_fixed_ = 0;

  cudaStream_t stream_ = nullptr;
  DevData d_{};
  CgLaunch cg_{};
  double* d_slice_part_ = nullptr;
  unsigned long long* d_ctr_ = nullptr;
  int cg_ndyn_ = 0;  // dynamically handed-out PCG slices (cg_sell.cu Phase)
  double* d_tg_ = nullptr;  // cg_onchip.cu remote transposed products (null: the on-chip solver is not used)
  double* d_ocm_ = nullptr;  // cg_onchip.cu gathered-vector buffers
  uint32_t* d_oc_meta_ = nullptr;  // cg_onchip.cu per-row slot masks over oc_off_
  int32_t oc_off_[7] = {0, 0, 0, 0, 0, 0, 0};
  int64_t oc_slot_blocks_[7] = {0, 0, 0, 0, 0, 0, 0};
  std::vector<void*> allocs_;
  int32_t* d_fixed_nodes_ = nullptr;
  BcStep* d_bcstep_ = nullptr;
  ColliderDev* d_cols_ = nullptr;
  double* d_load_ = nullptr;
  double* d_energy_partials_ = nullptr;  // block partials of the device reductions (metrics.cu)
  unsigned* d_red_ticket_ = nullptr;
  double* d_red_out_ = nullptr;
  // pinned staging
  BcStep* h_bcstep_ = nullptr;
  ColliderDev* h_cols_ = nullptr;
  double* h_stats_ = nullptr;  // [cg_out(4), load, newly_count]
  double* d_stats_ = nullptr;  // the same record on the device
  std::unique_ptr<RenderMesh> viz_;
  void feed_viz(std::vector<int32_t> ids);  // newly broken ids (any order) of the damage pass just run
  // profiling
  int profiling_ = 0;
  struct Pending { std::string name; cudaEvent_t a, b; double bytes; };
  std::vector<Pending> pending_;
  std::vector<cudaEvent_t> event_pool_;
  std::map<std::string, gf_kernel_time> ktimes_;
  cudaEvent_t timers_[8] = {};
  // CUDA-graph step (dynamic_step): one executable per profiling level (0, 2), the captured (name, bytes) list
  bool graphs_enabled_ = true;
  bool capturing_ = false;
  int replayed_ = 0;
  cudaGraphExec_t step_exec_[2] = {nullptr, nullptr};
  std::vector<std::pair<std::string, double>> capture_list_, step_list_[2];
  cudaEvent_t pcg_ev_[2] = {nullptr, nullptr};
};

double measure_bandwidth(int kind, int64_t bytes, int reps);

void cg_solve_csr(int32_t n, const int32_t* row_ptr, const int32_t* cols, const double* vals, const double* b,
                  double* x, double tol, int32_t max_iters, gf_cg_result* res);

}  // namespace gfb
