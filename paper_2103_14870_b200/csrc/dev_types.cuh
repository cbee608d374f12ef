// dev_types.cuh — HBM-resident data of one Simulation (plain device pointers) and kernel launchers.
//
// Layout: node vectors interleaved xyz (dof = 3*node+axis, 24 B contiguous per node so a
// gather is one sector); per-tet records AoS (B^-1 72 B, sigma 48 B) so scattered per-tet gathers are
// contiguous; the system matrix is a node-block CSR (BSR 3x3, row-major blocks, 72 B per block).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace gfb {

__host__ __device__ __forceinline__ size_t sell_addr(const int32_t* sell_ptr, int i, int c, int q) {
  return ((size_t)(sell_ptr[i >> 5] + c) * 9 + q) * 32 + (i & 31);
}
// value address of block (row i, CSR position c) for either format (symmetric: upper blocks only, c_u >= 0)

struct MatDev {
  double mu, lambda, alpha_nh;  // alpha_nh = 1 + mu/lambda - mu/(4 lambda) (material.cpp:65-67)
  double sigma_thres, chi_eps;  // chi_eps = 1e-12 * sigma_thres (fracture.cpp:132)
  int32_t model;                // 0 stable neo-hookean, 1 stvk
};

struct StepCoeffs {  // per-step scalars of solver.cpp:279-289
  double dt;
  double rhs_fint_scale;  // dt
  double rhs_mv_scale;    // dt*alpha
  double rhs_kv_scale;    // dt*beta + dt*dt
  double kscale;          // dt*beta + dt*dt
  double mscale;          // 1 + dt*alpha
  int32_t use_ext;        // 1: rhs includes f_ext + f_coll (dynamic); 0: internal forces only (quasi-static)
  int32_t fixed_zero;     // 1: Dirichlet rows prescribe 0 instead of fv (full-Newton iterations > 0, solver.cpp:291)
  const double* mdv;      // non-null: rhs -= M dv_total (full-Newton iterations > 0, solver.cpp:282)
};

// one entry per boundary condition, evaluated by the host each step (solver.cpp:22-29)
struct BcStep {
  int32_t kind;    // 0 translate, 1 rotate
  int32_t _pad;
  double d0[3], d1[3];   // translate: u(t), u(t+dt)
  double R0[9], R1[9];   // rotate: rotation matrices at t, t+dt (row-major)
  double axis_point[3];
};

struct ColliderDev {
  int32_t kind;  // 0 sphere, 1 halfspace
  int32_t _pad;
  double center[3], cvel[3];  // sphere centre / centre rate at the probe time
  double radius;
  double point[3], normal[3];
  double stiffness, restitution, friction;
};

struct DevData {
  int32_t nn, nt, ne, nb;  // nodes, tets, edges, node blocks (BSR nnz)
  // mesh (read-only)
  const double* X;          // 3nn
  const int4* tets;         // nt
  const double2* bv;        // 5nt: per tet B^-1 row-major (9 doubles) then V -- one 80-byte record, 5 x 16-byte loads
  const int32_t* tet_edges; // 6nt AoS
  const double* rest_len;   // ne
  int32_t rest_len_gt1;     // some rest length exceeds 1.0: build_T's degeneracy bound 1e-14 max(1, L) needs L
  const int32_t* et_ptr;    // ne+1 (edge -> tets, ascending)
  const int32_t* et_ids;
  const double* mass;       // nn (lumped node mass; all three dofs equal)
  const int32_t* node_bc;   // nn: bc index or -1
  // node -> tet incidence (ascending tet) with packed column slots
  const int32_t* nt_ptr;
  const int32_t* nt_tet;
  const int4* nt_nodes;     // per incidence entry: the tet's 4 node ids (a copy of tets[nt_tet]), so the assembly's
                            // displacement gathers issue with the tet's rest-record loads, one dependent round trip less
  // per block (CSR order) the contributions (pair l, local node k) as items l*4+k, ascending tet order
  const int32_t* contrib_ptr;  // nn+1: padded contribution items of row i start here (mx per column)
  const int32_t* big_rows;     // rows with > 32 incident tets or > 32 neighbour blocks (k_assemble_big)
  int32_t n_big;
  const uint8_t* contrib_item;
  // node-block pattern (CSR view: column ids per row, ascending)
  const int32_t* brow;      // nn+1
  const int32_t* bcol;      // nb
  // System matrix, symmetric SELL-32: slices of 32 consecutive node rows; only the upper blocks (j >= i) are
  // stored: slice s owns upper slots usp[s]..usp[s+1] (max upper degree of its rows), entry q of upper block
  // (i, c_u) at ((usp[i/32] + c_u) * 9 + q) * 32 + i%32, so a warp owning a slice reads every slot coalesced.
  // uslot[b] maps a CSR block (row i, column c) to c_u, or -1 when j < i (that block is (j,i)^T, stored by row
  // j). The SpMV slot list (SELL-32 over the full row in column order; slice s owns slots sell_ptr[s]..
  // sell_ptr[s+1]) holds packed (j << 6 | c) words (cg_sell.cu). For interior rows the neighbour offsets are
  // uniform across a slice, so both direct and transposed block reads coalesce.
  const int32_t* sell_ptr;  // nslices+1
  int32_t nslices;
  const int32_t* usp;       // nslices+1
  const int32_t* uslot;     // nb
  const uint32_t* sell_slot;  // 32 * total slots, packed (j << 6 | c) (cg_sell.cu)
  // non-local table (r_d > 0), sliced-ELL over 32 consecutive tets: entry j of tet e (slice s = e/32) is at
  // (nl_sptr[s] + j) * 32 + e%32, j < nl_len[e]; table order (ascending neighbour id) is preserved per tet
  const int64_t* nl_sptr;
  const int32_t* nl_len;
  const int32_t* nl_ids;
  const double* nl_w;
  // structured non-local layout (nl_tpl = 1; chosen at setup when the table is shift-invariant, e.g. box meshes):
  // a "template warp" holds 32 tets of one residue t = e mod 6 in consecutive cells q (e = 6 q + t); its slots
  // are the union of the lanes' neighbour shifts d = o - e in ascending order (so every lane still visits its
  // neighbours in table order). Slot j stores the sigma-plane position of lane 0's neighbour (lane k: + k) and
  // per lane the table weight (0 = not a neighbour of that lane). sigma_c is then stored in cell-major planes
  // (pos(e) = (e mod 6) * ncell + e / 6, three double2 planes) so the 32 lanes of a slot read 512 contiguous
  // bytes per plane instead of 32 scattered records.
  int32_t nl_tpl;
  int32_t nl_nwarps;
  int32_t nl_ncell;
  const int4* nl_warp;      // {t, q0, nlanes, first slot}; slot range ends at the next warp's first slot
  const int32_t* nl_spos;   // per slot
  const double* nl_tw;      // per (slot, lane)
  // cell template (nl_tpl = 2, the default structured layout): a warp holds G x 32 tets -- residues
  // [g G, g G + G) of 32 consecutive cells, one cell per lane (G = nl_group divides 6). Its slots are the union
  // over lanes and its residues of the neighbour offsets D = o - 6 q in ascending order (each tet still visits its
  // neighbours in table order); nl_cslot[slot] = {sigma-plane position of lane 0's neighbour, mask of the warp's
  // residues (bit t: residue g G + t) with a weight in this slot}; nl_tw then holds one 32-lane weight vector per
  // set mask bit, in slot-then-residue order, each warp's stream padded to a multiple of 8 vectors;
  // nl_warp = {q0, nlanes | g << 8, first slot, first weight vector}.
  const int2* nl_cslot;
  int32_t nl_group;
  int32_t* nl_flag;         // != 0: sigma_c holds a non-finite component (set by k_tet_stress, cleared by k_relabel)
  // state
  double* u;                // 3nn
  double* v;                // 3nn
  uint8_t* zeta;            // ne
  double* chi;              // nt
  // damage scratch
  double* sigc;             // 6nt
  double* sigf;             // 6nt
  uint8_t* deg;             // nt
  unsigned long long* scr_key;  // ne ordered-key max accumulator
  double* screening;        // ne (parity hooks only)
  int32_t* newly;           // ne
  int32_t* newly_count;     // 1
  // system
  double* bval;             // 9 * 32 * total slots (SELL-32 layout above)
  double* rhs;              // 3nn
  double* dinv;             // 3nn
  double* x;                // 3nn  (dv)
  double* fext;             // 3nn static part: m g + user load
  double* fcoll;            // 3nn collision part of the current step
  double* fv;               // 3nn fixed-dof prescribed dv (valid on BC nodes)
  double* utgt;             // 3nn pinned u(t+dt) (valid on BC nodes)
  double* vtgt;             // 3nn pinned v(t+dt)
  double* fint_out;         // 3nn optional (parity hook)
  double* absdiag;          // 3nn |diag| with fixed dofs zeroed (CG shift ladder)
  // CG work
  double* r;
  double* z;
  double* p0;
  double* Ap;
  double* cg_out;           // [iterations, converged, negcurv, relres]
  // edge-length element form (assemble.cu k_tet_edge; null = F-based row kernel)
  double* erec;             // 28 nt: chi V t_k (6), chi V M_kk' packed upper (21), fallback slot
  uint8_t* eflag;           // nt: 0 edge record, 1 F-based fallback rows, 2 no contribution (chi V = 0)
  double* efall;            // efall_cap x 4 rows x 39: F-based rows of the fallback tets
  int32_t* efall_tet;       // efall_cap
  int32_t* efall_count;     // 1 (device counter; the host reads it with the step's stats)
  int32_t efall_cap;
  double* eng_part;         // tet_edge_blocks(nt) block partials of the fused energy
  unsigned* eng_ticket;
  double* eng_out;          // total strain energy of the state the last assembly evaluated (both element forms)
  double* eng_row;          // nn: F-based form, per-row sums of the energies of the tets whose local node 0 is the row
  int32_t eng_sum;          // 1: k_integrate reduces eng_row into eng_out (F-based form's dynamic step)
  double* ecoef;            // 6 nt edge decomposition coefficients (parity hook)
  uint8_t* eok;             // nt
  // misc
  const BcStep* bcstep;
  const ColliderDev* colliders;
  int32_t n_colliders;
  double* coll_partials;
};

// ---- launchers (damage.cu, compiled with -fmad=false) ----
void launch_tet_stress(const DevData& d, const MatDev& m, bool local_screen, cudaStream_t s);
void launch_nonlocal(const DevData& d, cudaStream_t s);
void launch_relabel(const DevData& d, double sigma_thres, bool relabel, bool keep_values, cudaStream_t s);
void launch_chi(const DevData& d, const MatDev& m, cudaStream_t s);
void launch_reset_keys(const DevData& d, cudaStream_t s);
// ---- assemble.cu ----
enum AssembleMode { kAssembleSystem = 0, kAssembleRawK = 1, kAssembleForcesOnly = 2 };
void launch_assemble(const DevData& d, const MatDev& m, const StepCoeffs& c, int mode, cudaStream_t s);
int tet_edge_blocks(int nt);
// mode 0: edge records + fused energy (+ F-based fallback rows); mode 1: edge decomposition (ecoef, eok)
void launch_tet_edge(const DevData& d, const MatDev& m, int mode, cudaStream_t s);
// ---- cg.cu ----
struct CgLaunch {
  int32_t nrows;          // node rows (cg_sell.cu) or scalar rows (cg.cu)
  const int32_t* row_ptr; // cg_sell.cu: SELL-32 slice pointer (full-row slots); cg.cu: scalar CSR row pointer
  const int32_t* cols;    // cg_sell.cu: packed symmetric slots (uint32); cg.cu: CSR columns
  const double* vals;
  const double* b;
  double* x;
  const double* dinv;     // cg_sell.cu: from the assembly; cg.cu: computed from the diagonal
  double* r; double* z; double* p0; double* p1; double* Ap;  // p1: cg.cu only (double-buffered p)
  double* partials;       // cg.cu block partials
  double* out;            // [iterations, converged, negative_curvature, relative_residual]
  double tol;
  int32_t max_iters;
  int32_t nslices;        // cg_sell.cu: number of 32-row SELL slices
  const int32_t* usp;     // cg_sell.cu: upper-block slice pointer (slot decoding)
  int32_t zero_base;      // cg_sell.cu: value offset of the all-zero padding block
  const int32_t* cta_first;  // cg_sell.cu: slice range of each CTA (grid + 1 entries)
  unsigned long long* trace;  // optional per-phase %globaltimer stamps (GF_CG_TRACE)
  // cg_sell.cu: 1 when the initial guess is the assembly's projected one (prescribed values on Dirichlet rows,
  // zero elsewhere): those rows are identity rows and their columns are zero, so A x0 = x0 exactly (up to the
  // sign of zero) and the setup's SpMV is skipped. The solve_linear retries start from a solve's result: 0.
  int32_t x0_identity;
  int32_t pipelined;  // cg_sell.cu: 1 = the single-barrier pipelined solver (k_pcg_pipe) when the state fits on chip
  int32_t grid;       // cg_sell.cu: CTAs of the cooperative launch (0 = all co-resident)
  int32_t cluster;    // cg_sell.cu: 1 = the pipelined solve runs in ONE thread-block cluster of `grid` CTAs
  int32_t split;      // cg_sell.cu (cluster): warps sharing one slice's SpMV (1, 2, 3 or 4)
  int32_t onchip;     // cg_onchip.cu: 1 = the pipelined solve with the matrix held in TMEM + shared memory
  int32_t big;        // cg_sell.cu: 1 = the large-matrix instance k_pcg_big (round-robin static work, deferred x)
};
int cg_csr_grid();
void launch_pcg_csr(const CgLaunch& a, cudaStream_t s);  // scalar CSR (gf_cg_solve_csr)
// ---- cg_sell.cu (production solver on the symmetric SELL-32 matrix) ----
int pcg_sell_grid();
size_t pcg_sell_part_doubles(int ndyn);  // size of the partial work array (ndyn dynamic units)
int pcg_sell_warps_per_cta();
int pcg_dyn_warps_per_cta();  // the large-matrix instance's warps per CTA and co-resident CTAs
int pcg_dyn_grid();
int pcg_pipelined_default();  // GF_CG_PIPE (default 1)
int pcg_max_cluster();        // largest launchable cluster of the pipelined solver (0: none)
void launch_pcg_sell(const CgLaunch& a, double* part, int ndyn, unsigned long long* ctr, cudaStream_t s);
void launch_spmv_sym(const CgLaunch& a, const double* xin, double* y, cudaStream_t s);
// ---- cg_onchip.cu (the pipelined solve with the matrix on chip: at most 7 distinct positive column offsets (rows
// of <= 8 upper blocks), <= 24 slices per CTA, exactly symmetric diagonal blocks) ----
int pcg_onchip_grid();  // co-resident CTAs (0: not launchable on this device)
int pcg_onchip_max_cluster();  // largest launchable cluster of the on-chip solver (0: none)
int pcg_onchip_warps_per_cta();
int pcg_onchip_npad(int nslices);
size_t pcg_onchip_t_doubles(int nslices);  // the remote transposed-product buffers (zero-initialized)
size_t pcg_onchip_m_doubles(int nslices);  // the gathered vector's two buffers (zero-initialized)
// meta / off: the rows' structure over the matrix's (at most 7) distinct positive column offsets (cg_onchip.cu)
void launch_pcg_onchip(const CgLaunch& a, double* part, double* tg, double* gm, const uint32_t* meta,
                       const int32_t off[7], cudaStream_t s);
// ---- misc.cu ----
void launch_bc_targets(const DevData& d, int32_t n_fixed, const int32_t* fixed_nodes, double dt, cudaStream_t s);
int collide_blocks(const DevData& d);
void launch_collide(const DevData& d, int substep, double tau, double dt, int nsub, cudaStream_t s);
void launch_collide_load(const DevData& d, int nsub, double* out, cudaStream_t s);
void launch_integrate(const DevData& d, double dt, cudaStream_t s);
void launch_shift_diag(const DevData& d, double shift, cudaStream_t s);
void launch_absdiag(const DevData& d, cudaStream_t s);
void launch_bsr_dinv(const DevData& d, cudaStream_t s);
void launch_fill(double* p, double v, int64_t n, cudaStream_t s);
void launch_qs_bc(const DevData& d, int32_t n_fixed, const int32_t* fixed_nodes, cudaStream_t s);
void launch_qs_update(double* u, const double* saved, const double* dx, double step, int64_t n, cudaStream_t s);
// dynamic_full_newton (solver.cpp:296-303): dv_total += dv, v += dv, u = u_start + dt v; and the final BC pinning
void launch_newton_update(const DevData& d, double* dv_total, const double* u_start, double dt, cudaStream_t s);
void launch_pin_bc(const DevData& d, cudaStream_t s);
// ---- metrics.cu (device reductions; the last block writes the result) ----
size_t metrics_partial_doubles();
// out[0..4] = strain energy, kinetic energy, chi sum, broken edges, chi min
void launch_metrics(const DevData& d, const MatDev& m, double* partials, unsigned* ticket, double* out, cudaStream_t s);
void launch_dot(const double* a, const double* b, int64_t n, double* partials, unsigned* ticket, double* out,
                cudaStream_t s);

#ifdef __CUDACC__
// the tet's rest record: B^-1 (row-major) and volume V
__device__ __forceinline__ void load_rest(const DevData& d, int e, double B[9], double& vol) {
  const double2* r = d.bv + 5 * (size_t)e;
  const double2 a = __ldg(r), b = __ldg(r + 1), c = __ldg(r + 2), f = __ldg(r + 3), g = __ldg(r + 4);
  B[0] = a.x; B[1] = a.y; B[2] = b.x; B[3] = b.y; B[4] = c.x; B[5] = c.y; B[6] = f.x; B[7] = f.y; B[8] = g.x;
  vol = g.y;
}
#endif

}  // namespace gfb
