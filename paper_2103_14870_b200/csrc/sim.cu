// sim.cu — host orchestration of the B200 Simulation (solver.cpp:31-333 restated B200-first).
//
// Per dynamic_step (solver.cpp:219-333) the host issues, on one stream and with no intermediate sync:
//   damage    k_tet_stress [+ k_nonlocal_tpl | k_nonlocal] -> k_relabel -> k_chi  (solver.cpp:225, 90-103)
//   f_ext     [k_collide x substeps -> k_collide_load]                        (solver.cpp:229-250)
//   BCs       k_bc_targets                                                    (solver.cpp:255-262)
//   system    k_assemble (forces, K, K v, rhs, A, projection, D^-1, x0)       (solver.cpp:275-295)
//   solve     k_pcg_sell (one cooperative kernel for the whole CG)            (solver.cpp:105-136)
//   update    k_integrate (v += dv, u += dt v, pin; no-op unless converged)   (solver.cpp:296-328)
// and reads back one 48-byte stats record (CG result, newly-broken count, collider load); the
// reference's retry/shift ladder (solver.cpp:110-135) runs only when that record says the CG failed, after
// which the integration is enqueued again. quasi_static_step (solver.cpp:138-217) reuses the same kernels.
#include "sim.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <sstream>

namespace gfb {

#define GF_CUDA(x)                                                                          \
  do {                                                                                      \
    const cudaError_t _e = (x);                                                             \
    if (_e != cudaSuccess) throw CudaError(std::string(#x) + ": " + cudaGetErrorString(_e)); \
  } while (0)

void launch_reset_x(const DevData& d, cudaStream_t s);

// ---------------------------------------------------------------- schedules / BCs (host, per step)
void Schedule::eval(double time, double out[3]) const {  // Schedule3::eval (collision.cpp:8-18)
  if (t.empty()) {
    out[0] = out[1] = out[2] = 0.0;
    return;
  }
  if (time <= t.front()) {
    for (int a = 0; a < 3; ++a) out[a] = v[a];
    return;
  }
  if (time >= t.back()) {
    for (int a = 0; a < 3; ++a) out[a] = v[3 * (t.size() - 1) + a];
    return;
  }
  const size_t hi = (size_t)(std::upper_bound(t.begin(), t.end(), time) - t.begin()), lo = hi - 1;
  const double span = t[hi] - t[lo];
  const double w = span > 0.0 ? (time - t[lo]) / span : 0.0;
  for (int a = 0; a < 3; ++a) out[a] = (1.0 - w) * v[3 * lo + a] + w * v[3 * hi + a];
}

void Schedule::rate(double time, double out[3]) const {  // Schedule3::rate (collision.cpp:20-30)
  out[0] = out[1] = out[2] = 0.0;
  if (t.size() < 2 || time < t.front() || time > t.back()) return;
  size_t hi = (size_t)(std::upper_bound(t.begin(), t.end(), time) - t.begin());
  if (hi == 0) hi = 1;
  if (hi >= t.size()) hi = t.size() - 1;
  const size_t lo = hi - 1;
  const double span = t[hi] - t[lo];
  if (!(span > 0.0)) return;
  for (int a = 0; a < 3; ++a) out[a] = (v[3 * hi + a] - v[3 * lo + a]) / span;
}

// BoundaryCondition::displacement_at (solver.cpp:22-29): translate -> d; rotate -> R of AngleAxis
void HostBc::displacement_params(double time, double d[3], double R[9]) const {
  if (kind == 0) {
    sched.eval(time, d);
    return;
  }
  double ang[3];
  sched.eval(time, ang);
  const double nn = (axis_dir[0] * axis_dir[0] + axis_dir[1] * axis_dir[1]) + axis_dir[2] * axis_dir[2];
  double ax[3] = {axis_dir[0], axis_dir[1], axis_dir[2]};
  if (nn > 0.0) {
    const double l = std::sqrt(nn);
    for (int a = 0; a < 3; ++a) ax[a] = axis_dir[a] / l;
  }
  const double s = std::sin(ang[0]), c = std::cos(ang[0]);
  const double sa[3] = {s * ax[0], s * ax[1], s * ax[2]};
  const double ca[3] = {(1.0 - c) * ax[0], (1.0 - c) * ax[1], (1.0 - c) * ax[2]};
  double tmp = ca[0] * ax[1];
  R[1] = tmp - sa[2];
  R[3] = tmp + sa[2];
  tmp = ca[0] * ax[2];
  R[2] = tmp + sa[1];
  R[6] = tmp - sa[1];
  tmp = ca[1] * ax[2];
  R[5] = tmp - sa[0];
  R[7] = tmp + sa[0];
  for (int a = 0; a < 3; ++a) R[4 * a] = ca[a] * ax[a] + c;
}

// ---------------------------------------------------------------- construction (solver.cpp:31-60)
void* Simulation::dalloc(size_t bytes) {
  void* p = nullptr;
  if (bytes == 0) bytes = 8;
  GF_CUDA(cudaMalloc(&p, bytes));
  allocs_.push_back(p);
  return p;
}

// Structured non-local layout (DevData::nl_tpl): accepted when the table is shift-invariant over tets of one
// residue mod 6 in consecutive cells (the box generator's numbering, primitives.cpp:26-38), i.e. when the padded
// template slots cost at most 30% more warp steps than the sliced-ELL table. Any other mesh keeps the general
// table. Summation order per tet is unchanged (slots ascend in neighbour id).
template <class Up>
bool Simulation::build_template_layout(const NonlocalTable& tb, Up&& up) {
  const int32_t nt = mesh_.nt;
  if (nt % 6 != 0) return false;
  const int32_t nc = nt / 6;
  int64_t ell_steps = 0;
  for (int32_t sl = 0; sl < (nt + 31) / 32; ++sl) {
    int64_t mx = 0;
    for (int32_t e = 32 * sl; e < std::min(nt, 32 * sl + 32); ++e) mx = std::max(mx, tb.ptr[e + 1] - tb.ptr[e]);
    ell_steps += mx;
  }
  const int64_t budget = ell_steps + ell_steps * 3 / 10;
  std::vector<int4> warps;
  std::vector<int32_t> spos, sh;
  std::vector<double> tw;
  auto fdiv = [](int64_t a, int64_t b) { return a >= 0 ? a / b : -((-a + b - 1) / b); };
  // warp order: the six residues of one 32-cell range are consecutive (one CTA), so their neighbourhoods — the
  // same cells — are gathered while still in L1
  for (int32_t q0 = 0; q0 < nc; q0 += 32)
    for (int t = 0; t < 6; ++t) {
      const int n = (int)std::min<int32_t>(32, nc - q0);
      sh.clear();
      for (int k = 0; k < n; ++k) {
        const int64_t e = 6 * (int64_t)(q0 + k) + t;
        for (int64_t q = tb.ptr[e]; q < tb.ptr[e + 1]; ++q) sh.push_back((int32_t)(tb.ids[q] - e));
      }
      std::sort(sh.begin(), sh.end());
      sh.erase(std::unique(sh.begin(), sh.end()), sh.end());
      const int32_t s0 = (int32_t)spos.size();
      if ((int64_t)s0 + (int64_t)sh.size() > budget) return false;
      warps.push_back(make_int4(t, q0, n, s0));
      for (int32_t d : sh) {  // sigma-plane position of lane 0's neighbour o0 = e_0 + d (lane k: + k)
        const int64_t o0 = 6 * (int64_t)q0 + t + d;
        spos.push_back((int32_t)((o0 - 6 * fdiv(o0, 6)) * nc + fdiv(o0, 6)));
      }
      tw.resize(32 * spos.size(), 0.0);
      for (int k = 0; k < n; ++k) {
        const int64_t e = 6 * (int64_t)(q0 + k) + t;
        for (int64_t q = tb.ptr[e]; q < tb.ptr[e + 1]; ++q) {
          const int64_t j = std::lower_bound(sh.begin(), sh.end(), (int32_t)(tb.ids[q] - e)) - sh.begin();
          tw[32 * (size_t)(s0 + j) + k] = tb.w[q];
        }
      }
    }
  const int32_t nwarps = (int32_t)warps.size();
  warps.push_back(make_int4(0, 0, 0, (int32_t)spos.size()));
  d_.nl_tpl = 1;
  d_.nl_nwarps = nwarps;
  d_.nl_ncell = nc;
  d_.nl_warp = (const int4*)up(warps.data(), sizeof(int4) * warps.size());
  d_.nl_spos = (const int32_t*)up(spos.data(), 4 * spos.size());
  d_.nl_tw = (const double*)up(tw.data(), 8 * tw.size());
  nl_tpl_slots_ = (int64_t)spos.size();
  GF_CUDA(cudaStreamSynchronize(stream_));  // host staging goes out of scope
  return true;
}

// Cell template (DevData::nl_tpl == 2, dev_types.cuh): the same shift-invariance test and budget as the per-residue
// template -- a (slot, residue) pair here is exactly one slot of that layout -- but one thread owns a cell's six
// tets, so a gathered sigma record feeds up to six sums.
template <class Up>
bool Simulation::build_cell_layout(const NonlocalTable& tb, int G, Up&& up) {
  const int32_t nt = mesh_.nt;
  if (nt % 6 != 0 || G < 1 || 6 % G != 0) return false;
  const int32_t nc = nt / 6;
  int64_t ell_steps = 0;
  for (int32_t sl = 0; sl < (nt + 31) / 32; ++sl) {
    int64_t mx = 0;
    for (int32_t e = 32 * sl; e < std::min(nt, 32 * sl + 32); ++e) mx = std::max(mx, tb.ptr[e + 1] - tb.ptr[e]);
    ell_steps += mx;
  }
  const int64_t budget = ell_steps + ell_steps * 3 / 10;
  constexpr int kVec = 16;  // a multiple of damage.cu's kNcVec (weight vectors per bulk copy)
  const int ngroups = 6 / G;
  const int32_t nw = ((nc + 31) / 32) * ngroups;  // warps: the groups of one 32-cell range are consecutive
  std::vector<int4> warps(nw + 1);
  // pass 1 (parallel): per warp the sorted (offset, residue mask) list
  std::vector<std::vector<int2>> lists(nw);
  std::vector<int64_t> nvec(nw + 1, 0);
#pragma omp parallel
  {
    std::vector<int64_t> keys;
#pragma omp for schedule(dynamic, 16)
    for (int32_t r = 0; r < nw; ++r) {
      const int32_t q0 = 32 * (r / ngroups), n = std::min<int32_t>(32, nc - q0), g = r % ngroups;
      keys.clear();
      for (int k = 0; k < n; ++k)
        for (int t = 0; t < G; ++t) {
          const int64_t e = 6 * (int64_t)(q0 + k) + g * G + t;
          for (int64_t q = tb.ptr[e]; q < tb.ptr[e + 1]; ++q)
            keys.push_back(((int64_t)(tb.ids[q] - 6 * (int64_t)(q0 + k)) + (int64_t(1) << 40)) * 8 + t);
        }
      std::sort(keys.begin(), keys.end());
      keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
      std::vector<int2>& L = lists[r];
      for (int64_t key : keys) {
        const int32_t D = (int32_t)((key >> 3) - (int64_t(1) << 40)), t = (int32_t)(key & 7);
        if (L.empty() || L.back().x != D) L.push_back(make_int2(D, 0));
        L.back().y |= 1 << t;
      }
      nvec[r + 1] = ((int64_t)keys.size() + kVec - 1) / kVec * kVec;
    }
  }
  int64_t nslots = 0, pairs = 0;
  for (int32_t r = 0; r < nw; ++r) {
    const int32_t q0 = 32 * (r / ngroups);
    warps[r] = make_int4(q0, std::min<int32_t>(32, nc - q0) | ((r % ngroups) << 8), (int32_t)nslots, (int32_t)nvec[r]);
    nslots += (int64_t)lists[r].size();
    for (const int2& s : lists[r]) pairs += __builtin_popcount((unsigned)s.y);
    nvec[r + 1] += nvec[r];
    if (nvec[r + 1] > INT32_MAX || nslots > INT32_MAX) return false;
  }
  if (pairs > budget) return false;
  warps[nw] = make_int4(0, 0, (int32_t)nslots, (int32_t)nvec[nw]);
  std::vector<int2> cslot((size_t)nslots + 1, make_int2(0, 0));  // + one pad record (a warp without slots reads it)
  std::vector<double> tw(32 * (size_t)nvec[nw], 0.0);
  auto fdiv = [](int64_t a, int64_t b) { return a >= 0 ? a / b : -((-a + b - 1) / b); };
#pragma omp parallel for schedule(dynamic, 16)
  for (int32_t r = 0; r < nw; ++r) {
    const int32_t q0 = warps[r].x, n = warps[r].y & 255, g = warps[r].y >> 8;
    const std::vector<int2>& L = lists[r];
    std::vector<int32_t> first(L.size());  // first weight vector of each slot (relative to the warp's stream)
    int32_t acc = 0;
    for (size_t j = 0; j < L.size(); ++j) {
      first[j] = acc;
      acc += __builtin_popcount((unsigned)L[j].y);
      const int64_t o0 = 6 * (int64_t)q0 + L[j].x;  // lane 0's neighbour (lane k: + 6 k, i.e. plane position + k)
      cslot[(size_t)warps[r].z + j] = make_int2((int32_t)((o0 - 6 * fdiv(o0, 6)) * nc + fdiv(o0, 6)), L[j].y);
    }
    for (int k = 0; k < n; ++k)
      for (int t = 0; t < G; ++t) {
        const int64_t e = 6 * (int64_t)(q0 + k) + g * G + t;
        size_t j = 0;
        for (int64_t q = tb.ptr[e]; q < tb.ptr[e + 1]; ++q) {
          const int32_t D = (int32_t)(tb.ids[q] - 6 * (int64_t)(q0 + k));
          while (L[j].x != D) ++j;  // both ascend
          const int32_t vec = first[j] + __builtin_popcount((unsigned)L[j].y & ((1u << t) - 1u));
          tw[32 * ((size_t)warps[r].w + vec) + k] = tb.w[q];
        }
      }
  }
  d_.nl_tpl = 2;
  d_.nl_group = G;
  d_.nl_flag = (int32_t*)dalloc(4);
  GF_CUDA(cudaMemsetAsync(d_.nl_flag, 0, 4, stream_));
  d_.nl_nwarps = nw;
  d_.nl_ncell = nc;
  d_.nl_warp = (const int4*)up(warps.data(), sizeof(int4) * warps.size());
  d_.nl_cslot = (const int2*)up(cslot.data(), sizeof(int2) * cslot.size());
  d_.nl_tw = (const double*)up(tw.data(), 8 * tw.size());
  nl_tpl_slots_ = nvec[nw];
  GF_CUDA(cudaStreamSynchronize(stream_));  // host staging goes out of scope
  return true;
}

Simulation::Simulation(const HostMesh& mesh, const gf_material& mat, const gf_solver_config& cfg,
                       const gf_boundary_condition* bcs, int32_t n_bcs, const gf_collider* cols, int32_t n_cols)
    : mesh_(mesh), mat_(mat), cfg_(cfg) {
  using clk = std::chrono::steady_clock;
  const auto t_ctor = clk::now();
  auto secs = [](clk::time_point a) { return std::chrono::duration<double>(clk::now() - a).count(); };
  // validation in the reference's order (material.cpp:37-43, solver.cpp:10-20, collision.cpp:32-40, 46-56)
  if (!(mat.youngs > 0.0)) throw FormatError("youngs modulus must be positive");
  if (!(mat.poisson >= 0.0 && mat.poisson < 0.5)) throw FormatError("poisson ratio must be in [0, 0.5)");
  if (!(mat.density > 0.0)) throw FormatError("density must be positive");
  if (!(mat.sigma_thres > 0.0)) throw FormatError("sigma_thres must be positive");
  if (!(mat.r_d >= 0.0)) throw FormatError("r_d must be non-negative");
  if (!(cfg.dt > 0.0)) throw FormatError("dt must be positive");
  if (!(cfg.cg_tol > 0.0)) throw FormatError("cg_tol must be positive");
  if (cfg.newton_max_iters <= 0 || cfg.cg_max_iters <= 0) throw FormatError("iteration limits must be positive");
  if (!(cfg.ls_backtrack > 0.0 && cfg.ls_backtrack < 1.0))
    throw FormatError("line-search backtrack factor must be in (0, 1)");
  if (!(cfg.ls_sufficient_decrease > 0.0 && cfg.ls_sufficient_decrease < 1.0))
    throw FormatError("line-search sufficient-decrease constant must be in (0, 1)");
  if (cfg.collision_substeps < 1) throw FormatError("collision_substeps must be >= 1");
  for (int c = 0; c < n_cols; ++c) {
    const gf_collider& k = cols[c];
    const double nn = std::sqrt((k.normal[0] * k.normal[0] + k.normal[1] * k.normal[1]) + k.normal[2] * k.normal[2]);
    if (k.kind == 0 && !(k.radius > 0.0)) throw FormatError("sphere radius must be positive");
    if (k.kind == 1 && std::abs(nn - 1.0) > 1e-9) throw FormatError("halfspace normal must be unit length");
    if (!(k.stiffness > 0.0)) throw FormatError("collider stiffness must be positive");
    if (k.restitution < 0.0 || k.restitution > 1.0) throw FormatError("restitution must be in [0, 1]");
    if (k.friction < 0.0) throw FormatError("friction must be non-negative");
  }
  if (n_cols > 8) throw FormatError("at most 8 colliders are supported by the device collision kernel");
  std::vector<int32_t> node_bc(mesh_.nn, -1);
  for (int b = 0; b < n_bcs; ++b) {
    const std::string name = "bc" + std::to_string(b);
    if (bcs[b].n_nodes <= 0) throw FormatError("boundary condition '" + name + "' selects no nodes");
    for (int q = 0; q < bcs[b].n_nodes; ++q) {
      const int32_t n = bcs[b].nodes[q];
      if (n < 0 || n >= mesh_.nn) throw FormatError("boundary condition '" + name + "' references node out of range");
      if (node_bc[n] >= 0) throw FormatError("node " + std::to_string(n) + " appears in two boundary conditions");
      node_bc[n] = b;
    }
    HostBc hb;
    hb.kind = bcs[b].kind;
    hb.nodes.assign(bcs[b].nodes, bcs[b].nodes + bcs[b].n_nodes);
    hb.sched.t.assign(bcs[b].key_times, bcs[b].key_times + bcs[b].n_keys);
    hb.sched.v.assign(bcs[b].key_values, bcs[b].key_values + 3 * bcs[b].n_keys);
    for (int a = 0; a < 3; ++a) {
      hb.axis_point[a] = bcs[b].axis_point[a];
      hb.axis_dir[a] = bcs[b].axis_dir[a];
    }
    bcs_.push_back(std::move(hb));
  }
  for (int c = 0; c < n_cols; ++c) {
    HostCollider hc;
    hc.kind = cols[c].kind;
    hc.center.t.assign(cols[c].key_times, cols[c].key_times + cols[c].n_keys);
    hc.center.v.assign(cols[c].key_values, cols[c].key_values + 3 * cols[c].n_keys);
    hc.radius = cols[c].radius;
    for (int a = 0; a < 3; ++a) {
      hc.point[a] = cols[c].point[a];
      hc.normal[a] = cols[c].normal[a];
    }
    hc.stiffness = cols[c].stiffness;
    hc.restitution = cols[c].restitution;
    hc.friction = cols[c].friction;
    cols_.push_back(hc);
  }

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    throw CudaError("no CUDA device: the B200 hot path has no CPU fallback");
  }
  int dev = 0, major = 0;
  GF_CUDA(cudaGetDevice(&dev));
  GF_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  if (major < 10) throw CudaError("device is not sm_100 class (Blackwell); this build targets sm_100a only");

  // host setup: pattern, incidence, table, mass (fem.cpp:140-179, fracture.cpp:32-54)
  auto t_phase = clk::now();
  pat_ = make_node_pattern(mesh_);
  if (pat_.max_degree > 64) throw GeometryError("node rows with more than 64 neighbour blocks are not supported by the assembly kernel");
  const NodeTets ntets = make_node_tets(mesh_, pat_);
  if (ntets.max_valence > 84) throw GeometryError("nodes shared by more than 84 tets are not supported by the assembly kernel");
  hash_ = pat_.structure_hash(mesh_.nn);
  mass_.assign(mesh_.nn, 0.0);
  for (int32_t e = 0; e < mesh_.nt; ++e) {  // lumped_mass (fem.cpp:171-179), ascending tet order
    const double q = mat.density * mesh_.vol[e] / 4.0;
    for (int k = 0; k < 4; ++k) mass_[mesh_.tets[4 * (size_t)e + k]] += q;
  }
  md_.mu = mat.mu;
  md_.lambda = mat.lambda;
  md_.alpha_nh = 1.0 + mat.mu / mat.lambda - mat.mu / (4.0 * mat.lambda);
  md_.sigma_thres = mat.sigma_thres;
  md_.chi_eps = 1e-12 * mat.sigma_thres;
  md_.model = mat.energy_model;

  GF_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  const int32_t nn = mesh_.nn, nt = mesh_.nt, ne = mesh_.ne, nb = (int32_t)pat_.cols.size();
  auto up = [&](const void* src, size_t bytes) {
    void* p = dalloc(bytes);
    if (bytes) GF_CUDA(cudaMemcpyAsync(p, src, bytes, cudaMemcpyHostToDevice, stream_));
    return p;
  };
  d_.nn = nn; d_.nt = nt; d_.ne = ne; d_.nb = nb;
  d_.X = (const double*)up(mesh_.X.data(), 8 * mesh_.X.size());
  d_.tets = (const int4*)up(mesh_.tets.data(), 4 * mesh_.tets.size());
  {
    std::vector<double> rec(10 * (size_t)mesh_.nt);
    for (size_t e = 0; e < (size_t)mesh_.nt; ++e) {
      for (int q = 0; q < 9; ++q) rec[10 * e + q] = mesh_.binv[9 * e + q];
      rec[10 * e + 9] = mesh_.vol[e];
    }
    d_.bv = (const double2*)up(rec.data(), 8 * rec.size());
    GF_CUDA(cudaStreamSynchronize(stream_));  // host staging goes out of scope
  }
  d_.tet_edges = (const int32_t*)up(mesh_.tet_edges.data(), 4 * mesh_.tet_edges.size());
  d_.rest_len = (const double*)up(mesh_.rest_len.data(), 8 * mesh_.rest_len.size());
  d_.rest_len_gt1 = 0;
  for (double L : mesh_.rest_len) d_.rest_len_gt1 |= (1.0 < L) ? 1 : 0;
  d_.et_ptr = (const int32_t*)up(mesh_.et_ptr.data(), 4 * mesh_.et_ptr.size());
  d_.et_ids = (const int32_t*)up(mesh_.et_ids.data(), 4 * mesh_.et_ids.size());
  d_.mass = (const double*)up(mass_.data(), 8 * mass_.size());
  d_.node_bc = (const int32_t*)up(node_bc.data(), 4 * node_bc.size());
  d_.nt_ptr = (const int32_t*)up(ntets.ptr.data(), 4 * ntets.ptr.size());
  d_.nt_tet = (const int32_t*)up(ntets.tet.data(), 4 * ntets.tet.size());
  {
    std::vector<int32_t> nodes(4 * ntets.tet.size());
    for (size_t q = 0; q < ntets.tet.size(); ++q)
      for (int k = 0; k < 4; ++k) nodes[4 * q + k] = mesh_.tets[4 * (size_t)ntets.tet[q] + k];
    d_.nt_nodes = (const int4*)up(nodes.data(), 4 * nodes.size());
    GF_CUDA(cudaStreamSynchronize(stream_));  // host staging goes out of scope
  }
  {  // contribution lists of the assembly reduction (assemble.cu): per off-diagonal block, items 3 l + s
     // (lane l = incident tet, s = its off-diagonal block slot), ascending l; diagonal blocks are warp sums
    auto col_of = [&](int32_t q, int k) { return (int32_t)((ntets.slot[q] >> (8 * k)) & 0xff); };
    auto local_of = [&](int32_t i, int32_t q) {
      for (int k = 0; k < 4; ++k)
        if (pat_.cols[pat_.row_ptr[i] + col_of(q, k)] == i) return k;
      throw std::logic_error("incidence slot without the diagonal");
    };
    std::vector<int32_t> cnt(pat_.cols.size() + 1, 0);
    for (int32_t i = 0; i < nn; ++i)
      for (int32_t q = ntets.ptr[i]; q < ntets.ptr[i + 1]; ++q) {
        const int li = local_of(i, q);
        for (int k = 0; k < 4; ++k)
          if (k != li) cnt[pat_.row_ptr[i] + col_of(q, k) + 1]++;
      }
    for (size_t b = 0; b < pat_.cols.size(); ++b) cnt[b + 1] += cnt[b];
    std::vector<uint8_t> items(cnt.back());
    std::vector<int32_t> cur(cnt.begin(), cnt.end() - 1);
    for (int32_t i = 0; i < nn; ++i)
      for (int32_t q = ntets.ptr[i]; q < ntets.ptr[i + 1]; ++q) {
        const int li = local_of(i, q);
        for (int k = 0; k < 4; ++k)
          if (k != li)
            items[cur[pat_.row_ptr[i] + col_of(q, k)]++] = (uint8_t)(3 * (q - ntets.ptr[i]) + (k < li ? k : k - 1));
      }
    // padded per row: every column of row i gets mx_i items (the row's longest list), pad item 96 addresses a
    // zero block, so the kernel's reduction loop has a uniform trip count across the warp
    std::vector<int32_t> rptr(nn + 1, 0);
    for (int32_t i = 0; i < nn; ++i) {
      int32_t mx = 0;
      for (int32_t b = pat_.row_ptr[i]; b < pat_.row_ptr[i + 1]; ++b) mx = std::max(mx, cnt[b + 1] - cnt[b]);
      if (mx > 16) throw GeometryError("more than 16 tets around an edge are not supported by the assembly kernel");
      mx = (mx + 3) & ~3;  // lists padded to whole 4-item words (the kernel reads them as 32-bit words)
      rptr[i + 1] = rptr[i] + mx * (pat_.row_ptr[i + 1] - pat_.row_ptr[i]);
    }
    // rows beyond one warp's lanes (> 32 incident tets or > 32 neighbour blocks) go to k_assemble_big, whose
    // padding item is 255; the one-warp rows pad with 96 (the zero block after the 32 lanes' blocks)
    std::vector<int32_t> big;
    std::vector<uint8_t> padded(rptr[nn], 96);
    for (int32_t i = 0; i < nn; ++i) {
      const int32_t deg = pat_.row_ptr[i + 1] - pat_.row_ptr[i], mx = (rptr[i + 1] - rptr[i]) / std::max(1, deg);
      const bool is_big = ntets.ptr[i + 1] - ntets.ptr[i] > 32 || deg > 32;
      if (is_big) {
        big.push_back(i);
        std::fill(padded.begin() + rptr[i], padded.begin() + rptr[i + 1], (uint8_t)255);
      }
      for (int32_t c = 0; c < deg; ++c) {
        const int32_t b = pat_.row_ptr[i] + c;
        for (int32_t t = cnt[b]; t < cnt[b + 1]; ++t) padded[rptr[i] + c * mx + (t - cnt[b])] = items[t];
      }
    }
    d_.n_big = (int32_t)big.size();
    d_.big_rows = big.empty() ? nullptr : (const int32_t*)up(big.data(), 4 * big.size());
    d_.contrib_ptr = (const int32_t*)up(rptr.data(), 4 * rptr.size());
    d_.contrib_item = (const uint8_t*)up(padded.data(), std::max<size_t>(1, padded.size()));
    GF_CUDA(cudaStreamSynchronize(stream_));
  }
  d_.brow = (const int32_t*)up(pat_.row_ptr.data(), 4 * pat_.row_ptr.size());
  d_.bcol = (const int32_t*)up(pat_.cols.data(), 4 * pat_.cols.size());
  {
    // SELL-32 slices (dev_types.cuh): full-row slots per slice = max degree of its 32 rows
    const int32_t ns = (nn + 31) / 32;
    sell_ptr_.assign(ns + 1, 0);
    for (int32_t sl = 0; sl < ns; ++sl) {
      int32_t mx = 0;
      for (int32_t i = 32 * sl; i < std::min(nn, 32 * sl + 32); ++i) mx = std::max(mx, pat_.row_ptr[i + 1] - pat_.row_ptr[i]);
      sell_ptr_[sl + 1] = sell_ptr_[sl] + mx;
    }
    d_.sell_ptr = (const int32_t*)up(sell_ptr_.data(), 4 * sell_ptr_.size());
    d_.nslices = ns;
    sell_slots_ = sell_ptr_[ns];
    // symmetric format: upper blocks (j >= i) in upper-CSR order per row, SELL-32 over slices
    uslot_.assign(pat_.cols.size(), -1);
    std::vector<int32_t> ucount(nn, 0);
    for (int32_t i = 0; i < nn; ++i)
      for (int32_t q = pat_.row_ptr[i]; q < pat_.row_ptr[i + 1]; ++q)
        if (pat_.cols[q] >= i) uslot_[q] = ucount[i]++;
    for (int32_t i = 0; i < nn; ++i)
      if (ucount[i] > 63) throw GeometryError("node rows with more than 63 upper neighbour blocks are not supported");
    usp_.assign(ns + 1, 0);
    for (int32_t sl = 0; sl < ns; ++sl) {
      int32_t mx = 0;
      for (int32_t i = 32 * sl; i < std::min(nn, 32 * sl + 32); ++i) mx = std::max(mx, ucount[i]);
      usp_[sl + 1] = usp_[sl] + mx;
    }
    if ((int64_t)usp_[ns] * 288 >= (int64_t)1 << 31) throw GeometryError("symmetric value array exceeds 31-bit slot bases");
    // packed slot (j << 6 | c): column block j and the ordinal c of the stored upper block ((i, j) in row i
    // when j >= i, else (j, i) in row j); c = 63 marks padding (cg_sell.cu decodes the value base)
    if (nn >= (1 << 26)) throw GeometryError("symmetric slot packing supports < 2^26 nodes");
    std::vector<uint32_t> slot(32 * (size_t)sell_slots_);
    zero_base_ = (int32_t)((int64_t)usp_[ns] * 288);  // one extra all-zero 288-double group
    for (int32_t sl = 0; sl < ns; ++sl)
      for (int32_t l = 0; l < 32; ++l) {
        const int32_t i = 32 * sl + l;
        const int32_t deg = i < nn ? pat_.row_ptr[i + 1] - pat_.row_ptr[i] : 0;
        for (int32_t c = 0; c < sell_ptr_[sl + 1] - sell_ptr_[sl]; ++c) {
          uint32_t e = ((uint32_t)(i < nn ? i : 0) << 6) | 63u;  // padding: zero block, own row
          if (c < deg) {
            const int32_t q = pat_.row_ptr[i] + c, j = pat_.cols[q];
            if (j >= i) {
              e = ((uint32_t)j << 6) | (uint32_t)uslot_[q];
            } else {
              const auto jb = pat_.cols.begin() + pat_.row_ptr[j], je = pat_.cols.begin() + pat_.row_ptr[j + 1];
              const int32_t qj = pat_.row_ptr[j] + (int32_t)(std::lower_bound(jb, je, i) - jb);
              e = ((uint32_t)j << 6) | (uint32_t)uslot_[qj];
            }
          }
          slot[32 * (size_t)(sell_ptr_[sl] + c) + l] = e;
        }
      }
    d_.usp = (const int32_t*)up(usp_.data(), 4 * usp_.size());
    d_.uslot = (const int32_t*)up(uslot_.data(), 4 * uslot_.size());
    d_.sell_slot = (const uint32_t*)up(slot.data(), 4 * slot.size());
    GF_CUDA(cudaStreamSynchronize(stream_));
  }
  setup_s_[0] = secs(t_phase);
  if (mat.r_d > 0.0) {
    t_phase = clk::now();
    const NonlocalTable tb = make_nonlocal_table(mesh_, mat.r_d);
    setup_s_[1] = secs(t_phase);
    nl_entries_ = (int64_t)tb.ids.size();
    // GF_NL_LAYOUT: "general" forces the sliced-ELL table, "tet" the per-residue template (one tet per thread)
    const std::string nl_env = std::getenv("GF_NL_LAYOUT") ? std::getenv("GF_NL_LAYOUT") : "";
    const int nl_group = std::getenv("GF_NL_GROUP") ? std::atoi(std::getenv("GF_NL_GROUP")) : 3;
    if (nl_env != "general" && (nl_env == "tet" ? build_template_layout(tb, up) : build_cell_layout(tb, nl_group, up))) {
      GF_CUDA(cudaStreamSynchronize(stream_));
    } else {
    const int32_t ns = (nt + 31) / 32;
    std::vector<int64_t> sptr(ns + 1, 0);
    std::vector<int32_t> len(nt);
    for (int32_t e = 0; e < nt; ++e) len[e] = (int32_t)(tb.ptr[e + 1] - tb.ptr[e]);
    for (int32_t sl = 0; sl < ns; ++sl) {
      int32_t mx = 0;
      for (int32_t e = 32 * sl; e < std::min(nt, 32 * sl + 32); ++e) mx = std::max(mx, len[e]);
      sptr[sl + 1] = sptr[sl] + mx;
    }
    std::vector<int32_t> ids(32 * (size_t)sptr[ns], 0);
    std::vector<double> w(32 * (size_t)sptr[ns], 0.0);
    for (int32_t e = 0; e < nt; ++e) {
      const int64_t b = sptr[e >> 5] * 32 + (e & 31);
      for (int32_t j = 0; j < len[e]; ++j) {
        ids[b + 32 * (int64_t)j] = tb.ids[tb.ptr[e] + j];
        w[b + 32 * (int64_t)j] = tb.w[tb.ptr[e] + j];
      }
    }
    d_.nl_sptr = (const int64_t*)up(sptr.data(), 8 * sptr.size());
    d_.nl_len = (const int32_t*)up(len.data(), 4 * len.size());
    d_.nl_ids = (const int32_t*)up(ids.data(), 4 * ids.size());
    d_.nl_w = (const double*)up(w.data(), 8 * w.size());
    nl_ell_slots_ = 32 * sptr[ns];
    GF_CUDA(cudaStreamSynchronize(stream_));  // host staging goes out of scope
    }
  } else {
    nl_entries_ = nt;
  }
  const size_t nd = 3 * (size_t)nn;
  auto zeros = [&](size_t bytes) {
    void* p = dalloc(bytes);
    GF_CUDA(cudaMemsetAsync(p, 0, bytes, stream_));
    return p;
  };
  d_.u = (double*)zeros(8 * nd);
  d_.v = (double*)zeros(8 * nd);
  d_.zeta = (uint8_t*)zeros(ne);
  d_.chi = (double*)dalloc(8 * (size_t)nt);
  launch_fill(d_.chi, 1.0, nt, stream_);  // SimState::rest (fem.cpp:7-14)
  d_.sigc = (double*)zeros(48 * (size_t)nt);
  d_.sigf = (double*)zeros(48 * (size_t)nt);
  d_.deg = (uint8_t*)zeros(nt);
  d_.scr_key = (unsigned long long*)dalloc(8 * (size_t)ne);
  d_.screening = (double*)zeros(8 * (size_t)ne);
  d_.newly = (int32_t*)zeros(4 * (size_t)ne);
  // one 64-byte stats record read back once per step: [cg_out (4 doubles), collider load, newly-broken count]
  d_stats_ = (double*)zeros(64);
  d_.newly_count = reinterpret_cast<int32_t*>(d_stats_ + 5);
  bval_doubles_ = 288 * ((size_t)usp_[d_.nslices] + 1);  // + one all-zero padding group
  // GF_PAD_MB: allocation-placement experiment (tools/ab_pad.sh); the PCG time depends on where the system
  // matrix lands in physical memory by up to ~8%
  if (const char* e = std::getenv("GF_PAD_MB")) dalloc((size_t)std::atol(e) << 20);
  d_.bval = (double*)zeros(8 * bval_doubles_);  // padding slots / the extra zero block stay zero
  d_.rhs = (double*)zeros(8 * nd);
  d_.dinv = (double*)zeros(8 * nd);
  d_.x = (double*)zeros(8 * nd);
  d_.fext = (double*)zeros(8 * nd);
  d_.fcoll = (double*)zeros(8 * nd);
  d_.fv = (double*)zeros(8 * nd);
  d_.utgt = (double*)zeros(8 * nd);
  d_.vtgt = (double*)zeros(8 * nd);
  d_.absdiag = (double*)zeros(8 * nd);
  d_.r = (double*)zeros(8 * nd);
  d_.z = (double*)zeros(8 * nd);
  d_.p0 = (double*)zeros(8 * nd);
  d_.Ap = (double*)zeros(8 * nd);
  d_.cg_out = d_stats_;
  d_.n_colliders = (int32_t)cols_.size();
  const int nsub = cfg.collision_substeps;
  if (!cols_.empty()) {
    d_cols_ = (ColliderDev*)dalloc(sizeof(ColliderDev) * cols_.size() * nsub);
    d_.colliders = d_cols_;
    d_.coll_partials = (double*)zeros(8 * (size_t)nsub * cols_.size() * 3 * collide_blocks(d_));
    GF_CUDA(cudaMallocHost(&h_cols_, sizeof(ColliderDev) * cols_.size() * nsub));
  }
  d_load_ = d_stats_ + 4;
  {  // element form: GF_ELEMENT=edge selects the edge-length kernels (k_tet_edge + edge row kernel)
    const char* ef = std::getenv("GF_ELEMENT");
    edge_form_ = ef ? std::string(ef) == "edge" : kEdgeFormDefault;
    if (edge_form_) {
      d_.erec = (double*)zeros(8 * 28 * (size_t)nt);
      d_.eflag = (uint8_t*)zeros((size_t)nt);
      d_.efall_cap = std::max<int32_t>(1024, nt / 64);
      d_.efall = (double*)zeros(8 * 156 * (size_t)d_.efall_cap);
      d_.efall_tet = (int32_t*)zeros(4 * (size_t)d_.efall_cap);
      d_.efall_count = reinterpret_cast<int32_t*>(d_stats_ + 6);
      d_.eng_part = (double*)zeros(8 * (size_t)tet_edge_blocks(nt));
      d_.eng_ticket = (unsigned*)zeros(64);
    }
    d_.eng_out = d_stats_ + 7;
    d_.eng_row = (double*)zeros(8 * (size_t)nn);
    if (!edge_form_) {  // the F-based form's energy partials are reduced by k_integrate (misc.cu)
      d_.eng_part = (double*)zeros(8 * (size_t)((nn + 255) / 256));
      d_.eng_ticket = (unsigned*)zeros(64);
    }
  }
  d_energy_partials_ = (double*)zeros(8 * metrics_partial_doubles());
  d_red_ticket_ = (unsigned*)zeros(64);
  d_red_out_ = (double*)zeros(64);
  if (!bcs_.empty()) {
    d_bcstep_ = (BcStep*)dalloc(sizeof(BcStep) * bcs_.size());
    d_.bcstep = d_bcstep_;
    GF_CUDA(cudaMallocHost(&h_bcstep_, sizeof(BcStep) * bcs_.size()));
  }
  std::vector<int32_t> fixed;
  for (int32_t i = 0; i < nn; ++i)
    if (node_bc[i] >= 0) fixed.push_back(i);
  n_fixed_ = (int32_t)fixed.size();
  d_fixed_nodes_ = (int32_t*)up(fixed.data(), 4 * fixed.size());
  GF_CUDA(cudaMallocHost(&h_stats_, 8 * 8));
  GF_CUDA(cudaMallocHost(&h_partials_, 64));
  newton_tol_ = cfg_.newton_tol > 0.0 ? cfg_.newton_tol : 1e-6 * mat_.sigma_thres * mesh_.mean_face_area();  // solver.cpp:57-59
  // static external force: m g (solver.cpp:230-231)
  std::vector<double> fext(nd);
  for (int32_t i = 0; i < nn; ++i)
    for (int a = 0; a < 3; ++a) fext[3 * (size_t)i + a] = mass_[i] * cfg.gravity[a];
  GF_CUDA(cudaMemcpyAsync(d_.fext, fext.data(), 8 * nd, cudaMemcpyHostToDevice, stream_));
  launch_reset_keys(d_, stream_);

  cg_.nrows = nn;
  cg_.row_ptr = d_.sell_ptr;
  cg_.cols = reinterpret_cast<const int32_t*>(d_.sell_slot);
  cg_.usp = d_.usp;
  cg_.zero_base = zero_base_;
  cg_.nslices = d_.nslices;
  cg_.vals = d_.bval;
  cg_.b = d_.rhs;
  cg_.x = d_.x;
  cg_.dinv = d_.dinv;
  cg_.r = d_.r; cg_.z = d_.z; cg_.p0 = d_.p0; cg_.Ap = d_.Ap;
  cg_.out = d_.cg_out;
  {  // PCG work split (cg_sell.cu Phase): contiguous slice ranges of at most K slices per warp, balanced by the
     // slices' slot counts (interior slices carry ~1.5x the slots of boundary ones): the smallest per-CTA slot
     // budget that places the static slices. One slice per warp covers the matrix while it fits (c3: no
     // dynamic units); a larger matrix places one slice per warp statically and hands out the rest by ticket.
    const int ns = d_.nslices;
    // a matrix of at most one slice per resident warp keeps the solver state on chip (k_pcg_pipe / k_pcg_sell<false>);
    // a larger one runs the large-matrix instance with its own block size (k_pcg_sell<true>)
    // GF_CG_BIG=2 forces the large-matrix instance k_pcg_big on any matrix (tests); GF_CG_BIG=0 keeps k_pcg_sell<true>
    const char* be = std::getenv("GF_CG_BIG");
    const int big_env = be ? std::atoi(be) : 1;
    const bool dyn = ns > pcg_sell_grid() * pcg_sell_warps_per_cta() || big_env == 2;
    const int Gfull = dyn ? pcg_dyn_grid() : pcg_sell_grid(), W = dyn ? pcg_dyn_warps_per_cta() : pcg_sell_warps_per_cta();
    // CTAs of the cooperative solve: all co-resident ones by default; GF_CG_GRID=<n> asks for fewer (cheaper grid
    // barriers for small matrices), never fewer than one slice per warp needs
    int G = Gfull, want = 0;
    if (const char* e = std::getenv("GF_CG_GRID")) {
      want = std::atoi(e);
      if (want > 0) G = std::min(Gfull, std::max(want, (ns + W - 1) / W));
    }
    cg_.pipelined = pcg_pipelined_default();
    // the matrix on chip (cg_onchip.cu) when the pattern has at most 7 distinct positive column offsets (the box
    // meshes: +1, +nx, +nx+1, +nx ny, ...) and its slices fit one CTA per SM (GF_CG_ONCHIP=0 disables)
    std::vector<int32_t> offs;
    for (int32_t i = 0; i < nn && offs.size() <= 7; ++i)
      for (int32_t q = pat_.row_ptr[i]; q < pat_.row_ptr[i + 1]; ++q) {
        const int32_t d = pat_.cols[q] - i;
        if (d > 0 && std::find(offs.begin(), offs.end(), d) == offs.end()) offs.push_back(d);
      }
    const char* oe = std::getenv("GF_CG_ONCHIP");
    const bool onchip_ok = !(oe && std::atoi(oe) == 0) && cg_.pipelined && !dyn && offs.size() <= 7 &&
                           pcg_onchip_grid() >= G && W == pcg_onchip_warps_per_cta();
    // small matrices (c1): the whole pipelined solve in one thread-block cluster -- hardware cluster barriers and
    // DSMEM partial exchange instead of grid barriers through global memory (GF_CG_CLUSTER=0 disables); the on-chip
    // solver's cluster instance when it applies, else k_pcg_pipe's
    const char* ce = std::getenv("GF_CG_CLUSTER");
    const bool cluster_ok = !(ce && std::atoi(ce) == 0) && cg_.pipelined && !dyn;
    const int cmax_oc = cluster_ok && onchip_ok ? pcg_onchip_max_cluster() : 0;
    const int cmax = cluster_ok ? pcg_max_cluster() : 0;
    int Weff = W;
    if (cmax_oc > 0 && ns <= cmax_oc * W) {
      G = std::min(cmax_oc, ns);  // one CTA per slice up to the cluster size: more SMs, shorter latency chains
      if (want > 0) G = std::min(G, std::max(want, (ns + W - 1) / W));
      cg_.cluster = 1;
      cg_.onchip = 1;
      cg_.split = 1;  // k_pcg_pipe's cluster instance on this layout when a caller's matrix falls back (solve_system)
    } else if (cmax > 0 && ns <= cmax * W) {
      G = cmax;
      cg_.cluster = 1;
      // warps to spare: up to 4 warps share a slice's SpMV (shorter latency chains)
      int split = 4;
      if (const char* se = std::getenv("GF_CG_SPLIT")) split = std::max(1, std::min(4, std::atoi(se)));
      while (split > 1 && ns > cmax * (W / split)) --split;
      cg_.split = split;
      Weff = W / split;
    } else if (onchip_ok) {
      cg_.onchip = 1;
    }
    // large matrices: k_pcg_big (round-robin static slices, one partial per CTA, x deferred; GF_CG_BIG=0: the
    // ticketed k_pcg_sell<true>)
    if (dyn) cg_.big = big_env != 0;
    cg_.grid = G;
    const int64_t gw = (int64_t)G * Weff;
    double frac = 0.0;  // measured at c4 (28k slices): all-dynamic tail 22.5 ms, 50 % static 23.0, 80 % 26.2
    if (const char* e = std::getenv("GF_CG_STATIC")) frac = std::atof(e);  // static share of a large matrix
    const int32_t nstat = ns <= gw ? ns : (int32_t)std::min<int64_t>(ns, std::max<int64_t>(gw, (int64_t)(frac * ns)));
    const int64_t cap_n = (int64_t)Weff * std::max<int64_t>(1, (nstat + gw - 1) / gw);
    std::vector<int32_t> first(G + 1, 0);
    auto fill = [&](int64_t cap, bool write) {
      int32_t sl = 0;
      for (int b = 0; b < G; ++b) {
        if (write) first[b] = sl;
        int64_t acc = 0, cnt = 0;
        while (sl < nstat && cnt < cap_n && acc + (sell_ptr_[sl + 1] - sell_ptr_[sl]) <= cap) {
          acc += sell_ptr_[sl + 1] - sell_ptr_[sl];
          ++sl;
          ++cnt;
        }
      }
      if (write) first[G] = sl;
      return sl == nstat;
    };
    int64_t lo = 1, hi = cap_n * 64;  // slots per slice <= 63 (packed ordinals)
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (fill(mid, false)) hi = mid;
      else lo = mid + 1;
    }
    fill(lo, true);
    cg_ndyn_ = ns - nstat;
    d_slice_part_ = (double*)zeros(8 * pcg_sell_part_doubles(cg_ndyn_));
    d_ctr_ = (unsigned long long*)zeros(64);
    cg_.cta_first = (const int32_t*)up(first.data(), 4 * first.size());
    if (cg_.onchip) {  // per-row slot masks over the sorted offsets
      std::sort(offs.begin(), offs.end());
      for (size_t b = 0; b < offs.size(); ++b) oc_off_[b] = offs[b];
      auto bit = [&](int32_t d) { return (int)(std::lower_bound(offs.begin(), offs.end(), d) - offs.begin()); };
      std::vector<uint32_t> meta(nn, 0u);  // upper slot mask | lower slot mask << 8 (slot b: offset offs[b])
      for (int32_t i = 0; i < nn; ++i)
        for (int32_t q = pat_.row_ptr[i]; q < pat_.row_ptr[i + 1]; ++q) {
          const int32_t j = pat_.cols[q];
          if (j > i) {
            meta[i] |= 1u << bit(j - i);
            ++oc_slot_blocks_[bit(j - i)];
          }
          else if (j < i) meta[i] |= 1u << (8 + bit(i - j));
        }
      d_oc_meta_ = (uint32_t*)up(meta.data(), sizeof(uint32_t) * meta.size());
      d_tg_ = (double*)zeros(8 * pcg_onchip_t_doubles(ns));
      d_ocm_ = (double*)zeros(8 * pcg_onchip_m_doubles(ns));
    }
  }
  if (std::getenv("GF_CG_TRACE")) cg_.trace = (unsigned long long*)zeros(8 * 5000);
  if (const char* e = std::getenv("GF_GRAPH")) graphs_enabled_ = std::atoi(e) != 0;
  GF_CUDA(cudaEventCreate(&pcg_ev_[0]));
  GF_CUDA(cudaEventCreate(&pcg_ev_[1]));
  cg_.tol = cfg.cg_tol;
  GF_CUDA(cudaStreamSynchronize(stream_));
  GF_CUDA(cudaGetLastError());
  setup_s_[3] = secs(t_ctor);
  setup_s_[2] = setup_s_[3] - setup_s_[0] - setup_s_[1];
}

gf_sim_info Simulation::info() const {
  gf_sim_info o{};
  o.nodes = mesh_.nn;
  o.tets = mesh_.nt;
  o.edges = mesh_.ne;
  o.node_blocks = (int64_t)pat_.cols.size();
  o.upper_blocks = (o.node_blocks + o.nodes) / 2;
  o.upper_block_slots = 32 * (int64_t)usp_[d_.nslices];
  o.spmv_slots = 32 * sell_slots_;
  o.nl_entries = nl_entries_;
  o.nl_slots = mat_.r_d <= 0.0 ? 0 : d_.nl_tpl ? 32 * nl_tpl_slots_ : nl_ell_slots_;
  o.nl_layout = nonlocal_layout();
  o.pcg_dynamic_units = cg_ndyn_;
  o.pcg_solver = cg_.big ? 6 : cg_ndyn_ > 0 ? 4 : cg_.onchip ? (cg_.cluster ? 5 : 3) : !cg_.pipelined ? 0 : cg_.cluster ? 2 : 1;
  for (int b = 0; b < 7; ++b) {
    o.oc_slot_blocks[b] = cg_.onchip ? oc_slot_blocks_[b] : 0;
    o.oc_offsets[b] = cg_.onchip ? oc_off_[b] : 0;
  }
  for (int k = 0; k < 4; ++k) o.setup_s[k] = setup_s_[k];
  return o;
}

Simulation::~Simulation() {
  if (stream_) cudaStreamSynchronize(stream_);
  for (auto& e : step_exec_)
    if (e) cudaGraphExecDestroy(e);
  for (auto e : pcg_ev_)
    if (e) cudaEventDestroy(e);
  for (auto& p : pending_) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto e : event_pool_) cudaEventDestroy(e);
  for (auto e : timers_)
    if (e) cudaEventDestroy(e);
  for (void* p : allocs_) cudaFree(p);
  if (h_bcstep_) cudaFreeHost(h_bcstep_);
  if (h_cols_) cudaFreeHost(h_cols_);
  if (h_stats_) cudaFreeHost(h_stats_);
  if (h_partials_) cudaFreeHost(h_partials_);
  if (stream_) cudaStreamDestroy(stream_);
}

// ---------------------------------------------------------------- launch bookkeeping / profiling
template <class F>
void Simulation::launch(const char* name, double bytes, F&& f) {
  if (capturing_) {  // recorded into the step graph; counted at replay (dynamic_step)
    capture_list_.emplace_back(name, bytes);
    const bool ev = profiling_ == 2 && std::strcmp(name, "pcg") == 0;
    if (ev) GF_CUDA(cudaEventRecordWithFlags(pcg_ev_[0], stream_, cudaEventRecordExternal));  // an event node
    f();
    GF_CUDA(cudaGetLastError());
    if (ev) GF_CUDA(cudaEventRecordWithFlags(pcg_ev_[1], stream_, cudaEventRecordExternal));
    return;
  }
  if (!profiling_) {
    f();
    GF_CUDA(cudaGetLastError());
    return;
  }
  if (profiling_ == 2 && std::strcmp(name, "pcg") != 0) {  // launch count + bytes only, no events
    f();
    GF_CUDA(cudaGetLastError());
    auto& k = ktimes_[name];
    std::strncpy(k.name, name, sizeof(k.name) - 1);
    k.launches += 1;
    k.bytes += bytes;
    return;
  }
  auto take = [&]() {
    cudaEvent_t e;
    if (!event_pool_.empty()) {
      e = event_pool_.back();
      event_pool_.pop_back();
    } else {
      GF_CUDA(cudaEventCreate(&e));
    }
    return e;
  };
  Pending p{name, take(), take(), bytes};
  GF_CUDA(cudaEventRecord(p.a, stream_));
  f();
  GF_CUDA(cudaGetLastError());
  GF_CUDA(cudaEventRecord(p.b, stream_));
  pending_.push_back(p);
}

void Simulation::flush_events() {
  for (auto& p : pending_) {
    float ms = 0.f;
    GF_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
    auto& k = ktimes_[p.name];
    std::strncpy(k.name, p.name.c_str(), sizeof(k.name) - 1);
    k.launches += 1;
    k.total_ms += ms;
    k.bytes += p.bytes;
    event_pool_.push_back(p.a);
    event_pool_.push_back(p.b);
  }
  pending_.clear();
}

void Simulation::synchronize() {
  GF_CUDA(cudaStreamSynchronize(stream_));
  flush_events();
}

void Simulation::cg_trace(unsigned long long* out) {
  if (!cg_.trace) throw FormatError("CG trace disabled (set GF_CG_TRACE before creating the simulation)");
  GF_CUDA(cudaMemcpyAsync(out, cg_.trace, 8 * 5000, cudaMemcpyDeviceToHost, stream_));
  synchronize();
}

void Simulation::timer_record(int slot) {
  if (slot < 0 || slot >= 8) throw FormatError("timer slot must be in [0, 8)");
  if (!timers_[slot]) GF_CUDA(cudaEventCreate(&timers_[slot]));
  GF_CUDA(cudaEventRecord(timers_[slot], stream_));
}

double Simulation::timer_elapsed(int a, int b) {
  if (a < 0 || a >= 8 || b < 0 || b >= 8 || !timers_[a] || !timers_[b]) throw FormatError("timer slot not recorded");
  GF_CUDA(cudaEventSynchronize(timers_[b]));
  float ms = 0.f;
  GF_CUDA(cudaEventElapsedTime(&ms, timers_[a], timers_[b]));
  return ms;
}

std::vector<gf_kernel_time> Simulation::kernel_times() {
  synchronize();
  std::vector<gf_kernel_time> out;
  for (auto& kv : ktimes_) out.push_back(kv.second);
  return out;
}

// ---------------------------------------------------------------- damage pass (solver.cpp:90-103)
void Simulation::run_damage(bool relabel, bool keep_values, bool chi) {
  // algorithmic bytes: SURVEY.md §8(d) B_D = 16n + 128T + 10E + 12S + 4 n_new (n = 3N dofs), split by kernel
  const double n = 3.0 * mesh_.nn, T = mesh_.nt, E = mesh_.ne;
  const bool local = mat_.r_d <= 0.0;
  launch("tet_stress", 16 * n + 112 * T + 8 * E, [&] { launch_tet_stress(d_, md_, local, stream_); });
  if (!local) launch("nonlocal", 12.0 * nl_entries_, [&] { launch_nonlocal(d_, stream_); });
  launch("relabel", 2 * E, [&] { launch_relabel(d_, mat_.sigma_thres, relabel, keep_values, stream_); });
  if (chi) launch("chi", 16 * T, [&] { launch_chi(d_, md_, stream_); });
}

std::vector<int32_t> Simulation::damage_pass() {
  run_damage(true, false, true);
  int32_t n = 0;
  GF_CUDA(cudaMemcpyAsync(&n, d_.newly_count, 4, cudaMemcpyDeviceToHost, stream_));
  synchronize();
  std::vector<int32_t> ids(n);
  if (n) GF_CUDA(cudaMemcpy(ids.data(), d_.newly, 4 * (size_t)n, cudaMemcpyDeviceToHost));
  std::sort(ids.begin(), ids.end());  // update_damage returns ascending ids (fracture.hpp:48-50)
  if (viz_ && !ids.empty()) feed_viz(ids);
  return ids;
}

void Simulation::feed_viz(std::vector<int32_t> ids) {
  std::vector<uint8_t> zeta(mesh_.ne);
  GF_CUDA(cudaMemcpyAsync(zeta.data(), d_.zeta, zeta.size(), cudaMemcpyDeviceToHost, stream_));
  synchronize();
  std::sort(ids.begin(), ids.end());
  viz_->apply_splits(ids.data(), (int64_t)ids.size(), zeta.data());
}

RenderMesh& Simulation::viz() {
  if (!viz_) {
    viz_ = std::make_unique<RenderMesh>(mesh_);
    std::vector<uint8_t> zeta(mesh_.ne);
    GF_CUDA(cudaMemcpyAsync(zeta.data(), d_.zeta, zeta.size(), cudaMemcpyDeviceToHost, stream_));
    synchronize();
    std::vector<int32_t> broken;  // edges broken before the companion existed, ascending
    for (int32_t e = 0; e < mesh_.ne; ++e)
      if (zeta[e]) broken.push_back(e);
    viz_->apply_splits(broken.data(), (int64_t)broken.size(), zeta.data());
  }
  return *viz_;
}

// ---------------------------------------------------------------- dynamic step (solver.cpp:219-333)
void Simulation::upload_bc_step(double t, double dt) {
  for (size_t b = 0; b < bcs_.size(); ++b) {
    BcStep& s = h_bcstep_[b];
    std::memset(&s, 0, sizeof s);
    s.kind = bcs_[b].kind;
    bcs_[b].displacement_params(t, s.d0, s.R0);
    bcs_[b].displacement_params(t + dt, s.d1, s.R1);
    for (int a = 0; a < 3; ++a) s.axis_point[a] = bcs_[b].axis_point[a];
  }
  GF_CUDA(cudaMemcpyAsync(d_bcstep_, h_bcstep_, sizeof(BcStep) * bcs_.size(), cudaMemcpyHostToDevice, stream_));
}

void Simulation::launch_cg() {
  if (cg_.onchip) launch_pcg_onchip(cg_, d_slice_part_, d_tg_, d_ocm_, d_oc_meta_, oc_off_, stream_);
  else launch_pcg_sell(cg_, d_slice_part_, cg_ndyn_, d_ctr_, stream_);
}

double Simulation::run_cg(int max_iters) {
  cg_.max_iters = max_iters;
  const double N = mesh_.nn, NB = pat_.cols.size();
  // bytes are filled in after the run from the iteration count (see dynamic_step)
  launch("pcg", 0.0 * (N + NB), [&] { launch_cg(); });
  GF_CUDA(cudaMemcpyAsync(h_stats_, d_stats_, 64, cudaMemcpyDeviceToHost, stream_));  // the whole stats record
  synchronize();
  return h_stats_[0];
}

// solve_linear retries (solver.cpp:113-135) after a first attempt whose outcome is `ok`: 4x iterations, then
// cumulative diagonal shifts of |diag| (fixed dofs excluded) from 1e-8 up by 10x, 8 attempts, else SolveError
template <class Acc>
void Simulation::solve_ladder(bool ok, int32_t* iters, Acc&& account) {
  if (!ok) {
    *iters += (int32_t)run_cg(4 * cfg_.cg_max_iters);
    account(h_stats_[0]);
    ok = h_stats_[1] != 0.0;
  }
  if (!ok) {
    launch("absdiag", 0.0, [&] { launch_absdiag(d_, stream_); });
    double shift = 1e-8;
    for (int attempt = 0; attempt < 8 && !ok; ++attempt) {
      launch("shift_diag", 0.0, [&] { launch_shift_diag(d_, shift, stream_); });
      launch("bsr_dinv", 0.0, [&] { launch_bsr_dinv(d_, stream_); });
      launch("reset_x", 0.0, [&] { launch_reset_x(d_, stream_); });
      *iters += (int32_t)run_cg(cfg_.cg_max_iters);
      account(h_stats_[0]);
      ok = h_stats_[1] != 0.0;
      shift *= 10.0;
    }
    if (!ok) {
      std::ostringstream msg;
      msg << "linear solve failed: relative residual " << h_stats_[3] << " after " << (int)h_stats_[0]
          << " iterations" << (h_stats_[2] != 0.0 ? " (negative curvature)" : "");
      throw SolveError(msg.str());
    }
  }
}

// force + stiffness assembly (fem.cpp:96-169 fused with solver.cpp:275-295): the F-based row kernel, or the
// edge-length form (k_tet_edge once per tet -> records + fused energy, then the edge row kernel)
void Simulation::assemble(const StepCoeffs& c, int mode, const char* name, double bytes, bool energy_in_integrate) {
  if (edge_form_) {
    const double T = mesh_.nt, N = mesh_.nn;
    // reads conn 16, rest record 80, chi 8 per tet and X, u once (48 per node); writes the 224-byte record
    launch("tet_edge", 328.0 * T + 48.0 * N, [&] { launch_tet_edge(d_, md_, 0, stream_); });
  }
  launch(name, bytes, [&] { launch_assemble(d_, md_, c, mode, stream_); });
  // the F-based form's fused energy: per-row partials -> one deterministic sum, folded into the step's k_integrate
  // (dynamic_step) or a separate reduction (quasi-static Newton)
  if (!edge_form_ && mode == kAssembleSystem && !energy_in_integrate)
    launch("energy_sum", 8.0 * mesh_.nn,
           [&] { launch_dot(d_.eng_row, nullptr, mesh_.nn, d_energy_partials_, d_red_ticket_, d_.eng_out, stream_); });
}

void Simulation::check_edge_fallback() {  // h_stats_ holds the step's record
  if (!edge_form_) return;
  int32_t nf = 0;
  std::memcpy(&nf, h_stats_ + 6, 4);
  if (nf > d_.efall_cap)
    throw GeometryError("edge-length element form: " + std::to_string(nf) + " degenerate tets exceed the fallback capacity " +
                        std::to_string(d_.efall_cap) + " (use GF_ELEMENT=F)");
}

double Simulation::assembly_energy() {
  GF_CUDA(cudaMemcpyAsync(h_partials_, d_.eng_out, 8, cudaMemcpyDeviceToHost, stream_));
  synchronize();
  return h_partials_[0];
}

void Simulation::edge_forces(double* coeff6, uint8_t* ok) {  // edge_decomposed_forces (fem.cpp:57-94), every tet
  const size_t nt = (size_t)mesh_.nt;
  if (!d_.ecoef) {
    d_.ecoef = (double*)dalloc(48 * nt);
    d_.eok = (uint8_t*)dalloc(nt);
  }
  launch("edge_decomposition", 0.0, [&] { launch_tet_edge(d_, md_, 1, stream_); });
  GF_CUDA(cudaMemcpyAsync(coeff6, d_.ecoef, 48 * nt, cudaMemcpyDeviceToHost, stream_));
  GF_CUDA(cudaMemcpyAsync(ok, d_.eok, nt, cudaMemcpyDeviceToHost, stream_));
  synchronize();
}

// host-side per-step parameters (pinned records, read by the step's H2D copies): collider states at each substep
// probe time (solver.cpp:233-249, Schedule3 eval/rate) and the boundary-condition displacements at t and t + dt
// (solver.cpp:22-29, 255-262)
void Simulation::fill_step_params(double t, double dt) {
  const int nsub = cfg_.collision_substeps;
  const size_t nc = cols_.size();
  for (int s = 0; s < nsub && nc; ++s) {
    const double tau = dt * (double)s / (double)nsub;
    for (size_t c = 0; c < nc; ++c) {
      ColliderDev& k = h_cols_[s * nc + c];
      std::memset(&k, 0, sizeof k);
      k.kind = cols_[c].kind;
      if (k.kind == 0) {
        cols_[c].center.eval(t + tau, k.center);
        cols_[c].center.rate(t + tau, k.cvel);
      }
      k.radius = cols_[c].radius;
      for (int a = 0; a < 3; ++a) {
        k.point[a] = cols_[c].point[a];
        k.normal[a] = cols_[c].normal[a];
      }
      k.stiffness = cols_[c].stiffness;
      k.restitution = cols_[c].restitution;
      k.friction = cols_[c].friction;
    }
  }
  for (size_t b = 0; b < bcs_.size(); ++b) {
    BcStep& q = h_bcstep_[b];
    std::memset(&q, 0, sizeof q);
    q.kind = bcs_[b].kind;
    bcs_[b].displacement_params(t, q.d0, q.R0);
    bcs_[b].displacement_params(t + dt, q.d1, q.R1);
    for (int a = 0; a < 3; ++a) q.axis_point[a] = bcs_[b].axis_point[a];
  }
}

// the device work of one dynamic_step, enqueued on the stream (or captured into the step graph): no host decision
// inside, the only read-back is the 64-byte stats record at the end
void Simulation::enqueue_prologue(double dt) {  // damage pass, collider forces, BC targets (solver.cpp:225-262)
  run_damage(true, false, true);
  const int nsub = cfg_.collision_substeps;
  if (!cols_.empty()) {
    const size_t nc = cols_.size();
    GF_CUDA(cudaMemcpyAsync(d_cols_, h_cols_, sizeof(ColliderDev) * nc * nsub, cudaMemcpyHostToDevice, stream_));
    for (int s = 0; s < nsub; ++s) {
      const double tau = dt * (double)s / (double)nsub;
      launch("collide", 96.0 * mesh_.nn, [&] { launch_collide(d_, s, tau, dt, nsub, stream_); });
    }
    launch("collide_load", 0.0, [&] { launch_collide_load(d_, nsub, d_load_, stream_); });
  }
  if (!bcs_.empty()) {
    GF_CUDA(cudaMemcpyAsync(d_bcstep_, h_bcstep_, sizeof(BcStep) * bcs_.size(), cudaMemcpyHostToDevice, stream_));
    launch("bc_targets", 96.0 * n_fixed_, [&] { launch_bc_targets(d_, n_fixed_, d_fixed_nodes_, dt, stream_); });
  }
}

void Simulation::enqueue_step(double dt) {
  enqueue_prologue(dt);
  StepCoeffs c{};
  c.use_ext = 1;
  c.dt = dt;
  c.rhs_fint_scale = dt;
  c.rhs_mv_scale = dt * mat_.damp_mass_coeff;
  c.rhs_kv_scale = dt * mat_.damp_stiff_coeff + dt * dt;
  c.kscale = dt * mat_.damp_stiff_coeff + dt * dt;
  c.mscale = 1.0 + dt * mat_.damp_mass_coeff;
  // algorithmic bytes: SURVEY.md §8(d) B_F = 16n + 104T + 8Z (n = 3N dofs, Z scalar nonzeros)
  const double n = 3.0 * mesh_.nn, T = mesh_.nt, Z = 9.0 * pat_.cols.size();
  d_.fint_out = nullptr;
  assemble(c, kAssembleSystem, "assemble", 16 * n + 104 * T + 8 * Z, true);
  // solve_linear (solver.cpp:105-136): first attempt here; the 4x retry and the diagonal shifts run on the host
  // only when the stats record says this one failed
  cg_.max_iters = cfg_.cg_max_iters;
  cg_.x0_identity = 1;  // x0 from the assembly's epilogue (fixed rows: prescribed values, identity rows)
  launch("pcg", 0.0, [&] { launch_cg(); });
  cg_.x0_identity = 0;
  d_.eng_sum = edge_form_ ? 0 : 1;
  launch("integrate", 40 * n, [&] { launch_integrate(d_, dt, stream_); });  // B_int = 40n; no-op if not converged
  d_.eng_sum = 0;
  // cg_out, load, newly broken, edge-form fallback count, assembled-state energy
  GF_CUDA(cudaMemcpyAsync(h_stats_, d_stats_, 64, cudaMemcpyDeviceToHost, stream_));
}

// CUDA-graph step orchestration: the step's ~10 launches and copies are captured once per
// profiling level (0: none; 2: events around the PCG solve) and replayed; the per-step host parameters travel
// through pinned records that the graph's copy nodes read at replay time. Falls back to direct launches when the
// capture fails (GF_GRAPH=0 disables it).
bool Simulation::launch_step_graph(double dt) {
  if (!graphs_enabled_ || profiling_ == 1) return false;
  const int lvl = profiling_ == 2 ? 1 : 0;
  if (!step_exec_[lvl]) {
    capture_list_.clear();
    capturing_ = true;
    cudaGraph_t gr = nullptr;
    bool ok = cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    if (ok) {
      try {
        enqueue_step(dt);
      } catch (...) {
        ok = false;
      }
      ok = (cudaStreamEndCapture(stream_, &gr) == cudaSuccess) && ok;
    }
    capturing_ = false;
    if (ok) ok = cudaGraphInstantiate(&step_exec_[lvl], gr, 0) == cudaSuccess;
    if (gr) cudaGraphDestroy(gr);
    if (!ok) {
      cudaGetLastError();
      step_exec_[lvl] = nullptr;
      graphs_enabled_ = false;
      return false;
    }
    step_list_[lvl] = capture_list_;
  }
  GF_CUDA(cudaGraphLaunch(step_exec_[lvl], stream_));
  replayed_ = lvl + 1;
  return true;
}

// dynamic_full_newton (solver.cpp:264-313): Newton iterations on the backward-Euler residual
// M dv - dt (f_ext + f(u_start + dt v+) - B v+), each a fused assembly + PCG solve. The system assembled at a trial
// state is exactly the next iteration's (its rhs is -residual, fixed rows 0), so the residual norm is taken from it and
// it is reused -- one assembly per iteration where the reference assembles twice.
gf_step_stats Simulation::dynamic_step_full_newton() {
  gf_step_stats st{};
  const double t = time_, dt = cfg_.dt;
  const size_t nd = 3 * (size_t)mesh_.nn;
  if (!d_usave_) {
    d_usave_ = (double*)dalloc(8 * nd);
    d_ubackup_ = (double*)dalloc(8 * nd);
  }
  double* dv_total = d_ubackup_;
  fill_step_params(t, dt);
  enqueue_prologue(dt);
  GF_CUDA(cudaMemcpyAsync(d_usave_, d_.u, 8 * nd, cudaMemcpyDeviceToDevice, stream_));
  GF_CUDA(cudaMemsetAsync(dv_total, 0, 8 * nd, stream_));
  const double n = (double)nd, T = mesh_.nt, Z = 9.0 * pat_.cols.size();
  double msum = 0.0;
  for (double m : mass_) msum += 3.0 * m;
  const double tol = std::max(newton_tol_, 1e-12 * msum);
  auto coeffs = [&](int outer) {
    StepCoeffs c{};
    c.use_ext = 1;
    c.dt = dt;
    c.rhs_fint_scale = dt;
    c.rhs_mv_scale = dt * mat_.damp_mass_coeff;
    c.rhs_kv_scale = dt * mat_.damp_stiff_coeff + (outer == 0 ? dt * dt : 0.0);
    c.kscale = dt * mat_.damp_stiff_coeff + dt * dt;
    c.mscale = 1.0 + dt * mat_.damp_mass_coeff;
    c.fixed_zero = outer > 0;
    c.mdv = outer > 0 ? dv_total : nullptr;
    return c;
  };
  d_.fint_out = nullptr;
  assemble(coeffs(0), kAssembleSystem, "assemble", 16 * n + 104 * T + 8 * Z);
  for (int outer = 0; outer < cfg_.newton_max_iters; ++outer) {
    cg_.x0_identity = 1;
    st.cg_iterations += (int32_t)run_cg(cfg_.cg_max_iters);
    cg_.x0_identity = 0;
    if (outer == 0) {
      check_edge_fallback();
      int32_t newly = 0;
      std::memcpy(&newly, h_stats_ + 5, 4);
      st.newly_broken = newly;
      last_load_ = cols_.empty() ? 0.0 : h_stats_[4];
      st.load = last_load_;
    }
    solve_ladder(h_stats_[1] != 0.0, &st.cg_iterations, [](double) {});
    launch("newton_update", 56.0 * n, [&] { launch_newton_update(d_, dv_total, d_usave_, dt, stream_); });
    // the residual at the trial state = -(the next iteration's rhs), fixed dofs 0 (solver.cpp:298-312)
    assemble(coeffs(outer + 1), kAssembleSystem, "assemble", 16 * n + 104 * T + 8 * Z);
    st.newton_iterations = outer + 1;
    if (std::sqrt(device_dot(d_.rhs, d_.rhs, (int64_t)nd)) <= tol) break;
  }
  if (!bcs_.empty()) launch("pin_bc", 96.0 * n_fixed_, [&] { launch_pin_bc(d_, stream_); });
  if (viz_ && st.newly_broken > 0) {
    std::vector<int32_t> ids(st.newly_broken);
    GF_CUDA(cudaMemcpyAsync(ids.data(), d_.newly, 4 * (size_t)st.newly_broken, cudaMemcpyDeviceToHost, stream_));
    feed_viz(std::move(ids));
  }
  synchronize();
  time_ = t + dt;
  st.residual = 0.0;
  return st;
}

gf_step_stats Simulation::dynamic_step() {
  if (cfg_.dynamic_full_newton) return dynamic_step_full_newton();
  gf_step_stats st{};
  const double t = time_, dt = cfg_.dt;
  fill_step_params(t, dt);
  replayed_ = 0;
  if (!launch_step_graph(dt)) enqueue_step(dt);
  synchronize();
  if (replayed_ && profiling_) {  // launch counts, bytes and the PCG's event time of the replayed step
    for (const auto& it : step_list_[replayed_ - 1]) {
      auto& k = ktimes_[it.first];
      std::strncpy(k.name, it.first.c_str(), sizeof(k.name) - 1);
      k.launches += 1;
      k.bytes += it.second;
    }
    if (replayed_ == 2) {
      float ms = 0.f;
      GF_CUDA(cudaEventElapsedTime(&ms, pcg_ev_[0], pcg_ev_[1]));
      ktimes_["pcg"].total_ms += ms;
    }
  }
  const double n = 3.0 * mesh_.nn;
  // PCG algorithmic bytes per iteration for THIS format: every stored upper block and slot word
  // once, plus the vectors that leave the chip -- z gathered and written (24 B per node each) when the solver
  // state stays on chip (one slice per warp); p, q, x, r, D^-1 traffic as well when it does not (large
  // matrices). The reference's scalar-CSR model (SURVEY §8(d) B_CG = 12Z + 4(n+1) + 56n) is reported by bench.py
  // next to it.
  double cg_bytes_per_iter = 72.0 * ((double)pat_.cols.size() + mesh_.nn) / 2.0 + 4.0 * 32.0 * (double)sell_slots_ +
                             (cg_ndyn_ ? 312.0 : 48.0) * mesh_.nn;
  if (cg_.onchip) {  // the matrix stays on chip: per iteration the column gathers and the remote t (written and read)
                     // of slots 3..6, and m (bench.py pcg_models); the matrix load once per solve is added below
    double t = 0.0;
    for (int b = 3; b < 7; ++b) t += (double)oc_slot_blocks_[b];
    cg_bytes_per_iter = 72.0 * t + 24.0 * mesh_.nn;
  }
  // k_pcg_onchip loads the matrix (upper blocks incl. slice padding) once per solve
  const double cg_bytes_per_solve = cg_.onchip ? 72.0 * 32.0 * (double)usp_[d_.nslices] : 0.0;
  auto account = [&](double iters) {
    if (profiling_) ktimes_["pcg"].bytes += iters * cg_bytes_per_iter + cg_bytes_per_solve;
  };
  check_edge_fallback();
  int32_t newly = 0;
  std::memcpy(&newly, h_stats_ + 5, 4);
  st.newly_broken = newly;
  if (viz_ && newly > 0) {  // the render companion follows this step's damage pass (solver.cpp:94)
    std::vector<int32_t> ids(newly);
    GF_CUDA(cudaMemcpyAsync(ids.data(), d_.newly, 4 * (size_t)newly, cudaMemcpyDeviceToHost, stream_));
    feed_viz(std::move(ids));
  }
  last_load_ = cols_.empty() ? 0.0 : h_stats_[4];
  st.load = last_load_;
  st.cg_iterations = (int32_t)h_stats_[0];
  account(h_stats_[0]);
  if (h_stats_[1] == 0.0) {
    solve_ladder(false, &st.cg_iterations, account);
    launch("integrate", 40 * n, [&] { launch_integrate(d_, dt, stream_); });
  }
  time_ = t + dt;
  st.residual = 0.0;
  return st;
}

// ---------------------------------------------------------------- quasi-static step (solver.cpp:138-217)
double Simulation::device_dot(const double* a, const double* b, int64_t n) {
  launch("dot", 16.0 * n, [&] { launch_dot(a, b, n, d_energy_partials_, d_red_ticket_, d_red_out_, stream_); });
  GF_CUDA(cudaMemcpyAsync(h_partials_, d_red_out_, 8, cudaMemcpyDeviceToHost, stream_));
  synchronize();
  return h_partials_[0];
}

// k_metrics: [strain energy, kinetic energy, chi sum, broken edges, chi min] of the current state, one 40-byte read
void Simulation::device_metrics(double out[5]) {
  launch("metrics", 0.0, [&] { launch_metrics(d_, md_, d_energy_partials_, d_red_ticket_, d_red_out_, stream_); });
  GF_CUDA(cudaMemcpyAsync(h_partials_, d_red_out_, 40, cudaMemcpyDeviceToHost, stream_));
  synchronize();
  for (int k = 0; k < 5; ++k) out[k] = h_partials_[k];
}

double Simulation::device_strain_energy() {
  double m[5];
  device_metrics(m);
  return m[0];
}

void Simulation::apply_boundary_displacements(double t) {  // solver.cpp:74-77, plus zero Newton increments
  if (bcs_.empty()) return;
  upload_bc_step(t, 0.0);
  launch("qs_bc", 0.0, [&] { launch_qs_bc(d_, n_fixed_, d_fixed_nodes_, stream_); });
}

// newton_solve (solver.cpp:143-188): one fused assembly pass gives the residual (f_int, fixed dofs zeroed) and
// the projected tangent K; the norm check precedes the solve, so the final (converged) pass's matrix is unused
bool Simulation::newton_solve(gf_step_stats& st) {
  const size_t nd = 3 * (size_t)mesh_.nn;
  const double n = (double)nd, T = mesh_.nt, Z = 9.0 * pat_.cols.size();
  StepCoeffs c{};
  c.use_ext = 0;
  c.rhs_fint_scale = 1.0;
  c.kscale = 1.0;
  d_.fint_out = nullptr;
  auto account = [](double) {};
  for (int it = 0; it <= cfg_.newton_max_iters; ++it) {
    assemble(c, kAssembleSystem, "assemble", 16 * n + 104 * T + 8 * Z);
    const double rr = device_dot(d_.rhs, d_.rhs, (int64_t)nd);
    st.residual = std::sqrt(rr);
    st.newton_iterations = it;
    if (st.residual <= newton_tol_) return true;
    if (it == cfg_.newton_max_iters) return false;
    st.cg_iterations += (int32_t)run_cg(cfg_.cg_max_iters);
    solve_ladder(h_stats_[1] != 0.0, &st.cg_iterations, account);
    // line search on the degraded strain energy (solver.cpp:166-186)
    const double e0 = device_strain_energy();
    double slope = -device_dot(d_.rhs, d_.x, (int64_t)nd);
    if (slope >= 0.0) {  // steepest-descent fallback
      GF_CUDA(cudaMemcpyAsync(d_.x, d_.rhs, 8 * nd, cudaMemcpyDeviceToDevice, stream_));
      slope = -rr;
    }
    GF_CUDA(cudaMemcpyAsync(d_usave_, d_.u, 8 * nd, cudaMemcpyDeviceToDevice, stream_));
    double step = 1.0;
    bool accepted = false;
    for (int h = 0; h <= cfg_.ls_max_halvings; ++h) {
      launch("qs_update", 24.0 * n, [&] { launch_qs_update(d_.u, d_usave_, d_.x, step, (int64_t)nd, stream_); });
      const double e1 = device_strain_energy();
      if (e1 <= e0 + cfg_.ls_sufficient_decrease * step * slope) {
        accepted = true;
        break;
      }
      step *= cfg_.ls_backtrack;
    }
    if (!accepted) GF_CUDA(cudaMemcpyAsync(d_.u, d_usave_, 8 * nd, cudaMemcpyDeviceToDevice, stream_));
  }
  return false;
}

gf_step_stats Simulation::quasi_static_step(double t_load) {
  gf_step_stats st{};
  const size_t nd = 3 * (size_t)mesh_.nn;
  if (!d_usave_) {
    d_usave_ = (double*)dalloc(8 * nd);
    d_ubackup_ = (double*)dalloc(8 * nd);
  }
  double current = quasi_time_;
  double increment = t_load - current;
  if (increment <= 0.0) {
    apply_boundary_displacements(t_load);
    if (!newton_solve(st)) throw SolveError("equilibrium solve failed at fixed load");
  } else {
    int halvings = 0;
    // only the displacements change inside a load increment, so they are the whole backup (solver.cpp:195)
    GF_CUDA(cudaMemcpyAsync(d_ubackup_, d_.u, 8 * nd, cudaMemcpyDeviceToDevice, stream_));
    while (current < t_load - 1e-15) {
      const double target = std::min(t_load, current + increment);
      apply_boundary_displacements(target);
      if (newton_solve(st)) {
        current = target;
        GF_CUDA(cudaMemcpyAsync(d_ubackup_, d_.u, 8 * nd, cudaMemcpyDeviceToDevice, stream_));
      } else {
        GF_CUDA(cudaMemcpyAsync(d_.u, d_ubackup_, 8 * nd, cudaMemcpyDeviceToDevice, stream_));
        ++halvings;
        if (halvings > 10) {
          std::ostringstream msg;
          msg << "quasi-static step failed: Newton did not reach " << newton_tol_ << " (residual " << st.residual
              << ") after 10 load halvings at load time " << target;
          throw SolveError(msg.str());
        }
        increment *= 0.5;
      }
    }
  }
  quasi_time_ = t_load;
  time_ = t_load;
  st.newly_broken = (int32_t)damage_pass().size();
  return st;
}

// ---------------------------------------------------------------- state access
void Simulation::get_state(double* u, double* v, uint8_t* zeta, double* chi, double* time) {
  const size_t nd = 3 * (size_t)mesh_.nn;
  if (u) GF_CUDA(cudaMemcpyAsync(u, d_.u, 8 * nd, cudaMemcpyDeviceToHost, stream_));
  if (v) GF_CUDA(cudaMemcpyAsync(v, d_.v, 8 * nd, cudaMemcpyDeviceToHost, stream_));
  if (zeta) GF_CUDA(cudaMemcpyAsync(zeta, d_.zeta, mesh_.ne, cudaMemcpyDeviceToHost, stream_));
  if (chi) GF_CUDA(cudaMemcpyAsync(chi, d_.chi, 8 * (size_t)mesh_.nt, cudaMemcpyDeviceToHost, stream_));
  synchronize();
  if (time) *time = time_;
}

void Simulation::set_state(const double* u, const double* v, const uint8_t* zeta, const double* chi,
                           const double* time, bool async) {
  const size_t nd = 3 * (size_t)mesh_.nn;
  if (u) GF_CUDA(cudaMemcpyAsync(d_.u, u, 8 * nd, cudaMemcpyHostToDevice, stream_));
  if (v) GF_CUDA(cudaMemcpyAsync(d_.v, v, 8 * nd, cudaMemcpyHostToDevice, stream_));
  if (zeta) GF_CUDA(cudaMemcpyAsync(d_.zeta, zeta, mesh_.ne, cudaMemcpyHostToDevice, stream_));
  if (chi) GF_CUDA(cudaMemcpyAsync(d_.chi, chi, 8 * (size_t)mesh_.nt, cudaMemcpyHostToDevice, stream_));
  if (time) time_ = *time;
  if (!async) synchronize();  // async (pinned sources): the copies are stream-ordered before the next step
}

void Simulation::set_external_forces(const double* f3n) {
  const size_t nd = 3 * (size_t)mesh_.nn;
  std::vector<double> fext(nd);
  for (int32_t i = 0; i < mesh_.nn; ++i)
    for (int a = 0; a < 3; ++a) {
      const size_t k = 3 * (size_t)i + a;
      fext[k] = mass_[i] * cfg_.gravity[a];
      if (f3n) fext[k] += f3n[k];
    }
  GF_CUDA(cudaMemcpyAsync(d_.fext, fext.data(), 8 * nd, cudaMemcpyHostToDevice, stream_));
  synchronize();
}

int64_t Simulation::broken_edge_count() {  // SimState::broken_edge_count, a device reduction
  double m[5];
  device_metrics(m);
  return (int64_t)m[3];
}

void Simulation::mass(double* m3n) const {
  for (int32_t i = 0; i < mesh_.nn; ++i)
    for (int a = 0; a < 3; ++a) m3n[3 * (size_t)i + a] = mass_[i];
}

// ---------------------------------------------------------------- parity / microbench hooks
void Simulation::eval_forces(double* f3n) {
  const size_t nd = 3 * (size_t)mesh_.nn;
  StepCoeffs c{};
  d_.fint_out = d_.r;  // scratch
  assemble(c, kAssembleForcesOnly, "forces", 0.0);
  d_.fint_out = nullptr;
  GF_CUDA(cudaMemcpyAsync(f3n, d_.r, 8 * nd, cudaMemcpyDeviceToHost, stream_));
  synchronize();
}

void Simulation::bsr_to_csr(const std::vector<double>& bval, double* vals) const {
  for (int32_t i = 0; i < mesh_.nn; ++i) {
    const int32_t r0 = pat_.row_ptr[i], deg = pat_.row_ptr[i + 1] - r0;
    for (int32_t q = 0; q < deg; ++q) {
      const int32_t j = pat_.cols[r0 + q];
      double blk[9];
      if (j >= i) {
        for (int r = 0; r < 9; ++r) blk[r] = bval[sell_addr(usp_.data(), i, uslot_[r0 + q], r)];
      } else {  // (i,j) = (j,i)^T
        const auto jb = pat_.cols.begin() + pat_.row_ptr[j], je = pat_.cols.begin() + pat_.row_ptr[j + 1];
        const int32_t qj = pat_.row_ptr[j] + (int32_t)(std::lower_bound(jb, je, i) - jb);
        for (int a = 0; a < 3; ++a)
          for (int c = 0; c < 3; ++c) blk[3 * a + c] = bval[sell_addr(usp_.data(), j, uslot_[qj], 3 * c + a)];
      }
      for (int a = 0; a < 3; ++a)
        for (int c = 0; c < 3; ++c) vals[9 * (size_t)r0 + 3 * (size_t)a * deg + 3 * q + c] = blk[3 * a + c];
    }
  }
}

void Simulation::eval_stiffness(double* vals) {
  StepCoeffs c{};
  assemble(c, kAssembleRawK, "stiffness", 0.0);
  std::vector<double> b(bval_doubles_);
  GF_CUDA(cudaMemcpyAsync(b.data(), d_.bval, 8 * b.size(), cudaMemcpyDeviceToHost, stream_));
  synchronize();
  bsr_to_csr(b, vals);
}

void Simulation::last_system(double* vals, double* rhs) {
  std::vector<double> b(bval_doubles_);
  GF_CUDA(cudaMemcpyAsync(b.data(), d_.bval, 8 * b.size(), cudaMemcpyDeviceToHost, stream_));
  if (rhs) GF_CUDA(cudaMemcpyAsync(rhs, d_.rhs, 24 * (size_t)mesh_.nn, cudaMemcpyDeviceToHost, stream_));
  synchronize();
  if (vals) bsr_to_csr(b, vals);
}

void Simulation::eval_cauchy(double* sigma6) {
  launch("tet_stress", 0.0, [&] { launch_tet_stress(d_, md_, false, stream_); });
  if (!d_.nl_tpl) {
    GF_CUDA(cudaMemcpyAsync(sigma6, d_.sigc, 48 * (size_t)mesh_.nt, cudaMemcpyDeviceToHost, stream_));
    synchronize();
    return;
  }
  const size_t nt = (size_t)mesh_.nt;
  std::vector<double> planes(6 * nt);
  GF_CUDA(cudaMemcpyAsync(planes.data(), d_.sigc, 48 * nt, cudaMemcpyDeviceToHost, stream_));
  synchronize();
  for (size_t e = 0; e < nt; ++e) {
    const size_t pos = (e % 6) * (size_t)d_.nl_ncell + e / 6;
    for (int p = 0; p < 3; ++p)
      for (int c = 0; c < 2; ++c) sigma6[6 * e + 2 * p + c] = planes[2 * (p * nt + pos) + c];
  }
}

void Simulation::eval_screening(double* screening, double* sigma_f6, uint8_t* degenerate) {
  run_damage(false, true, false);
  if (screening) GF_CUDA(cudaMemcpyAsync(screening, d_.screening, 8 * (size_t)mesh_.ne, cudaMemcpyDeviceToHost, stream_));
  if (sigma_f6) GF_CUDA(cudaMemcpyAsync(sigma_f6, d_.sigf, 48 * (size_t)mesh_.nt, cudaMemcpyDeviceToHost, stream_));
  if (degenerate) GF_CUDA(cudaMemcpyAsync(degenerate, d_.deg, mesh_.nt, cudaMemcpyDeviceToHost, stream_));
  synchronize();
}

void Simulation::spmv(const double* x, double* y) {
  const size_t nd = 3 * (size_t)mesh_.nn;
  GF_CUDA(cudaMemcpyAsync(d_.z, x, 8 * nd, cudaMemcpyHostToDevice, stream_));
  launch("spmv", 0.0, [&] { launch_spmv_sym(cg_, d_.z, d_.Ap, stream_); });
  GF_CUDA(cudaMemcpyAsync(y, d_.Ap, 8 * nd, cudaMemcpyDeviceToHost, stream_));
  synchronize();
}

// the production PCG (k_pcg_sell) on a caller-provided matrix with the mesh's pattern (scalar-CSR order, symmetric:
// the upper blocks are stored, the lower ones implied) -- cg_solve (sparse.cpp:129-188) as a parity hook. Replaces
// the simulation's current system; D^-1 from the diagonal as sparse.cpp:133-136.
void Simulation::solve_system(const double* vals, const double* b, const double* x0, double tol, int32_t max_iters,
                              double* x, gf_cg_result* res) {
  if (max_iters < 0) throw FormatError("max_iters must be non-negative");
  const size_t nd = 3 * (size_t)mesh_.nn;
  std::vector<double> bv(bval_doubles_, 0.0), dinv(nd, 1.0);
  bool diag_sym = true;  // the on-chip solver stores the diagonal block's upper triangle only
  for (int32_t i = 0; i < mesh_.nn; ++i) {
    const int32_t r0 = pat_.row_ptr[i], deg = pat_.row_ptr[i + 1] - r0;
    for (int32_t q = 0; q < deg; ++q) {
      const int32_t j = pat_.cols[r0 + q];
      for (int a = 0; a < 3; ++a)
        for (int c = 0; c < 3; ++c) {
          const double v = vals[9 * (size_t)r0 + 3 * (size_t)a * deg + 3 * q + c];
          if (j >= i) bv[sell_addr(usp_.data(), i, uslot_[r0 + q], 3 * a + c)] = v;
          if (j == i && a == c) dinv[3 * (size_t)i + a] = std::fabs(v) > 1e-300 ? 1.0 / v : 1.0;
          if (j == i && c < a && v != vals[9 * (size_t)r0 + 3 * (size_t)c * deg + 3 * q + a]) diag_sym = false;
        }
    }
  }
  struct Restore {  // a caller's matrix with an asymmetric diagonal block takes k_pcg_pipe
    int32_t& flag;
    int32_t saved;
    ~Restore() { flag = saved; }
  } restore{cg_.onchip, cg_.onchip};
  if (!diag_sym) cg_.onchip = 0;
  GF_CUDA(cudaMemcpyAsync(d_.bval, bv.data(), 8 * bv.size(), cudaMemcpyHostToDevice, stream_));
  GF_CUDA(cudaMemcpyAsync(d_.dinv, dinv.data(), 8 * nd, cudaMemcpyHostToDevice, stream_));
  GF_CUDA(cudaMemcpyAsync(d_.rhs, b, 8 * nd, cudaMemcpyHostToDevice, stream_));
  if (x0) GF_CUDA(cudaMemcpyAsync(d_.x, x0, 8 * nd, cudaMemcpyHostToDevice, stream_));
  else GF_CUDA(cudaMemsetAsync(d_.x, 0, 8 * nd, stream_));
  const double tol0 = cg_.tol;
  cg_.tol = tol;
  cg_.x0_identity = 0;
  try {
    run_cg(max_iters);
  } catch (...) {
    cg_.tol = tol0;
    throw;
  }
  cg_.tol = tol0;
  GF_CUDA(cudaMemcpyAsync(x, d_.x, 8 * nd, cudaMemcpyDeviceToHost, stream_));
  synchronize();
  res->iterations = (int32_t)h_stats_[0];
  res->converged = h_stats_[1] != 0.0;
  res->negative_curvature = h_stats_[2] != 0.0;
  res->relative_residual = h_stats_[3];
}

double Simulation::reaction_load(const int32_t* nodes, int32_t n, const double axis[3]) {  // solver.cpp:335-340
  std::vector<double> f(3 * (size_t)mesh_.nn);
  eval_forces(f.data());
  double tot[3] = {0, 0, 0};
  for (int32_t q = 0; q < n; ++q)
    for (int a = 0; a < 3; ++a) tot[a] += f[3 * (size_t)nodes[q] + a];
  return -((tot[0] * axis[0] + tot[1] * axis[1]) + tot[2] * axis[2]);
}

void Simulation::energies(double* strain, double* kinetic) {  // total_strain_energy + kinetic_energy (fem.cpp:190-206)
  double m[5];
  device_metrics(m);
  if (strain) *strain = m[0];
  if (kinetic) *kinetic = m[1];
}

gf_step_metrics Simulation::step_metrics() {  // run_scenario's make_row + log_damage (scenario.cpp:640-672)
  double m[5];
  device_metrics(m);
  gf_step_metrics r{};
  r.strain_energy = m[0];
  r.kinetic_energy = m[1];
  r.chi_mean = m[2] / (double)mesh_.nt;
  r.broken_edges = (int64_t)m[3];
  r.chi_min = m[4];
  r.time = time_;
  return r;
}

}  // namespace gfb

namespace gfb {
// cg_solve on a caller-provided scalar CSR (sparse.cpp:129-188): the same cooperative kernel, B = 1
void cg_solve_csr(int32_t n, const int32_t* row_ptr, const int32_t* cols, const double* vals, const double* b,
                  double* x, double tol, int32_t max_iters, gf_cg_result* res) {
  cudaStream_t s;
  GF_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  const int64_t nnz = row_ptr[n];
  std::vector<void*> bufs;
  auto alloc = [&](size_t bytes) {
    void* p = nullptr;
    GF_CUDA(cudaMalloc(&p, bytes ? bytes : 8));
    bufs.push_back(p);
    return p;
  };
  auto cleanup = [&]() {
    for (void* p : bufs) cudaFree(p);
    cudaStreamDestroy(s);
  };
  try {
    CgLaunch a{};
    a.nrows = n;
    a.row_ptr = (const int32_t*)alloc(4 * (size_t)(n + 1));
    a.cols = (const int32_t*)alloc(4 * (size_t)nnz);
    a.vals = (const double*)alloc(8 * (size_t)nnz);
    a.b = (const double*)alloc(8 * (size_t)n);
    a.x = (double*)alloc(8 * (size_t)n);
    a.dinv = (const double*)alloc(8 * (size_t)n);
    a.r = (double*)alloc(8 * (size_t)n);
    a.z = (double*)alloc(8 * (size_t)n);
    a.p0 = (double*)alloc(8 * (size_t)n);
    a.p1 = (double*)alloc(8 * (size_t)n);
    a.Ap = (double*)alloc(8 * (size_t)n);
    a.partials = (double*)alloc(8 * 2 * 3 * (size_t)cg_csr_grid());
    a.out = (double*)alloc(8 * 4);
    a.tol = tol;
    a.max_iters = max_iters;
    GF_CUDA(cudaMemcpyAsync((void*)a.row_ptr, row_ptr, 4 * (size_t)(n + 1), cudaMemcpyHostToDevice, s));
    GF_CUDA(cudaMemcpyAsync((void*)a.cols, cols, 4 * (size_t)nnz, cudaMemcpyHostToDevice, s));
    GF_CUDA(cudaMemcpyAsync((void*)a.vals, vals, 8 * (size_t)nnz, cudaMemcpyHostToDevice, s));
    GF_CUDA(cudaMemcpyAsync((void*)a.b, b, 8 * (size_t)n, cudaMemcpyHostToDevice, s));
    GF_CUDA(cudaMemcpyAsync(a.x, x, 8 * (size_t)n, cudaMemcpyHostToDevice, s));
    launch_pcg_csr(a, s);
    double out[4];
    GF_CUDA(cudaMemcpyAsync(out, a.out, 32, cudaMemcpyDeviceToHost, s));
    GF_CUDA(cudaMemcpyAsync(x, a.x, 8 * (size_t)n, cudaMemcpyDeviceToHost, s));
    GF_CUDA(cudaStreamSynchronize(s));
    res->iterations = (int32_t)out[0];
    res->converged = out[1] != 0.0;
    res->negative_curvature = out[2] != 0.0;
    res->relative_residual = out[3];
  } catch (...) {
    cleanup();
    throw;
  }
  cleanup();
}
}  // namespace gfb
