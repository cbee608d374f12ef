// metrics.cu — per-step metrics and scalar reductions on the device: one small record is read
// back instead of O(N) / O(T) host copies.
//
//  k_metrics  the run loop's per-step row and damage-log statistics (scenario.cpp:640-650, 660-672):
//             total_strain_energy (fem.cpp:190-199: chi V Psi(F) of every tet with chi V != 0), kinetic_energy
//             (fem.cpp:201-206: 1/2 m |v|^2 per node), broken-edge count (SimState::broken_edge_count), chi min and
//             chi sum (log_damage's chi_min / chi_mean).
//  k_dot      a . b (the quasi-static Newton residual norm and line-search slope, solver.cpp:148, 168), or sum a
//             (b = null: the fused assembly energy's per-row partials).
// Deterministic: a fixed partition of kBlocks blocks (independent of the device), per-block fixed trees, and the
// last block to finish (ticket) sums the block partials in block order and writes the result, so the values are
// bit-reproducible run to run. They differ from the reference's serial ascending sums at rounding level only.
#include "device_math.cuh"

namespace gfb {
namespace {

constexpr int kTpb = 256;
constexpr int kBlocks = 296;
constexpr int kFields = 5;  // strain energy, kinetic energy, chi sum, broken edges, chi min

__device__ __forceinline__ double block_tree(double v, double* s, bool is_min) {
  s[threadIdx.x] = v;
  __syncthreads();
  for (int o = kTpb / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) s[threadIdx.x] = is_min ? fmin(s[threadIdx.x], s[threadIdx.x + o]) : s[threadIdx.x] + s[threadIdx.x + o];
    __syncthreads();
  }
  const double r = s[0];
  __syncthreads();
  return r;
}

// the last block of a kBlocks-block reduction: returns true in every thread of that block (after a fence)
__device__ __forceinline__ bool last_block(unsigned* ticket) {
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1u) == kBlocks - 1;
  __syncthreads();
  return s_last;
}

__global__ void __launch_bounds__(kTpb) k_metrics(DevData d, MatDev m, double* partials, unsigned* ticket, double* out) {
  __shared__ double s[kTpb];
  const int tid = blockIdx.x * kTpb + threadIdx.x, stride = kBlocks * kTpb;
  double en = 0.0, chi_sum = 0.0, chi_min = 1.0, ke = 0.0, broken = 0.0;
  for (int e = tid; e < d.nt; e += stride) {
    const double chi = d.chi[e];
    chi_sum += chi;
    chi_min = fmin(chi_min, chi);
    double B[9], vol;
    load_rest(d, e, B, vol);
    const double scale = chi * vol;
    if (scale == 0.0) continue;  // fem.cpp:194
    const int4 t = __ldg(d.tets + e);
    const int id[4] = {t.x, t.y, t.z, t.w};
    double du[9], F[9];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int r = 0; r < 3; ++r) du[3 * r + c] = d.u[3 * (size_t)id[c + 1] + r] - d.u[3 * (size_t)id[0] + r];
    def_grad(du, B, F);
    en += scale * energy_density(F, m);
  }
  for (int i = tid; i < d.nn; i += stride) {
    const double* v = d.v + 3 * (size_t)i;
    ke += 0.5 * __ldg(d.mass + i) * ((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]);
  }
  for (int k = tid; k < d.ne; k += stride) broken += d.zeta[k] ? 1.0 : 0.0;
  const double vals[kFields] = {en, ke, chi_sum, broken, chi_min};
#pragma unroll
  for (int f = 0; f < kFields; ++f) {
    const double r = block_tree(vals[f], s, f == 4);
    if (threadIdx.x == 0) partials[f * kBlocks + blockIdx.x] = r;
  }
  if (!last_block(ticket)) return;
  if ((int)threadIdx.x < kFields) {
    const int f = threadIdx.x;
    double acc = f == 4 ? 1.0 : 0.0;
    for (int b = 0; b < kBlocks; ++b) {
      const double p = __ldcg(partials + f * kBlocks + b);
      acc = f == 4 ? fmin(acc, p) : acc + p;
    }
    out[f] = acc;
  }
  if (threadIdx.x == 0) *ticket = 0u;
}

__global__ void __launch_bounds__(kTpb) k_dot(const double* a, const double* b, int64_t n, double* partials,
                                              unsigned* ticket, double* out) {
  __shared__ double s[kTpb];
  double acc = 0.0;
  for (int64_t k = (int64_t)blockIdx.x * kTpb + threadIdx.x; k < n; k += (int64_t)kBlocks * kTpb) acc += b ? a[k] * b[k] : a[k];
  const double r = block_tree(acc, s, false);
  if (threadIdx.x == 0) partials[blockIdx.x] = r;
  if (!last_block(ticket)) return;
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < kBlocks; ++q) t += __ldcg(partials + q);
    *out = t;
    *ticket = 0u;
  }
}

}  // namespace

size_t metrics_partial_doubles() { return (size_t)kFields * kBlocks; }

void launch_metrics(const DevData& d, const MatDev& m, double* partials, unsigned* ticket, double* out, cudaStream_t s) {
  k_metrics<<<kBlocks, kTpb, 0, s>>>(d, m, partials, ticket, out);
}

void launch_dot(const double* a, const double* b, int64_t n, double* partials, unsigned* ticket, double* out,
                cudaStream_t s) {
  k_dot<<<kBlocks, kTpb, 0, s>>>(a, b, n, partials, ticket, out);
}

}  // namespace gfb
