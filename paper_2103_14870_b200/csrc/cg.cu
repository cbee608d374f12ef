// cg.cu — Jacobi-preconditioned CG (cg_solve, sparse.cpp:129-188) on a caller-provided scalar CSR matrix
// (gf_cg_solve_csr, the parity hook for the reference's free function) as ONE persistent cooperative kernel.
//
// The simulation's own solver is cg_sell.cu (symmetric node-block SELL-32); this one keeps the reference's
// matrix format. The whole solve runs on the device: no host round-trip per iteration. Every block reaches the
// same scalars (alpha, beta, convergence) because block partial sums are reduced by every warp in one fixed
// order after a grid barrier — the run is bit-reproducible. Two grid barriers per iteration:
//   phase A  q = A p fused with p = z + beta p (each gathered p_j is recomputed from z_j and the previous p_j
//            with the same FMA the row owner uses to store it, double-buffered), partial p.q  -> barrier, pAp
//   phase B  x += alpha p, r -= alpha q, z = D^-1 r, partials r.r, r.z                      -> barrier, rr, rz
// Stopping tests are the reference's: pAp <= 0 exits (negative-curvature flag if < 0), ||r||/||b|| <= tol.
// SpMV: one half-warp per row, lanes stride over the row's nonzeros, shuffle reduction within the half-warp.
#include <cooperative_groups.h>

#include <stdexcept>
#include <string>

#include "dev_types.cuh"

namespace cg = cooperative_groups;

namespace gfb {
namespace {

constexpr int kThreads = 1024;  // one CTA per SM: fewer grid-barrier arrivals
constexpr int kMaxRed = 3;

// block-reduce NV values, publish per-block partials, grid barrier, then every warp sums all block partials in
// the same order. Two alternating partial buffers make the re-use race-free.
template <int NV, class Grid>
__device__ __forceinline__ void grid_reduce(double (&v)[NV], double* partials, int& parity, Grid& grid) {
  __shared__ double s_red[kThreads / 32][kMaxRed];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    double x = v[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) s_red[w][q] = x;
  }
  __syncthreads();
  double* slot = partials + (size_t)parity * kMaxRed * gridDim.x;
  if (threadIdx.x < NV) {
    double x = 0.0;
    for (int k = 0; k < kThreads / 32; ++k) x += s_red[k][threadIdx.x];
    slot[(size_t)threadIdx.x * gridDim.x + blockIdx.x] = x;
  }
  grid.sync();
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    double x = 0.0;
    for (int b = lane; b < (int)gridDim.x; b += 32) x += __ldcg(slot + (size_t)q * gridDim.x + b);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    v[q] = x;
  }
  parity ^= 1;
}

struct Gather {  // p_j = fused ? fma(beta, p_old_j, z_j) : src_j
  const double* src;
  const double* z;
  double beta;
  bool fused;
  __device__ __forceinline__ double operator()(size_t k) const {
    return fused ? __fma_rn(beta, __ldcg(src + k), __ldcg(z + k)) : __ldcg(src + k);
  }
};

// y = A * P over the rows owned by this half-warp; returns the owner's partial P_row * y_row. If `write_p`, the
// row owner stores P_row to `pout` (the fused p update).
__device__ __forceinline__ double spmv_csr(const CgLaunch& a, const Gather& P, double* y, double* pout,
                                           bool write_p) {
  const int sub = threadIdx.x & 15;
  const int half = (threadIdx.x >> 4) & 1;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarp = (gridDim.x * blockDim.x) >> 5;
  double dotp = 0.0;
  // warp-uniform loop over row pairs so the half-warp shuffles always run with all 32 lanes present
  for (int base = 2 * warp; base < a.nrows; base += 2 * nwarp) {
    const int row = base + half;
    const bool active = row < a.nrows;
    int k0 = 0, k1 = 0;
    if (active) {
      k0 = __ldg(a.row_ptr + row);
      k1 = __ldg(a.row_ptr + row + 1);
    }
    double acc = 0.0;
    for (int k = k0 + sub; k < k1; k += 16) acc = __fma_rn(__ldg(a.vals + k), P((size_t)__ldg(a.cols + k)), acc);
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (active && sub == 0) {
      const double pr = P((size_t)row);
      y[row] = acc;
      if (write_p) pout[row] = pr;
      dotp = __fma_rn(pr, acc, dotp);
    }
  }
  return dotp;
}

__global__ void __launch_bounds__(kThreads) k_pcg_csr(CgLaunch a) {
  cg::grid_group grid = cg::this_grid();
  const size_t n = (size_t)a.nrows;
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t nthr = (size_t)gridDim.x * blockDim.x;
  int parity = 0;
  double* dinv = const_cast<double*>(a.dinv);

  for (size_t i = tid; i < n; i += nthr) {  // Jacobi inverse from the diagonal (sparse.cpp:133-136)
    double dg = 0.0;
    for (int k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k)
      if (a.cols[k] == (int)i) dg = a.vals[k];
    dinv[i] = (fabs(dg) > 1e-300) ? 1.0 / dg : 1.0;
  }
  grid.sync();
  // setup: Ap = A x ; r = b - Ap ; z = D^-1 r ; p = z ; partials b.b, r.z, r.r
  spmv_csr(a, Gather{a.x, nullptr, 0.0, false}, a.Ap, nullptr, false);
  grid.sync();
  double red3[3] = {0.0, 0.0, 0.0};
  for (size_t i = tid; i < n; i += nthr) {
    const double bi = a.b[i];
    const double ri = bi - __ldcg(a.Ap + i);
    const double zi = __ldcg(dinv + i) * ri;
    a.r[i] = ri;
    a.z[i] = zi;
    a.p0[i] = zi;
    red3[0] = __fma_rn(bi, bi, red3[0]);
    red3[1] = __fma_rn(ri, zi, red3[1]);
    red3[2] = __fma_rn(ri, ri, red3[2]);
  }
  grid_reduce<3>(red3, a.partials, parity, grid);
  const double bnorm = sqrt(red3[0]);
  double rz = red3[1], rr = red3[2];
  int iterations = 0, converged = 0, negcurv = 0;
  double relres = 0.0;
  if (bnorm == 0.0) {  // sparse.cpp:145-150
    for (size_t i = tid; i < n; i += nthr) a.x[i] = 0.0;
    converged = 1;
  } else {
    double* pcur = a.p0;
    double* pnext = a.p1;
    double beta = 0.0;
    bool done = false;
    for (int it = 0; it < a.max_iters; ++it) {
      const bool fused = it > 0;
      double pap[1] = {spmv_csr(a, Gather{pcur, a.z, beta, fused}, a.Ap, pnext, fused)};
      if (fused) {
        double* t = pcur;
        pcur = pnext;
        pnext = t;
      }
      grid_reduce<1>(pap, a.partials, parity, grid);
      if (pap[0] <= 0.0) {  // sparse.cpp:160-168
        negcurv = pap[0] < 0.0;
        iterations = it;
        relres = sqrt(rr) / bnorm;
        converged = relres <= a.tol;
        done = true;
        break;
      }
      const double alpha = rz / pap[0];
      double red2[2] = {0.0, 0.0};
      for (size_t i = tid; i < n; i += nthr) {
        const double pi = __ldcg(pcur + i);
        a.x[i] = __fma_rn(alpha, pi, __ldcg(a.x + i));
        const double ri = __fma_rn(-alpha, __ldcg(a.Ap + i), __ldcg(a.r + i));
        a.r[i] = ri;
        const double zi = __ldcg(dinv + i) * ri;
        a.z[i] = zi;
        red2[0] = __fma_rn(ri, ri, red2[0]);
        red2[1] = __fma_rn(ri, zi, red2[1]);
      }
      grid_reduce<2>(red2, a.partials, parity, grid);
      rr = red2[0];
      iterations = it + 1;
      const double rnorm = sqrt(rr);
      if (rnorm / bnorm <= a.tol) {  // sparse.cpp:172-178
        relres = rnorm / bnorm;
        converged = 1;
        done = true;
        break;
      }
      beta = red2[1] / rz;
      rz = red2[1];
    }
    if (!done) {
      relres = sqrt(rr) / bnorm;
      converged = relres <= a.tol;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.out[0] = iterations;
    a.out[1] = converged;
    a.out[2] = negcurv;
    a.out[3] = relres;
  }
}

int g_grid = 0;

}  // namespace

int cg_csr_grid() {
  if (g_grid == 0) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_pcg_csr, kThreads, 0);
    g_grid = sms * (per > 0 ? per : 1);
  }
  return g_grid;
}

void launch_pcg_csr(const CgLaunch& a, cudaStream_t s) {
  CgLaunch arg = a;
  void* args[] = {&arg};
  const cudaError_t err = cudaLaunchCooperativeKernel((const void*)k_pcg_csr, cg_csr_grid(), kThreads, args, 0, s);
  if (err != cudaSuccess) {
    cudaGetLastError();
    throw std::runtime_error(std::string("cooperative CG launch failed: ") + cudaGetErrorString(err));
  }
}

}  // namespace gfb
