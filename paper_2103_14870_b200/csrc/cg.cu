// cg.cu — Jacobi-preconditioned CG (cg_solve, sparse.cpp:129-188) as ONE persistent cooperative kernel.
//
// The whole solve runs on the device: no host round-trip per iteration. Every block reaches the same
// scalars (alpha, beta, convergence) because block partial sums are reduced by every block in one fixed
// order after a grid barrier — the run is bit-reproducible. Two grid barriers per iteration:
//   phase A  q = A p fused with p = z + beta p (each gathered p_j is recomputed from z_j and the previous
//            p_j with the same FMA the row owner uses to store it, double-buffered, so no barrier is needed
//            between the p update and the SpMV), partial p.q          -> barrier, pAp
//   phase B  x += alpha p, r -= alpha q, z = D^-1 r, partials r.r, r.z -> barrier, rr, rz
// Stopping tests are the reference's: pAp <= 0 exits (negative-curvature flag if < 0), ||r||/||b|| <= tol.
// SpMV: node-block CSR (3x3 blocks), one half-warp per block row, lanes stride over the row's blocks
// (consecutive lanes read consecutive 72 B blocks: coalesced), shuffle reduction within the half-warp.
// B = 1 instantiates the same solver on a scalar CSR (gf_cg_solve_csr).
#include <cooperative_groups.h>

#include <stdexcept>
#include <string>

#include "dev_types.cuh"

namespace cg = cooperative_groups;


namespace gfb {
namespace {

constexpr int kThreads = 1024;  // one CTA per SM: fewer grid-barrier arrivals (148 vs 592)
constexpr int kMaxRed = 3;

// Grid barrier for a co-resident (cooperatively launched) grid: one release-atomic arrival per CTA on a
// counter, the last arrival resets it and publishes a new generation; the others spin on an acquire load.
// Data written before the barrier by other CTAs is read afterwards with ld.global.cg (L2), never from L1.
struct GridBarrier {
  unsigned* count;
  unsigned* gen;
  __device__ __forceinline__ void sync() const {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned g, arrived;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(gen) : "memory");
      __threadfence();
      asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;" : "=r"(arrived) : "l"(count) : "memory");
      if (arrived == gridDim.x - 1) {
        asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(count), "r"(0u) : "memory");
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(gen), "r"(g + 1) : "memory");
      } else {
        unsigned cur;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(gen) : "memory");
        } while (cur == g);
      }
    }
    __syncthreads();
  }
};

// block-reduce NV values, publish per-block partials, grid barrier, then every block sums all partials in
// the same order. Two alternating partial buffers make the re-use race-free (see header).
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
  // every warp sums all block partials itself, in the same fixed order: identical bits everywhere and no
  // second intra-block barrier on the critical path
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

template <int B>
struct Gather {  // p_j = fused ? fma(beta, p_old_j, z_j) : src_j
  const double* src;
  const double* z;
  double beta;
  bool fused;
  __device__ __forceinline__ double operator()(size_t k) const {
    return fused ? __fma_rn(beta, __ldcg(src + k), __ldcg(z + k)) : __ldcg(src + k);
  }
};

// y = A * P over all block rows owned by this half-warp; returns the owner's partial P_row . y_row.
// If `write_p`, the row owner stores P_row to `pout` (the fused p update).
template <int B>
__device__ __forceinline__ double spmv_csr(const CgLaunch& a, const Gather<B>& P, double* y, double* pout,
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
    double acc[B];
#pragma unroll
    for (int c = 0; c < B; ++c) acc[c] = 0.0;
    for (int k = k0 + sub; k < k1; k += 16) {
      const int j = __ldg(a.cols + k);
      double pj[B];
#pragma unroll
      for (int c = 0; c < B; ++c) pj[c] = P((size_t)B * j + c);
      const double* blk = a.vals + (size_t)B * B * k;
#pragma unroll
      for (int r = 0; r < B; ++r)
#pragma unroll
        for (int c = 0; c < B; ++c) acc[r] = __fma_rn(__ldg(blk + B * r + c), pj[c], acc[r]);
    }
#pragma unroll
    for (int r = 0; r < B; ++r)
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], o);
    if (active && sub == 0) {
#pragma unroll
      for (int r = 0; r < B; ++r) {
        const size_t dof = (size_t)B * row + r;
        const double pr = P(dof);
        y[dof] = acc[r];
        if (write_p) pout[dof] = pr;
        dotp = __fma_rn(pr, acc[r], dotp);
      }
    }
  }
  return dotp;
}

// SELL-32 node-block SpMV: one warp per 32-row slice, one lane per block row; every slot load (column id,
// 9 block entries) is a coalesced 128/256 B warp access; the 3 gathered p_j values are 24 contiguous bytes.
__device__ __forceinline__ double spmv_sell3(const CgLaunch& a, const Gather<3>& P, double* y, double* pout,
                                             bool write_p) {
  const int lane = threadIdx.x & 31;
  // each CTA owns one contiguous, equal run of slices (balanced over SMs, neighbouring rows stay on one SM so
  // the gathered p_j hit the same L1); warps of the CTA stride through the run
  int s_begin, s_end, s_step;
  if (a.mapping == 2) {
    const int per = (a.nslices + gridDim.x - 1) / gridDim.x;
    s_begin = blockIdx.x * per + (threadIdx.x >> 5);
    s_end = min(a.nslices, (blockIdx.x + 1) * per);
    s_step = blockDim.x >> 5;
  } else if (a.mapping == 1) {
    s_begin = (threadIdx.x >> 5) * gridDim.x + blockIdx.x;
    s_end = a.nslices;
    s_step = (gridDim.x * blockDim.x) >> 5;
  } else {
    s_begin = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    s_end = a.nslices;
    s_step = (gridDim.x * blockDim.x) >> 5;
  }
  double dotp = 0.0;
  for (int sl = s_begin; sl < s_end; sl += s_step) {
    const int row = sl * 32 + lane;
    const int k0 = __ldg(a.row_ptr + sl), k1 = __ldg(a.row_ptr + sl + 1);
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
#pragma unroll 2
    for (int k = k0; k < k1; ++k) {
      const size_t j = (size_t)__ldg(a.cols + (size_t)k * 32 + lane);
      const double* v = a.vals + (size_t)k * 288 + lane;
      const double p0 = P(3 * j), p1 = P(3 * j + 1), p2 = P(3 * j + 2);
      acc0 = __fma_rn(__ldg(v + 0), p0, acc0);
      acc0 = __fma_rn(__ldg(v + 32), p1, acc0);
      acc0 = __fma_rn(__ldg(v + 64), p2, acc0);
      acc1 = __fma_rn(__ldg(v + 96), p0, acc1);
      acc1 = __fma_rn(__ldg(v + 128), p1, acc1);
      acc1 = __fma_rn(__ldg(v + 160), p2, acc1);
      acc2 = __fma_rn(__ldg(v + 192), p0, acc2);
      acc2 = __fma_rn(__ldg(v + 224), p1, acc2);
      acc2 = __fma_rn(__ldg(v + 256), p2, acc2);
    }
    if (row < a.nrows) {
      const double acc[3] = {acc0, acc1, acc2};
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const size_t dof = 3 * (size_t)row + r;
        const double pr = P(dof);
        y[dof] = acc[r];
        if (write_p) pout[dof] = pr;
        dotp = __fma_rn(pr, acc[r], dotp);
      }
    }
  }
  return dotp;
}

template <int B>
__device__ __forceinline__ double spmv_phase(const CgLaunch& a, const Gather<B>& P, double* y, double* pout,
                                             bool write_p) {
  if constexpr (B == 3) return spmv_sell3(a, P, y, pout, write_p);
  else return spmv_csr<B>(a, P, y, pout, write_p);
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// optional phase trace (GF_CG_TRACE): block b in {0, last} thread 0 stamps %globaltimer at 5 points/iteration
#define CG_STAMP(k, point)                                                                              \
  do {                                                                                                  \
    if (a.trace && threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1) && (k) < 200)   \
      a.trace[((blockIdx.x == 0 ? 0 : 1) * 200 + (k)) * 5 + (point)] = gtimer();                     \
  } while (0)

template <int B>
__global__ void __launch_bounds__(kThreads) k_pcg(CgLaunch a) {
  cg::grid_group grid = cg::this_grid();
  const size_t n = (size_t)B * a.nrows;
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t nthr = (size_t)gridDim.x * blockDim.x;
  int parity = 0;
  double* dinv = const_cast<double*>(a.dinv);

  if (B == 1) {  // Jacobi inverse from the diagonal (sparse.cpp:133-136)
    for (size_t i = tid; i < n; i += nthr) {
      double dg = 0.0;
      for (int k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k)
        if (a.cols[k] == (int)i) dg = a.vals[k];
      dinv[i] = (fabs(dg) > 1e-300) ? 1.0 / dg : 1.0;
    }
    grid.sync();
  }
  // setup: Ap = A x ; r = b - Ap ; z = D^-1 r ; p = z ; partials b.b, r.z, r.r
  {
    Gather<B> gx{a.x, nullptr, 0.0, false};
    spmv_phase<B>(a, gx, a.Ap, nullptr, false);
  }
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
      CG_STAMP(it, 0);
      Gather<B> gp{pcur, a.z, beta, fused};
      double pap[1] = {spmv_phase<B>(a, gp, a.Ap, pnext, fused)};
      CG_STAMP(it, 1);
      if (a.trace && it == 10) {
        __syncthreads();
        if (threadIdx.x == 0) a.trace[3000 + blockIdx.x] = gtimer();
        if (threadIdx.x == 0 && blockIdx.x == 0) a.trace[4000] = gtimer();
      }
      if (fused) {
        double* t = pcur;
        pcur = pnext;
        pnext = t;
      }
      grid_reduce<1>(pap, a.partials, parity, grid);
      CG_STAMP(it, 2);
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
      CG_STAMP(it, 3);
      if (a.trace && it == 10) {  // per-block end of phase A/B at iteration 10 (diagnostics)
        __syncthreads();
        if (threadIdx.x == 0) a.trace[2000 + blockIdx.x] = gtimer();
      }
      grid_reduce<2>(red2, a.partials, parity, grid);
      CG_STAMP(it, 4);
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

template <int B>
__global__ void __launch_bounds__(kThreads) k_spmv(CgLaunch a, const double* xin, double* y) {
  Gather<B> g{xin, nullptr, 0.0, false};
  spmv_phase<B>(a, g, y, nullptr, false);
}

int g_grid[2] = {0, 0};

template <int B>
int grid_for() {
  int& gsz = g_grid[B == 3 ? 1 : 0];
  if (gsz == 0) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_pcg<B>, kThreads, 0);
    gsz = sms * (per > 0 ? per : 1);
  }
  return gsz;
}

template <int B>
void launch_pcg(const CgLaunch& a, cudaStream_t s) {
  const int grid = grid_for<B>();
  CgLaunch arg = a;
  void* args[] = {&arg};
  const cudaError_t err = cudaLaunchCooperativeKernel((const void*)k_pcg<B>, grid, kThreads, args, 0, s);
  if (err != cudaSuccess) {
    cudaGetLastError();
    throw std::runtime_error(std::string("cooperative CG launch failed: ") + cudaGetErrorString(err));
  }
}

}  // namespace

int cg_grid_size(int block_size) { return block_size == 3 ? grid_for<3>() : grid_for<1>(); }
void launch_pcg3(const CgLaunch& a, cudaStream_t s) { launch_pcg<3>(a, s); }
void launch_pcg1(const CgLaunch& a, cudaStream_t s) { launch_pcg<1>(a, s); }
void launch_spmv3(const CgLaunch& a, const double* xin, double* y, cudaStream_t s) {
  k_spmv<3><<<grid_for<3>(), kThreads, 0, s>>>(a, xin, y);
}

}  // namespace gfb

// ---------------------------------------------------------------- diagnostics: grid-barrier microbenchmark
namespace gfb {
namespace {
__global__ void k_bar_cg(int iters, double* sink) {
  cg::grid_group grid = cg::this_grid();
  double acc = 0.0;
  for (int i = 0; i < iters; ++i) {
    acc += (double)threadIdx.x;
    grid.sync();
  }
  if (acc < 0) sink[0] = acc;
}
__global__ void k_bar_custom(int iters, double* sink, unsigned* bar) {
  const GridBarrier grid{bar, bar + 1};
  double acc = 0.0;
  for (int i = 0; i < iters; ++i) {
    acc += (double)threadIdx.x;
    grid.sync();
  }
  if (acc < 0) sink[0] = acc;
}
}  // namespace

double barrier_bench(int variant, int iters, int blocks, int threads) {
  double* sink = nullptr;
  unsigned* bar = nullptr;
  cudaMalloc(&sink, 64);
  cudaMalloc(&bar, 64);
  cudaMemset(bar, 0, 64);
  void* args_cg[] = {&iters, &sink};
  void* args_cu[] = {&iters, &sink, &bar};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&]() {
    return variant == 0 ? cudaLaunchCooperativeKernel((const void*)k_bar_cg, blocks, threads, args_cg, 0, 0)
                        : cudaLaunchCooperativeKernel((const void*)k_bar_custom, blocks, threads, args_cu, 0, 0);
  };
  run();
  cudaEventRecord(a);
  const cudaError_t e = run();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaFree(sink);
  cudaFree(bar);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return -1.0;
  }
  return 1e3 * ms / iters;
}
}  // namespace gfb
