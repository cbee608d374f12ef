// cg_sell.cu — the production Jacobi-PCG (cg_solve, sparse.cpp:129-188) on the SELL-32 node-block matrix:
// ONE cooperative persistent kernel per solve, no host round-trip per iteration.
//
// Load balance: both vector phases are bandwidth bound and B200 SMs do not stream at equal rates (measured:
// up to 2.4x spread of per-SM SpMV time under a static split), so 32-row slices are handed out dynamically
// from a global atomic counter. Determinism is kept by never reducing per thread: every slice produces its
// own partial dot products (fixed lane-tree order) in a per-slice array, and after the grid barrier every CTA
// sums all slice partials in one fixed order. alpha, beta and the stopping decisions are therefore bit-identical
// in every CTA and from run to run, whatever the dynamic schedule.
//
// Per iteration (two grid barriers, the minimum for the reference's PCG recurrences):
//   phase A  q = A p, with p = z + beta p fused into the gathers (recomputed with one FMA from z and the
//            double-buffered previous p), partial p.q per slice               -> barrier, pAp
//   phase B  x += alpha p, r -= alpha q, z = D^-1 r, partials r.r and r.z     -> barrier, rr, rz
#include <cooperative_groups.h>

#include <cstdlib>
#include <stdexcept>
#include <string>

#include "dev_types.cuh"

#ifndef GF_SELL_THREADS
#define GF_SELL_THREADS 768
#endif

namespace cg = cooperative_groups;

namespace gfb {
namespace {

constexpr int kThreads = GF_SELL_THREADS;
constexpr int kWarpsPerCta = kThreads / 32;

struct SellArgs {
  CgLaunch a;
  int stream_matrix;        // 1: matrix loads use ld.global.cs (evict-first) so the vectors stay in L2
  unsigned long long* ctr;  // dynamic slice counter (zeroed by the host before the launch)
  double* slice_part;       // 2 parities x 3 values x nslices
};

__device__ __forceinline__ double lane_sum(double v) {  // fixed butterfly: same bits in every lane
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// every CTA sums all per-slice partials in the same order (thread stride, then a fixed block tree)
template <int NV>
__device__ __forceinline__ void sum_slices(const double* part, int ns, double (&out)[NV]) {
  __shared__ double s_w[kWarpsPerCta][3];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    double x = 0.0;
    for (int k = threadIdx.x; k < ns; k += blockDim.x) x += __ldcg(part + (size_t)q * ns + k);
    x = lane_sum(x);
    if (lane == 0) s_w[w][q] = x;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    double x = (lane < kWarpsPerCta) ? s_w[lane][q] : 0.0;
    out[q] = lane_sum(x);  // every warp computes the same total
  }
  __syncthreads();
}

struct Sched {  // dynamic slice hand-out; each warp overshoots exactly once per phase
  unsigned long long* ctr;
  unsigned long long base;
  unsigned long long stride;  // nslices + total warps
  __device__ __forceinline__ int next(int ns) const {
    unsigned long long t = 0;
    if ((threadIdx.x & 31) == 0) t = atomicAdd(ctr, 1ull);
    t = __shfl_sync(0xffffffffu, t, 0);
    const unsigned long long idx = t - base;
    return idx < (unsigned long long)ns ? (int)idx : -1;
  }
  __device__ __forceinline__ void advance() { base += stride; }
};

// y = A p for one slice (lane = row); p_j gathered as fused ? fma(beta, pold_j, z_j) : src_j
template <bool kStream>
__device__ __forceinline__ double ldm(const double* p) {
  if constexpr (kStream) return __ldcs(p);
  else return __ldg(p);
}

#ifndef GF_SELL_GROUP
#define GF_SELL_GROUP 2
#endif
constexpr int kGroup = GF_SELL_GROUP;
#ifndef GF_GATHER_L1
#define GF_GATHER_L1 1
#endif
// Vectors written in the previous phase are read through L1 (ld.global.nc): safe because every phase boundary
// is a cooperative-groups grid barrier, whose gpu-scope fence invalidates L1 (CCTL.IVALL), and within a phase
// the gathered vectors are read-only (the fused p update writes the other buffer).
__device__ __forceinline__ double ldv(const double* p) {
#if GF_GATHER_L1
  return __ldg(p);
#else
  return __ldcg(p);
#endif
}

// Software-pipelined: the column ids of the next group of kGroup slots are fetched while the current group's
// p_j gathers and block values are in flight, so each group costs one memory round trip instead of two
// (col -> gather dependency).
template <bool kStream>
__device__ __forceinline__ void slice_spmv(const CgLaunch& a, int sl, const double* src, const double* z, double beta,
                                           bool fused, double acc[3]) {
  const int lane = threadIdx.x & 31;
  const int k0 = __ldg(a.row_ptr + sl), k1 = __ldg(a.row_ptr + sl + 1);
  acc[0] = acc[1] = acc[2] = 0.0;
  auto col = [&](int k) -> int {
    return kStream ? __ldcs(a.cols + (size_t)k * 32 + lane) : __ldg(a.cols + (size_t)k * 32 + lane);
  };
  int jc[kGroup];
#pragma unroll
  for (int g = 0; g < kGroup; ++g) jc[g] = (k0 + g < k1) ? col(k0 + g) : 0;
  for (int kb = k0; kb < k1; kb += kGroup) {
    int jn[kGroup];
#pragma unroll
    for (int g = 0; g < kGroup; ++g) jn[g] = (kb + kGroup + g < k1) ? col(kb + kGroup + g) : 0;
#pragma unroll
    for (int g = 0; g < kGroup; ++g) {
      if (kb + g < k1) {
        const size_t j = (size_t)jc[g];
        const double* v = a.vals + (size_t)(kb + g) * 288 + lane;
        double p0, p1, p2;
        if (fused) {
          p0 = __fma_rn(beta, ldv(src + 3 * j), ldv(z + 3 * j));
          p1 = __fma_rn(beta, ldv(src + 3 * j + 1), ldv(z + 3 * j + 1));
          p2 = __fma_rn(beta, ldv(src + 3 * j + 2), ldv(z + 3 * j + 2));
        } else {
          p0 = ldv(src + 3 * j);
          p1 = ldv(src + 3 * j + 1);
          p2 = ldv(src + 3 * j + 2);
        }
        acc[0] = __fma_rn(ldm<kStream>(v + 0), p0, acc[0]);
        acc[0] = __fma_rn(ldm<kStream>(v + 32), p1, acc[0]);
        acc[0] = __fma_rn(ldm<kStream>(v + 64), p2, acc[0]);
        acc[1] = __fma_rn(ldm<kStream>(v + 96), p0, acc[1]);
        acc[1] = __fma_rn(ldm<kStream>(v + 128), p1, acc[1]);
        acc[1] = __fma_rn(ldm<kStream>(v + 160), p2, acc[1]);
        acc[2] = __fma_rn(ldm<kStream>(v + 192), p0, acc[2]);
        acc[2] = __fma_rn(ldm<kStream>(v + 224), p1, acc[2]);
        acc[2] = __fma_rn(ldm<kStream>(v + 256), p2, acc[2]);
      }
    }
#pragma unroll
    for (int g = 0; g < kGroup; ++g) jc[g] = jn[g];
  }
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// diagnostics (GF_CG_TRACE): CTA 0 stamps 5 points per iteration; at iteration 10 every CTA stamps the end of
// its phase-A and phase-B work (after a CTA barrier)
#define SELL_STAMP(k, point)                                                          \
  do {                                                                                \
    if (a.trace && threadIdx.x == 0 && blockIdx.x == 0 && (k) < 200)                 \
      a.trace[(k) * 5 + (point)] = gtimer();                                         \
  } while (0)
#define SELL_BLOCK_STAMP(k, slot)                                                     \
  do {                                                                                \
    if (a.trace && (k) == 10) {                                                       \
      __syncthreads();                                                                \
      if (threadIdx.x == 0) a.trace[(slot) + blockIdx.x] = gtimer();                 \
    }                                                                                 \
  } while (0)

// Symmetric format: slot (base | T<<31, j) of row i contributes A p_j (T = 0, upper block (i,j)) or A^T p_j
// (T = 1, block (j,i) stored by row j); entry q at vals[base + 32 q]. Half the matrix bytes of the full format;
// the upper blocks (~62 MB at c3) and the CG vectors can stay resident in the 126 MB L2 across iterations.
__device__ __forceinline__ void slice_spmv_sym(const CgLaunch& a, int sl, const double* src, const double* z,
                                               double beta, bool fused, double acc[3]) {
  const int lane = threadIdx.x & 31;
  const int k0 = __ldg(a.row_ptr + sl), k1 = __ldg(a.row_ptr + sl + 1);
  const int2* slots = reinterpret_cast<const int2*>(a.cols);
  acc[0] = acc[1] = acc[2] = 0.0;
  int2 sc[kGroup];
#pragma unroll
  for (int g = 0; g < kGroup; ++g) sc[g] = (k0 + g < k1) ? __ldg(slots + (size_t)(k0 + g) * 32 + lane) : make_int2(0, 0);
  for (int kb = k0; kb < k1; kb += kGroup) {
    int2 sn[kGroup];
#pragma unroll
    for (int g = 0; g < kGroup; ++g)
      sn[g] = (kb + kGroup + g < k1) ? __ldg(slots + (size_t)(kb + kGroup + g) * 32 + lane) : make_int2(0, 0);
#pragma unroll
    for (int g = 0; g < kGroup; ++g) {
      if (kb + g < k1) {
        const size_t j = (size_t)sc[g].y;
        const bool tr = sc[g].x < 0;
        const size_t base = (size_t)(sc[g].x & 0x7fffffff);
        double p0, p1, p2;
        if (fused) {
          p0 = __fma_rn(beta, ldv(src + 3 * j), ldv(z + 3 * j));
          p1 = __fma_rn(beta, ldv(src + 3 * j + 1), ldv(z + 3 * j + 1));
          p2 = __fma_rn(beta, ldv(src + 3 * j + 2), ldv(z + 3 * j + 2));
        } else {
          p0 = ldv(src + 3 * j);
          p1 = ldv(src + 3 * j + 1);
          p2 = ldv(src + 3 * j + 2);
        }
        const double* v = a.vals + base;
        double m[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) m[q] = __ldcg(v + 32 * q);
        if (!tr) {
          acc[0] = __fma_rn(m[0], p0, acc[0]); acc[0] = __fma_rn(m[1], p1, acc[0]); acc[0] = __fma_rn(m[2], p2, acc[0]);
          acc[1] = __fma_rn(m[3], p0, acc[1]); acc[1] = __fma_rn(m[4], p1, acc[1]); acc[1] = __fma_rn(m[5], p2, acc[1]);
          acc[2] = __fma_rn(m[6], p0, acc[2]); acc[2] = __fma_rn(m[7], p1, acc[2]); acc[2] = __fma_rn(m[8], p2, acc[2]);
        } else {
          acc[0] = __fma_rn(m[0], p0, acc[0]); acc[0] = __fma_rn(m[3], p1, acc[0]); acc[0] = __fma_rn(m[6], p2, acc[0]);
          acc[1] = __fma_rn(m[1], p0, acc[1]); acc[1] = __fma_rn(m[4], p1, acc[1]); acc[1] = __fma_rn(m[7], p2, acc[1]);
          acc[2] = __fma_rn(m[2], p0, acc[2]); acc[2] = __fma_rn(m[5], p1, acc[2]); acc[2] = __fma_rn(m[8], p2, acc[2]);
        }
      }
    }
#pragma unroll
    for (int g = 0; g < kGroup; ++g) sc[g] = sn[g];
  }
}

template <bool kStream, int kFmt>
__device__ __forceinline__ void spmv_fmt(const CgLaunch& a, int sl, const double* src, const double* z, double beta,
                                         bool fused, double acc[3]) {
  if constexpr (kFmt == 1) slice_spmv_sym(a, sl, src, z, beta, fused, acc);
  else slice_spmv<kStream>(a, sl, src, z, beta, fused, acc);
}

template <bool kStream, int kFmt>
__global__ void __launch_bounds__(kThreads) k_pcg_sell(SellArgs sa) {
  cg::grid_group grid = cg::this_grid();
  const CgLaunch& a = sa.a;
  const int ns = a.nslices, nrows = a.nrows, lane = threadIdx.x & 31;
  Sched sch{sa.ctr, 0ull, (unsigned long long)ns + (unsigned long long)((gridDim.x * blockDim.x) >> 5)};
  int parity = 0;
  auto part = [&](int q) { return sa.slice_part + ((size_t)parity * 3 + q) * ns; };

  // setup (sparse.cpp:145-157): r = b - A x, z = D^-1 r, p = z; partials b.b, r.z, r.r per slice
  for (int sl = sch.next(ns); sl >= 0; sl = sch.next(ns)) {
    double acc[3];
    spmv_fmt<kStream, kFmt>(a, sl, a.x, nullptr, 0.0, false, acc);
    const int row = sl * 32 + lane;
    double bb = 0.0, rz = 0.0, rr = 0.0;
    if (row < nrows) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const size_t dof = 3 * (size_t)row + c;
        const double bi = a.b[dof];
        const double ri = bi - acc[c];
        const double zi = __ldg(a.dinv + dof) * ri;
        a.r[dof] = ri;
        a.z[dof] = zi;
        a.p0[dof] = zi;
        bb = __fma_rn(bi, bi, bb);
        rz = __fma_rn(ri, zi, rz);
        rr = __fma_rn(ri, ri, rr);
      }
    }
    bb = lane_sum(bb);
    rz = lane_sum(rz);
    rr = lane_sum(rr);
    if (lane == 0) {
      part(0)[sl] = bb;
      part(1)[sl] = rz;
      part(2)[sl] = rr;
    }
  }
  sch.advance();
  grid.sync();
  double tot3[3];
  sum_slices<3>(part(0), ns, tot3);
  parity ^= 1;
  const double bnorm = sqrt(tot3[0]);
  double rz = tot3[1], rr = tot3[2];
  int iterations = 0, converged = 0, negcurv = 0;
  double relres = 0.0;
  if (bnorm == 0.0) {  // sparse.cpp:145-150
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < 3 * (size_t)nrows; i += (size_t)gridDim.x * blockDim.x)
      a.x[i] = 0.0;
    converged = 1;
  } else {
    double* pcur = a.p0;
    double* pnext = a.p1;
    double beta = 0.0;
    bool done = false;
    for (int it = 0; it < a.max_iters; ++it) {
      const bool fused = it > 0;
      SELL_STAMP(it, 0);
      // ---- phase A: q = A p
      for (int sl = sch.next(ns); sl >= 0; sl = sch.next(ns)) {
        double acc[3];
        spmv_fmt<kStream, kFmt>(a, sl, pcur, a.z, beta, fused, acc);
        const int row = sl * 32 + lane;
        double pq = 0.0;
        if (row < nrows) {
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const size_t dof = 3 * (size_t)row + c;
            const double pr = fused ? __fma_rn(beta, ldv(pcur + dof), ldv(a.z + dof)) : ldv(pcur + dof);
            a.Ap[dof] = acc[c];
            if (fused) pnext[dof] = pr;
            pq = __fma_rn(pr, acc[c], pq);
          }
        }
        pq = lane_sum(pq);
        if (lane == 0) part(0)[sl] = pq;
      }
      sch.advance();
      SELL_STAMP(it, 1);
      SELL_BLOCK_STAMP(it, 3000);
      if (fused) {
        double* t = pcur;
        pcur = pnext;
        pnext = t;
      }
      grid.sync();
      double pap[1];
      sum_slices<1>(part(0), ns, pap);
      parity ^= 1;
      SELL_STAMP(it, 2);
      if (pap[0] <= 0.0) {  // sparse.cpp:160-168
        negcurv = pap[0] < 0.0;
        iterations = it;
        relres = sqrt(rr) / bnorm;
        converged = relres <= a.tol;
        done = true;
        break;
      }
      const double alpha = rz / pap[0];
      // ---- phase B: x += alpha p, r -= alpha q, z = D^-1 r
      for (int sl = sch.next(ns); sl >= 0; sl = sch.next(ns)) {
        double r2 = 0.0, rzp = 0.0;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const int local = c * 32 + lane;  // 96 dofs of the slice, coalesced
          const size_t dof = (size_t)sl * 96 + local;
          if (dof < 3 * (size_t)nrows) {
            const double pi = __ldcg(pcur + dof);
            a.x[dof] = __fma_rn(alpha, pi, __ldcg(a.x + dof));
            const double ri = __fma_rn(-alpha, __ldcg(a.Ap + dof), __ldcg(a.r + dof));
            a.r[dof] = ri;
            const double zi = __ldg(a.dinv + dof) * ri;
            a.z[dof] = zi;
            r2 = __fma_rn(ri, ri, r2);
            rzp = __fma_rn(ri, zi, rzp);
          }
        }
        r2 = lane_sum(r2);
        rzp = lane_sum(rzp);
        if (lane == 0) {
          part(0)[sl] = r2;
          part(1)[sl] = rzp;
        }
      }
      sch.advance();
      SELL_STAMP(it, 3);
      SELL_BLOCK_STAMP(it, 2000);
      grid.sync();
      double red2[2];
      sum_slices<2>(part(0), ns, red2);
      parity ^= 1;
      SELL_STAMP(it, 4);
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

int pcg_sell_grid() {
  if (g_grid == 0) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_pcg_sell<true, 1>, kThreads, 0);
    g_grid = sms * (per > 0 ? per : 1);
  }
  return g_grid;
}

void launch_pcg_sell(const CgLaunch& a, unsigned long long* ctr, double* slice_part, cudaStream_t s, int mat_format) {
  static const int stream_matrix = [] {
    const char* e = std::getenv("GF_CG_STREAM");
    return e ? std::atoi(e) : 1;
  }();
  SellArgs sa{a, stream_matrix, ctr, slice_part};
  cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), s);
  void* args[] = {&sa};
  const void* fn = mat_format == 1 ? (const void*)k_pcg_sell<true, 1>
                   : stream_matrix ? (const void*)k_pcg_sell<true, 0> : (const void*)k_pcg_sell<false, 0>;
  const cudaError_t err = cudaLaunchCooperativeKernel(fn, pcg_sell_grid(), kThreads, args, 0, s);
  if (err != cudaSuccess) {
    cudaGetLastError();
    throw std::runtime_error(std::string("cooperative CG launch failed: ") + cudaGetErrorString(err));
  }
}

}  // namespace gfb

namespace gfb {
namespace {
template <int kFmt>
__global__ void __launch_bounds__(kThreads) k_spmv_fmt(CgLaunch a, const double* xin, double* y) {
  const int lane = threadIdx.x & 31;
  for (int sl = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; sl < a.nslices; sl += (gridDim.x * blockDim.x) >> 5) {
    double acc[3];
    spmv_fmt<true, kFmt>(a, sl, xin, nullptr, 0.0, false, acc);
    const int row = sl * 32 + lane;
    if (row < a.nrows)
      for (int c = 0; c < 3; ++c) y[3 * (size_t)row + c] = acc[c];
  }
}
}  // namespace
void launch_spmv_fmt(const CgLaunch& a, const double* xin, double* y, int mat_format, cudaStream_t s) {
  if (mat_format == 1) k_spmv_fmt<1><<<pcg_sell_grid(), kThreads, 0, s>>>(a, xin, y);
  else k_spmv_fmt<0><<<pcg_sell_grid(), kThreads, 0, s>>>(a, xin, y);
}
}  // namespace gfb
