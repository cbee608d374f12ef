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
__device__ __forceinline__ void sum_slices(const double* part, int ns, double (&out)[NV], size_t qstride) {
  __shared__ double s_w[kWarpsPerCta][4];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  constexpr int kB = 8;  // loads issued back to back per batch (one L2 round trip per batch, not per element)
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    double x = 0.0;
    for (int k0 = 0; k0 < ns; k0 += kB * (int)blockDim.x) {
      double v[kB];
#pragma unroll
      for (int b = 0; b < kB; ++b) {
        const int k = k0 + b * (int)blockDim.x + (int)threadIdx.x;
        v[b] = (k < ns) ? __ldcg(part + (size_t)q * qstride + k) : 0.0;
      }
#pragma unroll
      for (int b = 0; b < kB; ++b) x += v[b];
    }
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

struct Sched {  // dynamic work hand-out; each warp overshoots exactly once per phase
  unsigned long long* ctr;
  unsigned long long base;
  unsigned long long nwarps;
  __device__ __forceinline__ int next(int n) const {
    unsigned long long t = 0;
    if ((threadIdx.x & 31) == 0) t = atomicAdd(ctr, 1ull);
    t = __shfl_sync(0xffffffffu, t, 0);
    const unsigned long long idx = t - base;
    return idx < (unsigned long long)n ? (int)idx : -1;
  }
  __device__ __forceinline__ void advance(int n) { base += (unsigned long long)n + nwarps; }
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
#ifndef GF_QREC
#define GF_QREC 1
#endif
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
      a.trace[(k) * 8 + (point)] = gtimer();                                         \
  } while (0)
#define SELL_BLOCK_STAMP(k, slot) SELL_BLOCK_STAMP_AT(k, 10, slot)
#define SELL_BLOCK_STAMP_AT(k, at, slot)                                              \
  do {                                                                                \
    if (a.trace && (k) == (at)) {                                                     \
      __syncthreads();                                                                \
      if (threadIdx.x == 0) a.trace[(slot) + blockIdx.x] = gtimer();                 \
    }                                                                                 \
  } while (0)

// Symmetric format: the packed slot (j << 6 | c) of row i contributes A_ij p_j when j >= i (c = ordinal of the
// upper block (i, j) in row i) or A_ji^T p_j when j < i (block (j, i), ordinal c in row j's upper list); c = 63
// marks a padding slot (the all-zero block at zero_base). Entry q of a block at vals[base + 32 q] with
// base = (usp[owner / 32] + c) * 288 + owner % 32. 4 bytes per slot; half the matrix bytes of the full format:
// the upper blocks (~62 MB at c3), the slot list (~7 MB) and the CG vectors stay resident in the 126 MB L2.
#ifndef GF_MAT_L1
#define GF_MAT_L1 1  // block values through L1 (the transposed reads of neighbouring slices often hit)
#endif
__device__ __forceinline__ double ldmat(const double* p) {
#if GF_MAT_L1
  return __ldg(p);
#else
  return __ldcg(p);
#endif
}

template <class G>
__device__ __forceinline__ void slice_spmv_sym_g(const CgLaunch& a, int sl, const G& gat, double acc[3]) {
  const int lane = threadIdx.x & 31;
  const int row = sl * 32 + lane;
  const int k0 = __ldg(a.row_ptr + sl), k1 = __ldg(a.row_ptr + sl + 1);
  const uint32_t* slots = reinterpret_cast<const uint32_t*>(a.cols);
  const int own_base = __ldg(a.usp + sl) * 288 + lane;
  const int zero_base = a.zero_base + lane;
  acc[0] = acc[1] = acc[2] = 0.0;
  uint32_t sc[kGroup];
#pragma unroll
  for (int g = 0; g < kGroup; ++g) sc[g] = (k0 + g < k1) ? __ldg(slots + (size_t)(k0 + g) * 32 + lane) : 63u;
  for (int kb = k0; kb < k1; kb += kGroup) {
    uint32_t sn[kGroup];
#pragma unroll
    for (int g = 0; g < kGroup; ++g)
      sn[g] = (kb + kGroup + g < k1) ? __ldg(slots + (size_t)(kb + kGroup + g) * 32 + lane) : 63u;
#pragma unroll
    for (int g = 0; g < kGroup; ++g) {
      if (kb + g < k1) {
        const int j = (int)(sc[g] >> 6), c = (int)(sc[g] & 63u);
        const bool tr = j < row;
        const int base = c == 63 ? zero_base : tr ? (__ldg(a.usp + (j >> 5)) + c) * 288 + (j & 31) : own_base + 288 * c;
        const double3 p = gat((size_t)j);
        const double* v = a.vals + base;
        double m[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) m[q] = ldmat(v + 32 * q);
        if (!tr) {
          acc[0] = __fma_rn(m[0], p.x, acc[0]); acc[0] = __fma_rn(m[1], p.y, acc[0]); acc[0] = __fma_rn(m[2], p.z, acc[0]);
          acc[1] = __fma_rn(m[3], p.x, acc[1]); acc[1] = __fma_rn(m[4], p.y, acc[1]); acc[1] = __fma_rn(m[5], p.z, acc[1]);
          acc[2] = __fma_rn(m[6], p.x, acc[2]); acc[2] = __fma_rn(m[7], p.y, acc[2]); acc[2] = __fma_rn(m[8], p.z, acc[2]);
        } else {
          acc[0] = __fma_rn(m[0], p.x, acc[0]); acc[0] = __fma_rn(m[3], p.y, acc[0]); acc[0] = __fma_rn(m[6], p.z, acc[0]);
          acc[1] = __fma_rn(m[1], p.x, acc[1]); acc[1] = __fma_rn(m[4], p.y, acc[1]); acc[1] = __fma_rn(m[7], p.z, acc[1]);
          acc[2] = __fma_rn(m[2], p.x, acc[2]); acc[2] = __fma_rn(m[5], p.y, acc[2]); acc[2] = __fma_rn(m[8], p.z, acc[2]);
        }
      }
    }
#pragma unroll
    for (int g = 0; g < kGroup; ++g) sc[g] = sn[g];
  }
}

struct GatherX {
  const double* x;
  __device__ __forceinline__ double3 operator()(size_t j) const {
    return make_double3(ldv(x + 3 * j), ldv(x + 3 * j + 1), ldv(x + 3 * j + 2));
  }
};

struct GatherP {  // p_j = fused ? fma(beta, pold_j, z_j) : src_j
  const double* src;
  const double* z;
  double beta;
  bool fused;
  __device__ __forceinline__ double3 operator()(size_t j) const {
    if (fused)
      return make_double3(__fma_rn(beta, ldv(src + 3 * j), ldv(z + 3 * j)),
                          __fma_rn(beta, ldv(src + 3 * j + 1), ldv(z + 3 * j + 1)),
                          __fma_rn(beta, ldv(src + 3 * j + 2), ldv(z + 3 * j + 2)));
    return make_double3(ldv(src + 3 * j), ldv(src + 3 * j + 1), ldv(src + 3 * j + 2));
  }
};

// Symmetric format: slot (base | T<<31, j) of row i contributes A p_j (T = 0, upper block (i,j)) or A^T p_j
// (T = 1, block (j,i) stored by row j); entry q at vals[base + 32 q]. Half the matrix bytes of the full format;
// the upper blocks (~62 MB at c3) and the CG vectors can stay resident in the 126 MB L2 across iterations.
__device__ __forceinline__ void slice_spmv_sym(const CgLaunch& a, int sl, const double* src, const double* z,
                                               double beta, bool fused, double acc[3]) {
  slice_spmv_sym_g(a, sl, GatherP{src, z, beta, fused}, acc);
}

template <bool kStream, int kFmt>
__device__ __forceinline__ void spmv_fmt(const CgLaunch& a, int sl, const double* src, const double* z, double beta,
                                         bool fused, double acc[3]) {
  if constexpr (kFmt == 1) slice_spmv_sym(a, sl, src, z, beta, fused, acc);
  else slice_spmv<kStream>(a, sl, src, z, beta, fused, acc);
}

// Work distribution of one phase over n units, without per-unit atomics on the critical path: unit gw (the
// global warp id) is taken statically; the remaining n - nwarps units are handed out from the ticket counter,
// each warp requesting its next ticket BEFORE working on the current unit so the atomic's round trip hides
// behind the work (every warp takes exactly one overshooting ticket per phase). Statically taken units are
// reduced per CTA in warp order (one partial per CTA); dynamic units keep one partial each. After the grid
// barrier every CTA sums [CTA partials, dynamic-unit partials] in one fixed order, so alpha / beta / the stop
// tests are bit-identical in every CTA and run to run.
struct Phase {
  unsigned long long* ctr;
  unsigned long long base;
  int nwarps, gw;
  template <int NV, class Body>
  __device__ __forceinline__ void run(int n, double* const (&part)[NV], double* const (&cta)[NV], Body&& body) {
    __shared__ double s_acc[kWarpsPerCta][4];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned long long nd = n > nwarps ? (unsigned long long)(n - nwarps) : 0ull;
    unsigned long long tk = 0;
    if (nd && lane == 0) tk = atomicAdd(ctr, 1ull);
    double sv[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) sv[q] = 0.0;
    if (gw < n) body(gw, sv);
    if (nd) {
      for (;;) {
        const unsigned long long idx = __shfl_sync(0xffffffffu, tk, 0) - base;
        if (idx >= nd) break;
        if (lane == 0) tk = atomicAdd(ctr, 1ull);
        const int u = nwarps + (int)idx;
        double v[NV];
        body(u, v);
        if (lane == 0)
#pragma unroll
          for (int q = 0; q < NV; ++q) part[q][u] = v[q];
      }
      base += nd + (unsigned long long)nwarps;
    }
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < NV; ++q) s_acc[w][q] = sv[q];
    __syncthreads();
    if (threadIdx.x < NV) {
      double x = 0.0;
      for (int k = 0; k < kWarpsPerCta; ++k) x += s_acc[k][threadIdx.x];
      cta[threadIdx.x][blockIdx.x] = x;
    }
  }
};

// sum over [cta[0..G), part[nwarps..n)] in one fixed order (thread stride, then a fixed block tree)
template <int NV>
__device__ __forceinline__ void sum_phase(double* const (&part)[NV], double* const (&cta)[NV], int G, int nwarps,
                                          int n, double (&out)[NV]) {
  __shared__ double s_w[kWarpsPerCta][4];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nd = n > nwarps ? n - nwarps : 0, total = G + nd;
  constexpr int kB = 4;
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    double x = 0.0;
    for (int k0 = 0; k0 < total; k0 += kB * (int)blockDim.x) {
      double v[kB];
#pragma unroll
      for (int b = 0; b < kB; ++b) {
        const int k = k0 + b * (int)blockDim.x + (int)threadIdx.x;
        v[b] = (k < G) ? __ldcg(cta[q] + k) : (k < total) ? __ldcg(part[q] + nwarps + (k - G)) : 0.0;
      }
#pragma unroll
      for (int b = 0; b < kB; ++b) x += v[b];
    }
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

__host__ __device__ inline size_t part_stride(int ns) { return 4 * (size_t)ns + 1024; }

template <bool kStream, int kFmt>
__global__ void __launch_bounds__(kThreads) k_pcg_sell(SellArgs sa) {
  cg::grid_group grid = cg::this_grid();
  const CgLaunch& a = sa.a;
  const int ns = a.nslices, nrows = a.nrows, lane = threadIdx.x & 31;
  const int nwarps = (int)((gridDim.x * blockDim.x) >> 5), G = (int)gridDim.x;
  Phase ph{sa.ctr, 0ull, nwarps, (int)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5))};
  int parity = 0;
  const size_t qs = part_stride(ns);
  auto pq_ptr = [&](int q) { return sa.slice_part + ((size_t)parity * 4 + q) * qs; };
  auto ptrs1 = [&](double* (&u)[1], double* (&c)[1]) { u[0] = pq_ptr(0); c[0] = u[0] + 4 * (size_t)ns; };
  auto ptrs2 = [&](double* (&u)[2], double* (&c)[2]) {
    for (int q = 0; q < 2; ++q) { u[q] = pq_ptr(q); c[q] = u[q] + 4 * (size_t)ns; }
  };
  auto ptrs3 = [&](double* (&u)[3], double* (&c)[3]) {
    for (int q = 0; q < 3; ++q) { u[q] = pq_ptr(q); c[q] = u[q] + 4 * (size_t)ns; }
  };

  // setup (sparse.cpp:145-157): r = b - A x, z = D^-1 r, p = z; partials b.b, r.z, r.r per unit
  double tot3[3];
  {
    double *u3[3], *c3[3];
    ptrs3(u3, c3);
    ph.run<3>(ns, u3, c3, [&](int sl, double (&v)[3]) {
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
      v[0] = lane_sum(bb);
      v[1] = lane_sum(rz);
      v[2] = lane_sum(rr);
    });
    grid.sync();
    sum_phase<3>(u3, c3, G, nwarps, ns, tot3);
    parity ^= 1;
  }
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
      const int nunits = ns;
      double *uA[1], *cA[1];
      ptrs1(uA, cA);
      ph.run<1>(nunits, uA, cA, [&](int sl, double (&v)[1]) {
        double acc[3];
        int row;
        if constexpr (kFmt == 1 && GF_QREC) {
          // A p_{k+1} = A z_{k+1} + beta A p_k: only z is gathered (half the gather traffic of the L2-bound
          // phase); q = A p and p are then updated in place by their row owner.
          slice_spmv_sym_g(a, sl, GatherP{a.z, nullptr, 0.0, false}, acc);
          row = sl * 32 + lane;
          double pq = 0.0;
          if (row >= 0 && row < nrows) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              const size_t dof = 3 * (size_t)row + c;
              const double zi = ldv(a.z + dof);
              const double pr = fused ? __fma_rn(beta, ldv(pcur + dof), zi) : zi;
              const double qr = fused ? __fma_rn(beta, ldv(a.Ap + dof), acc[c]) : acc[c];
              pcur[dof] = pr;
              a.Ap[dof] = qr;
              pq = __fma_rn(pr, qr, pq);
            }
          }
          v[0] = lane_sum(pq);
          return;
        } else if constexpr (kFmt == 1) {
          slice_spmv_sym_g(a, sl, GatherP{pcur, a.z, beta, fused}, acc);
          row = sl * 32 + lane;
        } else {
          spmv_fmt<kStream, kFmt>(a, sl, pcur, a.z, beta, fused, acc);
          row = sl * 32 + lane;
        }
        double pq = 0.0;
        if (row >= 0 && row < nrows) {
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const size_t dof = 3 * (size_t)row + c;
            const double pr = fused ? __fma_rn(beta, ldv(pcur + dof), ldv(a.z + dof)) : ldv(pcur + dof);
            a.Ap[dof] = acc[c];
            if (fused) pnext[dof] = pr;
            pq = __fma_rn(pr, acc[c], pq);
          }
        }
        v[0] = lane_sum(pq);
      });
      SELL_STAMP(it, 1);
      SELL_BLOCK_STAMP(it, 3000);
      SELL_BLOCK_STAMP_AT(it, 20, 4000);
      if (fused && !(kFmt == 1 && GF_QREC)) {
        double* t = pcur;
        pcur = pnext;
        pnext = t;
      }
      double pap[1];
      grid.sync();
      SELL_STAMP(it, 5);
      sum_phase<1>(uA, cA, G, nwarps, nunits, pap);
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
      double *uB[2], *cB[2];
      ptrs2(uB, cB);
      ph.run<2>(ns, uB, cB, [&](int sl, double (&v)[2]) {
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
        v[0] = lane_sum(r2);
        v[1] = lane_sum(rzp);
      });
      SELL_STAMP(it, 3);
      SELL_BLOCK_STAMP(it, 2000);
      double red2[2];
      grid.sync();
      SELL_STAMP(it, 6);
      sum_phase<2>(uB, cB, G, nwarps, ns, red2);
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


// ---------------------------------------------------------------- single-barrier PCG (default)
// Chronopoulos-Gear form of the same Jacobi-PCG: one fused pass and ONE grid barrier per iteration.
//   given alpha_k, beta_k (identical in every CTA) and r_k, w_k = A z_k, s_{k-1}, p_{k-1}:
//     s_k = w_k + beta_k s_{k-1} (= A p_k),  p_k = z_k + beta_k p_{k-1},  x += alpha_k p_k,
//     r_{k+1} = r_k - alpha_k s_k,  z_{k+1} = D^-1 r_{k+1},  w_{k+1} = A z_{k+1}
//   where every gathered z_{k+1,j} is recomputed from (r_k, w_k, s_{k-1}, D^-1)_j with the same FMA sequence the
//   row owner uses (bit-identical), all four vectors double-buffered; per slice: partials r.z, z.w, r.r.
//   After the barrier: rr -> the reference's ||r||/||b|| <= tol test (sparse.cpp:172-178);
//   beta = rz'/rz, eta = zw' - beta rz'/alpha = (p_{k+1}, A p_{k+1}) -> the pAp <= 0 exit (sparse.cpp:160-168);
//   alpha = rz'/eta. Mathematically identical iterates to cg_solve; rounding differs at the 1e-16 level.
struct Cg1Vec {
  const double* r;   // r_k
  const double* w;   // w_k
  const double* s;   // s_{k-1}
  const double* dinv;
  double alpha, beta;
  __device__ __forceinline__ double znew(size_t d) const {
    const double sk = __fma_rn(beta, ldv(s + d), ldv(w + d));
    const double r1 = __fma_rn(-alpha, sk, ldv(r + d));
    return __ldg(dinv + d) * r1;
  }
  __device__ __forceinline__ double3 operator()(size_t j) const {
    return make_double3(znew(3 * j), znew(3 * j + 1), znew(3 * j + 2));
  }
};
struct GatherZ0 {  // z_0 = D^-1 r_0
  const double* r;
  const double* dinv;
  __device__ __forceinline__ double3 operator()(size_t j) const {
    return make_double3(__ldg(dinv + 3 * j) * ldv(r + 3 * j), __ldg(dinv + 3 * j + 1) * ldv(r + 3 * j + 1),
                        __ldg(dinv + 3 * j + 2) * ldv(r + 3 * j + 2));
  }
};

struct Cg1Args {
  CgLaunch a;
  unsigned long long* ctr;
  double* slice_part;   // 2 parities x 4 values x nslices
  double* r2;           // second buffers (3N each): r, w, s, p are double-buffered
  double* w0;
  double* w1;
  double* s0;
  double* s1;
};

__global__ void __launch_bounds__(kThreads) k_pcg_cg1(Cg1Args ca) {
  cg::grid_group grid = cg::this_grid();
  const CgLaunch& a = ca.a;
  const int ns = a.nslices, nrows = a.nrows, lane = threadIdx.x & 31;
  const int nwarps = (int)((gridDim.x * blockDim.x) >> 5), G = (int)gridDim.x;
  Phase ph{ca.ctr, 0ull, nwarps, (int)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5))};
  int parity = 0;
  const size_t qs = part_stride(ns);
  auto ptrs = [&](double* (&u)[3], double* (&c)[3]) {
    for (int q = 0; q < 3; ++q) {
      u[q] = ca.slice_part + ((size_t)parity * 4 + q) * qs;
      c[q] = u[q] + 4 * (size_t)ns;
    }
  };
  double* rb[2] = {a.r, ca.r2};
  double* wb[2] = {ca.w0, ca.w1};
  double* sb[2] = {ca.s0, ca.s1};
  double* pb[2] = {a.p0, a.p1};

  // setup 1: r0 = b - A x0; zero s_{-1}, p_{-1}; partial b.b
  double t1[3];
  {
    double *u[3], *c[3];
    ptrs(u, c);
    ph.run<3>(ns, u, c, [&](int sl, double (&v)[3]) {
      double acc[3];
      slice_spmv_sym_g(a, sl, GatherX{a.x}, acc);
      const int row = sl * 32 + lane;
      double bb = 0.0;
      if (row < nrows) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const size_t d = 3 * (size_t)row + c;
          const double bi = a.b[d];
          rb[0][d] = bi - acc[c];
          sb[0][d] = 0.0;
          pb[0][d] = 0.0;
          bb = __fma_rn(bi, bi, bb);
        }
      }
      v[0] = lane_sum(bb);
      v[1] = 0.0;
      v[2] = 0.0;
    });
    grid.sync();
    sum_phase<3>(u, c, G, nwarps, ns, t1);
    parity ^= 1;
  }
  // setup 2: w0 = A z0; partials r0.z0, z0.w0, r0.r0
  double t3[3];
  {
    double *u[3], *c[3];
    ptrs(u, c);
    ph.run<3>(ns, u, c, [&](int sl, double (&v)[3]) {
      double acc[3];
      slice_spmv_sym_g(a, sl, GatherZ0{rb[0], a.dinv}, acc);
      const int row = sl * 32 + lane;
      double rz = 0.0, zw = 0.0, rr = 0.0;
      if (row < nrows) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const size_t d = 3 * (size_t)row + c;
          const double ri = ldv(rb[0] + d);
          const double zi = __ldg(a.dinv + d) * ri;
          wb[0][d] = acc[c];
          rz = __fma_rn(ri, zi, rz);
          zw = __fma_rn(zi, acc[c], zw);
          rr = __fma_rn(ri, ri, rr);
        }
      }
      v[0] = lane_sum(rz);
      v[1] = lane_sum(zw);
      v[2] = lane_sum(rr);
    });
    grid.sync();
    sum_phase<3>(u, c, G, nwarps, ns, t3);
    parity ^= 1;
  }
  const double bnorm = sqrt(t1[0]);
  double rz = t3[0], eta = t3[1], rr = t3[2];
  int iterations = 0, converged = 0, negcurv = 0;
  double relres = 0.0;
  int cur = 0;
  if (bnorm == 0.0) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < 3 * (size_t)nrows; i += (size_t)gridDim.x * blockDim.x)
      a.x[i] = 0.0;
    converged = 1;
  } else {
    double beta = 0.0;
    bool done = false;
    for (int it = 0; it < a.max_iters; ++it) {
      if (eta <= 0.0) {  // (p_it, A p_it) <= 0  (sparse.cpp:160-168)
        negcurv = eta < 0.0;
        iterations = it;
        relres = sqrt(rr) / bnorm;
        converged = relres <= a.tol;
        done = true;
        break;
      }
      const double alpha = rz / eta;
      SELL_STAMP(it, 0);
      const int nx = cur ^ 1;
      const Cg1Vec gv{rb[cur], wb[cur], sb[cur], a.dinv, alpha, beta};
      double *u[3], *c[3];
      ptrs(u, c);
      ph.run<3>(ns, u, c, [&](int sl, double (&v)[3]) {
        double acc[3];
        slice_spmv_sym_g(a, sl, gv, acc);
        const int row = sl * 32 + lane;
        double prz = 0.0, pzw = 0.0, prr = 0.0;
        if (row < nrows) {
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const size_t d = 3 * (size_t)row + c;
            const double rk = ldv(rb[cur] + d), wk = ldv(wb[cur] + d), sprev = ldv(sb[cur] + d);
            const double di = __ldg(a.dinv + d);
            const double sk = __fma_rn(beta, sprev, wk);                 // s_k = w_k + beta s_{k-1}
            const double pk = __fma_rn(beta, ldv(pb[cur] + d), di * rk);  // p_k = z_k + beta p_{k-1}
            a.x[d] = __fma_rn(alpha, pk, ldv(a.x + d));
            const double r1 = __fma_rn(-alpha, sk, rk);                  // identical to Cg1Vec::znew
            const double z1 = di * r1;
            sb[nx][d] = sk;
            pb[nx][d] = pk;
            rb[nx][d] = r1;
            wb[nx][d] = acc[c];
            prz = __fma_rn(r1, z1, prz);
            pzw = __fma_rn(z1, acc[c], pzw);
            prr = __fma_rn(r1, r1, prr);
          }
        }
        v[0] = lane_sum(prz);
        v[1] = lane_sum(pzw);
        v[2] = lane_sum(prr);
      });
      SELL_STAMP(it, 1);
      SELL_BLOCK_STAMP(it, 3000);
      SELL_BLOCK_STAMP_AT(it, 20, 4000);
      grid.sync();
      double t[3];
      sum_phase<3>(u, c, G, nwarps, ns, t);
      parity ^= 1;
      SELL_STAMP(it, 2);
      cur = nx;
      rr = t[2];
      iterations = it + 1;
      const double rnorm = sqrt(rr);
      if (rnorm / bnorm <= a.tol) {
        relres = rnorm / bnorm;
        converged = 1;
        done = true;
        break;
      }
      beta = t[0] / rz;
      eta = t[1] - beta * t[0] / alpha;
      rz = t[0];
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

void launch_pcg_cg1(const CgLaunch& a, unsigned long long* ctr, double* slice_part, double* extra, cudaStream_t s) {
  const size_t n = 3 * (size_t)a.nrows;
  Cg1Args ca{a, ctr, slice_part, extra, extra + n, extra + 2 * n, extra + 3 * n, extra + 4 * n};
  cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), s);
  void* args[] = {&ca};
  const cudaError_t err = cudaLaunchCooperativeKernel((const void*)k_pcg_cg1, pcg_sell_grid(), kThreads, args, 0, s);
  if (err != cudaSuccess) {
    cudaGetLastError();
    throw std::runtime_error(std::string("cooperative CG launch failed: ") + cudaGetErrorString(err));
  }
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
#ifdef GF_CARVEOUT
  static bool carve = [fn] {
    cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, GF_CARVEOUT);
    return true;
  }();
  (void)carve;
#endif
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
