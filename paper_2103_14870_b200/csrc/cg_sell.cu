// cg_sell.cu — the production Jacobi-PCG (cg_solve, sparse.cpp:129-188) on the symmetric node-block SELL-32
// matrix: ONE cooperative persistent kernel per solve, no host round-trip per iteration.
//
// Per iteration (two grid barriers, the minimum for the reference's PCG recurrences):
//   phase A  q = A p_k through q_k = A z_k + beta q_{k-1} (only z is gathered; p and q are updated in place by
//            their row owner), partial p.q                                   -> barrier, pAp
//   phase B  x += alpha p, r -= alpha q, z = D^-1 r, partials r.r and r.z   -> barrier, rr, rz
// Work distribution (class Phase): CTA b owns the slice range [cta_first[b], cta_first[b+1]) (balanced by slot
// count on the host), its warps stride through it; no atomics. A matrix larger than one slice per warp takes
// one slice per warp statically and hands out the rest dynamically (a ticket counter, requested one unit
// ahead), which absorbs SM speed differences. Determinism: static unit values are summed per warp in unit order and per CTA in warp order,
// dynamic units keep one partial each, and after the barrier every CTA sums [CTA partials, unit partials] in
// one fixed order, so alpha, beta and the stop decisions are bit-identical in every CTA and run to run.
#include <cooperative_groups.h>

#include <algorithm>
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
#ifndef GF_DYN_THREADS
#define GF_DYN_THREADS 768  // large-matrix instance block size (measured at c4: 768 23.0 ms, 512 26.9, 384 + 12-deep 23.6)
#endif
constexpr int kDynThreads = GF_DYN_THREADS;
constexpr int kDynWarps = kDynThreads / 32;

struct SellArgs {
  CgLaunch a;
  double* cta_part;         // 2 parities x 4 values x kMaxGrid CTA partials
  double* dyn_part;         // 2 parities x 4 values x max(1, #dynamic units) unit partials
  unsigned long long* ctr;  // dynamic ticket counter
};

__device__ __forceinline__ double lane_sum(double v) {  // fixed butterfly: same bits in every lane
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

#ifndef GF_CG_REGS
#define GF_CG_REGS 2  // 1: x, r, D^-1 of the owner rows in registers; 2: also p, q and z
#endif
#ifndef GF_CG_DEFER
#define GF_CG_DEFER 1
#endif
#ifndef GF_CG_SMEM
#define GF_CG_SMEM 1  // per-lane solver state in shared memory: frees registers for the SpMV loads in flight
#endif
#ifndef GF_SELL_GROUP
#define GF_SELL_GROUP 4
#endif
#ifndef GF_GATHER_L1
#define GF_GATHER_L1 1
#endif
// Vectors written earlier in the same kernel are gathered with coherent L1-cached loads (ld.global.ca, not the
// read-only .nc path: the data changes during the kernel). Safe because every phase boundary is a cooperative-groups
// grid barrier, whose gpu-scope fence invalidates L1 (CCTL.IVALL), and within a phase the gathered vector is
// read-only (the pipelined solver double-buffers it).
__device__ __forceinline__ double ldv(const double* p) {
#if GF_GATHER_L1
  return __ldca(p);
#else
  return __ldcg(p);
#endif
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

#ifndef GF_CG_TRACE_SM
#define GF_CG_TRACE_SM 0  // diagnostics build (tools/cg_trace_pipe.py imbalance section): per-CTA stamps + %smid
#endif

#ifndef GF_SELL_GROUP_DYN
#define GF_SELL_GROUP_DYN 8  // the large-matrix (HBM-streaming) instance: more block loads in flight (c4: -0.8 %)
#endif
// part / split: this warp takes the part-th of `split` contiguous chunks of the slice's slots (small matrices whose
// slices are shared by several warps, k_pcg_pipe<true>); the owner adds the chunks' sums in chunk order
template <class G, int kGroup = GF_SELL_GROUP>
__device__ __forceinline__ void slice_spmv_sym_g(const CgLaunch& a, int sl, const G& gat, double acc[3], int part = 0,
                                                 int split = 1) {
  const int lane = threadIdx.x & 31;
  const int row = sl * 32 + lane;
  int k0 = __ldg(a.row_ptr + sl), k1 = __ldg(a.row_ptr + sl + 1);
  if (split > 1) {
    const int per = (k1 - k0 + split - 1) / split;
    k0 += part * per;
    k1 = min(k1, k0 + per);
  }
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

struct GatherZ {
  const double* z;
  __device__ __forceinline__ double3 operator()(size_t j) const {
    return make_double3(ldv(z + 3 * j), ldv(z + 3 * j + 1), ldv(z + 3 * j + 2));
  }
};

// gathers of the pipelined solver's m (and u): L1-cached after the grid barrier's invalidation; inside a cluster
// (whose barrier orders memory at cluster scope only) through L2
template <bool kL2>
struct GatherM {
  const double* z;
  __device__ __forceinline__ double3 operator()(size_t j) const {
    if (kL2) return make_double3(__ldcg(z + 3 * j), __ldcg(z + 3 * j + 1), __ldcg(z + 3 * j + 2));
    return make_double3(ldv(z + 3 * j), ldv(z + 3 * j + 1), ldv(z + 3 * j + 2));
  }
};

struct Phase {
  const int32_t* cta_first;  // static units (slices) of CTA b: [cta_first[b], cta_first[b + 1])
  int n;                     // all units; [cta_first[G], n) are handed out dynamically (large matrices only)
  unsigned long long* ctr;   // ticket counter of the dynamic units (zeroed before the launch)
  unsigned long long base;
  // warp w of the CTA takes static units first + w, first + w + W, ... (consecutive warps on consecutive
  // slices), then dynamic units by ticket (requested one unit ahead). Static unit values are summed per warp in
  // unit order and per CTA in warp order (one partial per CTA); dynamic units keep one partial each.
  template <bool kDyn, int NV, int W = kWarpsPerCta, class Body>
  __device__ __forceinline__ void run(double* const (&cta)[NV], double* const (&dyn)[NV], Body&& body) {
    __shared__ double s_acc[W][4];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int nst = kDyn ? __ldg(cta_first + gridDim.x) : n;
    const unsigned long long nd = (unsigned long long)(n - nst);
    double sv[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) sv[q] = 0.0;
    unsigned long long tk = 0;
    if (kDyn && lane == 0) tk = atomicAdd(ctr, 1ull);
    const int u1 = __ldg(cta_first + blockIdx.x + 1);
    for (int u = __ldg(cta_first + blockIdx.x) + w; u < u1; u += W) {
      double v[NV];
      body(u, v);
#pragma unroll
      for (int q = 0; q < NV; ++q) sv[q] += v[q];
    }
    if (kDyn) {
      for (;;) {
        const unsigned long long idx = __shfl_sync(0xffffffffu, tk, 0) - base;
        if (idx >= nd) break;
        if (lane == 0) tk = atomicAdd(ctr, 1ull);
        double v[NV];
        body(nst + (int)idx, v);
        if (lane == 0)
#pragma unroll
          for (int q = 0; q < NV; ++q) dyn[q][idx] = v[q];
      }
      base += nd + ((gridDim.x * blockDim.x) >> 5);  // every warp took exactly one overshooting ticket
    }
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < NV; ++q) s_acc[w][q] = sv[q];
    __syncthreads();
    if (threadIdx.x < NV) {
      double x = 0.0;
      for (int k = 0; k < W; ++k) x += s_acc[k][threadIdx.x];
      cta[threadIdx.x][blockIdx.x] = x;
    }
  }
};

// fixed lane and warp trees over the CTA's per-thread values; every thread gets the same totals
template <int NV, int W = kWarpsPerCta>
__device__ __forceinline__ void cta_tree(const double (&x)[NV], double (&out)[NV]) {
  __shared__ double s_w[W][4];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    const double t = lane_sum(x[q]);
    if (lane == 0) s_w[w][q] = t;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    const double t = (lane < W) ? s_w[lane][q] : 0.0;
    out[q] = lane_sum(t);  // every warp computes the same total
  }
  __syncthreads();
}

// sum of [CTA partials, dynamic-unit partials] in one fixed order (thread stride, fixed lane and warp trees)
template <bool kDyn, int NV, int W = kWarpsPerCta>
__device__ __forceinline__ void sum_phase(double* const (&cta)[NV], double* const (&dyn)[NV], int G, int nd,
                                          double (&out)[NV]) {
  double x[NV];
  // all values' CTA partials are loaded back to back (one L2 round trip), then reduced
#pragma unroll
  for (int q = 0; q < NV; ++q) x[q] = 0.0;
  for (int k = threadIdx.x; k < G; k += blockDim.x)
#pragma unroll
    for (int q = 0; q < NV; ++q) x[q] += __ldcg(cta[q] + k);
  if (kDyn) {
    constexpr int kB = 8;  // loads issued back to back per batch (one L2 round trip per batch)
#pragma unroll
    for (int q = 0; q < NV; ++q)
      for (int k0 = 0; k0 < nd; k0 += kB * (int)blockDim.x) {
        double v[kB];
#pragma unroll
        for (int b = 0; b < kB; ++b) {
          const int k = k0 + b * (int)blockDim.x + (int)threadIdx.x;
          v[b] = k < nd ? __ldcg(dyn[q] + k) : 0.0;
        }
#pragma unroll
        for (int b = 0; b < kB; ++b) x[q] += v[b];
      }
  }
  cta_tree<NV, W>(x, out);
}

constexpr int kMaxGrid = 1024;  // CTA partial slots per value

template <bool kDyn>
__global__ void __launch_bounds__(kDyn ? kDynThreads : kThreads) k_pcg_sell(SellArgs sa) {
  constexpr int W = kDyn ? kDynWarps : kWarpsPerCta;
  cg::grid_group grid = cg::this_grid();
  const CgLaunch& a = sa.a;
  const int ns = a.nslices, nrows = a.nrows, lane = threadIdx.x & 31;
  const int G = (int)gridDim.x;
  Phase ph{a.cta_first, ns, sa.ctr, 0ull};
  const int nd = ns - __ldg(a.cta_first + G);
  const size_t dstride = nd > 0 ? (size_t)nd : 1;
  int parity = 0;
  auto ptrs = [&](auto& c, auto& dp) {  // CTA and dynamic-unit partial arrays of the current parity
    for (int q = 0; q < (int)(sizeof(c) / sizeof(c[0])); ++q) {
      c[q] = sa.cta_part + ((size_t)parity * 4 + q) * kMaxGrid;
      dp[q] = sa.dyn_part + ((size_t)parity * 4 + q) * dstride;
    }
  };

  // One slice per warp (kRegs): the owner keeps x, r and D^-1 of its rows in registers for the whole solve
  // (they are never gathered), so phase B reads only p and q and writes only z; x is stored once at the end.
  constexpr bool kRegs = !kDyn && GF_CG_REGS;
  constexpr bool kRegs2 = kRegs && GF_CG_REGS >= 2;  // p, q and the owner's z in registers too
  constexpr bool kDefer = kRegs2 && GF_CG_DEFER;      // phase B's reduction overlapped with the next SpMV
#if GF_CG_SMEM
  // per-lane solver state in shared memory ([warp][field][component][lane]: conflict-free), leaving the
  // registers to the SpMV's loads in flight
  extern __shared__ double s_state[];
  const int wq = threadIdx.x >> 5;
#define GF_SV(f, c) s_state[((wq * 6 + (f)) * 3 + (c)) * 32 + lane]
#else
  double xv_[3] = {0.0, 0.0, 0.0}, rv_[3] = {0.0, 0.0, 0.0}, dv_[3] = {0.0, 0.0, 0.0};
  double pv_[3] = {0.0, 0.0, 0.0}, qv_[3] = {0.0, 0.0, 0.0}, zv_[3] = {0.0, 0.0, 0.0};
  double* const svp[6] = {xv_, rv_, dv_, pv_, qv_, zv_};
#define GF_SV(f, c) svp[f][c]
#endif
  int own_row = -1;
  // setup (sparse.cpp:145-157): r = b - A x, z = D^-1 r, p = z, q = 0; partials b.b, r.z, r.r per unit
  double tot3[3];
  {
    double *c3[3], *d3[3];
    ptrs(c3, d3);
    ph.run<kDyn, 3, W>(c3, d3, [&](int sl, double (&v)[3]) {
      double acc[3];
      const int row = sl * 32 + lane;
      if (a.x0_identity) {  // A x0 = x0 (see CgLaunch::x0_identity): no SpMV
#pragma unroll
        for (int c = 0; c < 3; ++c) acc[c] = row < nrows ? a.x[3 * (size_t)row + c] : 0.0;
      } else {
        slice_spmv_sym_g(a, sl, GatherX{a.x}, acc);
      }
      double bb = 0.0, rz = 0.0, rr = 0.0;
      if (row < nrows) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const size_t dof = 3 * (size_t)row + c;
          const double bi = a.b[dof];
          const double ri = bi - acc[c];
          const double di = __ldg(a.dinv + dof);
          const double zi = di * ri;
          if (kRegs) {
            GF_SV(0, c) = a.x[dof];
            GF_SV(1, c) = ri;
            GF_SV(2, c) = di;
            own_row = row;
          } else {
            a.r[dof] = ri;
          }
          a.z[dof] = zi;
          if (kRegs2) {
            GF_SV(5, c) = zi;
            GF_SV(3, c) = zi;
          } else {
            a.p0[dof] = zi;
          }
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
    sum_phase<kDyn, 3, W>(c3, d3, G, nd, tot3);
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
    double* const p = a.p0;
    double beta = 0.0;
    bool done = false;
    if constexpr (kDefer) {
      // Same recurrences and decisions as the loop below, with phase B's reduction (r.r -> stop test, r.z ->
      // beta) deferred into the next phase A: its partials are loaded before that phase's SpMV (which gathers
      // only z and needs no scalar) and reduced after it, so the reduction's L2 round trip overlaps the SpMV.
      // One slice per warp (kRegs): the warp's SpMV result waits in registers for beta.
      const int u0 = __ldg(a.cta_first + blockIdx.x) + (int)(threadIdx.x >> 5);
      const bool has = u0 < __ldg(a.cta_first + blockIdx.x + 1);
      double* cBp[2] = {nullptr, nullptr};
      for (int it = 0;; ++it) {
        SELL_STAMP(it, 0);
        double pb[2] = {0.0, 0.0};
        if (it > 0 && (int)threadIdx.x < G) {
          pb[0] = __ldcg(cBp[0] + threadIdx.x);
          pb[1] = __ldcg(cBp[1] + threadIdx.x);
        }
        double acc[3] = {0.0, 0.0, 0.0};
        if (has && it < a.max_iters) slice_spmv_sym_g(a, u0, GatherZ{a.z}, acc);
        if (it > 0) {  // previous iteration's phase-B totals
          double red2[2];
          cta_tree<2, W>(pb, red2);
          rr = red2[0];
          iterations = it;
          const double rnorm = sqrt(rr);
          if (rnorm / bnorm <= a.tol) {  // sparse.cpp:172-178
            relres = rnorm / bnorm;
            converged = 1;
            done = true;
            break;
          }
          if (it < a.max_iters) {
            beta = red2[1] / rz;
            rz = red2[1];
          }
        }
        if (it >= a.max_iters) break;
        const bool fused = it > 0;
        double *cA[1], *dA[1];
        ptrs(cA, dA);
        ph.run<false, 1, W>(cA, dA, [&](int sl, double (&v)[1]) {
          const int row = sl * 32 + lane;
          double pq = 0.0;
          if (row < nrows) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              const double pr = fused ? __fma_rn(beta, GF_SV(3, c), GF_SV(5, c)) : GF_SV(5, c);
              const double qr = fused ? __fma_rn(beta, GF_SV(4, c), acc[c]) : acc[c];
              GF_SV(3, c) = pr;
              GF_SV(4, c) = qr;
              pq = __fma_rn(pr, qr, pq);
            }
          }
          v[0] = lane_sum(pq);
        });
        SELL_STAMP(it, 1);
        SELL_BLOCK_STAMP(it, 3000);
        SELL_BLOCK_STAMP_AT(it, 20, 4000);
        double pap[1];
        grid.sync();
        SELL_STAMP(it, 5);
        sum_phase<false, 1, W>(cA, dA, G, 0, pap);
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
        double *cB[2], *dB[2];
        ptrs(cB, dB);
        ph.run<false, 2, W>(cB, dB, [&](int sl, double (&v)[2]) {
          double r2 = 0.0, rzp = 0.0;
          const int row = sl * 32 + lane;
          if (row < nrows) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              const size_t dof = 3 * (size_t)row + c;
              GF_SV(0, c) = __fma_rn(alpha, GF_SV(3, c), GF_SV(0, c));
              GF_SV(1, c) = __fma_rn(-alpha, GF_SV(4, c), GF_SV(1, c));
              const double zi = GF_SV(2, c) * GF_SV(1, c);
              GF_SV(5, c) = zi;
              a.z[dof] = zi;
              r2 = __fma_rn(GF_SV(1, c), GF_SV(1, c), r2);
              rzp = __fma_rn(GF_SV(1, c), zi, rzp);
            }
          }
          v[0] = lane_sum(r2);
          v[1] = lane_sum(rzp);
        });
        SELL_STAMP(it, 3);
        SELL_BLOCK_STAMP(it, 2000);
        grid.sync();
        SELL_STAMP(it, 6);
        SELL_STAMP(it, 4);
        cBp[0] = cB[0];
        cBp[1] = cB[1];
        parity ^= 1;
      }
      if (!done) {
        relres = sqrt(rr) / bnorm;
        converged = relres <= a.tol;
      }
    } else
    for (int it = 0; it < a.max_iters; ++it) {
      const bool fused = it > 0;
      SELL_STAMP(it, 0);
      // ---- phase A: q = A p via A p_{k+1} = A z_{k+1} + beta A p_k: only z is gathered (half the gather
      // traffic of the L2-bound phase); q and p are then updated in place by their row owner
      double *cA[1], *dA[1];
      ptrs(cA, dA);
      ph.run<kDyn, 1, W>(cA, dA, [&](int sl, double (&v)[1]) {
        double acc[3];
        slice_spmv_sym_g<GatherZ, kDyn ? GF_SELL_GROUP_DYN : GF_SELL_GROUP>(a, sl, GatherZ{a.z}, acc);
        const int row = sl * 32 + lane;
        double pq = 0.0;
        if (row < nrows) {
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const size_t dof = 3 * (size_t)row + c;
            if (kRegs2) {
              const double pr = fused ? __fma_rn(beta, GF_SV(3, c), GF_SV(5, c)) : GF_SV(5, c);
              const double qr = fused ? __fma_rn(beta, GF_SV(4, c), acc[c]) : acc[c];
              GF_SV(3, c) = pr;
              GF_SV(4, c) = qr;
              pq = __fma_rn(pr, qr, pq);
            } else {
              // own rows through L1: z_i was just gathered by this warp's SpMV (the diagonal slot), an L1 hit
              // (measured: L2-only loads here cost c4 9 %)
              const double zi = ldv(a.z + dof);
              const double pr = fused ? __fma_rn(beta, ldv(p + dof), zi) : zi;
              const double qr = fused ? __fma_rn(beta, ldv(a.Ap + dof), acc[c]) : acc[c];
              p[dof] = pr;
              a.Ap[dof] = qr;
              pq = __fma_rn(pr, qr, pq);
            }
          }
        }
        v[0] = lane_sum(pq);
      });
      SELL_STAMP(it, 1);
      SELL_BLOCK_STAMP(it, 3000);
      SELL_BLOCK_STAMP_AT(it, 20, 4000);
      double pap[1];
      grid.sync();
      SELL_STAMP(it, 5);
      sum_phase<kDyn, 1, W>(cA, dA, G, nd, pap);
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
      double *cB[2], *dB[2];
      ptrs(cB, dB);
      ph.run<kDyn, 2, W>(cB, dB, [&](int sl, double (&v)[2]) {
        double r2 = 0.0, rzp = 0.0;
        if (kRegs) {
          const int row = sl * 32 + lane;
          if (row < nrows) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              const size_t dof = 3 * (size_t)row + c;
              GF_SV(0, c) = __fma_rn(alpha, kRegs2 ? GF_SV(3, c) : __ldcg(p + dof), GF_SV(0, c));
              GF_SV(1, c) = __fma_rn(-alpha, kRegs2 ? GF_SV(4, c) : __ldcg(a.Ap + dof), GF_SV(1, c));
              const double zi = GF_SV(2, c) * GF_SV(1, c);
              if (kRegs2) GF_SV(5, c) = zi;
              a.z[dof] = zi;
              r2 = __fma_rn(GF_SV(1, c), GF_SV(1, c), r2);
              rzp = __fma_rn(GF_SV(1, c), zi, rzp);
            }
          }
        } else {
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const size_t dof = (size_t)sl * 96 + c * 32 + lane;  // 96 dofs of the slice, coalesced
            if (dof < 3 * (size_t)nrows) {
              const double pi = __ldcg(p + dof);
              a.x[dof] = __fma_rn(alpha, pi, __ldcg(a.x + dof));
              const double ri = __fma_rn(-alpha, __ldcg(a.Ap + dof), __ldcg(a.r + dof));
              a.r[dof] = ri;
              const double zi = __ldg(a.dinv + dof) * ri;
              a.z[dof] = zi;
              r2 = __fma_rn(ri, ri, r2);
              rzp = __fma_rn(ri, zi, rzp);
            }
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
      sum_phase<kDyn, 2, W>(cB, dB, G, nd, red2);
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
    if (kRegs && own_row >= 0)
#pragma unroll
      for (int c = 0; c < 3; ++c) a.x[3 * (size_t)own_row + c] = GF_SV(0, c);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.out[0] = iterations;
    a.out[1] = converged;
    a.out[2] = negcurv;
    a.out[3] = relres;
  }
}

// Large-matrix instance (HBM-streaming, c4): k_pcg_sell<true>'s recurrences with
//  * round-robin static work: warp w of CTA b takes slices b W + w, b W + w + G W, ... -- the grid sweeps the matrix
//    in slice order (a block's transposed re-read, one z-plane of slices later, still finds it in L2) without the
//    ticket atomics, and every CTA publishes ONE partial per value: the reduction after each barrier reads G values
//    instead of one per dynamic unit (~25k at c4);
//  * x += alpha p deferred into the next phase A, which reads p_k anyway to form p_{k+1}: phase B then reads only q,
//    r and D^-1 and writes r and z (the same fma, applied one phase later: bit-identical x), and an exit after a
//    phase B applies the pending update in one final pass. Per node and iteration 288 instead of 312 vector bytes.
template <int NV, class Body>
__device__ __forceinline__ void rr_run(int ns, double* const (&cta)[NV], Body&& body) {
  __shared__ double s_acc[kDynWarps][4];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int stride = (int)gridDim.x * kDynWarps;
  double sv[NV];
#pragma unroll
  for (int q = 0; q < NV; ++q) sv[q] = 0.0;
  for (int u = (int)blockIdx.x * kDynWarps + w; u < ns; u += stride) {
    double v[NV];
    body(u, v);
#pragma unroll
    for (int q = 0; q < NV; ++q) sv[q] += v[q];
  }
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < NV; ++q) s_acc[w][q] = sv[q];
  __syncthreads();
  if (threadIdx.x < NV) {
    double x = 0.0;
    for (int k = 0; k < kDynWarps; ++k) x += s_acc[k][threadIdx.x];
    cta[threadIdx.x][blockIdx.x] = x;
  }
}

__global__ void __launch_bounds__(kDynThreads) k_pcg_big(SellArgs sa) {
  constexpr int W = kDynWarps;
  cg::grid_group grid = cg::this_grid();
  const CgLaunch& a = sa.a;
  const int ns = a.nslices, nrows = a.nrows, lane = threadIdx.x & 31;
  const int G = (int)gridDim.x;
  double* const p = a.p0;
  int parity = 0;
  auto ptrs = [&](auto& c) {
    for (int q = 0; q < (int)(sizeof(c) / sizeof(c[0])); ++q) c[q] = sa.cta_part + ((size_t)parity * 4 + q) * kMaxGrid;
  };
  // setup (sparse.cpp:145-157): r = b - A x, z = D^-1 r, p = z; partials b.b, r.z, r.r
  double tot3[3];
  {
    double* c3[3];
    ptrs(c3);
    rr_run<3>(ns, c3, [&](int sl, double (&v)[3]) {
      double acc[3];
      const int row = sl * 32 + lane;
      if (a.x0_identity) {  // A x0 = x0 (see CgLaunch::x0_identity): no SpMV
#pragma unroll
        for (int c = 0; c < 3; ++c) acc[c] = row < nrows ? a.x[3 * (size_t)row + c] : 0.0;
      } else {
        slice_spmv_sym_g<GatherX, GF_SELL_GROUP_DYN>(a, sl, GatherX{a.x}, acc);
      }
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
          p[dof] = zi;
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
    sum_phase<false, 3, W>(c3, c3, G, 0, tot3);
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
    double beta = 0.0, alpha_prev = 0.0;
    bool done = false, pending = false;  // pending: x lacks alpha_prev p (applied by the next phase A or at the end)
    for (int it = 0; it < a.max_iters; ++it) {
      const bool fused = it > 0;
      SELL_STAMP(it, 0);
      // ---- phase A: q = A p via A p_{k+1} = A z_{k+1} + beta A p_k (only z gathered); x += alpha_k p_k on the way
      double* cA[1];
      ptrs(cA);
      rr_run<1>(ns, cA, [&](int sl, double (&v)[1]) {
        double acc[3];
        slice_spmv_sym_g<GatherZ, GF_SELL_GROUP_DYN>(a, sl, GatherZ{a.z}, acc);
        const int row = sl * 32 + lane;
        double pq = 0.0;
        if (row < nrows) {
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const size_t dof = 3 * (size_t)row + c;
            const double zi = ldv(a.z + dof);  // gathered by this warp's diagonal slot: an L1 hit
            double pr = zi, qr = acc[c];
            if (fused) {
              const double po = ldv(p + dof);
              a.x[dof] = __fma_rn(alpha_prev, po, __ldcg(a.x + dof));
              pr = __fma_rn(beta, po, zi);
              qr = __fma_rn(beta, ldv(a.Ap + dof), acc[c]);
            }
            p[dof] = pr;
            a.Ap[dof] = qr;
            pq = __fma_rn(pr, qr, pq);
          }
        }
        v[0] = lane_sum(pq);
      });
      pending = false;
      SELL_STAMP(it, 1);
      SELL_BLOCK_STAMP(it, 3000);
      SELL_BLOCK_STAMP_AT(it, 20, 4000);
      double pap[1];
      grid.sync();
      SELL_STAMP(it, 5);
      sum_phase<false, 1, W>(cA, cA, G, 0, pap);
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
      // ---- phase B: r -= alpha q, z = D^-1 r (coalesced over the slice's 96 dofs)
      double* cB[2];
      ptrs(cB);
      rr_run<2>(ns, cB, [&](int sl, double (&v)[2]) {
        double r2 = 0.0, rzp = 0.0;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const size_t dof = (size_t)sl * 96 + c * 32 + lane;
          if (dof < 3 * (size_t)nrows) {
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
      alpha_prev = alpha;
      pending = true;
      SELL_STAMP(it, 3);
      SELL_BLOCK_STAMP(it, 2000);
      double red2[2];
      grid.sync();
      SELL_STAMP(it, 6);
      sum_phase<false, 2, W>(cB, cB, G, 0, red2);
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
    if (pending)  // the last phase B's step: p_k was written before the last two barriers
      for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < 3 * (size_t)nrows; i += (size_t)gridDim.x * blockDim.x)
        a.x[i] = __fma_rn(alpha_prev, __ldcg(p + i), __ldcg(a.x + i));
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.out[0] = iterations;
    a.out[1] = converged;
    a.out[2] = negcurv;
    a.out[3] = relres;
  }
}

// Pipelined PCG (Ghysels & Vanroose 2014, preconditioned pipelined CG) for matrices of at most one slice per warp:
// ONE grid barrier per iteration. The recurrences carry s = A p, q = D^-1 s and z = A q next to x, r, u = D^-1 r and
// w = A u, so the only SpMV of an iteration is n = A m with m = D^-1 w -- and m is known at the END of the previous
// iteration, before alpha and beta are. The iteration's reduction (gamma = r.u, delta = w.u, r.r) is published at
// the same barrier as m, loaded before the SpMV and reduced after it:
//   [barrier] load partials -> n = A m (gather m) -> gamma, delta, r.r -> stop tests -> beta, alpha
//             -> z = n + beta z, q = m + beta q, s = w + beta s, p = u + beta p
//             -> x += alpha p, r -= alpha s, u -= alpha q, w -= alpha z, m' = D^-1 w, partials -> [barrier]
// Equivalent to the reference's PCG (sparse.cpp:129-188) in exact arithmetic, with its decisions mapped one to one:
// p.Ap = delta - beta gamma / alpha_prev (<= 0: negative curvature exit, sparse.cpp:160-168), ||r||/||b|| <= tol
// tested on every updated r (sparse.cpp:172-178), bnorm = 0 -> x = 0 (sparse.cpp:145-150), max_iters updates.
// Solver state (x, r, D^-1, u, w, p, s, q, z) lives in shared memory for the whole solve; m is double-buffered in
// global memory (a slow warp may still gather m_i while a fast one writes m_{i+1}); deterministic fixed-order
// reductions as in k_pcg_sell.
// solver state per lane in shared memory: x, r, D^-1, w, p, s, z (u = D^-1 r and q = D^-1 s are evaluated where
// needed instead of carried: the same quantities, and 37 KB more L1 per SM than 9 carried fields -- DESIGN.md §7)
constexpr int kPipeFields = 7;
// kCluster: the whole solve inside ONE thread-block cluster (small matrices, <= 16 x 24 slices): the grid barrier
// becomes the hardware cluster barrier and the CTA partials are exchanged through distributed shared memory
template <bool kCluster>
__global__ void __launch_bounds__(kThreads) k_pcg_pipe(SellArgs sa) {
  __shared__ double s_part[2][4];  // kCluster: this CTA's published partials, read by the cluster through DSMEM
  auto gsync = [&] {
    if constexpr (kCluster) cg::this_cluster().sync();
    else cg::this_grid().sync();
  };
  // a published CTA partial (CTA k, parity, value q)
  auto read_part = [&](int parity, int q, int k) -> double {
    if constexpr (kCluster) return *cg::this_cluster().map_shared_rank(&s_part[parity][q], k);
    else return __ldcg(sa.cta_part + ((size_t)parity * 4 + q) * kMaxGrid + k);
  };
  const CgLaunch& a = sa.a;
  const int nrows = a.nrows, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int G = (int)gridDim.x;
  // kCluster: `split` warps share a slice (part 0 owns its state; the others SpMV a chunk of its slots)
  const int split = kCluster ? a.split : 1;
  const int ws = kCluster ? w / split : w, part = kCluster ? w - ws * split : 0;
  const int cta_s0 = __ldg(a.cta_first + blockIdx.x), cta_s1 = __ldg(a.cta_first + blockIdx.x + 1);
  const int u0 = cta_s0 + ws;
  const bool has = u0 < cta_s1;
  const int row = u0 * 32 + lane;
  const bool live = has && part == 0 && row < nrows;
  extern __shared__ double s_state[];
  double* const s_split = s_state + kWarpsPerCta * kPipeFields * 96;  // kCluster, split > 1: chunk sums
  // the chunk sums of a shared slice, added by the owner in chunk order (deterministic)
  auto combine = [&](double (&v)[3]) {
    if (split == 1) return;
    if (has && part > 0)
#pragma unroll
      for (int c = 0; c < 3; ++c) s_split[((ws * (split - 1) + part - 1) * 3 + c) * 32 + lane] = v[c];
    __syncthreads();
    if (has && part == 0)
      for (int q = 1; q < split; ++q)
#pragma unroll
        for (int c = 0; c < 3; ++c) v[c] += s_split[((ws * (split - 1) + q - 1) * 3 + c) * 32 + lane];
  };
  enum { R = 0, D = 1, W = 2, P = 3, S = 4, Z = 5, X = 6 };
#define PV(f, c) s_state[((ws * kPipeFields + (f)) * 3 + (c)) * 32 + lane]
  auto DV = [&](int c) -> double { return PV(D, c); };
  __shared__ double s_acc[kWarpsPerCta][4];
  // double-buffered gathered vector (u during setup, then m): buffer k is a.z (k = 0) or a.p0 (k = 1)
  auto gm = [&](int k) { return k ? a.p0 : a.z; };

  // CTA partials of NV warp values (one slice per warp): warp sums in lane order, CTA sum in warp order
  // the CTA's partial of NV warp values: warp 0 reduces the warps' values with one fixed butterfly (not a serial
  // 24-term loop), lane q < NV publishes value q
  auto publish = [&](const double* v, int nv, int parity) {
    if (lane == 0)
      for (int q = 0; q < nv; ++q) s_acc[w][q] = v[q];
    __syncthreads();
    if constexpr (kCluster) {  // latency-bound small solves: one warp butterfly instead of a serial 24-term loop
      if (w == 0) {
        double x[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) x[q] = (q < nv && lane < kWarpsPerCta) ? s_acc[lane][q] : 0.0;
#pragma unroll
        for (int q = 0; q < 3; ++q) x[q] = lane_sum(x[q]);
        const double xl = lane == 0 ? x[0] : lane == 1 ? x[1] : x[2];
        if (lane < nv) s_part[parity][lane] = xl;
      }
    } else {  // (the butterfly costs the grid instance a register spill: measured neutral-to-worse at c3)
      if ((int)threadIdx.x < nv) {
        double x = 0.0;
        for (int k = 0; k < kWarpsPerCta; ++k) x += s_acc[k][threadIdx.x];
        sa.cta_part[((size_t)parity * 4 + threadIdx.x) * kMaxGrid + blockIdx.x] = x;
      }
    }
  };
  // totals of the published partials of all G CTAs: fixed lane and warp trees with ONE block barrier (the next
  // writer of s_tot is separated from these reads by the publish barrier and the grid / cluster barrier)
  __shared__ double s_tot[kWarpsPerCta][4];
  auto totals3 = [&](const double (&pbv)[3], double (&out)[3]) {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const double t = lane_sum(pbv[q]);
      if (lane == 0) s_tot[w][q] = t;
    }
    __syncthreads();
    const int nw = (G + 31) >> 5;  // warps holding partials (threads < G)
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      double t = 0.0;
      for (int k = 0; k < nw; ++k) t += s_tot[k][q];
      out[q] = t;
    }
  };

  // setup 1 (sparse.cpp:145-157): r = b - A x0, u = D^-1 r (gathered next), partial b.b
  double acc[3] = {0.0, 0.0, 0.0};
  if (has) {
    if (a.x0_identity) {  // A x0 = x0 (see CgLaunch::x0_identity): no SpMV
#pragma unroll
      for (int c = 0; c < 3; ++c) acc[c] = row < nrows ? a.x[3 * (size_t)row + c] : 0.0;
    } else {
      if constexpr (kCluster) slice_spmv_sym_g(a, u0, GatherX{a.x}, acc, part, split);
      else slice_spmv_sym_g(a, u0, GatherX{a.x}, acc);
    }
  }
  if (!a.x0_identity) combine(acc);
  double bb = 0.0;
  if (live) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const size_t dof = 3 * (size_t)row + c;
      const double bi = a.b[dof], ri = bi - acc[c], di = __ldg(a.dinv + dof), ui = di * ri;
      PV(X, c) = a.x[dof];
      PV(R, c) = ri;
      PV(D, c) = di;
      PV(P, c) = PV(S, c) = PV(Z, c) = 0.0;
      gm(0)[dof] = ui;
      bb = __fma_rn(bi, bi, bb);
    }
  }
  bb = lane_sum(bb);
  publish(&bb, 1, 0);
  gsync();
  double tot[1];
  {
    double x[1] = {(int)threadIdx.x < G ? read_part(0, 0, threadIdx.x) : 0.0};
    cta_tree<1>(x, tot);
  }
  const double bnorm = sqrt(tot[0]);
  int iterations = 0, converged = 0, negcurv = 0;
  double relres = 0.0;
  if (bnorm == 0.0) {  // sparse.cpp:145-150
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < 3 * (size_t)nrows; i += (size_t)gridDim.x * blockDim.x)
      a.x[i] = 0.0;
    converged = 1;
  } else {
    // setup 2: w = A u, m = D^-1 w (gathered by iteration 0), partials gamma_0, delta_0, r.r
    acc[0] = acc[1] = acc[2] = 0.0;
    if (has) {
      if constexpr (kCluster) slice_spmv_sym_g(a, u0, GatherM<kCluster>{gm(0)}, acc, part, split);
      else slice_spmv_sym_g(a, u0, GatherM<kCluster>{gm(0)}, acc);
    }
    combine(acc);
    double v3[3] = {0.0, 0.0, 0.0};
    if (live) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const size_t dof = 3 * (size_t)row + c;
        PV(W, c) = acc[c];
        gm(1)[dof] = DV(c) * acc[c];
        const double uc = DV(c) * PV(R, c);  // u_0 = D^-1 r_0
        v3[0] = __fma_rn(PV(R, c), uc, v3[0]);
        v3[1] = __fma_rn(acc[c], uc, v3[1]);
        v3[2] = __fma_rn(PV(R, c), PV(R, c), v3[2]);
      }
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) v3[q] = lane_sum(v3[q]);
    __syncthreads();  // s_acc reuse
    publish(v3, 3, 1);
    gsync();
    int pp = 1, cur = 1;
    double gam_prev = 1.0, alpha_prev = 1.0;
    for (int it = 0;; ++it) {
      SELL_STAMP(it, 0);
      double pb[3] = {0.0, 0.0, 0.0};
      if ((int)threadIdx.x < G) {
#pragma unroll
        for (int q = 0; q < 3; ++q) pb[q] = read_part(pp, q, threadIdx.x);
      }
      double n3[3] = {0.0, 0.0, 0.0};
      if (has && it < a.max_iters) {
        if constexpr (kCluster) slice_spmv_sym_g(a, u0, GatherM<kCluster>{gm(cur)}, n3, part, split);
        else slice_spmv_sym_g(a, u0, GatherM<kCluster>{gm(cur)}, n3);
      }
      combine(n3);
      SELL_STAMP(it, 1);
      SELL_BLOCK_STAMP(it, 3000);
#if GF_CG_TRACE_SM
      SELL_BLOCK_STAMP_AT(it, 20, 4000);
      if (a.trace && it == 10 && threadIdx.x == 0) {  // the SM each CTA runs on (imbalance diagnostics)
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        a.trace[1600 + blockIdx.x] = smid;
      }
#endif
      double red[3];
      if constexpr (kCluster) totals3(pb, red);  // gamma_it, delta_it, r_it.r_it
      else cta_tree<3>(pb, red);
      const double gam = red[0], del = red[1];
      relres = sqrt(red[2]) / bnorm;
      if (it > 0 && relres <= a.tol) {  // sparse.cpp:172-178 on the residual of update it
        iterations = it;
        converged = 1;
        break;
      }
      if (it >= a.max_iters) {
        iterations = it;
        converged = relres <= a.tol;
        break;
      }
      const double beta = it > 0 ? gam / gam_prev : 0.0;
      const double pap = it > 0 ? del - beta * gam / alpha_prev : del;  // = p.Ap
      if (pap <= 0.0) {  // sparse.cpp:160-168
        negcurv = pap < 0.0;
        iterations = it;
        converged = relres <= a.tol;
        break;
      }
      const double alpha = gam / pap;
      gam_prev = gam;
      alpha_prev = alpha;
      double v[3] = {0.0, 0.0, 0.0};
      if (live) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const size_t dof = 3 * (size_t)row + c;
          const double dvc = DV(c);
          const double zi = __fma_rn(beta, PV(Z, c), n3[c]);   // z = A q  = n + beta z
          const double si = __fma_rn(beta, PV(S, c), PV(W, c));  // s = A p  = w + beta s
          const double pi = __fma_rn(beta, PV(P, c), dvc * PV(R, c));  // p = u + beta p, u = D^-1 r
          PV(Z, c) = zi;
          PV(S, c) = si;
          PV(P, c) = pi;
          PV(X, c) = __fma_rn(alpha, pi, PV(X, c));
          const double ri = __fma_rn(-alpha, si, PV(R, c));
          const double ui = dvc * ri;                              // u = D^-1 r (q = D^-1 s is implied)
          const double wi = __fma_rn(-alpha, zi, PV(W, c));        // w -= alpha z
          PV(R, c) = ri;
          PV(W, c) = wi;
          gm(cur ^ 1)[dof] = dvc * wi;
          v[0] = __fma_rn(ri, ui, v[0]);
          v[1] = __fma_rn(wi, ui, v[1]);
          v[2] = __fma_rn(ri, ri, v[2]);
        }
      }
#pragma unroll
      for (int q = 0; q < 3; ++q) v[q] = lane_sum(v[q]);
      publish(v, 3, pp ^ 1);
      SELL_STAMP(it, 3);
      SELL_BLOCK_STAMP(it, 2000);
      pp ^= 1;
      cur ^= 1;
      gsync();
    }
    if (live)
#pragma unroll
      for (int c = 0; c < 3; ++c) a.x[3 * (size_t)row + c] = PV(X, c);
  }
#undef PV
  // no CTA of a cluster may exit while another can still read its shared memory (the last partial reads)
  if constexpr (kCluster) cg::this_cluster().sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.out[0] = iterations;
    a.out[1] = converged;
    a.out[2] = negcurv;
    a.out[3] = relres;
  }
}

// y = A x on the symmetric format (the FixedPatternSparse::multiply parity hook, sparse.cpp:49-58)
__global__ void __launch_bounds__(kThreads) k_spmv_sym(CgLaunch a, const double* xin, double* y) {
  const int lane = threadIdx.x & 31;
  for (int sl = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); sl < a.nslices;
       sl += (int)((gridDim.x * blockDim.x) >> 5)) {
    double acc[3];
    slice_spmv_sym_g(a, sl, GatherX{xin}, acc);
    const int row = sl * 32 + lane;
    if (row < a.nrows)
#pragma unroll
      for (int c = 0; c < 3; ++c) y[3 * (size_t)row + c] = acc[c];
  }
}

int g_grid = 0, g_dyn_per = 0;

constexpr size_t kSellSmem = GF_CG_SMEM ? (size_t)kWarpsPerCta * 6 * 3 * 32 * sizeof(double) : 0;
constexpr size_t kPipeSmem = (size_t)kWarpsPerCta * kPipeFields * 3 * 32 * sizeof(double);
constexpr size_t kSplitSmem = (size_t)1728 * sizeof(double);  // chunk sums of shared slices (split <= 4: 24 warps)

void set_smem_attributes() {
  static bool done = [] {
    cudaFuncSetAttribute((const void*)k_pcg_sell<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSellSmem);
    cudaFuncSetAttribute((const void*)k_pcg_sell<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSellSmem);
    cudaFuncSetAttribute((const void*)k_pcg_pipe<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPipeSmem);
    cudaFuncSetAttribute((const void*)k_pcg_pipe<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(kPipeSmem + kSplitSmem));
    cudaFuncSetAttribute((const void*)k_pcg_pipe<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    return true;
  }();
  (void)done;
}

}  // namespace

// co-resident CTAs of the cooperative solvers: the occupancy of every instance WITH its dynamic shared memory (the
// pipelined solver's 166 KB bounds it), one CTA per SM at 768 threads
int pcg_sell_grid() {
  if (g_grid == 0) {
    set_smem_attributes();
    int dev = 0, sms = 0, per = 1 << 30;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int q = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&q, k_pcg_sell<true>, kDynThreads, 0);
    g_dyn_per = q;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&q, k_pcg_big, kDynThreads, 0);
    g_dyn_per = std::min(g_dyn_per, q);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&q, k_pcg_sell<false>, kThreads, kSellSmem);
    per = std::min(per, q);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&q, k_pcg_pipe<false>, kThreads, kPipeSmem);
    per = std::min(per, q);
    if (per < 1) throw std::runtime_error("cooperative PCG kernels cannot be resident (occupancy 0)");
    g_grid = std::min(kMaxGrid, sms * per);
  }
  return g_grid;
}

size_t pcg_sell_part_doubles(int ndyn) { return 2 * 4 * ((size_t)kMaxGrid + (size_t)std::max(1, ndyn)); }
int pcg_sell_warps_per_cta() { return kWarpsPerCta; }
int pcg_dyn_warps_per_cta() { return kDynWarps; }
int pcg_dyn_grid() {  // co-resident CTAs of the large-matrix instance (its own block size, no dynamic smem)
  pcg_sell_grid();
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (g_dyn_per < 1) throw std::runtime_error("large-matrix PCG kernel cannot be resident (occupancy 0)");
  return std::min(kMaxGrid, sms * g_dyn_per);
}

// the largest cluster k_pcg_pipe<true> can be launched with on this device (0: clusters unavailable)
int pcg_max_cluster() {
  static int cached = -1;
  if (cached < 0) {
    set_smem_attributes();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16, 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = kPipeSmem + kSplitSmem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 16;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxPotentialClusterSize(&n, (const void*)k_pcg_pipe<true>, &cfg) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    cached = std::min(n, 16);
  }
  return cached;
}

int pcg_pipelined_default() {
  const char* e = std::getenv("GF_CG_PIPE");
  return e ? std::atoi(e) != 0 : 1;
}

void launch_pcg_sell(const CgLaunch& a, double* part, int ndyn, unsigned long long* ctr, cudaStream_t s) {
  SellArgs sa{a, part, part + 2 * 4 * (size_t)kMaxGrid, ctr};
  if (ndyn > 0) cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), s);
  void* args[] = {&sa};
  set_smem_attributes();
  const bool pipe = ndyn == 0 && a.pipelined;
  if (pipe && a.cluster > 0) {  // one thread-block cluster of a.grid CTAs (small matrices)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.grid, 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = kPipeSmem + kSplitSmem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = a.grid;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const cudaError_t err = cudaLaunchKernelEx(&cfg, k_pcg_pipe<true>, sa);
    if (err != cudaSuccess) {
      cudaGetLastError();
      throw std::runtime_error(std::string("cluster CG launch failed: ") + cudaGetErrorString(err));
    }
    return;
  }
  const void* fn = pipe ? (const void*)k_pcg_pipe<false>
                  : ndyn > 0 ? (a.big ? (const void*)k_pcg_big : (const void*)k_pcg_sell<true>)
                             : (const void*)k_pcg_sell<false>;
  const size_t smem = pipe ? kPipeSmem : ndyn > 0 ? 0 : kSellSmem;
  const int grid = a.grid > 0 ? a.grid : ndyn > 0 ? pcg_dyn_grid() : pcg_sell_grid();
  const cudaError_t err = cudaLaunchCooperativeKernel(fn, grid, ndyn > 0 ? kDynThreads : kThreads, args, smem, s);
  if (err != cudaSuccess) {
    cudaGetLastError();
    throw std::runtime_error(std::string("cooperative CG launch failed: ") + cudaGetErrorString(err));
  }
}

void launch_spmv_sym(const CgLaunch& a, const double* xin, double* y, cudaStream_t s) {
  k_spmv_sym<<<pcg_sell_grid(), kThreads, 0, s>>>(a, xin, y);
}

}  // namespace gfb
