// cg_onchip.cu — the pipelined Jacobi-PCG (cg_solve, sparse.cpp:129-188) with the system matrix held ON CHIP for
// the whole solve: each CTA loads the upper blocks of its rows once, into tensor memory (TMEM) and shared memory,
// and every iteration's SpMV then reads the matrix from on-chip storage instead of L2.
//
// Why: k_pcg_pipe (cg_sell.cu) streams every block of the full matrix from L2 each iteration (an upper block for its
// row, the same block transposed for its column's row): ~1.3 KB per node row and iteration at c3, which the L2 -> SM
// bandwidth (64 B/clk/SM measured) turns into ~8 of its ~15 us per iteration. On chip, per SM (one CTA owning up to
// 24 slices of 32 rows, as in k_pcg_pipe):
// The pattern must have at most 7 distinct positive column offsets off[0..6] (the box meshes' Freudenthal rows: +1,
// +nx, +nx+1, +nx ny, +nx ny+1, +nx ny+nx, +nx ny+nx+1); a row's upper block at offset off[b] lives in SLOT b (absent
// slots hold zero blocks), so a block's column, its transposed partner's slot and every route below are fixed by b:
//   TMEM (512 columns x 128 lanes; 3 warps share a lane quadrant, 84 columns per row): the diagonal block (symmetric:
//        6 values -- the assembly writes exactly symmetric diagonal blocks) and slots 3..6 (9 values each);
//        tcgen05.ld reads 425 B/clk/SM (measured, tools/tmem_bw.cu), 3.3x shared memory;
//   shared memory: slots 0..2 ([slot][entry][row]) -- readable by every thread of the CTA --, the m-cache (below)
//        and D^-1.
// 384 threads own two rows each (768 rows = 24 slices per CTA, slices cs0 + w and cs0 + w + 12): the registers of
// two rows' solver state plus their loads in flight fit 168 per thread, where one row per thread at 768 threads
// (80 registers) spills.
//
// Symmetric SpMV without reading a block twice from L2: block (i, b) of row i with column j = i + off[b] contributes
// B v_j to row i and t = B^T v_i to row j. Row i's thread computes the direct product; the transposed one reaches row
// j by one of three routes, decided identically on both sides from (b, lane, CTA range):
//   shuffle  slot 0 (offset +1), j = i + 1 in the same warp: t moves one lane up (shfl);
//   on chip  slots 0..2 with both rows in the CTA: row j's thread computes t itself from row i's shared-memory block
//            and the CTA's shared copy of the gathered vector (the m-cache, written with the global copy);
//   remote   everything else (slots 3..6, CTA edges): t = B^T m_i is computed by the owner at the END of the previous
//            iteration, as soon as its new m_i exists (the pipelined recurrences know m one iteration ahead), and
//            published through double-buffered global planes before the grid barrier -- so no extra barrier.
// Per row and iteration the L2 then carries the gathers of slots 3..6, the remote t (written and read) and m itself
// (~0.3 KB instead of ~1.3 KB).
//
// The recurrences, decisions and deterministic reductions are k_pcg_pipe's (Ghysels & Vanroose pipelined PCG; one
// grid barrier per iteration; decisions mapped one to one onto the reference's). Every row sums its contributions in
// one fixed order and the reductions use fixed trees, so the solve is bit-reproducible.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "dev_types.cuh"

namespace gfb {
namespace {

namespace cgx = cooperative_groups;

constexpr int kT = 384;                  // threads per CTA
constexpr int kW = kT / 32;              // 12 warps
constexpr int kRpt = 2;                  // node rows per thread
constexpr int kRows = kT * kRpt;         // 768 rows = 24 slices per CTA
constexpr int kTmCols = 84;              // TMEM columns per row: a warp's two rows take 168 of 512 (3 warps per quadrant)
constexpr int kTmSlot3 = 12;             // diagonal (6 doubles) at columns 0..11, slot b >= 3 at 12 + 18 (b - 3)
constexpr int kMaxGridOc = 1024;         // CTA partial slots per value (as cg_sell.cu)
constexpr size_t kBlkDoubles = 27 * (size_t)kRows;  // slots 0..2, [b][entry][local row]
constexpr size_t kMDoubles = 3 * (size_t)kRows;     // the CTA's rows of the gathered vector, [component][local row]
constexpr size_t kDDoubles = 3 * (size_t)kRows;     // D^-1, [component][local row]
constexpr size_t kOcSmem = (kBlkDoubles + kMDoubles + kDDoubles) * sizeof(double);

struct OcArgs {
  CgLaunch a;
  double* cta_part;       // 2 parities x 4 values x kMaxGridOc
  double* tg;             // remote t: 2 parities x 21 planes (slot b * 3 + component) x npad
  double* gm;             // the gathered vector m: 2 buffers x 3 component planes x npad
  const uint32_t* meta;   // per row: upper slot mask | lower slot mask << 8
  int32_t npad;           // >= nrows + 1: row index nrows of every plane / buffer is a zero entry (never written)
  int32_t shuf;           // off[0] == 1: slot 0's column is the next row (the shuffle route)
  int32_t off[7];         // the matrix's distinct positive column offsets, ascending
};

__device__ __forceinline__ unsigned long long gtimer_oc() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// diagnostics (GF_CG_TRACE, tools/cg_trace_oc.py): CTA 0 stamps 5 points of every iteration; at iteration 10 every CTA
// stamps the end of its SpMV (after a CTA barrier)
#define OC_SUB(point)                                                                         \
  do {                                                                                        \
    if (a.trace && sub_on && tid == 0 && blockIdx.x == 0 && h == 0) a.trace[4100 + (point)] = gtimer_oc(); \
  } while (0)
#define OC_STAMP(k, point)                                                   \
  do {                                                                       \
    if (a.trace && tid == 0 && blockIdx.x == 0 && (k) < 200)                 \
      a.trace[(k) * 8 + (point)] = gtimer_oc();                              \
  } while (0)

__device__ __forceinline__ int launder(int x) {  // an opaque copy: keeps the compiler from hoisting what depends on x
  asm volatile("" : "+r"(x));
  return x;
}
__device__ __forceinline__ uint32_t launder(uint32_t x) {
  asm volatile("" : "+r"(x));
  return x;
}
__device__ __forceinline__ double lane_sum_oc(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---- tensor memory (tcgen05) ----
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// 9 doubles (18 columns) of this thread's TMEM lane; the wait names the destination registers so that no use of
// them can be scheduled before the load completes
__device__ __forceinline__ void tm_ld9(uint32_t ta, double (&m)[9]) {
  uint32_t r[18];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(ta));
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];\n" : "=r"(r[16]), "=r"(r[17]) : "r"(ta + 16));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15]), "+r"(r[16]), "+r"(r[17]));
#pragma unroll
  for (int q = 0; q < 9; ++q) m[q] = __hiloint2double((int)r[2 * q + 1], (int)r[2 * q]);
}
__device__ __forceinline__ void tm_ld6(uint32_t ta, double (&m)[6]) {
  uint32_t r[12];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(ta));
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11])
               : "r"(ta + 8));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]));
#pragma unroll
  for (int q = 0; q < 6; ++q) m[q] = __hiloint2double((int)r[2 * q + 1], (int)r[2 * q]);
}
template <int N>
__device__ __forceinline__ void tm_st(uint32_t ta, const double* m) {  // N doubles (2N columns), N = 6 or 9
  uint32_t r[18];
#pragma unroll
  for (int q = 0; q < N; ++q) {
    r[2 * q] = (uint32_t)__double2loint(m[q]);
    r[2 * q + 1] = (uint32_t)__double2hiint(m[q]);
  }
  if (N == 9) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(ta),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};\n" ::"r"(ta + 16), "r"(r[16]), "r"(r[17])
                 : "memory");
  } else {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(ta), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(ta + 8), "r"(r[8]), "r"(r[9]),
                 "r"(r[10]), "r"(r[11])
                 : "memory");
  }
}

__device__ __forceinline__ void mv_add(const double (&B)[9], const double (&v)[3], double (&acc)[3]) {
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    acc[r] = __fma_rn(B[3 * r], v[0], acc[r]);
    acc[r] = __fma_rn(B[3 * r + 1], v[1], acc[r]);
    acc[r] = __fma_rn(B[3 * r + 2], v[2], acc[r]);
  }
}
__device__ __forceinline__ void mtv(const double (&B)[9], const double (&v)[3], double (&t)[3]) {  // t = B^T v
#pragma unroll
  for (int c = 0; c < 3; ++c) t[c] = __fma_rn(B[6 + c], v[2], __fma_rn(B[3 + c], v[1], B[c] * v[0]));
}

// kCluster: the whole solve in ONE thread-block cluster (small matrices, <= 16 x 24 slices): the hardware cluster
// barrier replaces the grid barrier, the CTA partials travel through distributed shared memory and the gathered
// vector is read through L2 (the cluster barrier orders memory at cluster scope; it does not invalidate L1)
template <bool kCluster>
__global__ void __launch_bounds__(kT, 1) k_pcg_onchip(OcArgs oa) {
  auto gsync = [] {
    if constexpr (kCluster) cgx::this_cluster().sync();
    else cgx::this_grid().sync();
  };
  __shared__ double s_part[2][4];  // kCluster: this CTA's published partials (read by the cluster through DSMEM)
  const CgLaunch& a = oa.a;
  extern __shared__ double s_dyn[];
  double* const s_blk = s_dyn;                          // [b][q][local row]
  double* const s_m = s_dyn + kBlkDoubles;              // the gathered vector of the CTA's rows [component][row]
  double* const s_d = s_dyn + kBlkDoubles + kMDoubles;  // D^-1 [component][local row]
  __shared__ uint32_t s_taddr;
  __shared__ double s_acc[kW][4];
  __shared__ double s_w[kW][4];
  __shared__ double s_x1[3][kT];  // x of each thread's second row (the register budget)
  __shared__ double s_p1[3][kT];  // p of each thread's second row
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, G = (int)gridDim.x;
  const int cs0 = __ldg(a.cta_first + blockIdx.x), cs1 = __ldg(a.cta_first + blockIdx.x + 1);
  const int r0 = cs0 * 32, r1 = cs1 * 32;  // this CTA's rows (rows >= nrows are never referenced)
  const int nrows = a.nrows, npad = oa.npad, ZP = nrows;  // ZP: the zero entry of every global plane
  const bool shuf = oa.shuf != 0;

  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_addr(&s_taddr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  for (int k = tid; k < (int)kMDoubles; k += kT) s_m[k] = 0.0;  // rows the CTA does not have stay zero
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");

  // this thread's two rows: slices cs0 + w + 12 h (local rows li), TMEM columns 84 h.. of its warp's 168
  int row[kRpt], li[kRpt];
  bool live[kRpt];
  uint32_t tmh[kRpt], pm[kRpt];  // pm: upper slot mask | lower slot mask << 8 (0 for dead rows)
#pragma unroll
  for (int h = 0; h < kRpt; ++h) {
    const int sl = cs0 + w + kW * h;
    row[h] = sl * 32 + lane;
    li[h] = (w + kW * h) * 32 + lane;
    live[h] = sl < cs1 && row[h] < nrows;
    tmh[h] = s_taddr + ((uint32_t)(32 * (w & 3)) << 16) + (uint32_t)((w >> 2) * 2 * kTmCols + h * kTmCols);
    pm[h] = live[h] ? __ldg(oa.meta + row[h]) : 0u;
    // the slice's upper blocks (ordinal c = 1 + the number of present slots below b) into their slots
    const int ub = live[h] ? __ldg(a.usp + sl) : 0;
    {
      double m[9];
#pragma unroll
      for (int q = 0; q < 9; ++q) m[q] = live[h] ? __ldcg(a.vals + ((size_t)ub * 9 + q) * 32 + lane) : 0.0;
      const double d6[6] = {m[0], m[1], m[2], m[4], m[5], m[8]};
      tm_st<6>(tmh[h], d6);
    }
#pragma unroll
    for (int b = 0; b < 7; ++b) {
      const bool pres = (pm[h] >> b) & 1u;
      const int c = 1 + __popc(pm[h] & ((1u << b) - 1u));
      double m[9];
#pragma unroll
      for (int q = 0; q < 9; ++q) m[q] = pres ? __ldcg(a.vals + ((size_t)(ub + c) * 9 + q) * 32 + lane) : 0.0;
      if (b <= 2) {
#pragma unroll
        for (int q = 0; q < 9; ++q) s_blk[(b * 9 + q) * kRows + li[h]] = m[q];
      } else {
        tm_st<9>(tmh[h] + kTmSlot3 + 18 * (b - 3), m);
      }
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) s_d[k * kRows + li[h]] = live[h] ? __ldg(a.dinv + 3 * (size_t)row[h] + k) : 0.0;
  }
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  __syncthreads();

  auto up = [&](int h, int b) -> bool { return (pm[h] >> b) & 1u; };
  auto lo = [&](int h, int b) -> bool { return (pm[h] >> (8 + b)) & 1u; };
  auto Dv = [&](int h, int k) -> double { return s_d[k * kRows + li[h]]; };
  double* const tg0 = oa.tg;
  auto tmem_block = [&](int h, int b, double (&B)[9]) { tm_ld9(tmh[h] + kTmSlot3 + 18 * (b - 3), B); };
  // routes of the transposed products, fixed by the slot b: slots 0..2 whose other row is in the CTA are computed
  // by the CONSUMER from the producer's shared-memory block and the CTA's copy of the gathered vector (slot 0 in
  // lanes 1..31: the previous lane's product, shuffled); everything else is remote -- the global t planes, written by
  // the producer at the end of the previous iteration
  auto up_remote = [&](int h, int b) -> bool {
    if (b <= 2) return up(h, b) && row[h] + oa.off[b] >= r1;
    return live[h];  // slots 3..6: always (absent slots store zeros that no row reads)
  };
  auto lo_remote = [&](int h, int b) -> bool { return lo(h, b) && (b >= 3 || row[h] - oa.off[b] < r0); };
  // the CTA's copy of the vector the next SpMV gathers (written with the global one; read after the grid barrier)
  auto put_m = [&](int h, const double (&v)[3]) {
#pragma unroll
    for (int k = 0; k < 3; ++k) s_m[k * kRows + li[h]] = v[k];
  };

  // remote transposed products of v (row h's value) for the NEXT SpMV, published before the grid barrier: slots
  // 3..6 every row (absent slots hold zero blocks), slots 0..2 at CTA edges only
  auto produce = [&](int h, const double (&v)[3], int par) {
    if (!__any_sync(0xffffffffu, live[h])) return;
    row[h] = launder(row[h]);
    li[h] = launder(li[h]);
    tmh[h] = launder(tmh[h]);
    double* const base = tg0 + (size_t)par * 21 * npad + row[h];
#pragma unroll
    for (int b = 0; b < 7; ++b) {
      const bool rem = up_remote(h, b);
      double B[9];
      if (b <= 2) {
        if (!__any_sync(0xffffffffu, rem)) continue;
#pragma unroll
        for (int q = 0; q < 9; ++q) B[q] = s_blk[(b * 9 + q) * kRows + li[h]];
      } else {
        tmem_block(h, b, B);
      }
      double t[3];
      mtv(B, v, t);
      if (rem)
#pragma unroll
        for (int k = 0; k < 3; ++k) base[(b * 3 + k) * npad] = t[k];
    }
  };

  // n = A v for both rows: v their own values, vg the published vector (zero at row ZP), par the parity of the
  // remote t of v; the CTA's rows of v are also in s_m. One accumulator per row in a fixed order: the diagonal, then
  // the on-chip products (slots 0..2 direct and, for rows of the CTA, transposed) while the first loads fly, then the
  // remote lower products and the direct products of slots 3..6 as their loads arrive. Loads go out in rounds of at
  // most four 24-byte items, one row at a time (the register budget).
  bool sub_on = false;
  auto spmv = [&](const double* vg, const double (&v)[kRpt][3], int par, double (&n)[kRpt][3]) {
#pragma unroll
    for (int h = 0; h < kRpt; ++h) {
      row[h] = launder(row[h]);
      li[h] = launder(li[h]);
      tmh[h] = launder(tmh[h]);
      pm[h] = launder(pm[h]);
    }
    par = launder(par);
    const double* const tgb = tg0 + (size_t)par * 21 * npad;
    auto lower_t = [&](int h, int b, double (&t)[3]) {  // remote lower product of slot b (zero entry otherwise)
      const int i = lo_remote(h, b) ? row[h] - oa.off[b] : ZP;
#pragma unroll
      for (int k = 0; k < 3; ++k) t[k] = __ldcg(tgb + (b * 3 + k) * npad + i);
    };
    auto gather = [&](int h, int b, double (&g)[3]) {  // v at slot b's column from global (zero entry if not taken)
      const int j = up(h, b) ? row[h] + oa.off[b] : ZP;
#pragma unroll
      for (int k = 0; k < 3; ++k) g[k] = kCluster ? __ldcg(vg + k * npad + j) : __ldca(vg + k * npad + j);
    };
    auto add3 = [&](int h, const double (&t)[3]) {
#pragma unroll
      for (int k = 0; k < 3; ++k) n[h][k] += t[k];
    };
    auto slot_tm = [&](int h, int b, const double (&g)[3]) {
      double B[9];
      tmem_block(h, b, B);
      mv_add(B, g, n[h]);
    };
#pragma unroll
    for (int h = 0; h < kRpt; ++h) {
      if (!__any_sync(0xffffffffu, live[h])) {  // a warp without this slice (CTAs of fewer than 24 slices)
#pragma unroll
        for (int k = 0; k < 3; ++k) n[h][k] = 0.0;
        continue;
      }
      double L[4][3];
      OC_SUB(0);
      // round 1: the remote lower products of slots 6..4 (and of slots 0..2 at CTA edges)
      lower_t(h, 6, L[0]);
      lower_t(h, 5, L[1]);
      lower_t(h, 4, L[2]);
      const double(&x)[3] = v[h];
      {
        double d[6];
        tm_ld6(tmh[h], d);
        n[h][0] = __fma_rn(d[2], x[2], __fma_rn(d[1], x[1], d[0] * x[0]));
        n[h][1] = __fma_rn(d[4], x[2], __fma_rn(d[3], x[1], d[1] * x[0]));
        n[h][2] = __fma_rn(d[5], x[2], __fma_rn(d[4], x[1], d[2] * x[0]));
      }
      // slots 0..2 on chip. Slot 0: the next row is the next lane (shuffle); lane 31 reads the next slice's row from
      // s_m (or global at the CTA's end); its transposed product reaches lanes 1..31 by shuffle
      {
        double vj[3], B[9], t1[3], tr[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) vj[k] = __shfl_down_sync(0xffffffffu, x[k], 1);
        if (!(shuf && lane < 31)) {
          const int j = row[h] + oa.off[0];
          const bool in = up(h, 0) && j < r1;
#pragma unroll
          for (int k = 0; k < 3; ++k)
            vj[k] = in ? s_m[k * kRows + li[h] + oa.off[0]] : __ldcg(vg + k * npad + (up(h, 0) ? j : ZP));
        }
#pragma unroll
        for (int q = 0; q < 9; ++q) B[q] = s_blk[q * kRows + li[h]];
        mv_add(B, vj, n[h]);
        mtv(B, x, t1);
#pragma unroll
        for (int k = 0; k < 3; ++k) tr[k] = __shfl_up_sync(0xffffffffu, t1[k], 1);
        if (shuf && lane > 0 && lo(h, 0)) add3(h, tr);
      }
#pragma unroll
      for (int b = 1; b <= 2; ++b) {  // direct products of slots 1, 2
        const int j = row[h] + oa.off[b];
        const bool in = j < r1;
        double g[3], B[9];
#pragma unroll
        for (int k = 0; k < 3; ++k)
          g[k] = in ? s_m[k * kRows + li[h] + oa.off[b]] : __ldcg(vg + k * npad + (up(h, b) ? j : ZP));
#pragma unroll
        for (int q = 0; q < 9; ++q) B[q] = s_blk[(b * 9 + q) * kRows + li[h]];
        mv_add(B, g, n[h]);
      }
      // transposed products of the CTA's rows: slot 0 for lane 0 (the previous slice's lane 31; without a +1
      // offset every lane), slots 1, 2
#pragma unroll
      for (int b = 0; b <= 2; ++b) {
        const int i = row[h] - oa.off[b];
        const bool take = lo(h, b) && i >= r0 && !(b == 0 && shuf && lane > 0);
        if (take) {
          const int src = li[h] - oa.off[b];
          double B[9], mi[3], t[3];
#pragma unroll
          for (int q = 0; q < 9; ++q) B[q] = s_blk[(b * 9 + q) * kRows + src];
#pragma unroll
          for (int k = 0; k < 3; ++k) mi[k] = s_m[k * kRows + src];
          mtv(B, mi, t);
          add3(h, t);
        }
      }
      OC_SUB(1);
      add3(h, L[0]);
      add3(h, L[1]);
      add3(h, L[2]);
      OC_SUB(2);
      // round 2: slot 3's remote lower product, the columns of slots 3, 4, and the CTA-edge remote lower products
      lower_t(h, 3, L[0]);
      gather(h, 3, L[1]);
      gather(h, 4, L[2]);
      double E[3][3];
      lower_t(h, 2, E[0]);
      lower_t(h, 1, E[1]);
      lower_t(h, 0, E[2]);
      add3(h, L[0]);
      slot_tm(h, 3, L[1]);
      slot_tm(h, 4, L[2]);
      add3(h, E[0]);
      add3(h, E[1]);
      add3(h, E[2]);
      OC_SUB(3);
      // round 3: the columns of slots 5, 6
      gather(h, 5, L[0]);
      gather(h, 6, L[1]);
      slot_tm(h, 5, L[0]);
      slot_tm(h, 6, L[1]);
      OC_SUB(4);
    }
  };

  auto publish = [&](const double* v, int nv, int parity) {
    if (lane == 0)
      for (int q = 0; q < nv; ++q) s_acc[w][q] = v[q];
    __syncthreads();
    if (tid < nv) {
      double x = 0.0;
      for (int k = 0; k < kW; ++k) x += s_acc[k][tid];
      if constexpr (kCluster) s_part[parity][tid] = x;
      else oa.cta_part[((size_t)parity * 4 + tid) * kMaxGridOc + blockIdx.x] = x;
    }
  };
  // the published CTA partials (thread k < G holds CTA k's), loaded before an SpMV and reduced after it
  auto load_parts = [&](int parity, int nv, double (&pb)[3]) {
#pragma unroll
    for (int q = 0; q < 3; ++q) pb[q] = 0.0;
    for (int k = tid; k < G; k += kT)
#pragma unroll
      for (int q = 0; q < 3; ++q)
        if (q < nv) {
          if constexpr (kCluster) pb[q] += *cgx::this_cluster().map_shared_rank(&s_part[parity][q], k);
          else pb[q] += __ldcg(oa.cta_part + ((size_t)parity * 4 + q) * kMaxGridOc + k);
        }
  };
  auto totals = [&](const double (&pb)[3], double (&out)[3]) {  // fixed lane and warp trees, identical everywhere
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const double t = lane_sum_oc(pb[q]);
      if (lane == 0) s_w[w][q] = t;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 3; ++q) out[q] = lane_sum_oc(lane < kW ? s_w[lane][q] : 0.0);
    // no trailing barrier: s_w is next written by the following totals(), which a publish() barrier precedes
  };

  // solver state of the two rows in registers (D^-1 in shared memory)
  double X[kRpt][3], R[kRpt][3], Wv[kRpt][3], P[kRpt][3], S[kRpt][3], Z[kRpt][3];
#pragma unroll
  for (int h = 0; h < kRpt; ++h)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      X[h][k] = live[h] ? a.x[3 * (size_t)row[h] + k] : 0.0;
      if (h == 1) {
        s_x1[k][tid] = X[h][k];
        s_p1[k][tid] = 0.0;
      }
      R[h][k] = Wv[h][k] = P[h][k] = S[h][k] = Z[h][k] = 0.0;
    }
  int tpar = 0;
  // the gathered vector's two buffers (row ZP of each a zero entry): x0 (setup 1) and m_{2k} in gm1, u and m_{2k+1}
  // in gm0 -- a buffer is rewritten only after a grid barrier that follows the last SpMV reading it
  double* const gm0 = oa.gm;
  double* const gm1 = oa.gm + 3 * (size_t)npad;
  // setup 1 (sparse.cpp:145-157): r = b - A x0, u = D^-1 r (gathered next), partial b.b
  double acc[kRpt][3];
  if (a.x0_identity) {  // A x0 = x0 (CgLaunch::x0_identity): no SpMV
#pragma unroll
    for (int h = 0; h < kRpt; ++h)
#pragma unroll
      for (int k = 0; k < 3; ++k) acc[h][k] = X[h][k];
  } else {
#pragma unroll
    for (int h = 0; h < kRpt; ++h) {
      if (live[h])
#pragma unroll
        for (int k = 0; k < 3; ++k) gm1[k * npad + row[h]] = X[h][k];
      put_m(h, X[h]);
      produce(h, X[h], tpar);
    }
    gsync();
    spmv(gm1, X, tpar, acc);
    tpar ^= 1;
    __syncthreads();  // every warp's SpMV has read s_m before it is rewritten
  }
  double bb = 0.0, U[kRpt][3];
#pragma unroll
  for (int h = 0; h < kRpt; ++h) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const size_t dof = 3 * (size_t)row[h] + k;
      const double bi = live[h] ? a.b[dof] : 0.0;
      R[h][k] = bi - acc[h][k];
      U[h][k] = Dv(h, k) * R[h][k];
      if (live[h]) gm0[k * npad + row[h]] = U[h][k];
      bb = __fma_rn(bi, bi, bb);
    }
    put_m(h, U[h]);
    produce(h, U[h], tpar);
  }
  bb = lane_sum_oc(bb);
  publish(&bb, 1, 0);
  gsync();
  double tot[3], pb0[3];
  load_parts(0, 1, pb0);
  totals(pb0, tot);
  const double bnorm = sqrt(tot[0]);
  int iterations = 0, converged = 0, negcurv = 0;
  double relres = 0.0;
  if (bnorm == 0.0) {  // sparse.cpp:145-150
#pragma unroll
    for (int h = 0; h < kRpt; ++h)
      if (live[h])
#pragma unroll
        for (int k = 0; k < 3; ++k) a.x[3 * (size_t)row[h] + k] = 0.0;
    converged = 1;
  } else {
    // setup 2: w = A u, m = D^-1 w (gathered by iteration 0), partials gamma_0, delta_0, r.r
    spmv(gm0, U, tpar, acc);
    tpar ^= 1;
    __syncthreads();  // every warp's SpMV has read s_m before it is rewritten
    double v3[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int h = 0; h < kRpt; ++h) {
      double M[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        Wv[h][k] = acc[h][k];
        M[k] = Dv(h, k) * acc[h][k];
        if (live[h]) gm1[k * npad + row[h]] = M[k];
        s_m[k * kRows + li[h]] = M[k];
        v3[0] = __fma_rn(R[h][k], U[h][k], v3[0]);
        v3[1] = __fma_rn(acc[h][k], U[h][k], v3[1]);
        v3[2] = __fma_rn(R[h][k], R[h][k], v3[2]);
      }
      produce(h, M, tpar);
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) v3[q] = lane_sum_oc(v3[q]);
    __syncthreads();  // s_acc reuse
    publish(v3, 3, 1);
    gsync();
    int pp = 1, cur = 1;
    // reciprocals of the previous iteration's gamma and gamma * alpha, formed off the critical path: beta and p.Ap
    // then cost multiplies, and the only division left between the reduction and the update is alpha's
    double inv_g = 1.0, inv_ga = 1.0;
    for (int it = 0;; ++it) {
      OC_STAMP(it, 0);
      double pb[3], red[3];
      load_parts(pp, 3, pb);
      double n3[kRpt][3];
      if (it < a.max_iters) {
        double m[kRpt][3];
#pragma unroll
        for (int h = 0; h < kRpt; ++h)
#pragma unroll
          for (int k = 0; k < 3; ++k) m[h][k] = Dv(h, k) * Wv[h][k];
        sub_on = it == 10;
        spmv(cur ? gm1 : gm0, m, tpar, n3);
        sub_on = false;
        tpar ^= 1;
      }
      OC_STAMP(it, 1);
      if (a.trace && it == 10) {
        __syncthreads();
        if (tid == 0) a.trace[3000 + blockIdx.x] = gtimer_oc();
      }
      totals(pb, red);  // gamma_it, delta_it, r_it.r_it
      OC_STAMP(it, 2);
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
      const double beta = it > 0 ? gam * inv_g : 0.0;                              // gamma / gamma_prev
      const double pap = it > 0 ? __fma_rn(-(gam * inv_ga), gam, del) : del;      // = p.Ap = delta - beta gamma / alpha_prev
      if (pap <= 0.0) {  // sparse.cpp:160-168
        negcurv = pap < 0.0;
        iterations = it;
        converged = relres <= a.tol;
        break;
      }
      const double alpha = gam / pap;
      inv_g = 1.0 / gam;
      inv_ga = 1.0 / (gam * alpha);
      double v[3] = {0.0, 0.0, 0.0};
      double* const gnext = cur ? gm0 : gm1;
      double M2[kRpt][3];
#pragma unroll
      for (int h = 0; h < kRpt; ++h) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const double dk = Dv(h, k);
          Z[h][k] = __fma_rn(beta, Z[h][k], n3[h][k]);      // z = A q = n + beta z
          S[h][k] = __fma_rn(beta, S[h][k], Wv[h][k]);      // s = A p = w + beta s
          double pk;  // p = u + beta p, u = D^-1 r
          if (h == 0) {
            pk = P[h][k] = __fma_rn(beta, P[h][k], dk * R[h][k]);
            X[h][k] = __fma_rn(alpha, pk, X[h][k]);
          } else {
            pk = s_p1[k][tid] = __fma_rn(beta, s_p1[k][tid], dk * R[h][k]);
            s_x1[k][tid] = __fma_rn(alpha, pk, s_x1[k][tid]);
          }
          R[h][k] = __fma_rn(-alpha, S[h][k], R[h][k]);
          const double uk = dk * R[h][k];
          Wv[h][k] = __fma_rn(-alpha, Z[h][k], Wv[h][k]);   // w -= alpha z
          M2[h][k] = dk * Wv[h][k];
          if (live[h]) gnext[k * npad + row[h]] = M2[h][k];
          s_m[k * kRows + li[h]] = M2[h][k];
          v[0] = __fma_rn(R[h][k], uk, v[0]);
          v[1] = __fma_rn(Wv[h][k], uk, v[1]);
          v[2] = __fma_rn(R[h][k], R[h][k], v[2]);
        }
      }
      OC_STAMP(it, 5);
#pragma unroll
      for (int h = 0; h < kRpt; ++h) produce(h, M2[h], tpar);
      OC_STAMP(it, 3);
#pragma unroll
      for (int q = 0; q < 3; ++q) v[q] = lane_sum_oc(v[q]);
      publish(v, 3, pp ^ 1);
      OC_STAMP(it, 4);
      if (a.trace && it == 10 && tid == 0) a.trace[2000 + blockIdx.x] = gtimer_oc();
      pp ^= 1;
      cur ^= 1;
      gsync();
    }
#pragma unroll
    for (int h = 0; h < kRpt; ++h)
      if (live[h])
#pragma unroll
        for (int k = 0; k < 3; ++k) a.x[3 * (size_t)row[h] + k] = h == 0 ? X[h][k] : s_x1[k][tid];
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  // no CTA of a cluster may exit while another can still read its shared memory (the last partial reads)
  if constexpr (kCluster) cgx::this_cluster().sync();
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(s_taddr));
  if (blockIdx.x == 0 && tid == 0) {
    a.out[0] = iterations;
    a.out[1] = converged;
    a.out[2] = negcurv;
    a.out[3] = relres;
  }
}

}  // namespace

// co-resident CTAs of k_pcg_onchip (one per SM: its shared memory), 0 when it cannot run here
int pcg_onchip_grid() {
  static int g = -1;
  if (g < 0) {
    cudaFuncSetAttribute((const void*)k_pcg_onchip<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kOcSmem);
    cudaFuncSetAttribute((const void*)k_pcg_onchip<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kOcSmem);
    cudaFuncSetAttribute((const void*)k_pcg_onchip<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int dev = 0, sms = 0, q = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&q, k_pcg_onchip<false>, kT, kOcSmem) != cudaSuccess) {
      cudaGetLastError();
      q = 0;
    }
    g = q >= 1 ? std::min(kMaxGridOc, sms) : 0;
  }
  return g;
}
// the largest cluster k_pcg_onchip<true> can be launched with (0: clusters unavailable)
int pcg_onchip_max_cluster() {
  static int cached = -1;
  if (cached < 0) {
    pcg_onchip_grid();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16, 1, 1);
    cfg.blockDim = dim3(kT, 1, 1);
    cfg.dynamicSmemBytes = kOcSmem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 16;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxPotentialClusterSize(&n, (const void*)k_pcg_onchip<true>, &cfg) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    cached = std::min(n, 16);
  }
  return cached;
}
int pcg_onchip_warps_per_cta() { return kRows / 32; }  // slices per CTA (two per warp)
int pcg_onchip_npad(int nslices) { return nslices * 32 + 32; }  // row nrows <= npad - 1 is the zero entry
size_t pcg_onchip_t_doubles(int nslices) { return 2 * 21 * (size_t)pcg_onchip_npad(nslices); }
size_t pcg_onchip_m_doubles(int nslices) { return 2 * 3 * (size_t)pcg_onchip_npad(nslices); }

void launch_pcg_onchip(const CgLaunch& a, double* part, double* tg, double* gm, const uint32_t* meta,
                       const int32_t off[7], cudaStream_t s) {
  OcArgs oa{a, part, tg, gm, meta, pcg_onchip_npad(a.nslices), off[0] == 1, {}};
  for (int b = 0; b < 7; ++b) oa.off[b] = off[b];
  pcg_onchip_grid();
  if (a.cluster) {  // one thread-block cluster of a.grid CTAs
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.grid, 1, 1);
    cfg.blockDim = dim3(kT, 1, 1);
    cfg.dynamicSmemBytes = kOcSmem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = a.grid;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const cudaError_t err = cudaLaunchKernelEx(&cfg, k_pcg_onchip<true>, oa);
    if (err != cudaSuccess) {
      cudaGetLastError();
      throw std::runtime_error(std::string("on-chip cluster CG launch failed: ") + cudaGetErrorString(err));
    }
    return;
  }
  void* args[] = {&oa};
  const cudaError_t err = cudaLaunchCooperativeKernel((const void*)k_pcg_onchip<false>, a.grid, kT, args, kOcSmem, s);
  if (err != cudaSuccess) {
    cudaGetLastError();
    throw std::runtime_error(std::string("on-chip CG launch failed: ") + cudaGetErrorString(err));
  }
}

}  // namespace gfb
