// damage.cu — per-timestep damage pass (Simulation::damage_pass, solver.cpp:90-103) on the GPU.
//
// BUILT WITH -fmad=false: every kernel here must reproduce the CPU oracle bit-for-bit (edge labels,
// newly-broken sets and chi are bit-exact from an identical state; north_star).
//
//  k_tet_stress  thread/tet: F, P, Cauchy six-vector sigma_c (per_tet_cauchy, solver.cpp:79-88), edge
//                transform T (build_T, fracture.cpp:16-28), local edge stresses sigma_f = T sigma_c
//                (fracture.cpp:74), degenerate flag; for r_d = 0 also the screened value T*(0 + 1*sigma_c)
//                reduced straight into the per-edge max (fracture.cpp:80-87) by an order-free atomic max.
//  k_nonlocal    thread/tet (r_d > 0): avg = sum_w w*sigma_c[o] in table order (fracture.cpp:75-76),
//                screened = T*avg (fracture.cpp:77), atomic max into the edges. k_nonlocal_cell (several tets of a
//                cell per thread, weights through a cp.async.bulk ring) and k_nonlocal_tpl are its structured-mesh
//                forms: the same sums in the same order.
//  k_relabel     thread/edge: decode the max (-inf -> 0, fracture.cpp:88-89), signed >= threshold relabel
//                of intact edges (update_damage, fracture.cpp:93-104), warp-ballot + one atomic per warp
//                compaction of the newly-broken ids (ascending order restored on read-back), key reset.
//  k_chi         thread/tet: compute_chi (fracture.cpp:127-157) incl. fragment_components
//                (fracture.cpp:106-125), degenerate -> 0, chi = min(chi_old, value) (solver.cpp:97-101).
#include "device_math.cuh"

namespace gfb {
namespace {

constexpr int kTpb = 256;
#ifndef GF_NL_MINB
#define GF_NL_MINB 3  // 3 x 256 threads per SM (<= 80 registers): the non-local gathers are latency bound
#endif

__device__ __forceinline__ void load_tet_positions(const DevData& d, int4 t, double x[4][3], double du[9]) {
  const int id[4] = {t.x, t.y, t.z, t.w};
  double u[4][3];
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      u[k][a] = __ldg(d.u + 3 * (size_t)id[k] + a);
      x[k][a] = __ldg(d.X + 3 * (size_t)id[k] + a) + u[k][a];
    }
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int r = 0; r < 3; ++r) du[3 * r + c] = u[c + 1][r] - u[0][r];
}

__device__ __forceinline__ void scatter_max(const DevData& d, const int te[6], const double scr[6]) {
#pragma unroll
  for (int k = 0; k < 6; ++k) atomicMax(d.scr_key + te[k], dkey(scr[k]));
}

#ifndef GF_NC_WARPS
#define GF_NC_WARPS 4  // cell-template warps per CTA (each with its own weight ring)
#endif
#ifndef GF_NC_MINB
#define GF_NC_MINB 3
#endif
#ifndef GF_TS_MINB
#define GF_TS_MINB 3  // 3 x 256 threads per SM (80 registers): measured faster than 2 at c3 and c4
#endif
__global__ void __launch_bounds__(kTpb, GF_TS_MINB) k_tet_stress(DevData d, MatDev m, int local_screen) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e == 0) *d.newly_count = 0;  // this pass's relabel compacts from zero (stream order: tet_stress first)
  if (e >= d.nt) return;
  const int4 t = __ldg(d.tets + e);
  double x[4][3], du[9], B[9], F[9], P[9], c6[6];
  load_tet_positions(d, t, x, du);
  double vol;
  load_rest(d, e, B, vol);
  def_grad(du, B, F);
  const double J = pk1(F, m, P);
  cauchy6(F, P, J, c6);
  if (d.nl_tpl) {  // cell-major double2 planes (see DevData::nl_tpl)
    double2* s2 = reinterpret_cast<double2*>(d.sigc);
    const size_t pos = (size_t)(e % 6) * d.nl_ncell + e / 6;
#pragma unroll
    for (int p = 0; p < 3; ++p) s2[(size_t)p * d.nt + pos] = make_double2(c6[2 * p], c6[2 * p + 1]);
    if (d.nl_tpl == 2) {  // a non-finite component (exponent all ones) sends the gather kernel down its exact path
      int fin = 0x7ff00000;
#pragma unroll
      for (int k = 0; k < 6; ++k) fin = min(fin, ~__double2hiint(c6[k]) & 0x7ff00000);
      if (fin == 0) *d.nl_flag = 1;
    }
  } else {
#pragma unroll
    for (int k = 0; k < 6; ++k) d.sigc[6 * (size_t)e + k] = c6[k];
  }

  // build_T (fracture.cpp:16-28) and T sigma_c (fracture.cpp:74) row by row: each row's operations in build_T's
  // and matvec6's order, without materialising T (fewer live registers); outputs only after every row passed
  // the degeneracy test, as build_T's early return implies
  int te[6];
  double sf[6], scr[6], avg[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) avg[k] = 0.0 + 1.0 * c6[k];  // r_d = 0: table {(e, 1.0)} -> avg = 0 + 1.0 sigma_c
  bool ok = true;
  constexpr int le[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    // std::max(1.0, rest length) is 1.0 for every edge unless some rest length exceeds 1 (flag set at setup): the
    // scattered rest-length gathers -- and, with the non-local table, the edge ids -- are then not needed here
    te[k] = (local_screen || d.rest_len_gt1) ? __ldg(d.tet_edges + 6 * (size_t)e + k) : 0;
    const double rl = d.rest_len_gt1 ? __ldg(d.rest_len + te[k]) : 0.0;
    const double dx = x[le[k][1]][0] - x[le[k][0]][0];
    const double dy = x[le[k][1]][1] - x[le[k][0]][1];
    const double dz = x[le[k][1]][2] - x[le[k][0]][2];
    const double len = sqrt((dx * dx + dy * dy) + dz * dz);
    const double mx = (1.0 < rl) ? rl : 1.0;  // std::max(1.0, rl)
    ok = ok && !(len < 1e-14 * mx);
    const double nx = dx / len, ny = dy / len, nz = dz / len;
    const double row[6] = {nx * nx, ny * ny, nz * nz, nx * ny, nx * nz, ny * nz};
    double a = row[0] * c6[0];
#pragma unroll
    for (int j = 1; j < 6; ++j) a = a + row[j] * c6[j];
    sf[k] = a;
    if (local_screen) {
      double b = row[0] * avg[0];
#pragma unroll
      for (int j = 1; j < 6; ++j) b = b + row[j] * avg[j];
      scr[k] = b;
    }
  }
  d.deg[e] = ok ? 0 : 1;
#pragma unroll
  for (int k = 0; k < 6; ++k) d.sigf[6 * (size_t)e + k] = ok ? sf[k] : 0.0;  // degenerate: tet_edge_stress stays Zero
  if (ok && local_screen) scatter_max(d, te, scr);
}

// screened values of one non-degenerate tet, T * avg (fracture.cpp:77), max-reduced into its edges
// (fracture.cpp:80-87): build_T + matvec6 row by row -- the same operations in the same order, without
// materialising T (fewer live registers in the gather kernels) and without the degeneracy test, which
// k_tet_stress already made with identical arithmetic (deg[e])
__device__ __forceinline__ void screen_tet(const DevData& d, int e, const double avg[6]) {
  const int4 t = __ldg(d.tets + e);
  const int id[4] = {t.x, t.y, t.z, t.w};
  double x[4][3];
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int a = 0; a < 3; ++a) x[k][a] = __ldg(d.X + 3 * (size_t)id[k] + a) + __ldg(d.u + 3 * (size_t)id[k] + a);
  constexpr int le[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    const double dx = x[le[k][1]][0] - x[le[k][0]][0];
    const double dy = x[le[k][1]][1] - x[le[k][0]][1];
    const double dz = x[le[k][1]][2] - x[le[k][0]][2];
    const double len = sqrt((dx * dx + dy * dy) + dz * dz);
    const double nx = dx / len, ny = dy / len, nz = dz / len;
    double acc = (nx * nx) * avg[0];
    acc = acc + (ny * ny) * avg[1];
    acc = acc + (nz * nz) * avg[2];
    acc = acc + (nx * ny) * avg[3];
    acc = acc + (nx * nz) * avg[4];
    acc = acc + (ny * nz) * avg[5];
    atomicMax(d.scr_key + __ldg(d.tet_edges + 6 * (size_t)e + k), dkey(acc));
  }
}

__global__ void __launch_bounds__(kTpb, GF_NL_MINB) k_nonlocal(DevData d) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= d.nt) return;
  if (d.deg[e]) return;
  // avg = sum_q w_q * sigma_c[o_q], strictly in table order (fracture.cpp:75-76); coalesced sliced-ELL reads
  double avg[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  const int64_t base = __ldg(d.nl_sptr + (e >> 5)) * 32 + (e & 31);
  const int len = __ldg(d.nl_len + e);
  for (int j = 0; j < len; ++j) {
    const int64_t q = base + 32 * (int64_t)j;
    const double w = __ldg(d.nl_w + q);
    const double2* so = reinterpret_cast<const double2*>(d.sigc + 6 * (size_t)__ldg(d.nl_ids + q));
    const double2 s01 = __ldg(so), s23 = __ldg(so + 1), s45 = __ldg(so + 2);
    avg[0] = avg[0] + w * s01.x;
    avg[1] = avg[1] + w * s01.y;
    avg[2] = avg[2] + w * s23.x;
    avg[3] = avg[3] + w * s23.y;
    avg[4] = avg[4] + w * s45.x;
    avg[5] = avg[5] + w * s45.y;
  }
  screen_tet(d, e, avg);  // non-degenerate (checked by k_tet_stress with identical arithmetic)
}

// structured layout: warp = template warp (DevData::nl_tpl); same sums in the same order as k_nonlocal
#ifndef GF_NL_TPB
#define GF_NL_TPB 384  // two 32-cell ranges x six residues per CTA
#endif
constexpr int kNlTpb = GF_NL_TPB;
#ifndef GF_NL_PRED
#define GF_NL_PRED 1
#endif
  // template warps per CTA x 32
__global__ void __launch_bounds__(kNlTpb, (GF_NL_MINB * 256) / kNlTpb) k_nonlocal_tpl(DevData d) {
  const int wid = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (wid >= d.nl_nwarps) return;
  const int4 info = __ldg(d.nl_warp + wid);
  if (lane >= info.z) return;
  const int e = 6 * (info.y + lane) + info.x;
  if (d.deg[e]) return;
  const int j0 = info.w, j1 = __ldg(&d.nl_warp[wid + 1].w);
  const double2* s2 = reinterpret_cast<const double2*>(d.sigc);
  const size_t plane = (size_t)d.nt;
  double avg[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  // loads are unconditional (absent slots read lane 0's record of plane position 0, one L1 line) so consecutive
  // slots pipeline; an absent slot leaves avg untouched (a predicated add, not a multiply-add: exact whatever it read).
  // Gathering at the template position regardless of the weight was measured slower.
#pragma unroll 4
  for (int j = j0; j < j1; ++j) {
    const double w = __ldcs(d.nl_tw + (size_t)j * 32 + lane);
    const bool present = w != 0.0;
    const size_t pos = present ? (size_t)__ldg(d.nl_spos + j) + lane : 0;
    const double2 s01 = __ldg(s2 + pos), s23 = __ldg(s2 + plane + pos), s45 = __ldg(s2 + 2 * plane + pos);
#if GF_NL_PRED
    if (present) {  // predicated adds: half the instructions of per-component selects
      avg[0] = avg[0] + w * s01.x;
      avg[1] = avg[1] + w * s01.y;
      avg[2] = avg[2] + w * s23.x;
      avg[3] = avg[3] + w * s23.y;
      avg[4] = avg[4] + w * s45.x;
      avg[5] = avg[5] + w * s45.y;
    }
#else
    avg[0] = present ? avg[0] + w * s01.x : avg[0];
    avg[1] = present ? avg[1] + w * s01.y : avg[1];
    avg[2] = present ? avg[2] + w * s23.x : avg[2];
    avg[3] = present ? avg[3] + w * s23.y : avg[3];
    avg[4] = present ? avg[4] + w * s45.x : avg[4];
    avg[5] = present ? avg[5] + w * s45.y : avg[5];
#endif
  }
  screen_tet(d, e, avg);
}

// ---- cell template (DevData::nl_tpl == 2): one thread owns G tets of a cell (G = 3 by default) ---------------
// A warp covers G residues of 32 consecutive cells; its slots are the union over lanes AND its residues of the
// neighbour offsets D = o - 6 q in ascending order, so each of a thread's G sums still runs in table order. One
// gathered sigma record (48 B per lane, three coalesced 512-byte reads per warp) feeds up to G sums instead of one:
// the L1 wavefronts per (tet, neighbour) fall ~2.3x at G = 3 -- they were the limiter of the per-tet template. The
// weights -- one 32-lane vector per (slot, residue) present in the slot's mask, stored in exactly the order the
// warp consumes them -- are the kernel's only DRAM stream: each warp pulls its own stream through a shared-memory
// ring with cp.async.bulk + mbarrier (kNcStages copies of kNcVec vectors, two in flight beyond the one being
// consumed), so the stream depends neither on registers nor on the warp's scoreboard. Measured design steps and
// rejected variants: DESIGN.md §7.
constexpr int kNcWarps = GF_NC_WARPS;
#ifndef GF_NC_WPIPE
#define GF_NC_WPIPE 1  // weights one slot ahead of the sums in registers
#endif
#ifndef GF_NC_RING
#define GF_NC_RING 1  // weights through the cp.async.bulk shared-memory ring (0: straight into registers + L2 prefetch)
#endif
#ifndef GF_NC_AHEAD
#define GF_NC_AHEAD 2
#endif
#ifndef GF_NC_DEPTH
#define GF_NC_DEPTH 3  // sigma gather buffers (register pipeline depth)
#endif
#ifndef GF_NC_VEC
#define GF_NC_VEC 8
#endif
#ifndef GF_NC_STAGES
#define GF_NC_STAGES 4
#endif
constexpr int kNcVec = GF_NC_VEC;  // weight vectors (256 B each) per bulk copy (sim.cu pads each stream to 16)
constexpr int kNcStages = GF_NC_STAGES;  // ring depth in copies (4 x 2 KB = 8 KB per warp)
constexpr uint32_t kNcCopyBytes = kNcVec * 256;
constexpr uint32_t kNcRingBytes = kNcStages * kNcCopyBytes;
static_assert((kNcRingBytes & (kNcRingBytes - 1)) == 0, "ring size must be a power of two");

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void nc_copy(uint32_t dst, const double* src, uint32_t bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(kNcCopyBytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(kNcCopyBytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void nc_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tNC_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@p bra NC_DONE;\n\tbra NC_WAIT;\n\tNC_DONE:\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// a += w * s where w != 0, as a predicated multiply and add (mul.rn + add.rn: no contraction, the oracle's two
// roundings); the compiler turns the equivalent C++ `if` over six components into a divergent branch per residue
__device__ __forceinline__ void nc_add(double& a, int nz, double w, double s) {
  asm("{\n\t.reg .pred p;\n\t.reg .f64 t;\n\tsetp.ne.s32 p, %1, 0;\n\tmul.rn.f64 t, %2, %3;\n\t@p add.rn.f64 %0, %0, t;\n\t}"
      : "+d"(a)
      : "r"(nz), "d"(w), "d"(s));
}
__device__ __forceinline__ void nc_accumulate(double (&a)[6], double w, double2 s01, double2 s23, double2 s45) {
  const int nz = (__double2hiint(w) << 1) | __double2loint(w);  // w != 0.0 (true for NaN too, like the C++ test)
  nc_add(a[0], nz, w, s01.x);
  nc_add(a[1], nz, w, s01.y);
  nc_add(a[2], nz, w, s23.x);
  nc_add(a[3], nz, w, s23.y);
  nc_add(a[4], nz, w, s45.x);
  nc_add(a[5], nz, w, s45.y);
}

// EXACT = false: the sums add w * sigma for every lane, a zero weight included -- bit-identical to skipping it while
// every gathered sigma is finite (avg + (+-0) = avg, and avg is never -0). k_tet_stress raises *nl_flag when it
// writes a non-finite sigma component; that sends the kernel down its EXACT = true twin (selects keep avg
// where w = 0, whatever was gathered); the kernel takes the twin the flag picks (one warp-uniform branch).
template <int G, bool EXACT>  // G residues per thread: the warp owns residues [g G, g G + G) of its 32 cells
__device__ __forceinline__ void nonlocal_cell_warp(const DevData& d, double (*ring)[kNcRingBytes / 8],
                                                   unsigned long long (*bars)[kNcStages]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wid = blockIdx.x * kNcWarps + warp;
  if (wid >= d.nl_nwarps) return;  // warps are independent: no CTA-wide barrier below
  const int4 info = __ldg(d.nl_warp + wid), next = __ldg(d.nl_warp + wid + 1);
  const int s0 = info.z, s1 = next.z;
  const int ncopies = (next.w - info.w) / kNcVec;
  const double* wsrc = d.nl_tw + (size_t)info.w * 32;
  const uint32_t ring0 = smem_addr(&ring[warp][0]), bar0 = smem_addr(&bars[warp][0]);
  if (lane == 0) {
#pragma unroll
    for (int c = 0; c < kNcStages; ++c) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8 * c));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#pragma unroll
    for (int c = 0; c < kNcStages - 2; ++c)
      if (c < ncopies) nc_copy(ring0 + c * kNcCopyBytes, wsrc + (size_t)c * kNcVec * 32, bar0 + 8 * c);
  }
  __syncwarp();
  const double2* s2 = reinterpret_cast<const double2*>(d.sigc);
  const int plane = d.nt, last = d.nt - 1;
  const int2* slots = d.nl_cslot;
  double avg[G][6];
#pragma unroll
  for (int t = 0; t < G; ++t)
#pragma unroll
    for (int k = 0; k < 6; ++k) avg[t][k] = 0.0;
  const uint32_t lane_base = ring0 + (uint32_t)(lane * 8);
  uint32_t off = 0;  // byte offset of the next weight vector in the warp's stream
  int cready = -1;   // last copy waited for
  // Software pipeline over slots, three sigma buffers deep: in the step of slot j the record of slot j + 3 is
  // requested (one uniform 8-byte load), the gathers of slot j + 2 are issued from the record requested one step
  // earlier, and slot j (gathered two steps earlier) is consumed. Indices past the end repeat the last slot
  // (harmless loads). A lane whose neighbour does not exist (mesh boundary, short last range) gathers a clamped
  // position: its weight is 0.
  auto record = [&](int j) { return __ldg(slots + max(min(j, s1 - 1), s0)); };  // (one pad record ends the array)
  auto gather = [&](int2 rec, double2& a, double2& b, double2& c) {
    const int p = min(max(rec.x + lane, 0), last);
    a = __ldg(s2 + p), b = __ldg(s2 + plane + p), c = __ldg(s2 + 2 * plane + p);
  };
  // the weights of a slot from the ring into registers, without branches over the residues (an absent (slot,
  // residue) has no vector and reads as 0, like a lane that lacks this neighbour)
  auto loadw = [&](int mask, double (&w)[G]) {
    // the slot's <= G (< kNcVec) vectors lie in copies cl - 1 and cl: on first touching copy cl, the stage of copy
    // cl - 2 is free (fully consumed; never used for cl < 2) and takes copy cl + kNcStages - 2
    const int cl = (int)((off + 256u * (uint32_t)__popc(mask) - 256u) / kNcCopyBytes);
    if (mask != 0 && cl > cready) {
      cready = cl;
      __syncwarp();
      const int cn = cl + kNcStages - 2;
      if (lane == 0 && cn < ncopies) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        nc_copy(ring0 + (cn % kNcStages) * kNcCopyBytes, wsrc + (size_t)cn * kNcVec * 32, bar0 + 8 * (cn % kNcStages));
      }
      nc_wait(bar0 + 8 * (cl % kNcStages), (uint32_t)((cl / kNcStages) & 1));
    }
#pragma unroll
    for (int t = 0; t < G; ++t) {
      const bool has = (mask >> t) & 1;
      w[t] = 0.0;
      if (has) asm volatile("ld.shared.f64 %0, [%1];" : "=d"(w[t]) : "r"(lane_base + (off & (kNcRingBytes - 1))));
      off += has ? 256u : 0u;
    }
  };
  auto sums = [&](const double (&w)[G], const double2& s01, const double2& s23, const double2& s45) {
#pragma unroll
    for (int t = 0; t < G; ++t) {
      if (EXACT) {
        nc_accumulate(avg[t], w[t], s01, s23, s45);
      } else {
        avg[t][0] = avg[t][0] + w[t] * s01.x;
        avg[t][1] = avg[t][1] + w[t] * s01.y;
        avg[t][2] = avg[t][2] + w[t] * s23.x;
        avg[t][3] = avg[t][3] + w[t] * s23.y;
        avg[t][4] = avg[t][4] + w[t] * s45.x;
        avg[t][5] = avg[t][5] + w[t] * s45.y;
      }
    }
  };
#if GF_NC_WPIPE
  // the weights run one slot ahead of the sums in registers: the shared-memory loads of slot j + 1 are issued before
  // the sums of slot j (mask 0 past the end: no loads, no ring progress)
  double2 a01, a23, a45, b01, b23, b45, c01, c23, c45;
  double wa[G], wb[G], wc[G];
  int2 rec = record(s0);
  int mb, mc;
  gather(rec, a01, a23, a45);
  loadw(rec.y, wa);
  rec = record(s0 + 1);
  mb = s0 + 1 < s1 ? rec.y : 0;
  gather(rec, b01, b23, b45);
  rec = record(s0 + 2);
  for (int j = s0; j < s1; j += 3) {
    int2 nrec = record(j + 3);
    mc = j + 2 < s1 ? rec.y : 0;
    gather(rec, c01, c23, c45);
    loadw(mb, wb);
    sums(wa, a01, a23, a45);
    if (j + 1 >= s1) break;
    rec = record(j + 4);
    const int ma = j + 3 < s1 ? nrec.y : 0;
    gather(nrec, a01, a23, a45);
    loadw(mc, wc);
    sums(wb, b01, b23, b45);
    if (j + 2 >= s1) break;
    nrec = record(j + 5);
    mb = j + 4 < s1 ? rec.y : 0;
    gather(rec, b01, b23, b45);
    loadw(ma, wa);
    sums(wc, c01, c23, c45);
    rec = nrec;
  }
#else
  auto consume = [&](int mask, const double2& s01, const double2& s23, const double2& s45) {
    double w[G];
    loadw(mask, w);
    sums(w, s01, s23, s45);
  };
#if GF_NC_DEPTH == 2
  double2 a01, a23, a45, b01, b23, b45;
  int2 rec = record(s0);
  int ma = rec.y, mb;
  gather(rec, a01, a23, a45);
  rec = record(s0 + 1);
  for (int j = s0; j < s1; j += 2) {  // two buffers: the gathers of slot j + 1 fly while slot j is summed
    int2 nrec = record(j + 2);
    mb = rec.y;
    gather(rec, b01, b23, b45);
    consume(ma, a01, a23, a45);
    if (j + 1 >= s1) break;
    rec = record(j + 3);
    ma = nrec.y;
    gather(nrec, a01, a23, a45);
    consume(mb, b01, b23, b45);
  }
#else
  double2 a01, a23, a45, b01, b23, b45, c01, c23, c45;
  int2 rec = record(s0);
  int ma = rec.y, mb, mc;
  gather(rec, a01, a23, a45);
  rec = record(s0 + 1);
  mb = rec.y;
  gather(rec, b01, b23, b45);
  rec = record(s0 + 2);
  for (int j = s0; j < s1; j += 3) {
    int2 nrec = record(j + 3);
    mc = rec.y;
    gather(rec, c01, c23, c45);
    consume(ma, a01, a23, a45);
    if (j + 1 >= s1) break;
    rec = record(j + 4);
    ma = nrec.y;
    gather(nrec, a01, a23, a45);
    consume(mb, b01, b23, b45);
    if (j + 2 >= s1) break;
    nrec = record(j + 5);
    mb = rec.y;
    gather(rec, b01, b23, b45);
    consume(mc, c01, c23, c45);
    rec = nrec;
  }
#endif
#endif  // GF_NC_WPIPE
  if (lane >= (info.y & 255)) return;
#pragma unroll
  for (int t = 0; t < G; ++t) {
    const int e = 6 * (info.x + lane) + (info.y >> 8) * G + t;
    if (!d.deg[e]) screen_tet(d, e, avg[t]);
  }
}

// Ring-free variant (GF_NC_RING=0): the weights are loaded straight into registers (coalesced streaming loads, issued
// with the slot's gathers, GF_NC_DEPTH - 1 slots ahead of their use) and the DRAM latency is taken by L2 prefetches
// that run kNcAhead 4-KB chunks ahead of the loads (one prefetch instruction per chunk: each lane one 128-byte
// line). No shared memory, no mbarrier bookkeeping.
constexpr int kNcAhead = GF_NC_AHEAD;
template <int G, bool EXACT>
__device__ __forceinline__ void nonlocal_cell_direct(const DevData& d) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wid = blockIdx.x * kNcWarps + warp;
  if (wid >= d.nl_nwarps) return;
  const int4 info = __ldg(d.nl_warp + wid), next = __ldg(d.nl_warp + wid + 1);
  const int s0 = info.z, s1 = next.z;
  const double* wp = d.nl_tw + (size_t)info.w * 32 + lane;  // this lane's entry of the next weight vector
  const char* const pf0 = reinterpret_cast<const char*>(d.nl_tw + (size_t)info.w * 32) + 128 * lane;
  const char* const pfend = reinterpret_cast<const char*>(d.nl_tw + (size_t)__ldg(&d.nl_warp[d.nl_nwarps].w) * 32);
  auto prefetch = [&](int chunk) {
    const char* p = pf0 + ((size_t)chunk << 12);
    if (p < pfend) asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
  };
#pragma unroll
  for (int c = 0; c <= kNcAhead; ++c) prefetch(c);
  const double2* s2 = reinterpret_cast<const double2*>(d.sigc);
  const int plane = d.nt, last = d.nt - 1;
  const int2* slots = d.nl_cslot;
  double avg[G][6];
#pragma unroll
  for (int t = 0; t < G; ++t)
#pragma unroll
    for (int k = 0; k < 6; ++k) avg[t][k] = 0.0;
  uint32_t off = 0;  // bytes of the warp's weight stream requested so far
  int cdone = 0;     // chunks up to cdone + kNcAhead are prefetched
  auto record = [&](int j) { return __ldg(slots + max(min(j, s1 - 1), s0)); };
  // the gathers of a slot and its weights (an absent (slot, residue) has no vector and reads as 0)
  auto fetch = [&](int2 rec, bool live, double2& a, double2& b, double2& c, double (&w)[G]) {
    const int p = min(max(rec.x + lane, 0), last);
    a = __ldg(s2 + p), b = __ldg(s2 + plane + p), c = __ldg(s2 + 2 * plane + p);
    const int mask = live ? rec.y : 0;  // slots past the end are repeated for their (unused) gathers only
#pragma unroll
    for (int t = 0; t < G; ++t) {
      const bool has = (mask >> t) & 1;
      w[t] = 0.0;
      if (has) w[t] = __ldcs(wp);
      wp += has ? 32 : 0;
    }
    off += 256u * (uint32_t)__popc(mask);
    const int c4 = (int)(off >> 12);
    if (c4 > cdone) {
      cdone = c4;
      prefetch(c4 + kNcAhead);
    }
  };
  auto consume = [&](const double (&w)[G], const double2& s01, const double2& s23, const double2& s45) {
#pragma unroll
    for (int t = 0; t < G; ++t) {
      if (EXACT) {
        nc_accumulate(avg[t], w[t], s01, s23, s45);
      } else {
        avg[t][0] = avg[t][0] + w[t] * s01.x;
        avg[t][1] = avg[t][1] + w[t] * s01.y;
        avg[t][2] = avg[t][2] + w[t] * s23.x;
        avg[t][3] = avg[t][3] + w[t] * s23.y;
        avg[t][4] = avg[t][4] + w[t] * s45.x;
        avg[t][5] = avg[t][5] + w[t] * s45.y;
      }
    }
  };
#if GF_NC_DEPTH == 2
  double2 a01, a23, a45, b01, b23, b45;
  double wa[G], wb[G];
  fetch(record(s0), true, a01, a23, a45, wa);
  int2 rec = record(s0 + 1);
  for (int j = s0; j < s1; j += 2) {
    int2 nrec = record(j + 2);
    fetch(rec, j + 1 < s1, b01, b23, b45, wb);
    consume(wa, a01, a23, a45);
    if (j + 1 >= s1) break;
    rec = record(j + 3);
    fetch(nrec, j + 2 < s1, a01, a23, a45, wa);
    consume(wb, b01, b23, b45);
  }
#else
  double2 a01, a23, a45, b01, b23, b45, c01, c23, c45;
  double wa[G], wb[G], wc[G];
  fetch(record(s0), true, a01, a23, a45, wa);
  fetch(record(s0 + 1), s0 + 1 < s1, b01, b23, b45, wb);
  int2 rec = record(s0 + 2);
  for (int j = s0; j < s1; j += 3) {
    int2 nrec = record(j + 3);
    fetch(rec, j + 2 < s1, c01, c23, c45, wc);
    consume(wa, a01, a23, a45);
    if (j + 1 >= s1) break;
    rec = record(j + 4);
    fetch(nrec, j + 3 < s1, a01, a23, a45, wa);
    consume(wb, b01, b23, b45);
    if (j + 2 >= s1) break;
    nrec = record(j + 5);
    fetch(rec, j + 4 < s1, b01, b23, b45, wb);
    consume(wc, c01, c23, c45);
    rec = nrec;
  }
#endif
  if (lane >= (info.y & 255)) return;
#pragma unroll
  for (int t = 0; t < G; ++t) {
    const int e = 6 * (info.x + lane) + (info.y >> 8) * G + t;
    if (!d.deg[e]) screen_tet(d, e, avg[t]);
  }
}

template <int G>
__global__ void __launch_bounds__(32 * kNcWarps, G == 6 ? GF_NC_MINB : G == 3 ? GF_NC_MINB + 1 : GF_NC_MINB + 2)
    k_nonlocal_cell(DevData d) {
#if GF_NC_RING
  __shared__ __align__(128) double ring[kNcWarps][kNcRingBytes / 8];
  __shared__ __align__(8) unsigned long long bars[kNcWarps][kNcStages];
  if (*d.nl_flag != 0) nonlocal_cell_warp<G, true>(d, ring, bars);
  else nonlocal_cell_warp<G, false>(d, ring, bars);
#else
  if (*d.nl_flag != 0) nonlocal_cell_direct<G, true>(d);
  else nonlocal_cell_direct<G, false>(d);
#endif
}

__global__ void __launch_bounds__(kTpb) k_relabel(DevData d, double thres, int relabel, int keep_values) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  bool broke = false;
  if (i < d.ne) {
    const unsigned long long key = d.scr_key[i];
    const double s = (key == kKeyNegInf) ? 0.0 : dkey_inv(key);
    if (keep_values) d.screening[i] = s;
    d.scr_key[i] = kKeyNegInf;
    if (i == 0 && d.nl_tpl == 2) *d.nl_flag = 0;  // this pass's gathers are done (stream order)
    if (relabel && !d.zeta[i] && s >= thres) {
      d.zeta[i] = 1;
      broke = true;
    }
  }
  const unsigned mask = __ballot_sync(0xffffffffu, broke);
  if (mask == 0) return;
  const int lane = threadIdx.x & 31;
  int base = 0;
  if (lane == 0) base = atomicAdd(d.newly_count, __popc(mask));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (broke) d.newly[base + __popc(mask & ((1u << lane) - 1u))] = i;
}

__global__ void __launch_bounds__(kTpb) k_chi(DevData d, MatDev m) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= d.nt) return;
  int te[6];
  bool dmg[6];
  int intact = 0;
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    te[k] = __ldg(d.tet_edges + 6 * (size_t)e + k);
    dmg[k] = d.zeta[te[k]] != 0;
    intact += dmg[k] ? 0 : 1;
  }
  double value;
  if (d.deg[e]) {
    value = 0.0;
  } else if (intact == 6) {
    value = 1.0;
  } else if (intact == 0) {
    value = 0.0;
  } else {
    constexpr int le[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
    int label[4] = {0, 1, 2, 3};
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      if (dmg[k]) continue;
      int a = le[k][0], b = le[k][1];
      while (label[a] != a) a = label[a];
      while (label[b] != b) b = label[b];
      if (a != b) label[a > b ? a : b] = a < b ? a : b;
    }
    int comps = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int r = i;
      while (label[r] != r) r = label[r];
      comps += (r == i) ? 1 : 0;
    }
    if (comps >= 2) {
      value = 0.0;
    } else {
      double surviving = 0.0, total = 0.0;
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        const double s = fabs(d.sigf[6 * (size_t)e + k]);
        total += s;
        if (!dmg[k]) surviving += s;
      }
      value = (total < m.chi_eps) ? (double)intact / 6.0 : surviving / total;
    }
  }
  const double old = d.chi[e];
  const double nv = std_min(old, value);
  if (__double_as_longlong(nv) != __double_as_longlong(old)) d.chi[e] = nv;
}

__global__ void k_reset_keys(unsigned long long* k, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) k[i] = kKeyNegInf;
}

inline int nblk(int64_t n) { return (int)((n + kTpb - 1) / kTpb); }

}  // namespace

void launch_tet_stress(const DevData& d, const MatDev& m, bool local_screen, cudaStream_t s) {
  k_tet_stress<<<nblk(d.nt), kTpb, 0, s>>>(d, m, local_screen ? 1 : 0);
}
void launch_nonlocal(const DevData& d, cudaStream_t s) {
  if (d.nl_tpl == 2) {
    const int grid = (d.nl_nwarps + kNcWarps - 1) / kNcWarps;
    switch (d.nl_group) {
#if GF_NC_VEC >= 8  // a slot's <= G vectors must be fewer than one copy's
      case 6: k_nonlocal_cell<6><<<grid, 32 * kNcWarps, 0, s>>>(d); break;
#endif
      case 3: k_nonlocal_cell<3><<<grid, 32 * kNcWarps, 0, s>>>(d); break;
      case 2: k_nonlocal_cell<2><<<grid, 32 * kNcWarps, 0, s>>>(d); break;
      default: k_nonlocal_cell<1><<<grid, 32 * kNcWarps, 0, s>>>(d); break;
    }
  }
  else if (d.nl_tpl) k_nonlocal_tpl<<<(int)((32 * (int64_t)d.nl_nwarps + kNlTpb - 1) / kNlTpb), kNlTpb, 0, s>>>(d);
  else k_nonlocal<<<nblk(d.nt), kTpb, 0, s>>>(d);
}
void launch_relabel(const DevData& d, double thres, bool relabel, bool keep_values, cudaStream_t s) {
  k_relabel<<<nblk(d.ne), kTpb, 0, s>>>(d, thres, relabel ? 1 : 0, keep_values ? 1 : 0);
}
void launch_chi(const DevData& d, const MatDev& m, cudaStream_t s) { k_chi<<<nblk(d.nt), kTpb, 0, s>>>(d, m); }
void launch_reset_keys(const DevData& d, cudaStream_t s) {
  k_reset_keys<<<nblk(d.ne), kTpb, 0, s>>>(d.scr_key, d.ne);
}

}  // namespace gfb
