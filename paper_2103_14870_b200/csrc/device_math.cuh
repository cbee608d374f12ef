// device_math.cuh — per-tet material math shared by the damage kernels (damage.cu, built with
// -fmad=false so every + and * below is a separately rounded IEEE op in the written order) and the
// assembly kernel (assemble.cu, FMA allowed: forces/matrix entries are held to 1e-9, not to bits).
//
// Operation orders are the contract with the CPU oracle (oracle/grafem_oracle.cpp header, rules R1,
// R2, R3, S9, N3 and the in-place symmetrisation of material.cpp:128); matrices are row-major [3r+c].
#pragma once

#include "dev_types.cuh"

namespace gfb {

#define GF_HD __host__ __device__ __forceinline__

// F = I + du * B^-1 (fem.cpp:22-31); du[3r+c] = (u_{c+1} - u_0)_r ; R1 product order
GF_HD void def_grad(const double du[9], const double B[9], double F[9]) {
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double c0 = (du[0] * B[c] + du[1] * B[3 + c]) + du[2] * B[6 + c];
    const double c1 = (du[3] * B[c] + du[4] * B[3 + c]) + du[5] * B[6 + c];
    const double c2 = du[6] * B[c] + (du[7] * B[3 + c] + du[8] * B[6 + c]);
    F[c] = (c == 0 ? 1.0 : 0.0) + c0;
    F[3 + c] = (c == 1 ? 1.0 : 0.0) + c1;
    F[6 + c] = (c == 2 ? 1.0 : 0.0) + c2;
  }
}

GF_HD double det3(const double m[9]) {  // bruteforce_det3_helper: (h0 - h1) + h2
  const double h0 = m[0] * (m[4] * m[8] - m[5] * m[7]);
  const double h1 = m[1] * (m[3] * m[8] - m[5] * m[6]);
  const double h2 = m[2] * (m[3] * m[7] - m[4] * m[6]);
  return (h0 - h1) + h2;
}

// S9 over the column-major linear order x0..x8 = F00,F10,F20,F01,F11,F21,F02,F12,F22
GF_HD double sqnorm9(const double F[9]) {
  const double l0 = (F[0] * F[0] + F[6] * F[6]) + (F[4] * F[4] + F[2] * F[2]);
  const double l1 = (F[3] * F[3] + F[1] * F[1]) + (F[7] * F[7] + F[5] * F[5]);
  return (l0 + l1) + F[8] * F[8];
}

// cofactor (material.cpp:48-54): column c = F.col(c+1) x F.col(c+2)
GF_HD void cofactor(const double F[9], double C[9]) {
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const int a = (c + 1) % 3, b = (c + 2) % 3;
    C[0 * 3 + c] = F[3 + a] * F[6 + b] - F[6 + a] * F[3 + b];
    C[1 * 3 + c] = F[6 + a] * F[0 + b] - F[0 + a] * F[6 + b];
    C[2 * 3 + c] = F[0 + a] * F[3 + b] - F[3 + a] * F[0 + b];
  }
}

// pk1 (material.cpp:86-95). Returns J = det F as a by-product (NH) or computes it (StVK).
GF_HD double pk1(const double F[9], const MatDev& p, double P[9]) {
  const double J = det3(F);
  if (p.model == 1) {
    double E[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double ftf = (F[r] * F[c] + F[3 + r] * F[3 + c]) + F[6 + r] * F[6 + c];  // R2
        E[3 * r + c] = 0.5 * (ftf - (r == c ? 1.0 : 0.0));
      }
    const double s2mu = 2.0 * p.mu;
    const double lt = p.lambda * (E[0] + (E[4] + E[8]));
    double S[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) S[q] = s2mu * E[q] + lt * ((q % 4 == 0) ? 1.0 : 0.0);
#pragma unroll
    for (int c = 0; c < 3; ++c) {  // P = F S, R1
      P[c] = (F[0] * S[c] + F[1] * S[3 + c]) + F[2] * S[6 + c];
      P[3 + c] = (F[3] * S[c] + F[4] * S[3 + c]) + F[5] * S[6 + c];
      P[6 + c] = F[6] * S[c] + (F[7] * S[3 + c] + F[8] * S[6 + c]);
    }
    return J;
  }
  const double ic = sqnorm9(F);
  const double s1 = p.mu * (1.0 - 1.0 / (ic + 1.0));
  const double s2 = p.lambda * (J - p.alpha_nh);
  double C[9];
  cofactor(F, C);
#pragma unroll
  for (int q = 0; q < 9; ++q) P[q] = s1 * F[q] + s2 * C[q];
  return J;
}

// energy_density (material.cpp:71-84): StVK invariants of C = F^T F; stable NH with log(I_C + 1)
GF_HD double energy_density(const double F[9], const MatDev& m) {
  if (m.model == 1) {
    double Cm[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) Cm[3 * r + c] = F[r] * F[c] + F[3 + r] * F[3 + c] + F[6 + r] * F[6 + c];
    const double ic = Cm[0] + Cm[4] + Cm[8];
    double iic = 0.0;
#pragma unroll
    for (int q = 0; q < 9; ++q) iic += Cm[q] * Cm[q];
    return 0.125 * m.lambda * (ic - 3.0) * (ic - 3.0) + 0.25 * m.mu * (iic - 2.0 * ic + 3.0);
  }
  const double ic = sqnorm9(F);
  const double j = det3(F);
  return 0.5 * m.mu * (ic - 3.0) + 0.5 * m.lambda * (j - m.alpha_nh) * (j - m.alpha_nh) - 0.5 * m.mu * log(ic + 1.0);
}

// cartesian_stress_sixvector (material.cpp:121-135): sigma = P F^T / J (R1), then the Release-build
// in-place column-major symmetrisation of material.cpp:128; det F <= 0 falls back to sym(P).
GF_HD void cauchy6(const double F[9], const double P[9], double J, double c6[6]) {
  if (J > 0.0) {
    double s[9];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      s[c] = ((P[0] * F[3 * c] + P[1] * F[3 * c + 1]) + P[2] * F[3 * c + 2]) / J;
      s[3 + c] = ((P[3] * F[3 * c] + P[4] * F[3 * c + 1]) + P[5] * F[3 * c + 2]) / J;
      s[6 + c] = (P[6] * F[3 * c] + (P[7] * F[3 * c + 1] + P[8] * F[3 * c + 2])) / J;
    }
    // traversal (0,0),(1,0),(2,0),(0,1),(1,1),(2,1),(0,2),(1,2),(2,2), reading updated entries
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int r = 0; r < 3; ++r) s[3 * r + c] = 0.5 * (s[3 * r + c] + s[3 * c + r]);
    c6[0] = s[0]; c6[1] = s[4]; c6[2] = s[8];
    c6[3] = 2.0 * s[1]; c6[4] = 2.0 * s[2]; c6[5] = 2.0 * s[5];
  } else {
    c6[0] = 0.5 * (P[0] + P[0]);
    c6[1] = 0.5 * (P[4] + P[4]);
    c6[2] = 0.5 * (P[8] + P[8]);
    c6[3] = 2.0 * (0.5 * (P[1] + P[3]));
    c6[4] = 2.0 * (0.5 * (P[2] + P[6]));
    c6[5] = 2.0 * (0.5 * (P[5] + P[7]));
  }
}

// build_T (fracture.cpp:16-28) for one tet from the 4 current positions x[4][3]. Returns false on a
// degenerate edge (len < 1e-14 * max(1, rest length)).
GF_HD bool build_T(const double x[4][3], const double rl[6], double T[6][6]) {
  constexpr int le[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    const double dx = x[le[k][1]][0] - x[le[k][0]][0];
    const double dy = x[le[k][1]][1] - x[le[k][0]][1];
    const double dz = x[le[k][1]][2] - x[le[k][0]][2];
    const double len = sqrt((dx * dx + dy * dy) + dz * dz);
    const double m = (1.0 < rl[k]) ? rl[k] : 1.0;  // std::max(1.0, rl)
    if (len < 1e-14 * m) return false;
    const double nx = dx / len, ny = dy / len, nz = dz / len;
    T[k][0] = nx * nx; T[k][1] = ny * ny; T[k][2] = nz * nz;
    T[k][3] = nx * ny; T[k][4] = nx * nz; T[k][5] = ny * nz;
  }
  return true;
}

GF_HD void matvec6(const double T[6][6], const double s[6], double out[6]) {  // R3 sequential
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    double acc = T[k][0] * s[0];
#pragma unroll
    for (int j = 1; j < 6; ++j) acc = acc + T[k][j] * s[j];
    out[k] = acc;
  }
}

// std::max(a, b) / std::min(a, b) semantics (first argument kept on ties / NaN)
GF_HD double std_max(double a, double b) { return (a < b) ? b : a; }
GF_HD double std_min(double a, double b) { return (b < a) ? b : a; }

// order-preserving map of a double to an unsigned key (for atomicMax); monotone for non-NaN values
__device__ __forceinline__ unsigned long long dkey(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double dkey_inv(unsigned long long k) {
  const unsigned long long b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}
constexpr unsigned long long kKeyNegInf = 0x000fffffffffffffull;  // dkey(-inf) = ~0xfff0000000000000

}  // namespace gfb
