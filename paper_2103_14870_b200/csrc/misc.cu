// misc.cu — per-node kernels of dynamic_step (solver.cpp:229-330). Built with -fmad=false so the pinned
// boundary values and the u += dt*v update round exactly like the oracle.
//   k_bc_targets  prescribed dv / u(t+dt) / v(t+dt) of BC nodes (solver.cpp:255-262, 322-328)
//   k_collide     per-vertex penalty + impulse + Coulomb response (detect_and_respond, collision.cpp:49-111)
//                 on the substep probe u + tau v (solver.cpp:233-249), block partials for the load
//   k_integrate   v += dv, u += dt v, then pin BC nodes (solver.cpp:296-328); no-op unless the PCG converged
//   k_qs_bc / k_qs_update  quasi-static Newton helpers (solver.cpp:138-217; the dots are in metrics.cu)
//   k_shift_diag  shift_diagonal on the node-block matrix (solver.cpp:119-129 ladder)
#include "device_math.cuh"

namespace gfb {
namespace {

constexpr int kTpb = 256;
inline int nblk(int64_t n) { return (int)((n + kTpb - 1) / kTpb); }

__device__ __forceinline__ const double* diag_block(const DevData& d, int i) {  // entry q at [32 q]
  return d.bval + sell_addr(d.usp, i, 0, 0);  // the diagonal is the first upper block of its row
}

__device__ __forceinline__ void bc_disp(const BcStep& b, const double* X, const double* R, const double* d,
                                        double out[3]) {
  if (b.kind == 0) {
    out[0] = d[0];
    out[1] = d[1];
    out[2] = d[2];
    return;
  }
  const double rel[3] = {X[0] - b.axis_point[0], X[1] - b.axis_point[1], X[2] - b.axis_point[2]};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double rr = (R[3 * a] * rel[0] + R[3 * a + 1] * rel[1]) + R[3 * a + 2] * rel[2];
    out[a] = (rr + b.axis_point[a]) - X[a];
  }
}

__global__ void k_bc_targets(DevData d, int n_fixed, const int32_t* fixed_nodes, double dt) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n_fixed) return;
  const int i = fixed_nodes[q];
  const BcStep& b = d.bcstep[d.node_bc[i]];
  const double* X = d.X + 3 * (size_t)i;
  double d0[3], d1[3];
  bc_disp(b, X, b.R0, b.d0, d0);
  bc_disp(b, X, b.R1, b.d1, d1);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double vt = (d1[a] - d0[a]) / dt;
    d.fv[3 * (size_t)i + a] = vt - d.v[3 * (size_t)i + a];
    d.utgt[3 * (size_t)i + a] = d1[a];
    d.vtgt[3 * (size_t)i + a] = vt;
  }
}

// one launch per substep; colliders for this substep at d.colliders[0..n)
__global__ void __launch_bounds__(kTpb) k_collide(DevData d, double tau, double dt, double sub, int first,
                                                  const ColliderDev* cols, double* partials) {
  __shared__ double s[kTpb / 32][8][3];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double fsum_c[8][3];
  for (int c = 0; c < 8; ++c) fsum_c[c][0] = fsum_c[c][1] = fsum_c[c][2] = 0.0;
  if (i < d.nn) {
    double x[3], v[3], ftot[3] = {0.0, 0.0, 0.0};
    for (int a = 0; a < 3; ++a) {
      const double u = d.u[3 * (size_t)i + a];
      v[a] = d.v[3 * (size_t)i + a];
      const double up = (tau != 0.0) ? u + tau * v[a] : u;
      x[a] = d.X[3 * (size_t)i + a] + up;
    }
    const double mi = d.mass[i];
    for (int c = 0; c < d.n_colliders && c < 8; ++c) {
      const ColliderDev& col = cols[c];
      double depth, nrm[3];
      if (col.kind == 0) {
        const double rel[3] = {x[0] - col.center[0], x[1] - col.center[1], x[2] - col.center[2]};
        const double dist = sqrt((rel[0] * rel[0] + rel[1] * rel[1]) + rel[2] * rel[2]);
        depth = col.radius - dist;
        if (depth <= 0.0) continue;
        if (dist > 1e-12) {
          nrm[0] = rel[0] / dist; nrm[1] = rel[1] / dist; nrm[2] = rel[2] / dist;
        } else {
          nrm[0] = 0.0; nrm[1] = 0.0; nrm[2] = 1.0;
        }
      } else {
        const double rel[3] = {x[0] - col.point[0], x[1] - col.point[1], x[2] - col.point[2]};
        depth = -((rel[0] * col.normal[0] + rel[1] * col.normal[1]) + rel[2] * col.normal[2]);
        if (depth <= 0.0) continue;
        nrm[0] = col.normal[0]; nrm[1] = col.normal[1]; nrm[2] = col.normal[2];
      }
      const double kd = col.stiffness * depth;
      double f[3] = {kd * nrm[0], kd * nrm[1], kd * nrm[2]};
      const double vr[3] = {v[0] - col.cvel[0], v[1] - col.cvel[1], v[2] - col.cvel[2]};
      const double vn = (vr[0] * nrm[0] + vr[1] * nrm[1]) + vr[2] * nrm[2];
      double imp = 0.0;
      if (vn < 0.0) {
        imp = -(1.0 + col.restitution) * vn * mi / dt;
        for (int a = 0; a < 3; ++a) f[a] += imp * nrm[a];
      }
      if (col.friction > 0.0) {
        const double vt[3] = {vr[0] - vn * nrm[0], vr[1] - vn * nrm[1], vr[2] - vn * nrm[2]};
        const double vtn = sqrt((vt[0] * vt[0] + vt[1] * vt[1]) + vt[2] * vt[2]);
        if (vtn > 1e-12) {
          const double cap = col.friction * (kd + imp);
          const double want = mi * vtn / dt;
          const double mag = (want < cap) ? want : cap;  // std::min(cap, want)
          for (int a = 0; a < 3; ++a) f[a] -= mag * (vt[a] / vtn);
        }
      }
      for (int a = 0; a < 3; ++a) {
        ftot[a] += f[a];
        fsum_c[c][a] = f[a];
      }
    }
    for (int a = 0; a < 3; ++a) {
      const double add = ftot[a] / sub;  // collision += hit.force / sub
      d.fcoll[3 * (size_t)i + a] = first ? 0.0 + add : d.fcoll[3 * (size_t)i + a] + add;
    }
  }
  // per-collider block partial of the force vector sum (load metric)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nc = d.n_colliders < 8 ? d.n_colliders : 8;
  for (int c = 0; c < nc; ++c)
    for (int a = 0; a < 3; ++a) {
      double x = fsum_c[c][a];
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (lane == 0) s[w][c][a] = x;
    }
  __syncthreads();
  if (threadIdx.x < 3 * nc) {
    const int c = threadIdx.x / 3, a = threadIdx.x % 3;
    double x = 0.0;
    for (int k = 0; k < kTpb / 32; ++k) x += s[k][c][a];
    partials[((size_t)c * 3 + a) * gridDim.x + blockIdx.x] = x;
  }
}

// load of each substep = sum_c |sum_i f_ic| (collision.cpp:110), last_collider_load = max over substeps
__global__ void k_collide_load(const double* partials, int nblocks, int nc, int nsub, double* out) {
  __shared__ double s[256];
  double best = 0.0;
  for (int sb = 0; sb < nsub; ++sb) {
    double load = 0.0;
    for (int c = 0; c < nc; ++c) {
      double v[3];
      for (int a = 0; a < 3; ++a) {
        const double* p = partials + (((size_t)sb * nc + c) * 3 + a) * nblocks;
        double x = 0.0;
        for (int b = threadIdx.x; b < nblocks; b += blockDim.x) x += p[b];
        s[threadIdx.x] = x;
        __syncthreads();
        for (int o = blockDim.x / 2; o > 0; o >>= 1) {
          if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
          __syncthreads();
        }
        v[a] = s[0];
        __syncthreads();
      }
      load += sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]);
    }
    best = (best < load) ? load : best;
  }
  if (threadIdx.x == 0) out[0] = best;
}

// enqueued right behind the PCG: it commits the step only when the solve converged (cg_out[1]), so the host
// needs no round trip before it; after a failed solve the host runs the ladder and enqueues it again
// also finishes the F-based assembly's fused energy (d.eng_sum): the per-row partials of the step's assembled state are
// summed by a fixed block tree, and the last block sums the block partials in block order (deterministic)
__global__ void __launch_bounds__(kTpb) k_integrate(DevData d, double dt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (d.cg_out[1] != 0.0 && i < d.nn) {
    const bool fixed = d.node_bc[i] >= 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const size_t k = 3 * (size_t)i + a;
      if (fixed) {
        d.u[k] = d.utgt[k];
        d.v[k] = d.vtgt[k];
      } else {
        const double v = d.v[k] + d.x[k];
        d.v[k] = v;
        d.u[k] = d.u[k] + dt * v;
      }
    }
  }
  if (!d.eng_sum) return;
  __shared__ double s[kTpb];
  __shared__ bool s_last;
  s[threadIdx.x] = i < d.nn ? d.eng_row[i] : 0.0;
  __syncthreads();
  for (int o = kTpb / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) s[threadIdx.x] = s[threadIdx.x] + s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) d.eng_part[blockIdx.x] = s[0];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(d.eng_ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  double acc = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += kTpb) acc = acc + __ldcg(d.eng_part + b);
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int o = kTpb / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) s[threadIdx.x] = s[threadIdx.x] + s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *d.eng_out = s[0];
    *d.eng_ticket = 0u;
  }
}

__global__ void k_absdiag(DevData d) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d.nn) return;
  const bool fixed = d.node_bc[i] >= 0;
  const double* A = diag_block(d, i);
  constexpr int st = 32;
#pragma unroll
  for (int a = 0; a < 3; ++a) d.absdiag[3 * (size_t)i + a] = fixed ? 0.0 : fabs(A[st * 4 * a]);
}

__global__ void k_shift_diag(DevData d, double shift) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d.nn) return;
  double* A = const_cast<double*>(diag_block(d, i));
  constexpr int st = 32;
#pragma unroll
  for (int a = 0; a < 3; ++a) A[st * 4 * a] += shift * d.absdiag[3 * (size_t)i + a];
}

__global__ void k_bsr_dinv(DevData d) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d.nn) return;
  const double* A = diag_block(d, i);
  constexpr int st = 32;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double dd = A[st * 4 * a];
    d.dinv[3 * (size_t)i + a] = (fabs(dd) > 1e-300) ? 1.0 / dd : 1.0;
  }
}

__global__ void k_reset_x(DevData d) {  // dx.setZero(); dx[fixed] = fixed_values (solver.cpp:124-125)
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d.nn) return;
  const bool fixed = d.node_bc[i] >= 0;
#pragma unroll
  for (int a = 0; a < 3; ++a) d.x[3 * (size_t)i + a] = fixed ? d.fv[3 * (size_t)i + a] : 0.0;
}

// quasi-static load step (solver.cpp:74-77 apply_boundary_displacements + the zero prescribed Newton increment)
__global__ void k_qs_bc(DevData d, int n_fixed, const int32_t* fixed_nodes) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n_fixed) return;
  const int i = fixed_nodes[q];
  const BcStep& b = d.bcstep[d.node_bc[i]];
  double u1[3];
  bc_disp(b, d.X + 3 * (size_t)i, b.R1, b.d1, u1);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    d.u[3 * (size_t)i + a] = u1[a];
    d.fv[3 * (size_t)i + a] = 0.0;
  }
}

// line-search trial point u = saved + step * dx (solver.cpp:176-177)
__global__ void k_qs_update(double* u, const double* saved, const double* dx, double step, int64_t n) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) u[k] = saved[k] + step * dx[k];
}

// per-block partial dot products a.b (fixed grid, deterministic order; summed on the host)
__global__ void k_fill(double* p, double v, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

// dynamic_full_newton update after each Newton solve (solver.cpp:296-303): dv_total += dv, v += dv on every dof
// (fixed dofs carry their prescribed dv), u = u_start + dt v
__global__ void k_newton_update(DevData d, double* dv_total, const double* u_start, double dt) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= 3 * (int64_t)d.nn) return;
  const double dv = d.x[k];
  dv_total[k] = dv_total[k] + dv;
  const double v = d.v[k] + dv;
  d.v[k] = v;
  d.u[k] = u_start[k] + dt * v;
}

__global__ void k_pin_bc(DevData d) {  // solver.cpp:322-328
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d.nn || d.node_bc[i] < 0) return;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    d.u[3 * (size_t)i + a] = d.utgt[3 * (size_t)i + a];
    d.v[3 * (size_t)i + a] = d.vtgt[3 * (size_t)i + a];
  }
}

}  // namespace

void launch_bc_targets(const DevData& d, int32_t n_fixed, const int32_t* fixed_nodes, double dt, cudaStream_t s) {
  if (n_fixed > 0) k_bc_targets<<<nblk(n_fixed), kTpb, 0, s>>>(d, n_fixed, fixed_nodes, dt);
}
int collide_blocks(const DevData& d) { return nblk(d.nn); }
void launch_collide(const DevData& d, int substep, double tau, double dt, int nsub, cudaStream_t s) {
  const int nb = nblk(d.nn);
  const int nc = d.n_colliders < 8 ? d.n_colliders : 8;
  k_collide<<<nb, kTpb, 0, s>>>(d, tau, dt, (double)nsub, substep == 0 ? 1 : 0, d.colliders + (size_t)substep * nc,
                                d.coll_partials + (size_t)substep * nc * 3 * nb);
}
void launch_collide_load(const DevData& d, int nsub, double* out, cudaStream_t s) {
  const int nc = d.n_colliders < 8 ? d.n_colliders : 8;
  k_collide_load<<<1, 256, 0, s>>>(d.coll_partials, nblk(d.nn), nc, nsub, out);
}
void launch_newton_update(const DevData& d, double* dv_total, const double* u_start, double dt, cudaStream_t s) {
  k_newton_update<<<nblk(3 * (int64_t)d.nn), kTpb, 0, s>>>(d, dv_total, u_start, dt);
}
void launch_pin_bc(const DevData& d, cudaStream_t s) { k_pin_bc<<<nblk(d.nn), kTpb, 0, s>>>(d); }
void launch_integrate(const DevData& d, double dt, cudaStream_t s) { k_integrate<<<nblk(d.nn), kTpb, 0, s>>>(d, dt); }
void launch_shift_diag(const DevData& d, double shift, cudaStream_t s) {
  k_shift_diag<<<nblk(d.nn), kTpb, 0, s>>>(d, shift);
}
void launch_absdiag(const DevData& d, cudaStream_t s) { k_absdiag<<<nblk(d.nn), kTpb, 0, s>>>(d); }
void launch_bsr_dinv(const DevData& d, cudaStream_t s) { k_bsr_dinv<<<nblk(d.nn), kTpb, 0, s>>>(d); }
void launch_reset_x(const DevData& d, cudaStream_t s) { k_reset_x<<<nblk(d.nn), kTpb, 0, s>>>(d); }
void launch_qs_bc(const DevData& d, int32_t n_fixed, const int32_t* fixed_nodes, cudaStream_t s) {
  if (n_fixed > 0) k_qs_bc<<<nblk(n_fixed), kTpb, 0, s>>>(d, n_fixed, fixed_nodes);
}
void launch_qs_update(double* u, const double* saved, const double* dx, double step, int64_t n, cudaStream_t s) {
  if (n > 0) k_qs_update<<<nblk(n), kTpb, 0, s>>>(u, saved, dx, step, n);
}
void launch_fill(double* p, double v, int64_t n, cudaStream_t s) {
  if (n > 0) k_fill<<<(int)((n + kTpb - 1) / kTpb), kTpb, 0, s>>>(p, v, n);
}

}  // namespace gfb
