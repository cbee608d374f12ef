// probe.cu — bandwidth probes for the roofline denominators (bench.py, tools/l2_roof.py).
//
//  kind 0  L2 read roof: every SM streams an L2-resident buffer with 16-byte ld.global.cg (L1 bypassed), four
//          independent loads in flight per thread; one warm pass, then `reps` timed passes. This is the roof of a
//          kernel whose working set stays in the 126 MB L2 (the c3 PCG: symmetric matrix + slots + vectors).
//  kind 1  HBM copy roof: y = x over buffers larger than L2, read + write bytes counted (MEASURED_PEAKS.json's
//          definition), so the number is directly comparable to the driver's measured peak.
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "dev_types.cuh"
#include "host_mesh.hpp"

namespace gfb {
namespace {

__global__ void __launch_bounds__(512) k_read_cg(const double2* __restrict__ p, size_t n, int reps, double* sink) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n; i += 4 * stride) {
      const double2 v0 = __ldcg(p + i), v1 = __ldcg(p + i + stride), v2 = __ldcg(p + i + 2 * stride),
                    v3 = __ldcg(p + i + 3 * stride);
      a0 += v0.x + v0.y;
      a1 += v1.x + v1.y;
      a2 += v2.x + v2.y;
      a3 += v3.x + v3.y;
    }
    for (; i < n; i += stride) {
      const double2 v = __ldcg(p + i);
      a0 += v.x + v.y;
    }
  }
  const double t = (a0 + a1) + (a2 + a3);
  if (t == 1234.5678) sink[0] = t;  // never true for the zero-filled buffer; keeps the loads alive
}

__global__ void __launch_bounds__(512) k_copy(const double2* __restrict__ x, double2* __restrict__ y, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) y[i] = __ldcs(x + i);
}

#define PB_CUDA(x)                                                                              \
  do {                                                                                          \
    const cudaError_t _e = (x);                                                                 \
    if (_e != cudaSuccess) throw CudaError(std::string(#x) + ": " + cudaGetErrorString(_e));     \
  } while (0)

}  // namespace

double measure_bandwidth(int kind, int64_t bytes, int reps) {
  if (bytes < (1 << 20) || reps < 1) throw FormatError("bandwidth probe: bytes >= 1 MiB and reps >= 1 required");
  int dev = 0, sms = 0;
  PB_CUDA(cudaGetDevice(&dev));
  PB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const size_t n = (size_t)bytes / 16;
  void *a = nullptr, *b = nullptr;
  double* sink = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  auto cleanup = [&] {
    if (a) cudaFree(a);
    if (b) cudaFree(b);
    if (sink) cudaFree(sink);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
  };
  double gbps = 0.0;
  try {
    PB_CUDA(cudaMalloc(&a, 16 * n));
    PB_CUDA(cudaMemset(a, 0, 16 * n));
    PB_CUDA(cudaMalloc(&sink, 8));
    PB_CUDA(cudaEventCreate(&e0));
    PB_CUDA(cudaEventCreate(&e1));
    float ms = 0.f;
    if (kind == 0) {
      const int grid = 4 * sms;  // 4 x 512 threads per SM
      k_read_cg<<<grid, 512>>>((const double2*)a, n, 1, sink);  // warm pass: the buffer lands in L2
      PB_CUDA(cudaEventRecord(e0));
      k_read_cg<<<grid, 512>>>((const double2*)a, n, reps, sink);
      PB_CUDA(cudaEventRecord(e1));
      PB_CUDA(cudaEventSynchronize(e1));
      PB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      gbps = 16.0 * (double)n * reps / (ms * 1e-3) / 1e9;
    } else if (kind == 1) {
      PB_CUDA(cudaMalloc(&b, 16 * n));
      const int grid = 4 * sms;
      k_copy<<<grid, 512>>>((const double2*)a, (double2*)b, n);
      float best = 1e30f;
      for (int r = 0; r < reps; ++r) {
        PB_CUDA(cudaEventRecord(e0));
        k_copy<<<grid, 512>>>((const double2*)a, (double2*)b, n);
        PB_CUDA(cudaEventRecord(e1));
        PB_CUDA(cudaEventSynchronize(e1));
        PB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        best = ms < best ? ms : best;
      }
      gbps = 32.0 * (double)n / (best * 1e-3) / 1e9;  // read + write
    } else {
      throw FormatError("bandwidth probe: kind must be 0 (L2 read) or 1 (HBM copy)");
    }
    PB_CUDA(cudaGetLastError());
  } catch (...) {
    cleanup();
    throw;
  }
  cleanup();
  return gbps;
}

}  // namespace gfb
