// fp64_peak.cu — measured FP64 FMA throughput of the CUDA cores (the compute roof of the fp64 kernels, SURVEY
// §8(d) asks for it: not in MEASURED_PEAKS.json). Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
// tools/fp64_peak.cu -o tools/fp64_peak ; run on a B200: prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_fma(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 1234.5) out[0] = s;  // keep the chains alive
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  const int blocks = sms * 8, threads = 256, iters = 8192;
  k_fma<<<blocks, threads>>>(out, 16, 0.999999, 1e-9);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k_fma<<<blocks, threads>>>(out, iters, 0.999999, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * 8.0 * (double)iters * blocks * threads;
  printf("{\"fp64_fma_tflops\": %.2f, \"sms\": %d, \"ms\": %.3f, \"how\": \"8 independent FMA chains x %d iterations, %d x %d threads, best of 5\"}\n",
         flops / (best * 1e-3) / 1e12, sms, best, iters, blocks, threads);
  return 0;
}
