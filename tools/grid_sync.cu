// Cost of one cooperative-groups grid barrier on this GPU (diagnostic for the PCG's per-iteration floor):
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/grid_sync tools/grid_sync.cu && /tmp/grid_sync
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_sync(int iters, double* part, int with_reduce) {
  cg::grid_group g = cg::this_grid();
  double acc = 0.0;
  for (int i = 0; i < iters; ++i) {
    if (with_reduce && threadIdx.x == 0) part[(i & 1) * 1024 + blockIdx.x] = i + blockIdx.x;
    g.sync();
    if (with_reduce && threadIdx.x < gridDim.x) acc += __ldcg(part + (i & 1) * 1024 + threadIdx.x);
  }
  if (acc == -1.0) part[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* part;
  cudaMalloc(&part, 8 * 2048);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int threads : {32, 256, 768})
    for (int grid : {4, 16, 64, sms})
      for (int red = 0; red < 2; ++red) {
        int iters = 2000;
        void* args[] = {&iters, &part, &red};
        cudaLaunchCooperativeKernel((void*)k_sync, grid, threads, args, 0, 0);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k_sync, grid, threads, args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("{\"threads\": %d, \"grid\": %d, \"reduce\": %d, \"us_per_sync\": %.3f}\n", threads, grid, red,
               1e3 * ms / iters);
      }
  return 0;
}
