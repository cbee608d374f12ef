// Read bandwidth of tensor memory (tcgen05.ld) and of shared memory from every SM, as general per-thread storage
// (the design question for an on-chip-resident PCG matrix):
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tmem_bw tools/tmem_bw.cu && /tmp/tmem_bw
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int N>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, uint32_t (&r)[N]);

template <>
__device__ __forceinline__ void tmem_ld<16>(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

template <int kCols>
__global__ void __launch_bounds__(768, 1) k_tmem_read(int iters, int wpq, unsigned* out, long long* cyc) {
  __shared__ uint32_t s_taddr;
  const int w = threadIdx.x >> 5;
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&s_taddr)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t base = s_taddr;
  const int quad = w & 3, slot = w >> 2;
  const int per = 512 / wpq;  // columns per warp of a quadrant
  const uint32_t ta = base + ((uint32_t)(32 * quad) << 16) + (uint32_t)(slot * per);
  unsigned acc = 0;
  const long long t0 = clock64();
  if (slot < wpq) {
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int c = 0; c + 16 <= kCols; c += 16) {
        uint32_t r[16];
        tmem_ld<16>(ta + c, r);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n");
#pragma unroll
        for (int k = 0; k < 16; ++k) acc += r[k];
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(base), "r"(512));
  if (acc == 0xdeadbeefu) out[0] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// shared memory: each thread reads kWords 32-bit words of its own [word][thread] column, 8 bytes at a time
template <int kDoubles>
__global__ void __launch_bounds__(768, 1) k_smem_read(int iters, unsigned* out, long long* cyc) {
  extern __shared__ double s[];
  for (int i = threadIdx.x; i < kDoubles * 768; i += blockDim.x) s[i] = i;
  __syncthreads();
  double acc = 0.0;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kDoubles; ++c) acc += s[c * 768 + threadIdx.x];
    __syncwarp();
  }
  __syncthreads();
  const long long t1 = clock64();
  if (acc == -1.0) out[0] = 1;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  unsigned* out;
  long long* cyc;
  cudaMalloc(&out, 64);
  cudaMalloc(&cyc, 8 * 1024);
  long long h[1024];
  const int iters = 2000;
  for (int threads : {128, 384, 768}) {
    const int wpq = threads / 128;
    k_tmem_read<80><<<sms, threads>>>(iters, wpq, out, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(h, cyc, 8 * sms, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
    const double bytes = (double)iters * 80 * 4 * threads;  // per SM
    printf("{\"kind\": \"tmem_ld_32x32b_x16\", \"threads\": %d, \"bytes_per_clk_per_sm\": %.1f}\n", threads,
           bytes / mx);
  }
  cudaFuncSetAttribute(k_smem_read<36>, cudaFuncAttributeMaxDynamicSharedMemorySize, 36 * 768 * 8);
  for (int threads : {384, 768}) {
    k_smem_read<36><<<sms, threads, 36 * 768 * 8>>>(iters, out, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(h, cyc, 8 * sms, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
    const double bytes = (double)iters * 36 * 8 * threads;
    printf("{\"kind\": \"smem_ld_f64\", \"threads\": %d, \"bytes_per_clk_per_sm\": %.1f}\n", threads, bytes / mx);
  }
  printf("{\"sm_clock_khz\": %d, \"sms\": %d}\n", clk, sms);
  return 0;
}
