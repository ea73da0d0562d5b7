// Microbenchmark: tcgen05.mma (M = 128, K = 16, bf16) throughput for the A-operand layouts
// the conv kernel uses -- SW128 K-major (im2col / tiled modes) vs the stem rows mode's
// no-swizzle layout with overlapping core matrices (LBO = 16 B: tap s+1 is the next
// pixel, 16 B on) -- at N = 64 / 128 / 256.  One CTA per SM, one thread issues ITER MMAs
// into one accumulator, commit, wait; cycles per MMA from clock64.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../../paper_2003_01538_b200/csrc/sm100.cuh"

using namespace eb;

constexpr int ITER = 4096;

__global__ void __launch_bounds__(128, 1) mma_bench(int mode, int N, int group, int nacc, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(8) uint64_t bar;
  uint8_t* a = smem;            // 64 KB of A
  uint8_t* b = smem + 65536;    // 32 KB of B
  for (int i = threadIdx.x; i < (65536 + 32768) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3f803f80u, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tmem_alloc(&tmem_slot, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = umma_idesc_bf16(128, N);
    const uint32_t sa = smem_u32(a), sb = smem_u32(b);
    // mode 0: SW128 K-major A (128 rows x 128 B, K steps +32 B); mode 1: stem rows
    // (no swizzle, LBO 16 B, SBO 128 B: row m = 16 B * m, K core matrix +16 B)
    const uint64_t bdesc0 = umma_desc_sw128(sb);
    long long t0 = clock64();
    uint32_t phase = 0;
    for (int i = 0; i < ITER; ++i) {
      const int k = i & 3;
      uint64_t adesc;
      if (mode == 0)
        adesc = umma_desc_sw128(sa) + 2 * k;
      else
        adesc = umma_desc(sa, 16, 128, 0) + 2 * k;  // taps 2k, 2k+1
      // nacc accumulators round-robin (columns N apart): independent MMA chains
      umma_bf16(tmem + (i % nacc) * N, adesc, bdesc0 + 2 * k, idesc, i >= nacc ? 1u : 0u);
      if (group > 0 && (i + 1) % group == 0) {  // per-tile commit + wait (latency chain)
        umma_commit(&bar);
        mbar_wait(&bar, phase);
        phase ^= 1;
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, phase);
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  const int smem = 65536 + 32768;
  cudaFuncSetAttribute(mma_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int nacc : {1, 2, 4})
    for (int mode = 0; mode < 2; ++mode)
      for (int N : {32, 64, 96, 128, 192, 256}) {
        if (N * nacc > 512) continue;
        mma_bench<<<148, 128, smem>>>(mode, N, 0, nacc, d);
        long long c = 0;
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        printf("%-12s N=%3d acc=%d: %6.1f cycles per MMA (floor 128*N/256 = %d)\n",
               mode ? "stem-rows A" : "SW128 A", N, nacc, double(c) / ITER, 128 * N / 256);
      }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
