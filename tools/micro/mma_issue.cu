// Microbenchmark: how fast can one CTA issue tcgen05.mma (M = 128, K = 16, bf16)?
//   v0: loop, descriptors rebuilt per MMA (as a generic loop would)
//   v1: unrolled groups of 12 MMAs, descriptors = base + compile-time offsets
//   v2: like v1 but two warps issue, each into its own accumulator
//   v3: groups of 6 MMAs (the VGG stem's tile), one commit to an mbarrier after each group
//   v4: groups of 6 MMAs, two commits per group (the stage slot and the accumulator)
//   v5: the fused VGG block-1 conv pattern: per row 3 SW128 A slots x 4 K16 steps, N = 192,
//       alternating accumulators, one commit per row -- random operand data
//   v6: v5 with zero operand data (data-dependence check)
// cycles per MMA over ITER MMAs per issuing warp, one CTA per SM.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../../paper_2003_01538_b200/csrc/sm100.cuh"

using namespace eb;

constexpr int ITER = 4800;  // multiple of 12

template <int V, int N>
__global__ void __launch_bounds__(128, 1) issue_bench(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(8) uint64_t bar[2];
  for (int i = threadIdx.x; i < 196608 / 16; i += blockDim.x) {
    if (V == 5) {  // pseudo-random bf16 in [-1, 1)
      uint32_t h = (i * 2654435761u) ^ 0x9e3779b9u, q[4];
      for (int e = 0; e < 4; ++e) {
        h = h * 1664525u + 1013904223u;
        const uint32_t lo = 0x3f80u | ((h >> 9) & 0x7fu) | ((h & 1u) << 15);
        const uint32_t hi = 0x3f00u | ((h >> 17) & 0x7fu) | ((h & 2u) << 14);
        q[e] = lo | (hi << 16);
      }
      reinterpret_cast<uint4*>(smem)[i] = make_uint4(q[0], q[1], q[2], q[3]);
    } else {
      reinterpret_cast<uint4*>(smem)[i] = make_uint4(V == 6 ? 0u : 0x3f803f80u, 0, 0, 0);
    }
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tmem_alloc(&tmem_slot, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  const int w = threadIdx.x >> 5;
  const int issuers = V == 2 ? 2 : 1;
  long long t0 = clock64();
  if (w < issuers && elect_one()) {
    constexpr uint32_t idesc = umma_idesc_bf16(128, N);
    const uint64_t a0 = umma_desc(smem_u32(smem), 16, 128, 0);
    const uint64_t b0 = umma_desc_sw128(smem_u32(smem + 65536));
    const uint32_t td = tmem + w * 256;
    if (V == 0) {
      for (int i = 0; i < ITER; ++i) {
        const int r = (i / 4) % 3, k = i & 3;
        const uint64_t ad = umma_desc(smem_u32(smem) + r * 4224, 16, 128, 0) + 2 * k;
        const uint64_t bd = umma_desc_sw128(smem_u32(smem + 65536) + r * 8192) + 2 * k;
        umma_bf16(td, ad, bd, idesc, i ? 1u : 0u);
      }
    } else if (V == 5 || V == 6) {
      // rows of 12 MMAs: A = 3 SW128 slots (16 KB) x K16 steps, B = 3 x 24 KB at 64 KB
      for (int i = 0; i < ITER; i += 12) {
        const uint32_t acc = tmem + ((i / 12) & 1) * 192;
#pragma unroll
        for (int j = 0; j < 12; ++j) {
          const int r = j / 4, k = j & 3;
          const uint64_t ad = umma_desc_sw128(smem_u32(smem) + r * 16384) + 2 * k;
          const uint64_t bd = umma_desc_sw128(smem_u32(smem + 65536) + r * 24576) + 2 * k;
          umma_bf16(acc, ad, bd, idesc, j ? 1u : 0u);
        }
        umma_commit(&bar[1]);
      }
    } else if (V == 3 || V == 4) {
      for (int i = 0; i < ITER; i += 6) {
#pragma unroll
        for (int j = 0; j < 6; ++j) {
          const int r = j / 2, k = j & 1;
          umma_bf16(td, a0 + r * 264 + 2 * k, b0 + r * 512 + 2 * k, idesc, (i | j) ? 1u : 0u);
        }
        umma_commit(&bar[1]);
        if (V == 4) umma_commit(&bar[1]);
      }
    } else {
      for (int i = 0; i < ITER; i += 12) {
#pragma unroll
        for (int j = 0; j < 12; ++j) {
          const int r = j / 4, k = j & 3;
          umma_bf16(td, a0 + r * 264 + 2 * k, b0 + r * 512 + 2 * k, idesc, (i | j) ? 1u : 0u);
        }
      }
    }
    umma_commit(&bar[w]);
    mbar_wait(&bar[w], 0);
  }
  __syncthreads();
  long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

template <int V, int N>
void run(long long* d) {
  const int smem = 196608;
  cudaFuncSetAttribute(issue_bench<V, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  issue_bench<V, N><<<148, 128, smem>>>(d);
  long long c = 0;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  const int total = ITER * (V == 2 ? 2 : 1);
  printf("v%d N=%3d: %6.1f cycles per MMA (%d MMAs), tensor floor %d\n", V, N, double(c) / total, total,
         128 * N / 256);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  run<0, 64>(d);
  run<1, 64>(d);
  run<2, 64>(d);
  run<0, 128>(d);
  run<1, 128>(d);
  run<2, 128>(d);
  run<1, 192>(d);
  run<2, 192>(d);
  run<1, 256>(d);
  run<3, 64>(d);
  run<4, 64>(d);
  run<3, 128>(d);
  run<5, 192>(d);
  run<6, 192>(d);
  run<1, 192>(d);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
