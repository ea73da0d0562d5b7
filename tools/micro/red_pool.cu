// Microbenchmark: 2x2 max-pool of an NHWC bf16 conv output by 16-byte red.global.max
// (REDG.E.MAX.BF16x8) vs. write full-res + separate pool read.  B=256, 112x112x128 -> 56x56.
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
__global__ void red_pool(uint4* out, int B, int H, int W, int C8, uint32_t v) {
  // one thread per (pixel, 8-channel group) of the full-res tensor, in NHWC order
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t total = (int64_t)B * H * W * C8;
  if (i >= total) return;
  int c = i % C8; int64_t p = i / C8; int w = p % W; int64_t q = p / W; int h = q % H; int b = q / H;
  int64_t o = (((int64_t)b * (H / 2) + h / 2) * (W / 2) + w / 2) * C8 + c;
  uint32_t x = v ^ (uint32_t)(i * 2654435761u) & 0x3f7f3f7fu;
  asm volatile("red.global.v4.bf16x2.max.noftz [%0], {%1,%2,%3,%4};" :: "l"(out + o), "r"(x), "r"(x), "r"(x), "r"(x) : "memory");
}
__global__ void plain_store(uint4* full, int64_t n, uint32_t v) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) full[i] = make_uint4(v, v, v, v);
}
int main() {
  int B = 256, H = 112, W = 112, C8 = 16;
  int64_t nfull = (int64_t)B * H * W * C8, npool = nfull / 4;
  uint4 *full, *pool;
  cudaMalloc(&full, nfull * 16); cudaMalloc(&pool, npool * 16);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    cudaMemsetAsync(pool, 0, npool * 16);
    red_pool<<<(nfull + 255) / 256, 256>>>(pool, B, H, W, C8, 0x3f003f00u + rep);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    cudaEventRecord(a);
    plain_store<<<(nfull + 255) / 256, 256>>>(full, nfull, rep);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms2; cudaEventElapsedTime(&ms2, a, b);
    printf("memset+red %.1f us (%.0f GB/s of reductions)   plain full-res store %.1f us\n", ms * 1e3,
           nfull * 16 / ms / 1e6, ms2 * 1e3);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
