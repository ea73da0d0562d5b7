// Microbenchmark: per-launch time of back-to-back dependent launches inside a CUDA graph,
// as a function of the launch configuration of an (almost) empty persistent kernel:
// dynamic shared memory, block size, parameter size (four 128-byte CUtensorMaps as
// __grid_constant__ like conv_umma_kernel), TMEM alloc/dealloc, and PDL.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o tools/micro/launch_gap \
//        tools/micro/launch_gap.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../../paper_2003_01538_b200/csrc/sm100.cuh"

using namespace eb;

struct Big {
  CUtensorMap m[4];
  char pad[512];
};

template <bool TMEM, bool PDL>
__global__ void __launch_bounds__(384, 1) k_big(const __grid_constant__ Big b, int* out) {
  extern __shared__ uint8_t smem[];
  __shared__ uint32_t slot;
  if (TMEM && threadIdx.x < 32) tmem_alloc(&slot, 512);
  if (PDL) {
    pdl_wait();
    pdl_launch_dependents();
  }
  __syncthreads();
  if (threadIdx.x == 0 && b.pad[0] == 7) out[blockIdx.x] = smem[0];
  __syncthreads();
  if (TMEM && threadIdx.x < 32) tmem_dealloc(slot, 512);
}

__global__ void k_small(int* out, int v) {
  if (threadIdx.x == 0 && v == 7) out[blockIdx.x] = v;
}

template <typename F>
float time_graph(cudaStream_t s, int n, F launch) {
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < n; ++i) launch();
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best * 1e3f / n;
}

template <bool TMEM, bool PDL>
float run_big(cudaStream_t s, int* out, int smem, int threads, int grid) {
  cudaFuncSetAttribute(k_big<TMEM, PDL>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  Big b = {};
  return time_graph(s, 200, [&] {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = PDL ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_big<TMEM, PDL>, b, out);
  });
}

int main() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  int* out;
  cudaMalloc(&out, 1 << 20);
  printf("small kernel, 148x128, 0 smem:            %.2f us/launch\n",
         time_graph(s, 200, [&] { k_small<<<148, 128, 0, s>>>(out, 1); }));
  const int smems[] = {0, 100 * 1024, 200 * 1024, 227 * 1024};
  for (int sm : smems) {
    printf("big params, 148x384, %3d KB smem:          %.2f us/launch\n", sm / 1024,
           run_big<false, false>(s, out, sm, 384, 148));
  }
  printf("big params, 148x384, 200 KB, TMEM 512:     %.2f us/launch\n",
         run_big<true, false>(s, out, 200 * 1024, 384, 148));
  printf("big params, 148x384, 200 KB, TMEM, PDL:    %.2f us/launch\n",
         run_big<true, true>(s, out, 200 * 1024, 384, 148));
  printf("big params, 148x384, 200 KB, PDL:          %.2f us/launch\n",
         run_big<false, true>(s, out, 200 * 1024, 384, 148));
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
