// tmap.cpp -- TMA tensor-map encoding for the conv/GEMM kernels.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>
#include <mutex>
#include <string>

#include "eb_internal.h"

namespace eb {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
using EncodeIm2colFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const int*, const int*,
                                    cuuint32_t, cuuint32_t, const cuuint32_t*,
                                    CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn g_tiled = nullptr;
static EncodeIm2colFn g_im2col = nullptr;
static int g_driver_version = 0;
static std::once_flag g_once;

static bool resolve(std::string* err) {
  std::call_once(g_once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_tiled = reinterpret_cast<EncodeTiledFn>(fn);
    fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_im2col = reinterpret_cast<EncodeIm2colFn>(fn);
    cudaDriverGetVersion(&g_driver_version);
  });
  if (!g_tiled || !g_im2col) {
    if (err) *err = "cuTensorMapEncode* entry points unavailable (no CUDA driver?)";
    return false;
  }
  return true;
}

bool encode_tiled_2d_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                          uint64_t ld_elems, uint32_t box_inner, uint32_t box_outer,
                          std::string* err, int swizzle_bytes) {
  if (!resolve(err)) return false;
  const CUtensorMapSwizzle swz = swizzle_bytes == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                                 : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                 : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                       : CU_TENSOR_MAP_SWIZZLE_NONE;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld_elems * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_tiled(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                       strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    if (err)
      *err = "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) +
             ") inner=" + std::to_string(inner) + " outer=" + std::to_string(outer) +
             " ld=" + std::to_string(ld_elems);
    return false;
  }
  return true;
}

bool encode_tiled_3d_bf16(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t d2,
                          uint64_t stride1_elems, uint64_t stride2_elems, uint32_t b0, uint32_t b1,
                          uint32_t b2, std::string* err, int swizzle_bytes) {
  if (!resolve(err)) return false;
  const CUtensorMapSwizzle swz = swizzle_bytes == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                                 : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                 : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                       : CU_TENSOR_MAP_SWIZZLE_NONE;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {stride1_elems * 2, stride2_elems * 2};
  cuuint32_t box[3] = {b0, b1, b2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_tiled(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims,
                       strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    if (err)
      *err = "cuTensorMapEncodeTiled (3d) failed (" + std::to_string(static_cast<int>(r)) + ")";
    return false;
  }
  return true;
}

bool encode_im2col_bf16(CUtensorMap* map, const void* base, int n, int h, int w, int c, int ldc,
                        int kh, int kw, int sh, int sw, int ph, int pw, int chans_per_pixel,
                        int pixels, bool swizzle128, std::string* err, int upper_w_extra,
                        int upper_h_extra) {
  if (!resolve(err)) return false;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(c), static_cast<cuuint64_t>(w),
                        static_cast<cuuint64_t>(h), static_cast<cuuint64_t>(n)};
  const uint64_t px = static_cast<uint64_t>(ldc) * 2;
  cuuint64_t strides[3] = {px, px * w, px * w * h};
  int lower[2] = {-pw, -ph};                       // [W, H]
  // upper_w_extra widens the traversal in W (tap-shift mode walks W + 2*pw positions)
  // (and upper_h_extra in H: tall taps-in-N walks Ho + kh - 1 rows per image)
  int upper[2] = {pw - (kw - 1) + upper_w_extra, ph - (kh - 1) + upper_h_extra};   // [W, H]
  cuuint32_t estr[4] = {1, static_cast<cuuint32_t>(sw), static_cast<cuuint32_t>(sh), 1};
  CUresult r = g_im2col(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims,
                        strides, lower, upper, static_cast<cuuint32_t>(chans_per_pixel),
                        static_cast<cuuint32_t>(pixels), estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    if (err)
      *err = "cuTensorMapEncodeIm2col failed (" + std::to_string(static_cast<int>(r)) + ") n=" +
             std::to_string(n) + " h=" + std::to_string(h) + " w=" + std::to_string(w) +
             " c=" + std::to_string(c) + " ldc=" + std::to_string(ldc);
    return false;
  }
  // Drivers up to 13.1 mis-handle an im2col descriptor flag for tensors under
  // 128 KiB; clearing bit 21 of the second descriptor word is the same
  // workaround CUTLASS's im2col TMA path applies.
  const uint64_t bytes = px * static_cast<uint64_t>(w) * h * n;
  if (g_driver_version <= 13010 && bytes < 131072) {
    reinterpret_cast<uint64_t*>(map)[1] &= ~(1ull << 21);
  }
  return true;
}

}  // namespace eb
