// eb_kernels.h -- host launchers for the non-GEMM kernels.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace eb {

cudaError_t k_preprocess_f32(const float* x, float* y, int B, int C, int64_t plane,
                             const float* mean, const float* stdv, int nms, cudaStream_t s);
cudaError_t k_preprocess_f32chw_to_nhwc(const float* x, __nv_bfloat16* y, int B, int C,
                                        int64_t plane, int cpad, const float* mean,
                                        const float* stdv, int nms, cudaStream_t s);
cudaError_t k_preprocess_u8hwc_to_nhwc(const uint8_t* x, __nv_bfloat16* y, int B, int C,
                                       int64_t plane, int cpad, const float* lut, cudaStream_t s);
cudaError_t k_preprocess_u8hwc_to_f32chw(const uint8_t* x, float* y, int B, int C, int64_t plane,
                                         const float* lut, cudaStream_t s);

// 8-channel NHWC image -> the zero-padded stem layout described by StemGeom (eb_internal.h):
// mode kAModeStemRows (stride 1) or kAModeStemPlanes (stride 2, even/odd column planes).
cudaError_t k_copy(const void* src, void* dst, size_t bytes, cudaStream_t s);
cudaError_t k_preprocess_u8_to_layout(const uint8_t* x, int B, int C, int H, int W, const float* lut,
                                      int ph, int pw, int mode, int Hq, int Wq, __nv_bfloat16* y,
                                      cudaStream_t s);
cudaError_t k_stem_relayout(const __nv_bfloat16* x, int B, int H, int W, int ph, int pw, int mode,
                            int Hq, int Wq, __nv_bfloat16* y, cudaStream_t s);

cudaError_t k_pool(const __nv_bfloat16* x, int ldx, __nv_bfloat16* y, int ldy, int y_off, int B,
                   int H, int W, int C, int Ho, int Wo, int k, int s, int pad, int mode,
                   const float* scale, const float* shift, cudaStream_t st);
cudaError_t k_bnrelu(const __nv_bfloat16* x, int ldx, __nv_bfloat16* y, int ldy, int64_t M, int C,
                     const float* scale, const float* shift, cudaStream_t st);
cudaError_t k_gap(const __nv_bfloat16* x, int ldx, __nv_bfloat16* y, int B, int HW, int C,
                  const float* scale, const float* shift, cudaStream_t st);
cudaError_t k_resize_bilinear(const __nv_bfloat16* x, int ldx, __nv_bfloat16* y, int ldy, int B,
                              int H, int W, int C, int Ho, int Wo, cudaStream_t st);
cudaError_t k_splitk_finalize(const float* ws, int splits, int64_t M, int N, const float* bias,
                              int relu, void* out, int ldo, int out_off, int out_f32,
                              cudaStream_t st);

cudaError_t k_combine(const float* l32, int ld32, const double* l64, int ld64, const int* kind,
                      const int* koff, const int* kcnt, int N, int B, int32_t* labels, int topk,
                      int32_t* topk_idx, float* topk_prob, int policy, int policy_k,
                      int32_t* combined, cudaStream_t s);
cudaError_t k_lin1(const float* x, const float* w, const float* bias, double* part,
                   double* logits, int B, int K, int64_t D, int nsplit, cudaStream_t s);

// fp32-faithful parity mode (ref32.cu): fp32 NHWC activations, CUDA-core kernels.
cudaError_t k32_preprocess_u8(const uint8_t* x, float* y, int B, int C, int64_t plane, int cpad,
                              const float* lut, cudaStream_t s);
cudaError_t k32_preprocess_f32chw(const float* x, float* y, int B, int C, int64_t plane, int cpad,
                                  const float* mean, const float* stdv, int nms, cudaStream_t s);
cudaError_t k32_conv(const float* x, int B, int H, int W, int ldx, int cin, int groups,
                     const float* w, const float* bias, const float* res, int ldr, float* y,
                     int ldy, int y_off, float* y2, int ldy2, int y2_off, int n_split, int cout,
                     int kh, int kw, int sh, int sw, int ph, int pw, int relu, int flatten,
                     const float* pre_scale, const float* pre_shift, cudaStream_t s);
cudaError_t k32_pool(const float* x, int ldx, float* y, int ldy, int y_off, int B, int H, int W,
                     int C, int Ho, int Wo, int k, int s, int pad, int mode, const float* scale,
                     const float* shift, cudaStream_t st);
cudaError_t k32_bnrelu(const float* x, int ldx, float* y, int ldy, int64_t M, int C,
                       const float* scale, const float* shift, cudaStream_t st);
cudaError_t k32_gap(const float* x, int ldx, float* y, int B, int HW, int C, const float* scale,
                    const float* shift, cudaStream_t st);
cudaError_t k32_resize(const float* x, int ldx, float* y, int ldy, int B, int H, int W, int C,
                       int Ho, int Wo, cudaStream_t st);

}  // namespace eb
