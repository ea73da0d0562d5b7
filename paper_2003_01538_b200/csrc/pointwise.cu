// pointwise.cu -- K1 (shared preprocess) and K4 (pooling / BN-ReLU) kernels.
//
// All activation tensors are NHWC bf16 with a row (pixel) stride `ld` that may
// exceed the channel count (channel slices of a concat buffer).  Channel work is
// vectorised by 8 (16-byte loads/stores); every channel count used by the
// supported model families is a multiple of 8.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "eb_internal.h"
#include "eb_kernels.h"

namespace eb {

static inline int grid_for(int64_t work, int threads) {
  int64_t g = (work + threads - 1) / threads;
  if (g > 148 * 64) g = 148 * 64;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

// ------------------------------------------------------------------ K1 preprocess

// Reference semantics (eg/models.py:254-259): y = (x - mean_c) / std_c in fp32,
// each op correctly rounded, same (B, C, H*W) layout.  No FMA can form here
// (there is no multiply), and '/' compiles to the IEEE divide without fast-math.
__global__ void preprocess_f32_kernel(const float* __restrict__ x, float* __restrict__ y,
                                      int64_t total, int C, int64_t plane,
                                      const float* __restrict__ mean,
                                      const float* __restrict__ stdv, int nms) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = (nms == 1) ? 0 : static_cast<int>((i / plane) % C);
    y[i] = __fdiv_rn(__fsub_rn(x[i], mean[c]), stdv[c]);
  }
}

// f32 CHW (already divided by pixel_scale on the wire, eg/wire.py:71) ->
// normalised fp32 -> bf16 NHWC with channels zero-padded to `cpad` (8).
__global__ void preprocess_f32chw_to_nhwc_kernel(const float* __restrict__ x,
                                                 __nv_bfloat16* __restrict__ y, int64_t pixels,
                                                 int C, int64_t plane, int cpad,
                                                 const float* __restrict__ mean,
                                                 const float* __restrict__ stdv, int nms) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < pixels;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = p / plane;
    const int64_t q = p - b * plane;
    __align__(16) __nv_bfloat16 v[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      float f = 0.f;
      if (c < C) {
        const int mc = (nms == 1) ? 0 : c;
        f = __fdiv_rn(__fsub_rn(x[(b * C + c) * plane + q], mean[mc]), stdv[mc]);
      }
      v[c] = __float2bfloat16_rn(f);
    }
    *reinterpret_cast<uint4*>(y + p * cpad) = *reinterpret_cast<uint4*>(v);
  }
}

// u8 HWC -> bf16 NHWC8 through a per-channel 256-entry LUT.  The LUT holds the
// reference's fp32 value ((u8 / pixel_scale) - mean_c) / std_c for every byte,
// computed on the host with numpy's own fp32 ops, so the kernel is exact by
// construction (no divides on the device).
__global__ void preprocess_u8hwc_to_nhwc_kernel(const uint8_t* __restrict__ x,
                                                __nv_bfloat16* __restrict__ y, int64_t pixels,
                                                int C, int cpad, const float* __restrict__ lut) {
  __shared__ float s_lut[8 * 256];
  for (int i = threadIdx.x; i < C * 256; i += blockDim.x) s_lut[i] = lut[i];
  __syncthreads();
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < pixels;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    __align__(16) __nv_bfloat16 v[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const float f = (c < C) ? s_lut[c * 256 + x[p * C + c]] : 0.f;
      v[c] = __float2bfloat16_rn(f);
    }
    *reinterpret_cast<uint4*>(y + p * cpad) = *reinterpret_cast<uint4*>(v);
  }
}

// u8 HWC -> fp32 CHW normalised (LIN1 members fed from u8 requests).
__global__ void preprocess_u8hwc_to_f32chw_kernel(const uint8_t* __restrict__ x,
                                                  float* __restrict__ y, int64_t pixels, int C,
                                                  int64_t plane, const float* __restrict__ lut) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < pixels;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = p / plane;
    const int64_t q = p - b * plane;
    for (int c = 0; c < C; ++c) y[(b * C + c) * plane + q] = lut[c * 256 + x[p * C + c]];
  }
}

cudaError_t k_preprocess_f32(const float* x, float* y, int B, int C, int64_t plane,
                             const float* mean, const float* stdv, int nms, cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(B) * C * plane;
  if (total == 0) return cudaSuccess;
  preprocess_f32_kernel<<<grid_for(total, 256), 256, 0, s>>>(x, y, total, C, plane, mean, stdv,
                                                             nms);
  return cudaGetLastError();
}

cudaError_t k_preprocess_f32chw_to_nhwc(const float* x, __nv_bfloat16* y, int B, int C,
                                        int64_t plane, int cpad, const float* mean,
                                        const float* stdv, int nms, cudaStream_t s) {
  const int64_t pixels = static_cast<int64_t>(B) * plane;
  if (pixels == 0) return cudaSuccess;
  preprocess_f32chw_to_nhwc_kernel<<<grid_for(pixels, 256), 256, 0, s>>>(x, y, pixels, C, plane,
                                                                         cpad, mean, stdv, nms);
  return cudaGetLastError();
}

cudaError_t k_preprocess_u8hwc_to_nhwc(const uint8_t* x, __nv_bfloat16* y, int B, int C,
                                       int64_t plane, int cpad, const float* lut,
                                       cudaStream_t s) {
  const int64_t pixels = static_cast<int64_t>(B) * plane;
  if (pixels == 0) return cudaSuccess;
  preprocess_u8hwc_to_nhwc_kernel<<<grid_for(pixels, 256), 256, 0, s>>>(x, y, pixels, C, cpad,
                                                                        lut);
  return cudaGetLastError();
}

cudaError_t k_preprocess_u8hwc_to_f32chw(const uint8_t* x, float* y, int B, int C,
                                         int64_t plane, const float* lut, cudaStream_t s) {
  const int64_t pixels = static_cast<int64_t>(B) * plane;
  if (pixels == 0) return cudaSuccess;
  preprocess_u8hwc_to_f32chw_kernel<<<grid_for(pixels, 256), 256, 0, s>>>(x, y, pixels, C,
                                                                          plane, lut);
  return cudaGetLastError();
}

// K1 straight into a stem layout (StemGeom): u8 HWC -> LUT -> bf16 8-channel pixels of
// the zero-padded rows / even-odd planes buffer.  Used instead of the NHWC8 image plus a
// relayout when a stem reads the preprocessed image (one pass, no intermediate).
// A work unit is kRows consecutive padded rows hq of one image (both planes in the planes
// mode, which read the same input rows): the unit's input rows are one contiguous run of
// bytes, staged into smem with 16-byte loads (all in flight at once), then every output
// pixel is formed from smem and written with one 16-byte store.
constexpr int kK1Rows = 8;
constexpr int kK1MaxRowBytes = 2048;  // W * C per input row staged (larger: direct loads)

template <int CT>  // CT: channel count when known at compile time (3), else 0
__global__ void __launch_bounds__(256)
    preprocess_u8_to_layout_kernel(const uint8_t* __restrict__ x, int B, int C_, int H, int W,
                                   const float* __restrict__ lut, int ph, int pw, int planes, int Hq,
                                   int Wq, int rpu, uint4* __restrict__ y) {
  const int C = CT ? CT : C_;
  // the LUT pre-rounded to bf16 (the value the output carries)
  __shared__ __nv_bfloat16 s_lut[8 * 256];
  __shared__ __align__(16) uint8_t s_in[kK1Rows * kK1MaxRowBytes];
  for (int i = threadIdx.x; i < C * 256; i += blockDim.x) s_lut[i] = __float2bfloat16_rn(lut[i]);
  const int row_bytes = W * C;
  const bool staged = row_bytes <= kK1MaxRowBytes;
  const int chunks = (Hq + rpu - 1) / rpu;
  const int units = B * chunks;
  const int nq = planes ? 2 : 1;
  const int warp = static_cast<int>(threadIdx.x) >> 5;
  const int lane = static_cast<int>(threadIdx.x) & 31;
  const __nv_bfloat16 zero = __float2bfloat16_rn(0.f);
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    const int b = u / chunks;
    const int hq0 = (u - b * chunks) * rpu;
    // input rows [ih0, ih1) of this unit that lie inside the image
    const int ih0 = max(hq0 - ph, 0);
    const int ih1 = min(hq0 + rpu - ph, H);
    const uint8_t* src = x + (static_cast<int64_t>(b) * H + ih0) * row_bytes;
    __syncthreads();  // (previous unit done with s_in; LUT staged)
    if (staged && ih1 > ih0) {
      const int n = (ih1 - ih0) * row_bytes;
      if (((reinterpret_cast<uintptr_t>(src) | static_cast<uintptr_t>(n)) & 15) == 0) {
        for (int i = threadIdx.x; i < n / 16; i += blockDim.x)
          reinterpret_cast<uint4*>(s_in)[i] = __ldg(reinterpret_cast<const uint4*>(src) + i);
      } else {
        for (int i = threadIdx.x; i < n; i += blockDim.x) s_in[i] = src[i];
      }
    }
    __syncthreads();
    // one warp per output row (plane q, padded row hq), 32 pixels per step
    for (int qr = warp; qr < nq * rpu; qr += 8) {
      const int q = qr / rpu;
      const int hq = hq0 + (qr - q * rpu);
      if (hq >= Hq) continue;
      const int ih = hq - ph;
      const bool hok = ih >= 0 && ih < H;
      uint4* yr = y + (static_cast<int64_t>(q * B + b) * Hq + hq) * Wq;
      const uint8_t* rowp = staged ? s_in + (ih - ih0) * row_bytes
                                   : x + (static_cast<int64_t>(b) * H + ih) * row_bytes;
      for (int j = lane; j < Wq; j += 32) {
        const int iw = planes ? 2 * j + q - pw : j - pw;
        const bool ok = hok && iw >= 0 && iw < W;
        const uint8_t* px = rowp + iw * C;
        __align__(16) __nv_bfloat16 v[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) v[c] = (ok && c < C) ? s_lut[c * 256 + px[c]] : zero;
        yr[j] = *reinterpret_cast<const uint4*>(v);
      }
    }
  }
}

cudaError_t k_preprocess_u8_to_layout(const uint8_t* x, int B, int C, int H, int W, const float* lut,
                                      int ph, int pw, int mode, int Hq, int Wq, __nv_bfloat16* y,
                                      cudaStream_t s) {
  const int planes = mode == kAModeStemPlanes ? 1 : 0;
  if (B == 0 || Hq == 0 || Wq == 0) return cudaSuccess;
  // rows per unit: kK1Rows, fewer when that would leave SMs idle (small batches)
  int rpu = kK1Rows;
  while (rpu > 1 && static_cast<int64_t>(B) * ((Hq + rpu - 1) / rpu) < 148 * 4) rpu /= 2;
  const int64_t units = static_cast<int64_t>(B) * ((Hq + rpu - 1) / rpu);
  const int grid = static_cast<int>(std::min<int64_t>(units, 148 * 8));
  if (C == 3)
    preprocess_u8_to_layout_kernel<3><<<grid, 256, 0, s>>>(x, B, C, H, W, lut, ph, pw, planes, Hq,
                                                           Wq, rpu, reinterpret_cast<uint4*>(y));
  else
    preprocess_u8_to_layout_kernel<0><<<grid, 256, 0, s>>>(x, B, C, H, W, lut, ph, pw, planes, Hq,
                                                           Wq, rpu, reinterpret_cast<uint4*>(y));
  return cudaGetLastError();
}

// ------------------------------------------------------------------ device copy
// SM copy for the pipelined forward's staging -> input move (a copy-engine D2D of a
// batch of images runs far below HBM bandwidth).
__global__ void copy16_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, int64_t n16) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n16;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

cudaError_t k_copy(const void* src, void* dst, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return cudaSuccess;
  if ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst) | bytes) & 15)
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s);
  const int64_t n16 = static_cast<int64_t>(bytes / 16);
  copy16_kernel<<<grid_for(n16, 256), 256, 0, s>>>(static_cast<const uint4*>(src),
                                                   static_cast<uint4*>(dst), n16);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ stem relayout
// One thread per 16-byte output pixel (8 bf16 channels); borders are written as zeros
// every time, so the destination needs no initialisation.
__global__ void __launch_bounds__(256)
    stem_relayout_kernel(const uint4* __restrict__ x, int B, int H, int W, int ph, int pw,
                         int planes, int Hq, int Wq, uint4* __restrict__ y) {
  // one CTA per padded row (plane q, image b, row hq); threads walk its Wq pixels
  const int row = blockIdx.x;  // (q * B + b) * Hq + hq
  const int hq = row % Hq;
  const int bq = row / Hq;
  const int q = bq / B;
  const int b = bq - q * B;
  const int ih = hq - ph;
  const bool hok = ih >= 0 && ih < H;
  const uint4* xr = x + (static_cast<int64_t>(b) * H + (hok ? ih : 0)) * W;
  uint4* yr = y + static_cast<int64_t>(row) * Wq;
  for (int j = threadIdx.x; j < Wq; j += blockDim.x) {
    const int iw = planes ? 2 * j + q - pw : j - pw;
    yr[j] = (hok && iw >= 0 && iw < W) ? xr[iw] : make_uint4(0, 0, 0, 0);
  }
}

cudaError_t k_stem_relayout(const __nv_bfloat16* x, int B, int H, int W, int ph, int pw, int mode,
                            int Hq, int Wq, __nv_bfloat16* y, cudaStream_t s) {
  const int planes = mode == kAModeStemPlanes ? 1 : 0;
  const int rows = (planes ? 2 : 1) * B * Hq;
  if (rows == 0 || Wq == 0) return cudaSuccess;
  stem_relayout_kernel<<<rows, 256, 0, s>>>(reinterpret_cast<const uint4*>(x), B, H, W, ph, pw,
                                            planes, Hq, Wq, reinterpret_cast<uint4*>(y));
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K4 pooling / BN-ReLU

struct Vec8 {
  float v[8];
};

__device__ __forceinline__ Vec8 load8(const __nv_bfloat16* p) {
  uint4 q = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&q);
  Vec8 r;
#pragma unroll
  for (int j = 0; j < 8; ++j) r.v[j] = __bfloat162float(h[j]);
  return r;
}
__device__ __forceinline__ void store8(__nv_bfloat16* p, const Vec8& r) {
  __align__(16) __nv_bfloat16 h[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) h[j] = __float2bfloat16_rn(r.v[j]);
  *reinterpret_cast<uint4*>(p) = *reinterpret_cast<uint4*>(h);
}
__device__ __forceinline__ void bnrelu8(Vec8& r, const float* scale, const float* shift, int c) {
#pragma unroll
  for (int j = 0; j < 8; ++j) r.v[j] = fmaxf(fmaf(r.v[j], __ldg(scale + c + j), __ldg(shift + c + j)), 0.f);
}

// mode 0 = max (padding ignored), 1 = avg count_include_pad, 2 = avg exclude pad.
// Optional per-channel BN-ReLU applied to every input element before pooling.
// One CTA per output row (image b, row oh); the CTA size is a multiple of the number
// of 8-channel groups, so each thread keeps one channel group (and its BN-ReLU
// constants, in registers) for the whole row and walks output columns -- 32-bit
// index math only.  The window loop is unrolled for the common K = 2 / 3 so all
// window loads are in flight together.
template <int KT>
__global__ void __launch_bounds__(256)
    pool_kernel(const __nv_bfloat16* __restrict__ x, int ldx, __nv_bfloat16* __restrict__ y,
                int ldy, int y_off, int H, int W, int C, int Ho, int Wo, int kdyn, int s, int pad,
                int mode, const float* __restrict__ scale, const float* __restrict__ shift) {
  const int k = KT > 0 ? KT : kdyn;
  const int cg = C >> 3;
  const int b = blockIdx.x / Ho;
  const int oh = blockIdx.x - b * Ho;
  const int per = blockDim.x / cg;  // output columns per pass (blockDim is a multiple of cg)
  const int c = static_cast<int>(threadIdx.x % cg) * 8;
  const int ow0 = static_cast<int>(threadIdx.x / cg);
  if (ow0 >= per) return;
  float sc[8], sf[8];
  if (scale) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      sc[j] = __ldg(scale + c + j);
      sf[j] = __ldg(shift + c + j);
    }
  }
  const __nv_bfloat16* xb = x + static_cast<int64_t>(b) * H * W * ldx + c;
  __nv_bfloat16* yb = y + (static_cast<int64_t>(b) * Ho + oh) * Wo * ldy + y_off + c;
  const int ih0 = oh * s - pad;
  for (int ow = ow0; ow < Wo; ow += per) {
    Vec8 acc;
#pragma unroll
    for (int j = 0; j < 8; ++j) acc.v[j] = (mode == 0) ? -INFINITY : 0.f;
    int cnt = 0;
    const int iw0 = ow * s - pad;
#pragma unroll
    for (int dh = 0; dh < (KT > 0 ? KT : 8); ++dh) {
      if (KT == 0 && dh >= k) break;
      const int ih = ih0 + dh;
#pragma unroll
      for (int dw = 0; dw < (KT > 0 ? KT : 8); ++dw) {
        if (KT == 0 && dw >= k) break;
        const int iw = iw0 + dw;
        if (ih < 0 || ih >= H || iw < 0 || iw >= W) continue;
        Vec8 v = load8(xb + (ih * W + iw) * ldx);
        if (scale) {
#pragma unroll
          for (int j = 0; j < 8; ++j) v.v[j] = fmaxf(fmaf(v.v[j], sc[j], sf[j]), 0.f);
        }
        ++cnt;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          acc.v[j] = (mode == 0) ? fmaxf(acc.v[j], v.v[j]) : acc.v[j] + v.v[j];
      }
    }
    if (mode == 1) {
      const float inv = 1.f / static_cast<float>(k * k);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc.v[j] *= inv;
    } else if (mode == 2) {
      const float inv = 1.f / static_cast<float>(cnt > 0 ? cnt : 1);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc.v[j] *= inv;
    }
    store8(yb + ow * ldy, acc);
  }
}

// K x K windows with the mode and the BN-ReLU fixed at compile time: every window load
// of a thread is issued (predicated, clamped address) before any is used, so a thread
// keeps K*K 16-byte loads in flight.  Same CTA/row mapping as pool_kernel.
__device__ __forceinline__ void unpack8(const uint4& q, float* f) {
  const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    f[2 * e] = __uint_as_float(w[e] << 16);
    f[2 * e + 1] = __uint_as_float(w[e] & 0xffff0000u);
  }
}
template <int K, int MODE, bool PRE>
__global__ void __launch_bounds__(256)
    pool_fixed_kernel(const __nv_bfloat16* __restrict__ x, int ldx, __nv_bfloat16* __restrict__ y,
                      int ldy, int y_off, int H, int W, int C, int Ho, int Wo, int s, int pad,
                      const float* __restrict__ scale, const float* __restrict__ shift) {
  const int cg = C >> 3;
  const int b = blockIdx.x / Ho;
  const int oh = blockIdx.x - b * Ho;
  const int per = blockDim.x / cg;
  const int c = static_cast<int>(threadIdx.x % cg) * 8;
  const int ow0 = static_cast<int>(threadIdx.x / cg);
  if (ow0 >= per) return;
  float sc[8], sf[8];
  if (PRE) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      sc[j] = __ldg(scale + c + j);
      sf[j] = __ldg(shift + c + j);
    }
  }
  const __nv_bfloat16* xb = x + static_cast<int64_t>(b) * H * W * ldx + c;
  __nv_bfloat16* yb = y + (static_cast<int64_t>(b) * Ho + oh) * Wo * ldy + y_off + c;
  const int ih0 = oh * s - pad;
  for (int ow = ow0; ow < Wo; ow += per) {
    const int iw0 = ow * s - pad;
    uint4 raw[K * K];
    bool ok[K * K];
#pragma unroll
    for (int dh = 0; dh < K; ++dh) {
#pragma unroll
      for (int dw = 0; dw < K; ++dw) {
        const int ih = ih0 + dh, iw = iw0 + dw;
        const bool v = ih >= 0 && ih < H && iw >= 0 && iw < W;
        ok[dh * K + dw] = v;
        const int off = v ? (ih * W + iw) * ldx : 0;
        raw[dh * K + dw] = *reinterpret_cast<const uint4*>(xb + off);
      }
    }
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = MODE == 0 ? -INFINITY : 0.f;
    int cnt = 0;
#pragma unroll
    for (int t = 0; t < K * K; ++t) {
      float f[8];
      unpack8(raw[t], f);
      if (PRE) {
#pragma unroll
        for (int j = 0; j < 8; ++j) f[j] = fmaxf(fmaf(f[j], sc[j], sf[j]), 0.f);
      }
      if (ok[t]) {
        ++cnt;
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = MODE == 0 ? fmaxf(acc[j], f[j]) : acc[j] + f[j];
      }
    }
    if (MODE != 0) {
      const float inv = MODE == 1 ? 1.f / static_cast<float>(K * K) : 1.f / static_cast<float>(cnt > 0 ? cnt : 1);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] *= inv;
    }
    Vec8 r;
#pragma unroll
    for (int j = 0; j < 8; ++j) r.v[j] = acc[j];
    store8(yb + ow * ldy, r);
  }
}

template <int K>
static void launch_pool_fixed(int mode, bool pre, int rows, int threads, cudaStream_t st,
                              const __nv_bfloat16* x, int ldx, __nv_bfloat16* y, int ldy, int y_off,
                              int H, int W, int C, int Ho, int Wo, int s, int pad, const float* scale,
                              const float* shift) {
#define EB_POOL_LAUNCH(M, P)                                                                    \
  pool_fixed_kernel<K, M, P><<<rows, threads, 0, st>>>(x, ldx, y, ldy, y_off, H, W, C, Ho, Wo, s, \
                                                       pad, scale, shift)
  if (mode == 0) {
    if (pre) EB_POOL_LAUNCH(0, true); else EB_POOL_LAUNCH(0, false);
  } else if (mode == 1) {
    if (pre) EB_POOL_LAUNCH(1, true); else EB_POOL_LAUNCH(1, false);
  } else {
    if (pre) EB_POOL_LAUNCH(2, true); else EB_POOL_LAUNCH(2, false);
  }
#undef EB_POOL_LAUNCH
}

cudaError_t k_pool(const __nv_bfloat16* x, int ldx, __nv_bfloat16* y, int ldy, int y_off, int B,
                   int H, int W, int C, int Ho, int Wo, int k, int s, int pad, int mode,
                   const float* scale, const float* shift, cudaStream_t st) {
  if (static_cast<int64_t>(B) * Ho * Wo * (C / 8) == 0) return cudaSuccess;
  if (k > 8 || C % 8 != 0 || C / 8 > 256) return cudaErrorInvalidValue;
  // in-image offsets are 32-bit
  if (static_cast<int64_t>(H) * W * ldx >= (1ll << 31)) return cudaErrorInvalidValue;
  const int cg = C / 8;
  const int threads = (256 / cg) * cg;
  const int rows = B * Ho;
  if (k == 2 && mode >= 0 && mode <= 2)
    launch_pool_fixed<2>(mode, scale != nullptr, rows, threads, st, x, ldx, y, ldy, y_off, H, W, C,
                         Ho, Wo, s, pad, scale, shift);
  else if (k == 3 && mode >= 0 && mode <= 2)
    launch_pool_fixed<3>(mode, scale != nullptr, rows, threads, st, x, ldx, y, ldy, y_off, H, W, C,
                         Ho, Wo, s, pad, scale, shift);
  else
    pool_kernel<0><<<rows, threads, 0, st>>>(x, ldx, y, ldy, y_off, H, W, C, Ho, Wo, k, s, pad,
                                             mode, scale, shift);
  return cudaGetLastError();
}

// y[m, c] = relu(x[m, c] * scale[c] + shift[c]) for c < C (DenseNet pre-activation).
__global__ void bnrelu_kernel(const __nv_bfloat16* __restrict__ x, int ldx,
                              __nv_bfloat16* __restrict__ y, int ldy, int64_t M, int C,
                              const float* __restrict__ scale, const float* __restrict__ shift) {
  const int cg = C / 8;
  const int64_t total = M * cg;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % cg) * 8;
    const int64_t m = i / cg;
    Vec8 v = load8(x + m * ldx + c);
    bnrelu8(v, scale, shift, c);
    store8(y + m * ldy + c, v);
  }
}

cudaError_t k_bnrelu(const __nv_bfloat16* x, int ldx, __nv_bfloat16* y, int ldy, int64_t M, int C,
                     const float* scale, const float* shift, cudaStream_t st) {
  const int64_t total = M * (C / 8);
  if (total == 0) return cudaSuccess;
  bnrelu_kernel<<<grid_for(total, 256), 256, 0, st>>>(x, ldx, y, ldy, M, C, scale, shift);
  return cudaGetLastError();
}

// Global average pool over H*W (optionally BN-ReLU first) -> bf16 [B, C].
__global__ void gap_kernel(const __nv_bfloat16* __restrict__ x, int ldx,
                           __nv_bfloat16* __restrict__ y, int B, int HW, int C,
                           const float* __restrict__ scale, const float* __restrict__ shift) {
  const int cg = C / 8;
  const int64_t total = static_cast<int64_t>(B) * cg;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % cg) * 8;
    const int64_t b = i / cg;
    Vec8 acc;
#pragma unroll
    for (int j = 0; j < 8; ++j) acc.v[j] = 0.f;
    // 8 pixels' loads in flight per step (the sum keeps its sequential order); the BN-ReLU
    // constants of the thread's 8 channels are loaded once
    float sc[8], sh[8];
    if (scale) {
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        sc[jj] = __ldg(scale + c + jj);
        sh[jj] = __ldg(shift + c + jj);
      }
    }
    const __nv_bfloat16* xb = x + b * HW * ldx + c;
    for (int p0 = 0; p0 < HW; p0 += 8) {
      uint4 q[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (p0 + u < HW) q[u] = __ldg(reinterpret_cast<const uint4*>(xb + static_cast<int64_t>(p0 + u) * ldx));
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (p0 + u >= HW) break;
        const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&q[u]);
        Vec8 v;
#pragma unroll
        for (int j = 0; j < 8; ++j) v.v[j] = __bfloat162float(h[j]);
        if (scale) {
#pragma unroll
          for (int j = 0; j < 8; ++j) v.v[j] = fmaxf(fmaf(v.v[j], sc[j], sh[j]), 0.f);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) acc.v[j] += v.v[j];
      }
    }
    const float inv = 1.f / static_cast<float>(HW);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc.v[j] *= inv;
    store8(y + b * C + c, acc);
  }
}

cudaError_t k_gap(const __nv_bfloat16* x, int ldx, __nv_bfloat16* y, int B, int HW, int C,
                  const float* scale, const float* shift, cudaStream_t st) {
  const int64_t total = static_cast<int64_t>(B) * (C / 8);
  if (total == 0) return cudaSuccess;
  gap_kernel<<<grid_for(total, 128), 128, 0, st>>>(x, ldx, y, B, HW, C, scale, shift);
  return cudaGetLastError();
}

// Bilinear resize of an NHWC bf16 image (align_corners=False, no antialias: the
// semantics of torch.nn.functional.interpolate(mode="bilinear")), 8 channels per thread.
// K1's second output for members whose native resolution differs from the request's.
__global__ void resize_bilinear_kernel(const __nv_bfloat16* __restrict__ x, int ldx,
                                       __nv_bfloat16* __restrict__ y, int ldy, int B, int H, int W,
                                       int C, int Ho, int Wo) {
  const int cg = C / 8;
  const int64_t total = static_cast<int64_t>(B) * Ho * Wo * cg;
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= total) return;
  const int c = static_cast<int>(i % cg) * 8;
  int64_t t = i / cg;
  const int ox = static_cast<int>(t % Wo);
  t /= Wo;
  const int oy = static_cast<int>(t % Ho);
  const int b = static_cast<int>(t / Ho);
  const float sy = fmaxf((oy + 0.5f) * (static_cast<float>(H) / Ho) - 0.5f, 0.f);
  const float sx = fmaxf((ox + 0.5f) * (static_cast<float>(W) / Wo) - 0.5f, 0.f);
  const int y0 = min(static_cast<int>(sy), H - 1), x0 = min(static_cast<int>(sx), W - 1);
  const int y1 = min(y0 + 1, H - 1), x1 = min(x0 + 1, W - 1);
  const float ly = sy - y0, lx = sx - x0;
  const __nv_bfloat16* xb = x + static_cast<int64_t>(b) * H * W * ldx + c;
  const Vec8 a = load8(xb + (static_cast<int64_t>(y0) * W + x0) * ldx);
  const Vec8 bq = load8(xb + (static_cast<int64_t>(y0) * W + x1) * ldx);
  const Vec8 cq = load8(xb + (static_cast<int64_t>(y1) * W + x0) * ldx);
  const Vec8 d = load8(xb + (static_cast<int64_t>(y1) * W + x1) * ldx);
  Vec8 o;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float top = a.v[j] + lx * (bq.v[j] - a.v[j]);
    const float bot = cq.v[j] + lx * (d.v[j] - cq.v[j]);
    o.v[j] = top + ly * (bot - top);
  }
  store8(y + (static_cast<int64_t>(b) * Ho * Wo + static_cast<int64_t>(oy) * Wo + ox) * ldy + c, o);
}

cudaError_t k_resize_bilinear(const __nv_bfloat16* x, int ldx, __nv_bfloat16* y, int ldy, int B,
                              int H, int W, int C, int Ho, int Wo, cudaStream_t st) {
  const int64_t total = static_cast<int64_t>(B) * Ho * Wo * (C / 8);
  if (total == 0) return cudaSuccess;
  resize_bilinear_kernel<<<(total + 255) / 256, 256, 0, st>>>(x, ldx, y, ldy, B, H, W, C, Ho, Wo);
  return cudaGetLastError();
}

// Split-K finalisation: y = act(sum_z ws[z] + bias), slices added in ascending z
// (deterministic, independent of scheduling) -> bf16 slice or fp32.
__global__ void splitk_finalize_kernel(const float* __restrict__ ws, int splits, int64_t M, int N,
                                       const float* __restrict__ bias, int relu, void* out,
                                       int ldo, int out_off, int out_f32) {
  const int64_t total = M * N;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int n = static_cast<int>(i % N);
    const int64_t m = i / N;
    float v = 0.f;
    for (int z = 0; z < splits; ++z) v += ws[z * total + i];
    if (bias) v += bias[n];
    if (relu) v = fmaxf(v, 0.f);
    if (out_f32)
      reinterpret_cast<float*>(out)[m * ldo + out_off + n] = v;
    else
      reinterpret_cast<__nv_bfloat16*>(out)[m * ldo + out_off + n] = __float2bfloat16_rn(v);
  }
}

// 4 columns per thread (float4 partial loads, all slices' loads in flight together),
// one wave of CTAs striding over the elements: the one-element-per-thread version was
// bound by launching CTAs (FC 256 x 4096, 4 slices: 14.7 us)
__global__ void __launch_bounds__(256)
    splitk_finalize4_kernel(const float4* __restrict__ ws, int splits, int total4, int N4,
                            const float* __restrict__ bias, int relu, void* out, int ldo,
                            int out_off, int out_f32) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total4; i += gridDim.x * blockDim.x) {
    const int m = i / N4;
    const int n = (i - m * N4) * 4;
    float4 v = ws[i];
    for (int z = 1; z < splits; ++z) {
      const float4 w = ws[static_cast<int64_t>(z) * total4 + i];
      v.x += w.x;
      v.y += w.y;
      v.z += w.z;
      v.w += w.w;
    }
    if (bias) {
      v.x += bias[n];
      v.y += bias[n + 1];
      v.z += bias[n + 2];
      v.w += bias[n + 3];
    }
    if (relu) {
      v.x = fmaxf(v.x, 0.f);
      v.y = fmaxf(v.y, 0.f);
      v.z = fmaxf(v.z, 0.f);
      v.w = fmaxf(v.w, 0.f);
    }
    const int64_t o = static_cast<int64_t>(m) * ldo + out_off + n;
    if (out_f32) {
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + o) = v;
    } else {
      __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
      uint2 u;
      u.x = *reinterpret_cast<uint32_t*>(&a);
      u.y = *reinterpret_cast<uint32_t*>(&b);
      *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(out) + o) = u;
    }
  }
}

cudaError_t k_splitk_finalize(const float* ws, int splits, int64_t M, int N, const float* bias,
                              int relu, void* out, int ldo, int out_off, int out_f32,
                              cudaStream_t st) {
  const int64_t total = M * N;
  if (total == 0) return cudaSuccess;
  if (N % 4 == 0 && ldo % 4 == 0 && out_off % 4 == 0 && total / 4 < (1ll << 31) &&
      (reinterpret_cast<uintptr_t>(ws) & 15) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
    const int total4 = static_cast<int>(total / 4);
    const int grid = std::min((total4 + 255) / 256, 148 * 8);
    splitk_finalize4_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const float4*>(ws), splits, total4,
                                                  N / 4, bias, relu, out, ldo, out_off, out_f32);
    return cudaGetLastError();
  }
  splitk_finalize_kernel<<<grid_for(total, 256), 256, 0, st>>>(ws, splits, M, N, bias, relu, out,
                                                               ldo, out_off, out_f32);
  return cudaGetLastError();
}

}  // namespace eb
