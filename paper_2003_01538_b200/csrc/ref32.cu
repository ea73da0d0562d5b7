// ref32.cu -- the fp32-faithful parity mode (EB_PREC_F32): every CNN op in fp32 on the
// CUDA cores, so that top-k class indices reproduce the fp32 CPU oracle on every sample
// ("an fp32-faithful parity mode with bf16 operands off").
//
// Same op list, same NHWC activation layout (row stride ld, channel slices) as the bf16
// tcgen05 path; only the element type and the kernels differ.  Every dot product is a
// sequential fp32 FFMA chain over K in (filter row, filter column, channel) order, so the
// result of a sample never depends on its batch or on the launch geometry.  The reference
// arithmetic this restates is torchvision's fp32 eager CPU forward (oracle/cnn.py); the
// only differences are summation order and BN folded into the conv weights (both at the
// 1e-6 relative level).
//
// Weights: fp32 [Cout][kh][kw][Cin_g] (packing.pack_conv_weight_f32); an FC after a
// feature map (flatten) is [Cout][H*W*C] in NHWC order, i.e. a 1x1 conv over one
// H*W*C-channel pixel.
#include <cuda_runtime.h>

#include <cstdint>

#include "eb_kernels.h"

namespace eb {

namespace {

inline int grid_for32(int64_t work, int threads) {
  int64_t g = (work + threads - 1) / threads;
  if (g > 148 * 64) g = 148 * 64;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

// ------------------------------------------------------------------ preprocess

// u8 HWC -> fp32 NHWC with channels zero-padded to cpad, through the exact LUT
// (packing.u8_lut: eg/wire.py:71 then eg/models.py:254-259).
__global__ void pre32_u8_kernel(const uint8_t* __restrict__ x, float* __restrict__ y,
                                int64_t pixels, int C, int cpad, const float* __restrict__ lut) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < pixels;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x)
    for (int c = 0; c < cpad; ++c) y[p * cpad + c] = c < C ? __ldg(lut + c * 256 + x[p * C + c]) : 0.f;
}

// f32 CHW (already / pixel_scale) -> (x - mean) / std in the reference's op order -> NHWC.
__global__ void pre32_f32chw_kernel(const float* __restrict__ x, float* __restrict__ y,
                                    int64_t pixels, int C, int64_t plane, int cpad,
                                    const float* __restrict__ mean, const float* __restrict__ stdv,
                                    int nms) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < pixels;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = p / plane;
    const int64_t q = p - b * plane;
    for (int c = 0; c < cpad; ++c) {
      float f = 0.f;
      if (c < C) {
        const int mc = nms == 1 ? 0 : c;
        f = __fdiv_rn(__fsub_rn(x[(b * C + c) * plane + q], mean[mc]), stdv[mc]);
      }
      y[p * cpad + c] = f;
    }
  }
}

// ------------------------------------------------------------------ convolution

struct Conv32 {
  const float* x;  // first channel of the source slice
  int H, W, ldx, cin_g;
  const float* w;  // [cout][kh][kw][cin_g]
  const float* bias;
  const float* res;
  int ldr;
  float* y;
  int ldy, y_off;
  float* y2;
  int ldy2, y2_off, n_split;
  int cout_g, kh, kw, sh, sw, ph, pw, Ho, Wo, relu;
  const float* pre_scale;  // per source channel (ungrouped convs only)
  const float* pre_shift;
  int K;      // kh * kw * cin_g
  int64_t M;  // B * Ho * Wo
};

constexpr int kTM = 64, kTN = 64, kTK = 16;

// Implicit GEMM on the CUDA cores: a 64 x 64 output tile per CTA (blockIdx.z = group),
// 256 threads with 4 x 4 outputs each, K staged 16 at a time through shared memory.
// Thread t loads A rows m = t/16 + 16 i (k = t % 16, consecutive channels: coalesced) and
// B columns n = t/16 + 16 j; it computes rows ty + 16 i, columns tx + 16 j.
__global__ void __launch_bounds__(256) conv32_kernel(Conv32 p) {
  __shared__ float As[kTK][kTM + 4];
  __shared__ float Bs[kTK][kTN + 4];
  const int t = threadIdx.x;
  const int tx = t & 15, ty = t >> 4;
  const int g = blockIdx.z;
  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * kTM;
  const int n0 = blockIdx.y * kTN;
  // the 4 A rows this thread loads
  const float* xrow[4];
  int ih0[4], iw0[4];
  bool mval[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = m0 + ty + 16 * i;
    mval[i] = m < p.M;
    const int64_t mm = mval[i] ? m : 0;
    const int wo = static_cast<int>(mm % p.Wo);
    const int64_t r = mm / p.Wo;
    const int ho = static_cast<int>(r % p.Ho);
    const int64_t b = r / p.Ho;
    xrow[i] = p.x + b * p.H * p.W * p.ldx + static_cast<int64_t>(g) * p.cin_g;
    ih0[i] = ho * p.sh - p.ph;
    iw0[i] = wo * p.sw - p.pw;
  }
  const float* wbase = p.w + static_cast<int64_t>(g) * p.cout_g * p.K;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < p.K; k0 += kTK) {
    const int k = k0 + tx;
    const bool kval = k < p.K;
    int c = 0, r = 0, s = 0;
    if (kval) {
      c = k % p.cin_g;
      const int rs = k / p.cin_g;
      s = rs % p.kw;
      r = rs / p.kw;
    }
    float sc = 1.f, sf = 0.f;
    if (p.pre_scale && kval) {
      sc = __ldg(p.pre_scale + c);
      sf = __ldg(p.pre_shift + c);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float v = 0.f;
      const int ih = ih0[i] + r, iw = iw0[i] + s;
      if (kval && mval[i] && ih >= 0 && ih < p.H && iw >= 0 && iw < p.W) {
        v = __ldg(xrow[i] + (static_cast<int64_t>(ih) * p.W + iw) * p.ldx + c);
        if (p.pre_scale) v = fmaxf(fmaf(v, sc, sf), 0.f);
      }
      As[tx][ty + 16 * i] = v;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + ty + 16 * j;
      Bs[tx][ty + 16 * j] = (kval && n < p.cout_g) ? __ldg(wbase + static_cast<int64_t>(n) * p.K + k) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kTK; ++kk) {
      float a[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = m0 + ty + 16 * i;
    if (m >= p.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int nl = n0 + tx + 16 * j;
      if (nl >= p.cout_g) continue;
      const int n = g * p.cout_g + nl;
      float v = acc[i][j];
      if (p.bias) v += __ldg(p.bias + n);
      if (p.res) v += __ldg(p.res + m * p.ldr + n);
      if (p.relu) v = fmaxf(v, 0.f);
      if (p.n_split > 0 && n >= p.n_split)
        p.y2[m * p.ldy2 + p.y2_off + (n - p.n_split)] = v;
      else
        p.y[m * p.ldy + p.y_off + n] = v;
    }
  }
}

// ------------------------------------------------------------------ pooling etc.

// One thread per output element.  mode 0 max (padding ignored), 1 avg with the padded
// window count (torch count_include_pad=True), 2 avg over valid elements; the sum runs in
// row-major window order and is divided once, as torch's CPU kernel does.
__global__ void pool32_kernel(const float* __restrict__ x, int ldx, float* __restrict__ y, int ldy,
                              int y_off, int B, int H, int W, int C, int Ho, int Wo, int k, int s,
                              int pad, int mode, const float* __restrict__ scale,
                              const float* __restrict__ shift) {
  const int64_t total = static_cast<int64_t>(B) * Ho * Wo * C;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % C);
    int64_t q = i / C;
    const int ow = static_cast<int>(q % Wo);
    q /= Wo;
    const int oh = static_cast<int>(q % Ho);
    const int64_t b = q / Ho;
    const float sc = scale ? __ldg(scale + c) : 1.f, sf = scale ? __ldg(shift + c) : 0.f;
    float acc = mode == 0 ? -INFINITY : 0.f;
    int cnt = 0;
    const int hs = oh * s - pad, ws = ow * s - pad;
    for (int dh = 0; dh < k; ++dh) {
      const int ih = hs + dh;
      if (ih < 0 || ih >= H) continue;
      for (int dw = 0; dw < k; ++dw) {
        const int iw = ws + dw;
        if (iw < 0 || iw >= W) continue;
        float v = __ldg(x + ((b * H + ih) * W + iw) * ldx + c);
        if (scale) v = fmaxf(fmaf(v, sc, sf), 0.f);
        acc = mode == 0 ? fmaxf(acc, v) : acc + v;
        ++cnt;
      }
    }
    if (mode == 1) {
      // torch: the window clipped to the padded input
      const int he = min(hs + k, H + pad), we = min(ws + k, W + pad);
      acc = acc / static_cast<float>((he - hs) * (we - ws));
    } else if (mode == 2) {
      acc = acc / static_cast<float>(cnt > 0 ? cnt : 1);
    }
    y[((b * Ho + oh) * Wo + ow) * ldy + y_off + c] = acc;
  }
}

__global__ void bnrelu32_kernel(const float* __restrict__ x, int ldx, float* __restrict__ y,
                                int ldy, int64_t M, int C, const float* __restrict__ scale,
                                const float* __restrict__ shift) {
  const int64_t total = M * C;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % C);
    const int64_t m = i / C;
    y[m * ldy + c] = fmaxf(fmaf(x[m * ldx + c], __ldg(scale + c), __ldg(shift + c)), 0.f);
  }
}

// Global average pool: sequential fp32 sum over the H*W positions, one division.
__global__ void gap32_kernel(const float* __restrict__ x, int ldx, float* __restrict__ y, int B,
                             int HW, int C, const float* __restrict__ scale,
                             const float* __restrict__ shift) {
  const int64_t total = static_cast<int64_t>(B) * C;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % C);
    const int64_t b = i / C;
    const float sc = scale ? __ldg(scale + c) : 1.f, sf = scale ? __ldg(shift + c) : 0.f;
    const float* xb = x + b * HW * ldx + c;
    float acc = 0.f;
    for (int q = 0; q < HW; ++q) {
      float v = __ldg(xb + static_cast<int64_t>(q) * ldx);
      if (scale) v = fmaxf(fmaf(v, sc, sf), 0.f);
      acc += v;
    }
    y[b * C + c] = acc / static_cast<float>(HW);
  }
}

// Bilinear, align_corners=False, no antialias, in torch's CPU formula: source index
// (dst + 0.5) * in/out - 0.5 clamped at 0, lambdas l1 = src - i0, l0 = 1 - l1,
// out = h0 * (w0 * a + w1 * b) + h1 * (w0 * c + w1 * d).
__global__ void resize32_kernel(const float* __restrict__ x, int ldx, float* __restrict__ y,
                                int ldy, int B, int H, int W, int C, int Ho, int Wo) {
  const int64_t total = static_cast<int64_t>(B) * Ho * Wo * C;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % C);
    int64_t q = i / C;
    const int ox = static_cast<int>(q % Wo);
    q /= Wo;
    const int oy = static_cast<int>(q % Ho);
    const int64_t b = q / Ho;
    const float sy = fmaxf((oy + 0.5f) * (static_cast<float>(H) / Ho) - 0.5f, 0.f);
    const float sx = fmaxf((ox + 0.5f) * (static_cast<float>(W) / Wo) - 0.5f, 0.f);
    const int y0 = min(static_cast<int>(sy), H - 1), x0 = min(static_cast<int>(sx), W - 1);
    const int yp = y0 < H - 1 ? 1 : 0, xp = x0 < W - 1 ? 1 : 0;
    const float h1 = sy - y0, h0 = 1.f - h1, w1 = sx - x0, w0 = 1.f - w1;
    const float* xb = x + b * H * W * ldx + c;
    const float a = xb[(static_cast<int64_t>(y0) * W + x0) * ldx];
    const float bq = xb[(static_cast<int64_t>(y0) * W + x0 + xp) * ldx];
    const float cq = xb[(static_cast<int64_t>(y0 + yp) * W + x0) * ldx];
    const float d = xb[(static_cast<int64_t>(y0 + yp) * W + x0 + xp) * ldx];
    y[((b * Ho + oy) * Wo + ox) * ldy + c] = h0 * (w0 * a + w1 * bq) + h1 * (w0 * cq + w1 * d);
  }
}

}  // namespace

cudaError_t k32_preprocess_u8(const uint8_t* x, float* y, int B, int C, int64_t plane, int cpad,
                              const float* lut, cudaStream_t s) {
  const int64_t pixels = static_cast<int64_t>(B) * plane;
  if (pixels == 0) return cudaSuccess;
  pre32_u8_kernel<<<grid_for32(pixels, 256), 256, 0, s>>>(x, y, pixels, C, cpad, lut);
  return cudaGetLastError();
}

cudaError_t k32_preprocess_f32chw(const float* x, float* y, int B, int C, int64_t plane, int cpad,
                                  const float* mean, const float* stdv, int nms, cudaStream_t s) {
  const int64_t pixels = static_cast<int64_t>(B) * plane;
  if (pixels == 0) return cudaSuccess;
  pre32_f32chw_kernel<<<grid_for32(pixels, 256), 256, 0, s>>>(x, y, pixels, C, plane, cpad, mean,
                                                              stdv, nms);
  return cudaGetLastError();
}

cudaError_t k32_conv(const float* x, int B, int H, int W, int ldx, int cin, int groups,
                     const float* w, const float* bias, const float* res, int ldr, float* y,
                     int ldy, int y_off, float* y2, int ldy2, int y2_off, int n_split, int cout,
                     int kh, int kw, int sh, int sw, int ph, int pw, int relu, int flatten,
                     const float* pre_scale, const float* pre_shift, cudaStream_t s) {
  Conv32 p{};
  if (groups < 1 || cin % groups || cout % groups) return cudaErrorInvalidValue;
  if (flatten) {  // FC over an H x W x C map: one pixel of H*W*C channels (NHWC order)
    if (ldx != cin || groups != 1 || pre_scale) return cudaErrorInvalidValue;
    p.H = p.W = 1;
    p.cin_g = H * W * cin;
    p.ldx = p.cin_g;
    p.kh = p.kw = p.sh = p.sw = 1;
    p.ph = p.pw = 0;
  } else {
    p.H = H;
    p.W = W;
    p.cin_g = cin / groups;
    p.ldx = ldx;
    p.kh = kh;
    p.kw = kw;
    p.sh = sh;
    p.sw = sw;
    p.ph = ph;
    p.pw = pw;
  }
  if (pre_scale && groups != 1) return cudaErrorInvalidValue;
  p.Ho = (p.H + 2 * p.ph - p.kh) / p.sh + 1;
  p.Wo = (p.W + 2 * p.pw - p.kw) / p.sw + 1;
  p.M = static_cast<int64_t>(B) * p.Ho * p.Wo;
  p.K = p.kh * p.kw * p.cin_g;
  p.x = x;
  p.w = w;
  p.bias = bias;
  p.res = res;
  p.ldr = ldr;
  p.y = y;
  p.ldy = ldy;
  p.y_off = y_off;
  p.y2 = y2;
  p.ldy2 = ldy2;
  p.y2_off = y2_off;
  p.n_split = n_split;
  p.cout_g = cout / groups;
  p.relu = relu;
  p.pre_scale = pre_scale;
  p.pre_shift = pre_shift;
  if (p.M == 0) return cudaSuccess;
  const int64_t mt = (p.M + kTM - 1) / kTM;
  if (mt > 0x7fffffff) return cudaErrorInvalidValue;
  dim3 grid(static_cast<unsigned>(mt), (p.cout_g + kTN - 1) / kTN, groups);
  conv32_kernel<<<grid, 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t k32_pool(const float* x, int ldx, float* y, int ldy, int y_off, int B, int H, int W,
                     int C, int Ho, int Wo, int k, int s, int pad, int mode, const float* scale,
                     const float* shift, cudaStream_t st) {
  const int64_t total = static_cast<int64_t>(B) * Ho * Wo * C;
  if (total == 0) return cudaSuccess;
  pool32_kernel<<<grid_for32(total, 256), 256, 0, st>>>(x, ldx, y, ldy, y_off, B, H, W, C, Ho, Wo,
                                                        k, s, pad, mode, scale, shift);
  return cudaGetLastError();
}

cudaError_t k32_bnrelu(const float* x, int ldx, float* y, int ldy, int64_t M, int C,
                       const float* scale, const float* shift, cudaStream_t st) {
  if (M * C == 0) return cudaSuccess;
  bnrelu32_kernel<<<grid_for32(M * C, 256), 256, 0, st>>>(x, ldx, y, ldy, M, C, scale, shift);
  return cudaGetLastError();
}

cudaError_t k32_gap(const float* x, int ldx, float* y, int B, int HW, int C, const float* scale,
                    const float* shift, cudaStream_t st) {
  const int64_t total = static_cast<int64_t>(B) * C;
  if (total == 0) return cudaSuccess;
  gap32_kernel<<<grid_for32(total, 128), 128, 0, st>>>(x, ldx, y, B, HW, C, scale, shift);
  return cudaGetLastError();
}

cudaError_t k32_resize(const float* x, int ldx, float* y, int ldy, int B, int H, int W, int C,
                       int Ho, int Wo, cudaStream_t st) {
  const int64_t total = static_cast<int64_t>(B) * Ho * Wo * C;
  if (total == 0) return cudaSuccess;
  resize32_kernel<<<grid_for32(total, 256), 256, 0, st>>>(x, ldx, y, ldy, B, H, W, C, Ho, Wo);
  return cudaGetLastError();
}

}  // namespace eb
