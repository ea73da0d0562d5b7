// eb_internal.h -- types shared by the kernels and the native runtime.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

namespace eb {

enum AMode : int {
  kAModeTiled = 0,     // A is a plain [M, K] matrix (1x1 stride-1 conv, FC)
  kAModeIm2col = 1,    // TMA im2col, 64-channel chunks, 128B swizzle
  kAModeGatherC8 = 2,  // stem (Cin <= 8): cp.async gather, one K block per filter row
  kAModeTapShift = 3,  // 3-wide stride-1 filters: one load per filter row, taps by row shift
  kAModeTapC8 = 4,     // stem (Cin <= 8): per filter row, one TMA im2col load of 8-channel
                       // pixels per horizontal tap into a no-swizzle K-major tile
  kAModeTapN = 5,      // 3-wide stride-1 filters, Cout <= 64: the 3 taps stacked along N
};

enum OutMode : int {
  kOutBF16 = 0,       // bf16 NHWC slice, bias/residual/ReLU fused
  kOutF32 = 1,        // fp32 (logits), bias/ReLU fused
  kOutPartialF32 = 2,  // fp32 split-K partial of slice blockIdx.z (deterministic reduce after)
};

struct ConvParams {
  int M, N;
  int num_kb, kb_per_split;
  int a_mode;
  int Ho, Wo, sh, sw, ph, pw, kw, taps, cchunks;
  int H, W;                  // input geometry (gather mode)
  int Wp;                    // padded-grid width (tap-shift mode): Wo + kw - 1
  int grouped;               // grouped conv: N tile t reads input channels [t*BN, t*BN + BN)
  int n_split;               // grouped launch: columns >= n_split are stored through map_res
  int mcast;                 // 2-CTA cluster: M-tile pairs share the B tile via TMA multicast
  int pair;                  // with mcast: 2-SM MMA (cta_group::2), M = 256 per CTA pair
  int resb;                  // single N tile: all K blocks of B resident in smem (loaded once)
  const __nv_bfloat16* x;    // input base (gather mode), NHWC with 8 channels
  void* out;
  int ldo, out_off;
  const __nv_bfloat16* res;
  int ldr;
  const float* bias;
  int relu;
  int out_mode;
  int vec_ok;  // 16-byte aligned rows/offsets: vector epilogue stores allowed
  // optional pre-activation on A (DenseNet BN-ReLU on the concatenated input):
  // a = relu(a * pre_scale[k] + pre_shift[k]); arrays padded with zeros to 64
  const float* pre_scale;
  const float* pre_shift;
};

cudaError_t conv_umma_launch(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mo,
                             const CUtensorMap& mr, const ConvParams& p, int block_n, int grid,
                             cudaStream_t stream);
int conv_umma_chunk(int block_n);
// pipeline stages the kernel instance for this plan would get (host-side layout query)
int conv_umma_stages(const ConvParams& p, int block_n);

// Driver entry point for tensor-map encoding (resolved through the runtime so the
// library does not link libcuda directly).
bool encode_tiled_2d_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                          uint64_t ld_elems, uint32_t box_inner, uint32_t box_outer,
                          std::string* err, int swizzle_bytes = 128);
bool encode_im2col_bf16(CUtensorMap* map, const void* base, int n, int h, int w, int c, int ldc,
                        int kh, int kw, int sh, int sw, int ph, int pw, int chans_per_pixel,
                        int pixels, bool swizzle128, std::string* err, int upper_w_extra = 0);

void set_error(const std::string& msg);

}  // namespace eb
