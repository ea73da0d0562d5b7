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
  kAModeStemRows = 6,  // stem, stride 1: zero-padded 8-channel image, one contiguous load
                       // of 136 pixels per filter row; taps = overlapping core matrices
  kAModeStemPlanes = 7,  // stem, stride 2: even/odd padded column planes, two such loads
};

// Padded source layouts for the stem modes (written by k_stem_relayout).  A tile is 128
// consecutive positions of a per-image output grid of width Wg; rows of the grid with
// ow >= Wo (and positions past Ho) are computed and dropped.
//   rows   (stride 1): buffer [B][Hq][Wq][8], padded pixel (ih + ph, iw + pw); Wg = Wq
//   planes (stride 2): buffer [2][B][Hq][Wq][8], plane q holds padded columns 2j + q;
//                      Wg = 128 * ceil(Wo / 128)
#ifndef EB_STEM_ALIGN
#define EB_STEM_ALIGN 8  // rows mode: padded row width multiple (128: a tile never straddles rows)
#endif
struct StemGeom {
  int mode;        // kAModeStemRows / kAModeStemPlanes
  int Hq, Wq, Wg;  // padded rows / width per image, output grid width
  int Mi;          // output grid positions per image (multiple of 128)
  int64_t plane_px;  // pixels per plane (planes mode)
  int64_t bytes;
};
inline bool stem_geom(int B, int H, int W, int kh, int kw, int sh, int sw, int ph, int pw,
                      StemGeom* g) {
  if (kw > 8 || sh != sw || (sh != 1 && sh != 2)) return false;
  const int Ho = (H + 2 * ph - kh) / sh + 1;
  const int Wo = (W + 2 * pw - kw) / sw + 1;
  if (Ho <= 0 || Wo <= 0) return false;
  if (sh == 1) {
    g->mode = kAModeStemRows;
    // a multiple of 8: an epilogue warp's 32-row slab meets at most one grid-row boundary,
    // at an 8-row-aligned offset (the second part is stored in 8-row boxes); taps >= kw
    // meet zero weights
    g->Wq = (W + 2 * pw + EB_STEM_ALIGN - 1) / EB_STEM_ALIGN * EB_STEM_ALIGN;
    g->Wg = g->Wq;
    g->Mi = (Ho * g->Wg + 127) / 128 * 128;
    // the last tile's loads reach Mi - 1 + 7 + (kh - 1) * Wq
    g->Hq = (g->Mi + 8 + (kh - 1) * g->Wq + g->Wq - 1) / g->Wq;
    if (g->Hq < H + 2 * ph) g->Hq = H + 2 * ph;
    g->plane_px = static_cast<int64_t>(B) * g->Hq * g->Wq;
    g->bytes = g->plane_px * 16;
  } else {
    g->mode = kAModeStemPlanes;
    g->Wg = (Wo + 127) / 128 * 128;
    g->Wq = g->Wg + 8;                       // plane columns reach Wg - 1 + (kw - 1) / 2
    g->Mi = Ho * g->Wg;
    g->Hq = 2 * (Ho - 1) + kh;               // plane rows reach 2 (Ho - 1) + kh - 1
    if (g->Hq < H + 2 * ph) g->Hq = H + 2 * ph;
    g->plane_px = static_cast<int64_t>(B) * g->Hq * g->Wq;
    g->bytes = 2 * g->plane_px * 16;
  }
  return true;
}

enum OutMode : int {
  kOutBF16 = 0,       // bf16 NHWC slice, bias/residual/ReLU fused
  kOutF32 = 1,        // fp32 (logits), bias/ReLU fused
  kOutPartialF32 = 2,  // fp32 split-K partial of slice blockIdx.z (deterministic reduce after)
};

// Division by a run-time constant for 0 <= n < 2^31 (multiply-high + add + shift):
// s = ceil(log2 d), m = floor(2^32 (2^s - d) / d) + 1, q = (umulhi(n, m) + n) >> s.
struct FastDiv {
  uint32_t d, m, s;
};
inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f{d, 0, 0};
  if (d == 0) return f;
  while ((1ull << f.s) < d) ++f.s;
  f.m = static_cast<uint32_t>(((1ull << 32) * ((1ull << f.s) - d)) / d + 1);
  return f;
}
#ifdef __CUDACC__
__device__ __forceinline__ int fdiv(int n, const FastDiv& f) {
  const uint32_t t = __umulhi(static_cast<uint32_t>(n), f.m);
  return static_cast<int>((t + static_cast<uint32_t>(n)) >> f.s);
}
#endif

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
  int stem_tma;              // stem modes: epilogue stores 32-pixel slabs with a clipped 3-D map
  int kbs;                   // stem modes: filter rows (64-wide K blocks) per pipeline stage
  int early_release;         // epilogue frees the accumulator right after its TMEM loads
  int stem_lines;            // tall stems: lines of the one load per plane (0: a load per filter row)
  int tall_rows;             // tall taps-in-N: rows of the one A load per channel chunk (0: off)
  int ring_half;             // plain tiles, no residual: half the epilogue ring (one buffer per warp)
  int tapn_alt;              // taps-in-N, 64 columns: epilogue groups take alternate tiles
  int tapn2;                 // taps-in-N (unpaired): tap 2 folded into plane 0 by a 2-row A shift
  int pool2;                 // taps-in-N: 2x2/2 max-pool fused (out is the pooled tensor)
  int nseg, Ho2, Wo2;        // pool2: 60-column segments per row pair, pooled geometry
  int dbg;                   // timing experiments only (EB_DBG); 0 in production
  long long* trace;          // timing experiments only (EB_TRACE): per-role event clocks of CTA 0
  const __nv_bfloat16* x;    // input base (gather mode), NHWC with 8 channels
  int Wg, Mi, Hq, Wq;        // stem rows / planes modes (see StemGeom)
  // epilogue row decode, padded-grid modes: grid positions per image and per grid row
  // (tap-shift / taps-in-N: Ho * Wp and Wp; stems: Mi and Wg)
  FastDiv fd_img, fd_row;
  long long plane_px;
  void* out2;                // grouped launch, direct-store modes: columns >= n_split
  int ldo2, out2_off;
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

// VGG block 1 fused (block1.cu): conv3x3(3->64)+ReLU, conv3x3(64->64)+ReLU, 2x2/2 max-pool;
// input = the stem rows layout ([B][Hq][Wq][8], padding 1), output pooled NHWC
struct Block1Params {
  int H, W, Hq;                // image (= both convs' output) size; padded rows per image
  int bh, nbands, nseg;        // strips: image x band of bh rows x 120-column segment
  int strips;
  const float* bias1;          // conv1_1 bias [64]
  const float* bias2;          // conv1_2 bias [64]
  __nv_bfloat16* out;          // pooled [B][H/2][W/2][ldo] at channel offset out_off
  int ldo, out_off;
};
cudaError_t block1_launch(const CUtensorMap& mx, const CUtensorMap& mw1, const CUtensorMap& mw2,
                          const Block1Params& p, int grid, cudaStream_t stream);
bool pdl_enabled();

// 7x7/2 stem of one member or two (grouped) + the 3x3/2 (pad 1) max-pools (stem_pool.cu); input =
// the stem planes layout with the tall-box line map, output = the two pooled tensors
struct StemPoolParams {
  int ncol;                    // 64 (one member) or 128 (two)
  int Ho, Wo;                  // stem output size (Wo <= 128: one planes tile per row)
  int Hq, Wq;                  // padded rows per image / plane width of the planes layout
  long long plane_px;          // pixels per plane
  int lines;                   // 128-byte lines of one tall box (7 filter rows of a plane)
  int pb, nbands, strips;      // strips: image x band of pb pooled rows
  const float* bias;           // [128]: member 0's 64, then member 1's
  __nv_bfloat16* out0;         // member 0 pooled [B][Ho/2][Wo/2][ld0] at off0
  int ld0, off0;
  __nv_bfloat16* out1;         // member 1 pooled
  int ld1, off1;
};
cudaError_t stem_pool_launch(const CUtensorMap& ma, const CUtensorMap& mb, const StemPoolParams& p,
                             int grid, cudaStream_t stream);

cudaError_t conv_umma_launch(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mo,
                             const CUtensorMap& mr, const ConvParams& p, int block_n, int grid,
                             cudaStream_t stream);
int conv_umma_chunk(int block_n);
int conv_umma_stem_chunk(int block_n);  // the stem instances' epilogue chunk
// batch of the forward being enqueued on this thread (0 = unknown): gates PDL
void set_pdl_batch(int batch);
// pipeline stages the kernel instance for this plan would get (host-side layout query)
int conv_umma_stages(const ConvParams& p, int block_n);

// Driver entry point for tensor-map encoding (resolved through the runtime so the
// library does not link libcuda directly).
bool encode_tiled_2d_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                          uint64_t ld_elems, uint32_t box_inner, uint32_t box_outer,
                          std::string* err, int swizzle_bytes = 128);
// 3-D tiled map (d0 innermost, contiguous); strides in elements
bool encode_tiled_3d_bf16(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t d2,
                          uint64_t stride1_elems, uint64_t stride2_elems, uint32_t b0, uint32_t b1,
                          uint32_t b2, std::string* err, int swizzle_bytes = 128);
bool encode_im2col_bf16(CUtensorMap* map, const void* base, int n, int h, int w, int c, int ldc,
                        int kh, int kw, int sh, int sw, int ph, int pw, int chans_per_pixel,
                        int pixels, bool swizzle128, std::string* err, int upper_w_extra = 0,
                        int upper_h_extra = 0);

void set_error(const std::string& msg);

}  // namespace eb
