// conv_umma.cu -- K2/K3: implicit-GEMM convolution and fully-connected layers
// on the sm_100a 5th-generation tensor cores.
//
//   D[M, N] = A[M, K] * W[N, K]^T       (bf16 operands, fp32 accumulate in TMEM)
//   M = output pixels (B*Ho*Wo, NHWC order), N = output channels, K = taps*Cin
//
// A is never materialised: a TMA im2col load brings, per (filter tap, 64-channel
// chunk), 128 consecutive output pixels' receptive-field samples straight into
// 128B-swizzled shared memory (zero-filled at the padded borders and past the
// last image).  1x1/stride-1 convolutions and FC layers use a plain 2-D TMA
// tile instead.  The stem (Cin=3, padded to 8 channels by the preprocess
// kernel) uses 16-byte im2col columns in the non-swizzled canonical layout, one
// TMA per tap, eight taps per 64-wide K block.
//
// Warp roles (192 threads): warp 0 = TMA producer, warp 1 = TMEM owner + MMA
// issuer (one elected lane), warps 2..5 = epilogue (TMEM -> registers ->
// bias / residual / ReLU -> bf16 NHWC store, or fp32 logits / split-K partial slices).
// The epilogue writes into a channel slice of a wider NHWC buffer, which is how
// DenseNet concatenation and Inception branch concatenation are realised
// without a copy.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "eb_internal.h"
#include "sm100.cuh"

namespace eb {

constexpr int kBlockM = 128;
constexpr int kBlockK = 64;  // one 128-byte swizzle atom of bf16
constexpr int kThreads = 192;
constexpr int kABytes = kBlockM * kBlockK * 2;  // 16 KiB

template <int BN>
struct ConvSmem {
  static constexpr int kBBytes = BN * kBlockK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = (BN >= 256) ? 4 : (BN >= 128 ? 6 : 8);
  static constexpr int kBarOffset = kStages * kStageBytes;
  static constexpr int kBytes = kBarOffset + 256 + 1024;  // barriers + alignment slack
};

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    conv_umma_kernel(const __grid_constant__ CUtensorMap map_a,
                     const __grid_constant__ CUtensorMap map_b, const ConvParams p) {
  using S = ConvSmem<BN>;
  extern __shared__ uint8_t smem_raw[];
  // 128B swizzle needs 1024-byte aligned tiles
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::kBarOffset);
  uint64_t* empty = full + S::kStages;
  uint64_t* accum_full = empty + S::kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum_full + 1);

  const uint32_t warp = warp_id();
  const int tile_m = blockIdx.x;
  const int tile_n = blockIdx.y;
  const int kb_begin = blockIdx.z * p.kb_per_split;
  int kb_end = kb_begin + p.kb_per_split;
  if (kb_end > p.num_kb) kb_end = p.num_kb;
  const int nkb = kb_end - kb_begin;

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
    for (int s = 0; s < S::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accum_full, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, BN < 32 ? 32 : BN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (elect_one()) {
      const int m0 = tile_m * kBlockM;
      int img = 0, oh = 0, ow = 0;
      if (p.a_mode != kAModeTiled) {
        const int hw = p.Ho * p.Wo;
        img = m0 / hw;
        const int rem = m0 - img * hw;
        oh = rem / p.Wo;
        ow = rem - oh * p.Wo;
      }
      const int base_w = ow * p.sw - p.pw;
      const int base_h = oh * p.sh - p.ph;
      const int n0 = tile_n * BN;
      int stage = 0;
      uint32_t phase = 0;
      for (int i = 0; i < nkb; ++i) {
        const int kb = kb_begin + i;
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* sa = smem + stage * S::kStageBytes;
        uint8_t* sb = sa + kABytes;
        mbar_arrive_expect_tx(&full[stage], S::kStageBytes);
        if (p.a_mode == kAModeTiled) {
          tma_load_2d(sa, &map_a, &full[stage], kb * kBlockK, m0);
        } else if (p.a_mode == kAModeIm2col) {
          const int tap = kb / p.cchunks;
          const int cc = kb - tap * p.cchunks;
          const int r = tap / p.kw;
          const int s = tap - r * p.kw;
          tma_load_im2col_4d(sa, &map_a, &full[stage], cc * kBlockK, base_w, base_h, img,
                             static_cast<uint16_t>(s), static_cast<uint16_t>(r));
        } else {  // kAModeIm2colC8: eight 8-channel taps per K block
#pragma unroll 1
          for (int j = 0; j < 8; ++j) {
            int tap = kb * 8 + j;
            if (tap >= p.taps) tap = 0;  // weights are zero there; any finite data works
            const int r = tap / p.kw;
            const int s = tap - r * p.kw;
            tma_load_im2col_4d(sa + j * (kBlockM * 16), &map_a, &full[stage], 0, base_w, base_h,
                               img, static_cast<uint16_t>(s), static_cast<uint16_t>(r));
          }
        }
        tma_load_2d(sb, &map_b, &full[stage], kb * kBlockK, n0);
        if (++stage == S::kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = umma_idesc_bf16(kBlockM, BN);
    int stage = 0;
    uint32_t phase = 0;
    for (int i = 0; i < nkb; ++i) {
      mbar_wait(&full[stage], phase);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sa = smem_u32(smem + stage * S::kStageBytes);
        const uint32_t sb = sa + kABytes;
#pragma unroll
        for (int k = 0; k < kBlockK / 16; ++k) {
          uint64_t adesc;
          if (p.a_mode == kAModeIm2colC8) {
            // two 8-channel tap columns per K=16 step; core matrices 128 B apart along M,
            // 2 KiB apart along K
            adesc = umma_desc(sa + k * 2 * (kBlockM * 16), kBlockM * 16, 128, 0);
          } else {
            adesc = umma_desc_sw128(sa + k * 32);
          }
          const uint64_t bdesc = umma_desc_sw128(sb + k * 32);
          umma_bf16(tmem_base, adesc, bdesc, idesc, (i > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit(&empty[stage]);
        if (i == nkb - 1) umma_commit(accum_full);
      }
      __syncwarp();
      if (++stage == S::kStages) {
        stage = 0;
        phase ^= 1;
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const uint32_t quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int row = static_cast<int>(quarter * 32 + lane_id());
    const int m = tile_m * kBlockM + row;
    const bool row_ok = m < p.M;
    mbar_wait(accum_full, 0);
    tc_fence_after();
    const int n_tile0 = tile_n * BN;
#pragma unroll 1
    for (int c = 0; c < BN; c += 16) {
      const int n = n_tile0 + c;
      if (n >= p.N) break;  // warp-uniform
      uint32_t r[16];
      tmem_ld16(tmem_base + ((quarter * 32) << 16) + c, r);
      tmem_ld_wait();
      if (!row_ok) continue;
      float v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
      const int nvalid = (p.N - n) < 16 ? (p.N - n) : 16;
      const bool vec = p.vec_ok && nvalid == 16;
      if (p.out_mode == kOutPartialF32) {
        float* o = reinterpret_cast<float*>(p.out) +
                   (static_cast<size_t>(blockIdx.z) * p.M + m) * p.ldo + n;
        if (vec) {
#pragma unroll
          for (int j = 0; j < 16; j += 4)
            *reinterpret_cast<float4*>(o + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        } else {
          for (int j = 0; j < nvalid; ++j) o[j] = v[j];
        }
        continue;
      }
      if (p.bias) {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] += (j < nvalid) ? __ldg(p.bias + n + j) : 0.f;
      }
      if (p.res) {
        const __nv_bfloat16* rp = p.res + static_cast<size_t>(m) * p.ldr + n;
        if (vec) {
          uint4 q0 = *reinterpret_cast<const uint4*>(rp);
          uint4 q1 = *reinterpret_cast<const uint4*>(rp + 8);
          const __nv_bfloat16* h0 = reinterpret_cast<const __nv_bfloat16*>(&q0);
          const __nv_bfloat16* h1 = reinterpret_cast<const __nv_bfloat16*>(&q1);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            v[j] += __bfloat162float(h0[j]);
            v[j + 8] += __bfloat162float(h1[j]);
          }
        } else {
          for (int j = 0; j < nvalid; ++j) v[j] += __bfloat162float(rp[j]);
        }
      }
      if (p.relu) {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = fmaxf(v[j], 0.f);
      }
      if (p.out_mode == kOutF32) {
        float* o = reinterpret_cast<float*>(p.out) + static_cast<size_t>(m) * p.ldo + p.out_off + n;
        if (vec) {
#pragma unroll
          for (int j = 0; j < 16; j += 4)
            *reinterpret_cast<float4*>(o + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        } else {
          for (int j = 0; j < nvalid; ++j) o[j] = v[j];
        }
      } else {
        __nv_bfloat16* o =
            reinterpret_cast<__nv_bfloat16*>(p.out) + static_cast<size_t>(m) * p.ldo + p.out_off + n;
        if (vec) {
          uint4 q0, q1;
          q0.x = pack_bf16x2(v[0], v[1]);
          q0.y = pack_bf16x2(v[2], v[3]);
          q0.z = pack_bf16x2(v[4], v[5]);
          q0.w = pack_bf16x2(v[6], v[7]);
          q1.x = pack_bf16x2(v[8], v[9]);
          q1.y = pack_bf16x2(v[10], v[11]);
          q1.z = pack_bf16x2(v[12], v[13]);
          q1.w = pack_bf16x2(v[14], v[15]);
          *reinterpret_cast<uint4*>(o) = q0;
          *reinterpret_cast<uint4*>(o + 8) = q1;
        } else {
          for (int j = 0; j < nvalid; ++j) o[j] = __float2bfloat16_rn(v[j]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem_base, BN < 32 ? 32 : BN);
}

// ---------------------------------------------------------------- host side

template <int BN>
static cudaError_t launch_bn(const CUtensorMap& ma, const CUtensorMap& mb, const ConvParams& p,
                             dim3 grid, cudaStream_t stream) {
  using S = ConvSmem<BN>;
  static bool configured = false;  // attribute is per-function; idempotent
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(conv_umma_kernel<BN>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, S::kBytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  conv_umma_kernel<BN><<<grid, kThreads, S::kBytes, stream>>>(ma, mb, p);
  return cudaGetLastError();
}

cudaError_t conv_umma_launch(const CUtensorMap& ma, const CUtensorMap& mb, const ConvParams& p,
                             int block_n, dim3 grid, cudaStream_t stream) {
  switch (block_n) {
    case 32: return launch_bn<32>(ma, mb, p, grid, stream);
    case 64: return launch_bn<64>(ma, mb, p, grid, stream);
    case 128: return launch_bn<128>(ma, mb, p, grid, stream);
    case 256: return launch_bn<256>(ma, mb, p, grid, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace eb
