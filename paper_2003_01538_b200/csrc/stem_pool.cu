// stem_pool.cu -- the 7x7/2 stem of one member, or the grouped stem of two (ResNet / ResNeXt
// / DenseNet: conv 3->64 + bias + ReLU each, N = 64 or 128 concatenated), with the members'
// 3x3/2 (pad 1) max-pools in one kernel: the 112 x 112 stem output (411 MB per member and
// 256 images) is pooled in registers and never written.
//
// Work unit ("strip"): one image, a band of pb pooled rows (conv rows 2 p0 - 1 .. 2 p1 - 1;
// the first band starts at conv row 0).  A conv row is one stem tile exactly (the planes
// grid is 128 wide, Wo = 112), computed with the stem planes mode's descriptors: two tall
// TMA boxes (even / odd column planes, all 7 filter rows) and 28 MMAs (K16 steps: even taps
// 0-2, 4-6 then odd taps 1-3, 5-(7); N = 128).  The epilogue (16 warps: lane quarter x
// 32-channel group) rounds each value exactly as the stem kernel does (bias, ReLU, bf16),
// runs the vertical max over conv rows (2y-1, 2y, 2y+1) in registers and then the max of
// positions (2x-1, 2x, 2x+1) once per pooled row -- lane shuffles, and one smem hand-over
// of lane 31 to the next quarter.  Max is exact in any order, so the pooled tensors are bitwise the unfused pair's.
#include "eb_internal.h"
#include "sm100.cuh"

namespace eb {

#ifndef EB_SP_DBG
#define EB_SP_DBG 0  // timing probe (variant builds only; results wrong): 1 epilogue hand-shakes only
#endif
namespace {
#ifndef EB_SP_EPI
#define EB_SP_EPI 16  // epilogue warps: 8 or 16
#endif
constexpr int kEpiW = EB_SP_EPI;
constexpr int kThreadsSP = 64 + 32 * kEpiW;  // producer, MMA, epilogue warps
constexpr int kSPStages = 3;
constexpr int kSPAcc = 4;             // TMEM accumulators (NCOL columns each)
constexpr int kSPMaxStage = 31 * 1024;  // two tall boxes of <= 124 lines, 1024-aligned
// NCOL = 64 * members (one or two members' stems)
template <int NCOL>
struct SPCfg {
  static constexpr int kCh = NCOL / (kEpiW / 4);  // channels per epilogue warp
  static constexpr int kWords = kCh / 2;          // bf16x2 words per lane
  static constexpr int kBRow = NCOL * 128;        // weights of one filter row: NCOL N x 64 K (SW128)
  static constexpr int kB = 7 * kBRow;            // resident
  static constexpr int kOffB = 0;
  static constexpr int kOffStage = kOffB + kB;
  static constexpr int kOffBias = kOffStage + kSPStages * kSPMaxStage;
  static constexpr int kOffXch = kOffBias + 128 * 4;  // [group][quarter][parity] kCh * 2 B
  static constexpr int kOffBar = kOffXch + (kEpiW / 4) * 4 * 2 * kCh * 2;
  static constexpr int kBars = 2 * kSPStages + 2 * kSPAcc + 1;
  static constexpr int kSmem = kOffBar + kBars * 8 + 16 + 1024;
  static_assert(kSmem <= 232448, "stem_pool shared memory");
  static_assert(kCh % 16 == 0, "epilogue channel groups of 16");
};
}  // namespace

template <int NCOL>
__global__ void __launch_bounds__(kThreadsSP, 1)
    stem_pool_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                     const StemPoolParams p) {
  using C = SPCfg<NCOL>;
  constexpr int kCh = C::kCh;
  constexpr int kWords = C::kWords;
  constexpr int kSPBRow = C::kBRow;
  constexpr int kSPB = C::kB;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* bres_s = smem + C::kOffB;
  uint8_t* stage_s = smem + C::kOffStage;
  float* bias = reinterpret_cast<float*>(smem + C::kOffBias);
  uint32_t* xch = reinterpret_cast<uint32_t*>(smem + C::kOffXch);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* empty = full + kSPStages;
  uint64_t* tfull = empty + kSPStages;
  uint64_t* tempty = tfull + kSPAcc;
  uint64_t* bres = tempty + kSPAcc;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bres + 1);

  const uint32_t warp = warp_id();
  const int lane = static_cast<int>(lane_id());
  const int ns = (p.strips - static_cast<int>(blockIdx.x) + static_cast<int>(gridDim.x) - 1) /
                 static_cast<int>(gridDim.x);
  const int Hp = p.Ho >> 1;  // pooled rows (3x3/2, pad 1, even Ho)
  // strip i of this CTA -> image, first and last conv row
  auto strip = [&](int i, int& b, int& y0, int& y1) {
    const int s = static_cast<int>(blockIdx.x) + i * static_cast<int>(gridDim.x);
    b = s / p.nbands;
    const int band = s - b * p.nbands;
    const int p0 = band * p.pb;
    y0 = p0 > 0 ? 2 * p0 - 1 : 0;
    y1 = 2 * (p0 + p.pb) - 1;
  };

  if (threadIdx.x < NCOL) bias[threadIdx.x] = p.bias[threadIdx.x];
  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
    for (int i = 0; i < kSPStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < kSPAcc; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], kEpiW);
    }
    mbar_init(bres, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (warp == 0 && elect_one()) {  // weights: never written inside the graph
    mbar_arrive_expect_tx(bres, kSPB);
    for (int r = 0; r < 7; ++r) tma_load_2d(bres_s + r * kSPBRow, &map_b, bres, r * 64, 0);
  }
  pdl_wait();
  pdl_launch_dependents();

  if (warp == 0) {
    // ---------------------------------------------------------------- producer
    if (elect_one()) {
      int st = 0;
      uint32_t ph = 0;
      const int plane_lines = static_cast<int>(p.plane_px >> 3);
      for (int i = 0; i < ns; ++i) {
        int b, y0, y1;
        strip(i, b, y0, y1);
        for (int y = y0; y <= y1; ++y) {
          mbar_wait(&empty[st], ph ^ 1);
          mbar_arrive_expect_tx(&full[st], 2 * p.lines * 128);
          // padded row 2y (filter row 0) .. 2y + 6 of both column planes, whole rows
          const int line = ((b * p.Hq + 2 * y) * p.Wq) >> 3;
          uint8_t* dst = stage_s + st * kSPMaxStage;
          tma_load_2d(dst, &map_a, &full[st], 0, line);
          tma_load_2d(dst + p.lines * 128, &map_a, &full[st], 0, line + plane_lines);
          if (++st == kSPStages) {
            st = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    // (a second issuer taking alternate rows measured no faster: 0.317 vs 0.314 ms)
    constexpr uint32_t idesc = umma_idesc_bf16(128, NCOL);
    const uint64_t b0 = umma_desc_sw128(smem_u32(bres_s));
    const uint32_t odd16 = static_cast<uint32_t>(p.lines * 8);  // the odd plane's box
    const uint32_t koff[4] = {0u, 2u, odd16, odd16 + 2u};
    int j = 0;
    mbar_wait(bres, 0);
    for (int i = 0; i < ns; ++i) {
      int b, y0, y1;
      strip(i, b, y0, y1);
      for (int y = y0; y <= y1; ++y, ++j) {
        const int a = j % kSPAcc;
        const int st = j % kSPStages;
        const uint32_t ph = static_cast<uint32_t>((j / kSPStages) & 1);
        mbar_wait(&tempty[a], ((j / kSPAcc) & 1) ^ 1);
        mbar_wait(&full[st], ph);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t a0 = umma_desc(smem_u32(stage_s + st * kSPMaxStage), 16, 128, 0);
          for (int r = 0; r < 7; ++r)
#pragma unroll
            for (int k = 0; k < 4; ++k)
              umma_bf16(tmem_base + a * NCOL, a0 + r * static_cast<uint32_t>(p.Wq) + koff[k],
                        b0 + r * (kSPBRow >> 4) + 2 * k, idesc, (r | k) ? 1u : 0u);
          umma_commit(&empty[st]);
          umma_commit(&tfull[a]);
        }
        __syncwarp();
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue
    const uint32_t quarter = warp & 3;
    const int grp = (static_cast<int>(warp) - 2) >> 2;  // channels kCh * grp .. + kCh - 1
    const int col0 = kCh * grp;
    const int member = col0 >> 6;
    const int pos = static_cast<int>(quarter) * 32 + lane;  // output column of the conv row
    const uint32_t lane_off = (quarter * 32) << 16;
    const float2* bias2 = reinterpret_cast<const float2*>(bias + col0);
    __nv_bfloat16* out = member ? p.out1 : p.out0;
    const int ldo = member ? p.ld1 : p.ld0;
    const int ooff = (member ? p.off1 : p.off0) + (col0 & 63);
    uint32_t prev[kWords], acc[kWords];
#pragma unroll
    for (int i = 0; i < kWords; ++i) prev[i] = acc[i] = 0u;
    int j = 0, xn = 0;
    for (int i = 0; i < ns; ++i) {
      int b, y0, y1;
      strip(i, b, y0, y1);
      for (int y = y0; y <= y1; ++y, ++j) {
        const int a = j % kSPAcc;
        mbar_wait(&tfull[a], (j / kSPAcc) & 1);
        tc_fence_after();
        if (EB_SP_DBG & 1) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[a]);
          continue;
        }
        uint32_t h[kWords];  // this position's channels, rounded as the stem kernel stores them
#pragma unroll
        for (int qd = 0; qd < kCh / 16; ++qd) {  // 16 channels at a time (register budget)
          uint32_t r[16];
          tmem_ld16(tmem_base + lane_off + a * NCOL + col0 + 16 * qd, r);
          tmem_ld_wait();
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float2 v = __fadd2_rn(make_float2(__uint_as_float(r[2 * q]), __uint_as_float(r[2 * q + 1])),
                                        bias2[8 * qd + q]);
            h[8 * qd + q] = pack_bf16x2_relu(v.x, v.y);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[a]);
        // vertical first, per lane: pooled row py = max(conv rows 2py - 1, 2py, 2py + 1)
        // (max is exact in any order); the horizontal window then runs once per pooled row
        if ((y & 1) == 0) {
#pragma unroll
          for (int c = 0; c < kWords; ++c) {
            if (y == 0) {
              acc[c] = h[c];
            } else {
              __nv_bfloat162 m2 = __hmax2(*reinterpret_cast<const __nv_bfloat162*>(&prev[c]),
                                          *reinterpret_cast<const __nv_bfloat162*>(&h[c]));
              acc[c] = *reinterpret_cast<uint32_t*>(&m2);
            }
          }
          continue;
        }
        if (y == y0) {  // a band's first (odd) row only primes the next pooled row
#pragma unroll
          for (int c = 0; c < kWords; ++c) prev[c] = h[c];
          continue;
        }
        uint32_t v[kWords];
#pragma unroll
        for (int c = 0; c < kWords; ++c) {
          __nv_bfloat162 m2 = __hmax2(*reinterpret_cast<const __nv_bfloat162*>(&acc[c]),
                                      *reinterpret_cast<const __nv_bfloat162*>(&h[c]));
          v[c] = *reinterpret_cast<uint32_t*>(&m2);
          prev[c] = h[c];
        }
        // horizontal: max of positions pos - 1, pos, pos + 1 (even pos); position -1 is
        // padding, positions >= Wo never enter an even position's window (Wo even); lane 31
        // hands its column to the next quarter's lane 0 through shared memory
        uint32_t* xw = xch + ((grp * 4 + static_cast<int>(quarter)) * 2 + (xn & 1)) * kWords;
        if (lane == 31 && quarter < 3) {
#pragma unroll
          for (int c4 = 0; c4 < kWords / 4; ++c4)
            reinterpret_cast<uint4*>(xw)[c4] = make_uint4(v[4 * c4], v[4 * c4 + 1], v[4 * c4 + 2], v[4 * c4 + 3]);
        }
        named_bar_sync(1 + grp, 128);
        const uint32_t* xr = xch + ((grp * 4 + static_cast<int>(quarter) - 1) * 2 + (xn & 1)) * kWords;
        ++xn;
        uint32_t o[kWords];
#pragma unroll
        for (int c = 0; c < kWords; ++c) {
          uint32_t up = __shfl_up_sync(0xffffffffu, v[c], 1);
          const uint32_t dn = __shfl_down_sync(0xffffffffu, v[c], 1);
          if (lane == 0) up = quarter > 0 ? xr[c] : v[c];
          __nv_bfloat162 m2 = __hmax2(*reinterpret_cast<const __nv_bfloat162*>(&up),
                                      *reinterpret_cast<const __nv_bfloat162*>(&v[c]));
          m2 = __hmax2(m2, *reinterpret_cast<const __nv_bfloat162*>(&dn));
          o[c] = *reinterpret_cast<uint32_t*>(&m2);
        }
        if (!(lane & 1) && pos < p.Wo) {
          const size_t orow = (static_cast<size_t>(b) * Hp + (y >> 1)) * (p.Wo >> 1) + (pos >> 1);
          uint4* o4 = reinterpret_cast<uint4*>(out + orow * ldo + ooff);
#pragma unroll
          for (int c4 = 0; c4 < kWords / 4; ++c4)
            o4[c4] = make_uint4(o[4 * c4], o[4 * c4 + 1], o[4 * c4 + 2], o[4 * c4 + 3]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem_base, 512);
}

template <int NCOL>
static cudaError_t launch_sp(const CUtensorMap& ma, const CUtensorMap& mb, const StemPoolParams& p, int grid,
                             cudaStream_t stream) {
  static bool configured = false;
  if (!configured) {
    const cudaError_t e = cudaFuncSetAttribute(stem_pool_kernel<NCOL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               SPCfg<NCOL>::kSmem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreadsSP);
  cfg.dynamicSmemBytes = SPCfg<NCOL>::kSmem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, stem_pool_kernel<NCOL>, ma, mb, p);
}

cudaError_t stem_pool_launch(const CUtensorMap& ma, const CUtensorMap& mb, const StemPoolParams& p,
                             int grid, cudaStream_t stream) {
  if (2 * p.lines * 128 > kSPMaxStage) return cudaErrorInvalidValue;
  if (p.ncol == 128) return launch_sp<128>(ma, mb, p, grid, stream);
  if (p.ncol == 64) return launch_sp<64>(ma, mb, p, grid, stream);
  return cudaErrorInvalidValue;
}

}  // namespace eb
