// block1.cu -- VGG block 1 in one kernel: conv3x3(3->64)+ReLU -> conv3x3(64->64)+ReLU ->
// maxpool 2x2/2.  The 64-channel full-resolution intermediate (1.6 GB per 256 images)
// never leaves shared memory.
//
// Work unit ("strip"): one image, a band of bh output rows, one 120-column segment.  A
// CTA walks its strips top to bottom; every conv1_2 output row ("tile") is one taps-in-N
// MMA group (M = 128 grid positions, N = 3 x 64: the three horizontal taps stacked) whose
// A operands are three conv1_1 row segments held in a ring of shared-memory slots.  Each
// new conv1_1 row segment is computed once per strip by the stem MMAs (rows mode:
// overlapping 16-byte core matrices over a 136-pixel run of the 8-channel padded image)
// and written by the epilogue warps straight into a ring slot in the 128B-swizzled
// K-major layout the conv1_2 MMAs read -- the layout TMA im2col writes in the unfused
// kernel.  Every arithmetic step (MMA K order, fp32 bias adds, tap combination order,
// max-before-bias pooling, rounding) is the unfused pair's (conv_umma.cu stem rows mode,
// taps-in-N + fused pool), so the pooled output is bitwise the same.
//
// Roles: warp 0 TMA producer (stem input runs; resident weights), warp 1 conv1_2 MMA
// issuer, warp 14 stem MMA issuer, warps 2-9 conv1_2 epilogue (quarter = warp & 3 owns
// TMEM lanes 32q..32q+31; the two groups take channels 0-31 / 32-63), warps 10-13 stem
// epilogue (one per lane quarter, all 64 channels) -- the two epilogues run side by side.
// Job order (identical in all roles): before conv1_2 tile t of the CTA's tile sequence,
// every ring job (conv1_1 row) up to tile t's third row + kLook -- the stem epilogue
// then has kLook tiles of MMA time to deliver a row; the look-ahead also reaches into the
// next strip at the end of a strip.
#include "eb_internal.h"
#include "sm100.cuh"

namespace eb {

namespace {
constexpr int kThreads1 = 480;  // producer, conv MMA, 8 conv1_2-epilogue, 4 stem-epilogue, stem MMA warps
#ifndef EB_B1_LOOK
#define EB_B1_LOOK 2
#endif
constexpr int kLook = EB_B1_LOOK;  // conv1_1 rows computed ahead of the tile that reads them
// EB_B1_DBG: timing probes (variant builds only; results wrong): 1 no tap shuffles, 2 no
// ring stores, 4 conv planes 1-2 not loaded from TMEM, 8 epilogues hand-shake only (16 the
// stem epilogue only, 32 the conv epilogue only)
#ifndef EB_B1_DBG
#define EB_B1_DBG 0
#endif
constexpr int kRing = 3 + kLook + 1;         // conv1_1 row slots: 3 read + kLook written ahead + 1
constexpr int kSlotBytes = 128 * 128;        // 128 grid rows x 64 channels bf16 (SW128 K-major)
constexpr int kRunBytes = 136 * 16;          // one filter row's run: 136 padded pixels x 8 ch
constexpr int kStemStage = 3 * kRunBytes;    // the 3 filter rows of one conv1_1 row segment
constexpr int kStemStages = 4;
constexpr int kBStem = 3 * 64 * 128;         // stem weights: 3 filter rows x [64 N][64 K]
constexpr int kBConvRow = 3 * 64 * 128;      // conv1_2 weights per filter row: 3 taps x [64][64]
constexpr int kBConv = 3 * kBConvRow;
constexpr int kOffRing = 0;
constexpr int kOffBConv = kOffRing + kRing * kSlotBytes;
constexpr int kOffBStem = kOffBConv + kBConv;
constexpr int kOffStem = kOffBStem + kBStem;
constexpr int kOffBias = kOffStem + kStemStages * kStemStage;
constexpr int kOffBar = kOffBias + 2 * 64 * 4;
constexpr int kNumBars = 2 * kStemStages + 2 + 2 + 2 * kRing + 2 + 2 + 1;
constexpr int kSmemBytes = kOffBar + kNumBars * 8 + 16 + 1024;  // + TMEM slot + alignment slack
// TMEM columns: conv1_2 accumulators (192 each) at 0 / 192, stem accumulators at 384 / 448
constexpr uint32_t kConvAcc = 192, kStemAcc0 = 384;
static_assert(kSmemBytes <= 232448, "block1 shared memory");
}  // namespace

__global__ void __launch_bounds__(kThreads1, 1)
    block1_kernel(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_w1,
                  const __grid_constant__ CUtensorMap map_w2, const Block1Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* ring = smem + kOffRing;
  uint8_t* bconv = smem + kOffBConv;
  uint8_t* bstem = smem + kOffBStem;
  uint8_t* stem = smem + kOffStem;
  float* bias1 = reinterpret_cast<float*>(smem + kOffBias);
  float* bias2 = bias1 + 64;
  uint64_t* sfull = reinterpret_cast<uint64_t*>(smem + kOffBar);  // [kStemStages] stem input landed
  uint64_t* sempty = sfull + kStemStages;                         // [kStemStages] stem input consumed
  uint64_t* afull = sempty + kStemStages;                         // [2] stem accumulator ready
  uint64_t* aempty = afull + 2;                                   // [2] stem accumulator drained
  uint64_t* rfull = aempty + 2;                                   // [kRing] conv1_1 row written
  uint64_t* rempty = rfull + kRing;                               // [kRing] conv1_1 row no longer read
  uint64_t* tfull = rempty + kRing;                               // [2] conv1_2 accumulator ready
  uint64_t* tempty = tfull + 2;                                   // [2] conv1_2 accumulator drained
  uint64_t* bres = tempty + 2;                                    // resident weights landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bres + 1);

  const uint32_t warp = warp_id();
  const int lane = static_cast<int>(lane_id());
  // this CTA's strips: blockIdx.x + i * gridDim.x
  const int ns = (p.strips - static_cast<int>(blockIdx.x) + static_cast<int>(gridDim.x) - 1) /
                 static_cast<int>(gridDim.x);
  const int rj = p.bh + 2;  // ring jobs (conv1_1 rows y0-1 .. y0+bh) per strip
  const int nring = ns * rj;
  const int ntile = ns * p.bh;
  const int per_img = p.nbands * p.nseg;

  if (threadIdx.x < 128) {
    if (threadIdx.x < 64)
      bias1[threadIdx.x] = p.bias1[threadIdx.x];
    else
      bias2[threadIdx.x - 64] = p.bias2[threadIdx.x - 64];
  }
  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&map_x);
    tma_prefetch_desc(&map_w1);
    tma_prefetch_desc(&map_w2);
    for (int i = 0; i < kStemStages; ++i) {
      mbar_init(&sfull[i], 1);
      mbar_init(&sempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&afull[i], 1);
      mbar_init(&aempty[i], 4);
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 8);
    }
    for (int i = 0; i < kRing; ++i) {
      mbar_init(&rfull[i], 4);
      mbar_init(&rempty[i], 1);
    }
    mbar_init(bres, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (warp == 0 && elect_one()) {
    // weights are never written inside the graph: fetched before the PDL wait
    mbar_arrive_expect_tx(bres, kBConv + kBStem);
    for (int r = 0; r < 3; ++r) {
      for (int s = 0; s < 3; ++s)
        tma_load_2d(bconv + r * kBConvRow + s * 64 * 128, &map_w2, bres, (r * 3 + s) * 64, 0);
      tma_load_2d(bstem + r * 64 * 128, &map_w1, bres, r * 64, 0);
    }
  }
  pdl_wait();
  pdl_launch_dependents();

  // ring job j -> image, conv1_1 row k (y0 - 1 .. y0 + bh), segment start column x0
  auto ring_job = [&](int j, int& b, int& k, int& x0) {
    const int i = j / rj;
    const int s = static_cast<int>(blockIdx.x) + i * static_cast<int>(gridDim.x);
    b = s / per_img;
    const int rem = s - b * per_img;
    const int band = rem / p.nseg;
    x0 = 120 * (rem - band * p.nseg);
    k = band * p.bh - 1 + (j - i * rj);
  };
  // the shared job order: ring jobs up to one row past each tile's third row, then the tile
  auto walk = [&](auto&& on_ring, auto&& on_tile) {
    int next = 0;
    for (int g = 0; g < ntile; ++g) {
      const int i = g / p.bh;
      const int t = g - i * p.bh;
      const int need = min(i * rj + t + 2 + kLook, nring - 1);
      for (; next <= need; ++next) on_ring(next);
      on_tile(i, t);
    }
  };

  if (warp == 0) {
    // ---------------------------------------------------------------- producer
    if (elect_one()) {
      int st = 0;
      uint32_t ph = 0;
      walk(
          [&](int j) {
            int b, k, x0;
            ring_job(j, b, k, x0);
            if (k < 0 || k >= p.H) return;  // border rows of conv1_2's padding: no stem work
            mbar_wait(&sempty[st], ph ^ 1);
            mbar_arrive_expect_tx(&sfull[st], kStemStage);
            uint8_t* dst = stem + st * kStemStage;
            // filter row r of conv1_1 row k: padded row k + r; grid position m (conv1_1
            // column x0 - 1 + m) at padded column x0 - 1 + m (+ tap); column -1 is TMA
            // zero fill (its output is conv1_2 padding and never used)
            for (int r = 0; r < 3; ++r)
              tma_load_3d(dst + r * kRunBytes, &map_x, &sfull[st], 0, x0 - 1, b * p.Hq + k + r);
            if (++st == kStemStages) {
              st = 0;
              ph ^= 1;
            }
          },
          [&](int, int) {});
    }
  } else if (warp == 1 || warp == 14) {
    // ---------------------------------------------------------------- MMA issuers
    // (two: warp 14 the stem MMAs, warp 1 the conv1_2 MMAs -- one issuing thread cannot
    // keep the tensor core fed through the hand-shakes and descriptor math of both)
    const bool stem_issuer = warp == 14;
    constexpr uint32_t idesc1 = umma_idesc_bf16(128, 64);
    constexpr uint32_t idesc2 = umma_idesc_bf16(128, 192);
    const uint64_t bstem_d = umma_desc_sw128(smem_u32(bstem));
    const uint64_t bconv_d = umma_desc_sw128(smem_u32(bconv));
    int st = 0, sj = 0, tj = 0;
    uint32_t ph = 0;
    mbar_wait(bres, 0);
    walk(
        [&](int j) {
          if (!stem_issuer) return;
          int b, k, x0;
          ring_job(j, b, k, x0);
          if (k < 0 || k >= p.H) return;
          const int a = sj & 1;
          mbar_wait(&aempty[a], ((sj >> 1) & 1) ^ 1);
          mbar_wait(&sfull[st], ph);
          tc_fence_after();
          if (elect_one()) {
            // stem rows mode: taps are core matrices 16 B apart (LBO = 16); K16 step k
            // covers taps 2k, 2k + 1 (tap 3 meets zero weights)
            const uint64_t a0 = umma_desc(smem_u32(stem + st * kStemStage), 16, 128, 0);
            for (int r = 0; r < 3; ++r)
#pragma unroll
              for (int kk = 0; kk < 2; ++kk)
                umma_bf16(tmem_base + kStemAcc0 + a * 64, a0 + r * (kRunBytes >> 4) + 2 * kk,
                          bstem_d + r * ((64 * 128) >> 4) + 2 * kk, idesc1, (r | kk) ? 1u : 0u);
            umma_commit(&sempty[st]);
            umma_commit(&afull[a]);
          }
          __syncwarp();
          ++sj;
          if (++st == kStemStages) {
            st = 0;
            ph ^= 1;
          }
        },
        [&](int i, int t) {
          if (stem_issuer) return;
          const int a = tj & 1;
          const int j0 = i * rj + t;  // the tile's conv1_1 rows are ring jobs j0 .. j0 + 2
          mbar_wait(&tempty[a], ((tj >> 1) & 1) ^ 1);
          for (int q = 0; q < 3; ++q) mbar_wait(&rfull[(j0 + q) % kRing], ((j0 + q) / kRing) & 1);
          tc_fence_after();
          if (elect_one()) {
            for (int r = 0; r < 3; ++r) {
              const uint64_t ad = umma_desc_sw128(smem_u32(ring + ((j0 + r) % kRing) * kSlotBytes));
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
                umma_bf16(tmem_base + a * kConvAcc, ad + 2 * kk, bconv_d + r * (kBConvRow >> 4) + 2 * kk,
                          idesc2, (r | kk) ? 1u : 0u);
            }
            umma_commit(&tfull[a]);
            // row j0 is read by no later tile; a strip's last tile also frees its last two
            umma_commit(&rempty[j0 % kRing]);
            if (t == p.bh - 1) {
              umma_commit(&rempty[(j0 + 1) % kRing]);
              umma_commit(&rempty[(j0 + 2) % kRing]);
            }
          }
          __syncwarp();
          ++tj;
        });
  } else if (warp >= 10) {  // (10 .. 13)
    // ---------------------------------------------------------------- stem epilogue
    const uint32_t quarter = warp & 3;
    const int m = static_cast<int>(quarter) * 32 + lane;  // TMEM lane = grid position
    const uint32_t lane_off = (quarter * 32) << 16;
    float2 bias_r[32];  // in registers: shared-memory bandwidth is what bounds this kernel
#pragma unroll
    for (int i = 0; i < 32; ++i) bias_r[i] = make_float2(bias1[2 * i], bias1[2 * i + 1]);
    int sj = 0;
    walk(
        [&](int j) {
          int b, k, x0;
          ring_job(j, b, k, x0);
          const int slot = j % kRing;
          if (j >= kRing) mbar_wait(&rempty[slot], ((j / kRing) - 1) & 1);
          const bool live = k >= 0 && k < p.H;
          const int col = x0 - 1 + m;  // conv1_1 column; outside the image it is padding
          const bool inside = live && col >= 0 && col < p.W;
          const int a = sj & 1;
          if (live) {
            mbar_wait(&afull[a], (sj >> 1) & 1);
            tc_fence_after();
          }
          if (EB_B1_DBG & (8 | 16)) {  // (probe: hand-shakes only)
            if (live) {
              __syncwarp();
              if (lane == 0) mbar_arrive(&aempty[a]);
              ++sj;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&rfull[slot]);
            return;
          }
          uint8_t* sb = ring + slot * kSlotBytes;
          const int qh = m / 30;
#pragma unroll
          for (int half = 0; half < 2; ++half) {  // channels 32 * half .. + 31
            uint32_t pk[16];
            if (live) {
              uint32_t r[32];
              tmem_ld32(tmem_base + lane_off + kStemAcc0 + a * 64 + 32 * half, r);
              tmem_ld_wait();
              if (half == 1) {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&aempty[a]);
              }
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const float2 v = __fadd2_rn(make_float2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1])),
                                            bias_r[16 * half + i]);
                pk[i] = inside ? pack_bf16x2_relu(v.x, v.y) : 0u;
              }
            } else {
#pragma unroll
              for (int i = 0; i < 16; ++i) pk[i] = 0u;
            }
            // grid position m is A row m + 2q of every quarter q it belongs to (quarter q
            // covers positions 30q .. 30q + 31: the taps-in-N rows overlap by two)
#pragma unroll
            for (int d = 0; d < 2; ++d) {
              const int q = qh - d;
              if (q < 0 || q > 3 || m - 30 * q > 31) continue;
              const int R = m + 2 * q;
              uint8_t* rowp = sb + (R >> 3) * 1024 + (R & 7) * 128;
#pragma unroll
              for (int c4 = 0; c4 < 4; ++c4) {
                const int chunk = 4 * half + c4;  // 16-byte chunk (8 channels) of the 128-byte row
                if (!(EB_B1_DBG & 2))
                  *reinterpret_cast<uint4*>(rowp + ((chunk ^ (R & 7)) << 4)) =
                      make_uint4(pk[4 * c4], pk[4 * c4 + 1], pk[4 * c4 + 2], pk[4 * c4 + 3]);
              }
            }
          }
          if (live) ++sj;
          fence_proxy_async_smem();  // generic-proxy writes, read by the MMAs (async proxy)
          __syncwarp();
          if (lane == 0) mbar_arrive(&rfull[slot]);
        },
        [&](int, int) {});
  } else if (warp >= 2) {
    // ---------------------------------------------------------------- conv1_2 epilogue
    const uint32_t quarter = warp & 3;
    const int half = (static_cast<int>(warp) - 2) >> 2;  // channels 32 * half .. + 31
    const uint32_t lane_off = (quarter * 32) << 16;
    int tj = 0;
    float2 bias_r[16];  // this group's 32 channels, in registers
#pragma unroll
    for (int i = 0; i < 16; ++i) bias_r[i] = make_float2(bias2[32 * half + 2 * i], bias2[32 * half + 2 * i + 1]);
    float2 keep[16];  // an even conv1_2 row's tap-combined values (fp32, pre-bias)
#pragma unroll
    for (int i = 0; i < 16; ++i) keep[i] = make_float2(0.f, 0.f);
    walk(
        [&](int) {},
        [&](int i, int t) {
          const int a = tj & 1;
          mbar_wait(&tfull[a], (tj >> 1) & 1);
          tc_fence_after();
          if (EB_B1_DBG & (8 | 32)) {  // (probe: hand-shakes only)
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[a]);
            ++tj;
            return;
          }
          const uint32_t tb = tmem_base + lane_off + a * kConvAcc + 32 * half;
          const int s = static_cast<int>(blockIdx.x) + i * static_cast<int>(gridDim.x);
          const int b = s / per_img;
          const int rem = s - b * per_img;
          const int band = rem / p.nseg;
          const int x = 120 * (rem - band * p.nseg) + 30 * static_cast<int>(quarter) + lane;
          const int y = band * p.bh + t;
          const bool store = (t & 1) && !(lane & 1) && lane < 30 && x < p.W;
          uint4* o4 = nullptr;
          if (store) {
            const size_t orow = (static_cast<size_t>(b) * (p.H >> 1) + (y >> 1)) * (p.W >> 1) + (x >> 1);
            o4 = reinterpret_cast<uint4*>(p.out + orow * p.ldo + p.out_off + 32 * half);
          }
#pragma unroll
          for (int sub = 0; sub < 2; ++sub) {  // 16 channels at a time (register budget)
            uint32_t r0[16], r1[16], r2[16];
            tmem_ld16(tb + 16 * sub, r0);
#if EB_B1_DBG & 4  // (probe: planes 1-2 not read -- TMEM read bandwidth)
#pragma unroll
            for (int q = 0; q < 16; ++q) r1[q] = r2[q] = r0[q];
#else
            tmem_ld16(tb + 64 + 16 * sub, r1);
            tmem_ld16(tb + 128 + 16 * sub, r2);
#endif
            tmem_ld_wait();
            if (sub == 1) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&tempty[a]);
            }
            // out[m] = (D0[m] + D1[m+1]) + D2[m+2]
            float2 v2[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
#if EB_B1_DBG & 1
              const float2 d1 = make_float2(__uint_as_float(r1[2 * q]), __uint_as_float(r1[2 * q + 1]));
              const float2 d2 = make_float2(__uint_as_float(r2[2 * q]), __uint_as_float(r2[2 * q + 1]));
#else
              const float2 d1 = make_float2(__shfl_down_sync(0xffffffffu, __uint_as_float(r1[2 * q]), 1),
                                            __shfl_down_sync(0xffffffffu, __uint_as_float(r1[2 * q + 1]), 1));
              const float2 d2 = make_float2(__shfl_down_sync(0xffffffffu, __uint_as_float(r2[2 * q]), 2),
                                            __shfl_down_sync(0xffffffffu, __uint_as_float(r2[2 * q + 1]), 2));
#endif
              v2[q] = __fadd2_rn(
                  __fadd2_rn(make_float2(__uint_as_float(r0[2 * q]), __uint_as_float(r0[2 * q + 1])), d1), d2);
            }
            if ((t & 1) == 0) {
#pragma unroll
              for (int q = 0; q < 8; ++q) keep[8 * sub + q] = v2[q];
            } else {
              // the 2x2 max (vertical, then lanes (2k, 2k+1): max is exact in any order, the
              // unfused kernel's horizontal-first order gives the same value), then bias,
              // ReLU, rounding -- the shuffle runs once per row pair
              uint32_t pk[8];
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                float2 w = make_float2(fmaxf(keep[8 * sub + q].x, v2[q].x), fmaxf(keep[8 * sub + q].y, v2[q].y));
                w.x = fmaxf(w.x, __shfl_down_sync(0xffffffffu, w.x, 1));
                w.y = fmaxf(w.y, __shfl_down_sync(0xffffffffu, w.y, 1));
                w = __fadd2_rn(w, bias_r[8 * sub + q]);
                pk[q] = pack_bf16x2_relu(w.x, w.y);
              }
              if (store) {
                o4[2 * sub] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                o4[2 * sub + 1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
              }
            }
          }
          ++tj;
        });
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem_base, 512);
}

cudaError_t block1_launch(const CUtensorMap& mx, const CUtensorMap& mw1, const CUtensorMap& mw2,
                          const Block1Params& p, int grid, cudaStream_t stream) {
  static bool configured = false;
  if (!configured) {
    const cudaError_t e =
        cudaFuncSetAttribute(block1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads1);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, block1_kernel, mx, mw1, mw2, p);
}

}  // namespace eb
