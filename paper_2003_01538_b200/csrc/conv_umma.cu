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
// kernel) is gathered with cp.async by four extra warps: per filter row, the 8
// consecutive input pixels of a receptive-field row are one 128-byte A row.
//
// Persistent, warp-specialised (192 threads, one CTA per SM):
//   warp 0      TMA producer: a smem ring of (A, B) stages that runs across tiles
//   warp 1      TMEM owner + MMA issuer (one elected lane); two accumulator
//               buffers in TMEM so tile i+1's MMAs overlap tile i's epilogue
//   warps 2..5  epilogue: TMEM -> registers -> bias / residual / ReLU -> bf16 ->
//               128B-swizzled smem staging -> TMA bulk store (coalesced), or
//               direct fp32 stores for logits and split-K partial slices.
// The output map addresses a channel slice of a wider NHWC buffer, which is how
// DenseNet / Inception concatenation is realised without a copy; TMA clips the
// stores at the slice's N and at M.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "eb_internal.h"
#include "sm100.cuh"

namespace eb {

bool pdl_enabled();

constexpr int kBlockM = 128;
constexpr int kBlockK = 64;  // one 128-byte swizzle atom of bf16
// 2 control warps + 8 epilogue warps (or 4 epilogue + 4 stem-gather / 6 pre-activation
// warps).  Twelve warps cost no registers over ten: three warps per SM sub-partition
// either way caps a thread at 168 registers.
constexpr int kThreads = 384;
#ifndef EB_XFORM_THREADS
#define EB_XFORM_THREADS 64
#endif
constexpr int kXformThreads = EB_XFORM_THREADS;  // pre-activation transform: the last warps
// (128 -- four transform warps beside a four-warp epilogue -- hangs on B200 as of round 2's
// end; only the 64-thread configuration is maintained)
static_assert(EB_XFORM_THREADS == 64, "EB_XFORM_THREADS: only 64 is maintained");
constexpr int kTapC8Bytes = kBlockM * 16;  // tap-C8 mode: one tap = 128 pixels x 8 bf16
#ifndef EB_MAX_ACC
#define EB_MAX_ACC 4  // TMEM accumulators per CTA at most (8: measured no gain on the stems)
#endif
#ifndef EB_STEM_CW
#define EB_STEM_CW 64
#endif
#ifndef EB_STEM_NB
#define EB_STEM_NB 1  // stems: epilogue chunk buffers per warp (1 or 2)
#endif

// TS = filter taps consumed per pipeline stage: 1 (one TMA im2col load per tap)
// or 3 (tap-shift mode: one 136-row load per filter row serves its 3 horizontal taps).
// PAIR: 2-SM mode (cta_group::2) -- the CTA pair of a cluster runs one M=256 x BN MMA
// per K step; each CTA stages its own 128 A rows and half of the B tile.
// TAPN: taps-in-N mode for 3-wide stride-1 filters with small Cout -- one MMA per K block
// with the 3 horizontal taps' weights stacked along N (N = 3 x BN); the epilogue adds the
// tap planes shifted by 0/1/2 rows.  The A tile is 4 x 32 rows overlapping by 2, so each
// lane quarter can form its 30 outputs with warp shuffles; tiles advance 120 rows.
// STEM: the stem rows / planes modes (direct row stores; separate instances so the
// other kernels do not carry their code)
template <int BN, int TS, bool PAIR, int TAPN = 0, bool STEM = false>
struct ConvSmem {
  static_assert(BN == 32 || BN == 64 || BN == 128 || BN == 256, "tile width");
  static constexpr int kBN = BN;
  static constexpr int kARows = TS == 1 ? kBlockM : kBlockM + 8;    // +8: row shifts 0..2
  static constexpr int kALoadBytes = kARows * 128;                  // bytes TMA delivers
  static constexpr int kABytes = (kALoadBytes + 1023) / 1024 * 1024;
  static constexpr int kBRows = PAIR ? BN / 2 : BN;                 // B rows held per tap
  static constexpr int kBTapBytes = kBRows * kBlockK * 2;
  static constexpr int kBBytes = (TAPN ? 3 : TS) * kBTapBytes;
  // epilogue chunk (columns); stems: EB_STEM_CW (32: both epilogue warp groups take half
  // of every tile's columns instead of alternating tiles)
  static constexpr int kCW = STEM ? (BN < EB_STEM_CW ? BN : EB_STEM_CW) : (BN < 64 ? BN : 64);
  // one warp's 32-row chunk; tap-shift tiles store directly (no staging, no residual)
  static constexpr int kStageOutBytes = (TS == 1 && !TAPN) ? 32 * kCW * 2 : 0;
  // pre-activation scale/shift cache (DenseNet 1x1 convs, cout = 128): 2 x 2048 floats
  static constexpr int kPreMax = (BN == 128 && TS == 1 && !PAIR && !TAPN && !STEM) ? 2048 : 0;
  // ring: 16 chunk buffers (4 warps x 4 or 8 warps x 2); tap-shift / taps-in-N tiles
  // instead stage 32 rows x 32 columns per warp for coalesced row stores
  static constexpr int kRowStageBytes = 32 * 32 * 2;
  // (stems: one chunk buffer per warp -- their whole-filter stages need the space)
  static constexpr int kRingArea = STEM ? (8 * EB_STEM_NB * kStageOutBytes > 8 * kRowStageBytes
                                              ? 8 * EB_STEM_NB * kStageOutBytes
                                              : 8 * kRowStageBytes)
                                   : (TS == 1 && !TAPN) ? 16 * kStageOutBytes
                                                        : 8 * kRowStageBytes;
  // tall taps-in-N: per epilogue group, two tile-parity buffers of the boundary rows three
  // lane quarters hand to the quarter above (96 floats each)
  static constexpr int kXchBytes = (TAPN & 8) ? 2 * 2 * 3 * 96 * 4 : 0;
  // bias cache: 8 warps x BN floats
  static constexpr int kEpiBytes = kRingArea + 8 * BN * 4 + 2 * kPreMax * 4 + kXchBytes;
  // dynamic smem: everything (one CTA per SM); 1 KiB alignment slack + barrier block
  static constexpr int kBytes = 232448;
  // up to 32 stages x 3 + 2 x 4 accumulators + 16 + 2 mbarriers (EB_MAX_ACC=8 needs 1088)
  static constexpr int kBarBytes = EB_MAX_ACC >= 8 ? 1088 : 1024;
  static constexpr int kBudget = kBytes - 1024 - kBarBytes;
  // barrier block: 3 x 32 + 21 mbarriers + TMEM slot; small stages (stems) run deep rings
  static constexpr int kMaxStages = 32;
  static_assert((kBudget - kEpiBytes) / (kABytes + kBBytes) >= 2, "pipeline needs two stages");
};

// Shared-memory layout, chosen per launch: [resident B (optional)] [stage ring of A (+B)]
// [epilogue rings] [bias caches] [pre-activation cache] [barriers].  With resident B
// (single N tile, short K) the weights are loaded once per CTA and the ring holds A only,
// so the same space buys a deeper A pipeline.
struct SmemLayout {
  int resb_bytes, stage_bytes, stages, out_off, bias_off, pre_off, xch_off, bar_off;
};
// A bytes per stage: the stem modes stage one (rows) or two (planes) 136-pixel runs
// A bytes per stage: the stem modes stage one (rows) or two (planes) 136-pixel runs per
// filter row, kbs filter rows per stage
constexpr int kStemPlaneOff = 2304;  // planes mode: the odd-column run's offset in a row block
__host__ __device__ inline int stem_run_bytes(int a_mode) {
  return a_mode == kAModeStemRows ? 2304 : a_mode == kAModeStemPlanes ? 4608 : 0;
}
__host__ __device__ inline int stem_a_bytes(int a_mode, int kbs) {
  const int b = stem_run_bytes(a_mode) * (kbs > 0 ? kbs : 1);
  return (b + 1023) / 1024 * 1024;
}
// stem stage A bytes: kbs row runs, or (tall stems) one stem_lines-line load per plane
__host__ __device__ inline int stem_stage_bytes(const ConvParams& p, int kbs) {
  if (p.stem_lines) {
    const int b = p.stem_lines * 128 * (p.a_mode == kAModeStemPlanes ? 2 : 1);
    return (b + 1023) / 1024 * 1024;
  }
  return stem_a_bytes(p.a_mode, kbs);
}
template <class S>
__host__ __device__ inline SmemLayout make_layout(const ConvParams& p) {
  SmemLayout L;
  const int kbs = p.kbs > 0 ? p.kbs : 1;
  // A bytes of one stage: stems their row runs; tall taps-in-N one tall_rows-row load per
  // channel chunk (every filter row of it resident, kh B tiles per chunk)
  const int ab = stem_run_bytes(p.a_mode) ? stem_stage_bytes(p, kbs) : p.tall_rows * 128 * kbs;
  const int bb = S::kBBytes * kbs;  // B bytes of one stage
  L.resb_bytes = p.resb ? p.num_kb * bb * (p.tall_rows ? p.taps / p.kw : 1) : 0;
  L.stage_bytes = (ab ? ab : S::kABytes * kbs) + (p.resb ? 0 : bb);
  int st = (S::kBudget - S::kEpiBytes + (p.ring_half ? S::kRingArea / 2 : 0) - L.resb_bytes) / L.stage_bytes;
  L.stages = st > S::kMaxStages ? S::kMaxStages : st;
  L.out_off = L.resb_bytes + L.stages * L.stage_bytes;
  // (ring_half: plain tiles without a residual keep one chunk buffer per epilogue warp and
  // give the other half of the ring to the A/B stages)
  L.bias_off = L.out_off + (p.ring_half ? S::kRingArea / 2 : S::kRingArea);
  L.pre_off = L.bias_off + 8 * S::kBN * 4;
  L.xch_off = L.pre_off + 2 * S::kPreMax * 4;
  L.bar_off = L.xch_off + S::kXchBytes;
  return L;
}
// Persistent tile walk t = t_first, t_first + t_step, ...; t = (z * mtp + pm) * nt + tn.
// Advanced incrementally (the step is decomposed once) so no warp divides per tile.
struct TileWalk {
  int tn, pm, z;
  int dn, dm, dz, nt, mtp;
  __device__ __forceinline__ void init(int t, int step, int nt_, int mtp_) {
    nt = nt_;
    mtp = mtp_;
    tn = t % nt;
    pm = (t / nt) % mtp;
    z = t / nt / mtp;
    dn = step % nt;
    dm = (step / nt) % mtp;
    dz = step / nt / mtp;
  }
  __device__ __forceinline__ void next() {
    tn += dn;
    int c = 0;
    if (tn >= nt) {
      tn -= nt;
      c = 1;
    }
    pm += dm + c;
    c = 0;
    if (pm >= mtp) {
      pm -= mtp;
      c = 1;
    }
    z += dz + c;
  }
};

// Coalesced store of a warp's 32 rows x 32 bf16 columns whose output rows are not
// contiguous (tap-shift / taps-in-N tiles walk a padded pixel grid).  Each lane stages
// its row (4 x 16 B, XOR-swizzled against bank conflicts), then the warp writes 8 rows
// x 64 B per instruction using the row addresses of the lanes that own them (null =
// row not stored).
// base: the warp's column origin (out + out_off + n); my_row: this lane's output row
// (pixel index) or -1 when the row is not stored.
__device__ __forceinline__ void stage_store_rows32(uint8_t* buf, const uint32_t* pk, int lane,
                                                   __nv_bfloat16* base, int ld, int my_row) {
  const int sw = (lane >> 1) & 3;
#pragma unroll
  for (int u = 0; u < 4; ++u)
    *reinterpret_cast<uint4*>(buf + lane * 64 + ((u ^ sw) * 16)) =
        make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
  __syncwarp();
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const int row = it * 8 + (lane >> 2);
    const int u = lane & 3;
    const int orow = __shfl_sync(0xffffffffu, my_row, row);
    const uint4 q = *reinterpret_cast<const uint4*>(buf + row * 64 + ((u ^ ((row >> 1) & 3)) * 16));
    if (orow >= 0) {
      uint4* dst = reinterpret_cast<uint4*>(base + static_cast<size_t>(orow) * ld + u * 8);
      asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "r"(q.x), "r"(q.y),
                   "r"(q.z), "r"(q.w)
                   : "memory");
    }
  }
  __syncwarp();
}

// EB_TRACE timing probe: role r (0 producer, 1 MMA, 2 epilogue warp 2) of CTA 0 records
// up to 1024 (tag, clock) events
// Compiled in only with -DEB_ENABLE_TRACE (EB_BUILD_TRACE=1 python -m ...build): the
// probes cost instruction-cache space in the hot loops.
__device__ __forceinline__ void trace_ev(long long* tr, int role, int& n, int tag) {
#ifndef EB_ENABLE_TRACE
  return;
#endif
  if (tr && blockIdx.x == 0 && n < 1024) {
    const long long clk = clock64();
    tr[(role * 1024 + n) * 2] = (static_cast<long long>(tag) << 48) | (clk & 0xFFFFFFFFFFFFll);
    tr[(role * 1024 + n) * 2 + 1] = 0;
    ++n;
  }
}

// EB_TRACE CTA span probe: every CTA (< 1024) records global-timer stamps at entry (0),
// after its prologue (1) and at exit (2)
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void trace_cta(long long* tr, int which) {
#ifndef EB_ENABLE_TRACE
  return;
#endif
  if (tr && threadIdx.x == 0 && blockIdx.x < 1024)
    tr[3 * 1024 * 2 + blockIdx.x * 4 + which] = static_cast<long long>(global_ns());
}

// EB_DBG timing probes (trace build only): 2 = MMA does not wait for the stem gather,
// 3 = no pre-activation transform, 5 = no TMA output stores, 6 = epilogue loads TMEM
// and releases it, nothing else, 7 = stems: no A loads, 8 = 6 and 7, 9 = return at entry.  Results are wrong under a
// probe; timing only.
__device__ __forceinline__ bool dbg_probe(const ConvParams& p, int which) {
#ifdef EB_ENABLE_TRACE
  return p.dbg == which;
#else
  return false;
#endif
}

__device__ __forceinline__ int swz_chunk(int chunk, int row, int cw) {
  // TMA SWIZZLE_128B (128 B rows): 16 B chunk ^= row % 8
  // TMA SWIZZLE_64B  (64 B rows):  16 B chunk ^= (row / 2) % 4
  return cw == 64 ? (chunk ^ (row & 7)) : (chunk ^ ((row >> 1) & 3));
}

template <int BN, int TS, bool PAIR, int TAPN, bool STEM>
__global__ void __launch_bounds__(kThreads, 1)
    conv_umma_kernel(const __grid_constant__ CUtensorMap map_a,
                     const __grid_constant__ CUtensorMap map_b,
                     const __grid_constant__ CUtensorMap map_out,
                     const __grid_constant__ CUtensorMap map_res, const ConvParams p) {
  using S = ConvSmem<BN, TS, PAIR, TAPN, STEM>;
  extern __shared__ uint8_t smem_raw[];
  // 128B swizzle needs 1024-byte aligned tiles
  // (offset arithmetic on the __shared__ array keeps the address space visible to the
  // compiler, so staging accesses compile to STS/LDS rather than generic ST/LD)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const SmemLayout L = make_layout<S>(p);
  constexpr bool stem_direct = STEM;  // a_mode is kAModeStemRows / kAModeStemPlanes
  const int kbs = p.kbs > 0 ? p.kbs : 1;  // 64-wide K blocks per stage (stems, taps-in-N)
  constexpr bool tall = (TAPN & 8) != 0;  // tall taps-in-N (one load per channel chunk)
  const int a_chunk = tall ? p.tall_rows * 128 : S::kABytes;  // A bytes of one K block
  const int a_stage = stem_direct ? stem_stage_bytes(p, kbs) : a_chunk * kbs;  // B follows A
  const int b_stage = S::kBBytes * kbs;
  uint8_t* const ring_base = smem + L.resb_bytes;  // stage s at ring_base + s * stage_bytes
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar_off);
  uint64_t* empty = full + L.stages;
  // TMEM accumulators: four when they fit the 512 columns (the MMA may then run up to three
  // tiles ahead of a slow epilogue), else two
  constexpr int kAccCols = TAPN ? 3 * BN : BN;  // TMEM columns per accumulator
  constexpr int kNAcc = (EB_MAX_ACC >= 8 && 8 * kAccCols <= 512)   ? 8
                        : (EB_MAX_ACC >= 4 && 4 * kAccCols <= 512) ? 4
                                                                    : 2;
  uint64_t* tfull = empty + L.stages;  // [kNAcc] accumulator ready
  uint64_t* tempty = tfull + kNAcc;      // [kNAcc] accumulator drained
  uint64_t* rfull = tempty + kNAcc;      // [4 warps][4] residual chunk landed in ring buffer
  uint64_t* xfull = rfull + 16;          // [stages] A tile transformed (pre-activation)
  uint64_t* bres = xfull + L.stages;     // resident B landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bres + 1);

  trace_cta(p.trace, 0);
  if (dbg_probe(p, 9)) return;  // (probe 9: launch cost only)
  const uint32_t warp = warp_id();
  constexpr int kTileRows = tall ? 126 : TAPN ? 120 : kBlockM;  // output rows a tile advances
  constexpr int kAccAll = kNAcc * kAccCols;
  constexpr int kTmemCols = kAccAll <= 32 ? 32 : kAccAll <= 64 ? 64 : kAccAll <= 128 ? 128
                          : kAccAll <= 256 ? 256 : 512;
  const int mt = (p.M + kTileRows - 1) / kTileRows;
  const int nt = (p.N + BN - 1) / BN;
  const int splits = (p.num_kb + p.kb_per_split - 1) / p.kb_per_split;
  // Tile walk.  In cluster modes the two CTAs of a cluster take the two M tiles of a
  // pair (same N tile, same K range).  Multicast mode: each CTA loads half of the shared
  // B tile into both CTAs and runs its own M=128 MMAs.  PAIR mode: each CTA loads half
  // of B into its own smem and the leader (rank 0) issues M=256 2-SM MMAs for both.
  const uint32_t crank = p.mcast ? cluster_ctarank() : 0;
  const int mtp = p.mcast ? (mt + 1) / 2 : mt;
  const int total = mtp * nt * splits;
  const int t_first = p.mcast ? static_cast<int>(blockIdx.x) / 2 : static_cast<int>(blockIdx.x);
  const int t_step = p.mcast ? static_cast<int>(gridDim.x) / 2 : static_cast<int>(gridDim.x);
  // warps 6..9 help with A (stem gather / pre-activation) or, otherwise, double the epilogue
  const bool a_helper = p.a_mode == kAModeGatherC8 || (p.pre_scale != nullptr && kXformThreads > 64);
  const int n_epi = a_helper ? 4 : 8;

  if (p.a_mode == kAModeTapC8) {
    // K groups >= kw are never loaded: make them finite (zero) once
    for (int i = threadIdx.x; i < L.stages * (S::kABytes / 16); i += kThreads) {
      const int st = i / (S::kABytes / 16);
      const int off = i - st * (S::kABytes / 16);
      *reinterpret_cast<uint4*>(ring_base + st * L.stage_bytes + off * 16) = make_uint4(0, 0, 0, 0);
    }
    fence_proxy_async_smem();
  }
  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
    if (p.out_mode == kOutBF16) tma_prefetch_desc(&map_out);
    if (p.res || p.n_split) tma_prefetch_desc(&map_res);
    mbar_init(bres, 1);
    for (int s = 0; s < L.stages; ++s) {
      mbar_init(&full[s], 1);
      // multicast: both CTAs' MMAs free a slot; PAIR: the leader's MMAs free it in both
      mbar_init(&empty[s], (p.mcast && !PAIR) ? 2 : 1);
    }
    for (int a = 0; a < kNAcc; ++a) {
      mbar_init(&tfull[a], 1);
      // arrivals that drain one accumulator: the epilogue warps that read it (8 when the
      // two epilogue groups split each tile's chunks), doubled in PAIR mode where the
      // leader waits for both CTAs' epilogues
      const uint32_t drain =
          (n_epi == 8 && (TAPN ? (BN == 64 && !p.tapn_alt) : BN / S::kCW > 1)) ? 8u : 4u;
      mbar_init(&tempty[a], PAIR ? 2 * drain : drain);
    }
    for (int a = 0; a < 16; ++a) mbar_init(&rfull[a], 1);
    // A-gather mode: 128 per-thread cp.async arrivals; A-transform mode: one arrive per warp
    const uint32_t xcount = p.a_mode == kAModeGatherC8 ? 128u : kXformThreads / 32;
    for (int s = 0; s < L.stages; ++s) mbar_init(&xfull[s], xcount);
    fence_mbar_init();
  }
  if (warp == 1) {
    if constexpr (PAIR)
      tmem_alloc_pair(tmem_slot, kTmemCols);
    else
      tmem_alloc(tmem_slot, kTmemCols);
  }
  tc_fence_before();
  __syncthreads();
  if (p.mcast) cluster_sync();  // the peer's barriers exist before we multicast into it
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (warp == 0 && elect_one()) {
    // resident weights: no earlier kernel of the graph writes them, so they are fetched
    // before the PDL wait and land while the previous layer drains
    if (p.resb && PAIR) {
      // 2-SM taps-in-N: each CTA keeps its half of the stacked [tap0; tap1; tap2] rows
      // (rows 1.5*BN*crank .. +1.5*BN, as three BN/2-row boxes); both halves complete
      // on the leader's barrier
      const uint32_t rb = mapa_shared(smem_u32(bres), 0);
      if (crank == 0) mbar_arrive_expect_tx(bres, 2u * L.resb_bytes);
      for (int kb = 0; kb < p.num_kb * kbs; ++kb) {
        uint8_t* sb = smem + kb * S::kBBytes;
        const int r = kb / p.cchunks;
        const int cc = kb - r * p.cchunks;
        for (int box = 0; box < 3; ++box) {
          const int R = (3 * static_cast<int>(crank) + box) * (BN / 2);  // stacked row
          const int tap = R / BN;
          tma_load_2d_pair(sb + box * S::kBTapBytes, &map_b, rb,
                           ((r * p.kw + tap) * p.cchunks + cc) * kBlockK, R - tap * BN);
        }
      }
    } else if (p.resb) {
      // resident B (single N tile): every K block's weights, once per CTA
      mbar_arrive_expect_tx(bres, L.resb_bytes);
      // (stems: kbs K blocks per stage; tall taps-in-N: kh filter rows per channel chunk)
      const int n_res = p.num_kb * kbs * (tall ? p.taps / p.kw : 1);
      for (int kb = 0; kb < n_res; ++kb) {
        uint8_t* sb = smem + kb * S::kBBytes;
        if (TAPN || TS > 1) {
          const int r = kb / p.cchunks;
          const int cc = kb - r * p.cchunks;
          for (int s2 = 0; s2 < (TAPN ? 3 : TS); ++s2)
            tma_load_2d(sb + s2 * S::kBTapBytes, &map_b, bres,
                        ((r * p.kw + s2) * p.cchunks + cc) * kBlockK, 0);
        } else {
          tma_load_2d(sb, &map_b, bres, kb * kBlockK, 0);
        }
      }
    }
  }
  // PDL: everything above overlapped the previous layer's tail; from here on we read
  // its output.  Let the next layer's CTAs start their own prologue as SMs free up.
  pdl_wait();
  pdl_launch_dependents();
  trace_cta(p.trace, 1);

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      int tr_n = 0;
      TileWalk tw;
      tw.init(t_first, t_step, nt, mtp);
      for (int t = t_first; t < total; t += t_step, tw.next()) {
        const int tile_n = tw.tn;
        const int tile_m = p.mcast ? 2 * tw.pm + static_cast<int>(crank) : tw.pm;
        const int z = tw.z;
        const int kb0 = z * p.kb_per_split;
        const int kb1 = min(kb0 + p.kb_per_split, p.num_kb);
        const int m0 = tile_m * kBlockM;
        int img = 0, oh = 0, ow = 0;
        if (p.a_mode != kAModeTiled && !stem_direct && !TAPN) {
          const int gw = TS > 1 ? p.Wp : p.Wo;  // tap-shift tiles walk the padded grid
          const int hw = p.Ho * gw;
          img = m0 / hw;
          const int rem = m0 - img * hw;
          oh = rem / gw;
          ow = rem - oh * gw;
        }
        const int base_w = ow * p.sw - p.pw;
        const int base_h = oh * p.sh - p.ph;
        const int n0 = tile_n * BN;
        // grouped conv (block-diagonal weights): this N tile's input channel window
        const int c_base = p.grouped ? n0 : 0;
        // stem rows / planes: first 128-byte line of this tile's filter row 0 (per tile)
        int stem_line0 = 0;
        const int stem_plane_lines = static_cast<int>(p.plane_px >> 3);
        if constexpr (stem_direct) {
          const int b = m0 / p.Mi;
          const int local = m0 - b * p.Mi;
          long long px;
          if (p.a_mode == kAModeStemRows) {
            px = static_cast<long long>(b) * p.Hq * p.Wq + local;
          } else {
            const int oh = local / p.Wg;
            px = (static_cast<long long>(b) * p.Hq + 2 * oh) * p.Wq + (local - oh * p.Wg);
          }
          stem_line0 = static_cast<int>(px >> 3);
        }
        // taps-in-N: receptive-field origins of the four 32-row quarter loads (per tile)
        int qw[4] = {0, 0, 0, 0}, qh[4] = {0, 0, 0, 0}, qi[4] = {0, 0, 0, 0};
        if constexpr (tall) {
          // the tile's first grid position (rows of Ho + kh - 1 per image) at filter row 0
          const int hwq = (p.Ho + p.taps / p.kw - 1) * p.Wp;
          const int m0 = tile_m * kTileRows;
          qi[0] = m0 / hwq;
          const int rem = m0 - qi[0] * hwq;
          qh[0] = rem / p.Wp;
          qw[0] = rem - qh[0] * p.Wp - p.pw;
          qh[0] -= p.ph;
        } else if constexpr (TAPN) {
          if constexpr ((TAPN & 4) != 0) {
            // fused 2x2 max-pool: a tile is output rows 2r, 2r+1 x columns [60 sg, 60 sg + 60)
            // of one image; quarters 0/1 = row 2r (30 columns each), 2/3 = row 2r + 1
            const int sg = tile_m % p.nseg;
            const int rowp = tile_m / p.nseg;
            const int img = rowp / p.Ho2;
            const int r = rowp - img * p.Ho2;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              qi[q] = img;
              qh[q] = 2 * r + (q >> 1) - p.ph;
              // (a quarter that starts past the row's end only feeds junk lanes: load the
              // segment's first one again rather than hand the TMA an out-of-range origin)
              const int c0 = 60 * sg + 30 * (q & 1);
              qw[q] = (c0 < p.Wo ? c0 : 60 * sg) - p.pw;
            }
          } else {
          const int hw = p.Ho * p.Wp;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int mq = tile_m * kTileRows + 30 * q;
            qi[q] = mq / hw;
            const int qrem = mq - qi[q] * hw;
            qh[q] = qrem / p.Wp;
            qw[q] = qrem - qh[q] * p.Wp - p.pw;
            qh[q] -= p.ph;
          }
          }
        }
        // K-block coordinates, advanced incrementally: kb = (row_or_tap * cchunks + cc), and
        // for im2col tap = r * kw + s
        int cc = kb0 % p.cchunks;
        int outer = kb0 / p.cchunks;
        int rr = outer / p.kw;
        int ss = outer - rr * p.kw;
        auto next_k = [&] {
          if (++cc == p.cchunks) {
            cc = 0;
            ++outer;
            if (++ss == p.kw) {
              ss = 0;
              ++rr;
            }
          }
        };
        for (int kb = kb0; kb < kb1; ++kb, next_k()) {
          mbar_wait(&empty[stage], phase ^ 1);
          trace_ev(p.trace, 0, tr_n, 1);
          uint8_t* sa = ring_base + stage * L.stage_bytes;
          uint8_t* sb = p.resb ? smem + kb * b_stage : sa + a_stage;
          if constexpr (TAPN) {
            // filter row r, channel chunk cc: lane quarter q's 32 rows are the padded-grid
            // pixels m0 + 30q ..; B = the row's 3 taps stacked along N
            // (kbs K blocks per stage: block g = kb * kbs + sub)
            if constexpr (PAIR) {
              // 2-SM: each CTA stages its own tile's A; B is resident (halves per CTA);
              // both CTAs' loads complete on the leader's barrier
              const uint32_t fb = mapa_shared(smem_u32(&full[stage]), 0);
              if (crank == 0) mbar_arrive_expect_tx(&full[stage], 2u * kbs * (4 * 32 * 128));
              for (int sub = 0; sub < kbs; ++sub) {
                const int g = kb * kbs + sub;
                const int r = g / p.cchunks;
                const int gc = g - r * p.cchunks;
#pragma unroll
                for (int q = 0; q < 4; ++q)
                  tma_load_im2col_4d_pair(sa + sub * S::kABytes + q * 4096, &map_a, fb, gc * kBlockK,
                                          qw[q], qh[q], qi[q], 0, static_cast<uint16_t>(r));
              }
            } else if constexpr (tall) {
              // one load per channel chunk: tall_rows grid positions at filter row 0; filter
              // row r reads the same rows r * Wp further (B resident)
              mbar_arrive_expect_tx(&full[stage], kbs * p.tall_rows * 128);
              for (int sub = 0; sub < kbs; ++sub)
                tma_load_im2col_4d(sa + sub * a_chunk, &map_a, &full[stage], (kb * kbs + sub) * kBlockK,
                                   qw[0], qh[0], qi[0], 0, 0);
            } else {
            mbar_arrive_expect_tx(&full[stage], kbs * (4 * 32 * 128 + (p.resb ? 0 : S::kBBytes)));
            for (int sub = 0; sub < kbs; ++sub) {
              const int g = kb * kbs + sub;
              const int r = g / p.cchunks;
              const int gc = g - r * p.cchunks;
#pragma unroll
              for (int q = 0; q < 4; ++q)
                tma_load_im2col_4d(sa + sub * S::kABytes + q * 4096, &map_a, &full[stage], gc * kBlockK,
                                   qw[q], qh[q], qi[q], 0, static_cast<uint16_t>(r));
              if (!p.resb) {
#pragma unroll
                for (int s2 = 0; s2 < 3; ++s2)
                  tma_load_2d(sb + sub * S::kBBytes + s2 * S::kBTapBytes, &map_b, &full[stage],
                              ((r * p.kw + s2) * p.cchunks + gc) * kBlockK, n0);
              }
            }
            }
            if (++stage == L.stages) {
              stage = 0;
              phase ^= 1;
            }
            continue;
          }
          if constexpr (PAIR) {
            // both CTAs' loads complete on the leader's barrier, which expects them all
            const uint32_t fb = mapa_shared(smem_u32(&full[stage]), 0);
            if (crank == 0) mbar_arrive_expect_tx(&full[stage], 2u * (S::kALoadBytes + S::kBBytes));
            const int nb = n0 + static_cast<int>(crank) * S::kBRows;
            if (TS > 1) {
              const int r = outer;
              tma_load_im2col_4d_pair(sa, &map_a, fb, c_base + cc * kBlockK, base_w, base_h, img, 0,
                                      static_cast<uint16_t>(r));
#pragma unroll
              for (int s2 = 0; s2 < TS; ++s2)
                tma_load_2d_pair(sb + s2 * S::kBTapBytes, &map_b, fb,
                                 ((r * p.kw + s2) * p.cchunks + cc) * kBlockK, nb);
            } else {
              if (p.a_mode == kAModeTiled) {
                tma_load_2d_pair(sa, &map_a, fb, kb * kBlockK, m0);
              } else {
                tma_load_im2col_4d_pair(sa, &map_a, fb, c_base + cc * kBlockK, base_w, base_h, img,
                                        static_cast<uint16_t>(ss), static_cast<uint16_t>(rr));
              }
              tma_load_2d_pair(sb, &map_b, fb, kb * kBlockK, nb);
            }
            if (++stage == L.stages) {
              stage = 0;
              phase ^= 1;
            }
            continue;
          }
          {
            const uint32_t bbytes = p.resb ? 0u : static_cast<uint32_t>(S::kBBytes);
            const uint32_t abytes = p.a_mode == kAModeGatherC8 ? 0u
                                    : p.a_mode == kAModeTapC8
                                        ? static_cast<uint32_t>(p.kw * kTapC8Bytes)
                                    : p.stem_lines ? static_cast<uint32_t>(p.stem_lines * 128 *
                                                                           (p.a_mode == kAModeStemPlanes ? 2 : 1))
                                    : p.a_mode == kAModeStemRows   ? 2176u * kbs
                                    : p.a_mode == kAModeStemPlanes ? 4352u * kbs
                                                                   : static_cast<uint32_t>(S::kALoadBytes);
            // (gather mode with resident B: this stage only waits for the cp.async arrivals)
            mbar_arrive_expect_tx(&full[stage], (dbg_probe(p, 7) || dbg_probe(p, 8)) && stem_direct ? bbytes : abytes + bbytes);
          }
          if (TS > 1) {
            // filter row r, channel chunk cc: 136 consecutive padded-grid pixels at tap (r, 0);
            // tap (r, s) is the same buffer shifted down by s rows
            const int r = outer;
            tma_load_im2col_4d(sa, &map_a, &full[stage], c_base + cc * kBlockK, base_w, base_h,
                               img, 0, static_cast<uint16_t>(r));
            if (!p.resb) {
#pragma unroll
              for (int s2 = 0; s2 < TS; ++s2)
                tma_load_2d(sb + s2 * S::kBTapBytes, &map_b, &full[stage],
                            ((r * p.kw + s2) * p.cchunks + cc) * kBlockK, n0);
            }
          } else if (p.a_mode == kAModeTiled) {
            tma_load_2d(sa, &map_a, &full[stage], kb * kBlockK, m0);
          } else if (p.a_mode == kAModeIm2col) {
            tma_load_im2col_4d(sa, &map_a, &full[stage], c_base + cc * kBlockK, base_w, base_h,
                               img, static_cast<uint16_t>(ss), static_cast<uint16_t>(rr));
          } else if (stem_direct) {
            // filter row kb of a 128-position tile: contiguous 136-pixel runs (17 lines of
            // 8 pixels x 8 channels) of the padded layout; the next filter row is Wq
            // pixels further in both layouts
            const int run = stem_run_bytes(p.a_mode);
            if (dbg_probe(p, 7) || dbg_probe(p, 8)) {
              // (probe 7/8: no A loads -- the MMAs read stale smem; timing only)
            } else if (p.stem_lines) {
              // tall stem: one load per plane covers every filter row of the tile (row r is
              // Wq pixels = Wq / 8 lines further); the odd plane follows the even one
              const int line = stem_line0 + kb * kbs * (p.Wq >> 3);
              tma_load_2d(sa, &map_a, &full[stage], 0, line);
              if (p.a_mode == kAModeStemPlanes)
                tma_load_2d(sa + p.stem_lines * 128, &map_a, &full[stage], 0, line + stem_plane_lines);
            } else
            for (int r = 0; r < kbs; ++r) {
              const int line = stem_line0 + (kb * kbs + r) * (p.Wq >> 3);
              tma_load_2d(sa + r * run, &map_a, &full[stage], 0, line);
              if (p.a_mode == kAModeStemPlanes)
                tma_load_2d(sa + r * run + kStemPlaneOff, &map_a, &full[stage], 0, line + stem_plane_lines);
            }
            trace_ev(p.trace, 0, tr_n, 2);
          } else if (p.a_mode == kAModeTapC8) {
            // filter row kb: tap s brings 128 pixels x 8 channels (16 B) = the K group s
            // column of core matrices (2 KiB, no swizzle); groups s >= kw keep stale
            // finite data that meets zero weights
            for (int s = 0; s < p.kw; ++s) {
              const int g = p.sw == 2 ? ((s & 1) ? 4 + (s >> 1) : (s >> 1)) : s;
              tma_load_im2col_4d(sa + g * kTapC8Bytes, &map_a, &full[stage], 0, base_w, base_h, img,
                                 static_cast<uint16_t>(s), static_cast<uint16_t>(kb));
            }
          }  // kAModeGatherC8: A is gathered by warps 6..9
          if (stem_direct && !p.resb) {
            for (int r = 0; r < kbs; ++r)
              tma_load_2d(sb + r * S::kBBytes, &map_b, &full[stage], (kb * kbs + r) * kBlockK, n0);
          } else if (TS == 1 && !p.resb) {
            if (p.mcast)  // our half of B, written into both CTAs
              tma_load_2d_mcast(sb + crank * (BN / 2) * 128, &map_b, &full[stage], kb * kBlockK,
                                n0 + static_cast<int>(crank) * (BN / 2), 0x3);
            else
              tma_load_2d(sb, &map_b, &full[stage], kb * kBlockK, n0);
          }
          if (++stage == L.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      if (p.mcast) {
        // producer tail: every MMA commit aimed at this CTA's empty barriers (some come
        // from the peer) has landed before the cluster may tear down
        for (int i = 0; i < L.stages; ++i) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (++stage == L.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = umma_idesc_bf16(PAIR ? 2 * kBlockM : kBlockM, TAPN ? 3 * BN : BN);
    constexpr uint32_t idesc_2bn = umma_idesc_bf16(kBlockM, 2 * BN);
    constexpr uint32_t idesc_bn = umma_idesc_bf16(kBlockM, BN);
    int stage = 0;
    uint32_t phase = 0;
    int j = 0;  // local tile counter
    // PAIR: the peer's MMA warp idles; the leader issues for both CTAs
    const int t_mma_end = (PAIR && crank != 0) ? 0 : total;
    if (p.resb && t_first < t_mma_end) mbar_wait(bres, 0);
    // K16 steps per K block that carry nonzero weights (step 0 always does), and the A
    // start-address offset of each step (16-byte units):
    //   128B-swizzled tiles: 32 B per step;  tap-C8: 2 KiB K groups, 4 KiB per step;
    //   stem rows/planes: taps are core matrices 16 B apart (overlapping, LBO = 16), the
    //   planes mode's odd-column run starts kStemPlaneOff into the stage.
    uint32_t kmask = 0xFu;
    uint32_t a_koff[4] = {0, 2, 4, 6};
    uint64_t a_desc_hi = umma_desc_sw128(0);
    const uint64_t b_desc_hi = umma_desc_sw128(0);
    if (p.a_mode == kAModeTapC8) {
      a_desc_hi = umma_desc(0, kTapC8Bytes, 128, 0);
      for (int k = 0; k < 4; ++k) a_koff[k] = k * 2 * kTapC8Bytes / 16;
    } else if (p.a_mode == kAModeStemRows) {
      a_desc_hi = umma_desc(0, 16, 128, 0);
      kmask = (1u << ((p.kw + 1) / 2)) - 1u;
    } else if (p.a_mode == kAModeStemPlanes) {
      a_desc_hi = umma_desc(0, 16, 128, 0);
      const int ne = ((p.kw + 1) / 2 + 1) / 2;  // even taps -> K groups 0..3
      const int no = (p.kw / 2 + 1) / 2;        // odd taps  -> K groups 4..7
      kmask = ((1u << ne) - 1u) | (((1u << no) - 1u) << 2);
      const uint32_t odd16 = p.stem_lines ? static_cast<uint32_t>(p.stem_lines * 8) : kStemPlaneOff / 16;
      a_koff[2] = odd16;
      a_koff[3] = odd16 + 2;
    }
    TileWalk tw;
    tw.init(t_first, t_step, nt, mtp);
    int tr_n = 0;
    for (int t = t_first; t < t_mma_end; t += t_step, ++j, tw.next()) {
      const int z = tw.z;
      const int kb0 = z * p.kb_per_split;
      const int kb1 = min(kb0 + p.kb_per_split, p.num_kb);
      const int acc = j % kNAcc;
      const uint32_t tmem_d = tmem_base + acc * kAccCols;
      mbar_wait(&tempty[acc], ((j / kNAcc) & 1) ^ 1);
      if (lane_id() == 0) trace_ev(p.trace, 1, tr_n, 10);
      tc_fence_after();
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(p.pre_scale ? &xfull[stage] : &full[stage], phase);
        if (p.a_mode == kAModeGatherC8 && !dbg_probe(p, 2)) mbar_wait(&xfull[stage], phase);
        if (lane_id() == 0) trace_ev(p.trace, 1, tr_n, 11);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sa = smem_u32(ring_base + stage * L.stage_bytes);
          const uint32_t sb = p.resb ? smem_u32(smem + kb * b_stage) : sa + a_stage;
          // descriptors: the per-kernel fields (LBO/SBO/layout) are fixed, so a K step or
          // a row shift only adds to the 14-bit start-address field (16-byte units)
          const uint64_t a0 = a_desc_hi | ((sa >> 4) & 0x3FFF);
          const uint64_t b0 = b_desc_hi | ((sb >> 4) & 0x3FFF);
          if constexpr (stem_direct) {
            // kbs filter rows per stage: row block r's run / B tile follow each other
            const uint32_t run16 = p.stem_lines ? static_cast<uint32_t>(p.Wq) : stem_run_bytes(p.a_mode) >> 4;
            for (int r = 0; r < kbs; ++r) {
#pragma unroll
              for (int k = 0; k < kBlockK / 16; ++k) {
                if (!((kmask >> k) & 1u)) continue;
                const uint64_t adesc = a0 + r * run16 + a_koff[k];
                const uint64_t bdesc = b0 + r * (S::kBBytes >> 4) + 2 * k;
                umma_bf16(tmem_d, adesc, bdesc, idesc, (kb > kb0 || r > 0 || k > 0) ? 1u : 0u);
              }
            }
          } else {
          if constexpr (tall) {
            // channel chunk cc's tall tile serves filter row r from r * Wp rows on; B of
            // (r, cc) is resident tile r * cchunks + cc
            const uint32_t wp16 = static_cast<uint32_t>(p.Wp) * 8;  // Wp rows of 128 B, 16 B units
            const uint32_t bres16 = (smem_u32(smem) >> 4) & 0x3FFF;
            for (int sub = 0; sub < kbs; ++sub) {
              const int cc = kb * kbs + sub;
#pragma unroll
              for (int r = 0; r < 3; ++r) {
                const uint64_t bt = b_desc_hi + bres16 + (r * p.cchunks + cc) * (S::kBBytes >> 4);
#pragma unroll
                for (int k = 0; k < kBlockK / 16; ++k) {
                  const uint64_t adesc = a0 + sub * (a_chunk >> 4) + r * wp16 + 2 * k;
                  const uint32_t accum = (kb > kb0 || sub > 0 || r > 0 || k > 0) ? 1u : 0u;
                  umma_bf16(tmem_d, adesc, bt + 2 * k, idesc, accum);
                }
              }
            }
          } else
          for (int sub = 0; sub < kbs; ++sub) {  // (kbs > 1: taps-in-N only)
#pragma unroll
          for (int s2 = 0; s2 < TS; ++s2) {
#pragma unroll
            for (int k = 0; k < kBlockK / 16; ++k) {
              // a shift of s2 rows is a start address 128 B further: the 128B swizzle is
              // applied on absolute smem address bits (base offset field stays 0), which
              // is also what the TMA used when it wrote the tile (verified on B200)
              if (!((kmask >> k) & 1u)) continue;  // (stems: all-zero weight steps)
              const uint64_t adesc = a0 + sub * (S::kABytes >> 4) + s2 * 8 + a_koff[k];
              const uint64_t bdesc = b0 + sub * (S::kBBytes >> 4) + s2 * (S::kBTapBytes >> 4) + 2 * k;
              const uint32_t accum = (kb > kb0 || sub > 0 || s2 > 0 || k > 0) ? 1u : 0u;
              if constexpr (PAIR) {
                umma_bf16_pair(tmem_d, adesc, bdesc, idesc, accum);
              } else if constexpr (TAPN) {
                if constexpr ((TAPN & 3) == 2) {
                  // planes 0|1 = A x [tap0; tap1]; plane 0 += (A two rows on) x tap2: the
                  // epilogue then adds one shifted plane instead of two
                  umma_bf16(tmem_d, adesc, bdesc, idesc_2bn, accum);
                  umma_bf16(tmem_d, adesc + 16, bdesc + (2 * BN * 128 >> 4), idesc_bn, 1u);
                } else {
                  umma_bf16(tmem_d, adesc, bdesc, idesc, accum);
                }
              } else {
                umma_bf16(tmem_d, adesc, bdesc, idesc, accum);
              }
            }
          }
          }
          }
          if constexpr (PAIR) {
            umma_commit_pair_mcast(&empty[stage], 0x3);
            if (kb == kb1 - 1) umma_commit_pair_mcast(&tfull[acc], 0x3);
          } else {
            if (p.mcast)
              umma_commit_mcast(&empty[stage], 0x3);  // the slot is free in both CTAs
            else
              umma_commit(&empty[stage]);
            if (kb == kb1 - 1) umma_commit(&tfull[acc]);
          }
        }
        __syncwarp();
        if (lane_id() == 0) trace_ev(p.trace, 1, tr_n, 12);
        if (++stage == L.stages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (TAPN && warp < 2 + n_epi) {
    // ------------------------------------------------------------ epilogue, taps-in-N
    // Lane l of quarter q owns padded-grid row m = tile*120 + 30q + l; its output is
    //   out[m] = D0[m] + D1[m+1] + D2[m+2]   (D_s = the tap-s column block)
    // (tapn2: the MMA warp already accumulated D2[m+2] into plane 0 through a 2-row
    // shifted A descriptor, so only plane 1 is shuffled)
    // and rows m+1, m+2 live in lanes l+1, l+2 of the same warp (quarters overlap by 2
    // rows, lanes 30/31 only feed their neighbours).  With 64 output channels the two
    // epilogue groups split every tile's columns (32 each: the accumulator is released as
    // soon as both have loaded their half); with 32 they take alternate tiles.  Row
    // stores are staged per warp (rows are not contiguous in the output).
    const int ew = static_cast<int>(warp) - 2;
    const int half = ew >> 2;
    const uint32_t quarter = warp & 3;
    const int lane = static_cast<int>(lane_id());
    const bool split_cols = n_epi == 8 && BN == 64 && !p.tapn_alt;
    const bool alt = n_epi == 8 && !split_cols;
    const int c_lo = split_cols ? 32 * half : 0;
    const int c_hi = split_cols ? c_lo + 32 : BN;
    const __nv_bfloat162 zero2 = __floats2bfloat162_rn(0.f, 0.f);
    const int hw = p.Ho * p.Wp;
    int tr_n = 0;
    float* bias_s = reinterpret_cast<float*>(smem + L.bias_off) + ew * BN;
    int pool_round = 0;  // fused pool: vertical exchanges done (upper quarters)
    int cached_n = -1;
    const int j0 = alt ? half : 0;
    const int jstep = alt ? 2 : 1;
    int j = j0;
    TileWalk tw;
    tw.init(t_first + j0 * t_step, jstep * t_step, nt, mtp);
    for (int t = t_first + j0 * t_step; t < total; t += jstep * t_step, j += jstep, tw.next()) {
      if (tw.tn != cached_n) {
        __syncwarp();
        for (int i = lane; i < BN; i += 32)
          bias_s[i] = (p.bias && tw.tn * BN + i < p.N) ? __ldg(p.bias + tw.tn * BN + i) : 0.f;
        __syncwarp();
        cached_n = tw.tn;
      }
      const int acc = j % kNAcc;
      const int tile_m = p.mcast ? 2 * tw.pm + static_cast<int>(crank) : tw.pm;
      bool ok;
      size_t orow;
      if constexpr ((TAPN & 4) != 0) {
        // pooled pixel (r, 30 sg + 15 (quarter & 1) + lane / 2), held by the even lanes of
        // the row-2r quarters (0, 1) after the max over the 2x2 window
        const int sg = tile_m % p.nseg;
        const int rowp = tile_m / p.nseg;
        const int ow = 60 * sg + 30 * static_cast<int>(quarter & 1) + lane;
        ok = lane < 30 && !(lane & 1) && ow < p.Wo;
        orow = static_cast<size_t>(rowp) * p.Wo2 + (ow >> 1);
      } else if constexpr (tall) {
        // 126-row tiles of the (Ho + kh - 1) x Wp grid: every lane of quarters 0-2 and lanes
        // 0-29 of quarter 3 own a grid position; the 2 extra rows per image are junk
        const int m = tile_m * kTileRows + static_cast<int>(quarter) * 32 + lane;
        const int img = fdiv(m, p.fd_img);
        const int rem = m - img * static_cast<int>(p.fd_img.d);
        const int oh = fdiv(rem, p.fd_row);
        const int owp = rem - oh * p.Wp;
        ok = (quarter < 3 || lane < 30) && m < p.M && oh < p.Ho && owp < p.Wo;
        orow = (static_cast<size_t>(img) * p.Ho + oh) * p.Wo + owp;
      } else {
        const int m = tile_m * kTileRows + static_cast<int>(quarter) * 30 + lane;
        const int img = fdiv(m, p.fd_img);
        const int rem = m - img * hw;
        const int oh = fdiv(rem, p.fd_row);
        const int owp = rem - oh * p.Wp;
        ok = lane < 30 && m < p.M && owp < p.Wo;
        orow = (static_cast<size_t>(img) * p.Ho + oh) * p.Wo + owp;
      }
      const int n_tile0 = tw.tn * BN;
      if (warp == 2 && lane == 0) trace_ev(p.trace, 2, tr_n, 20);
      mbar_wait(&tfull[acc], (j / kNAcc) & 1);
      if (warp == 2 && lane == 0) trace_ev(p.trace, 2, tr_n, 21);
      tc_fence_after();
      const uint32_t tb = tmem_base + acc * kAccCols + ((quarter * 32) << 16);
#pragma unroll
      for (int c = c_lo; c < c_hi; c += 32) {
        const int n = n_tile0 + c;
        uint32_t r0[32], r1[32], r2[32];
        constexpr bool two = !PAIR && (TAPN & 3) == 2;
        tmem_ld32(tb + c, r0);
        tmem_ld32(tb + BN + c, r1);
        if constexpr (!two) tmem_ld32(tb + 2 * BN + c, r2);
        tmem_ld_wait();
        if (c + 32 >= c_hi && p.early_release) {  // last TMEM read of the tile: hand it back now
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (PAIR && crank != 0)  // the leader's MMAs write our TMEM: release it there
              mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));
            else
              mbar_arrive(&tempty[acc]);
          }
        }
        // ((D0 + D1') + D2') + bias on fp32 pairs (FADD2), the shifted planes by shuffle
        float2 v2[16];
        if constexpr (tall) {
          // rows m+1, m+2 of lanes 31 / 30-31 live in the next quarter's warp: each quarter
          // above 0 hands its lanes 0-1 of planes 1-2 down through smem (double-buffered by
          // tile parity; one named barrier per tile and group)
          float* xb = reinterpret_cast<float*>(smem + L.xch_off) + (half * 2 + ((j >> 1) & 1)) * 3 * 96;
          if (quarter > 0 && lane < 2) {
            float4* dst = reinterpret_cast<float4*>(xb + (quarter - 1) * 96);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              if (lane == 0)
                dst[i] = make_float4(__uint_as_float(r1[4 * i]), __uint_as_float(r1[4 * i + 1]),
                                     __uint_as_float(r1[4 * i + 2]), __uint_as_float(r1[4 * i + 3]));
              dst[8 + 8 * lane + i] = make_float4(__uint_as_float(r2[4 * i]), __uint_as_float(r2[4 * i + 1]),
                                                  __uint_as_float(r2[4 * i + 2]), __uint_as_float(r2[4 * i + 3]));
            }
          }
          named_bar_sync(2 + half, 128);
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            r1[i] = __shfl_down_sync(0xffffffffu, r1[i], 1);
            r2[i] = __shfl_down_sync(0xffffffffu, r2[i], 2);
          }
          if (quarter < 3 && lane >= 30) {
            const float4* src = reinterpret_cast<const float4*>(xb + quarter * 96);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              if (lane == 31) {
                const float4 a = src[i];
                r1[4 * i] = __float_as_uint(a.x);
                r1[4 * i + 1] = __float_as_uint(a.y);
                r1[4 * i + 2] = __float_as_uint(a.z);
                r1[4 * i + 3] = __float_as_uint(a.w);
              }
              const float4 b = src[8 + 8 * (lane - 30) + i];
              r2[4 * i] = __float_as_uint(b.x);
              r2[4 * i + 1] = __float_as_uint(b.y);
              r2[4 * i + 2] = __float_as_uint(b.z);
              r2[4 * i + 3] = __float_as_uint(b.w);
            }
          }
#pragma unroll
          for (int i = 0; i < 16; ++i)
            v2[i] = __fadd2_rn(__fadd2_rn(make_float2(__uint_as_float(r0[2 * i]), __uint_as_float(r0[2 * i + 1])),
                                          make_float2(__uint_as_float(r1[2 * i]), __uint_as_float(r1[2 * i + 1]))),
                               make_float2(__uint_as_float(r2[2 * i]), __uint_as_float(r2[2 * i + 1])));
        } else if constexpr (two) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float2 d1 = make_float2(__shfl_down_sync(0xffffffffu, __uint_as_float(r1[2 * i]), 1),
                                          __shfl_down_sync(0xffffffffu, __uint_as_float(r1[2 * i + 1]), 1));
            v2[i] = __fadd2_rn(make_float2(__uint_as_float(r0[2 * i]), __uint_as_float(r0[2 * i + 1])), d1);
          }
        } else
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float2 d1 = make_float2(__shfl_down_sync(0xffffffffu, __uint_as_float(r1[2 * i]), 1),
                                        __shfl_down_sync(0xffffffffu, __uint_as_float(r1[2 * i + 1]), 1));
          const float2 d2 = make_float2(__shfl_down_sync(0xffffffffu, __uint_as_float(r2[2 * i]), 2),
                                        __shfl_down_sync(0xffffffffu, __uint_as_float(r2[2 * i + 1]), 2));
          v2[i] = __fadd2_rn(__fadd2_rn(make_float2(__uint_as_float(r0[2 * i]), __uint_as_float(r0[2 * i + 1])),
                                        d1),
                             d2);
        }
        if constexpr ((TAPN & 4) != 0) {
          // max over the 2x2 window before bias / ReLU / rounding (all monotone, so this
          // equals pooling the rounded conv output): horizontal pairs are lanes (2k, 2k+1);
          // vertical pairs are quarters q and q + 2, exchanged through the upper quarter's
          // staging slot (float4 chunks XOR-swizzled by pair index)
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            v2[i].x = fmaxf(v2[i].x, __shfl_down_sync(0xffffffffu, v2[i].x, 1));
            v2[i].y = fmaxf(v2[i].y, __shfl_down_sync(0xffffffffu, v2[i].y, 1));
          }
          const bool upper = quarter >= 2;
          float4* xb = reinterpret_cast<float4*>(smem + L.out_off + (upper ? ew : ew - 2) * S::kRowStageBytes);
          const int h = lane >> 1;
          const int bar_id = 2 + half * 2 + static_cast<int>(quarter & 1);
          if (upper) {
            if (pool_round > 0) named_bar_sync(bar_id + 4, 64);  // reader done with the last tile
            if (!(lane & 1) && lane < 30)
#pragma unroll
              for (int c4 = 0; c4 < 8; ++c4)
                xb[h * 8 + (c4 ^ (h & 7))] = make_float4(v2[2 * c4].x, v2[2 * c4].y, v2[2 * c4 + 1].x, v2[2 * c4 + 1].y);
            named_bar_arrive(bar_id, 64);
            ++pool_round;
            continue;
          }
          named_bar_sync(bar_id, 64);
          if (!(lane & 1) && lane < 30)
#pragma unroll
            for (int c4 = 0; c4 < 8; ++c4) {
              const float4 o = xb[h * 8 + (c4 ^ (h & 7))];
              v2[2 * c4].x = fmaxf(v2[2 * c4].x, o.x);
              v2[2 * c4].y = fmaxf(v2[2 * c4].y, o.y);
              v2[2 * c4 + 1].x = fmaxf(v2[2 * c4 + 1].x, o.z);
              v2[2 * c4 + 1].y = fmaxf(v2[2 * c4 + 1].y, o.w);
            }
          named_bar_arrive(bar_id + 4, 64);
        }
#pragma unroll
        for (int i = 0; i < (dbg_probe(p, 4) ? 0 : 8); ++i) {
          const float4 b4 = *reinterpret_cast<const float4*>(bias_s + c + 4 * i);
          v2[2 * i] = __fadd2_rn(v2[2 * i], make_float2(b4.x, b4.y));
          v2[2 * i + 1] = __fadd2_rn(v2[2 * i + 1], make_float2(b4.z, b4.w));
        }
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
          pk[i] = p.relu ? pack_bf16x2_relu(v2[i].x, v2[i].y) : pack_bf16x2(v2[i].x, v2[i].y);
        __nv_bfloat16* const col0 = reinterpret_cast<__nv_bfloat16*>(p.out) + p.out_off + n;
        __nv_bfloat16* o = col0 + orow * p.ldo;
        if constexpr ((TAPN & 4) != 0) {  // (vec_ok and N % 32 == 0 checked by the plan): 64 B per pooled pixel
          if (ok) {
            uint4* o4 = reinterpret_cast<uint4*>(o);
#pragma unroll
            for (int i = 0; i < 4; ++i)
              o4[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
          }
        } else if (p.vec_ok && n + 32 <= p.N) {
          stage_store_rows32(smem + L.out_off + ew * S::kRowStageBytes, pk, lane, col0, p.ldo,
                             ok ? static_cast<int>(orow) : -1);
        } else if (ok && n < p.N) {
          {
            const __nv_bfloat16* hv = reinterpret_cast<const __nv_bfloat16*>(pk);
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (n + i < p.N) o[i] = hv[i];
          }
        }
      }
      if (!p.early_release) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (PAIR && crank != 0)
            mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));
          else
            mbar_arrive(&tempty[acc]);
        }
      }
      if (warp == 2 && lane == 0) trace_ev(p.trace, 2, tr_n, 22);
    }
  } else if (warp < 2 + n_epi) {
    // ------------------------------------------------------------ epilogue
    // All per-element loops are fully unrolled with predicates so the chunk stays in
    // registers; the math runs on fp32 pairs (FADD2) and packed bf16 pairs (ReLU after
    // rounding is exact: rounding preserves sign).  The bias of the current N tile is
    // cached in smem per warp.  Each warp owns a ring of swizzled 32 x CW chunk
    // buffers: the residual of every chunk it will handle in a tile is TMA-loaded into
    // the ring as soon as the tile starts (overlapping its MMAs), the result is written
    // back in place and TMA-stored from there.
    // With 8 epilogue warps (no A helper in this mode) two warps share each TMEM lane
    // quarter: they split every tile's chunks, or -- one chunk per tile -- take
    // alternate tiles (and so alternate accumulator buffers).
    const int ew = static_cast<int>(warp) - 2;
    const int half = ew >> 2;
    const uint32_t quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int lane = static_cast<int>(lane_id());
    const int row = static_cast<int>(quarter * 32) + lane;
    constexpr int CW = S::kCW;
    constexpr int NCH = BN / CW;
    const bool wide = n_epi == 8;
    const bool alt_tiles = wide && NCH == 1;
    const int c_first = (wide && NCH > 1) ? half : 0;
    const int c_step = (wide && NCH > 1) ? 2 : 1;
    const int nb = (STEM ? EB_STEM_NB : wide ? 2 : 4) >> (p.ring_half ? 1 : 0);  // ring buffers per warp
    uint8_t* ring = smem + L.out_off + ew * nb * S::kStageOutBytes;
    float* bias_s = reinterpret_cast<float*>(smem + L.bias_off) + ew * BN;
    uint64_t* rbar = rfull + ew * nb;
    uint32_t rphase = 0;  // bit b: parity of ring buffer b's residual barrier
    uint32_t seq = 0;     // chunks this warp has staged so far (ring position)
    int tr_n = 0;
    const bool has_res = p.res != nullptr && p.out_mode == kOutBF16;
    const __nv_bfloat162 zero2 = __floats2bfloat162_rn(0.f, 0.f);
    int cached_n = -1;
    // alternate-tile groups walk every other tile of the CTA directly
    const int j0 = alt_tiles ? half : 0;
    const int jstep = alt_tiles ? 2 : 1;
    int j = j0;
    TileWalk tw;
    tw.init(t_first + j0 * t_step, jstep * t_step, nt, mtp);
    for (int t = t_first + j0 * t_step; t < total; t += jstep * t_step, j += jstep, tw.next()) {
      const int tile_n = tw.tn;
      const int tile_m = p.mcast ? 2 * tw.pm + static_cast<int>(crank) : tw.pm;
      const int z = tw.z;
      const int acc = j % kNAcc;
      const int m = tile_m * kBlockM + row;
      bool row_ok = m < p.M;
      size_t orow = static_cast<size_t>(m);
      if (TS > 1 || stem_direct) {
        // padded grid position -> output pixel (tap-shift: Ho x (Wo + kw - 1) per image, the
        // kw-1 junk columns dropped; stems: Mi positions per image, rows of Wg)
        const int img = fdiv(m, p.fd_img);
        const int local = m - img * static_cast<int>(p.fd_img.d);
        const int oh = fdiv(local, p.fd_row);
        const int ow = local - oh * static_cast<int>(p.fd_row.d);
        row_ok = row_ok && oh < p.Ho && ow < p.Wo;
        orow = (static_cast<size_t>(img) * p.Ho + oh) * p.Wo + ow;
      }
      const int n_tile0 = tile_n * BN;
      const int m_slab = tile_m * kBlockM + static_cast<int>(quarter) * 32;
      if (p.bias && tile_n != cached_n) {
        __syncwarp();
        for (int i = lane; i < BN; i += 32) bias_s[i] = (n_tile0 + i < p.N) ? __ldg(p.bias + n_tile0 + i) : 0.f;
        __syncwarp();
        cached_n = tile_n;
      }
      if (has_res && lane == 0) {
        // every earlier store has finished reading the ring -> prefetch this tile's
        // residual chunks now, while its MMAs run
        bulk_wait_read<0>();
        uint32_t k = 0;
        for (int ci = c_first; ci < NCH && n_tile0 + ci * CW < p.N; ci += c_step, ++k) {
          const uint32_t b = (seq + k) & (nb - 1);
          mbar_arrive_expect_tx(&rbar[b], S::kStageOutBytes);
          tma_load_2d(ring + b * S::kStageOutBytes, &map_res, &rbar[b], n_tile0 + ci * CW, m_slab);
        }
      }
      if (warp == 2 && lane == 0) trace_ev(p.trace, 2, tr_n, 20);
      mbar_wait(&tfull[acc], (j / kNAcc) & 1);
      if (warp == 2 && lane == 0) trace_ev(p.trace, 2, tr_n, 21);
      tc_fence_after();
      const uint32_t tbase = tmem_base + acc * BN + ((quarter * 32) << 16);
      // The accumulator is released as soon as this warp's last TMEM load of the tile
      // has completed -- before its math and stores -- so the MMAs of tile j+2 overlap
      // the epilogue of tile j.
      bool released = false;
      auto release = [&] {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (PAIR && crank != 0)  // the leader's MMAs write our TMEM: release it there
            mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));
          else
            mbar_arrive(&tempty[acc]);
        }
        released = true;
      };
      int last_ci = c_first;
      while (last_ci + c_step < NCH && n_tile0 + (last_ci + c_step) * CW < p.N) last_ci += c_step;
#pragma unroll 1
      for (int ci = c_first; ci < NCH; ci += c_step) {
        const int c = ci * CW;
        const int n = n_tile0 + c;
        if (n >= p.N) break;  // warp-uniform
        const bool full_chunk = n + CW <= p.N;
        uint32_t r[CW];
#pragma unroll
        for (int q = 0; q < CW; q += 32) tmem_ld32(tbase + c + q, r + q);
        tmem_ld_wait();
        if (warp == 2 && lane == 0) trace_ev(p.trace, 2, tr_n, 23);
        if (ci == last_ci && p.early_release) release();
        if (dbg_probe(p, 6) || dbg_probe(p, 8)) {  // (probe 6/8: TMEM load + release only)
          ++seq;
          continue;
        }
        if (p.out_mode != kOutBF16) {
          // fp32 logits or a split-K partial slice: direct stores (small outputs)
          if (row_ok) {
            float* o;
            const bool logits = p.out_mode == kOutF32;
            if (!logits)
              o = reinterpret_cast<float*>(p.out) + (static_cast<size_t>(z) * p.M + m) * p.ldo + n;
            else
              o = reinterpret_cast<float*>(p.out) + static_cast<size_t>(m) * p.ldo + p.out_off + n;
            float v[CW];
#pragma unroll
            for (int i = 0; i < CW; ++i) {
              float x = __uint_as_float(r[i]);
              if (logits && p.bias) x += bias_s[c + i];
              if (logits && p.relu) x = fmaxf(x, 0.f);
              v[i] = x;
            }
            if (p.vec_ok && full_chunk) {
#pragma unroll
              for (int i = 0; i < CW; i += 4)
                *reinterpret_cast<float4*>(o + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
            } else {
#pragma unroll
              for (int i = 0; i < CW; ++i)
                if (n + i < p.N) o[i] = v[i];
            }
          }
          continue;
        }
        float2 v2[CW / 2];
#pragma unroll
        for (int i = 0; i < CW / 2; ++i) v2[i] = make_float2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
        if (p.bias && !dbg_probe(p, 4)) {
#pragma unroll
          for (int i = 0; i < CW; i += 4) {
            const float4 b4 = *reinterpret_cast<const float4*>(bias_s + c + i);
            v2[i / 2] = __fadd2_rn(v2[i / 2], make_float2(b4.x, b4.y));
            v2[i / 2 + 1] = __fadd2_rn(v2[i / 2 + 1], make_float2(b4.z, b4.w));
          }
        }
        const uint32_t b = seq & (nb - 1);
        uint8_t* buf = ring + b * S::kStageOutBytes;
        uint8_t* rowp = buf + lane * (CW * 2);
        if (has_res) {
          mbar_wait(&rbar[b], (rphase >> b) & 1u);
          rphase ^= 1u << b;
#pragma unroll
          for (int ch = 0; ch < CW / 8; ++ch) {
            const uint4 q = *reinterpret_cast<const uint4*>(rowp + swz_chunk(ch, lane, CW) * 16);
            const uint32_t qq[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int e = 0; e < 4; ++e)  // bf16 -> fp32 is a 16-bit shift
              v2[ch * 4 + e] = __fadd2_rn(v2[ch * 4 + e], make_float2(__uint_as_float(qq[e] << 16),
                                                                      __uint_as_float(qq[e] & 0xffff0000u)));
          }
        }
        uint32_t pk[CW / 2];
#pragma unroll
        for (int i = 0; i < CW / 2; ++i)
          pk[i] = p.relu ? pack_bf16x2_relu(v2[i].x, v2[i].y) : pack_bf16x2(v2[i].x, v2[i].y);
        if (TS > 1 || (stem_direct && !p.stem_tma)) {
          // tap-shift / stem tiles are not contiguous in the output (padded grids): row
          // stores; a grouped stem launch sends columns >= n_split to the second tensor
          const bool second = p.n_split > 0 && n >= p.n_split;
          __nv_bfloat16* const col0 =
              second ? reinterpret_cast<__nv_bfloat16*>(p.out2) + p.out2_off + (n - p.n_split)
                     : reinterpret_cast<__nv_bfloat16*>(p.out) + p.out_off + n;
          const int ldd = second ? p.ldo2 : p.ldo;
          __nv_bfloat16* o = col0 + orow * ldd;
          if (warp == 2 && lane == 0) trace_ev(p.trace, 2, tr_n, 24);
          if (dbg_probe(p, 1)) continue;  // (trace build: no stores)
          if (full_chunk && p.vec_ok && CW % 32 == 0) {
            uint8_t* stg = smem + L.out_off + ew * S::kRowStageBytes;
#pragma unroll
            for (int h = 0; h < CW / 32; ++h)
              stage_store_rows32(stg, pk + 16 * h, lane, col0 + 32 * h, ldd,
                                 row_ok ? static_cast<int>(orow) : -1);
          } else if (row_ok) {
            {
              const __nv_bfloat16* hv = reinterpret_cast<const __nv_bfloat16*>(pk);
#pragma unroll
              for (int i = 0; i < CW; ++i)
                if (n + i < p.N) o[i] = hv[i];
            }
          }
          continue;
        }
        if (warp == 2 && lane == 0) trace_ev(p.trace, 2, tr_n, 25);
        if (!has_res) {
          // the store that last used this ring buffer (nb chunks ago) has read it
          if (lane == 0) {
            if (nb == 1)
              bulk_wait_read<0>();
            else if (nb == 2)
              bulk_wait_read<1>();
            else
              bulk_wait_read<3>();
          }
          __syncwarp();
        }
        // (with a residual each lane rewrites the row it just read, in place)
#pragma unroll
        for (int ch = 0; ch < CW / 8; ++ch)
          *reinterpret_cast<uint4*>(rowp + swz_chunk(ch, lane, CW) * 16) =
              make_uint4(pk[ch * 4], pk[ch * 4 + 1], pk[ch * 4 + 2], pk[ch * 4 + 3]);
        if (warp == 2 && lane == 0) trace_ev(p.trace, 2, tr_n, 26);
        fence_proxy_async_smem();
        __syncwarp();
        if (warp == 2 && lane == 0) trace_ev(p.trace, 2, tr_n, 27);
        if (lane == 0 && !dbg_probe(p, 5)) {  // (probe 5: no output stores, timing only)
          // a grouped launch (members sharing a stem) writes its second column range
          // to another tensor through the residual map slot
          if (stem_direct) {
            // the warp's 32 grid positions lie in one output row: a 3-D (C, Wo, B*Ho) store
            // clipped at Wo drops the junk columns; slabs wholly past Wo / Ho are skipped
            const int img = fdiv(m_slab, p.fd_img);
            const int local = m_slab - img * static_cast<int>(p.fd_img.d);
            const int oh = fdiv(local, p.fd_row);
            const int ow0 = local - oh * static_cast<int>(p.fd_row.d);
            if (m_slab < p.M && oh < p.Ho) {
              if (ow0 < p.Wo) tma_store_3d(&map_out, buf, n, ow0, img * p.Ho + oh);
              const int k = static_cast<int>(p.fd_row.d) - ow0;  // rows left in this grid row
              if (k < 32 && oh + 1 < p.Ho) {
                // the slab's tail starts the next output row: 8-row boxes (map_res slot)
                for (int r8 = k; r8 < 32; r8 += 8)
                  tma_store_3d(&map_res, buf + r8 * (CW * 2), n, r8 - k, img * p.Ho + oh + 1);
              }
            }
          } else if (p.n_split > 0 && n >= p.n_split) {
            tma_store_2d(&map_res, buf, n - p.n_split, m_slab);
          } else {
            tma_store_2d(&map_out, buf, n, m_slab);
          }
          bulk_commit();
        }
        ++seq;
      }
      if (!released) release();  // (no chunk of this tile fell inside N)
      if (warp == 2 && lane == 0) trace_ev(p.trace, 2, tr_n, 22);
    }
    if (lane == 0) bulk_wait<0>();
  } else if (p.a_mode == kAModeGatherC8 && warp < 10) {
    // ------------------------------------------------------------ A gather (stem)
    // Thread r builds A row r: for filter row kb, the 8 consecutive input pixels
    // starting at the receptive field's left edge are 8 x 16 B = one 128-byte
    // swizzled smem row (pixels beyond kw meet zero weights; outside the image
    // they are zero-filled).  Completion is signalled asynchronously with
    // cp.async.mbarrier.arrive, so each thread streams as many stages as the ring
    // has free slots.
    const int r = static_cast<int>(threadIdx.x) - 192;  // 0..127
    int stage = 0;
    uint32_t phase = 0;
    TileWalk tw;
    tw.init(t_first, t_step, nt, mtp);
    for (int t = t_first; t < total; t += t_step, tw.next()) {
      const int tile_m = p.mcast ? 2 * tw.pm + static_cast<int>(crank) : tw.pm;
      const int z = tw.z;
      const int kb0 = z * p.kb_per_split;
      const int kb1 = min(kb0 + p.kb_per_split, p.num_kb);
      const int m = tile_m * kBlockM + r;
      const bool row_ok = m < p.M;
      const int hw = p.Ho * p.Wo;
      const int img = row_ok ? m / hw : 0;
      const int rem = m - img * hw;
      const int oh = rem / p.Wo;
      const int ow = rem - oh * p.Wo;
      const int iw0 = ow * p.sw - p.pw;
      // per tile: the 8 pixel columns of this row (K group j <- tap; stride-2 stem weights
      // list the even taps first, then the odd) and which of them lie inside the image
      uint32_t wmask = 0;
      int coff[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int tap = p.sw == 2 ? (j < 4 ? 2 * j : 2 * (j - 4) + 1) : j;
        const int iw = iw0 + tap;
        const bool ok = iw >= 0 && iw < p.W;
        wmask |= (ok ? 1u : 0u) << j;
        coff[j] = (ok ? iw : 0) * 8;
      }
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* rowp = ring_base + stage * L.stage_bytes + r * 128;
        const int ih = oh * p.sh - p.ph + kb;
        const bool hok = row_ok && ih >= 0 && ih < p.H;
        const __nv_bfloat16* src = p.x + ((static_cast<int64_t>(img) * p.H + (hok ? ih : 0)) * p.W) * 8;
        const uint32_t m8 = hok ? wmask : 0u;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          cp_async_16(rowp + ((j ^ (r & 7)) * 16), src + coff[j], ((m8 >> j) & 1u) ? 16u : 0u);
        cp_async_arrive_noinc(&xfull[stage]);
        if (++stage == L.stages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    cp_async_wait<0>();
  } else if (p.pre_scale) {
    // ------------------------------------------------------------ A transform
    // relu(a * scale[k] + shift[k]) in place on the swizzled A tile, then a proxy
    // fence so the tensor core sees the result.  Thread t owns logical 16-byte chunk
    // j = t % 8 (8 channels) of rows t/8, t/8 + 24, ...: its scale/shift are read once
    // per stage (from an smem copy of the whole vector), and each warp's accesses
    // cover whole 128-byte rows (conflict-free).
    if constexpr (S::kPreMax > 0) {
      const int t = static_cast<int>(threadIdx.x) - (kThreads - kXformThreads);  // 0 .. kXformThreads-1
      const int j = t & 7;
      constexpr int kRowStep = kXformThreads / 8;         // rows apart
      // scale/shift rounded to bf16 once (the math is bf16x2 FMA anyway)
      __nv_bfloat16* sc_s = reinterpret_cast<__nv_bfloat16*>(smem + L.pre_off);
      __nv_bfloat16* sh_s = sc_s + S::kPreMax;
      const int kpad = p.num_kb * kBlockK;
      for (int i = t; i < kpad; i += kXformThreads) {
        sc_s[i] = __float2bfloat16_rn(__ldg(p.pre_scale + i));
        sh_s[i] = __float2bfloat16_rn(__ldg(p.pre_shift + i));
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kXformThreads) : "memory");  // transform warps only
      int stage = 0;
      uint32_t phase = 0;
      TileWalk tw;
      tw.init(t_first, t_step, nt, mtp);
      for (int tt = t_first; tt < total; tt += t_step, tw.next()) {
        const int z = tw.z;
        const int kb0 = z * p.kb_per_split;
        const int kb1 = min(kb0 + p.kb_per_split, p.num_kb);
        for (int kb = kb0; kb < kb1; ++kb) {
          const int c0 = kb * kBlockK + j * 8;
          // one HFMA2.RELU per channel pair
          const uint4 sq = *reinterpret_cast<const uint4*>(sc_s + c0);
          const uint4 tq = *reinterpret_cast<const uint4*>(sh_s + c0);
          const __nv_bfloat162* sc2 = reinterpret_cast<const __nv_bfloat162*>(&sq);
          const __nv_bfloat162* sh2 = reinterpret_cast<const __nv_bfloat162*>(&tq);
          mbar_wait(&full[stage], phase);
          uint8_t* tile = ring_base + stage * L.stage_bytes;
          // all of this thread's rows are loaded before any is stored (the loads are
          // then in flight together; interleaved, each store fenced the next load)
          constexpr int kRowsPer = (kBlockM + kRowStep - 1) / kRowStep;
          static_assert(kRowStep % 8 == 0, "rows of one thread must share the 128B swizzle phase");
          const int r0 = t >> 3;  // rows r0 + i * kRowStep share one swizzle phase
          uint8_t* const col = tile + r0 * 128 + ((j ^ (r0 & 7)) * 16);
          uint4 xs[kRowsPer];
#pragma unroll
          for (int i = 0; i < kRowsPer; ++i)
            if (r0 + i * kRowStep < kBlockM) xs[i] = *reinterpret_cast<const uint4*>(col + i * kRowStep * 128);
#pragma unroll
          for (int i = 0; i < kRowsPer; ++i) {
            __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&xs[i]);
#pragma unroll
            for (int e = 0; e < 4; ++e) h[e] = __hfma2_relu(h[e], sc2[e], sh2[e]);
          }
#pragma unroll
          for (int i = 0; i < (dbg_probe(p, 3) ? 0 : kRowsPer); ++i)
            if (r0 + i * kRowStep < kBlockM) *reinterpret_cast<uint4*>(col + i * kRowStep * 128) = xs[i];
          fence_proxy_async_smem();
          __syncwarp();
          if ((t & 31) == 0) mbar_arrive(&xfull[stage]);
          if (++stage == L.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  trace_cta(p.trace, 2);
  if (p.mcast) cluster_sync();  // no CTA leaves while its peer may still write into it
  if (warp == 1) {
    if constexpr (PAIR)
      tmem_dealloc_pair(tmem_base, kTmemCols);
    else
      tmem_dealloc(tmem_base, kTmemCols);
  }
}

// ---------------------------------------------------------------- host side

template <int BN, int TS, bool PAIR, int TAPN = 0, bool STEM = false>
static cudaError_t launch_bn(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mo,
                             const CUtensorMap& mr, const ConvParams& p, int grid,
                             cudaStream_t stream) {
  using S = ConvSmem<BN, TS, PAIR, TAPN, STEM>;
  static bool configured = false;  // attribute is per-function; idempotent
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(conv_umma_kernel<BN, TS, PAIR, TAPN, STEM>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, S::kBytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = S::kBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = p.mcast ? 2 : 1;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, conv_umma_kernel<BN, TS, PAIR, TAPN, STEM>, ma, mb, mo, mr, p);
}

int conv_umma_chunk(int block_n) { return block_n < 64 ? block_n : 64; }
int conv_umma_stem_chunk(int block_n) { return block_n < EB_STEM_CW ? block_n : EB_STEM_CW; }

template <int BN, int TS, bool PAIR, int TAPN = 0, bool STEM = false>
static int stages_of(const ConvParams& p) {
  return make_layout<ConvSmem<BN, TS, PAIR, TAPN, STEM>>(p).stages;
}
int conv_umma_stages(const ConvParams& p, int block_n) {
  const bool ts = p.a_mode == kAModeTapShift;
  if (p.a_mode == kAModeStemRows || p.a_mode == kAModeStemPlanes)
    return block_n == 32 ? stages_of<32, 1, false, 0, true>(p)
           : block_n == 64 ? stages_of<64, 1, false, 0, true>(p)
           : block_n == 128 ? stages_of<128, 1, false, 0, true>(p)
                            : stages_of<256, 1, false, 0, true>(p);
  if (p.a_mode == kAModeTapN) {
    if (p.pair) return block_n == 32 ? stages_of<32, 1, true, 1>(p) : stages_of<64, 1, true, 1>(p);
    // TAPN template value: 1 = three planes, 2 = two (tap 2 folded by the MMA), +4 = fused pool
    if (p.tall_rows) return block_n == 32 ? stages_of<32, 1, false, 9>(p) : 0;
    const int tv = (p.tapn2 ? 2 : 1) + (p.pool2 ? 4 : 0);
    switch (tv + (block_n == 32 ? 0 : 8)) {
      case 1: return stages_of<32, 1, false, 1>(p);
      case 2: return stages_of<32, 1, false, 2>(p);
      case 5: return stages_of<32, 1, false, 5>(p);
      case 6: return stages_of<32, 1, false, 6>(p);
      case 9: return stages_of<64, 1, false, 1>(p);
      case 10: return stages_of<64, 1, false, 2>(p);
      case 13: return stages_of<64, 1, false, 5>(p);
      default: return stages_of<64, 1, false, 6>(p);
    }
  }
  if (p.pair) {
    if (ts) return block_n == 64 ? stages_of<64, 3, true>(p) : stages_of<128, 3, true>(p);
    return block_n == 64 ? stages_of<64, 1, true>(p) : block_n == 128 ? stages_of<128, 1, true>(p) : stages_of<256, 1, true>(p);
  }
  if (ts) return block_n == 32 ? stages_of<32, 3, false>(p) : block_n == 64 ? stages_of<64, 3, false>(p) : stages_of<128, 3, false>(p);
  switch (block_n) {
    case 32: return stages_of<32, 1, false>(p);
    case 64: return stages_of<64, 1, false>(p);
    case 128: return stages_of<128, 1, false>(p);
    default: return stages_of<256, 1, false>(p);
  }
}

// Programmatic dependent launch: the next layer's CTAs start their prologue while the
// current one drains.  It shortens small-batch (latency-bound) forwards, but at large
// batch the early CTAs of one member's next layer sit on SMs waiting for their
// predecessor while the other members' lanes could use them (measured on B200, C2
// B = 256: 17.0k img/s with PDL vs 17.4k without; B = 1: 1.24-1.35 ms vs 1.38-1.46 ms).
// So it is on for forwards of at most EB_PDL_MAX_BATCH images (default 32).
thread_local int t_pdl_batch = 0;
void set_pdl_batch(int batch) { t_pdl_batch = batch; }
bool pdl_enabled() {
  static const bool on = [] {
    const char* v = getenv("EB_PDL");
    return !(v && (v[0] == '0' || v[0] == 'n' || v[0] == 'N'));
  }();
  static const int max_b = [] {
    const char* v = getenv("EB_PDL_MAX_BATCH");
    return (v && *v) ? atoi(v) : 32;
  }();
  return on && t_pdl_batch > 0 && t_pdl_batch <= max_b;
}

cudaError_t conv_umma_launch(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mo,
                             const CUtensorMap& mr, const ConvParams& p, int block_n, int grid,
                             cudaStream_t stream) {
  if (p.a_mode == kAModeStemRows || p.a_mode == kAModeStemPlanes) {
    if (p.mcast || p.pair) return cudaErrorInvalidValue;
    switch (block_n) {
      case 32: return launch_bn<32, 1, false, 0, true>(ma, mb, mo, mr, p, grid, stream);
      case 64: return launch_bn<64, 1, false, 0, true>(ma, mb, mo, mr, p, grid, stream);
      case 128: return launch_bn<128, 1, false, 0, true>(ma, mb, mo, mr, p, grid, stream);
      case 256: return launch_bn<256, 1, false, 0, true>(ma, mb, mo, mr, p, grid, stream);
      default: return cudaErrorInvalidValue;
    }
  }
  if (p.a_mode == kAModeTapN) {
    if (p.pair) {
      if (!p.mcast || !p.resb) return cudaErrorInvalidValue;
      switch (block_n) {
        case 32: return launch_bn<32, 1, true, 1>(ma, mb, mo, mr, p, grid, stream);
        case 64: return launch_bn<64, 1, true, 1>(ma, mb, mo, mr, p, grid, stream);
        default: return cudaErrorInvalidValue;
      }
    }
    if (p.mcast) return cudaErrorInvalidValue;
    switch (block_n) {
      case 32:
      case 64: {
        if (p.tall_rows)
          return block_n == 32 ? launch_bn<32, 1, false, 9>(ma, mb, mo, mr, p, grid, stream)
                               : cudaErrorInvalidValue;
        const int tv = (p.tapn2 ? 2 : 1) + (p.pool2 ? 4 : 0);
        switch (tv + (block_n == 32 ? 0 : 8)) {
          case 1: return launch_bn<32, 1, false, 1>(ma, mb, mo, mr, p, grid, stream);
          case 2: return launch_bn<32, 1, false, 2>(ma, mb, mo, mr, p, grid, stream);
          case 5: return launch_bn<32, 1, false, 5>(ma, mb, mo, mr, p, grid, stream);
          case 6: return launch_bn<32, 1, false, 6>(ma, mb, mo, mr, p, grid, stream);
          case 9: return launch_bn<64, 1, false, 1>(ma, mb, mo, mr, p, grid, stream);
          case 10: return launch_bn<64, 1, false, 2>(ma, mb, mo, mr, p, grid, stream);
          case 13: return launch_bn<64, 1, false, 5>(ma, mb, mo, mr, p, grid, stream);
          default: return launch_bn<64, 1, false, 6>(ma, mb, mo, mr, p, grid, stream);
        }
      }
      default: return cudaErrorInvalidValue;
    }
  }
  if (p.pair) {
    if (!p.mcast) return cudaErrorInvalidValue;
    if (p.a_mode == kAModeTapShift) {
      switch (block_n) {
        case 64: return launch_bn<64, 3, true>(ma, mb, mo, mr, p, grid, stream);
        case 128: return launch_bn<128, 3, true>(ma, mb, mo, mr, p, grid, stream);
        default: return cudaErrorInvalidValue;
      }
    }
    switch (block_n) {
      case 64: return launch_bn<64, 1, true>(ma, mb, mo, mr, p, grid, stream);
      case 128: return launch_bn<128, 1, true>(ma, mb, mo, mr, p, grid, stream);
      case 256: return launch_bn<256, 1, true>(ma, mb, mo, mr, p, grid, stream);
      default: return cudaErrorInvalidValue;
    }
  }
  if (p.a_mode == kAModeTapShift) {
    switch (block_n) {
      case 32: return launch_bn<32, 3, false>(ma, mb, mo, mr, p, grid, stream);
      case 64: return launch_bn<64, 3, false>(ma, mb, mo, mr, p, grid, stream);
      case 128: return launch_bn<128, 3, false>(ma, mb, mo, mr, p, grid, stream);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (block_n) {
    case 32: return launch_bn<32, 1, false>(ma, mb, mo, mr, p, grid, stream);
    case 64: return launch_bn<64, 1, false>(ma, mb, mo, mr, p, grid, stream);
    case 128: return launch_bn<128, 1, false>(ma, mb, mo, mr, p, grid, stream);
    case 256: return launch_bn<256, 1, false>(ma, mb, mo, mr, p, grid, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace eb
