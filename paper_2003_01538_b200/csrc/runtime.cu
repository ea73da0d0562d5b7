// runtime.cu -- the native engine behind include/ensemble_b200.h.
//
// An engine owns, for one GPU: the weight pool (one allocation for every
// member), the activation arena (one buffer per plan tensor, max_batch deep),
// the op list of every member, and a cache of instantiated CUDA graphs keyed by
// (batch size, input encoding).  eb_forward = H2D input copy -> graph replay
// (K1 preprocess, every member's layers on its own concurrency lane) -> K5
// combine -> D2H copy of labels / top-k / policy output.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/ensemble_b200.h"
#include "eb_internal.h"
#include "eb_kernels.h"

namespace eb {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

}  // namespace eb

using namespace eb;

#define EB_CUDA(call)                                                                  \
  do {                                                                                 \
    cudaError_t _e = (call);                                                           \
    if (_e != cudaSuccess) {                                                           \
      set_error(std::string(#call) + ": " + cudaGetErrorString(_e));                   \
      return EB_E_CUDA;                                                                \
    }                                                                                  \
  } while (0)

#define EB_FAIL(code, msg)   \
  do {                       \
    set_error(msg);          \
    return (code);           \
  } while (0)

namespace {

constexpr int kLanes = 4;
// split-K partial slices: splits * tiles <= 2 * 148 by construction (plan_conv)
constexpr size_t kSplitWsFloats = static_cast<size_t>(2 * 148) * 128 * 256;
constexpr int kMaxGraphs = 256;

struct Tensor {
  int h, w, c, dtype;
  void* dev = nullptr;
};

struct Member {
  int kind, tensor, koff, k;
};

size_t dsize(int dtype) { return dtype == EB_BF16 ? 2 : (dtype == EB_F32 ? 4 : 8); }

// ------------------------------------------------------------------ conv planning

struct ConvArgs {
  const void* x;  // first channel of the slice
  int B, H, W, ldx, cin;
  const void* w;
  const float* bias;
  const void* res;
  int ldr;
  void* y;
  int ldy, y_off, cout;
  int kh, kw, sh, sw, ph, pw;
  int relu, out_f32, c8_stem, flatten;
  void* y2 = nullptr;  // grouped launch: columns >= n_split are written here
  int ldy2 = 0, y2_off = 0, n_split = 0;
  int split_k;  // 0 = auto
  int block_n;  // 0 = auto
  int groups = 1;                    // grouped conv (block-diagonal weights per N tile)
  const float* pre_scale = nullptr;  // pre-activation on A (tiled mode only)
  const float* pre_shift = nullptr;
  int pool2 = 0;  // fused 2x2/2 max-pool: y is the pooled (Ho/2 x Wo/2) tensor
  int max_ctas = 0;  // persistent grid cap (0 = every SM): the SM share of the op's lane
};

// EB_LANE_SMS=a,b,c,d: the persistent conv grids of lane l use at most that many SMs, so
// members on different lanes run side by side on disjoint SM sets (one CTA per SM) instead
// of each grid taking the whole GPU in turn.  Unset / 0: every lane uses every SM.
int lane_sms(int lane) {
  static int v[4] = {-1, -1, -1, -1};
  if (v[0] < 0) {
    for (int& x : v) x = 0;
    if (const char* e = getenv("EB_LANE_SMS")) {
      int i = 0;
      for (const char* q = e; *q && i < 4; ++i) {
        v[i] = atoi(q);
        while (*q && *q != ',') ++q;
        if (*q == ',') ++q;
      }
    }
  }
  return (lane >= 0 && lane < 4) ? v[lane] : 0;
}

int conv_out(int in, int k, int s, int p) { return (in + 2 * p - k) / s + 1; }

int pick_block_n(int cout) {
  if (cout <= 32) return 32;
  if (cout <= 64) return 64;
  if (cout <= 128) return 128;
  return (cout % 256 == 0) ? 256 : 128;
}

// K extent (elements) of the packed weight rows for a conv of this geometry.
int64_t packed_k(int cin, int kh, int kw, bool c8, bool flatten, int H, int W) {
  if (flatten) return ((static_cast<int64_t>(H) * W * cin + 63) / 64) * 64;
  if (c8) return static_cast<int64_t>(kh) * 64;  // one K block (8 px x 8 ch) per filter row
  return static_cast<int64_t>(kh) * kw * ((cin + 63) / 64) * 64;
}

bool env_flag(const char* name, bool dflt) {
  const char* v = getenv(name);
  if (!v || !*v) return dflt;
  return !(v[0] == '0' || v[0] == 'n' || v[0] == 'N' || v[0] == 'f' || v[0] == 'F');
}
bool mcast_enabled() {
  static const bool on = env_flag("EB_MCAST", true);
  return on;
}
bool pair_enabled() {
  static const bool on = env_flag("EB_PAIR", true);
  return on;
}
int pair_min_kb_ts() {
  static const int v = [] {
    const char* e = getenv("EB_PAIR_TS_KB");
    return (e && *e) ? atoi(e) : 4;
  }();
  return v;
}
int tapn_max_cout() {
  static const int v = [] {
    const char* e = getenv("EB_TAPN_MAX_COUT");
    return (e && *e) ? atoi(e) : 64;
  }();
  return v;
}
bool pair_tapn_enabled() {
  // correct but slower (B200, B = 256): 224x224 64->64 1600 vs 1120 us, 56x56 107 vs 65 us,
  // growth conv 76.4 vs 77.1 us -- the pair's lock-step per one-stage tile costs more than
  // the halved B reads save.  Opt-in.
  static const bool on = env_flag("EB_PAIR_TAPN", false);
  return on;
}
bool resb_enabled() {
  static const bool on = env_flag("EB_RESB", true);
  return on;
}
bool tall_enabled() {
  return env_flag("EB_TAPN_TALL", true);  // (read per plan: tests pin the mode of a reference conv)
}
bool tapn_enabled() {
  static const bool on = env_flag("EB_TAPN", true);
  return on;
}
bool stem_rows_per_stage_all() {
  static const bool on = env_flag("EB_STEM_KBS", true);
  return on;
}
bool stem_tma_store_enabled() {
  static const bool on = env_flag("EB_STEM_TMA_STORE", true);
  return on;
}
bool stem_rows_enabled() {
  // measured on B200 (B = 256): VGG stem 556 us (+ K1 writes the layout) vs 843 us gathered;
  // grouped 7x7/2 stem 361 us vs 470 us; C2 step 14.8-14.9 vs 15.1 ms
  static const bool on = env_flag("EB_STEM_ROWS", true);
  return on;
}
bool stem_tma_enabled() {
  // measured on B200: the cp.async gather is as fast for the 3x3/s1 stem and 1.6x faster
  // for the 7x7/s2 one (16-byte im2col elements are TMA-request bound)
  static const bool on = env_flag("EB_STEM_TMA", false);
  return on;
}
bool tap_shift_enabled() {
  static const bool on = env_flag("EB_TAPSHIFT", true);
  return on;
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
  }
  return n;
}

struct ConvPlan {
  CUtensorMap ma, mb, mo, mr;
  ConvParams p;
  int grid;
  int block_n;
  int splits;
  size_t ws_floats;
};

int plan_conv(const ConvArgs& a, ConvPlan* out) {
  const bool tiled = a.groups == 1 &&
                     (a.flatten || (a.kh == 1 && a.kw == 1 && a.sh == 1 && a.sw == 1 &&
                                    a.ph == 0 && a.pw == 0 && !a.c8_stem));
  const int Ho = a.flatten ? 1 : conv_out(a.H, a.kh, a.sh, a.ph);
  const int Wo = a.flatten ? 1 : conv_out(a.W, a.kw, a.sw, a.pw);
  if (Ho <= 0 || Wo <= 0) EB_FAIL(EB_E_SHAPE, "conv output would be empty");
  // grouped convs (block-diagonal N tiles): 64-wide tiles whenever a group fits -- a
  // tile's K window is its own channel block, so the zero off-diagonal blocks shrink with
  // the tile (B200, ResNeXt-50 at B = 128: 3x3 grouped 94.7 -> 80.3 us at 56x56, 24.1 ->
  // 18.7 us at 7x7 against 128-wide tiles; 32-wide tiles are slower again)
  const int bn_guess = a.block_n ? a.block_n
                                 : (a.groups > 1 ? (a.cout / a.groups <= 64 ? std::min(64, pick_block_n(a.cout))
                                                                            : std::min(128, pick_block_n(a.cout)))
                                                 : pick_block_n(a.cout));
  if (a.groups > 1) {
    // block-diagonal grouped conv: an N tile of BN outputs reads the BN input channels of
    // its own groups, so groups must not straddle tiles and Cin == Cout
    const int cpg = a.cout / a.groups;
    if (a.cin != a.cout || a.cout % a.groups != 0 || bn_guess % cpg != 0 || bn_guess > 128 ||
        a.c8_stem || a.flatten || a.res)
      EB_FAIL(EB_E_INVALID, "unsupported grouped convolution geometry");
  }
  // (pw 0 or 1: the padded grid is Wo + 2 columns wide either way -- W + 2 or W; the
  // im2col map's traversal box covers it, unpadded Inception convs included)
  const bool tap_shift = !tiled && !a.c8_stem && !a.flatten && a.kw == 3 && (a.pw == 1 || a.pw == 0) &&
                         a.sh == 1 && a.sw == 1 && !a.res && !a.out_f32 && bn_guess <= 128 &&
                         tap_shift_enabled();
  // taps-in-N: small Cout (the MMA would otherwise re-read A from smem per 32 columns).
  // Measured on B200 (B=256): 3x3 128->32 at 56x56 152 -> 105 us, at 28x28 45 -> 32 us;
  // 3x3 64->64 at 56x56 92 -> 83 us.
  const bool tapn = tap_shift && a.cout <= std::min(64, tapn_max_cout()) && a.groups == 1 && !a.pre_scale && a.n_split == 0 &&
                    tapn_enabled();
  // tall taps-in-N: one A load per channel chunk covers all kh filter rows (filter row r
  // reads the same buffer r * Wp rows on), over a grid padded to Ho + kh - 1 rows per image
  // so that the shifted rows stay inside their image; 126-row tiles, neighbouring quarters
  // exchange their boundary rows in the epilogue.  For 32-column layers with more than one
  // channel chunk (DenseNet growth convs) whose tall load fits one 256-row TMA box.
  const int tall_wp = Wo + a.kw - 1;
  const int tall_rows = (128 + (a.kh - 1) * tall_wp + 7) / 8 * 8;
  // (not when its 2 extra grid rows per image cost more than ~12 % more tiles than the
  // plain taps-in-N walk: 7x7 images, 135 -> 165 tiles at B = 256.  Decided from the
  // per-image geometry only -- never from B -- because the two modes accumulate the
  // K blocks in different orders and a sample's logits must not depend on its batch,
  // SPEC.md:166,174)
  const bool tall_pays = static_cast<int64_t>(Ho + a.kh - 1) * 120 * 100 <= static_cast<int64_t>(Ho) * 126 * 112;
  // (and only while its resident weights -- kh x chunks x 12 KB -- leave room for two
  // one-chunk stages: Cin <= 192)
  const int64_t tall_smem = 3ll * ((a.cin + 63) / 64) * (3 * 32 * 128) + 2ll * tall_rows * 128 + 24 * 1024;
  const bool tall = tapn && bn_guess == 32 && a.cin > 64 && !a.pool2 && a.kh == 3 && tall_rows <= 256 &&
                    tall_smem <= 220 * 1024 && tall_pays && tall_enabled();
  // stem rows / planes: x is the padded layout of an 8-channel image (k_stem_relayout)
  const bool stem_direct = a.c8_stem == 2;
  StemGeom sg{};
  if (stem_direct && !stem_geom(a.B, a.H, a.W, a.kh, a.kw, a.sh, a.sw, a.ph, a.pw, &sg))
    EB_FAIL(EB_E_INVALID, "unsupported stem layout geometry");
  const int64_t M64 = stem_direct ? static_cast<int64_t>(a.B) * sg.Mi
                    : tall     ? static_cast<int64_t>(a.B) * (Ho + a.kh - 1) * tall_wp
                               : static_cast<int64_t>(a.B) * Ho * (tap_shift ? Wo + a.kw - 1 : Wo);
  if (M64 > (1ll << 31) - 1) EB_FAIL(EB_E_INVALID, "conv M too large");
  const int M = static_cast<int>(M64);
  const int64_t kpad =
      a.groups > 1 ? static_cast<int64_t>(a.kh) * a.kw * ((bn_guess + 63) / 64 * 64)
                   : packed_k(a.cin, a.kh, a.kw, a.c8_stem, a.flatten, a.H, a.W);
  std::string err;
  ConvPlan& pl = *out;
  memset(&pl.p, 0, sizeof(pl.p));
  if (a.flatten) {
    const int64_t feat = static_cast<int64_t>(a.H) * a.W * a.cin;
    if (a.ldx != a.cin) EB_FAIL(EB_E_INVALID, "flatten needs a dense source tensor");
    if (!encode_tiled_2d_bf16(&pl.ma, a.x, feat, a.B, feat, 64, 128, &err))
      EB_FAIL(EB_E_INVALID, err);
    pl.p.a_mode = kAModeTiled;
  } else if (tiled) {
    if (!encode_tiled_2d_bf16(&pl.ma, a.x, a.cin, M64, a.ldx, 64, 128, &err))
      EB_FAIL(EB_E_INVALID, err);
    pl.p.a_mode = kAModeTiled;
  } else if (a.c8_stem) {
    if (a.cin != 8 || a.ldx != 8) EB_FAIL(EB_E_INVALID, "stem mode expects an 8-channel image");
    if (a.kw > 8) EB_FAIL(EB_E_INVALID, "stem mode needs kw <= 8");
    pl.p.x = static_cast<const __nv_bfloat16*>(a.x);
    pl.p.H = a.H;
    pl.p.W = a.W;
    if (stem_direct) {
      // the layout as rows of 128 bytes (8 pixels x 8 channels); a load = 17 such lines
      if (!encode_tiled_2d_bf16(&pl.ma, a.x, 64, static_cast<uint64_t>(sg.bytes / 128), 64, 64, 17,
                                &err, 0))
        EB_FAIL(EB_E_INVALID, err);
      pl.p.a_mode = sg.mode;
      pl.p.kbs = 1;  // (raised below to the whole filter when the smem ring stays deep)
      pl.p.Wg = sg.Wg;
      pl.p.Mi = sg.Mi;
      pl.p.Hq = sg.Hq;
      pl.p.Wq = sg.Wq;
      pl.p.plane_px = sg.plane_px;
    } else if (stem_tma_enabled()) {
      // per filter row: one TMA im2col load per horizontal tap, 128 pixels x 8 channels
      if (!encode_im2col_bf16(&pl.ma, a.x, a.B, a.H, a.W, 8, 8, a.kh, a.kw, a.sh, a.sw, a.ph,
                              a.pw, 8, 128, false, &err))
        EB_FAIL(EB_E_INVALID, err);
      pl.p.a_mode = kAModeTapC8;
    } else {
      pl.ma = {};
      pl.p.a_mode = kAModeGatherC8;
    }
  } else if (tap_shift) {
    // one 136-pixel load per (filter row, channel chunk) serves taps s = 0..2 by row shift
    // (taps-in-N: four 32-pixel loads); tiles walk the padded grid (Wo + 2 columns per
    // row, the 2 extra are dropped)
    if (!encode_im2col_bf16(&pl.ma, a.x, a.B, a.H, a.W, a.cin, a.ldx, a.kh, a.kw, a.sh, a.sw, a.ph,
                            a.pw, 64, tall ? tall_rows : tapn ? 32 : 136, true, &err, a.kw - 1,
                            tall ? a.kh - 1 : 0))
      EB_FAIL(EB_E_INVALID, err);
    pl.p.a_mode = tapn ? kAModeTapN : kAModeTapShift;
    pl.p.Wp = Wo + a.kw - 1;
  } else {
    if (!encode_im2col_bf16(&pl.ma, a.x, a.B, a.H, a.W, a.cin, a.ldx, a.kh, a.kw, a.sh, a.sw, a.ph,
                            a.pw, 64, 128, true, &err))
      EB_FAIL(EB_E_INVALID, err);
    pl.p.a_mode = kAModeIm2col;
  }
  const int bn = bn_guess;
  if (!encode_tiled_2d_bf16(&pl.mb, a.w, kpad, a.cout, kpad, 64, bn, &err))
    EB_FAIL(EB_E_INVALID, err);
  // tap-shift stages cover all kw taps of one filter row; a grouped tile sees BN channels
  const int cin_tile = a.groups > 1 ? bn : a.cin;
  const int num_kb = tall ? (cin_tile + 63) / 64
                   : tap_shift ? a.kh * ((cin_tile + 63) / 64) : static_cast<int>(kpad / 64);
  const int mt = tall ? (M + 125) / 126
                 : (tapn && a.pool2) ? a.B * (Ho / 2) * ((Wo + 59) / 60)
                                   : tapn ? (M + 119) / 120 : (M + 127) / 128;
  const int nt = (a.cout + bn - 1) / bn;
  int splits = a.split_k;
  if (splits <= 0) {
    // Split K only when one image's tile grid leaves most SMs idle AND each split keeps a
    // long K loop: the partial slices cost an extra pass and a second launch.  The count
    // is a function of the layer shape alone (one image's rows, N, K), never of B: split
    // and unsplit sum K in different orders, and a sample's logits must be bitwise the
    // same whatever batch it arrives in (eg/models.py:273-274).  Only
    // FC layers (one row per image) qualify by default: their partials stay small at any
    // batch.  EB_SPLIT_MAX_ROWS=64 also splits the 7x7 convs (ResNet-50 layer4): B = 1
    // latency 1.22-1.24 -> 1.13-1.15 ms, but the fp32 partials of those layers cost the
    // B = 256 step 3 % (13.74-13.83 -> 14.17-14.33 ms; interleaved A/B on one B200).
    splits = 1;
    static const int max_rows = getenv("EB_SPLIT_MAX_ROWS") ? atoi(getenv("EB_SPLIT_MAX_ROWS")) : 1;
    const int64_t rows_img = a.flatten ? 1 : static_cast<int64_t>(Ho) * Wo;
    const int64_t tiles1 = ((rows_img + 127) / 128) * nt;
    static const int cap = getenv("EB_SPLIT_CAP") ? atoi(getenv("EB_SPLIT_CAP")) : 32;
    if (!a.res && !tap_shift && rows_img <= max_rows && tiles1 * 4 <= 148 && num_kb >= 32) {
      splits = static_cast<int>(std::min<int64_t>(148 / tiles1, num_kb / 16));
      // (conv layers -- several rows per image -- at most EB_SPLIT_CAP slices)
      splits = std::max(1, std::min(splits, rows_img > 1 ? cap : 32));
    }
  }
  if (splits > num_kb) splits = num_kb;
  const int kb_per = (num_kb + splits - 1) / splits;
  splits = (num_kb + kb_per - 1) / kb_per;
  if (splits > 1 && a.res) EB_FAIL(EB_E_INVALID, "split-K with a residual is not supported");
  pl.p.M = M;
  pl.p.N = a.cout;
  pl.p.num_kb = num_kb;
  pl.p.kb_per_split = kb_per;
  pl.p.Ho = Ho;
  pl.p.Wo = Wo;
  pl.p.sh = a.sh;
  pl.p.sw = a.sw;
  pl.p.ph = a.ph;
  pl.p.pw = a.pw;
  pl.p.kw = a.kw;
  pl.p.taps = a.kh * a.kw;
  pl.p.cchunks = (cin_tile + 63) / 64;
  pl.p.grouped = a.groups > 1 ? 1 : 0;
  pl.p.res = static_cast<const __nv_bfloat16*>(a.res);
  pl.p.ldr = a.ldr;
  pl.p.bias = a.bias;
  pl.p.relu = a.relu;
  pl.p.out = a.y;
  pl.p.ldo = a.ldy;
  pl.p.out_off = a.y_off;
  pl.p.out_mode = a.out_f32 ? kOutF32 : kOutBF16;
  pl.p.pre_scale = a.pre_scale;
  pl.p.pre_shift = a.pre_shift;

  if (a.pre_scale && (pl.p.a_mode != kAModeTiled || !a.pre_shift))
    EB_FAIL(EB_E_INVALID, "pre-activation is only supported on 1x1 (tiled) convolutions");
  if (a.pre_scale && (bn != 128 || num_kb * 64 > 2048))
    EB_FAIL(EB_E_INVALID, "pre-activation needs cout in (64, 128] and Cin <= 2048");
  {
    const int q = a.out_f32 ? 4 : 8;  // elements per 16 bytes
    pl.p.vec_ok = (a.ldy % q == 0) && (a.y_off % q == 0) && (!a.res || a.ldr % 8 == 0);
  }
  pl.block_n = bn;
  pl.splits = splits;
  pl.ws_floats = splits > 1 ? static_cast<size_t>(splits) * M * a.cout : 0;
  // 2-CTA clusters for MMA-heavy tiles.  Preferred: 2-SM MMAs (cta_group::2), where each
  // SM stages its 128 A rows and half of B and the pair runs M=256 MMAs -- per-SM smem
  // operand traffic per MMA drops from (A + B) to (A + B/2), which is what limits
  // SS-mode MMAs at N >= 128.  Otherwise M-tile pairs share B by TMA multicast.
  const bool plain_a = pl.p.a_mode == kAModeTiled || pl.p.a_mode == kAModeIm2col;
  // (short K loops stay unpaired: the pair's lock-step costs more than it saves when the
  // layer is memory-bound -- measured on B200, 1x1 256->64 at 56x56: 79 us single vs 107 us)
  bool pair = pair_enabled() && splits == 1 && mt >= 2 && !a.pre_scale && !tapn &&
                    (tap_shift ? ((bn == 64 || bn == 128) && num_kb >= pair_min_kb_ts())
                               : (plain_a && bn >= 64 && num_kb >= 8));
  bool mcast = pair || (mcast_enabled() && splits == 1 && bn >= 128 && mt >= 2 &&
                              num_kb >= 8 && !a.pre_scale && plain_a);
  pl.p.mcast = mcast ? 1 : 0;
  pl.p.pair = pair ? 1 : 0;
  if (stem_direct) {
    pl.p.fd_img = make_fastdiv(sg.Mi);
    pl.p.fd_row = make_fastdiv(sg.Wg);
  } else if (tap_shift) {
    pl.p.fd_img = make_fastdiv(static_cast<uint32_t>(tall ? Ho + a.kh - 1 : Ho) * (Wo + a.kw - 1));
    pl.p.fd_row = make_fastdiv(Wo + a.kw - 1);
  }
  static const bool early = env_flag("EB_EARLY_REL", true);
  pl.p.early_release = early ? 1 : 0;
  // tap 2 folded by a shifted A (2 MMAs per K step, one plane less to combine): pays
  // where the epilogue bounds the layer (one 64-channel K block per filter row); with
  // more K blocks the layer is MMA-issue bound and the extra MMAs cost more.
  // EB_TAPN2: 0 off, 1 auto, 2 always
  // (read per plan, not cached: tests pin the plane mode of a reference conv)
  const int tapn2 = getenv("EB_TAPN2") ? atoi(getenv("EB_TAPN2")) : 1;
  // (not with the fused pool, whose epilogue is lighter: three planes measured 999-1021 vs
  // 1048-1111 us on VGG conv1_2 + pool1 -- the second MMA re-reads A from smem)
  pl.p.tapn2 = (tapn && !tall && !pair &&
                (tapn2 == 2 || (tapn2 == 1 && num_kb <= a.kh && !a.pool2))) ? 1 : 0;
  if (a.pool2) {
    // fused max-pool (VGG): taps-in-N tiles re-cut as 2 output rows x 60 columns so that
    // each 2x2 window lies inside one tile
    if (!tapn || Ho % 2 || Wo % 2 || a.cout % 32 || !pl.p.vec_ok || a.res || a.out_f32 ||
        a.n_split || splits != 1 || pair)
      EB_FAIL(EB_E_INVALID, "max-pool fusion needs a taps-in-N conv with even output size");
    pl.p.pool2 = 1;
    pl.p.Ho2 = Ho / 2;
    pl.p.Wo2 = Wo / 2;
    pl.p.nseg = (Wo + 59) / 60;
    const int64_t mt2 = static_cast<int64_t>(a.B) * pl.p.Ho2 * pl.p.nseg;
    if (mt2 * 120 > (1ll << 31) - 1) EB_FAIL(EB_E_INVALID, "conv M too large");
    pl.p.M = static_cast<int>(mt2 * 120);  // (the kernel derives its tile count as M / 120)
  }
  // 64-column taps-in-N: the two epilogue groups take alternate tiles (each warp then has
  // two independent 32-column chunks per tile to overlap) rather than splitting columns:
  // B200, B = 256: 224x224 64->64 (+ fused pool) 1185 -> 1080 us, 56x56 72.6 -> 67.2 us
  // pre-activation 1x1 convs (DenseNet): one epilogue chunk buffer per warp, the other half
  // of the ring to the A/B stages (their ring is short -- B streams with A): 56x56 224->128
  // 109 -> 93 us, 28x28 480->128 54 -> 50 us; plain 1x1 convs without the transform were
  // measured neutral (BN 128) or slower (BN 64: 81 -> 89 us)
  static const bool ring_half = env_flag("EB_RING_HALF", true);
  pl.p.ring_half = (ring_half && a.pre_scale && plain_a && !a.res && !a.out_f32 && a.n_split == 0 &&
                    !pair && !mcast && bn <= 128) ? 1 : 0;
  static const bool tapn_alt = env_flag("EB_TAPN_ALT", true);
  pl.p.tapn_alt = tapn_alt ? 1 : 0;
  static const int dbg = getenv("EB_DBG") ? atoi(getenv("EB_DBG")) : 0;
  pl.p.dbg = dbg;
  if (tall) {
    // tall: the whole tile (every channel chunk) per stage when two such stages fit beside
    // the resident weights, else one chunk per stage
    ConvParams q = pl.p;
    q.tall_rows = tall_rows;
    q.resb = 1;
    q.kbs = num_kb;
    q.num_kb = q.kb_per_split = 1;
    if (conv_umma_stages(q, bn) < 2) {
      q.kbs = 1;
      q.num_kb = q.kb_per_split = num_kb;
    }
    if (conv_umma_stages(q, bn) < 2) EB_FAIL(EB_E_INVALID, "tall taps-in-N does not fit shared memory");
    pl.p = q;
  } else if (tapn) {
    // taps-in-N: several K blocks per stage (one 4-MMA K block at N = 3*Cout is only a few
    // hundred cycles of tensor work, less than a stage's fixed sync cost); kbs divides
    // the kh*cchunks K blocks
    static const int kbs_env = getenv("EB_KBS") ? atoi(getenv("EB_KBS")) : 0;
    // measured on B200 (B = 256): Cout 32, Cin 128 (6 K blocks): kbs 1/2/3 = 101/77/85 us at
    // 56x56; Cout 64, Cin 64 (3 K blocks): kbs 1/3 = 1197/1028 us at 224x224, 71/64 at 56x56
    int want = kbs_env > 0 ? kbs_env : (bn <= 32 ? 2 : 3);
    while (want > 1 && num_kb % want != 0) --want;
    ConvParams q = pl.p;
    q.kbs = want;
    q.num_kb = num_kb / want;
    q.kb_per_split = q.num_kb;
    // 2-SM taps-in-N: the MMA re-reads the stacked 3-tap B for every K step; a CTA pair
    // halves that per SM.  Requires resident B (each CTA keeps its half).
    bool tp = pair_tapn_enabled() && splits == 1 && mt >= 2 && nt == 1 && resb_enabled() &&
              !a.pool2;  // (the fused pool's tile re-cut has no 2-SM form)
    if (tp) {
      q.pair = 1;
      q.mcast = 1;
      q.resb = 1;
      if (conv_umma_stages(q, bn) < 2) tp = false;
    }
    if (tp) {
      pl.p = q;  // resident B decided here (the generic pass below skips cluster modes)
      pair = mcast = true;
    } else if (want > 1) {
      q.pair = q.mcast = 0;
      q.resb = 1;
      if (conv_umma_stages(q, bn) >= 2) {
        q.resb = 0;  // (decided below)
        pl.p = q;
      }
    }
  }
  bool stem_whole = false;
  if (stem_direct && stem_rows_per_stage_all()) {
    // stems: all kh filter rows of a tile in one stage (one wait / one commit per tile);
    // prefer resident weights, accept a 2-deep ring (a stage is a whole tile of MMAs)
    ConvParams q = pl.p;
    q.kbs = a.kh;
    q.num_kb = 1;
    q.kb_per_split = 1;
    q.resb = nt == 1 ? 1 : 0;
    if (conv_umma_stages(q, bn) < 2) q.resb = 0;
    if (conv_umma_stages(q, bn) >= 2) {
      pl.p = q;
      stem_whole = true;
    }
    // tall stem: the whole filter's rows of a plane as ONE load (17 + (kh-1) * Wq/8 lines)
    // instead of kh loads of 17 lines -- fewer TMA operations per tile
    const int lines = 17 + (a.kh - 1) * (sg.Wq >> 3);
    if (stem_whole && lines <= 256 && env_flag("EB_STEM_TALL", true)) {
      ConvParams t = pl.p;
      t.stem_lines = lines;
      CUtensorMap mt;
      if (conv_umma_stages(t, bn) >= 2 &&
          encode_tiled_2d_bf16(&mt, a.x, 64, static_cast<uint64_t>(sg.bytes / 128), 64, 64, lines, &err, 0)) {
        pl.p = t;
        pl.ma = mt;
      }
    }
  }
  // Resident B: with a single N tile every CTA re-streams the same weights per tile; keep
  // them in smem instead when they fit and the A ring stays deep (it gets all the space).
  if (resb_enabled() && nt == 1 && splits == 1 && !mcast && !stem_whole && !tall) {
    const int s_stream = conv_umma_stages(pl.p, bn);
    pl.p.resb = 1;
    const int s_res = conv_umma_stages(pl.p, bn);
    const int64_t rb = static_cast<int64_t>(pl.p.num_kb) * (pl.p.kbs > 1 ? pl.p.kbs : 1) *
                       (tap_shift ? 3 : 1) * bn * 128;
    // (up to 160 KB of weights when at least three A stages stay: VGG conv2_1, 112x112
    // 64->128 tap-shift, 147 KB resident, 464 -> 418 us -- streamed, each tile re-read 48 KB
    // of B per filter row from L2)
    static const int max_kb = getenv("EB_RESB_MAX_KB") ? atoi(getenv("EB_RESB_MAX_KB")) : 160;
    static const int min_st = getenv("EB_RESB_MIN_STAGES") ? atoi(getenv("EB_RESB_MIN_STAGES")) : 3;
    const int min_stages = pl.p.kbs > 1 ? 2 : min_st;  // (multi-block stages are long)
    if (rb > max_kb * 1024 || s_res < min_stages || s_res < s_stream) pl.p.resb = 0;
  }
  if (mcast) {
    if (!encode_tiled_2d_bf16(&pl.mb, a.w, kpad, a.cout, kpad, 64, bn / 2, &err))
      EB_FAIL(EB_E_INVALID, err);
    const int sms = a.max_ctas > 0 ? std::min(a.max_ctas, num_sms()) : num_sms();
    const int64_t pairs = static_cast<int64_t>((mt + 1) / 2) * nt;
    pl.grid = 2 * static_cast<int>(std::min<int64_t>(pairs, std::max(1, sms / 2)));
  } else {
    const int sms = a.max_ctas > 0 ? std::min(a.max_ctas, num_sms()) : num_sms();
    const int64_t total = static_cast<int64_t>(mt) * nt * splits;
    pl.grid = static_cast<int>(std::min<int64_t>(total, sms));
  }
  if (tap_shift && splits != 1) EB_FAIL(EB_E_INVALID, "tap-shift mode does not split K");
  if (a.n_split > 0 && (a.res || a.out_f32 || splits != 1 || tap_shift ||
                        a.n_split % conv_umma_chunk(bn) != 0 || a.n_split >= a.cout))
    EB_FAIL(EB_E_INVALID, "unsupported grouped-launch split");
  pl.p.n_split = a.n_split;
  if (a.n_split > 0) {  // direct-store modes write the second column range themselves
    pl.p.out2 = a.y2;
    pl.p.ldo2 = a.ldy2;
    pl.p.out2_off = a.y2_off;
    if (a.ldy2 % 8 != 0 || a.y2_off % 8 != 0) pl.p.vec_ok = 0;
  }
  if (stem_direct && !a.out_f32 && a.n_split == 0 && pl.p.vec_ok && stem_tma_store_enabled()) {
    // stems: 32-pixel slabs stored through a (C, Wo, B*Ho) map that clips the junk columns
    const int cw = conv_umma_stem_chunk(bn);
    for (int box : {32, 8}) {  // (8-row boxes: a slab's part in the next output row)
      if (!encode_tiled_3d_bf16(box == 32 ? &pl.mo : &pl.mr,
                                static_cast<const __nv_bfloat16*>(a.y) + a.y_off, a.cout, Wo,
                                static_cast<uint64_t>(a.B) * Ho, a.ldy,
                                static_cast<uint64_t>(a.ldy) * Wo, cw, box, 1, &err, cw * 2))
        EB_FAIL(EB_E_INVALID, err);
    }
    pl.p.stem_tma = 1;
  } else if (!a.out_f32 && splits == 1 && !tap_shift && !stem_direct) {
    const int cw = conv_umma_chunk(bn);
    const int n1 = a.n_split > 0 ? a.n_split : a.cout;
    if (!encode_tiled_2d_bf16(&pl.mo, static_cast<const __nv_bfloat16*>(a.y) + a.y_off, n1, M64,
                              a.ldy, cw, 32, &err, cw * 2))
      EB_FAIL(EB_E_INVALID, err);
  } else {
    pl.mo = pl.mb;  // unused: fp32 outputs are stored directly
  }
  if (!pl.p.stem_tma) pl.mr = pl.mb;  // (stems with 3-D stores use the slot for 8-row boxes)
  if (a.n_split > 0) {
    const int cw = conv_umma_chunk(bn);
    if (!encode_tiled_2d_bf16(&pl.mr, static_cast<const __nv_bfloat16*>(a.y2) + a.y2_off,
                              a.cout - a.n_split, M64, a.ldy2, cw, 32, &err, cw * 2))
      EB_FAIL(EB_E_INVALID, err);
  }
  if (a.res) {
    const int cw = conv_umma_chunk(bn);
    if (a.out_f32 || a.ldr % 8 != 0) EB_FAIL(EB_E_INVALID, "residual needs a bf16 output, ldr % 8 == 0");
    if (!encode_tiled_2d_bf16(&pl.mr, a.res, a.cout, M64, a.ldr, cw, 32, &err, cw * 2))
      EB_FAIL(EB_E_INVALID, err);
  }
  return EB_OK;
}

int run_conv_plan(ConvPlan& pl, float* ws, size_t ws_cap, const ConvArgs& a, cudaStream_t s,
                  int* launches) {
  if (pl.splits > 1) {
    if (!ws || pl.ws_floats > ws_cap) EB_FAIL(EB_E_INVALID, "split-K workspace too small");
    ConvParams p = pl.p;
    p.out = ws;
    p.ldo = a.cout;
    p.out_off = 0;
    p.out_mode = kOutPartialF32;
    p.vec_ok = (a.cout % 4 == 0);
    p.bias = nullptr;
    p.relu = 0;
    EB_CUDA(conv_umma_launch(pl.ma, pl.mb, pl.mo, pl.mr, p, pl.block_n, pl.grid, s));
    EB_CUDA(k_splitk_finalize(ws, pl.splits, pl.p.M, a.cout, a.bias, a.relu, a.y, a.ldy, a.y_off,
                              a.out_f32, s));
    if (launches) *launches += 2;
  } else {
    EB_CUDA(conv_umma_launch(pl.ma, pl.mb, pl.mo, pl.mr, pl.p, pl.block_n, pl.grid, s));
    if (launches) *launches += 1;
  }
  return EB_OK;
}

}  // namespace

struct eb_engine {
  int device = 0;
  int max_batch = 0;
  bool f32 = false;  // EB_PREC_F32: fp32-faithful parity mode (ref32.cu)
  int C = 0, H = 0, W = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t lanes[kLanes] = {};
  cudaEvent_t ev_fork = nullptr;
  cudaEvent_t ev_join[kLanes] = {};
  void* pool = nullptr;
  uint64_t pool_bytes = 0;
  // the weight pool is shared by an engine and its execution-context clones
  // (eb_engine_clone): freed when the last of them is destroyed
  std::shared_ptr<void> pool_ref;
  std::vector<Tensor> tensors;
  std::vector<eb_op_desc> ops;
  std::vector<Member> members;
  bool finalized = false;
  bool have_pre = false;
  float* d_mean = nullptr;
  float* d_std = nullptr;
  float* d_lut = nullptr;
  int nms = 1;
  uint8_t* d_in_u8 = nullptr;
  float* d_in_f32 = nullptr;
  // eb_forward with pageable host input: pinned staging slots filled by host threads
  // while the previous slot's DMA runs (upload_pageable)
  uint8_t* h_slot[2] = {nullptr, nullptr};
  cudaEvent_t ev_slot[2] = {nullptr, nullptr};
  // eb_forward_batches: a staging buffer filled on a copy stream while the previous
  // batch computes
  void* d_stage = nullptr;
  size_t d_stage_bytes = 0;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_staged = nullptr, ev_stage_free = nullptr;
  float* ws[kLanes] = {};
  size_t ws_floats[kLanes] = {};  // split-K partials, sized at finalize for max_batch
  double* lin_part = nullptr;
  int lin_nsplit = 1;
  int32_t* d_labels = nullptr;
  int32_t* d_topk_idx = nullptr;
  float* d_topk_prob = nullptr;
  int32_t* d_combined = nullptr;
  int* d_kind = nullptr;
  int* d_koff = nullptr;
  int* d_kcnt = nullptr;
  int max_topk = 16;
  int l32_tensor = -1, l64_tensor = -1;
  bool any_cnn = false, any_lin = false;
  std::map<std::pair<int, int>, cudaGraphExec_t> graphs;
  std::map<std::pair<int, int>, int> launch_counts;
  std::mutex mu;
  // profiling: when set, every op runs on the main stream bracketed by events
  std::vector<cudaEvent_t>* prof = nullptr;
  int prof_repeat = 1;
  // stem convs reading an 8-channel image: padded-layout scratch (stem rows / planes modes)
  std::map<const eb_op_desc*, void*> stem_buf;
  // u8 input: stems reading the preprocessed image get their layout straight from K1;
  // the NHWC8 image itself is then written only if something else reads it
  bool img8_needed = true;
  bool layouts_fused = false;  // set per enqueue (u8 input)
  // conv -> 2x2/2 max-pool pairs fused at finalize: op_pool[i] = index of the pool op whose
  // output conv i writes directly (-1 if none); op_skip marks the absorbed pool ops
  std::vector<int> op_pool;
  std::vector<uint8_t> op_skip;
  // VGG block 1 fused at finalize (block1.cu): op_block1[i] = the stem conv whose output
  // conv i (3x3 64->64 + fused pool) computes itself; block1_stem marks that stem op.  The
  // fused kernel runs at batch sizes with enough strips (block1_bh); below, both ops run
  // as declared.
  std::vector<int> op_block1;
  std::vector<uint8_t> block1_stem;
  // grouped 7x7/2 stem + both members' 3x3/2 max-pools fused (stem_pool.cu): for the stem
  // op, the indices of the two absorbed pool ops (-1: none); stempool_pool marks them
  std::vector<std::pair<int, int>> op_stempool;
  std::vector<uint8_t> stempool_pool;
};

namespace {

bool is_prefork(const eb_op_desc& op) { return op.kind == EB_OP_RESIZE || op.prefork; }

// The ConvArgs of a conv op at batch B.  *relayout_dst is set when the op reads the
// padded stem layout of an 8-channel image (written by K1 or by k_stem_relayout).
void conv_args_for(eb_engine* e, const eb_op_desc& op, int B, int fused_pool, ConvArgs* out,
                   const void** relayout_dst) {
  const uint8_t* pool = static_cast<const uint8_t*>(e->pool);
  auto P = [&](uint64_t off) -> const void* {
    return off == EB_NO_OFFSET ? nullptr : static_cast<const void*>(pool + off);
  };
  Tensor& src = e->tensors[op.src];
  Tensor& dst = e->tensors[op.dst];
  const size_t es = dsize(src.dtype);
  const void* x = static_cast<const uint8_t*>(src.dev) + static_cast<size_t>(op.src_c_off) * es;
  ConvArgs& a = *out;
  a.x = x;
  a.B = B;
  a.H = src.h;
  a.W = src.w;
  a.ldx = src.c;
  a.cin = op.src_c;
  a.w = P(op.w_off);
  a.bias = static_cast<const float*>(P(op.b_off));
  if (op.res >= 0) {
    a.res = e->tensors[op.res].dev;
    a.ldr = e->tensors[op.res].c;
  }
  a.y = dst.dev;
  a.ldy = dst.c;
  a.y_off = op.dst_c_off;
  a.cout = op.cout;
  if (fused_pool >= 0) {  // the conv writes the pooled tensor of the absorbed pool op
    const eb_op_desc& po = e->ops[fused_pool];
    a.y = e->tensors[po.dst].dev;
    a.ldy = e->tensors[po.dst].c;
    a.y_off = po.dst_c_off;
    a.pool2 = 1;
  }
  if (op.n_split > 0) {  // grouped launch: columns >= n_split go to dst2
    const Tensor& d2 = e->tensors[op.dst2];
    a.y2 = d2.dev;
    a.ldy2 = d2.c;
    a.y2_off = op.dst2_c_off;
    a.n_split = op.n_split;
  }
  a.kh = op.kh;
  a.kw = op.kw;
  a.sh = op.sh;
  a.sw = op.sw;
  a.ph = op.ph;
  a.pw = op.pw;
  a.relu = op.relu;
  a.out_f32 = dst.dtype == EB_F32;
  // an 8-channel source is a (possibly resized) K1 image: stem mode -- relaid out into
  // the padded rows / planes layout when this op owns such a scratch, else gathered
  a.c8_stem = src.c == 8 && op.src_c == 8 && op.src_c_off == 0;
  *relayout_dst = nullptr;
  if (a.c8_stem) {
    auto it = e->stem_buf.find(&op);
    StemGeom g;
    if (it != e->stem_buf.end() &&
        stem_geom(B, src.h, src.w, op.kh, op.kw, op.sh, op.sw, op.ph, op.pw, &g)) {
      *relayout_dst = it->second;
      a.x = it->second;
      a.c8_stem = 2;
    }
  }
  a.flatten = op.flatten;
  a.groups = op.groups > 1 ? op.groups : 1;
  a.pre_scale = static_cast<const float*>(P(op.scale_off));
  a.pre_shift = static_cast<const float*>(P(op.shift_off));
  a.max_ctas = is_prefork(op) ? 0 : lane_sms(op.stream);
}

// One op of the fp32-faithful mode (ref32.cu) on stream ls.
int enqueue_op_f32(eb_engine* e, const eb_op_desc& op, int B, cudaStream_t ls, int* launches) {
  const uint8_t* pool = static_cast<const uint8_t*>(e->pool);
  auto P = [&](uint64_t off) -> const float* {
    return off == EB_NO_OFFSET ? nullptr : reinterpret_cast<const float*>(pool + off);
  };
  const Tensor& src = e->tensors[op.src];
  const Tensor& dst = e->tensors[op.dst];
  const float* x = static_cast<const float*>(src.dev) + op.src_c_off;
  float* y = static_cast<float*>(dst.dev);
  switch (op.kind) {
    case EB_OP_CONV: {
      const float* res = op.res >= 0 ? static_cast<const float*>(e->tensors[op.res].dev) : nullptr;
      const int ldr = op.res >= 0 ? e->tensors[op.res].c : 0;
      float* y2 = nullptr;
      int ldy2 = 0;
      if (op.n_split > 0) {
        y2 = static_cast<float*>(e->tensors[op.dst2].dev);
        ldy2 = e->tensors[op.dst2].c;
      }
      EB_CUDA(k32_conv(x, B, src.h, src.w, src.c, op.src_c, op.groups > 1 ? op.groups : 1, P(op.w_off),
                       P(op.b_off), res, ldr, y, dst.c, op.dst_c_off, y2, ldy2, op.dst2_c_off,
                       op.n_split, op.cout, op.kh, op.kw, op.sh, op.sw, op.ph, op.pw, op.relu,
                       op.flatten, P(op.scale_off), P(op.shift_off), ls));
      break;
    }
    case EB_OP_POOL:
      EB_CUDA(k32_pool(x, src.c, y, dst.c, op.dst_c_off, B, src.h, src.w, op.src_c, dst.h, dst.w,
                       op.kh, op.sh, op.ph, op.pool_mode, P(op.scale_off), P(op.shift_off), ls));
      break;
    case EB_OP_BNRELU:
      EB_CUDA(k32_bnrelu(x, src.c, y + op.dst_c_off, dst.c, static_cast<int64_t>(B) * src.h * src.w,
                         op.src_c, P(op.scale_off), P(op.shift_off), ls));
      break;
    case EB_OP_GAP:
      EB_CUDA(k32_gap(x, src.c, y, B, src.h * src.w, op.src_c, P(op.scale_off), P(op.shift_off), ls));
      break;
    case EB_OP_RESIZE:
      EB_CUDA(k32_resize(x, src.c, y, dst.c, B, src.h, src.w, op.src_c, dst.h, dst.w, ls));
      break;
    default:
      EB_FAIL(EB_E_INVALID, "unknown op kind");
  }
  ++*launches;
  return EB_OK;
}

// One op on stream ls.
// Band height of the fused VGG block 1 at batch B (0: run the two convs unfused).  The
// fused and unfused paths compute bitwise the same values, so this may depend on B.
int block1_bh(int B, int H, int W) {
  const int nseg = (W + 119) / 120;
  for (int bh : {112, 56, 28}) {
    if (H % bh || bh % 2) continue;
    if (static_cast<int64_t>(B) * (H / bh) * nseg >= 2 * num_sms()) return bh;
  }
  if (H % 28 == 0 && static_cast<int64_t>(B) * (H / 28) * nseg >= num_sms()) return 28;
  return 0;
}

// Pooled rows per strip of the fused stem + pools at batch B (0: unfused).  Bitwise the
// same values either way, so this may depend on B.
int stempool_pb(int B, int Hp) {
  for (int pb : {14, 7}) {
    if (Hp % pb) continue;
    if (static_cast<int64_t>(B) * (Hp / pb) >= num_sms()) return pb;
  }
  return 0;
}

int enqueue_stem_pool(eb_engine* e, const eb_op_desc& g, int B, int pb, cudaStream_t ls, int* launches) {
  const auto pools = e->op_stempool[static_cast<size_t>(&g - e->ops.data())];
  ConvArgs a{};
  const void* rd = nullptr;
  conv_args_for(e, g, B, -1, &a, &rd);
  const Tensor& src = e->tensors[g.src];
  StemGeom sg;
  if (!rd || !stem_geom(B, src.h, src.w, 7, 7, 2, 2, 3, 3, &sg) || sg.mode != kAModeStemPlanes)
    EB_FAIL(EB_E_STATE, "fused stem + pools needs the stem planes layout");
  if (!(e->layouts_fused && g.src == EB_T_IMAGE_NHWC8)) {  // else K1 wrote the layout
    const void* x = static_cast<const uint8_t*>(src.dev) + static_cast<size_t>(g.src_c_off) * 2;
    EB_CUDA(k_stem_relayout(static_cast<const __nv_bfloat16*>(x), B, src.h, src.w, 3, 3, sg.mode, sg.Hq,
                            sg.Wq, static_cast<__nv_bfloat16*>(const_cast<void*>(rd)), ls));
    ++*launches;
  }
  ConvPlan pl;
  const int rc = plan_conv(a, &pl);
  if (rc != EB_OK) return rc;
  if (pl.p.a_mode != kAModeStemPlanes || pl.block_n != g.cout || pl.p.stem_lines <= 0 || pl.p.kbs != 7)
    EB_FAIL(EB_E_STATE, "fused stem + pools: unexpected stem plan");
  const eb_op_desc& q0 = e->ops[pools.first];
  const eb_op_desc& q1 = e->ops[pools.second >= 0 ? pools.second : pools.first];
  const Tensor& d0 = e->tensors[q0.dst];
  const Tensor& d1 = e->tensors[q1.dst];
  StemPoolParams p{};
  p.ncol = g.cout;
  p.Ho = e->tensors[g.dst].h;
  p.Wo = e->tensors[g.dst].w;
  p.Hq = sg.Hq;
  p.Wq = sg.Wq;
  p.plane_px = sg.plane_px;
  p.lines = pl.p.stem_lines;
  p.pb = pb;
  p.nbands = (p.Ho / 2) / pb;
  p.strips = B * p.nbands;
  p.bias = a.bias;
  p.out0 = static_cast<__nv_bfloat16*>(d0.dev);
  p.ld0 = d0.c;
  p.off0 = q0.dst_c_off;
  p.out1 = static_cast<__nv_bfloat16*>(d1.dev);
  p.ld1 = d1.c;
  p.off1 = q1.dst_c_off;
  EB_CUDA(stem_pool_launch(pl.ma, pl.mb, p, std::min(p.strips, num_sms()), ls));
  ++*launches;
  return EB_OK;
}

// The fused VGG block 1 (block1.cu) for stem conv sop -> conv c (+ its fused pool).
int enqueue_block1(eb_engine* e, const eb_op_desc& sop, const eb_op_desc& c, int fused_pool, int B,
                   int bh, cudaStream_t ls, int* launches) {
  ConvArgs as{}, ac{};
  const void* rd = nullptr;
  const void* rd_c = nullptr;
  conv_args_for(e, sop, B, -1, &as, &rd);
  conv_args_for(e, c, B, fused_pool, &ac, &rd_c);
  const Tensor& src = e->tensors[sop.src];
  StemGeom g;
  if (!rd || !stem_geom(B, src.h, src.w, 3, 3, 1, 1, 1, 1, &g) || g.mode != kAModeStemRows)
    EB_FAIL(EB_E_STATE, "fused VGG block 1 needs the stem rows layout");
  if (!(e->layouts_fused && sop.src == EB_T_IMAGE_NHWC8)) {  // else K1 wrote the layout
    const void* x = static_cast<const uint8_t*>(src.dev) + static_cast<size_t>(sop.src_c_off) * 2;
    EB_CUDA(k_stem_relayout(static_cast<const __nv_bfloat16*>(x), B, src.h, src.w, 1, 1, g.mode, g.Hq,
                            g.Wq, static_cast<__nv_bfloat16*>(const_cast<void*>(rd)), ls));
    ++*launches;
  }
  ConvPlan ps, pc;
  int rc = plan_conv(as, &ps);
  if (rc != EB_OK) return rc;
  rc = plan_conv(ac, &pc);
  if (rc != EB_OK) return rc;
  if (ps.p.a_mode != kAModeStemRows || ps.block_n != 64 || ps.p.kbs != 3 || pc.p.a_mode != kAModeTapN ||
      !pc.p.pool2 || pc.block_n != 64 || pc.p.tapn2 || pc.p.tall_rows || pc.p.pair)
    EB_FAIL(EB_E_STATE, "fused VGG block 1: unexpected conv plans");
  CUtensorMap mx;
  std::string err;
  // the padded image rows: (8 channels, Wq pixels, B * Hq rows), 136-pixel runs, zero fill
  if (!encode_tiled_3d_bf16(&mx, rd, 8, g.Wq, static_cast<uint64_t>(B) * g.Hq, 8,
                            static_cast<uint64_t>(g.Wq) * 8, 8, 136, 1, &err, 0))
    EB_FAIL(EB_E_INVALID, err);
  Block1Params p{};
  p.H = src.h;
  p.W = src.w;
  p.Hq = g.Hq;
  p.bh = bh;
  p.nbands = src.h / bh;
  p.nseg = (src.w + 119) / 120;
  p.strips = B * p.nbands * p.nseg;
  p.bias1 = as.bias;
  p.bias2 = ac.bias;
  p.out = static_cast<__nv_bfloat16*>(ac.y);
  p.ldo = ac.ldy;
  p.out_off = ac.y_off;
  EB_CUDA(block1_launch(mx, ps.mb, pc.mb, p, std::min(p.strips, num_sms()), ls));
  ++*launches;
  return EB_OK;
}

int enqueue_op(eb_engine* e, const eb_op_desc& op, int B, cudaStream_t ls, int* launches) {
  const uint8_t* pool = static_cast<const uint8_t*>(e->pool);
  auto P = [&](uint64_t off) -> const void* {
    return off == EB_NO_OFFSET ? nullptr : static_cast<const void*>(pool + off);
  };
  const size_t op_idx = static_cast<size_t>(&op - e->ops.data());
  if (op_idx < e->op_skip.size() && e->op_skip[op_idx]) return EB_OK;  // fused into its conv
  if (op_idx < e->block1_stem.size() && e->block1_stem[op_idx] &&
      block1_bh(B, e->tensors[op.dst].h, e->tensors[op.dst].w) > 0)
    return EB_OK;  // computed inside the next op's fused VGG block-1 kernel
  if (op_idx < e->stempool_pool.size() && e->stempool_pool[op_idx] &&
      stempool_pb(B, e->tensors[op.dst].h) > 0)
    return EB_OK;  // pooled inside the fused stem launch
  if (op_idx < e->op_stempool.size() && e->op_stempool[op_idx].first >= 0 && !e->f32) {
    const int pb = stempool_pb(B, e->tensors[op.dst].h / 2);
    if (pb > 0) return enqueue_stem_pool(e, op, B, pb, ls, launches);
  }
  const int fused_pool = op_idx < e->op_pool.size() ? e->op_pool[op_idx] : -1;
  if (op_idx < e->op_block1.size() && e->op_block1[op_idx] >= 0 && !e->f32) {
    const int bh = block1_bh(B, e->tensors[op.src].h, e->tensors[op.src].w);
    if (bh > 0) return enqueue_block1(e, e->ops[e->op_block1[op_idx]], op, fused_pool, B, bh, ls, launches);
  }
  Tensor& src = e->tensors[op.src];
  Tensor& dst = e->tensors[op.dst];
  const size_t es = dsize(src.dtype);
  const void* x = static_cast<const uint8_t*>(src.dev) + static_cast<size_t>(op.src_c_off) * es;
  if (e->f32 && op.kind != EB_OP_LIN1) return enqueue_op_f32(e, op, B, ls, launches);
  switch (op.kind) {
    case EB_OP_CONV: {
      ConvArgs a{};
      const void* relayout_dst = nullptr;
      conv_args_for(e, op, B, fused_pool, &a, &relayout_dst);
      if (relayout_dst && !(e->layouts_fused && op.src == EB_T_IMAGE_NHWC8)) {  // else K1 wrote it
        StemGeom g;
        stem_geom(B, src.h, src.w, op.kh, op.kw, op.sh, op.sw, op.ph, op.pw, &g);
        EB_CUDA(k_stem_relayout(static_cast<const __nv_bfloat16*>(x), B, src.h, src.w, op.ph,
                                op.pw, g.mode, g.Hq, g.Wq,
                                static_cast<__nv_bfloat16*>(const_cast<void*>(relayout_dst)), ls));
        ++*launches;
      }
      ConvPlan pl;
      int rc = plan_conv(a, &pl);
      if (rc != EB_OK) return rc;
      static const bool dbg = env_flag("EB_DEBUG_PLAN", false);
      if (dbg)
        fprintf(stderr, "[eb] conv src=%d dst=%d mode=%d bn=%d grid=%d splits=%d M=%d N=%d kb=%d cl=%d pair=%d resb=%d\n",
                op.src, op.dst, pl.p.a_mode, pl.block_n, pl.grid, pl.splits, pl.p.M, pl.p.N,
                pl.p.num_kb, pl.p.mcast, pl.p.pair, pl.p.resb);
      return run_conv_plan(pl, e->ws[op.stream], e->ws_floats[op.stream], a, ls, launches);
    }
    case EB_OP_POOL: {
      const int Ho = conv_out(src.h, op.kh, op.sh, op.ph);
      const int Wo = conv_out(src.w, op.kw, op.sw, op.pw);
      EB_CUDA(k_pool(static_cast<const __nv_bfloat16*>(x), src.c,
                     static_cast<__nv_bfloat16*>(dst.dev), dst.c, op.dst_c_off, B, src.h, src.w,
                     op.src_c, Ho, Wo, op.kh, op.sh, op.ph, op.pool_mode,
                     static_cast<const float*>(P(op.scale_off)),
                     static_cast<const float*>(P(op.shift_off)), ls));
      ++*launches;
      return EB_OK;
    }
    case EB_OP_BNRELU: {
      EB_CUDA(k_bnrelu(static_cast<const __nv_bfloat16*>(x), src.c,
                       static_cast<__nv_bfloat16*>(dst.dev) + op.dst_c_off, dst.c,
                       static_cast<int64_t>(B) * src.h * src.w, op.src_c,
                       static_cast<const float*>(P(op.scale_off)),
                       static_cast<const float*>(P(op.shift_off)), ls));
      ++*launches;
      return EB_OK;
    }
    case EB_OP_GAP: {
      EB_CUDA(k_gap(static_cast<const __nv_bfloat16*>(x), src.c,
                    static_cast<__nv_bfloat16*>(dst.dev), B, src.h * src.w, op.src_c,
                    static_cast<const float*>(P(op.scale_off)),
                    static_cast<const float*>(P(op.shift_off)), ls));
      ++*launches;
      return EB_OK;
    }
    case EB_OP_RESIZE: {
      EB_CUDA(k_resize_bilinear(static_cast<const __nv_bfloat16*>(x), src.c,
                                static_cast<__nv_bfloat16*>(dst.dev), dst.c, B, src.h, src.w,
                                op.src_c, dst.h, dst.w, ls));
      ++*launches;
      return EB_OK;
    }
    case EB_OP_LIN1: {
      const int64_t D = static_cast<int64_t>(src.c) * src.h * src.w;
      EB_CUDA(k_lin1(static_cast<const float*>(src.dev), static_cast<const float*>(P(op.w_off)),
                     static_cast<const float*>(P(op.b_off)), e->lin_part,
                     static_cast<double*>(dst.dev), B, op.cout, D, e->lin_nsplit, ls));
      *launches += 2;
      return EB_OK;
    }
    default:
      EB_FAIL(EB_E_INVALID, "unknown op kind");
  }
}

// Enqueue preprocess + every op for batch B on e->stream (fork/join over lanes).
int enqueue_layers(
eb_engine* e, int input_kind, int B, int* launches) {
  cudaStream_t s = e->stream;
  set_pdl_batch(B);
  const int64_t plane = static_cast<int64_t>(e->H) * e->W;
  Tensor& img8 = e->tensors[EB_T_IMAGE_NHWC8];
  Tensor& imgf = e->tensors[EB_T_IMAGE_F32];
  e->layouts_fused = false;
  if (e->f32 && e->any_cnn) {
    if (input_kind == EB_IN_U8_HWC)
      EB_CUDA(k32_preprocess_u8(e->d_in_u8, static_cast<float*>(img8.dev), B, e->C, plane, 8,
                                e->d_lut, s));
    else
      EB_CUDA(k32_preprocess_f32chw(e->d_in_f32, static_cast<float*>(img8.dev), B, e->C, plane, 8,
                                    e->d_mean, e->d_std, e->nms, s));
    ++*launches;
  }
  if (input_kind == EB_IN_U8_HWC) {
    if (e->any_cnn && !e->f32) {
      if (e->img8_needed) {
        EB_CUDA(k_preprocess_u8hwc_to_nhwc(e->d_in_u8, static_cast<__nv_bfloat16*>(img8.dev), B,
                                           e->C, plane, 8, e->d_lut, s));
        ++*launches;
      }
      // stems on the preprocessed image: K1 writes their padded layouts directly
      for (const auto& kv : e->stem_buf) {
        const eb_op_desc& op = *kv.first;
        if (op.src != EB_T_IMAGE_NHWC8) continue;
        StemGeom g;
        if (!stem_geom(B, e->H, e->W, op.kh, op.kw, op.sh, op.sw, op.ph, op.pw, &g))
          EB_FAIL(EB_E_INVALID, "stem layout geometry");
        EB_CUDA(k_preprocess_u8_to_layout(e->d_in_u8, B, e->C, e->H, e->W, e->d_lut, op.ph, op.pw,
                                          g.mode, g.Hq, g.Wq, static_cast<__nv_bfloat16*>(kv.second),
                                          s));
        ++*launches;
        e->layouts_fused = true;
      }
    }
    if (e->any_lin) {
      EB_CUDA(k_preprocess_u8hwc_to_f32chw(e->d_in_u8, static_cast<float*>(imgf.dev), B, e->C,
                                           plane, e->d_lut, s));
      ++*launches;
    }
  } else {
    if (e->any_cnn && !e->f32) {
      EB_CUDA(k_preprocess_f32chw_to_nhwc(e->d_in_f32, static_cast<__nv_bfloat16*>(img8.dev), B,
                                          e->C, plane, 8, e->d_mean, e->d_std, e->nms, s));
      ++*launches;
    }
    if (e->any_lin) {
      EB_CUDA(k_preprocess_f32(e->d_in_f32, static_cast<float*>(imgf.dev), B, e->C, plane,
                               e->d_mean, e->d_std, e->nms, s));
      ++*launches;
    }
  }
  if (e->prof) {
    // profiling: every op serialised on the main stream in declaration order,
    // bracketed by events (one elapsed time per op)
    // (prof_repeat > 1: each op launched that many times back to back -- every op is a
    // pure function of tensors it does not write -- so a short op's time is its own, not
    // the host's launch latency; the caller divides)
    for (const auto& op : e->ops) {
      cudaEvent_t ev;
      EB_CUDA(cudaEventCreate(&ev));
      e->prof->push_back(ev);
      EB_CUDA(cudaEventRecord(ev, s));
      for (int r = 0; r < e->prof_repeat; ++r) {
        const int rc = enqueue_op(e, op, B, s, launches);
        if (rc != EB_OK) return rc;
      }
    }
    cudaEvent_t ev;
    EB_CUDA(cudaEventCreate(&ev));
    e->prof->push_back(ev);
    EB_CUDA(cudaEventRecord(ev, s));
    return EB_OK;
  }
  // Inputs shared by members on several lanes (K1's resized copies, grouped stems) are
  // produced on the main stream before the fork.
  for (const auto& op : e->ops) {
    if (!is_prefork(op)) continue;
    const int rc = enqueue_op(e, op, B, s, launches);
    if (rc != EB_OK) return rc;
  }
  bool used[kLanes] = {};
  for (const auto& op : e->ops)
    if (!is_prefork(op)) used[op.stream] = true;
  EB_CUDA(cudaEventRecord(e->ev_fork, s));
  for (int l = 1; l < kLanes; ++l)
    if (used[l]) EB_CUDA(cudaStreamWaitEvent(e->lanes[l], e->ev_fork, 0));
  for (const auto& op : e->ops) {
    if (is_prefork(op)) continue;
    const int rc = enqueue_op(e, op, B, op.stream == 0 ? s : e->lanes[op.stream], launches);
    if (rc != EB_OK) return rc;
  }
  for (int l = 1; l < kLanes; ++l) {
    if (!used[l]) continue;
    EB_CUDA(cudaEventRecord(e->ev_join[l], e->lanes[l]));
    EB_CUDA(cudaStreamWaitEvent(s, e->ev_join[l], 0));
  }
  return EB_OK;
}

// Flexible batching: a batch runs through the graph of its size bucket -- exact up to 8,
// then multiples of 16 up to 128, of 32 up to 512, of 64 beyond (at most 12 % padding) --
// so a stream of arbitrary request sizes needs a few dozen graphs, not one per size.
// Rows past B compute on whatever the input buffer holds and are never read back: every
// op is per-sample and the conv plans do not depend on B (plan_conv), so the first B
// rows are bitwise what an exact-size run gives (tests/test_gpu_batch_invariance.py).
// EB_BUCKETS=0: one graph per exact size.
int bucket_of(const eb_engine* e, int B) {
  static const bool on = env_flag("EB_BUCKETS", true);
  if (!on || B <= 8) return B;
  const int q = B <= 128 ? 16 : B <= 512 ? 32 : 64;
  return std::min(e->max_batch, (B + q - 1) / q * q);
}

int run_layers(eb_engine* e, int input_kind, int B) {
  B = bucket_of(e, B);
  const auto key = std::make_pair(B, input_kind);
  auto it = e->graphs.find(key);
  if (it != e->graphs.end()) {
    EB_CUDA(cudaGraphLaunch(it->second, e->stream));
    return EB_OK;
  }
  int launches = 0;
  static const bool no_graph = env_flag("EB_NO_GRAPH", false);
  if (no_graph || static_cast<int>(e->graphs.size()) >= kMaxGraphs) {
    return enqueue_layers(e, input_kind, B, &launches);  // plain launches
  }
  EB_CUDA(cudaStreamBeginCapture(e->stream, cudaStreamCaptureModeThreadLocal));
  int rc = enqueue_layers(e, input_kind, B, &launches);
  cudaGraph_t g = nullptr;
  cudaError_t ce = cudaStreamEndCapture(e->stream, &g);
  if (rc != EB_OK) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  if (ce != cudaSuccess) EB_FAIL(EB_E_CUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
  cudaGraphExec_t ex = nullptr;
  ce = cudaGraphInstantiate(&ex, g, 0);
  cudaGraphDestroy(g);
  if (ce != cudaSuccess)
    EB_FAIL(EB_E_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(ce));
  e->graphs[key] = ex;
  e->launch_counts[key] = launches;
  EB_CUDA(cudaGraphLaunch(ex, e->stream));
  return EB_OK;
}

int check_batch(eb_engine* e, int batch) {
  if (!e) EB_FAIL(EB_E_INVALID, "null engine");
  if (!e->finalized) EB_FAIL(EB_E_STATE, "engine not finalized");
  if (batch == 0) EB_FAIL(EB_E_EMPTY, "batch has no samples");
  if (batch < 0) EB_FAIL(EB_E_INVALID, "negative batch");
  if (batch > e->max_batch)
    EB_FAIL(EB_E_TOO_LARGE, "batch size " + std::to_string(batch) + " exceeds max_batch " +
                                std::to_string(e->max_batch));
  return EB_OK;
}

int check_policy(eb_engine* e, int policy, int policy_k) {
  if (policy == EB_POLICY_NONE) return EB_OK;
  if (policy < 0 || policy > EB_POLICY_AT_LEAST) EB_FAIL(EB_E_INVALID, "unknown policy");
  for (const auto& m : e->members)
    if (m.k != 2) EB_FAIL(EB_E_POLICY, "policy unavailable: every model must be binary");
  const int n = static_cast<int>(e->members.size());
  if (policy == EB_POLICY_AT_LEAST && (policy_k < 1 || policy_k > n))
    EB_FAIL(EB_E_BAD_K, "k must be between 1 and " + std::to_string(n) +
                            " for this ensemble, got " + std::to_string(policy_k));
  return EB_OK;
}

int enqueue_combine(eb_engine* e, int B, int topk, int policy, int policy_k) {
  const float* l32 = nullptr;
  const double* l64 = nullptr;
  int ld32 = 0, ld64 = 0;
  if (e->l32_tensor >= 0) {
    l32 = static_cast<const float*>(e->tensors[e->l32_tensor].dev);
    ld32 = e->tensors[e->l32_tensor].c;
  }
  if (e->l64_tensor >= 0) {
    l64 = static_cast<const double*>(e->tensors[e->l64_tensor].dev);
    ld64 = e->tensors[e->l64_tensor].c;
  }
  EB_CUDA(k_combine(l32, ld32, l64, ld64, e->d_kind, e->d_koff, e->d_kcnt,
                    static_cast<int>(e->members.size()), B, e->d_labels, topk, e->d_topk_idx,
                    e->d_topk_prob, policy, policy_k, e->d_combined, e->stream));
  return EB_OK;
}

}  // namespace

// Host -> device copy of a request from ordinary (pageable) memory.  The driver stages
// pageable copies through its own small pinned buffers with one thread (~12 GB/s for the
// reference's f32 samples, 154 MB per 256 images); here kHostCopyThreads threads copy
// kSlotBytes chunks into two pinned slots while the previous slot's DMA runs (B200 box,
// C2 B = 256, f32: drop-in forward 9.9k -> 12.5k images/s with 4 threads).
constexpr size_t kSlotBytes = 16u << 20;
constexpr int kMaxHostCopyThreads = 16;
int host_copy_threads() {  // EB_HOST_COPY_THREADS (default 4)
  static const int n = [] {
    const char* v = getenv("EB_HOST_COPY_THREADS");
    const int k = (v && *v) ? atoi(v) : 4;
    return std::max(1, std::min(k, kMaxHostCopyThreads));
  }();
  return n;
}

static bool is_pageable(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

static int upload_pageable(eb_engine* e, void* dst, const void* src, size_t bytes) {
  for (int i = 0; i < 2; ++i) {
    if (!e->h_slot[i]) {
      if (cudaHostAlloc(reinterpret_cast<void**>(&e->h_slot[i]), kSlotBytes, cudaHostAllocDefault) !=
          cudaSuccess) {
        cudaGetLastError();
        e->h_slot[i] = nullptr;
        EB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, e->stream));  // plain path
        return EB_OK;
      }
      EB_CUDA(cudaEventCreateWithFlags(&e->ev_slot[i], cudaEventDisableTiming));
    }
  }
  const uint8_t* s = static_cast<const uint8_t*>(src);
  uint8_t* d = static_cast<uint8_t*>(dst);
  int slot = 0;
  bool used[2] = {false, false};
  for (size_t off = 0; off < bytes; off += kSlotBytes, slot ^= 1) {
    const size_t n = std::min(kSlotBytes, bytes - off);
    if (used[slot]) EB_CUDA(cudaEventSynchronize(e->ev_slot[slot]));  // its last DMA is done
    uint8_t* h = e->h_slot[slot];
    const int nt = host_copy_threads();
    const size_t part = (n / nt + 63) / 64 * 64;
    std::thread th[kMaxHostCopyThreads];
    for (int t = 1; t < nt; ++t) {
      const size_t a = std::min(n, t * part), b = std::min(n, (t + 1) * part);
      th[t] = std::thread([=] { if (b > a) memcpy(h + a, s + off + a, b - a); });
    }
    memcpy(h, s + off, std::min(n, part));
    for (int t = 1; t < nt; ++t) th[t].join();
    EB_CUDA(cudaMemcpyAsync(d + off, h, n, cudaMemcpyHostToDevice, e->stream));
    EB_CUDA(cudaEventRecord(e->ev_slot[slot], e->stream));
    used[slot] = true;
  }
  return EB_OK;
}

// ====================================================================== C ABI

extern "C" {

const char* eb_last_error(void) { return g_err.c_str(); }
int eb_abi_version(void) { return 1; }

int eb_engine_create(int device, int max_batch, int in_c, int in_h, int in_w, eb_engine** out) {
  if (!out || max_batch < 1 || in_c < 1 || in_h < 1 || in_w < 1)
    EB_FAIL(EB_E_INVALID, "bad engine geometry");
  EB_CUDA(cudaSetDevice(device));
  eb_engine* e = new eb_engine();
  e->device = device;
  e->max_batch = max_batch;
  e->C = in_c;
  e->H = in_h;
  e->W = in_w;
  if (cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete e;
    EB_FAIL(EB_E_CUDA, "stream create failed");
  }
  {
    // EB_LANE_PRIO=<lane>: that lane's stream gets the highest priority (experiment)
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    const char* pr = getenv("EB_LANE_PRIO");
    const int prio_lane = (pr && *pr) ? atoi(pr) : -1;
    for (int l = 1; l < kLanes; ++l)
      cudaStreamCreateWithPriority(&e->lanes[l], cudaStreamNonBlocking, l == prio_lane ? hi : lo);
  }
  e->lanes[0] = e->stream;
  cudaEventCreateWithFlags(&e->ev_fork, cudaEventDisableTiming);
  for (int l = 0; l < kLanes; ++l) cudaEventCreateWithFlags(&e->ev_join[l], cudaEventDisableTiming);
  e->tensors.push_back(Tensor{in_h, in_w, 8, EB_BF16, nullptr});
  e->tensors.push_back(Tensor{in_h, in_w, in_c, EB_F32, nullptr});  // (C,H,W) layout
  *out = e;
  return EB_OK;
}

int eb_engine_set_precision(eb_engine* e, int precision) {
  if (!e) EB_FAIL(EB_E_INVALID, "null engine");
  if (e->finalized || e->tensors.size() != 2 || !e->ops.empty())
    EB_FAIL(EB_E_STATE, "precision must be set before tensors and ops are declared");
  if (precision != EB_PREC_BF16 && precision != EB_PREC_F32) EB_FAIL(EB_E_INVALID, "unknown precision");
  e->f32 = precision == EB_PREC_F32;
  e->tensors[EB_T_IMAGE_NHWC8].dtype = e->f32 ? EB_F32 : EB_BF16;
  return EB_OK;
}

int eb_engine_destroy(eb_engine* e) {
  if (!e) return EB_OK;
  cudaSetDevice(e->device);
  cudaStreamSynchronize(e->stream);
  for (auto& kv : e->graphs) cudaGraphExecDestroy(kv.second);
  for (auto& t : e->tensors) cudaFree(t.dev);
  for (auto& kv : e->stem_buf) cudaFree(kv.second);
  e->pool_ref.reset();
  cudaFree(e->d_mean);
  cudaFree(e->d_std);
  cudaFree(e->d_lut);
  cudaFree(e->d_in_u8);
  cudaFree(e->d_in_f32);
  cudaFree(e->d_stage);
  if (e->copy_stream) cudaStreamDestroy(e->copy_stream);
  for (int i = 0; i < 2; ++i) {
    if (e->h_slot[i]) cudaFreeHost(e->h_slot[i]);
    if (e->ev_slot[i]) cudaEventDestroy(e->ev_slot[i]);
  }
  if (e->ev_staged) cudaEventDestroy(e->ev_staged);
  if (e->ev_stage_free) cudaEventDestroy(e->ev_stage_free);
  for (int l = 0; l < kLanes; ++l) cudaFree(e->ws[l]);
  cudaFree(e->lin_part);
  cudaFree(e->d_labels);
  cudaFree(e->d_topk_idx);
  cudaFree(e->d_topk_prob);
  cudaFree(e->d_combined);
  cudaFree(e->d_kind);
  cudaFree(e->d_koff);
  cudaFree(e->d_kcnt);
  for (int l = 1; l < kLanes; ++l) cudaStreamDestroy(e->lanes[l]);
  cudaEventDestroy(e->ev_fork);
  for (int l = 0; l < kLanes; ++l) cudaEventDestroy(e->ev_join[l]);
  cudaStreamDestroy(e->stream);
  delete e;
  return EB_OK;
}

int eb_engine_clone(eb_engine* src, eb_engine** out) {
  if (!src || !out) EB_FAIL(EB_E_INVALID, "null argument");
  if (!src->finalized) EB_FAIL(EB_E_STATE, "clone needs a finalized engine");
  eb_engine* e = nullptr;
  int rc = eb_engine_create(src->device, src->max_batch, src->C, src->H, src->W, &e);
  if (rc != EB_OK) return rc;
  e->f32 = src->f32;
  e->tensors = src->tensors;
  for (auto& t : e->tensors) t.dev = nullptr;
  e->ops = src->ops;
  e->members = src->members;
  e->l32_tensor = src->l32_tensor;
  e->l64_tensor = src->l64_tensor;
  e->any_cnn = src->any_cnn;
  e->any_lin = src->any_lin;
  e->pool = src->pool;
  e->pool_bytes = src->pool_bytes;
  e->pool_ref = src->pool_ref;
  e->nms = src->nms;
  cudaSetDevice(e->device);
  const size_t c = static_cast<size_t>(e->C);
  bool ok = cudaMalloc(&e->d_mean, c * sizeof(float)) == cudaSuccess &&
            cudaMalloc(&e->d_std, c * sizeof(float)) == cudaSuccess &&
            cudaMalloc(&e->d_lut, c * 256 * sizeof(float)) == cudaSuccess &&
            cudaMemcpy(e->d_mean, src->d_mean, c * sizeof(float), cudaMemcpyDeviceToDevice) == cudaSuccess &&
            cudaMemcpy(e->d_std, src->d_std, c * sizeof(float), cudaMemcpyDeviceToDevice) == cudaSuccess &&
            cudaMemcpy(e->d_lut, src->d_lut, c * 256 * sizeof(float), cudaMemcpyDeviceToDevice) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    eb_engine_destroy(e);
    EB_FAIL(EB_E_NOMEM, "clone: preprocess constants");
  }
  e->have_pre = true;
  rc = eb_finalize(e);
  if (rc != EB_OK) {
    const std::string msg = eb_last_error();
    eb_engine_destroy(e);
    EB_FAIL(rc, msg);
  }
  *out = e;
  return EB_OK;
}

int eb_set_preprocess(eb_engine* e, const float* host_mean, const float* host_std, int n,
                      const float* host_lut_u8) {
  if (!e || !host_mean || !host_std || !host_lut_u8) EB_FAIL(EB_E_INVALID, "null argument");
  if (n != 1 && n != e->C)
    EB_FAIL(EB_E_SHAPE, "mean/std have " + std::to_string(n) + " entries; input has " +
                            std::to_string(e->C) + " channel(s)");
  cudaSetDevice(e->device);
  if (!e->d_mean) {
    EB_CUDA(cudaMalloc(&e->d_mean, e->C * sizeof(float)));
    EB_CUDA(cudaMalloc(&e->d_std, e->C * sizeof(float)));
    EB_CUDA(cudaMalloc(&e->d_lut, e->C * 256 * sizeof(float)));
  }
  EB_CUDA(cudaMemcpy(e->d_mean, host_mean, n * sizeof(float), cudaMemcpyHostToDevice));
  EB_CUDA(cudaMemcpy(e->d_std, host_std, n * sizeof(float), cudaMemcpyHostToDevice));
  EB_CUDA(cudaMemcpy(e->d_lut, host_lut_u8, e->C * 256 * sizeof(float), cudaMemcpyHostToDevice));
  e->nms = n;
  e->have_pre = true;
  return EB_OK;
}

int eb_pool_reserve(eb_engine* e, uint64_t bytes) {
  if (!e || e->pool) EB_FAIL(EB_E_STATE, "pool already reserved");
  cudaSetDevice(e->device);
  if (cudaMalloc(&e->pool, bytes ? bytes : 256) != cudaSuccess) {
    cudaGetLastError();
    EB_FAIL(EB_E_NOMEM, "cannot allocate a " + std::to_string(bytes) + "-byte weight pool");
  }
  {
    const int dev = e->device;
    e->pool_ref = std::shared_ptr<void>(e->pool, [dev](void* p) {
      cudaSetDevice(dev);
      cudaFree(p);
    });
  }
  e->pool_bytes = bytes;
  return EB_OK;
}

int eb_pool_write(eb_engine* e, uint64_t offset, const void* host_src, uint64_t bytes) {
  if (!e || !e->pool) EB_FAIL(EB_E_STATE, "pool not reserved");
  if (offset + bytes > e->pool_bytes) EB_FAIL(EB_E_INVALID, "pool write out of range");
  cudaSetDevice(e->device);
  EB_CUDA(cudaMemcpy(static_cast<uint8_t*>(e->pool) + offset, host_src, bytes,
                     cudaMemcpyHostToDevice));
  return EB_OK;
}

int eb_pool_bytes(eb_engine* e, uint64_t* bytes) {
  if (!e || !bytes) EB_FAIL(EB_E_INVALID, "null argument");
  *bytes = e->pool_bytes;
  return EB_OK;
}

int eb_tensor(eb_engine* e, int h, int w, int c, int dtype, int* id_out) {
  if (!e || e->finalized) EB_FAIL(EB_E_STATE, "engine finalized");
  if (h < 1 || w < 1 || c < 1 || dtype < EB_BF16 || dtype > EB_F64)
    EB_FAIL(EB_E_INVALID, "bad tensor shape");
  if (dtype == EB_BF16 && c % 8 != 0) EB_FAIL(EB_E_INVALID, "bf16 tensors need c % 8 == 0");
  e->tensors.push_back(Tensor{h, w, c, dtype, nullptr});
  *id_out = static_cast<int>(e->tensors.size()) - 1;
  return EB_OK;
}

int eb_add_op(eb_engine* e, const eb_op_desc* op) {
  if (!e || !op || e->finalized) EB_FAIL(EB_E_STATE, "engine finalized");
  const int nt = static_cast<int>(e->tensors.size());
  if (op->src < 0 || op->src >= nt || op->dst < 0 || op->dst >= nt || op->res >= nt)
    EB_FAIL(EB_E_INVALID, "op references an unknown tensor");
  if (op->stream < 0 || op->stream >= kLanes) EB_FAIL(EB_E_INVALID, "bad lane");
  const Tensor& src = e->tensors[op->src];
  const Tensor& dst = e->tensors[op->dst];
  if (op->src_c_off < 0 || op->src_c < 1 || op->src_c_off + op->src_c > src.c)
    EB_FAIL(EB_E_INVALID, "source channel slice out of range");
  if (op->kind == EB_OP_CONV) {
    if (e->f32 ? (src.dtype != EB_F32 || dst.dtype != EB_F32 ||
                  (op->res >= 0 && e->tensors[op->res].dtype != EB_F32))
               : (src.dtype != EB_BF16 || (dst.dtype != EB_BF16 && dst.dtype != EB_F32)))
      EB_FAIL(EB_E_INVALID, "conv dtypes");
    if (op->dst_c_off < 0 || op->dst_c_off + op->cout > dst.c)
      EB_FAIL(EB_E_INVALID, "conv output slice out of range");
    const int Ho = op->flatten ? 1 : conv_out(src.h, op->kh, op->sh, op->ph);
    const int Wo = op->flatten ? 1 : conv_out(src.w, op->kw, op->sw, op->pw);
    if (Ho != dst.h || Wo != dst.w)
      EB_FAIL(EB_E_SHAPE, "conv output geometry " + std::to_string(Ho) + "x" +
                              std::to_string(Wo) + " does not match the destination tensor");
    if (op->w_off == EB_NO_OFFSET || op->w_off % 16 != 0) EB_FAIL(EB_E_INVALID, "weights offset");
    if (op->src_c_off % 8 != 0 || op->dst_c_off % 8 != 0)
      EB_FAIL(EB_E_INVALID, "channel slices must start at multiples of 8");
    if (dst.dtype == EB_BF16 && op->cout % 8 != 0)
      EB_FAIL(EB_E_INVALID, "bf16 conv outputs need cout % 8 == 0");
    if (e->f32 && op->groups > 1 && (op->src_c % op->groups || op->cout % op->groups))
      EB_FAIL(EB_E_INVALID, "grouped conv channels must divide by groups");
    if (op->res >= 0 && (e->tensors[op->res].h != dst.h || e->tensors[op->res].w != dst.w))
      EB_FAIL(EB_E_SHAPE, "residual geometry");
    if (op->n_split > 0) {
      if (op->dst2 < 0 || op->dst2 >= nt || op->res >= 0 || op->n_split >= op->cout)
        EB_FAIL(EB_E_INVALID, "grouped launch needs dst2 and no residual");
      const Tensor& d2 = e->tensors[op->dst2];
      if (d2.h != dst.h || d2.w != dst.w || d2.dtype != dst.dtype ||
          op->dst2_c_off + (op->cout - op->n_split) > d2.c || op->dst2_c_off % 8 != 0)
        EB_FAIL(EB_E_SHAPE, "grouped launch: second destination geometry");
    }
  } else if (op->kind == EB_OP_LIN1) {
    if (op->src != EB_T_IMAGE_F32 || dst.dtype != EB_F64 || dst.c != op->cout)
      EB_FAIL(EB_E_INVALID, "LIN1 op must read the f32 image and write fp64 scores");
  } else if (op->kind == EB_OP_RESIZE) {
    const int dt = e->f32 ? EB_F32 : EB_BF16;
    if (src.dtype != dt || dst.dtype != dt || op->src_c % 8 != 0 || op->dst_c_off != 0)
      EB_FAIL(EB_E_INVALID, "resize works on NHWC images with 8-channel groups");
  } else if (op->kind == EB_OP_POOL || op->kind == EB_OP_BNRELU || op->kind == EB_OP_GAP) {
    const int dt = e->f32 ? EB_F32 : EB_BF16;
    if (src.dtype != dt || dst.dtype != dt) EB_FAIL(EB_E_INVALID, "pool dtypes");
    if (op->src_c % 8 != 0 || op->src_c_off % 8 != 0 || op->dst_c_off % 8 != 0)
      EB_FAIL(EB_E_INVALID, "channel slices must be multiples of 8");
    if (op->kind == EB_OP_POOL) {
      const int Ho = conv_out(src.h, op->kh, op->sh, op->ph);
      const int Wo = conv_out(src.w, op->kw, op->sw, op->pw);
      if (Ho != dst.h || Wo != dst.w || op->kh != op->kw || op->sh != op->sw || op->ph != op->pw)
        EB_FAIL(EB_E_SHAPE, "pool geometry");
    }
    if (op->kind == EB_OP_GAP && (dst.h != 1 || dst.w != 1 || dst.c != op->src_c))
      EB_FAIL(EB_E_SHAPE, "gap destination must be (1, 1, C)");
  } else {
    EB_FAIL(EB_E_INVALID, "unknown op kind");
  }
  e->ops.push_back(*op);
  return EB_OK;
}

int eb_add_member(eb_engine* e, int kind, int logits_tensor, int k_off, int k) {
  if (!e || e->finalized) EB_FAIL(EB_E_STATE, "engine finalized");
  if (logits_tensor < 0 || logits_tensor >= static_cast<int>(e->tensors.size()) || k < 1 ||
      k_off < 0 || k_off + k > e->tensors[logits_tensor].c)
    EB_FAIL(EB_E_INVALID, "bad member logits slice");
  const Tensor& t = e->tensors[logits_tensor];
  if (kind == EB_MEMBER_CNN) {
    if (t.dtype != EB_F32) EB_FAIL(EB_E_INVALID, "CNN logits must be fp32");
    if (e->C > 8) EB_FAIL(EB_E_INVALID, "CNN members need at most 8 input channels");
    if (e->l32_tensor >= 0 && e->l32_tensor != logits_tensor)
      EB_FAIL(EB_E_INVALID, "all CNN members must share one logits tensor");
    e->l32_tensor = logits_tensor;
    e->any_cnn = true;
  } else if (kind == EB_MEMBER_LIN1) {
    if (t.dtype != EB_F64) EB_FAIL(EB_E_INVALID, "LIN1 logits must be fp64");
    if (e->l64_tensor >= 0 && e->l64_tensor != logits_tensor)
      EB_FAIL(EB_E_INVALID, "all LIN1 members must share one logits tensor");
    e->l64_tensor = logits_tensor;
    e->any_lin = true;
  } else {
    EB_FAIL(EB_E_INVALID, "unknown member kind");
  }
  e->members.push_back(Member{kind, logits_tensor, k_off, k});
  return EB_OK;
}

namespace {
// Peephole at finalize: a taps-in-N conv whose only reader is the next op on its lane, a
// 2x2/2 max-pool over the whole tensor, writes the pooled tensor itself (VGG: conv1_2 +
// pool1 at 224x224 is 1.46 ms unfused, 1.11-1.15 ms fused on B200, B = 256).  EB_POOL_FUSE=0
// keeps them apart.
void fuse_conv_pools(eb_engine* e) {
  const size_t n = e->ops.size();
  e->op_pool.assign(n, -1);
  e->op_skip.assign(n, 0);
  static const bool on = env_flag("EB_POOL_FUSE", true);
  if (!on || !tap_shift_enabled() || !tapn_enabled()) return;
  for (size_t i = 0; i + 1 < n; ++i) {
    const eb_op_desc& c = e->ops[i];
    const eb_op_desc& po = e->ops[i + 1];
    if (c.kind != EB_OP_CONV || po.kind != EB_OP_POOL || po.src != c.dst) continue;
    if (po.pool_mode != EB_POOL_MAX || po.kh != 2 || po.kw != 2 || po.sh != 2 || po.sw != 2 ||
        po.ph || po.pw || po.stream != c.stream || is_prefork(po) || is_prefork(c))
      continue;
    const Tensor& src = e->tensors[c.src];
    const Tensor& t = e->tensors[c.dst];
    const Tensor& pd = e->tensors[po.dst];
    if (t.dtype != EB_BF16 || pd.dtype != EB_BF16 || c.dst_c_off != 0 || c.cout != t.c ||
        po.src_c_off != 0 || po.src_c != t.c || pd.c % 8 || po.dst_c_off % 8)
      continue;
    // the taps-in-N geometry (plan_conv): 3x3/s1/p1, Cout <= 64 in 32s, even output, plain
    if (c.kh != 3 || c.kw != 3 || c.sh != 1 || c.sw != 1 || c.ph != 1 || c.pw != 1 ||
        c.cout % 32 || c.cout > std::min(64, tapn_max_cout()) || c.groups > 1 || c.res >= 0 ||
        c.scale_off != EB_NO_OFFSET || c.n_split || c.flatten || src.c == 8 || t.h % 2 || t.w % 2)
      continue;
    bool other = false;  // nobody else reads the full-resolution output
    for (size_t k = 0; k < n; ++k)
      if (k != i + 1 && (e->ops[k].src == c.dst || e->ops[k].res == c.dst)) other = true;
    for (const auto& m : e->members)
      if (m.tensor == c.dst) other = true;
    if (other) continue;
    e->op_pool[i] = static_cast<int>(i + 1);
    e->op_skip[i + 1] = 1;
    ++i;
  }
}

// Peephole at finalize, after fuse_conv_pools: a stem conv (3x3/s1/p1 over the 8-channel
// image in the rows layout, 64 outputs, ReLU) whose only reader is the next op on its
// lane, a taps-in-N 3x3 64->64 conv with a fused 2x2 max-pool, becomes one kernel
// (block1.cu).  EB_BLOCK1=0 keeps them apart (read per finalize: tests compare both).
// Peephole at finalize: a 7x7/2/p3 stem over the 8-channel image in the planes layout with
// ReLU -- a member's own (64 outputs) or a grouped launch of two members (64 + 64 channels
// of one tensor) -- each 64-channel part of whose output is read only by one 3x3/2/p1
// max-pool becomes one kernel that writes the pooled tensors (stem_pool.cu).
// EB_STEM_POOL=0 keeps them apart (read per finalize).
void fuse_stem_pools(eb_engine* e) {
  const size_t n = e->ops.size();
  e->op_stempool.assign(n, {-1, -1});
  e->stempool_pool.assign(n, 0);
  if (!env_flag("EB_STEM_POOL", true) || !stem_rows_enabled() || e->f32) return;
  for (size_t i = 0; i < n; ++i) {
    const eb_op_desc& g = e->ops[i];
    if (g.kind != EB_OP_CONV || g.n_split != 0 || (g.cout != 128 && g.cout != 64) ||
        (g.cout == 128 && !g.prefork) || g.kh != 7 || g.kw != 7 || g.sh != 2 || g.sw != 2 ||
        g.ph != 3 || g.pw != 3 || !g.relu || g.res >= 0 || g.groups > 1 || g.flatten ||
        g.b_off == EB_NO_OFFSET || g.scale_off != EB_NO_OFFSET || g.dst_c_off != 0 ||
        e->op_pool[i] >= 0 || e->op_skip[i])
      continue;
    const Tensor& src = e->tensors[g.src];
    const Tensor& t = e->tensors[g.dst];
    if (!(src.c == 8 && g.src_c == 8 && g.src_c_off == 0) || t.c != g.cout || t.dtype != EB_BF16 ||
        t.h % 2 || t.w % 2 || t.w > 128)
      continue;
    const int parts = g.cout / 64;
    int pool_of[2] = {-1, -1};
    bool ok = true;
    for (size_t k = 0; k < n && ok; ++k) {
      const eb_op_desc& o = e->ops[k];
      if (k == i || (o.src != g.dst && o.res != g.dst)) continue;
      const int half = o.src_c_off == 0 ? 0 : o.src_c_off == 64 ? 1 : -1;
      const Tensor& d = e->tensors[o.dst];
      if (o.kind != EB_OP_POOL || o.res == g.dst || half < 0 || half >= parts || o.src_c != 64 ||
          pool_of[half] >= 0 || o.pool_mode != EB_POOL_MAX || o.kh != 3 || o.kw != 3 || o.sh != 2 ||
          o.sw != 2 || o.ph != 1 || o.pw != 1 || o.scale_off != EB_NO_OFFSET || e->op_skip[k] ||
          d.dtype != EB_BF16 || d.c % 8 || o.dst_c_off % 8)
        ok = false;
      else
        pool_of[half] = static_cast<int>(k);
    }
    for (const auto& m : e->members)
      if (m.tensor == g.dst) ok = false;
    if (!ok || pool_of[0] < 0 || (parts == 2 && pool_of[1] < 0)) continue;
    e->op_stempool[i] = {pool_of[0], pool_of[1]};
    for (int h = 0; h < parts; ++h) e->stempool_pool[pool_of[h]] = 1;
  }
}

void fuse_block1(eb_engine* e) {
  const size_t n = e->ops.size();
  e->op_block1.assign(n, -1);
  e->block1_stem.assign(n, 0);
  if (!env_flag("EB_BLOCK1", true) || !stem_rows_enabled() || e->f32) return;
  for (size_t i = 0; i + 1 < n; ++i) {
    const eb_op_desc& sop = e->ops[i];
    const eb_op_desc& c = e->ops[i + 1];
    if (sop.kind != EB_OP_CONV || c.kind != EB_OP_CONV || e->op_skip[i] || e->op_pool[i] >= 0 ||
        e->op_pool[i + 1] < 0 || c.src != sop.dst || c.stream != sop.stream || is_prefork(sop))
      continue;
    const Tensor& src = e->tensors[sop.src];
    const Tensor& mid = e->tensors[sop.dst];
    if (!(src.c == 8 && sop.src_c == 8 && sop.src_c_off == 0) || sop.kh != 3 || sop.kw != 3 ||
        sop.sh != 1 || sop.sw != 1 || sop.ph != 1 || sop.pw != 1 || sop.cout != 64 || !sop.relu ||
        sop.res >= 0 || sop.groups > 1 || sop.n_split || sop.flatten || sop.scale_off != EB_NO_OFFSET ||
        sop.b_off == EB_NO_OFFSET || sop.dst_c_off != 0 || mid.c != 64 || mid.dtype != EB_BF16)
      continue;
    if (c.cout != 64 || c.src_c != 64 || c.src_c_off != 0 || !c.relu || c.b_off == EB_NO_OFFSET ||
        mid.h % 2 || mid.w % 2 || mid.h < 28)
      continue;
    bool other = false;  // the conv1_1 output has no other reader
    for (size_t k = 0; k < n; ++k)
      if (k != i + 1 && (e->ops[k].src == sop.dst || e->ops[k].res == sop.dst)) other = true;
    for (const auto& m : e->members)
      if (m.tensor == sop.dst) other = true;
    if (other) continue;
    e->op_block1[i + 1] = static_cast<int>(i);
    e->block1_stem[i] = 1;
    ++i;
  }
}
}  // namespace

int eb_finalize(eb_engine* e) {
  if (!e || e->finalized) EB_FAIL(EB_E_STATE, "engine already finalized");
  if (e->members.empty()) EB_FAIL(EB_E_INVALID, "no members");
  if (!e->have_pre) EB_FAIL(EB_E_STATE, "preprocess not set");
  cudaSetDevice(e->device);
  const int mb = e->max_batch;
  fuse_conv_pools(e);
  if (e->f32) {  // the fp32 kernels take every op as declared
    e->op_pool.assign(e->ops.size(), -1);
    e->op_skip.assign(e->ops.size(), 0);
  }
  fuse_block1(e);
  fuse_stem_pools(e);
  std::vector<uint8_t> t_read(e->tensors.size(), 0);  // tensors some op or member reads
  for (size_t i = 0; i < e->ops.size(); ++i) {
    if (e->op_skip[i]) continue;
    const eb_op_desc& op = e->ops[i];
    t_read[op.src] = 1;
    if (op.res >= 0) t_read[op.res] = 1;
  }
  for (const auto& m : e->members) t_read[m.tensor] = 1;
  for (size_t i = 0; i < e->tensors.size(); ++i) {
    Tensor& t = e->tensors[i];
    // a fused conv's full-resolution output is never materialised
    bool absorbed = false;
    for (size_t k = 0; k < e->ops.size(); ++k)
      if (e->op_pool[k] >= 0 && e->ops[k].dst == static_cast<int>(i)) absorbed = true;
    if (absorbed && !t_read[i]) continue;
    if (i == EB_T_IMAGE_NHWC8 && !e->any_cnn) continue;
    if (i == EB_T_IMAGE_F32 && !e->any_lin) continue;
    const size_t bytes = static_cast<size_t>(mb) * t.h * t.w * t.c * dsize(t.dtype);
    if (cudaMalloc(&t.dev, bytes) != cudaSuccess) {
      cudaGetLastError();
      EB_FAIL(EB_E_NOMEM, "activation arena allocation failed");
    }
    EB_CUDA(cudaMemset(t.dev, 0, bytes));
  }
  const size_t img = static_cast<size_t>(mb) * e->C * e->H * e->W;
  EB_CUDA(cudaMalloc(&e->d_in_u8, img));
  EB_CUDA(cudaMalloc(&e->d_in_f32, img * sizeof(float)));
  if (stem_rows_enabled() && !e->f32) {
    for (const auto& op : e->ops) {
      if (op.kind != EB_OP_CONV) continue;
      const Tensor& src = e->tensors[op.src];
      StemGeom g;
      if (!(src.c == 8 && op.src_c == 8 && op.src_c_off == 0)) continue;
      if (!stem_geom(mb, src.h, src.w, op.kh, op.kw, op.sh, op.sw, op.ph, op.pw, &g)) continue;
      void* buf = nullptr;
      if (cudaMalloc(&buf, static_cast<size_t>(g.bytes)) != cudaSuccess) {
        cudaGetLastError();
        EB_FAIL(EB_E_NOMEM, "stem layout allocation failed");
      }
      e->stem_buf[&op] = buf;
    }
  }
  e->img8_needed = false;
  for (const auto& op : e->ops)
    if (op.src == EB_T_IMAGE_NHWC8 && !e->stem_buf.count(&op)) e->img8_needed = true;
  // split-K partial slices per lane: the largest split layer at max_batch (split counts
  // are a function of the layer shape only, plan_conv)
  for (size_t i = 0; i < e->ops.size(); ++i) {
    const eb_op_desc& op = e->ops[i];
    if (op.kind != EB_OP_CONV || e->op_skip[i] || e->f32) continue;
    ConvArgs a{};
    const void* rd = nullptr;
    conv_args_for(e, op, mb, e->op_pool[i], &a, &rd);
    ConvPlan pl;
    const int rc = plan_conv(a, &pl);
    if (rc != EB_OK) return rc;
    e->ws_floats[op.stream] = std::max(e->ws_floats[op.stream], pl.ws_floats);
  }
  for (int l = 0; l < kLanes; ++l)
    if (e->ws_floats[l] > 0 && cudaMalloc(&e->ws[l], e->ws_floats[l] * sizeof(float)) != cudaSuccess) {
      cudaGetLastError();
      EB_FAIL(EB_E_NOMEM, "split-K workspace allocation failed");
    }
  // LIN1 d-slices: a function of D only (never of the batch); models.lin1_splits.
  int64_t lin_k = 0;
  for (const auto& op : e->ops)
    if (op.kind == EB_OP_LIN1) lin_k = std::max<int64_t>(lin_k, op.cout);
  if (lin_k > 0) {
    const int64_t D = static_cast<int64_t>(e->C) * e->H * e->W;
    const int64_t ns = std::max<int64_t>(1, std::min<int64_t>(148, D / 1024));
    e->lin_nsplit = static_cast<int>(ns);
    EB_CUDA(cudaMalloc(&e->lin_part, static_cast<size_t>(ns) * mb * lin_k * sizeof(double)));
  }
  const int n = static_cast<int>(e->members.size());
  std::vector<int> kind(n), koff(n), kcnt(n);
  for (int i = 0; i < n; ++i) {
    kind[i] = e->members[i].kind;
    koff[i] = e->members[i].koff;
    kcnt[i] = e->members[i].k;
  }
  EB_CUDA(cudaMalloc(&e->d_kind, n * sizeof(int)));
  EB_CUDA(cudaMalloc(&e->d_koff, n * sizeof(int)));
  EB_CUDA(cudaMalloc(&e->d_kcnt, n * sizeof(int)));
  EB_CUDA(cudaMemcpy(e->d_kind, kind.data(), n * sizeof(int), cudaMemcpyHostToDevice));
  EB_CUDA(cudaMemcpy(e->d_koff, koff.data(), n * sizeof(int), cudaMemcpyHostToDevice));
  EB_CUDA(cudaMemcpy(e->d_kcnt, kcnt.data(), n * sizeof(int), cudaMemcpyHostToDevice));
  EB_CUDA(cudaMalloc(&e->d_labels, static_cast<size_t>(n) * mb * sizeof(int32_t)));
  EB_CUDA(cudaMalloc(&e->d_topk_idx, static_cast<size_t>(n) * mb * e->max_topk * sizeof(int32_t)));
  EB_CUDA(cudaMalloc(&e->d_topk_prob, static_cast<size_t>(n) * mb * e->max_topk * sizeof(float)));
  EB_CUDA(cudaMalloc(&e->d_combined, static_cast<size_t>(mb) * sizeof(int32_t)));
  // The arena memsets above run on the legacy default stream, which does not order
  // against the engine's non-blocking streams: drain them before any forward.
  EB_CUDA(cudaDeviceSynchronize());
  e->finalized = true;
  return EB_OK;
}

int eb_forward_device(eb_engine* e, int input_kind, int batch, int topk, int policy,
                      int policy_k) {
  int rc = check_batch(e, batch);
  if (rc != EB_OK) return rc;
  if (input_kind != EB_IN_F32_CHW && input_kind != EB_IN_U8_HWC)
    EB_FAIL(EB_E_INVALID, "unknown input encoding");
  if (topk < 0 || topk > e->max_topk) EB_FAIL(EB_E_INVALID, "topk out of range");
  rc = check_policy(e, policy, policy_k);
  if (rc != EB_OK) return rc;
  cudaSetDevice(e->device);
  rc = run_layers(e, input_kind, batch);
  if (rc != EB_OK) return rc;
  return enqueue_combine(e, batch, topk, policy, policy_k);
}

int eb_forward(eb_engine* e, const void* host_input, int input_kind, int batch,
               int32_t* host_labels, float* host_logits, int topk, int32_t* host_topk_idx,
               float* host_topk_prob, int policy, int policy_k, int32_t* host_combined) {
  int rc = check_batch(e, batch);
  if (rc != EB_OK) return rc;
  if (!host_input || !host_labels) EB_FAIL(EB_E_INVALID, "null input/labels");
  if (topk > 0 && (!host_topk_idx || !host_topk_prob)) EB_FAIL(EB_E_INVALID, "null top-k out");
  if (policy != EB_POLICY_NONE && !host_combined) EB_FAIL(EB_E_INVALID, "null combined out");
  rc = check_policy(e, policy, policy_k);
  if (rc != EB_OK) return rc;
  std::lock_guard<std::mutex> lock(e->mu);
  cudaSetDevice(e->device);
  const size_t px = static_cast<size_t>(batch) * e->C * e->H * e->W;
  if (input_kind != EB_IN_U8_HWC && input_kind != EB_IN_F32_CHW)
    EB_FAIL(EB_E_INVALID, "unknown input encoding");
  void* d_in = input_kind == EB_IN_U8_HWC ? static_cast<void*>(e->d_in_u8) : static_cast<void*>(e->d_in_f32);
  const size_t in_bytes = input_kind == EB_IN_U8_HWC ? px : px * sizeof(float);
  static const bool staged_up = env_flag("EB_PAGEABLE_STAGING", true);
  if (staged_up && in_bytes >= (4u << 20) && is_pageable(host_input)) {
    rc = upload_pageable(e, d_in, host_input, in_bytes);
    if (rc != EB_OK) return rc;
  } else {
    EB_CUDA(cudaMemcpyAsync(d_in, host_input, in_bytes, cudaMemcpyHostToDevice, e->stream));
  }
  rc = eb_forward_device(e, input_kind, batch, topk, policy, policy_k);
  if (rc != EB_OK) return rc;
  const int n = static_cast<int>(e->members.size());
  EB_CUDA(cudaMemcpyAsync(host_labels, e->d_labels, static_cast<size_t>(n) * batch * sizeof(int32_t),
                          cudaMemcpyDeviceToHost, e->stream));
  if (topk > 0) {
    EB_CUDA(cudaMemcpyAsync(host_topk_idx, e->d_topk_idx,
                            static_cast<size_t>(n) * batch * topk * sizeof(int32_t),
                            cudaMemcpyDeviceToHost, e->stream));
    EB_CUDA(cudaMemcpyAsync(host_topk_prob, e->d_topk_prob,
                            static_cast<size_t>(n) * batch * topk * sizeof(float),
                            cudaMemcpyDeviceToHost, e->stream));
  }
  if (policy != EB_POLICY_NONE)
    EB_CUDA(cudaMemcpyAsync(host_combined, e->d_combined, static_cast<size_t>(batch) * sizeof(int32_t),
                            cudaMemcpyDeviceToHost, e->stream));
  // fp32 member logits are copied row by row into [N][B][Kmax]; LIN1 members' fp64
  // scores land in a host staging buffer and are narrowed to fp32 after the sync
  int kmax = 0;
  for (const auto& m : e->members) kmax = std::max(kmax, m.k);
  std::vector<double> l64_host;
  if (host_logits) {
    for (int i = 0; i < n; ++i) {
      const Member& m = e->members[i];
      const Tensor& t = e->tensors[m.tensor];
      if (m.kind == EB_MEMBER_CNN) {
        EB_CUDA(cudaMemcpy2DAsync(host_logits + static_cast<size_t>(i) * batch * kmax,
                                  kmax * sizeof(float),
                                  static_cast<const float*>(t.dev) + m.koff, t.c * sizeof(float),
                                  m.k * sizeof(float), batch, cudaMemcpyDeviceToHost, e->stream));
      } else if (l64_host.empty()) {
        l64_host.resize(static_cast<size_t>(batch) * t.c);
        EB_CUDA(cudaMemcpyAsync(l64_host.data(), t.dev, l64_host.size() * sizeof(double),
                                cudaMemcpyDeviceToHost, e->stream));
      }
    }
  }
  EB_CUDA(cudaStreamSynchronize(e->stream));
  if (!l64_host.empty()) {
    for (int i = 0; i < n; ++i) {
      const Member& m = e->members[i];
      if (m.kind != EB_MEMBER_LIN1) continue;
      const int ld = e->tensors[m.tensor].c;
      for (int b = 0; b < batch; ++b)
        for (int k = 0; k < m.k; ++k)
          host_logits[(static_cast<size_t>(i) * batch + b) * kmax + k] =
              static_cast<float>(l64_host[static_cast<size_t>(b) * ld + m.koff + k]);
    }
  }
  return EB_OK;
}

int eb_forward_batches(eb_engine* e, const void* const* host_inputs, int n_batches, int input_kind,
                       int batch, int32_t* const* host_labels) {
  int rc = check_batch(e, batch);
  if (rc != EB_OK) return rc;
  if (n_batches < 0 || (n_batches > 0 && (!host_inputs || !host_labels)))
    EB_FAIL(EB_E_INVALID, "null inputs/labels");
  if (input_kind != EB_IN_U8_HWC && input_kind != EB_IN_F32_CHW)
    EB_FAIL(EB_E_INVALID, "unknown input encoding");
  for (int i = 0; i < n_batches; ++i)
    if (!host_inputs[i] || !host_labels[i]) EB_FAIL(EB_E_INVALID, "null input/labels entry");
  std::lock_guard<std::mutex> lock(e->mu);
  cudaSetDevice(e->device);
  const size_t bytes = static_cast<size_t>(batch) * e->C * e->H * e->W *
                       (input_kind == EB_IN_U8_HWC ? 1 : sizeof(float));
  void* d_in = input_kind == EB_IN_U8_HWC ? static_cast<void*>(e->d_in_u8) : static_cast<void*>(e->d_in_f32);
  if (e->d_stage_bytes < bytes) {
    cudaFree(e->d_stage);
    e->d_stage = nullptr;
    e->d_stage_bytes = 0;
    const size_t cap = static_cast<size_t>(e->max_batch) * e->C * e->H * e->W * sizeof(float);
    if (cudaMalloc(&e->d_stage, cap) != cudaSuccess) {
      cudaGetLastError();
      EB_FAIL(EB_E_NOMEM, "staging buffer allocation failed");
    }
    e->d_stage_bytes = cap;
  }
  if (!e->copy_stream) {
    EB_CUDA(cudaStreamCreateWithFlags(&e->copy_stream, cudaStreamNonBlocking));

    EB_CUDA(cudaEventCreateWithFlags(&e->ev_staged, cudaEventDisableTiming));
    EB_CUDA(cudaEventCreateWithFlags(&e->ev_stage_free, cudaEventDisableTiming));
  }
  const int n = static_cast<int>(e->members.size());
  // copy stream: H2D of batch i into the staging buffer (after batch i-1 left it);
  // engine stream: staging -> input buffer, forward, D2H of labels.  So batch i+1's
  // transfer overlaps batch i's forward.
  if (n_batches > 0) {
    EB_CUDA(cudaMemcpyAsync(e->d_stage, host_inputs[0], bytes, cudaMemcpyHostToDevice, e->copy_stream));
    EB_CUDA(cudaEventRecord(e->ev_staged, e->copy_stream));
  }
  for (int i = 0; i < n_batches; ++i) {
    EB_CUDA(cudaStreamWaitEvent(e->stream, e->ev_staged, 0));
    EB_CUDA(k_copy(e->d_stage, d_in, bytes, e->stream));
    EB_CUDA(cudaEventRecord(e->ev_stage_free, e->stream));
    if (i + 1 < n_batches) {
      EB_CUDA(cudaStreamWaitEvent(e->copy_stream, e->ev_stage_free, 0));
      EB_CUDA(cudaMemcpyAsync(e->d_stage, host_inputs[i + 1], bytes, cudaMemcpyHostToDevice,
                              e->copy_stream));
      EB_CUDA(cudaEventRecord(e->ev_staged, e->copy_stream));
    }
    rc = eb_forward_device(e, input_kind, batch, 0, EB_POLICY_NONE, 0);
    if (rc != EB_OK) return rc;
    EB_CUDA(cudaMemcpyAsync(host_labels[i], e->d_labels, static_cast<size_t>(n) * batch * sizeof(int32_t),
                            cudaMemcpyDeviceToHost, e->stream));
  }
  EB_CUDA(cudaStreamSynchronize(e->stream));
  return EB_OK;
}

int eb_profile_ops(eb_engine* e, int input_kind, int batch, float* host_ms, int n_ops) {
  return eb_profile_ops_repeat(e, input_kind, batch, host_ms, n_ops, 1);
}

int eb_profile_ops_repeat(eb_engine* e, int input_kind, int batch, float* host_ms, int n_ops,
                          int repeat) {
  int rc = check_batch(e, batch);
  if (rc != EB_OK) return rc;
  if (!host_ms || n_ops != static_cast<int>(e->ops.size()))
    EB_FAIL(EB_E_INVALID, "host_ms must hold one float per op");
  if (repeat < 1 || repeat > 100) EB_FAIL(EB_E_INVALID, "repeat must be 1..100");
  std::lock_guard<std::mutex> lock(e->mu);
  cudaSetDevice(e->device);
  std::vector<cudaEvent_t> evs;
  e->prof = &evs;
  e->prof_repeat = repeat;
  int launches = 0;
  rc = enqueue_layers(e, input_kind, batch, &launches);
  e->prof = nullptr;
  e->prof_repeat = 1;
  cudaError_t ce = cudaStreamSynchronize(e->stream);
  if (rc == EB_OK && ce != cudaSuccess) {
    set_error(std::string("profile run: ") + cudaGetErrorString(ce));
    rc = EB_E_CUDA;
  }
  if (rc == EB_OK) {
    for (int i = 0; i < n_ops && i + 1 < static_cast<int>(evs.size()); ++i) {
      cudaEventElapsedTime(&host_ms[i], evs[i], evs[i + 1]);
      host_ms[i] /= static_cast<float>(repeat);
    }
  }
  for (auto ev : evs) cudaEventDestroy(ev);
  return rc;
}

int eb_engine_warmup(eb_engine* e, int input_kind, int max_b) {
  if (!e || !e->finalized) EB_FAIL(EB_E_STATE, "engine not finalized");
  if (input_kind != EB_IN_F32_CHW && input_kind != EB_IN_U8_HWC)
    EB_FAIL(EB_E_INVALID, "unknown input encoding");
  std::lock_guard<std::mutex> lock(e->mu);
  cudaSetDevice(e->device);
  const int top = (max_b > 0 && max_b < e->max_batch) ? max_b : e->max_batch;
  int last = 0;
  for (int b = 1; b <= top; ++b) {
    const int q = bucket_of(e, b);
    if (q == last) continue;
    last = q;
    const int rc = run_layers(e, input_kind, q);
    if (rc != EB_OK) return rc;
  }
  EB_CUDA(cudaStreamSynchronize(e->stream));
  return EB_OK;
}

int eb_input_buffer(eb_engine* e, int input_kind, void** dev_ptr) {
  if (!e || !dev_ptr || !e->finalized) EB_FAIL(EB_E_STATE, "engine not finalized");
  *dev_ptr = input_kind == EB_IN_U8_HWC ? static_cast<void*>(e->d_in_u8)
                                        : static_cast<void*>(e->d_in_f32);
  return EB_OK;
}

int eb_output_labels(eb_engine* e, int32_t** dev_labels) {
  if (!e || !dev_labels || !e->finalized) EB_FAIL(EB_E_STATE, "engine not finalized");
  *dev_labels = e->d_labels;
  return EB_OK;
}

int eb_tensor_ptr(eb_engine* e, int id, void** dev_ptr, int* h, int* w, int* c, int* dtype) {
  if (!e || id < 0 || id >= static_cast<int>(e->tensors.size()))
    EB_FAIL(EB_E_INVALID, "bad tensor id");
  const Tensor& t = e->tensors[id];
  if (dev_ptr) *dev_ptr = t.dev;
  if (h) *h = t.h;
  if (w) *w = t.w;
  if (c) *c = t.c;
  if (dtype) *dtype = t.dtype;
  return EB_OK;
}

int eb_engine_stream(eb_engine* e, void** stream) {
  if (!e || !stream) EB_FAIL(EB_E_INVALID, "null argument");
  *stream = e->stream;
  return EB_OK;
}

int eb_launch_count(eb_engine* e, int input_kind, int batch, int* count) {
  if (!e || !count) EB_FAIL(EB_E_INVALID, "null argument");
  auto it = e->launch_counts.find(std::make_pair(bucket_of(e, batch), input_kind));
  if (it == e->launch_counts.end()) EB_FAIL(EB_E_STATE, "no graph captured for this batch");
  *count = it->second + 1;  // + combine
  return EB_OK;
}

// ------------------------------------------------------------------ kernel-level ABI

int eb_k_preprocess_f32(const float* dev_x, float* dev_y, int batch, int c, int64_t plane,
                        const float* dev_mean, const float* dev_std, int n, void* stream) {
  EB_CUDA(k_preprocess_f32(dev_x, dev_y, batch, c, plane, dev_mean, dev_std, n,
                           static_cast<cudaStream_t>(stream)));
  return EB_OK;
}

int eb_k_preprocess_u8_nhwc8(const uint8_t* dev_x, void* dev_y_bf16, int batch, int c,
                             int64_t plane, const float* dev_lut, void* stream) {
  if (c < 1 || c > 8) EB_FAIL(EB_E_INVALID, "channels must be 1..8");
  EB_CUDA(k_preprocess_u8hwc_to_nhwc(dev_x, static_cast<__nv_bfloat16*>(dev_y_bf16), batch, c,
                                     plane, 8, dev_lut, static_cast<cudaStream_t>(stream)));
  return EB_OK;
}

namespace {
int k_conv_abi(const void* dev_x, int batch, int h, int w, int ldx, int cin, const void* dev_w,
               const float* dev_bias, const void* dev_res, int ldr, void* dev_y, int ldy,
               int y_off, int cout, int kh, int kw, int sh, int sw, int ph, int pw, int relu,
               int out_f32, int c8_stem, int split_k, int block_n, int groups,
               void* dev_workspace, const float* dev_pre_scale, const float* dev_pre_shift,
               void* stream, int pool2) {
  ConvArgs a{};
  a.pool2 = pool2;
  a.groups = groups > 1 ? groups : 1;
  a.pre_scale = dev_pre_scale;
  a.pre_shift = dev_pre_shift;
  a.x = dev_x;
  a.B = batch;
  a.H = h;
  a.W = w;
  a.ldx = ldx;
  a.cin = cin;
  a.w = dev_w;
  a.bias = dev_bias;
  a.res = dev_res;
  a.ldr = ldr;
  a.y = dev_y;
  a.ldy = ldy;
  a.y_off = y_off;
  a.cout = cout;
  a.kh = kh;
  a.kw = kw;
  a.sh = sh;
  a.sw = sw;
  a.ph = ph;
  a.pw = pw;
  a.relu = relu;
  a.out_f32 = out_f32;
  a.c8_stem = c8_stem;
  a.flatten = 0;
  a.split_k = split_k;
  a.block_n = block_n;
  set_pdl_batch(batch);  // (same PDL policy as the engine)
  ConvPlan pl;
  int rc = plan_conv(a, &pl);
  if (rc != EB_OK) return rc;
  if (env_flag("EB_DEBUG_PLAN", false))
    fprintf(stderr, "[eb] conv mode=%d bn=%d grid=%d splits=%d M=%d N=%d kb=%d kbs=%d cl=%d pair=%d resb=%d stages=%d\n",
            pl.p.a_mode, pl.block_n, pl.grid, pl.splits, pl.p.M, pl.p.N, pl.p.num_kb, pl.p.kbs, pl.p.mcast,
            pl.p.pair, pl.p.resb, conv_umma_stages(pl.p, pl.block_n));
  // EB_TRACE=<file>: timing probe (per-role event clocks of CTA 0, appended as text)
  static const char* trace_path = getenv("EB_TRACE");
  constexpr size_t kTraceLongs = 3 * 1024 * 2 + 1024 * 4;
  static long long* d_trace = nullptr;
  if (trace_path) {
    if (!d_trace) EB_CUDA(cudaMalloc(&d_trace, kTraceLongs * sizeof(long long)));
    EB_CUDA(cudaMemset(d_trace, 0, kTraceLongs * sizeof(long long)));
    pl.p.trace = d_trace;
  }
  rc = run_conv_plan(pl, static_cast<float*>(dev_workspace), kSplitWsFloats, a,
                     static_cast<cudaStream_t>(stream), nullptr);
  if (rc == EB_OK && trace_path) {
    std::vector<long long> h(kTraceLongs);
    EB_CUDA(cudaMemcpy(h.data(), d_trace, h.size() * sizeof(long long), cudaMemcpyDeviceToHost));
    if (FILE* f = fopen(trace_path, "w")) {
      for (int r = 0; r < 3; ++r)
        for (int i = 0; i < 1024; ++i) {
          const long long v = h[(r * 1024 + i) * 2];
          if (v == 0) break;
          fprintf(f, "%d %lld %lld %lld\n", r, v >> 48, v & 0xFFFFFFFFFFFFll, h[(r * 1024 + i) * 2 + 1]);
        }
      // CTA spans: "3 <cta> <entry ns> <prologue done ns> <exit ns>"
      for (int c = 0; c < 1024; ++c) {
        const long long* q = &h[3 * 1024 * 2 + c * 4];
        if (q[0] == 0) break;
        fprintf(f, "3 %d %lld %lld %lld\n", c, q[0], q[1], q[2]);
      }
      fclose(f);
    }
  }
  return rc;
}
}  // namespace

int eb_k_conv(const void* dev_x, int batch, int h, int w, int ldx, int cin, const void* dev_w,
              const float* dev_bias, const void* dev_res, int ldr, void* dev_y, int ldy,
              int y_off, int cout, int kh, int kw, int sh, int sw, int ph, int pw, int relu,
              int out_f32, int c8_stem, int split_k, int block_n, int groups,
              void* dev_workspace, const float* dev_pre_scale, const float* dev_pre_shift,
              void* stream) {
  return k_conv_abi(dev_x, batch, h, w, ldx, cin, dev_w, dev_bias, dev_res, ldr, dev_y, ldy, y_off,
                    cout, kh, kw, sh, sw, ph, pw, relu, out_f32, c8_stem, split_k, block_n, groups,
                    dev_workspace, dev_pre_scale, dev_pre_shift, stream, 0);
}

int eb_k_conv_maxpool2(const void* dev_x, int batch, int h, int w, int ldx, int cin,
                       const void* dev_w, const float* dev_bias, void* dev_y, int ldy, int y_off,
                       int cout, int kh, int kw, int ph, int pw, int relu, void* stream) {
  return k_conv_abi(dev_x, batch, h, w, ldx, cin, dev_w, dev_bias, nullptr, 0, dev_y, ldy, y_off,
                    cout, kh, kw, 1, 1, ph, pw, relu, 0, 0, 0, 0, 1, nullptr, nullptr, nullptr,
                    stream, 1);
}

int eb_k_resize(const void* dev_x, int ldx, void* dev_y, int ldy, int batch, int h, int w, int c,
                int ho, int wo, void* stream) {
  EB_CUDA(k_resize_bilinear(static_cast<const __nv_bfloat16*>(dev_x), ldx,
                            static_cast<__nv_bfloat16*>(dev_y), ldy, batch, h, w, c, ho, wo,
                            static_cast<cudaStream_t>(stream)));
  return EB_OK;
}

int eb_k_stem_layout(int batch, int h, int w, int kh, int kw, int sh, int sw, int ph, int pw,
                     uint64_t* bytes) {
  StemGeom g;
  if (!stem_geom(batch, h, w, kh, kw, sh, sw, ph, pw, &g)) EB_FAIL(EB_E_INVALID, "no stem layout");
  if (bytes) *bytes = static_cast<uint64_t>(g.bytes);
  return EB_OK;
}

int eb_k_stem_relayout(const void* dev_x, int batch, int h, int w, int kh, int kw, int sh, int sw,
                       int ph, int pw, void* dev_y, void* stream) {
  StemGeom g;
  if (!stem_geom(batch, h, w, kh, kw, sh, sw, ph, pw, &g)) EB_FAIL(EB_E_INVALID, "no stem layout");
  EB_CUDA(k_stem_relayout(static_cast<const __nv_bfloat16*>(dev_x), batch, h, w, ph, pw, g.mode,
                          g.Hq, g.Wq, static_cast<__nv_bfloat16*>(dev_y),
                          static_cast<cudaStream_t>(stream)));
  return EB_OK;
}

int eb_k_preprocess_u8_layout(const uint8_t* dev_x, int batch, int c, int h, int w,
                              const float* dev_lut, int kh, int kw, int sh, int sw, int ph, int pw,
                              void* dev_y, void* stream) {
  StemGeom g;
  if (c < 1 || c > 8) EB_FAIL(EB_E_INVALID, "1..8 channels");
  if (!stem_geom(batch, h, w, kh, kw, sh, sw, ph, pw, &g)) EB_FAIL(EB_E_INVALID, "no stem layout");
  EB_CUDA(k_preprocess_u8_to_layout(dev_x, batch, c, h, w, dev_lut, ph, pw, g.mode, g.Hq, g.Wq,
                                    static_cast<__nv_bfloat16*>(dev_y),
                                    static_cast<cudaStream_t>(stream)));
  return EB_OK;
}

int eb_k_pool(const void* dev_x, int ldx, void* dev_y, int ldy, int y_off, int batch, int h,
              int w, int c, int k, int s, int pad, int mode, const float* dev_scale,
              const float* dev_shift, void* stream) {
  const int Ho = conv_out(h, k, s, pad), Wo = conv_out(w, k, s, pad);
  EB_CUDA(k_pool(static_cast<const __nv_bfloat16*>(dev_x), ldx, static_cast<__nv_bfloat16*>(dev_y),
                 ldy, y_off, batch, h, w, c, Ho, Wo, k, s, pad, mode, dev_scale, dev_shift,
                 static_cast<cudaStream_t>(stream)));
  return EB_OK;
}

int eb_k_gap(const void* dev_x, int ldx, void* dev_y, int batch, int hw, int c,
             const float* dev_scale, const float* dev_shift, void* stream) {
  EB_CUDA(k_gap(static_cast<const __nv_bfloat16*>(dev_x), ldx, static_cast<__nv_bfloat16*>(dev_y),
                batch, hw, c, dev_scale, dev_shift, static_cast<cudaStream_t>(stream)));
  return EB_OK;
}

int eb_k_lin1(const float* dev_x, const float* dev_w, const float* dev_bias, double* dev_part,
              double* dev_logits, int batch, int k, int64_t d, int nsplit, void* stream) {
  EB_CUDA(k_lin1(dev_x, dev_w, dev_bias, dev_part, dev_logits, batch, k, d, nsplit,
                 static_cast<cudaStream_t>(stream)));
  return EB_OK;
}

int eb_k_combine(const float* dev_l32, int ld32, const double* dev_l64, int ld64,
                 const int* dev_kind, const int* dev_koff, const int* dev_kcnt, int n, int batch,
                 int32_t* dev_labels, int topk, int32_t* dev_topk_idx, float* dev_topk_prob,
                 int policy, int policy_k, int32_t* dev_combined, void* stream) {
  EB_CUDA(k_combine(dev_l32, ld32, dev_l64, ld64, dev_kind, dev_koff, dev_kcnt, n, batch,
                    dev_labels, topk, dev_topk_idx, dev_topk_prob, policy, policy_k,
                    dev_combined, static_cast<cudaStream_t>(stream)));
  return EB_OK;
}

}  // extern "C"
