// combine.cu -- K5 (per-member argmax / softmax / top-k + ensemble policy) and
// K6 (LIN1 members: fp64 linear scores).
#include <cuda_runtime.h>

#include <cstdint>

#include "eb_kernels.h"

namespace eb {

// ------------------------------------------------------------------ K5 combine
//
// One warp per (sample, member) row.  Per row:
//   label  = argmax over the member's K logits, lowest index on ties
//            (np.argmax semantics, eg/models.py:279)
//   top-k  = indices ordered by (logit desc, index asc), with softmax
//            probabilities computed in fp32 from the logits
// Then (policy requests only) a second pass applies the sensitivity policy over the N
// binary votes of each sample (eg/policy.py:66-76): any = max, all = min, at_least =
// count >= k.

template <typename T>
__device__ __forceinline__ bool better(T v, int i, T bv, int bi) {
  return v > bv || (v == bv && i < bi);
}

template <typename T>
__device__ void warp_argmax_excluding(const T* row, int K, bool have_prev, T pv, int pi, T* out_v,
                                      int* out_i) {
  T bv = 0;
  int bi = -1;
  for (int i = threadIdx.x & 31; i < K; i += 32) {
    const T v = row[i];
    // candidates strictly after (pv, pi) in (value desc, index asc) order
    if (have_prev && !(v < pv || (v == pv && i > pi))) continue;
    if (bi < 0 || better(v, i, bv, bi)) {
      bv = v;
      bi = i;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const T ov = __shfl_xor_sync(0xffffffffu, bv, off);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
    if (oi >= 0 && (bi < 0 || better(ov, oi, bv, bi))) {
      bv = ov;
      bi = oi;
    }
  }
  *out_v = bv;
  *out_i = bi;
}

template <typename T>
__device__ void member_outputs(const T* row, int K, int lane, int mem, int B, int b,
                               int32_t* labels, int* s_lab, int topk, int32_t* topk_idx,
                               float* topk_prob) {
  T bv;
  int bi;
  warp_argmax_excluding(row, K, false, T(0), 0, &bv, &bi);
  if (lane == 0) {
    labels[static_cast<int64_t>(mem) * B + b] = bi;
    if (s_lab) s_lab[mem] = bi;
  }
  if (topk > 0) {
    // softmax denominator in fp32, max-subtracted
    const float mx = static_cast<float>(bv);
    float sum = 0.f;
    for (int i = lane; i < K; i += 32) sum += __expf(static_cast<float>(row[i]) - mx);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
    const float inv = 1.f / sum;
    T pv = bv;
    int pi = bi;
    const int64_t base = (static_cast<int64_t>(mem) * B + b) * topk;
    for (int j = 0; j < topk; ++j) {
      T v = pv;
      int idx = pi;
      if (j > 0) warp_argmax_excluding(row, K, true, pv, pi, &v, &idx);
      if (lane == 0) {
        topk_idx[base + j] = idx;
        topk_prob[base + j] = (idx >= 0) ? __expf(static_cast<float>(v) - mx) * inv : 0.f;
      }
      pv = v;
      pi = idx;
    }
  }
}

// Fast path for fp32 members with K <= 32 * VPL: the warp reads the row ONCE into
// registers (lane l holds elements l, l + 32, ...; each load instruction is one
// coalesced 128-byte line), then argmax, the softmax denominator and the top-k rounds
// all run on registers.  Each top-k round: every lane offers its best remaining
// (value, index), a 5-step shuffle reduction picks the winner (value desc, index asc),
// and the owning lane retires that slot.
template <int VPL>
__device__ void member_outputs_reg(const float* row, int K, int lane, int mem, int B, int b,
                                   int32_t* labels, int* s_lab, int topk, int32_t* topk_idx,
                                   float* topk_prob) {
  float v[VPL];
#pragma unroll
  for (int j = 0; j < VPL; ++j) {
    const int i = lane + 32 * j;
    v[j] = i < K ? __ldg(row + i) : -INFINITY;
  }
  auto local_best = [&](float& bv, int& bj) {
    bv = v[0];
    bj = 0;
#pragma unroll
    for (int j = 1; j < VPL; ++j)
      if (v[j] > bv) {  // strict: equal values keep the lower j (= lower index)
        bv = v[j];
        bj = j;
      }
  };
  auto warp_best = [&](float bv, int bi, float& wv, int& wi) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (oi >= 0 && (bi < 0 || ov > bv || (ov == bv && oi < bi))) {
        bv = ov;
        bi = oi;
      }
    }
    wv = bv;
    wi = bi;
  };
  float bv;
  int bj;
  local_best(bv, bj);
  int bi = (bv == -INFINITY) ? -1 : lane + 32 * bj;
  float wv;
  int wi;
  warp_best(bv, bi, wv, wi);
  if (lane == 0) {
    labels[static_cast<int64_t>(mem) * B + b] = wi;
    if (s_lab) s_lab[mem] = wi;
  }
  if (topk <= 0) return;
  const float mx = wv;
  float sum = 0.f;
#pragma unroll
  for (int j = 0; j < VPL; ++j)
    if (lane + 32 * j < K) sum += __expf(v[j] - mx);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
  const float inv = 1.f / sum;
  const int64_t base = (static_cast<int64_t>(mem) * B + b) * topk;
  for (int r = 0; r < topk; ++r) {
    if (lane == 0) {
      topk_idx[base + r] = wi;
      topk_prob[base + r] = (wi >= 0) ? __expf(wv - mx) * inv : 0.f;
    }
    if (r + 1 == topk) break;
    if (wi >= 0 && (wi & 31) == lane) {  // the winner retires its slot
      const int wj = wi >> 5;
#pragma unroll
      for (int j = 0; j < VPL; ++j)
        if (j == wj) v[j] = -INFINITY;
      local_best(bv, bj);
      bi = (bv == -INFINITY) ? -1 : lane + 32 * bj;
    }
    warp_best(bv, bi, wv, wi);
  }
}

// Monotone map float -> uint32 (a < b  <=>  key(a) < key(b) for non-NaN values).
__device__ __forceinline__ uint32_t ord_key(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord_value(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}
// 2^x on the SFU (MUFU.EX2, flush-to-zero): the softmax terms; x <= 0 here.
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// fp32 rows with K <= 1024, K % 4 == 0 and 16-byte aligned rows: the row is read with
// 16-byte loads, 8 per lane (lane l holds elements 128 j + 4 l + e, j < 8, e < 4 --
// each load instruction of the warp is 512 contiguous bytes).  One pass over a lane's 32
// registers keeps its best and second-best (value desc, index asc: slots are visited in
// increasing index order with strict '>'); the softmax denominator is a second pass (one
// ex2 per element).  Warp-wide best: two redux.sync (max of a monotone unsigned image of
// the value, then min index among the lanes holding it).  Top-k round r: every lane
// offers its current best, the winning lane promotes its second-best -- and only if it
// wins again does it rescan its registers for the element after it (rare: the top-5 of a
// row rarely share a lane).  ncu (B = 4096, 3 x 1000 logits): 1750 -> 850 instructions per
// row, 36 -> 20.6 us (a variant that prunes candidates below the k-th largest lane maximum
// executed as many instructions and ran 22 us).
__device__ void member_outputs_vec(const float* row, int K, int lane, int mem, int B, int b,
                                   int32_t* labels, int topk, int32_t* topk_idx,
                                   float* topk_prob) {
  float v[32];
  const float4* row4 = reinterpret_cast<const float4*>(row);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int i0 = 128 * j + 4 * lane;
    float4 q = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
    if (i0 < K) q = __ldg(row4 + 32 * j + lane);
    v[4 * j + 0] = q.x;
    v[4 * j + 1] = q.y;
    v[4 * j + 2] = q.z;
    v[4 * j + 3] = q.w;
  }
  auto idx_of = [&](int slot) { return 128 * (slot >> 2) + 4 * lane + (slot & 3); };
  // best / second-best slot of this lane
  float b1 = v[0], b2 = -INFINITY;
  int s1 = 0, s2 = -1;
#pragma unroll
  for (int t = 1; t < 32; ++t) {
    const float x = v[t];
    if (x > b1) {
      b2 = b1;
      s2 = s1;
      b1 = x;
      s1 = t;
    } else if (x > b2) {
      b2 = x;
      s2 = t;
    }
  }
  auto warp_best = [&](float bv, int bi, float& wv, int& wi) {
    const uint32_t key = ord_key(bv + 0.f);  // (+0.f: -0 ties with +0, as in np.argmax)
    const uint32_t kmax = __reduce_max_sync(0xffffffffu, key);
    const uint32_t cand = (key == kmax && bi >= 0) ? static_cast<uint32_t>(bi) : 0xffffffffu;
    const uint32_t imin = __reduce_min_sync(0xffffffffu, cand);
    wv = ord_value(kmax);
    wi = imin == 0xffffffffu ? -1 : static_cast<int>(imin);
  };
  int i1 = b1 == -INFINITY ? -1 : idx_of(s1);
  float wv;
  int wi;
  warp_best(b1, i1, wv, wi);
  if (lane == 0) labels[static_cast<int64_t>(mem) * B + b] = wi;
  if (topk <= 0) return;
  const float l2e = 1.4426950408889634f;
  const float mxl = wv * l2e;
  float sum = 0.f;
#pragma unroll
  for (int t = 0; t < 32; ++t) sum += ex2_approx(fmaf(v[t], l2e, -mxl));  // (-inf slots add 0)
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
  const float inv = 1.f / sum;
  int my_idx = -1;
  float my_prob = 0.f;
  bool have2 = true;  // b2/s2 hold this lane's next element
  for (int r = 0; r < topk; ++r) {
    if (r == lane) {
      my_idx = wi;
      my_prob = wi >= 0 ? ex2_approx(fmaf(wv, l2e, -mxl)) * inv : 0.f;
    }
    if (r + 1 == topk) break;
    if (wi >= 0 && wi == i1) {  // this lane won: promote its next element
      if (!have2) {
        // rescan: the best element strictly after (b1, i1) in (value desc, index asc)
        float nb = -INFINITY;
        int ns = -1;
#pragma unroll
        for (int t = 0; t < 32; ++t) {
          const float x = v[t];
          const int it = idx_of(t);
          const bool after = x < b1 || (x == b1 && it > i1);
          if (after && (ns < 0 || x > nb)) {
            nb = x;
            ns = t;
          }
        }
        b2 = nb;
        s2 = ns;
      }
      b1 = b2;
      i1 = (s2 < 0 || b2 == -INFINITY) ? -1 : idx_of(s2);
      have2 = false;
    }
    warp_best(b1, i1, wv, wi);
  }
  if (lane < topk) {
    const int64_t base = (static_cast<int64_t>(mem) * B + b) * topk;
    topk_idx[base + lane] = my_idx;
    topk_prob[base + lane] = my_prob;
  }
}

// One warp per (sample, member) row, 8 rows per CTA (rows of one sample adjacent).
// Member m reads logits from the fp32 buffer (CNN members) when kind[m] == 0, else
// from the fp64 buffer (LIN1 members); koff[m] is its column offset.
__global__ void __launch_bounds__(256, 4)
    combine_rows_kernel(const float* __restrict__ l32, int ld32, const double* __restrict__ l64,
                        int ld64, const int* __restrict__ kind, const int* __restrict__ koff,
                        const int* __restrict__ kcnt, int N, int B, int32_t* labels, int topk,
                        int32_t* topk_idx, float* topk_prob) {
  const int lane = threadIdx.x & 31;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (r >= static_cast<int64_t>(B) * N) return;
  const int b = static_cast<int>(r / N);
  const int mem = static_cast<int>(r - static_cast<int64_t>(b) * N);
  const int K = kcnt[mem];
  if (kind[mem] == 0) {
    const float* row = l32 + static_cast<int64_t>(b) * ld32 + koff[mem];
    if (K <= 1024 && (K & 3) == 0 && (reinterpret_cast<uintptr_t>(row) & 15) == 0)
      member_outputs_vec(row, K, lane, mem, B, b, labels, topk, topk_idx, topk_prob);
    else if (K <= 1024)
      member_outputs_reg<32>(row, K, lane, mem, B, b, labels, nullptr, topk, topk_idx, topk_prob);
    else
      member_outputs(row, K, lane, mem, B, b, labels, nullptr, topk, topk_idx, topk_prob);
  } else {
    member_outputs(l64 + static_cast<int64_t>(b) * ld64 + koff[mem], K, lane, mem, B, b, labels,
                   nullptr, topk, topk_idx, topk_prob);
  }
}

// The sensitivity policy over the N binary votes of each sample (eg/policy.py:66-76):
// any = max, all = min, at_least = count >= k.
__global__ void policy_kernel(const int32_t* __restrict__ labels, int N, int B, int policy,
                              int policy_k, int32_t* __restrict__ combined) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  int lo = 1, hi = 0, sum = 0;
  for (int mem = 0; mem < N; ++mem) {
    const int v = labels[static_cast<int64_t>(mem) * B + b];
    lo = min(lo, v);
    hi = max(hi, v);
    sum += v;
  }
  int out = 0;
  if (policy == 1) out = hi;             // any
  else if (policy == 2) out = lo;        // all
  else out = (sum >= policy_k) ? 1 : 0;  // at_least
  combined[b] = out;
}

cudaError_t k_combine(const float* l32, int ld32, const double* l64, int ld64, const int* kind,
                      const int* koff, const int* kcnt, int N, int B, int32_t* labels, int topk,
                      int32_t* topk_idx, float* topk_prob, int policy, int policy_k,
                      int32_t* combined, cudaStream_t s) {
  if (B == 0 || N == 0) return cudaSuccess;
  const int64_t rows = static_cast<int64_t>(B) * N;
  combine_rows_kernel<<<static_cast<unsigned>((rows + 7) / 8), 256, 0, s>>>(
      l32, ld32, l64, ld64, kind, koff, kcnt, N, B, labels, topk, topk_idx, topk_prob);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || policy <= 0) return e;
  policy_kernel<<<(B + 255) / 256, 256, 0, s>>>(labels, N, B, policy, policy_k, combined);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K6 LIN1 scores
//
// logits[b, k] = sum_d f64(x[b, d]) * f64(W[k, d])  (+ bias[k] afterwards),
// eg/models.py:275-278.  Products of two fp32 values are exact in fp64, so the
// only rounding is in the summation.  The d range is cut into `nsplit` fixed
// slices that depend on D only; each slice is summed in a fixed order (below), and
// slices are added in ascending order by the reduce kernel.  A
// sample's logits are therefore bitwise independent of the batch it arrives in
// (the reference's batch == concatenated singles property, eg/models.py:273-274).

// Small sum-K (binary members: 2 per member): one warp per sample and d-slice; lane l sums
// d = d0 + l, d0 + l + 32, ... of the slice in ascending order for every k, then a fixed
// shuffle tree adds the 32 lane sums (lane 0's result is kept) -- deterministic and a
// function of D only.  x is read once, coalesced; the 8 warps of a CTA (8 samples) share
// the slice of W through L1.  KS = sum K is a template value (no predication, the K
// weight rows' addresses hoisted out of the d loop).
constexpr int kLinSmallK = 16;
constexpr int kLinSmallChunk = 256;
// SPW samples per warp (8 warps: 8 * SPW samples per CTA): each fp64 weight read from
// shared memory feeds SPW FMAs (B200, B = 256, D = 150528, sum K = 6: SPW 1 / 2 / 4 =
// 116 / 124 / 113 us -- fp64-FMA bound; the first version without the fp64 weight stage
// and with predicated K ran 961 us)
template <int KS, int SPW>
__global__ void __launch_bounds__(256)
    lin1_small_kernel(const float* __restrict__ x, const float* __restrict__ w,
                      double* __restrict__ part, int B, int64_t D, int64_t dslice) {
  // the slice's weights, converted to fp64 once per CTA (not once per sample), chunk by chunk
  __shared__ double sw[KS][kLinSmallChunk];
  const int lane = threadIdx.x & 31;
  const int bw = (blockIdx.x * 8 + (threadIdx.x >> 5)) * SPW;  // the warp's first sample
  const int64_t d0 = blockIdx.y * dslice;
  const int n = static_cast<int>((d0 + dslice < D ? d0 + dslice : D) - d0);
  double acc[SPW][KS];
#pragma unroll
  for (int j = 0; j < SPW; ++j)
#pragma unroll
    for (int k = 0; k < KS; ++k) acc[j][k] = 0.0;
  const float* xb[SPW];
#pragma unroll
  for (int j = 0; j < SPW; ++j) xb[j] = x + static_cast<int64_t>(bw + j < B ? bw + j : 0) * D + d0;
  for (int c0 = 0; c0 < n; c0 += kLinSmallChunk) {
    const int cn = n - c0 < kLinSmallChunk ? n - c0 : kLinSmallChunk;
    __syncthreads();
    for (int t = threadIdx.x; t < KS * kLinSmallChunk; t += 256) {
      const int k = t / kLinSmallChunk, i = t - k * kLinSmallChunk;
      sw[k][i] = i < cn ? static_cast<double>(__ldg(w + k * D + d0 + c0 + i)) : 0.0;
    }
    __syncthreads();
    if (bw < B) {
      // all of the chunk's x loads of this lane in flight at once (8 per sample)
      float xr[SPW][kLinSmallChunk / 32];
#pragma unroll
      for (int q = 0; q < kLinSmallChunk / 32; ++q) {
        const int i = lane + 32 * q;
#pragma unroll
        for (int j = 0; j < SPW; ++j) xr[j][q] = i < cn ? __ldg(xb[j] + c0 + i) : 0.f;
      }
#pragma unroll
      for (int q = 0; q < kLinSmallChunk / 32; ++q) {
        const int i = lane + 32 * q;
#pragma unroll
        for (int k = 0; k < KS; ++k) {
          const double wv = sw[k][i];
#pragma unroll
          for (int j = 0; j < SPW; ++j) acc[j][k] = fma(static_cast<double>(xr[j][q]), wv, acc[j][k]);
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < SPW; ++j) {
    if (bw + j >= B) break;
#pragma unroll
    for (int k = 0; k < KS; ++k) {
      double v = acc[j][k];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
      if (lane == 0) part[(static_cast<int64_t>(blockIdx.y) * B + bw + j) * KS + k] = v;
    }
  }
}

// Small sum-K reduction: one warp per (b, k); lane l adds slices l, l + 32, ... in
// ascending order, a fixed shuffle tree adds the lanes, then the bias (after the sum,
// eg/models.py:278).  The order is a function of the slice count only.
__global__ void lin1_reduce_warp_kernel(const double* __restrict__ part,
                                        const float* __restrict__ bias,
                                        double* __restrict__ logits, int B, int K, int nsplit) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t total = static_cast<int64_t>(B) * K;
  if (i >= total) return;
  double s = 0.0;
  for (int z = lane; z < nsplit; z += 32) s += part[z * total + i];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
  if (lane == 0) logits[i] = s + static_cast<double>(bias[i % K]);
}

// Larger sum-K: 64 samples x 64 classes per CTA, 4 x 4 fp64 accumulators per thread, the
// slice walked in chunks of 16 d staged (transposed) in shared memory so each thread reads
// its 4 samples and 4 classes with one 16-byte load each.  Each (b, k) of a slice is summed
// in ascending d by one thread.
constexpr int kLinTB = 64, kLinTK = 64, kLinChunk = 16;
__global__ void __launch_bounds__(256)
    lin1_partial_kernel(const float* __restrict__ x, const float* __restrict__ w,
                        double* __restrict__ part, int B, int K, int64_t D, int64_t dslice) {
  __shared__ __align__(16) float sx[kLinChunk][kLinTB + 4];
  __shared__ __align__(16) float sw[kLinChunk][kLinTK + 4];
  const int tx = threadIdx.x & 15;  // class quad
  const int ty = threadIdx.x >> 4;  // sample quad
  const int b0 = blockIdx.x * kLinTB;
  const int k0 = blockIdx.y * kLinTK;
  const int64_t d0 = blockIdx.z * dslice;
  const int64_t d1 = d0 + dslice < D ? d0 + dslice : D;
  double acc[4][4] = {};
  // loader: thread t loads rows t / 16 + 16 i (i < 4), column t % 16 of the chunk
  const int lc = threadIdx.x & 15, lr = threadIdx.x >> 4;
  for (int64_t dc = d0; dc < d1; dc += kLinChunk) {
    const int64_t d = dc + lc;
    const bool dok = d < d1;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = lr + 16 * i;
      sx[lc][r] = (dok && b0 + r < B) ? __ldg(x + static_cast<int64_t>(b0 + r) * D + d) : 0.f;
      sw[lc][r] = (dok && k0 + r < K) ? __ldg(w + static_cast<int64_t>(k0 + r) * D + d) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < kLinChunk; ++c) {
      const float4 xa = *reinterpret_cast<const float4*>(&sx[c][4 * ty]);
      const float4 wa = *reinterpret_cast<const float4*>(&sw[c][4 * tx]);
      const double xv[4] = {xa.x, xa.y, xa.z, xa.w};
      const double wv[4] = {wa.x, wa.y, wa.z, wa.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(xv[i], wv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int b = b0 + 4 * ty + i;
      const int k = k0 + 4 * tx + j;
      if (b < B && k < K) part[(static_cast<int64_t>(blockIdx.z) * B + b) * K + k] = acc[i][j];
    }
}

__global__ void lin1_reduce_kernel(const double* __restrict__ part, const float* __restrict__ bias,
                                   double* __restrict__ logits, int B, int K, int nsplit) {
  const int64_t total = static_cast<int64_t>(B) * K;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int z = 0; z < nsplit; ++z) s += part[z * total + i];
    logits[i] = s + static_cast<double>(bias[i % K]);
  }
}

cudaError_t k_lin1(const float* x, const float* w, const float* bias, double* part,
                   double* logits, int B, int K, int64_t D, int nsplit, cudaStream_t s) {
  if (B == 0 || K == 0) return cudaSuccess;
  const int64_t dslice = (D + nsplit - 1) / nsplit;
  if (K <= kLinSmallK) {
    switch (K) {
#define EB_LIN_SMALL(k, spw)                                                              \
  case k:                                                                                 \
    lin1_small_kernel<k, spw><<<dim3((B + 8 * spw - 1) / (8 * spw), nsplit), 256, 0, s>>>( \
        x, w, part, B, D, dslice);                                                        \
    break;
      EB_LIN_SMALL(1, 1) EB_LIN_SMALL(2, 1) EB_LIN_SMALL(3, 1) EB_LIN_SMALL(4, 1)
      EB_LIN_SMALL(5, 1) EB_LIN_SMALL(6, 1) EB_LIN_SMALL(7, 1) EB_LIN_SMALL(8, 1)
      EB_LIN_SMALL(9, 1) EB_LIN_SMALL(10, 1) EB_LIN_SMALL(11, 1) EB_LIN_SMALL(12, 1)
      EB_LIN_SMALL(13, 1) EB_LIN_SMALL(14, 1) EB_LIN_SMALL(15, 1) EB_LIN_SMALL(16, 1)
#undef EB_LIN_SMALL
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const int64_t warps = static_cast<int64_t>(B) * K;
    lin1_reduce_warp_kernel<<<static_cast<unsigned>((warps + 7) / 8), 256, 0, s>>>(part, bias, logits,
                                                                                  B, K, nsplit);
    return cudaGetLastError();
  } else {
    dim3 grid((B + kLinTB - 1) / kLinTB, (K + kLinTK - 1) / kLinTK, nsplit);
    lin1_partial_kernel<<<grid, 256, 0, s>>>(x, w, part, B, K, D, dslice);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int64_t total = static_cast<int64_t>(B) * K;
  int g = static_cast<int>((total + 255) / 256);
  if (g > 148 * 16) g = 148 * 16;
  lin1_reduce_kernel<<<g, 256, 0, s>>>(part, bias, logits, B, K, nsplit);
  return cudaGetLastError();
}

}  // namespace eb
