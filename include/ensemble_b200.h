/* ensemble_b200.h -- C ABI of the B200-native ensemble forward path.
 *
 * This library replaces the compute behind ensemblegate's forward boundary:
 *
 *   ensemblegate.ensemble.forward(ensemble, raw) -> EnsembleOutput
 *       (pkg/src/ensemblegate/ensemble.py:232-250)
 *     = validation (ensemble.py:238-247)
 *     + preprocess once                (models.py:238-260)      -> K1
 *     + every member in manifest order (models.py:263-279)      -> K2/K3/K4 (CNN), K6 (LIN1)
 *   followed, in the gateway, by
 *     votes_from_output + apply_policy (policy.py:53-92)        -> K5
 *
 * The reference has no FFI of its own (it is pure Python/NumPy);
 * these entry points are what a ctypes binding of that boundary needs, and are
 * bound by paper_2003_01538_b200/_lib.py.
 *
 * Conventions: every function returns an eb_status; on failure a thread-local
 * message is available from eb_last_error().  No C++ exception crosses the ABI.
 * Pointers named host_* are host memory (pageable or pinned); pointers named
 * dev_* are device memory on the engine's GPU.
 */
#ifndef ENSEMBLE_B200_H
#define ENSEMBLE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  The Python wrapper maps them onto ensemblegate.errors:
 *   EB_E_EMPTY      -> EmptyBatch        (ensemble.py:239-240)
 *   EB_E_TOO_LARGE  -> BatchTooLarge     (ensemble.py:241-242)
 *   EB_E_SHAPE      -> ShapeMismatch     (ensemble.py:243-247)
 *   EB_E_POLICY     -> PolicyUnavailable (policy.py:88-91)
 *   EB_E_BAD_K      -> BadK              (policy.py:74-75)
 *   anything else   -> a generic internal error (gateway.py:85-88: never leaked) */
typedef enum {
  EB_OK = 0,
  EB_E_INVALID = 1,
  EB_E_CUDA = 2,
  EB_E_SHAPE = 3,
  EB_E_EMPTY = 4,
  EB_E_TOO_LARGE = 5,
  EB_E_POLICY = 6,
  EB_E_BAD_K = 7,
  EB_E_NOMEM = 8,
  EB_E_STATE = 9
} eb_status;

/* Input encodings accepted by eb_forward. */
enum {
  EB_IN_F32_CHW = 0, /* SampleBatch.data: (B, C*H*W) float32, already /pixel_scale (wire.py:71) */
  EB_IN_U8_HWC = 1   /* raw pixels, (B, H, W, C) uint8; /pixel_scale fused into K1 */
};

/* Tensor element types. */
enum { EB_BF16 = 0, EB_F32 = 1, EB_F64 = 2 };

/* Reserved tensor ids created by eb_engine_create. */
enum {
  EB_T_IMAGE_NHWC8 = 0, /* bf16 (H, W, 8): preprocessed image, channels >= C are zero */
  EB_T_IMAGE_F32 = 1    /* f32 (C, H, W): preprocessed image in the reference layout */
};

/* Operation kinds. */
enum {
  EB_OP_CONV = 0,   /* implicit-GEMM conv / FC on tcgen05; bias, residual, ReLU fused */
  EB_OP_POOL = 1,   /* max / avg pooling, optional per-channel BN-ReLU on the input */
  EB_OP_BNRELU = 2, /* y = relu(x * scale + shift) per channel */
  EB_OP_GAP = 3,    /* global average pool (optional BN-ReLU first) -> (1, 1, C) */
  EB_OP_LIN1 = 4,   /* fp64 linear scores of all LIN1 members: (C*H*W) -> (sum K) */
  EB_OP_RESIZE = 5  /* bilinear resize (align_corners=False) of an NHWC image to dst's H x W */
};

enum { EB_POOL_MAX = 0, EB_POOL_AVG = 1, EB_POOL_AVG_EXCL_PAD = 2 };

enum { EB_POLICY_NONE = 0, EB_POLICY_ANY = 1, EB_POLICY_ALL = 2, EB_POLICY_AT_LEAST = 3 };

enum { EB_MEMBER_CNN = 0, EB_MEMBER_LIN1 = 1 };

#define EB_NO_OFFSET UINT64_MAX

/* One node of a member's network.  Offsets are byte offsets into the engine's
 * weight pool.  Activations are NHWC; an op reads channels
 * [src_c_off, src_c_off + src_c) of `src` and writes channels
 * [dst_c_off, dst_c_off + cout) of `dst` (this is how concatenation is done). */
typedef struct {
  int32_t kind;
  int32_t src, dst, res; /* tensor ids; res = -1 for none */
  int32_t src_c_off, src_c;
  int32_t dst_c_off, cout;
  int32_t kh, kw, sh, sw, ph, pw;
  int32_t relu;
  int32_t pool_mode;
  int32_t flatten; /* CONV: treat src (H, W, C) as one row of H*W*C features */
  int32_t stream;  /* concurrency lane (0..3); ops on different lanes may overlap */
  int32_t groups;  /* CONV: grouped convolution (Cin == Cout, block-diagonal per N tile) */
  int32_t prefork; /* run on the main stream before the lanes fork (shared inputs) */
  int32_t dst2, dst2_c_off, n_split; /* CONV grouped launch: columns >= n_split -> dst2 */
  /* CONV: scale/shift = optional per-input-channel BN-ReLU applied to A inside
   * the kernel (1x1 only; arrays zero-padded to a multiple of 64).
   * POOL/GAP/BNRELU: the same BN-ReLU applied to the input elements. */
  uint64_t w_off, b_off, scale_off, shift_off;
} eb_op_desc;

typedef struct eb_engine eb_engine;

const char* eb_last_error(void);
int eb_abi_version(void);

/* Engine lifecycle.  The image geometry is the ensemble's shared input shape
 * (ensemble.py:202-208). */
int eb_engine_create(int device, int max_batch, int in_c, int in_h, int in_w, eb_engine** out);
/* Arithmetic precision of the CNN members, before any tensor or op is declared.
 * EB_PREC_BF16 (default): bf16 activations and weights, fp32 accumulation, tcgen05.
 * EB_PREC_F32: the fp32-faithful parity mode -- fp32 activations (tensors declared
 * EB_F32, the K1 image included), fp32 weights packed [Cout][kh][kw][Cin/groups],
 * every op on the CUDA cores with a sequential fp32 sum per output (SURVEY.md
 * §7.3 (iii)); top-k equals the fp32 CPU oracle's up to summation order. */
enum { EB_PREC_BF16 = 0, EB_PREC_F32 = 1 };
int eb_engine_set_precision(eb_engine* e, int precision);
/* A second execution context of a finalized engine: same device, ops and weight pool
 * (shared, freed with the last engine using it), its own activation arena, streams,
 * split-K workspaces and graph cache.  Concurrent requests lease one context each
 * (the reference re-enters forward from its worker threads, eg/gateway.py:222-257)
 * instead of serialising on one engine. */
int eb_engine_clone(eb_engine* src, eb_engine** out);
/* Capture the CUDA graphs of every batch-size bucket up to max_b (<= 0: max_batch) so
 * that no request pays a capture.  Buckets: exact up to 8, then multiples of 16 / 32 /
 * 64 (runtime.cu bucket_of); a request runs through its bucket's graph. */
int eb_engine_warmup(eb_engine* e, int input_kind, int max_b);
int eb_engine_destroy(eb_engine* e);

/* Normalisation: mean/std have 1 or C entries (models.py:247-253).  lut_u8 is
 * C*256 floats: the reference's fp32 value of ((v / pixel_scale) - mean) / std
 * for every byte v, computed on the host by the caller (exact by construction). */
int eb_set_preprocess(eb_engine* e, const float* host_mean, const float* host_std, int n,
                      const float* host_lut_u8);

/* One device allocation holds every member's weights (the shared pool of
 * ensemble.py:215-220, here in real device bytes). */
int eb_pool_reserve(eb_engine* e, uint64_t bytes);
int eb_pool_write(eb_engine* e, uint64_t offset, const void* host_src, uint64_t bytes);
int eb_pool_bytes(eb_engine* e, uint64_t* bytes);

/* Activation tensor of per-sample shape (h, w, c); storage is max_batch deep. */
int eb_tensor(eb_engine* e, int h, int w, int c, int dtype, int* id_out);
int eb_add_op(eb_engine* e, const eb_op_desc* op);
/* Register an output member: its logits are columns [k_off, k_off + k) of
 * `logits_tensor` (fp32 for CNN members, fp64 for LIN1). Manifest order. */
int eb_add_member(eb_engine* e, int kind, int logits_tensor, int k_off, int k);
int eb_finalize(eb_engine* e);

/* The forward boundary.  host_labels: int32 [N][batch] (EnsembleOutput.per_model
 * layout).  Optional outputs (NULL to skip): host_logits fp32 [N][batch][Kmax]
 * (zero padded), top-k indices/probabilities [N][batch][topk], combined policy
 * output [batch].  Host<->device copies are inside this call. */
/* A pipelined sequence of forwards (bulk serving; bench.py's end-to-end figure): batch
 * i (host_inputs[i], `batch` samples, one encoding) is copied host->device on a
 * separate copy stream while batch i-1 computes; its labels ([N][batch] int32) land
 * in host_labels[i].  Every batch's transfers are inside the call, which returns when
 * all batches are done.  Same validation and errors as eb_forward. */
int eb_forward_batches(eb_engine* e, const void* const* host_inputs, int n_batches, int input_kind,
                       int batch, int32_t* const* host_labels);
int eb_forward(eb_engine* e, const void* host_input, int input_kind, int batch,
               int32_t* host_labels, float* host_logits, int topk, int32_t* host_topk_idx,
               float* host_topk_prob, int policy, int policy_k, int32_t* host_combined);

/* Device-resident variant used for kernel-only timing: the input is already in
 * the engine's device staging buffer (see eb_input_buffer) and outputs stay on
 * the device (see eb_output_labels). */
int eb_forward_device(eb_engine* e, int input_kind, int batch, int topk, int policy, int policy_k);
int eb_input_buffer(eb_engine* e, int input_kind, void** dev_ptr);
int eb_output_labels(eb_engine* e, int32_t** dev_labels);
int eb_tensor_ptr(eb_engine* e, int id, void** dev_ptr, int* h, int* w, int* c, int* dtype);
int eb_engine_stream(eb_engine* e, void** stream);
/* Per-op device time (ms) of one eager, fully serialised run of the layers
 * (CUDA events around every op on one stream); host_ms holds one float per op
 * in eb_add_op order.  Used for the roofline of each kernel class. */
int eb_profile_ops(eb_engine* e, int input_kind, int batch, float* host_ms, int n_ops);
/* As eb_profile_ops with every op launched `repeat` times back to back (1..100); host_ms
 * gets the mean per launch, so short ops are timed without the host's launch latency. */
int eb_profile_ops_repeat(eb_engine* e, int input_kind, int batch, float* host_ms, int n_ops,
                          int repeat);
/* Number of kernels one eb_forward_device launches for this batch size. */
int eb_launch_count(eb_engine* e, int input_kind, int batch, int* count);

/* F1 wire fast path (host): decode a well-formed f32le /v1/predict body
 * (eg/wire.py:76-109) straight into host_out (n x prod(dims) floats, e.g. pinned),
 * base64 decoded in parallel, finiteness checked.  Returns EB_E_INVALID for anything
 * it does not accept (the caller then uses the reference decoder for its exact error).
 * The optional "policy" member is returned as a byte range of body. */
int eb_decode_request(const char* body, uint64_t len, const int32_t* dims, int ndims,
                      float* host_out, int max_samples, int* n_samples, uint64_t* policy_off,
                      uint64_t* policy_len);
/* As eb_decode_request, and also the "pgm" encoding (eg/wire.py:60-72) when
 * pixel_scale > 0 and dims = [1, H, W]: P5 parsed as eg/pgm.py:16-59, raster /
 * pixel_scale in fp32 (eg/wire.py:71). */
int eb_decode_request2(const char* body, uint64_t len, const int32_t* dims, int ndims,
                       float pixel_scale, float* out, int max_samples, int* n_samples,
                       uint64_t* policy_off, uint64_t* policy_len);
/* F4: the /v1/predict response body, byte-identical to the reference's
 * dumps_canonical(render_prediction(...)) (eg/wire.py:136-143, eg/jsonio.py:28-36).
 * key_json: the JSON-encoded keys in sorted order; key_kind[i] = -1 "_batch_size",
 * -2 "_combined", m >= 0 model m; label_json[m] + label_off[m][v] .. [v + 1]: model m's
 * label v JSON-encoded.  EB_E_TOO_LARGE (with *out_len set) when cap is too small. */
int eb_render_prediction(const int32_t* labels, int n_models, int batch, const int32_t* combined,
                         const char* const* key_json, const int32_t* key_kind, int n_keys,
                         const char* const* label_json, const int64_t* const* label_off,
                         const int32_t* n_labels, char* out, uint64_t cap, uint64_t* out_len);

/* Kernel-level entry points on caller-owned device memory (used by the parity
 * tests; `stream` is a cudaStream_t, NULL = legacy default stream). */
int eb_k_preprocess_f32(const float* dev_x, float* dev_y, int batch, int c, int64_t plane,
                        const float* dev_mean, const float* dev_std, int n, void* stream);
int eb_k_preprocess_u8_nhwc8(const uint8_t* dev_x, void* dev_y_bf16, int batch, int c,
                             int64_t plane, const float* dev_lut, void* stream);
int eb_k_conv(const void* dev_x, int batch, int h, int w, int ldx, int cin, const void* dev_w,
              const float* dev_bias, const void* dev_res, int ldr, void* dev_y, int ldy,
              int y_off, int cout, int kh, int kw, int sh, int sw, int ph, int pw, int relu,
              int out_f32, int c8_stem, int split_k, int block_n, int groups,
              void* dev_workspace, const float* dev_pre_scale, const float* dev_pre_shift,
              void* stream);
/* (eb_k_conv c8_stem: 0 = regular input, 1 = 8-channel NHWC image (gathered stem),
 *  2 = the image already in its eb_k_stem_relayout layout; h, w stay the image's.) */
/* eb_k_conv_maxpool2: a stride-1 conv followed by a 2x2 / stride-2 max-pool, fused
 * (eb_k_conv then eb_k_pool with kernel 2, stride 2, EB_POOL_MAX; bit-identical).  dev_y
 * is the pooled NHWC tensor (Ho/2 x Wo/2, row stride ldy, channel offset y_off).  Only the
 * taps-in-N geometry (3x3, pad 1, Cout <= 64 and a multiple of 32, even Ho and Wo, ldy and
 * y_off multiples of 8); EB_E_INVALID otherwise. */
int eb_k_conv_maxpool2(const void* dev_x, int batch, int h, int w, int ldx, int cin,
                       const void* dev_w, const float* dev_bias, void* dev_y, int ldy, int y_off,
                       int cout, int kh, int kw, int ph, int pw, int relu, void* stream);
int eb_k_resize(const void* dev_x, int ldx, void* dev_y, int ldy, int batch, int h, int w, int c,
                int ho, int wo, void* stream);
/* Stem layouts: eb_k_stem_layout reports the bytes of the zero-padded layout a stem conv
 * of this geometry reads with c8_stem = 2 (stride 1: padded rows; stride 2: even/odd
 * column planes), or EB_E_INVALID if the geometry has none; eb_k_stem_relayout writes it
 * from the 8-channel NHWC image (bf16). */
int eb_k_stem_layout(int batch, int h, int w, int kh, int kw, int sh, int sw, int ph, int pw,
                     uint64_t* bytes);
int eb_k_stem_relayout(const void* dev_x, int batch, int h, int w, int kh, int kw, int sh, int sw,
                       int ph, int pw, void* dev_y, void* stream);
/* K1 straight into a stem layout: u8 HWC pixels (c <= 8 channels) -> per-channel LUT ->
 * the padded layout eb_k_stem_relayout would produce from the NHWC8 image (identical
 * bytes, one pass; what the engine runs for stems on a u8 request). */
int eb_k_preprocess_u8_layout(const uint8_t* dev_x, int batch, int c, int h, int w,
                              const float* dev_lut, int kh, int kw, int sh, int sw, int ph, int pw,
                              void* dev_y, void* stream);
int eb_k_pool(const void* dev_x, int ldx, void* dev_y, int ldy, int y_off, int batch, int h,
              int w, int c, int k, int s, int pad, int mode, const float* dev_scale,
              const float* dev_shift, void* stream);
int eb_k_gap(const void* dev_x, int ldx, void* dev_y, int batch, int hw, int c,
             const float* dev_scale, const float* dev_shift, void* stream);
int eb_k_lin1(const float* dev_x, const float* dev_w, const float* dev_bias, double* dev_part,
              double* dev_logits, int batch, int k, int64_t d, int nsplit, void* stream);
int eb_k_combine(const float* dev_l32, int ld32, const double* dev_l64, int ld64,
                 const int* dev_kind, const int* dev_koff, const int* dev_kcnt, int n, int batch,
                 int32_t* dev_labels, int topk, int32_t* dev_topk_idx, float* dev_topk_prob,
                 int policy, int policy_k, int32_t* dev_combined, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ENSEMBLE_B200_H */
