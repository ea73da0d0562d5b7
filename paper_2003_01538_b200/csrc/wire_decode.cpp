// wire_decode.cpp -- F1: native fast path for the /v1/predict request body.
//
// The reference decodes requests with json.loads + base64.b64decode + np.frombuffer +
// np.stack (eg/wire.py:76-109), ~8 ms per 224x224 RGB f32le sample.  This scanner
// accepts exactly the well-formed f32le case of that protocol:
//
//   {"samples": [{"encoding": "f32le", "shape": [...], "data": "<base64>"}, ...],
//    "policy": {...}}                               (keys in any order, any whitespace)
//
// (and, given the ensemble's pixel scale, the "pgm" encoding of a [1, H, W] shape: the
// P5 header parsed as eg/pgm.py does, raster / pixel_scale in fp32) and base64-decodes
// every sample straight into one caller-provided (pinned) buffer,
// in parallel across samples, checking finiteness.  Anything else -- another
// encoding, an unexpected key, a duplicate key, an escape sequence, a shape or length
// mismatch, invalid base64, a non-finite value -- returns EB_E_INVALID and the caller
// falls back to the reference decoder, which produces the reference's exact error.
// The optional "policy" value is returned as a byte range for the caller to parse.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/ensemble_b200.h"
#include "eb_internal.h"

namespace {

struct Scanner {
  const char* p;
  const char* end;
  bool ok = true;

  void ws() {
    while (p < end && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) ++p;
  }
  bool lit(char c) {
    ws();
    if (p < end && *p == c) {
      ++p;
      return true;
    }
    return false;
  }
  // a JSON string without escapes; returns [b, e)
  bool str(const char** b, const char** e) {
    ws();
    if (p >= end || *p != '"') return false;
    const char* s = ++p;
    const char* q = static_cast<const char*>(memchr(p, '"', end - p));
    if (!q) return false;
    if (memchr(s, '\\', q - s)) return false;  // escapes: leave to the reference
    *b = s;
    *e = q;
    p = q + 1;
    return true;
  }
  bool integer(long long* v) {
    ws();
    const char* s = p;
    if (p < end && *p == '-') ++p;
    if (p >= end || *p < '0' || *p > '9') return false;
    // strict JSON: no leading zeros ("007", "-0..."), and no "-0" either -- anything the
    // reference's loads_strict might judge differently goes to the reference decoder
    if (*p == '0' && (*s == '-' || (p + 1 < end && p[1] >= '0' && p[1] <= '9'))) return false;
    long long x = 0;
    while (p < end && *p >= '0' && *p <= '9') {
      x = x * 10 + (*p - '0');
      if (x > (1ll << 40)) return false;
      ++p;
    }
    if (p < end && (*p == '.' || *p == 'e' || *p == 'E')) return false;
    *v = (*s == '-') ? -x : x;
    return true;
  }
  // skip any JSON value (used for "policy"); strings may not contain escapes
  bool skip_value() {
    ws();
    if (p >= end) return false;
    if (*p == '"') {
      const char *b, *e;
      return str(&b, &e);
    }
    if (*p == '{' || *p == '[') {
      const char open = *p, close = (*p == '{') ? '}' : ']';
      ++p;
      if (lit(close)) return true;
      for (;;) {
        if (open == '{') {
          const char *b, *e;
          if (!str(&b, &e) || !lit(':')) return false;
        }
        if (!skip_value()) return false;
        if (lit(',')) continue;
        return lit(close);
      }
    }
    while (p < end && *p != ',' && *p != '}' && *p != ']' && *p != ' ' && *p != '\n' &&
           *p != '\r' && *p != '\t')
      ++p;
    return true;
  }
};

bool key_is(const char* b, const char* e, const char* k) {
  const size_t n = strlen(k);
  return static_cast<size_t>(e - b) == n && memcmp(b, k, n) == 0;
}

int8_t kB64[256];
bool b64_init() {
  memset(kB64, -1, sizeof(kB64));
  const char* a = "ABCDEFGHIJKLMNOPQRSTUVWXYZabcdefghijklmnopqrstuvwxyz0123456789+/";
  for (int i = 0; i < 64; ++i) kB64[static_cast<unsigned char>(a[i])] = static_cast<int8_t>(i);
  return true;
}
const bool kB64Ready = b64_init();

// strict base64 (as base64.b64decode(validate=True)) into exactly n_out bytes
bool b64_decode(const char* s, size_t len, uint8_t* out, size_t n_out) {
  if (len % 4 != 0) return false;
  size_t pad = 0;
  if (len >= 1 && s[len - 1] == '=') ++pad;
  if (len >= 2 && s[len - 2] == '=') ++pad;
  if (len / 4 * 3 - pad != n_out) return false;
  size_t o = 0;
  for (size_t i = 0; i < len; i += 4) {
    const int a = kB64[static_cast<unsigned char>(s[i])];
    const int b = kB64[static_cast<unsigned char>(s[i + 1])];
    const bool last = (i + 4 == len);
    const int c = (last && pad >= 2) ? 0 : kB64[static_cast<unsigned char>(s[i + 2])];
    const int d = (last && pad >= 1) ? 0 : kB64[static_cast<unsigned char>(s[i + 3])];
    if ((a | b | c | d) < 0) return false;
    const uint32_t v = (a << 18) | (b << 12) | (c << 6) | d;
    out[o++] = static_cast<uint8_t>(v >> 16);
    if (o < n_out) out[o++] = static_cast<uint8_t>(v >> 8);
    if (o < n_out) out[o++] = static_cast<uint8_t>(v);
  }
  return true;
}

struct Sample {
  const char* data_b;
  const char* data_e;
  bool pgm;  // "encoding": "pgm" (eg/wire.py:60-72): P5 raster / pixel_scale, shape [1, H, W]
};

// The reference's parse_pgm (eg/pgm.py:16-59) on a decoded P5 document, then
// u8 / pixel_scale in fp32 (eg/wire.py:71).  false for anything it would reject (or
// anything this restatement is unsure about: very long header tokens) -- the caller then
// falls back to the reference decoder for the exact error.
bool is_pgm_ws(uint8_t c) { return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == 0x0b || c == 0x0c; }
bool pgm_to_f32(const uint8_t* d, size_t n, int h_want, int w_want, float pixel_scale, float* out) {
  size_t pos = 0;
  auto token = [&](size_t* b, size_t* e) {
    while (pos < n && is_pgm_ws(d[pos])) ++pos;
    *b = pos;
    while (pos < n && !is_pgm_ws(d[pos])) ++pos;
    *e = pos;
    return *e > *b;
  };
  size_t b, e;
  if (!token(&b, &e) || e - b != 2 || d[b] != 'P' || d[b + 1] != '5') return false;
  long long v[3];
  for (int i = 0; i < 3; ++i) {
    if (!token(&b, &e) || e - b > 9) return false;
    long long x = 0;
    for (size_t k = b; k < e; ++k) {
      if (d[k] < '0' || d[k] > '9') return false;
      x = x * 10 + (d[k] - '0');
    }
    v[i] = x;
  }
  const long long width = v[0], height = v[1], maxval = v[2];
  if (width < 1 || height < 1 || maxval < 1 || maxval > 255) return false;
  if (pos >= n || !is_pgm_ws(d[pos])) return false;
  ++pos;
  if (width != w_want || height != h_want || static_cast<long long>(n - pos) != width * height) return false;
  const uint8_t* px = d + pos;
  const int64_t np = width * height;
  for (int64_t k = 0; k < np; ++k) {
    if (px[k] > maxval) return false;
    out[k] = static_cast<float>(px[k]) / pixel_scale;
  }
  return true;
}

}  // namespace

extern "C" int eb_decode_request2(const char* body, uint64_t len, const int32_t* dims, int ndims,
                                  float pixel_scale, float* out, int max_samples, int* n_samples,
                                  uint64_t* policy_off, uint64_t* policy_len);

extern "C" int eb_decode_request(const char* body, uint64_t len, const int32_t* dims, int ndims,
                                 float* out, int max_samples, int* n_samples,
                                 uint64_t* policy_off, uint64_t* policy_len) {
  return eb_decode_request2(body, len, dims, ndims, 0.f, out, max_samples, n_samples, policy_off,
                            policy_len);
}

extern "C" int eb_decode_request2(const char* body, uint64_t len, const int32_t* dims, int ndims,
                                  float pixel_scale, float* out, int max_samples, int* n_samples,
                                  uint64_t* policy_off, uint64_t* policy_len) {
  // pgm samples only with a pixel scale and a [1, H, W] ensemble shape
  const bool pgm_ok = pixel_scale > 0.f && ndims == 3 && dims[0] == 1;
  if (!body || !dims || !out || !n_samples || ndims < 1 || ndims > 3) return EB_E_INVALID;
  int64_t D = 1;
  for (int i = 0; i < ndims; ++i) D *= dims[i];
  Scanner sc{body, body + len};
  std::vector<Sample> samples;
  bool have_samples = false, have_policy = false;
  *policy_off = 0;
  *policy_len = 0;
  if (!sc.lit('{')) return EB_E_INVALID;
  if (!sc.lit('}')) {
    for (;;) {
      const char *kb, *ke;
      if (!sc.str(&kb, &ke) || !sc.lit(':')) return EB_E_INVALID;
      if (key_is(kb, ke, "samples")) {
        if (have_samples) return EB_E_INVALID;
        have_samples = true;
        if (!sc.lit('[')) return EB_E_INVALID;
        if (sc.lit(']')) return EB_E_INVALID;  // empty: reference error path
        for (;;) {
          if (!sc.lit('{')) return EB_E_INVALID;
          bool h_enc = false, h_shape = false, h_data = false;
          Sample smp{};
          for (;;) {
            const char *fb, *fe;
            if (!sc.str(&fb, &fe) || !sc.lit(':')) return EB_E_INVALID;
            if (key_is(fb, fe, "encoding")) {
              const char *vb, *ve;
              if (h_enc || !sc.str(&vb, &ve)) return EB_E_INVALID;
              if (key_is(vb, ve, "pgm") && pgm_ok)
                smp.pgm = true;
              else if (!key_is(vb, ve, "f32le"))
                return EB_E_INVALID;
              h_enc = true;
            } else if (key_is(fb, fe, "shape")) {
              if (h_shape || !sc.lit('[')) return EB_E_INVALID;
              for (int i = 0; i < ndims; ++i) {
                long long v;
                if (!sc.integer(&v) || v != dims[i]) return EB_E_INVALID;
                if (i + 1 < ndims && !sc.lit(',')) return EB_E_INVALID;
              }
              if (!sc.lit(']')) return EB_E_INVALID;
              h_shape = true;
            } else if (key_is(fb, fe, "data")) {
              if (h_data || !sc.str(&smp.data_b, &smp.data_e)) return EB_E_INVALID;
              h_data = true;
            } else {
              return EB_E_INVALID;
            }
            if (sc.lit(',')) continue;
            if (!sc.lit('}')) return EB_E_INVALID;
            break;
          }
          // f32le: encoding, shape, data; pgm: encoding, data (eg/wire.py:26-27)
          if (!(h_enc && h_data) || h_shape == smp.pgm) return EB_E_INVALID;
          samples.push_back(smp);
          if (static_cast<int>(samples.size()) > max_samples) return EB_E_TOO_LARGE;
          if (sc.lit(',')) continue;
          if (!sc.lit(']')) return EB_E_INVALID;
          break;
        }
      } else if (key_is(kb, ke, "policy")) {
        if (have_policy) return EB_E_INVALID;
        have_policy = true;
        sc.ws();
        const char* vb = sc.p;
        if (!sc.skip_value()) return EB_E_INVALID;
        *policy_off = static_cast<uint64_t>(vb - body);
        *policy_len = static_cast<uint64_t>(sc.p - vb);
      } else {
        return EB_E_INVALID;
      }
      if (sc.lit(',')) continue;
      if (!sc.lit('}')) return EB_E_INVALID;
      break;
    }
  }
  sc.ws();
  if (sc.p != sc.end || !have_samples) return EB_E_INVALID;

  const int n = static_cast<int>(samples.size());
  const size_t nbytes = static_cast<size_t>(D) * 4;
  std::vector<char> bad(n, 0);
  auto work = [&](int lo, int hi) {
    std::vector<uint8_t> doc;
    for (int i = lo; i < hi; ++i) {
      float* dst = out + static_cast<size_t>(i) * D;
      if (samples[i].pgm) {
        const size_t l = samples[i].data_e - samples[i].data_b;
        if (l % 4 != 0 || l == 0) {
          bad[i] = 1;
          continue;
        }
        const char* q = samples[i].data_b;
        const size_t pad = (q[l - 1] == '=') + (l >= 2 && q[l - 2] == '=');
        doc.resize(l / 4 * 3 - pad);
        if (!b64_decode(q, l, doc.data(), doc.size()) ||
            !pgm_to_f32(doc.data(), doc.size(), dims[1], dims[2], pixel_scale, dst))
          bad[i] = 1;
        continue;
      }
      if (!b64_decode(samples[i].data_b, samples[i].data_e - samples[i].data_b,
                      reinterpret_cast<uint8_t*>(dst), nbytes)) {
        bad[i] = 1;
        continue;
      }
      for (int64_t k = 0; k < D; ++k)
        if (!std::isfinite(dst[k])) {
          bad[i] = 1;
          break;
        }
    }
  };
  const int hw = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  const int nt = std::min({n, hw, 32});
  if (nt <= 1 || static_cast<int64_t>(n) * D < (1 << 20)) {
    work(0, n);
  } else {
    std::vector<std::thread> th;
    const int per = (n + nt - 1) / nt;
    for (int t = 0; t < nt; ++t) th.emplace_back(work, t * per, std::min(n, (t + 1) * per));
    for (auto& t : th) t.join();
  }
  for (int i = 0; i < n; ++i)
    if (bad[i]) return EB_E_INVALID;
  *n_samples = n;
  return EB_OK;
}

// ---------------------------------------------------------------------------------------
// F4: the response body of /v1/predict, byte-identical to
//   dumps_canonical(render_prediction(ensemble, output, combined))   (eg/wire.py:136-143,
//   eg/jsonio.py:28-36: sorted keys, compact separators, ensure_ascii)
// The caller passes every key already JSON-encoded, in sorted order, and every model's
// labels JSON-encoded (json.dumps(label, ensure_ascii=True) on the host, once per
// ensemble); key_kind[i] = -1: "_batch_size", -2: "_combined", m >= 0: model m.
extern "C" int eb_render_prediction(const int32_t* labels, int n_models, int batch,
                                    const int32_t* combined, const char* const* key_json,
                                    const int32_t* key_kind, int n_keys,
                                    const char* const* label_json, const int64_t* const* label_off,
                                    const int32_t* n_labels, char* out, uint64_t cap,
                                    uint64_t* out_len) {
  if (!labels || !key_json || !key_kind || !out_len || n_models < 0 || batch < 0) return EB_E_INVALID;
  static const char* kBin[2] = {"\"absent\"", "\"present\""};
  std::string s;
  s.reserve(64 + static_cast<size_t>(batch) * (n_models + 1) * 12);
  s.push_back('{');
  for (int i = 0; i < n_keys; ++i) {
    if (i) s.push_back(',');
    s.append(key_json[i]);
    s.push_back(':');
    const int k = key_kind[i];
    if (k == -1) {
      s.append(std::to_string(batch));
    } else if (k == -2) {
      if (!combined) return EB_E_INVALID;
      s.push_back('[');
      for (int b = 0; b < batch; ++b) {
        if (b) s.push_back(',');
        const int v = combined[b];
        if (v < 0 || v > 1) return EB_E_INVALID;
        s.append(kBin[v]);
      }
      s.push_back(']');
    } else if (k >= 0 && k < n_models) {
      const int32_t* row = labels + static_cast<int64_t>(k) * batch;
      s.push_back('[');
      for (int b = 0; b < batch; ++b) {
        if (b) s.push_back(',');
        const int v = row[b];
        if (v < 0 || v >= n_labels[k]) return EB_E_INVALID;
        s.append(label_json[k] + label_off[k][v], label_json[k] + label_off[k][v + 1]);
      }
      s.push_back(']');
    } else {
      return EB_E_INVALID;
    }
  }
  s.push_back('}');
  *out_len = s.size();
  if (!out || s.size() > cap) return EB_E_TOO_LARGE;
  memcpy(out, s.data(), s.size());
  return EB_OK;
}
