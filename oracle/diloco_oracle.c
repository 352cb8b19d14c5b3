/*
 * diloco_oracle.c — CPU restatement of the reference DiLoCo hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity *checker*: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  The product path (paper_2407_07852_b200, libdiloco_cuda.so)
 * never links or calls it and fails loudly when its CUDA library is missing.
 *
 * Every function restates one reference function, cited file:line against
 * /root/reference/proj.  Arithmetic is plain FP32 in the reference's evaluation
 * order; build with -ffp-contract=off like the reference (proj/CMakeLists.txt:18)
 * so no multiply-add is contracted.
 *
 * Pinning: tests/test_oracle.py checks this restatement bit-for-bit against the
 * reference compiled from its own sources (oracle/_ref, see oracle/Makefile)
 * and against the committed golden vectors in tests/golden/ generated from it.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <string.h>

#define ORC_OK 0
#define ORC_ESHAPE 1
#define ORC_ECONFIG 2
#define ORC_ENUMERIC 3
#define ORC_ECOLLECTIVE 4

static inline uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static inline float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

/* ---- counter RNG: proj/include/diloco/rng.hpp:17-74 --------------------- */

uint64_t orc_splitmix64(uint64_t x) { /* rng.hpp:17-22 */
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

uint64_t orc_fnv1a64(const char* s) { /* rng.hpp:24-31 */
  uint64_t h = 0xCBF29CE484222325ull;
  for (; *s; ++s) { h ^= (uint8_t)*s; h *= 0x100000001B3ull; }
  return h;
}

/* CounterRng(seed, purpose, index) initial state, rng.hpp:40-41,66-71. */
uint64_t orc_rng_key(uint64_t seed, const char* purpose, uint64_t index) {
  uint64_t h = orc_splitmix64(seed ^ 0x6A09E667F3BCC909ull);
  h = orc_splitmix64(h ^ orc_fnv1a64(purpose));
  h = orc_splitmix64(h ^ index);
  return h;
}

/* The (i+1)-th next_uniform(lo, hi) draw of a CounterRng whose state is
 * `key` (rng.hpp:43-56): state += golden (i+1 times), splitmix, top 24 bits.
 * Stateless in i, so a GPU thread can produce element i on its own. */
float orc_rng_uniform_at(uint64_t key, uint64_t i, float lo, float hi) {
  const uint64_t st = key + (i + 1) * 0x9E3779B97F4A7C15ull;
  const float u = (float)(orc_splitmix64(st) >> 40) * 0x1p-24f;
  return lo + (hi - lo) * u;
}

void orc_rng_fill(uint64_t key, uint64_t first, size_t n, float lo, float hi,
                  float* out) {
  for (size_t i = 0; i < n; ++i) out[i] = orc_rng_uniform_at(key, first + i, lo, hi);
}

/* ---- binary16 codec: proj/src/fp16.cpp:13-85 ----------------------------- */

static inline uint32_t shift_rne(uint32_t m, int shift) { /* fp16.cpp:13-21 */
  uint32_t q = m >> shift;
  const uint32_t rem = m & ((1u << shift) - 1u);
  const uint32_t half = 1u << (shift - 1);
  if (rem > half || (rem == half && (q & 1u))) ++q;
  return q;
}

uint16_t orc_fp16_encode(float value) { /* fp16.cpp:25-63 */
  const uint32_t x = f2u(value);
  const uint16_t sign = (uint16_t)((x >> 16) & 0x8000u);
  const uint32_t mag = x & 0x7FFFFFFFu;
  if (mag >= 0x7F800000u) return mag == 0x7F800000u ? (sign | 0x7C00u) : (sign | 0x7E00u);
  if (mag >= 0x477FF000u) return sign | 0x7C00u;   /* >= 65520 -> inf */
  if (mag <= 0x33000000u) return sign;             /* <= 2^-25 -> 0 */
  if (mag < 0x38800000u) {                         /* subnormal half */
    const uint32_t significand = (mag & 0x007FFFFFu) | 0x00800000u;
    const int exp = (int)(mag >> 23);
    return sign | (uint16_t)shift_rne(significand, 126 - exp);
  }
  uint32_t code = (((mag >> 23) - 127 + 15) << 10) | ((mag & 0x007FFFFFu) >> 13);
  const uint32_t rem = mag & 0x1FFFu;
  if (rem > 0x1000u || (rem == 0x1000u && (code & 1u))) ++code;
  return sign | (uint16_t)code;
}

float orc_fp16_decode(uint16_t bits) { /* fp16.cpp:65-85 */
  const uint32_t sign = (uint32_t)(bits & 0x8000u) << 16;
  const uint32_t exp = (bits >> 10) & 0x1Fu;
  const uint32_t mant = bits & 0x3FFu;
  if (exp == 0) {
    if (mant == 0) return u2f(sign);
    return u2f(sign | f2u((float)mant * 0x1p-24f));
  }
  if (exp == 31) {
    if (mant == 0) return u2f(sign | 0x7F800000u);
    return u2f(sign | 0x7FC00000u | (mant << 13));
  }
  return u2f(sign | ((exp - 15 + 127) << 23) | (mant << 13));
}

static inline int fp16_is_nonfinite(uint16_t b) { return (b & 0x7C00u) == 0x7C00u; } /* fp16.hpp:24-26 */

/* encode_fp16, tensor.cpp:131-140: returns the overflow signal. */
int orc_encode_fp16(const float* v, size_t n, uint16_t* out) {
  int overflow = 0;
  for (size_t i = 0; i < n; ++i) {
    out[i] = orc_fp16_encode(v[i]);
    overflow |= fp16_is_nonfinite(out[i]);
  }
  return overflow;
}

void orc_decode_fp16(const uint16_t* b, size_t n, float* out) { /* tensor.cpp:142-154 */
  for (size_t i = 0; i < n; ++i) out[i] = orc_fp16_decode(b[i]);
}

/* ---- tensor helpers: proj/src/tensor.cpp ---------------------------------- */

int orc_all_finite(const float* v, size_t n) { /* tensor.cpp:97-104 */
  for (size_t i = 0; i < n; ++i) if (!isfinite(v[i])) return 0;
  return 1;
}

void orc_axpy(float alpha, const float* x, const float* y, size_t n, float* out) {
  for (size_t i = 0; i < n; ++i) out[i] = y[i] + alpha * x[i]; /* tensor.cpp:125-127 */
}

/* ---- optimizers: proj/src/optim.cpp --------------------------------------- */

float orc_lr_at(uint64_t warmup, uint64_t total, float base_lr, int cosine,
                uint64_t step) { /* optim.cpp:37-56 */
  const float base = base_lr;
  if (warmup > 0 && step <= warmup) return base * (float)step / (float)warmup;
  if (!cosine || total == 0 || total <= warmup) return base;
  const float floor_lr = 0.1f * base;
  if (step >= total) return floor_lr;
  const double progress = (double)(step - warmup) / (double)(total - warmup);
  const double c = 0.5 * (1.0 + cos(progress * M_PI));
  return (float)(floor_lr + (base - floor_lr) * c);
}

/* Bias corrections at step t, optim.cpp:73-76 (host powf, float exponent). */
void orc_bias_corrections(float b1, float b2, uint64_t t, float* c1, float* c2) {
  *c1 = 1.0f - powf(b1, (float)t);
  *c2 = 1.0f - powf(b2, (float)t);
}

/* adamw_step, optim.cpp:58-93.  p -> out (out of place), m/v in place,
 * *step_count advanced on success only. */
int orc_adamw_step(const float* p, const float* g, float* m, float* v, size_t n,
                   float b1, float b2, float eps, float wd, uint64_t* step_count,
                   float lr, float* out) {
  if (lr < 0.0f) return ORC_ECONFIG;                 /* :63-65 */
  if (!orc_all_finite(g, n)) return ORC_ENUMERIC;    /* :66-68 */
  *step_count += 1;                                   /* :69 */
  float corr1, corr2;
  orc_bias_corrections(b1, b2, *step_count, &corr1, &corr2);
  for (size_t i = 0; i < n; ++i) {                    /* :83-91 */
    m[i] = b1 * m[i] + (1.0f - b1) * g[i];
    v[i] = b2 * v[i] + (1.0f - b2) * g[i] * g[i];
    const float m_hat = m[i] / corr1;
    const float v_hat = v[i] / corr2;
    const float update = m_hat / (sqrtf(v_hat) + eps) + wd * p[i];
    out[i] = p[i] - lr * update;
  }
  return ORC_OK;
}

/* nesterov_step, optim.cpp:95-115. */
int orc_nesterov_step(const float* p, const float* g, float* buf, size_t n,
                      float lr, float mu, float* out) {
  if (!orc_all_finite(g, n)) return ORC_ENUMERIC;    /* :101-103 */
  for (size_t i = 0; i < n; ++i) {                    /* :110-113 */
    buf[i] = mu * buf[i] + g[i];
    out[i] = p[i] - lr * (g[i] + mu * buf[i]);
  }
  return ORC_OK;
}

/* scale_gradient, engine.cpp:20-27 (closed-form backward of the scaled loss). */
void orc_scale_gradient(const float* g, float scale, size_t n, float* out) {
  for (size_t i = 0; i < n; ++i) out[i] = g[i] * scale;
}

/* scaler_unscale_and_check, optim.cpp:121-135: returns overflow. */
int orc_scaler_unscale_and_check(float scale, const float* g, size_t n, float* out) {
  const float inv = 1.0f / scale;
  int overflow = 0;
  for (size_t i = 0; i < n; ++i) {
    out[i] = g[i] * inv;
    if (!isfinite(out[i])) overflow = 1;
  }
  return overflow;
}

/* scaler_update, optim.cpp:137-148 (clamps at optim.cpp:13-14). */
void orc_scaler_update(float* scale, uint64_t* good, uint64_t growth, int overflow) {
  if (overflow) {
    const float s = *scale * 0.5f;
    *scale = s > 0x1p-20f ? s : 0x1p-20f;
    *good = 0;
    return;
  }
  *good += 1;
  if (*good >= growth) {
    const float s = *scale * 2.0f;
    *scale = s < 0x1p24f ? s : 0x1p24f;
    *good = 0;
  }
}

/* apply_inner_step minus the (out-of-scope) gradient producer,
 * engine.cpp:50-69: scale -> unscale/check -> (clean) lr_at + adamw -> scaler.
 * `params` is updated in place (engine assigns the returned vector).
 * `tmp` is scratch of 2n floats.  Returns 1 when the step was skipped. */
int orc_inner_step(float* params, const float* grad, float* m, float* v, size_t n,
                   float b1, float b2, float eps, float wd, uint64_t* step_count,
                   uint64_t warmup, uint64_t total, float base_lr, int cosine,
                   float* scale, uint64_t* good, uint64_t growth, float* tmp,
                   float* lr_out) {
  float* scaled = tmp;
  float* unscaled = tmp + n;
  orc_scale_gradient(grad, *scale, n, scaled);
  const int overflow = orc_scaler_unscale_and_check(*scale, scaled, n, unscaled);
  *lr_out = 0.0f;
  if (!overflow) {
    *lr_out = orc_lr_at(warmup, total, base_lr, cosine, *step_count + 1);
    orc_adamw_step(params, unscaled, m, v, n, b1, b2, eps, wd, step_count, *lr_out, params);
  }
  orc_scaler_update(scale, good, growth, overflow);
  return overflow;
}

/* ---- reduction: proj/src/reduce.cpp --------------------------------------- */

void orc_partition_ranges(size_t n, size_t k, size_t* offsets, size_t* lengths) {
  const size_t base = k == 0 ? 0 : n / k;           /* reduce.cpp:20-31 */
  const size_t rem = k == 0 ? 0 : n % k;
  size_t off = 0;
  for (size_t i = 0; i < k; ++i) {
    lengths[i] = base + (i < rem ? 1 : 0);
    offsets[i] = off;
    off += lengths[i];
  }
}

void orc_fold_mean(const float* const* slices, size_t k, size_t n, float* out) {
  const float divisor = (float)k;                   /* reduce.cpp:33-44 */
  for (size_t i = 0; i < n; ++i) {
    float acc = slices[0][i];
    for (size_t j = 1; j < k; ++j) acc += slices[j][i];
    out[i] = acc / divisor;
  }
}

/* reduce_average, reduce.cpp:46-89.  precision 0 = fp32, 1 = fp16.
 * `scratch` must hold k*n floats for the fp16 path (may be NULL for fp32). */
int orc_reduce_average(const float* const* contribs, size_t k, size_t n,
                       int precision, float* scratch, float* out) {
  if (k == 0) return ORC_ECOLLECTIVE;
  if (precision == 0) { orc_fold_mean(contribs, k, n, out); return ORC_OK; }
  const float* slices[256];
  if (k > 256) return ORC_ECONFIG;
  for (size_t j = 0; j < k; ++j) {
    float* d = scratch + j * n;
    for (size_t i = 0; i < n; ++i) d[i] = orc_fp16_decode(orc_fp16_encode(contribs[j][i]));
    slices[j] = d;
  }
  orc_fold_mean(slices, k, n, out);
  for (size_t i = 0; i < n; ++i) out[i] = orc_fp16_decode(orc_fp16_encode(out[i]));
  return ORC_OK;
}

uint64_t orc_per_peer_reduce_bytes(size_t n, size_t k, size_t rank, int precision) {
  if (k <= 1) return 0;                             /* reduce.cpp:91-104 */
  const uint64_t w = precision ? 2 : 4;
  const size_t base = n / k, rem = n % k;
  const size_t own = base + (rank < rem ? 1 : 0);
  const size_t nxt = (rank + 1) % k;
  const size_t succ = base + (nxt < rem ? 1 : 0);
  return (uint64_t)(n - own) * w + (uint64_t)(n - succ) * w;
}

uint64_t orc_fleet_reduce_bytes(size_t n, size_t k, int precision) {
  if (k <= 1) return 0;                             /* reduce.cpp:106-111 */
  return 2ull * (k - 1) * (uint64_t)n * (precision ? 2 : 4);
}

/* ---- outer step: engine.cpp:115-146 ---------------------------------------- */

/* compute_pseudo_gradient, engine.cpp:115-126 -> axpy(-1, theta_local, theta_t). */
void orc_pseudo_gradient(const float* theta_t, const float* theta_local, size_t n,
                         float* delta) {
  orc_axpy(-1.0f, theta_local, theta_t, n, delta);
}

/* DilocoEngine::outer_step after the epoch guard, engine.cpp:136-144:
 * Nesterov on theta_t when the reduction is finite, theta_local := theta_t
 * always.  Returns 1 when applied. */
int orc_outer_step(float* theta_t, float* theta_local, float* buf, const float* dbar,
                   size_t n, float lr, float mu) {
  int applied = 0;
  if (orc_all_finite(dbar, n)) {
    orc_nesterov_step(theta_t, dbar, buf, n, lr, mu, theta_t);
    applied = 1;
  }
  memcpy(theta_local, theta_t, n * sizeof(float));
  return applied;
}

/* ---- wire codec: proj/src/wire.cpp:10-104, proj/src/collective.cpp:63-152,
 *      1318-1345 ----------------------------------------- */

#define ORC_ESERIAL 5   /* SerializationError, errors.hpp:48 */
#define ORC_EAGAIN 6    /* FrameParser::next() == nullopt: frame incomplete */

static size_t put_le(uint8_t* out, uint64_t v, int nbytes) {
  for (int i = 0; i < nbytes; ++i) out[i] = (uint8_t)(v >> (8 * i));
  return (size_t)nbytes;
}

static uint64_t get_le(const uint8_t* in, int nbytes) {
  uint64_t v = 0;
  for (int i = 0; i < nbytes; ++i) v |= (uint64_t)in[i] << (8 * i);
  return v;
}

/* encode_frame, wire.cpp:10-22: "ODLC" | version 1 | type | u64 LE length | payload.
 * out == NULL: size only. */
size_t orc_encode_frame(uint8_t type, const uint8_t* payload, size_t len, uint8_t* out) {
  if (out) {
    memcpy(out, "ODLC", 4);
    out[4] = 1; /* kWireVersion, wire.hpp:27 */
    out[5] = type;
    put_le(out + 6, len, 8);
    if (len) memcpy(out + 14, payload, len);
  }
  return 14 + len;
}

/* encode_reduce_payload, wire.cpp:74-88: epoch u64 | chunk_index u32 | precision u8 | segment. */
size_t orc_encode_reduce_payload(uint64_t epoch, uint32_t chunk_index, uint8_t precision,
                                 const uint8_t* seg, size_t seglen, uint8_t* out) {
  if (out) {
    put_le(out, epoch, 8);
    put_le(out + 8, chunk_index, 4);
    out[12] = precision;
    if (seglen) memcpy(out + 13, seg, seglen);
  }
  return 13 + seglen;
}

/* encode_chunk_segment, collective.cpp:63-81: u64 1 | u64 name_len | name |
 * u64 offset | u64 length | scalars (the tensor-core layout header of one segment). */
size_t orc_encode_chunk_segment(const char* name, size_t name_len, uint64_t offset, uint64_t length,
                                const uint8_t* scalars, size_t nbytes, uint8_t* out) {
  if (out) {
    uint8_t* o = out;
    o += put_le(o, 1, 8);
    o += put_le(o, name_len, 8);
    memcpy(o, name, name_len);
    o += name_len;
    o += put_le(o, offset, 8);
    o += put_le(o, length, 8);
    if (nbytes) memcpy(o, scalars, nbytes);
  }
  return 32 + name_len + nbytes;
}

/* chunk_name, collective.cpp:126-131 with PeerId::hex, collective.cpp:214-220:
 * "a<attempt>.p<partition>.f<%016llx%016llx>".  Returns the length (< 80). */
size_t orc_chunk_name(uint32_t attempt, uint32_t partition, uint64_t hi, uint64_t lo, char* out) {
  char buf[96];
  /* snprintf is not in string.h; build the decimal fields by hand */
  size_t n = 0;
  char dec[16];
  int d;
  buf[n++] = 'a';
  d = 0;
  do { dec[d++] = (char)('0' + attempt % 10); attempt /= 10; } while (attempt);
  while (d) buf[n++] = dec[--d];
  buf[n++] = '.';
  buf[n++] = 'p';
  do { dec[d++] = (char)('0' + partition % 10); partition /= 10; } while (partition);
  while (d) buf[n++] = dec[--d];
  buf[n++] = '.';
  buf[n++] = 'f';
  static const char* hx = "0123456789abcdef";
  for (int i = 15; i >= 0; --i) buf[n++] = hx[(hi >> (4 * i)) & 0xF];
  for (int i = 15; i >= 0; --i) buf[n++] = hx[(lo >> (4 * i)) & 0xF];
  memcpy(out, buf, n);
  return n;
}

/* The byte stream send_chunk_span puts on one connection (collective.cpp:1318-1345):
 * max_elems = max(1, chunk_size_bytes / width) elements per frame, chunk_index
 * counting from 0, each chunk's global offset = global_offset + start.
 * `scalars` holds elems * width bytes.  out == NULL: size only. */
size_t orc_send_chunk_span(uint8_t type, uint64_t epoch, const char* name, size_t name_len, int precision,
                           uint64_t global_offset, const uint8_t* scalars, uint64_t elems,
                           uint64_t chunk_size_bytes, uint8_t* out) {
  const uint64_t width = precision ? 2 : 4;
  uint64_t max_elems = chunk_size_bytes / width;
  if (max_elems < 1) max_elems = 1;
  size_t used = 0;
  uint32_t chunk_index = 0;
  for (uint64_t start = 0; start < elems; start += max_elems) {
    const uint64_t count = (elems - start < max_elems) ? elems - start : max_elems;
    const size_t seg = 32 + name_len + count * width;
    const size_t payload = 13 + seg;
    if (out) {
      uint8_t* f = out + used;
      orc_encode_frame(type, NULL, 0, f);
      put_le(f + 6, payload, 8);
      orc_encode_reduce_payload(epoch, chunk_index, (uint8_t)(precision ? 1 : 0), NULL, 0, f + 14);
      orc_encode_chunk_segment(name, name_len, global_offset + start, count, scalars + start * width,
                               count * width, f + 27);
    }
    chunk_index++;
    used += 14 + payload;
  }
  return used;
}

/* One frame off the front of a byte stream: FrameParser::next (wire.cpp:38-72),
 * decode_reduce_payload (wire.cpp:90-104), decode_chunk_segment
 * (collective.cpp:90-119).  ORC_EAGAIN when the frame is incomplete. */
int orc_parse_chunk_frame(const uint8_t* in, size_t avail, size_t* frame_bytes, uint8_t* type,
                          uint64_t* epoch, uint32_t* chunk_index, uint8_t* precision, size_t* name_off,
                          size_t* name_len, uint64_t* offset, uint64_t* length, size_t* scalars_off,
                          size_t* scalars_bytes) {
  if (avail < 14) return ORC_EAGAIN;
  if (memcmp(in, "ODLC", 4) != 0) return ORC_ESERIAL;           /* bad frame magic */
  if (in[4] != 1) return ORC_ESERIAL;                           /* unsupported wire version */
  const uint64_t len = get_le(in + 6, 8);
  if (len > (1ull << 33)) return ORC_ESERIAL;                   /* implausible frame length */
  if (avail < 14 + len) return ORC_EAGAIN;
  if (in[5] < 1 || in[5] > 9) return ORC_ESERIAL;               /* unknown message type */
  *type = in[5];
  *frame_bytes = 14 + len;
  const uint8_t* p = in + 14;
  if (len < 13) return ORC_ESERIAL;                             /* truncated reduce payload */
  *epoch = get_le(p, 8);
  *chunk_index = (uint32_t)get_le(p + 8, 4);
  *precision = p[12];
  const uint8_t* s = p + 13;
  const size_t slen = len - 13;
  size_t c = 0;
  if (c + 8 > slen) return ORC_ESERIAL;                         /* truncated chunk segment */
  if (get_le(s, 8) != 1) return ORC_ESERIAL;                    /* exactly one segment */
  c += 8;
  if (c + 8 > slen) return ORC_ESERIAL;
  const uint64_t nl = get_le(s + c, 8);
  c += 8;
  if (nl > slen - c) return ORC_ESERIAL;                        /* truncated chunk segment name */
  *name_off = (size_t)(s - in) + c;
  *name_len = nl;
  c += nl;
  if (c + 16 > slen) return ORC_ESERIAL;
  *offset = get_le(s + c, 8);
  *length = get_le(s + c + 8, 8);
  c += 16;
  *scalars_off = (size_t)(s - in) + c;
  *scalars_bytes = slen - c;
  return ORC_OK;
}
