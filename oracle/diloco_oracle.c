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
