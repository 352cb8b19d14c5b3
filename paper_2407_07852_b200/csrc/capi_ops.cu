// capi_ops.cu — section 1 of include/diloco_cuda.h: the reference's free
// functions over HOST buffers, staged through the calling thread's device.
//
// Each call mirrors the reference function's checks in the same order and
// leaves caller-owned state untouched when it fails (e.g. adamw_step's
// NumericError leaves m, v and step_count as they were, optim.cpp:66-69).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "engine_impl.hpp"

namespace dlc {

namespace {
thread_local std::string t_err;

// Per-thread staging context: device, stream, a growable device arena and a
// pinned flag word.
struct ThreadCtx {
  int device = -1;
  cudaStream_t stream = nullptr;
  char* arena = nullptr;
  size_t cap = 0;
  int* hflag = nullptr;

  ~ThreadCtx() {
    if (device >= 0) {
      cudaSetDevice(device);
      if (arena) cudaFree(arena);
      if (stream) cudaStreamDestroy(stream);
      if (hflag) cudaFreeHost(hflag);
    }
  }
};
thread_local ThreadCtx t_ctx;

ThreadCtx& ctx() {
  int dev = 0;
  DLC_CUDA(cudaGetDevice(&dev));
  if (t_ctx.device != dev) {
    if (t_ctx.device >= 0) {
      cudaSetDevice(t_ctx.device);
      if (t_ctx.arena) cudaFree(t_ctx.arena);
      if (t_ctx.stream) cudaStreamDestroy(t_ctx.stream);
      if (t_ctx.hflag) cudaFreeHost(t_ctx.hflag);
      cudaSetDevice(dev);
    }
    t_ctx = ThreadCtx{};
    t_ctx.device = dev;
    DLC_CUDA(cudaStreamCreateWithFlags(&t_ctx.stream, cudaStreamNonBlocking));
    DLC_CUDA(cudaMallocHost(&t_ctx.hflag, 64));
  }
  return t_ctx;
}

// Carves `bytes` (256-B aligned pieces) out of the thread arena.
struct Arena {
  ThreadCtx& c;
  size_t used = 0;
  explicit Arena(ThreadCtx& cx, size_t total) : c(cx) {
    if (total > c.cap) {
      if (c.arena) DLC_CUDA(cudaFree(c.arena));
      c.arena = nullptr;
      c.cap = 0;
      DLC_CUDA(cudaMalloc(&c.arena, total));
      c.cap = total;
    }
  }
  template <typename T>
  T* take(size_t count) {
    T* p = reinterpret_cast<T*>(c.arena + used);
    used += (count * sizeof(T) + 255) & ~size_t(255);
    return p;
  }
};

size_t al(size_t bytes) { return (bytes + 255) & ~size_t(255); }

void need(const void* p, size_t n, const char* what) {
  if (n > 0 && p == nullptr) fail(DLC_EINVAL, std::string(what) + ": null pointer");
}

void h2d(void* d, const void* h, size_t bytes, cudaStream_t s) {
  if (bytes) DLC_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s));
}
void d2h(void* h, const void* d, size_t bytes, cudaStream_t s) {
  if (bytes) DLC_CUDA(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s));
}
void finish(ThreadCtx& c) {
  DLC_LAUNCHED("kernel launch");
  DLC_CUDA(cudaStreamSynchronize(c.stream));
}

}  // namespace

void set_error(const std::string& msg) { t_err = msg; }
void clear_error() { t_err.clear(); }

}  // namespace dlc

using namespace dlc;

extern "C" {

int dlc_abi_version(void) { return DLC_ABI_VERSION; }

const char* dlc_last_error(void) { return t_err.c_str(); }

int dlc_device_count(int* count) {
  return guard([&] {
    need(count, 1, "dlc_device_count");
    *count = 0;
    DLC_CUDA(cudaGetDeviceCount(count));
  });
}

int dlc_set_device(int device) { return guard([&] { DLC_CUDA(cudaSetDevice(device)); }); }

int dlc_axpy(float alpha, const float* x, const float* y, size_t n, float* out) {
  return guard([&] {
    need(x, n, "axpy x");
    need(y, n, "axpy y");
    need(out, n, "axpy out");
    if (n == 0) return;
    ThreadCtx& c = ctx();
    Arena a(c, 3 * al(n * 4));
    float *dx = a.take<float>(n), *dy = a.take<float>(n), *dout = a.take<float>(n);
    h2d(dx, x, n * 4, c.stream);
    h2d(dy, y, n * 4, c.stream);
    launch_axpy(alpha, dx, dy, dout, n, c.stream);
    d2h(out, dout, n * 4, c.stream);
    finish(c);
  });
}

int dlc_encode_fp16(const float* v, size_t n, uint16_t* out, int* overflow) {
  return guard([&] {
    need(v, n, "encode_fp16 v");
    need(out, n, "encode_fp16 out");
    if (overflow) *overflow = 0;
    if (n == 0) return;
    ThreadCtx& c = ctx();
    Arena a(c, al(n * 4) + al(n * 2) + 256);
    float* dv = a.take<float>(n);
    uint16_t* dout = a.take<uint16_t>(n);
    int* dflag = a.take<int>(1);
    DLC_CUDA(cudaMemsetAsync(dflag, 0, 4, c.stream));
    h2d(dv, v, n * 4, c.stream);
    launch_encode(dv, dout, dflag, n, c.stream);
    d2h(out, dout, n * 2, c.stream);
    d2h(c.hflag, dflag, 4, c.stream);
    finish(c);
    if (overflow) *overflow = *c.hflag ? 1 : 0;
  });
}

int dlc_decode_fp16(const uint16_t* bits, size_t n, float* out) {
  return guard([&] {
    need(bits, n, "decode_fp16 bits");
    need(out, n, "decode_fp16 out");
    if (n == 0) return;
    ThreadCtx& c = ctx();
    Arena a(c, al(n * 4) + al(n * 2));
    uint16_t* db = a.take<uint16_t>(n);
    float* dout = a.take<float>(n);
    h2d(db, bits, n * 2, c.stream);
    launch_decode(db, dout, n, c.stream);
    d2h(out, dout, n * 4, c.stream);
    finish(c);
  });
}

int dlc_all_finite(const float* v, size_t n, int* all_finite) {
  return guard([&] {
    need(v, n, "all_finite v");
    need(all_finite, 1, "all_finite out");
    *all_finite = 1;
    if (n == 0) return;
    ThreadCtx& c = ctx();
    Arena a(c, al(n * 4) + 256);
    float* dv = a.take<float>(n);
    int* dflag = a.take<int>(1);
    DLC_CUDA(cudaMemsetAsync(dflag, 0, 4, c.stream));
    h2d(dv, v, n * 4, c.stream);
    launch_nonfinite(dv, dflag, n, c.stream);
    d2h(c.hflag, dflag, 4, c.stream);
    finish(c);
    *all_finite = *c.hflag ? 0 : 1;
  });
}

float dlc_lr_at(const dlc_lr_schedule* s, uint64_t step) {
  // optim.cpp:37-56, host scalar (FP32 warmup ramp, FP64 cosine).
  const float base = s->base_lr;
  if (s->warmup_steps > 0 && step <= s->warmup_steps) {
    return base * static_cast<float>(step) / static_cast<float>(s->warmup_steps);
  }
  if (s->decay == DLC_LR_NONE || s->total_steps == 0 || s->total_steps <= s->warmup_steps) return base;
  const float floor_lr = 0.1f * base;
  if (step >= s->total_steps) return floor_lr;
  const double progress = static_cast<double>(step - s->warmup_steps) /
                          static_cast<double>(s->total_steps - s->warmup_steps);
  const double cosine = 0.5 * (1.0 + std::cos(progress * M_PI));
  return static_cast<float>(floor_lr + (base - floor_lr) * cosine);
}

int dlc_adamw_step(dlc_adamw_state* st, const float* params, const float* grad, size_t n, float lr,
                   float* out) {
  return guard([&] {
    need(st, 1, "adamw_step state");
    need(params, n, "adamw_step params");
    need(grad, n, "adamw_step grad");
    need(out, n, "adamw_step out");
    need(st->m, n, "adamw_step m");
    need(st->v, n, "adamw_step v");
    if (lr < 0.0f) fail(DLC_ECONFIG, "adamw_step: negative learning rate");  // optim.cpp:63-65
    // optim.cpp:73-76: bias corrections from host powf at the new step count.
    const uint64_t t = st->step_count + 1;
    AdamWPlain a{st->beta1, st->beta2, st->eps, st->weight_decay, 1.0f - st->beta1, 1.0f - st->beta2,
                 1.0f - std::pow(st->beta1, static_cast<float>(t)),
                 1.0f - std::pow(st->beta2, static_cast<float>(t)), lr};
    int nonfinite = 0;
    if (n > 0) {
      ThreadCtx& c = ctx();
      Arena ar(c, 6 * al(n * 4) + 256);
      float *dp = ar.take<float>(n), *dg = ar.take<float>(n), *dm = ar.take<float>(n),
            *dv = ar.take<float>(n), *dout = ar.take<float>(n);
      int* dflag = ar.take<int>(1);
      DLC_CUDA(cudaMemsetAsync(dflag, 0, 4, c.stream));
      h2d(dg, grad, n * 4, c.stream);
      h2d(dp, params, n * 4, c.stream);
      h2d(dm, st->m, n * 4, c.stream);
      h2d(dv, st->v, n * 4, c.stream);
      launch_nonfinite(dg, dflag, n, c.stream);  // optim.cpp:66-68
      launch_adamw_plain(dp, dg, dm, dv, dout, n, a, c.stream);
      d2h(c.hflag, dflag, 4, c.stream);
      finish(c);
      nonfinite = *c.hflag;
      if (nonfinite) fail(DLC_ENUMERIC, "adamw_step: non-finite gradient");
      d2h(out, dout, n * 4, c.stream);
      d2h(st->m, dm, n * 4, c.stream);
      d2h(st->v, dv, n * 4, c.stream);
      finish(c);
    }
    st->step_count = t;  // optim.cpp:69
  });
}

int dlc_nesterov_step(dlc_nesterov_state* st, const float* params, const float* pg, size_t n, float* out) {
  return guard([&] {
    need(st, 1, "nesterov_step state");
    need(params, n, "nesterov_step params");
    need(pg, n, "nesterov_step pseudo_grad");
    need(out, n, "nesterov_step out");
    need(st->momentum_buf, n, "nesterov_step momentum_buf");
    if (n == 0) return;
    ThreadCtx& c = ctx();
    Arena ar(c, 4 * al(n * 4) + 256);
    float *dp = ar.take<float>(n), *dg = ar.take<float>(n), *db = ar.take<float>(n), *dout = ar.take<float>(n);
    int* dflag = ar.take<int>(1);
    DLC_CUDA(cudaMemsetAsync(dflag, 0, 4, c.stream));
    h2d(dg, pg, n * 4, c.stream);
    h2d(dp, params, n * 4, c.stream);
    h2d(db, st->momentum_buf, n * 4, c.stream);
    launch_nonfinite(dg, dflag, n, c.stream);  // optim.cpp:101-103
    launch_nesterov_plain(dp, dg, db, dout, n, st->lr, st->momentum, c.stream);
    d2h(c.hflag, dflag, 4, c.stream);
    finish(c);
    if (*c.hflag) fail(DLC_ENUMERIC, "nesterov_step: non-finite pseudo-gradient");
    d2h(out, dout, n * 4, c.stream);
    d2h(st->momentum_buf, db, n * 4, c.stream);
    finish(c);
  });
}

float dlc_scaler_scale_loss(const dlc_loss_scaler* s, float loss) { return loss * s->scale; }

int dlc_scaler_unscale_and_check(const dlc_loss_scaler* s, const float* grad, size_t n, float* out,
                                 int* overflow) {
  return guard([&] {
    need(s, 1, "unscale scaler");
    need(grad, n, "unscale grad");
    need(out, n, "unscale out");
    if (overflow) *overflow = 0;
    if (n == 0) return;
    ThreadCtx& c = ctx();
    Arena ar(c, 2 * al(n * 4) + 256);
    float *dg = ar.take<float>(n), *dout = ar.take<float>(n);
    int* dflag = ar.take<int>(1);
    DLC_CUDA(cudaMemsetAsync(dflag, 0, 4, c.stream));
    h2d(dg, grad, n * 4, c.stream);
    launch_unscale(dg, 1.0f / s->scale, dout, dflag, n, c.stream);  // optim.cpp:124
    d2h(out, dout, n * 4, c.stream);
    d2h(c.hflag, dflag, 4, c.stream);
    finish(c);
    if (overflow) *overflow = *c.hflag ? 1 : 0;
  });
}

void dlc_scaler_update(dlc_loss_scaler* s, int overflow) {
  // optim.cpp:137-148 (clamps optim.cpp:13-14)
  if (overflow) {
    s->scale = std::max(s->scale * 0.5f, 0x1p-20f);
    s->consecutive_good = 0;
    return;
  }
  s->consecutive_good += 1;
  if (s->consecutive_good >= s->growth_interval) {
    s->scale = std::min(s->scale * 2.0f, 0x1p24f);
    s->consecutive_good = 0;
  }
}

int dlc_reduce_average(const float* const* contributions, size_t k, size_t n, int precision, float* out) {
  return guard([&] {
    if (k == 0) fail(DLC_ECOLLECTIVE, "reduce_average: no contributions");  // reduce.cpp:48-50
    need(contributions, k, "reduce_average contributions");
    for (size_t j = 0; j < k; ++j) need(contributions[j], n, "reduce_average contribution");
    need(out, n, "reduce_average out");
    if (precision != DLC_FP32 && precision != DLC_FP16) fail(DLC_ECONFIG, "reduce_average: unknown precision");
    if (n == 0) return;
    ThreadCtx& c = ctx();
    Arena ar(c, (k + 1) * al(n * 4) + al(k * sizeof(void*)));
    std::vector<const float*> dptr(k);
    for (size_t j = 0; j < k; ++j) {
      float* d = ar.take<float>(n);
      h2d(d, contributions[j], n * 4, c.stream);
      dptr[j] = d;
    }
    float* dout = ar.take<float>(n);
    const float** dlist = ar.take<const float*>(k);
    h2d(dlist, dptr.data(), k * sizeof(void*), c.stream);
    launch_fold_many(dlist, k, precision == DLC_FP16, dout, n, c.stream);
    d2h(out, dout, n * 4, c.stream);
    finish(c);
  });
}

void dlc_partition_ranges(size_t n, size_t k, size_t* offsets, size_t* lengths) {
  // reduce.cpp:20-31: first n % k ranges one longer.
  const size_t base = k == 0 ? 0 : n / k, rem = k == 0 ? 0 : n % k;
  size_t off = 0;
  for (size_t i = 0; i < k; ++i) {
    lengths[i] = base + (i < rem ? 1 : 0);
    offsets[i] = off;
    off += lengths[i];
  }
}

uint64_t dlc_per_peer_reduce_bytes(size_t n, size_t k, size_t rank, int precision) {
  // reduce.cpp:91-104: direct scatter + ring relay of the all-gather.
  if (k <= 1) return 0;
  const uint64_t w = precision == DLC_FP16 ? 2 : 4;
  const size_t base = n / k, rem = n % k;
  const size_t own = base + (rank < rem ? 1 : 0);
  const size_t nxt = (rank + 1) % k;
  const size_t succ = base + (nxt < rem ? 1 : 0);
  return (uint64_t)(n - own) * w + (uint64_t)(n - succ) * w;
}

uint64_t dlc_fleet_reduce_bytes(size_t n, size_t k, int precision) {
  if (k <= 1) return 0;  // reduce.cpp:106-111
  return 2ull * (k - 1) * (uint64_t)n * (precision == DLC_FP16 ? 2 : 4);
}

uint64_t dlc_rng_key(uint64_t seed, const char* purpose, uint64_t index) {
  // CounterRng::mix over fnv1a64(purpose), rng.hpp:17-31,66-71.
  auto sm = [](uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
  };
  uint64_t h = 0xCBF29CE484222325ull;
  for (const char* p = purpose; p && *p; ++p) {
    h ^= (uint8_t)*p;
    h *= 0x100000001B3ull;
  }
  uint64_t k = sm(seed ^ 0x6A09E667F3BCC909ull);
  k = sm(k ^ h);
  return sm(k ^ index);
}

int dlc_fp16_encode_bits(uint32_t start, size_t n, uint16_t* out) {
  return guard([&] {
    need(out, n, "fp16_encode_bits out");
    if (n == 0) return;
    if ((uint64_t)start + n > (1ull << 32)) fail(DLC_EINVAL, "fp16_encode_bits: range exceeds 2^32");
    ThreadCtx& c = ctx();
    Arena ar(c, al(n * 2));
    uint16_t* d = ar.take<uint16_t>(n);
    launch_encode_bits_range(start, d, n, c.stream);
    d2h(out, d, n * 2, c.stream);
    finish(c);
  });
}

int dlc_fold_push_probe(const void* const* contribs, int k, size_t n, int precision, int tma, void* out,
                        int* nonfinite) {
  return guard([&] {
    if (k < 1 || k > kMaxK) fail(DLC_EINVAL, "fold_push_probe: k must be 1..32");
    if (tma < 0 || tma > 2) fail(DLC_EINVAL, "fold_push_probe: tma must be 0, 1 or 2");
    if (precision != DLC_FP32 && precision != DLC_FP16) fail(DLC_ECONFIG, "unknown precision");
    if (n % 64) fail(DLC_ESHAPE, "fold_push_probe: n must be a multiple of 64");
    if (!contribs || !nonfinite) fail(DLC_EINVAL, "fold_push_probe: null argument");
    need(out, n, "fold_push_probe out");
    const size_t w = precision == DLC_FP16 ? 2 : 4, b = al(n * w);
    ThreadCtx& c = ctx();
    Arena ar(c, b * (k + 1) + 256);
    PtrList in{}, outs{}, flags{};
    for (int j = 0; j < k; ++j) {
      need(contribs[j], n, "fold_push_probe contribution");
      void* d = ar.take<uint8_t>(b);
      h2d(d, contribs[j], n * w, c.stream);
      in.ptr[j] = d;
    }
    void* d_out = ar.take<uint8_t>(b);
    int* d_flag = ar.take<int>(64);
    DLC_CUDA(cudaMemsetAsync(d_flag, 0, sizeof(int), c.stream));
    outs.ptr[0] = d_out;
    flags.ptr[0] = d_flag;
    if (!(tma && launch_fold_push_tma(in, k, precision, outs, 1, flags, 1, n, tma_ctas(k), tma_threads(k), tma - 1,
                                      c.stream)))
      launch_fold_push(in, k, precision, outs, 1, flags, 1, n, 0, c.stream);
    d2h(out, d_out, n * w, c.stream);
    d2h(nonfinite, d_flag, sizeof(int), c.stream);
    finish(c);
  });
}

int dlc_p2p_kernels_probe(int k, size_t n, int precision, int reps, float* ms3) {
  return dlc_p2p_overlap_probe(k, n, precision, reps, 0, ms3, nullptr);
}

int dlc_p2p_overlap_probe(int k, size_t n, int precision, int reps, int fold_ctas, float* ms3, float* overlap_ms) {
  return guard([&] {
    if (k < 2 || k > kMaxK) fail(DLC_EINVAL, "p2p_kernels_probe: k must be 2..32");
    if (precision != DLC_FP32 && precision != DLC_FP16) fail(DLC_ECONFIG, "unknown precision");
    if (n == 0 || reps < 1 || !ms3) fail(DLC_EINVAL, "p2p_kernels_probe: bad argument");
    const size_t w = precision == DLC_FP16 ? 2 : 4;
    const size_t quantum = 64 * 8;  // the engine's owner-slot quantum (engine_impl.hpp kMaxPieces)
    const size_t S = ((n + k - 1) / k + quantum - 1) / quantum * quantum;
    ThreadCtx& c = ctx();
    // dedicated allocations (full-size vectors do not belong in the staging arena)
    std::vector<void*> owned;
    auto dmalloc = [&](size_t bytes) {
      void* p = nullptr;
      DLC_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 256)));
      owned.push_back(p);
      return p;
    };
    cudaEvent_t ev[2] = {nullptr, nullptr};
    try {
      float* tt[2] = {(float*)dmalloc(n * 4), (float*)dmalloc(n * 4)};
      float* bf[2] = {(float*)dmalloc(n * 4), (float*)dmalloc(n * 4)};
      float* x = (float*)dmalloc(n * 4);
      char* send = (char*)dmalloc((size_t)k * S * w);
      char* gather = (char*)dmalloc((size_t)k * S * w);
      int* flags = (int*)dmalloc(kMaxK * sizeof(int));
      DevState* st = (DevState*)dmalloc(sizeof(DevState));
      DLC_CUDA(cudaMemsetAsync(st, 0, sizeof(DevState), c.stream));
      DLC_CUDA(cudaMemsetAsync(flags, 0, kMaxK * sizeof(int), c.stream));
      DLC_CUDA(cudaMemsetAsync(bf[0], 0, n * 4, c.stream));
      launch_rng_fill(1, 0, -0.05f, 0.05f, tt[0], n, c.stream);
      launch_rng_fill(2, 0, -0.05f, 0.05f, x, n, c.stream);
      const Pair ttp{{tt[0], tt[1]}, 0}, bufp{{bf[0], bf[1]}, 0};
      const Pair src{{x, x}, 0}, follow{{x, x}, 1};
      // owner r's view, emulated on one device: the K contributions to a slot are
      // the K rows of the send buffer, the mean goes to K gather rows -- the same
      // DRAM bytes one GPU serves and receives in the real exchange
      PtrList in{}, outs{}, fl{}, slots{};
      for (int j = 0; j < k; ++j) {
        in.ptr[j] = send + (size_t)j * S * w;
        outs.ptr[j] = gather + (size_t)j * S * w;
        fl.ptr[j] = flags + j;
        slots.ptr[j] = gather + (size_t)j * S * w;
      }
      DLC_CUDA(cudaEventCreate(&ev[0]));
      DLC_CUDA(cudaEventCreate(&ev[1]));
      auto timed = [&](auto&& launch) {
        launch();  // warm
        DLC_CUDA(cudaEventRecord(ev[0], c.stream));
        for (int i = 0; i < reps; ++i) launch();
        DLC_CUDA(cudaEventRecord(ev[1], c.stream));
        DLC_CUDA(cudaEventSynchronize(ev[1]));
        float ms = 0.f;
        DLC_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[1]));
        DLC_CUDA(cudaGetLastError());
        return ms / (float)reps;
      };
      ms3[0] = timed([&] {
        launch_pseudo_grad_piece(ttp, src, st, send, precision, k, S, 0, S, n, 0, c.stream);
      });
      ms3[1] = timed([&] {
        if (!launch_fold_push_tma(in, k, precision, outs, k, fl, k, S, tma_ctas(k), tma_threads(k), fold_kernel(),
                                  c.stream))
          launch_fold_push(in, k, precision, outs, k, fl, k, S, kFoldCtas, c.stream);
      });
      ms3[2] = timed([&] {
        launch_nesterov_p2p_piece(ttp, bufp, follow, slots, k, S, 0, S, precision, st, 0.7f, 0.9f, n, 0, c.stream);
      });
      if (overlap_ms) {
        // K4 on the staging stream while the fold (fold_ctas CTAs) runs back to
        // back on a second stream for at least as long: on-chip interference
        // between the two, without NVLink in the picture
        cudaStream_t s2 = nullptr;
        DLC_CUDA(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
        cudaEvent_t f0 = nullptr, f1 = nullptr;
        DLC_CUDA(cudaEventCreate(&f0));
        DLC_CUDA(cudaEventCreate(&f1));
        const int freps = std::max(1, (int)std::ceil(3.0 * reps * ms3[2] / std::max(ms3[1], 1e-3f)));
        DLC_CUDA(cudaStreamSynchronize(c.stream));
        DLC_CUDA(cudaEventRecord(f0, s2));
        for (int i = 0; i < freps; ++i)
          if (!launch_fold_push_tma(in, k, precision, outs, k, fl, k, S, fold_ctas > 0 ? fold_ctas : tma_ctas(k),
                                    tma_threads(k), fold_kernel(), s2))
            launch_fold_push(in, k, precision, outs, k, fl, k, S, fold_ctas > 0 ? fold_ctas : kFoldCtas, s2);
        DLC_CUDA(cudaEventRecord(f1, s2));
        DLC_CUDA(cudaEventRecord(ev[0], c.stream));
        for (int i = 0; i < reps; ++i)
          launch_nesterov_p2p_piece(ttp, bufp, follow, slots, k, S, 0, S, precision, st, 0.7f, 0.9f, n, 0, c.stream);
        DLC_CUDA(cudaEventRecord(ev[1], c.stream));
        DLC_CUDA(cudaEventSynchronize(ev[1]));
        DLC_CUDA(cudaEventSynchronize(f1));
        float a = 0.f, b = 0.f;
        DLC_CUDA(cudaEventElapsedTime(&a, ev[0], ev[1]));
        DLC_CUDA(cudaEventElapsedTime(&b, f0, f1));
        overlap_ms[0] = a / (float)reps;   // K4 per launch while the fold runs
        overlap_ms[1] = b / (float)freps;  // fold per launch (partly alone at the end)
        cudaEventDestroy(f0);
        cudaEventDestroy(f1);
        cudaStreamDestroy(s2);
      }
    } catch (...) {
      for (cudaEvent_t e : ev)
        if (e) cudaEventDestroy(e);
      for (void* p : owned) cudaFree(p);
      throw;
    }
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
    for (void* p : owned) DLC_CUDA(cudaFree(p));
  });
}

}  // extern "C"
