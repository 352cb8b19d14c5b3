// device.cuh — device helpers shared by the kernel translation units: grid
// shapes (streaming window, persistent), thread indexing, the counter RNG and
// the per-element arithmetic of SURVEY.md Appendix A (FP32 evaluation order of
// the reference, explicit round-to-nearest ops).
#pragma once

#include <algorithm>
#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "kernels.cuh"

namespace dlc {

namespace {

// Wall-clock nanoseconds (%globaltimer), independent of the SM clock.
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Persistent grid for the setup / host-staged helpers (not on the hot path).
template <typename Kern>
int grid_persist(Kern kernel, size_t work) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> per_sm;
  int bps;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = per_sm.find((const void*)kernel);
    if (it == per_sm.end()) {
      int b = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, kThreads, 0);
      it = per_sm.emplace((const void*)kernel, std::max(b, 1)).first;
    }
    bps = it->second;
  }
  const size_t cap = (size_t)num_sms() * (size_t)bps;
  const size_t need = (work + kThreads - 1) / kThreads;
  return (int)std::max<size_t>(1, std::min(cap, need));
}

// Streaming-window grid: one CTA per kThreads*U work items.
template <int U>
int grid_window(size_t items) {
  return (int)std::max<size_t>(1, (items + (size_t)kThreads * U - 1) / ((size_t)kThreads * U));
}

__device__ __forceinline__ size_t gtid() { return (size_t)blockIdx.x * blockDim.x + threadIdx.x; }
__device__ __forceinline__ size_t gstride() { return (size_t)gridDim.x * blockDim.x; }
// first work item of this thread in the streaming window (items u*kThreads apart)
template <int U>
__device__ __forceinline__ size_t wbase() {
  return (size_t)blockIdx.x * kThreads * U + threadIdx.x;
}

// ---- counter RNG, rng.hpp:17-56 ---------------------------------------------
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ float rng_uniform_at(uint64_t key, uint64_t i, float lo, float hi) {
  const float u = __fmul_rn((float)(splitmix64(key + (i + 1) * 0x9E3779B97F4A7C15ull) >> 40), 0x1p-24f);
  return __fadd_rn(lo, __fmul_rn(__fsub_rn(hi, lo), u));
}

// ---- per-element arithmetic, Appendix A of SURVEY.md ------------------------
struct AdamScalars {
  float b1, b2, eps, wd, omb1, omb2, c1, c2, lr;
};

// optim.cpp:84-90 for one element; p is the OLD parameter.
__device__ __forceinline__ float adamw_elem(float p, float g, float& m, float& v, const AdamScalars& s) {
  m = __fadd_rn(__fmul_rn(s.b1, m), __fmul_rn(s.omb1, g));
  v = __fadd_rn(__fmul_rn(s.b2, v), __fmul_rn(__fmul_rn(s.omb2, g), g));
  const float mh = __fdiv_rn(m, s.c1);
  const float vh = __fdiv_rn(v, s.c2);
  const float upd = __fadd_rn(__fdiv_rn(mh, __fadd_rn(__fsqrt_rn(vh), s.eps)), __fmul_rn(s.wd, p));
  return __fsub_rn(p, __fmul_rn(s.lr, upd));
}

// optim.cpp:111-112 for one element.
__device__ __forceinline__ float nesterov_elem(float p, float g, float& buf, float lr, float mu) {
  buf = __fadd_rn(__fmul_rn(mu, buf), g);
  return __fsub_rn(p, __fmul_rn(lr, __fadd_rn(g, __fmul_rn(mu, buf))));
}

// tensor.cpp:126 with alpha = -1: theta_t + (-1 * theta_local).
__device__ __forceinline__ float delta_elem(float tt, float tl) { return __fadd_rn(tt, __fmul_rn(-1.0f, tl)); }

__device__ __forceinline__ float4 decode4(uint2 w) {
  return make_float4(fp16_decode(lo16(w.x)), fp16_decode(hi16(w.x)), fp16_decode(lo16(w.y)), fp16_decode(hi16(w.y)));
}

__device__ __forceinline__ float* sel(const Pair& p, int i) { return i ? p.ptr[1] : p.ptr[0]; }

// theta_local as held right now: theta_t[ocur] while the two are equal by
// construction (Pair::follow + DevState::lalias), else the live p buffer.
__device__ __forceinline__ const float* local_src(const Pair& tl, const Pair& tt, const DevState* st) {
  return (tl.follow && st->lalias) ? sel(tt, st->ocur) : sel(tl, st->cur);
}

// One thread after K1 (and after the fused window boundary): the skip decision,
// step counter, lr record and scaler_update (engine.cpp:57-67, optim.cpp:69,
// optim.cpp:137-148 with clamps :13-14).
__device__ __forceinline__ void inner_finalize(DevState* st, const float* lr_tab, int pingpong, int fused) {
  const int fi = st->found_inf;
  // a fused delta is the outer step's input only if p' became theta_local
  st->delta_ready = fused && !fi;
  const uint64_t t = st->step_count + 1;
  if (!fi) {
    if (pingpong) st->cur ^= 1;  // the freshly written buffers become live
    st->lalias = 0;              // theta_local now lives in p[cur]
    st->step_count = t;
    st->last_lr = lr_tab[t];
  } else {
    st->last_lr = 0.0f;
    st->overflow_skips += 1;
  }
  st->last_overflow = fi;
  if (fi) {
    const float s = __fmul_rn(st->scale, 0.5f);
    st->scale = (s < 0x1p-20f) ? 0x1p-20f : s;
    st->good = 0;
  } else {
    st->good += 1;
    if (st->good >= st->growth) {
      const float s = __fmul_rn(st->scale, 2.0f);
      st->scale = (0x1p24f < s) ? 0x1p24f : s;
      st->good = 0;
    }
  }
  st->inner_step += 1;  // data cursor always advances (engine.cpp:103)
  st->found_inf = 0;
}

// After an outer step, applied or skipped: theta_local := theta_t
// (engine.cpp:141-143, recorded as DevState::lalias for PINGPONG engines),
// the result and the epoch (engine.cpp:144).
__device__ __forceinline__ void k4_finalize(DevState* st, bool applied, const Pair& tl) {
  if (tl.follow) st->lalias = 1;  // theta_local := theta_t (engine.cpp:141-143) without the copy
  st->last_applied = applied ? 1 : 0;
  st->outer_skips += applied ? 0 : 1;
  st->outer_epoch += 1;  // engine.cpp:144
}

// K2 of a single worker in the reduce precision: the delta as the outer step
// sees it (FP16: encoded once at the source; the mean of one contribution
// re-encodes to the same code), non-finite OR into `bad`.
template <int PREC>
__device__ __forceinline__ float solo_delta(float tt, float tl, bool& bad) {
  const float d = delta_elem(tt, tl);  // engine.cpp:122
  if (PREC == 0) {
    bad |= !finite_f(d);
    return d;
  }
  const uint16_t h = fp16_encode(d);
  bad |= fp16_nonfinite(h);
  return fp16_decode(h);
}

}  // namespace

}  // namespace dlc
