// kernels.cu — DiLoCo hot-path kernels for B200 (sm_100a).
//
// Memory-bound elementwise and reduction work: no tensor cores.  The hot
// kernels use the streaming-window distribution described in kernels.cuh: one
// CTA per 256*U consecutive 128-bit vectors, evict-first (.cs) loads/stores, a
// scalar tail on CTA 0, and CTA-level OR reductions (__syncthreads_or + one
// atomicOr per CTA that saw a non-finite value) for the global flags.
//
// Arithmetic follows the reference's FP32 evaluation order exactly (see
// common.cuh); citations are to /root/reference/proj.
#include <algorithm>
#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "kernels.cuh"

namespace dlc {

namespace {

int g_sms = 0;

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

// =============================================================================
// K1: fused unscale + overflow OR + AdamW.
// =============================================================================

constexpr int kU1 = 1;  // vectors per thread (tools/tune_stream: best for 4R3W)

__global__ void __launch_bounds__(kThreads) adamw_kernel(AdamWArgs a) {
  DevState* st = a.st;
  // INPLACE mode: the pre-pass already decided; an overflowed step writes nothing.
  if (!a.pingpong && *(volatile int*)&st->found_inf != 0) return;
  const int cur = a.pingpong ? st->cur : 0;
  const int nxt = a.pingpong ? (cur ^ 1) : 0;
  const uint64_t t = st->step_count + 1;
  const AdamScalars s{a.b1, a.b2, a.eps, a.wd, a.omb1, a.omb2, a.corr1[t], a.corr2[t], a.lr[t]};
  const float inv = __fdiv_rn(1.0f, st->scale);  // optim.cpp:124 (exact: power of two)
  const float* pc = (a.pingpong && st->lalias) ? (st->ocur ? a.tt[1] : a.tt[0]) : (cur ? a.p[1] : a.p[0]);
  const float* mc = cur ? a.m[1] : a.m[0];
  const float* vc = cur ? a.v[1] : a.v[0];
  float* pn = nxt ? a.p[1] : a.p[0];
  float* mn = nxt ? a.m[1] : a.m[0];
  float* vn = nxt ? a.v[1] : a.v[0];
  bool bad = false;
  const size_t n4 = a.n / 4, b = wbase<kU1>();
  float4 p[kU1], g[kU1], m[kU1], v[kU1];
#pragma unroll
  for (int u = 0; u < kU1; ++u) {
    const size_t j = b + u * kThreads;
    if (j < n4) {
      g[u] = ld_stream(reinterpret_cast<const float4*>(a.g) + j);
      p[u] = ld_stream(reinterpret_cast<const float4*>(pc) + j);
      m[u] = ld_stream(reinterpret_cast<const float4*>(mc) + j);
      v[u] = ld_stream(reinterpret_cast<const float4*>(vc) + j);
    }
  }
#pragma unroll
  for (int u = 0; u < kU1; ++u) {
    const size_t j = b + u * kThreads;
    if (j < n4) {
      const float4 gu = make_float4(__fmul_rn(g[u].x, inv), __fmul_rn(g[u].y, inv), __fmul_rn(g[u].z, inv),
                                    __fmul_rn(g[u].w, inv));
      bad |= !(finite_f(gu.x) && finite_f(gu.y) && finite_f(gu.z) && finite_f(gu.w));
      float4 po;
      po.x = adamw_elem(p[u].x, gu.x, m[u].x, v[u].x, s);
      po.y = adamw_elem(p[u].y, gu.y, m[u].y, v[u].y, s);
      po.z = adamw_elem(p[u].z, gu.z, m[u].z, v[u].z, s);
      po.w = adamw_elem(p[u].w, gu.w, m[u].w, v[u].w, s);
      st_stream(reinterpret_cast<float4*>(pn) + j, po);
      st_stream(reinterpret_cast<float4*>(mn) + j, m[u]);
      st_stream(reinterpret_cast<float4*>(vn) + j, v[u]);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < a.n - n4 * 4) {
    const size_t e = n4 * 4 + threadIdx.x;
    const float gu = __fmul_rn(a.g[e], inv);
    bad |= !finite_f(gu);
    float mm = mc[e], vv = vc[e];
    pn[e] = adamw_elem(pc[e], gu, mm, vv, s);
    mn[e] = mm;
    vn[e] = vv;
  }
  if (a.pingpong) block_or_flag(bad, &st->found_inf);
}

// One thread: the skip decision, step counter, lr record and scaler_update
// (engine.cpp:57-67, optim.cpp:69, optim.cpp:137-148 with clamps :13-14).
__global__ void adamw_finalize_kernel(DevState* st, const float* lr_tab, int pingpong) {
  const int fi = st->found_inf;
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

// INPLACE pre-pass (optim.cpp:127-132): found_inf |= !isfinite(g * (1/scale)).
__global__ void __launch_bounds__(kThreads) unscale_check_kernel(const float* g, DevState* st, size_t n) {
  const float inv = __fdiv_rn(1.0f, st->scale);
  bool bad = false;
  const size_t n4 = n / 4, b = wbase<2>();
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const size_t j = b + u * kThreads;
    if (j < n4) {
      const float4 x = ld_stream(reinterpret_cast<const float4*>(g) + j);
      bad |= !(finite_f(__fmul_rn(x.x, inv)) && finite_f(__fmul_rn(x.y, inv)) && finite_f(__fmul_rn(x.z, inv)) &&
               finite_f(__fmul_rn(x.w, inv)));
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < n - n4 * 4) bad |= !finite_f(__fmul_rn(g[n4 * 4 + threadIdx.x], inv));
  block_or_flag(bad, &st->found_inf);
}

// Out-of-place AdamW on an already unscaled, finite gradient (adamw_step with
// the host-side checks done by the caller; optim.cpp:83-91).
__global__ void __launch_bounds__(kThreads) adamw_plain_kernel(const float* p, const float* g, float* m, float* v,
                                                               float* out, size_t n, AdamWPlain a) {
  const AdamScalars s{a.b1, a.b2, a.eps, a.wd, a.omb1, a.omb2, a.corr1, a.corr2, a.lr};
  for (size_t e = gtid(); e < n; e += gstride()) {
    float mm = m[e], vv = v[e];
    out[e] = adamw_elem(p[e], g[e], mm, vv, s);
    m[e] = mm;
    v[e] = vv;
  }
}

// =============================================================================
// K2: pseudo-gradient into the collective send buffer.
// =============================================================================

constexpr int kU2 = 2;

template <int PREC>
__global__ void __launch_bounds__(kThreads) pseudo_grad_kernel(Pair ttp, Pair tl, const DevState* st, void* out,
                                                               int* flag, size_t off, size_t len) {
  const float* T = sel(ttp, st->ocur) + off;
  const float* L = local_src(tl, ttp, st) + off;
  bool bad = false;
  const size_t n4 = len / 4, b = wbase<kU2>();
  float4 x[kU2], y[kU2];
#pragma unroll
  for (int u = 0; u < kU2; ++u) {
    const size_t j = b + u * kThreads;
    if (j < n4) {
      x[u] = ld_stream(reinterpret_cast<const float4*>(T) + j);
      y[u] = ld_stream(reinterpret_cast<const float4*>(L) + j);
    }
  }
#pragma unroll
  for (int u = 0; u < kU2; ++u) {
    const size_t j = b + u * kThreads;
    if (j < n4) {
      const float4 d = make_float4(delta_elem(x[u].x, y[u].x), delta_elem(x[u].y, y[u].y),
                                   delta_elem(x[u].z, y[u].z), delta_elem(x[u].w, y[u].w));
      if (PREC == 0) {
        bad |= !(finite_f(d.x) && finite_f(d.y) && finite_f(d.z) && finite_f(d.w));
        st_stream(reinterpret_cast<float4*>(static_cast<float*>(out) + off) + j, d);
      } else {
        const uint16_t h0 = fp16_encode(d.x), h1 = fp16_encode(d.y), h2 = fp16_encode(d.z), h3 = fp16_encode(d.w);
        bad |= fp16_nonfinite(h0) | fp16_nonfinite(h1) | fp16_nonfinite(h2) | fp16_nonfinite(h3);
        st_stream(reinterpret_cast<uint2*>(static_cast<uint16_t*>(out) + off) + j,
                  make_uint2(pack2(h0, h1), pack2(h2, h3)));
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < len - n4 * 4) {
    const size_t e = n4 * 4 + threadIdx.x;
    const float d = delta_elem(T[e], L[e]);
    if (PREC == 0) {
      bad |= !finite_f(d);
      static_cast<float*>(out)[off + e] = d;
    } else {
      const uint16_t h = fp16_encode(d);
      bad |= fp16_nonfinite(h);
      static_cast<uint16_t*>(out)[off + e] = h;
    }
  }
  block_or_flag(bad, flag);
}

// =============================================================================
// K3: ordered fold of K contributions (reduce.cpp:33-44 / 70-88).
// Each thread owns 8 consecutive elements; contributions are visited in rank
// order 0..K-1 so the FP32 sum is bit-identical to fold_mean.  Contributions
// may live in peer GPUs' memory (DLC_MODE_P2P): the loads then travel NVLink.
// =============================================================================

template <int IN>
__device__ __forceinline__ void load8(const void* base, size_t e8, float (&x)[8]) {
  if (IN == 1) {
    const uint4 w = ld_stream(reinterpret_cast<const uint4*>(base) + e8);
    x[0] = fp16_decode(lo16(w.x)); x[1] = fp16_decode(hi16(w.x));
    x[2] = fp16_decode(lo16(w.y)); x[3] = fp16_decode(hi16(w.y));
    x[4] = fp16_decode(lo16(w.z)); x[5] = fp16_decode(hi16(w.z));
    x[6] = fp16_decode(lo16(w.w)); x[7] = fp16_decode(hi16(w.w));
  } else {
    const float4 a = ld_stream(reinterpret_cast<const float4*>(base) + 2 * e8);
    const float4 b = ld_stream(reinterpret_cast<const float4*>(base) + 2 * e8 + 1);
    x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
    x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
    if (IN == 2) {
#pragma unroll
      for (int q = 0; q < 8; ++q) x[q] = fp16_decode(fp16_encode(x[q]));
    }
  }
}

// Raw 8-element group of one contribution (16 B of FP16 codes, 32 B of FP32),
// loaded first and decoded later, so the K loads of a group are all in flight
// together (for peer memory they are NVLink round trips).
template <int IN>
struct Raw8 {
  float4 a, b;
};
template <>
struct Raw8<1> {
  uint4 w;
};

// volatile: the K loads of a group stay adjacent (the scheduler would
// otherwise interleave the decode of load j with the issue of load j + 1)
__device__ __forceinline__ uint4 ld_cs_v4(const void* p) {
  uint4 v;
  asm volatile("ld.global.cs.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

template <int IN>
__device__ __forceinline__ void ld_raw(const void* base, size_t e8, Raw8<IN>& r) {
  if constexpr (IN == 1) {
    r.w = ld_cs_v4(reinterpret_cast<const uint4*>(base) + e8);
  } else {
    const uint4 a = ld_cs_v4(reinterpret_cast<const float4*>(base) + 2 * e8);
    const uint4 b = ld_cs_v4(reinterpret_cast<const float4*>(base) + 2 * e8 + 1);
    r.a = make_float4(__uint_as_float(a.x), __uint_as_float(a.y), __uint_as_float(a.z), __uint_as_float(a.w));
    r.b = make_float4(__uint_as_float(b.x), __uint_as_float(b.y), __uint_as_float(b.z), __uint_as_float(b.w));
  }
}

template <int IN>
__device__ __forceinline__ void unpack(const Raw8<IN>& r, float (&x)[8]) {
  if constexpr (IN == 1) {
    x[0] = fp16_decode(lo16(r.w.x)); x[1] = fp16_decode(hi16(r.w.x));
    x[2] = fp16_decode(lo16(r.w.y)); x[3] = fp16_decode(hi16(r.w.y));
    x[4] = fp16_decode(lo16(r.w.z)); x[5] = fp16_decode(hi16(r.w.z));
    x[6] = fp16_decode(lo16(r.w.w)); x[7] = fp16_decode(hi16(r.w.w));
  } else {
    x[0] = r.a.x; x[1] = r.a.y; x[2] = r.a.z; x[3] = r.a.w;
    x[4] = r.b.x; x[5] = r.b.y; x[6] = r.b.z; x[7] = r.b.w;
    if (IN == 2) {
#pragma unroll
      for (int q = 0; q < 8; ++q) x[q] = fp16_decode(fp16_encode(x[q]));
    }
  }
}

template <int IN>
__device__ __forceinline__ float load1(const void* base, size_t e) {
  if (IN == 1) return fp16_decode(reinterpret_cast<const uint16_t*>(base)[e]);
  const float x = reinterpret_cast<const float*>(base)[e];
  return IN == 2 ? fp16_decode(fp16_encode(x)) : x;
}

template <int OUT>
__device__ __forceinline__ bool store1(void* out, size_t e, float mean) {
  if (OUT == 1) {
    const uint16_t h = fp16_encode(mean);
    reinterpret_cast<uint16_t*>(out)[e] = h;
    return fp16_nonfinite(h);
  }
  const float y = OUT == 2 ? fp16_decode(fp16_encode(mean)) : mean;
  reinterpret_cast<float*>(out)[e] = y;
  return !finite_f(y);
}

template <int IN, int OUT>
__global__ void __launch_bounds__(kThreads) fold_kernel(const __grid_constant__ PtrList in, int k, void* out,
                                                        int* flag, size_t n) {
  const float divisor = (float)k;  // reduce.cpp:36
  bool bad = false;
  const size_t n8 = n / 8, i = gtid();
  if (i < n8) {
    float acc[8], x[8];
    load8<IN>(in.ptr[0], i, acc);
    for (int j = 1; j < k; ++j) {
      load8<IN>(in.ptr[j], i, x);
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = __fadd_rn(acc[q], x[q]);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = __fdiv_rn(acc[q], divisor);
    if (OUT == 1) {
      uint16_t h[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        h[q] = fp16_encode(acc[q]);
        bad |= fp16_nonfinite(h[q]);
      }
      st_stream(reinterpret_cast<uint4*>(out) + i,
                make_uint4(pack2(h[0], h[1]), pack2(h[2], h[3]), pack2(h[4], h[5]), pack2(h[6], h[7])));
    } else {
      if (OUT == 2) {
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = fp16_decode(fp16_encode(acc[q]));
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) bad |= !finite_f(acc[q]);
      float4* o = reinterpret_cast<float4*>(out) + 2 * i;
      st_stream(o, make_float4(acc[0], acc[1], acc[2], acc[3]));
      st_stream(o + 1, make_float4(acc[4], acc[5], acc[6], acc[7]));
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < n - n8 * 8) {
    const size_t e = n8 * 8 + threadIdx.x;
    float acc = load1<IN>(in.ptr[0], e);
    for (int j = 1; j < k; ++j) acc = __fadd_rn(acc, load1<IN>(in.ptr[j], e));
    bad |= store1<OUT>(out, e, __fdiv_rn(acc, divisor));
  }
  if (flag) block_or_flag(bad, flag);
}

// K3 fused with the all-gather: the owner pushes its mean to every rank.
// KK > 0: the contributor count at compile time, so the KK loads of a group
// are issued back to back (KK NVLink round trips in flight per thread instead
// of one); KK == 0: any k, one load at a time.
template <int PREC, int KK>
__global__ void __launch_bounds__(kThreads) fold_push_kernel(const __grid_constant__ PtrList in, int k,
                                                             const __grid_constant__ PtrList outs, int nout,
                                                             const __grid_constant__ PtrList flags, size_t n) {
  const float divisor = (float)k;  // reduce.cpp:36
  bool bad = false;
  const size_t n8 = n / 8;
  // grid-stride: a persistent grid of a few CTAs leaves the other SMs to the
  // HBM-bound K2 / K4 pieces running concurrently on the main stream
  for (size_t i = gtid(); i < n8; i += gstride()) {
    float acc[8], x[8];
    if constexpr (KK > 0) {
      Raw8<PREC> raw[KK];
#pragma unroll
      for (int j = 0; j < KK; ++j) ld_raw<PREC>(in.ptr[j], i, raw[j]);
      unpack<PREC>(raw[0], acc);
#pragma unroll
      for (int j = 1; j < KK; ++j) {  // rank order (reduce.cpp:37-43)
        unpack<PREC>(raw[j], x);
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = __fadd_rn(acc[q], x[q]);
      }
    } else {
      load8<PREC>(in.ptr[0], i, acc);
      for (int j = 1; j < k; ++j) {
        load8<PREC>(in.ptr[j], i, x);
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = __fadd_rn(acc[q], x[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = __fdiv_rn(acc[q], divisor);
    if (PREC == 1) {
      uint16_t h[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        h[q] = fp16_encode(acc[q]);
        bad |= fp16_nonfinite(h[q]);
      }
      const uint4 w = make_uint4(pack2(h[0], h[1]), pack2(h[2], h[3]), pack2(h[4], h[5]), pack2(h[6], h[7]));
      for (int o = 0; o < nout; ++o) st_stream(reinterpret_cast<uint4*>(const_cast<void*>(outs.ptr[o])) + i, w);
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) bad |= !finite_f(acc[q]);
      const float4 a = make_float4(acc[0], acc[1], acc[2], acc[3]), b = make_float4(acc[4], acc[5], acc[6], acc[7]);
      for (int o = 0; o < nout; ++o) {
        float4* d = reinterpret_cast<float4*>(const_cast<void*>(outs.ptr[o])) + 2 * i;
        st_stream(d, a);
        st_stream(d + 1, b);
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < n - n8 * 8) {
    const size_t e = n8 * 8 + threadIdx.x;
    float acc = load1<PREC>(in.ptr[0], e);
    for (int j = 1; j < k; ++j) acc = __fadd_rn(acc, load1<PREC>(in.ptr[j], e));
    const float mean = __fdiv_rn(acc, divisor);
    for (int o = 0; o < nout; ++o) bad |= store1<PREC>(const_cast<void*>(outs.ptr[o]), e, mean);
  }
  if (__syncthreads_or(bad ? 1 : 0) && threadIdx.x == 0) {
    for (int o = 0; o < nout; ++o) *reinterpret_cast<volatile int*>(const_cast<void*>(flags.ptr[o])) = 1;
  }
  // The CTA's pushed slots are visible system-wide before the barrier that
  // follows: the __syncthreads_or above orders every thread's stores before
  // this (cumulative) system-scope fence of one thread.
  if (threadIdx.x == 0) __threadfence_system();
}

// ---- K3 fused with the all-gather, TMA version -------------------------------
// The same rank-ordered fold as fold_push_kernel, with the data moved by the
// bulk-copy engine (cp.async.bulk) instead of per-thread loads and stores:
// one elected thread streams 8 KB tiles of the KK inputs (peer memory over
// NVLink, or local HBM) into a STAGES-deep shared-memory ring, arming an
// mbarrier with the expected bytes; 128 threads fold the tile in rank order
// into an output tile, which the elected thread bulk-stores into every
// destination (the owners' mean slots in every rank's gather buffer).  Each CTA
// keeps STAGES * KK * 8 KB of NVLink reads in flight with a handful of
// instructions, so a few dozen CTAs saturate the links and leave the SMs to the
// HBM-bound K2 / K4 pieces.
constexpr int kTmaThreads = 128;
constexpr int kTmaTileBytes = 8192;
constexpr int kTmaStages = 3;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_load(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst_smem)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void bulk_store(void* dst, const void* src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src_smem)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

template <int PREC, int KK>
__global__ void __launch_bounds__(kTmaThreads) fold_push_tma_kernel(const __grid_constant__ PtrList in,
                                                                    const __grid_constant__ PtrList outs, int nout,
                                                                    const __grid_constant__ PtrList flags,
                                                                    size_t n) {
  constexpr int W = PREC == 1 ? 2 : 4;
  constexpr int TILE = kTmaTileBytes / W;  // elements per tile
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* in_buf = smem;                                          // [STAGES][KK][8 KB]
  uint8_t* out_buf = smem + kTmaStages * KK * kTmaTileBytes;       // [STAGES][8 KB]
  uint64_t* bar = reinterpret_cast<uint64_t*>(out_buf + kTmaStages * kTmaTileBytes);  // [STAGES]
  const float divisor = (float)KK;  // reduce.cpp:36
  const size_t ntiles = (n + TILE - 1) / TILE;
  const size_t mine = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const bool leader = threadIdx.x == 0;
  auto tile_of = [&](size_t i) { return blockIdx.x + i * gridDim.x; };
  auto tile_bytes = [&](size_t t) {
    const size_t e = t * (size_t)TILE;
    return (uint32_t)((n - e < (size_t)TILE ? n - e : (size_t)TILE) * W);
  };
  auto issue = [&](size_t i) {  // tile i of this CTA into stage i % STAGES
    const int st = (int)(i % kTmaStages);
    const size_t t = tile_of(i);
    const uint32_t bytes = tile_bytes(t);
    mbar_expect_tx(&bar[st], bytes * KK);
#pragma unroll
    for (int j = 0; j < KK; ++j)
      bulk_load(in_buf + ((size_t)st * KK + j) * kTmaTileBytes,
                static_cast<const uint8_t*>(in.ptr[j]) + t * (size_t)kTmaTileBytes, bytes, &bar[st]);
  };
  if (leader) {
    for (int st = 0; st < kTmaStages; ++st) mbar_init(&bar[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (leader)
    for (size_t i = 0; i < mine && i < (size_t)kTmaStages; ++i) issue(i);
  bool bad = false;
  for (size_t i = 0; i < mine; ++i) {
    const int st = (int)(i % kTmaStages);
    const size_t t = tile_of(i);
    const uint32_t bytes = tile_bytes(t);
    if (leader && i >= (size_t)kTmaStages) bulk_wait_read<kTmaStages - 1>();  // out_buf[st] read by its store
    __syncthreads();
    mbar_wait(&bar[st], (uint32_t)((i / kTmaStages) & 1));
    const uint8_t* src = in_buf + (size_t)st * KK * kTmaTileBytes;
    uint8_t* dst = out_buf + (size_t)st * kTmaTileBytes;
    for (uint32_t off = threadIdx.x * 16; off < bytes; off += kTmaThreads * 16) {  // 16 B per thread and step
      constexpr int E = 16 / W;  // 8 FP16 or 4 FP32 elements
      float acc[E], x[E];
#pragma unroll
      for (int j = 0; j < KK; ++j) {  // rank order (reduce.cpp:37-43)
        const uint4 v = *reinterpret_cast<const uint4*>(src + (size_t)j * kTmaTileBytes + off);
        if constexpr (PREC == 1) {
          x[0] = fp16_decode(lo16(v.x)); x[1] = fp16_decode(hi16(v.x));
          x[2] = fp16_decode(lo16(v.y)); x[3] = fp16_decode(hi16(v.y));
          x[4] = fp16_decode(lo16(v.z)); x[5] = fp16_decode(hi16(v.z));
          x[6] = fp16_decode(lo16(v.w)); x[7] = fp16_decode(hi16(v.w));
        } else {
          x[0] = __uint_as_float(v.x); x[1] = __uint_as_float(v.y);
          x[2] = __uint_as_float(v.z); x[3] = __uint_as_float(v.w);
        }
#pragma unroll
        for (int q = 0; q < E; ++q) acc[q] = j == 0 ? x[q] : __fadd_rn(acc[q], x[q]);
      }
      uint4 o;
      if constexpr (PREC == 1) {
        uint16_t h[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          h[q] = fp16_encode(__fdiv_rn(acc[q], divisor));
          bad |= fp16_nonfinite(h[q]);
        }
        o = make_uint4(pack2(h[0], h[1]), pack2(h[2], h[3]), pack2(h[4], h[5]), pack2(h[6], h[7]));
      } else {
        float m[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          m[q] = __fdiv_rn(acc[q], divisor);
          bad |= !finite_f(m[q]);
        }
        o = make_uint4(__float_as_uint(m[0]), __float_as_uint(m[1]), __float_as_uint(m[2]), __float_as_uint(m[3]));
      }
      *reinterpret_cast<uint4*>(dst + off) = o;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // our smem writes -> the bulk store's reads
    __syncthreads();  // every thread is done with in_buf[st] and out_buf[st]
    if (leader) {
      for (int o = 0; o < nout; ++o)
        bulk_store(static_cast<uint8_t*>(const_cast<void*>(outs.ptr[o])) + t * (size_t)kTmaTileBytes, dst, bytes);
      bulk_commit();
      if (i + kTmaStages < mine) issue(i + kTmaStages);  // in_buf[st] is free again
    }
  }
  if (__syncthreads_or(bad ? 1 : 0) && threadIdx.x == 0) {
    for (int o = 0; o < nout; ++o) *reinterpret_cast<volatile int*>(const_cast<void*>(flags.ptr[o])) = 1;
  }
  if (leader) {
    bulk_wait_all();  // every bulk store of this CTA has landed
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __threadfence_system();  // ... and is visible system-wide before the barrier that follows
  }
}

size_t fold_push_tma_smem(int k) { return (size_t)kTmaStages * (k + 1) * kTmaTileBytes + kTmaStages * 8; }

// Scatter half of the push/push P2P mover: row q of `src` (this rank's piece of
// owner q's slot, in local HBM) is stored into row `me` of owner q's receive
// buffer over NVLink.  Consecutive 16-byte vectors go to different owners so
// every link carries traffic at once.
__global__ void __launch_bounds__(kThreads) scatter_push_kernel(const __grid_constant__ PtrList src,
                                                                const __grid_constant__ PtrList dst, int nrow,
                                                                size_t bytes) {
  const size_t n16 = bytes / 16, total = n16 * (size_t)nrow;
  for (size_t i = gtid(); i < total; i += gstride()) {
    const int q = (int)(i % (size_t)nrow);
    const size_t j = i / (size_t)nrow;
    const uint4 v = ld_stream(reinterpret_cast<const uint4*>(src.ptr[q]) + j);
    st_stream(reinterpret_cast<uint4*>(const_cast<void*>(dst.ptr[q])) + j, v);
  }
  __syncthreads();
  if (threadIdx.x == 0) __threadfence_system();  // the CTA's stores land before the barrier that follows
}

// =============================================================================
// K4: finite-gated Nesterov on theta_t + theta_local refresh (engine.cpp:136-144).
// =============================================================================

// one 4-element vector of K4: applied -> Nesterov + three stores, else copy
// (L4 == nullptr: theta_local follows theta_t, no refresh store)
__device__ __forceinline__ void k4_vec(bool applied, float4* T4, float4* B4, float4* L4, float4 d, float lr,
                                       float mu) {
  if (!applied && !L4) return;
  const float4 t = ld_stream(T4);
  if (applied) {
    float4 b = ld_stream(B4), o;
    o.x = nesterov_elem(t.x, d.x, b.x, lr, mu);
    o.y = nesterov_elem(t.y, d.y, b.y, lr, mu);
    o.z = nesterov_elem(t.z, d.z, b.z, lr, mu);
    o.w = nesterov_elem(t.w, d.w, b.w, lr, mu);
    st_stream(T4, o);
    st_stream(B4, b);
    if (L4) st_stream(L4, o);
  } else if (L4) {
    st_stream(L4, t);
  }
}

__device__ __forceinline__ void k4_scalar(bool applied, float* T, float* B, float* L, float d, float lr, float mu) {
  if (applied) {
    float b = *B;
    const float o = nesterov_elem(*T, d, b, lr, mu);
    *T = o;
    *B = b;
    if (L) *L = o;
  } else if (L) {
    *L = *T;
  }
}

__device__ __forceinline__ void k4_finalize(DevState* st, bool applied, const Pair& tl) {
  if (tl.follow) st->lalias = 1;  // theta_local := theta_t (engine.cpp:141-143) without the copy
  st->last_applied = applied ? 1 : 0;
  st->outer_skips += applied ? 0 : 1;
  st->outer_epoch += 1;  // engine.cpp:144
}

template <int PREC>
__global__ void __launch_bounds__(kThreads) nesterov_outer_kernel(Pair ttp, Pair bufp, Pair tl, const void* dbar,
                                                                  const int* flags, int nflags, DevState* st,
                                                                  float lr, float mu, size_t n) {
  __shared__ int s_nonfinite;
  if (threadIdx.x == 0) {
    int nf = 0;
    for (int j = 0; j < nflags; ++j) nf |= flags[j];
    s_nonfinite = nf;
  }
  __syncthreads();
  const bool applied = s_nonfinite == 0;
  float* tt = sel(ttp, st->ocur);
  float* buf = sel(bufp, st->ocur);
  float* L = tl.follow ? nullptr : sel(tl, st->cur);
  const size_t n4 = n / 4, j = gtid();
  if (j < n4) {
    float4 d = make_float4(0.f, 0.f, 0.f, 0.f);
    if (applied) {
      d = PREC == 0 ? ld_stream(reinterpret_cast<const float4*>(dbar) + j)
                    : decode4(ld_stream(reinterpret_cast<const uint2*>(dbar) + j));
    }
    k4_vec(applied, reinterpret_cast<float4*>(tt) + j, reinterpret_cast<float4*>(buf) + j,
           L ? reinterpret_cast<float4*>(L) + j : nullptr, d, lr, mu);
  }
  if (blockIdx.x == 0 && threadIdx.x < n - n4 * 4) {
    const size_t e = n4 * 4 + threadIdx.x;
    const float d = PREC == 0 ? reinterpret_cast<const float*>(dbar)[e]
                              : fp16_decode(reinterpret_cast<const uint16_t*>(dbar)[e]);
    k4_scalar(applied, tt + e, buf + e, L ? L + e : nullptr, d, lr, mu);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) k4_finalize(st, applied, tl);
}

// ---- NVLink flag barrier ----------------------------------------------------
__global__ void flag_barrier_kernel(const __grid_constant__ PtrList remote, const uint64_t* local, int k, int me,
                                    uint64_t epoch, int* err) {
  const int j = threadIdx.x;
  if (j < k && j != me) {
    __threadfence_system();  // everything this GPU wrote before the barrier is visible first
    *reinterpret_cast<volatile unsigned long long*>(const_cast<void*>(remote.ptr[j])) = epoch;
    const long long start = clock64();
    const volatile unsigned long long* mine = reinterpret_cast<const volatile unsigned long long*>(local + j);
    while (*mine < epoch) {
      if (clock64() - start > (1ll << 35)) {  // ~17 s at 2 GHz: a peer is gone
        atomicExch(err, 1);
        break;
      }
    }
    __threadfence_system();
  }
  __syncthreads();
}

// ---- pipelined P2P pieces ----------------------------------------------------
// CTA b covers owner q = b % K, vectors [(b / K) * 256, ...) of that owner's
// piece, so every piece launch spreads over all slots.

template <int PREC>
__device__ __forceinline__ void pseudo_grad_piece_block(const float* T, const float* L, void* send, size_t blk, int k,
                                                        size_t S, size_t po, size_t plen, size_t n) {
  const int q = (int)(blk % (unsigned)k);
  const size_t j = (blk / (unsigned)k) * kThreads + threadIdx.x;
  const size_t e0 = (size_t)q * S + po + 4 * j;
  if (4 * j >= plen || e0 >= n) return;
  if (e0 + 3 < n) {
    const float4 x = ld_stream(reinterpret_cast<const float4*>(T + e0));
    const float4 y = ld_stream(reinterpret_cast<const float4*>(L + e0));
    const float4 d = make_float4(delta_elem(x.x, y.x), delta_elem(x.y, y.y), delta_elem(x.z, y.z),
                                 delta_elem(x.w, y.w));
    if (PREC == 0) {
      st_stream(reinterpret_cast<float4*>(static_cast<float*>(send) + e0), d);
    } else {
      st_stream(reinterpret_cast<uint2*>(static_cast<uint16_t*>(send) + e0),
                make_uint2(pack2(fp16_encode(d.x), fp16_encode(d.y)), pack2(fp16_encode(d.z), fp16_encode(d.w))));
    }
  } else {
    for (size_t e = e0; e < n; ++e) {
      const float d = delta_elem(T[e], L[e]);
      if (PREC == 0)
        static_cast<float*>(send)[e] = d;
      else
        static_cast<uint16_t*>(send)[e] = fp16_encode(d);
    }
  }
}

// `nblk` logical blocks (one 256-vector window of one owner slot each) over a
// grid that may be smaller (DLC_P2P_PIECE_CTAS), leaving SMs to the fold.
template <int PREC>
__global__ void __launch_bounds__(kThreads) pseudo_grad_piece_kernel(Pair ttp, Pair tl, const DevState* st,
                                                                     void* send, int k, size_t S, size_t po,
                                                                     size_t plen, size_t n, size_t nblk) {
  const float* T = sel(ttp, st->ocur);
  const float* L = local_src(tl, ttp, st);
  for (size_t b = blockIdx.x; b < nblk; b += gridDim.x) pseudo_grad_piece_block<PREC>(T, L, send, b, k, S, po, plen, n);
}

template <int PREC>
__global__ void __launch_bounds__(kThreads) pseudo_grad_push_piece_kernel(Pair ttp, Pair tl, const DevState* st,
                                                                          const __grid_constant__ PtrList rows, int k,
                                                                          size_t S, size_t po, size_t plen,
                                                                          size_t n) {
  const int q = (int)(blockIdx.x % (unsigned)k);
  const size_t j = (size_t)(blockIdx.x / (unsigned)k) * kThreads + threadIdx.x;
  const size_t e0 = (size_t)q * S + po + 4 * j;  // global element
  const size_t o0 = po + 4 * j;                  // offset inside owner q's row
  void* row = const_cast<void*>(rows.ptr[q]);
  if (4 * j < plen && e0 < n) {
    const float* T = sel(ttp, st->ocur);
    const float* L = local_src(tl, ttp, st);
    if (e0 + 3 < n) {
      const float4 x = ld_stream(reinterpret_cast<const float4*>(T + e0));
      const float4 y = ld_stream(reinterpret_cast<const float4*>(L + e0));
      const float4 d = make_float4(delta_elem(x.x, y.x), delta_elem(x.y, y.y), delta_elem(x.z, y.z),
                                   delta_elem(x.w, y.w));
      if (PREC == 0) {
        st_stream(reinterpret_cast<float4*>(static_cast<float*>(row) + o0), d);
      } else {
        st_stream(reinterpret_cast<uint2*>(static_cast<uint16_t*>(row) + o0),
                  make_uint2(pack2(fp16_encode(d.x), fp16_encode(d.y)), pack2(fp16_encode(d.z), fp16_encode(d.w))));
      }
    } else {
      for (size_t e = e0; e < n; ++e) {
        const float d = delta_elem(T[e], L[e]);
        if (PREC == 0)
          static_cast<float*>(row)[o0 + (e - e0)] = d;
        else
          static_cast<uint16_t*>(row)[o0 + (e - e0)] = fp16_encode(d);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) __threadfence_system();  // the CTA's stores land before the barrier that follows
}

template <int PREC>
__device__ __forceinline__ void nesterov_p2p_piece_block(const float* T, const float* B, float* To, float* Bo, float* L,
                                                         const PtrList& slots, size_t blk, int k, size_t S, size_t po,
                                                         size_t plen, float lr, float mu, size_t n) {
  const int q = (int)(blk % (unsigned)k);
  const size_t j = (blk / (unsigned)k) * kThreads + threadIdx.x;
  const size_t e0 = (size_t)q * S + po + 4 * j;
  if (4 * j >= plen || e0 >= n) return;
  const void* dbar = slots.ptr[q];
  const size_t o0 = po + 4 * j;  // offset inside owner q's mean slot
  if (e0 + 3 < n) {
    const float4 d = PREC == 0 ? ld_stream(reinterpret_cast<const float4*>(static_cast<const float*>(dbar) + o0))
                               : decode4(ld_stream(reinterpret_cast<const uint2*>(
                                     static_cast<const uint16_t*>(dbar) + o0)));
    const float4 t = ld_stream(reinterpret_cast<const float4*>(T + e0));
    float4 b = ld_stream(reinterpret_cast<const float4*>(B + e0)), o;
    o.x = nesterov_elem(t.x, d.x, b.x, lr, mu);
    o.y = nesterov_elem(t.y, d.y, b.y, lr, mu);
    o.z = nesterov_elem(t.z, d.z, b.z, lr, mu);
    o.w = nesterov_elem(t.w, d.w, b.w, lr, mu);
    st_stream(reinterpret_cast<float4*>(To + e0), o);
    st_stream(reinterpret_cast<float4*>(Bo + e0), b);
    if (L) st_stream(reinterpret_cast<float4*>(L + e0), o);
  } else {
    for (size_t e = e0; e < n; ++e) {
      const size_t o = o0 + (e - e0);
      const float d = PREC == 0 ? static_cast<const float*>(dbar)[o]
                                : fp16_decode(static_cast<const uint16_t*>(dbar)[o]);
      float b = B[e];
      const float v = nesterov_elem(T[e], d, b, lr, mu);
      To[e] = v;
      Bo[e] = b;
      if (L) L[e] = v;
    }
  }
}

template <int PREC>
__global__ void __launch_bounds__(kThreads) nesterov_p2p_piece_kernel(Pair ttp, Pair bufp, Pair tl,
                                                                      const __grid_constant__ PtrList slots, int k,
                                                                      size_t S, size_t po, size_t plen,
                                                                      DevState* st, float lr, float mu, size_t n,
                                                                      size_t nblk) {
  const int oc = st->ocur;
  const float* T = sel(ttp, oc);
  const float* B = sel(bufp, oc);
  float* To = sel(ttp, oc ^ 1);
  float* Bo = sel(bufp, oc ^ 1);
  float* L = tl.follow ? nullptr : sel(tl, st->cur);
  for (size_t b = blockIdx.x; b < nblk; b += gridDim.x)
    nesterov_p2p_piece_block<PREC>(T, B, To, Bo, L, slots, b, k, S, po, plen, lr, mu, n);
}

// Gate of the pipelined P2P step: flip `ocur` when all K owner flags are clean
// (engine.cpp:136-139), else theta_local := theta_t (engine.cpp:143).
__global__ void __launch_bounds__(kThreads) p2p_finish_kernel(Pair ttp, Pair tl, const __grid_constant__ PtrList flags,
                                                              int k, DevState* st, size_t n) {
  __shared__ int s_skip;
  if (threadIdx.x == 0) {
    int nf = 0;
    for (int j = 0; j < k; ++j) nf |= *reinterpret_cast<const volatile int*>(flags.ptr[j]);
    s_skip = nf;
  }
  __syncthreads();
  const int skip = s_skip;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (!skip) st->ocur ^= 1;
    k4_finalize(st, !skip, tl);
  }
  if (!skip || tl.follow) return;
  const float* T = sel(ttp, st->ocur);  // unchanged on a skip
  float* L = sel(tl, st->cur);
  for (size_t e = gtid(); e < n; e += gstride()) L[e] = T[e];
}

// ---- K2 + K4 fused for K = 1 -------------------------------------------------
// Speculative: the new theta_t and momentum go to the idle buffers of their
// ping-pong pairs, so a skip only has to leave `ocur` unflipped.
template <int PREC>
__device__ __forceinline__ float solo_delta(float tt, float tl, bool& bad) {
  const float d = delta_elem(tt, tl);  // engine.cpp:122
  if (PREC == 0) {
    bad |= !finite_f(d);
    return d;
  }
  const uint16_t h = fp16_encode(d);  // encode once at the source; the mean of one
  bad |= fp16_nonfinite(h);           // contribution re-encodes to the same code
  return fp16_decode(h);
}

template <int PREC>
__global__ void __launch_bounds__(kThreads) outer_solo_kernel(Pair ttp, Pair bufp, Pair tl, const float* src,
                                                              DevState* st, float lr, float mu, size_t off,
                                                              size_t len) {
  const int oc = st->ocur;
  const float* T = sel(ttp, oc) + off;
  const float* B = sel(bufp, oc) + off;
  float* To = sel(ttp, oc ^ 1) + off;
  float* Bo = sel(bufp, oc ^ 1) + off;
  float* Ld = tl.follow ? nullptr : sel(tl, st->cur) + off;
  const float* Ls = src ? src + off : local_src(tl, ttp, st) + off;
  bool bad = false;
  const size_t n4 = len / 4, j = gtid();
  if (j < n4) {
    const float4 t = ld_stream(reinterpret_cast<const float4*>(T) + j);
    const float4 l = ld_stream(reinterpret_cast<const float4*>(Ls) + j);
    float4 b = ld_stream(reinterpret_cast<const float4*>(B) + j), o;
    o.x = nesterov_elem(t.x, solo_delta<PREC>(t.x, l.x, bad), b.x, lr, mu);
    o.y = nesterov_elem(t.y, solo_delta<PREC>(t.y, l.y, bad), b.y, lr, mu);
    o.z = nesterov_elem(t.z, solo_delta<PREC>(t.z, l.z, bad), b.z, lr, mu);
    o.w = nesterov_elem(t.w, solo_delta<PREC>(t.w, l.w, bad), b.w, lr, mu);
    st_stream(reinterpret_cast<float4*>(To) + j, o);
    st_stream(reinterpret_cast<float4*>(Bo) + j, b);
    if (Ld) st_stream(reinterpret_cast<float4*>(Ld) + j, o);
  }
  if (blockIdx.x == 0 && threadIdx.x < len - n4 * 4) {
    const size_t e = n4 * 4 + threadIdx.x;
    float bb = B[e];
    const float o = nesterov_elem(T[e], solo_delta<PREC>(T[e], Ls[e], bad), bb, lr, mu);
    To[e] = o;
    Bo[e] = bb;
    if (Ld) Ld[e] = o;
  }
  block_or_flag(bad, &st->delta_nonfinite);
}

// After all chunks: flip `ocur` when every delta was finite (engine.cpp:136-139);
// on a skip, theta_local := theta_t (engine.cpp:143).  The skip path is rare, so
// the grid is small and persistent; applied steps exit at once.
__global__ void __launch_bounds__(kThreads) outer_solo_finish_kernel(Pair ttp, Pair tl, DevState* st, size_t n) {
  const int skip = *reinterpret_cast<volatile int*>(&st->delta_nonfinite);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (!skip) st->ocur ^= 1;
    k4_finalize(st, !skip, tl);
  }
  if (!skip || tl.follow) return;
  const float* T = sel(ttp, st->ocur);  // unchanged on a skip
  float* L = sel(tl, st->cur);
  for (size_t e = gtid(); e < n; e += gstride()) L[e] = T[e];
}

__global__ void __launch_bounds__(kThreads) nesterov_plain_kernel(const float* p, const float* g, float* buf,
                                                                  float* out, size_t n, float lr, float mu) {
  for (size_t e = gtid(); e < n; e += gstride()) {
    float b = buf[e];
    out[e] = nesterov_elem(p[e], g[e], b, lr, mu);
    buf[e] = b;
  }
}

// =============================================================================
// elementwise helpers (host-staged API, synthetic inputs, probes)
// =============================================================================

__global__ void __launch_bounds__(kThreads) axpy_kernel(float alpha, const float* x, const float* y, float* out,
                                                        size_t n) {
  for (size_t e = gtid(); e < n; e += gstride()) out[e] = __fadd_rn(y[e], __fmul_rn(alpha, x[e]));
}

__global__ void __launch_bounds__(kThreads) encode_kernel(const float* x, uint16_t* out, int* flag, size_t n) {
  bool bad = false;
  for (size_t e = gtid(); e < n; e += gstride()) {
    const uint16_t h = fp16_encode(x[e]);
    bad |= fp16_nonfinite(h);
    out[e] = h;
  }
  if (flag) block_or_flag(bad, flag);
}

__global__ void __launch_bounds__(kThreads) decode_kernel(const uint16_t* b, float* out, size_t n) {
  for (size_t e = gtid(); e < n; e += gstride()) out[e] = fp16_decode(b[e]);
}

__global__ void __launch_bounds__(kThreads) nonfinite_kernel(const float* x, int* flag, size_t n) {
  bool bad = false;
  for (size_t e = gtid(); e < n; e += gstride()) bad |= !finite_f(x[e]);
  block_or_flag(bad, flag);
}

__global__ void __launch_bounds__(kThreads) nonfinite_codes_kernel(const uint16_t* b, int* flag, size_t n) {
  bool bad = false;
  for (size_t e = gtid(); e < n; e += gstride()) bad |= fp16_nonfinite(b[e]);
  block_or_flag(bad, flag);
}

// reduce.cpp:46-89 for any k: contributions visited in index order.
__global__ void __launch_bounds__(kThreads) fold_many_kernel(const float* const* ptrs, size_t k, int fp16,
                                                             float* out, size_t n) {
  const float divisor = (float)k;
  for (size_t e = gtid(); e < n; e += gstride()) {
    float acc = ptrs[0][e];
    if (fp16) acc = fp16_decode(fp16_encode(acc));
    for (size_t j = 1; j < k; ++j) {
      const float x = ptrs[j][e];
      acc = __fadd_rn(acc, fp16 ? fp16_decode(fp16_encode(x)) : x);
    }
    const float mean = __fdiv_rn(acc, divisor);
    out[e] = fp16 ? fp16_decode(fp16_encode(mean)) : mean;
  }
}

__global__ void __launch_bounds__(kThreads) unscale_kernel(const float* g, float inv, float* out, int* flag,
                                                           size_t n) {
  bool bad = false;
  for (size_t e = gtid(); e < n; e += gstride()) {
    const float y = __fmul_rn(g[e], inv);
    bad |= !finite_f(y);
    out[e] = y;
  }
  block_or_flag(bad, flag);
}

__global__ void __launch_bounds__(kThreads) scale_gradient_kernel(const float* g, const DevState* st, float* out,
                                                                  size_t n) {
  const float s = st->scale;
  const size_t n4 = n / 4, j = gtid();
  if (j < n4) {
    const float4 x = ld_stream(reinterpret_cast<const float4*>(g) + j);
    st_stream(reinterpret_cast<float4*>(out) + j,
              make_float4(__fmul_rn(x.x, s), __fmul_rn(x.y, s), __fmul_rn(x.z, s), __fmul_rn(x.w, s)));
  }
  if (blockIdx.x == 0 && threadIdx.x < n - n4 * 4) out[n4 * 4 + threadIdx.x] = __fmul_rn(g[n4 * 4 + threadIdx.x], s);
}

__global__ void __launch_bounds__(kThreads) rng_fill_kernel(uint64_t key, uint64_t first, float lo, float hi,
                                                            float* out, size_t n) {
  for (size_t e = gtid(); e < n; e += gstride()) out[e] = rng_uniform_at(key, first + e, lo, hi);
}

__global__ void __launch_bounds__(kThreads) rng_perturb_kernel(const float* tt, uint64_t key, float lo, float hi,
                                                               float* out, size_t n) {
  for (size_t e = gtid(); e < n; e += gstride()) out[e] = __fsub_rn(tt[e], rng_uniform_at(key, e, lo, hi));
}

__global__ void __launch_bounds__(kThreads) encode_bits_kernel(uint32_t start, uint16_t* out, size_t n) {
  for (size_t e = gtid(); e < n; e += gstride()) out[e] = fp16_encode(__uint_as_float(start + (uint32_t)e));
}

__global__ void __launch_bounds__(kThreads) copy_kernel(const float* src, float* dst, size_t n) {
  const size_t n4 = n / 4, j = gtid();
  if (j < n4) st_stream(reinterpret_cast<float4*>(dst) + j, ld_stream(reinterpret_cast<const float4*>(src) + j));
  if (blockIdx.x == 0 && threadIdx.x < n - n4 * 4) dst[n4 * 4 + threadIdx.x] = src[n4 * 4 + threadIdx.x];
}

}  // namespace

// ---- launchers ----------------------------------------------------------------

int num_sms() {
  if (g_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms <= 0) g_sms = 148;
  }
  return g_sms;
}

void launch_adamw(const AdamWArgs& a, cudaStream_t s) {
  if (!a.pingpong)
    unscale_check_kernel<<<grid_window<2>(a.n / 4), kThreads, 0, s>>>(a.g, a.st, a.n);
  adamw_kernel<<<grid_window<kU1>(a.n / 4), kThreads, 0, s>>>(a);
  adamw_finalize_kernel<<<1, 1, 0, s>>>(a.st, a.lr, a.pingpong);
}

void launch_adamw_plain(const float* p, const float* g, float* m, float* v, float* out, size_t n,
                        const AdamWPlain& a, cudaStream_t s) {
  if (n == 0) return;
  adamw_plain_kernel<<<grid_persist(adamw_plain_kernel, n), kThreads, 0, s>>>(p, g, m, v, out, n, a);
}

void launch_pseudo_grad(Pair tt, Pair tl, const DevState* st, void* out, int precision, int* flag, size_t off,
                        size_t len, cudaStream_t s) {
  const int grid = grid_window<kU2>(len / 4);
  if (precision == 0)
    pseudo_grad_kernel<0><<<grid, kThreads, 0, s>>>(tt, tl, st, out, flag, off, len);
  else
    pseudo_grad_kernel<1><<<grid, kThreads, 0, s>>>(tt, tl, st, out, flag, off, len);
}

void launch_fold(const PtrList& in, int k, int in_kind, void* out, int out_kind, int* flag, size_t n,
                 cudaStream_t s) {
  const int grid = grid_window<1>(n / 8);
#define DLC_FOLD(I, O)                                                      \
  if (in_kind == I && out_kind == O) {                                      \
    fold_kernel<I, O><<<grid, kThreads, 0, s>>>(in, k, out, flag, n);       \
    return;                                                                 \
  }
  DLC_FOLD(0, 0) DLC_FOLD(0, 1) DLC_FOLD(0, 2) DLC_FOLD(1, 0) DLC_FOLD(1, 1) DLC_FOLD(1, 2)
  DLC_FOLD(2, 0) DLC_FOLD(2, 1) DLC_FOLD(2, 2)
#undef DLC_FOLD
}

void launch_nesterov_outer(Pair tt, Pair buf, Pair tl, const void* dbar, int precision, const int* flags,
                           int nflags, DevState* st, float lr, float mu, size_t n, cudaStream_t s) {
  const int grid = grid_window<1>(n / 4);
  if (precision == 0)
    nesterov_outer_kernel<0><<<grid, kThreads, 0, s>>>(tt, buf, tl, dbar, flags, nflags, st, lr, mu, n);
  else
    nesterov_outer_kernel<1><<<grid, kThreads, 0, s>>>(tt, buf, tl, dbar, flags, nflags, st, lr, mu, n);
}

void launch_fold_push(const PtrList& in, int k, int precision, const PtrList& outs, int nout, const PtrList& flags,
                      size_t n, int ctas, cudaStream_t s) {
  const int grid = ctas > 0 ? std::min(ctas, grid_window<1>(n / 8)) : grid_window<1>(n / 8);
#define DLC_FOLD_PUSH(P, KK) fold_push_kernel<P, KK><<<grid, kThreads, 0, s>>>(in, k, outs, nout, flags, n)
#define DLC_FOLD_PUSH_K(P)      \
  switch (k) {                  \
    case 2: DLC_FOLD_PUSH(P, 2); break; \
    case 3: DLC_FOLD_PUSH(P, 3); break; \
    case 4: DLC_FOLD_PUSH(P, 4); break; \
    case 5: DLC_FOLD_PUSH(P, 5); break; \
    case 6: DLC_FOLD_PUSH(P, 6); break; \
    case 7: DLC_FOLD_PUSH(P, 7); break; \
    case 8: DLC_FOLD_PUSH(P, 8); break; \
    default: DLC_FOLD_PUSH(P, 0); break; \
  }
  if (precision == 0) {
    DLC_FOLD_PUSH_K(0)
  } else {
    DLC_FOLD_PUSH_K(1)
  }
#undef DLC_FOLD_PUSH_K
#undef DLC_FOLD_PUSH
}

bool launch_fold_push_tma(const PtrList& in, int k, int precision, const PtrList& outs, int nout,
                          const PtrList& flags, size_t n, int ctas, cudaStream_t s) {
  const size_t smem = fold_push_tma_smem(k);
  const int W = precision == 1 ? 2 : 4;
  const size_t ntiles = (n + kTmaTileBytes / W - 1) / (kTmaTileBytes / W);
  const int grid = (int)std::max<size_t>(1, std::min<size_t>(ctas > 0 ? ctas : num_sms(), ntiles));
#define DLC_TMA(P, KK)                                                                                   \
  {                                                                                                      \
    static unsigned attr_devices = 0; /* per-device function attribute, set once */                      \
    int dev = 0;                                                                                         \
    cudaGetDevice(&dev);                                                                                 \
    if (!(attr_devices & (1u << (dev & 31)))) {                                                          \
      cudaFuncSetAttribute(fold_push_tma_kernel<P, KK>, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                           (int)fold_push_tma_smem(KK));                                                 \
      attr_devices |= 1u << (dev & 31);                                                                  \
    }                                                                                                    \
    fold_push_tma_kernel<P, KK><<<grid, kTmaThreads, smem, s>>>(in, outs, nout, flags, n);               \
    return true;                                                                                         \
  }
#define DLC_TMA_K(P)             \
  switch (k) {                   \
    case 2: DLC_TMA(P, 2)        \
    case 3: DLC_TMA(P, 3)        \
    case 4: DLC_TMA(P, 4)        \
    case 5: DLC_TMA(P, 5)        \
    case 6: DLC_TMA(P, 6)        \
    case 7: DLC_TMA(P, 7)        \
    case 8: DLC_TMA(P, 8)        \
    default: return false;       \
  }
  if (precision == 0) {
    DLC_TMA_K(0)
  } else {
    DLC_TMA_K(1)
  }
#undef DLC_TMA_K
#undef DLC_TMA
}

void launch_scatter_push(const PtrList& src, const PtrList& dst, int nrow, size_t bytes, int ctas, cudaStream_t s) {
  const size_t vecs = bytes / 16 * (size_t)nrow;
  const int grid = (int)std::max<size_t>(1, std::min<size_t>(ctas > 0 ? ctas : 4 * num_sms(), (vecs + kThreads - 1) / kThreads));
  scatter_push_kernel<<<grid, kThreads, 0, s>>>(src, dst, nrow, bytes);
}

void launch_flag_barrier(const PtrList& remote, const uint64_t* local, int k, int me, uint64_t epoch, int* err,
                         cudaStream_t s) {
  flag_barrier_kernel<<<1, 32, 0, s>>>(remote, local, k, me, epoch, err);
}

void launch_pseudo_grad_piece(Pair tt, Pair tl, const DevState* st, void* send, int precision, int k, size_t S,
                              size_t po, size_t plen, size_t n, int ctas, cudaStream_t s) {
  const size_t nblk = std::max<size_t>(1, (plen / 4 + kThreads - 1) / kThreads) * (size_t)k;
  const int grid = (int)(ctas > 0 ? std::min<size_t>(nblk, (size_t)ctas) : nblk);
  if (precision == 0)
    pseudo_grad_piece_kernel<0><<<grid, kThreads, 0, s>>>(tt, tl, st, send, k, S, po, plen, n, nblk);
  else
    pseudo_grad_piece_kernel<1><<<grid, kThreads, 0, s>>>(tt, tl, st, send, k, S, po, plen, n, nblk);
}

void launch_pseudo_grad_push_piece(Pair tt, Pair tl, const DevState* st, const PtrList& rows, int precision, int k,
                                   size_t S, size_t po, size_t plen, size_t n, cudaStream_t s) {
  const int grid = (int)(std::max<size_t>(1, (plen / 4 + kThreads - 1) / kThreads) * (size_t)k);
  if (precision == 0)
    pseudo_grad_push_piece_kernel<0><<<grid, kThreads, 0, s>>>(tt, tl, st, rows, k, S, po, plen, n);
  else
    pseudo_grad_push_piece_kernel<1><<<grid, kThreads, 0, s>>>(tt, tl, st, rows, k, S, po, plen, n);
}

void launch_nesterov_p2p_piece(Pair tt, Pair buf, Pair tl, const PtrList& slots, int k, size_t S, size_t po,
                               size_t plen, int precision, DevState* st, float lr, float mu, size_t n, int ctas,
                               cudaStream_t s) {
  const size_t nblk = std::max<size_t>(1, (plen / 4 + kThreads - 1) / kThreads) * (size_t)k;
  const int grid = (int)(ctas > 0 ? std::min<size_t>(nblk, (size_t)ctas) : nblk);
  if (precision == 0)
    nesterov_p2p_piece_kernel<0><<<grid, kThreads, 0, s>>>(tt, buf, tl, slots, k, S, po, plen, st, lr, mu, n, nblk);
  else
    nesterov_p2p_piece_kernel<1><<<grid, kThreads, 0, s>>>(tt, buf, tl, slots, k, S, po, plen, st, lr, mu, n, nblk);
}

void launch_p2p_finish(Pair tt, Pair tl, const PtrList& flags, int k, DevState* st, size_t n, cudaStream_t s) {
  p2p_finish_kernel<<<num_sms() * 4, kThreads, 0, s>>>(tt, tl, flags, k, st, n);
}

void launch_outer_solo_chunk(Pair tt, Pair buf, Pair tl, const float* src, int precision, DevState* st, float lr,
                             float mu, size_t off, size_t len, cudaStream_t s) {
  const int grid = grid_window<1>(len / 4);
  if (precision == 0)
    outer_solo_kernel<0><<<grid, kThreads, 0, s>>>(tt, buf, tl, src, st, lr, mu, off, len);
  else
    outer_solo_kernel<1><<<grid, kThreads, 0, s>>>(tt, buf, tl, src, st, lr, mu, off, len);
}

void launch_outer_solo_finish(Pair tt, Pair tl, DevState* st, size_t n, cudaStream_t s) {
  outer_solo_finish_kernel<<<num_sms() * 4, kThreads, 0, s>>>(tt, tl, st, n);
}

void launch_outer_solo_fused(Pair tt, Pair buf, Pair tl, const float* src, int precision, DevState* st, float lr,
                             float mu, size_t n, cudaStream_t s) {
  launch_outer_solo_chunk(tt, buf, tl, src, precision, st, lr, mu, 0, n, s);
  launch_outer_solo_finish(tt, tl, st, n, s);
}

void launch_nesterov_plain(const float* p, const float* g, float* buf, float* out, size_t n, float lr, float mu,
                           cudaStream_t s) {
  if (n == 0) return;
  nesterov_plain_kernel<<<grid_persist(nesterov_plain_kernel, n), kThreads, 0, s>>>(p, g, buf, out, n, lr, mu);
}

void launch_axpy(float alpha, const float* x, const float* y, float* out, size_t n, cudaStream_t s) {
  if (n == 0) return;
  axpy_kernel<<<grid_persist(axpy_kernel, n), kThreads, 0, s>>>(alpha, x, y, out, n);
}

void launch_encode(const float* x, uint16_t* out, int* flag, size_t n, cudaStream_t s) {
  if (n == 0) return;
  encode_kernel<<<grid_persist(encode_kernel, n), kThreads, 0, s>>>(x, out, flag, n);
}

void launch_decode(const uint16_t* b, float* out, size_t n, cudaStream_t s) {
  if (n == 0) return;
  decode_kernel<<<grid_persist(decode_kernel, n), kThreads, 0, s>>>(b, out, n);
}

void launch_nonfinite(const float* x, int* flag, size_t n, cudaStream_t s) {
  if (n == 0) return;
  nonfinite_kernel<<<grid_persist(nonfinite_kernel, n), kThreads, 0, s>>>(x, flag, n);
}

void launch_nonfinite_codes(const uint16_t* b, int* flag, size_t n, cudaStream_t s) {
  if (n == 0) return;
  nonfinite_codes_kernel<<<grid_persist(nonfinite_codes_kernel, n), kThreads, 0, s>>>(b, flag, n);
}

void launch_fold_many(const float* const* ptrs, size_t k, int fp16, float* out, size_t n, cudaStream_t s) {
  if (n == 0 || k == 0) return;
  fold_many_kernel<<<grid_persist(fold_many_kernel, n), kThreads, 0, s>>>(ptrs, k, fp16, out, n);
}

void launch_unscale(const float* g, float inv, float* out, int* flag, size_t n, cudaStream_t s) {
  if (n == 0) return;
  unscale_kernel<<<grid_persist(unscale_kernel, n), kThreads, 0, s>>>(g, inv, out, flag, n);
}

void launch_scale_gradient(const float* g, const DevState* st, float* out, size_t n, cudaStream_t s) {
  scale_gradient_kernel<<<grid_window<1>(n / 4), kThreads, 0, s>>>(g, st, out, n);
}

void launch_rng_fill(uint64_t key, uint64_t first, float lo, float hi, float* out, size_t n, cudaStream_t s) {
  if (n == 0) return;
  rng_fill_kernel<<<grid_persist(rng_fill_kernel, n), kThreads, 0, s>>>(key, first, lo, hi, out, n);
}

void launch_rng_perturb(const float* tt, uint64_t key, float lo, float hi, float* out, size_t n,
                        cudaStream_t s) {
  if (n == 0) return;
  rng_perturb_kernel<<<grid_persist(rng_perturb_kernel, n), kThreads, 0, s>>>(tt, key, lo, hi, out, n);
}

void launch_encode_bits_range(uint32_t start, uint16_t* out, size_t n, cudaStream_t s) {
  if (n == 0) return;
  encode_bits_kernel<<<grid_persist(encode_bits_kernel, n), kThreads, 0, s>>>(start, out, n);
}

void launch_copy(const float* src, float* dst, size_t n, cudaStream_t s) {
  if (n == 0) return;
  copy_kernel<<<grid_window<1>(n / 4), kThreads, 0, s>>>(src, dst, n);
}

}  // namespace dlc
