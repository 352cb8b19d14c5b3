// kernels.cu — DiLoCo hot-path kernels for B200 (sm_100a).
//
// Memory-bound elementwise and reduction work: no tensor cores.  Every kernel
// is a persistent grid-stride loop (grid = #SM x resident CTAs) over 128-bit
// vectors with U independent vectors in flight per thread, evict-first
// streaming hints, a scalar tail, and CTA-level OR reductions
// (__syncthreads_or + one atomicOr per CTA) for the global non-finite flags.
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

constexpr int kU = 2;  // vectors per thread per grid-stride iteration

int g_sms = 0;

template <typename Kern>
int grid_for(Kern kernel, size_t work, int smem = 0) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> per_sm;
  int bps;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = per_sm.find((const void*)kernel);
    if (it == per_sm.end()) {
      int b = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, kThreads, smem);
      it = per_sm.emplace((const void*)kernel, std::max(b, 1)).first;
    }
    bps = it->second;
  }
  const size_t cap = (size_t)num_sms() * (size_t)bps;
  const size_t need = (work + kThreads - 1) / kThreads;
  return (int)std::max<size_t>(1, std::min(cap, need));
}

__device__ __forceinline__ size_t gtid() { return (size_t)blockIdx.x * blockDim.x + threadIdx.x; }
__device__ __forceinline__ size_t gstride() { return (size_t)gridDim.x * blockDim.x; }

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

#define F4_APPLY(OUT, EXPR_X, EXPR_Y, EXPR_Z, EXPR_W) \
  OUT.x = (EXPR_X);                                   \
  OUT.y = (EXPR_Y);                                   \
  OUT.z = (EXPR_Z);                                   \
  OUT.w = (EXPR_W)

// =============================================================================
// K1: fused unscale + overflow OR + AdamW, with device-side skip semantics.
// =============================================================================

__device__ __forceinline__ void adamw_finalize(const AdamWArgs& a, int fi, uint64_t t, float lr) {
  DevState* st = a.st;
  if (!fi) {                       // engine.cpp:57-61: step only when clean
    if (a.pingpong) st->cur ^= 1;  // the freshly written buffers become live
    st->step_count = t;            // optim.cpp:69
    st->last_lr = lr;
  } else {
    st->last_lr = 0.0f;
    st->overflow_skips += 1;
  }
  st->last_overflow = fi;
  // scaler_update, optim.cpp:137-148 (clamps optim.cpp:13-14)
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
  st->done_blocks = 0;
}

__global__ void __launch_bounds__(kThreads) adamw_kernel(AdamWArgs a) {
  DevState* st = a.st;
  const int cur = a.pingpong ? st->cur : 0;
  const int nxt = a.pingpong ? (cur ^ 1) : 0;
  const bool gated_skip = !a.pingpong && (*(volatile int*)&st->found_inf != 0);
  const uint64_t t = st->step_count + 1;
  AdamScalars s{a.b1, a.b2, a.eps, a.wd, a.omb1, a.omb2, a.corr1[t], a.corr2[t], a.lr[t]};
  const float inv = __fdiv_rn(1.0f, st->scale);  // optim.cpp:124 (exact: power of two)
  bool bad = false;
  if (!gated_skip) {
    float* const pc = cur ? a.p[1] : a.p[0];
    float* const mc = cur ? a.m[1] : a.m[0];
    float* const vc = cur ? a.v[1] : a.v[0];
    float* const pn = nxt ? a.p[1] : a.p[0];
    float* const mn = nxt ? a.m[1] : a.m[0];
    float* const vn = nxt ? a.v[1] : a.v[0];
    const float4* P = reinterpret_cast<const float4*>(pc);
    const float4* M = reinterpret_cast<const float4*>(mc);
    const float4* V = reinterpret_cast<const float4*>(vc);
    const float4* G = reinterpret_cast<const float4*>(a.g);
    float4* Po = reinterpret_cast<float4*>(pn);
    float4* Mo = reinterpret_cast<float4*>(mn);
    float4* Vo = reinterpret_cast<float4*>(vn);
    const size_t n4 = a.n / 4, stride = gstride();
    for (size_t i = gtid(); i < n4; i += stride * kU) {
      float4 p[kU], g[kU], m[kU], v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const size_t j = i + u * stride;
        if (j < n4) {
          g[u] = ld_stream(G + j);
          p[u] = ld_stream(P + j);
          m[u] = ld_stream(M + j);
          v[u] = ld_stream(V + j);
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const size_t j = i + u * stride;
        if (j < n4) {
          float4 gu, po;
          F4_APPLY(gu, __fmul_rn(g[u].x, inv), __fmul_rn(g[u].y, inv), __fmul_rn(g[u].z, inv),
                   __fmul_rn(g[u].w, inv));
          bad |= !(finite_f(gu.x) && finite_f(gu.y) && finite_f(gu.z) && finite_f(gu.w));
          po.x = adamw_elem(p[u].x, gu.x, m[u].x, v[u].x, s);
          po.y = adamw_elem(p[u].y, gu.y, m[u].y, v[u].y, s);
          po.z = adamw_elem(p[u].z, gu.z, m[u].z, v[u].z, s);
          po.w = adamw_elem(p[u].w, gu.w, m[u].w, v[u].w, s);
          st_stream(Po + j, po);
          st_stream(Mo + j, m[u]);
          st_stream(Vo + j, v[u]);
        }
      }
    }
    const size_t tail = a.n - n4 * 4, i = gtid();
    if (i < tail) {
      const size_t e = n4 * 4 + i;
      const float gu = __fmul_rn(a.g[e], inv);
      bad |= !finite_f(gu);
      float m = mc[e], v = vc[e];
      pn[e] = adamw_elem(pc[e], gu, m, v, s);
      mn[e] = m;
      vn[e] = v;
    }
  }
  block_or_flag(bad, &st->found_inf);
  __shared__ bool last;
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(&st->done_blocks, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    adamw_finalize(a, atomicAdd(&st->found_inf, 0), t, s.lr);
  }
}

// In-place mode, pass 1 (optim.cpp:127-132): found_inf |= !isfinite(g / scale).
__global__ void __launch_bounds__(kThreads) unscale_check_kernel(const float* g, const DevState* st,
                                                                 int* flag, size_t n) {
  const float inv = __fdiv_rn(1.0f, st->scale);
  bool bad = false;
  const float4* G = reinterpret_cast<const float4*>(g);
  const size_t n4 = n / 4, stride = gstride();
  for (size_t i = gtid(); i < n4; i += stride * kU) {
    float4 x[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (i + u * stride < n4) x[u] = ld_stream(G + i + u * stride);
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (i + u * stride < n4)
        bad |= !(finite_f(__fmul_rn(x[u].x, inv)) && finite_f(__fmul_rn(x[u].y, inv)) &&
                 finite_f(__fmul_rn(x[u].z, inv)) && finite_f(__fmul_rn(x[u].w, inv)));
  }
  const size_t i = gtid();
  if (i < n - n4 * 4) bad |= !finite_f(__fmul_rn(g[n4 * 4 + i], inv));
  block_or_flag(bad, flag);
}

// Out-of-place AdamW on an already unscaled, finite gradient (adamw_step with
// the host-side checks done by the caller; optim.cpp:83-91).
__global__ void __launch_bounds__(kThreads) adamw_plain_kernel(const float* p, const float* g, float* m,
                                                               float* v, float* out, size_t n, AdamWPlain a) {
  AdamScalars s{a.b1, a.b2, a.eps, a.wd, a.omb1, a.omb2, a.corr1, a.corr2, a.lr};
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

template <int PREC>
__global__ void __launch_bounds__(kThreads) pseudo_grad_kernel(Pair ttp, Pair tl, const DevState* st,
                                                               void* out, int* flag, size_t n) {
  const float* tt = st->ocur ? ttp.ptr[1] : ttp.ptr[0];
  const float* L = st->cur ? tl.ptr[1] : tl.ptr[0];
  const float4* T4 = reinterpret_cast<const float4*>(tt);
  const float4* L4 = reinterpret_cast<const float4*>(L);
  bool bad = false;
  const size_t n4 = n / 4, stride = gstride();
  for (size_t i = gtid(); i < n4; i += stride * kU) {
    float4 a[kU], b[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (i + u * stride < n4) {
        a[u] = ld_stream(T4 + i + u * stride);
        b[u] = ld_stream(L4 + i + u * stride);
      }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const size_t j = i + u * stride;
      if (j < n4) {
        float4 d;
        F4_APPLY(d, delta_elem(a[u].x, b[u].x), delta_elem(a[u].y, b[u].y), delta_elem(a[u].z, b[u].z),
                 delta_elem(a[u].w, b[u].w));
        if (PREC == 0) {
          bad |= !(finite_f(d.x) && finite_f(d.y) && finite_f(d.z) && finite_f(d.w));
          st_stream(reinterpret_cast<float4*>(out) + j, d);
        } else {
          const uint16_t h0 = fp16_encode(d.x), h1 = fp16_encode(d.y), h2 = fp16_encode(d.z),
                         h3 = fp16_encode(d.w);
          bad |= fp16_nonfinite(h0) | fp16_nonfinite(h1) | fp16_nonfinite(h2) | fp16_nonfinite(h3);
          st_stream(reinterpret_cast<uint2*>(out) + j, make_uint2(pack2(h0, h1), pack2(h2, h3)));
        }
      }
    }
  }
  const size_t i = gtid();
  if (i < n - n4 * 4) {
    const size_t e = n4 * 4 + i;
    const float d = delta_elem(tt[e], L[e]);
    if (PREC == 0) {
      bad |= !finite_f(d);
      reinterpret_cast<float*>(out)[e] = d;
    } else {
      const uint16_t h = fp16_encode(d);
      bad |= fp16_nonfinite(h);
      reinterpret_cast<uint16_t*>(out)[e] = h;
    }
  }
  block_or_flag(bad, flag);
}

// =============================================================================
// K3: ordered fold of K contributions (reduce.cpp:33-44 / 70-88).
// Each thread owns 8 consecutive elements; contributions are visited in rank
// order 0..K-1 so the FP32 sum is bit-identical to fold_mean.
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
__global__ void __launch_bounds__(kThreads) fold_kernel(const __grid_constant__ PtrList in, int k, void* out, int* flag, size_t n) {
  const float divisor = (float)k;  // reduce.cpp:36
  bool bad = false;
  const size_t n8 = n / 8, stride = gstride();
  for (size_t i = gtid(); i < n8; i += stride) {
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
  const size_t i = gtid();
  if (i < n - n8 * 8) {
    const size_t e = n8 * 8 + i;
    float acc = load1<IN>(in.ptr[0], e);
    for (int j = 1; j < k; ++j) acc = __fadd_rn(acc, load1<IN>(in.ptr[j], e));
    bad |= store1<OUT>(out, e, __fdiv_rn(acc, divisor));
  }
  if (flag) block_or_flag(bad, flag);
}

// =============================================================================
// K4: finite-gated Nesterov on theta_t + theta_local refresh (engine.cpp:136-144).
// =============================================================================

template <int PREC>
__global__ void __launch_bounds__(kThreads) nesterov_outer_kernel(Pair ttp, Pair bufp, Pair tl,
                                                                  const void* dbar, const int* flags, int nflags,
                                                                  DevState* st, float lr, float mu, size_t n) {
  float* tt = st->ocur ? ttp.ptr[1] : ttp.ptr[0];
  float* buf = st->ocur ? bufp.ptr[1] : bufp.ptr[0];
  int nonfinite = 0;
  for (int j = 0; j < nflags; ++j) nonfinite |= flags[j];
  const bool applied = nonfinite == 0;
  float* L = st->cur ? tl.ptr[1] : tl.ptr[0];
  float4* T4 = reinterpret_cast<float4*>(tt);
  float4* B4 = reinterpret_cast<float4*>(buf);
  float4* L4 = reinterpret_cast<float4*>(L);
  const size_t n4 = n / 4, stride = gstride();
  if (applied) {
    for (size_t i = gtid(); i < n4; i += stride * kU) {
      float4 t[kU], b[kU], d[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const size_t j = i + u * stride;
        if (j < n4) {
          if (PREC == 0) {
            d[u] = ld_stream(reinterpret_cast<const float4*>(dbar) + j);
          } else {
            const uint2 w = ld_stream(reinterpret_cast<const uint2*>(dbar) + j);
            F4_APPLY(d[u], fp16_decode(lo16(w.x)), fp16_decode(hi16(w.x)), fp16_decode(lo16(w.y)),
                     fp16_decode(hi16(w.y)));
          }
          t[u] = ld_stream(T4 + j);
          b[u] = ld_stream(B4 + j);
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const size_t j = i + u * stride;
        if (j < n4) {
          float4 o;
          o.x = nesterov_elem(t[u].x, d[u].x, b[u].x, lr, mu);
          o.y = nesterov_elem(t[u].y, d[u].y, b[u].y, lr, mu);
          o.z = nesterov_elem(t[u].z, d[u].z, b[u].z, lr, mu);
          o.w = nesterov_elem(t[u].w, d[u].w, b[u].w, lr, mu);
          st_stream(T4 + j, o);
          st_stream(B4 + j, b[u]);
          st_stream(L4 + j, o);
        }
      }
    }
  } else {  // skip: keep theta_t, discard local progress (engine.cpp:140-143)
    for (size_t i = gtid(); i < n4; i += stride * kU) {
      float4 t[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (i + u * stride < n4) t[u] = ld_stream(T4 + i + u * stride);
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (i + u * stride < n4) st_stream(L4 + i + u * stride, t[u]);
    }
  }
  const size_t i = gtid();
  if (i < n - n4 * 4) {
    const size_t e = n4 * 4 + i;
    if (applied) {
      const float d = PREC == 0 ? reinterpret_cast<const float*>(dbar)[e]
                                : fp16_decode(reinterpret_cast<const uint16_t*>(dbar)[e]);
      float b = buf[e];
      const float o = nesterov_elem(tt[e], d, b, lr, mu);
      tt[e] = o;
      buf[e] = b;
      L[e] = o;
    } else {
      L[e] = tt[e];
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->last_applied = applied ? 1 : 0;
    st->outer_skips += applied ? 0 : 1;
    st->outer_epoch += 1;  // engine.cpp:144
  }
}

// K2 + K4 fused for K = 1 (see kernels.cuh).  Speculative: the new theta_t and
// momentum go to the idle buffers of their ping-pong pairs, so a skip only has
// to leave `ocur` unflipped.
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
                                                              DevState* st, float lr, float mu, size_t n) {
  const int oc = st->ocur;
  const float4* T = reinterpret_cast<const float4*>(oc ? ttp.ptr[1] : ttp.ptr[0]);
  const float4* B = reinterpret_cast<const float4*>(oc ? bufp.ptr[1] : bufp.ptr[0]);
  float4* To = reinterpret_cast<float4*>(oc ? ttp.ptr[0] : ttp.ptr[1]);
  float4* Bo = reinterpret_cast<float4*>(oc ? bufp.ptr[0] : bufp.ptr[1]);
  float* Ld = st->cur ? tl.ptr[1] : tl.ptr[0];
  const float4* Ls = reinterpret_cast<const float4*>(src ? src : Ld);
  float4* L4 = reinterpret_cast<float4*>(Ld);
  bool bad = false;
  const size_t n4 = n / 4, stride = gstride();
  for (size_t i = gtid(); i < n4; i += stride * kU) {
    float4 t[kU], b[kU], l[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const size_t j = i + u * stride;
      if (j < n4) {
        t[u] = ld_stream(T + j);
        l[u] = ld_stream(Ls + j);
        b[u] = ld_stream(B + j);
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const size_t j = i + u * stride;
      if (j < n4) {
        float4 o;
        o.x = nesterov_elem(t[u].x, solo_delta<PREC>(t[u].x, l[u].x, bad), b[u].x, lr, mu);
        o.y = nesterov_elem(t[u].y, solo_delta<PREC>(t[u].y, l[u].y, bad), b[u].y, lr, mu);
        o.z = nesterov_elem(t[u].z, solo_delta<PREC>(t[u].z, l[u].z, bad), b[u].z, lr, mu);
        o.w = nesterov_elem(t[u].w, solo_delta<PREC>(t[u].w, l[u].w, bad), b[u].w, lr, mu);
        st_stream(To + j, o);
        st_stream(Bo + j, b[u]);
        st_stream(L4 + j, o);
      }
    }
  }
  const size_t i = gtid();
  if (i < n - n4 * 4) {
    const size_t e = n4 * 4 + i;
    const float* Tf = reinterpret_cast<const float*>(T);
    float bb = reinterpret_cast<const float*>(B)[e];
    const float t0 = Tf[e];
    const float o = nesterov_elem(t0, solo_delta<PREC>(t0, reinterpret_cast<const float*>(Ls)[e], bad), bb, lr, mu);
    reinterpret_cast<float*>(To)[e] = o;
    reinterpret_cast<float*>(Bo)[e] = bb;
    Ld[e] = o;
  }
  block_or_flag(bad, &st->delta_nonfinite);
  __shared__ bool last;
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(&st->done_blocks, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    const int skip = atomicAdd(&st->delta_nonfinite, 0);
    if (!skip) st->ocur ^= 1;  // engine.cpp:136-139: apply only a finite reduction
    st->last_applied = skip ? 0 : 1;
    st->outer_skips += skip ? 1 : 0;
    st->outer_epoch += 1;  // engine.cpp:144
    st->done_blocks = 0;
  }
}

// After a skipped solo step: theta_local := theta_t (engine.cpp:143).
__global__ void __launch_bounds__(kThreads) outer_solo_recover_kernel(Pair ttp, Pair tl, const DevState* st,
                                                                      size_t n) {
  if (st->last_applied) return;
  const float* T = st->ocur ? ttp.ptr[1] : ttp.ptr[0];
  float* L = st->cur ? tl.ptr[1] : tl.ptr[0];
  for (size_t e = gtid(); e < n; e += gstride()) L[e] = T[e];
}

// K4 over NVLink peer memory (DLC_MODE_P2P): the mean slot of owner q is read
// in place from q's HBM; the K owner flags are read once per CTA.
template <int PREC>
__global__ void __launch_bounds__(kThreads) nesterov_outer_p2p_kernel(Pair ttp, Pair bufp, Pair tl,
                                                                      const __grid_constant__ PtrList slots,
                                                                      const __grid_constant__ PtrList flags, int k,
                                                                      size_t S, DevState* st, float lr, float mu,
                                                                      size_t n) {
  __shared__ int s_nonfinite;
  if (threadIdx.x == 0) {
    int nf = 0;
    for (int j = 0; j < k; ++j) nf |= *reinterpret_cast<const volatile int*>(flags.ptr[j]);
    s_nonfinite = nf;
  }
  __syncthreads();
  const bool applied = s_nonfinite == 0;
  float* tt = st->ocur ? ttp.ptr[1] : ttp.ptr[0];
  float* buf = st->ocur ? bufp.ptr[1] : bufp.ptr[0];
  float* L = st->cur ? tl.ptr[1] : tl.ptr[0];
  const size_t stride = gstride();
  for (int q = 0; q < k; ++q) {
    const size_t base = (size_t)q * S;
    if (base >= n) break;
    const size_t len = n - base < S ? n - base : S;
    const size_t len4 = len / 4;
    float4* T4 = reinterpret_cast<float4*>(tt + base);
    float4* B4 = reinterpret_cast<float4*>(buf + base);
    float4* L4 = reinterpret_cast<float4*>(L + base);
    const void* dbar = slots.ptr[q];
    if (applied) {
      for (size_t i = gtid(); i < len4; i += stride * kU) {
        float4 t[kU], b[kU], d[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const size_t j = i + u * stride;
          if (j < len4) {
            if (PREC == 0) {
              d[u] = ld_stream(reinterpret_cast<const float4*>(dbar) + j);
            } else {
              const uint2 w = ld_stream(reinterpret_cast<const uint2*>(dbar) + j);
              F4_APPLY(d[u], fp16_decode(lo16(w.x)), fp16_decode(hi16(w.x)), fp16_decode(lo16(w.y)),
                       fp16_decode(hi16(w.y)));
            }
            t[u] = ld_stream(T4 + j);
            b[u] = ld_stream(B4 + j);
          }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const size_t j = i + u * stride;
          if (j < len4) {
            float4 o;
            o.x = nesterov_elem(t[u].x, d[u].x, b[u].x, lr, mu);
            o.y = nesterov_elem(t[u].y, d[u].y, b[u].y, lr, mu);
            o.z = nesterov_elem(t[u].z, d[u].z, b[u].z, lr, mu);
            o.w = nesterov_elem(t[u].w, d[u].w, b[u].w, lr, mu);
            st_stream(T4 + j, o);
            st_stream(B4 + j, b[u]);
            st_stream(L4 + j, o);
          }
        }
      }
    } else {
      for (size_t i = gtid(); i < len4; i += stride) st_stream(L4 + i, ld_stream(T4 + i));
    }
    const size_t i = gtid();
    if (i < len - len4 * 4) {
      const size_t e = len4 * 4 + i;
      float* te = tt + base;
      if (applied) {
        const float d = PREC == 0 ? reinterpret_cast<const float*>(dbar)[e]
                                  : fp16_decode(reinterpret_cast<const uint16_t*>(dbar)[e]);
        float b = buf[base + e];
        const float o = nesterov_elem(te[e], d, b, lr, mu);
        te[e] = o;
        buf[base + e] = b;
        L[base + e] = o;
      } else {
        L[base + e] = te[e];
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->last_applied = applied ? 1 : 0;
    st->outer_skips += applied ? 0 : 1;
    st->outer_epoch += 1;  // engine.cpp:144
  }
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
// elementwise helpers
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
  const float4* G = reinterpret_cast<const float4*>(g);
  float4* O = reinterpret_cast<float4*>(out);
  const size_t n4 = n / 4;
  for (size_t i = gtid(); i < n4; i += gstride()) {
    const float4 x = ld_stream(G + i);
    st_stream(O + i, make_float4(__fmul_rn(x.x, s), __fmul_rn(x.y, s), __fmul_rn(x.z, s), __fmul_rn(x.w, s)));
  }
  const size_t i = gtid();
  if (i < n - n4 * 4) out[n4 * 4 + i] = __fmul_rn(g[n4 * 4 + i], s);
}

__global__ void __launch_bounds__(kThreads) rng_fill_kernel(uint64_t key, uint64_t first, float lo, float hi,
                                                            float* out, size_t n) {
  for (size_t e = gtid(); e < n; e += gstride()) out[e] = rng_uniform_at(key, first + e, lo, hi);
}

__global__ void __launch_bounds__(kThreads) rng_perturb_kernel(const float* tt, uint64_t key, float lo, float hi,
                                                               float* out, size_t n) {
  for (size_t e = gtid(); e < n; e += gstride())
    out[e] = __fsub_rn(tt[e], rng_uniform_at(key, e, lo, hi));
}

__global__ void __launch_bounds__(kThreads) encode_bits_kernel(uint32_t start, uint16_t* out, size_t n) {
  for (size_t e = gtid(); e < n; e += gstride()) out[e] = fp16_encode(__uint_as_float(start + (uint32_t)e));
}

__global__ void __launch_bounds__(kThreads) copy_kernel(const float* src, float* dst, size_t n) {
  const float4* S = reinterpret_cast<const float4*>(src);
  float4* D = reinterpret_cast<float4*>(dst);
  const size_t n4 = n / 4;
  for (size_t i = gtid(); i < n4; i += gstride()) st_stream(D + i, ld_stream(S + i));
  const size_t i = gtid();
  if (i < n - n4 * 4) dst[n4 * 4 + i] = src[n4 * 4 + i];
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
  adamw_kernel<<<grid_for(adamw_kernel, std::max<size_t>(a.n / 4, 1) / kU + 1), kThreads, 0, s>>>(a);
}

void launch_unscale_check(const float* g, const DevState* st, int* flag, size_t n, cudaStream_t s) {
  unscale_check_kernel<<<grid_for(unscale_check_kernel, n / 4 / kU + 1), kThreads, 0, s>>>(g, st, flag, n);
}

void launch_adamw_plain(const float* p, const float* g, float* m, float* v, float* out, size_t n,
                        const AdamWPlain& a, cudaStream_t s) {
  if (n == 0) return;
  adamw_plain_kernel<<<grid_for(adamw_plain_kernel, n), kThreads, 0, s>>>(p, g, m, v, out, n, a);
}

void launch_pseudo_grad(Pair tt, Pair tl, const DevState* st, void* out, int precision, int* flag,
                        size_t n, cudaStream_t s) {
  if (precision == 0)
    pseudo_grad_kernel<0><<<grid_for(pseudo_grad_kernel<0>, n / 4 / kU + 1), kThreads, 0, s>>>(tt, tl, st, out,
                                                                                                 flag, n);
  else
    pseudo_grad_kernel<1><<<grid_for(pseudo_grad_kernel<1>, n / 4 / kU + 1), kThreads, 0, s>>>(tt, tl, st, out,
                                                                                                 flag, n);
}

void launch_fold(const PtrList& in, int k, int in_kind, void* out, int out_kind, int* flag, size_t n,
                 cudaStream_t s) {
  const size_t work = n / 8 + 1;
#define DLC_FOLD(I, O)                                                                      \
  if (in_kind == I && out_kind == O) {                                                      \
    fold_kernel<I, O><<<grid_for(fold_kernel<I, O>, work), kThreads, 0, s>>>(in, k, out, flag, n); \
    return;                                                                                 \
  }
  DLC_FOLD(0, 0) DLC_FOLD(0, 1) DLC_FOLD(0, 2) DLC_FOLD(1, 0) DLC_FOLD(1, 1) DLC_FOLD(1, 2)
  DLC_FOLD(2, 0) DLC_FOLD(2, 1) DLC_FOLD(2, 2)
#undef DLC_FOLD
}

void launch_nesterov_outer(Pair tt, Pair buf, Pair tl, const void* dbar, int precision, const int* flags,
                           int nflags, DevState* st, float lr, float mu, size_t n, cudaStream_t s) {
  const size_t work = n / 4 / kU + 1;
  if (precision == 0)
    nesterov_outer_kernel<0><<<grid_for(nesterov_outer_kernel<0>, work), kThreads, 0, s>>>(
        tt, buf, tl, dbar, flags, nflags, st, lr, mu, n);
  else
    nesterov_outer_kernel<1><<<grid_for(nesterov_outer_kernel<1>, work), kThreads, 0, s>>>(
        tt, buf, tl, dbar, flags, nflags, st, lr, mu, n);
}

void launch_outer_solo_fused(Pair tt, Pair buf, Pair tl, const float* src, int precision, DevState* st, float lr,
                             float mu, size_t n, cudaStream_t s) {
  const size_t work = n / 4 / kU + 1;
  if (precision == 0)
    outer_solo_kernel<0><<<grid_for(outer_solo_kernel<0>, work), kThreads, 0, s>>>(tt, buf, tl, src, st, lr, mu, n);
  else
    outer_solo_kernel<1><<<grid_for(outer_solo_kernel<1>, work), kThreads, 0, s>>>(tt, buf, tl, src, st, lr, mu, n);
  outer_solo_recover_kernel<<<grid_for(outer_solo_recover_kernel, n), kThreads, 0, s>>>(tt, tl, st, n);
}

void launch_nesterov_outer_p2p(Pair tt, Pair buf, Pair tl, const PtrList& slots, const PtrList& flags, int k,
                               size_t S, int precision, DevState* st, float lr, float mu, size_t n,
                               cudaStream_t s) {
  const size_t work = n / 4 / kU + 1;
  if (precision == 0)
    nesterov_outer_p2p_kernel<0><<<grid_for(nesterov_outer_p2p_kernel<0>, work), kThreads, 0, s>>>(
        tt, buf, tl, slots, flags, k, S, st, lr, mu, n);
  else
    nesterov_outer_p2p_kernel<1><<<grid_for(nesterov_outer_p2p_kernel<1>, work), kThreads, 0, s>>>(
        tt, buf, tl, slots, flags, k, S, st, lr, mu, n);
}

void launch_nesterov_plain(const float* p, const float* g, float* buf, float* out, size_t n, float lr, float mu,
                           cudaStream_t s) {
  if (n == 0) return;
  nesterov_plain_kernel<<<grid_for(nesterov_plain_kernel, n), kThreads, 0, s>>>(p, g, buf, out, n, lr, mu);
}

void launch_axpy(float alpha, const float* x, const float* y, float* out, size_t n, cudaStream_t s) {
  if (n == 0) return;
  axpy_kernel<<<grid_for(axpy_kernel, n), kThreads, 0, s>>>(alpha, x, y, out, n);
}

void launch_encode(const float* x, uint16_t* out, int* flag, size_t n, cudaStream_t s) {
  if (n == 0) return;
  encode_kernel<<<grid_for(encode_kernel, n), kThreads, 0, s>>>(x, out, flag, n);
}

void launch_decode(const uint16_t* b, float* out, size_t n, cudaStream_t s) {
  if (n == 0) return;
  decode_kernel<<<grid_for(decode_kernel, n), kThreads, 0, s>>>(b, out, n);
}

void launch_nonfinite(const float* x, int* flag, size_t n, cudaStream_t s) {
  if (n == 0) return;
  nonfinite_kernel<<<grid_for(nonfinite_kernel, n), kThreads, 0, s>>>(x, flag, n);
}

void launch_nonfinite_codes(const uint16_t* b, int* flag, size_t n, cudaStream_t s) {
  if (n == 0) return;
  nonfinite_codes_kernel<<<grid_for(nonfinite_codes_kernel, n), kThreads, 0, s>>>(b, flag, n);
}

void launch_fold_many(const float* const* ptrs, size_t k, int fp16, float* out, size_t n, cudaStream_t s) {
  if (n == 0 || k == 0) return;
  fold_many_kernel<<<grid_for(fold_many_kernel, n), kThreads, 0, s>>>(ptrs, k, fp16, out, n);
}

void launch_unscale(const float* g, float inv, float* out, int* flag, size_t n, cudaStream_t s) {
  if (n == 0) return;
  unscale_kernel<<<grid_for(unscale_kernel, n), kThreads, 0, s>>>(g, inv, out, flag, n);
}

void launch_scale_gradient(const float* g, const DevState* st, float* out, size_t n, cudaStream_t s) {
  scale_gradient_kernel<<<grid_for(scale_gradient_kernel, n / 4 + 1), kThreads, 0, s>>>(g, st, out, n);
}

void launch_rng_fill(uint64_t key, uint64_t first, float lo, float hi, float* out, size_t n, cudaStream_t s) {
  if (n == 0) return;
  rng_fill_kernel<<<grid_for(rng_fill_kernel, n), kThreads, 0, s>>>(key, first, lo, hi, out, n);
}

void launch_rng_perturb(const float* tt, uint64_t key, float lo, float hi, float* out, size_t n,
                        cudaStream_t s) {
  if (n == 0) return;
  rng_perturb_kernel<<<grid_for(rng_perturb_kernel, n), kThreads, 0, s>>>(tt, key, lo, hi, out, n);
}

void launch_encode_bits_range(uint32_t start, uint16_t* out, size_t n, cudaStream_t s) {
  if (n == 0) return;
  encode_bits_kernel<<<grid_for(encode_bits_kernel, n), kThreads, 0, s>>>(start, out, n);
}

void launch_copy(const float* src, float* dst, size_t n, cudaStream_t s) {
  if (n == 0) return;
  copy_kernel<<<grid_for(copy_kernel, n / 4 + 1), kThreads, 0, s>>>(src, dst, n);
}

}  // namespace dlc
