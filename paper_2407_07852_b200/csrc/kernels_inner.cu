// kernels_inner.cu — K1: the fused inner step (unscale + overflow check +
// AdamW, one HBM pass) with its one-thread finalize (skip decision, step
// counter, lr record, scaler update), the INPLACE pre-pass and the host-staged
// adamw_step (optim.cpp:58-148, engine.cpp:50-69).
#include <algorithm>
#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "device.cuh"
#include "kernels.cuh"

namespace dlc {

namespace {

// =============================================================================
// K1: fused unscale + overflow OR + AdamW.
// =============================================================================

// vectors per thread (tools/tune_stream: best for 4R3W).  Round 2 A/B of
// builds (profiles/r2_ab_k1_builds.jsonl): 2 vectors with >= 4 CTAs per SM,
// or 1 vector with >= 8 CTAs per SM (32 registers), run within 1% of this one.
constexpr int kU1 = 1;

// FUSE 0: plain K1.  FUSE 1 / 2: K2 fused in (the last inner step of a window,
// K > 1, dlc_engine_set_fused_delta): delta = theta_t[ocur] - p' (tensor.cpp:126,
// the same explicit-RN op as pseudo_grad_kernel) stored as FP32 / binary16 into
// a.delta, +4 B read and +4 / 2 B written per parameter instead of K2's
// separate 12 / 10 B pass.  While theta_local follows theta_t
// (DevState::lalias) the theta_t read is the p read.
template <int FUSE>
__device__ __forceinline__ void store_delta(void* out, size_t j, float4 t, float4 p) {
  const float4 d = make_float4(delta_elem(t.x, p.x), delta_elem(t.y, p.y), delta_elem(t.z, p.z), delta_elem(t.w, p.w));
  if (FUSE == 1) {
    st_stream(reinterpret_cast<float4*>(out) + j, d);
  } else {
    st_stream(reinterpret_cast<uint2*>(out) + j,
              make_uint2(pack2(fp16_encode(d.x), fp16_encode(d.y)), pack2(fp16_encode(d.z), fp16_encode(d.w))));
  }
}

template <int FUSE>
__global__ void __launch_bounds__(kThreads) adamw_kernel(AdamWArgs a) {
  DevState* st = a.st;
  // INPLACE mode: the pre-pass already decided; an overflowed step writes nothing.
  if (!a.pingpong && *(volatile int*)&st->found_inf != 0) return;
  const int cur = a.pingpong ? st->cur : 0;
  const int nxt = a.pingpong ? (cur ^ 1) : 0;
  const uint64_t t = st->step_count + 1;
  const AdamScalars s{a.b1, a.b2, a.eps, a.wd, a.omb1, a.omb2, a.corr1[t], a.corr2[t], a.lr[t]};
  const float inv = __fdiv_rn(1.0f, st->scale);  // optim.cpp:124 (exact: power of two)
  const bool follow = a.pingpong && st->lalias;
  const float* tc = st->ocur ? a.tt[1] : a.tt[0];
  const float* pc = follow ? tc : (cur ? a.p[1] : a.p[0]);
  const float* mc = cur ? a.m[1] : a.m[0];
  const float* vc = cur ? a.v[1] : a.v[0];
  float* pn = nxt ? a.p[1] : a.p[0];
  float* mn = nxt ? a.m[1] : a.m[0];
  float* vn = nxt ? a.v[1] : a.v[0];
  bool bad = false;
  const size_t n4 = a.n / 4, b = wbase<kU1>();
  float4 p[kU1], g[kU1], m[kU1], v[kU1], tt[kU1];
#pragma unroll
  for (int u = 0; u < kU1; ++u) {
    const size_t j = b + u * kThreads;
    if (j < n4) {
      g[u] = ld_stream(reinterpret_cast<const float4*>(a.g) + j);
      p[u] = ld_stream(reinterpret_cast<const float4*>(pc) + j);
      m[u] = ld_stream(reinterpret_cast<const float4*>(mc) + j);
      v[u] = ld_stream(reinterpret_cast<const float4*>(vc) + j);
      if (FUSE) tt[u] = follow ? p[u] : ld_stream(reinterpret_cast<const float4*>(tc) + j);
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
      if (FUSE) store_delta<FUSE>(a.delta, j, tt[u], po);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < a.n - n4 * 4) {
    const size_t e = n4 * 4 + threadIdx.x;
    const float gu = __fmul_rn(a.g[e], inv);
    bad |= !finite_f(gu);
    float mm = mc[e], vv = vc[e];
    const float po = adamw_elem(pc[e], gu, mm, vv, s);
    pn[e] = po;
    mn[e] = mm;
    vn[e] = vv;
    if (FUSE == 1) static_cast<float*>(a.delta)[e] = delta_elem(tc[e], po);
    if (FUSE == 2) static_cast<uint16_t*>(a.delta)[e] = fp16_encode(delta_elem(tc[e], po));
  }
  if (a.pingpong) block_or_flag(bad, &st->found_inf);
}

// One thread: the skip decision, step counter, lr record and scaler_update
// (inner_finalize, device.cuh).
__global__ void adamw_finalize_kernel(DevState* st, const float* lr_tab, int pingpong, int fused) {
  inner_finalize(st, lr_tab, pingpong, fused);
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

}  // namespace

void launch_adamw(const AdamWArgs& a, cudaStream_t s) {
  if (!a.pingpong)
    unscale_check_kernel<<<grid_window<2>(a.n / 4), kThreads, 0, s>>>(a.g, a.st, a.n);
  const int grid = grid_window<kU1>(a.n / 4);
  if (!a.delta)
    adamw_kernel<0><<<grid, kThreads, 0, s>>>(a);
  else if (!a.delta_fp16)
    adamw_kernel<1><<<grid, kThreads, 0, s>>>(a);
  else
    adamw_kernel<2><<<grid, kThreads, 0, s>>>(a);
  adamw_finalize_kernel<<<1, 1, 0, s>>>(a.st, a.lr, a.pingpong, a.delta != nullptr);
}

void launch_unscale_check(const float* g, DevState* st, size_t n, cudaStream_t s) {
  unscale_check_kernel<<<grid_window<2>(n / 4), kThreads, 0, s>>>(g, st, n);
}

void launch_adamw_plain(const float* p, const float* g, float* m, float* v, float* out, size_t n,
                        const AdamWPlain& a, cudaStream_t s) {
  if (n == 0) return;
  adamw_plain_kernel<<<grid_persist(adamw_plain_kernel, n), kThreads, 0, s>>>(p, g, m, v, out, n, a);
}

}  // namespace dlc
