// kernels_boundary.cu — the window boundary of a single worker in one HBM pass:
// the window's last inner step (K1: unscale + overflow OR + AdamW,
// engine.cpp:50-69, optim.cpp:58-148) with the SoloCollective outer step fused
// into it (K2 + K4: delta, Nesterov, theta_local := theta_t; engine.cpp:115-146,
// reduce.cpp:113-126), as DilocoOptimizer::step runs them back to back at
// inner_step % H == 0 (engine.cpp:162-174).
#include "common.cuh"
#include "device.cuh"
#include "kernels.cuh"

namespace dlc {

namespace {

// One 4-element vector per thread in address order (the streaming window of
// K1).  Every value is the one the two separate steps would compute: p' by
// adamw_elem, the delta from p' (solo_delta: FP16 encode / decode once), the
// Nesterov update of theta_t from it.  m', v' go to the idle moments (flipped
// in by the finalize when the inner step applies), theta_t' and momentum' to
// the idle outer pair (flipped in when the inner step applied and every delta
// was finite).
#ifndef DLC_BOUNDARY_MINB  // min resident CTAs per SM (6: 40 registers; r2 A/B: 6.28 vs 6.49 ms at 1.1B)
#define DLC_BOUNDARY_MINB 6
#endif
#if DLC_BOUNDARY_MINB > 0
#define DLC_BOUNDARY_BOUNDS __launch_bounds__(kThreads, DLC_BOUNDARY_MINB)
#else
#define DLC_BOUNDARY_BOUNDS __launch_bounds__(kThreads)
#endif
template <int PREC>
__global__ void DLC_BOUNDARY_BOUNDS boundary_solo_kernel(AdamWArgs a, Pair ttp, Pair bufp, float lr, float mu) {
  DevState* st = a.st;
  const int cur = st->cur, nxt = cur ^ 1, oc = st->ocur;
  const uint64_t t = st->step_count + 1;
  const AdamScalars s{a.b1, a.b2, a.eps, a.wd, a.omb1, a.omb2, a.corr1[t], a.corr2[t], a.lr[t]};
  const float inv = __fdiv_rn(1.0f, st->scale);  // optim.cpp:124 (exact: power of two)
  const bool follow = st->lalias;                // theta_local == theta_t[ocur]: one read for both
  const float* T = sel(ttp, oc);
  const float* B = sel(bufp, oc);
  float* To = sel(ttp, oc ^ 1);
  float* Bo = sel(bufp, oc ^ 1);
  const float* pc = follow ? T : (cur ? a.p[1] : a.p[0]);
  const float* mc = cur ? a.m[1] : a.m[0];
  const float* vc = cur ? a.v[1] : a.v[0];
  float* mn = nxt ? a.m[1] : a.m[0];
  float* vn = nxt ? a.v[1] : a.v[0];
  bool bad_in = false, bad_out = false;
  const size_t n4 = a.n / 4, j = gtid();
  if (j < n4) {
    const float4 g = ld_stream(reinterpret_cast<const float4*>(a.g) + j);
    const float4 tt = ld_stream(reinterpret_cast<const float4*>(T) + j);
    const float4 p = follow ? tt : ld_stream(reinterpret_cast<const float4*>(pc) + j);
    float4 m = ld_stream(reinterpret_cast<const float4*>(mc) + j);
    float4 v = ld_stream(reinterpret_cast<const float4*>(vc) + j);
    float4 b = ld_stream(reinterpret_cast<const float4*>(B) + j);
    const float4 gu = make_float4(__fmul_rn(g.x, inv), __fmul_rn(g.y, inv), __fmul_rn(g.z, inv), __fmul_rn(g.w, inv));
    bad_in |= !(finite_f(gu.x) && finite_f(gu.y) && finite_f(gu.z) && finite_f(gu.w));
    float4 pn, o;
    pn.x = adamw_elem(p.x, gu.x, m.x, v.x, s);
    pn.y = adamw_elem(p.y, gu.y, m.y, v.y, s);
    pn.z = adamw_elem(p.z, gu.z, m.z, v.z, s);
    pn.w = adamw_elem(p.w, gu.w, m.w, v.w, s);
    o.x = nesterov_elem(tt.x, solo_delta<PREC>(tt.x, pn.x, bad_out), b.x, lr, mu);
    o.y = nesterov_elem(tt.y, solo_delta<PREC>(tt.y, pn.y, bad_out), b.y, lr, mu);
    o.z = nesterov_elem(tt.z, solo_delta<PREC>(tt.z, pn.z, bad_out), b.z, lr, mu);
    o.w = nesterov_elem(tt.w, solo_delta<PREC>(tt.w, pn.w, bad_out), b.w, lr, mu);
    st_stream(reinterpret_cast<float4*>(mn) + j, m);
    st_stream(reinterpret_cast<float4*>(vn) + j, v);
    st_stream(reinterpret_cast<float4*>(To) + j, o);
    st_stream(reinterpret_cast<float4*>(Bo) + j, b);
  }
  if (blockIdx.x == 0 && threadIdx.x < a.n - n4 * 4) {
    const size_t e = n4 * 4 + threadIdx.x;
    const float gu = __fmul_rn(a.g[e], inv);
    bad_in |= !finite_f(gu);
    float mm = mc[e], vv = vc[e], bb = B[e];
    const float pn = adamw_elem(pc[e], gu, mm, vv, s);
    const float o = nesterov_elem(T[e], solo_delta<PREC>(T[e], pn, bad_out), bb, lr, mu);
    mn[e] = mm;
    vn[e] = vv;
    To[e] = o;
    Bo[e] = bb;
  }
  block_or_flag(bad_in, &st->found_inf);
  block_or_flag(bad_out, &st->delta_nonfinite);
}

// One thread: the inner step's finalize, then the outer step's gate, or the
// rerun mark when the inner step overflowed.
__global__ void boundary_solo_finalize_kernel(DevState* st, const float* lr_tab) {
  const int fi = st->found_inf;
  inner_finalize(st, lr_tab, 1, 0);
  if (fi) {  // theta_local unchanged: the outer step reruns from it (boundary_solo_redo_kernel)
    st->redo = 1;
    st->delta_nonfinite = 0;
    return;
  }
  const int skip = st->delta_nonfinite;
  if (!skip) st->ocur ^= 1;  // engine.cpp:136-139
  k4_finalize(st, !skip, Pair{{nullptr, nullptr}, 1});
}

// The solo outer step after an overflowed inner step, over the whole vector
// (persistent grid; every CTA returns at once when there is nothing to redo).
template <int PREC>
__global__ void __launch_bounds__(kThreads) boundary_solo_redo_kernel(Pair ttp, Pair bufp, Pair tl, DevState* st,
                                                                      float lr, float mu, size_t n) {
  if (!*reinterpret_cast<volatile int*>(&st->redo)) return;
  const int oc = st->ocur;
  const float* T = sel(ttp, oc);
  const float* B = sel(bufp, oc);
  float* To = sel(ttp, oc ^ 1);
  float* Bo = sel(bufp, oc ^ 1);
  const float* L = local_src(tl, ttp, st);
  bool bad = false;
  for (size_t e = gtid(); e < n; e += gstride()) {
    float bb = B[e];
    To[e] = nesterov_elem(T[e], solo_delta<PREC>(T[e], L[e], bad), bb, lr, mu);
    Bo[e] = bb;
  }
  block_or_flag(bad, &st->delta_nonfinite);
}

__global__ void boundary_solo_redo_finish_kernel(DevState* st) {
  if (!st->redo) return;
  const int skip = st->delta_nonfinite;
  if (!skip) st->ocur ^= 1;
  k4_finalize(st, !skip, Pair{{nullptr, nullptr}, 1});
  st->redo = 0;
}

// DLC_INNER_INPLACE: the pre-pass has decided the overflow (found_inf), so one
// pass applies the inner step or not, then the outer step from the resulting
// theta_local, and stores theta_t' speculatively into the idle outer pair AND
// into theta_local (its fixed address; the finish restores it on a skip).
template <int PREC>
#ifdef DLC_INPLACE_MINB  // A/B build knob (tools/): min resident CTAs per SM of the in-place pass
#define DLC_INPLACE_BOUNDS __launch_bounds__(kThreads, DLC_INPLACE_MINB)
#else
#define DLC_INPLACE_BOUNDS __launch_bounds__(kThreads)
#endif
__global__ void DLC_INPLACE_BOUNDS boundary_solo_inplace_kernel(AdamWArgs a, Pair ttp, Pair bufp, float lr,
                                                                 float mu) {
  DevState* st = a.st;
  const bool skip_inner = *(volatile int*)&st->found_inf != 0;
  const int oc = st->ocur;
  const uint64_t t = st->step_count + 1;
  const AdamScalars s{a.b1, a.b2, a.eps, a.wd, a.omb1, a.omb2, a.corr1[t], a.corr2[t], a.lr[t]};
  const float inv = __fdiv_rn(1.0f, st->scale);
  const float* T = sel(ttp, oc);
  const float* B = sel(bufp, oc);
  float* To = sel(ttp, oc ^ 1);
  float* Bo = sel(bufp, oc ^ 1);
  float* P = a.p[0];
  float* M = a.m[0];
  float* V = a.v[0];
  bool bad_out = false;
  const size_t n4 = a.n / 4, j = gtid();
  if (j < n4) {
    const float4 tt = ld_stream(reinterpret_cast<const float4*>(T) + j);
    float4 p = ld_stream(reinterpret_cast<const float4*>(P) + j);
    float4 b = ld_stream(reinterpret_cast<const float4*>(B) + j), o;
    if (!skip_inner) {
      const float4 g = ld_stream(reinterpret_cast<const float4*>(a.g) + j);
      float4 m = ld_stream(reinterpret_cast<const float4*>(M) + j);
      float4 v = ld_stream(reinterpret_cast<const float4*>(V) + j);
      p.x = adamw_elem(p.x, __fmul_rn(g.x, inv), m.x, v.x, s);
      p.y = adamw_elem(p.y, __fmul_rn(g.y, inv), m.y, v.y, s);
      p.z = adamw_elem(p.z, __fmul_rn(g.z, inv), m.z, v.z, s);
      p.w = adamw_elem(p.w, __fmul_rn(g.w, inv), m.w, v.w, s);
      st_stream(reinterpret_cast<float4*>(M) + j, m);
      st_stream(reinterpret_cast<float4*>(V) + j, v);
    }
    o.x = nesterov_elem(tt.x, solo_delta<PREC>(tt.x, p.x, bad_out), b.x, lr, mu);
    o.y = nesterov_elem(tt.y, solo_delta<PREC>(tt.y, p.y, bad_out), b.y, lr, mu);
    o.z = nesterov_elem(tt.z, solo_delta<PREC>(tt.z, p.z, bad_out), b.z, lr, mu);
    o.w = nesterov_elem(tt.w, solo_delta<PREC>(tt.w, p.w, bad_out), b.w, lr, mu);
    st_stream(reinterpret_cast<float4*>(To) + j, o);
    st_stream(reinterpret_cast<float4*>(Bo) + j, b);
    st_stream(reinterpret_cast<float4*>(P) + j, o);
  }
  if (blockIdx.x == 0 && threadIdx.x < a.n - n4 * 4) {
    const size_t e = n4 * 4 + threadIdx.x;
    float pp = P[e], bb = B[e];
    if (!skip_inner) {
      float mm = M[e], vv = V[e];
      pp = adamw_elem(pp, __fmul_rn(a.g[e], inv), mm, vv, s);
      M[e] = mm;
      V[e] = vv;
    }
    const float o = nesterov_elem(T[e], solo_delta<PREC>(T[e], pp, bad_out), bb, lr, mu);
    To[e] = o;
    Bo[e] = bb;
    P[e] = o;
  }
  block_or_flag(bad_out, &st->delta_nonfinite);
}

// One thread: the inner step's finalize (the pre-pass decided the skip)
__global__ void boundary_inplace_finalize_kernel(DevState* st, const float* lr_tab) {
  inner_finalize(st, lr_tab, 0, 0);
}

}  // namespace

void launch_boundary_solo(const AdamWArgs& a, Pair tt, Pair buf, int precision, float lr, float mu,
                          cudaStream_t s) {
  const int grid = grid_window<1>(a.n / 4);
  const Pair tl{{a.p[0], a.p[1]}, 1};
  if (precision == 0)
    boundary_solo_kernel<0><<<grid, kThreads, 0, s>>>(a, tt, buf, lr, mu);
  else
    boundary_solo_kernel<1><<<grid, kThreads, 0, s>>>(a, tt, buf, lr, mu);
  boundary_solo_finalize_kernel<<<1, 1, 0, s>>>(a.st, a.lr);
  if (precision == 0)
    boundary_solo_redo_kernel<0><<<num_sms() * 4, kThreads, 0, s>>>(tt, buf, tl, a.st, lr, mu, a.n);
  else
    boundary_solo_redo_kernel<1><<<num_sms() * 4, kThreads, 0, s>>>(tt, buf, tl, a.st, lr, mu, a.n);
  boundary_solo_redo_finish_kernel<<<1, 1, 0, s>>>(a.st);
}

void launch_boundary_solo_inplace(const AdamWArgs& a, Pair tt, Pair buf, int precision, float lr, float mu,
                                  cudaStream_t s) {
  launch_unscale_check(a.g, a.st, a.n, s);
  const int grid = grid_window<1>(a.n / 4);
  if (precision == 0)
    boundary_solo_inplace_kernel<0><<<grid, kThreads, 0, s>>>(a, tt, buf, lr, mu);
  else
    boundary_solo_inplace_kernel<1><<<grid, kThreads, 0, s>>>(a, tt, buf, lr, mu);
  boundary_inplace_finalize_kernel<<<1, 1, 0, s>>>(a.st, a.lr);
  // the outer gate: flip theta_t / momentum in, or restore theta_local := theta_t
  launch_outer_solo_finish(tt, Pair{{a.p[0], a.p[1]}, 0}, a.st, a.n, s);
}

}  // namespace dlc
