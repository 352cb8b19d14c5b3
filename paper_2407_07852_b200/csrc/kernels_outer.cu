// kernels_outer.cu — the outer step's elementwise kernels: K2 pseudo-gradient
// (engine.cpp:115-126), K4 finite-gated Nesterov + theta_local refresh
// (engine.cpp:128-146), their pieces for the pipelined P2P step with the
// speculative write and finish gate, and K2+K4 fused for one worker.
#include <algorithm>
#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "device.cuh"
#include "kernels.cuh"

namespace dlc {

namespace {

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

// The outer step's K2 after a fused K1: nothing to do when the window's last
// step wrote the delta (DevState::delta_ready); else the whole delta, grid-stride.
template <int PREC>
__global__ void __launch_bounds__(kThreads) pseudo_grad_gated_kernel(Pair ttp, Pair tl, const DevState* st, void* out,
                                                                     size_t n) {
  if (*(volatile const int*)&st->delta_ready) return;
  const float* T = sel(ttp, st->ocur);
  const float* L = local_src(tl, ttp, st);
  const size_t n4 = n / 4;
  for (size_t j = gtid(); j < n4; j += gstride()) {
    const float4 x = ld_stream(reinterpret_cast<const float4*>(T) + j);
    const float4 y = ld_stream(reinterpret_cast<const float4*>(L) + j);
    const float4 d = make_float4(delta_elem(x.x, y.x), delta_elem(x.y, y.y), delta_elem(x.z, y.z),
                                 delta_elem(x.w, y.w));
    if (PREC == 0)
      st_stream(reinterpret_cast<float4*>(out) + j, d);
    else
      st_stream(reinterpret_cast<uint2*>(out) + j,
                make_uint2(pack2(fp16_encode(d.x), fp16_encode(d.y)), pack2(fp16_encode(d.z), fp16_encode(d.w))));
  }
  if (blockIdx.x == 0 && threadIdx.x < n - n4 * 4) {
    const size_t e = n4 * 4 + threadIdx.x;
    const float d = delta_elem(T[e], L[e]);
    if (PREC == 0)
      static_cast<float*>(out)[e] = d;
    else
      static_cast<uint16_t*>(out)[e] = fp16_encode(d);
  }
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
      st_exchange(reinterpret_cast<float4*>(static_cast<float*>(send) + e0), d);
    } else {
      st_exchange(reinterpret_cast<uint2*>(static_cast<uint16_t*>(send) + e0),
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
    const float4 d = PREC == 0 ? ld_exchange(reinterpret_cast<const float4*>(static_cast<const float*>(dbar) + o0))
                               : decode4(ld_exchange(reinterpret_cast<const uint2*>(
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
                                                              int k, DevState* st, size_t n, const int* abort) {
  // a failed round (abort) changes nothing: no flip, no epoch, no theta_local
  if (abort && *reinterpret_cast<const volatile int*>(abort)) return;
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

}  // namespace

void launch_pseudo_grad(Pair tt, Pair tl, const DevState* st, void* out, int precision, int* flag, size_t off,
                        size_t len, cudaStream_t s) {
  const int grid = grid_window<kU2>(len / 4);
  if (precision == 0)
    pseudo_grad_kernel<0><<<grid, kThreads, 0, s>>>(tt, tl, st, out, flag, off, len);
  else
    pseudo_grad_kernel<1><<<grid, kThreads, 0, s>>>(tt, tl, st, out, flag, off, len);
}

void launch_pseudo_grad_gated(Pair tt, Pair tl, const DevState* st, void* send, int precision, size_t n,
                              cudaStream_t s) {
  const int grid = num_sms() * 8;
  if (precision == 0)
    pseudo_grad_gated_kernel<0><<<grid, kThreads, 0, s>>>(tt, tl, st, send, n);
  else
    pseudo_grad_gated_kernel<1><<<grid, kThreads, 0, s>>>(tt, tl, st, send, n);
}

void launch_nesterov_outer(Pair tt, Pair buf, Pair tl, const void* dbar, int precision, const int* flags,
                           int nflags, DevState* st, float lr, float mu, size_t n, cudaStream_t s) {
  const int grid = grid_window<1>(n / 4);
  if (precision == 0)
    nesterov_outer_kernel<0><<<grid, kThreads, 0, s>>>(tt, buf, tl, dbar, flags, nflags, st, lr, mu, n);
  else
    nesterov_outer_kernel<1><<<grid, kThreads, 0, s>>>(tt, buf, tl, dbar, flags, nflags, st, lr, mu, n);
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

void launch_p2p_finish(Pair tt, Pair tl, const PtrList& flags, int k, DevState* st, size_t n, const int* abort,
                       cudaStream_t s) {
  p2p_finish_kernel<<<num_sms() * 4, kThreads, 0, s>>>(tt, tl, flags, k, st, n, abort);
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

}  // namespace dlc
