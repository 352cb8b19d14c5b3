// kernels.cuh — launch interface of the DiLoCo hot-path kernels (sm_100a).
//
//   K1  adamw       fused grad-scaler unscale + overflow OR + AdamW
//                   (proj/src/optim.cpp:58-93,121-148; engine.cpp:50-69)
//   K2  pseudo_grad delta = theta_t - theta_local, FP32 or FP16-encoded
//                   (engine.cpp:115-126 -> tensor.cpp:118-140)
//   K3  fold        owner fold of K contributions in rank order, / K, encode
//                   once (reduce.cpp:33-89; collective.cpp:1444-1489)
//   K4  nesterov    finite-gated outer Nesterov + theta_local refresh
//                   (engine.cpp:128-146 -> optim.cpp:95-115)
//
// Work distribution (measured, profiles/r1_tune_stream_v2.log): one CTA per
// 256*U consecutive 128-bit vectors, launched in address order, so the CTAs
// resident at any instant stream through one compact window of every buffer.
// That beats a persistent grid-stride loop by 12-18% on these shapes (K1
// 7.0 vs 5.9 TB/s).  Global decisions that need every element (overflow skip,
// non-finite outer step) are taken by a one-CTA finalize kernel that follows.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace dlc {

constexpr int kMaxK = 32;  // largest worker count a single fold launch takes

struct PtrList {
  const void* ptr[kMaxK];
};

// Device-resident engine scalars (EngineState, engine.hpp:48-56; AdamWState
// step_count, optim.hpp:20; LossScaler, optim.hpp:52-56).  Kept on the GPU so
// the inner loop never waits on the host: the overflow decision, step counter
// and loss scale are all updated by the K1 finalize kernel.
struct DevState {
  uint64_t step_count;      // applied AdamW steps
  uint64_t inner_step;      // batches consumed (data cursor, always advances)
  uint64_t good;            // scaler consecutive_good
  uint64_t growth;          // scaler growth_interval
  uint64_t outer_epoch;
  uint64_t overflow_skips;  // inner steps skipped on overflow
  uint64_t outer_skips;     // outer steps skipped on a non-finite reduction
  float scale;              // loss scale (power of two)
  float last_lr;            // lr of the last inner step (0 when skipped)
  int cur;                  // live buffer of the p/m/v ping-pong pair
  int found_inf;            // K1 scratch: OR of !isfinite(g / scale)
  int lalias;               // theta_local == theta_t[ocur] by construction (see Pair::follow)
  int last_overflow;        // InnerStepResult::overflow_skipped
  int delta_nonfinite;      // K2 / solo: non-finite delta (or FP16 encode overflow)
  int last_applied;         // OuterStepResult::applied
  int ocur;                 // live buffer of the theta_t / momentum pair (solo fused outer step)
  int delta_ready;          // the send buffer holds theta_t - theta_local of the live state: written by
                            // the window's last K1 (AdamWArgs::delta) when that step was applied
  int redo;                 // fused single-worker boundary: its inner step overflowed, so the outer
                            // step reruns from the unchanged theta_local (launch_boundary_solo)
};

struct AdamWArgs {
  float* p[2];
  float* m[2];
  float* v[2];
  const float* g;      // scaled gradient (loss-scaled backward output)
  const float* corr1;  // host tables indexed by the 1-based step t
  const float* corr2;
  const float* lr;
  DevState* st;
  size_t n;
  float b1, b2, eps, wd, omb1, omb2;  // omb = 1.0f - b, rounded as optim.cpp:84-85
  int pingpong;                       // 1: read [cur], write [cur^1]; 0: in place, gated
  float* tt[2];                       // theta_t pair: the source while DevState::lalias (pingpong only)
  // K2 fused into the last inner step of a window (K > 1): besides p', write
  // delta = theta_t[ocur] - p' into `delta` (FP32, or binary16 codes when
  // delta_fp16) and let the finalize set DevState::delta_ready = !overflow.
  void* delta;                        // nullptr: plain K1
  int delta_fp16;
};

// Scalars of one out-of-place AdamW call whose gradient is already unscaled
// and checked (host-staged drop-in of adamw_step, optim.hpp:61-62).
struct AdamWPlain {
  float b1, b2, eps, wd, omb1, omb2, corr1, corr2, lr;
};


// The two buffers of a ping-pong pair; DevState::cur / ocur selects the live one.
struct Pair {
  float* ptr[2];
  // theta_local pair only (PINGPONG engines): every outer step ends with
  // theta_local := theta_t (engine.cpp:141-143).  Instead of copying, the engine
  // records the equality (DevState::lalias) and reads theta_local from
  // theta_t[ocur] until the next applied inner step writes a fresh p buffer.
  int follow;
};

int num_sms();

// K1 --------------------------------------------------------------------------
// PINGPONG: one pass (reads [cur], writes [cur^1]) + finalize.  INPLACE: an
// overflow pre-pass over g, the gated in-place update, finalize.
void launch_adamw(const AdamWArgs& a, cudaStream_t s);
void launch_adamw_plain(const float* p, const float* g, float* m, float* v, float* out,
                        size_t n, const AdamWPlain& a, cudaStream_t s);

// K1 + K2 + K4 for one worker at a window boundary ------------------------------
// DilocoOptimizer::step at inner_step % H == 0 (engine.cpp:162-174) with the
// SoloCollective (reduce.cpp:113-126), PINGPONG engines: ONE HBM pass reads
// theta_local (p, or theta_t while DevState::lalias), g, m, v, theta_t and
// momentum and writes m', v' and the speculative theta_t', momentum' (40 B per
// parameter instead of K1's 28 + the solo outer step's 20).  theta_local' is
// never stored: after the outer step theta_local follows theta_t.  A one-thread
// finalize applies the inner step's skip decision and scaler update, then the
// outer step's finite gate.  If the inner step overflowed, the fused outer
// values came from a rejected theta_local: a gated persistent pass reruns the
// solo outer step from the unchanged one (DevState::redo; ~10 us when idle).
void launch_boundary_solo(const AdamWArgs& a, Pair theta_t, Pair buf, int precision, float lr, float mu,
                          cudaStream_t s);
// The same for DLC_INNER_INPLACE engines (fixed theta_local / m / v addresses):
// the overflow pre-pass first (4 B/param), then ONE in-place pass that applies
// the inner step unless it overflowed and the outer step from the resulting
// theta_local, storing theta_t' into theta_local as well (44 B/param; 48 with
// the pre-pass, against 32 + 24 as two steps); a skipped outer step restores
// theta_local := theta_t in the finish (outer_solo_finish_kernel).
void launch_boundary_solo_inplace(const AdamWArgs& a, Pair theta_t, Pair buf, int precision, float lr, float mu,
                                  cudaStream_t s);
// INPLACE K1's pre-pass: found_inf |= !isfinite(g * (1 / scale)).
void launch_unscale_check(const float* g, DevState* st, size_t n, cudaStream_t s);

// K2 --------------------------------------------------------------------------
// The outer step's K2 after a fused K1 (AdamWArgs::delta): a persistent grid
// that returns at once when DevState::delta_ready (the usual case) and
// otherwise (the window's last step overflowed, so theta_local kept its old
// value) writes delta = theta_t - theta_local over [0, n) of `send`.
void launch_pseudo_grad_gated(Pair theta_t, Pair theta_local, const DevState* st, void* send, int precision,
                              size_t n, cudaStream_t s);
// Elements [off, off + len) of delta = theta_t - theta_local into `out`
// (float* for precision 0, binary16 codes for 1); non-finite OR into *flag.
void launch_pseudo_grad(Pair theta_t, Pair theta_local, const DevState* st, void* out,
                        int precision, int* flag, size_t off, size_t len, cudaStream_t s);

// K3 --------------------------------------------------------------------------
// in_kind 0: FP32 contributions, 1: FP16 codes, 2: FP32 contributions that go
// through one encode/decode each (reduce_average's FP16 path on FP32 inputs).
// out_kind 0: FP32 mean, 1: FP16 code of the mean, 2: FP32 decode(encode(mean)).
void launch_fold(const PtrList& in, int k, int in_kind, void* out, int out_kind, int* flag,
                 size_t n, cudaStream_t s);

// K4 --------------------------------------------------------------------------
void launch_nesterov_outer(Pair theta_t, Pair buf, Pair theta_local,
                           const void* dbar, int precision, const int* flags, int nflags,
                           DevState* st, float lr, float mu, size_t n, cudaStream_t s);
// Pipelined DLC_MODE_P2P pieces.  Piece p of the outer step is the sub-range
// [q*S + po, q*S + po + plen) of every owner slot q (po = p*plen).  K2 writes a
// piece of the send buffer; K4 consumes a piece of every owner's mean slot and
// writes theta_t / momentum speculatively into the idle ping-pong buffers (the
// non-finite gate is only known after the last piece); p2p_finish then flips
// `ocur` when every owner flag is clean, else restores theta_local := theta_t.
// Owner fold fused with the all-gather (DLC_MODE_P2P): contributions `in`
// (peer send buffers, pulled over NVLink) folded in rank order exactly as
// launch_fold, the encoded mean stored to all `nout` destinations (this rank's
// slot in every peer's gather buffer, posted NVLink writes) and a non-finite
// mean marked by storing 1 to every `flags` entry; ends with a system fence.
// `ctas` > 0 runs a persistent grid of that many CTAs (0: one CTA per window).
void launch_fold_push(const PtrList& in, int k, int precision, const PtrList& outs, int nout,
                      const PtrList& flags, int nflags, size_t n, int ctas, cudaStream_t s);
// fold_push with the bulk-copy engine (TMA) moving the tiles, `threads`
// folding threads per CTA (128 / 256 / 512); kernel 0: one leader thread
// issues the copies between its share of the fold, 1: warp-specialised (a
// producer warp + the folding warps).  False when k is outside 2..8 (the caller then
// uses launch_fold_push).
bool launch_fold_push_tma(const PtrList& in, int k, int precision, const PtrList& outs, int nout,
                          const PtrList& flags, int nflags, size_t n, int ctas, int threads, int kernel,
                          cudaStream_t s);
// Fleet barrier over NVLink flags (DLC_MODE_P2P): one CTA stores the barrier's
// signal into slot `me` of every peer's signal array (`remote`, after a system
// fence), then waits until every peer's signal has landed in `local`.  A peer
// silent for `timeout_ns` (globaltimer; NodeOptions::reduce_timeout_ms,
// collective.hpp) sets *err and the kernel exits instead of hanging the GPU;
// once *err is set (this round already failed) later barriers neither signal
// nor wait.  A signal is (epoch << 1) | error bit.  `commit` (the last barrier
// of a step): a failed rank still signals, with its error bit set, and a rank
// that receives an error bit sets *err, so every rank's finish gate sees the
// failure.  `stall` (fault injection, the reference's set_stage_hook) makes
// this rank stop arriving: it sets *err without signalling its peers.
void launch_flag_barrier(const PtrList& remote, const uint64_t* local, int k, int me, uint64_t epoch,
                         int* err, uint64_t timeout_ns, bool stall, bool commit, cudaStream_t s);
void launch_pseudo_grad_piece(Pair theta_t, Pair theta_local, const DevState* st, void* send,
                              int precision, int k, size_t S, size_t po, size_t plen, size_t n,
                              int ctas, cudaStream_t s);
void launch_nesterov_p2p_piece(Pair theta_t, Pair buf, Pair theta_local, const PtrList& slots,
                               int k, size_t S, size_t po, size_t plen, int precision,
                               DevState* st, float lr, float mu, size_t n, int ctas, cudaStream_t s);
// `abort` (nullable): a failed round (a barrier timed out) leaves every state
// buffer and counter as it was, so the round can be retried on a shrunk world.
void launch_p2p_finish(Pair theta_t, Pair theta_local, const PtrList& flags, int k, DevState* st,
                       size_t n, const int* abort, cudaStream_t s);
// K2+K4 fused for a single worker (SoloCollective, reduce.cpp:113-126): one
// HBM pass reading theta_t[ocur], buf[ocur], theta_local and writing
// theta_t[ocur^1], buf[ocur^1], theta_local (24 B/param), then a finish kernel
// that flips `ocur` only when every delta was finite and otherwise restores
// theta_local := theta_t (engine.cpp:136-144).  `src` (nullable) overrides the
// theta_local input.  The chunk / finish split lets host copies overlap.
void launch_outer_solo_fused(Pair theta_t, Pair buf, Pair theta_local, const float* src,
                             int precision, DevState* st, float lr, float mu, size_t n,
                             cudaStream_t s);
void launch_outer_solo_chunk(Pair theta_t, Pair buf, Pair theta_local, const float* src,
                             int precision, DevState* st, float lr, float mu, size_t off,
                             size_t len, cudaStream_t s);
void launch_outer_solo_finish(Pair theta_t, Pair theta_local, DevState* st, size_t n,
                              cudaStream_t s);
void launch_nesterov_plain(const float* p, const float* g, float* buf, float* out, size_t n,
                           float lr, float mu, cudaStream_t s);

// elementwise helpers -----------------------------------------------------------
void launch_axpy(float alpha, const float* x, const float* y, float* out, size_t n,
                 cudaStream_t s);
void launch_encode(const float* x, uint16_t* out, int* flag, size_t n, cudaStream_t s);
void launch_decode(const uint16_t* b, float* out, size_t n, cudaStream_t s);
void launch_nonfinite(const float* x, int* flag, size_t n, cudaStream_t s);
void launch_nonfinite_codes(const uint16_t* b, int* flag, size_t n, cudaStream_t s);
// Ordered fold over an arbitrary number of FP32 contributions whose pointers
// live in device memory (host-staged reduce_average for any k).
void launch_fold_many(const float* const* ptrs, size_t k, int fp16, float* out, size_t n,
                      cudaStream_t s);
void launch_unscale(const float* g, float inv, float* out, int* flag, size_t n, cudaStream_t s);
// g_scaled = g * scale where scale is read from the device state (engine.cpp:20-27).
void launch_scale_gradient(const float* g, const DevState* st, float* out, size_t n,
                           cudaStream_t s);
// out[i] = CounterRng(key) draw first+i, uniform in [lo, hi) (rng.hpp:43-56).
void launch_rng_fill(uint64_t key, uint64_t first, float lo, float hi, float* out, size_t n,
                     cudaStream_t s);
// theta_local = theta_t - U(lo, hi) keyed draw (synthetic end-of-window weights).
void launch_rng_perturb(const float* theta_t, uint64_t key, float lo, float hi, float* out,
                        size_t n, cudaStream_t s);
// codes for the consecutive FP32 bit patterns [start, start + n)
void launch_encode_bits_range(uint32_t start, uint16_t* out, size_t n, cudaStream_t s);
void launch_copy(const float* src, float* dst, size_t n, cudaStream_t s);
// *dst |= *src (one thread)
void launch_or_word(int* dst, const int* src, cudaStream_t s);

}  // namespace dlc
