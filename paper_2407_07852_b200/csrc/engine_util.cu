// engine_util.cu — engine internals shared by the engine translation units:
// allocation, runtime knobs, per-phase timing and tracing, the per-step lr /
// bias-correction tables, the live-buffer view of the ping-pong pairs, the
// inner step (K1) and the pieces of the outer step used by every mode.
#include <chrono>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "engine_impl.hpp"

namespace dlc {

void* dalloc(dlc_engine* e, size_t bytes) {
  void* p = nullptr;
  DLC_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 256)));
  e->allocs.push_back(p);
  return p;
}

// ---- P2P tuning: measured defaults, overridable for sweeps (dlc_p2p_set_tuning) ----
namespace {
std::mutex g_tuning_mu;
dlc_p2p_tuning g_tuning{};  // all zero: the measured defaults
dlc_p2p_tuning tuning() {
  std::lock_guard<std::mutex> lock(g_tuning_mu);
  return g_tuning;
}
}  // namespace

// Piece boundaries inside an owner slot of S elements (S a multiple of 64):
// relative piece weights, boundaries rounded down to whole 64-element vectors.
std::vector<size_t> piece_plan(size_t S, size_t n, bool host_path) {
  const dlc_p2p_tuning t = tuning();
  std::vector<size_t> w;
  if (t.plan_len > 0) {
    w.assign(t.plan, t.plan + std::min<uint32_t>(t.plan_len, 32));
  } else if (host_path) {
    w.assign(16, 1);
  } else if (n < kSmallStepElems) {
    w = {1, 2, 2, 1};
  } else {
    w = {1, 2, 3, 2, 1};  // short first and last pieces shrink the pipeline's fill and drain
  }
  size_t sum = 0;
  for (size_t x : w) sum += x;
  std::vector<size_t> b{0};
  size_t cum = 0;
  for (size_t x : w) {
    cum += x;
    b.push_back(cum == sum ? S : (S / 64) * cum / sum * 64);
  }
  return b;
}

// Each TMA fold CTA keeps 3 stages x K inputs x 8 KB of reads in flight; about
// 7.5 MB in flight per GPU saturates the links, hence ~320 / K CTAs
// (profiles/r1_sweep_p2p_*_tma.log).
int tma_ctas(size_t k) {
  const dlc_p2p_tuning t = tuning();
  return t.fold_ctas > 0 ? t.fold_ctas : (int)std::max<size_t>(16, 320 / std::max<size_t>(k, 1));
}

// Threads per TMA fold CTA.  An owner decodes about N contributions per step
// whatever K is, but the CTA count falls as 320 / K, so the fold needs more
// warps per CTA as K grows.  At K = 4 the 4-GPU A/B put the optimum at about
// 80 "128-thread CTA equivalents" (80 x 128 or 48 x 512; 48 x 128 and 64 x 128
// were 20% / 12% slower, profiles/r1_ab_tma_threads_ctas_4gpu.log); K >= 5 keeps
// that capacity with 256 / 512 threads.
int tma_threads(size_t k) {
  const dlc_p2p_tuning t = tuning();
  if (t.fold_threads > 0) return t.fold_threads;
  return k <= 4 ? 128 : (k <= 6 ? 256 : 512);
}

// CTAs of the K2 / K4 piece kernels running beside the fold (0: one per window)
int piece_ctas() { return tuning().piece_ctas; }

// TMA fold kernel: 0 single leader thread (default: fastest inside the 4-GPU
// step, profiles/r2_ab_fold_kernel_*.log), 1 warp-specialised (fastest alone)
int fold_kernel() { return tuning().fold_kernel; }


void ensure_copy_streams(dlc_engine* e) {
  if (!e->h2d) DLC_CUDA(cudaStreamCreateWithFlags(&e->h2d, cudaStreamNonBlocking));
  if (!e->d2h) DLC_CUDA(cudaStreamCreateWithFlags(&e->d2h, cudaStreamNonBlocking));
}

void ensure_chunk_events(dlc_engine* e, size_t count) {
  while (e->chunk_ev.size() < count) {
    cudaEvent_t ev;
    DLC_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    e->chunk_ev.push_back(ev);
  }
}

void harvest(dlc_engine* e) {
  if (e->pending.empty()) return;
  stream_wait(e);
  for (const auto& mk : e->pending) {
    float ms = 0.0f;
    DLC_CUDA(cudaEventElapsedTime(&ms, mk.a, mk.b));
    e->phase_ms[mk.phase] += ms;
    e->phase_n[mk.phase] += 1;
    e->pool.push_back(mk.a);
    e->pool.push_back(mk.b);
  }
  e->pending.clear();
}

cudaEvent_t pooled_event(dlc_engine* e) {
  if (e->pool.empty()) {
    cudaEvent_t ev;
    DLC_CUDA(cudaEventCreate(&ev));
    return ev;
  }
  cudaEvent_t ev = e->pool.back();
  e->pool.pop_back();
  return ev;
}

// Bounds the pending timing events.  Called at the entry of a step, never
// between its launches: a host wait inside a P2P step could block on a peer's
// barrier that is not enqueued yet.
void harvest_if_full(dlc_engine* e) {
  if (e->pending.size() > 8192) harvest(e);
}

// Brackets one phase on the engine stream when timing is on.
void phase_begin(dlc_engine* e) {
  if (!e->timing) return;
  e->open_ev = pooled_event(e);
  DLC_CUDA(cudaEventRecord(e->open_ev, e->stream));
}

void phase_end(dlc_engine* e, int phase) {
  if (!e->timing) return;
  cudaEvent_t b = pooled_event(e);
  DLC_CUDA(cudaEventRecord(b, e->stream));
  e->pending.push_back({phase, e->open_ev, b});
}

// DLC_TRACE=1: events around every op of the pipelined P2P step, printed to
// stderr as a timeline (ms from the step start) once the step completes.
bool tracing() {
  static const bool on = [] {
    const char* s = std::getenv("DLC_TRACE");
    return s && s[0] == '1';
  }();
  return on;
}

cudaEvent_t trace_begin(dlc_engine* e, cudaStream_t s) {
  if (!tracing()) return nullptr;
  cudaEvent_t a = pooled_event(e);
  DLC_CUDA(cudaEventRecord(a, s));
  return a;
}

void trace_end(dlc_engine* e, cudaStream_t s, const char* label, int piece, cudaEvent_t a) {
  if (!a) return;
  cudaEvent_t b = pooled_event(e);
  DLC_CUDA(cudaEventRecord(b, s));
  e->trace.push_back({label, piece, a, b});
}

void trace_dump(dlc_engine* e, cudaEvent_t origin) {
  if (!origin) return;
  DLC_CUDA(cudaDeviceSynchronize());
  for (const auto& m : e->trace) {
    float t0 = 0, t1 = 0;
    DLC_CUDA(cudaEventElapsedTime(&t0, origin, m.a));
    DLC_CUDA(cudaEventElapsedTime(&t1, origin, m.b));
    std::fprintf(stderr, "[dlc trace dev%d] %-10s p%-2d %8.3f -> %8.3f ms (%.3f)\n", e->device, m.label, m.piece, t0,
                 t1, t1 - t0);
    e->pool.push_back(m.a);
    e->pool.push_back(m.b);
  }
  e->trace.clear();
  e->pool.push_back(origin);
}

// Host tables of the per-step scalars the reference computes on the host:
// corr1/corr2 from std::pow(float, float) (optim.cpp:73-76) and lr_at
// (optim.cpp:37-56, indexed as engine.cpp:64).  Index = the 1-based step t.
void ensure_tables(dlc_engine* e, uint64_t t_max) {
  if (t_max < e->tab_cap) return;
  size_t cap = std::max<size_t>(e->tab_cap * 2, 4096);
  while (cap <= t_max) cap *= 2;
  std::vector<float> h(3 * cap);
  const float b1 = e->hyper.beta1, b2 = e->hyper.beta2;
  dlc_lr_schedule sch{e->hyper.warmup_steps, e->cfg.total_inner_steps, e->hyper.inner_lr, e->hyper.lr_decay};
  for (size_t t = 0; t < cap; ++t) {
    h[t] = 1.0f - std::pow(b1, static_cast<float>(t));
    h[cap + t] = 1.0f - std::pow(b2, static_cast<float>(t));
    h[2 * cap + t] = dlc_lr_at(&sch, t);
  }
  float* fresh = nullptr;
  DLC_CUDA(cudaMalloc(&fresh, 3 * cap * sizeof(float)));
  DLC_CUDA(cudaMemcpyAsync(fresh, h.data(), 3 * cap * sizeof(float), cudaMemcpyHostToDevice, e->stream));
  stream_wait(e);  // in-flight K1 launches still read the old table
  if (e->tab) cudaFree(e->tab);
  e->tab = fresh;
  e->tab_cap = cap;
}

void unwatch(dlc_engine* e) {
  if (!e->watch_coll) return;
  auto& v = e->watch_coll->watchers;
  v.erase(std::remove(v.begin(), v.end(), e), v.end());
  e->watch_coll = nullptr;
}

void watch_round(dlc_engine* e, dlc_collective* c) {
  if (!e->watch_ev) DLC_CUDA(cudaEventCreateWithFlags(&e->watch_ev, cudaEventDisableTiming));
  DLC_CUDA(cudaEventRecord(e->watch_ev, e->stream));
  if (e->watch_coll != c) {
    unwatch(e);
    e->watch_coll = c;
    c->watchers.push_back(e);
  }
  e->watched = true;
  e->watch_ms = c->timeout_ms;
  e->deadline = std::chrono::steady_clock::now() + std::chrono::milliseconds(c->timeout_ms);
}

void stream_wait(dlc_engine* e) {
  while (e->watched) {
    const cudaError_t q = cudaEventQuery(e->watch_ev);
    if (q == cudaSuccess) {
      e->watched = false;
      break;
    }
    if (q != cudaErrorNotReady) check_cuda(q, "cudaEventQuery (watched NCCL round)");
    if (std::chrono::steady_clock::now() > e->deadline) {
      // a peer stopped participating: mark the round failed on the device (a
      // side stream; the engine stream is blocked inside NCCL), so its commit
      // gate changes nothing once the caller's shrink with DLC_SHRINK_ABORT
      // releases it (collective.cpp:1368-1440 restarts over the survivors)
      e->watched = false;
      e->nccl_failed = true;
      e->failed_tries += 1;
      if (e->watch_coll) e->watch_coll->broken = true;  // its peers are gone: destroy aborts it
      ensure_copy_streams(e);
      DLC_CUDA(cudaMemsetAsync(e->sig_err, 1, 1, e->h2d));
      DLC_CUDA(cudaStreamSynchronize(e->h2d));
      fail(DLC_ECOLLECTIVE, "outer round timed out after " + std::to_string(e->watch_ms) +
                                " ms: a peer rank stopped participating; the state is unchanged once the round is "
                                "released: shrink the collective with DLC_SHRINK_ABORT and retry");
    }
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
  DLC_CUDA(cudaStreamSynchronize(e->stream));
}

void drain_failed_round(dlc_engine* e) {
  if (!e->nccl_failed) return;
  DLC_CUDA(cudaStreamSynchronize(e->stream));
  if (e->cstream) DLC_CUDA(cudaStreamSynchronize(e->cstream));
  DLC_CUDA(cudaMemset(e->sig_err, 0, 2 * sizeof(int)));
  e->nccl_failed = false;
}

DevState read_state(dlc_engine* e) {
  DevState s;
  stream_wait(e);
  DLC_CUDA(cudaMemcpy(&s, e->st, sizeof(DevState), cudaMemcpyDeviceToHost));
  return s;
}

float* live(dlc_engine* e, int which) {
  if (which == DLC_GRAD) return e->grad;  // not part of a ping-pong pair: no host wait
  const DevState s = read_state(e);
  const int cur = s.cur, oc = s.ocur;
  switch (which) {
    case DLC_THETA_T: return e->theta_t[oc];
    case DLC_THETA_LOCAL: return s.lalias ? e->theta_t[oc] : e->p[cur];
    case DLC_ADAM_M: return e->m[cur];
    case DLC_ADAM_V: return e->v[cur];
    case DLC_MOMENTUM: return e->buf[oc];
    case DLC_GRAD: return e->grad;
  }
  fail(DLC_EINVAL, "unknown engine buffer " + std::to_string(which));
}

// Before a caller writes theta_t or theta_local: give theta_local its own copy
// again (one D2D copy; every kernel path keeps the follow state consistent).
void unalias(dlc_engine* e) {
  DevState s = read_state(e);
  if (!s.lalias) return;
  DLC_CUDA(cudaMemcpyAsync(e->p[s.cur], e->theta_t[s.ocur], e->n * sizeof(float), cudaMemcpyDeviceToDevice,
                           e->stream));
  const int zero = 0;
  DLC_CUDA(cudaMemcpyAsync(&e->st->lalias, &zero, sizeof(int), cudaMemcpyHostToDevice, e->stream));
  DLC_CUDA(cudaStreamSynchronize(e->stream));
}

// live() for a caller that writes through the pointer
float* writable(dlc_engine* e, int which) {
  if (which == DLC_THETA_T || which == DLC_THETA_LOCAL) {
    e->delta_fused = false;  // a fused delta no longer matches the weights
    unalias(e);
  }
  return live(e, which);
}

// K1's arguments for the engine's live state; the gradient is scaled on the
// device first when the caller passes a raw one (engine.cpp:56).
static AdamWArgs inner_args(dlc_engine* e, const float* grad, int grad_is_scaled) {
  harvest_if_full(e);
  if (e->issued_inner >= e->cfg.total_inner_steps) fail(DLC_EINVAL, "inner_step called after total_inner_steps");
  ensure_tables(e, e->issued_inner + 2);
  const float* g = grad;
  if (!grad_is_scaled) {  // engine.cpp:56: closed-form backward of the scaled loss
    launch_scale_gradient(grad, e->st, e->grad, e->n, e->stream);
    g = e->grad;
  }
  AdamWArgs a{};
  for (int i = 0; i < 2; ++i) {
    a.p[i] = e->p[i];
    a.m[i] = e->m[i];
    a.v[i] = e->v[i];
    a.tt[i] = e->theta_t[i];
  }
  a.g = g;
  a.corr1 = e->tab;
  a.corr2 = e->tab + e->tab_cap;
  a.lr = e->tab + 2 * e->tab_cap;
  a.st = e->st;
  a.n = e->n;
  a.b1 = e->hyper.beta1;
  a.b2 = e->hyper.beta2;
  a.eps = e->hyper.adam_eps;
  a.wd = e->hyper.weight_decay;
  a.omb1 = 1.0f - e->hyper.beta1;
  a.omb2 = 1.0f - e->hyper.beta2;
  a.pingpong = e->inner_mode == DLC_INNER_PINGPONG;
  return a;
}

void engine_inner(dlc_engine* e, const float* grad, int grad_is_scaled) {
  AdamWArgs a = inner_args(e, grad, grad_is_scaled);
  // fused delta (opt-in): the last step of a window at K > 1 also writes the
  // pseudo-gradient (engine.cpp:115-126) into the send buffer, so the outer
  // step starts with the exchange; a single worker fuses its whole outer step
  // into the boundary instead (engine_boundary_solo)
  const bool fuse = e->fuse_delta && e->k > 1 && (e->issued_inner + 1) % e->cfg.local_steps_h == 0;
  a.delta = fuse ? e->send : nullptr;
  a.delta_fp16 = e->prec == DLC_FP16;
  phase_begin(e);
  launch_adamw(a, e->stream);
  phase_end(e, DLC_PHASE_INNER);
  launched("adamw");
  e->issued_inner += 1;
  e->delta_fused = fuse;
}

bool boundary_solo_ok(const dlc_engine* e, const dlc_collective* c) {
  return e->fuse_delta && e->k == 1 && (!c || c->kind == 0) &&
         (e->issued_inner + 1) % e->cfg.local_steps_h == 0 && e->issued_inner < e->cfg.total_inner_steps;
}

void engine_boundary_solo(dlc_engine* e, const float* grad, int grad_is_scaled) {
  const AdamWArgs a = inner_args(e, grad, grad_is_scaled);
  e->delta_fused = false;
  DLC_CUDA(cudaMemsetAsync(&e->st->delta_nonfinite, 0, sizeof(int), e->stream));
  phase_begin(e);
  if (e->inner_mode == DLC_INNER_PINGPONG)
    launch_boundary_solo(a, tt_pair(e), buf_pair(e), e->prec, e->hyper.outer_lr, e->hyper.outer_momentum, e->stream);
  else
    launch_boundary_solo_inplace(a, tt_pair(e), buf_pair(e), e->prec, e->hyper.outer_lr, e->hyper.outer_momentum,
                                 e->stream);
  phase_end(e, DLC_PHASE_INNER);
  launched("boundary_solo");
  e->issued_inner += 1;
}


void reset_flags(dlc_engine* e) {
  DLC_CUDA(cudaMemsetAsync(e->flags, 0, kMaxK * sizeof(int), e->stream));
  DLC_CUDA(cudaMemsetAsync(&e->st->delta_nonfinite, 0, sizeof(int), e->stream));
}

// K2 from an explicit theta_local pair (the engine's own, or a staging buffer).
void pseudo_grad(dlc_engine* e, Pair tl) {
  phase_begin(e);
  launch_pseudo_grad(tt_pair(e), tl, e->st, e->send, e->prec, &e->st->delta_nonfinite, 0, e->n, e->stream);
  phase_end(e, DLC_PHASE_PSEUDO);
  launched("pseudo_grad");
}

void pseudo_grad_step(dlc_engine* e, Pair tl, bool fused) {
  if (!fused) {
    pseudo_grad(e, tl);
    return;
  }
  phase_begin(e);
  launch_pseudo_grad_gated(tt_pair(e), tl, e->st, e->send, e->prec, e->n, e->stream);
  phase_end(e, DLC_PHASE_PSEUDO);
  launched("pseudo_grad_gated");
}

void nesterov(dlc_engine* e, const void* dbar, const int* flags, int nflags) {
  phase_begin(e);
  launch_nesterov_outer(tt_pair(e), buf_pair(e), local_pair(e), dbar, e->prec, flags, nflags, e->st,
                        e->hyper.outer_lr, e->hyper.outer_momentum, e->n, e->stream);
  phase_end(e, DLC_PHASE_OUTER);
  launched("nesterov_outer");
}

void fill_report(dlc_engine* e, dlc_collective* c, dlc_reduce_report* rep, uint64_t epoch) {
  if (!rep) return;
  *rep = dlc_reduce_report{};
  rep->outer_epoch = epoch;
  rep->contributors = e->k;  // the survivor count after a membership change (collective.cpp:1378-1389)
  rep->attempts = 1 + e->failed_tries;
  if (e->k > 1) {
    // data bytes: the reference's exact per-peer accounting over
    // partition_ranges (reduce.cpp:91-104); wire bytes: what this transport
    // moved, the owner slots padded to 512 elements (2(K-1) S w each way)
    const int rank = c ? c->rank : 0;
    rep->data_bytes_sent = dlc_per_peer_reduce_bytes(e->n, e->k, (size_t)rank, e->prec);
    rep->data_bytes_received = per_peer_reduce_bytes_received(e->n, e->k, (size_t)rank, e->prec);
    rep->wire_bytes_sent = rep->wire_bytes_received = 2ull * (e->k - 1) * e->S * elem_width(e->prec);
    stream_wait(e);  // raises when a watched NCCL round timed out (its events never complete)
    DLC_CUDA(cudaEventSynchronize(e->ev1));
    float ms = 0;
    DLC_CUDA(cudaEventElapsedTime(&ms, e->ev0, e->ev1));
    rep->wall_ms = ms;
  }
}

// What one peer receives in the reference's round: its own range from each of
// the K - 1 others (scatter), then every other range once (ring all-gather);
// summed over the fleet it equals the bytes sent, 2(K-1) * payload
// (fleet_reduce_bytes, reduce.cpp:106-111).
uint64_t per_peer_reduce_bytes_received(size_t n, size_t k, size_t rank, int precision) {
  if (k <= 1) return 0;
  const uint64_t len = n / k + (rank < n % k ? 1 : 0);  // partition_ranges, reduce.cpp:20-31
  return ((k - 1) * len + (n - len)) * elem_width(precision);
}

// Owner slot S for k workers: ceil(n / k) rounded up to 64 elements per P2P piece.
size_t slot_elems(size_t n, size_t k) {
  const size_t quantum = 64 * kMaxPieces;
  return ((n + k - 1) / k + quantum - 1) / quantum * quantum;
}

// Membership change: lay the collective buffers out for a
// fleet of k workers (k <= k_cap, so the buffers made at creation suffice).
// Padding must read as zero again and the P2P peer mappings are rebuilt by
// the next bind over the new communicator.
void relayout(dlc_engine* e, size_t k) {
  if (k == e->k) return;
  if (k < 1 || k > e->k_cap) fail(DLC_ECOLLECTIVE, "membership of " + std::to_string(k) + " workers exceeds the " +
                                                       std::to_string(e->k_cap) + " this engine was made for");
  stream_wait(e);
  if (e->cstream) DLC_CUDA(cudaStreamSynchronize(e->cstream));
  p2p_unbind(e);
  e->delta_fused = false;
  const size_t pb = e->slot_cap * elem_width(e->prec);
  DLC_CUDA(cudaMemsetAsync(e->send, 0, pb, e->stream));
  if (e->gather) DLC_CUDA(cudaMemsetAsync(e->gather, 0, pb, e->stream));
  if (e->recv) DLC_CUDA(cudaMemsetAsync(e->recv, 0, pb, e->stream));
  DLC_CUDA(cudaMemsetAsync(e->flags, 0, kMaxK * sizeof(int), e->stream));
  DLC_CUDA(cudaStreamSynchronize(e->stream));
  e->k = k;
  e->S = slot_elems(e->n, k);
}

void check_collective(dlc_engine* e, dlc_collective* c) {
  drain_failed_round(e);  // a timed-out NCCL round, released by the caller's shrink
  const size_t world = c ? (size_t)c->world : 1;
  if (world != e->k && c && c->shrunk && c->kind == 1 && world <= e->k_cap &&
      e->issued_inner % e->cfg.local_steps_h == 0)
    relayout(e, world);  // the fleet lost members: survivor slots and divisor
  if (world != e->k)
    fail(DLC_ECOLLECTIVE, "collective world size " + std::to_string(world) + " != num_workers_k " +
                              std::to_string(e->k));
  if (c && c->kind == 1 && c->device != e->device) fail(DLC_ECOLLECTIVE, "collective and engine devices differ");
  if (e->issued_inner % e->cfg.local_steps_h != 0)  // engine.cpp:116-120
    fail(DLC_EINVAL, "pseudo-gradient requested mid-window (inner_step " + std::to_string(e->issued_inner) +
                         ", H " + std::to_string(e->cfg.local_steps_h) + ")");
}

// A flag barrier that timed out (a peer never arrived) surfaces as CollectiveError.
// The round then changed nothing (p2p_finish_kernel's abort gate): the caller
// shrinks the collective around the silent peer and retries the same epoch,
// as Node::Impl::all_reduce restarts with the suspect excluded
// (collective.cpp:1369-1440).  The barrier epochs of the failed round are
// abandoned: the next bind (over the new communicator) agrees on fresh ones.
void check_barrier(dlc_engine* e) {
  if (!e->sig_err || e->nccl_failed) return;  // (a timed-out NCCL round was reported already)
  int err = 0;
  stream_wait(e);
  if (e->cstream) DLC_CUDA(cudaStreamSynchronize(e->cstream));
  DLC_CUDA(cudaMemcpy(&err, e->sig_err, sizeof(int), cudaMemcpyDeviceToHost));
  if (!err) return;
  DLC_CUDA(cudaMemset(e->sig_err, 0, sizeof(int)));
  if (e->p2p_bound) const_cast<dlc_collective*>(e->p2p_bound)->broken = true;
  p2p_unbind(e);
  e->failed_tries += 1;
  if (e->inner_mode != DLC_INNER_PINGPONG)
    fail(DLC_ECOLLECTIVE, "outer round failed: a peer rank stopped participating (DLC_INNER_INPLACE: theta_local "
                          "was overwritten, restore it before retrying)");
  fail(DLC_ECOLLECTIVE, "outer round failed: a peer rank stopped participating; state unchanged, shrink the "
                        "collective and retry");
}

void outer_result(dlc_engine* e, dlc_outer_result* res) {
  if (!res) return;  // asynchronous call: nothing is synchronised here
  check_barrier(e);
  e->failed_tries = 0;
  const DevState s = read_state(e);
  res->applied = s.last_applied;
  res->outer_epoch = s.outer_epoch;
}

}  // namespace dlc

using namespace dlc;

extern "C" {

int dlc_p2p_set_tuning(const dlc_p2p_tuning* t) {
  return guard([&] {
    dlc_p2p_tuning v{};
    if (t) {
      v = *t;
      if (v.plan_len > 32) fail(DLC_ECONFIG, "p2p tuning: at most 32 pieces");
      for (uint32_t i = 0; i < v.plan_len; ++i)
        if (v.plan[i] == 0 || v.plan[i] > 1024) fail(DLC_ECONFIG, "p2p tuning: piece weights must be 1..1024");
      if (v.fold_threads != 0 && v.fold_threads != 128 && v.fold_threads != 256 && v.fold_threads != 512)
        fail(DLC_ECONFIG, "p2p tuning: fold_threads must be 128, 256 or 512");
      if (v.fold_ctas < 0 || v.piece_ctas < 0) fail(DLC_ECONFIG, "p2p tuning: negative CTA count");
      if (v.fold_kernel != 0 && v.fold_kernel != 1) fail(DLC_ECONFIG, "p2p tuning: fold_kernel must be 0 or 1");
    }
    std::lock_guard<std::mutex> lock(g_tuning_mu);
    g_tuning = v;
  });
}

int dlc_p2p_get_tuning(dlc_p2p_tuning* t) {
  return guard([&] {
    if (!t) fail(DLC_EINVAL, "dlc_p2p_get_tuning: null argument");
    *t = tuning();
  });
}

}  // extern "C"
