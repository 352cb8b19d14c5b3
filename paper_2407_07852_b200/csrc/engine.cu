// engine.cu — sections 2 and 3 of include/diloco_cuda.h: the collective plugin
// (class Collective, reduce.hpp:86-97) and the device-resident DilocoEngine
// (engine.hpp:76-157).
//
// HBM layout of one engine (one worker, one GPU), every buffer 256-B aligned:
//   theta_t[2][N], buf[2][N]       outer weights, momentum  FP32 ping-pong pair
//   p[2][N], m[2][N], v[2][N]      theta_local + AdamW      FP32 ping-pong pair
//                                  (one buffer each in INPLACE mode; theta_local
//                                  may follow theta_t[ocur], Pair::follow)
//   grad[N]                        gradient staging          FP32
//   send[K*S]                      pseudo-gradient, padded   FP32 | FP16 codes
//   recv[K*S], gather[K*S]         scatter / all-gather      (K > 1)
//   flags[kMaxK], DevState, lr/corr tables
// S = ceil(N / K) rounded up to 512 elements: rank r owns send[r*S, (r+1)*S).
// The partition differs from partition_ranges (reduce.cpp:20-31) only by the
// padding; results are independent of the split because the fold is
// elementwise, and the scalar bytes on the wire are the same
// 2(K-1)/K*N*{4,2} per peer.
#include <chrono>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "internal.hpp"
#include "kernels.cuh"

using namespace dlc;

struct dlc_collective {
  int kind = 0;  // 0 solo, 1 nccl
  int rank = 0;
  int world = 1;
  int device = 0;
  int mode = DLC_MODE_ORDERED;
  ncclComm_t comm = nullptr;
  cudaStream_t stream = nullptr;  // used only by the host-buffer plugin call
  bool in_world = false;          // one of the K collectives of a dlc_world (one host thread)
};

struct dlc_engine {
  int device = 0;
  cudaStream_t stream = nullptr;
  dlc_config cfg{};
  dlc_hyperparams hyper{};
  int inner_mode = DLC_INNER_PINGPONG;
  size_t n = 0, k = 1, S = 0;
  int prec = DLC_FP32;
  // theta_t / momentum: a ping-pong pair for a single worker (fused solo outer
  // step, DevState::ocur selects the live one); both entries alias for K > 1.
  float* theta_t[2] = {nullptr, nullptr};
  float* p[2] = {nullptr, nullptr};
  float* m[2] = {nullptr, nullptr};
  float* v[2] = {nullptr, nullptr};
  float* buf[2] = {nullptr, nullptr};
  float* grad = nullptr;
  void* send = nullptr;
  void* recv = nullptr;
  void* gather = nullptr;
  int* flags = nullptr;
  DevState* st = nullptr;
  float* tab = nullptr;  // corr1 | corr2 | lr, tab_cap entries each
  size_t tab_cap = 0;
  uint64_t issued_inner = 0;  // host mirror of the data cursor (always advances)
  std::vector<void*> allocs;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // per-phase event timing (dlc_engine_set_timing)
  struct Mark {
    int phase;
    cudaEvent_t a, b;
  };
  bool timing = false;
  std::vector<Mark> pending;
  std::vector<cudaEvent_t> pool;
  double phase_ms[4] = {0, 0, 0, 0};
  uint64_t phase_n[4] = {0, 0, 0, 0};
  cudaEvent_t open_ev = nullptr;
  // DLC_MODE_P2P: every rank's send buffer, gather buffer and flag array mapped
  // into this process through CUDA IPC (own entries are local).
  int* barrier_buf = nullptr;
  const dlc_collective* p2p_bound = nullptr;
  void* peer_send[kMaxK] = {};
  void* peer_gather[kMaxK] = {};
  int* peer_flags[kMaxK] = {};
  void* peer_recv[kMaxK] = {};  // "push" mover: owners' recv buffers
  uint64_t* sig = nullptr;  // flag-barrier signal slots, one per rank
  uint64_t* peer_sig[kMaxK] = {};
  uint64_t sig_epoch = 0;
  int* sig_err = nullptr;
  std::vector<void*> ipc_opened;
  // host-buffer path: copy streams and per-chunk events
  cudaStream_t h2d = nullptr, d2h = nullptr;
  std::vector<cudaEvent_t> chunk_ev;
  // pipelined P2P: high-priority stream for barriers + owner folds, per-piece events
  cudaStream_t cstream = nullptr;
  cudaStream_t sstream = nullptr;  // "push2" mover: scatter kernels, concurrent with the folds
  struct TraceMark {
    const char* label;
    int piece;
    cudaEvent_t a, b;
  };
  std::vector<TraceMark> trace;  // DLC_TRACE=1: per-op timeline of the P2P step
  cudaStream_t pull[kMaxK] = {};  // copy-engine pulls of peers' delta slices
  cudaStream_t gath[kMaxK] = {};  // copy-engine pulls of owners' mean slices
  std::vector<cudaEvent_t> piece_ev;
  // wire rounds (dlc_engine_wire_*): fold rows of the owned range, `wire_stride` elements each
  void* wire_rows = nullptr;
  size_t wire_rows_bytes = 0;
  uint64_t wire_stride = 0;
};

namespace {

size_t elem_width(int prec) { return prec == DLC_FP16 ? 2 : 4; }

void* dalloc(dlc_engine* e, size_t bytes) {
  void* p = nullptr;
  DLC_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 256)));
  e->allocs.push_back(p);
  return p;
}

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) DLC_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

void launched(const char* what) { DLC_LAUNCHED(what); }

// Host <-> device chunk of the host-buffer outer step (64 MB of FP32).
constexpr size_t kHostChunk = size_t(16) << 20;
// Pieces of the pipelined P2P outer step (DLC_MODE_P2P).
// Owner slots are a multiple of 64 * kMaxPieces elements; the split actually
// used comes from DLC_P2P_PLAN / DLC_P2P_PIECES (profiles/r1_sweep_p2p_*.log).
constexpr size_t kMaxPieces = 8;

// (read on every step so a tuning sweep can change them in-process)
size_t p2p_pieces() {
  const char* s = std::getenv("DLC_P2P_PIECES");
  const long v = s ? std::strtol(s, nullptr, 10) : 4;
  size_t p = 1;  // a power of two <= kMaxPieces, so every piece is a whole number of 64-element vectors
  while (p * 2 <= (size_t)std::min<long>(std::max<long>(v, 1), (long)kMaxPieces)) p *= 2;
  return p;
}

// Piece boundaries inside an owner slot of S elements (S a multiple of
// 64 * kMaxPieces): DLC_P2P_PLAN lists piece weights in eighths of a slot
// (default "1,1,2,2,1,1": short first and last pieces shrink the pipeline's
// fill (K2 of piece 0) and drain (K4 of the last piece)); DLC_P2P_PIECES asks
// for equal pieces instead.
std::vector<size_t> piece_plan(size_t S) {
  std::vector<size_t> w;
  const char* plan = std::getenv("DLC_P2P_PLAN");
  if (plan || !std::getenv("DLC_P2P_PIECES")) {
    std::string str = plan ? plan : "1,1,2,2,1,1";
    size_t pos = 0, sum = 0;
    while (pos <= str.size()) {
      const size_t comma = str.find(',', pos);
      const std::string tok = str.substr(pos, comma == std::string::npos ? std::string::npos : comma - pos);
      const long v = std::strtol(tok.c_str(), nullptr, 10);
      if (v <= 0) {
        w.clear();
        break;
      }
      w.push_back((size_t)v);
      sum += (size_t)v;
      if (comma == std::string::npos) break;
      pos = comma + 1;
    }
    if (sum != kMaxPieces) w.clear();
  }
  if (w.empty()) w.assign(p2p_pieces(), kMaxPieces / p2p_pieces());
  std::vector<size_t> b{0};
  for (size_t x : w) b.push_back(b.back() + x * (S / kMaxPieces));
  return b;
}

// Who moves the bytes in DLC_MODE_P2P: "sm" (default) = a persistent fold
// kernel pulling deltas and pushing means over NVLink; "ce" = DMA copy engines.
bool p2p_mover_sm() {
  const char* s = std::getenv("DLC_P2P_COPY");
  return !(s && std::string(s) == "ce");
}

// "push": the scatter is fused into K2 (deltas stored straight into the
// owners' recv rows over NVLink), so every NVLink byte is a posted store.
bool p2p_mover_push() {
  const char* s = std::getenv("DLC_P2P_COPY");
  return s && std::string(s) == "push";
}
// push/push: K2 writes locally, a scatter kernel on the comm stream pushes the
// rows to their owners, the owners fold locally and push the means
bool p2p_mover_push2() {
  const char* s = std::getenv("DLC_P2P_COPY");
  return s && std::string(s) == "push2";
}

// CTAs of the persistent SM mover (0 = one CTA per window, no SM partitioning);
// default 384 of the 1184 resident CTA slots (profiles/r1_sweep_p2p_*_barrier.log).
int comm_ctas() {
  const char* s = std::getenv("DLC_COMM_CTAS");
  return s ? (int)std::strtol(s, nullptr, 10) : 256;  // profiles/r1_sweep_p2p_4gpu_kk.log
}
// SM mover fold on the bulk-copy engine (fold_push_tma_kernel), and its CTAs
bool fold_tma() {
  const char* s = std::getenv("DLC_FOLD_TMA");
  return !(s && std::string(s) == "0");
}
// Each TMA fold CTA keeps 3 stages x K inputs x 8 KB of reads in flight; about
// 7.5 MB in flight per GPU saturates the links, hence ~320 / K CTAs
// (profiles/r1_sweep_p2p_*_tma.log).
int tma_ctas(size_t k) {
  const char* s = std::getenv("DLC_TMA_CTAS");
  return s ? (int)std::strtol(s, nullptr, 10) : (int)std::max<size_t>(16, 320 / std::max<size_t>(k, 1));
}
// CTAs of the K2 / K4 piece kernels running beside the fold (0: one per window)
int piece_ctas() {
  const char* s = std::getenv("DLC_P2P_PIECE_CTAS");
  return s ? (int)std::strtol(s, nullptr, 10) : 0;
}

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
  DLC_CUDA(cudaStreamSynchronize(e->stream));
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

// Brackets one phase on the engine stream when timing is on.
void phase_begin(dlc_engine* e) {
  if (!e->timing) return;
  if (e->pending.size() > 8192) harvest(e);
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
  const char* s = std::getenv("DLC_TRACE");
  return s && s[0] == '1';
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
  DLC_CUDA(cudaStreamSynchronize(e->stream));  // in-flight K1 launches still read the old table
  if (e->tab) cudaFree(e->tab);
  e->tab = fresh;
  e->tab_cap = cap;
}

DevState read_state(dlc_engine* e) {
  DevState s;
  DLC_CUDA(cudaStreamSynchronize(e->stream));
  DLC_CUDA(cudaMemcpy(&s, e->st, sizeof(DevState), cudaMemcpyDeviceToHost));
  return s;
}

float* live(dlc_engine* e, int which) {
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
  if (which == DLC_THETA_T || which == DLC_THETA_LOCAL) unalias(e);
  return live(e, which);
}

void engine_inner(dlc_engine* e, const float* grad, int grad_is_scaled) {
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
  phase_begin(e);
  launch_adamw(a, e->stream);
  phase_end(e, DLC_PHASE_INNER);
  launched("adamw");
  e->issued_inner += 1;
}

// PINGPONG: theta_local follows theta_t after every outer step (Pair::follow).
Pair local_pair(dlc_engine* e) { return Pair{{e->p[0], e->p[1]}, e->inner_mode == DLC_INNER_PINGPONG}; }

Pair tt_pair(dlc_engine* e) { return Pair{{e->theta_t[0], e->theta_t[1]}}; }
Pair buf_pair(dlc_engine* e) { return Pair{{e->buf[0], e->buf[1]}}; }

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

void nesterov(dlc_engine* e, const void* dbar, const int* flags, int nflags) {
  phase_begin(e);
  launch_nesterov_outer(tt_pair(e), buf_pair(e), local_pair(e), dbar, e->prec, flags, nflags, e->st,
                        e->hyper.outer_lr, e->hyper.outer_momentum, e->n, e->stream);
  phase_end(e, DLC_PHASE_OUTER);
  launched("nesterov_outer");
}

// The whole outer step: fused K2+K4 for one worker, else K2 -> C1/K3 -> K4.
// `src` (nullable) supplies theta(t+h) from a caller buffer.
void outer_round(dlc_engine* e, dlc_collective* c, const float* src, dlc_reduce_report* rep);

ncclDataType_t nccl_type(int prec) { return prec == DLC_FP16 ? ncclFloat16 : ncclFloat32; }

void p2p_unbind(dlc_engine* e) {
  for (void* p : e->ipc_opened) cudaIpcCloseMemHandle(p);
  e->ipc_opened.clear();
  e->p2p_bound = nullptr;
}

// Maps every rank's send buffer, owner slot and owner flag into this process:
// IPC handles are all-gathered over the collective's own NCCL communicator.
void p2p_bind(dlc_engine* e, dlc_collective* c) {
  if (e->p2p_bound == c) return;
  p2p_unbind(e);
  const int K = (int)e->k, r = c->rank;
  struct Handles {
    cudaIpcMemHandle_t send, gather, flags, sig, recv;
  };
  Handles mine;
  DLC_CUDA(cudaIpcGetMemHandle(&mine.recv, e->recv));
  DLC_CUDA(cudaIpcGetMemHandle(&mine.send, e->send));
  DLC_CUDA(cudaIpcGetMemHandle(&mine.gather, e->gather));
  DLC_CUDA(cudaIpcGetMemHandle(&mine.flags, e->flags));
  DLC_CUDA(cudaIpcGetMemHandle(&mine.sig, e->sig));
  const size_t sz = sizeof(Handles);
  char* dbuf = nullptr;
  DLC_CUDA(cudaMalloc(&dbuf, K * sz));
  std::vector<Handles> all(K);
  try {
    DLC_CUDA(cudaMemcpyAsync(dbuf + r * sz, &mine, sz, cudaMemcpyHostToDevice, e->stream));
    DLC_NCCL(ncclAllGather(dbuf + r * sz, dbuf, sz, ncclUint8, c->comm, e->stream));
    DLC_CUDA(cudaMemcpyAsync(all.data(), dbuf, K * sz, cudaMemcpyDeviceToHost, e->stream));
    DLC_CUDA(cudaStreamSynchronize(e->stream));
  } catch (...) {
    cudaFree(dbuf);
    throw;
  }
  cudaFree(dbuf);
  for (int j = 0; j < K; ++j) {
    if (j == r) {
      e->peer_send[j] = e->send;
      e->peer_gather[j] = e->gather;
      e->peer_flags[j] = e->flags;
      e->peer_sig[j] = e->sig;
      e->peer_recv[j] = e->recv;
      continue;
    }
    void* precv = nullptr;
    check_cuda(cudaIpcOpenMemHandle(&precv, all[j].recv, cudaIpcMemLazyEnablePeerAccess),
               "cudaIpcOpenMemHandle (recv rows)");
    e->ipc_opened.push_back(precv);
    e->peer_recv[j] = precv;
    void* psig = nullptr;
    check_cuda(cudaIpcOpenMemHandle(&psig, all[j].sig, cudaIpcMemLazyEnablePeerAccess),
               "cudaIpcOpenMemHandle (signal slots)");
    e->ipc_opened.push_back(psig);
    e->peer_sig[j] = (uint64_t*)psig;
    void* ps = nullptr;
    void* pg = nullptr;
    void* pf = nullptr;
    const char* what = "cudaIpcOpenMemHandle (DLC_MODE_P2P needs one process per GPU with NVLink peer access)";
    check_cuda(cudaIpcOpenMemHandle(&ps, all[j].send, cudaIpcMemLazyEnablePeerAccess), what);
    e->ipc_opened.push_back(ps);
    check_cuda(cudaIpcOpenMemHandle(&pg, all[j].gather, cudaIpcMemLazyEnablePeerAccess), what);
    e->ipc_opened.push_back(pg);
    check_cuda(cudaIpcOpenMemHandle(&pf, all[j].flags, cudaIpcMemLazyEnablePeerAccess), what);
    e->ipc_opened.push_back(pf);
    e->peer_send[j] = ps;
    e->peer_gather[j] = pg;
    e->peer_flags[j] = (int*)pf;
  }
  e->p2p_bound = c;
}

// Stream-ordered fleet barrier: a 4-byte NCCL all-reduce.
void fleet_barrier(dlc_engine* e, dlc_collective* c) {
  DLC_NCCL(ncclAllReduce(e->barrier_buf, e->barrier_buf, 1, ncclInt32, ncclSum, c->comm, e->stream));
}

// Phase barrier of the P2P step on stream `s`: NVLink flags by default
// (one CTA, a few microseconds), DLC_P2P_BARRIER=nccl for the NCCL all-reduce.
void p2p_barrier(dlc_engine* e, dlc_collective* c, cudaStream_t s) {
  const char* b = std::getenv("DLC_P2P_BARRIER");
  if (b && std::string(b) == "nccl" && !c->in_world) {  // (one thread drives a world: flags only)
    DLC_NCCL(ncclAllReduce(e->barrier_buf, e->barrier_buf, 1, ncclInt32, ncclSum, c->comm, s));
    return;
  }
  PtrList remote{};
  for (size_t j = 0; j < e->k; ++j) remote.ptr[j] = e->peer_sig[j] + c->rank;
  e->sig_epoch += 1;
  launch_flag_barrier(remote, e->sig, (int)e->k, c->rank, e->sig_epoch, e->sig_err, s);
  launched("flag_barrier");
}

// C1 + K3 on the engine's send buffer, then K4.  Everything is enqueued on the
// engine stream; NCCL calls are stream-ordered with the kernels around them.
void outer_collective(dlc_engine* e, dlc_collective* c, dlc_reduce_report* rep) {
  const size_t K = e->k, S = e->S, w = elem_width(e->prec);
  char* send = static_cast<char*>(e->send);
  if (K == 1) {  // SoloCollective: the mean of one contribution is itself (reduce.cpp:113-126)
    nesterov(e, e->send, &e->st->delta_nonfinite, 1);
    return;
  }
  const int r = c->rank;
  if (rep) DLC_CUDA(cudaEventRecord(e->ev0, e->stream));
  phase_begin(e);
  if (c->mode == DLC_MODE_ORDERED) {
    char* recv = static_cast<char*>(e->recv);
    char* gather = static_cast<char*>(e->gather);
    // scatter: partition j of my delta goes to its owner j (collective.cpp:1400-1426)
    DLC_NCCL(ncclGroupStart());
    for (size_t j = 0; j < K; ++j) {
      if ((int)j == r) continue;
      DLC_NCCL(ncclSend(send + j * S * w, S, nccl_type(e->prec), (int)j, c->comm, e->stream));
      DLC_NCCL(ncclRecv(recv + j * S * w, S, nccl_type(e->prec), (int)j, c->comm, e->stream));
    }
    DLC_NCCL(ncclGroupEnd());
    // owner fold in rank order (collective.cpp:1444-1489)
    PtrList in{};
    for (size_t j = 0; j < K; ++j) in.ptr[j] = ((int)j == r) ? send + r * S * w : recv + j * S * w;
    launch_fold(in, (int)K, e->prec, gather + r * S * w, e->prec, e->flags + r, S, e->stream);
    launched("fold");
    // all-gather of the owner means and their non-finite flags (collective.cpp:1491-1531)
    DLC_NCCL(ncclGroupStart());
    DLC_NCCL(ncclAllGather(gather + r * S * w, gather, S, nccl_type(e->prec), c->comm, e->stream));
    DLC_NCCL(ncclAllGather(e->flags + r, e->flags, 1, ncclInt32, c->comm, e->stream));
    DLC_NCCL(ncclGroupEnd());
    phase_end(e, DLC_PHASE_COLLECTIVE);
    if (rep) DLC_CUDA(cudaEventRecord(e->ev1, e->stream));
    nesterov(e, e->gather, e->flags, (int)K);
  } else {
    DLC_NCCL(ncclAllReduce(send, send, K * S, nccl_type(e->prec), ncclAvg, c->comm, e->stream));
    if (e->prec == DLC_FP16)
      launch_nonfinite_codes(static_cast<const uint16_t*>(e->send), e->flags, e->n, e->stream);
    else
      launch_nonfinite(static_cast<const float*>(e->send), e->flags, e->n, e->stream);
    launched("nonfinite");
    phase_end(e, DLC_PHASE_COLLECTIVE);
    if (rep) DLC_CUDA(cudaEventRecord(e->ev1, e->stream));
    nesterov(e, e->send, e->flags, 1);
  }
}

// DLC_MODE_P2P: the rank-ordered owner fold fused with its own data movement
// over NVLink peer memory (CUDA IPC), pipelined over the pieces of piece_plan()
// (piece p = the same sub-range of every owner slot):
//   main     K2(p) into my send buffer                                 -> evK2[p]
//   cstream  wait evK2[p]; barrier A_p (every rank's K2(p) is done);
//            fold_push(p): the owner pulls piece p of slot r from every rank,
//            folds in rank order, pushes the mean + a non-finite mark into
//            slot r of every rank's gather buffer; barrier B_p          -> evB[p]
//   main     wait evB[p]; K4(p) speculative into the idle theta_t / momentum;
//            ...; finish (flip ocur when every owner flag is clean)
// The fold kernel keeps DLC_COMM_CTAS CTAs, so the NVLink time of piece p
// overlaps the HBM-bound K2 / K4 pieces on the other SMs.  Other movers
// (DLC_P2P_COPY): "ce" pulls / gathers with the copy engines around a local
// fold; "push" stores K2's rows straight into the owners' receive buffers;
// "push2" pushes them from a scatter kernel on the comm stream.  A_p orders
// every rank's K2(p) (and, for p = 0, every rank's previous finish) before
// anyone reads them; B_p orders every push of piece p before any K4(p).  With
// host buffers (`hsrc` / `hdst`) piece p is also copied in before K2(p) and its
// new theta_t copied out after K4(p).
void outer_p2p_pipelined(dlc_engine* e, dlc_collective* c, const float* src, dlc_reduce_report* rep,
                         const float* hsrc, float* hdst, int oc_host) {
  p2p_bind(e, c);
  const size_t K = e->k, S = e->S, w = elem_width(e->prec), n = e->n;
  const int r = c->rank;
  if (!e->cstream) {
    int lo = 0, hi = 0;
    DLC_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    DLC_CUDA(cudaStreamCreateWithPriority(&e->cstream, cudaStreamNonBlocking, hi));
    DLC_CUDA(cudaStreamCreateWithPriority(&e->sstream, cudaStreamNonBlocking, hi));
    for (size_t j = 0; j < K; ++j) {
      DLC_CUDA(cudaStreamCreateWithFlags(&e->pull[j], cudaStreamNonBlocking));
      DLC_CUDA(cudaStreamCreateWithFlags(&e->gath[j], cudaStreamNonBlocking));
    }
  }
  const std::vector<size_t> pb = piece_plan(S);  // piece boundaries inside a slot
  const size_t P = pb.size() - 1;
  auto po = [&](size_t p) { return pb[p]; };
  auto pl = [&](size_t p) { return pb[p + 1] - pb[p]; };
  const size_t nev = 5 * P + 2 * K * P + 1;
  while (e->piece_ev.size() < nev) {
    cudaEvent_t ev;
    DLC_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    e->piece_ev.push_back(ev);
  }
  cudaEvent_t* evK2 = e->piece_ev.data();
  cudaEvent_t* evA = evK2 + P;
  cudaEvent_t* evB = evA + P;
  cudaEvent_t* evH = evB + P;
  cudaEvent_t* evK4 = evH + P;
  cudaEvent_t* evPull = evK4 + P;       // [j * P + p]
  cudaEvent_t* evGath = evPull + K * P;  // [q * P + p]
  cudaEvent_t evStart = evGath[K * P];
  float* s = const_cast<float*>(src);
  const Pair tl = s ? Pair{{s, s}} : local_pair(e);
  const float lr = e->hyper.outer_lr, mu = e->hyper.outer_momentum;
  char* send = static_cast<char*>(e->send);
  char* recv = static_cast<char*>(e->recv);
  char* gather = static_cast<char*>(e->gather);
  const bool push_mover = p2p_mover_push();
  auto rows = [&](size_t p, auto&& fn) {  // piece p of every owner slot, clipped to n
    for (size_t q = 0; q < K; ++q) {
      const size_t lo = q * S + po(p);
      if (lo >= n) break;
      fn(lo, std::min(pl(p), n - lo));
    }
  };
  if (rep) DLC_CUDA(cudaEventRecord(e->ev0, e->stream));
  // SM mover: owners push non-finite marks into this array after A_0, which
  // every rank reaches only after this memset (it precedes our K2(0))
  if (p2p_mover_sm()) DLC_CUDA(cudaMemsetAsync(e->flags, 0, kMaxK * sizeof(int), e->stream));
  cudaEvent_t origin = trace_begin(e, e->stream);
  DLC_CUDA(cudaEventRecord(evStart, e->stream));
  if (hsrc) {
    ensure_copy_streams(e);
    DLC_CUDA(cudaStreamWaitEvent(e->h2d, evStart, 0));  // staging buffer free
  }
  phase_begin(e);
  for (size_t p = 0; p < P; ++p) {
    if (hsrc) {
      rows(p, [&](size_t lo, size_t len) {
        DLC_CUDA(cudaMemcpyAsync(s + lo, hsrc + lo, len * sizeof(float), cudaMemcpyHostToDevice, e->h2d));
      });
      DLC_CUDA(cudaEventRecord(evH[p], e->h2d));
      DLC_CUDA(cudaStreamWaitEvent(e->stream, evH[p], 0));
    }
    cudaEvent_t t0 = trace_begin(e, e->stream);
    if (push_mover) {
      PtrList rows{};  // my row in every owner's recv buffer
      for (size_t q = 0; q < K; ++q) rows.ptr[q] = static_cast<char*>(e->peer_recv[q]) + r * S * w;
      launch_pseudo_grad_push_piece(tt_pair(e), tl, e->st, rows, e->prec, (int)K, S, po(p), pl(p), n, e->stream);
    } else {
      launch_pseudo_grad_piece(tt_pair(e), tl, e->st, e->send, e->prec, (int)K, S, po(p), pl(p), n, piece_ctas(),
                               e->stream);
    }
    trace_end(e, e->stream, "K2", (int)p, t0);
    DLC_CUDA(cudaEventRecord(evK2[p], e->stream));
  }
  launched("pseudo_grad_piece");
  phase_end(e, DLC_PHASE_PSEUDO);
  DLC_CUDA(cudaStreamWaitEvent(e->cstream, evStart, 0));
  cudaEvent_t c0 = pooled_event(e), c1 = pooled_event(e);
  DLC_CUDA(cudaEventRecord(c0, e->cstream));
  const bool sm_mover = p2p_mover_sm();
  const bool push2 = p2p_mover_push2();
  cudaEvent_t* evS = evA;  // (evA is only used by the copy-engine mover)
  for (size_t p = 0; p < P && push2; ++p) {
    // push/push: our piece of every foreign slot into its owner's recv row r, on
    // its own stream so that scatter(p + 1) overlaps fold(p): every NVLink byte
    // is a remote store and both link directions stay busy
    DLC_CUDA(cudaStreamWaitEvent(e->sstream, evK2[p], 0));
    PtrList src{}, dst{};
    int nrow = 0;
    for (size_t q = 0; q < K; ++q) {
      if ((int)q == r) continue;
      src.ptr[nrow] = send + (q * S + po(p)) * w;
      dst.ptr[nrow] = static_cast<char*>(e->peer_recv[q]) + (r * S + po(p)) * w;
      ++nrow;
    }
    cudaEvent_t ts = trace_begin(e, e->sstream);
    launch_scatter_push(src, dst, nrow, pl(p) * w, comm_ctas(), e->sstream);
    trace_end(e, e->sstream, "scatter", (int)p, ts);
    DLC_CUDA(cudaEventRecord(evS[p], e->sstream));
  }
  for (size_t p = 0; p < P && sm_mover; ++p) {
    // SM mover: a persistent fold kernel on a few CTAs pulls slot r / piece p of
    // every rank's delta and pushes the mean (and a non-finite mark) into slot r
    // of every rank's gather buffer (flags reset by each rank before its K2(0)).
    DLC_CUDA(cudaStreamWaitEvent(e->cstream, push2 ? evS[p] : evK2[p], 0));
    cudaEvent_t ta = trace_begin(e, e->cstream);
    p2p_barrier(e, c, e->cstream);  // A_p
    trace_end(e, e->cstream, "barrierA", (int)p, ta);
    PtrList in{}, outs{}, pfl{};
    for (size_t j = 0; j < K; ++j) {
      in.ptr[j] = (int)j == r && push2 ? send + (r * S + po(p)) * w  // own row stays local
                  : (push_mover || push2) ? recv + (j * S + po(p)) * w   // rows already pushed here
                                          : static_cast<char*>(e->peer_send[j]) + (r * S + po(p)) * w;
      outs.ptr[j] = static_cast<char*>(e->peer_gather[j]) + (r * S + po(p)) * w;
      pfl.ptr[j] = e->peer_flags[j] + r;
    }
    cudaEvent_t tf = trace_begin(e, e->cstream);
    if (!(fold_tma() && launch_fold_push_tma(in, (int)K, e->prec, outs, (int)K, pfl, pl(p), tma_ctas(K), e->cstream)))
      launch_fold_push(in, (int)K, e->prec, outs, (int)K, pfl, pl(p), comm_ctas(), e->cstream);
    trace_end(e, e->cstream, "fold_push", (int)p, tf);
    cudaEvent_t tb = trace_begin(e, e->cstream);
    p2p_barrier(e, c, e->cstream);  // B_p
    trace_end(e, e->cstream, "barrierB", (int)p, tb);
    DLC_CUDA(cudaEventRecord(evB[p], e->cstream));
  }
  for (size_t p = 0; p < P && !sm_mover; ++p) {
    DLC_CUDA(cudaStreamWaitEvent(e->cstream, evK2[p], 0));
    p2p_barrier(e, c, e->cstream);  // A_p
    if (p == 0) DLC_CUDA(cudaMemsetAsync(e->flags + r, 0, sizeof(int), e->cstream));
    DLC_CUDA(cudaEventRecord(evA[p], e->cstream));
    for (size_t j = 0; j < K; ++j) {  // scatter: pull slot r, piece p of every peer's delta
      if ((int)j == r) continue;
      DLC_CUDA(cudaStreamWaitEvent(e->pull[j], evA[p], 0));
      DLC_CUDA(cudaMemcpyAsync(recv + (j * S + po(p)) * w, static_cast<char*>(e->peer_send[j]) + (r * S + po(p)) * w,
                               pl(p) * w, cudaMemcpyDefault, e->pull[j]));
      DLC_CUDA(cudaEventRecord(evPull[j * P + p], e->pull[j]));
      DLC_CUDA(cudaStreamWaitEvent(e->cstream, evPull[j * P + p], 0));
    }
    PtrList in{};  // owner fold in rank order (collective.cpp:1444-1489)
    for (size_t j = 0; j < K; ++j)  // my own contribution straight from my send buffer
      in.ptr[j] = ((int)j == r ? send + (r * S + po(p)) * w : recv + (j * S + po(p)) * w);
    launch_fold(in, (int)K, e->prec, gather + (r * S + po(p)) * w, e->prec, e->flags + r, pl(p), e->cstream);
    p2p_barrier(e, c, e->cstream);  // B_p
    DLC_CUDA(cudaEventRecord(evB[p], e->cstream));
    for (size_t q = 0; q < K; ++q) {  // all-gather: pull piece p of every owner's mean slot
      if ((int)q == r) continue;
      DLC_CUDA(cudaStreamWaitEvent(e->gath[q], evB[p], 0));
      DLC_CUDA(cudaMemcpyAsync(gather + (q * S + po(p)) * w,
                               static_cast<char*>(e->peer_gather[q]) + (q * S + po(p)) * w, pl(p) * w,
                               cudaMemcpyDefault, e->gath[q]));
      DLC_CUDA(cudaEventRecord(evGath[q * P + p], e->gath[q]));
    }
  }
  launched("fold_p2p");
  DLC_CUDA(cudaEventRecord(c1, e->cstream));
  if (e->timing) {
    e->pending.push_back({DLC_PHASE_COLLECTIVE, c0, c1});
  } else {
    e->pool.push_back(c0);
    e->pool.push_back(c1);
  }
  if (rep) DLC_CUDA(cudaEventRecord(e->ev1, e->cstream));
  // K4 pieces on the local gather buffer, speculative into the idle theta_t / momentum
  PtrList slots{}, fl{};
  for (size_t q = 0; q < K; ++q) {
    slots.ptr[q] = gather + q * S * w;
    // SM mover: owners pushed their marks into my flag array; CE mover: owner
    // q's flag lives in owner q's memory
    fl.ptr[q] = sm_mover ? e->flags + q : e->peer_flags[q] + q;
  }
  phase_begin(e);
  for (size_t p = 0; p < P; ++p) {
    DLC_CUDA(cudaStreamWaitEvent(e->stream, evB[p], 0));
    for (size_t q = 0; q < K && !sm_mover; ++q)
      if ((int)q != r) DLC_CUDA(cudaStreamWaitEvent(e->stream, evGath[q * P + p], 0));
    cudaEvent_t t4 = trace_begin(e, e->stream);
    launch_nesterov_p2p_piece(tt_pair(e), buf_pair(e), local_pair(e), slots, (int)K, S, po(p), pl(p), e->prec, e->st,
                              lr, mu, n, piece_ctas(), e->stream);
    trace_end(e, e->stream, "K4", (int)p, t4);
    if (hdst) {
      DLC_CUDA(cudaEventRecord(evK4[p], e->stream));
      DLC_CUDA(cudaStreamWaitEvent(e->d2h, evK4[p], 0));
      rows(p, [&](size_t lo, size_t len) {
        DLC_CUDA(cudaMemcpyAsync(hdst + lo, e->theta_t[oc_host ^ 1] + lo, len * sizeof(float),
                                 cudaMemcpyDeviceToHost, e->d2h));
      });
    }
  }
  launch_p2p_finish(tt_pair(e), local_pair(e), fl, (int)K, e->st, n, e->stream);
  phase_end(e, DLC_PHASE_OUTER);
  launched("nesterov_p2p_piece");
  trace_dump(e, origin);
}

// DLC_MODE_ALLREDUCE, pipelined: ncclAllReduce(ncclAvg) of contiguous pieces of
// the flat pseudo-gradient on the high-priority comm stream, overlapped with
// K2 of the next piece and the speculative K4 of the previous one:
//   main     K2(p) -> evK2[p]
//   cstream  wait evK2[p]; ncclAllReduce(piece p, in place); non-finite(p) -> evB[p]
//   main     wait evB[p]; K4(p) into the idle theta_t / momentum; ...; finish
// (DLC_AR_SERIAL=1: the unpipelined K2 -> all-reduce -> K4 of outer_collective.)
bool allreduce_pipelined() {
  const char* s = std::getenv("DLC_AR_SERIAL");
  return !(s && std::string(s) == "1");
}

void outer_allreduce_pipelined(dlc_engine* e, dlc_collective* c, const float* src, dlc_reduce_report* rep) {
  const size_t n = e->n, w = elem_width(e->prec);
  if (!e->cstream) {
    int lo = 0, hi = 0;
    DLC_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    DLC_CUDA(cudaStreamCreateWithPriority(&e->cstream, cudaStreamNonBlocking, hi));
  }
  std::vector<size_t> pb = piece_plan((n + 511) / 512 * 512);  // contiguous pieces of [0, n)
  for (size_t& b : pb) b = std::min(b, n);
  const size_t P = pb.size() - 1;
  while (e->piece_ev.size() < 2 * P + 1) {
    cudaEvent_t ev;
    DLC_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    e->piece_ev.push_back(ev);
  }
  cudaEvent_t* evK2 = e->piece_ev.data();
  cudaEvent_t* evB = evK2 + P;
  cudaEvent_t evStart = evB[P];
  float* s = const_cast<float*>(src);
  const Pair tl = s ? Pair{{s, s}} : local_pair(e);
  char* send = static_cast<char*>(e->send);
  if (rep) DLC_CUDA(cudaEventRecord(e->ev0, e->stream));
  DLC_CUDA(cudaMemsetAsync(e->flags, 0, sizeof(int), e->stream));
  DLC_CUDA(cudaEventRecord(evStart, e->stream));
  phase_begin(e);
  for (size_t p = 0; p < P; ++p) {  // k = 1: piece p is the contiguous range [pb[p], pb[p+1])
    launch_pseudo_grad_piece(tt_pair(e), tl, e->st, e->send, e->prec, 1, 0, pb[p], pb[p + 1] - pb[p], n, 0,
                             e->stream);
    DLC_CUDA(cudaEventRecord(evK2[p], e->stream));
  }
  launched("pseudo_grad_piece");
  phase_end(e, DLC_PHASE_PSEUDO);
  DLC_CUDA(cudaStreamWaitEvent(e->cstream, evStart, 0));
  cudaEvent_t c0 = pooled_event(e), c1 = pooled_event(e);
  DLC_CUDA(cudaEventRecord(c0, e->cstream));
  for (size_t p = 0; p < P; ++p) {
    const size_t len = pb[p + 1] - pb[p];
    DLC_CUDA(cudaStreamWaitEvent(e->cstream, evK2[p], 0));
    if (len) {
      char* x = send + pb[p] * w;
      DLC_NCCL(ncclAllReduce(x, x, len, nccl_type(e->prec), ncclAvg, c->comm, e->cstream));
      if (e->prec == DLC_FP16)  // engine.cpp:136 on the piece
        launch_nonfinite_codes(reinterpret_cast<const uint16_t*>(x), e->flags, len, e->cstream);
      else
        launch_nonfinite(reinterpret_cast<const float*>(x), e->flags, len, e->cstream);
    }
    DLC_CUDA(cudaEventRecord(evB[p], e->cstream));
  }
  launched("nonfinite");
  DLC_CUDA(cudaEventRecord(c1, e->cstream));
  if (e->timing) {
    e->pending.push_back({DLC_PHASE_COLLECTIVE, c0, c1});
  } else {
    e->pool.push_back(c0);
    e->pool.push_back(c1);
  }
  if (rep) DLC_CUDA(cudaEventRecord(e->ev1, e->cstream));
  PtrList slots{}, fl{};
  slots.ptr[0] = send;
  fl.ptr[0] = e->flags;
  phase_begin(e);
  for (size_t p = 0; p < P; ++p) {
    DLC_CUDA(cudaStreamWaitEvent(e->stream, evB[p], 0));
    launch_nesterov_p2p_piece(tt_pair(e), buf_pair(e), local_pair(e), slots, 1, 0, pb[p], pb[p + 1] - pb[p],
                              e->prec, e->st, e->hyper.outer_lr, e->hyper.outer_momentum, n, 0, e->stream);
  }
  launch_p2p_finish(tt_pair(e), local_pair(e), fl, 1, e->st, n, e->stream);
  phase_end(e, DLC_PHASE_OUTER);
  launched("nesterov_p2p_piece");
}

void outer_round(dlc_engine* e, dlc_collective* c, const float* src, dlc_reduce_report* rep) {
  if (e->k > 1 && c->mode == DLC_MODE_P2P) {  // manages its own flag (read remotely by peers)
    outer_p2p_pipelined(e, c, src, rep, nullptr, nullptr, 0);
    return;
  }
  if (e->k > 1 && c->mode == DLC_MODE_ALLREDUCE && allreduce_pipelined()) {
    outer_allreduce_pipelined(e, c, src, rep);
    return;
  }
  reset_flags(e);
  if (e->k == 1) {
    phase_begin(e);
    launch_outer_solo_fused(tt_pair(e), buf_pair(e), local_pair(e), src, e->prec, e->st, e->hyper.outer_lr,
                            e->hyper.outer_momentum, e->n, e->stream);
    phase_end(e, DLC_PHASE_OUTER);
    launched("outer_solo");
    return;
  }
  float* s = const_cast<float*>(src);
  pseudo_grad(e, s ? Pair{{s, s}} : local_pair(e));
  outer_collective(e, c, rep);
}

void fill_report(dlc_engine* e, dlc_collective* c, dlc_reduce_report* rep, uint64_t epoch) {
  if (!rep) return;
  *rep = dlc_reduce_report{};
  rep->outer_epoch = epoch;
  rep->contributors = e->k;
  rep->attempts = 1;
  if (e->k > 1) {
    const uint64_t bytes = 2ull * (e->k - 1) * e->S * elem_width(e->prec);
    rep->data_bytes_sent = rep->data_bytes_received = bytes;
    rep->wire_bytes_sent = rep->wire_bytes_received = bytes;
    DLC_CUDA(cudaEventSynchronize(e->ev1));
    float ms = 0;
    DLC_CUDA(cudaEventElapsedTime(&ms, e->ev0, e->ev1));
    rep->wall_ms = ms;
  }
  (void)c;
}

void check_collective(dlc_engine* e, dlc_collective* c) {
  const size_t world = c ? (size_t)c->world : 1;
  if (world != e->k)
    fail(DLC_ECOLLECTIVE, "collective world size " + std::to_string(world) + " != num_workers_k " +
                              std::to_string(e->k));
  if (c && c->kind == 1 && c->device != e->device) fail(DLC_ECOLLECTIVE, "collective and engine devices differ");
  if (e->issued_inner % e->cfg.local_steps_h != 0)  // engine.cpp:116-120
    fail(DLC_EINVAL, "pseudo-gradient requested mid-window (inner_step " + std::to_string(e->issued_inner) +
                         ", H " + std::to_string(e->cfg.local_steps_h) + ")");
}

// A flag barrier that timed out (a peer never arrived) surfaces as CollectiveError.
void check_barrier(dlc_engine* e) {
  if (!e->sig_err) return;
  int err = 0;
  DLC_CUDA(cudaStreamSynchronize(e->stream));
  if (e->cstream) DLC_CUDA(cudaStreamSynchronize(e->cstream));
  DLC_CUDA(cudaMemcpy(&err, e->sig_err, sizeof(int), cudaMemcpyDeviceToHost));
  if (err) fail(DLC_ECOLLECTIVE, "P2P barrier timed out: a peer rank stopped participating");
}

void outer_result(dlc_engine* e, dlc_outer_result* res) {
  if (!res) return;  // asynchronous call: nothing is synchronised here
  check_barrier(e);
  const DevState s = read_state(e);
  res->applied = s.last_applied;
  res->outer_epoch = s.outer_epoch;
}

}  // namespace

extern "C" {

void dlc_hyperparams_default(dlc_hyperparams* h) {
  // OptimHyperparams defaults, engine.hpp:34-46
  h->inner_lr = 4e-4f;
  h->warmup_steps = 1000;
  h->lr_decay = DLC_LR_NONE;
  h->weight_decay = 0.1f;
  h->beta1 = 0.9f;
  h->beta2 = 0.95f;
  h->adam_eps = 1e-8f;
  h->outer_lr = 0.7f;
  h->outer_momentum = 0.9f;
  h->scaler_init_scale = 65536.0f;
  h->scaler_growth_interval = 2000;
}

int dlc_engine_create(const dlc_config* cfg, const dlc_hyperparams* hyper, size_t n, int device, int inner_mode,
                      dlc_engine** out) {
  dlc_engine* e = nullptr;
  const int st = guard([&] {
    if (!cfg || !hyper || !out) fail(DLC_EINVAL, "dlc_engine_create: null argument");
    *out = nullptr;
    // DilocoConfig::validate, engine.cpp:31-48
    if (cfg->local_steps_h < 1) fail(DLC_ECONFIG, "local_steps must be >= 1");
    if (cfg->num_workers_k < 1) fail(DLC_ECONFIG, "num_workers must be >= 1");
    if (cfg->total_inner_steps == 0 || cfg->total_inner_steps % cfg->local_steps_h != 0)
      fail(DLC_ECONFIG, "total_inner_steps (" + std::to_string(cfg->total_inner_steps) +
                            ") must be a positive multiple of local_steps (" + std::to_string(cfg->local_steps_h) +
                            ")");
    if (cfg->num_workers_k > (size_t)kMaxK) fail(DLC_ECONFIG, "num_workers_k exceeds 32");
    if (cfg->reduce_precision != DLC_FP32 && cfg->reduce_precision != DLC_FP16)
      fail(DLC_ECONFIG, "unknown reduce precision");
    if (inner_mode != DLC_INNER_PINGPONG && inner_mode != DLC_INNER_INPLACE) fail(DLC_ECONFIG, "unknown inner mode");
    DeviceGuard dg(device);
    e = new dlc_engine();
    e->device = device;
    e->cfg = *cfg;
    e->hyper = *hyper;
    e->inner_mode = inner_mode;
    e->n = n;
    e->k = cfg->num_workers_k;
    e->prec = cfg->reduce_precision;
    // owner slot: a multiple of 64 elements per P2P piece
    const size_t quantum = 64 * kMaxPieces;
    e->S = (((n + e->k - 1) / e->k) + quantum - 1) / quantum * quantum;
    DLC_CUDA(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
    DLC_CUDA(cudaEventCreate(&e->ev0));
    DLC_CUDA(cudaEventCreate(&e->ev1));
    const size_t vb = n * sizeof(float);
    // theta_t / momentum ping-pong: the fused solo step (K = 1) and the pipelined
    // P2P step (K > 1) write the new values speculatively into the idle buffer
    for (int i = 0; i < 2; ++i) {
      e->theta_t[i] = (float*)dalloc(e, vb);
      e->buf[i] = (float*)dalloc(e, vb);
    }
    const int pairs = inner_mode == DLC_INNER_PINGPONG ? 2 : 1;
    for (int i = 0; i < pairs; ++i) {
      e->p[i] = (float*)dalloc(e, vb);
      e->m[i] = (float*)dalloc(e, vb);
      e->v[i] = (float*)dalloc(e, vb);
    }
    if (pairs == 1) {
      e->p[1] = e->p[0];
      e->m[1] = e->m[0];
      e->v[1] = e->v[0];
    }
    e->grad = (float*)dalloc(e, vb);
    const size_t pb = e->k * e->S * elem_width(e->prec);
    e->send = dalloc(e, pb);
    DLC_CUDA(cudaMemsetAsync(e->send, 0, pb, e->stream));  // padding stays zero
    if (e->k > 1) {
      e->recv = dalloc(e, pb);
      e->gather = dalloc(e, pb);
      DLC_CUDA(cudaMemsetAsync(e->gather, 0, pb, e->stream));
      e->barrier_buf = (int*)dalloc(e, 256);
      e->sig = (uint64_t*)dalloc(e, kMaxK * sizeof(uint64_t));
      e->sig_err = (int*)dalloc(e, 256);
      DLC_CUDA(cudaMemsetAsync(e->sig, 0, kMaxK * sizeof(uint64_t), e->stream));
      DLC_CUDA(cudaMemsetAsync(e->sig_err, 0, 256, e->stream));
    }
    e->flags = (int*)dalloc(e, kMaxK * sizeof(int));
    e->st = (DevState*)dalloc(e, sizeof(DevState));
    for (int i = 0; i < pairs; ++i) {
      DLC_CUDA(cudaMemsetAsync(e->p[i], 0, vb, e->stream));
      DLC_CUDA(cudaMemsetAsync(e->m[i], 0, vb, e->stream));  // AdamWState::init zeros, optim.cpp:17-27
      DLC_CUDA(cudaMemsetAsync(e->v[i], 0, vb, e->stream));
    }
    for (int i = 0; i < 2; ++i) {
      DLC_CUDA(cudaMemsetAsync(e->theta_t[i], 0, vb, e->stream));
      DLC_CUDA(cudaMemsetAsync(e->buf[i], 0, vb, e->stream));  // NesterovState::init, optim.cpp:29-35
    }
    DLC_CUDA(cudaMemsetAsync(e->flags, 0, kMaxK * sizeof(int), e->stream));
    DevState s{};
    s.scale = hyper->scaler_init_scale;
    s.growth = hyper->scaler_growth_interval;
    DLC_CUDA(cudaMemcpyAsync(e->st, &s, sizeof(s), cudaMemcpyHostToDevice, e->stream));
    ensure_tables(e, std::min<uint64_t>(cfg->total_inner_steps + 2, 1u << 16));
    DLC_CUDA(cudaStreamSynchronize(e->stream));
    *out = e;
  });
  if (st != DLC_OK && e) dlc_engine_destroy(e);
  return st;
}

int dlc_engine_destroy(dlc_engine* e) {
  if (!e) return DLC_OK;
  return guard([&] {
    DeviceGuard dg(e->device);
    if (e->stream) cudaStreamSynchronize(e->stream);
    if (e->p2p_bound) {
      // peers may still be reading this engine's slot / send buffer: wait for
      // the whole fleet (engines are destroyed collectively, before their collective)
      fleet_barrier(e, const_cast<dlc_collective*>(e->p2p_bound));
      cudaStreamSynchronize(e->stream);
    }
    p2p_unbind(e);
    for (void* p : e->allocs) cudaFree(p);
    if (e->wire_rows) cudaFree(e->wire_rows);
    for (const auto& mk : e->pending) {
      cudaEventDestroy(mk.a);
      cudaEventDestroy(mk.b);
    }
    for (cudaEvent_t ev : e->pool) cudaEventDestroy(ev);
    if (e->tab) cudaFree(e->tab);
    if (e->ev0) cudaEventDestroy(e->ev0);
    if (e->ev1) cudaEventDestroy(e->ev1);
    for (cudaEvent_t ev : e->chunk_ev) cudaEventDestroy(ev);
    for (cudaEvent_t ev : e->piece_ev) cudaEventDestroy(ev);
    for (size_t j = 0; j < (size_t)kMaxK; ++j) {
      if (e->pull[j]) cudaStreamDestroy(e->pull[j]);
      if (e->gath[j]) cudaStreamDestroy(e->gath[j]);
    }
    if (e->cstream) cudaStreamDestroy(e->cstream);
    if (e->sstream) cudaStreamDestroy(e->sstream);
    if (e->h2d) cudaStreamDestroy(e->h2d);
    if (e->d2h) cudaStreamDestroy(e->d2h);
    if (e->stream) cudaStreamDestroy(e->stream);
    delete e;
  });
}

size_t dlc_engine_size(const dlc_engine* e) { return e ? e->n : 0; }

int dlc_engine_stream(dlc_engine* e, void** stream) {
  return guard([&] {
    if (!e || !stream) fail(DLC_EINVAL, "dlc_engine_stream: null argument");
    *stream = (void*)e->stream;
  });
}

int dlc_engine_upload(dlc_engine* e, int which, const float* host, size_t n) {
  return guard([&] {
    if (!e || (n && !host)) fail(DLC_EINVAL, "dlc_engine_upload: null argument");
    if (n != e->n) fail(DLC_ESHAPE, "upload length " + std::to_string(n) + " != engine size " + std::to_string(e->n));
    DeviceGuard dg(e->device);
    float* d = writable(e, which);
    DLC_CUDA(cudaMemcpyAsync(d, host, n * sizeof(float), cudaMemcpyHostToDevice, e->stream));
    DLC_CUDA(cudaStreamSynchronize(e->stream));
  });
}

int dlc_engine_download(dlc_engine* e, int which, float* host, size_t n) {
  return guard([&] {
    if (!e || (n && !host)) fail(DLC_EINVAL, "dlc_engine_download: null argument");
    if (n != e->n) fail(DLC_ESHAPE, "download length " + std::to_string(n) + " != engine size " + std::to_string(e->n));
    DeviceGuard dg(e->device);
    float* d = live(e, which);
    DLC_CUDA(cudaMemcpyAsync(host, d, n * sizeof(float), cudaMemcpyDeviceToHost, e->stream));
    DLC_CUDA(cudaStreamSynchronize(e->stream));
  });
}

int dlc_engine_download_range(dlc_engine* e, int which, size_t offset, float* host, size_t count) {
  return guard([&] {
    if (!e || (count && !host)) fail(DLC_EINVAL, "dlc_engine_download_range: null argument");
    if (offset > e->n || count > e->n - offset)
      fail(DLC_ESHAPE, "download range [" + std::to_string(offset) + ", +" + std::to_string(count) + ") outside " +
                           std::to_string(e->n) + " elements");
    DeviceGuard dg(e->device);
    const float* d = live(e, which);
    DLC_CUDA(cudaMemcpyAsync(host, d + offset, count * sizeof(float), cudaMemcpyDeviceToHost, e->stream));
    DLC_CUDA(cudaStreamSynchronize(e->stream));
  });
}

int dlc_engine_upload_range(dlc_engine* e, int which, size_t offset, const float* host, size_t count) {
  return guard([&] {
    if (!e || (count && !host)) fail(DLC_EINVAL, "dlc_engine_upload_range: null argument");
    if (offset > e->n || count > e->n - offset)
      fail(DLC_ESHAPE, "upload range [" + std::to_string(offset) + ", +" + std::to_string(count) + ") outside " +
                           std::to_string(e->n) + " elements");
    DeviceGuard dg(e->device);
    float* d = writable(e, which);
    DLC_CUDA(cudaMemcpyAsync(d + offset, host, count * sizeof(float), cudaMemcpyHostToDevice, e->stream));
    DLC_CUDA(cudaStreamSynchronize(e->stream));
  });
}

int dlc_engine_device_ptr(dlc_engine* e, int which, float** dev) {
  return guard([&] {
    if (!e || !dev) fail(DLC_EINVAL, "dlc_engine_device_ptr: null argument");
    DeviceGuard dg(e->device);
    *dev = writable(e, which);  // the caller may write through it
  });
}

int dlc_engine_get_scalars(dlc_engine* e, dlc_engine_scalars* out) {
  return guard([&] {
    if (!e || !out) fail(DLC_EINVAL, "dlc_engine_get_scalars: null argument");
    DeviceGuard dg(e->device);
    const DevState s = read_state(e);
    out->step_count = s.step_count;
    out->inner_step = s.inner_step;
    out->outer_epoch = s.outer_epoch;
    out->scale = s.scale;
    out->consecutive_good = s.good;
    out->overflow_skips = s.overflow_skips;
    out->outer_skips = s.outer_skips;
    out->last_lr = s.last_lr;
    out->last_overflow = s.last_overflow;
    out->last_applied = s.last_applied;
  });
}

int dlc_engine_set_scalars(dlc_engine* e, const dlc_engine_scalars* in) {
  return guard([&] {
    if (!e || !in) fail(DLC_EINVAL, "dlc_engine_set_scalars: null argument");
    if (in->inner_step > e->cfg.total_inner_steps) fail(DLC_ECONFIG, "inner_step beyond total_inner_steps");
    DeviceGuard dg(e->device);
    DevState s = read_state(e);
    s.step_count = in->step_count;
    s.inner_step = in->inner_step;
    s.outer_epoch = in->outer_epoch;
    s.scale = in->scale;
    s.good = in->consecutive_good;
    s.overflow_skips = in->overflow_skips;
    s.outer_skips = in->outer_skips;
    s.last_lr = in->last_lr;
    s.last_overflow = in->last_overflow;
    s.last_applied = in->last_applied;
    ensure_tables(e, in->step_count + 2);
    DLC_CUDA(cudaMemcpy(e->st, &s, sizeof(s), cudaMemcpyHostToDevice));
    e->issued_inner = in->inner_step;
  });
}

int dlc_engine_synchronize(dlc_engine* e) {
  return guard([&] {
    if (!e) fail(DLC_EINVAL, "dlc_engine_synchronize: null engine");
    DeviceGuard dg(e->device);
    DLC_CUDA(cudaStreamSynchronize(e->stream));
    check_barrier(e);
  });
}

int dlc_engine_inner_step(dlc_engine* e, const float* grad, int grad_is_scaled, dlc_inner_result* result) {
  return guard([&] {
    if (!e || (e->n && !grad)) fail(DLC_EINVAL, "dlc_engine_inner_step: null argument");
    DeviceGuard dg(e->device);
    engine_inner(e, grad, grad_is_scaled);
    if (result) {
      const DevState s = read_state(e);
      result->lr = s.last_lr;
      result->overflow_skipped = s.last_overflow;
    }
  });
}

int dlc_engine_inner_step_host(dlc_engine* e, const float* host_grad, int grad_is_scaled,
                               dlc_inner_result* result) {
  return guard([&] {
    if (!e || (e->n && !host_grad)) fail(DLC_EINVAL, "dlc_engine_inner_step_host: null argument");
    DeviceGuard dg(e->device);
    DLC_CUDA(cudaMemcpyAsync(e->grad, host_grad, e->n * sizeof(float), cudaMemcpyHostToDevice, e->stream));
    engine_inner(e, e->grad, grad_is_scaled);
    if (result) {
      const DevState s = read_state(e);
      result->lr = s.last_lr;
      result->overflow_skipped = s.last_overflow;
    }
  });
}

int dlc_engine_outer_step(dlc_engine* e, dlc_collective* c, dlc_outer_result* result, dlc_reduce_report* report) {
  return guard([&] {
    if (!e) fail(DLC_EINVAL, "dlc_engine_outer_step: null engine");
    if (c && c->kind == 0) c = nullptr;
    check_collective(e, c);
    DeviceGuard dg(e->device);
    const uint64_t epoch = report ? read_state(e).outer_epoch : 0;
    outer_round(e, c, nullptr, report);
    fill_report(e, c, report, epoch);
    outer_result(e, result);
  });
}

int dlc_engine_outer_step_from(dlc_engine* e, dlc_collective* c, const float* theta_local_dev,
                               dlc_outer_result* result, dlc_reduce_report* report) {
  return guard([&] {
    if (!e || (e->n && !theta_local_dev)) fail(DLC_EINVAL, "dlc_engine_outer_step_from: null argument");
    if (c && c->kind == 0) c = nullptr;
    check_collective(e, c);
    DeviceGuard dg(e->device);
    const uint64_t epoch = report ? read_state(e).outer_epoch : 0;
    float* src = const_cast<float*>(theta_local_dev);
    outer_round(e, c, src, report);
    fill_report(e, c, report, epoch);
    outer_result(e, result);
  });
}

int dlc_engine_set_timing(dlc_engine* e, int on) {
  return guard([&] {
    if (!e) fail(DLC_EINVAL, "dlc_engine_set_timing: null engine");
    DeviceGuard dg(e->device);
    harvest(e);
    e->timing = on != 0;
  });
}

int dlc_engine_phase_times(dlc_engine* e, double total_ms[4], uint64_t count[4]) {
  return guard([&] {
    if (!e || !total_ms || !count) fail(DLC_EINVAL, "dlc_engine_phase_times: null argument");
    DeviceGuard dg(e->device);
    harvest(e);
    for (int i = 0; i < 4; ++i) {
      total_ms[i] = e->phase_ms[i];
      count[i] = e->phase_n[i];
      e->phase_ms[i] = 0.0;
      e->phase_n[i] = 0;
    }
  });
}

int dlc_engine_outer_step_host(dlc_engine* e, dlc_collective* c, const float* host_theta_local, float* host_theta_t,
                               dlc_outer_result* result) {
  return guard([&] {
    if (!e || (e->n && (!host_theta_local || !host_theta_t))) fail(DLC_EINVAL, "dlc_engine_outer_step_host: null argument");
    if (c && c->kind == 0) c = nullptr;
    check_collective(e, c);
    DeviceGuard dg(e->device);
    // theta_local arrives chunk by chunk in the staging buffer (copy stream);
    // each chunk's kernel starts as soon as its bytes land, and for a single
    // worker each finished chunk of the new theta_t streams back on a second
    // copy stream, so H2D, compute and D2H overlap.  K4 refreshes the engine's
    // own theta_local from the new theta_t.
    ensure_copy_streams(e);
    const DevState s0 = read_state(e);
    if (e->k > 1 && c->mode == DLC_MODE_P2P) {  // piece-pipelined H2D / step / D2H
      outer_p2p_pipelined(e, c, e->grad, nullptr, host_theta_local, host_theta_t, s0.ocur);
      DLC_CUDA(cudaStreamSynchronize(e->h2d));
      DLC_CUDA(cudaStreamSynchronize(e->d2h));
      const DevState s1 = read_state(e);
      if (!s1.last_applied)  // skipped: theta_t did not move
        DLC_CUDA(cudaMemcpy(host_theta_t, e->theta_t[s1.ocur], e->n * sizeof(float), cudaMemcpyDeviceToHost));
      outer_result(e, result);
      return;
    }
    const size_t n = e->n, C = kHostChunk, nch = (n + C - 1) / C;
    ensure_chunk_events(e, 2 * nch + 1);
    reset_flags(e);
    DLC_CUDA(cudaEventRecord(e->chunk_ev[2 * nch], e->stream));  // staging buffer free to overwrite
    DLC_CUDA(cudaStreamWaitEvent(e->h2d, e->chunk_ev[2 * nch], 0));
    float* staged = e->grad;
    for (size_t ci = 0; ci < nch; ++ci) {
      const size_t off = ci * C, len = std::min(C, n - off);
      DLC_CUDA(cudaMemcpyAsync(staged + off, host_theta_local + off, len * sizeof(float), cudaMemcpyHostToDevice,
                               e->h2d));
      DLC_CUDA(cudaEventRecord(e->chunk_ev[2 * ci], e->h2d));
      DLC_CUDA(cudaStreamWaitEvent(e->stream, e->chunk_ev[2 * ci], 0));
      if (e->k == 1) {
        launch_outer_solo_chunk(tt_pair(e), buf_pair(e), local_pair(e), staged, e->prec, e->st, e->hyper.outer_lr,
                                e->hyper.outer_momentum, off, len, e->stream);
        launched("outer_solo_chunk");
        DLC_CUDA(cudaEventRecord(e->chunk_ev[2 * ci + 1], e->stream));
        DLC_CUDA(cudaStreamWaitEvent(e->d2h, e->chunk_ev[2 * ci + 1], 0));
        // speculative: the idle theta_t buffer holds the new weights if the step applies
        DLC_CUDA(cudaMemcpyAsync(host_theta_t + off, e->theta_t[s0.ocur ^ 1] + off, len * sizeof(float),
                                 cudaMemcpyDeviceToHost, e->d2h));
      } else {
        launch_pseudo_grad(tt_pair(e), Pair{{staged, staged}}, e->st, e->send, e->prec, &e->st->delta_nonfinite,
                           off, len, e->stream);
        launched("pseudo_grad_chunk");
      }
    }
    if (e->k == 1) {
      launch_outer_solo_finish(tt_pair(e), local_pair(e), e->st, n, e->stream);
      launched("outer_solo_finish");
    } else {
      outer_collective(e, c, nullptr);  // ORDERED / ALLREDUCE: K4 in place on theta_t[ocur]
      DLC_CUDA(cudaMemcpyAsync(host_theta_t, e->theta_t[s0.ocur], n * sizeof(float), cudaMemcpyDeviceToHost,
                               e->stream));
    }
    DLC_CUDA(cudaStreamSynchronize(e->h2d));
    DLC_CUDA(cudaStreamSynchronize(e->d2h));
    const DevState s1 = read_state(e);
    if (e->k == 1 && !s1.last_applied)  // skipped: theta_t did not move
      DLC_CUDA(cudaMemcpy(host_theta_t, e->theta_t[s1.ocur], n * sizeof(float), cudaMemcpyDeviceToHost));
    outer_result(e, result);
  });
}

int dlc_engine_compute_pseudo_gradient(dlc_engine* e, float* host_delta, uint64_t* outer_epoch) {
  return guard([&] {
    if (!e || (e->n && !host_delta)) fail(DLC_EINVAL, "dlc_engine_compute_pseudo_gradient: null argument");
    if (e->issued_inner % e->cfg.local_steps_h != 0)  // engine.cpp:116-120
      fail(DLC_EINVAL, "pseudo-gradient requested mid-window (inner_step " + std::to_string(e->issued_inner) +
                           ", H " + std::to_string(e->cfg.local_steps_h) + ")");
    DeviceGuard dg(e->device);
    // raw FP32 delta (axpy(-1, theta_local, theta_t), engine.cpp:122) into the staging buffer
    launch_pseudo_grad(tt_pair(e), local_pair(e), e->st, e->grad, DLC_FP32, &e->st->delta_nonfinite, 0, e->n,
                       e->stream);
    launched("pseudo_grad");
    DLC_CUDA(cudaMemcpyAsync(host_delta, e->grad, e->n * sizeof(float), cudaMemcpyDeviceToHost, e->stream));
    const DevState s = read_state(e);
    if (outer_epoch) *outer_epoch = s.outer_epoch;
  });
}

int dlc_engine_apply_outer_step(dlc_engine* e, const float* host_mean, uint64_t outer_epoch,
                                dlc_outer_result* result) {
  return guard([&] {
    if (!e || (e->n && !host_mean)) fail(DLC_EINVAL, "dlc_engine_apply_outer_step: null argument");
    DeviceGuard dg(e->device);
    const DevState s = read_state(e);
    if (outer_epoch != s.outer_epoch)  // engine.cpp:129-134
      fail(DLC_ECOLLECTIVE, "outer_step: reduced pseudo-gradient from epoch " + std::to_string(outer_epoch) +
                                " applied at epoch " + std::to_string(s.outer_epoch));
    DLC_CUDA(cudaMemcpyAsync(e->grad, host_mean, e->n * sizeof(float), cudaMemcpyHostToDevice, e->stream));
    DLC_CUDA(cudaMemsetAsync(e->flags, 0, sizeof(int), e->stream));
    launch_nonfinite(e->grad, e->flags, e->n, e->stream);  // engine.cpp:136
    launch_nesterov_outer(tt_pair(e), buf_pair(e), local_pair(e), e->grad, DLC_FP32, e->flags, 1, e->st,
                          e->hyper.outer_lr, e->hyper.outer_momentum, e->n, e->stream);
    launched("apply_outer_step");
    outer_result(e, result);
  });
}

int dlc_engines_outer_step_local(dlc_engine* const* engines, size_t k, dlc_outer_result* result) {
  return guard([&] {
    if (!engines || k == 0) fail(DLC_ECOLLECTIVE, "outer_step_local: no engines");
    if (k > (size_t)kMaxK) fail(DLC_ECONFIG, "outer_step_local: more than 32 engines");
    dlc_engine* e0 = engines[0];
    for (size_t j = 0; j < k; ++j) {
      dlc_engine* e = engines[j];
      if (!e) fail(DLC_EINVAL, "outer_step_local: null engine");
      if (e->n != e0->n || e->prec != e0->prec || e->device != e0->device)
        fail(DLC_ESHAPE, "outer_step_local: engines differ in size, precision or device");  // reduce.cpp:52-56
      if (e->k != k) fail(DLC_ECOLLECTIVE, "outer_step_local: num_workers_k != fleet size");
      if (e->issued_inner % e->cfg.local_steps_h != 0) fail(DLC_EINVAL, "pseudo-gradient requested mid-window");
    }
    DeviceGuard dg(e0->device);
    cudaEvent_t ev;
    DLC_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    for (size_t j = 1; j < k; ++j) {  // everything below runs on engine 0's stream
      DLC_CUDA(cudaEventRecord(ev, engines[j]->stream));
      DLC_CUDA(cudaStreamWaitEvent(e0->stream, ev, 0));
    }
    cudaStream_t s = e0->stream;
    for (size_t j = 0; j < k; ++j)
      DLC_CUDA(cudaMemsetAsync(&engines[j]->st->delta_nonfinite, 0, sizeof(int), s));
    PtrList in{};
    for (size_t j = 0; j < k; ++j) {
      dlc_engine* e = engines[j];
      launch_pseudo_grad(tt_pair(e), local_pair(e), e->st, e->send, e->prec, &e->st->delta_nonfinite, 0, e->n,
                         s);
      in.ptr[j] = e->send;
    }
    DLC_CUDA(cudaMemsetAsync(e0->flags, 0, kMaxK * sizeof(int), s));
    void* dbar = k > 1 ? e0->gather : e0->send;
    if (k > 1) {
      launch_fold(in, (int)k, e0->prec, e0->gather, e0->prec, e0->flags, e0->n, s);
    } else {
      DLC_CUDA(cudaMemcpyAsync(e0->flags, &e0->st->delta_nonfinite, sizeof(int), cudaMemcpyDeviceToDevice, s));
    }
    for (size_t j = 0; j < k; ++j) {
      dlc_engine* e = engines[j];
      launch_nesterov_outer(tt_pair(e), buf_pair(e), local_pair(e), dbar, e->prec, e0->flags, 1, e->st,
                            e->hyper.outer_lr, e->hyper.outer_momentum, e->n, s);
    }
    launched("outer_step_local");
    DLC_CUDA(cudaEventRecord(ev, s));
    for (size_t j = 1; j < k; ++j) DLC_CUDA(cudaStreamWaitEvent(engines[j]->stream, ev, 0));
    DLC_CUDA(cudaEventDestroy(ev));
    outer_result(e0, result);
  });
}

int dlc_optimizer_step(dlc_engine* e, dlc_collective* c, const float* grad, int grad_is_scaled, int* round_completed) {
  return guard([&] {
    if (!e || (e->n && !grad)) fail(DLC_EINVAL, "dlc_optimizer_step: null argument");
    if (c && c->kind == 0) c = nullptr;
    DeviceGuard dg(e->device);
    engine_inner(e, grad, grad_is_scaled);  // engine.cpp:163
    const bool boundary = e->issued_inner % e->cfg.local_steps_h == 0;
    if (round_completed) *round_completed = boundary ? 1 : 0;
    if (boundary) {  // engine.cpp:165-172
      check_collective(e, c);
      outer_round(e, c, nullptr, nullptr);
    }
  });
}

int dlc_rng_fill_device(dlc_engine* e, int which, uint64_t key, uint64_t first, float lo, float hi) {
  return guard([&] {
    if (!e) fail(DLC_EINVAL, "dlc_rng_fill_device: null engine");
    DeviceGuard dg(e->device);
    float* d = writable(e, which);
    launch_rng_fill(key, first, lo, hi, d, e->n, e->stream);
    launched("rng_fill");
  });
}

int dlc_rng_perturb(dlc_engine* e, float* dst, uint64_t key, float lo, float hi) {
  return guard([&] {
    if (!e) fail(DLC_EINVAL, "dlc_rng_perturb: null engine");
    DeviceGuard dg(e->device);
    float* d = dst ? dst : writable(e, DLC_THETA_LOCAL);
    launch_rng_perturb(live(e, DLC_THETA_T), key, lo, hi, d, e->n, e->stream);
    launched("rng_perturb");
  });
}

// ---- collectives ---------------------------------------------------------------

int dlc_nccl_unique_id(uint8_t id[128]) {
  return guard([&] {
    if (!id) fail(DLC_EINVAL, "dlc_nccl_unique_id: null id");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId u;
    DLC_NCCL(ncclGetUniqueId(&u));
    std::memcpy(id, &u, 128);
  });
}

int dlc_collective_create_nccl(int rank, int world, const uint8_t id[128], int device, int mode,
                               dlc_collective** out) {
  return guard([&] {
    if (!id || !out) fail(DLC_EINVAL, "dlc_collective_create_nccl: null argument");
    if (world < 1 || rank < 0 || rank >= world) fail(DLC_ECONFIG, "bad rank/world");
    if (mode != DLC_MODE_ORDERED && mode != DLC_MODE_ALLREDUCE && mode != DLC_MODE_P2P) fail(DLC_ECONFIG, "unknown reduce mode");
    DeviceGuard dg(device);
    auto* c = new dlc_collective();
    c->kind = 1;
    c->rank = rank;
    c->world = world;
    c->device = device;
    c->mode = mode;
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    const ncclResult_t r = ncclCommInitRank(&c->comm, world, u, rank);
    if (r != ncclSuccess) {
      delete c;
      fail(DLC_ENCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    }
    cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    *out = c;
  });
}

int dlc_collective_create_solo(int device, dlc_collective** out) {
  return guard([&] {
    if (!out) fail(DLC_EINVAL, "dlc_collective_create_solo: null out");
    auto* c = new dlc_collective();
    c->device = device;
    *out = c;
  });
}

int dlc_collective_destroy(dlc_collective* c) {
  if (!c) return DLC_OK;
  return guard([&] {
    if (c->kind == 1) {
      DeviceGuard dg(c->device);
      if (c->stream) cudaStreamDestroy(c->stream);
      ncclCommDestroy(c->comm);
    }
    delete c;
  });
}

size_t dlc_collective_world_size(const dlc_collective* c) { return c ? (size_t)c->world : 1; }
int dlc_collective_rank(const dlc_collective* c) { return c ? c->rank : 0; }

int dlc_collective_all_reduce_avg(dlc_collective* c, const float* local, size_t n, int precision,
                                  uint64_t outer_epoch, float* out, dlc_reduce_report* report) {
  return guard([&] {
    if (!c || (n && (!local || !out))) fail(DLC_EINVAL, "all_reduce_avg: null argument");
    if (precision != DLC_FP32 && precision != DLC_FP16) fail(DLC_ECONFIG, "unknown precision");
    const auto t0 = std::chrono::steady_clock::now();
    if (c->kind == 0 || c->world == 1) {  // SoloCollective, reduce.cpp:113-126
      const float* one[1] = {local};
      const int st = dlc_reduce_average(one, 1, n, precision, out);
      if (st != DLC_OK) fail(st, dlc_last_error());
    } else {
      // Host pseudo-gradient through a transient device engine-less pipeline:
      // encode -> scatter -> ordered fold -> all-gather -> decode.
      DeviceGuard dg(c->device);
      const size_t K = c->world, w = precision == DLC_FP16 ? 2 : 4;
      const size_t S = (((n + K - 1) / K) + 63) / 64 * 64;
      std::vector<void*> allocs;
      auto take = [&](size_t b) {
        void* p = nullptr;
        DLC_CUDA(cudaMalloc(&p, std::max<size_t>(b, 256)));
        allocs.push_back(p);
        return (char*)p;
      };
      try {
        char* src = take(n * 4);
        char* send = take(K * S * w);
        char* recv = take(K * S * w);
        char* gather = take(K * S * w);
        float* res = (float*)take(K * S * 4);
        cudaStream_t s = c->stream;
        DLC_CUDA(cudaMemsetAsync(send, 0, K * S * w, s));
        DLC_CUDA(cudaMemcpyAsync(src, local, n * 4, cudaMemcpyHostToDevice, s));
        if (precision == DLC_FP16)
          launch_encode((const float*)src, (uint16_t*)send, nullptr, n, s);  // collective.cpp:1356-1366
        else
          DLC_CUDA(cudaMemcpyAsync(send, src, n * 4, cudaMemcpyDeviceToDevice, s));
        const int r = c->rank;
        if (c->mode != DLC_MODE_ALLREDUCE) {  // ORDERED and P2P: rank-order fold
          DLC_NCCL(ncclGroupStart());
          for (size_t j = 0; j < K; ++j) {
            if ((int)j == r) continue;
            DLC_NCCL(ncclSend(send + j * S * w, S, nccl_type(precision), (int)j, c->comm, s));
            DLC_NCCL(ncclRecv(recv + j * S * w, S, nccl_type(precision), (int)j, c->comm, s));
          }
          DLC_NCCL(ncclGroupEnd());
          PtrList in{};
          for (size_t j = 0; j < K; ++j) in.ptr[j] = ((int)j == r) ? send + r * S * w : recv + j * S * w;
          launch_fold(in, (int)K, precision, gather + r * S * w, precision, nullptr, S, s);
          DLC_NCCL(ncclAllGather(gather + r * S * w, gather, S, nccl_type(precision), c->comm, s));
        } else {
          DLC_NCCL(ncclAllReduce(send, gather, K * S, nccl_type(precision), ncclAvg, c->comm, s));
        }
        if (precision == DLC_FP16)
          launch_decode((const uint16_t*)gather, res, n, s);
        else
          DLC_CUDA(cudaMemcpyAsync(res, gather, n * 4, cudaMemcpyDeviceToDevice, s));
        DLC_CUDA(cudaMemcpyAsync(out, res, n * 4, cudaMemcpyDeviceToHost, s));
        DLC_LAUNCHED("all_reduce_avg");
        DLC_CUDA(cudaStreamSynchronize(s));
      } catch (...) {
        for (void* p : allocs) cudaFree(p);
        throw;
      }
      for (void* p : allocs) cudaFree(p);
    }
    if (report) {
      *report = dlc_reduce_report{};
      report->outer_epoch = outer_epoch;
      report->contributors = (size_t)c->world;
      report->attempts = 1;
      const uint64_t b = c->world > 1 ? dlc_per_peer_reduce_bytes(n, c->world, c->rank, precision) : 0;
      report->data_bytes_sent = report->data_bytes_received = b;
      report->wire_bytes_sent = report->wire_bytes_received = b;
      report->wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
  });
}

}  // extern "C"

// ---- checkpoint / resume, ODLCKPT1 (checkpoint.cpp:17-198) -------------------------

namespace {

constexpr char kCkptMagic[8] = {'O', 'D', 'L', 'C', 'K', 'P', 'T', '1'};
constexpr size_t kCkptStage = size_t(16) << 20;  // floats per staging round trip

struct File {
  FILE* f = nullptr;
  std::string path;
  File(const char* p, const char* mode) : path(p) {
    f = std::fopen(p, mode);
    if (!f) fail(DLC_ECONFIG, std::string("cannot open checkpoint file '") + p + "'");
  }
  ~File() {
    if (f) std::fclose(f);
  }
  void write(const void* d, size_t b) {
    if (b && std::fwrite(d, 1, b, f) != b) fail(DLC_EINVAL, "checkpoint write failed: " + path);
  }
  void read(void* d, size_t b) {
    if (b && std::fread(d, 1, b, f) != b) fail(DLC_ESERIAL, "checkpoint truncated: " + path);  // checkpoint.cpp:45,60
  }
  void u64(uint64_t v) {
    uint8_t b[8];
    for (int i = 0; i < 8; ++i) b[i] = (uint8_t)(v >> (8 * i));
    write(b, 8);
  }
  uint64_t u64() {
    uint8_t b[8];
    read(b, 8);
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= (uint64_t)b[i] << (8 * i);
    return v;
  }
  void f64(double d) {
    uint64_t v;
    std::memcpy(&v, &d, 8);
    u64(v);
  }
  double f64() {
    const uint64_t v = u64();
    double d;
    std::memcpy(&d, &v, 8);
    return d;
  }
};

struct Seg {
  std::string name;
  uint64_t offset, length;
};

// scalar_header, checkpoint.cpp:74-91 (same printf formats, FP64 text).
std::string ckpt_header(const dlc_engine* e, const DevState& s) {
  char buf[512];
  std::snprintf(buf, sizeof(buf),
                "step_count=%" PRIu64 "\nbeta1=%.17g\nbeta2=%.17g\neps=%.17g\n"
                "weight_decay=%.17g\nouter_lr=%.17g\nouter_momentum=%.17g\n"
                "scale=%.17g\ngrowth_interval=%" PRIu64 "\nconsecutive_good=%" PRIu64
                "\ninner_step=%" PRIu64 "\nouter_epoch=%" PRIu64 "\n",
                s.step_count, (double)e->hyper.beta1, (double)e->hyper.beta2, (double)e->hyper.adam_eps,
                (double)e->hyper.weight_decay, (double)e->hyper.outer_lr, (double)e->hyper.outer_momentum,
                (double)s.scale, s.growth, s.good, s.inner_step, s.outer_epoch);
  return buf;
}

// serialize_layout + FP32 payload (tensor.cpp:156-200), streamed from the device.
void ckpt_write_vector(File& f, const std::vector<Seg>& segs, const float* dev, size_t n, float* stage,
                       cudaStream_t s) {
  uint64_t layout_bytes = 8;
  for (const Seg& g : segs) layout_bytes += 8 + g.name.size() + 16;
  f.u64(layout_bytes + 4 * (uint64_t)n);  // put_block length prefix (checkpoint.cpp:31-34)
  f.u64(segs.size());
  for (const Seg& g : segs) {
    f.u64(g.name.size());
    f.write(g.name.data(), g.name.size());
    f.u64(g.offset);
    f.u64(g.length);
  }
  for (size_t off = 0; off < n; off += kCkptStage) {  // little-endian FP32 (x86 host order)
    const size_t len = std::min(kCkptStage, n - off);
    DLC_CUDA(cudaMemcpyAsync(stage, dev + off, len * 4, cudaMemcpyDeviceToHost, s));
    DLC_CUDA(cudaStreamSynchronize(s));
    f.write(stage, len * 4);
  }
}

// deserialize_param_vector (tensor.cpp:202-218) into a device buffer of n.
void ckpt_read_vector(File& f, float* dev, size_t n, float* stage, cudaStream_t s) {
  const uint64_t block = f.u64();
  const uint64_t nseg = f.u64();
  uint64_t used = 8, total = 0, expect = 0;
  for (uint64_t i = 0; i < nseg; ++i) {
    const uint64_t len = f.u64();
    if (len > (1u << 20)) fail(DLC_ESERIAL, "checkpoint: implausible segment name");  // tensor.cpp:169-176
    std::string name(len, '\0');
    f.read(name.data(), len);
    const uint64_t off = f.u64(), length = f.u64();
    if (off != expect) fail(DLC_ESHAPE, "checkpoint: segments must be contiguous and ordered");  // tensor.cpp:36-47
    expect += length;
    total += length;
    used += 8 + len + 16;
  }
  if (total != n) fail(DLC_ESHAPE, "checkpoint vector of " + std::to_string(total) + " scalars, engine holds " +
                                       std::to_string(n));
  if (block != used + 4 * total) fail(DLC_ESHAPE, "checkpoint: block length mismatch");
  for (size_t off = 0; off < n; off += kCkptStage) {
    const size_t len = std::min(kCkptStage, n - off);
    f.read(stage, len * 4);
    DLC_CUDA(cudaMemcpyAsync(dev + off, stage, len * 4, cudaMemcpyHostToDevice, s));
    DLC_CUDA(cudaStreamSynchronize(s));
  }
}

struct Pinned {
  float* p = nullptr;
  Pinned() { DLC_CUDA(cudaMallocHost(&p, kCkptStage * 4)); }
  ~Pinned() { cudaFreeHost(p); }
};

}  // namespace

extern "C" {

int dlc_checkpoint_save(dlc_engine* const* engines, size_t count, const char* path, const dlc_checkpoint_meta* meta,
                        const char* const* seg_names, const uint64_t* seg_lengths, size_t nseg) {
  return guard([&] {
    if (!engines || !path || !meta) fail(DLC_EINVAL, "dlc_checkpoint_save: null argument");
    if (meta->ledger_workers && !meta->ledger) fail(DLC_EINVAL, "dlc_checkpoint_save: ledger missing");
    for (size_t i = 0; i < count; ++i)
      if (!engines[i]) fail(DLC_EINVAL, "dlc_checkpoint_save: null engine");
    File f(path, "wb");
    f.write(kCkptMagic, 8);  // save_checkpoint, checkpoint.cpp:131-160
    f.u64(meta->config_hash);
    f.u64(meta->completed_rounds);
    f.f64(meta->clock_seconds);
    f.u64(meta->reduce_data_bytes);
    f.u64(meta->ledger_workers);
    for (size_t w = 0; w < meta->ledger_workers; ++w)
      for (int j = 0; j < 3; ++j) f.f64(meta->ledger[3 * w + j]);
    f.u64(count);
    Pinned stage;
    for (size_t i = 0; i < count; ++i) {
      dlc_engine* e = engines[i];
      DeviceGuard dg(e->device);
      std::vector<Seg> segs;
      if (seg_names && nseg) {
        uint64_t off = 0;
        for (size_t j = 0; j < nseg; ++j) {
          segs.push_back({seg_names[j], off, seg_lengths[j]});
          off += seg_lengths[j];
        }
        if (off != e->n) fail(DLC_ESHAPE, "checkpoint layout does not cover the engine's vector");
      } else {
        segs.push_back({"p", 0, e->n});
      }
      const DevState s = read_state(e);
      const std::string header = ckpt_header(e, s);
      f.u64(header.size());
      f.write(header.data(), header.size());
      for (int which : {DLC_THETA_T, DLC_THETA_LOCAL, DLC_ADAM_M, DLC_ADAM_V, DLC_MOMENTUM})
        ckpt_write_vector(f, segs, live(e, which), e->n, stage.p, e->stream);
    }
  });
}

int dlc_checkpoint_load(dlc_engine* const* engines, size_t count, const char* path, dlc_checkpoint_meta* meta_out) {
  return guard([&] {
    if (!engines || !path) fail(DLC_EINVAL, "dlc_checkpoint_load: null argument");
    File f(path, "rb");
    char magic[8];
    f.read(magic, 8);
    if (std::memcmp(magic, kCkptMagic, 8) != 0) fail(DLC_ESERIAL, "not a checkpoint file: bad magic");  // checkpoint.cpp:170
    dlc_checkpoint_meta m{};
    m.config_hash = f.u64();
    m.completed_rounds = f.u64();
    m.clock_seconds = f.f64();
    m.reduce_data_bytes = f.u64();
    m.ledger_workers = f.u64();
    for (size_t w = 0; w < 3 * m.ledger_workers; ++w) (void)f.f64();
    const uint64_t n_eng = f.u64();
    if (n_eng != count)
      fail(DLC_ESHAPE, "checkpoint holds " + std::to_string(n_eng) + " engines, " + std::to_string(count) + " given");
    Pinned stage;
    for (size_t i = 0; i < count; ++i) {
      dlc_engine* e = engines[i];
      if (!e) fail(DLC_EINVAL, "dlc_checkpoint_load: null engine");
      DeviceGuard dg(e->device);
      const uint64_t hl = f.u64();
      if (hl > 4096) fail(DLC_ESERIAL, "checkpoint: implausible scalar header");
      std::string text(hl, '\0');
      f.read(text.data(), hl);
      std::map<std::string, std::string> kv;  // parse_scalar_header, checkpoint.cpp:93-129
      size_t pos = 0;
      while (pos < text.size()) {
        const size_t nl = text.find('\n', pos);
        const std::string line = text.substr(pos, nl == std::string::npos ? std::string::npos : nl - pos);
        pos = nl == std::string::npos ? text.size() : nl + 1;
        const size_t eq = line.find('=');
        if (eq != std::string::npos) kv[line.substr(0, eq)] = line.substr(eq + 1);
      }
      auto need = [&](const char* key) {
        const auto it = kv.find(key);
        if (it == kv.end()) fail(DLC_ESERIAL, std::string("checkpoint header missing '") + key + "'");  // checkpoint.cpp:109
        return it->second;
      };
      unalias(e);
      DevState s = read_state(e);
      s.step_count = std::stoull(need("step_count"));
      e->hyper.beta1 = (float)std::stod(need("beta1"));
      e->hyper.beta2 = (float)std::stod(need("beta2"));
      e->hyper.adam_eps = (float)std::stod(need("eps"));
      e->hyper.weight_decay = (float)std::stod(need("weight_decay"));
      e->hyper.outer_lr = (float)std::stod(need("outer_lr"));
      e->hyper.outer_momentum = (float)std::stod(need("outer_momentum"));
      s.scale = (float)std::stod(need("scale"));
      s.growth = std::stoull(need("growth_interval"));
      e->hyper.scaler_growth_interval = s.growth;
      s.good = std::stoull(need("consecutive_good"));
      s.inner_step = std::stoull(need("inner_step"));
      s.outer_epoch = std::stoull(need("outer_epoch"));
      s.found_inf = 0;
      s.delta_nonfinite = 0;
      if (s.inner_step > e->cfg.total_inner_steps) fail(DLC_ECONFIG, "checkpoint inner_step beyond total_inner_steps");
      for (int which : {DLC_THETA_T, DLC_THETA_LOCAL, DLC_ADAM_M, DLC_ADAM_V, DLC_MOMENTUM})
        ckpt_read_vector(f, live(e, which), e->n, stage.p, e->stream);
      // betas may differ from the engine's: rebuild the per-step tables
      if (e->tab) cudaFree(e->tab);
      e->tab = nullptr;
      e->tab_cap = 0;
      ensure_tables(e, std::max<uint64_t>(s.step_count + 2, e->issued_inner + 2));
      DLC_CUDA(cudaMemcpy(e->st, &s, sizeof(s), cudaMemcpyHostToDevice));
      e->issued_inner = s.inner_step;
    }
    if (meta_out) *meta_out = m;
  });
}

}  // extern "C"

// ---- wire rounds for cross-box transports (include/diloco_cuda.h section 5) ------

namespace {

void check_window(dlc_engine* e) {
  if (e->issued_inner % e->cfg.local_steps_h != 0)  // engine.cpp:116-120
    fail(DLC_EINVAL, "pseudo-gradient requested mid-window (inner_step " + std::to_string(e->issued_inner) +
                         ", H " + std::to_string(e->cfg.local_steps_h) + ")");
}

// DELTA lives in the gradient staging buffer (4N bytes), MEAN in the send
// buffer (K*S >= N elements of the engine's width); both are contiguous [0, N).
char* wire_vector(dlc_engine* e, int which) {
  if (which == DLC_WIRE_DELTA) return reinterpret_cast<char*>(e->grad);
  if (which == DLC_WIRE_MEAN) return static_cast<char*>(e->send);
  fail(DLC_EINVAL, "wire: unknown buffer " + std::to_string(which));
}

// Fold rows are stored 8 elements apart at least (16-byte aligned vectors for
// the fold kernel, whatever the owned range's length).
uint64_t row_stride(uint64_t capacity) { return (capacity + 7) / 8 * 8; }

// Grows the row buffer to `rows` rows of the current stride, keeping its contents.
char* wire_rows(dlc_engine* e, size_t rows) {
  const size_t need = std::max<size_t>(rows * row_stride(e->wire_stride) * elem_width(e->prec), 256);
  if (need > e->wire_rows_bytes) {
    DLC_CUDA(cudaStreamSynchronize(e->stream));
    void* fresh = nullptr;
    DLC_CUDA(cudaMalloc(&fresh, need));
    if (e->wire_rows) {
      DLC_CUDA(cudaMemcpy(fresh, e->wire_rows, e->wire_rows_bytes, cudaMemcpyDeviceToDevice));
      cudaFree(e->wire_rows);
    }
    e->wire_rows = fresh;
    e->wire_rows_bytes = need;
  }
  return static_cast<char*>(e->wire_rows);
}

void check_range(dlc_engine* e, uint64_t offset, uint64_t length) {
  if (offset > e->n || length > e->n - offset)
    fail(DLC_ESHAPE, "wire: range [" + std::to_string(offset) + ", +" + std::to_string(length) +
                         ") outside the engine's " + std::to_string(e->n) + " elements");
}

}  // namespace

int dlc_engine_wire_begin(dlc_engine* e, uint64_t* outer_epoch) {
  return guard([&] {
    if (!e) fail(DLC_EINVAL, "dlc_engine_wire_begin: null engine");
    check_window(e);
    DeviceGuard dg(e->device);
    // encode once at the source (collective.cpp:1356-1366): FP16 codes or FP32 deltas
    launch_pseudo_grad(tt_pair(e), local_pair(e), e->st, e->grad, e->prec, &e->st->delta_nonfinite, 0, e->n,
                       e->stream);
    launched("pseudo_grad");
    const DevState s = read_state(e);
    if (outer_epoch) *outer_epoch = s.outer_epoch;
  });
}

int dlc_engine_wire_encode(dlc_engine* e, int which, uint64_t offset, uint64_t length, const dlc_wire_tags* tags,
                           uint8_t* host_out, size_t cap, size_t* used) {
  return guard([&] {
    if (!e || !tags) fail(DLC_EINVAL, "dlc_engine_wire_encode: null argument");
    if (tags->precision != e->prec) fail(DLC_ECONFIG, "wire encode: tag precision differs from the engine's");
    check_range(e, offset, length);
    DeviceGuard dg(e->device);
    const char* base = wire_vector(e, which);
    wire_encode_impl(base + offset * elem_width(e->prec), offset, length, tags, host_out, cap, used, e->stream);
  });
}

int dlc_engine_wire_decode(dlc_engine* e, int which, int row, uint64_t base_offset, uint64_t capacity,
                           const uint8_t* host_in, size_t bytes, dlc_wire_chunk* chunks, size_t max_chunks,
                           size_t* n_chunks, size_t* consumed) {
  return guard([&] {
    if (!e) fail(DLC_EINVAL, "dlc_engine_wire_decode: null engine");
    check_range(e, base_offset, capacity);
    DeviceGuard dg(e->device);
    const size_t w = elem_width(e->prec);
    char* dst = nullptr;
    if (which == DLC_WIRE_ROW) {  // contributor `row`'s slice of the owned range
      if (row < 0 || row >= kMaxK) fail(DLC_EINVAL, "wire decode: row out of range");
      e->wire_stride = capacity;  // a new range (round / membership) makes earlier rows stale
      dst = wire_rows(e, (size_t)row + 1) + (size_t)row * row_stride(capacity) * w;
    } else if (which == DLC_WIRE_MEAN || which == DLC_WIRE_DELTA) {
      dst = wire_vector(e, which) + base_offset * w;
    } else {
      fail(DLC_EINVAL, "wire: unknown buffer " + std::to_string(which));
    }
    wire_decode_impl(host_in, bytes, e->prec, base_offset, capacity, dst, chunks, max_chunks, n_chunks, consumed,
                     e->stream);
  });
}

int dlc_engine_wire_fold(dlc_engine* e, int rank, int k, uint64_t offset, uint64_t length) {
  return guard([&] {
    if (!e) fail(DLC_EINVAL, "dlc_engine_wire_fold: null engine");
    if (k < 1 || k > kMaxK || rank < 0 || rank >= k) fail(DLC_EINVAL, "wire fold: bad rank / contributor count");
    check_range(e, offset, length);
    if (k > 1 && length != e->wire_stride && e->wire_rows)
      fail(DLC_ESHAPE, "wire fold: rows were decoded for a range of " + std::to_string(e->wire_stride) +
                           " elements, fold asks for " + std::to_string(length));
    if (k > 1 && !e->wire_rows) fail(DLC_EINVAL, "wire fold: no contributions decoded");
    DeviceGuard dg(e->device);
    const size_t w = elem_width(e->prec);
    e->wire_stride = length;
    const size_t stride = row_stride(length) * w;
    char* rows = wire_rows(e, (size_t)k + 1);  // k contributions + an aligned output row
    char* own = reinterpret_cast<char*>(e->grad) + offset * w;
    char* out = static_cast<char*>(e->send) + offset * w;
    const bool aligned = (offset * w) % 16 == 0;  // vector loads / stores of the fold kernel
    if (!aligned && length)  // our own slice joins the rows
      DLC_CUDA(cudaMemcpyAsync(rows + (size_t)rank * stride, own, length * w, cudaMemcpyDeviceToDevice, e->stream));
    PtrList in{};
    for (int j = 0; j < k; ++j)  // peer-sorted order; our own slice from DELTA (collective.cpp:1460-1474)
      in.ptr[j] = (j == rank && aligned) ? own : rows + (size_t)j * stride;
    DLC_CUDA(cudaMemsetAsync(e->flags, 0, sizeof(int), e->stream));
    if (length) {
      char* dst = aligned ? out : rows + (size_t)k * stride;
      launch_fold(in, k, e->prec, dst, e->prec, e->flags, length, e->stream);
      launched("fold");
      if (!aligned) DLC_CUDA(cudaMemcpyAsync(out, dst, length * w, cudaMemcpyDeviceToDevice, e->stream));
    }
    DLC_CUDA(cudaStreamSynchronize(e->stream));
  });
}

int dlc_engine_wire_finish(dlc_engine* e, uint64_t outer_epoch, dlc_outer_result* result) {
  return guard([&] {
    if (!e) fail(DLC_EINVAL, "dlc_engine_wire_finish: null engine");
    DeviceGuard dg(e->device);
    const DevState s = read_state(e);
    if (outer_epoch != s.outer_epoch)  // engine.cpp:129-134
      fail(DLC_ECOLLECTIVE, "outer_step: reduced pseudo-gradient from epoch " + std::to_string(outer_epoch) +
                                " applied at epoch " + std::to_string(s.outer_epoch));
    DLC_CUDA(cudaMemsetAsync(e->flags, 0, sizeof(int), e->stream));
    if (e->prec == DLC_FP16)  // engine.cpp:136 on the decoded mean: non-finite <=> inf/NaN code
      launch_nonfinite_codes(static_cast<const uint16_t*>(e->send), e->flags, e->n, e->stream);
    else
      launch_nonfinite(static_cast<const float*>(e->send), e->flags, e->n, e->stream);
    launch_nesterov_outer(tt_pair(e), buf_pair(e), local_pair(e), e->send, e->prec, e->flags, 1, e->st,
                          e->hyper.outer_lr, e->hyper.outer_momentum, e->n, e->stream);
    launched("wire_outer_step");
    outer_result(e, result);
  });
}

// ---- single-process multi-GPU world (include/diloco_cuda.h section 3) ----------

struct dlc_world {
  int k = 0;
  int mode = DLC_MODE_P2P;
  std::vector<int> devices;
  std::vector<dlc_engine*> engines;
  std::vector<dlc_collective*> colls;
};

namespace {

// Every engine's peer tables point straight at the other engines' buffers
// (one address space, peer access enabled): no IPC, no handle exchange.
void world_bind_p2p(dlc_world* w) {
  for (int a = 0; a < w->k; ++a) {
    DeviceGuard dg(w->devices[a]);
    for (int b = 0; b < w->k; ++b) {
      if (a == b || w->devices[a] == w->devices[b]) continue;
      const cudaError_t st = cudaDeviceEnablePeerAccess(w->devices[b], 0);
      if (st == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
      } else if (st != cudaSuccess) {
        fail(DLC_ECUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(st));
      }
    }
  }
  for (int r = 0; r < w->k; ++r) {
    dlc_engine* e = w->engines[r];
    for (int j = 0; j < w->k; ++j) {
      dlc_engine* q = w->engines[j];
      e->peer_send[j] = q->send;
      e->peer_gather[j] = q->gather;
      e->peer_flags[j] = q->flags;
      e->peer_sig[j] = q->sig;
      e->peer_recv[j] = q->recv;
    }
    e->p2p_bound = w->colls[r];
  }
}

// DLC_MODE_ORDERED from one thread: the per-rank NCCL calls of
// outer_collective, grouped across the K communicators.
void world_outer_nccl(dlc_world* w) {
  const int K = w->k;
  dlc_engine* e0 = w->engines[0];
  const size_t S = e0->S, wd = elem_width(e0->prec);
  const ncclDataType_t type = nccl_type(e0->prec);
  for (int r = 0; r < K; ++r) {
    DeviceGuard dg(w->devices[r]);
    dlc_engine* e = w->engines[r];
    reset_flags(e);
    pseudo_grad(e, local_pair(e));
  }
  if (w->mode == DLC_MODE_ORDERED) {
    DLC_NCCL(ncclGroupStart());
    for (int r = 0; r < K; ++r) {
      dlc_engine* e = w->engines[r];
      char* send = static_cast<char*>(e->send);
      char* recv = static_cast<char*>(e->recv);
      for (int j = 0; j < K; ++j) {
        if (j == r) continue;
        DLC_NCCL(ncclSend(send + j * S * wd, S, type, j, w->colls[r]->comm, e->stream));
        DLC_NCCL(ncclRecv(recv + j * S * wd, S, type, j, w->colls[r]->comm, e->stream));
      }
    }
    DLC_NCCL(ncclGroupEnd());
    for (int r = 0; r < K; ++r) {  // owner fold in rank order (collective.cpp:1444-1489)
      DeviceGuard dg(w->devices[r]);
      dlc_engine* e = w->engines[r];
      char* send = static_cast<char*>(e->send);
      char* recv = static_cast<char*>(e->recv);
      PtrList in{};
      for (int j = 0; j < K; ++j) in.ptr[j] = j == r ? send + r * S * wd : recv + j * S * wd;
      launch_fold(in, K, e->prec, static_cast<char*>(e->gather) + r * S * wd, e->prec, e->flags + r, S, e->stream);
      launched("fold");
    }
    DLC_NCCL(ncclGroupStart());
    for (int r = 0; r < K; ++r) {
      dlc_engine* e = w->engines[r];
      char* gather = static_cast<char*>(e->gather);
      DLC_NCCL(ncclAllGather(gather + r * S * wd, gather, S, type, w->colls[r]->comm, e->stream));
      DLC_NCCL(ncclAllGather(e->flags + r, e->flags, 1, ncclInt32, w->colls[r]->comm, e->stream));
    }
    DLC_NCCL(ncclGroupEnd());
    for (int r = 0; r < K; ++r) {
      DeviceGuard dg(w->devices[r]);
      nesterov(w->engines[r], w->engines[r]->gather, w->engines[r]->flags, K);
    }
  } else {  // DLC_MODE_ALLREDUCE
    DLC_NCCL(ncclGroupStart());
    for (int r = 0; r < K; ++r) {
      dlc_engine* e = w->engines[r];
      DLC_NCCL(ncclAllReduce(e->send, e->send, K * S, type, ncclAvg, w->colls[r]->comm, e->stream));
    }
    DLC_NCCL(ncclGroupEnd());
    for (int r = 0; r < K; ++r) {
      DeviceGuard dg(w->devices[r]);
      dlc_engine* e = w->engines[r];
      if (e->prec == DLC_FP16)
        launch_nonfinite_codes(static_cast<const uint16_t*>(e->send), e->flags, e->n, e->stream);
      else
        launch_nonfinite(static_cast<const float*>(e->send), e->flags, e->n, e->stream);
      launched("nonfinite");
      nesterov(e, e->send, e->flags, 1);
    }
  }
}

}  // namespace

int dlc_world_create(const dlc_config* cfg, const dlc_hyperparams* hyper, size_t n_params, const int* devices,
                     int inner_mode, int mode, dlc_world** out) {
  dlc_world* w = nullptr;
  const int st = guard([&] {
    if (!cfg || !hyper || !devices || !out) fail(DLC_EINVAL, "dlc_world_create: null argument");
    *out = nullptr;
    if (mode != DLC_MODE_ORDERED && mode != DLC_MODE_ALLREDUCE && mode != DLC_MODE_P2P)
      fail(DLC_ECONFIG, "unknown reduce mode");
    const int k = (int)cfg->num_workers_k;
    if (k < 1 || k > kMaxK) fail(DLC_ECONFIG, "world size must be 1..32");
    w = new dlc_world();
    w->k = k;
    w->mode = mode;
    w->devices.assign(devices, devices + k);
    for (int r = 0; r < k; ++r) {
      dlc_engine* e = nullptr;
      const int s2 = dlc_engine_create(cfg, hyper, n_params, devices[r], inner_mode, &e);
      if (s2 != DLC_OK) fail(s2, std::string("world engine ") + std::to_string(r) + ": " + dlc_last_error());
      w->engines.push_back(e);
    }
    std::vector<ncclComm_t> comms(k, nullptr);
    if (k > 1) {
      for (int r = 1; r < k; ++r)
        for (int q = 0; q < r; ++q)
          if (devices[q] == devices[r]) fail(DLC_ECONFIG, "world ranks need distinct devices");
      DLC_NCCL(ncclCommInitAll(comms.data(), k, devices));
    }
    for (int r = 0; r < k; ++r) {
      auto* c = new dlc_collective();
      c->kind = k > 1 ? 1 : 0;
      c->rank = r;
      c->world = k;
      c->device = devices[r];
      c->mode = mode;
      c->comm = comms[r];
      c->in_world = true;
      w->colls.push_back(c);
    }
    if (k > 1 && mode == DLC_MODE_P2P) world_bind_p2p(w);
    *out = w;
  });
  if (st != DLC_OK && w) dlc_world_destroy(w);
  return st;
}

int dlc_world_destroy(dlc_world* w) {
  if (!w) return DLC_OK;
  return guard([&] {
    for (size_t r = 0; r < w->engines.size(); ++r) {  // everything in flight on every GPU first
      DeviceGuard dg(w->devices[r]);
      cudaDeviceSynchronize();
    }
    for (dlc_engine* e : w->engines) {
      e->p2p_bound = nullptr;  // direct pointers: nothing to unmap, no fleet barrier
      dlc_engine_destroy(e);
    }
    for (size_t r = 0; r < w->colls.size(); ++r) {
      DeviceGuard dg(w->devices[r]);
      if (w->colls[r]->comm) ncclCommDestroy(w->colls[r]->comm);
      delete w->colls[r];
    }
    delete w;
  });
}

int dlc_world_engine(dlc_world* w, int rank, dlc_engine** e) {
  return guard([&] {
    if (!w || !e) fail(DLC_EINVAL, "dlc_world_engine: null argument");
    if (rank < 0 || rank >= w->k) fail(DLC_EINVAL, "dlc_world_engine: rank out of range");
    *e = w->engines[rank];
  });
}

int dlc_world_outer_step(dlc_world* w, dlc_outer_result* result) {
  return guard([&] {
    if (!w) fail(DLC_EINVAL, "dlc_world_outer_step: null world");
    for (int r = 0; r < w->k; ++r) check_collective(w->engines[r], w->k > 1 ? w->colls[r] : nullptr);
    if (w->k == 1) {
      DeviceGuard dg(w->devices[0]);
      outer_round(w->engines[0], nullptr, nullptr, nullptr);
    } else if (w->mode == DLC_MODE_P2P) {
      // every rank's pipelined step is enqueued without a host wait; the
      // flag barriers inside synchronise the GPUs with each other
      for (int r = 0; r < w->k; ++r) {
        DeviceGuard dg(w->devices[r]);
        outer_p2p_pipelined(w->engines[r], w->colls[r], nullptr, nullptr, nullptr, nullptr, 0);
      }
    } else {
      world_outer_nccl(w);
    }
    if (result) {
      dlc_outer_result r0{};
      for (int r = 0; r < w->k; ++r) {
        DeviceGuard dg(w->devices[r]);
        dlc_outer_result rr{};
        outer_result(w->engines[r], &rr);
        if (r == 0) r0 = rr;
        if (rr.applied != r0.applied || rr.outer_epoch != r0.outer_epoch)
          fail(DLC_ECOLLECTIVE, "world ranks disagree on the outer step");
      }
      *result = r0;
    }
  });
}
