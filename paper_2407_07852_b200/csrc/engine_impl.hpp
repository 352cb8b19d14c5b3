// engine_impl.hpp — the engine and collective state shared by the engine's
// translation units (engine.cu: the C ABI of the device engine; engine_util.cu:
// buffers, tables, timing, inner step; p2p.cu: the outer step's collectives;
// collective.cu, checkpoint.cu, wire_engine.cu, world.cu).  Internal: nothing
// here is exported from libdiloco_cuda.so.
#pragma once

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <string>
#include <vector>

#include "internal.hpp"
#include "kernels.cuh"

struct dlc_engine;

struct dlc_collective {
  int kind = 0;  // 0 solo, 1 nccl
  int rank = 0;
  int world = 1;
  int device = 0;
  int mode = DLC_MODE_ORDERED;
  ncclComm_t comm = nullptr;
  cudaStream_t stream = nullptr;  // used only by the host-buffer plugin call
  bool in_world = false;          // one of the K collectives of a dlc_world (one host thread)
  // membership: members[i] = rank in the ORIGINAL world of
  // this communicator's rank i (the reference's sorted contributor list)
  int members[dlc::kMaxK] = {};
  bool shrunk = false;                 // made by dlc_collective_shrink (engines re-layout for it)
  bool broken = false;                 // a round failed on it, or ranks were excluded from it: abort on destroy
  uint64_t timeout_ms = 20000;         // NodeOptions::reduce_timeout_ms: P2P barrier failure detector
  int64_t stall_at = -1;               // fault injection: stop arriving from this barrier on (-1 off)
  int64_t barriers = 0;                // P2P barriers issued on this collective
  std::vector<dlc_engine*> bound;      // engines whose peer tables map this collective's members
  std::vector<dlc_engine*> watchers;   // engines whose last NCCL round on it is watched (engine::watch_coll)
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
  dlc::DevState* st = nullptr;
  float* tab = nullptr;  // corr1 | corr2 | lr, tab_cap entries each
  size_t tab_cap = 0;
  uint64_t issued_inner = 0;  // host mirror of the data cursor (always advances)
  // K2 fused into the last inner step of a window (dlc_engine_set_fused_delta;
  // K = 1: the whole solo outer step fused into it by dlc_optimizer_step /
  // dlc_run_training, on by default; K > 1:
  // delta_fused = that K1 wrote the send buffer and nothing has touched theta_t,
  // theta_local or the send buffer since; the outer step then runs only the gated K2.
  bool fuse_delta = false;
  bool delta_fused = false;
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
  // into this process through CUDA IPC (own entries are local; a dlc_world
  // points them straight at the other engines' buffers).
  int* barrier_buf = nullptr;
  const dlc_collective* p2p_bound = nullptr;
  void* peer_send[dlc::kMaxK] = {};
  void* peer_gather[dlc::kMaxK] = {};
  int* peer_flags[dlc::kMaxK] = {};
  uint64_t* sig = nullptr;  // flag-barrier signal slots, one per rank
  uint64_t* peer_sig[dlc::kMaxK] = {};
  uint64_t sig_epoch = 0;
  int* sig_err = nullptr;
  size_t k_cap = 1;      // collective buffers hold any layout k' <= k_cap (membership changes)
  size_t slot_cap = 0;   // elements per collective buffer: max over k' <= k_cap of k' * S(k')
  uint64_t failed_tries = 0;  // consecutive failed rounds at the current epoch (ReduceReport::attempts - 1)
  // Failure detector of the NCCL modes (ORDERED / ALLREDUCE, one process per
  // GPU; NCCL itself never times out): the round's device work is watched
  // through an event until reduce_timeout_ms after it was enqueued; a host wait
  // past that deadline declares the round failed (stream_wait).
  bool watched = false;
  std::chrono::steady_clock::time_point deadline{};
  uint64_t watch_ms = 0;
  cudaEvent_t watch_ev = nullptr;
  dlc_collective* watch_coll = nullptr;  // marked broken on a timeout (its destroy then aborts, not waits)
  bool nccl_failed = false;  // reported; drained and reset at the next outer step
  std::vector<void*> ipc_opened;
  // host-buffer path: copy streams and per-chunk events
  cudaStream_t h2d = nullptr, d2h = nullptr;
  std::vector<cudaEvent_t> chunk_ev;
  // pipelined P2P: high-priority stream for barriers + owner folds, per-piece events
  cudaStream_t cstream = nullptr;
  struct TraceMark {
    const char* label;
    int piece;
    cudaEvent_t a, b;
  };
  std::vector<TraceMark> trace;  // DLC_TRACE=1: per-op timeline of the P2P step
  std::vector<cudaEvent_t> piece_ev;
  // dlc_run_training: pinned ring of device-scalar snapshots + per-step events,
  // made on the first call and kept (no allocation inside a training loop)
  static constexpr int kRing = 4;
  dlc::DevState* ring_host = nullptr;
  cudaEvent_t ring_a[kRing] = {}, ring_b[kRing] = {};
  // wire rounds (dlc_engine_wire_*): fold rows of the owned range, `wire_stride` elements each
  void* wire_rows = nullptr;
  size_t wire_rows_bytes = 0;
  uint64_t wire_stride = 0;
};


namespace dlc {

inline size_t elem_width(int prec) { return prec == DLC_FP16 ? 2 : 4; }

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) DLC_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

inline void launched(const char* what) { DLC_LAUNCHED(what); }

inline ncclDataType_t nccl_type(int prec) { return prec == DLC_FP16 ? ncclFloat16 : ncclFloat32; }

// Host <-> device chunk of the host-buffer outer step (64 MB of FP32).
constexpr size_t kHostChunk = size_t(16) << 20;
// Pieces of the pipelined P2P outer step (DLC_MODE_P2P).
// Owner slots are a multiple of 64 * kMaxPieces elements.
constexpr size_t kMaxPieces = 8;
// CTAs of the per-thread fold (K > 8, where the TMA fold has no instance);
// 256 from profiles/r1_sweep_p2p_{2,4}gpu_kk.log
constexpr int kFoldCtas = 256;

// ---- engine_util.cu ----
void* dalloc(dlc_engine* e, size_t bytes);
// Piece boundaries inside an owner slot of S elements, for a vector of n
// elements per worker.  Measured defaults (dlc_p2p_set_tuning overrides):
// 1,2,3,2,1 ninths (r2: 6.22 vs 6.27 ms at 4 GPUs, 5.88 vs 5.96 at 2 against
// round 1's 1,1,2,2,1,1, profiles/r2_ab_plan_1p1b_*), or 1,2,2,1 below 400M
// elements per worker, where the
// step is ~1 ms and per-piece costs outweigh a shorter fill / drain (150M:
// 0.99 vs 1.07 ms at 4 GPUs, 0.88 vs 0.95 ms at 2 against the 1.1B plan;
// 1,3,3,1 1.00 / 0.90 ms; profiles/r1_sweep_150m_*, r2_sweep_150m_*).
// host_path: the e2e call with host buffers, where the step is PCIe-bound and
// the pipeline fill / drain is one piece of H2D / D2H: 16 equal pieces.
constexpr size_t kSmallStepElems = 400000000;
std::vector<size_t> piece_plan(size_t S, size_t n, bool host_path = false);
int tma_ctas(size_t k);
int tma_threads(size_t k);
int piece_ctas();
int fold_kernel();
void ensure_copy_streams(dlc_engine* e);
void ensure_chunk_events(dlc_engine* e, size_t count);
void harvest(dlc_engine* e);
void harvest_if_full(dlc_engine* e);
cudaEvent_t pooled_event(dlc_engine* e);
void phase_begin(dlc_engine* e);
void phase_end(dlc_engine* e, int phase);
bool tracing();
cudaEvent_t trace_begin(dlc_engine* e, cudaStream_t s);
void trace_end(dlc_engine* e, cudaStream_t s, const char* label, int piece, cudaEvent_t a);
void trace_dump(dlc_engine* e, cudaEvent_t origin);
void ensure_tables(dlc_engine* e, uint64_t t_max);
DevState read_state(dlc_engine* e);
// cudaStreamSynchronize of the engine stream that raises CollectiveError when a
// watched NCCL round passes its deadline (the stream may then stay blocked
// until the caller shrinks the collective with DLC_SHRINK_ABORT).
void stream_wait(dlc_engine* e);
void watch_round(dlc_engine* e, dlc_collective* c);
void unwatch(dlc_engine* e);
// The failed round's commit gate: ncclAllReduce(MAX) of the error word, so
// every rank's finish takes the same decision, then the speculative K4 of
// the whole vector and the finish (abort = the error word).
void drain_failed_round(dlc_engine* e);
float* live(dlc_engine* e, int which);
void unalias(dlc_engine* e);
float* writable(dlc_engine* e, int which);
void engine_inner(dlc_engine* e, const float* grad, int grad_is_scaled);
// The window boundary of a single worker as one fused pass (launch_boundary_solo):
// usable when the next inner step completes a window, K = 1 (either inner mode), and the
// collective is the solo one.  engine_boundary_solo = that inner step + the
// outer step (engine.cpp:162-174).
bool boundary_solo_ok(const dlc_engine* e, const dlc_collective* c);
void engine_boundary_solo(dlc_engine* e, const float* grad, int grad_is_scaled);
// The outer step's K2 input: true (and cleared) when the window's last K1 wrote
// the delta into the send buffer (DevState::delta_ready then tells the device
// whether it still holds).
inline bool take_fused_delta(dlc_engine* e) {
  const bool f = e->delta_fused;
  e->delta_fused = false;
  return f;
}
// K2 of an outer step: the gated fallback after a fused K1, else the full pass.
void pseudo_grad_step(dlc_engine* e, Pair tl, bool fused);
// PINGPONG: theta_local follows theta_t after every outer step (Pair::follow).
inline Pair local_pair(dlc_engine* e) { return Pair{{e->p[0], e->p[1]}, e->inner_mode == DLC_INNER_PINGPONG}; }
inline Pair tt_pair(dlc_engine* e) { return Pair{{e->theta_t[0], e->theta_t[1]}}; }
inline Pair buf_pair(dlc_engine* e) { return Pair{{e->buf[0], e->buf[1]}}; }
void reset_flags(dlc_engine* e);
void pseudo_grad(dlc_engine* e, Pair tl);
void nesterov(dlc_engine* e, const void* dbar, const int* flags, int nflags);

// ---- p2p.cu ----
void p2p_unbind(dlc_engine* e);
void p2p_bind(dlc_engine* e, dlc_collective* c);
void fleet_barrier(dlc_engine* e, dlc_collective* c);
void p2p_barrier(dlc_engine* e, dlc_collective* c, cudaStream_t s, bool commit);
void outer_collective(dlc_engine* e, dlc_collective* c, dlc_reduce_report* rep);
// One pipelined DLC_MODE_P2P outer step of one engine, in stages.  Ranks
// synchronise between the stages: flag barriers (outer_p2p_pipelined) or
// event dependencies (world.cu).
struct P2PStep {
  dlc_engine* e = nullptr;
  int rank = 0;
  size_t K = 0, S = 0, w = 0, n = 0, P = 0;
  std::vector<size_t> pb;  // piece boundaries inside an owner slot
  Pair tl{};               // theta_local source (the engine's, or a staging buffer)
  const float* hsrc = nullptr;
  float* hdst = nullptr;
  int oc_host = 0;
  bool rep = false;
  cudaEvent_t *evK2 = nullptr, *evB = nullptr, *evH = nullptr, *evK4 = nullptr;
  cudaEvent_t evStart = nullptr, evCommit = nullptr, c0 = nullptr, c1 = nullptr, origin = nullptr;
  PtrList slots{}, fl{};
};
P2PStep p2p_begin(dlc_engine* e, int rank, const float* src, bool rep, const float* hsrc, float* hdst, int oc_host);
void p2p_k2(P2PStep& s, size_t p);
void p2p_k2_all(P2PStep& s, bool fused);
void p2p_fold_begin(P2PStep& s);
void p2p_fold(P2PStep& s, size_t p);
void p2p_fold_end(P2PStep& s);
void p2p_k4(P2PStep& s, size_t p);
void p2p_finish(P2PStep& s, const int* abort);
void outer_p2p_pipelined(dlc_engine* e, dlc_collective* c, const float* src, dlc_reduce_report* rep,
                         const float* hsrc, float* hdst, int oc_host, bool fused = false);
void outer_allreduce_pipelined(dlc_engine* e, dlc_collective* c, const float* src, dlc_reduce_report* rep,
                               bool fused = false);
void outer_round(dlc_engine* e, dlc_collective* c, const float* src, dlc_reduce_report* rep);

// ---- engine_util.cu (results) ----
void fill_report(dlc_engine* e, dlc_collective* c, dlc_reduce_report* rep, uint64_t epoch);
uint64_t per_peer_reduce_bytes_received(size_t n, size_t k, size_t rank, int precision);
void check_collective(dlc_engine* e, dlc_collective* c);
void check_barrier(dlc_engine* e);
size_t slot_elems(size_t n, size_t k);
void relayout(dlc_engine* e, size_t k);
void outer_result(dlc_engine* e, dlc_outer_result* res);

}  // namespace dlc
