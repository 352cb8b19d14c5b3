// p2p.cu — the outer step's cross-worker average on device buffers: the NCCL
// modes (ORDERED: grouped send/recv + rank-ordered fold + all-gather;
// ALLREDUCE: ncclAllReduce, pipelined over pieces) and DLC_MODE_P2P (the fold
// fused with its data movement over NVLink peer memory, CUDA-IPC mapped),
// with the flag barriers and the pipelined K2 / fold / K4 schedule.
#include <chrono>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "engine_impl.hpp"

namespace dlc {

void p2p_unbind(dlc_engine* e) {
  for (void* p : e->ipc_opened) cudaIpcCloseMemHandle(p);
  e->ipc_opened.clear();
  if (e->p2p_bound) {
    auto& b = const_cast<dlc_collective*>(e->p2p_bound)->bound;
    b.erase(std::remove(b.begin(), b.end(), e), b.end());
  }
  e->p2p_bound = nullptr;
}

// Maps every rank's send buffer, owner slot and owner flag into this process:
// IPC handles are all-gathered over the collective's own NCCL communicator.
void p2p_bind(dlc_engine* e, dlc_collective* c) {
  if (e->p2p_bound == c) return;
  p2p_unbind(e);
  const int K = (int)e->k, r = c->rank;
  struct Handles {
    cudaIpcMemHandle_t send, gather, flags, sig;
    uint64_t sig_epoch;
  };
  Handles mine;
  mine.sig_epoch = e->sig_epoch;
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
  // Barrier epochs continue above every epoch any rank has used, so a signal
  // left over from an abandoned round (or an earlier membership) never
  // satisfies a barrier of this one.
  for (int j = 0; j < K; ++j) e->sig_epoch = std::max(e->sig_epoch, all[j].sig_epoch);
  for (int j = 0; j < K; ++j) {
    if (j == r) {
      e->peer_send[j] = e->send;
      e->peer_gather[j] = e->gather;
      e->peer_flags[j] = e->flags;
      e->peer_sig[j] = e->sig;
      continue;
    }
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
  c->bound.push_back(e);
}

// Stream-ordered fleet barrier: a 4-byte NCCL all-reduce.
void fleet_barrier(dlc_engine* e, dlc_collective* c) {
  DLC_NCCL(ncclAllReduce(e->barrier_buf, e->barrier_buf, 1, ncclInt32, ncclSum, c->comm, e->stream));
}

// Phase barrier of the P2P step on stream `s`: NVLink flags (one CTA, a few
// microseconds), also the failure detector.  `commit`: the last barrier of a
// step, whose signals carry the ranks' error bits (every rank's finish gate
// then aborts if any rank's round failed).
void p2p_barrier(dlc_engine* e, dlc_collective* c, cudaStream_t s, bool commit) {
  PtrList remote{};
  for (size_t j = 0; j < e->k; ++j) remote.ptr[j] = e->peer_sig[j] + c->rank;
  e->sig_epoch += 1;
  const bool stall = c->stall_at >= 0 && c->barriers >= c->stall_at;
  c->barriers += 1;
  launch_flag_barrier(remote, e->sig, (int)e->k, c->rank, e->sig_epoch, e->sig_err, c->timeout_ms * 1000000ull, stall,
                      commit, s);
  launched("flag_barrier");
}

// The end of an NCCL-mode round (ORDERED / ALLREDUCE, one process per GPU):
// the ranks' error words are OR-ed (ncclAllReduce MAX) so every finish gate
// takes the same decision, K4 runs speculatively into the idle theta_t /
// momentum over `nslots` mean slots (`slots`, `S` elements apart) and the finish
// flips them in only when every mark is clean and no rank's round failed; the
// round is watched by the NCCL-mode failure detector (stream_wait).
// The OR lands in a second word (sig_err[1]) and is folded into the local one
// after the all-reduce: a round released by an abort leaves that buffer
// undefined, and the local word (set by the failure detector) must survive.
static void nccl_error_or(dlc_engine* e, dlc_collective* c, cudaStream_t s) {
  DLC_NCCL(ncclAllReduce(e->sig_err, e->sig_err + 1, 1, ncclInt32, ncclMax, c->comm, s));
  launch_or_word(e->sig_err, e->sig_err + 1, s);
  launched("or_word");
}

static void nccl_round_commit(dlc_engine* e, dlc_collective* c, const PtrList& slots, int nslots, size_t S,
                              const PtrList& marks, int nmarks, cudaStream_t err_stream) {
  nccl_error_or(e, c, err_stream);
  if (err_stream != e->stream) {
    cudaEvent_t ev = pooled_event(e);
    DLC_CUDA(cudaEventRecord(ev, err_stream));
    DLC_CUDA(cudaStreamWaitEvent(e->stream, ev, 0));
    e->pool.push_back(ev);
  }
  phase_begin(e);
  if (nslots > 0)
    launch_nesterov_p2p_piece(tt_pair(e), buf_pair(e), local_pair(e), slots, nslots, S, 0, nslots > 1 ? S : e->n,
                              e->prec, e->st, e->hyper.outer_lr, e->hyper.outer_momentum, e->n, 0, e->stream);
  launch_p2p_finish(tt_pair(e), local_pair(e), marks, nmarks, e->st, e->n, e->sig_err, e->stream);
  phase_end(e, DLC_PHASE_OUTER);
  launched("nesterov_p2p_piece");
  if (c->kind == 1 && !c->in_world) watch_round(e, c);
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
  PtrList slots{}, marks{};
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
    for (size_t q = 0; q < K; ++q) {
      slots.ptr[q] = gather + q * S * w;
      marks.ptr[q] = e->flags + q;
    }
    nccl_round_commit(e, c, slots, (int)K, S, marks, (int)K, e->stream);
  } else {
    DLC_NCCL(ncclAllReduce(send, send, K * S, nccl_type(e->prec), ncclAvg, c->comm, e->stream));
    if (e->prec == DLC_FP16)
      launch_nonfinite_codes(static_cast<const uint16_t*>(e->send), e->flags, e->n, e->stream);
    else
      launch_nonfinite(static_cast<const float*>(e->send), e->flags, e->n, e->stream);
    launched("nonfinite");
    phase_end(e, DLC_PHASE_COLLECTIVE);
    if (rep) DLC_CUDA(cudaEventRecord(e->ev1, e->stream));
    slots.ptr[0] = send;
    marks.ptr[0] = e->flags;
    nccl_round_commit(e, c, slots, 1, 0, marks, 1, e->stream);
  }
}

// ---- DLC_MODE_P2P: the pipelined outer step, in stages ----------------------
// The rank-ordered owner fold fused with its own data movement over NVLink peer
// memory, pipelined over the pieces of piece_plan() (piece p = the same
// sub-range of every owner slot):
//   main     K2(p) into my send buffer                               -> evK2[p]
//   cstream  [every rank's K2(p) done]; fold(p): the owner pulls piece p of
//            slot r from every rank (TMA bulk copies over NVLink), folds in
//            rank order, pushes the mean + a non-finite mark into slot r of
//            every rank's gather buffer                              -> evB[p]
//   main     [every rank's fold(p) done]; K4(p) speculative into the idle
//            theta_t / momentum; ...; finish (flip ocur when every owner
//            flag is clean)
// The two "every rank" conditions are the only synchronisation.  One process
// per GPU (outer_p2p_pipelined) makes them NVLink flag barriers on the comm
// stream: barrier A_p before fold(p), B_p after it, B_p doubling as A_{p+1}
// once our K2(p+1) is done, plus a commit barrier that exchanges the ranks'
// error bits before the finish gate.  One thread driving every rank
// (world.cu) makes them cudaEvent dependencies between the ranks' streams,
// so any number of ranks may share a device.  The fold keeps a few dozen CTAs,
// so its NVLink time overlaps the HBM-bound K2 / K4 pieces on the other SMs.
// With host buffers (`hsrc` / `hdst`) piece p is also copied in before K2(p)
// and its new theta_t copied out after K4(p).
P2PStep p2p_begin(dlc_engine* e, int rank, const float* src, bool rep, const float* hsrc, float* hdst,
                  int oc_host) {
  P2PStep s;
  s.e = e;
  s.rank = rank;
  s.K = e->k;
  s.S = e->S;
  s.w = elem_width(e->prec);
  s.n = e->n;
  s.hsrc = hsrc;
  s.hdst = hdst;
  s.oc_host = oc_host;
  s.rep = rep;
  if (!e->cstream) {
    int lo = 0, hi = 0;
    DLC_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    DLC_CUDA(cudaStreamCreateWithPriority(&e->cstream, cudaStreamNonBlocking, hi));
  }
  s.pb = piece_plan(s.S, s.n, hsrc != nullptr);
  s.P = s.pb.size() - 1;
  const size_t nev = 4 * s.P + 2;
  while (e->piece_ev.size() < nev) {
    cudaEvent_t ev;
    DLC_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    e->piece_ev.push_back(ev);
  }
  s.evK2 = e->piece_ev.data();
  s.evB = s.evK2 + s.P;
  s.evH = s.evB + s.P;
  s.evK4 = s.evH + s.P;
  s.evStart = s.evK4[s.P];
  s.evCommit = s.evK4[s.P + 1];
  float* sp = const_cast<float*>(src);
  s.tl = sp ? Pair{{sp, sp}} : local_pair(e);
  for (size_t q = 0; q < s.K; ++q) {  // K4 reads the means from the local gather buffer
    s.slots.ptr[q] = static_cast<char*>(e->gather) + q * s.S * s.w;
    s.fl.ptr[q] = e->flags + q;  // owner q's non-finite mark, pushed here by owner q
  }
  if (rep) DLC_CUDA(cudaEventRecord(e->ev0, e->stream));
  // owners push their marks into this array after every rank's K2(0), which
  // follows this memset on every rank
  DLC_CUDA(cudaMemsetAsync(e->flags, 0, kMaxK * sizeof(int), e->stream));
  s.origin = trace_begin(e, e->stream);
  DLC_CUDA(cudaEventRecord(s.evStart, e->stream));
  if (hsrc) {
    ensure_copy_streams(e);
    DLC_CUDA(cudaStreamWaitEvent(e->h2d, s.evStart, 0));  // staging buffer free
  }
  return s;
}

// piece p of every owner slot, clipped to n
template <typename F>
static void piece_rows(const P2PStep& s, size_t p, F&& fn) {
  for (size_t q = 0; q < s.K; ++q) {
    const size_t lo = q * s.S + s.pb[p];
    if (lo >= s.n) break;
    fn(lo, std::min(s.pb[p + 1] - s.pb[p], s.n - lo));
  }
}

void p2p_k2(P2PStep& s, size_t p) {
  dlc_engine* e = s.e;
  if (s.hsrc) {
    float* stage = s.tl.ptr[0];
    piece_rows(s, p, [&](size_t lo, size_t len) {
      DLC_CUDA(cudaMemcpyAsync(stage + lo, s.hsrc + lo, len * sizeof(float), cudaMemcpyHostToDevice, e->h2d));
    });
    DLC_CUDA(cudaEventRecord(s.evH[p], e->h2d));
    DLC_CUDA(cudaStreamWaitEvent(e->stream, s.evH[p], 0));
  }
  cudaEvent_t t0 = trace_begin(e, e->stream);
  launch_pseudo_grad_piece(tt_pair(e), s.tl, e->st, e->send, e->prec, (int)s.K, s.S, s.pb[p], s.pb[p + 1] - s.pb[p],
                           s.n, piece_ctas(), e->stream);
  trace_end(e, e->stream, "K2", (int)p, t0);
  DLC_CUDA(cudaEventRecord(s.evK2[p], e->stream));
}

// Every K2 piece of a device-buffer step; after a fused K1 (the delta is
// already in the send buffer) only the gated fallback, whose completion then
// releases every piece's fold at once.
void p2p_k2_all(P2PStep& s, bool fused) {
  dlc_engine* e = s.e;
  if (!fused) {
    for (size_t p = 0; p < s.P; ++p) p2p_k2(s, p);
    launched("pseudo_grad_piece");
    return;
  }
  cudaEvent_t t0 = trace_begin(e, e->stream);
  launch_pseudo_grad_gated(tt_pair(e), s.tl, e->st, e->send, e->prec, s.n, e->stream);
  launched("pseudo_grad_gated");
  trace_end(e, e->stream, "K2gated", 0, t0);
  for (size_t p = 0; p < s.P; ++p) DLC_CUDA(cudaEventRecord(s.evK2[p], e->stream));
}

void p2p_fold_begin(P2PStep& s) {
  dlc_engine* e = s.e;
  s.c0 = pooled_event(e);
  s.c1 = pooled_event(e);
  DLC_CUDA(cudaStreamWaitEvent(e->cstream, s.evStart, 0));
  DLC_CUDA(cudaEventRecord(s.c0, e->cstream));
}

// The owner fold of piece p on the comm stream (the caller orders it after
// every rank's K2(p)): slot r / piece p of every rank's delta in, the mean and
// the non-finite mark out to every rank.
void p2p_fold(P2PStep& s, size_t p) {
  dlc_engine* e = s.e;
  const size_t K = s.K, S = s.S, w = s.w, po = s.pb[p], plen = s.pb[p + 1] - s.pb[p];
  const int r = s.rank;
  PtrList in{}, outs{}, pfl{};
  for (size_t j = 0; j < K; ++j) {
    in.ptr[j] = static_cast<char*>(e->peer_send[j]) + (r * S + po) * w;
    outs.ptr[j] = static_cast<char*>(e->peer_gather[j]) + (r * S + po) * w;
    pfl.ptr[j] = e->peer_flags[j] + r;
  }
  cudaEvent_t tf = trace_begin(e, e->cstream);
  if (!launch_fold_push_tma(in, (int)K, e->prec, outs, (int)K, pfl, (int)K, plen, tma_ctas(K), tma_threads(K),
                            fold_kernel(), e->cstream))
    launch_fold_push(in, (int)K, e->prec, outs, (int)K, pfl, (int)K, plen, kFoldCtas, e->cstream);
  launched("fold_push");
  trace_end(e, e->cstream, "fold_push", (int)p, tf);
}

void p2p_fold_end(P2PStep& s) {
  dlc_engine* e = s.e;
  DLC_CUDA(cudaEventRecord(s.c1, e->cstream));
  if (e->timing) {
    e->pending.push_back({DLC_PHASE_COLLECTIVE, s.c0, s.c1});
  } else {
    e->pool.push_back(s.c0);
    e->pool.push_back(s.c1);
  }
  if (s.rep) DLC_CUDA(cudaEventRecord(e->ev1, e->cstream));
}

// K4 of piece p on the local gather buffer, speculative into the idle theta_t /
// momentum; ordered after our own evB[p] (the caller adds the other ranks').
void p2p_k4(P2PStep& s, size_t p) {
  dlc_engine* e = s.e;
  DLC_CUDA(cudaStreamWaitEvent(e->stream, s.evB[p], 0));
  cudaEvent_t t4 = trace_begin(e, e->stream);
  // device buffers: each piece is timed on its own (after its wait), so the
  // OUTER phase sums K4's busy time, not the waits for the means
  const bool piece_timing = e->timing && !s.hsrc;
  if (piece_timing) phase_begin(e);
  launch_nesterov_p2p_piece(tt_pair(e), buf_pair(e), local_pair(e), s.slots, (int)s.K, s.S, s.pb[p],
                            s.pb[p + 1] - s.pb[p], e->prec, e->st, e->hyper.outer_lr, e->hyper.outer_momentum, s.n,
                            piece_ctas(), e->stream);
  launched("nesterov_p2p_piece");
  if (piece_timing) phase_end(e, DLC_PHASE_OUTER);
  trace_end(e, e->stream, "K4", (int)p, t4);
  if (s.hdst) {
    DLC_CUDA(cudaEventRecord(s.evK4[p], e->stream));
    DLC_CUDA(cudaStreamWaitEvent(e->d2h, s.evK4[p], 0));
    piece_rows(s, p, [&](size_t lo, size_t len) {
      DLC_CUDA(cudaMemcpyAsync(s.hdst + lo, e->theta_t[s.oc_host ^ 1] + lo, len * sizeof(float),
                               cudaMemcpyDeviceToHost, e->d2h));
    });
  }
}

// The finish gate: flip ocur when every owner's mark is clean; `abort`
// (nullable) = the round failed on some rank, change nothing.
void p2p_finish(P2PStep& s, const int* abort) {
  dlc_engine* e = s.e;
  if (!s.hsrc) phase_begin(e);
  launch_p2p_finish(tt_pair(e), local_pair(e), s.fl, (int)s.K, e->st, s.n, abort, e->stream);
  launched("p2p_finish");
  phase_end(e, DLC_PHASE_OUTER);
  trace_dump(e, s.origin);
}

// One process per GPU: the stages above ordered by NVLink flag barriers.
void outer_p2p_pipelined(dlc_engine* e, dlc_collective* c, const float* src, dlc_reduce_report* rep,
                         const float* hsrc, float* hdst, int oc_host, bool fused) {
  harvest_if_full(e);  // never inside the step: a host wait there could block on a peer's barrier
  p2p_bind(e, c);
  P2PStep s = p2p_begin(e, c->rank, src, rep != nullptr, hsrc, hdst, oc_host);
  const size_t P = s.P;
  // barrier B_p (= A_{p+1} once our K2(p+1) is done) after fold(p); the last
  // one is followed by the commit barrier, which exchanges the error bits so
  // that every rank's finish gate takes the same decision
  auto fold_piece = [&](size_t p) {
    DLC_CUDA(cudaStreamWaitEvent(e->cstream, s.evK2[p], 0));
    if (p == 0) {
      cudaEvent_t ta = trace_begin(e, e->cstream);
      p2p_barrier(e, c, e->cstream, false);  // A_0
      trace_end(e, e->cstream, "barrierA", 0, ta);
    }
    p2p_fold(s, p);
    if (p + 1 < P) DLC_CUDA(cudaStreamWaitEvent(e->cstream, s.evK2[p + 1], 0));
    cudaEvent_t tb = trace_begin(e, e->cstream);
    p2p_barrier(e, c, e->cstream, false);  // B_p
    trace_end(e, e->cstream, "barrierB", (int)p, tb);
    DLC_CUDA(cudaEventRecord(s.evB[p], e->cstream));
    if (p + 1 == P) {
      p2p_barrier(e, c, e->cstream, true);  // commit
      DLC_CUDA(cudaEventRecord(s.evCommit, e->cstream));
    }
  };
  if (!hsrc) {
    // device buffers: every K2 piece first (the folds of the early pieces run
    // beside the later K2 pieces), then the K4 pieces as their means land
    phase_begin(e);
    p2p_k2_all(s, fused);
    phase_end(e, DLC_PHASE_PSEUDO);
    p2p_fold_begin(s);
    for (size_t p = 0; p < P; ++p) fold_piece(p);
    p2p_fold_end(s);
    for (size_t p = 0; p < P; ++p) p2p_k4(s, p);
  } else {
    // host buffers: K2(p+1) then K4(p) on the engine stream, so the D2H of
    // piece p's new theta_t starts while later pieces are still arriving (H2D
    // and D2H overlap on the two copy streams instead of running back to back).
    // Issue order keeps every event recorded before a stream waits on it: the
    // merged barrier after fold(p) waits on K2(p + 1), K4(p) on fold(p).
    p2p_k2(s, 0);
    p2p_fold_begin(s);
    for (size_t p = 0; p < P; ++p) {
      if (p + 1 < P) p2p_k2(s, p + 1);
      fold_piece(p);
      p2p_k4(s, p);
    }
    launched("pseudo_grad_piece");
    p2p_fold_end(s);
  }
  DLC_CUDA(cudaStreamWaitEvent(e->stream, s.evCommit, 0));
  p2p_finish(s, e->sig_err);
}

// DLC_MODE_ALLREDUCE, pipelined: ncclAllReduce(ncclAvg) of contiguous pieces of
// the flat pseudo-gradient on the high-priority comm stream, overlapped with
// K2 of the next piece and the speculative K4 of the previous one:
//   main     K2(p) -> evK2[p]
//   cstream  wait evK2[p]; ncclAllReduce(piece p, in place); non-finite(p) -> evB[p]
//   main     wait evB[p]; K4(p) into the idle theta_t / momentum; ...; finish
// (measured 9.66 ms against 11.2 ms for the unpipelined K2 -> all-reduce -> K4
// of outer_collective at 4 GPUs, profiles/r1_bench_4gpu_allreduce*.json)
void outer_allreduce_pipelined(dlc_engine* e, dlc_collective* c, const float* src, dlc_reduce_report* rep,
                               bool fused) {
  harvest_if_full(e);
  const size_t n = e->n, w = elem_width(e->prec);
  if (!e->cstream) {
    int lo = 0, hi = 0;
    DLC_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    DLC_CUDA(cudaStreamCreateWithPriority(&e->cstream, cudaStreamNonBlocking, hi));
  }
  std::vector<size_t> pb = piece_plan((n + 511) / 512 * 512, n);  // contiguous pieces of [0, n)
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
  if (fused) {  // the delta is in the send buffer already (fused K1), the gated K2 covers an overflow
    launch_pseudo_grad_gated(tt_pair(e), tl, e->st, e->send, e->prec, n, e->stream);
    launched("pseudo_grad_gated");
  }
  for (size_t p = 0; p < P; ++p) {  // k = 1: piece p is the contiguous range [pb[p], pb[p+1])
    if (!fused)
      launch_pseudo_grad_piece(tt_pair(e), tl, e->st, e->send, e->prec, 1, 0, pb[p], pb[p + 1] - pb[p], n, 0,
                               e->stream);
    DLC_CUDA(cudaEventRecord(evK2[p], e->stream));
  }
  if (!fused) launched("pseudo_grad_piece");
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
  // the commit gate's error OR on the comm stream after the last piece, then
  // K4 of every piece as its mean lands, the finish and the watch
  nccl_error_or(e, c, e->cstream);
  cudaEvent_t evErr = pooled_event(e);
  DLC_CUDA(cudaEventRecord(evErr, e->cstream));
  phase_begin(e);
  for (size_t p = 0; p < P; ++p) {
    DLC_CUDA(cudaStreamWaitEvent(e->stream, evB[p], 0));
    launch_nesterov_p2p_piece(tt_pair(e), buf_pair(e), local_pair(e), slots, 1, 0, pb[p], pb[p + 1] - pb[p],
                              e->prec, e->st, e->hyper.outer_lr, e->hyper.outer_momentum, n, 0, e->stream);
  }
  DLC_CUDA(cudaStreamWaitEvent(e->stream, evErr, 0));
  e->pool.push_back(evErr);
  launch_p2p_finish(tt_pair(e), local_pair(e), fl, 1, e->st, n, e->sig_err, e->stream);
  phase_end(e, DLC_PHASE_OUTER);
  launched("nesterov_p2p_piece");
  if (!c->in_world) watch_round(e, c);
}

void outer_round(dlc_engine* e, dlc_collective* c, const float* src, dlc_reduce_report* rep) {
  const bool fused = take_fused_delta(e) && !src;  // an explicit theta_local source needs the full K2
  if (e->k > 1 && c->mode == DLC_MODE_P2P) {  // manages its own flag (read remotely by peers)
    outer_p2p_pipelined(e, c, src, rep, nullptr, nullptr, 0, fused);
    return;
  }
  if (e->k > 1 && c->mode == DLC_MODE_ALLREDUCE) {
    outer_allreduce_pipelined(e, c, src, rep, fused);
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
  pseudo_grad_step(e, s ? Pair{{s, s}} : local_pair(e), fused);
  outer_collective(e, c, rep);
}

}  // namespace dlc
