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
    uint64_t sig_epoch;
  };
  Handles mine;
  mine.sig_epoch = e->sig_epoch;
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
bool flag_barriers(const dlc_collective* c) {
  const char* b = std::getenv("DLC_P2P_BARRIER");
  return !(b && std::string(b) == "nccl" && !c->in_world);  // (one thread drives a world: flags only)
}

void p2p_barrier(dlc_engine* e, dlc_collective* c, cudaStream_t s) {
  if (!flag_barriers(c)) {
    DLC_NCCL(ncclAllReduce(e->barrier_buf, e->barrier_buf, 1, ncclInt32, ncclSum, c->comm, s));
    return;
  }
  PtrList remote{};
  for (size_t j = 0; j < e->k; ++j) remote.ptr[j] = e->peer_sig[j] + c->rank;
  e->sig_epoch += 1;
  const bool stall = c->stall_at >= 0 && c->barriers >= c->stall_at;
  c->barriers += 1;
  launch_flag_barrier(remote, e->sig, (int)e->k, c->rank, e->sig_epoch, e->sig_err, c->timeout_ms * 1000000ull, stall,
                      s);
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
  }
  if (!p2p_mover_sm() && !e->pull[0]) {  // copy-engine mover: one pull and one gather stream per peer
    for (size_t j = 0; j < K; ++j) {
      DLC_CUDA(cudaStreamCreateWithFlags(&e->pull[j], cudaStreamNonBlocking));
      DLC_CUDA(cudaStreamCreateWithFlags(&e->gath[j], cudaStreamNonBlocking));
    }
  }
  const std::vector<size_t> pb = piece_plan(S, n, hsrc != nullptr);  // piece boundaries inside a slot
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
  const bool sm_mover = p2p_mover_sm();
  const bool push2 = p2p_mover_push2();
  const bool k4_pull = sm_mover && p2p_k4_pull();
  const bool merge = p2p_merge_barriers();
  cudaEvent_t* evS = evA;  // (evA is only used by the copy-engine mover)
  auto k2_piece = [&](size_t p) {
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
  };
  auto scatter_piece = [&](size_t p) {
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
  };
  auto fold_piece = [&](size_t p) {
    if (sm_mover) {
      // SM mover: a persistent fold kernel on a few CTAs pulls slot r / piece p of
      // every rank's delta and pushes the mean (and a non-finite mark) into slot r
      // of every rank's gather buffer (flags reset by each rank before its K2(0)).
      DLC_CUDA(cudaStreamWaitEvent(e->cstream, push2 ? evS[p] : evK2[p], 0));
      if (!merge || p == 0) {
        cudaEvent_t ta = trace_begin(e, e->cstream);
        p2p_barrier(e, c, e->cstream);  // A_p
        trace_end(e, e->cstream, "barrierA", (int)p, ta);
      }
      PtrList in{}, outs{}, pfl{};
      for (size_t j = 0; j < K; ++j) {
        in.ptr[j] = (int)j == r && push2 ? send + (r * S + po(p)) * w  // own row stays local
                    : (push_mover || push2) ? recv + (j * S + po(p)) * w   // rows already pushed here
                                            : static_cast<char*>(e->peer_send[j]) + (r * S + po(p)) * w;
        outs.ptr[j] = static_cast<char*>(e->peer_gather[j]) + (r * S + po(p)) * w;
        pfl.ptr[j] = e->peer_flags[j] + r;
      }
      cudaEvent_t tf = trace_begin(e, e->cstream);
      // K4 pull: the mean stays in the owner's own gather slot; every rank's K4
      // reads it from there over NVLink (no remote stores of means)
      const int nout = k4_pull ? 1 : (int)K;
      if (k4_pull) outs.ptr[0] = gather + (r * S + po(p)) * w;
      if (!(fold_tma() && launch_fold_push_tma(in, (int)K, e->prec, outs, nout, pfl, (int)K, pl(p), tma_ctas(K),
                                               e->cstream)))
        launch_fold_push(in, (int)K, e->prec, outs, nout, pfl, (int)K, pl(p), comm_ctas(), e->cstream);
      trace_end(e, e->cstream, "fold_push", (int)p, tf);
      // merged barriers: B_p also serves as A_{p+1} once our K2(p+1) is done
      // (it precedes K4(p) on the main stream anyway, so K4(p) waits no longer)
      if (merge && p + 1 < P) DLC_CUDA(cudaStreamWaitEvent(e->cstream, push2 ? evS[p + 1] : evK2[p + 1], 0));
      cudaEvent_t tb = trace_begin(e, e->cstream);
      p2p_barrier(e, c, e->cstream);  // B_p
      trace_end(e, e->cstream, "barrierB", (int)p, tb);
      DLC_CUDA(cudaEventRecord(evB[p], e->cstream));
      return;
    }
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
  };
  // K4 pieces on the local gather buffer, speculative into the idle theta_t / momentum
  PtrList slots{}, fl{};
  for (size_t q = 0; q < K; ++q) {
    slots.ptr[q] = k4_pull ? static_cast<char*>(e->peer_gather[q]) + q * S * w : gather + q * S * w;
    // SM mover: owners pushed their marks into my flag array; CE mover: owner
    // q's flag lives in owner q's memory
    fl.ptr[q] = sm_mover ? e->flags + q : e->peer_flags[q] + q;
  }
  auto k4_piece = [&](size_t p) {
    DLC_CUDA(cudaStreamWaitEvent(e->stream, evB[p], 0));
    for (size_t q = 0; q < K && !sm_mover; ++q)
      if ((int)q != r) DLC_CUDA(cudaStreamWaitEvent(e->stream, evGath[q * P + p], 0));
    cudaEvent_t t4 = trace_begin(e, e->stream);
    // device buffers: time each piece's launch on its own (after its wait), so
    // the OUTER phase sums K4's busy time, not the waits for the means
    const bool piece_timing = e->timing && !hsrc;
    if (piece_timing) phase_begin(e);
    launch_nesterov_p2p_piece(tt_pair(e), buf_pair(e), local_pair(e), slots, (int)K, S, po(p), pl(p), e->prec, e->st,
                              lr, mu, n, piece_ctas(), e->stream);
    if (piece_timing) phase_end(e, DLC_PHASE_OUTER);
    trace_end(e, e->stream, "K4", (int)p, t4);
    if (hdst) {
      DLC_CUDA(cudaEventRecord(evK4[p], e->stream));
      DLC_CUDA(cudaStreamWaitEvent(e->d2h, evK4[p], 0));
      rows(p, [&](size_t lo, size_t len) {
        DLC_CUDA(cudaMemcpyAsync(hdst + lo, e->theta_t[oc_host ^ 1] + lo, len * sizeof(float),
                                 cudaMemcpyDeviceToHost, e->d2h));
      });
    }
  };
  cudaEvent_t c0 = pooled_event(e), c1 = pooled_event(e);
  auto fold_begin = [&] {
    DLC_CUDA(cudaStreamWaitEvent(e->cstream, evStart, 0));
    DLC_CUDA(cudaEventRecord(c0, e->cstream));
  };
  auto fold_end = [&] {
    launched("fold_p2p");
    DLC_CUDA(cudaEventRecord(c1, e->cstream));
    if (e->timing) {
      e->pending.push_back({DLC_PHASE_COLLECTIVE, c0, c1});
    } else {
      e->pool.push_back(c0);
      e->pool.push_back(c1);
    }
    if (rep) DLC_CUDA(cudaEventRecord(e->ev1, e->cstream));
  };
  const char* il = std::getenv("DLC_P2P_INTERLEAVE");  // device buffers: A/B knob (default 0)
  if (!hsrc && !(il && il[0] == '1')) {
    // device buffers: every K2 piece first (the folds of the early pieces run
    // beside the later K2 pieces), then the K4 pieces as their means land
    phase_begin(e);
    for (size_t p = 0; p < P; ++p) k2_piece(p);
    launched("pseudo_grad_piece");
    phase_end(e, DLC_PHASE_PSEUDO);
    fold_begin();
    for (size_t p = 0; p < P && push2; ++p) scatter_piece(p);
    for (size_t p = 0; p < P; ++p) fold_piece(p);
    fold_end();
    for (size_t p = 0; p < P; ++p) k4_piece(p);
    phase_begin(e);  // the finish gate below is one more OUTER interval
  } else {
    // host buffers: K2(p+1) then K4(p) on the engine stream, so the D2H of
    // piece p's new theta_t starts while later pieces are still arriving (H2D
    // and D2H overlap on the two copy streams instead of running back to back).
    // Issue order keeps every event recorded before a stream waits on it: the
    // merged barrier after fold(p) waits on K2(p + 1), K4(p) on fold(p).
    phase_begin(e);
    k2_piece(0);
    if (push2) scatter_piece(0);
    fold_begin();
    for (size_t p = 0; p < P; ++p) {
      if (p + 1 < P) {
        k2_piece(p + 1);
        if (push2) scatter_piece(p + 1);
      }
      fold_piece(p);
      k4_piece(p);
    }
    launched("pseudo_grad_piece");
    fold_end();
  }
  launch_p2p_finish(tt_pair(e), local_pair(e), fl, (int)K, e->st, n, flag_barriers(c) ? e->sig_err : nullptr,
                    e->stream);
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
  launch_p2p_finish(tt_pair(e), local_pair(e), fl, 1, e->st, n, nullptr, e->stream);
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

}  // namespace dlc
