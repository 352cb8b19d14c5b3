// world.cu — the single-process multi-GPU world (dlc_world_*): K engines on
// K GPUs driven by one host thread.
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

using namespace dlc;

// ---- single-process multi-GPU world (include/diloco_cuda.h section 3) ----------

struct dlc_world {
  int k = 0;
  int mode = DLC_MODE_P2P;
  std::vector<int> devices;
  std::vector<dlc_engine*> engines;
  std::vector<dlc_collective*> colls;
  std::vector<int> members;  // original rank of each current rank (dlc_world_shrink)
};

namespace {

// Every engine's peer tables point straight at the other engines' buffers
// (one address space; peer access enabled between distinct devices, ranks on
// the same device read each other's buffers as local memory): no IPC, no
// handle exchange, no signal slots.
void world_bind_p2p(dlc_world* w) {
  for (int a = 0; a < w->k; ++a) {
    DeviceGuard dg(w->devices[a]);
    for (int b = 0; b < w->k; ++b) {
      if (w->devices[a] == w->devices[b]) continue;
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
    p2p_unbind(e);
    for (int j = 0; j < w->k; ++j) {
      dlc_engine* q = w->engines[j];
      e->peer_send[j] = q->send;
      e->peer_gather[j] = q->gather;
      e->peer_flags[j] = q->flags;
    }
    e->p2p_bound = w->colls[r];
    w->colls[r]->bound.push_back(e);
  }
}

// DLC_MODE_P2P from one thread: every rank's staged step (p2p.cu), the
// "every rank" conditions as cudaEvent dependencies between the ranks'
// streams instead of flag barriers.  Nothing spins, so ranks may share a
// device (the driver's one-GPU box runs any K), and a stream never waits on
// an event that is not recorded yet: each stage is enqueued for every rank
// before the next stage waits on it.
//   fold_r(p) waits for K2_j(p) of every rank j (owner r reads slot r of
//             every rank's send buffer);
//   K4_r(p)   waits for fold_j(p) of every rank j (owner j pushed its mean
//             and mark into rank r's gather buffer and flags).
// The next step's K2 / flag reset on rank j follow rank j's K4 pieces on its
// stream, hence every fold of this step: no buffer is rewritten early.
void world_outer_p2p(dlc_world* w) {
  const int K = w->k;
  std::vector<P2PStep> st;
  st.reserve(K);
  for (int r = 0; r < K; ++r) {
    DeviceGuard dg(w->devices[r]);
    dlc_engine* e = w->engines[r];
    harvest_if_full(e);
    if (e->p2p_bound != w->colls[r]) world_bind_p2p(w);
    st.push_back(p2p_begin(e, r, nullptr, false, nullptr, nullptr, 0));
  }
  const size_t P = st[0].P;
  for (int r = 0; r < K; ++r) {
    DeviceGuard dg(w->devices[r]);
    dlc_engine* e = w->engines[r];
    phase_begin(e);
    p2p_k2_all(st[r], take_fused_delta(e));
    phase_end(e, DLC_PHASE_PSEUDO);
    p2p_fold_begin(st[r]);
  }
  for (size_t p = 0; p < P; ++p) {
    for (int r = 0; r < K; ++r) {
      DeviceGuard dg(w->devices[r]);
      dlc_engine* e = w->engines[r];
      for (int j = 0; j < K; ++j) DLC_CUDA(cudaStreamWaitEvent(e->cstream, st[j].evK2[p], 0));
      p2p_fold(st[r], p);
      DLC_CUDA(cudaEventRecord(st[r].evB[p], e->cstream));
    }
  }
  for (int r = 0; r < K; ++r) {
    DeviceGuard dg(w->devices[r]);
    p2p_fold_end(st[r]);
  }
  for (size_t p = 0; p < P; ++p) {
    for (int r = 0; r < K; ++r) {
      DeviceGuard dg(w->devices[r]);
      dlc_engine* e = w->engines[r];
      for (int j = 0; j < K; ++j)
        if (j != r) DLC_CUDA(cudaStreamWaitEvent(e->stream, st[j].evB[p], 0));
      p2p_k4(st[r], p);
    }
  }
  for (int r = 0; r < K; ++r) {
    DeviceGuard dg(w->devices[r]);
    p2p_finish(st[r], nullptr);
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
    pseudo_grad_step(e, local_pair(e), take_fused_delta(e));
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
    for (int r = 0; r < k; ++r) w->members.push_back(r);
    for (int r = 0; r < k; ++r) {
      dlc_engine* e = nullptr;
      const int s2 = dlc_engine_create(cfg, hyper, n_params, devices[r], inner_mode, &e);
      if (s2 != DLC_OK) fail(s2, std::string("world engine ") + std::to_string(r) + ": " + dlc_last_error());
      w->engines.push_back(e);
    }
    // P2P synchronises the ranks with events, so ranks may share a device;
    // NCCL communicators need one device per rank
    bool shared = false;
    for (int r = 1; r < k; ++r)
      for (int q = 0; q < r; ++q) shared |= devices[q] == devices[r];
    if (shared && mode != DLC_MODE_P2P)
      fail(DLC_ECONFIG, "world ranks sharing a device need DLC_MODE_P2P (NCCL needs one device per rank)");
    std::vector<ncclComm_t> comms(k, nullptr);
    if (k > 1 && mode != DLC_MODE_P2P) DLC_NCCL(ncclCommInitAll(comms.data(), k, devices));  // P2P needs none
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
      p2p_unbind(e);  // direct pointers: nothing to unmap, no fleet barrier
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

int dlc_world_shrink(dlc_world* w, const int* exclude_ranks, size_t n_exclude, size_t quorum_min) {
  return guard([&] {
    if (!w || (n_exclude && !exclude_ranks)) fail(DLC_EINVAL, "dlc_world_shrink: null argument");
    std::vector<int> ex(exclude_ranks, exclude_ranks + n_exclude);
    std::sort(ex.begin(), ex.end());
    ex.erase(std::unique(ex.begin(), ex.end()), ex.end());
    for (int r : ex)
      if (r < 0 || r >= w->k) fail(DLC_ECONFIG, "dlc_world_shrink: rank " + std::to_string(r) + " not in the world");
    const int k2 = w->k - (int)ex.size();
    if ((size_t)k2 < std::max<size_t>(quorum_min, 1))  // collective.cpp:1376-1378
      fail(DLC_EQUORUM, "contributor set below quorum");
    for (dlc_engine* e : w->engines)  // engine.cpp:116-120: membership changes between rounds
      if (e->issued_inner % e->cfg.local_steps_h != 0) fail(DLC_EINVAL, "dlc_world_shrink: mid-window");
    if (ex.empty()) return;
    for (int r = 0; r < w->k; ++r) {  // nothing in flight on any rank
      DeviceGuard dg(w->devices[r]);
      DLC_CUDA(cudaDeviceSynchronize());
    }
    std::vector<dlc_engine*> engines;
    std::vector<int> devices, members;
    for (int r = 0; r < w->k; ++r) {
      if (std::binary_search(ex.begin(), ex.end(), r)) continue;
      engines.push_back(w->engines[r]);
      devices.push_back(w->devices[r]);
      members.push_back(w->members[r]);
    }
    // the survivors' communicators first: if that fails, the world is unchanged
    std::vector<ncclComm_t> comms(k2, nullptr);
    if (k2 > 1 && w->mode != DLC_MODE_P2P) DLC_NCCL(ncclCommInitAll(comms.data(), k2, devices.data()));
    for (int r = 0; r < w->k; ++r) {
      p2p_unbind(w->engines[r]);  // before their collectives go away (unbind edits the collective's list)
      if (std::binary_search(ex.begin(), ex.end(), r)) dlc_engine_destroy(w->engines[r]);
    }
    for (size_t r = 0; r < w->colls.size(); ++r) {
      DeviceGuard dg(w->devices[r]);
      if (w->colls[r]->comm) ncclCommDestroy(w->colls[r]->comm);
      delete w->colls[r];
    }
    w->colls.clear();
    w->engines = engines;
    w->devices = devices;
    w->members = members;
    w->k = k2;
    for (int r = 0; r < k2; ++r) {
      auto* c = new dlc_collective();
      c->kind = k2 > 1 ? 1 : 0;
      c->rank = r;
      c->world = k2;
      c->device = w->devices[r];
      c->mode = w->mode;
      c->comm = comms[r];
      c->in_world = true;
      c->shrunk = true;
      for (int j = 0; j < k2; ++j) c->members[j] = w->members[j];
      w->colls.push_back(c);
    }
    for (dlc_engine* e : w->engines) {
      DeviceGuard dg(e->device);
      relayout(e, (size_t)k2);  // survivor slots and divisor
    }
    if (k2 > 1 && w->mode == DLC_MODE_P2P) world_bind_p2p(w);
  });
}

size_t dlc_world_members(const dlc_world* w, int* ranks, size_t cap) {
  if (!w) return 0;
  for (size_t i = 0; i < w->members.size() && i < cap && ranks; ++i) ranks[i] = w->members[i];
  return w->members.size();
}

int dlc_world_outer_step(dlc_world* w, dlc_outer_result* result) {
  return guard([&] {
    if (!w) fail(DLC_EINVAL, "dlc_world_outer_step: null world");
    for (int r = 0; r < w->k; ++r) check_collective(w->engines[r], w->k > 1 ? w->colls[r] : nullptr);
    if (w->k == 1) {
      DeviceGuard dg(w->devices[0]);
      outer_round(w->engines[0], nullptr, nullptr, nullptr);
    } else if (w->mode == DLC_MODE_P2P) {
      world_outer_p2p(w);
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
