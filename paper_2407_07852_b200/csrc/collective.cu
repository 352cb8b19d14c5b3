// collective.cu — section 2 of include/diloco_cuda.h: the collective plugin
// (class Collective, reduce.hpp:86-97) over NCCL, and its host-buffer
// all_reduce_avg.
#include <chrono>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <map>
#include <string>
#include <vector>

#include "engine_impl.hpp"

using namespace dlc;

extern "C" {

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
    for (int i = 0; i < world && i < kMaxK; ++i) c->members[i] = i;
    *out = c;
  });
}

// Membership change.  The reference's barrier picks the
// round's contributors from the live members minus the suspects, checks the
// quorum, renumbers them in sorted order and divides by their count
// (collective.cpp:1369-1395).  On one NVLink box the same step is an
// ncclCommShrink of the communicator: the survivors call it, the excluded
// ranks do not, NCCL keeps the survivors' relative order, and the engines
// re-lay their owner slots for the new fleet at their next outer step.
int dlc_collective_shrink(dlc_collective* c, const int* exclude_ranks, size_t n_exclude, size_t quorum_min,
                          int flags, dlc_collective** out) {
  return guard([&] {
    if (!c || !out || (n_exclude && !exclude_ranks)) fail(DLC_EINVAL, "dlc_collective_shrink: null argument");
    *out = nullptr;
    if (c->kind != 1) fail(DLC_ECONFIG, "dlc_collective_shrink: only an NCCL collective has a membership");
    if (c->in_world) fail(DLC_ECONFIG, "dlc_collective_shrink: a dlc_world's collectives are fixed");
    if (flags != DLC_SHRINK_DEFAULT && flags != DLC_SHRINK_ABORT) fail(DLC_ECONFIG, "unknown shrink flags");
    std::vector<int> ex(exclude_ranks, exclude_ranks + n_exclude);
    std::sort(ex.begin(), ex.end());
    ex.erase(std::unique(ex.begin(), ex.end()), ex.end());
    for (int r : ex)
      if (r < 0 || r >= c->world) fail(DLC_ECONFIG, "dlc_collective_shrink: rank " + std::to_string(r) + " not in the world");
    if (std::binary_search(ex.begin(), ex.end(), c->rank)) {  // collective.cpp:1382-1386
      c->broken = true;
      fail(DLC_ECOLLECTIVE, "excluded from round");
    }
    const int survivors = c->world - (int)ex.size();
    if ((size_t)survivors < std::max<size_t>(quorum_min, 1))  // collective.cpp:1376-1378
      fail(DLC_EQUORUM, "contributor set below quorum");
    DeviceGuard dg(c->device);
    auto* n = new dlc_collective();
    n->kind = 1;
    n->device = c->device;
    n->mode = c->mode;
    n->timeout_ms = c->timeout_ms;
    n->shrunk = true;
    const ncclResult_t r = ncclCommShrink(c->comm, ex.data(), (int)ex.size(), &n->comm, nullptr,
                                          flags == DLC_SHRINK_ABORT ? NCCL_SHRINK_ABORT : NCCL_SHRINK_DEFAULT);
    if (r != ncclSuccess) {
      delete n;
      fail(DLC_ENCCL, std::string("ncclCommShrink: ") + ncclGetErrorString(r));
    }
    int nr = -1, nw = 0;
    ncclCommUserRank(n->comm, &nr);
    ncclCommCount(n->comm, &nw);
    int j = 0;
    for (int i = 0; i < c->world; ++i)
      if (!std::binary_search(ex.begin(), ex.end(), i)) n->members[j++] = c->members[i];
    const int want = c->rank - (int)(std::lower_bound(ex.begin(), ex.end(), c->rank) - ex.begin());
    if (nw != survivors || nr != want) {
      ncclCommAbort(n->comm);
      delete n;
      fail(DLC_ENCCL, "ncclCommShrink: unexpected rank " + std::to_string(nr) + " of " + std::to_string(nw));
    }
    n->rank = nr;
    n->world = nw;
    c->broken = true;  // its peers are gone: destroying it must not wait for them
    cudaStreamCreateWithFlags(&n->stream, cudaStreamNonBlocking);
    *out = n;
  });
}

size_t dlc_collective_members(const dlc_collective* c, int* ranks, size_t cap) {
  if (!c) return 0;
  const size_t w = c->kind == 1 ? (size_t)c->world : 1;
  for (size_t i = 0; i < w && i < cap && ranks; ++i) ranks[i] = c->kind == 1 ? c->members[i] : 0;
  return w;
}

int dlc_collective_set_reduce_timeout_ms(dlc_collective* c, uint64_t ms) {
  return guard([&] {
    if (!c) fail(DLC_EINVAL, "dlc_collective_set_reduce_timeout_ms: null collective");
    if (ms == 0) fail(DLC_ECONFIG, "reduce_timeout_ms must be > 0");
    c->timeout_ms = ms;
  });
}

int dlc_collective_inject_stall(dlc_collective* c, int64_t barrier_index) {
  return guard([&] {
    if (!c) fail(DLC_EINVAL, "dlc_collective_inject_stall: null collective");
    c->stall_at = barrier_index < 0 ? -1 : c->barriers + barrier_index;
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
    // engines still bound to it lose their peer mappings (no fleet barrier:
    // the communicator is going away; their next P2P step binds again)
    while (!c->bound.empty()) {
      dlc_engine* e = c->bound.back();
      DeviceGuard dg(e->device);
      cudaStreamSynchronize(e->stream);
      if (e->cstream) cudaStreamSynchronize(e->cstream);
      p2p_unbind(e);  // removes e from c->bound
    }
    while (!c->watchers.empty()) unwatch(c->watchers.back());
    if (c->kind == 1) {
      DeviceGuard dg(c->device);
      if (c->stream) cudaStreamDestroy(c->stream);
      if (c->broken)
        ncclCommAbort(c->comm);  // some peers are gone: do not wait for them
      else
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
      if (c->world > 1) {
        report->data_bytes_sent = dlc_per_peer_reduce_bytes(n, c->world, c->rank, precision);
        report->data_bytes_received = per_peer_reduce_bytes_received(n, c->world, c->rank, precision);
        const uint64_t S = (((n + c->world - 1) / c->world) + 63) / 64 * 64;
        report->wire_bytes_sent = report->wire_bytes_received =
            2ull * (c->world - 1) * S * (precision == DLC_FP16 ? 2 : 4);
      }
      report->wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
  });
}

}  // extern "C"
