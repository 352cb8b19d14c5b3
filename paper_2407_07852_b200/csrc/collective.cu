// collective.cu — section 2 of include/diloco_cuda.h: the collective plugin
// (class Collective, reduce.hpp:86-97) over NCCL, and its host-buffer
// all_reduce_avg.
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
