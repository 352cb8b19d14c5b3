// wire_engine.cu — the engine side of the cross-box wire codec (section 5 of
// include/diloco_cuda.h; the framing itself is wire.cu).
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
    stream_wait(e);
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
    e->delta_fused = false;  // the wire round decodes the means into the send buffer
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
    stream_wait(e);
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
