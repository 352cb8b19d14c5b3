// internal.hpp — status/error plumbing shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <string>

#include "../../include/diloco_cuda.h"

namespace dlc {

// Thread-local message behind dlc_last_error().
void set_error(const std::string& msg);
void clear_error();

// Carries a status through C++ code; converted to an int at the C boundary.
struct Failure {
  int status;
  std::string msg;
};

[[noreturn]] inline void fail(int status, const std::string& msg) { throw Failure{status, msg}; }

inline void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(DLC_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

inline void check_nccl(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(DLC_ENCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

#define DLC_CUDA(expr) ::dlc::check_cuda((expr), #expr)
#define DLC_NCCL(expr) ::dlc::check_nccl((expr), #expr)
// Launch-error check right after a kernel launch.
#define DLC_LAUNCHED(what) ::dlc::check_cuda(cudaGetLastError(), what)

// Runs f() and converts a Failure / std::exception into a status code.
template <typename F>
int guard(F&& f) {
  try {
    f();
    return DLC_OK;
  } catch (const Failure& x) {
    set_error(x.msg);
    return x.status;
  } catch (const std::exception& x) {
    set_error(x.what());
    return DLC_ECUDA;
  }
}

// wire.cu: the reference's reduce-chunk framing from / into device memory
void wire_encode_impl(const void* dev, uint64_t global_offset, uint64_t elems, const dlc_wire_tags* t,
                      uint8_t* host_out, size_t cap, size_t* used, cudaStream_t stream);
void wire_decode_impl(const uint8_t* in, size_t bytes, int precision, uint64_t base, uint64_t capacity, void* dev_out,
                      dlc_wire_chunk* chunks, size_t max_chunks, size_t* n_chunks, size_t* consumed,
                      cudaStream_t stream);

}  // namespace dlc
