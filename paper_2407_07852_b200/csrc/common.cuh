// common.cuh — device helpers shared by the DiLoCo hot-path kernels (sm_100a).
//
// Bitwise parity rules (SURVEY.md §7 "Hard parts", Appendix A): the reference
// is built with -ffp-contract=off (proj/CMakeLists.txt:18), so every FP32
// product/sum here is an explicitly rounded __fmul_rn/__fadd_rn/__fsub_rn (never
// contracted into an FFMA), division is IEEE __fdiv_rn and sqrt is IEEE
// __fsqrt_rn.  The library is additionally compiled with -fmad=false.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace dlc {

constexpr int kThreads = 256;  // 8 warps per CTA

// ---- streaming 128-bit global access --------------------------------------
// Every byte of the optimizer state is touched once per launch and the vectors
// are far larger than L2 (4.4 GB each at 1.1B params), so loads and stores use
// the evict-first streaming hint (.cs) to keep L2 for the reduction buffers.
__device__ __forceinline__ float4 ld_stream(const float4* p) { return __ldcs(p); }
__device__ __forceinline__ void st_stream(float4* p, float4 v) { __stcs(p, v); }
__device__ __forceinline__ uint2 ld_stream(const uint2* p) { return __ldcs(p); }
__device__ __forceinline__ void st_stream(uint2* p, uint2 v) { __stcs(p, v); }
__device__ __forceinline__ uint4 ld_stream(const uint4* p) { return __ldcs(p); }
__device__ __forceinline__ void st_stream(uint4* p, uint4 v) { __stcs(p, v); }

// The exchange's FP16 / FP32 delta stores (K2 pieces) and the mean loads (K4
// pieces).  DLC_EXCHANGE_L2 (an A/B build, tools/): default caching, so a
// piece may still sit in L2 when the owners pull it / after the owners pushed it.
#ifdef DLC_EXCHANGE_L2
__device__ __forceinline__ void st_exchange(float4* p, float4 v) { *p = v; }
__device__ __forceinline__ void st_exchange(uint2* p, uint2 v) { *p = v; }
__device__ __forceinline__ float4 ld_exchange(const float4* p) { return *p; }
__device__ __forceinline__ uint2 ld_exchange(const uint2* p) { return *p; }
#else
__device__ __forceinline__ void st_exchange(float4* p, float4 v) { st_stream(p, v); }
__device__ __forceinline__ void st_exchange(uint2* p, uint2 v) { st_stream(p, v); }
__device__ __forceinline__ float4 ld_exchange(const float4* p) { return ld_stream(p); }
__device__ __forceinline__ uint2 ld_exchange(const uint2* p) { return ld_stream(p); }
#endif

__device__ __forceinline__ bool finite_f(float x) {
  return (__float_as_uint(x) & 0x7F800000u) != 0x7F800000u;
}

// ---- binary16 codec, bit-identical to proj/src/fp16.cpp:25-85 ---------------
// Encode: cvt.rn.f16.f32 is IEEE round-to-nearest-even with overflow to
// +/-inf and gradual underflow, which is exactly fp16_encode for every non-NaN
// input (fp16.cpp:36-62; pinned exhaustively over all 2^32 inputs by
// tests/test_gpu_parity.py::test_fp16_encode_exhaustive).  NaN inputs map to
// sign|0x7E00 as in fp16.cpp:30-35 (the hardware would give 0x7FFF).
__device__ __forceinline__ uint16_t fp16_encode(float x) {
  const uint32_t u = __float_as_uint(x);
  uint16_t h = __half_as_ushort(__float2half_rn(x));
  if ((u & 0x7FFFFFFFu) > 0x7F800000u) h = (uint16_t)(((u >> 16) & 0x8000u) | 0x7E00u);
  return h;
}

// Decode: exact widening.  NaN payloads follow fp16.cpp:79-81
// (sign | 0x7FC00000 | mant << 13) rather than the hardware's canonical NaN.
__device__ __forceinline__ float fp16_decode(uint16_t h) {
  const uint32_t e = h & 0x7C00u;
  if (e == 0x7C00u && (h & 0x3FFu)) {
    return __uint_as_float(((uint32_t)(h & 0x8000u) << 16) | 0x7FC00000u | ((uint32_t)(h & 0x3FFu) << 13));
  }
  return __half2float(__ushort_as_half(h));
}

__device__ __forceinline__ bool fp16_nonfinite(uint16_t h) { return (h & 0x7C00u) == 0x7C00u; }

// Pack / unpack 4 codes <-> uint2 and 8 codes <-> uint4.
__device__ __forceinline__ uint32_t pack2(uint16_t a, uint16_t b) { return (uint32_t)a | ((uint32_t)b << 16); }
__device__ __forceinline__ uint16_t lo16(uint32_t w) { return (uint16_t)(w & 0xFFFFu); }
__device__ __forceinline__ uint16_t hi16(uint32_t w) { return (uint16_t)(w >> 16); }

// ---- the mean's division, reduce.cpp:43 (acc / (float)K) --------------------
// For K a power of two, 1/K is exact, and RN(acc * 2^-m) is the same real value
// as RN(acc / 2^m) rounded once: bit-identical for every finite, infinite and
// subnormal result (NaNs stay NaNs; payloads compare by class), at
// one FMUL instead of the IEEE division sequence.  Other K divide.
struct MeanDiv {
  float divisor, inv;  // inv = 1/K for power-of-two K, else 0
};
__host__ __device__ inline MeanDiv mean_div(int k) {
  return MeanDiv{(float)k, (k > 0 && (k & (k - 1)) == 0) ? 1.0f / (float)k : 0.0f};
}
__device__ __forceinline__ float div_mean(float acc, const MeanDiv& d) {
  return d.inv != 0.0f ? __fmul_rn(acc, d.inv) : __fdiv_rn(acc, d.divisor);
}

// Block-wide OR of a predicate, then one atomicOr per CTA into *flag.
__device__ __forceinline__ void block_or_flag(bool pred, int* flag) {
  const int any = __syncthreads_or(pred ? 1 : 0);
  if (any && threadIdx.x == 0) atomicOr(flag, 1);
}

}  // namespace dlc
