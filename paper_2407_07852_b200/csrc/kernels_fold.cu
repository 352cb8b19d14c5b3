// kernels_fold.cu — K3: the rank-ordered fold of the cross-worker average
// (reduce.cpp:33-89, collective.cpp:1444-1489) on local rows, fused with the
// push of the mean to every rank (per-thread and TMA bulk-copy versions), and
// the NVLink flag barrier of the P2P step.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "device.cuh"
#include "kernels.cuh"

namespace dlc {

namespace {

// =============================================================================
// K3: ordered fold of K contributions (reduce.cpp:33-44 / 70-88).
// Each thread owns 8 consecutive elements; contributions are visited in rank
// order 0..K-1 so the FP32 sum is bit-identical to fold_mean.  Contributions
// may live in peer GPUs' memory (DLC_MODE_P2P): the loads then travel NVLink.
// =============================================================================

template <int IN>
__device__ __forceinline__ void load8(const void* base, size_t e8, float (&x)[8]) {
  if (IN == 1) {
    const uint4 w = ld_stream(reinterpret_cast<const uint4*>(base) + e8);
    x[0] = fp16_decode(lo16(w.x)); x[1] = fp16_decode(hi16(w.x));
    x[2] = fp16_decode(lo16(w.y)); x[3] = fp16_decode(hi16(w.y));
    x[4] = fp16_decode(lo16(w.z)); x[5] = fp16_decode(hi16(w.z));
    x[6] = fp16_decode(lo16(w.w)); x[7] = fp16_decode(hi16(w.w));
  } else {
    const float4 a = ld_stream(reinterpret_cast<const float4*>(base) + 2 * e8);
    const float4 b = ld_stream(reinterpret_cast<const float4*>(base) + 2 * e8 + 1);
    x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
    x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
    if (IN == 2) {
#pragma unroll
      for (int q = 0; q < 8; ++q) x[q] = fp16_decode(fp16_encode(x[q]));
    }
  }
}

// Raw 8-element group of one contribution (16 B of FP16 codes, 32 B of FP32),
// loaded first and decoded later, so the K loads of a group are all in flight
// together (for peer memory they are NVLink round trips).
template <int IN>
struct Raw8 {
  float4 a, b;
};
template <>
struct Raw8<1> {
  uint4 w;
};

// volatile: the K loads of a group stay adjacent (the scheduler would
// otherwise interleave the decode of load j with the issue of load j + 1)
__device__ __forceinline__ uint4 ld_cs_v4(const void* p) {
  uint4 v;
  asm volatile("ld.global.cs.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

template <int IN>
__device__ __forceinline__ void ld_raw(const void* base, size_t e8, Raw8<IN>& r) {
  if constexpr (IN == 1) {
    r.w = ld_cs_v4(reinterpret_cast<const uint4*>(base) + e8);
  } else {
    const uint4 a = ld_cs_v4(reinterpret_cast<const float4*>(base) + 2 * e8);
    const uint4 b = ld_cs_v4(reinterpret_cast<const float4*>(base) + 2 * e8 + 1);
    r.a = make_float4(__uint_as_float(a.x), __uint_as_float(a.y), __uint_as_float(a.z), __uint_as_float(a.w));
    r.b = make_float4(__uint_as_float(b.x), __uint_as_float(b.y), __uint_as_float(b.z), __uint_as_float(b.w));
  }
}

template <int IN>
__device__ __forceinline__ void unpack(const Raw8<IN>& r, float (&x)[8]) {
  if constexpr (IN == 1) {
    x[0] = fp16_decode(lo16(r.w.x)); x[1] = fp16_decode(hi16(r.w.x));
    x[2] = fp16_decode(lo16(r.w.y)); x[3] = fp16_decode(hi16(r.w.y));
    x[4] = fp16_decode(lo16(r.w.z)); x[5] = fp16_decode(hi16(r.w.z));
    x[6] = fp16_decode(lo16(r.w.w)); x[7] = fp16_decode(hi16(r.w.w));
  } else {
    x[0] = r.a.x; x[1] = r.a.y; x[2] = r.a.z; x[3] = r.a.w;
    x[4] = r.b.x; x[5] = r.b.y; x[6] = r.b.z; x[7] = r.b.w;
    if (IN == 2) {
#pragma unroll
      for (int q = 0; q < 8; ++q) x[q] = fp16_decode(fp16_encode(x[q]));
    }
  }
}

template <int IN>
__device__ __forceinline__ float load1(const void* base, size_t e) {
  if (IN == 1) return fp16_decode(reinterpret_cast<const uint16_t*>(base)[e]);
  const float x = reinterpret_cast<const float*>(base)[e];
  return IN == 2 ? fp16_decode(fp16_encode(x)) : x;
}

template <int OUT>
__device__ __forceinline__ bool store1(void* out, size_t e, float mean) {
  if (OUT == 1) {
    const uint16_t h = fp16_encode(mean);
    reinterpret_cast<uint16_t*>(out)[e] = h;
    return fp16_nonfinite(h);
  }
  const float y = OUT == 2 ? fp16_decode(fp16_encode(mean)) : mean;
  reinterpret_cast<float*>(out)[e] = y;
  return !finite_f(y);
}

template <int IN, int OUT>
__global__ void __launch_bounds__(kThreads) fold_kernel(const __grid_constant__ PtrList in, int k, void* out,
                                                        int* flag, size_t n) {
  const MeanDiv divisor = mean_div(k);  // reduce.cpp:36, 43
  bool bad = false;
  const size_t n8 = n / 8, i = gtid();
  if (i < n8) {
    float acc[8], x[8];
    load8<IN>(in.ptr[0], i, acc);
    for (int j = 1; j < k; ++j) {
      load8<IN>(in.ptr[j], i, x);
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = __fadd_rn(acc[q], x[q]);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = div_mean(acc[q], divisor);
    if (OUT == 1) {
      uint16_t h[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        h[q] = fp16_encode(acc[q]);
        bad |= fp16_nonfinite(h[q]);
      }
      st_stream(reinterpret_cast<uint4*>(out) + i,
                make_uint4(pack2(h[0], h[1]), pack2(h[2], h[3]), pack2(h[4], h[5]), pack2(h[6], h[7])));
    } else {
      if (OUT == 2) {
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = fp16_decode(fp16_encode(acc[q]));
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) bad |= !finite_f(acc[q]);
      float4* o = reinterpret_cast<float4*>(out) + 2 * i;
      st_stream(o, make_float4(acc[0], acc[1], acc[2], acc[3]));
      st_stream(o + 1, make_float4(acc[4], acc[5], acc[6], acc[7]));
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < n - n8 * 8) {
    const size_t e = n8 * 8 + threadIdx.x;
    float acc = load1<IN>(in.ptr[0], e);
    for (int j = 1; j < k; ++j) acc = __fadd_rn(acc, load1<IN>(in.ptr[j], e));
    bad |= store1<OUT>(out, e, div_mean(acc, divisor));
  }
  if (flag) block_or_flag(bad, flag);
}

// K3 fused with the all-gather: the owner pushes its mean to every rank.
// KK > 0: the contributor count at compile time, so the KK loads of a group
// are issued back to back (KK NVLink round trips in flight per thread instead
// of one); KK == 0: any k, one load at a time.
template <int PREC, int KK>
__global__ void __launch_bounds__(kThreads) fold_push_kernel(const __grid_constant__ PtrList in, int k,
                                                             const __grid_constant__ PtrList outs, int nout,
                                                             const __grid_constant__ PtrList flags, int nflags,
                                                             size_t n) {
  const MeanDiv divisor = mean_div(k);  // reduce.cpp:36, 43
  bool bad = false;
  const size_t n8 = n / 8;
  // grid-stride: a persistent grid of a few CTAs leaves the other SMs to the
  // HBM-bound K2 / K4 pieces running concurrently on the main stream
  for (size_t i = gtid(); i < n8; i += gstride()) {
    float acc[8], x[8];
    if constexpr (KK > 0) {
      Raw8<PREC> raw[KK];
#pragma unroll
      for (int j = 0; j < KK; ++j) ld_raw<PREC>(in.ptr[j], i, raw[j]);
      unpack<PREC>(raw[0], acc);
#pragma unroll
      for (int j = 1; j < KK; ++j) {  // rank order (reduce.cpp:37-43)
        unpack<PREC>(raw[j], x);
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = __fadd_rn(acc[q], x[q]);
      }
    } else {
      load8<PREC>(in.ptr[0], i, acc);
      for (int j = 1; j < k; ++j) {
        load8<PREC>(in.ptr[j], i, x);
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = __fadd_rn(acc[q], x[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = div_mean(acc[q], divisor);
    if (PREC == 1) {
      uint16_t h[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        h[q] = fp16_encode(acc[q]);
        bad |= fp16_nonfinite(h[q]);
      }
      const uint4 w = make_uint4(pack2(h[0], h[1]), pack2(h[2], h[3]), pack2(h[4], h[5]), pack2(h[6], h[7]));
      for (int o = 0; o < nout; ++o) st_stream(reinterpret_cast<uint4*>(const_cast<void*>(outs.ptr[o])) + i, w);
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) bad |= !finite_f(acc[q]);
      const float4 a = make_float4(acc[0], acc[1], acc[2], acc[3]), b = make_float4(acc[4], acc[5], acc[6], acc[7]);
      for (int o = 0; o < nout; ++o) {
        float4* d = reinterpret_cast<float4*>(const_cast<void*>(outs.ptr[o])) + 2 * i;
        st_stream(d, a);
        st_stream(d + 1, b);
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < n - n8 * 8) {
    const size_t e = n8 * 8 + threadIdx.x;
    float acc = load1<PREC>(in.ptr[0], e);
    for (int j = 1; j < k; ++j) acc = __fadd_rn(acc, load1<PREC>(in.ptr[j], e));
    const float mean = div_mean(acc, divisor);
    for (int o = 0; o < nout; ++o) bad |= store1<PREC>(const_cast<void*>(outs.ptr[o]), e, mean);
  }
  if (__syncthreads_or(bad ? 1 : 0) && threadIdx.x == 0) {
    for (int o = 0; o < nflags; ++o) *reinterpret_cast<volatile int*>(const_cast<void*>(flags.ptr[o])) = 1;
  }
  // The CTA's pushed slots are visible system-wide before the barrier that
  // follows: the __syncthreads_or above orders every thread's stores before
  // this (cumulative) system-scope fence of one thread.
  if (threadIdx.x == 0) __threadfence_system();
}

// ---- K3 fused with the all-gather, TMA version -------------------------------
// The same rank-ordered fold as fold_push_kernel, with the data moved by the
// bulk-copy engine (cp.async.bulk) instead of per-thread loads and stores:
// one elected thread streams 8 KB tiles of the KK inputs (peer memory over
// NVLink, or local HBM) into a STAGES-deep shared-memory ring, arming an
// mbarrier with the expected bytes; NT threads fold the tile in rank order
// into an output tile, which the elected thread bulk-stores into every
// destination (the owners' mean slots in every rank's gather buffer).  Each CTA
// keeps STAGES * KK * 8 KB of NVLink reads in flight with a handful of
// instructions, so a few dozen CTAs saturate the links and leave the SMs to the
// HBM-bound K2 / K4 pieces.
// NT threads per CTA (tma_threads(): 128 for K <= 4, more as the CTA count
// falls with K): the fold's decode / add / encode work is latency-bound with one
// warp per scheduler (ncu: 1.15 IPC per SM at 128 threads).
constexpr int kTmaThreads = 128;
constexpr int kTmaTileBytes = 8192;
constexpr int kTmaStages = 3;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_load(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst_smem)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void bulk_store(void* dst, const void* src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src_smem)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

template <int PREC, int KK, int NT>
__global__ void __launch_bounds__(NT) fold_push_tma_kernel(const __grid_constant__ PtrList in,
                                                                    const __grid_constant__ PtrList outs, int nout,
                                                                    const __grid_constant__ PtrList flags,
                                                                    int nflags, size_t n, MeanDiv divisor) {
  constexpr int W = PREC == 1 ? 2 : 4;
  constexpr int TILE = kTmaTileBytes / W;  // elements per tile
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* in_buf = smem;                                          // [STAGES][KK][8 KB]
  uint8_t* out_buf = smem + kTmaStages * KK * kTmaTileBytes;       // [STAGES][8 KB]
  uint64_t* bar = reinterpret_cast<uint64_t*>(out_buf + kTmaStages * kTmaTileBytes);  // [STAGES]
  const size_t ntiles = (n + TILE - 1) / TILE;
  const size_t mine = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const bool leader = threadIdx.x == 0;
  auto tile_of = [&](size_t i) { return blockIdx.x + i * gridDim.x; };
  auto tile_bytes = [&](size_t t) {
    const size_t e = t * (size_t)TILE;
    return (uint32_t)((n - e < (size_t)TILE ? n - e : (size_t)TILE) * W);
  };
  auto issue = [&](size_t i) {  // tile i of this CTA into stage i % STAGES
    const int st = (int)(i % kTmaStages);
    const size_t t = tile_of(i);
    const uint32_t bytes = tile_bytes(t);
    mbar_expect_tx(&bar[st], bytes * KK);
#pragma unroll
    for (int j = 0; j < KK; ++j)
      bulk_load(in_buf + ((size_t)st * KK + j) * kTmaTileBytes,
                static_cast<const uint8_t*>(in.ptr[j]) + t * (size_t)kTmaTileBytes, bytes, &bar[st]);
  };
  if (leader) {
    for (int st = 0; st < kTmaStages; ++st) mbar_init(&bar[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (leader)
    for (size_t i = 0; i < mine && i < (size_t)kTmaStages; ++i) issue(i);
  bool bad = false;
  for (size_t i = 0; i < mine; ++i) {
    const int st = (int)(i % kTmaStages);
    const size_t t = tile_of(i);
    const uint32_t bytes = tile_bytes(t);
    if (leader && i >= (size_t)kTmaStages) bulk_wait_read<kTmaStages - 1>();  // out_buf[st] read by its store
    __syncthreads();
    mbar_wait(&bar[st], (uint32_t)((i / kTmaStages) & 1));
    const uint8_t* src = in_buf + (size_t)st * KK * kTmaTileBytes;
    uint8_t* dst = out_buf + (size_t)st * kTmaTileBytes;
    for (uint32_t off = threadIdx.x * 16; off < bytes; off += NT * 16) {  // 16 B per thread and step
      constexpr int E = 16 / W;  // 8 FP16 or 4 FP32 elements
      float acc[E], x[E];
#pragma unroll
      for (int j = 0; j < KK; ++j) {  // rank order (reduce.cpp:37-43)
        const uint4 v = *reinterpret_cast<const uint4*>(src + (size_t)j * kTmaTileBytes + off);
        if constexpr (PREC == 1) {
          x[0] = fp16_decode(lo16(v.x)); x[1] = fp16_decode(hi16(v.x));
          x[2] = fp16_decode(lo16(v.y)); x[3] = fp16_decode(hi16(v.y));
          x[4] = fp16_decode(lo16(v.z)); x[5] = fp16_decode(hi16(v.z));
          x[6] = fp16_decode(lo16(v.w)); x[7] = fp16_decode(hi16(v.w));
        } else {
          x[0] = __uint_as_float(v.x); x[1] = __uint_as_float(v.y);
          x[2] = __uint_as_float(v.z); x[3] = __uint_as_float(v.w);
        }
#pragma unroll
        for (int q = 0; q < E; ++q) acc[q] = j == 0 ? x[q] : __fadd_rn(acc[q], x[q]);
      }
      uint4 o;
      if constexpr (PREC == 1) {
        uint16_t h[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          h[q] = fp16_encode(div_mean(acc[q], divisor));
          bad |= fp16_nonfinite(h[q]);
        }
        o = make_uint4(pack2(h[0], h[1]), pack2(h[2], h[3]), pack2(h[4], h[5]), pack2(h[6], h[7]));
      } else {
        float m[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          m[q] = div_mean(acc[q], divisor);
          bad |= !finite_f(m[q]);
        }
        o = make_uint4(__float_as_uint(m[0]), __float_as_uint(m[1]), __float_as_uint(m[2]), __float_as_uint(m[3]));
      }
      *reinterpret_cast<uint4*>(dst + off) = o;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // our smem writes -> the bulk store's reads
    __syncthreads();  // every thread is done with in_buf[st] and out_buf[st]
    if (leader) {
      for (int o = 0; o < nout; ++o)
        bulk_store(static_cast<uint8_t*>(const_cast<void*>(outs.ptr[o])) + t * (size_t)kTmaTileBytes, dst, bytes);
      bulk_commit();
      if (i + kTmaStages < mine) issue(i + kTmaStages);  // in_buf[st] is free again
    }
  }
  if (__syncthreads_or(bad ? 1 : 0) && threadIdx.x == 0) {
    for (int o = 0; o < nflags; ++o) *reinterpret_cast<volatile int*>(const_cast<void*>(flags.ptr[o])) = 1;
  }
  if (leader) {
    bulk_wait_all();  // every bulk store of this CTA has landed
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __threadfence_system();  // ... and is visible system-wide before the barrier that follows
  }
}

size_t fold_push_tma_smem(int k) { return (size_t)kTmaStages * (k + 1) * kTmaTileBytes + kTmaStages * 8; }

// ---- K3 fused with the all-gather, warp-specialised TMA version --------------
// The same fold again, with the roles split across warps so no thread both
// issues copies and computes:
//   warp 0 (one elected lane): producer.  Streams 8 KB tiles of the KK inputs
//     into a kWsStages-deep ring (bulk copies, mbarrier full[s] with the
//     expected bytes); reuses stage s once the consumers release it (empty[s]).
//   warps 1..NC: consumers.  Wait full[s], fold the tile 16 B per thread and
//     step (decode 2 codes per conversion, rank-ordered FP32 adds, the mean,
//     encode 2 per conversion), release in_buf[s] (empty[s]), write the mean
//     tile into one of two output buffers; one elected consumer bulk-stores it
//     to every destination (the owner's slot in every rank's gather buffer).
// Only the consumers meet at a named barrier, once per tile.  FP16 decode is
// the plain hardware widening (exact for every finite and infinite code; a NaN
// contribution makes the mean NaN whatever its payload, and NaNs compare by
// class); encode is cvt.rn.f16x2.f32 (RNE with overflow to inf,
// fp16.cpp:25-63) with the reference's NaN code sign|0x7E00 patched on the
// rare path where a code is non-finite.
constexpr int kWsStages = 3;
constexpr int kWsOutStages = 2;

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void consumer_sync(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

__device__ __forceinline__ float2 h2_to_f2(uint32_t w) {
  return __half22float2(*reinterpret_cast<const __half2*>(&w));
}

__device__ __forceinline__ uint32_t f2_to_h2(float lo, float hi) {
  const __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&h);
}

__device__ __forceinline__ bool h2_nonfinite(uint32_t w) {
  return ((w & 0x7C00u) == 0x7C00u) | ((w & 0x7C000000u) == 0x7C000000u);
}

template <int PREC, int KK, int NC>
__global__ void __launch_bounds__(32 * (NC + 1)) fold_push_ws_kernel(const __grid_constant__ PtrList in,
                                                                     const __grid_constant__ PtrList outs, int nout,
                                                                     const __grid_constant__ PtrList flags,
                                                                     int nflags, size_t n, MeanDiv divisor) {
  constexpr int W = PREC == 1 ? 2 : 4;
  constexpr int TILE = kTmaTileBytes / W;  // elements per tile
  constexpr int NCT = NC * 32;             // consumer threads
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* in_buf = smem;                                       // [kWsStages][KK][8 KB]
  uint8_t* out_buf = smem + kWsStages * KK * kTmaTileBytes;     // [kWsOutStages][8 KB]
  uint64_t* full = reinterpret_cast<uint64_t*>(out_buf + kWsOutStages * kTmaTileBytes);  // [kWsStages]
  uint64_t* empty = full + kWsStages;                                                     // [kWsStages]
  __shared__ int s_bad;
  const size_t ntiles = (n + TILE - 1) / TILE;
  const size_t mine = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto tile_bytes = [&](size_t t) {
    const size_t e = t * (size_t)TILE;
    return (uint32_t)((n - e < (size_t)TILE ? n - e : (size_t)TILE) * W);
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < kWsStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NC);  // one arrival per consumer warp
    }
    s_bad = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {  // ---- producer ----
    if (lane == 0) {
      for (size_t i = 0; i < mine; ++i) {
        const int s = (int)(i % kWsStages);
        if (i >= (size_t)kWsStages) mbar_wait(&empty[s], (uint32_t)(((i / kWsStages) + 1) & 1));
        const size_t t = blockIdx.x + i * gridDim.x;
        const uint32_t bytes = tile_bytes(t);
        mbar_expect_tx(&full[s], bytes * KK);
#pragma unroll
        for (int j = 0; j < KK; ++j)
          bulk_load(in_buf + ((size_t)s * KK + j) * kTmaTileBytes,
                    static_cast<const uint8_t*>(in.ptr[j]) + t * (size_t)kTmaTileBytes, bytes, &full[s]);
      }
    }
    return;
  }
  // ---- consumers ----
  const int ct = threadIdx.x - 32;
  const bool storer = ct == 0;
  bool bad = false;
  for (size_t i = 0; i < mine; ++i) {
    const int s = (int)(i % kWsStages);
    const size_t t = blockIdx.x + i * gridDim.x;
    const uint32_t bytes = tile_bytes(t);
    uint8_t* dst = out_buf + (size_t)(i % kWsOutStages) * kTmaTileBytes;  // free: see the wait below
    mbar_wait(&full[s], (uint32_t)((i / kWsStages) & 1));
    const uint8_t* src = in_buf + (size_t)s * KK * kTmaTileBytes;
    for (uint32_t off = ct * 16; off < bytes; off += NCT * 16) {
      uint4 o;
      if constexpr (PREC == 1) {
        float a[8];
#pragma unroll
        for (int j = 0; j < KK; ++j) {  // rank order (reduce.cpp:37-43)
          const uint4 v = *reinterpret_cast<const uint4*>(src + (size_t)j * kTmaTileBytes + off);
          const float2 x0 = h2_to_f2(v.x), x1 = h2_to_f2(v.y), x2 = h2_to_f2(v.z), x3 = h2_to_f2(v.w);
          if (j == 0) {
            a[0] = x0.x; a[1] = x0.y; a[2] = x1.x; a[3] = x1.y;
            a[4] = x2.x; a[5] = x2.y; a[6] = x3.x; a[7] = x3.y;
          } else {
            a[0] = __fadd_rn(a[0], x0.x); a[1] = __fadd_rn(a[1], x0.y);
            a[2] = __fadd_rn(a[2], x1.x); a[3] = __fadd_rn(a[3], x1.y);
            a[4] = __fadd_rn(a[4], x2.x); a[5] = __fadd_rn(a[5], x2.y);
            a[6] = __fadd_rn(a[6], x3.x); a[7] = __fadd_rn(a[7], x3.y);
          }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) a[q] = div_mean(a[q], divisor);
        o = make_uint4(f2_to_h2(a[0], a[1]), f2_to_h2(a[2], a[3]), f2_to_h2(a[4], a[5]), f2_to_h2(a[6], a[7]));
        if (h2_nonfinite(o.x) | h2_nonfinite(o.y) | h2_nonfinite(o.z) | h2_nonfinite(o.w)) {
          bad = true;  // rare: the reference's exact codes (NaN -> sign|0x7E00)
          o = make_uint4(pack2(fp16_encode(a[0]), fp16_encode(a[1])), pack2(fp16_encode(a[2]), fp16_encode(a[3])),
                         pack2(fp16_encode(a[4]), fp16_encode(a[5])), pack2(fp16_encode(a[6]), fp16_encode(a[7])));
        }
      } else {
        float a[4];
#pragma unroll
        for (int j = 0; j < KK; ++j) {
          const uint4 v = *reinterpret_cast<const uint4*>(src + (size_t)j * kTmaTileBytes + off);
          const float x[4] = {__uint_as_float(v.x), __uint_as_float(v.y), __uint_as_float(v.z), __uint_as_float(v.w)};
#pragma unroll
          for (int q = 0; q < 4; ++q) a[q] = j == 0 ? x[q] : __fadd_rn(a[q], x[q]);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          a[q] = div_mean(a[q], divisor);
          bad |= !finite_f(a[q]);
        }
        o = make_uint4(__float_as_uint(a[0]), __float_as_uint(a[1]), __float_as_uint(a[2]), __float_as_uint(a[3]));
      }
      *reinterpret_cast<uint4*>(dst + off) = o;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // in_buf[s] is read: the producer may refill it
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // our smem writes -> the bulk store's reads
    // before the next tile overwrites the other output buffer, the store that
    // read it (issued one tile ago) must be done reading
    if (storer) bulk_wait_read<kWsOutStages - 2>();
    consumer_sync(NCT);  // every consumer's share of dst is written
    if (storer) {
      for (int o = 0; o < nout; ++o)
        bulk_store(static_cast<uint8_t*>(const_cast<void*>(outs.ptr[o])) + t * (size_t)kTmaTileBytes, dst, bytes);
      bulk_commit();
    }
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&s_bad, 1);
  consumer_sync(NCT);
  if (storer) {
    if (s_bad)
      for (int o = 0; o < nflags; ++o) *reinterpret_cast<volatile int*>(const_cast<void*>(flags.ptr[o])) = 1;
    bulk_wait_all();  // every bulk store of this CTA has landed
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __threadfence_system();  // ... and is visible system-wide before the barrier that follows
  }
}

size_t fold_push_ws_smem(int k) {
  return (size_t)kWsStages * k * kTmaTileBytes + kWsOutStages * kTmaTileBytes + 2 * kWsStages * 8;
}


// ---- NVLink flag barrier ----------------------------------------------------
__global__ void flag_barrier_kernel(const __grid_constant__ PtrList remote, const uint64_t* local, int k, int me,
                                    uint64_t epoch, int* err, uint64_t timeout_ns, int stall, int commit) {
  const int j = threadIdx.x;
  __shared__ int s_failed;
  if (j == 0) {
    s_failed = *reinterpret_cast<volatile int*>(err);
    if (stall) {  // fault injection: stop arriving, fail this rank's round
      atomicExch(err, 1);
      s_failed = 2;
    }
  }
  __syncthreads();
  const int failed = s_failed;
  if (failed) {
    // the round already failed here: no wait; at the commit barrier tell the
    // peers (a stalled rank stays silent, as a dead peer would)
    if (commit && failed == 1 && j < k && j != me) {
      __threadfence_system();
      *reinterpret_cast<volatile unsigned long long*>(const_cast<void*>(remote.ptr[j])) = (epoch << 1) | 1ull;
    }
    return;
  }
  if (j < k && j != me) {
    __threadfence_system();  // everything this GPU wrote before the barrier is visible first
    *reinterpret_cast<volatile unsigned long long*>(const_cast<void*>(remote.ptr[j])) = epoch << 1;
    const uint64_t start = globaltimer_ns();
    const volatile unsigned long long* mine = reinterpret_cast<const volatile unsigned long long*>(local + j);
    unsigned long long v;
    while (((v = *mine) >> 1) < epoch) {
      if (globaltimer_ns() - start > timeout_ns) {  // a peer stopped participating
        atomicExch(err, 1);
        break;
      }
    }
    if (commit && (v >> 1) == epoch && (v & 1ull)) atomicExch(err, 1);  // a peer's round failed
    __threadfence_system();
  }
  __syncthreads();
}

}  // namespace

void launch_fold(const PtrList& in, int k, int in_kind, void* out, int out_kind, int* flag, size_t n,
                 cudaStream_t s) {
  const int grid = grid_window<1>(n / 8);
#define DLC_FOLD(I, O)                                                      \
  if (in_kind == I && out_kind == O) {                                      \
    fold_kernel<I, O><<<grid, kThreads, 0, s>>>(in, k, out, flag, n);       \
    return;                                                                 \
  }
  DLC_FOLD(0, 0) DLC_FOLD(0, 1) DLC_FOLD(0, 2) DLC_FOLD(1, 0) DLC_FOLD(1, 1) DLC_FOLD(1, 2)
  DLC_FOLD(2, 0) DLC_FOLD(2, 1) DLC_FOLD(2, 2)
#undef DLC_FOLD
}

void launch_fold_push(const PtrList& in, int k, int precision, const PtrList& outs, int nout, const PtrList& flags,
                      int nflags,
                      size_t n, int ctas, cudaStream_t s) {
  const int grid = ctas > 0 ? std::min(ctas, grid_window<1>(n / 8)) : grid_window<1>(n / 8);
#define DLC_FOLD_PUSH(P, KK) fold_push_kernel<P, KK><<<grid, kThreads, 0, s>>>(in, k, outs, nout, flags, nflags, n)
#define DLC_FOLD_PUSH_K(P)      \
  switch (k) {                  \
    case 2: DLC_FOLD_PUSH(P, 2); break; \
    case 3: DLC_FOLD_PUSH(P, 3); break; \
    case 4: DLC_FOLD_PUSH(P, 4); break; \
    case 5: DLC_FOLD_PUSH(P, 5); break; \
    case 6: DLC_FOLD_PUSH(P, 6); break; \
    case 7: DLC_FOLD_PUSH(P, 7); break; \
    case 8: DLC_FOLD_PUSH(P, 8); break; \
    default: DLC_FOLD_PUSH(P, 0); break; \
  }
  if (precision == 0) {
    DLC_FOLD_PUSH_K(0)
  } else {
    DLC_FOLD_PUSH_K(1)
  }
#undef DLC_FOLD_PUSH_K
#undef DLC_FOLD_PUSH
}

namespace {

// One instance of the TMA fold: WS = the warp-specialised kernel (NT consumer
// threads + a producer warp), else the single-leader one (NT threads).
template <int P, int KK, int NT, bool WS>
void launch_tma_inst(int grid, cudaStream_t s, const PtrList& in, const PtrList& outs, int nout, const PtrList& flags,
                     int nflags, size_t n, MeanDiv md) {
  auto* kern = WS ? fold_push_ws_kernel<P, KK, NT / 32> : fold_push_tma_kernel<P, KK, NT>;
  const size_t smem = WS ? fold_push_ws_smem(KK) : fold_push_tma_smem(KK);
  // per-device function attribute, set once (rank threads may launch concurrently)
  static std::atomic<unsigned> attr_devices{0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_devices.load() & (1u << (dev & 31)))) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);  // failures surface at launch
    attr_devices.fetch_or(1u << (dev & 31));
  }
  kern<<<grid, WS ? NT + 32 : NT, smem, s>>>(in, outs, nout, flags, nflags, n, md);
}

template <int P, int KK>
void launch_tma_k(int nt, bool ws, int grid, cudaStream_t s, const PtrList& in, const PtrList& outs, int nout,
                  const PtrList& flags, int nflags, size_t n, MeanDiv md) {
#define DLC_TMA_NT(NT)                                                                     \
  (ws ? launch_tma_inst<P, KK, NT, true>(grid, s, in, outs, nout, flags, nflags, n, md)    \
      : launch_tma_inst<P, KK, NT, false>(grid, s, in, outs, nout, flags, nflags, n, md))
  if (nt >= 512)
    DLC_TMA_NT(512);
  else if (nt >= 256)
    DLC_TMA_NT(256);
  else
    DLC_TMA_NT(128);
#undef DLC_TMA_NT
}

template <int P>
bool launch_tma_p(int k, int nt, bool ws, int grid, cudaStream_t s, const PtrList& in, const PtrList& outs, int nout,
                  const PtrList& flags, int nflags, size_t n, MeanDiv md) {
  switch (k) {
    case 2: launch_tma_k<P, 2>(nt, ws, grid, s, in, outs, nout, flags, nflags, n, md); return true;
    case 3: launch_tma_k<P, 3>(nt, ws, grid, s, in, outs, nout, flags, nflags, n, md); return true;
    case 4: launch_tma_k<P, 4>(nt, ws, grid, s, in, outs, nout, flags, nflags, n, md); return true;
    case 5: launch_tma_k<P, 5>(nt, ws, grid, s, in, outs, nout, flags, nflags, n, md); return true;
    case 6: launch_tma_k<P, 6>(nt, ws, grid, s, in, outs, nout, flags, nflags, n, md); return true;
    case 7: launch_tma_k<P, 7>(nt, ws, grid, s, in, outs, nout, flags, nflags, n, md); return true;
    case 8: launch_tma_k<P, 8>(nt, ws, grid, s, in, outs, nout, flags, nflags, n, md); return true;
    default: return false;
  }
}

}  // namespace

bool launch_fold_push_tma(const PtrList& in, int k, int precision, const PtrList& outs, int nout,
                          const PtrList& flags, int nflags, size_t n, int ctas, int threads, int kernel,
                          cudaStream_t s) {
  const MeanDiv md = mean_div(k);  // reduce.cpp:36, 43
  const int W = precision == 1 ? 2 : 4;
  const size_t ntiles = (n + kTmaTileBytes / W - 1) / (kTmaTileBytes / W);
  const int grid = (int)std::max<size_t>(1, std::min<size_t>(ctas > 0 ? ctas : num_sms(), ntiles));
  const bool ws = kernel == 1;
  return precision == 0 ? launch_tma_p<0>(k, threads, ws, grid, s, in, outs, nout, flags, nflags, n, md)
                        : launch_tma_p<1>(k, threads, ws, grid, s, in, outs, nout, flags, nflags, n, md);
}

void launch_flag_barrier(const PtrList& remote, const uint64_t* local, int k, int me, uint64_t epoch, int* err,
                         uint64_t timeout_ns, bool stall, bool commit, cudaStream_t s) {
  flag_barrier_kernel<<<1, 32, 0, s>>>(remote, local, k, me, epoch, err, timeout_ns, stall ? 1 : 0, commit ? 1 : 0);
}

}  // namespace dlc
