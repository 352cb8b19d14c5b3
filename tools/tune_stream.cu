// tune_stream.cu — HBM streaming micro-benchmark used to pick the grid /
// work-distribution policy of the hot-path kernels (development tool, not part
// of the product).  Random-initialised buffers of N = 1.1e9 FP32 (every stream
// >> L2); patterns with the hot-path traffic shapes and the real arithmetic:
//   copy  1R1W    adam 4R3W (K1)    nest 3R3W (K4/solo)    pg 2R + half W (K2)
// Work-distribution policies:
//   gs  : persistent grid-stride (grid = #SM x occupancy), U vectors per trip
//   full: one CTA per 256*U vectors, every thread U vectors (non-persistent)
//   blk : persistent, each CTA owns one contiguous range
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o tune_stream tune_stream.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                                \
  do {                                                                                       \
    cudaError_t e = (x);                                                                     \
    if (e != cudaSuccess) {                                                                  \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);    \
      std::exit(1);                                                                          \
    }                                                                                        \
  } while (0)

enum { GS = 0, FULL = 1, BLK = 2 };

__global__ void fill(float* p, size_t n, unsigned seed, float lo, float hi) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned x = (unsigned)i * 2654435761u ^ seed;
    x ^= x >> 13;
    x *= 0x5bd1e995;
    x ^= x >> 15;
    p[i] = lo + (hi - lo) * (x & 0xFFFFFF) * (1.0f / 16777216.0f);
  }
}

struct Ar {
  const float4* in[4];
  float4* out[3];
  size_t n4;
};

__device__ __forceinline__ float adam1(float p, float g, float& m, float& v) {
  g = __fmul_rn(g, 1.0f / 65536.0f);
  m = __fadd_rn(__fmul_rn(0.9f, m), __fmul_rn(0.1f, g));
  v = __fadd_rn(__fmul_rn(0.95f, v), __fmul_rn(__fmul_rn(0.05f, g), g));
  const float mh = __fdiv_rn(m, 0.1f), vh = __fdiv_rn(v, 0.05f);
  return __fsub_rn(p, __fmul_rn(4e-4f, __fadd_rn(__fdiv_rn(mh, __fadd_rn(__fsqrt_rn(vh), 1e-8f)), __fmul_rn(0.1f, p))));
}
__device__ __forceinline__ float nest1(float t, float d, float& b) {
  b = __fadd_rn(__fmul_rn(0.9f, b), d);
  return __fsub_rn(t, __fmul_rn(0.7f, __fadd_rn(d, __fmul_rn(0.9f, b))));
}

// one vector of work for pattern PAT at vector index j
template <int PAT>
__device__ __forceinline__ void work(const Ar& a, size_t j, bool& bad) {
  if (PAT == 0) {  // copy
    __stcs(a.out[0] + j, __ldcs(a.in[0] + j));
  } else if (PAT == 1) {  // adam
    float4 p = __ldcs(a.in[0] + j), g = __ldcs(a.in[1] + j), m = __ldcs(a.in[2] + j), v = __ldcs(a.in[3] + j), o;
    o.x = adam1(p.x, g.x, m.x, v.x);
    o.y = adam1(p.y, g.y, m.y, v.y);
    o.z = adam1(p.z, g.z, m.z, v.z);
    o.w = adam1(p.w, g.w, m.w, v.w);
    bad |= !isfinite(o.x + o.y + o.z + o.w);
    __stcs(a.out[0] + j, o);
    __stcs(a.out[1] + j, m);
    __stcs(a.out[2] + j, v);
  } else if (PAT == 2) {  // nesterov solo: t, l, b -> t', b', l'
    float4 t = __ldcs(a.in[0] + j), l = __ldcs(a.in[1] + j), b = __ldcs(a.in[2] + j), o;
    o.x = nest1(t.x, __fsub_rn(t.x, l.x), b.x);
    o.y = nest1(t.y, __fsub_rn(t.y, l.y), b.y);
    o.z = nest1(t.z, __fsub_rn(t.z, l.z), b.z);
    o.w = nest1(t.w, __fsub_rn(t.w, l.w), b.w);
    __stcs(a.out[0] + j, o);
    __stcs(a.out[1] + j, b);
    __stcs(a.out[2] + j, o);
  } else {  // pseudo-grad fp16: t, l -> 4 codes
    float4 t = __ldcs(a.in[0] + j), l = __ldcs(a.in[1] + j);
    __half2 h0 = __floats2half2_rn(t.x - l.x, t.y - l.y), h1 = __floats2half2_rn(t.z - l.z, t.w - l.w);
    uint2 w = make_uint2(*reinterpret_cast<unsigned*>(&h0), *reinterpret_cast<unsigned*>(&h1));
    __stcs(reinterpret_cast<uint2*>(a.out[0]) + j, w);
  }
}

template <int PAT, int POL, int U>
__global__ void __launch_bounds__(256) kern(Ar a, int* flag) {
  bool bad = false;
  if (POL == GS) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n4; i += stride * U) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (i + u * stride < a.n4) work<PAT>(a, i + u * stride, bad);
    }
  } else if (POL == FULL) {
    const size_t base = (size_t)blockIdx.x * blockDim.x * U + threadIdx.x;
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (base + u * blockDim.x < a.n4) work<PAT>(a, base + u * blockDim.x, bad);
  } else {
    const size_t per = (a.n4 + gridDim.x - 1) / gridDim.x;
    const size_t lo = blockIdx.x * per, hi = lo + per < a.n4 ? lo + per : a.n4;
    for (size_t i = lo + threadIdx.x; i < hi; i += (size_t)blockDim.x * U) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (i + u * blockDim.x < hi) work<PAT>(a, i + u * blockDim.x, bad);
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

int main(int argc, char** argv) {
  const size_t n = argc > 1 ? strtoull(argv[1], nullptr, 10) : 1100000000ull;
  const size_t n4 = n / 4;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  std::vector<float*> buf(7);
  for (int i = 0; i < 7; ++i) {
    CK(cudaMalloc(&buf[i], n * 4));
    fill<<<4096, 256>>>(buf[i], n, 1234u + i, i == 3 ? 0.0f : -1.0f, 1.0f);
  }
  CK(cudaDeviceSynchronize());
  int* flag;
  CK(cudaMalloc(&flag, 4));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const double bytes[4] = {8.0, 28.0, 24.0, 10.0};
  const char* pn[4] = {"copy", "adam", "nest", "pg16"};

#define RUN(PAT, POL, U, MULT)                                                                         \
  {                                                                                                    \
    auto k = kern<PAT, POL, U>;                                                                        \
    int occ = 0;                                                                                       \
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 256, 0));                                \
    int grid = POL == FULL ? (int)((n4 + 256 * U - 1) / (256 * U)) : sms * occ * MULT;                 \
    Ar a;                                                                                              \
    for (int i = 0; i < 4; ++i) a.in[i] = (const float4*)buf[i];                                       \
    for (int i = 0; i < 3; ++i) a.out[i] = (float4*)buf[4 + i];                                        \
    a.n4 = n4;                                                                                         \
    for (int w = 0; w < 2; ++w) k<<<grid, 256>>>(a, flag);                                              \
    CK(cudaDeviceSynchronize());                                                                       \
    CK(cudaEventRecord(e0));                                                                           \
    for (int r = 0; r < 8; ++r) k<<<grid, 256>>>(a, flag);                                              \
    CK(cudaEventRecord(e1));                                                                           \
    CK(cudaEventSynchronize(e1));                                                                      \
    float ms = 0;                                                                                      \
    CK(cudaEventElapsedTime(&ms, e0, e1));                                                             \
    ms /= 8;                                                                                           \
    std::printf("%-5s %-4s U%d x%d occ%d grid%-8d %8.3f ms %8.1f GB/s\n", pn[PAT],                     \
                POL == GS ? "gs" : POL == FULL ? "full" : "blk", U, MULT, occ, grid, ms,               \
                bytes[PAT] * n / (ms * 1e-3) / 1e9);                                                   \
  }
#define PATSET(P)    \
  RUN(P, GS, 1, 1)   \
  RUN(P, GS, 2, 1)   \
  RUN(P, GS, 2, 2)   \
  RUN(P, GS, 4, 1)   \
  RUN(P, FULL, 1, 1) \
  RUN(P, FULL, 2, 1) \
  RUN(P, FULL, 4, 1) \
  RUN(P, BLK, 1, 1)  \
  RUN(P, BLK, 2, 1)  \
  RUN(P, BLK, 2, 4)
  PATSET(0)
  PATSET(1)
  PATSET(2)
  PATSET(3)
  return 0;
}
