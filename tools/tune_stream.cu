// tune_stream.cu — HBM streaming micro-benchmark used to pick the K1/K4 access
// pattern (development tool, not part of the product).
//
// Measures, over N = 1.1e9 FP32 elements (every stream >> L2):
//   copy 1R1W with several access variants, and the AdamW traffic shape (4R3W)
//   with the real AdamW arithmetic, under different load/store cache hints,
//   vectors-in-flight U, CTA size and grid policy.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o tune_stream tune_stream.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      std::exit(1);                                                             \
    }                                                                           \
  } while (0)

enum { LD_DEF = 0, LD_CS = 1, LD_NC_NA = 2, LD_LU = 3 };
enum { ST_DEF = 0, ST_CS = 1, ST_NA = 2 };

template <int LD>
__device__ __forceinline__ float4 ld4(const float4* p) {
  if (LD == LD_CS) return __ldcs(p);
  if (LD == LD_LU) return __ldlu(p);
  if (LD == LD_NC_NA) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
  }
  return *p;
}

template <int ST>
__device__ __forceinline__ void st4(float4* p, float4 v) {
  if (ST == ST_CS) {
    __stcs(p, v);
  } else if (ST == ST_NA) {
    asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w));
  } else {
    *p = v;
  }
}

template <int LD, int ST, int U>
__global__ void copy_k(const float4* __restrict__ a, float4* __restrict__ b, size_t n4) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride * U) {
    float4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i + u * stride < n4) x[u] = ld4<LD>(a + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i + u * stride < n4) st4<ST>(b + i + u * stride, x[u]);
  }
}

struct S {
  float b1, b2, eps, wd, omb1, omb2, c1, c2, lr, inv;
};

__device__ __forceinline__ float adam1(float p, float g, float& m, float& v, const S& s) {
  g = __fmul_rn(g, s.inv);
  m = __fadd_rn(__fmul_rn(s.b1, m), __fmul_rn(s.omb1, g));
  v = __fadd_rn(__fmul_rn(s.b2, v), __fmul_rn(__fmul_rn(s.omb2, g), g));
  const float mh = __fdiv_rn(m, s.c1), vh = __fdiv_rn(v, s.c2);
  return __fsub_rn(p, __fmul_rn(s.lr, __fadd_rn(__fdiv_rn(mh, __fadd_rn(__fsqrt_rn(vh), s.eps)), __fmul_rn(s.wd, p))));
}

// AdamW traffic: read p,g,m,v ; write p2,m2,v2 (ping-pong)
template <int LD, int ST, int U, bool MATH>
__global__ void adam_k(const float4* __restrict__ P, const float4* __restrict__ G, const float4* __restrict__ M,
                       const float4* __restrict__ V, float4* __restrict__ Po, float4* __restrict__ Mo,
                       float4* __restrict__ Vo, size_t n4, S s, int* flag) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  bool bad = false;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride * U) {
    float4 p[U], g[U], m[U], v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i + u * stride < n4) {
        g[u] = ld4<LD>(G + i + u * stride);
        p[u] = ld4<LD>(P + i + u * stride);
        m[u] = ld4<LD>(M + i + u * stride);
        v[u] = ld4<LD>(V + i + u * stride);
      }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i + u * stride < n4) {
        float4 o;
        if (MATH) {
          o.x = adam1(p[u].x, g[u].x, m[u].x, v[u].x, s);
          o.y = adam1(p[u].y, g[u].y, m[u].y, v[u].y, s);
          o.z = adam1(p[u].z, g[u].z, m[u].z, v[u].z, s);
          o.w = adam1(p[u].w, g[u].w, m[u].w, v[u].w, s);
          bad |= !isfinite(o.x);
        } else {
          o = make_float4(p[u].x + g[u].x, p[u].y + g[u].y, p[u].z + g[u].z, p[u].w + g[u].w);
        }
        st4<ST>(Po + i + u * stride, o);
        st4<ST>(Mo + i + u * stride, m[u]);
        st4<ST>(Vo + i + u * stride, v[u]);
      }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

template <typename K>
int occ(K k, int threads) {
  int b = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, threads, 0));
  return b;
}

int main(int argc, char** argv) {
  const size_t n = argc > 1 ? strtoull(argv[1], nullptr, 10) : 1100000000ull;
  const size_t n4 = n / 4;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  std::vector<float*> buf(7);
  for (auto& b : buf) {
    CK(cudaMalloc(&b, n * 4));
    CK(cudaMemset(b, 0, n * 4));
  }
  int* flag;
  CK(cudaMalloc(&flag, 4));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  S s{0.9f, 0.95f, 1e-8f, 0.1f, 0.1f, 0.05f, 0.1f, 0.05f, 4e-4f, 1.0f / 65536.0f};

  auto timeit = [&](const char* name, double bytes, auto launch) {
    for (int w = 0; w < 2; ++w) launch();
    CK(cudaDeviceSynchronize());
    const int reps = 8;
    CK(cudaEventRecord(e0));
    for (int r = 0; r < reps; ++r) launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    ms /= reps;
    std::printf("%-48s %8.3f ms  %8.1f GB/s\n", name, ms, bytes / (ms * 1e-3) / 1e9);
  };

#define COPY(LD, ST, U, T, PERSIST)                                                                   \
  {                                                                                                   \
    auto k = copy_k<LD, ST, U>;                                                                       \
    const int grid = PERSIST ? sms * occ(k, T) : (int)((n4 / U + T - 1) / T);                         \
    char nm[96];                                                                                      \
    std::snprintf(nm, sizeof nm, "copy ld%d st%d U%d T%d %s", LD, ST, U, T, PERSIST ? "persist" : "full"); \
    timeit(nm, 8.0 * n, [&] { k<<<grid, T>>>((const float4*)buf[0], (float4*)buf[1], n4); });      \
  }
  COPY(LD_DEF, ST_DEF, 1, 256, false)
  COPY(LD_DEF, ST_DEF, 2, 256, true)
  COPY(LD_CS, ST_CS, 2, 256, true)
  COPY(LD_NC_NA, ST_DEF, 2, 256, true)
  COPY(LD_CS, ST_CS, 4, 256, true)
  COPY(LD_CS, ST_CS, 4, 512, true)
  COPY(LD_NC_NA, ST_NA, 4, 256, true)

#define ADAM(LD, ST, U, T, PERSIST, MATH)                                                               \
  {                                                                                                     \
    auto k = adam_k<LD, ST, U, MATH>;                                                                   \
    const int grid = PERSIST ? sms * occ(k, T) : (int)((n4 / U + T - 1) / T);                          \
    char nm[96];                                                                                        \
    std::snprintf(nm, sizeof nm, "adam%s ld%d st%d U%d T%d %s", MATH ? "" : "-nomath", LD, ST, U, T,   \
                  PERSIST ? "persist" : "full");                                                        \
    timeit(nm, 28.0 * n, [&] {                                                                          \
      k<<<grid, T>>>((const float4*)buf[0], (const float4*)buf[1], (const float4*)buf[2],               \
                     (const float4*)buf[3], (float4*)buf[4], (float4*)buf[5], (float4*)buf[6], n4, s, flag); \
    });                                                                                                 \
  }
  ADAM(LD_CS, ST_CS, 2, 256, true, true)
  ADAM(LD_CS, ST_CS, 2, 256, true, false)
  ADAM(LD_DEF, ST_DEF, 2, 256, true, true)
  ADAM(LD_NC_NA, ST_DEF, 2, 256, true, true)
  ADAM(LD_NC_NA, ST_NA, 2, 256, true, true)
  ADAM(LD_CS, ST_CS, 1, 256, true, true)
  ADAM(LD_CS, ST_CS, 4, 256, true, true)
  ADAM(LD_CS, ST_CS, 2, 512, true, true)
  ADAM(LD_CS, ST_CS, 2, 128, true, true)
  ADAM(LD_CS, ST_CS, 2, 256, false, true)
  ADAM(LD_CS, ST_DEF, 2, 256, true, true)
  ADAM(LD_DEF, ST_CS, 2, 256, true, true)
  ADAM(LD_LU, ST_CS, 2, 256, true, true)
  return 0;
}
