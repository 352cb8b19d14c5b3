// tune_p2p.cu — NVLink peer-access micro-benchmark (development tool, not part
// of the product).  One process drives all visible GPUs with peer access
// enabled; every GPU moves `bytes` to/from every other GPU at once:
//   pull   kernel loads of peer memory (uint4, U in flight per thread)
//   push   kernel stores into peer memory
//   ce     cudaMemcpyPeerAsync, one stream per peer
// Reports per-GPU ingress / egress GB/s.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tune_p2p tune_p2p.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                             \
  do {                                                                                    \
    cudaError_t err_ = (x);                                                                  \
    if (err_ != cudaSuccess) {                                                               \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(err_), __FILE__, __LINE__); \
      std::exit(1);                                                                       \
    }                                                                                     \
  } while (0)

constexpr int kMaxG = 8;
struct Ptrs {
  uint4* p[kMaxG];
};

// every GPU pulls its slot from every peer: dst[j-th row] <- peer j's src (row me)
template <int U>
__global__ void pull_k(Ptrs src, uint4* dst, int g, int me, size_t n16) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride * U) {
    uint4 v[kMaxG][U];
#pragma unroll
    for (int j = 0; j < kMaxG; ++j)
      if (j < g && j != me)
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (i + u * stride < n16) v[j][u] = __ldcs(src.p[j] + (size_t)me * n16 + i + u * stride);
#pragma unroll
    for (int j = 0; j < kMaxG; ++j)
      if (j < g && j != me)
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (i + u * stride < n16) __stcs(dst + (size_t)j * n16 + i + u * stride, v[j][u]);
  }
}

// every GPU pushes its row to every peer: peer j's dst (row me) <- src
template <int U>
__global__ void push_k(const uint4* src, Ptrs dst, int g, int me, size_t n16) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i + u * stride < n16) v[u] = __ldcs(src + i + u * stride);
#pragma unroll
    for (int j = 0; j < kMaxG; ++j)
      if (j < g && j != me)
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (i + u * stride < n16) __stcs(dst.p[j] + (size_t)me * n16 + i + u * stride, v[u]);
  }
}

int main(int argc, char** argv) {
  int g = 0;
  CK(cudaGetDeviceCount(&g));
  if (g < 2) {
    std::printf("need >= 2 GPUs\n");
    return 0;
  }
  g = std::min(g, kMaxG);
  const size_t bytes = argc > 1 ? strtoull(argv[1], nullptr, 10) : (size_t(512) << 20);  // per peer pair
  const size_t n16 = bytes / 16;
  std::vector<uint4*> src(g), dst(g);
  std::vector<cudaStream_t> st(g);
  std::vector<std::vector<cudaStream_t>> ps(g, std::vector<cudaStream_t>(g));
  for (int d = 0; d < g; ++d) {  // every primary context exists before peers are enabled
    CK(cudaSetDevice(d));
    CK(cudaFree(nullptr));
  }
  for (int d = 0; d < g; ++d) {
    CK(cudaSetDevice(d));
    for (int e = 0; e < g; ++e)
      if (e != d) CK(cudaDeviceEnablePeerAccess(e, 0));
    CK(cudaMalloc(&src[d], bytes * g));
    CK(cudaMalloc(&dst[d], bytes * g));
    CK(cudaMemset(src[d], d + 1, bytes * g));
    CK(cudaStreamCreate(&st[d]));
    for (int e = 0; e < g; ++e) CK(cudaStreamCreate(&ps[d][e]));
  }
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  Ptrs all_src{}, all_dst{};
  for (int d = 0; d < g; ++d) {
    all_src.p[d] = src[d];
    all_dst.p[d] = dst[d];
  }
  auto sync_all = [&] {
    for (int d = 0; d < g; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaDeviceSynchronize());
    }
  };
  auto run = [&](const char* name, auto launch) {
    launch();
    sync_all();
    cudaEvent_t a, b;
    CK(cudaSetDevice(0));
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    const int reps = 5;
    sync_all();
    CK(cudaSetDevice(0));
    CK(cudaEventRecord(a, st[0]));
    for (int r = 0; r < reps; ++r) launch();
    sync_all();
    CK(cudaSetDevice(0));
    CK(cudaEventRecord(b, st[0]));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    ms /= reps;
    const double per_gpu = (double)bytes * (g - 1);
    std::printf("%-36s g=%d  %8.3f ms  %7.1f GB/s per GPU per direction\n", name, g, ms, per_gpu / (ms * 1e-3) / 1e9);
  };
  for (int ctas : {148, 296, 592, 1184}) {
    char nm[64];
    std::snprintf(nm, sizeof nm, "pull U1 ctas=%d", ctas);
    run(nm, [&] {
      for (int d = 0; d < g; ++d) {
        CK(cudaSetDevice(d));
        pull_k<1><<<ctas, 256, 0, st[d]>>>(all_src, dst[d], g, d, n16);
      }
    });
    std::snprintf(nm, sizeof nm, "pull U4 ctas=%d", ctas);
    run(nm, [&] {
      for (int d = 0; d < g; ++d) {
        CK(cudaSetDevice(d));
        pull_k<4><<<ctas, 256, 0, st[d]>>>(all_src, dst[d], g, d, n16);
      }
    });
    std::snprintf(nm, sizeof nm, "push U1 ctas=%d", ctas);
    run(nm, [&] {
      for (int d = 0; d < g; ++d) {
        CK(cudaSetDevice(d));
        push_k<1><<<ctas, 256, 0, st[d]>>>(src[d], all_dst, g, d, n16);
      }
    });
    std::snprintf(nm, sizeof nm, "push U4 ctas=%d", ctas);
    run(nm, [&] {
      for (int d = 0; d < g; ++d) {
        CK(cudaSetDevice(d));
        push_k<4><<<ctas, 256, 0, st[d]>>>(src[d], all_dst, g, d, n16);
      }
    });
  }
  run("ce pull (memcpyPeer, stream per peer)", [&] {
    for (int d = 0; d < g; ++d) {
      CK(cudaSetDevice(d));
      for (int e = 0; e < g; ++e)
        if (e != d)
          CK(cudaMemcpyPeerAsync(dst[d] + (size_t)e * n16, d, src[e] + (size_t)d * n16, e, bytes, ps[d][e]));
    }
  });
  run("ce push (memcpyPeer, stream per peer)", [&] {
    for (int d = 0; d < g; ++d) {
      CK(cudaSetDevice(d));
      for (int e = 0; e < g; ++e)
        if (e != d)
          CK(cudaMemcpyPeerAsync(dst[e] + (size_t)d * n16, e, src[d], d, bytes, ps[d][e]));
    }
  });
  return 0;
}
