// p2p_probe.cu — report what peer access this box allows (development tool).
#include <cuda_runtime.h>
#include <cstdio>
int main() {
  int g = 0;
  cudaGetDeviceCount(&g);
  for (int a = 0; a < g; ++a)
    for (int b = 0; b < g; ++b) {
      if (a == b) continue;
      int can = -1, acc = -1, atom = -1, perf = -1;
      cudaDeviceCanAccessPeer(&can, a, b);
      cudaDeviceGetP2PAttribute(&acc, cudaDevP2PAttrAccessSupported, a, b);
      cudaDeviceGetP2PAttribute(&atom, cudaDevP2PAttrNativeAtomicSupported, a, b);
      cudaDeviceGetP2PAttribute(&perf, cudaDevP2PAttrPerformanceRank, a, b);
      cudaSetDevice(a);
      cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      std::printf("%d->%d canAccessPeer=%d accessSupported=%d atomics=%d perfRank=%d enable=%s\n", a, b, can, acc,
                  atom, perf, cudaGetErrorString(e));
    }
  return 0;
}
