// kernels.cu — DiLoCo kernels for B200 (sm_100a): the SM count and the
// host-staged / setup kernels; the hot path is kernels_inner.cu (K1),
// kernels_outer.cu (K2, K4) and kernels_fold.cu (K3).
//
// Memory-bound elementwise and reduction work: no tensor cores.  The hot
// kernels use the streaming-window distribution described in kernels.cuh: one
// CTA per 256*U consecutive 128-bit vectors, evict-first (.cs) loads/stores, a
// scalar tail on CTA 0, and CTA-level OR reductions (__syncthreads_or + one
// atomicOr per CTA that saw a non-finite value) for the global flags.
//
// Arithmetic follows the reference's FP32 evaluation order exactly (see
// common.cuh); citations are to /root/reference/proj.
#include <algorithm>
#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "device.cuh"
#include "kernels.cuh"

namespace dlc {

namespace {

int g_sms = 0;

// =============================================================================
// elementwise helpers (host-staged API, synthetic inputs, probes)
// =============================================================================

__global__ void __launch_bounds__(kThreads) axpy_kernel(float alpha, const float* x, const float* y, float* out,
                                                        size_t n) {
  for (size_t e = gtid(); e < n; e += gstride()) out[e] = __fadd_rn(y[e], __fmul_rn(alpha, x[e]));
}

__global__ void __launch_bounds__(kThreads) encode_kernel(const float* x, uint16_t* out, int* flag, size_t n) {
  bool bad = false;
  for (size_t e = gtid(); e < n; e += gstride()) {
    const uint16_t h = fp16_encode(x[e]);
    bad |= fp16_nonfinite(h);
    out[e] = h;
  }
  if (flag) block_or_flag(bad, flag);
}

__global__ void __launch_bounds__(kThreads) decode_kernel(const uint16_t* b, float* out, size_t n) {
  for (size_t e = gtid(); e < n; e += gstride()) out[e] = fp16_decode(b[e]);
}

__global__ void __launch_bounds__(kThreads) nonfinite_kernel(const float* x, int* flag, size_t n) {
  bool bad = false;
  for (size_t e = gtid(); e < n; e += gstride()) bad |= !finite_f(x[e]);
  block_or_flag(bad, flag);
}

__global__ void __launch_bounds__(kThreads) nonfinite_codes_kernel(const uint16_t* b, int* flag, size_t n) {
  bool bad = false;
  for (size_t e = gtid(); e < n; e += gstride()) bad |= fp16_nonfinite(b[e]);
  block_or_flag(bad, flag);
}

// reduce.cpp:46-89 for any k: contributions visited in index order.
__global__ void __launch_bounds__(kThreads) fold_many_kernel(const float* const* ptrs, size_t k, int fp16,
                                                             float* out, size_t n) {
  const MeanDiv divisor = mean_div(k);
  for (size_t e = gtid(); e < n; e += gstride()) {
    float acc = ptrs[0][e];
    if (fp16) acc = fp16_decode(fp16_encode(acc));
    for (size_t j = 1; j < k; ++j) {
      const float x = ptrs[j][e];
      acc = __fadd_rn(acc, fp16 ? fp16_decode(fp16_encode(x)) : x);
    }
    const float mean = div_mean(acc, divisor);
    out[e] = fp16 ? fp16_decode(fp16_encode(mean)) : mean;
  }
}

__global__ void __launch_bounds__(kThreads) unscale_kernel(const float* g, float inv, float* out, int* flag,
                                                           size_t n) {
  bool bad = false;
  for (size_t e = gtid(); e < n; e += gstride()) {
    const float y = __fmul_rn(g[e], inv);
    bad |= !finite_f(y);
    out[e] = y;
  }
  block_or_flag(bad, flag);
}

__global__ void __launch_bounds__(kThreads) scale_gradient_kernel(const float* g, const DevState* st, float* out,
                                                                  size_t n) {
  const float s = st->scale;
  const size_t n4 = n / 4, j = gtid();
  if (j < n4) {
    const float4 x = ld_stream(reinterpret_cast<const float4*>(g) + j);
    st_stream(reinterpret_cast<float4*>(out) + j,
              make_float4(__fmul_rn(x.x, s), __fmul_rn(x.y, s), __fmul_rn(x.z, s), __fmul_rn(x.w, s)));
  }
  if (blockIdx.x == 0 && threadIdx.x < n - n4 * 4) out[n4 * 4 + threadIdx.x] = __fmul_rn(g[n4 * 4 + threadIdx.x], s);
}

__global__ void __launch_bounds__(kThreads) rng_fill_kernel(uint64_t key, uint64_t first, float lo, float hi,
                                                            float* out, size_t n) {
  for (size_t e = gtid(); e < n; e += gstride()) out[e] = rng_uniform_at(key, first + e, lo, hi);
}

__global__ void __launch_bounds__(kThreads) rng_perturb_kernel(const float* tt, uint64_t key, float lo, float hi,
                                                               float* out, size_t n) {
  for (size_t e = gtid(); e < n; e += gstride()) out[e] = __fsub_rn(tt[e], rng_uniform_at(key, e, lo, hi));
}

__global__ void __launch_bounds__(kThreads) encode_bits_kernel(uint32_t start, uint16_t* out, size_t n) {
  for (size_t e = gtid(); e < n; e += gstride()) out[e] = fp16_encode(__uint_as_float(start + (uint32_t)e));
}

__global__ void __launch_bounds__(kThreads) copy_kernel(const float* src, float* dst, size_t n) {
  const size_t n4 = n / 4, j = gtid();
  if (j < n4) st_stream(reinterpret_cast<float4*>(dst) + j, ld_stream(reinterpret_cast<const float4*>(src) + j));
  if (blockIdx.x == 0 && threadIdx.x < n - n4 * 4) dst[n4 * 4 + threadIdx.x] = src[n4 * 4 + threadIdx.x];
}

}  // namespace

int num_sms() {
  if (g_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms <= 0) g_sms = 148;
  }
  return g_sms;
}

void launch_axpy(float alpha, const float* x, const float* y, float* out, size_t n, cudaStream_t s) {
  if (n == 0) return;
  axpy_kernel<<<grid_persist(axpy_kernel, n), kThreads, 0, s>>>(alpha, x, y, out, n);
}

void launch_encode(const float* x, uint16_t* out, int* flag, size_t n, cudaStream_t s) {
  if (n == 0) return;
  encode_kernel<<<grid_persist(encode_kernel, n), kThreads, 0, s>>>(x, out, flag, n);
}

void launch_decode(const uint16_t* b, float* out, size_t n, cudaStream_t s) {
  if (n == 0) return;
  decode_kernel<<<grid_persist(decode_kernel, n), kThreads, 0, s>>>(b, out, n);
}

void launch_nonfinite(const float* x, int* flag, size_t n, cudaStream_t s) {
  if (n == 0) return;
  nonfinite_kernel<<<grid_persist(nonfinite_kernel, n), kThreads, 0, s>>>(x, flag, n);
}

void launch_nonfinite_codes(const uint16_t* b, int* flag, size_t n, cudaStream_t s) {
  if (n == 0) return;
  nonfinite_codes_kernel<<<grid_persist(nonfinite_codes_kernel, n), kThreads, 0, s>>>(b, flag, n);
}

void launch_fold_many(const float* const* ptrs, size_t k, int fp16, float* out, size_t n, cudaStream_t s) {
  if (n == 0 || k == 0) return;
  fold_many_kernel<<<grid_persist(fold_many_kernel, n), kThreads, 0, s>>>(ptrs, k, fp16, out, n);
}

void launch_unscale(const float* g, float inv, float* out, int* flag, size_t n, cudaStream_t s) {
  if (n == 0) return;
  unscale_kernel<<<grid_persist(unscale_kernel, n), kThreads, 0, s>>>(g, inv, out, flag, n);
}

void launch_scale_gradient(const float* g, const DevState* st, float* out, size_t n, cudaStream_t s) {
  scale_gradient_kernel<<<grid_window<1>(n / 4), kThreads, 0, s>>>(g, st, out, n);
}

void launch_rng_fill(uint64_t key, uint64_t first, float lo, float hi, float* out, size_t n, cudaStream_t s) {
  if (n == 0) return;
  rng_fill_kernel<<<grid_persist(rng_fill_kernel, n), kThreads, 0, s>>>(key, first, lo, hi, out, n);
}

void launch_rng_perturb(const float* tt, uint64_t key, float lo, float hi, float* out, size_t n,
                        cudaStream_t s) {
  if (n == 0) return;
  rng_perturb_kernel<<<grid_persist(rng_perturb_kernel, n), kThreads, 0, s>>>(tt, key, lo, hi, out, n);
}

void launch_encode_bits_range(uint32_t start, uint16_t* out, size_t n, cudaStream_t s) {
  if (n == 0) return;
  encode_bits_kernel<<<grid_persist(encode_bits_kernel, n), kThreads, 0, s>>>(start, out, n);
}

void launch_copy(const float* src, float* dst, size_t n, cudaStream_t s) {
  if (n == 0) return;
  copy_kernel<<<grid_window<1>(n / 4), kThreads, 0, s>>>(src, dst, n);
}

namespace {
__global__ void or_word_kernel(int* dst, const int* src) { *dst |= *src; }
}  // namespace

void launch_or_word(int* dst, const int* src, cudaStream_t s) { or_word_kernel<<<1, 1, 0, s>>>(dst, src); }

}  // namespace dlc
