// Measurement utilities exported through the C-ABI (used by bench.py):
//  * vx_probe_pipe_rates: FP64 DADD and FP32 FADD issue rates of this GPU,
//    the roofline denominator for the ball kernel's evaluations
//    (MEASURED_PEAKS.json carries only HBM and bf16 figures).
//  * vx_label_fingerprint: SURVEY.md App. B FNV-style label fingerprint.
#include <cuda_runtime.h>

#include "voxellate_b200.h"

namespace {

constexpr int kIters = 4096;
constexpr int kChains = 8;

template <class T>
__global__ void add_chain_kernel(T* out, T seed) {
  T a[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) a[c] = seed + (T)(threadIdx.x + c);
  const T inc = seed * (T)1e-9;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) a[c] = a[c] + inc;
  }
  T s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += a[c];
  if (s == (T)-1) out[0] = s;  // never true; keeps the chains alive
}

template <class T>
double rate(int device) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  T* out = nullptr;
  if (cudaMalloc(&out, sizeof(T)) != cudaSuccess) return 0.0;
  const int blocks = sms * 8, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  add_chain_kernel<T><<<blocks, threads>>>(out, (T)1.0);  // warm-up (clocks up)
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    add_chain_kernel<T><<<blocks, threads>>>(out, (T)1.0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  const double ops = (double)blocks * threads * kIters * kChains;
  return ops / (best * 1e-3);
}

}  // namespace

extern "C" int vx_probe_pipe_rates(int device, double* dadd_per_s, double* fadd_per_s) {
  int prev = 0;
  cudaGetDevice(&prev);
  if (cudaSetDevice(device) != cudaSuccess) return VX_ECUDA;
  if (dadd_per_s) *dadd_per_s = rate<double>(device);
  if (fadd_per_s) *fadd_per_s = rate<float>(device);
  const cudaError_t e = cudaGetLastError();
  cudaSetDevice(prev);
  return e == cudaSuccess ? VX_OK : VX_ECUDA;
}

extern "C" uint64_t vx_label_fingerprint(const int32_t* labels, int64_t n) {
  uint64_t h = 1469598103934665603ull;
  for (int64_t i = 0; i < n; ++i) {
    h ^= (uint32_t)labels[i];
    h *= 1099511628211ull;
  }
  return h;
}
