// Measurement utilities exported through the C-ABI (used by bench.py):
//  * vx_probe_pipe_rates: FP64 DADD and FP32 FADD issue rates of this GPU,
//    the roofline denominator for the ball kernel's evaluations
//    (MEASURED_PEAKS.json carries only HBM and bf16 figures).
//  * vx_label_fingerprint: SURVEY.md App. B FNV-style label fingerprint.
//  * vx_probe_exact_arith: the call-free exact sqrt / division of the eval
//    kernel (vx_internal.cuh) against __dsqrt_rn / __ddiv_rn, bit for bit.
#include <cuda_runtime.h>

#include "voxellate_b200.h"
#include "vx_internal.cuh"

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

__device__ __forceinline__ unsigned long long splitmix(unsigned long long& z) {
  z += 0x9e3779b97f4a7c15ull;
  unsigned long long x = z;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// random doubles with uniform exponent in [e0, e1) and uniform mantissa
__device__ __forceinline__ double rand_exp(unsigned long long& z, int e0, int e1) {
  const unsigned long long r = splitmix(z);
  const int e = e0 + (int)((r >> 52) % (unsigned)(e1 - e0));
  return __longlong_as_double(((unsigned long long)(e + 1023) << 52) | (r & 0xfffffffffffffull));
}

__global__ void exact_arith_kernel(unsigned long long n, unsigned long long seed, double G,
                                   unsigned long long* bad) {
  const double y = __drcp_rn(G);
  unsigned long long nb_sqrt = 0, nb_div = 0;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    unsigned long long z = seed ^ (i * 0xd1b54a32d192ed03ull);
    // squared distances: three squared coordinate differences (uniform mantissas,
    // exponents over the whole fast range), and plain doubles over the range
    double x;
    if (i & 1) {
      const double u = rand_exp(z, -174, 101), v = rand_exp(z, -174, 101), w = rand_exp(z, -174, 101);
      x = __dadd_rn(__dadd_rn(__dmul_rn(w, w), __dmul_rn(v, v)), __dmul_rn(u, u));
    } else {
      x = rand_exp(z, -348, 210);
    }
    if ((i & 1023) == 0) x = 0.0;  // exact zeros (a site on a voxel centre)
    if (__double_as_longlong(vxb::sqrt_rn_nc(x)) != __double_as_longlong(__dsqrt_rn(x))) ++nb_sqrt;
    const double a = (i & 2) ? __dsqrt_rn(x) : x;
    if (__double_as_longlong(vxb::div_rn_nc(a, G, y)) != __double_as_longlong(__ddiv_rn(a, G))) ++nb_div;
  }
  if (nb_sqrt) atomicAdd(&bad[0], nb_sqrt);
  if (nb_div) atomicAdd(&bad[1], nb_div);
}

}  // namespace

extern "C" int vx_probe_exact_arith(int device, uint64_t n, uint64_t seed, double growth,
                                    uint64_t* sqrt_mismatches, uint64_t* div_mismatches) {
  int prev = 0;
  cudaGetDevice(&prev);
  if (cudaSetDevice(device) != cudaSuccess) return VX_ECUDA;
  unsigned long long* bad = nullptr;
  if (cudaMalloc(&bad, 2 * sizeof(unsigned long long)) != cudaSuccess) return VX_ECUDA;
  cudaMemset(bad, 0, 2 * sizeof(unsigned long long));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  exact_arith_kernel<<<sms * 8, 256>>>(n, seed, growth, bad);
  unsigned long long h[2] = {0, 0};
  const cudaError_t e = cudaMemcpy(h, bad, sizeof(h), cudaMemcpyDeviceToHost);
  cudaFree(bad);
  cudaSetDevice(prev);
  if (e != cudaSuccess) return VX_ECUDA;
  if (sqrt_mismatches) *sqrt_mismatches = h[0];
  if (div_mismatches) *div_mismatches = h[1];
  return VX_OK;
}

// H2D copy time of a host buffer through this library's runtime (diagnostics)
extern "C" int vx_probe_h2d(int device, const void* host, uint64_t bytes, int use_null_stream, float* ms_out) {
  int prev = 0;
  cudaGetDevice(&prev);
  if (cudaSetDevice(device) != cudaSuccess) return VX_ECUDA;
  void* d = nullptr;
  if (cudaMalloc(&d, bytes) != cudaSuccess) return VX_ECUDA;
  cudaStream_t s = nullptr;
  if (!use_null_stream) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0, s);
    cudaMemcpyAsync(d, host, bytes, cudaMemcpyHostToDevice, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (s) cudaStreamDestroy(s);
  cudaFree(d);
  cudaSetDevice(prev);
  if (ms_out) *ms_out = best;
  return cudaGetLastError() == cudaSuccess ? VX_OK : VX_ECUDA;
}

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
