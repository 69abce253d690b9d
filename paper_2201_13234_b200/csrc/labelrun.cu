// Run-coded label transport for host-buffer calls.
//
// A host-buffer call's cost is the PCIe copy of the int32 label image (4 GB at
// cfg5, ~55 GB/s: 73 ms against 5.4 ms of labelling).  Label images are runs
// of equal labels along x (a Voronoi cell spans ~7 voxels of a row at cfg5),
// so each labelled z-chunk is coded on the device as runs -- per x-row an
// (offset, count) record, per run its label (int32) and first x (uint16), or,
// when the label and x fit 32 bits together (xbits = bits of n0 - 1, labels
// below 2^(32 - xbits): cfg5's 10^6 sites in rows of 1000), one packed word
// `label << xbits | x` -- only the runs cross PCIe (~0.6 GB at cfg5 packed,
// ~0.9 GB unpacked), and host threads expand them
// into the caller's buffer row by row with streaming stores while the next
// chunk's runs are in flight.  The caller's image is the same int32 array as
// before; a chunk whose runs would not fit 1/4 of its voxels (average run
// < 4 voxels) is copied raw instead.
//
// The reference writes its image into host memory directly
// (`tessellate.cpp:160-174`, `make_result`); this is only how the same bytes
// reach the caller's buffer.
#include <cuda_runtime.h>


#include "vx_internal.cuh"

namespace vxb {

namespace {

constexpr int kRowsPerBlock = 8;  // one warp per x-row

// Per x-row: warp-wide run starts (label differs from the voxel before it) by
// ballot; one global atomic per block reserves the block's run slots.
__global__ void __launch_bounds__(32 * kRowsPerBlock)
    run_encode_kernel(const int* __restrict__ lab, long long nrows, int n0, int2* __restrict__ rows,
                      int* __restrict__ rlab, unsigned short* __restrict__ rx, long long cap,
                      unsigned long long* __restrict__ cnt, int xbits) {
  __shared__ int wc[kRowsPerBlock];
  __shared__ unsigned long long sbase;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long r = (long long)blockIdx.x * kRowsPerBlock + w;
  const int* row = lab + r * (long long)n0;
  int c = 0;
  if (r < nrows) {
    int prev = 0;
    unsigned wide = 0;  // packed mode: a label that does not fit sends the chunk raw
    for (int x0 = 0; x0 < n0; x0 += 32) {
      const int x = x0 + lane;
      const int v = x < n0 ? __ldg(row + x) : 0;
      wide |= (unsigned)v;
      int up = __shfl_up_sync(0xffffffffu, v, 1);
      if (lane == 0) up = prev;
      c += __popc(__ballot_sync(0xffffffffu, x < n0 && (x == 0 || v != up)));
      prev = __shfl_sync(0xffffffffu, v, 31);
    }
    if (xbits > 0 && __any_sync(0xffffffffu, (wide >> (32 - xbits)) != 0u)) c = -1;
  }
  if (lane == 0) wc[w] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long tot = 0;
    for (int i = 0; i < kRowsPerBlock; ++i) tot += wc[i] < 0 ? (1ull << 40) : (unsigned long long)wc[i];
    sbase = atomicAdd(cnt, tot);
  }
  __syncthreads();
  if (r >= nrows) return;
  unsigned long long base = sbase;
  for (int i = 0; i < w; ++i) base += wc[i] < 0 ? (1ull << 40) : (unsigned long long)wc[i];
  if (c < 0) c = 0, base = 1ull << 40;
  if (lane == 0) rows[r] = make_int2((int)min(base, (unsigned long long)cap), c);
  if (base + (unsigned long long)c > (unsigned long long)cap) return;  // chunk goes raw
  long long k = (long long)base;
  int prev = 0;
  const unsigned lt = (1u << lane) - 1u;
  for (int x0 = 0; x0 < n0; x0 += 32) {
    const int x = x0 + lane;
    const int v = x < n0 ? row[x] : 0;
    int up = __shfl_up_sync(0xffffffffu, v, 1);
    if (lane == 0) up = prev;
    const bool b = x < n0 && (x == 0 || v != up);
    const unsigned m = __ballot_sync(0xffffffffu, b);
    if (b) {
      const long long o = k + __popc(m & lt);
      if (xbits > 0) {
        rlab[o] = (int)(((unsigned)v << xbits) | (unsigned)x);
      } else {
        rlab[o] = v;
        rx[o] = (unsigned short)x;
      }
    }
    k += __popc(m);
    prev = __shfl_sync(0xffffffffu, v, 31);
  }
}

// The chunk's run count into mapped host memory: the host reads it without a
// copy-engine transfer (which would queue behind the previous chunks' runs).
__global__ void run_publish_kernel(const unsigned long long* __restrict__ cnt, volatile unsigned long long* host_cnt) {
  *host_cnt = *cnt;
  __threadfence_system();
}

}  // namespace

int launch_run_publish(const unsigned long long* cnt, unsigned long long* host_cnt, cudaStream_t st) {
  run_publish_kernel<<<1, 1, 0, st>>>(cnt, host_cnt);
  return 1;
}

int launch_run_encode(const int* lab, long long nrows, int n0, int2* rows, int* rlab, unsigned short* rx,
                      long long cap, unsigned long long* cnt, int xbits, cudaStream_t st) {
  if (nrows <= 0) return 0;
  cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), st);
  const long long nb = (nrows + kRowsPerBlock - 1) / kRowsPerBlock;
  run_encode_kernel<<<(unsigned)nb, 32 * kRowsPerBlock, 0, st>>>(lab, nrows, n0, rows, rlab, rx, cap, cnt, xbits);
  return 1;
}

}  // namespace vxb
