// K0 ingest + K1 site binning.
//
// The reference has no spatial index (its step 1 scatters each site's ball,
// ball_scan.hpp:55-124).  The gather-form engine needs one: sites are sorted
// by the id of a uniform cell grid (axis 0 fastest, like the voxels) with a
// stable LSD radix sort, so each cell -- and each x-row of cells -- is a
// contiguous, ascending-site-index range of the SoA arrays bx/by/bz/bt/bidx.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <cstdlib>

#include "vx_internal.cuh"

namespace vxb {

// Copies the caller's d-interleaved positions into the internal 3-D AoS
// buffer (padding axes >= d with the exact mid-coordinate 0.5), converts
// Laguerre weights to times t = -(w)/G (sites.cpp:101), and checks
// SiteSet::validate's position rule (sites.cpp:54-57): finite, 0 < x < L.
__global__ void ingest_kernel(Geo g, Len16 len, int dim_in, const double* __restrict__ pos_in,
                              const double* __restrict__ times_in,
                              const double* __restrict__ weights_in, double* __restrict__ p3,
                              double* __restrict__ t_out, DevCounters* ctr) {
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= g.n_sites) return;
  bool bad = false;
  for (int a = 0; a < dim_in; ++a) {
    const double v = pos_in[s * dim_in + a];
    bad |= !(isfinite(v) && v > 0.0 && v < len.L[a]);
  }
  if (p3 && dim_in <= 3) {
    double q[3] = {0.5, 0.5, 0.5};
    for (int a = 0; a < dim_in; ++a) q[g.emb[a]] = pos_in[s * dim_in + a];
#pragma unroll
    for (int a = 0; a < 3; ++a) p3[3 * s + a] = q[a];
  }
  if (g.kind != kVoronoi && t_out) {
    double t;
    if (times_in) t = times_in[s];
    else t = __ddiv_rn(-weights_in[s], g.growth);
    t_out[s] = t;
  }
  if (bad) atomicOr(&ctr->bad_site, 1u);
}

__device__ __forceinline__ int cell_of(double v, double inv_cw, int m) {
  int c = (int)(v * inv_cw);
  return c < 0 ? 0 : (c >= m ? m - 1 : c);
}

__global__ void keys_kernel(Geo g, const double* __restrict__ p3, const double* __restrict__ t,
                            const uint8_t* __restrict__ dropped, unsigned* __restrict__ keys,
                            int* __restrict__ vals, int* __restrict__ counts, DevParams* prm,
                            unsigned* ctr_bad) {
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  bool alive = false;
  double tv = 0.0;
  if (s < g.n_sites) {
    if (g.validate_in_keys) {  // sites.cpp:54-57: finite, strictly inside (0, L)
      bool bad = false;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double v = p3[3 * s + a];
        bad |= !(isfinite(v) && v > 0.0 && v < g.L[a]);
      }
      if (bad) atomicOr(&ctr_bad[0], 1u);
    }
    alive = !(dropped && dropped[s]);
    if (alive && g.win_on) {  // slab window (multi-GPU ranks): bin the slab's neighbourhood only
      double u = p3[3 * s + 2] - g.win_c;
      if (g.periodic) u -= floor(u * g.invL[2] + 0.5) * g.L[2];
      alive = fabs(u) <= g.win_half;
    }
    unsigned key = (unsigned)g.n_cells;
    if (alive) {
      const int cx = cell_of(p3[3 * s + 0], g.inv_cw[0], g.m[0]);
      const int cy = cell_of(p3[3 * s + 1], g.inv_cw[1], g.m[1]);
      const int cz = cell_of(p3[3 * s + 2], g.inv_cw[2], g.m[2]);
      key = (unsigned)(cx + (long long)g.m[0] * (cy + (long long)g.m[1] * cz));
      if (t) tv = t[s];
      atomicAdd(&counts[key], 1);  // sites per cell; their exclusive scan is cell_start
    }
    keys[s] = key;
    vals[s] = (int)s;
  }
  if (t) {  // min / max birth time over alive sites
    unsigned long long kmin = alive ? dkey(tv) : ~0ull, kmax = alive ? dkey(tv) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
      kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    }
    if ((threadIdx.x & 31) == 0) {
      if (kmin != ~0ull) atomicMin(&prm->tmin_key, kmin);
      if (kmax != 0ull) atomicMax(&prm->tmax_key, kmax);
    }
  }
}

// Counting sort (Voronoi): each alive site takes the next free slot of its cell
// (cell_start = exclusive scan of the counts).  The order inside a cell is
// then arbitrary -- every consumer orders candidates by site index (the ball
// kernels' rank sort) or compares (prox, index) lexicographically (shell,
// sub-brick shell), and pruning is an OR -- so labels do not depend on it.
__global__ void place_kernel(long long n, const unsigned* __restrict__ keys, const int* __restrict__ cell_start,
                             int* __restrict__ fill, int* __restrict__ vals_out, long long n_cells) {
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= n) return;
  const unsigned k = keys[s];
  if (k >= (unsigned)n_cells) return;  // dropped / outside the slab window
  vals_out[cell_start[k] + atomicAdd(&fill[k], 1)] = (int)s;
}

__global__ void gather_kernel(long long n, const int* __restrict__ vals,
                              const double* __restrict__ p3, const double* __restrict__ t,
                              double* __restrict__ bx, double* __restrict__ by,
                              double* __restrict__ bz, double* __restrict__ bt,
                              int* __restrict__ bidx, float4* __restrict__ f4,
                              const int* __restrict__ cell_start, long long n_cells, DevCounters* ctr) {
  const long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long n_alive = cell_start[n_cells];
  if (p == 0) ctr->n_alive = (unsigned long long)n_alive;  // dropped sites sort last (radix) / are not placed
  if (p >= n || p >= n_alive) return;
  const int s = vals[p];
  const double x = p3[3 * (long long)s + 0], y = p3[3 * (long long)s + 1],
               z = p3[3 * (long long)s + 2];
  bx[p] = x;
  by[p] = y;
  bz[p] = z;
  const double tv = t ? t[s] : 0.0;
  if (t) bt[p] = tv;
  bidx[p] = s;
  if (f4) f4[p] = make_float4((float)x, (float)y, (float)z, (float)tv);
}

static int key_bits(long long n_cells) {
  int b = 1;
  while ((1ll << b) <= n_cells) ++b;
  return b;
}

size_t bin_tmp_bytes(long long n_sites, long long n_cells) {
  size_t bytes = 0, scan = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (unsigned*)nullptr, (unsigned*)nullptr,
                                  (int*)nullptr, (int*)nullptr, (int)n_sites, 0, 32);
  cub::DeviceScan::ExclusiveSum(nullptr, scan, (int*)nullptr, (int*)nullptr, (int)(n_cells + 1));
  return bytes > scan ? bytes : scan;
}

int launch_ingest(const Geo& g, const Len16& len, int dim_in, const double* pos_in,
                  const double* times_in, const double* weights_in, double* p3, double* t_out,
                  DevCounters* ctr, cudaStream_t st) {
  const int T = 256;
  ingest_kernel<<<(unsigned)((g.n_sites + T - 1) / T), T, 0, st>>>(g, len, dim_in, pos_in, times_in,
                                                                  weights_in, p3, t_out, ctr);
  return 1;
}

int launch_bin(const Geo& g, const double* p3, const double* t, const uint8_t* dropped,
               void* cub_tmp, size_t cub_tmp_bytes, unsigned* keys_a, unsigned* keys_b,
               int* vals_a, int* vals_b, double* bx, double* by, double* bz, double* bt,
               int* bidx, float4* f4, int* cell_start, int* fill, DevParams* prm, DevCounters* ctr,
               cudaStream_t st) {
  const int T = 256;
  const unsigned nb = (unsigned)((g.n_sites + T - 1) / T);
  // cell_start = exclusive scan of the per-cell site counts (counted in place)
  cudaError_t e = cudaMemsetAsync(cell_start, 0, sizeof(int) * (size_t)(g.n_cells + 1), st);
  if (e != cudaSuccess) return -1000 - (int)e;
  keys_kernel<<<nb, T, 0, st>>>(g, p3, t, dropped, keys_a, vals_a, cell_start, prm, &ctr->bad_site);
  size_t bytes = cub_tmp_bytes;
  // counting sort (no radix passes); VX_RADIX_BIN=1: the stable radix sort
  static const bool radix_env = std::getenv("VX_RADIX_BIN") != nullptr;
  const bool counting = fill != nullptr && !radix_env;
  int passes = 0;
  if (!counting) {
    // stable: equal cells keep ascending site order
    e = cub::DeviceRadixSort::SortPairs(cub_tmp, bytes, keys_a, keys_b, vals_a, vals_b,
                                        (int)g.n_sites, 0, key_bits(g.n_cells), st);
    if (e != cudaSuccess) return -1000 - (int)e;
    passes = 2 * ((key_bits(g.n_cells) + 7) / 8);
  }
  bytes = cub_tmp_bytes;
  e = cub::DeviceScan::ExclusiveSum(cub_tmp, bytes, cell_start, cell_start, (int)(g.n_cells + 1), st);
  if (e != cudaSuccess) return -1000 - (int)e;
  if (counting) {
    e = cudaMemsetAsync(fill, 0, sizeof(int) * (size_t)g.n_cells, st);
    if (e != cudaSuccess) return -1000 - (int)e;
    place_kernel<<<nb, T, 0, st>>>(g.n_sites, keys_a, cell_start, fill, vals_b, g.n_cells);
    passes = 1;
  }
  gather_kernel<<<nb, T, 0, st>>>(g.n_sites, vals_b, p3, t, bx, by, bz, bt, bidx, f4, cell_start, g.n_cells,
                                  ctr);
  return 4 + passes;  // ours + the sort / placement and scan passes (approx.)
}

}  // namespace vxb
