// K4: widening-shell exact search for the voxels the ball phase left
// unresolved (reference step 2: resolve_voxels_impl<K,P> with
// only_unassigned=true, tessellate.cpp:36-75, an all-sites scan per voxel).
//
// One warp per voxel.  Ring r is the set of cells at Chebyshev distance r from
// the voxel's cell (periodic axes wrap; an axis whose window reaches the whole
// period is "full").  Each lane evaluates the exact reference ranking value of
// the sites in its cells and keeps the lexicographic minimum of (prox, index)
// -- the order-independent form of the reference's ascending strict-< scan.
// After each ring the search stops once a conservative lower bound of prox over
// every site outside the scanned window exceeds the current best (strictly, so
// a tie with a lower-index site further out is still found).
//
// The unresolved list comes from the ball kernel's fused compaction.  If it
// overflowed its capacity, the kernel instead compacts on the fly from the
// label image (sentinel -1), which needs no host round trip.
#include "vx_internal.cuh"

namespace vxb {

constexpr int kShellThreads = 256;

__device__ __forceinline__ long long wrapm(long long c, long long m) {
  const long long r = c % m;
  return r < 0 ? r + m : r;
}
// c in (-m, 2m): the periodic cell index in [0, m)
__device__ __forceinline__ int wrap1(int c, int m) { return c < 0 ? c + m : (c >= m ? c - m : c); }

// Few sites (n_alive <= kShellBrute): every alive site, 32 lanes at a time, is
// cheaper than the ring bookkeeping; the same exact (prox, index) minimum.
constexpr int kShellBrute = 2048;

template <int KIND, bool PER>
__device__ void shell_all(const Geo& g, const Bins& bins, int n_alive, long long lin, int* labels,
                          double* dist, unsigned long long* hist, unsigned long long* evals) {
  const int lane = threadIdx.x & 31;
  const long long kx = lin % g.n[0];
  const long long ky = (lin / g.n[0]) % g.n[1];
  const long long kz = lin / (g.n[0] * g.n[1]);
  const double c[3] = {center(kx, g.sp[0]), center(ky, g.sp[1]), center(kz, g.sp[2])};
  const bool g1 = g.g_is_one;
  double best = __longlong_as_double(0x7ff0000000000000ll);
  int bi = 0x7fffffff;
  for (int p = lane; p < n_alive; p += 32) {
    // reference fold: s = 0; s += w_z^2; s += w_y^2; s += w_x^2
    const double az = axis_sq<PER>(bins.z[p], c[2], g.L[2], g.invL[2]);
    const double ay = axis_sq<PER>(bins.y[p], c[1], g.L[1], g.invL[1]);
    const double ax = axis_sq<PER>(bins.x[p], c[0], g.L[0], g.invL[0]);
    const double dsq = __dadd_rn(__dadd_rn(az, ay), ax);
    const double pr = prox_from_dsq<KIND>(dsq, g.growth, g1, KIND == kVoronoi ? 0.0 : bins.t[p]);
    const int id = bins.idx[p];
    if (pr < best || (pr == best && id < bi)) {
      best = pr;
      bi = id;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ob < best || (ob == best && oi < bi)) {
      best = ob;
      bi = oi;
    }
  }
  if (KIND == kVoronoi && bins.win_r2 > 0.0 && !(best < bins.win_r2)) {
    // an unbinned site (beyond the slab window) may be nearer: all sites
    double b2 = __longlong_as_double(0x7ff0000000000000ll);
    int i2 = 0x7fffffff;
    for (long long s = lane; s < bins.n_all; s += 32) {
      const double* q = bins.all_p3 + 3 * s;
      const double dsq = __dadd_rn(__dadd_rn(axis_sq<PER>(q[2], c[2], g.L[2], g.invL[2]),
                                             axis_sq<PER>(q[1], c[1], g.L[1], g.invL[1])),
                                   axis_sq<PER>(q[0], c[0], g.L[0], g.invL[0]));
      if (dsq < b2 || (dsq == b2 && (int)s < i2)) {
        b2 = dsq;
        i2 = (int)s;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, b2, o);
      const int oi = __shfl_xor_sync(0xffffffffu, i2, o);
      if (ob < b2 || (ob == b2 && oi < i2)) {
        b2 = ob;
        i2 = oi;
      }
    }
    best = b2;
    bi = i2;
  }
  if (lane == 0) {
    const long long out = lin - g.z_begin * g.n[0] * g.n[1];
    labels[out] = bi;
    if (dist) dist[out] = KIND == kVoronoi ? __dsqrt_rn(best) : best;
    if (hist) atomicAdd(&hist[bi], 1ull);
    *evals += (unsigned long long)n_alive;
  }
}

template <int KIND, bool PER>
__device__ void shell_one(const Geo& g, const Bins& bins, const DevParams* prm, long long lin,
                          int* labels, double* dist, unsigned long long* hist,
                          unsigned long long* evals) {
  const int lane = threadIdx.x & 31;
  const long long kx = lin % g.n[0];
  const long long ky = (lin / g.n[0]) % g.n[1];
  const long long kz = lin / (g.n[0] * g.n[1]);
  const double c[3] = {center(kx, g.sp[0]), center(ky, g.sp[1]), center(kz, g.sp[2])};
  long long cv[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    long long q = (long long)(c[a] * g.inv_cw[a]);
    cv[a] = q < 0 ? 0 : (q >= g.m[a] ? g.m[a] - 1 : q);
  }
  const double t_min = prm->t_min;
  const bool g1 = g.g_is_one;
  double best = __longlong_as_double(0x7ff0000000000000ll);
  int bi = 0x7fffffff;
  unsigned long long ne = 0;
  long long plo[3] = {0, 0, 0}, phi[3] = {-1, -1, -1};
  bool pfull[3] = {false, false, false};
  for (long long r = 0;; ++r) {
    long long lo[3], hi[3];
    bool full[3];
    bool allfull = true;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      lo[a] = cv[a] - r;
      hi[a] = cv[a] + r;
      full[a] = false;
      if (PER) {
        if (hi[a] - lo[a] + 1 >= g.m[a]) {
          lo[a] = 0;
          hi[a] = g.m[a] - 1;
          full[a] = true;
        }
      } else {
        if (lo[a] < 0) lo[a] = 0;
        if (hi[a] > g.m[a] - 1) hi[a] = g.m[a] - 1;
        full[a] = lo[a] == 0 && hi[a] == g.m[a] - 1;
      }
      allfull &= full[a];
    }
    // 32-bit cell arithmetic: m <= 4096 per axis, windows never exceed the
    // grid (n_cells <= 2^26), and |index| < 2m so one conditional wraps it
    const int sx = (int)(hi[0] - lo[0] + 1), sy = (int)(hi[1] - lo[1] + 1), sz = (int)(hi[2] - lo[2] + 1);
    const int ncell = sx * sy * sz;
    for (int f = lane; f < ncell; f += 32) {
      const int fyz = f / sx;
      const int ix = (int)lo[0] + (f - fyz * sx), iy = (int)lo[1] + fyz % sy, iz = (int)lo[2] + fyz / sy;
      const int w[3] = {PER ? wrap1(ix, g.m[0]) : ix, PER ? wrap1(iy, g.m[1]) : iy, PER ? wrap1(iz, g.m[2]) : iz};
      if (r > 0) {  // skip cells of the previous window
        bool inside = true;
        const int u[3] = {ix, iy, iz};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          bool in_a;
          if (pfull[a]) in_a = true;
          else if (PER) in_a = wrap1(w[a] - (int)plo[a], g.m[a]) <= (int)(phi[a] - plo[a]);
          else in_a = u[a] >= plo[a] && u[a] <= phi[a];
          inside &= in_a;
        }
        if (inside) continue;
      }
      const long long cell = w[0] + (long long)g.m[0] * (w[1] + (long long)g.m[1] * w[2]);
      VXCHK(cell >= 0 && cell < g.n_cells, "cell %lld w %lld %lld %lld r %lld lin %lld", cell,
            w[0], w[1], w[2], r, lin);
      const int pb = bins.cell_start[cell], pe = bins.cell_start[cell + 1];
      VXCHK(pb >= 0 && pe <= g.n_sites && pb <= pe, "pb %d pe %d", pb, pe);
      for (int p = pb; p < pe; ++p) {
        // reference fold: s = 0; s += w_z^2; s += w_y^2; s += w_x^2
        const double az = axis_sq<PER>(bins.z[p], c[2], g.L[2], g.invL[2]);
        const double ay = axis_sq<PER>(bins.y[p], c[1], g.L[1], g.invL[1]);
        const double ax = axis_sq<PER>(bins.x[p], c[0], g.L[0], g.invL[0]);
        const double dsq = __dadd_rn(__dadd_rn(az, ay), ax);
        const double pr = prox_from_dsq<KIND>(dsq, g.growth, g1, KIND == kVoronoi ? 0.0 : bins.t[p]);
        const int id = bins.idx[p];
        if (pr < best || (pr == best && id < bi)) {
          best = pr;
          bi = id;
        }
        ++ne;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob < best || (ob == best && oi < bi)) {
        best = ob;
        bi = oi;
      }
    }
    if (allfull) break;
    // distance from the voxel centre to the outside of the scanned window
    double lbd = __longlong_as_double(0x7ff0000000000000ll);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (full[a]) continue;
      if (PER || lo[a] > 0) lbd = fmin(lbd, c[a] - lo[a] * g.cw[a]);
      if (PER || hi[a] < g.m[a] - 1) lbd = fmin(lbd, (hi[a] + 1) * g.cw[a] - c[a]);
    }
    lbd = lbd * (1.0 - 1e-9) - 1e-12 * g.lmax;
    if (lbd > 0.0 && bi != 0x7fffffff) {
      double lbp;
      if (KIND == kVoronoi) lbp = lbd * lbd;
      else if (KIND == kJohnsonMehl) lbp = lbd / g.growth + t_min;
      else lbp = lbd * lbd / g.growth + t_min;
      const double slack = KIND == kVoronoi ? 0.0 : 1e-12 * (fabs(t_min) + g.lmax * g.lmax / g.growth + g.lmax / g.growth);
      if (lbp - slack > best) break;
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      plo[a] = lo[a];
      phi[a] = hi[a];
      pfull[a] = full[a];
    }
  }
  if (KIND == kVoronoi && bins.win_r2 > 0.0 && !(best < bins.win_r2)) {
    // an unbinned site (beyond the slab window) may be nearer: all sites, lanes striding
    double b2 = __longlong_as_double(0x7ff0000000000000ll);
    int i2 = 0x7fffffff;
    for (long long s = lane; s < bins.n_all; s += 32) {
      const double* q = bins.all_p3 + 3 * s;
      const double dsq = __dadd_rn(__dadd_rn(axis_sq<PER>(q[2], c[2], g.L[2], g.invL[2]),
                                             axis_sq<PER>(q[1], c[1], g.L[1], g.invL[1])),
                                   axis_sq<PER>(q[0], c[0], g.L[0], g.invL[0]));
      if (dsq < b2 || (dsq == b2 && (int)s < i2)) {
        b2 = dsq;
        i2 = (int)s;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, b2, o);
      const int oi = __shfl_xor_sync(0xffffffffu, i2, o);
      if (ob < b2 || (ob == b2 && oi < i2)) {
        b2 = ob;
        i2 = oi;
      }
    }
    best = b2;
    bi = i2;
    ne += (unsigned long long)bins.n_all;
  }
  if (lane == 0) {
    const long long out = lin - g.z_begin * g.n[0] * g.n[1];
    VXCHK(out >= 0 && out < (g.z_end - g.z_begin) * g.n[0] * g.n[1] && bi >= 0 && bi < g.n_sites,
          "out %lld bi %d lin %lld", out, bi, lin);
    labels[out] = bi;
    if (dist) dist[out] = KIND == kVoronoi ? __dsqrt_rn(best) : best;
    if (hist) atomicAdd(&hist[bi], 1ull);
  }
  *evals += ne;
}

// The search is a chain of dependent L2 loads per voxel: occupancy pays even
// at the price of spills -- Voronoi / JM at 64 registers, 4 blocks (32 warps)
// per SM (cfg2 shell 0.075 -> 0.055 ms, cfg4 0.054 -> 0.038, cfg5 0.068 ->
// 0.055); Laguerre at 128 registers, 2 resident blocks (64: 0.077 -> 0.093)
#ifndef VX_SHELL_MINB
#define VX_SHELL_MINB 4
#endif
#ifndef VX_SHELL_MINB_L
#define VX_SHELL_MINB_L 2
#endif
template <int KIND, bool PER>
__global__ void __launch_bounds__(kShellThreads, KIND == kLaguerre ? VX_SHELL_MINB_L : VX_SHELL_MINB)
    shell_kernel(Geo g, Bins bins, const DevParams* __restrict__ prm, int* __restrict__ labels,
                 double* __restrict__ dist, unsigned long long* __restrict__ hist,
                 const long long* __restrict__ unres, long long unres_cap, DevCounters* ctr) {
  const long long nwarps = (long long)gridDim.x * (kShellThreads / 32);
  const long long w = blockIdx.x * (long long)(kShellThreads / 32) + (threadIdx.x >> 5);
  const long long n = (long long)ctr->n_unres;
  const int n_alive = (int)ctr->n_alive;  // binned (prune-surviving) sites
  unsigned long long ne = 0;
  if (n <= unres_cap) {
    for (long long i = w; i < n; i += nwarps) {
      VXCHK(unres[i] >= 0 && unres[i] < g.n[0] * g.n[1] * g.n[2], "unres[%lld]=%lld n=%lld", i,
            unres[i], n);
      if (n_alive <= kShellBrute) shell_all<KIND, PER>(g, bins, n_alive, unres[i], labels, dist, hist, &ne);
      else shell_one<KIND, PER>(g, bins, prm, unres[i], labels, dist, hist, &ne);
    }
  } else {
    // overflow: compact directly from the image (label sentinel -1)
    const long long nvs = (g.z_end - g.z_begin) * g.n[0] * g.n[1];
    const long long base = g.z_begin * g.n[0] * g.n[1];
    const int lane = threadIdx.x & 31;
    for (long long c0 = w * 32; c0 < nvs; c0 += nwarps * 32) {
      const long long v = c0 + lane;
      const bool un = v < nvs && labels[v] == -1;
      unsigned mask = __ballot_sync(0xffffffffu, un);
      while (mask) {
        const int src = __ffs(mask) - 1;
        mask &= mask - 1;
        if (n_alive <= kShellBrute) shell_all<KIND, PER>(g, bins, n_alive, base + c0 + src, labels, dist, hist, &ne);
        else shell_one<KIND, PER>(g, bins, prm, base + c0 + src, labels, dist, hist, &ne);
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ne += __shfl_xor_sync(0xffffffffu, ne, o);
  if ((threadIdx.x & 31) == 0 && ne) atomicAdd(&ctr->shell_evals, ne);
}

template <int KIND>
static void launch_k(const Geo& g, const Bins& bins, const DevParams* prm, int* labels,
                     double* dist, unsigned long long* hist, const long long* unres,
                     long long cap, DevCounters* ctr, cudaStream_t st) {
  const int blocks = sm_count() * 4;
  if (g.periodic)
    shell_kernel<KIND, true><<<blocks, kShellThreads, 0, st>>>(g, bins, prm, labels, dist, hist,
                                                               unres, cap, ctr);
  else
    shell_kernel<KIND, false><<<blocks, kShellThreads, 0, st>>>(g, bins, prm, labels, dist, hist,
                                                                unres, cap, ctr);
}

int launch_shell(const Geo& g, const Bins& bins, const DevParams* prm, int* labels, double* dist,
                 unsigned long long* hist, const long long* unres, long long unres_cap,
                 DevCounters* ctr, cudaStream_t st) {
  switch (g.kind) {
    case kVoronoi: launch_k<kVoronoi>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, st); break;
    case kJohnsonMehl: launch_k<kJohnsonMehl>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, st); break;
    default: launch_k<kLaguerre>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, st); break;
  }
  return 1;
}

}  // namespace vxb
