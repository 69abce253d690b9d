// Overflow fallback of the ball phase: a widening-shell search per 8x8x4
// sub-brick (instead of per voxel) for the sub-bricks whose lists overflowed
// the ball phase's caps -- very dense sites (spacing below ~7 voxels) or
// strongly anisotropic voxels.
//
// One warp per sub-brick, 8 voxels per lane (the eval kernel's mapping).  Ring r
// is the set of cells at Chebyshev distance r from the block of cells covering
// the sub-brick (periodic axes wrap; an axis whose window reaches the whole
// period is "full").  Every site of a ring is evaluated with the reference's
// exact f64 fold at all voxels (site data broadcast from the lane that found
// it), keeping the lexicographic minimum of (prox, index) -- the
// order-independent form of the reference's ascending strict-< scan
// (tessellate.cpp:36-75).  After each ring the search stops once a
// conservative lower bound of prox over every site outside the scanned window
// exceeds the largest current best of the sub-brick (strictly, so a tie with a
// lower-index site further out is still found).  Same contract as shell.cu,
// amortised over 256 voxels.
#include "vx_internal.cuh"

namespace vxb {
namespace ssh {

constexpr int kThreads = 128;

__device__ __forceinline__ long long wrapm(long long c, long long m) {
  const long long r = c % m;
  return r < 0 ? r + m : r;
}

template <int KIND, bool PER>
__global__ void __launch_bounds__(kThreads)
    subshell_kernel(Geo g, Bins bins, const DevParams* __restrict__ prm, const int* __restrict__ ovf,
                    const unsigned long long* __restrict__ n_ovf, int* __restrict__ labels,
                    double* __restrict__ dist, unsigned long long* __restrict__ hist, DevCounters* ctr) {
  const int lane = threadIdx.x & 31;
  const long long nw = (long long)gridDim.x * (kThreads / 32);
  const long long n = (long long)*n_ovf;
  const long long nsbx = (g.n[0] + 7) / 8, nsby = (g.n[1] + 7) / 8;
  const int qx = (lane & 1) * 4, vy = (lane >> 1) & 3, vz = lane >> 3;
  const double t_min = prm->t_min;
  const bool g1 = g.g_is_one;
  const long long slab_base = g.z_begin * g.n[0] * g.n[1];
  unsigned long long ne = 0;
  for (long long k = blockIdx.x * (long long)(kThreads / 32) + (threadIdx.x >> 5); k < n; k += nw) {
    const long long sb = ovf[k];
    const long long sbx = sb % nsbx, sby = (sb / nsbx) % nsby, sbz = sb / (nsbx * nsby);
    const long long x0 = sbx * 8, y0 = sby * 8, z0 = g.z_begin + sbz * 4;
    const int sext[3] = {(int)min(8ll, g.n[0] - x0), (int)min(8ll, g.n[1] - y0), (int)min(4ll, g.z_end - z0)};
    // my voxels' exact centres (geometry.hpp:58-60); voxels beyond the grid
    // repeat the last centre (they are never stored)
    double cxs[4], cys[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) cxs[i] = center(x0 + min(qx + i, sext[0] - 1), g.sp[0]);
#pragma unroll
    for (int h = 0; h < 2; ++h) cys[h] = center(y0 + min(vy + 4 * h, sext[1] - 1), g.sp[1]);
    const double czs = center(z0 + min(vz, sext[2] - 1), g.sp[2]);
    // the box of voxel centres and the block of cells covering it
    double blo[3], bhi[3];
    long long clo[3], chi[3];
    const long long o3[3] = {x0, y0, z0};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      blo[a] = center(o3[a], g.sp[a]);
      bhi[a] = center(o3[a] + sext[a] - 1, g.sp[a]);
      long long q0 = (long long)(blo[a] * g.inv_cw[a]), q1 = (long long)(bhi[a] * g.inv_cw[a]);
      clo[a] = q0 < 0 ? 0 : (q0 >= g.m[a] ? g.m[a] - 1 : q0);
      chi[a] = q1 < 0 ? 0 : (q1 >= g.m[a] ? g.m[a] - 1 : q1);
    }
    double best[8];
    int bi[8];
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      best[v] = __longlong_as_double(0x7ff0000000000000ll);
      bi[v] = 0x7fffffff;
    }
    long long plo[3] = {0, 0, 0}, phi[3] = {-1, -1, -1};
    bool pfull[3] = {false, false, false};
    for (long long r = 0;; ++r) {
      long long lo[3], hi[3];
      bool full[3];
      bool allfull = true;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        lo[a] = clo[a] - r;
        hi[a] = chi[a] + r;
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
      const long long sx = hi[0] - lo[0] + 1, sy = hi[1] - lo[1] + 1, sz = hi[2] - lo[2] + 1;
      const long long ncell = sx * sy * sz;
      for (long long f0 = 0; f0 < ncell; f0 += 32) {
        const long long f = f0 + lane;
        int pb = 0, pe = 0;
        if (f < ncell) {
          const long long ix = lo[0] + f % sx, iy = lo[1] + (f / sx) % sy, iz = lo[2] + f / (sx * sy);
          const long long w[3] = {PER ? wrapm(ix, g.m[0]) : ix, PER ? wrapm(iy, g.m[1]) : iy,
                                  PER ? wrapm(iz, g.m[2]) : iz};
          bool inside = r > 0;  // cells of the previous window are done
          if (inside) {
            const long long u[3] = {ix, iy, iz};
#pragma unroll
            for (int a = 0; a < 3; ++a) {
              bool in_a;
              if (pfull[a]) in_a = true;
              else if (PER) in_a = wrapm(w[a] - plo[a], g.m[a]) <= phi[a] - plo[a];
              else in_a = u[a] >= plo[a] && u[a] <= phi[a];
              inside &= in_a;
            }
          }
          if (!inside) {
            const long long cell = w[0] + (long long)g.m[0] * (w[1] + (long long)g.m[1] * w[2]);
            pb = bins.cell_start[cell];
            pe = bins.cell_start[cell + 1];
          }
        }
        // every lane evaluates every site found by any lane
        for (;;) {
          const unsigned m = __ballot_sync(0xffffffffu, pb < pe);
          if (!m) break;
          const int src = __ffs(m) - 1;
          const int p = __shfl_sync(0xffffffffu, pb, src);
          if (lane == src) ++pb;
          const double sxp = bins.x[p], syp = bins.y[p], szp = bins.z[p];
          const int id = bins.idx[p];
          const double tp = KIND == kVoronoi ? 0.0 : bins.t[p];
          const double az = axis_sq<PER>(szp, czs, g.L[2], g.invL[2]);
          double ay[2], ax[4];
#pragma unroll
          for (int h = 0; h < 2; ++h) ay[h] = axis_sq<PER>(syp, cys[h], g.L[1], g.invL[1]);
#pragma unroll
          for (int i = 0; i < 4; ++i) ax[i] = axis_sq<PER>(sxp, cxs[i], g.L[0], g.invL[0]);
#pragma unroll
          for (int v = 0; v < 8; ++v) {
            // reference fold: s = 0; s += w_z^2; s += w_y^2; s += w_x^2
            const double dsq = __dadd_rn(__dadd_rn(az, ay[v >> 2]), ax[v & 3]);
            const double pr = prox_from_dsq<KIND>(dsq, g.growth, g1, tp);
            if (pr < best[v] || (pr == best[v] && id < bi[v])) {
              best[v] = pr;
              bi[v] = id;
            }
          }
          ++ne;
        }
      }
      if (allfull) break;
      // the sub-brick's worst voxel against everything outside the window
      double mb = best[0];
#pragma unroll
      for (int v = 1; v < 8; ++v) mb = fmax(mb, best[v]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mb = fmax(mb, __shfl_xor_sync(0xffffffffu, mb, o));
      double lbd = __longlong_as_double(0x7ff0000000000000ll);
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        if (full[a]) continue;
        if (PER || lo[a] > 0) lbd = fmin(lbd, blo[a] - lo[a] * g.cw[a]);
        if (PER || hi[a] < g.m[a] - 1) lbd = fmin(lbd, (hi[a] + 1) * g.cw[a] - bhi[a]);
      }
      lbd = lbd * (1.0 - 1e-9) - 1e-12 * g.lmax;
      if (lbd > 0.0 && mb < __longlong_as_double(0x7ff0000000000000ll)) {
        double lbp;
        if (KIND == kVoronoi) lbp = lbd * lbd;
        else if (KIND == kJohnsonMehl) lbp = lbd / g.growth + t_min;
        else lbp = lbd * lbd / g.growth + t_min;
        const double slack =
            KIND == kVoronoi ? 0.0 : 1e-12 * (fabs(t_min) + g.lmax * g.lmax / g.growth + g.lmax / g.growth);
        if (lbp - slack > mb) break;
      }
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        plo[a] = lo[a];
        phi[a] = hi[a];
        pfull[a] = full[a];
      }
    }
    if (KIND == kVoronoi && bins.win_r2 > 0.0) {  // slab window: unbinned sites may be nearer
#pragma unroll
      for (int v = 0; v < 8; ++v)
        if (!(best[v] < bins.win_r2)) {
          const double cv[3] = {cxs[v & 3], cys[v >> 2], czs};
          double b2;
          int i2;
          allsites_min<PER>(g, bins, cv, b2, i2);
          best[v] = b2;
          bi[v] = i2;
        }
    }
    // stores (voxels of the grid only) and histogram runs
    const long long lin0 = x0 + qx + g.n[0] * (y0 + vy + g.n[1] * (z0 + vz)) - slab_base;
    int run_id = -1;
    unsigned long long run_n = 0;
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const int i = v & 3, h = v >> 2;
      if (qx + i >= sext[0] || vy + 4 * h >= sext[1] || vz >= sext[2]) continue;
      const long long o = lin0 + (long long)h * 4 * g.n[0] + i;
      labels[o] = bi[v];
      if (dist) dist[o] = KIND == kVoronoi ? __dsqrt_rn(best[v]) : best[v];
      if (hist) {
        if (bi[v] != run_id) {
          if (run_n) atomicAdd(&hist[run_id], run_n);
          run_id = bi[v];
          run_n = 0;
        }
        ++run_n;
      }
    }
    if (hist && run_n) atomicAdd(&hist[run_id], run_n);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ne += __shfl_xor_sync(0xffffffffu, ne, o);
  if (lane == 0 && ne) atomicAdd(&ctr->shell_evals, ne * 8ull);
}

}  // namespace ssh

int launch_subshell(const Geo& g, const Bins& bins, const DevParams* prm, const int* ovf,
                    const unsigned long long* n_ovf, int* labels, double* dist, unsigned long long* hist,
                    DevCounters* ctr, cudaStream_t st) {
  if (g.z_end <= g.z_begin) return 0;
  const unsigned blocks = (unsigned)sm_count() * 8;  // persistent warps walk the overflow list
#define VX_SS(K, P) \
  ssh::subshell_kernel<K, P><<<blocks, ssh::kThreads, 0, st>>>(g, bins, prm, ovf, n_ovf, labels, dist, hist, ctr)
  switch (g.kind * 2 + (g.periodic ? 1 : 0)) {
    case 0: VX_SS(kVoronoi, false); break;
    case 1: VX_SS(kVoronoi, true); break;
    case 2: VX_SS(kJohnsonMehl, false); break;
    case 3: VX_SS(kJohnsonMehl, true); break;
    case 4: VX_SS(kLaguerre, false); break;
    default: VX_SS(kLaguerre, true); break;
  }
#undef VX_SS
  return 1;
}

}  // namespace vxb
