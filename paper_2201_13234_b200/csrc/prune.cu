// K6: prune_ineffective_sites (reference: sites.cpp:113-171, O(N_s^2) OpenMP).
//
// Same predicate, same f64 expressions, evaluated only against the sites that
// can possibly satisfy it:
//  * JM drops s iff some o has sqrt(d(s,o)^2)/G + t_o < t_s (or == with o < s),
//    which needs d(s,o) <= G (t_s - t_min).
//  * Laguerre drops s iff G(t_s - t_o) + sum_i axis_min_sq_diff_i > 0 (or == 0
//    with o < s).  Every axis term is <= -(wrapped delta_i)^2 (both for the
//    periodic and the clamped form of sites.cpp:27-37), so o must lie within
//    sqrt(G (t_s - t_min)) of s.
// The candidate o are enumerated from the cell grid inside that (inflated)
// radius; since "dropped" is an OR over o, the enumeration order is irrelevant
// and the result is identical to the reference's full double loop.
#include "vx_internal.cuh"

namespace vxb {

__device__ __forceinline__ double axis_min_sq_diff(double a, double b, double L, double invL,
                                                   bool periodic) {
  if (periodic) {
    const double half = __dmul_rn(0.5, L);
    const double w = wrap_delta(__dadd_rn(__dsub_rn(b, a), half), L, invL);
    return __dsub_rn(__dmul_rn(w, w), __dmul_rn(half, half));
  }
  const double delta = __dsub_rn(b, a);
  const double at0 = __dmul_rn(delta, __dsub_rn(-a, b));
  const double atL = __dmul_rn(delta, __dsub_rn(__dsub_rn(__dmul_rn(2.0, L), a), b));
  return at0 < atL ? at0 : atL;
}

// One warp per site: the lanes split the cells of its reach box (one cell per
// lane, its sites in turn); a ballot ORs the verdicts.
constexpr int kPruneThreads = 128;

template <bool PER>
__global__ void __launch_bounds__(kPruneThreads)
    prune_kernel(Geo g, Bins bins, const double* __restrict__ p3, const double* __restrict__ times,
                 const DevParams* prm, uint8_t* __restrict__ dropped) {
  const long long s = blockIdx.x * (long long)(kPruneThreads / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (s >= g.n_sites) return;
  const double xs[3] = {p3[3 * s], p3[3 * s + 1], p3[3 * s + 2]};
  const double ts = times[s];
  const double t_min = dkey_inv(prm->tmin_key);
  const double t_max = dkey_inv(prm->tmax_key);
  const double G = g.growth;
  double rho;
  if (g.kind == kJohnsonMehl) {
    rho = G * (ts - t_min) * (1.0 + 1e-9) + 1e-12 * g.lmax;
  } else {
    const double tabs = fmax(fabs(t_min), fabs(t_max));
    const double e = 1e-12 * (3.0 * g.lmax * g.lmax + G * tabs);
    rho = sqrt(fmax(G * (ts - t_min), 0.0) + e) * (1.0 + 1e-9) + 1e-12 * g.lmax;
  }
  long long lo[3], hi[3];
  for (int a = 0; a < 3; ++a) {
    lo[a] = (long long)floor((xs[a] - rho) * g.inv_cw[a] - 1e-6);
    hi[a] = (long long)floor((xs[a] + rho) * g.inv_cw[a] + 1e-6);
    if (PER) {
      if (hi[a] - lo[a] + 1 >= g.m[a]) {
        lo[a] = 0;
        hi[a] = g.m[a] - 1;
      }
    } else {
      lo[a] = lo[a] < 0 ? 0 : lo[a];
      hi[a] = hi[a] >= g.m[a] ? g.m[a] - 1 : hi[a];
    }
  }
  const long long nx = hi[0] - lo[0] + 1, ny = hi[1] - lo[1] + 1, nz = hi[2] - lo[2] + 1;
  const long long ncell = nx > 0 && ny > 0 && nz > 0 ? nx * ny * nz : 0;
  bool drop = false;
  for (long long c0 = 0; c0 < ncell; c0 += 32) {
    const long long c = c0 + lane;
    if (c < ncell) {
      const long long cx = lo[0] + c % nx, cy = lo[1] + (c / nx) % ny, cz = lo[2] + c / (nx * ny);
      const long long wx = PER ? ((cx % g.m[0]) + g.m[0]) % g.m[0] : cx;
      const long long wy = PER ? ((cy % g.m[1]) + g.m[1]) % g.m[1] : cy;
      const long long wz = PER ? ((cz % g.m[2]) + g.m[2]) % g.m[2] : cz;
      const long long cell = wx + (long long)g.m[0] * (wy + (long long)g.m[1] * wz);
      const int b = bins.cell_start[cell], e = bins.cell_start[cell + 1];
      for (int p = b; p < e && !drop; ++p) {
        const long long o = bins.idx[p];
        if (o == s) continue;
        const double xo[3] = {bins.x[p], bins.y[p], bins.z[p]};
        const double to = bins.t[p];
        if (g.kind == kJohnsonMehl) {
          // l_periodic_distance_sq(xs, xo): a = xs, b = xo (sites.cpp:136-139)
          double acc = 0.0;
          for (int i = 2; i >= 0; --i) acc = __dadd_rn(acc, axis_sq<PER>(xo[i], xs[i], g.L[i], g.invL[i]));
          double reach = __dsqrt_rn(acc);
          if (!g.g_is_one) reach = __ddiv_rn(reach, G);
          reach = __dadd_rn(reach, to);
          drop = reach < ts || (reach == ts && o < s);
        } else {
          // ascending axis order; a padded axis adds exactly +0 (see Geo)
          double margin = __dmul_rn(G, __dsub_rn(ts, to));
          for (int i = 0; i < 3; ++i)
            margin = __dadd_rn(margin, axis_min_sq_diff(xs[i], xo[i], g.L[i], g.invL[i], PER));
          drop = margin > 0.0 || (margin == 0.0 && o < s);
        }
      }
    }
    if (__any_sync(0xffffffffu, drop)) {
      drop = true;
      break;
    }
  }
  if (lane == 0) dropped[s] = drop ? 1 : 0;
}

// Any dimension (d >= 4 path): the reference's full O(N_s^2) double loop.
struct PruneDims {
  double L[16], invL[16];
};

template <bool PER>
__global__ void prune_generic_kernel(int kind, int dim, PruneDims pd, double G, int g_one,
                                     const double* __restrict__ pos, const double* __restrict__ t,
                                     long long n, uint8_t* __restrict__ dropped) {
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= n) return;
  const double* xs = pos + s * dim;
  const double ts = t[s];
  bool drop = false;
  for (long long o = 0; o < n && !drop; ++o) {
    if (o == s) continue;
    const double* xo = pos + o * dim;
    if (kind == kJohnsonMehl) {
      double acc = 0.0;
      for (int i = dim - 1; i >= 0; --i) acc = __dadd_rn(acc, axis_sq<PER>(xo[i], xs[i], pd.L[i], pd.invL[i]));
      double reach = __dsqrt_rn(acc);
      if (!g_one) reach = __ddiv_rn(reach, G);
      reach = __dadd_rn(reach, t[o]);
      drop = reach < ts || (reach == ts && o < s);
    } else {
      double margin = __dmul_rn(G, __dsub_rn(ts, t[o]));
      for (int i = 0; i < dim; ++i)
        margin = __dadd_rn(margin, axis_min_sq_diff(xs[i], xo[i], pd.L[i], pd.invL[i], PER));
      drop = margin > 0.0 || (margin == 0.0 && o < s);
    }
  }
  dropped[s] = drop ? 1 : 0;
}

int launch_prune_generic(int kind, int periodic, int dim, const double* lengths, double growth,
                         const double* pos, const double* t, long long n_sites, uint8_t* dropped,
                         cudaStream_t st) {
  PruneDims pd;
  for (int i = 0; i < dim; ++i) {
    pd.L[i] = lengths[i];
    pd.invL[i] = 1.0 / lengths[i];
  }
  const int T = 128;
  const unsigned nb = (unsigned)((n_sites + T - 1) / T);
  if (periodic)
    prune_generic_kernel<true><<<nb, T, 0, st>>>(kind, dim, pd, growth, growth == 1.0, pos, t, n_sites, dropped);
  else
    prune_generic_kernel<false><<<nb, T, 0, st>>>(kind, dim, pd, growth, growth == 1.0, pos, t, n_sites, dropped);
  return 1;
}

int launch_prune(const Geo& g, const Bins& bins, const double* p3, const double* times,
                 const DevParams* prm, uint8_t* dropped, cudaStream_t st) {
  const int T = kPruneThreads;
  const unsigned nb = (unsigned)((g.n_sites + T / 32 - 1) / (T / 32));
  if (g.periodic) prune_kernel<true><<<nb, T, 0, st>>>(g, bins, p3, times, prm, dropped);
  else prune_kernel<false><<<nb, T, 0, st>>>(g, bins, p3, times, prm, dropped);
  return 1;
}

}  // namespace vxb
