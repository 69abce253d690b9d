// Parameter choice for the ball phase (reference: tessellate.cpp:217-260).
//
// Labels never depend on r0 / t0 (test_tessellate.cpp:
// 218-246), so these only size the gather.  Voronoi uses the reference's
// closed-form r0 (computed on the host with the reference's formula, cost.cpp:
// 28-39).  For timed kinds the reference runs a serial 257-point scan plus 60
// golden-section steps of growth_cost (cost.cpp:56-146); here the same cost
// model is evaluated on the device, 256 candidate t0 per pass in parallel
// (one CTA each), two passes (coarse bracket, then the neighbours of the best
// point).  Everything stays in device memory: no host round trip.
#include "vx_internal.cuh"

namespace vxb {

constexpr int kScan = 256;
constexpr long long kCostSample = 4096;

__global__ void init_kernel(DevParams* prm, DevCounters* ctr) {
  prm->tmin_key = ~0ull;
  prm->tmax_key = 0ull;
  prm->t_min = prm->t_max = 0.0;
  ctr->n_unres = ctr->ball_evals = ctr->shell_evals = ctr->overflow_bricks = 0;
  ctr->n_alive = 0;
  ctr->bad_site = 0;
  ctr->n_unres_done = 0;
  ctr->n_ovf_sb = 0;
}

__global__ void chunk_roll_kernel(DevCounters* ctr) {
  ctr->n_unres_done += ctr->n_unres;
  ctr->n_unres = 0;
}

__global__ void voronoi_params_kernel(DevParams* prm, double R, double lmax) {
  prm->param = R;
  prm->cutoff = R * R;
  prm->gather_r = fmin(R * (1.0 + 1e-9) + 1e-12 * lmax, 4.0 * lmax);
  prm->eps = 1e-12 * 3.0 * lmax * lmax;
}

struct CostArgs {
  int kind, dim;
  double growth, volume, unit;  // unit-ball volume in the true dimension
  double width;                 // t0_bracket width (cost.cpp:78-96)
};

__device__ double site_frac(const CostArgs& a, double t0, double ts) {
  const double dt = t0 - ts;
  double r = 0.0;
  if (dt > 0.0) r = a.kind == kJohnsonMehl ? a.growth * dt : sqrt(a.growth * dt);
  double rd = 1.0;
  for (int i = 0; i < a.dim; ++i) rd *= r;
  const double v = fmin(a.volume, a.unit * rd);
  return v / a.volume;
}

__device__ void scan_range(const CostArgs& a, const DevParams* prm, const double* costs0,
                           int pass, double* lo, double* hi) {
  const double t_min = dkey_inv(prm->tmin_key);
  const double blo = t_min, bhi = t_min + a.width;
  if (pass == 0) {
    *lo = blo;
    *hi = bhi;
    return;
  }
  const int best = (int)costs0[2 * kScan];  // pass 0's arg-min (argmin_kernel)
  const double step = (bhi - blo) / (kScan - 1);
  const double bt = blo + (bhi - blo) * best / (kScan - 1);
  *lo = fmax(blo, bt - step);
  *hi = fmin(bhi, bt + step);
}

// first arg-min of costs[0, kScan) (lowest index on ties, as a serial scan),
// by one warp
__device__ void argmin_warp(const double* c, int* out) {
  const int lane = threadIdx.x & 31;
  double bv = __longlong_as_double(0x7ff0000000000000ll);
  int bi = 0x7fffffff;
  for (int i = lane; i < kScan; i += 32)
    if (c[i] < bv) {
      bv = c[i];
      bi = i;
    }
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov < bv || (ov == bv && oi < bi)) {
      bv = ov;
      bi = oi;
    }
  }
  *out = bi == 0x7fffffff ? 0 : bi;
}
__device__ void argmin_pair(const double* costs, int* b0, int* b1) {
  argmin_warp(costs, b0);
  argmin_warp(costs + kScan, b1);
}
__global__ void argmin_kernel(double* costs) {  // after pass 0: its arg-min for pass 1's bracket
  int b;
  argmin_warp(costs, &b);
  if (threadIdx.x == 0) costs[2 * kScan] = (double)b;
}

// growth_cost(t0)/N_v = sum v'_s/V + N_s * prod(1 - v'_s/V), one CTA per t0.
__global__ void cost_scan_kernel(CostArgs a, const double* __restrict__ t_orig, const uint8_t* __restrict__ dropped,
                                 long long n_sites, const DevCounters* ctr, const DevParams* prm, double* costs,
                                 int pass) {
  __shared__ double s_sum[32], s_log[32];
  __shared__ int s_cnt[32];
  double lo, hi;
  scan_range(a, prm, costs, pass, &lo, &hi);
  const double t0 = lo + (hi - lo) * blockIdx.x / (kScan - 1);
  const long long n = (long long)ctr->n_alive;
  // t0 only sizes the ball phase (labels never depend on it): an evenly
  // strided sample of <= kCostSample sites in ORIGINAL order (independent of
  // the binned order, so the choice is reproducible), pruned ones skipped,
  // scaled back to the n alive sites
  const long long m = n_sites < kCostSample ? n_sites : kCostSample;
  double sum = 0.0, lg = 0.0;
  int cnt = 0;
  for (long long i = threadIdx.x; i < m; i += blockDim.x) {
    const long long s = i * n_sites / m;
    if (dropped && dropped[s]) continue;
    const double f = site_frac(a, t0, t_orig[s]);
    sum += f;
    lg += log1p(-f);
    ++cnt;
  }
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0) s_cnt[threadIdx.x >> 5] = cnt;
  for (int o = 16; o > 0; o >>= 1) {
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
    lg += __shfl_xor_sync(0xffffffffu, lg, o);
  }
  if ((threadIdx.x & 31) == 0) {
    s_sum[threadIdx.x >> 5] = sum;
    s_log[threadIdx.x >> 5] = lg;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double S = 0.0, Lg = 0.0;
    long long C = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      S += s_sum[w];
      Lg += s_log[w];
      C += s_cnt[w];
    }
    if (C > 0 && C < n) {
      S *= (double)n / (double)C;
      Lg *= (double)n / (double)C;
    }
    costs[pass * kScan + blockIdx.x] = S + (double)n * exp(Lg);
  }
}

__global__ void timed_finalize_kernel(CostArgs a, DevParams* prm, const DevCounters* ctr,
                                      const double* costs, int has_override, double override_t0,
                                      double lmax) {  // one warp
  int b0 = 0, b1 = 0;
  if (!has_override && ctr->n_alive > 1) argmin_pair(costs, &b0, &b1);
  if (threadIdx.x != 0) return;
  const double t_min = dkey_inv(prm->tmin_key);
  prm->t_min = t_min;
  prm->t_max = dkey_inv(prm->tmax_key);
  double t0;
  if (has_override) {
    t0 = override_t0;
  } else if (ctr->n_alive <= 1) {
    t0 = t_min + a.width;  // t0_bracket(...).hi, tessellate.cpp:232-233
  } else {
    double lo0, hi0, lo1, hi1;
    scan_range(a, prm, costs, 0, &lo0, &hi0);
    scan_range(a, prm, costs, 1, &lo1, &hi1);

    t0 = costs[kScan + b1] <= costs[b0] ? lo1 + (hi1 - lo1) * b1 / (kScan - 1)
                                        : lo0 + (hi0 - lo0) * b0 / (kScan - 1);
  }
  prm->param = t0;
  prm->cutoff = t0;
  double dt = t0 - t_min;
  if (!(dt > 0.0)) dt = 0.0;
  const double r = a.kind == kJohnsonMehl ? a.growth * dt : sqrt(a.growth * dt);
  prm->gather_r = fmin(r * (1.0 + 1e-9) + 1e-12 * lmax, 4.0 * lmax);
  const double tabs = fmax(fabs(prm->t_min), fabs(prm->t_max)) + fabs(t0);
  prm->eps = 1e-12 * (tabs + (a.kind == kJohnsonMehl ? 2.0 * lmax / a.growth
                                                      : 3.0 * lmax * lmax / a.growth));
}

int launch_params(const Geo& g, const double* t_orig, const uint8_t* dropped, DevParams* prm,
                  const DevCounters* ctr, int has_override, double override_param, double r0, double ball_scale,
                  double* scratch, cudaStream_t st) {
  if (g.kind == kVoronoi) {
    const double R = has_override ? override_param : r0 * ball_scale;
    voronoi_params_kernel<<<1, 1, 0, st>>>(prm, R, g.lmax);
    return 1;
  }
  CostArgs a;
  a.kind = g.kind;
  a.dim = g.dim;
  a.growth = g.growth;
  const double sum_l2 = g.suml2_true;
  a.volume = g.vol_true;
  a.unit = pow(M_PI, 0.5 * g.dim) / tgamma(0.5 * g.dim + 1.0);
  if (g.kind == kJohnsonMehl) {
    const double reach = sqrt(sum_l2);
    a.width = g.periodic ? reach / (2.0 * g.growth) : reach / g.growth;
  } else {
    a.width = g.periodic ? sum_l2 / (4.0 * g.growth) : sum_l2 / g.growth;
  }
  int n = 1;
  if (!has_override) {
    cost_scan_kernel<<<kScan, 256, 0, st>>>(a, t_orig, dropped, g.n_sites, ctr, prm, scratch, 0);
    argmin_kernel<<<1, 32, 0, st>>>(scratch);
    cost_scan_kernel<<<kScan, 256, 0, st>>>(a, t_orig, dropped, g.n_sites, ctr, prm, scratch, 1);
    n += 3;
  }
  timed_finalize_kernel<<<1, 32, 0, st>>>(a, prm, ctr, scratch, has_override, override_param,
                                          g.lmax);
  return n;
}

int launch_init(DevParams* prm, DevCounters* ctr, cudaStream_t st) {
  init_kernel<<<1, 1, 0, st>>>(prm, ctr);
  return 1;
}

int launch_chunk_roll(DevCounters* ctr, cudaStream_t st) {
  chunk_roll_kernel<<<1, 1, 0, st>>>(ctr);
  return 1;
}

}  // namespace vxb
