// K2: the ball phase in gather form (+ fused K3 compaction and the per-CTA
// grain-volume histogram).
//
// Reference: step1_scan (tessellate.cpp:103-144) scatters every site's
// investigation ball over the image (for_each_window_voxel, ball_scan.hpp:
// 55-124) and keeps, per voxel, the strict-< minimum of the ranking value over
// sites whose prox <= cutoff.  Here one CTA owns an 8x8x8 voxel brick and
// gathers instead:
//
//  1. rows:  the x-rows of the cell grid that intersect brick (+) ball(R) are
//            turned into contiguous ranges of the cell-sorted site arrays;
//  2. tau:   every gathered site gets conservative bounds lbp <= prox <= ubp
//            over the brick; tau = min ubp (its site is s0);
//  3. cull:  sites with lbp > tau + eps can never win in the brick; of the
//            rest, those whose bisector test against s0 shows they lose
//            everywhere in the brick are dropped too (separable per-axis
//            minimum; JM via the ratio form |x-s|-|x-s0| = N/D);
//  4. exact: the survivors (sorted by site index) get the reference's exact
//            per-axis squared residual tables (ball_scan.hpp:89-96 hoisting),
//            every voxel folds (wz^2 + wy^2) + wx^2 and keeps a strict-<
//            minimum -> lowest index wins ties (tessellate.cpp:65,132);
//  5. resolve: a voxel is resolved iff best prox <= cutoff (the reference's
//            step-1 membership test, tessellate.cpp:130): every site that could
//            reach it within the cutoff lies within R of the brick and was
//            gathered.  Unresolved voxels are compacted (warp ballot + scan +
//            one atomic per warp) for the widening-shell search (shell.cu).
// Culling only removes sites that lose strictly (by >> f64 rounding) at every
// voxel of the brick, so labels and values are bit-identical to the reference.
#include "vx_internal.cuh"

namespace vxb {

struct BrickGeom {
  double cc[3];    // brick centre (voxel-centre box)
  double half[3];  // half extent, slightly inflated
};

// Conservative per-axis distance bounds of a site to the brick's voxel-centre
// box; u = nearest-image residual site - centre.
template <bool PER>
__device__ __forceinline__ void axis_bounds(const Geo& g, const BrickGeom& b, int a, double s,
                                            double* u_out, double* mn, double* mx) {
  double u = s - b.cc[a];
  if (PER) u = u - floor(u * g.invL[a] + 0.5) * g.L[a];
  const double au = fabs(u);
  double lo = fmax(au - b.half[a], 0.0), hi = au + b.half[a];
  if (PER) {
    if (b.half[a] >= g.halfL[a]) lo = 0.0;
    hi = fmin(hi, g.halfL[a]);
  }
  *u_out = u;
  *mn = lo;
  *mx = hi;
}

template <int KIND>
__device__ __forceinline__ double prox_bound(const Geo& g, double dsq, double t) {
  if (KIND == kVoronoi) return dsq;
  const double v = KIND == kJohnsonMehl ? sqrt(dsq) : dsq;
  return v / g.growth + t;
}

template <int KIND, bool PER>
__device__ __forceinline__ void site_bounds(const Geo& g, const BrickGeom& b, const Bins& bins,
                                            int p, double* lbp, double* ubp) {
  const double s[3] = {bins.x[p], bins.y[p], bins.z[p]};
  const double t = KIND == kVoronoi ? 0.0 : bins.t[p];
  double lb = 0.0, ub = 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double u, mn, mx;
    axis_bounds<PER>(g, b, a, s[a], &u, &mn, &mx);
    lb += mn * mn;
    ub += mx * mx;
  }
  *lbp = prox_bound<KIND>(g, lb, t);
  *ubp = prox_bound<KIND>(g, ub, t);
}

__device__ __forceinline__ long long wrapi(long long c, long long m) {
  const long long r = c % m;
  return r < 0 ? r + m : r;
}

// Block-wide exclusive scan of n <= kMaxSegs ints in place; returns the total.
__device__ int block_exclusive_scan(int* v, int n, int* s_warp) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int PER_T = kMaxSegs / kBallThreads;
  int loc[PER_T];
  int sum = 0;
#pragma unroll
  for (int i = 0; i < PER_T; ++i) {
    const int k = tid * PER_T + i;
    loc[i] = k < n ? v[k] : 0;
    sum += loc[i];
  }
  int inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s_warp[wid] = inc;
  __syncthreads();
  int wbase = 0, total = 0;
#pragma unroll
  for (int w = 0; w < kBallThreads / 32; ++w) {
    if (w < wid) wbase += s_warp[w];
    total += s_warp[w];
  }
  int run = wbase + inc - sum;
#pragma unroll
  for (int i = 0; i < PER_T; ++i) {
    const int k = tid * PER_T + i;
    if (k < n) v[k] = run;
    run += loc[i];
  }
  __syncthreads();
  return total;
}

template <int KIND, bool PER>
__global__ void __launch_bounds__(kBallThreads)
    ball_kernel(Geo g, Bins bins, const DevParams* __restrict__ prm, int* __restrict__ labels,
                double* __restrict__ dist, unsigned long long* __restrict__ hist,
                long long* __restrict__ unres, long long unres_cap, DevCounters* ctr) {
  __shared__ int s_seg_start[kMaxSegs];
  __shared__ int s_seg_off[kMaxSegs + 1];
  __shared__ int s_cand1[kCap1];
  __shared__ int s_upos[kCap2];
  __shared__ int s_uidx[kCap2];
  __shared__ int s_fidx[kCap2];
  __shared__ int s_fpos[kCap2];
  __shared__ int s_cnt[kCap2];
  __shared__ double s_ft[kCap2];
  __shared__ __align__(16) double s_wx[kCap2][BX];
  __shared__ double s_wy[kCap2][BY];
  __shared__ double s_wz[kCap2][BZ];
  __shared__ double s_red_v[kBallThreads / 32];
  __shared__ int s_red_p[kBallThreads / 32];
  __shared__ int s_warp[kBallThreads / 32];
  __shared__ int s_n1, s_n2, s_overflow;

  const int tid = threadIdx.x;
  const long long bid = blockIdx.x;
  const long long bxi = bid % g.nbx, rr = bid / g.nbx;
  const long long byi = rr % g.nby, bzi = rr / g.nby;
  const long long k0[3] = {bxi * BX, byi * BY, g.z_begin + bzi * BZ};
  const int ext[3] = {(int)min((long long)BX, g.n[0] - k0[0]), (int)min((long long)BY, g.n[1] - k0[1]),
                      (int)min((long long)BZ, g.z_end - k0[2])};
  BrickGeom b;
  double blo[3], bhi[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    blo[a] = center(k0[a], g.sp[a]);
    bhi[a] = center(k0[a] + ext[a] - 1, g.sp[a]);
    b.cc[a] = 0.5 * (blo[a] + bhi[a]);
    b.half[a] = 0.5 * (bhi[a] - blo[a]) + 1e-13 * g.lmax;
  }
  const double R = prm->gather_r;
  const double cutoff = prm->cutoff;
  const double eps = prm->eps;
  if (tid == 0) {
    s_n1 = 0;
    s_n2 = 0;
    s_overflow = 0;
  }

  // ---- 1. bin rows -> contiguous site segments ----
  long long cl[3], ch[3];
  bool full[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    cl[a] = (long long)floor((blo[a] - R) * g.inv_cw[a] - 1e-6);
    ch[a] = (long long)floor((bhi[a] + R) * g.inv_cw[a] + 1e-6);
    full[a] = false;
    if (PER) {
      if (ch[a] - cl[a] + 1 >= g.m[a]) {
        cl[a] = 0;
        ch[a] = g.m[a] - 1;
        full[a] = true;
      }
    } else {
      cl[a] = max(cl[a], 0ll);
      ch[a] = min(ch[a], (long long)g.m[a] - 1);
    }
  }
  const int nry = (int)(ch[1] - cl[1] + 1), nrz = (int)(ch[2] - cl[2] + 1);
  const int nrows = nry * nrz;
  const bool rows_ok = nrows <= kMaxRows && nry > 0 && nrz > 0;
  const double R2 = R * R;
  if (rows_ok) {
    for (int r = tid; r < nrows; r += kBallThreads) {
      const long long cy = cl[1] + r % nry, cz = cl[2] + r / nry;
      double dy = 0.0, dz = 0.0;
      if (!full[1]) dy = fmax(0.0, fmax(cy * g.cw[1] - bhi[1], blo[1] - (cy + 1) * g.cw[1]));
      if (!full[2]) dz = fmax(0.0, fmax(cz * g.cw[2] - bhi[2], blo[2] - (cz + 1) * g.cw[2]));
      const double dyz = dy * dy + dz * dz;
      int st0 = 0, n0 = 0, st1 = 0, n1 = 0;
      if (dyz <= R2 * (1.0 + 1e-9)) {
        const double exr = sqrt(fmax(R2 - dyz, 0.0)) * (1.0 + 1e-9) + 1e-12 * g.lmax;
        long long cx0 = (long long)floor((blo[0] - exr) * g.inv_cw[0] - 1e-6);
        long long cx1 = (long long)floor((bhi[0] + exr) * g.inv_cw[0] + 1e-6);
        const long long wy = PER ? wrapi(cy, g.m[1]) : cy, wz = PER ? wrapi(cz, g.m[2]) : cz;
        const long long base = (long long)g.m[0] * (wy + (long long)g.m[1] * wz);
        const int mx = g.m[0];
        long long a0 = 0, a1 = -1, c0 = 0, c1 = -1;  // up to two cell ranges [a0,a1], [c0,c1]
        if (PER) {
          if (cx1 - cx0 + 1 >= mx) {
            a0 = 0;
            a1 = mx - 1;
          } else {
            const long long w0 = wrapi(cx0, mx), len = cx1 - cx0 + 1;
            if (w0 + len <= mx) {
              a0 = w0;
              a1 = w0 + len - 1;
            } else {
              a0 = w0;
              a1 = mx - 1;
              c0 = 0;
              c1 = len - (mx - w0) - 1;
            }
          }
        } else {
          a0 = max(cx0, 0ll);
          a1 = min(cx1, (long long)mx - 1);
        }
        if (a1 >= a0) {
          st0 = bins.cell_start[base + a0];
          n0 = bins.cell_start[base + a1 + 1] - st0;
        }
        if (c1 >= c0) {
          st1 = bins.cell_start[base + c0];
          n1 = bins.cell_start[base + c1 + 1] - st1;
        }
      }
      s_seg_start[2 * r] = st0;
      s_seg_off[2 * r] = n0;
      s_seg_start[2 * r + 1] = st1;
      s_seg_off[2 * r + 1] = n1;
    }
  }
  __syncthreads();
  const int nseg = rows_ok ? 2 * nrows : 0;
  const int total = block_exclusive_scan(s_seg_off, nseg, s_warp);
  if (tid == 0) s_seg_off[nseg] = total;
  __syncthreads();

  // ---- 2. tau = min over gathered sites of the upper bound ----
  auto seg_of = [&](int f) {
    int lo = 0, hi = nseg - 1;  // largest k with off[k] <= f
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_seg_off[mid] <= f) lo = mid;
      else hi = mid - 1;
    }
    return s_seg_start[lo] + (f - s_seg_off[lo]);
  };
  double my_ub = __longlong_as_double(0x7ff0000000000000ll);
  int my_p = -1;
  for (int f = tid; f < total; f += kBallThreads) {
    const int p = seg_of(f);
    double lbp, ubp;
    site_bounds<KIND, PER>(g, b, bins, p, &lbp, &ubp);
    if (ubp < my_ub) {
      my_ub = ubp;
      my_p = p;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double v = __shfl_xor_sync(0xffffffffu, my_ub, o);
    const int q = __shfl_xor_sync(0xffffffffu, my_p, o);
    if (v < my_ub || (v == my_ub && q > my_p)) {
      my_ub = v;
      my_p = q;
    }
  }
  if ((tid & 31) == 0) {
    s_red_v[tid >> 5] = my_ub;
    s_red_p[tid >> 5] = my_p;
  }
  __syncthreads();
  double tau = s_red_v[0];
  int p0 = s_red_p[0];
#pragma unroll
  for (int w = 1; w < kBallThreads / 32; ++w) {
    if (s_red_v[w] < tau || (s_red_v[w] == tau && s_red_p[w] > p0)) {
      tau = s_red_v[w];
      p0 = s_red_p[w];
    }
  }
  bool ok = rows_ok && p0 >= 0;

  // ---- 3. tau cull ----
  if (ok) {
    const double lim = tau + eps;
    for (int f = tid; f < total; f += kBallThreads) {
      const int p = seg_of(f);
      double lbp, ubp;
      site_bounds<KIND, PER>(g, b, bins, p, &lbp, &ubp);
      if (lbp <= lim) {
        const int k = atomicAdd(&s_n1, 1);
        if (k < kCap1) s_cand1[k] = p;
        else s_overflow = 1;
      }
    }
  }
  __syncthreads();
  ok = ok && !s_overflow;

  // ---- 4. bisector cull against s0 ----
  if (ok) {
    const int n1 = s_n1;
    double u0[3], mn0[3], mx0[3];
    const double s0[3] = {bins.x[p0], bins.y[p0], bins.z[p0]};
    const double t0s = KIND == kVoronoi ? 0.0 : bins.t[p0];
#pragma unroll
    for (int a = 0; a < 3; ++a) axis_bounds<PER>(g, b, a, s0[a], &u0[a], &mn0[a], &mx0[a]);
    for (int j = tid; j < n1; j += kBallThreads) {
      const int p = s_cand1[j];
      const double ss[3] = {bins.x[p], bins.y[p], bins.z[p]};
      double nmin = 0.0, dmn = 0.0, dmx = 0.0, dmn0 = 0.0, dmx0 = 0.0;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        double u, mn, mx;
        axis_bounds<PER>(g, b, a, ss[a], &u, &mn, &mx);
        const bool wrapcase =
            PER && (fabs(u0[a]) + b.half[a] > g.halfL[a] * (1.0 - 1e-12) ||
                    fabs(u) + b.half[a] > g.halfL[a] * (1.0 - 1e-12));
        // min over the brick of w_s^2 - w_s0^2 along this axis
        nmin += wrapcase ? mn * mn - mx0[a] * mx0[a]
                         : u * u - u0[a] * u0[a] - 2.0 * b.half[a] * fabs(u - u0[a]);
        dmn += mn * mn;
        dmx += mx * mx;
        dmn0 += mn0[a] * mn0[a];
        dmx0 += mx0[a] * mx0[a];
      }
      if (KIND == kJohnsonMehl) nmin -= 3e-13 * g.lmax * g.lmax;  // rounding slack before the ratio
      double lbdiff;  // lower bound of prox_s - prox_s0 over the brick
      if (KIND == kVoronoi) {
        lbdiff = nmin;
      } else if (KIND == kLaguerre) {
        lbdiff = nmin / g.growth + (bins.t[p] - t0s);
      } else {  // |x-s| - |x-s0| = N / (|x-s| + |x-s0|)
        const double dlo = sqrt(dmn) + sqrt(dmn0), dhi = sqrt(dmx) + sqrt(dmx0);
        double q;
        if (nmin >= 0.0) q = nmin / dhi;
        else q = dlo > 0.0 ? nmin / dlo : -__longlong_as_double(0x7ff0000000000000ll);
        lbdiff = q / g.growth + (bins.t[p] - t0s);
      }
      if (lbdiff <= eps || p == p0) {
        const int k = atomicAdd(&s_n2, 1);
        if (k < kCap2) s_upos[k] = p;
        else s_overflow = 1;
      }
    }
  }
  __syncthreads();
  ok = ok && !s_overflow;
  const int n2 = ok ? s_n2 : 0;

  // ---- sort survivors by site index; exact per-axis tables ----
  if (ok) {
    for (int j = tid; j < n2; j += kBallThreads) s_uidx[j] = bins.idx[s_upos[j]];
    __syncthreads();
    for (int j = tid; j < n2; j += kBallThreads) {
      const int me = s_uidx[j];
      int rank = 0;
      for (int k = 0; k < n2; ++k) rank += s_uidx[k] < me;
      s_fidx[rank] = me;
      s_fpos[rank] = s_upos[j];
      s_cnt[rank] = 0;
    }
    __syncthreads();
    for (int e = tid; e < n2 * (BX + BY + BZ); e += kBallThreads) {
      const int j = e / (BX + BY + BZ), r = e % (BX + BY + BZ);
      const int p = s_fpos[j];
      if (r < BX) {
        s_wx[j][r] = axis_sq<PER>(bins.x[p], center(k0[0] + r, g.sp[0]), g.L[0], g.invL[0]);
      } else if (r < BX + BY) {
        s_wy[j][r - BX] = axis_sq<PER>(bins.y[p], center(k0[1] + r - BX, g.sp[1]), g.L[1], g.invL[1]);
      } else {
        s_wz[j][r - BX - BY] =
            axis_sq<PER>(bins.z[p], center(k0[2] + r - BX - BY, g.sp[2]), g.L[2], g.invL[2]);
      }
      if (r == 0 && KIND != kVoronoi) s_ft[j] = bins.t[p];
    }
  }
  __syncthreads();

  // ---- 5. exact per-voxel evaluation (4 voxels per thread along x) ----
  const int qx = (tid & 1) * 4, vy = (tid >> 1) & 7, vz = tid >> 4;
  double best[4];
  int bj[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    best[q] = __longlong_as_double(0x7ff0000000000000ll);
    bj[q] = -1;
  }
  const bool g1 = g.g_is_one;
  for (int j = 0; j < n2; ++j) {
    const double a = __dadd_rn(s_wz[j][vz], s_wy[j][vy]);  // 0 + wz^2 == wz^2 exactly
    const double2 w01 = *reinterpret_cast<const double2*>(&s_wx[j][qx]);
    const double2 w23 = *reinterpret_cast<const double2*>(&s_wx[j][qx + 2]);
    const double tj = KIND == kVoronoi ? 0.0 : s_ft[j];
    const double d[4] = {__dadd_rn(a, w01.x), __dadd_rn(a, w01.y), __dadd_rn(a, w23.x),
                         __dadd_rn(a, w23.y)};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double pr = prox_from_dsq<KIND>(d[q], g.growth, g1, tj);
      if (pr < best[q]) {
        best[q] = pr;
        bj[q] = j;
      }
    }
  }

  // ---- resolve, store, compact unresolved ----
  const bool rowvalid = vy < ext[1] && vz < ext[2];
  const long long ky = k0[1] + vy, kz = k0[2] + vz;
  const long long slab_base = g.z_begin * g.n[0] * g.n[1];
  const long long lin0 = k0[0] + qx + g.n[0] * (ky + g.n[1] * kz);
  int lab[4];
  long long mylins[4];
  int nun = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const bool valid = rowvalid && (qx + q) < ext[0];
    lab[q] = -1;
    if (valid) {
      if (bj[q] >= 0 && best[q] <= cutoff) {
        lab[q] = s_fidx[bj[q]];
        atomicAdd(&s_cnt[bj[q]], 1);
      } else {
        mylins[nun++] = lin0 + q;
      }
    }
  }
  if (rowvalid) {
    int* out = labels + (lin0 - slab_base);
    if (qx + 4 <= ext[0] && g.vec_store) {
      *reinterpret_cast<int4*>(out) = make_int4(lab[0], lab[1], lab[2], lab[3]);
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (qx + q < ext[0]) out[q] = lab[q];
    }
    if (dist) {
      double* dout = dist + (lin0 - slab_base);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (qx + q < ext[0] && lab[q] >= 0)
          dout[q] = KIND == kVoronoi ? __dsqrt_rn(best[q]) : best[q];
    }
  }
  // warp-aggregated push of unresolved voxels
  {
    const int lane = tid & 31;
    int inc = nun;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    const int wtot = __shfl_sync(0xffffffffu, inc, 31);
    unsigned long long base = 0;
    if (wtot > 0) {
      if (lane == 31) base = atomicAdd(&ctr->n_unres, (unsigned long long)wtot);
      base = __shfl_sync(0xffffffffu, base, 31);
      const long long off = (long long)base + inc - nun;
      for (int i = 0; i < nun; ++i)
        if (off + i < unres_cap) unres[off + i] = mylins[i];
    }
  }
  __syncthreads();
  if (hist) {
    for (int j = tid; j < n2; j += kBallThreads)
      if (s_cnt[j]) atomicAdd(&hist[s_fidx[j]], (unsigned long long)s_cnt[j]);
  }
  if (tid == 0) {
    const long long nvox = (long long)ext[0] * ext[1] * ext[2];
    if (n2 > 0) atomicAdd(&ctr->ball_evals, (unsigned long long)n2 * nvox);
    if (!ok) atomicAdd(&ctr->overflow_bricks, 1ull);
  }
}

template <int KIND>
static void launch_kind(const Geo& g, const Bins& bins, const DevParams* prm, int* labels,
                        double* dist, unsigned long long* hist, long long* unres,
                        long long unres_cap, DevCounters* ctr, cudaStream_t st) {
  const long long nblocks = g.nbx * g.nby * g.nbz;
  if (g.periodic)
    ball_kernel<KIND, true><<<(unsigned)nblocks, kBallThreads, 0, st>>>(g, bins, prm, labels, dist,
                                                                       hist, unres, unres_cap, ctr);
  else
    ball_kernel<KIND, false><<<(unsigned)nblocks, kBallThreads, 0, st>>>(
        g, bins, prm, labels, dist, hist, unres, unres_cap, ctr);
}

int launch_ball(const Geo& g, const Bins& bins, const DevParams* prm, int* labels, double* dist,
                unsigned long long* hist, long long* unres, long long unres_cap, DevCounters* ctr,
                cudaStream_t st) {
  if (g.nbx * g.nby * g.nbz == 0) return 0;
  switch (g.kind) {
    case kVoronoi: launch_kind<kVoronoi>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, st); break;
    case kJohnsonMehl: launch_kind<kJohnsonMehl>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, st); break;
    default: launch_kind<kLaguerre>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, st); break;
  }
  return 1;
}

}  // namespace vxb
