// K2 (v12, default): the ball phase of tessellate_fast in gather form
// (reference step 1, tessellate.cpp:103-144 + ball_scan.hpp:55-124), as two
// kernels.
//
// Contract (as ball.cu): labels/values bit-identical to the reference, because
// every culled site loses strictly -- by far more than f64 rounding -- at every
// voxel of the box it was culled for, and the survivors are evaluated with the
// reference's exact f64 fold in ascending site order.  f32 bounds are widened
// by kRel (1e-5) of their terms' magnitude plus an absolute coordinate slack
// e_d; float rounding is ~1e-7 relative.
//
// cull12 (CTA = 8 warps = a 16 x 16 x 16nbb super-brick; nbb = 1, 2 or 4 chosen
// by the host from the site density and, for periodic z, the period):
//   gather : x-rows of cells within R of the super-brick -> shared memory
//            (f32 coordinates relative to the super-brick centre, time, binned
//            position, periodic-ambiguity flags); sites that cannot reach any
//            voxel within the cutoff are dropped; the kept sites are
//            rank-sorted by site index once (a carry-chain count) and moved
//            into index order.
//   column : each warp owns a column of nbb 8^3 bricks: one pass computes every
//            site's upper bound of prox for all bricks of the column (the x/y
//            terms are shared) -> per-brick tau; a second pass the lower bounds
//            -> a per-site keep mask; the column's brick lists are ballots
//            over the mask bits, all built in one pass, in site-index order.
//   sub-brick : per 8 x 8 x 4 sub-brick, tau + bisector cull against the site
//            with the least upper bound -> the survivors' binned positions, in
//            site order, into 16 fixed slots (longer lists: an overflow list),
//            (offset, count) per sub-brick.  Dense mode (spacing < ~8.5
//            voxels) allows brick lists of 256 and sub-brick lists of 128 with a
//            two-pass chunked cull.  Sub-bricks over every cap are listed for
//            the sub-brick shell (subshell.cu).
// eval12 (warp = one 8 x 8 x 4 sub-brick, 3-D grid): exact per-axis f64 tables
//   (one lane per (site, axis)), exact evaluation of 8 voxels per lane in two
//   y-rows sharing the x table (dense mode: in passes of 32 candidates),
//   resolve (prox <= cutoff), int4 label stores, optional exact distances,
//   per-candidate histogram counts, warp-aggregated compaction of unresolved
//   voxels for the shell search (shell.cu).
// Split at the sub-brick lists, both kernels fit 64 registers and run at 4
// CTAs/SM; the lists cost ~0.7 GB of HBM traffic at cfg5.
#include <algorithm>
#include <type_traits>
#include <atomic>
#include <cmath>
#include <cstdlib>

#include "vx_internal.cuh"

// VX_STATS=1 in the environment: per-level list sizes into eval_slots[64..70]
#define VX_STATS_ON (g.stats_on != 0)

namespace vxb {
namespace v12 {

constexpr int kSB = 16;           // super-brick edge along x and y (voxels)
constexpr int kMaxBB = 4;         // bricks per warp column (super-brick z = 16 nbb <= 64)
constexpr int kSZ = 16 * kMaxBB;
constexpr int kB2Threads = 256;   // 8 warps, one 8^3 brick each
constexpr int kTcap = 512;        // sites kept per super-brick (else the CTA falls back)
constexpr int kWcap = 64;         // brick-level survivors per warp (2 slots per lane)
constexpr int kFcap = 32;         // sub-brick survivors the eval kernel evaluates
constexpr int kLcap = 64;         // sub-brick list capacity (<= the brick list's kWcap)
// dense mode (site spacing below ~8.5 voxels, chosen on the host): longer
// brick lists, a two-pass chunked sub-brick cull and a chunked eval
constexpr int kWcapD = 256;
constexpr int kLcapD = 128;
constexpr int kSlot = 16;         // fixed list slots per sub-brick (longer lists: overflow list)
constexpr int kRows2 = 256;       // cell rows per super-brick
constexpr float kRel = 1e-5f;
#ifndef VX_COLSTAGE_V
#define VX_COLSTAGE_V 0  // Voronoi keeps the per-brick loop (column stage: cfg5 +6.6 %, 44 B of spills)
#endif

struct FBox {
  float c[3];  // centre relative to the super-brick centre
  float h[3];  // half extent (+ slack)
};

struct __align__(16) WarpSmem {
  int W[kWcapD];       // brick list (gather slots), ascending site index
  union {
    int L[kLcapD];     // dense mode: a sub-brick's survivors (binned positions)
    struct {           // standard lists, column brick stage: per brick the two references
      float zrefb[kMaxBB][16];
      float zref2b[kMaxBB][16];
    };
  };
  float4 bxy;          // the column's x/y box (c[0], c[1], h[0], h[1]), shared by its sub-bricks
  unsigned evals;      // exact evaluations the eval kernel will do for this warp's sub-bricks
  int nw[4];           // standard lists: the column's brick-list lengths
  alignas(16) float zref2[16]; // the second reference (VX_TWO_REFS)
  alignas(16) float zref[16];  // the sub-brick's reference site: SiteF fields + flags (written by its lane)
  float2 bzb[kMaxBB];   // each brick's z box (centre, half extent): box_sub's values
};

// eval12: per warp (one sub-brick); LC = list capacity
template <int LC>
struct __align__(16) EvalSmemT {
  double T[kFcap][20]; // exact w^2 of one pass of kFcap candidates: [0,8) x, [8,16) y, [16,20) z
  double C[24];        // the sub-brick's voxel centres: [0,8) x, [8,16) y, [16,24) z
  double Ft[LC];
  int P[LC];           // binned positions
  int Fidx[LC];
  int cnt[LC];
};
using EvalSmem = EvalSmemT<kFcap>;

struct Smem2 {
  float4 rel[kTcap];   // (ux, uy, uz, t) relative to the super-brick centre
  float4 reln[kTcap];  // periodic: the same with the ambiguous axes (flag bits 0..2) as NaN (column passes)
  int p[kTcap];        // binned position
  int idx[kTcap];      // original site index
  unsigned char flag[kTcap];  // bit a: periodic image ambiguous on axis a
  unsigned char mk[kB2Threads / 32][kTcap];  // per warp: bit b = kept for brick b of its column
  int seg_start[2 * kRows2];
  int seg_off[2 * kRows2 + 1];
  int warp_tot[kB2Threads / 32];
  int n_total;
  int n_kept;
  double cx[kSB], cy[kSB], cz[kSZ];  // exact voxel centres of the super-brick
  union {
    WarpSmem w[kB2Threads / 32];
    struct {  // the gather's staging arrays (dead once the sites are in index order)
      float4 rel[kTcap];
      int p[kTcap];
      unsigned char flag[kTcap];
    } g;
  };
};

__device__ __forceinline__ float lo_add(float a, float b) {
  return (a + b) - kRel * (fabsf(a) + fabsf(b));
}
__device__ __forceinline__ float hi_add(float a, float b) {
  return (a + b) + kRel * (fabsf(a) + fabsf(b));
}

struct SiteF {
  float v[3], mn[3], mx[3];
  float t;
  float lbp, ubp;
  float lb, ub;  // squared distance bounds
};

// Conservative prox bounds of one gathered site over box B.
template <int KIND, bool PER>
__device__ __forceinline__ void fbounds(const float4 s, unsigned flags, const FBox& B,
                                        const float* halfL, float invG, SiteF& o) {
  const float u[3] = {s.x, s.y, s.z};
  float lb = 0.f, ub = 0.f;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float va = u[a] - B.c[a];
    const float av = fabsf(va);
    float lo = fmaxf(av - B.h[a], 0.f), hi = av + B.h[a];
    if (PER) {
      if (flags & (1u << a)) {
        lo = 0.f;
        hi = halfL[a];
      } else {
        hi = fminf(hi, halfL[a]);
      }
    }
    o.v[a] = va;
    o.mn[a] = lo;
    o.mx[a] = hi;
    lb = __fmaf_rn(lo, lo, lb);
    ub = __fmaf_rn(hi, hi, ub);
  }
  lb *= (1.f - kRel);
  ub *= (1.f + kRel);
  o.lb = lb;
  o.ub = ub;
  o.t = s.w;
  if (KIND == kVoronoi) {
    o.lbp = lb;
    o.ubp = ub;
  } else {
    const float tl = s.w - kRel * fabsf(s.w), th = s.w + kRel * fabsf(s.w);
    const float dl = KIND == kJohnsonMehl ? sqrtf(lb) : lb;
    const float dh = KIND == kJohnsonMehl ? sqrtf(ub) : ub;
    o.lbp = lo_add(dl * invG * (1.f - kRel), tl);
    o.ubp = hi_add(dh * invG * (1.f + kRel), th);
  }
}

// The reference-site terms of bisector_keep, once per box: Z2 = |z|^2 and
// Kz = sum_a (|z_a| + 2 h_a) + 3 e_d.
__device__ __forceinline__ void ref_consts(const SiteF& z, const FBox& B, float e_d, float& Z2, float& Kz) {
  Z2 = 0.f;
  Kz = 3.f * e_d;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    Z2 = __fmaf_rn(z.v[a], z.v[a], Z2);
    Kz += fabsf(z.v[a]) + 2.f * B.h[a];
  }
}

// true iff s may beat (or tie) s0 somewhere in B: lower bound of prox_s - prox_s0 <= 0.
// min over x in B of |s - x|^2 - |z - x|^2 = sum_a s_a^2 - z_a^2 - 2 h_a |s_a - z_a|
// (x relative to the box centre); f32 rounding of the sums is covered by
// kRel x their magnitude, and the f32 coordinates' own error (|err| <= e_d
// per coordinate, e_d >= 16x the rounding of the relative coordinates) by
// pert = 2 e_d sum_a (|s_a| + |z_a| + 2 h_a + e_d), subtracted in full.
template <int KIND, bool PER>
__device__ __forceinline__ bool bisector_keep(const SiteF& s, unsigned fs, const SiteF& z,
                                              unsigned f0, const FBox& B, const float* halfL,
                                              float invG, float e_d, float Z2, float Kz) {
  float D, mag, pert;
  // neither site near half a period (flag bits 3..5): no axis needs the wrap bound
  const bool anyrisk = PER && ((fs | f0) & 0x38u) != 0u;
  if (!anyrisk) {
    float S2 = 0.f, Hs = 0.f, As = 0.f;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float dv = fabsf(s.v[a] - z.v[a]);
      S2 = __fmaf_rn(s.v[a], s.v[a], S2);
      Hs = __fmaf_rn(2.f * B.h[a], dv, Hs);
      As += fabsf(s.v[a]);
    }
    D = (S2 - Z2) - Hs;
    mag = (S2 + Z2) + Hs;
    pert = 2.f * e_d * (As + Kz);
  } else {
    D = 0.f, mag = 0.f, pert = 0.f;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const bool wrapcase = ((fs | f0) >> a) & 1u || fabsf(s.v[a]) + B.h[a] > halfL[a] * (1.f - 1e-5f) ||
                            fabsf(z.v[a]) + B.h[a] > halfL[a] * (1.f - 1e-5f);
      float term, m;
      if (wrapcase) {
        term = s.mn[a] * s.mn[a] - z.mx[a] * z.mx[a];
        m = s.mn[a] * s.mn[a] + z.mx[a] * z.mx[a];
      } else {
        const float dv = fabsf(s.v[a] - z.v[a]);
        term = s.v[a] * s.v[a] - z.v[a] * z.v[a] - 2.f * B.h[a] * dv;
        m = s.v[a] * s.v[a] + z.v[a] * z.v[a] + 2.f * B.h[a] * dv;
      }
      D += term;
      mag += m;
      pert += 2.f * e_d * (fabsf(s.v[a]) + fabsf(z.v[a]) + 2.f * B.h[a] + e_d);
    }
  }
  const float Dlo = D - kRel * mag - pert;  // lower bound of min_B (d_s^2 - d_s0^2)
  if (KIND == kVoronoi) return Dlo <= 0.f;
  const float dt = lo_add(s.t - kRel * fabsf(s.t), -(z.t + kRel * fabsf(z.t)));
  if (KIND == kLaguerre) {
    const float q = Dlo >= 0.f ? Dlo * invG * (1.f - kRel) : Dlo * invG * (1.f + kRel);
    return lo_add(q, dt) <= 0.f;
  }
  // JM: |x-s| - |x-s0| = N / (|x-s| + |x-s0|)
  float q;
  if (Dlo >= 0.f) {
    const float dhi = (sqrtf(s.ub) + sqrtf(z.ub)) * (1.f + kRel);
    q = Dlo / dhi * (1.f - kRel);
  } else {
    const float dlo = (sqrtf(s.lb) + sqrtf(z.lb)) * (1.f - kRel);
    if (!(dlo > 0.f)) return true;
    q = Dlo / dlo * (1.f + kRel);
  }
  q = q >= 0.f ? q * invG * (1.f - kRel) : q * invG * (1.f + kRel);
  return lo_add(q, dt) <= 0.f;
}

// a reference site's bounds through shared memory (16 floats: SiteF fields,
// flags, ref_consts), written by its owner lane, read by every lane of its box
__device__ __forceinline__ void put_ref(float* zr, const SiteF& o, unsigned fl, const FBox& B, float e_d) {
  zr[0] = o.v[0], zr[1] = o.v[1], zr[2] = o.v[2];
  zr[3] = o.mn[0], zr[4] = o.mn[1], zr[5] = o.mn[2];
  zr[6] = o.mx[0], zr[7] = o.mx[1], zr[8] = o.mx[2];
  zr[9] = o.t, zr[10] = o.lb, zr[11] = o.ub, zr[12] = o.ubp;
  zr[13] = __uint_as_float(fl);
  ref_consts(o, B, e_d, zr[14], zr[15]);
}
__device__ __forceinline__ void get_ref(const float* zr, SiteF& z, float4& q3) {
  const float4 q0 = *reinterpret_cast<const float4*>(&zr[0]);
  const float4 q1 = *reinterpret_cast<const float4*>(&zr[4]);
  const float4 q2 = *reinterpret_cast<const float4*>(&zr[8]);
  q3 = *reinterpret_cast<const float4*>(&zr[12]);
  z.v[0] = q0.x, z.v[1] = q0.y, z.v[2] = q0.z;
  z.mn[0] = q0.w, z.mn[1] = q1.x, z.mn[2] = q1.y;
  z.mx[0] = q1.z, z.mx[1] = q1.w, z.mx[2] = q2.x;
  z.t = q2.y, z.lb = q2.z, z.ub = q2.w;
  z.ubp = q3.x;
}

__device__ __forceinline__ long long wrapi2(long long c, long long m) {
  // the gather windows are narrower than a period, so c lies in (-m, 2m):
  // one conditional add or subtract (the 64-bit remainder is a ~70
  // instruction subroutine); anything else takes the remainder
  if (c >= -m && c < 2 * m) return c < 0 ? c + m : (c >= m ? c - m : c);
  const long long r = c % m;
  return r < 0 ? r + m : r;
}

// BL: standard lists per 8^3 brick (evaluated by eval16) instead of per 8 x 8 x 4 sub-brick
template <int KIND, bool PER, bool DENSE, bool BL>
__global__ void __launch_bounds__(kB2Threads, 4)
    cull12_kernel(Geo g, Bins bins, const DevParams* __restrict__ prm, int2* __restrict__ info,
                  int* __restrict__ slots16, int* __restrict__ list, long long list_cap,
                  unsigned long long* __restrict__ list_count, int* __restrict__ ovf,
                  DevCounters* ctr, unsigned long long* __restrict__ eval_slots, int nbb, unsigned by0) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem2& S = *reinterpret_cast<Smem2*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

  const long long K0[3] = {(long long)blockIdx.x * kSB, (long long)(by0 + blockIdx.y) * kSB,
                           g.z_begin + (long long)blockIdx.z * (16 * nbb)};
  int ext[3];
  ext[0] = (int)min((long long)kSB, g.n[0] - K0[0]);
  ext[1] = (int)min((long long)kSB, g.n[1] - K0[1]);
  ext[2] = (int)min((long long)(16 * nbb), g.z_end - K0[2]);
  double blo[3], bhi[3], cc[3], hs[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    blo[a] = center(K0[a], g.sp[a]);
    bhi[a] = center(K0[a] + ext[a] - 1, g.sp[a]);
    cc[a] = 0.5 * (blo[a] + bhi[a]);
    hs[a] = 0.5 * (bhi[a] - blo[a]);
  }
  const long long nsbx = g.nsbx, nsby = g.nsby;
  auto sb_id = [&](long long x, long long y, long long z) {  // 8x8x4 sub-brick at voxel (x, y, z)
    return (x >> 3) + nsbx * ((y >> 3) + nsby * ((z - g.z_begin) >> 2));
  };
  const double R = prm->gather_r;
  const double cutoff = prm->cutoff;
  // the cutoff rounded up to f32: a site whose lower bound exceeds it over a
  // brick has prox > cutoff at every voxel there, so it can neither win a
  // resolved voxel nor matter at an unresolved one -- every cull level is
  // clamped to it (a partly uncovered brick keeps only reachable sites)
  const float tcf = __double2float_ru(cutoff + 1e-9 * fabs(cutoff));
  float halfLf[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) halfLf[a] = (float)g.halfL[a];
  const float invG = KIND == kVoronoi ? 1.f : (float)(1.0 / g.growth);
  // absolute slack for f32 coordinates relative to the super-brick centre
  const float e_d = (float)(1e-6 * (R + hs[0] + hs[1] + hs[2] + g.cw[0] + g.cw[1] + g.cw[2]));

  // ---------------- G: gather ----------------
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
  const bool rows_ok = nry > 0 && nrz > 0 && nrows <= kRows2;
  const double R2 = R * R;
  if (rows_ok) {
    for (int r = tid; r < nrows; r += kB2Threads) {
      const long long cy = cl[1] + r % nry, cz = cl[2] + r / nry;
      double dy = 0.0, dz = 0.0;
      if (!full[1]) dy = fmax(0.0, fmax(cy * g.cw[1] - bhi[1], blo[1] - (cy + 1) * g.cw[1]));
      if (!full[2]) dz = fmax(0.0, fmax(cz * g.cw[2] - bhi[2], blo[2] - (cz + 1) * g.cw[2]));
      const double dyz = dy * dy + dz * dz;
      int st0 = 0, n0 = 0, st1 = 0, n1 = 0;
      if (dyz <= R2 * (1.0 + 1e-9)) {
        const double exr = sqrt(fmax(R2 - dyz, 0.0)) * (1.0 + 1e-9) + 1e-12 * g.lmax;
        const long long cx0 = (long long)floor((blo[0] - exr) * g.inv_cw[0] - 1e-6);
        const long long cx1 = (long long)floor((bhi[0] + exr) * g.inv_cw[0] + 1e-6);
        const long long wy = PER ? wrapi2(cy, g.m[1]) : cy, wz = PER ? wrapi2(cz, g.m[2]) : cz;
        const long long base = (long long)g.m[0] * (wy + (long long)g.m[1] * wz);
        const int mx = g.m[0];
        long long a0 = 0, a1 = -1, c0 = 0, c1 = -1;
        if (PER) {
          if (cx1 - cx0 + 1 >= mx) {
            a0 = 0;
            a1 = mx - 1;
          } else {
            const long long w0 = wrapi2(cx0, mx), len = cx1 - cx0 + 1;
            a0 = w0;
            if (w0 + len <= mx) {
              a1 = w0 + len - 1;
            } else {
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
      S.seg_start[2 * r] = st0;
      S.seg_off[2 * r] = n0;
      S.seg_start[2 * r + 1] = st1;
      S.seg_off[2 * r + 1] = n1;
    }
  }
  __syncthreads();
  // exclusive scan of the segment counts (2 per thread)
  const int nseg = rows_ok ? 2 * nrows : 0;
  {
    const int k0 = 2 * tid;
    const int c0 = k0 < nseg ? S.seg_off[k0] : 0, c1 = k0 + 1 < nseg ? S.seg_off[k0 + 1] : 0;
    int inc = c0 + c1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) S.warp_tot[wid] = inc;
    __syncthreads();
    int base = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kB2Threads / 32; ++w) {
      base += w < wid ? S.warp_tot[w] : 0;
      tot += S.warp_tot[w];
    }
    const int ex = base + inc - c0 - c1;
    if (k0 < nseg) S.seg_off[k0] = ex;
    if (k0 + 1 < nseg) S.seg_off[k0 + 1] = ex + c0;
    if (tid == 0) {
      S.seg_off[nseg] = tot;
      S.n_total = tot;
    }
  }
  if (tid == 0) S.n_kept = 0;
  for (int k = tid; k < kTcap; k += kB2Threads) S.idx[k] = 0x7fffffff;  // sort padding
  if (tid < 2 * kSB + 16 * nbb) {  // exact voxel centres (geometry.hpp:58-60)
    const int a = tid < kSB ? 0 : (tid < 2 * kSB ? 1 : 2), k = tid - a * kSB;
    (a == 0 ? S.cx : a == 1 ? S.cy : S.cz)[k] = center(K0[a] + k, g.sp[a]);
  }
  __syncthreads();
  const int Traw = S.n_total;
  bool cta_ok = rows_ok && Traw > 0;
  if (cta_ok) {
    // Only sites that can reach some voxel of the super-brick within the
    // cutoff are kept: a site whose prox exceeds the cutoff everywhere can
    // neither be the winner of a resolved voxel nor make one unresolved.
    const double tc = cutoff + 1e-9 * fabs(cutoff);
    for (int f0 = 0; f0 < Traw; f0 += kB2Threads) {
      const int f = f0 + tid;
      bool keep = false;
      int p = 0;
      float uf[3] = {0.f, 0.f, 0.f};
      unsigned fl = 0;
      double tv = 0.0;
      if (f < Traw) {
        int lo = 0, hi = nseg - 1;  // largest k with off[k] <= f
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (S.seg_off[mid] <= f) lo = mid;
          else hi = mid - 1;
        }
        p = S.seg_start[lo] + (f - S.seg_off[lo]);
        const double sv[3] = {bins.x[p], bins.y[p], bins.z[p]};
        double lb = 0.0;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          double u = sv[a] - cc[a];
          if (PER) {
            u = u - floor(u * g.invL[a] + 0.5) * g.L[a];
            if (fabs(u) + hs[a] >= g.halfL[a] * (1.0 - 1e-7) - 4.0 * e_d) fl |= 1u << a;
            // bit 3 + a: some box inside the super-brick may see the site near
            // half a period (a superset of bisector_keep's per-axis test)
            if (fabs(u) + hs[a] + 8.0 * e_d >= g.halfL[a] * (1.0 - 2e-5)) fl |= 8u << a;
          }
          uf[a] = (float)u;
          const double m = ((fl >> a) & 1u) ? 0.0 : fmax(fabs(u) - hs[a], 0.0);
          lb += m * m;
        }
        double lbp = lb * (1.0 - 1e-9);
        if (KIND != kVoronoi) {
          tv = bins.t[p];
          const double A = (KIND == kJohnsonMehl ? sqrt(lbp) : lbp) / g.growth * (1.0 - 1e-9);
          lbp = A + tv - 1e-9 * fabs(tv);
        }
        keep = lbp <= tc;
      }
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      int base = 0;
      if (lane == 0 && m) base = atomicAdd(&S.n_kept, __popc(m));
      base = __shfl_sync(0xffffffffu, base, 0);
      const int pos = base + __popc(m & ((1u << lane) - 1u));
      if (keep && pos < kTcap) {
        S.g.rel[pos] = make_float4(uf[0], uf[1], uf[2], (float)tv);
        S.g.p[pos] = p;
        S.g.flag[pos] = (unsigned char)fl;
        S.idx[pos] = bins.idx[p];
      }
    }
  }
  __syncthreads();
  const int T = S.n_kept;
  if (T <= kTcap) {  // rank sort of the kept sites by site index (ties impossible)
    for (int f = tid; f < T; f += kB2Threads) {
      const int me = S.idx[f];
      const int4* idx4 = reinterpret_cast<const int4*>(S.idx);  // padded with INT_MAX
      // the carry of v - me (v + ~me + 1) is set iff v >= me: a carry chain
      // counts them at 1.5 instructions per comparison (ptxas pairs two carries
      // per IADD3.X); rank = the padded count minus that
      const int nk = (T + 3) >> 2;
      unsigned ge = 0;
      for (int k = 0; k < nk; ++k) {
        const int4 v = idx4[k];
        unsigned t;
        asm("sub.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %1, 0;\n\t"
            "sub.cc.u32 %0, %4, %3;\n\taddc.u32 %1, %1, 0;\n\t"
            "sub.cc.u32 %0, %5, %3;\n\taddc.u32 %1, %1, 0;\n\t"
            "sub.cc.u32 %0, %6, %3;\n\taddc.u32 %1, %1, 0;"
            : "=&r"(t), "+r"(ge)
            : "r"(v.x), "r"(me), "r"(v.y), "r"(v.z), "r"(v.w));
      }
      const unsigned rank = 4u * (unsigned)nk - ge;
      VXCHK(rank < (unsigned)T);
      // the kept sites move into site-index order
      const float4 rv = S.g.rel[f];
      const unsigned fv = S.g.flag[f];
      S.rel[rank] = rv;
      S.p[rank] = S.g.p[f];
      S.flag[rank] = (unsigned char)fv;
      if (PER) {
        const float qn = __int_as_float(0x7fffffff);
        S.reln[rank] = make_float4(fv & 1u ? qn : rv.x, fv & 2u ? qn : rv.y, fv & 4u ? qn : rv.z, rv.w);
      }
    }
  }
  __syncthreads();
  if (VX_STATS_ON && tid == 0) {  // diagnostics: gathered sites per CTA
    atomicAdd(&eval_slots[64], (unsigned long long)Traw);
    atomicAdd(&eval_slots[65], (unsigned long long)T);
    atomicAdd(&eval_slots[66], 1ull);
    atomicMax(&eval_slots[71], (unsigned long long)T);
  }
  // no site reaches the super-brick within the cutoff (T == 0): every voxel
  // is outside every ball (the reference's step-2 set) -- empty brick lists,
  // not an overflow
  const bool lists_ok = rows_ok && T <= kTcap;
  cta_ok = cta_ok && T > 0 && T <= kTcap;

  // ---------------- W + S: per-warp column of nbb bricks ----------------
  WarpSmem& ws = S.w[wid];
  if (lane == 0) ws.evals = 0;  // lane 0 alone updates it
  const int bxo = (wid & 1) * 8, byo = ((wid >> 1) & 1) * 8;

  auto box_of = [&](int x0, int y0, int z0, int nx, int ny, int nz) {
    FBox B;
    const int o[3] = {x0, y0, z0}, n[3] = {nx, ny, nz};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double* ct = a == 0 ? S.cx : (a == 1 ? S.cy : S.cz);
      const double l = ct[o[a]], h = ct[o[a] + n[a] - 1];
      B.c[a] = (float)(0.5 * (l + h) - cc[a]);
      B.h[a] = (float)(0.5 * (h - l)) * (1.f + kRel) + 2.f * e_d;
    }
    return B;
  };

  // merged tau / keep-mask passes over the gathered sites for all bricks of the column
  const int ex0 = min(8, ext[0] - bxo), ex1 = min(8, ext[1] - byo);
  float bzc[kMaxBB], bzh[kMaxBB], tau[kMaxBB];
  bool bval[kMaxBB];
  // the column's x/y extent once (an empty column, ex0 or ex1 <= 0, returns
  // below: the indices stay inside cx / cy), each brick's z extent
  const FBox Bxy = box_of(bxo, byo, 0, max(ex0, 1), max(ex1, 1), 1);
#pragma unroll
  for (int b = 0; b < kMaxBB; ++b) {
    const int bzo = (wid >> 2) * 8 + 16 * b;
    const int ez = min(8, ext[2] - bzo);
    bval[b] = b < nbb && ex0 > 0 && ex1 > 0 && ez > 0;
    bzc[b] = 0.f;
    bzh[b] = 0.f;
    tau[b] = -1.f;
    if (bval[b]) {
      const double l = S.cz[bzo], h = S.cz[bzo + ez - 1];
      bzc[b] = (float)(0.5 * (l + h) - cc[2]);
      bzh[b] = (float)(0.5 * (h - l)) * (1.f + kRel) + 2.f * e_d;
    }
  }
  bool col_any = false;
#pragma unroll
  for (int b = 0; b < kMaxBB; ++b) col_any |= bval[b];
  if (lane == 0) {
    ws.bxy = make_float4(Bxy.c[0], Bxy.c[1], Bxy.h[0], Bxy.h[1]);
    if (BL && !DENSE && (KIND != kVoronoi || VX_COLSTAGE_V)) {  // the column brick stage's boxes
#pragma unroll
      for (int b = 0; b < kMaxBB; ++b) ws.bzb[b] = make_float2(bzc[b], bzh[b]);
    }
  }
  __syncwarp();
  // a sub-brick's box: the column's x/y extent (every sub-brick of the column
  // shares it) and its own z extent -- the values box_of would give
  auto box_sub = [&](int z0, int nz) {
    FBox B;
    const float4 xy = ws.bxy;
    B.c[0] = xy.x;
    B.c[1] = xy.y;
    B.h[0] = xy.z;
    B.h[1] = xy.w;
    const double l = S.cz[z0], h = S.cz[z0 + nz - 1];
    B.c[2] = (float)(0.5 * (l + h) - cc[2]);
    B.h[2] = (float)(0.5 * (h - l)) * (1.f + kRel) + 2.f * e_d;
    return B;
  };
  if (!col_any) return;  // no barrier follows
  if (cta_ok) {
    // Column passes.  A periodic-ambiguous axis (flag bit a) is fed in as a
    // NaN coordinate: the site drops out of the upper bounds' minimum and
    // fmaxf(NaN, 0) = 0 makes the lower bound's axis term 0, so no per-brick
    // flag test.  For
    // Voronoi the (1 + kRel) widening commutes with the minimum (RN(x c) is
    // monotone in x) and the lower-bound test lb (1 - kRel) <= tau is replaced
    // by the weaker lb <= tau / (1 - kRel) (1 + 1e-6): a superset is kept.
    float myub[kMaxBB];
#pragma unroll
    for (int b = 0; b < kMaxBB; ++b) myub[b] = __int_as_float(0x7f800000);
    // full columns (nbb = kMaxBB, the common case) without per-brick count tests
    auto pass1 = [&](auto nb_tag) {
    constexpr int NB = decltype(nb_tag)::value;
    for (int f = lane; f < T; f += 32) {
      const float4 s = PER ? S.reln[f] : S.rel[f];  // NaN-coded ambiguous axes
      const float sx = s.x, sy = s.y, sz = s.z;
      // no L/2 cap: on an unflagged axis |s - c| + h < L/2 already (up to the
      // widening, which only raises the bound), and a flagged (NaN) axis makes
      // the bound NaN, which fminf ignores -- a site left out of the minimum
      // only raises tau, so the cull stays conservative
      const float mx = fabsf(sx - Bxy.c[0]) + Bxy.h[0];
      const float my = fabsf(sy - Bxy.c[1]) + Bxy.h[1];
      const float bxy = __fmaf_rn(my, my, mx * mx);
#pragma unroll
      for (int b = 0; b < kMaxBB; ++b) {
        if (NB == 0 && b >= nbb) break;
        const float mz = fabsf(sz - bzc[b]) + bzh[b];
        const float u2 = __fmaf_rn(mz, mz, bxy);
        myub[b] = fminf(myub[b], KIND == kVoronoi ? u2
                                                  : hi_add((KIND == kJohnsonMehl ? sqrtf(u2 * (1.f + kRel)) : u2 * (1.f + kRel)) * invG * (1.f + kRel),
                                                           s.w + kRel * fabsf(s.w)));
      }
    }
    };
    if (nbb == kMaxBB) pass1(std::integral_constant<int, kMaxBB>{});
    else pass1(std::integral_constant<int, 0>{});
    float tlb[kMaxBB];  // Voronoi: the lower-bound threshold
#pragma unroll
    for (int b = 0; b < kMaxBB; ++b) {
      float t = myub[b];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t = fminf(t, __shfl_xor_sync(0xffffffffu, t, o));
      if (KIND == kVoronoi) t *= 1.f + kRel;
      tau[b] = bval[b] ? fminf(t, tcf) : __int_as_float(0xff800000);  // -inf: keeps nothing
      tlb[b] = KIND == kVoronoi ? tau[b] * ((1.f + 1e-6f) / (1.f - kRel)) : tau[b];
    }
    // the lower-bound pass; standard lists: fused with the lists of every
    // brick of the column (brick b in W[64 b, 64 b + 64)), in site-index
    // order (dense mode: the mask bits to shared memory, lists per brick below)
    auto pass2 = [&](auto nb_tag) {
    constexpr int NB = decltype(nb_tag)::value;
    int nWb[kMaxBB] = {0, 0, 0, 0};
    const unsigned lt = (1u << lane) - 1u;
    for (int f0 = 0; f0 < T; f0 += 32) {
      const int f = f0 + lane;
      unsigned m = 0;
      if (f < T) {
      const float4 s = PER ? S.reln[f] : S.rel[f];  // NaN-coded ambiguous axes
      const float sx = s.x, sy = s.y, sz = s.z;
      const float lx = fmaxf(fabsf(sx - Bxy.c[0]) - Bxy.h[0], 0.f);
      const float ly = fmaxf(fabsf(sy - Bxy.c[1]) - Bxy.h[1], 0.f);
      const float bxy = __fmaf_rn(ly, ly, lx * lx);
#pragma unroll
      for (int b = 0; b < kMaxBB; ++b) {
        if (NB == 0 && b >= nbb) break;
        const float lz = fmaxf(fabsf(sz - bzc[b]) - bzh[b], 0.f);
        const float l2 = __fmaf_rn(lz, lz, bxy);
        const float lbp = KIND == kVoronoi ? l2
                                           : lo_add((KIND == kJohnsonMehl ? sqrtf(l2 * (1.f - kRel)) : l2 * (1.f - kRel)) * invG * (1.f - kRel),
                                                    s.w - kRel * fabsf(s.w));
        if (lbp <= tlb[b]) m |= 1u << b;
      }
      if (DENSE) S.mk[wid][f] = (unsigned char)m;
      }
      if constexpr (!DENSE) {
#pragma unroll
        for (int b = 0; b < kMaxBB; ++b) {
          if (NB == 0 && b >= nbb) break;
          const bool keep = (m >> b) & 1u;
          const unsigned bm = __ballot_sync(0xffffffffu, keep);
          const int pos = nWb[b] + __popc(bm & lt);
          if (keep && pos < kWcap) ws.W[b * kWcap + pos] = f;
          nWb[b] += __popc(bm);
        }
      }
    }
    if (!DENSE && lane == 0) {
#pragma unroll
      for (int b = 0; b < kMaxBB; ++b) ws.nw[b] = nWb[b];
    }
    };
    if (nbb == kMaxBB) pass2(std::integral_constant<int, kMaxBB>{});
    else pass2(std::integral_constant<int, 0>{});
    __syncwarp();
  } else if (!DENSE && lists_ok) {  // no site reaches the super-brick: empty lists
    if (lane == 0) {
#pragma unroll
      for (int b = 0; b < kMaxBB; ++b) ws.nw[b] = 0;
    }
    __syncwarp();
  }

  // Column brick stage (brick lists): the refinement of every brick of the
  // column in one pass -- brick b's list occupies slots [off_b, off_b + nW_b)
  // of at most 64 (two per lane), arg-mins by warp reductions per brick,
  // references through shared memory per brick.  Per site the same keep
  // predicate, reference choice and slot order as the per-brick loop below
  // (which handles columns whose lists total more than 64).
  bool col_done = false;
  if constexpr (BL && !DENSE && (KIND != kVoronoi || VX_COLSTAGE_V)) {
    int nWe[kMaxBB];
    bool bok[kMaxBB];
#pragma unroll
    for (int b = 0; b < kMaxBB; ++b) {
      const int nwb = lists_ok && bval[b] ? ws.nw[b] : 0;
      bok[b] = bval[b] && lists_ok && nwb <= kWcap;
      nWe[b] = bok[b] ? nwb : 0;
    }
    const int o1 = nWe[0], o2 = o1 + nWe[1], o3 = o2 + nWe[2], M = o3 + nWe[3];
    if (M <= 64) {
      col_done = true;
      auto okey = [](float v) -> unsigned {
        const unsigned b = __float_as_uint(v);
        return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
      };
      auto bzo_of = [&](int b) { return (wid >> 2) * 8 + 16 * b; };
      auto boxb = [&](int b) {  // == box_sub(bzo_of(b), min(8, ext[2] - bzo_of(b)))
        FBox B;
        const float4 xy = ws.bxy;
        const float2 z = ws.bzb[b];
        B.c[0] = xy.x, B.c[1] = xy.y, B.c[2] = z.x;
        B.h[0] = xy.z, B.h[1] = xy.w, B.h[2] = z.y;
        return B;
      };
      SiteF sv[2];
      int fv[2], bv[2], kv[2];
      unsigned flv[2];
      bool vv[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int e = lane + 32 * i;
        vv[i] = e < M;
        const int b = (e >= o1) + (e >= o2) + (e >= o3);
        bv[i] = b;
        kv[i] = e - (b == 0 ? 0 : b == 1 ? o1 : b == 2 ? o2 : o3);
        fv[i] = vv[i] ? ws.W[b * kWcap + kv[i]] : 0;
        flv[i] = vv[i] ? S.flag[fv[i]] : 0u;
        if (i == 1 && M <= 32) continue;
        fbounds<KIND, PER>(S.rel[fv[i]], flv[i], boxb(b), halfLf, invG, sv[i]);
      }
      // per-brick packed (upper bound, slot) arg-min: one warp reduction per
      // brick and iteration (REDUX), lanes of other bricks contribute ~0
      auto brick_min = [&](const unsigned (&key)[2], unsigned (&res)[2]) {
        unsigned km[kMaxBB];
#pragma unroll
        for (int b = 0; b < kMaxBB; ++b) {
          km[b] = __reduce_min_sync(0xffffffffu, bv[0] == b ? key[0] : 0xffffffffu);
          if (M > 32) km[b] = min(km[b], __reduce_min_sync(0xffffffffu, bv[1] == b ? key[1] : 0xffffffffu));
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) res[i] = bv[i] == 0 ? km[0] : bv[i] == 1 ? km[1] : bv[i] == 2 ? km[2] : km[3];
      };
      unsigned key[2], r0v[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) key[i] = vv[i] ? (okey(sv[i].ubp) & ~63u) | (unsigned)kv[i] : 0xffffffffu;
      brick_min(key, r0v);
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        r0v[i] &= 63u;
        if (vv[i] && (unsigned)kv[i] == r0v[i]) put_ref(ws.zrefb[bv[i]], sv[i], flv[i], boxb(bv[i]), e_d);
      }
      unsigned r1v[2] = {0xffffffffu, 0xffffffffu};
      if constexpr (KIND == kVoronoi) {  // the second reference, the next-least upper bound
        unsigned key2[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) key2[i] = (unsigned)kv[i] != r0v[i] ? key[i] : 0xffffffffu;
        brick_min(key2, r1v);
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const unsigned k2 = r1v[i];
          if (vv[i] && k2 != 0xffffffffu && (unsigned)kv[i] == (k2 & 63u))
            put_ref(ws.zref2b[bv[i]], sv[i], flv[i], boxb(bv[i]), e_d);
        }
      }
      __syncwarp();
      bool kp[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        kp[i] = false;
        if (i == 1 && M <= 32) continue;
        const FBox Bs = boxb(bv[i]);
        SiteF z;
        float4 q3;
        get_ref(ws.zrefb[bv[i]], z, q3);
        const float tau = fminf(z.ubp, tcf);
        bool k = vv[i] && ((unsigned)kv[i] == r0v[i] ||
                           (sv[i].lbp <= tau &&
                            bisector_keep<KIND, PER>(sv[i], flv[i], z, __float_as_uint(q3.y), Bs, halfLf, invG, e_d,
                                                     q3.z, q3.w)));
        if constexpr (KIND == kVoronoi) {
          const unsigned k2 = r1v[i];
          if (k && (unsigned)kv[i] != r0v[i] && k2 != 0xffffffffu && (unsigned)kv[i] != (k2 & 63u)) {
            SiteF z2;
            float4 q3b;
            get_ref(ws.zref2b[bv[i]], z2, q3b);
            k = bisector_keep<KIND, PER>(sv[i], flv[i], z2, __float_as_uint(q3b.y), Bs, halfLf, invG, e_d, q3b.z,
                                         q3b.w);
          }
        }
        kp[i] = k;
      }
      const unsigned m0 = __ballot_sync(0xffffffffu, kp[0]), m1 = __ballot_sync(0xffffffffu, kp[1]);
      // brick b's slots in iteration i: lanes [off_b - 32 i, off_b+1 - 32 i) clamped to [0, 32)
      auto seg = [](int lo, int hi) -> unsigned {
        lo = max(0, min(32, lo));
        hi = max(0, min(32, hi));
        const unsigned mh = hi >= 32 ? 0xffffffffu : ((1u << hi) - 1u);
        const unsigned ml = lo >= 32 ? 0xffffffffu : ((1u << lo) - 1u);
        return mh & ~ml;
      };
      auto off_of = [&](int b) { return b == 0 ? 0 : b == 1 ? o1 : b == 2 ? o2 : b == 3 ? o3 : M; };
      // lanes 0 .. kMaxBB-1: brick lane's bookkeeping (list space, info, overflow)
      long long bbase = 0;
      int bn2 = 0;
      bool bokl = false;
      int* bdst = list;
      unsigned ev = 0;
      if (lane < kMaxBB) {
        const int b = lane;
        const bool valid = b == 0 ? bval[0] : b == 1 ? bval[1] : b == 2 ? bval[2] : bval[3];
        const bool okb = b == 0 ? bok[0] : b == 1 ? bok[1] : b == 2 ? bok[2] : bok[3];
        if (valid) {
          const int bz = bzo_of(b);
          const int ez = min(8, ext[2] - bz);
          const long long sbi = (long long)(bxo + K0[0]) / 8 +
                                (long long)nsbx * ((K0[1] + byo) / 8 + nsby * ((K0[2] + bz - g.z_begin) >> 3));
          if (VX_STATS_ON && lists_ok) {
            const int nwb = ws.nw[b];
            atomicAdd(&eval_slots[67], (unsigned long long)nwb);
            atomicAdd(&eval_slots[68], 1ull);
            atomicMax(&eval_slots[72], (unsigned long long)nwb);
          }
          if (okb) {
            const int lo = off_of(b), hi = off_of(b + 1);
            bn2 = __popc(m0 & seg(lo, hi)) + __popc(m1 & seg(lo - 32, hi - 32));
            if (bn2 > kSlot && bn2 <= kLcap) bbase = (long long)atomicAdd(list_count, (unsigned long long)bn2);
            bokl = bn2 <= kLcap && (bn2 <= kSlot || bbase + bn2 <= list_cap);
            info[sbi] = bokl ? make_int2((int)bbase, bn2) : make_int2(0, -1);
            bdst = bn2 <= kSlot ? slots16 + sbi * kSlot : list + bbase;
            if (VX_STATS_ON) {
              atomicAdd(&eval_slots[69], (unsigned long long)bn2);
              atomicAdd(&eval_slots[70], 1ull);
              atomicMax(&eval_slots[73], (unsigned long long)bn2);
            }
            if (bokl && bn2 <= kFcap) ev = (unsigned)(bn2 * ex0 * ex1 * ez);
          } else {
            info[sbi] = make_int2(0, -1);
            atomicAdd(&ctr->overflow_bricks, 1ull);
          }
          if (!okb || !bokl) {  // the sub-brick shell labels it, 8 x 8 x 4 at a time
            ovf[atomicAdd(&ctr->n_ovf_sb, 1ull)] = (int)sb_id(K0[0] + bxo, K0[1] + byo, K0[2] + bz);
            if (ez > 4) ovf[atomicAdd(&ctr->n_ovf_sb, 1ull)] = (int)sb_id(K0[0] + bxo, K0[1] + byo, K0[2] + bz + 4);
          }
        }
      }
      ev += __shfl_xor_sync(0xffffffffu, ev, 1);
      ev += __shfl_xor_sync(0xffffffffu, ev, 2);
      if (lane == 0) ws.evals += ev;
      // survivors -> their brick's slots (or overflow list), in slot order
      const unsigned lt = (1u << lane) - 1u;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        if (i == 1 && M <= 32) continue;
        const int b = bv[i] & 3;
        int* dst = reinterpret_cast<int*>(__shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(bdst), b));
        const bool okl = __shfl_sync(0xffffffffu, bokl, b);
        if (kp[i] && okl) {
          const int lo = off_of(b), hi = off_of(b + 1);
          const int rank = i == 0 ? __popc(m0 & seg(lo, hi) & lt)
                                  : __popc(m0 & seg(lo, hi)) + __popc(m1 & seg(lo - 32, hi - 32) & lt);
          dst[rank] = S.p[fv[i]];
        }
      }
    }
  }

  if (!col_done)
  for (int bb = 0; bb < nbb; ++bb) {  // no barrier below: warps run independently
  const int bzo = (wid >> 2) * 8 + 16 * bb;
  const int bext[3] = {ex0, ex1, min(8, ext[2] - bzo)};
  if (bext[0] <= 0 || bext[1] <= 0 || bext[2] <= 0) continue;

  int nW = 0;
  bool brick_ok = lists_ok;
  const int* Wl = ws.W;  // this brick's list
  if (!DENSE) {
    nW = lists_ok ? ws.nw[bb] : 0;
    Wl = ws.W + bb * kWcap;
    brick_ok = lists_ok && nW <= kWcap;
    if (VX_STATS_ON && lane == 0 && lists_ok) {
      atomicAdd(&eval_slots[67], (unsigned long long)nW);
      atomicAdd(&eval_slots[68], 1ull);
      atomicMax(&eval_slots[72], (unsigned long long)nW);
    }
  } else if (brick_ok) {
    for (int f0 = 0; f0 < T; f0 += 32) {
      const int f = f0 + lane < T ? f0 + lane : 0;
      const bool keep = f0 + lane < T && ((S.mk[wid][f] >> bb) & 1u);
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      const int pos = nW + __popc(m & ((1u << lane) - 1u));
      if (keep && pos < (DENSE ? kWcapD : kWcap)) ws.W[pos] = f;  // ballot order = ord order = site order
      nW += __popc(m);
    }
    brick_ok = nW <= (DENSE ? kWcapD : kWcap);
    if (VX_STATS_ON && lane == 0) {
      atomicAdd(&eval_slots[67], (unsigned long long)nW);
      atomicAdd(&eval_slots[68], 1ull);
      atomicMax(&eval_slots[72], (unsigned long long)nW);
    }
  }
  __syncwarp();

  // brick lists (standard lists only): one list per 8^3 brick instead of
  // one per 8 x 8 x 4 sub-brick
  constexpr bool BM = BL && !DENSE;
  for (int q = 0; q < (BM ? 1 : 2); ++q) {
    const int sy = byo, sz = bzo + q * 4;
    const int sext[3] = {bext[0], bext[1], min(BM ? 8 : 4, ext[2] - sz)};
    if (sext[1] <= 0 || sext[2] <= 0) continue;
    // overflowed lists go to the sub-brick shell, 8 x 8 x 4 at a time
    auto push_ovf = [&](void) {
      ovf[atomicAdd(&ctr->n_ovf_sb, 1ull)] = (int)sb_id(K0[0] + bxo, K0[1] + sy, K0[2] + sz);
      if (BM && sext[2] > 4) ovf[atomicAdd(&ctr->n_ovf_sb, 1ull)] = (int)sb_id(K0[0] + bxo, K0[1] + sy, K0[2] + sz + 4);
    };
    auto list_id = [&](void) -> long long {  // (K0 and the offsets are >= 0)
      return BM ? ((K0[0] + bxo) >> 3) + nsbx * (((K0[1] + sy) >> 3) + nsby * ((K0[2] + sz - g.z_begin) >> 3))
                : sb_id(K0[0] + bxo, K0[1] + sy, K0[2] + sz);
    };
    int n2 = 0;
    if (DENSE && brick_ok) {
      // two passes over the brick list in chunks of 32: arg-min of the upper
      // bounds (the reference s0), then tau + bisector cull and compaction in
      // slot (= site index) order
      const FBox Bs = box_sub(sz, sext[2]);
      auto okey = [](float v) -> unsigned {
        const unsigned b = __float_as_uint(v);
        return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
      };
      unsigned km = 0xffffffffu;
      for (int c0 = 0; c0 < nW; c0 += 32) {
        const int k = c0 + lane;
        if (k < nW) {
          const int f = ws.W[k];
          SiteF t;
          fbounds<KIND, PER>(S.rel[f], S.flag[f], Bs, halfLf, invG, t);
          km = min(km, (okey(t.ubp) & ~255u) | (unsigned)k);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) km = min(km, __shfl_xor_sync(0xffffffffu, km, o));
      const int r0 = (int)(km & 255u);
      const int fr = nW > 0 ? ws.W[r0] : 0;  // empty list (n2 = 0): any in-bounds slot
      const unsigned fl0 = S.flag[fr];
      SiteF z;  // every lane derives the reference's bounds itself
      fbounds<KIND, PER>(S.rel[fr], fl0, Bs, halfLf, invG, z);
      float zZ2, zKz;
      ref_consts(z, Bs, e_d, zZ2, zKz);
      const float tau = fminf(z.ubp, tcf);  // >= the minimum upper bound: a valid cull level
      for (int c0 = 0; c0 < nW; c0 += 32) {
        const int k = c0 + lane;
        bool keep = false;
        int f = 0;
        if (k < nW) {
          f = ws.W[k];
          const unsigned fl = S.flag[f];
          SiteF t;
          fbounds<KIND, PER>(S.rel[f], fl, Bs, halfLf, invG, t);
          keep = k == r0 || (t.lbp <= tau && bisector_keep<KIND, PER>(t, fl, z, fl0, Bs, halfLf, invG, e_d, zZ2, zKz));
        }
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        const int pos = n2 + __popc(m & ((1u << lane) - 1u));
        if (keep && pos < kLcapD) ws.L[pos] = S.p[f];
        n2 += __popc(m);
      }
      __syncwarp();
      const long long sbi = sb_id(K0[0] + bxo, K0[1] + sy, K0[2] + sz);
      // 64-bit list offsets: the counter keeps growing past list_cap, and
      // only offsets with base + n2 <= list_cap (< 2^31) are ever written
      long long base = 0;
      if (lane == 0 && n2 > kSlot && n2 <= kLcapD) base = (long long)atomicAdd(list_count, (unsigned long long)n2);
      base = __shfl_sync(0xffffffffu, base, 0);
      const bool ok = n2 <= kLcapD && (n2 <= kSlot || base + n2 <= list_cap);
      if (ok) {
        int* dst = n2 <= kSlot ? slots16 + sbi * kSlot : list + base;
        for (int i = lane; i < n2; i += 32) dst[i] = ws.L[i];
      }
      __syncwarp();
      if (VX_STATS_ON && lane == 0) {
        atomicAdd(&eval_slots[69], (unsigned long long)n2);
        atomicAdd(&eval_slots[70], 1ull);
        atomicMax(&eval_slots[73], (unsigned long long)n2);
      }
      if (lane == 0) {
        info[sbi] = ok ? make_int2((int)base, n2) : make_int2(0, -1);
        if (!ok) ovf[atomicAdd(&ctr->n_ovf_sb, 1ull)] = (int)sbi;
        if (ok) ws.evals += (unsigned)(n2 * sext[0] * sext[1] * sext[2]);
      }
    } else if (brick_ok) {
      const FBox Bs = box_sub(sz, sext[2]);
      // one bound evaluation per brick-list site, kept in registers (slots
      // lane and lane + 32; nW <= 64)
      const bool va = lane < nW, vb = lane + 32 < nW;
      const int fa = va ? Wl[lane] : 0, fb = vb ? Wl[lane + 32] : 0;
      const unsigned fla = va ? S.flag[fa] : 0u, flb = vb ? S.flag[fb] : 0u;
      SiteF sa, sb;
      fbounds<KIND, PER>(S.rel[fa], fla, Bs, halfLf, invG, sa);
      if (vb) fbounds<KIND, PER>(S.rel[fb], flb, Bs, halfLf, invG, sb);
      // packed (upper bound, slot) arg-min -> reference s0 and tau = its ubp
      // (Voronoi: ubp >= 0, whose bits already order as unsigned integers)
      auto okey = [](float v) -> unsigned {
        const unsigned b = __float_as_uint(v);
        if (KIND == kVoronoi) return b;
        return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
      };
      unsigned km = min(va ? ((okey(sa.ubp) & ~63u) | (unsigned)lane) : 0xffffffffu,
                        vb ? ((okey(sb.ubp) & ~63u) | (unsigned)(lane + 32)) : 0xffffffffu);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) km = min(km, __shfl_xor_sync(0xffffffffu, km, o));
      const int r0 = (int)(km & 63u), rl = r0 & 31;
      const bool rhi = r0 >= 32;
      // the reference's bounds through shared memory, written by its owner lane
      if (lane == rl) {
        const SiteF& o = rhi ? sb : sa;
        float* zr = ws.zref;
        zr[0] = o.v[0], zr[1] = o.v[1], zr[2] = o.v[2];
        zr[3] = o.mn[0], zr[4] = o.mn[1], zr[5] = o.mn[2];
        zr[6] = o.mx[0], zr[7] = o.mx[1], zr[8] = o.mx[2];
        zr[9] = o.t, zr[10] = o.lb, zr[11] = o.ub, zr[12] = o.ubp;
        zr[13] = __uint_as_float(rhi ? flb : fla);
        ref_consts(o, Bs, e_d, zr[14], zr[15]);
      }
      // Voronoi brick lists: a second reference, the next-least upper bound
      // (cfg2 -2.4 %, cfg5 -1.6 %; JM / Laguerre spill with it), published
      // before the same barrier as the first
      bool two = false;
      int r1 = 0;
      if constexpr (KIND == kVoronoi && BM) {
      unsigned km2 = min(va && lane != r0 ? ((okey(sa.ubp) & ~63u) | (unsigned)lane) : 0xffffffffu,
                         vb && lane + 32 != r0 ? ((okey(sb.ubp) & ~63u) | (unsigned)(lane + 32)) : 0xffffffffu);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) km2 = min(km2, __shfl_xor_sync(0xffffffffu, km2, o));
      two = km2 != 0xffffffffu;
      r1 = (int)(km2 & 63u);
      const int rl1 = r1 & 31;
      const bool rhi1 = r1 >= 32;
      if (two && lane == rl1) {
        const SiteF& o = rhi1 ? sb : sa;
        float* zr = ws.zref2;
        zr[0] = o.v[0], zr[1] = o.v[1], zr[2] = o.v[2];
        zr[3] = o.mn[0], zr[4] = o.mn[1], zr[5] = o.mn[2];
        zr[6] = o.mx[0], zr[7] = o.mx[1], zr[8] = o.mx[2];
        zr[9] = o.t, zr[10] = o.lb, zr[11] = o.ub, zr[12] = o.ubp;
        zr[13] = __uint_as_float(rhi1 ? flb : fla);
        ref_consts(o, Bs, e_d, zr[14], zr[15]);
      }
      }
      __syncwarp();
      SiteF z;
      float4 q3;
      {
        const float4 q0 = *reinterpret_cast<const float4*>(&ws.zref[0]);
        const float4 q1 = *reinterpret_cast<const float4*>(&ws.zref[4]);
        const float4 q2 = *reinterpret_cast<const float4*>(&ws.zref[8]);
        q3 = *reinterpret_cast<const float4*>(&ws.zref[12]);
        z.v[0] = q0.x, z.v[1] = q0.y, z.v[2] = q0.z;
        z.mn[0] = q0.w, z.mn[1] = q1.x, z.mn[2] = q1.y;
        z.mx[0] = q1.z, z.mx[1] = q1.w, z.mx[2] = q2.x;
        z.t = q2.y, z.lb = q2.z, z.ub = q2.w;
        z.ubp = q3.x;
      }
      const float tau = fminf(z.ubp, tcf);
      const unsigned fl0 = __float_as_uint(q3.y);
      const float zZ2 = q3.z, zKz = q3.w;
      bool ka, kb;
      if constexpr (KIND == kVoronoi && BM) {
      auto keep2 = [&](const SiteF& sx, unsigned flx, int slot) {
        if (!two || slot == r1) return true;
        SiteF z2;
        const float4 q0 = *reinterpret_cast<const float4*>(&ws.zref2[0]);
        const float4 q1 = *reinterpret_cast<const float4*>(&ws.zref2[4]);
        const float4 q2 = *reinterpret_cast<const float4*>(&ws.zref2[8]);
        z2.v[0] = q0.x, z2.v[1] = q0.y, z2.v[2] = q0.z;
        z2.mn[0] = q0.w, z2.mn[1] = q1.x, z2.mn[2] = q1.y;
        z2.mx[0] = q1.z, z2.mx[1] = q1.w, z2.mx[2] = q2.x;
        z2.t = q2.y, z2.lb = q2.z, z2.ub = q2.w;
        const float4 q3b = *reinterpret_cast<const float4*>(&ws.zref2[12]);
        return bisector_keep<KIND, PER>(sx, flx, z2, __float_as_uint(q3b.y), Bs, halfLf, invG, e_d, q3b.z, q3b.w);
      };
      ka = va && (lane == r0 || (sa.lbp <= tau &&
                                            bisector_keep<KIND, PER>(sa, fla, z, fl0, Bs, halfLf, invG, e_d, zZ2, zKz) &&
                                            keep2(sa, fla, lane)));
      kb = vb && (lane + 32 == r0 || (sb.lbp <= tau &&
                                                 bisector_keep<KIND, PER>(sb, flb, z, fl0, Bs, halfLf, invG, e_d, zZ2, zKz) &&
                                                 keep2(sb, flb, lane + 32)));
      } else {
      ka = va && (lane == r0 || (sa.lbp <= tau &&
                                            bisector_keep<KIND, PER>(sa, fla, z, fl0, Bs, halfLf, invG, e_d, zZ2, zKz)));
      kb = vb && (lane + 32 == r0 || (sb.lbp <= tau &&
                                                 bisector_keep<KIND, PER>(sb, flb, z, fl0, Bs, halfLf, invG, e_d, zZ2, zKz)));
      }
#ifdef VX_NO_BSTAGE  // experiment: the column pass's brick lists unrefined
      ka = va;
      kb = vb;
#endif
      // survivors -> the sub-brick's kSlot fixed slots (or the overflow
      // list when longer), in slot (= site index) order
      const long long sbi = list_id();
      const unsigned ma = __ballot_sync(0xffffffffu, ka), mb = __ballot_sync(0xffffffffu, kb);
      n2 = __popc(ma) + __popc(mb);
      long long base = 0;
      if (lane == 0 && n2 > kSlot && n2 <= kLcap) base = (long long)atomicAdd(list_count, (unsigned long long)n2);
      base = __shfl_sync(0xffffffffu, base, 0);
      const bool ok = n2 <= kLcap && (n2 <= kSlot || base + n2 <= list_cap);
      if (ok) {
        const unsigned lt = (1u << lane) - 1u;
        int* dst = n2 <= kSlot ? slots16 + sbi * kSlot : list + base;
        if (ka) dst[__popc(ma & lt)] = S.p[fa];
        if (kb) dst[__popc(ma) + __popc(mb & lt)] = S.p[fb];
      }
      if (VX_STATS_ON && lane == 0) {
        atomicAdd(&eval_slots[69], (unsigned long long)n2);
        atomicAdd(&eval_slots[70], 1ull);
        atomicMax(&eval_slots[73], (unsigned long long)n2);
      }
      if (lane == 0) {
        info[sbi] = ok ? make_int2((int)base, n2) : make_int2(0, -1);
        if (!ok) push_ovf();
        if (ok && n2 <= kFcap) ws.evals += (unsigned)(n2 * sext[0] * sext[1] * sext[2]);
      }
    } else if (lane == 0) {
      info[list_id()] = make_int2(0, -1);
      push_ovf();
    }
  }
  if (lane == 0 && !brick_ok) atomicAdd(&ctr->overflow_bricks, 1ull);
  }  // bb
  // the ball-phase evaluation counter (EvalCounters::step1_evals), one atomic per warp
  if (lane == 0 && ws.evals)
    atomicAdd(&eval_slots[(blockIdx.x + 8 * blockIdx.y + wid) & 63], (unsigned long long)ws.evals);
}

// exact per-axis tables (the reference arithmetic): one lane per (site, axis)
// computes w^2 at the sub-brick's 8 (z: 4) voxel centres; u = site - centre
// (geometry.hpp:58-60) is wrapped only when |u| >= 0.49 L -- below that
// floor(u/L + 0.5) == 0 and the reference's wrap returns u itself
template <bool PER, class ES>
__device__ __forceinline__ void exact_tables(ES& ws, const Bins& bins, const Geo& g, int lane, int c0, int m) {
  for (int e = lane; e < 3 * m; e += 32) {
    const int a = e >= 2 * m ? 2 : (e >= m ? 1 : 0);
    const int j = e - a * m;
    const int p = ws.P[c0 + j];
    const double sv = bins.x[p + a * bins.stride];  // x, y, z arrays are contiguous
    const double* cr = &ws.C[a * 8];
    double u[8];
    const double La = PER ? (a == 0 ? g.L[0] : (a == 1 ? g.L[1] : g.L[2])) : 0.0;
    const double lim = 0.49 * La;
#pragma unroll
    for (int r = 0; r < 8; ++r) u[r] = __dsub_rn(sv, cr[r]);
    // u is monotone in the (increasing) centres: |u| peaks at an end (for z
    // the 4th centre repeats as entries 4..7 when a sub-brick is short)
    if (PER && (!(fabs(u[0]) < lim) || !(fabs(u[7]) < lim) || !(fabs(u[3]) < lim))) {  // rare: ~half a period away
      const double iLa = a == 0 ? g.invL[0] : (a == 1 ? g.invL[1] : g.invL[2]);
#pragma unroll
      for (int r = 0; r < 8; ++r)
        if (!(fabs(u[r]) < lim)) u[r] = wrap_delta(u[r], La, iLa);
    }
    double* trow = &ws.T[j][a * 8];
#pragma unroll
    for (int r = 0; r < 8; ++r)
      if (r < 4 || a != 2) trow[r] = __dmul_rn(u[r], u[r]);
  }
}

// one sub-brick (warp) per CTA: a CTA slot frees as soon as its sub-brick is
// done (1 / 2 / 4 warps per CTA: cfg5 eval+cull 6.79 / 6.92 / 6.97 ms)
#ifndef VX_EVAL_WARPS
#define VX_EVAL_WARPS 1
#endif
constexpr int kEvalWarps = VX_EVAL_WARPS;  // sub-bricks along y per CTA
constexpr unsigned kMaxGridY = 65535;      // gridDim.y limit: taller grids launch in y-chunks
#ifndef VX_EVAL16_MINB
#define VX_EVAL16_MINB 24  // 80 registers, no spills (20: 92 registers, 28: spills; cfg5 6.63 / 7.05 / 7.20 ms)
#endif

// One warp per 8x8x4 sub-brick (the tail of v11's sub-brick loop: exact
// tables, evaluation, stores, histogram, unresolved compaction).  The site
// index load is issued before the tables and consumed at the store.
template <int KIND, bool PER, bool DENSE, bool FA>
__global__ void __launch_bounds__(kEvalWarps * 32, 32 / kEvalWarps)
    eval12_kernel(Geo g, Bins bins, const DevParams* __restrict__ prm, const int2* __restrict__ info,
                  const int* __restrict__ slots16, const int* __restrict__ list, int* __restrict__ labels,
                  double* __restrict__ dist,
                  unsigned long long* __restrict__ hist, long long* __restrict__ unres, long long unres_cap,
                  DevCounters* ctr, unsigned long long* __restrict__ eval_slots, long long nsb, unsigned sby0) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  using ES = EvalSmemT<DENSE ? kLcapD : kFcap>;
  ES& ws = reinterpret_cast<ES*>(smem_raw)[wid];
  const unsigned nsbx = g.nsbx, nsby = g.nsby;
  const double cutoff = prm->cutoff;
  const int qx = (lane & 1) * 4, vy = (lane >> 1) & 3, vz = lane >> 3;
  // grid (nsbx, ceil(nsby / 8), nsbz): no index division
  const unsigned sbx = blockIdx.x, sby = sby0 + blockIdx.y * kEvalWarps + wid, sbz = blockIdx.z;
  if (sby >= nsby) return;
  const long long sb = (long long)sbx + (long long)nsbx * ((long long)sby + (long long)nsby * sbz);
  const int2 inf = info[sb];
  const int ps = lane < kSlot ? slots16[sb * kSlot + lane] : 0;  // issued with info, not after it
  const int pl = inf.y > kSlot ? (lane < inf.y ? list[inf.x + lane] : 0) : ps;
  if (inf.y < 0) return;  // overflowed the ball phase's caps: the sub-brick shell labels it
  {
    const int x0 = (int)sbx * 8, y0 = (int)sby * 8;
    const long long z0 = g.z_begin + (long long)sbz * 4;
    const int sext[3] = {min(8, (int)g.n[0] - x0), min(8, (int)g.n[1] - y0), (int)min(4ll, g.z_end - z0)};
    // lists longer than the tables (a few per image at the benchmark densities)
    // send their voxels to the per-voxel shell search
    const int n2 = inf.y <= (DENSE ? kLcapD : kFcap) ? inf.y : 0;
    int fidx = 0;
    if constexpr (DENSE) {
      for (int i = lane; i < n2; i += 32) {
        const int p = n2 <= kSlot ? slots16[sb * kSlot + i] : list[inf.x + i];
        ws.P[i] = p;
        ws.cnt[i] = 0;
        ws.Fidx[i] = bins.idx[p];
        if (KIND != kVoronoi) ws.Ft[i] = bins.t[p];
      }
    } else {
      if (lane < n2) {
        ws.P[lane] = pl;
        ws.cnt[lane] = 0;
        fidx = bins.idx[pl];
        if (KIND != kVoronoi) ws.Ft[lane] = bins.t[pl];
      }
    }
    if (lane < 24 && n2 > 0) {  // the sub-brick's voxel centres, once (geometry.hpp:58-60)
      const int a = lane >> 3;
      // beyond the grid the last centre repeats (never stored); z entries 4..7 repeat the 4th
      const int k = min(lane & 7, (a == 0 ? sext[0] : (a == 1 ? sext[1] : sext[2])) - 1);
      const long long k0 = a == 0 ? (long long)x0 : (a == 1 ? (long long)y0 : z0);
      ws.C[lane] = center(k0 + k, a == 0 ? g.sp[0] : (a == 1 ? g.sp[1] : g.sp[2]));
    }
    __syncwarp();
    auto store_tail = [&](double (&best)[8], int (&bj)[8]) {
    // resolve + store + compaction of unresolved voxels
    if constexpr (!DENSE) {
      if (lane < n2) ws.Fidx[lane] = fidx;  // its load was issued before the tables
    }
    __syncwarp();

    // voxel offset inside the slab (the unresolved list holds absolute indices)
    const long long lrel = (long long)(sbz * 4 + vz) * g.plane + (long long)(y0 + vy) * g.n[0] + x0 + qx;
    const long long rstep = 4 * g.n[0];  // row vy -> vy + 4
    // bit k: voxel k of this lane lies inside the grid
    const int xr = sext[0] - qx;
    const unsigned xm = xr >= 4 ? 0xFu : (xr > 0 ? (1u << xr) - 1u : 0u);
    const unsigned vmask = vz < sext[2] ? ((vy < sext[1] ? xm : 0u) | (vy + 4 < sext[1] ? xm << 4 : 0u)) : 0u;
    int lab[8];
    unsigned umask = 0;  // bit k: voxel k valid but unresolved
    // sub-bricks entirely inside the grid skip the per-voxel validity tests
    auto resolve = [&](auto full_tag) {
      constexpr bool FULL = decltype(full_tag)::value;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        lab[k] = -1;
        if (FULL || ((vmask >> k) & 1u)) {
          if (best[k] <= cutoff) {  // best = +inf when there is no candidate
            lab[k] = ws.Fidx[bj[k]];
            if (hist) atomicAdd(&ws.cnt[bj[k]], 1);
          } else {
            umask |= 1u << k;
          }
        }
      }
    };
    bool allin = true;  // every voxel of the lane within the cutoff
#pragma unroll
    for (int k = 0; k < 8; ++k) allin &= best[k] <= cutoff;
    if (__all_sync(0xffffffffu, vmask == 0xFFu && allin)) {  // the common case: straight-line
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        lab[k] = ws.Fidx[bj[k]];
        if (hist) atomicAdd(&ws.cnt[bj[k]], 1);
      }
    } else if (vmask == 0xFFu) {
      resolve(std::true_type{});
    } else {
      resolve(std::false_type{});
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (!((vmask >> (4 * h)) & 0xFu)) continue;
      int* out = labels + (lrel + h * rstep);
      if (xm == 0xFu && g.vec_store) {
        *reinterpret_cast<int4*>(out) = make_int4(lab[4 * h], lab[4 * h + 1], lab[4 * h + 2], lab[4 * h + 3]);
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if ((xm >> k) & 1u) out[k] = lab[4 * h + k];
      }
      if (dist) {
        double* dout = dist + (lrel + h * rstep);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (((xm >> k) & 1u) && lab[4 * h + k] >= 0)
            dout[k] = KIND == kVoronoi ? __dsqrt_rn(best[4 * h + k]) : best[4 * h + k];
      }
    }
    if (__any_sync(0xffffffffu, umask != 0)) {  // K3: compaction of unresolved voxels
      const int nun = __popc(umask);
      int inc = nun;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      const int wtot = __shfl_sync(0xffffffffu, inc, 31);
      unsigned long long base = 0;
      if (lane == 31) base = atomicAdd(&ctr->n_unres, (unsigned long long)wtot);
      base = __shfl_sync(0xffffffffu, base, 31);
      const long long off = (long long)base + inc - nun;
      unsigned mm = umask;
      for (int i = 0; i < nun; ++i) {
        const int k = __ffs(mm) - 1;
        mm &= mm - 1;
        if (off + i < unres_cap) unres[off + i] = g.z_begin * g.plane + lrel + (k < 4 ? 0 : rstep) + (k & 3);
      }
    }
    if (hist && n2 > 0) {
      __syncwarp();
      for (int i = lane; i < (DENSE ? n2 : min(n2, 32)); i += 32)
        if (ws.cnt[i]) atomicAdd(&hist[ws.Fidx[i]], (unsigned long long)ws.cnt[i]);
    }
    };
    if constexpr (DENSE) {
      double best[8];
      int bj[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        best[k] = __longlong_as_double(0x7ff0000000000000ll);
        bj[k] = 0;  // any in-range slot: unresolved voxels never read it
      }
      const bool g1 = g.g_is_one;
      // candidates in passes of kFcap tables; the running minimum carries
      // over, so the scan order is still ascending site index
      for (int c0 = 0; c0 < n2; c0 += kFcap) {
        const int m = min(kFcap, n2 - c0);
    exact_tables<PER>(ws, bins, g, lane, c0, m);
    __syncwarp();
    // exact evaluation: lane -> 4 voxels along x in rows vy and vy + 4
    for (int j = 0; j < m; ++j) {
      const double wz = ws.T[j][16 + vz];
      const double a0 = __dadd_rn(wz, ws.T[j][8 + vy]);  // 0 + wz^2 == wz^2
      const double a1 = __dadd_rn(wz, ws.T[j][12 + vy]);
      const double2 w01 = *reinterpret_cast<const double2*>(&ws.T[j][qx]);
      const double2 w23 = *reinterpret_cast<const double2*>(&ws.T[j][qx + 2]);
      const double tj = KIND == kVoronoi ? 0.0 : ws.Ft[c0 + j];
      const double d[8] = {__dadd_rn(a0, w01.x), __dadd_rn(a0, w01.y), __dadd_rn(a0, w23.x),
                           __dadd_rn(a0, w23.y), __dadd_rn(a1, w01.x), __dadd_rn(a1, w01.y),
                           __dadd_rn(a1, w23.x), __dadd_rn(a1, w23.y)};
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const double pr = FA ? prox_from_dsq_nc<KIND>(d[k], g.growth, g1, tj, g.inv_growth_rn)
                                : prox_from_dsq<KIND>(d[k], g.growth, g1, tj);
        if (pr < best[k]) {
          best[k] = pr;
          bj[k] = c0 + j;
        }
      }
    }
        __syncwarp();  // the next pass rewrites the tables
      }
      store_tail(best, bj);
    } else {
    exact_tables<PER>(ws, bins, g, lane, 0, n2);
    __syncwarp();
    // exact evaluation: lane -> 4 voxels along x in rows vy and vy + 4
    double best[8];
    int bj[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      best[k] = __longlong_as_double(0x7ff0000000000000ll);
      bj[k] = 0;  // any in-range slot: unresolved voxels never read it
    }
    const bool g1 = g.g_is_one;
    for (int j = 0; j < n2; ++j) {
      const double wz = ws.T[j][16 + vz];
      const double a0 = __dadd_rn(wz, ws.T[j][8 + vy]);  // 0 + wz^2 == wz^2
      const double a1 = __dadd_rn(wz, ws.T[j][12 + vy]);
      const double2 w01 = *reinterpret_cast<const double2*>(&ws.T[j][qx]);
      const double2 w23 = *reinterpret_cast<const double2*>(&ws.T[j][qx + 2]);
      const double tj = KIND == kVoronoi ? 0.0 : ws.Ft[j];
      const double d[8] = {__dadd_rn(a0, w01.x), __dadd_rn(a0, w01.y), __dadd_rn(a0, w23.x),
                           __dadd_rn(a0, w23.y), __dadd_rn(a1, w01.x), __dadd_rn(a1, w01.y),
                           __dadd_rn(a1, w23.x), __dadd_rn(a1, w23.y)};
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const double pr = FA ? prox_from_dsq_nc<KIND>(d[k], g.growth, g1, tj, g.inv_growth_rn)
                                : prox_from_dsq<KIND>(d[k], g.growth, g1, tj);
        if (pr < best[k]) {
          best[k] = pr;
          bj[k] = j;
        }
      }
    }
      store_tail(best, bj);
    }
  }
}


// eval16 (standard lists per 8^3 brick): one warp per brick, 16 voxels per
// lane -- 4 along x in rows (vy, vy + 4) of planes (vz, vz + 4) -- so the x
// table, the y-z sums and the per-brick setup are shared by twice the voxels
// of eval12.  Same exact arithmetic, ascending-index strict-< scan, resolve,
// stores, histogram and compaction.
struct __align__(16) Eval16Smem {
  double T[kFcap][24]; // exact w^2: [0,8) x, [8,16) y, [16,24) z (Voronoi / Laguerre: y, z in the order 0 4 1 5 2 6 3 7)
  double C[24];
  double Ft[kFcap];
  int P[kFcap];
  int Fidx[kFcap];
  int cnt[kFcap];
};

#ifndef VX_JM_BRICKS
#define VX_JM_BRICKS 1
#endif
#ifndef VX_E16_PACK
#define VX_E16_PACK 1  // 0: one slot register per voxel (A/B)
#endif
// strict-< update of one voxel's best prox; its winner slot is byte SEL of
// bjp (prmt selector: that byte from jj = j * 0x01010101, the others kept),
// both under the compare's predicate
template <unsigned SEL>
__device__ __forceinline__ void upd_slot(unsigned& bjp, double& best, double pr, unsigned jj) {
  asm("{\n\t.reg .pred p;\n\tsetp.lt.f64 p, %2, %1;\n\t@p mov.f64 %1, %2;\n\t"
      "@p prmt.b32 %0, %0, %3, %4;\n\t}"
      : "+r"(bjp), "+d"(best)
      : "d"(pr), "r"(jj), "n"(SEL));
}
#ifndef VX_E16_UNROLL
#define VX_E16_UNROLL 1
#endif
constexpr int kE16Unroll = VX_E16_UNROLL;
#ifndef VX_EVAL16_MINB_V
// Voronoi / Laguerre (packed slots): 72 registers (Voronoi no spills: cfg5
// -1.3 %, cfg2 -3.1 %; Laguerre 4 B of spills: cfg3 -2.6 %); JM keeps 80
#define VX_EVAL16_MINB_V 28
#endif
template <int KIND, bool PER, bool FA>
__global__ void __launch_bounds__(32, KIND == kJohnsonMehl ? VX_EVAL16_MINB : VX_EVAL16_MINB_V)
    eval16_kernel(Geo g, Bins bins, const DevParams* __restrict__ prm, const int2* __restrict__ info,
                  const int* __restrict__ slots16, const int* __restrict__ list, int* __restrict__ labels,
                  double* __restrict__ dist, unsigned long long* __restrict__ hist, long long* __restrict__ unres,
                  long long unres_cap, DevCounters* ctr, unsigned by0) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Eval16Smem& ws = *reinterpret_cast<Eval16Smem*>(smem_raw);
  const int lane = threadIdx.x & 31;
  const unsigned nsbx = g.nsbx, nsby = g.nsby;
  const double cutoff = prm->cutoff;
  const int qx = (lane & 1) * 4, vy = (lane >> 1) & 3, vz = lane >> 3;
  const unsigned bx = blockIdx.x, by = by0 + blockIdx.y, bz = blockIdx.z;
  if (by >= nsby) return;
  const long long bi = (long long)bx + (long long)nsbx * ((long long)by + (long long)nsby * bz);
  const int2 inf = info[bi];
  const int ps = lane < kSlot ? slots16[bi * kSlot + lane] : 0;
  const int pl = inf.y > kSlot ? (lane < inf.y ? list[inf.x + lane] : 0) : ps;
  if (inf.y < 0) return;  // overflowed: the sub-brick shell labels it
  const int x0 = (int)bx * 8, y0 = (int)by * 8;
  const long long z0 = g.z_begin + (long long)bz * 8;
  const int bext[3] = {min(8, (int)g.n[0] - x0), min(8, (int)g.n[1] - y0), (int)min(8ll, g.z_end - z0)};
  const int n2 = inf.y <= kFcap ? inf.y : 0;  // longer lists: the per-voxel shell
  int fidx = 0;
  if (lane < n2) {
    ws.P[lane] = pl;
    ws.cnt[lane] = 0;
    fidx = bins.idx[pl];
    if (KIND != kVoronoi) ws.Ft[lane] = bins.t[pl];
  }
  if (lane < 24 && n2 > 0) {  // the brick's voxel centres (geometry.hpp:58-60)
    // y and z in the order 0 4 1 5 2 6 3 7, so a lane's two rows / planes
    // (v, v + 4) are adjacent in the tables (one 16-byte load each); the
    // first and last entries stay the extremes the wrap test looks at
    const int a = lane >> 3, s8 = lane & 7;
    const int kk = a == 0 || KIND == kJohnsonMehl ? s8 : (s8 >> 1) + 4 * (s8 & 1);  // JM: natural order (+1.4 % interleaved)
    const int k = min(kk, (a == 0 ? bext[0] : (a == 1 ? bext[1] : bext[2])) - 1);
    const long long k0 = a == 0 ? (long long)x0 : (a == 1 ? (long long)y0 : z0);
    ws.C[lane] = center(k0 + k, a == 0 ? g.sp[0] : (a == 1 ? g.sp[1] : g.sp[2]));
  }
  __syncwarp();
  // exact tables: one lane per (site, axis), 8 entries each
  for (int e = lane; e < 3 * n2; e += 32) {
    const int a = e >= 2 * n2 ? 2 : (e >= n2 ? 1 : 0);
    const int j = e - a * n2;
    const double sv = bins.x[ws.P[j] + a * bins.stride];
    const double* cr = &ws.C[a * 8];
    double u[8];
    const double La = PER ? (a == 0 ? g.L[0] : (a == 1 ? g.L[1] : g.L[2])) : 0.0;
    const double lim = 0.49 * La;
#pragma unroll
    for (int r = 0; r < 8; ++r) u[r] = __dsub_rn(sv, cr[r]);
    if (PER && (!(fabs(u[0]) < lim) || !(fabs(u[7]) < lim))) {
      const double iLa = a == 0 ? g.invL[0] : (a == 1 ? g.invL[1] : g.invL[2]);
#pragma unroll
      for (int r = 0; r < 8; ++r)
        if (!(fabs(u[r]) < lim)) u[r] = wrap_delta(u[r], La, iLa);
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) ws.T[j][a * 8 + r] = __dmul_rn(u[r], u[r]);
  }
  if (lane < n2) ws.Fidx[lane] = fidx;
  __syncwarp();
  // voxel k = 8 zh + 4 yh + i: x = qx + i, y = vy + 4 yh, z = vz + 4 zh
  // the winner slots as bytes of bjp (4 registers instead of 16): Voronoi
  // and Laguerre run at 72 registers / 28 warps per SM, JM's in-loop sqrt
  // fits 80 without spills
  constexpr bool PACK = VX_E16_PACK != 0;
  double best[16];
  unsigned bjp[4] = {0u, 0u, 0u, 0u};
  int bj[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    best[k] = __longlong_as_double(0x7ff0000000000000ll);
    bj[k] = 0;
  }
  const bool g1 = g.g_is_one;
#pragma unroll kE16Unroll
  for (int j = 0; j < n2; ++j) {
    // packed slots hold byte offsets 4 j (< 128) into the int arrays Fidx / cnt
    const unsigned jj = PACK ? (unsigned)j * 0x04040404u : (unsigned)j * 0x01010101u;
    double wz0, wz1, wy0, wy1;
    if constexpr (KIND != kJohnsonMehl) {
      const double2 wz = *reinterpret_cast<const double2*>(&ws.T[j][16 + 2 * vz]);  // planes vz, vz + 4
      const double2 wy = *reinterpret_cast<const double2*>(&ws.T[j][8 + 2 * vy]);   // rows vy, vy + 4
      wz0 = wz.x, wz1 = wz.y, wy0 = wy.x, wy1 = wy.y;
    } else {
      wz0 = ws.T[j][16 + vz], wz1 = ws.T[j][20 + vz];
      wy0 = ws.T[j][8 + vy], wy1 = ws.T[j][12 + vy];
    }
    const double a[4] = {__dadd_rn(wz0, wy0), __dadd_rn(wz0, wy1), __dadd_rn(wz1, wy0), __dadd_rn(wz1, wy1)};
    const double2 w01 = *reinterpret_cast<const double2*>(&ws.T[j][qx]);
    const double2 w23 = *reinterpret_cast<const double2*>(&ws.T[j][qx + 2]);
    const double wx[4] = {w01.x, w01.y, w23.x, w23.y};
    const double tj = KIND == kVoronoi ? 0.0 : ws.Ft[j];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if constexpr (PACK) {
        double pr[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const double d = __dadd_rn(a[r], wx[i]);
          pr[i] = FA ? prox_from_dsq_nc<KIND>(d, g.growth, g1, tj, g.inv_growth_rn)
                     : prox_from_dsq<KIND>(d, g.growth, g1, tj);
        }
        upd_slot<0x3214>(bjp[r], best[4 * r + 0], pr[0], jj);
        upd_slot<0x3240>(bjp[r], best[4 * r + 1], pr[1], jj);
        upd_slot<0x3410>(bjp[r], best[4 * r + 2], pr[2], jj);
        upd_slot<0x4210>(bjp[r], best[4 * r + 3], pr[3], jj);
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const double d = __dadd_rn(a[r], wx[i]);
          const double pr = FA ? prox_from_dsq_nc<KIND>(d, g.growth, g1, tj, g.inv_growth_rn)
                               : prox_from_dsq<KIND>(d, g.growth, g1, tj);
          const int k = 4 * r + i;  // r = 2 zh + yh
          if (pr < best[k]) {
            best[k] = pr;
            bj[k] = j;
          }
        }
      }
    }
  }
  // the winner's index / count slot of voxel k: packed, one PRMT (byte k & 3
  // of bjp[k >> 2], zero-extended) gives the byte offset itself
  auto fidx_of = [&](int k) -> int {
    if constexpr (PACK)
      return *reinterpret_cast<const int*>(reinterpret_cast<const char*>(ws.Fidx) +
                                           __byte_perm(bjp[k >> 2], 0u, 0x4440u + (unsigned)(k & 3)));
    else
      return ws.Fidx[bj[k]];
  };
  auto cnt_of = [&](int k) -> int* {
    if constexpr (PACK)
      return reinterpret_cast<int*>(reinterpret_cast<char*>(ws.cnt) +
                                    __byte_perm(bjp[k >> 2], 0u, 0x4440u + (unsigned)(k & 3)));
    else
      return &ws.cnt[bj[k]];
  };
  // ---- resolve + store + compaction ----
  const int xr = bext[0] - qx;
  const unsigned xm = xr >= 4 ? 0xFu : (xr > 0 ? (1u << xr) - 1u : 0u);
  unsigned vmask = 0xFFFFu;  // bricks inside the grid (warp-uniform test)
  if (bext[0] < 8 || bext[1] < 8 || bext[2] < 8) {
    vmask = 0;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int yy = vy + 4 * (r & 1), zz = vz + 4 * (r >> 1);
      if (yy < bext[1] && zz < bext[2]) vmask |= xm << (4 * r);
    }
  }
  int lab[16];
  unsigned umask = 0;
  // bricks entirely inside the grid (all but the boundary layers) skip the
  // per-voxel validity tests
  auto resolve = [&](auto full_tag) {
    constexpr bool FULL = decltype(full_tag)::value;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      lab[k] = -1;
      if (FULL || ((vmask >> k) & 1u)) {
        if (best[k] <= cutoff) {
          lab[k] = fidx_of(k);
          if (hist) atomicAdd(cnt_of(k), 1);
        } else {
          umask |= 1u << k;
        }
      }
    }
  };
  bool allin = true;  // every voxel of the lane within the cutoff
#pragma unroll
  for (int k = 0; k < 16; ++k) allin &= best[k] <= cutoff;
  if (__all_sync(0xffffffffu, vmask == 0xFFFFu && allin)) {
    // the common case (whole brick inside the grid and inside the balls):
    // straight-line label lookups and histogram counts
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      lab[k] = fidx_of(k);
      if (hist) atomicAdd(cnt_of(k), 1);
    }
  } else if (vmask == 0xFFFFu) {
    resolve(std::true_type{});
  } else {
    resolve(std::false_type{});
  }
  const long long slab_z = (long long)bz * 8 + vz;  // z inside the slab
  // row r = 2 zh + yh: voxel offset of its first x, rows 4 planes / 4 rows apart
  const long long vox0 = slab_z * g.plane + (long long)(y0 + vy) * g.n[0] + x0 + qx;
  const long long ystep = 4 * g.n[0], zstep = 4 * g.plane;
  auto vox = [&](int r) -> long long { return vox0 + (r >> 1) * zstep + (r & 1) * ystep; };
  const bool full = vmask == 0xFFFFu;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    if (!full && !((vmask >> (4 * r)) & 0xFu)) continue;
    int* out = labels + vox(r);
    if ((full || xm == 0xFu) && g.vec_store) {
      *reinterpret_cast<int4*>(out) = make_int4(lab[4 * r], lab[4 * r + 1], lab[4 * r + 2], lab[4 * r + 3]);
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if ((xm >> i) & 1u) out[i] = lab[4 * r + i];
    }
    if (dist) {
      double* dout = dist + vox(r);
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (((xm >> i) & 1u) && lab[4 * r + i] >= 0)
          dout[i] = KIND == kVoronoi ? __dsqrt_rn(best[4 * r + i]) : best[4 * r + i];
    }
  }
  if (__any_sync(0xffffffffu, umask != 0)) {
    const int nun = __popc(umask);
    int inc = nun;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    const int wtot = __shfl_sync(0xffffffffu, inc, 31);
    unsigned long long base = 0;
    if (lane == 31) base = atomicAdd(&ctr->n_unres, (unsigned long long)wtot);
    base = __shfl_sync(0xffffffffu, base, 31);
    const long long off = (long long)base + inc - nun;
    unsigned mm = umask;
    for (int i = 0; i < nun; ++i) {
      const int k = __ffs(mm) - 1;
      mm &= mm - 1;
      if (off + i < unres_cap) unres[off + i] = g.z_begin * g.plane + vox(k >> 2) + (k & 3);
    }
  }
  if (hist && n2 > 0) {
    __syncwarp();
    for (int i = lane; i < n2; i += 32)
      if (ws.cnt[i]) atomicAdd(&hist[ws.Fidx[i]], (unsigned long long)ws.cnt[i]);
  }
}

}  // namespace v12

__global__ void ball12_publish_kernel(const unsigned long long* slots, DevCounters* ctr) {
  unsigned long long s = 0;
  for (int i = threadIdx.x; i < 64; i += 32) s += slots[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (threadIdx.x == 0) ctr->ball_evals += s;
}

// Bricks per warp column: the tallest column (fewest gathers) whose expected
// gathered list stays well inside kTcap.  Sites per super-brick ~ density x
// (super-brick + a gather margin of ~1.6 site spacings on every side).
static int choose_nbb12(const Geo& g) {
  double L3 = 1.0;
  for (int a = 0; a < 3; ++a) L3 *= g.L[a];
  const double lambda = (double)g.n_sites / L3;
  const double spacing = pow(g.vol_true / (double)(g.n_sites > 0 ? g.n_sites : 1), 1.0 / g.dim);
  const double R = 1.6 * spacing;
  for (int nbb = v12::kMaxBB; nbb > 1; nbb >>= 1) {
    // periodic: a gathered site is within hs + R of the super-brick centre, and
    // the culling bounds need |u| + hs < L/2 (else the axis is treated as
    // ambiguous and nothing is culled along it)
    if (g.periodic && (double)(16 * nbb) * g.sp[2] + R >= 0.45 * g.L[2]) continue;
    double vol = 1.0;
    for (int a = 0; a < 3; ++a) {
      const long long ev = a < 2 ? v12::kSB : 16 * nbb;
      const double e = (double)(g.n[a] < ev ? g.n[a] : ev) * g.sp[a] + (g.n[a] > 1 ? 2.0 * R : 0.0);
      vol *= e < g.L[a] ? e : g.L[a];
    }
    if (0.7 * lambda * vol <= 0.5 * v12::kTcap) return nbb;
  }
  return 1;
}

long long ball12_subbricks(const Geo& g) {
  return ((g.n[0] + 7) / 8) * ((g.n[1] + 7) / 8) * ((g.z_end - g.z_begin + 3) / 4);
}

// Dense mode when the mean site spacing is below ~8.5 voxels (on the finest
// true axis): an 8^3 brick then sees more than ~60 sites (VX_DENSE=0/1 forces).
bool ball12_dense(const Geo& g) {
  const char* ev = std::getenv("VX_DENSE");  // read per call: tests switch it
  const int env = ev ? std::atoi(ev) : -1;
  if (env == 0 || env == 1) return env == 1;
  double sp = 1e300;
  for (int a = 0; a < 3; ++a)
    if (g.n[a] > 1) sp = std::min(sp, g.sp[a]);
  const double spacing = pow(g.vol_true / (double)(g.n_sites > 0 ? g.n_sites : 1), 1.0 / g.dim);
  if (sp < 1e300 && spacing < 8.5 * sp) return true;
  if (g.dim != 3) return false;
  // anisotropic voxels: expected sites reaching an 8 x 8 x 4 sub-brick from its
  // physical extents (+ ~1.2 site spacings of reach per axis); thick slices
  // make it elongated and its lists long at moderate density.  Measured on
  // 512^2 x (512 / r) with 10-voxel in-plane spacing (scripts/aniso_check.py):
  // dense mode wins from r ~ 3 (this estimate 9.5) on -- r = 4: 26 -> 50, r = 8:
  // 5.5 -> 29 Gvox/s -- and loses below (r = 2, estimate 8.0: 88 vs 73).
  const double lambda = (double)g.n_sites / g.vol_true;
  const double ext[3] = {8.0 * g.sp[0], 8.0 * g.sp[1], 4.0 * g.sp[2]};
  double e = lambda;
  for (int a = 0; a < 3; ++a) e *= ext[a] + 1.2 * spacing;
  return e > 9.5;
}

template <int KIND, bool PER, bool DENSE>
static int launch12(const Geo& g, const Bins& bins, const DevParams* prm, int* labels, double* dist,
                     unsigned long long* hist, long long* unres, long long cap, DevCounters* ctr,
                     unsigned long long* slots, int2* info, int* slots16, int* list, long long list_cap,
                     unsigned long long* list_count, int* ovf, int nbb, cudaStream_t st) {
  // the dynamic-smem opt-in is per device: remember it per device ordinal
  static std::atomic<unsigned long long> attr_done{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  const bool attr = (attr_done.load() & bit) != 0;
  const size_t sh_c = sizeof(v12::Smem2);
  const size_t sh_e = sizeof(v12::EvalSmemT<DENSE ? v12::kLcapD : v12::kFcap>) * v12::kEvalWarps;
  // brick lists + eval16 for every kind (JM: with the packed winner slots its
  // in-loop sqrt fits eval16's 80 registers, cfg4 -1.2 %); dense mode and
  // VX_SUBBRICK_LISTS=1 use sub-brick lists + eval12
  static const bool sub_env = std::getenv("VX_SUBBRICK_LISTS") != nullptr;
  const bool bl = !DENSE && (KIND != kJohnsonMehl || VX_JM_BRICKS) && !sub_env;
  if (!attr) {
    cudaFuncSetAttribute(v12::cull12_kernel<KIND, PER, DENSE, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sh_c);
    cudaFuncSetAttribute(v12::cull12_kernel<KIND, PER, DENSE, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sh_c);
    cudaFuncSetAttribute(v12::eval12_kernel<KIND, PER, DENSE, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh_e);
    if (KIND != kVoronoi)
      cudaFuncSetAttribute(v12::eval12_kernel<KIND, PER, DENSE, KIND != kVoronoi>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh_e);
    attr_done.fetch_or(bit);
  }
  int launches = 0;
  // super-brick rows along y in chunks of gridDim.y <= 65535
  const long long sbrows = (g.n[1] + v12::kSB - 1) / v12::kSB;
  for (long long y0 = 0; y0 < sbrows; y0 += v12::kMaxGridY, ++launches) {
    const dim3 grid((unsigned)((g.n[0] + v12::kSB - 1) / v12::kSB),
                    (unsigned)std::min<long long>(v12::kMaxGridY, sbrows - y0),
                    (unsigned)((g.z_end - g.z_begin + 16 * nbb - 1) / (16 * nbb)));
    if (bl)
      v12::cull12_kernel<KIND, PER, DENSE, true><<<grid, v12::kB2Threads, sh_c, st>>>(
          g, bins, prm, info, slots16, list, list_cap, list_count, ovf, ctr, slots, nbb, (unsigned)y0);
    else
      v12::cull12_kernel<KIND, PER, DENSE, false><<<grid, v12::kB2Threads, sh_c, st>>>(
          g, bins, prm, info, slots16, list, list_cap, list_count, ovf, ctr, slots, nbb, (unsigned)y0);
  }
  const long long nsb = ball12_subbricks(g);
  if constexpr (KIND != kJohnsonMehl || VX_JM_BRICKS) if (bl) {
    const size_t sh16 = sizeof(v12::Eval16Smem);
    if (!attr) {
      cudaFuncSetAttribute(v12::eval16_kernel<KIND, PER, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh16);
      cudaFuncSetAttribute(v12::eval16_kernel<KIND, PER, KIND != kVoronoi>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sh16);
    }
    const long long brows = (g.n[1] + 7) / 8;
    for (long long r0 = 0; r0 < brows; r0 += v12::kMaxGridY, ++launches) {
      const dim3 eg((unsigned)((g.n[0] + 7) / 8), (unsigned)std::min<long long>(v12::kMaxGridY, brows - r0),
                    (unsigned)((g.z_end - g.z_begin + 7) / 8));
      if (KIND != kVoronoi && g.fast_arith)
        v12::eval16_kernel<KIND, PER, KIND != kVoronoi><<<eg, 32, sh16, st>>>(g, bins, prm, info, slots16, list, labels, dist,
                                                                              hist, unres, cap, ctr, (unsigned)r0);
      else
        v12::eval16_kernel<KIND, PER, false><<<eg, 32, sh16, st>>>(g, bins, prm, info, slots16, list, labels, dist, hist,
                                                                   unres, cap, ctr, (unsigned)r0);
    }
    launch_subshell(g, bins, prm, ovf, &ctr->n_ovf_sb, labels, dist, hist, ctr, st);
    return launches - 2;
  }
  const long long rows = ((g.n[1] + 7) / 8 + v12::kEvalWarps - 1) / v12::kEvalWarps;  // CTA rows along y
  for (long long r0 = 0; r0 < rows; r0 += v12::kMaxGridY, ++launches) {
    const dim3 eg((unsigned)((g.n[0] + 7) / 8), (unsigned)std::min<long long>(v12::kMaxGridY, rows - r0),
                  (unsigned)((g.z_end - g.z_begin + 3) / 4));
    const unsigned sby0 = (unsigned)(r0 * v12::kEvalWarps);
    if (KIND != kVoronoi && g.fast_arith)  // call-free exact sqrt / division (vx_internal.cuh)
      v12::eval12_kernel<KIND, PER, DENSE, KIND != kVoronoi><<<eg, v12::kEvalWarps * 32, sh_e, st>>>(
          g, bins, prm, info, slots16, list, labels, dist, hist, unres, cap, ctr, slots, nsb, sby0);
    else
      v12::eval12_kernel<KIND, PER, DENSE, false><<<eg, v12::kEvalWarps * 32, sh_e, st>>>(
          g, bins, prm, info, slots16, list, labels, dist, hist, unres, cap, ctr, slots, nsb, sby0);
  }
  launch_subshell(g, bins, prm, ovf, &ctr->n_ovf_sb, labels, dist, hist, ctr, st);
  return launches - 2;  // cull / eval launches beyond the first of each
}

int launch_ball12(const Geo& g, const Bins& bins, const DevParams* prm, int* labels, double* dist,
                  unsigned long long* hist, long long* unres, long long unres_cap, DevCounters* ctr,
                  unsigned long long* slots, int2* info, int* slots16, int* list, long long list_cap,
                  unsigned long long* list_count, int* ovf, cudaStream_t st) {
  if (g.z_end <= g.z_begin) return 0;
  cudaMemsetAsync(&ctr->n_ovf_sb, 0, sizeof(unsigned long long), st);
  cudaMemsetAsync(slots, 0, 128 * sizeof(unsigned long long), st);
  cudaMemsetAsync(list_count, 0, sizeof(unsigned long long), st);
  static const int nbb_env = std::getenv("VX_NBB") ? std::atoi(std::getenv("VX_NBB")) : 0;
  const int nbb = nbb_env == 1 || nbb_env == 2 || nbb_env == 4 ? nbb_env : choose_nbb12(g);
  const bool dense = ball12_dense(g);
  int extra = 0;
#define VX_L12(K, P)                                                                                          \
  extra = (dense ? launch12<K, P, true>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, slots, info, slots16, \
                                list, list_cap, list_count, ovf, nbb, st)                                     \
         : launch12<K, P, false>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, slots, info, slots16, \
                                 list, list_cap, list_count, ovf, nbb, st))
  switch (g.kind * 2 + (g.periodic ? 1 : 0)) {
    case 0: VX_L12(kVoronoi, false); break;
    case 1: VX_L12(kVoronoi, true); break;
    case 2: VX_L12(kJohnsonMehl, false); break;
    case 3: VX_L12(kJohnsonMehl, true); break;
    case 4: VX_L12(kLaguerre, false); break;
    default: VX_L12(kLaguerre, true); break;
  }
#undef VX_L12
  ball12_publish_kernel<<<1, 32, 0, st>>>(slots, ctr);
  return 4 + extra;
}

}  // namespace vxb
