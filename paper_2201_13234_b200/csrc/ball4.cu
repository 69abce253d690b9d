// K2 (v4): the ball phase in gather form, two warp-level cull levels.
//
// Same contract as ball.cu: labels and values are bit-identical to the
// reference because every culled site loses strictly (by far more than f64
// rounding) at every voxel of the box it was culled for, and the survivors are
// evaluated with the reference's exact f64 fold (ball_scan.hpp:89-96 hoisting,
// geometry.hpp:106-123 order) in ascending site-index order with a strict <
// (tessellate.cpp:65,132).
//
// One CTA (8 warps) owns a 16^3 super-brick; warp w owns the 8^3 brick
// (w&1, (w>>1)&1, w>>2), processed as two 8x8x4 sub-bricks.
//   G (CTA)   : cell rows within R of the super-brick -> gathered sites in smem
//               (f32 coordinates relative to the super-brick centre, f32 time,
//               binned position, site index) + the exact f64 voxel-centre
//               coordinates of the super-brick (geometry.hpp:58-60).  1 barrier.
//   B (warp)  : tau_b = min over gathered sites of an upper bound of prox over
//               the brick; W = {lower bound <= tau_b}.
//   S (warp)  : per sub-brick: tau cull of W, then a multi-reference bisector
//               test (the kRefs sites with the smallest upper bounds; strict
//               dominance is transitive, so a culled reference still culls).
//   E (warp)  : survivors sorted by site index, exact per-axis f64 tables, exact
//               evaluation of 8 voxels per lane (4 x 2 z), resolve (prox <=
//               cutoff), int4 label stores, unresolved push and per-candidate
//               histogram counts only when needed.
// f32 bounds are widened by kRel = 1e-5 of the magnitude of their terms plus
// an absolute coordinate slack e_d (>> f32 rounding of the relative coords).
#include "vx_internal.cuh"

namespace vxb {
namespace v4 {

constexpr int kThreads = 256;
constexpr int kTcap = 768;
constexpr int kWcap = 96;
constexpr int kFcap = 32;
constexpr int kRefs = 4;
constexpr int kRows = 256;
constexpr float kRel = 1e-5f;
constexpr int NT = 8 + 8 + 4;  // table entries per candidate (x8, y8, z4)

__device__ __forceinline__ float lo_add(float a, float b) {
  return (a + b) - kRel * (fabsf(a) + fabsf(b));
}
__device__ __forceinline__ float hi_add(float a, float b) {
  return (a + b) + kRel * (fabsf(a) + fabsf(b));
}

struct __align__(16) WarpS {
  double T[kFcap][NT];      // first: 16-byte aligned rows (NT*8 = 160 B)
  float4 Wv[kWcap];         // relative coords (sub-brick centre) + t
  double Ft[kFcap];
  int W[kWcap];             // gathered slot of each brick-level survivor
  float Wlb[kWcap], Wub[kWcap], Wubp[kWcap];
  int refs[kRefs];
  int F[kFcap];
  int Fs[kFcap];
  int Fidx[kFcap];
  int cnt[kFcap];
  unsigned char Wfl[kWcap];
};

struct __align__(16) Smem {
  WarpS w[kThreads / 32];
  float4 rel[kTcap];
  int p[kTcap];
  int idx[kTcap];
  unsigned char flag[kTcap];
  double cx[16], cy[16], cz[16];  // exact voxel centres of the super-brick
  int seg_start[2 * kRows];
  int seg_off[2 * kRows + 1];
  int warp_tot[kThreads / 32];
  int n_total;
  int any_flag;
};
static_assert(sizeof(WarpS) % 16 == 0, "WarpS must keep 16-byte alignment");

template <bool PER, bool FLAGS>
__device__ __forceinline__ void axis_b(float u, float c, float h, float halfL, unsigned fl,
                                       float& v, float& mn, float& mx) {
  v = u - c;
  const float av = fabsf(v);
  mn = fmaxf(av - h, 0.f);
  mx = av + h;
  if (PER) {
    mx = fminf(mx, halfL);
    if (FLAGS && fl) {
      mn = 0.f;
      mx = halfL;
    }
  }
}

template <int KIND>
__device__ __forceinline__ float lbp_of(float lb, float t, float invG) {
  if (KIND == kVoronoi) return lb;
  const float tl = t - kRel * fabsf(t);
  const float dl = KIND == kJohnsonMehl ? sqrtf(lb) : lb;
  return lo_add(dl * invG * (1.f - kRel), tl);
}
template <int KIND>
__device__ __forceinline__ float ubp_of(float ub, float t, float invG) {
  if (KIND == kVoronoi) return ub;
  const float th = t + kRel * fabsf(t);
  const float dh = KIND == kJohnsonMehl ? sqrtf(ub) : ub;
  return hi_add(dh * invG * (1.f + kRel), th);
}

// squared-distance bounds of site s over box (c, h); v = coords relative to c
template <bool PER, bool FLAGS>
__device__ __forceinline__ void box_bounds(const float4 s, unsigned fl, const float* c,
                                           const float* h, const float* halfL, float4& v,
                                           float& lb, float& ub) {
  float vv[3], mn[3], mx[3];
  const float u[3] = {s.x, s.y, s.z};
#pragma unroll
  for (int a = 0; a < 3; ++a) axis_b<PER, FLAGS>(u[a], c[a], h[a], halfL[a], (fl >> a) & 1u, vv[a], mn[a], mx[a]);
  lb = __fmaf_rn(mn[2], mn[2], __fmaf_rn(mn[1], mn[1], mn[0] * mn[0])) * (1.f - kRel);
  ub = __fmaf_rn(mx[2], mx[2], __fmaf_rn(mx[1], mx[1], mx[0] * mx[0])) * (1.f + kRel);
  v = make_float4(vv[0], vv[1], vv[2], s.w);
}

// true iff r beats s strictly (by >> f64 rounding) at every point of the box
template <int KIND, bool PER>
__device__ __forceinline__ bool dominated(const float4 s, unsigned fs, float lbs, float ubs,
                                          const float4 r, unsigned fr, float lbr, float ubr,
                                          const float* h, const float* halfL, float invG,
                                          float e_d) {
  float D = 0.f, mag = 0.f;
  const float sv[3] = {s.x, s.y, s.z}, rv[3] = {r.x, r.y, r.z};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const bool wrapcase =
        PER && ((((fs | fr) >> a) & 1u) || fabsf(sv[a]) + h[a] > halfL[a] * (1.f - 1e-5f) ||
                fabsf(rv[a]) + h[a] > halfL[a] * (1.f - 1e-5f));
    if (wrapcase) {
      const float mn2 = (fs >> a) & 1u ? 0.f : fmaxf(fabsf(sv[a]) - h[a], 0.f);
      const float mx2 = (fr >> a) & 1u ? halfL[a] : fminf(fabsf(rv[a]) + h[a], halfL[a]);
      D += mn2 * mn2 - mx2 * mx2;
      mag += mn2 * mn2 + mx2 * mx2;
    } else {
      const float dv = fabsf(sv[a] - rv[a]);
      D += sv[a] * sv[a] - rv[a] * rv[a] - 2.f * h[a] * dv;
      mag += sv[a] * sv[a] + rv[a] * rv[a] + 2.f * h[a] * dv;
    }
    mag += 2.f * e_d * (fabsf(sv[a]) + fabsf(rv[a]) + 2.f * h[a] + e_d);
  }
  const float Dlo = D - kRel * mag;
  if (KIND == kVoronoi) return Dlo > 0.f;
  const float dt = lo_add(s.w - kRel * fabsf(s.w), -(r.w + kRel * fabsf(r.w)));
  float q;
  if (KIND == kLaguerre) {
    q = Dlo >= 0.f ? Dlo * invG * (1.f - kRel) : Dlo * invG * (1.f + kRel);
  } else {  // |x-s| - |x-r| = N / (|x-s| + |x-r|)
    if (Dlo >= 0.f) {
      q = Dlo / ((sqrtf(ubs) + sqrtf(ubr)) * (1.f + kRel)) * (1.f - kRel);
    } else {
      const float dlo = (sqrtf(lbs) + sqrtf(lbr)) * (1.f - kRel);
      if (!(dlo > 0.f)) return false;
      q = Dlo / dlo * (1.f + kRel);
    }
    q = q >= 0.f ? q * invG * (1.f - kRel) : q * invG * (1.f + kRel);
  }
  return lo_add(q, dt) > 0.f;
}

__device__ __forceinline__ long long wrapl(long long c, long long m) {
  const long long r = c % m;
  return r < 0 ? r + m : r;
}

template <int KIND, bool PER, bool FLAGS>
__device__ __forceinline__ void brick(const Geo& g, const Bins& bins, double cutoff, int* labels,
                                      double* dist, unsigned long long* hist, long long* unres,
                                      long long unres_cap, DevCounters* ctr,
                                      unsigned long long* eval_slots, Smem& S, const long long* K0,
                                      const int* ext, const double* cc, float e_d, int T,
                                      bool cta_ok) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WarpS& ws = S.w[wid];
  const int bo[3] = {(wid & 1) * 8, ((wid >> 1) & 1) * 8, (wid >> 2) * 8};
  const int be[3] = {min(8, ext[0] - bo[0]), min(8, ext[1] - bo[1]), min(8, ext[2] - bo[2])};
  if (be[0] <= 0 || be[1] <= 0 || be[2] <= 0) return;
  float halfL[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) halfL[a] = (float)g.halfL[a];
  const float invG = KIND == kVoronoi ? 1.f : (float)(1.0 / g.growth);
  // box (centre relative to cc, half extent + slack) of voxel range [o, o+n) per axis
  auto box_of = [&](const int* o, const int* n, float* c, float* h) {
    const double* ctab[3] = {S.cx, S.cy, S.cz};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double l = ctab[a][o[a]], r = ctab[a][o[a] + n[a] - 1];
      c[a] = (float)(0.5 * (l + r) - cc[a]);
      h[a] = (float)(0.5 * (r - l)) * (1.f + kRel) + 2.f * e_d;
    }
  };

  // ---- B: brick-level tau cull ----
  int nW = 0;
  bool ok = cta_ok;
  if (ok) {
    float cb[3], hb[3];
    box_of(bo, be, cb, hb);
    float mu = __int_as_float(0x7f800000);
    for (int f = lane; f < T; f += 32) {
      const float4 s = S.rel[f];
      const unsigned fl = FLAGS ? S.flag[f] : 0u;
      float ub = 0.f;
      const float u[3] = {s.x, s.y, s.z};
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        float v, mn, mx;
        axis_b<PER, FLAGS>(u[a], cb[a], hb[a], halfL[a], (fl >> a) & 1u, v, mn, mx);
        ub = __fmaf_rn(mx, mx, ub);
      }
      mu = fminf(mu, ubp_of<KIND>(ub * (1.f + kRel), s.w, invG));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mu = fminf(mu, __shfl_xor_sync(0xffffffffu, mu, o));
    for (int f0 = 0; f0 < T; f0 += 32) {
      const int f = f0 + lane;
      bool keep = false;
      if (f < T) {
        const float4 s = S.rel[f];
        const unsigned fl = FLAGS ? S.flag[f] : 0u;
        float lb = 0.f;
        const float u[3] = {s.x, s.y, s.z};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          float v, mn, mx;
          axis_b<PER, FLAGS>(u[a], cb[a], hb[a], halfL[a], (fl >> a) & 1u, v, mn, mx);
          lb = __fmaf_rn(mn, mn, lb);
        }
        keep = lbp_of<KIND>(lb * (1.f - kRel), s.w, invG) <= mu;
      }
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      const int pos = nW + __popc(m & ((1u << lane) - 1u));
      if (keep && pos < kWcap) ws.W[pos] = f;
      nW += __popc(m);
    }
    ok = nW <= kWcap;
  }
  __syncwarp();

  const long long slab_base = g.z_begin * g.n[0] * g.n[1];
  const int qx = (lane & 1) * 4, vy = (lane >> 1) & 7, zp = (lane >> 4) * 2;
  unsigned long long evals = 0;
  const bool g1 = g.g_is_one;
  for (int half = 0; half < 2; ++half) {
    const int so[3] = {bo[0], bo[1], bo[2] + 4 * half};
    const int se[3] = {be[0], be[1], min(4, ext[2] - so[2])};
    if (se[2] <= 0) break;
    int nF = 0;
    bool sok = ok;
    if (sok) {
      float cs[3], hs[3];
      box_of(so, se, cs, hs);
      // bounds of the brick survivors over the sub-brick, cached in smem
      float mu = __int_as_float(0x7f800000);
      for (int i = lane; i < nW; i += 32) {
        const int f = ws.W[i];
        const unsigned fl = FLAGS ? S.flag[f] : 0u;
        float4 v;
        float lb, ub;
        box_bounds<PER, FLAGS>(S.rel[f], fl, cs, hs, halfL, v, lb, ub);
        const float ubp = ubp_of<KIND>(ub, v.w, invG);
        ws.Wv[i] = v;
        ws.Wlb[i] = lb;
        ws.Wub[i] = ub;
        ws.Wubp[i] = ubp;
        ws.Wfl[i] = (unsigned char)fl;
        mu = fminf(mu, ubp);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mu = fminf(mu, __shfl_xor_sync(0xffffffffu, mu, o));
      __syncwarp();
      // references: the kRefs smallest upper bounds
      const int nref = min(kRefs, nW);
      for (int i = lane; i < nW; i += 32) {
        const float u = ws.Wubp[i];
        int rank = 0;
        for (int k = 0; k < nW; ++k) {
          const float uk = ws.Wubp[k];
          rank += (uk < u) || (uk == u && k < i);
        }
        if (rank < kRefs) ws.refs[rank] = i;
      }
      __syncwarp();
      for (int i0 = 0; i0 < nW; i0 += 32) {
        const int i = i0 + lane;
        bool keep = false;
        if (i < nW) {
          const float4 sv = ws.Wv[i];
          const float lbs = ws.Wlb[i];
          keep = lbp_of<KIND>(lbs, sv.w, invG) <= mu;
          const unsigned fs = ws.Wfl[i];
          const float ubs = ws.Wub[i];
          for (int r = 0; r < nref && keep; ++r) {
            const int j = ws.refs[r];
            if (j != i && dominated<KIND, PER>(sv, fs, lbs, ubs, ws.Wv[j], ws.Wfl[j], ws.Wlb[j],
                                               ws.Wub[j], hs, halfL, invG, e_d))
              keep = false;
          }
        }
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        const int pos = nF + __popc(m & ((1u << lane) - 1u));
        if (keep && pos < kFcap) ws.F[pos] = ws.W[i];
        nF += __popc(m);
      }
      sok = nF <= kFcap;
      if (!sok) nF = 0;
      __syncwarp();
      if (nF > 0) {
        // sort by site index (one survivor per lane)
        const int me = lane < nF ? S.idx[ws.F[lane]] : 0x7fffffff;
        int rank = 0;
        for (int k = 0; k < nF; ++k) rank += __shfl_sync(0xffffffffu, me, k) < me;
        if (lane < nF) {
          ws.Fs[rank] = ws.F[lane];
          ws.Fidx[rank] = me;
          ws.cnt[rank] = 0;
        }
        __syncwarp();
        // exact per-axis tables: the reference's w^2 for each candidate and voxel centre
        for (int e = lane; e < nF * NT; e += 32) {
          const int j = e / NT, r = e - j * NT;
          const int p = S.p[ws.Fs[j]];
          double w2;
          if (r < 8)
            w2 = axis_sq<PER>(bins.x[p], S.cx[so[0] + r], g.L[0], g.invL[0]);
          else if (r < 16)
            w2 = axis_sq<PER>(bins.y[p], S.cy[so[1] + r - 8], g.L[1], g.invL[1]);
          else
            w2 = axis_sq<PER>(bins.z[p], S.cz[so[2] + r - 16], g.L[2], g.invL[2]);
          ws.T[j][r] = w2;
          if (r == 0 && KIND != kVoronoi) ws.Ft[j] = bins.t[p];
        }
        __syncwarp();
      }
    }
    // ---- E: exact evaluation, lane -> 4 x-voxels x 2 z-planes of one y row ----
    double best[2][4];
    int bj[2][4];
#pragma unroll
    for (int zz = 0; zz < 2; ++zz)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        best[zz][k] = __longlong_as_double(0x7ff0000000000000ll);
        bj[zz][k] = -1;
      }
    for (int j = 0; j < nF; ++j) {
      const double wy = ws.T[j][8 + vy];
      const double2 w01 = *reinterpret_cast<const double2*>(&ws.T[j][qx]);
      const double2 w23 = *reinterpret_cast<const double2*>(&ws.T[j][qx + 2]);
      const double2 wz = *reinterpret_cast<const double2*>(&ws.T[j][16 + zp]);
      const double tj = KIND == kVoronoi ? 0.0 : ws.Ft[j];
#pragma unroll
      for (int zz = 0; zz < 2; ++zz) {
        const double a = __dadd_rn(zz ? wz.y : wz.x, wy);  // 0 + wz^2 == wz^2 exactly
        const double d[4] = {__dadd_rn(a, w01.x), __dadd_rn(a, w01.y), __dadd_rn(a, w23.x),
                             __dadd_rn(a, w23.y)};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const double pr = prox_from_dsq<KIND>(d[k], g.growth, g1, tj);
          if (pr < best[zz][k]) {
            best[zz][k] = pr;
            bj[zz][k] = j;
          }
        }
      }
    }
    // ---- resolve + store ----
    int nun = 0;
    int lab[2][4];
#pragma unroll
    for (int zz = 0; zz < 2; ++zz) {
      const bool rowvalid = vy < se[1] && zp + zz < se[2];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        lab[zz][k] = -1;
        if (rowvalid && qx + k < se[0]) {
          if (bj[zz][k] >= 0 && best[zz][k] <= cutoff) lab[zz][k] = ws.Fidx[bj[zz][k]];
          else ++nun;
        }
      }
      if (!rowvalid) continue;
      const long long ky = K0[1] + so[1] + vy, kz = K0[2] + so[2] + zp + zz;
      const long long lin0 = K0[0] + so[0] + qx + g.n[0] * (ky + g.n[1] * kz);
      int* out = labels + (lin0 - slab_base);
      if (qx + 4 <= se[0] && g.vec_store) {
        *reinterpret_cast<int4*>(out) = make_int4(lab[zz][0], lab[zz][1], lab[zz][2], lab[zz][3]);
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (qx + k < se[0]) out[k] = lab[zz][k];
      }
      if (dist) {
        double* dout = dist + (lin0 - slab_base);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (qx + k < se[0] && lab[zz][k] >= 0)
            dout[k] = KIND == kVoronoi ? __dsqrt_rn(best[zz][k]) : best[zz][k];
      }
    }
    if (__any_sync(0xffffffffu, nun > 0)) {  // compaction of unresolved voxels
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
      long long off = (long long)base + inc - nun;
#pragma unroll
      for (int zz = 0; zz < 2; ++zz) {
        const long long ky = K0[1] + so[1] + vy, kz = K0[2] + so[2] + zp + zz;
        const long long lin0 = K0[0] + so[0] + qx + g.n[0] * (ky + g.n[1] * kz);
        const bool rowvalid = vy < se[1] && zp + zz < se[2];
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (rowvalid && qx + k < se[0] && lab[zz][k] < 0) {
            if (off < unres_cap) unres[off] = lin0 + k;
            ++off;
          }
      }
    }
    if (hist && nF > 0) {
#pragma unroll
      for (int zz = 0; zz < 2; ++zz)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (lab[zz][k] >= 0) atomicAdd(&ws.cnt[bj[zz][k]], 1);
      __syncwarp();
      if (lane < nF && ws.cnt[lane]) atomicAdd(&hist[ws.Fidx[lane]], (unsigned long long)ws.cnt[lane]);
    }
    evals += (unsigned long long)nF * (se[0] * se[1] * se[2]);
    if (lane == 0 && !sok) atomicAdd(&ctr->overflow_bricks, 1ull);
    __syncwarp();
  }
  if (lane == 0 && evals)
    atomicAdd(&eval_slots[(blockIdx.x + 7 * blockIdx.y + 13 * blockIdx.z + wid) & 63], evals);
}

template <int KIND, bool PER>
__global__ void __launch_bounds__(kThreads, 2)
    ball4_kernel(Geo g, Bins bins, const DevParams* __restrict__ prm, int* __restrict__ labels,
                 double* __restrict__ dist, unsigned long long* __restrict__ hist,
                 long long* __restrict__ unres, long long unres_cap, DevCounters* ctr,
                 unsigned long long* __restrict__ eval_slots) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const long long K0[3] = {(long long)blockIdx.x * 16, (long long)blockIdx.y * 16,
                           g.z_begin + (long long)blockIdx.z * 16};
  const int ext[3] = {(int)min(16ll, g.n[0] - K0[0]), (int)min(16ll, g.n[1] - K0[1]),
                      (int)min(16ll, g.z_end - K0[2])};
  if (tid < 48) {  // exact voxel centres (geometry.hpp:58-60)
    const int a = tid >> 4, k = tid & 15;
    const double c = center(K0[a] + k, g.sp[a]);
    (a == 0 ? S.cx : a == 1 ? S.cy : S.cz)[k] = c;
  }
  if (tid == 0) S.any_flag = 0;
  __syncthreads();
  double blo[3], bhi[3], cc[3];
  blo[0] = S.cx[0];
  blo[1] = S.cy[0];
  blo[2] = S.cz[0];
  bhi[0] = S.cx[ext[0] - 1];
  bhi[1] = S.cy[ext[1] - 1];
  bhi[2] = S.cz[ext[2] - 1];
#pragma unroll
  for (int a = 0; a < 3; ++a) cc[a] = 0.5 * (blo[a] + bhi[a]);
  const double R = prm->gather_r;
  const float e_d = (float)(1e-6 * (R + (bhi[0] - blo[0]) + (bhi[1] - blo[1]) + (bhi[2] - blo[2]) +
                                    g.cw[0] + g.cw[1] + g.cw[2]));

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
  const bool rows_ok = nry > 0 && nrz > 0 && nrows <= kRows;
  if (rows_ok && tid < nrows) {
    const int r = tid;
    const long long cy = cl[1] + r % nry, cz = cl[2] + r / nry;
    double dy = 0.0, dz = 0.0;
    if (!full[1]) dy = fmax(0.0, fmax(cy * g.cw[1] - bhi[1], blo[1] - (cy + 1) * g.cw[1]));
    if (!full[2]) dz = fmax(0.0, fmax(cz * g.cw[2] - bhi[2], blo[2] - (cz + 1) * g.cw[2]));
    const double dyz = dy * dy + dz * dz, R2 = R * R;
    int st0 = 0, n0 = 0, st1 = 0, n1 = 0;
    if (dyz <= R2 * (1.0 + 1e-9)) {
      const double exr = sqrt(fmax(R2 - dyz, 0.0)) * (1.0 + 1e-9) + 1e-12 * g.lmax;
      const long long cx0 = (long long)floor((blo[0] - exr) * g.inv_cw[0] - 1e-6);
      const long long cx1 = (long long)floor((bhi[0] + exr) * g.inv_cw[0] + 1e-6);
      const long long wy = PER ? wrapl(cy, g.m[1]) : cy, wz = PER ? wrapl(cz, g.m[2]) : cz;
      const long long base = (long long)g.m[0] * (wy + (long long)g.m[1] * wz);
      const int mx = g.m[0];
      long long a0 = 0, a1 = -1, c0 = 0, c1 = -1;
      if (PER) {
        if (cx1 - cx0 + 1 >= mx) {
          a0 = 0;
          a1 = mx - 1;
        } else {
          const long long w0 = wrapl(cx0, mx), len = cx1 - cx0 + 1;
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
  __syncthreads();
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
    for (int w = 0; w < kThreads / 32; ++w) {
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
  __syncthreads();
  const int T = S.n_total;
  const bool cta_ok = rows_ok && T > 0 && T <= kTcap;
  if (cta_ok) {
    const double hs[3] = {0.5 * (bhi[0] - blo[0]), 0.5 * (bhi[1] - blo[1]), 0.5 * (bhi[2] - blo[2])};
    int seg = 0;
    unsigned anyf = 0;
    for (int f = tid; f < T; f += kThreads) {
      while (seg + 1 < nseg && S.seg_off[seg + 1] <= f) ++seg;
      const int p = S.seg_start[seg] + (f - S.seg_off[seg]);
      const double sv[3] = {bins.x[p], bins.y[p], bins.z[p]};
      float uf[3];
      unsigned fl = 0;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        double u = sv[a] - cc[a];
        if (PER) {
          u = u - floor(u * g.invL[a] + 0.5) * g.L[a];
          if (fabs(u) + hs[a] >= g.halfL[a] * (1.0 - 1e-7) - 4.0 * e_d) fl |= 1u << a;
        }
        uf[a] = (float)u;
      }
      S.rel[f] = make_float4(uf[0], uf[1], uf[2], KIND == kVoronoi ? 0.f : (float)bins.t[p]);
      S.p[f] = p;
      S.idx[f] = bins.idx[p];
      S.flag[f] = (unsigned char)fl;
      anyf |= fl;
    }
    if (anyf) S.any_flag = 1;
  }
  __syncthreads();
  const double cutoff = prm->cutoff;
  if (PER && S.any_flag)
    brick<KIND, PER, true>(g, bins, cutoff, labels, dist, hist, unres, unres_cap, ctr, eval_slots,
                           S, K0, ext, cc, e_d, T, cta_ok);
  else
    brick<KIND, PER, false>(g, bins, cutoff, labels, dist, hist, unres, unres_cap, ctr, eval_slots,
                            S, K0, ext, cc, e_d, T, cta_ok);
}

}  // namespace v4

__global__ void ball4_publish_kernel(const unsigned long long* slots, DevCounters* ctr) {
  unsigned long long s = 0;
  for (int i = threadIdx.x; i < 64; i += 32) s += slots[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (threadIdx.x == 0) ctr->ball_evals += s;
}

template <int KIND, bool PER>
static void launch4(const Geo& g, const Bins& bins, const DevParams* prm, int* labels,
                    double* dist, unsigned long long* hist, long long* unres, long long cap,
                    DevCounters* ctr, unsigned long long* slots, cudaStream_t st) {
  static bool attr = false;
  const size_t sh = sizeof(v4::Smem);
  if (!attr) {
    cudaFuncSetAttribute(v4::ball4_kernel<KIND, PER>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sh);
    attr = true;
  }
  const dim3 grid((unsigned)((g.n[0] + 15) / 16), (unsigned)((g.n[1] + 15) / 16),
                  (unsigned)((g.z_end - g.z_begin + 15) / 16));
  v4::ball4_kernel<KIND, PER><<<grid, v4::kThreads, sh, st>>>(g, bins, prm, labels, dist, hist,
                                                             unres, cap, ctr, slots);
}

int launch_ball4(const Geo& g, const Bins& bins, const DevParams* prm, int* labels, double* dist,
                 unsigned long long* hist, long long* unres, long long unres_cap,
                 DevCounters* ctr, unsigned long long* slots, cudaStream_t st) {
  if (g.z_end <= g.z_begin) return 0;
  cudaMemsetAsync(slots, 0, 64 * sizeof(unsigned long long), st);
  switch (g.kind * 2 + (g.periodic ? 1 : 0)) {
    case 0: launch4<kVoronoi, false>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, slots, st); break;
    case 1: launch4<kVoronoi, true>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, slots, st); break;
    case 2: launch4<kJohnsonMehl, false>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, slots, st); break;
    case 3: launch4<kJohnsonMehl, true>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, slots, st); break;
    case 4: launch4<kLaguerre, false>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, slots, st); break;
    default: launch4<kLaguerre, true>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, slots, st); break;
  }
  ball4_publish_kernel<<<1, 32, 0, st>>>(slots, ctr);
  return 2;
}

}  // namespace vxb
