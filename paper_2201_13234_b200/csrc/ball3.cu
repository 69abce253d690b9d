// K2 (v3): the ball phase in gather form -- one cull level per warp brick with
// a multi-reference bisector test.
//
// Same contract as ball.cu / ball2.cu: labels and values are bit-identical to
// the reference because every culled site loses strictly (by far more than f64
// rounding) at every voxel of the brick, and the survivors are evaluated with
// the reference's exact f64 fold in ascending site-index order (strict <).
//
// One CTA (8 warps) owns a 16 x 16 x (2*BZW) super-brick; warp w owns the
// 8 x 8 x BZW brick (w&1, (w>>1)&1, w>>2).
//   G (CTA) : cell rows within R of the super-brick -> gathered sites in smem
//             (f32 coordinates relative to the super-brick centre, f32 time,
//             binned position, site index).  One barrier.
//   C (warp): tau = min over gathered sites of an upper bound of prox over the
//             brick; W = {lower bound <= tau}; the (up to) kRefs W sites with
//             the smallest upper bounds are references; a W site is culled if
//             some reference beats it everywhere in the brick (bisector bound).
//             Strict dominance is transitive, so culling by a reference that is
//             itself culled is still sound.
//   E (warp): survivors sorted by site index, exact per-axis f64 tables
//             (ball_scan.hpp:89-96 hoisting), exact evaluation (lane: 4 x-voxels
//             x BZW/2 z-planes of one y row), resolve (prox <= cutoff), int4
//             label stores, warp-aggregated unresolved push, per-candidate
//             histogram counts.
#include "vx_internal.cuh"

namespace vxb {
namespace v3 {

constexpr int kThreads = 256;  // 8 warps
constexpr int kTcap = 768;     // gathered sites per super-brick
constexpr int kWcap = 96;      // tau survivors per warp
constexpr int kFcap = 32;      // final candidates per warp
constexpr int kRefs = 8;
constexpr int kRows = 256;
constexpr float kRel = 1e-5f;

__device__ __forceinline__ float lo_add(float a, float b) {
  return (a + b) - kRel * (fabsf(a) + fabsf(b));
}
__device__ __forceinline__ float hi_add(float a, float b) {
  return (a + b) + kRel * (fabsf(a) + fabsf(b));
}

template <int BZW>
struct WarpS {
  int W[kWcap];           // gathered slot of each tau survivor
  float4 Wv[kWcap];       // (vx, vy, vz, t): coordinates relative to the brick centre
  float Wlb[kWcap], Wub[kWcap], Wubp[kWcap];
  unsigned char Wfl[kWcap];
  int refs[kRefs];
  int F[kFcap];           // unsorted survivors (index into W)
  int Fs[kFcap];          // sorted (gathered slot)
  int Fidx[kFcap];
  int cnt[kFcap];
  double Ft[kFcap];
  double T[kFcap][8 + 8 + BZW];  // exact w^2: x[8], y[8], z[BZW]
};

template <int BZW>
struct Smem {
  float4 rel[kTcap];
  int p[kTcap];
  int idx[kTcap];
  unsigned char flag[kTcap];
  int seg_start[2 * kRows];
  int seg_off[2 * kRows + 1];
  int warp_tot[kThreads / 32];
  int n_total;
  int any_flag;
  WarpS<BZW> w[kThreads / 32];
};

// per-axis bounds of a site (relative coords u) over a box (centre c, half h)
template <bool PER, bool FLAGS>
__device__ __forceinline__ void axis_b(float u, float c, float h, float halfL, bool fl, float& v,
                                       float& mn, float& mx) {
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
__device__ __forceinline__ void prox_b(float lb, float ub, float t, float invG, float& lbp,
                                       float& ubp) {
  if (KIND == kVoronoi) {
    lbp = lb;
    ubp = ub;
  } else {
    const float tl = t - kRel * fabsf(t), th = t + kRel * fabsf(t);
    const float dl = KIND == kJohnsonMehl ? sqrtf(lb) : lb;
    const float dh = KIND == kJohnsonMehl ? sqrtf(ub) : ub;
    lbp = lo_add(dl * invG * (1.f - kRel), tl);
    ubp = hi_add(dh * invG * (1.f + kRel), th);
  }
}

template <int KIND, bool PER, bool FLAGS>
__device__ __forceinline__ void site_box(const float4 s, unsigned fl, const float* c,
                                         const float* h, const float* halfL, float invG,
                                         float4& v, float& lb, float& ub, float& lbp, float& ubp) {
  float vv[3], mn[3], mx[3];
  const float u[3] = {s.x, s.y, s.z};
#pragma unroll
  for (int a = 0; a < 3; ++a) axis_b<PER, FLAGS>(u[a], c[a], h[a], halfL[a], (fl >> a) & 1u, vv[a], mn[a], mx[a]);
  lb = __fmaf_rn(mn[2], mn[2], __fmaf_rn(mn[1], mn[1], mn[0] * mn[0])) * (1.f - kRel);
  ub = __fmaf_rn(mx[2], mx[2], __fmaf_rn(mx[1], mx[1], mx[0] * mx[0])) * (1.f + kRel);
  v = make_float4(vv[0], vv[1], vv[2], s.w);
  prox_b<KIND>(lb, ub, s.w, invG, lbp, ubp);
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
    const bool wrapcase = PER && ((((fs | fr) >> a) & 1u) || fabsf(sv[a]) + h[a] > halfL[a] * (1.f - 1e-5f) ||
                                  fabsf(rv[a]) + h[a] > halfL[a] * (1.f - 1e-5f));
    if (wrapcase) {
      // min w_s^2 - max w_r^2 along this axis
      const float mns = fmaxf(fabsf(sv[a]) - h[a], 0.f);
      const float mxr = fminf(fabsf(rv[a]) + h[a], halfL[a]);
      const float mn2 = (fs >> a) & 1u ? 0.f : mns;
      const float mx2 = (fr >> a) & 1u ? halfL[a] : mxr;
      D += mn2 * mn2 - mx2 * mx2;
      mag += mn2 * mn2 + mx2 * mx2;
    } else {
      const float dv = fabsf(sv[a] - rv[a]);
      D += sv[a] * sv[a] - rv[a] * rv[a] - 2.f * h[a] * dv;
      mag += sv[a] * sv[a] + rv[a] * rv[a] + 2.f * h[a] * dv;
    }
    mag += 2.f * e_d * (fabsf(sv[a]) + fabsf(rv[a]) + 2.f * h[a] + e_d);
  }
  const float Dlo = D - kRel * mag;  // lower bound over the box of d_s^2 - d_r^2
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

template <int KIND, bool PER, bool FLAGS, int BZW>
__device__ __forceinline__ void ball3_warp(const Geo& g, const Bins& bins,
                                           const DevParams* __restrict__ prm, int* labels,
                                           double* dist, unsigned long long* hist,
                                           long long* unres, long long unres_cap,
                                           DevCounters* ctr, unsigned long long* eval_slots,
                                           Smem<BZW>& S, const long long* K0, const int* ext,
                                           const double* cc, float e_d, int T, bool cta_ok) {
  constexpr int NT = 16 + BZW;  // table entries per candidate
  constexpr int NZ = BZW / 2;   // z planes per lane
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WarpS<BZW>& ws = S.w[wid];
  const int bo[3] = {(wid & 1) * 8, ((wid >> 1) & 1) * 8, (wid >> 2) * BZW};
  const int be[3] = {min(8, ext[0] - bo[0]), min(8, ext[1] - bo[1]), min(BZW, ext[2] - bo[2])};
  if (be[0] <= 0 || be[1] <= 0 || be[2] <= 0) return;
  float c3[3], h3[3], halfL[3];
  {
    double cv = 0.0, hv = 0.0;
    if (lane < 3) {
      const int a = lane;
      const double l = center(K0[a] + bo[a], g.sp[a]), h = center(K0[a] + bo[a] + be[a] - 1, g.sp[a]);
      cv = 0.5 * (l + h) - cc[a];
      hv = 0.5 * (h - l);
    }
    const float cf = (float)cv, hf = (float)hv * (1.f + kRel) + 2.f * e_d;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      c3[a] = __shfl_sync(0xffffffffu, cf, a);
      h3[a] = __shfl_sync(0xffffffffu, hf, a);
      halfL[a] = (float)g.halfL[a];
    }
  }
  const float invG = KIND == kVoronoi ? 1.f : (float)(1.0 / g.growth);
  const double cutoff = prm->cutoff;

  int nF = 0;
  bool ok = cta_ok;
  if (ok) {
    float mu = __int_as_float(0x7f800000);
    for (int f = lane; f < T; f += 32) {
      float4 v;
      float lb, ub, lbp, ubp;
      site_box<KIND, PER, FLAGS>(S.rel[f], FLAGS ? S.flag[f] : 0u, c3, h3, halfL, invG, v, lb, ub,
                                 lbp, ubp);
      mu = fminf(mu, ubp);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mu = fminf(mu, __shfl_xor_sync(0xffffffffu, mu, o));
    const float tau = mu;
    int nW = 0;
    for (int f0 = 0; f0 < T; f0 += 32) {
      const int f = f0 + lane;
      bool keep = false;
      float4 v;
      float lb = 0.f, ub = 0.f, lbp = 0.f, ubp = 0.f;
      unsigned fl = 0;
      if (f < T) {
        fl = FLAGS ? S.flag[f] : 0u;
        site_box<KIND, PER, FLAGS>(S.rel[f], fl, c3, h3, halfL, invG, v, lb, ub, lbp, ubp);
        keep = lbp <= tau;
      }
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      const int pos = nW + __popc(m & ((1u << lane) - 1u));
      if (keep && pos < kWcap) {
        ws.W[pos] = f;
        ws.Wv[pos] = v;
        ws.Wlb[pos] = lb;
        ws.Wub[pos] = ub;
        ws.Wubp[pos] = ubp;
        ws.Wfl[pos] = (unsigned char)fl;
      }
      nW += __popc(m);
    }
    ok = nW <= kWcap;
    __syncwarp();
    if (ok) {
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
          keep = true;
          const float4 sv = ws.Wv[i];
          const unsigned fs = ws.Wfl[i];
          const float lbs = ws.Wlb[i], ubs = ws.Wub[i];
          for (int r = 0; r < nref && keep; ++r) {
            const int j = ws.refs[r];
            if (j != i && dominated<KIND, PER>(sv, fs, lbs, ubs, ws.Wv[j], ws.Wfl[j], ws.Wlb[j],
                                               ws.Wub[j], h3, halfL, invG, e_d))
              keep = false;
          }
        }
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        const int pos = nF + __popc(m & ((1u << lane) - 1u));
        if (keep && pos < kFcap) ws.F[pos] = i;
        nF += __popc(m);
      }
      ok = nF <= kFcap;
    }
  }
  if (!ok) nF = 0;
  __syncwarp();
  if (nF > 0) {
    for (int i = lane; i < nF; i += 32) {
      const int f = ws.W[ws.F[i]];
      const int me = S.idx[f];
      int rank = 0;
      for (int k = 0; k < nF; ++k) rank += S.idx[ws.W[ws.F[k]]] < me;
      ws.Fs[rank] = f;
      ws.Fidx[rank] = me;
      ws.cnt[rank] = 0;
    }
    __syncwarp();
    for (int e = lane; e < nF * NT; e += 32) {
      const int j = e / NT, r = e - j * NT;
      const int p = S.p[ws.Fs[j]];
      double w2;
      if (r < 8)
        w2 = axis_sq<PER>(bins.x[p], center(K0[0] + bo[0] + r, g.sp[0]), g.L[0], g.invL[0]);
      else if (r < 16)
        w2 = axis_sq<PER>(bins.y[p], center(K0[1] + bo[1] + (r - 8), g.sp[1]), g.L[1], g.invL[1]);
      else
        w2 = axis_sq<PER>(bins.z[p], center(K0[2] + bo[2] + (r - 16), g.sp[2]), g.L[2], g.invL[2]);
      ws.T[j][r] = w2;
      if (r == 0 && KIND != kVoronoi) ws.Ft[j] = bins.t[p];
    }
    __syncwarp();
  }

  // ---- exact evaluation: lane -> 4 x-voxels x NZ z-planes of one y row ----
  const int qx = (lane & 1) * 4, vy = (lane >> 1) & 7, z0 = (lane >> 4) * NZ;
  double best[NZ][4];
  int bj[NZ][4];
#pragma unroll
  for (int zz = 0; zz < NZ; ++zz)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      best[zz][k] = __longlong_as_double(0x7ff0000000000000ll);
      bj[zz][k] = -1;
    }
  const bool g1 = g.g_is_one;
  for (int j = 0; j < nF; ++j) {
    const double wy = ws.T[j][8 + vy];
    const double2 w01 = *reinterpret_cast<const double2*>(&ws.T[j][qx]);
    const double2 w23 = *reinterpret_cast<const double2*>(&ws.T[j][qx + 2]);
    const double tj = KIND == kVoronoi ? 0.0 : ws.Ft[j];
#pragma unroll
    for (int zz = 0; zz < NZ; ++zz) {
      const double a = __dadd_rn(ws.T[j][16 + z0 + zz], wy);  // 0 + wz^2 == wz^2 exactly
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

  // ---- resolve, store, compact unresolved ----
  const long long slab_base = g.z_begin * g.n[0] * g.n[1];
  long long mylins[4 * NZ];
  int nun = 0, nvalid = 0;
#pragma unroll
  for (int zz = 0; zz < NZ; ++zz) {
    const bool rowvalid = vy < be[1] && z0 + zz < be[2];
    if (!rowvalid) continue;
    const long long ky = K0[1] + bo[1] + vy, kz = K0[2] + bo[2] + z0 + zz;
    const long long lin0 = K0[0] + bo[0] + qx + g.n[0] * (ky + g.n[1] * kz);
    int lab[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      lab[k] = -1;
      if (qx + k < be[0]) {
        ++nvalid;
        if (bj[zz][k] >= 0 && best[zz][k] <= cutoff) {
          lab[k] = ws.Fidx[bj[zz][k]];
          atomicAdd(&ws.cnt[bj[zz][k]], 1);
        } else {
          mylins[nun++] = lin0 + k;
        }
      }
    }
    int* out = labels + (lin0 - slab_base);
    if (qx + 4 <= be[0] && g.vec_store) {
      *reinterpret_cast<int4*>(out) = make_int4(lab[0], lab[1], lab[2], lab[3]);
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (qx + k < be[0]) out[k] = lab[k];
    }
    if (dist) {
      double* dout = dist + (lin0 - slab_base);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (qx + k < be[0] && lab[k] >= 0)
          dout[k] = KIND == kVoronoi ? __dsqrt_rn(best[zz][k]) : best[zz][k];
    }
  }
  {
    int inc = nun;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    const int wtot = __shfl_sync(0xffffffffu, inc, 31);
    if (wtot > 0) {
      unsigned long long base = 0;
      if (lane == 31) base = atomicAdd(&ctr->n_unres, (unsigned long long)wtot);
      base = __shfl_sync(0xffffffffu, base, 31);
      const long long off = (long long)base + inc - nun;
      for (int i = 0; i < nun; ++i)
        if (off + i < unres_cap) unres[off + i] = mylins[i];
    }
  }
  __syncwarp();
  if (hist)
    for (int i = lane; i < nF; i += 32)
      if (ws.cnt[i]) atomicAdd(&hist[ws.Fidx[i]], (unsigned long long)ws.cnt[i]);
  int nv = nvalid;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nv += __shfl_xor_sync(0xffffffffu, nv, o);
  if (lane == 0) {
    if (nF)
      atomicAdd(&eval_slots[(blockIdx.x + 7 * blockIdx.y + 13 * blockIdx.z + wid) & 63],
                (unsigned long long)nF * nv);
    if (!ok) atomicAdd(&ctr->overflow_bricks, 1ull);
  }
}

template <int KIND, bool PER, int BZW>
__global__ void __launch_bounds__(kThreads, 2)
    ball3_kernel(Geo g, Bins bins, const DevParams* __restrict__ prm, int* __restrict__ labels,
                 double* __restrict__ dist, unsigned long long* __restrict__ hist,
                 long long* __restrict__ unres, long long unres_cap, DevCounters* ctr,
                 unsigned long long* __restrict__ eval_slots) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem<BZW>& S = *reinterpret_cast<Smem<BZW>*>(smem_raw);
  constexpr int SBZ = 2 * BZW;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

  const long long K0[3] = {(long long)blockIdx.x * 16, (long long)blockIdx.y * 16,
                           g.z_begin + (long long)blockIdx.z * SBZ};
  const int ext[3] = {(int)min(16ll, g.n[0] - K0[0]), (int)min(16ll, g.n[1] - K0[1]),
                      (int)min((long long)SBZ, g.z_end - K0[2])};
  double blo[3], bhi[3], cc[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    blo[a] = center(K0[a], g.sp[a]);
    bhi[a] = center(K0[a] + ext[a] - 1, g.sp[a]);
    cc[a] = 0.5 * (blo[a] + bhi[a]);
  }
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
  if (tid == 0) S.any_flag = 0;
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
    for (int f = tid; f < T; f += kThreads) {
      while (seg + 1 < nseg && S.seg_off[seg + 1] <= f) ++seg;  // f increases per thread
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
      if (fl) S.any_flag = 1;
    }
  }
  __syncthreads();
  if (PER && S.any_flag) {
    ball3_warp<KIND, PER, true, BZW>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr,
                                     eval_slots, S, K0, ext, cc, e_d, T, cta_ok);
  } else {
    ball3_warp<KIND, PER, false, BZW>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr,
                                      eval_slots, S, K0, ext, cc, e_d, T, cta_ok);
  }
}

}  // namespace v3

__global__ void ball3_publish_kernel(const unsigned long long* slots, DevCounters* ctr) {
  unsigned long long s = 0;
  for (int i = threadIdx.x; i < 64; i += 32) s += slots[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (threadIdx.x == 0) ctr->ball_evals += s;
}

template <int KIND, bool PER, int BZW>
static void launch3(const Geo& g, const Bins& bins, const DevParams* prm, int* labels,
                    double* dist, unsigned long long* hist, long long* unres, long long cap,
                    DevCounters* ctr, unsigned long long* slots, cudaStream_t st) {
  static bool attr = false;
  const size_t sh = sizeof(v3::Smem<BZW>);
  if (!attr) {
    cudaFuncSetAttribute(v3::ball3_kernel<KIND, PER, BZW>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh);
    attr = true;
  }
  const dim3 grid((unsigned)((g.n[0] + 15) / 16), (unsigned)((g.n[1] + 15) / 16),
                  (unsigned)((g.z_end - g.z_begin + 2 * BZW - 1) / (2 * BZW)));
  v3::ball3_kernel<KIND, PER, BZW><<<grid, v3::kThreads, sh, st>>>(g, bins, prm, labels, dist, hist,
                                                                  unres, cap, ctr, slots);
}

template <int BZW>
static void dispatch3(const Geo& g, const Bins& bins, const DevParams* prm, int* labels,
                      double* dist, unsigned long long* hist, long long* unres, long long cap,
                      DevCounters* ctr, unsigned long long* slots, cudaStream_t st) {
  switch (g.kind * 2 + (g.periodic ? 1 : 0)) {
    case 0: launch3<kVoronoi, false, BZW>(g, bins, prm, labels, dist, hist, unres, cap, ctr, slots, st); break;
    case 1: launch3<kVoronoi, true, BZW>(g, bins, prm, labels, dist, hist, unres, cap, ctr, slots, st); break;
    case 2: launch3<kJohnsonMehl, false, BZW>(g, bins, prm, labels, dist, hist, unres, cap, ctr, slots, st); break;
    case 3: launch3<kJohnsonMehl, true, BZW>(g, bins, prm, labels, dist, hist, unres, cap, ctr, slots, st); break;
    case 4: launch3<kLaguerre, false, BZW>(g, bins, prm, labels, dist, hist, unres, cap, ctr, slots, st); break;
    default: launch3<kLaguerre, true, BZW>(g, bins, prm, labels, dist, hist, unres, cap, ctr, slots, st); break;
  }
}

int launch_ball3(const Geo& g, const Bins& bins, const DevParams* prm, int* labels, double* dist,
                 unsigned long long* hist, long long* unres, long long unres_cap,
                 DevCounters* ctr, unsigned long long* slots, int bzw, cudaStream_t st) {
  if (g.z_end <= g.z_begin) return 0;
  cudaMemsetAsync(slots, 0, 64 * sizeof(unsigned long long), st);
  if (bzw == 8) dispatch3<8>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, slots, st);
  else dispatch3<4>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, slots, st);
  ball3_publish_kernel<<<1, 32, 0, st>>>(slots, ctr);
  return 2;
}

}  // namespace vxb
