// K2 (v7): the ball phase in gather form -- one warp per 8^3 brick, f32
// packed-key evaluation with an exact f64 fallback.
//
// Contract (as ball.cu): labels and values bit-identical to the reference.
//  * Culling only removes sites that lose strictly (by far more than f64
//    rounding) at every voxel of the brick (tau bound + bisector bounds against
//    the kRefs sites with the smallest upper bounds; strict dominance is
//    transitive).
//  * Per voxel the survivors are ranked in f32: prox_f from f32 copies of the
//    *exact* f64 per-axis residuals w (ball_scan.hpp:89-96 hoisting, computed
//    with the reference's wrap), keyed as (order-preserving f32 bits with the
//    low 6 bits replaced by the slot).  The lane keeps the best and second-best
//    keys.  If the decoded gap exceeds a rigorous bound on the f32 error (+ key
//    truncation), the f32 winner IS the exact lexicographic winner (unique, no
//    tie possible).  Otherwise (rare: near-equidistant voxels) the voxel is
//    re-ranked exactly: the reference's f64 fold over all survivors with the
//    (prox, site index) tie rule (tessellate.cpp:65,132).
//  * Resolved (prox <= cutoff, tessellate.cpp:130): decided in f32 when the
//    margin allows, else from the exact f64 value of the winner.
//  * Distances (optional): exact f64 value of the winner (geometry.hpp:106-135).
#include "vx_internal.cuh"

namespace vxb {
namespace v7 {

constexpr int kWarps = 4;
constexpr int kRowCap = 64;
constexpr int kGcap = 256;   // gathered sites per brick
constexpr int kWcap = 64;    // survivors per brick (2 slots per lane)
constexpr int kRefs = 4;
constexpr float kRel = 1e-5f;
constexpr float kAmb = 4e-5f;  // ambiguity margin (relative): >> f32 error + key truncation

__device__ __forceinline__ float lo_add(float a, float b) {
  return (a + b) - kRel * (fabsf(a) + fabsf(b));
}
__device__ __forceinline__ float hi_add(float a, float b) {
  return (a + b) + kRel * (fabsf(a) + fabsf(b));
}

struct __align__(16) WarpS {
  float4 fx[kWcap][2];     // f32 w^2 along x for the 8 voxel columns
  float4 fy[kWcap][2];
  float4 fz[kWcap][2];
  float ft[kWcap];         // f32 birth time
  double cx[8], cy[8], cz[8];
  float4 Wv[kWcap];        // f32 coords relative to the brick centre, t (culling)
  float Wlb[kWcap], Wub[kWcap], Wubp[kWcap];
  int G[kGcap];
  int Wp[kWcap];           // binned position of each survivor slot
  int Widx[kWcap];         // site index
  int cnt[kWcap];
  int rs0[kRowCap], rn0[kRowCap], rs1[kRowCap], rn1[kRowCap];
  int dec[16][32];         // per-voxel decision: winner slot or -1 (unresolved)
};

template <int KIND>
__device__ __forceinline__ float lbp_of(float lb, float t, float invG) {
  if (KIND == kVoronoi) return lb;
  const float dl = KIND == kJohnsonMehl ? sqrtf(lb) : lb;
  return lo_add(dl * invG * (1.f - kRel), t - kRel * fabsf(t));
}
template <int KIND>
__device__ __forceinline__ float ubp_of(float ub, float t, float invG) {
  if (KIND == kVoronoi) return ub;
  const float dh = KIND == kJohnsonMehl ? sqrtf(ub) : ub;
  return hi_add(dh * invG * (1.f + kRel), t + kRel * fabsf(t));
}

template <bool PER>
__device__ __forceinline__ float relc(float s, float c, float L, float invL) {
  float v = s - c;
  if (PER) v = v - L * rintf(v * invL);
  return v;
}

// true iff r beats s strictly (by >> f64 rounding) everywhere in the brick (centre 0, half h)
template <int KIND, bool PER>
__device__ __forceinline__ bool dominated(const float4 s, float lbs, float ubs, const float4 r,
                                          float lbr, float ubr, const float* h,
                                          const float* halfL, float invG, float e_d) {
  const float sv[3] = {s.x, s.y, s.z}, rv[3] = {r.x, r.y, r.z};
  float D = 0.f, mag = 0.f;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (PER && (fabsf(sv[a]) + h[a] > halfL[a] * (1.f - 1e-5f) ||
                fabsf(rv[a]) + h[a] > halfL[a] * (1.f - 1e-5f)))
      return false;  // periodic image may change inside the brick: keep
    const float dv = fabsf(sv[a] - rv[a]);
    D += (sv[a] - rv[a]) * (sv[a] + rv[a]) - 2.f * h[a] * dv;
    mag += fabsf(sv[a]) + fabsf(rv[a]) + h[a];
  }
  const float Dlo = D - mag * (mag * 2.f * kRel + 4.f * e_d);
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

__device__ __forceinline__ int wrapi(int c, int m) {
  const int r = c % m;
  return r < 0 ? r + m : r;
}

// order-preserving f32 -> u32
__device__ __forceinline__ unsigned okey(float v) {
  const unsigned b = __float_as_uint(v);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float okey_inv(unsigned k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

template <int KIND>
__device__ __forceinline__ float proxf(float d, float t, float invG) {
  if (KIND == kVoronoi) return d;
  if (KIND == kJohnsonMehl) return __fmaf_rn(sqrtf(d), invG, t);
  return __fmaf_rn(d, invG, t);
}

// The reference's exact f64 ranking of one voxel over the slots in `mset`:
// fold (wz^2 + wy^2) + wx^2 (geometry.hpp:106-123), lexicographic (prox, site).
template <int KIND, bool PER>
__device__ __noinline__ double exact_voxel(const Geo& g, const Bins& bins, const WarpS& ws,
                                           unsigned long long mset, double cx, double cy,
                                           double cz, int* bj_out) {
  double best = __longlong_as_double(0x7ff0000000000000ll);
  int bi = 0x7fffffff, bj = -1;
  while (mset) {
    const int jj = __ffsll((long long)mset) - 1;
    mset &= mset - 1;
    const int p = ws.Wp[jj];
    const double az = axis_sq<PER>(bins.z[p], cz, g.L[2], g.invL[2]);
    const double ay = axis_sq<PER>(bins.y[p], cy, g.L[1], g.invL[1]);
    const double ax = axis_sq<PER>(bins.x[p], cx, g.L[0], g.invL[0]);
    const double dsq = __dadd_rn(__dadd_rn(az, ay), ax);
    const double pr = prox_from_dsq<KIND>(dsq, g.growth, g.g_is_one,
                                          KIND == kVoronoi ? 0.0 : bins.t[p]);
    const int id = ws.Widx[jj];
    if (pr < best || (pr == best && id < bi)) {
      best = pr;
      bi = id;
      bj = jj;
    }
  }
  *bj_out = bj;
  return best;
}

template <int KIND, bool PER>
__global__ void __launch_bounds__(kWarps * 32, 4)
    ball7_kernel(Geo g, Bins bins, const DevParams* __restrict__ prm, int* __restrict__ labels,
                 double* __restrict__ dist, unsigned long long* __restrict__ hist,
                 long long* __restrict__ unres, long long unres_cap, DevCounters* ctr,
                 unsigned long long* __restrict__ eval_slots) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WarpS& ws = reinterpret_cast<WarpS*>(smem_raw)[wid];
  const long long brick = (long long)blockIdx.x * kWarps + wid;
  if (brick >= g.nbx * g.nby * g.nbz) return;
  const int bxi = (int)(brick % g.nbx);
  const long long rr = brick / g.nbx;
  const int byi = (int)(rr % g.nby), bzi = (int)(rr / g.nby);
  const long long K0[3] = {8ll * bxi, 8ll * byi, g.z_begin + 8ll * bzi};
  const int be[3] = {(int)min(8ll, g.n[0] - K0[0]), (int)min(8ll, g.n[1] - K0[1]),
                     (int)min(8ll, g.z_end - K0[2])};
  if (lane < 24) {  // exact voxel centres (geometry.hpp:58-60)
    const int a = lane >> 3, k = lane & 7;
    (a == 0 ? ws.cx : a == 1 ? ws.cy : ws.cz)[k] = center(K0[a] + k, g.sp[a]);
  }
  __syncwarp();
  const double* ctab[3] = {ws.cx, ws.cy, ws.cz};
  const double R = prm->gather_r, cutoff = prm->cutoff;
  double blo[3], bhi[3];
  float bc[3], bh[3], halfL[3], Lf[3], iLf[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    blo[a] = ctab[a][0];
    bhi[a] = ctab[a][be[a] - 1];
  }
  const float e_d =
      (float)(1e-6 * (g.lmax + R + (bhi[0] - blo[0]) + (bhi[1] - blo[1]) + (bhi[2] - blo[2])));
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    bc[a] = (float)(0.5 * (blo[a] + bhi[a]));
    bh[a] = (float)(0.5 * (bhi[a] - blo[a])) * (1.f + kRel) + 2.f * e_d;
    halfL[a] = (float)g.halfL[a];
    Lf[a] = (float)g.L[a];
    iLf[a] = (float)g.invL[a];
  }
  const float invG = KIND == kVoronoi ? 1.f : (float)(1.0 / g.growth);

  // ---- rows -> gathered list G ----
  int cl[3], ch[3];
  bool full[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    long long lo = (long long)floor((blo[a] - R) * g.inv_cw[a] - 1e-6);
    long long hi = (long long)floor((bhi[a] + R) * g.inv_cw[a] + 1e-6);
    full[a] = false;
    if (PER) {
      if (hi - lo + 1 >= g.m[a]) {
        lo = 0;
        hi = g.m[a] - 1;
        full[a] = true;
      }
    } else {
      lo = max(lo, 0ll);
      hi = min(hi, (long long)g.m[a] - 1);
    }
    cl[a] = (int)lo;
    ch[a] = (int)hi;
  }
  const int nry = ch[1] - cl[1] + 1, nrz = ch[2] - cl[2] + 1;
  const int nrows = nry * nrz;
  bool ok = nry > 0 && nrz > 0 && nrows <= kRowCap;
  int T = 0;
  if (ok) {
    const double R2 = R * R;
    int st[4] = {0, 0, 0, 0}, sn[4] = {0, 0, 0, 0};
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      const int r = lane + 32 * h2;
      if (r < nrows) {
        const int cy = cl[1] + r % nry, cz = cl[2] + r / nry;
        double dy = 0.0, dz = 0.0;
        if (!full[1]) dy = fmax(0.0, fmax(cy * g.cw[1] - bhi[1], blo[1] - (cy + 1) * g.cw[1]));
        if (!full[2]) dz = fmax(0.0, fmax(cz * g.cw[2] - bhi[2], blo[2] - (cz + 1) * g.cw[2]));
        const double dyz = dy * dy + dz * dz;
        if (dyz <= R2 * (1.0 + 1e-9)) {
          const double exr = sqrt(fmax(R2 - dyz, 0.0)) * (1.0 + 1e-9) + 1e-12 * g.lmax;
          const int cx0 = (int)floor((blo[0] - exr) * g.inv_cw[0] - 1e-6);
          const int cx1 = (int)floor((bhi[0] + exr) * g.inv_cw[0] + 1e-6);
          const int wy = PER ? wrapi(cy, g.m[1]) : cy, wz = PER ? wrapi(cz, g.m[2]) : cz;
          const int base = g.m[0] * (wy + g.m[1] * wz);
          const int mx = g.m[0];
          int a0 = 0, a1 = -1, c0 = 0, c1 = -1;
          if (PER) {
            if (cx1 - cx0 + 1 >= mx) {
              a0 = 0;
              a1 = mx - 1;
            } else {
              const int w0 = wrapi(cx0, mx), len = cx1 - cx0 + 1;
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
            a0 = max(cx0, 0);
            a1 = min(cx1, mx - 1);
          }
          if (a1 >= a0) {
            st[2 * h2] = bins.cell_start[base + a0];
            sn[2 * h2] = bins.cell_start[base + a1 + 1] - st[2 * h2];
          }
          if (c1 >= c0) {
            st[2 * h2 + 1] = bins.cell_start[base + c0];
            sn[2 * h2 + 1] = bins.cell_start[base + c1 + 1] - st[2 * h2 + 1];
          }
        }
      }
    }
    const int mine = sn[0] + sn[1] + sn[2] + sn[3];
    int inc = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    T = __shfl_sync(0xffffffffu, inc, 31);
    ok = T > 0 && T <= kGcap;
    if (ok) {
      int off = inc - mine;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        for (int i = 0; i < sn[q]; ++i) ws.G[off++] = st[q] + i;
    }
  }
  __syncwarp();

  // ---- brick-level cull: tau, then bisector against kRefs references ----
  int nW = 0;
  if (ok) {
    float mu = __int_as_float(0x7f800000);
    for (int f = lane; f < T; f += 32) {
      const float4 s = bins.f4[ws.G[f]];
      const float u[3] = {s.x, s.y, s.z};
      float ub = 0.f;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const float av = fabsf(relc<PER>(u[a], bc[a], Lf[a], iLf[a]));
        float mx = av + bh[a];
        if (PER) mx = fminf(mx, halfL[a]);
        ub = __fmaf_rn(mx, mx, ub);
      }
      mu = fminf(mu, ubp_of<KIND>(ub * (1.f + kRel), s.w, invG));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mu = fminf(mu, __shfl_xor_sync(0xffffffffu, mu, o));
    for (int f0 = 0; f0 < T; f0 += 32) {
      const int f = f0 + lane;
      bool keep = false;
      int p = 0;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      float lb = 0.f, ub = 0.f;
      if (f < T) {
        p = ws.G[f];
        const float4 s = bins.f4[p];
        const float u[3] = {s.x, s.y, s.z};
        float vv[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          vv[a] = relc<PER>(u[a], bc[a], Lf[a], iLf[a]);
          const float av = fabsf(vv[a]);
          const float mn = fmaxf(av - bh[a], 0.f);
          float mx = av + bh[a];
          if (PER) mx = fminf(mx, halfL[a]);
          lb = __fmaf_rn(mn, mn, lb);
          ub = __fmaf_rn(mx, mx, ub);
        }
        lb *= (1.f - kRel);
        ub *= (1.f + kRel);
        v = make_float4(vv[0], vv[1], vv[2], s.w);
        keep = lbp_of<KIND>(lb, s.w, invG) <= mu;
      }
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      const int pos = nW + __popc(m & ((1u << lane) - 1u));
      if (keep && pos < kWcap) {
        ws.Wp[pos] = p;
        ws.Wv[pos] = v;
        ws.Wlb[pos] = lb;
        ws.Wub[pos] = ub;
        ws.Wubp[pos] = ubp_of<KIND>(ub, v.w, invG);
      }
      nW += __popc(m);
    }
    ok = nW <= kWcap;
  }
  __syncwarp();
  unsigned long long keepmask = 0ull;
  if (ok) {
    // references: kRefs rounds of a packed (ubp, slot) warp arg-min
    int refs[kRefs];
    const bool v0 = lane < nW, v1 = lane + 32 < nW;
    const float u0 = v0 ? ws.Wubp[lane] : __int_as_float(0x7f800000);
    const float u1 = v1 ? ws.Wubp[lane + 32] : __int_as_float(0x7f800000);
    unsigned k0 = (okey(u0) & ~63u) | (unsigned)lane, k1 = (okey(u1) & ~63u) | (unsigned)(lane + 32);
    const int nref = min(kRefs, nW);
#pragma unroll
    for (int r = 0; r < kRefs; ++r) {
      unsigned km = min(k0, k1);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) km = min(km, __shfl_xor_sync(0xffffffffu, km, o));
      refs[r] = (int)(km & 63u);
      if (k0 == km) k0 = 0xffffffffu;
      if (k1 == km) k1 = 0xffffffffu;
    }
    bool keep0 = v0, keep1 = v1;
    const float4 s0 = v0 ? ws.Wv[lane] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 s1 = v1 ? ws.Wv[lane + 32] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float lb0 = v0 ? ws.Wlb[lane] : 0.f, ub0 = v0 ? ws.Wub[lane] : 0.f;
    const float lb1 = v1 ? ws.Wlb[lane + 32] : 0.f, ub1 = v1 ? ws.Wub[lane + 32] : 0.f;
#pragma unroll
    for (int r = 0; r < kRefs; ++r) {
      if (r >= nref) break;
      const int j = refs[r];
      const float4 rv = ws.Wv[j];
      const float rlb = ws.Wlb[j], rub = ws.Wub[j];
      if (keep0 && j != lane && dominated<KIND, PER>(s0, lb0, ub0, rv, rlb, rub, bh, halfL, invG, e_d))
        keep0 = false;
      if (keep1 && j != lane + 32 && dominated<KIND, PER>(s1, lb1, ub1, rv, rlb, rub, bh, halfL, invG, e_d))
        keep1 = false;
    }
    keepmask = (unsigned long long)__ballot_sync(0xffffffffu, keep0) |
               ((unsigned long long)__ballot_sync(0xffffffffu, keep1) << 32);
    // f32 copies of the exact per-axis residual squares for the kept slots
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      const int j = lane + 32 * h2;
      if ((keepmask >> j) & 1ull) {
        const int p = ws.Wp[j];
        const double sx[3] = {bins.x[p], bins.y[p], bins.z[p]};
        ws.Widx[j] = bins.idx[p];
        ws.cnt[j] = 0;
        ws.ft[j] = KIND == kVoronoi ? 0.f : ws.Wv[j].w;
        float4* dst[3] = {ws.fx[j], ws.fy[j], ws.fz[j]};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const double* c = ctab[a];
          const double uu0 = __dsub_rn(sx[a], c[0]), uu7 = __dsub_rn(sx[a], c[be[a] - 1]);
          const bool fixed = !PER || (fabs(uu0) < 0.49 * g.L[a] && fabs(uu7) < 0.49 * g.L[a]);
          float w2[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            double w;
            if (fixed) {
              w = __dsub_rn(sx[a], c[k]);  // floor(u*invL + 0.5) == 0: w == u exactly
            } else {
              w = __dsub_rn(sx[a], c[k]);
              w = wrap_delta(w, g.L[a], g.invL[a]);
            }
            const float wf = (float)w;
            w2[k] = wf * wf;
          }
          dst[a][0] = make_float4(w2[0], w2[1], w2[2], w2[3]);
          dst[a][1] = make_float4(w2[4], w2[5], w2[6], w2[7]);
        }
      }
    }
  }
  __syncwarp();

  // ---- per-voxel f32 ranking: lane -> 4 x-voxels x 4 z-planes of one y row ----
  // Keys rank prox - tmin >= 0 (tmin = min birth time of the candidates), so
  // the f32 bit pattern is order-preserving and one LOP3 builds the key.
  float tabs = 0.f, tmin = 0.f;  // max |t|, min t over the candidates (timed kinds)
  if (KIND != kVoronoi) {
    tmin = __int_as_float(0x7f800000);
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      const int j = lane + 32 * h2;
      if ((keepmask >> j) & 1ull) {
        tabs = fmaxf(tabs, fabsf(ws.ft[j]));
        tmin = fminf(tmin, ws.ft[j]);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      tabs = fmaxf(tabs, __shfl_xor_sync(0xffffffffu, tabs, o));
      tmin = fminf(tmin, __shfl_xor_sync(0xffffffffu, tmin, o));
    }
  }
  const int xh = lane & 1, vy = (lane >> 1) & 7, zh = lane >> 4;
  unsigned b1[4][4], b2[4][4];  // [z][x]
#pragma unroll
  for (int z = 0; z < 4; ++z)
#pragma unroll
    for (int x = 0; x < 4; ++x) b1[z][x] = b2[z][x] = 0xffffffffu;
  {
    unsigned long long mm = keepmask;
    while (mm) {
      const int j = __ffsll((long long)mm) - 1;
      mm &= mm - 1;
      const float4 wx = ws.fx[j][xh];
      const float wy = reinterpret_cast<const float*>(ws.fy[j])[vy];
      const float4 wz = ws.fz[j][zh];
      const float tj = ws.ft[j] - tmin;
      const float az[4] = {wz.x + wy, wz.y + wy, wz.z + wy, wz.w + wy};
      const float wxa[4] = {wx.x, wx.y, wx.z, wx.w};
#pragma unroll
      for (int z = 0; z < 4; ++z)
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          float pf = proxf<KIND>(az[z] + wxa[x], tj, invG);
          if (KIND != kVoronoi) pf = fmaxf(pf, 0.f);
          const unsigned k = (__float_as_uint(pf) & ~63u) | (unsigned)j;
          b2[z][x] = min(b2[z][x], max(b1[z][x], k));
          b1[z][x] = min(b1[z][x], k);
        }
    }
  }
  // ---- decide, store ----
  // Voronoi: integer decision.  Keys are non-negative f32 bits; a bit gap of
  // >= 512 ulps (relative >= 3e-5) between the runner-up's truncated key and
  // the winner's key ceiling exceeds the f32 error (<= 3e-7 relative) of both.
  const float cf = (float)cutoff;
  const unsigned ck_lo = __float_as_uint(fmaxf(cf * (1.f - 1e-4f), 0.f));
  const unsigned ck_hi = __float_as_uint(cf * (1.f + 1e-4f));
  const long long slab_base = g.z_begin * g.n[0] * g.n[1];
  unsigned amb = 0, valm = 0;  // voxel bits: ambiguous ranking / exact value needed
  // pass 1: decisions (winner slot, or -1 = unresolved) into ws.dec[v][lane]
#pragma unroll
  for (int z = 0; z < 4; ++z)
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const int v = 4 * z + x;
      const unsigned k1 = b1[z][x], k2 = b2[z][x];
      int dj = -1;
      if (k1 != 0xffffffffu) {
        if (KIND == kVoronoi) {
          if (k2 != 0xffffffffu && (k2 & ~63u) < (k1 | 63u) + 512u) {
            amb |= 1u << v;
          } else {
            dj = (int)(k1 & 63u);
            if ((k1 & ~63u) > ck_hi) dj = -1;             // certainly beyond the cutoff
            else if (!((k1 | 63u) < ck_lo)) valm |= 1u << v;  // borderline
          }
        } else {
          // [lo1, hi1] brackets the winner's f32 prox; every other candidate's
          // f32 prox is >= lo2 (keys rank prox - tmin)
          const float lo1 = __uint_as_float(k1 & ~63u) + tmin, hi1 = __uint_as_float(k1 | 63u) + tmin;
          const float lo2 = __uint_as_float(k2 & ~63u) + tmin;
          // f32 error of any candidate's prox <= 3e-7 (|prox| + 2 max|t|); kAmb >> that
          const float m1 = kAmb * (fabsf(hi1) + fabsf(lo1) + 2.f * tabs) + 1e-30f;
          if (k2 != 0xffffffffu && !(lo2 - hi1 > m1 + kAmb * fabsf(lo2))) {
            amb |= 1u << v;
          } else {
            dj = (int)(k1 & 63u);
            const float cm = 1e-6f * fabsf(cf) + 1e-30f;
            if (lo1 - m1 > cf + cm) dj = -1;
            else if (!(hi1 + m1 < cf - cm)) valm |= 1u << v;
          }
        }
      }
      ws.dec[v][lane] = dj;
    }
  if (dist) {  // exact values of every resolved winner
#pragma unroll
    for (int v = 0; v < 16; ++v)
      if (ws.dec[v][lane] >= 0) valm |= 1u << v;
  }
  // pass 2 (rare unless distances are requested): exact f64 re-ranking
  {
    unsigned todo = amb | valm;
#pragma unroll 1
    while (todo) {
      const int v = __ffs(todo) - 1;
      todo &= todo - 1;
      const int z = v >> 2, x = v & 3, oz = zh * 4 + z;
      const bool valid = vy < be[1] && oz < be[2] && xh * 4 + x < be[0];
      if (!valid) continue;
      const unsigned long long mset = ((amb >> v) & 1u) ? keepmask : (1ull << ws.dec[v][lane]);
      int bj = -1;
      const double best = exact_voxel<KIND, PER>(g, bins, ws, mset, ws.cx[xh * 4 + x], ws.cy[vy],
                                                 ws.cz[oz], &bj);
      const bool res = bj >= 0 && best <= cutoff;
      ws.dec[v][lane] = res ? bj : -1;
      if (dist && res) {
        const long long lin = K0[0] + xh * 4 + x + g.n[0] * ((K0[1] + vy) + g.n[1] * (K0[2] + oz));
        dist[lin - slab_base] = KIND == kVoronoi ? __dsqrt_rn(best) : best;
      }
    }
  }
  // pass 3: label stores, histogram counts, unresolved list
  int nun = 0;
  long long ulins[16];
#pragma unroll
  for (int z = 0; z < 4; ++z) {
    const int oz = zh * 4 + z;
    const bool rowvalid = vy < be[1] && oz < be[2];
    if (!rowvalid) continue;
    const long long lin0 = K0[0] + xh * 4 + g.n[0] * ((K0[1] + vy) + g.n[1] * (K0[2] + oz));
    int lab[4];
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      lab[x] = -1;
      if (xh * 4 + x >= be[0]) continue;
      const int j = ws.dec[4 * z + x][lane];
      if (j >= 0) {
        lab[x] = ws.Widx[j];
        if (hist) atomicAdd(&ws.cnt[j], 1);
      } else {
        ulins[nun++] = lin0 + x;
      }
    }
    int* out = labels + (lin0 - slab_base);
    if (xh * 4 + 4 <= be[0] && g.vec_store) {
      *reinterpret_cast<int4*>(out) = make_int4(lab[0], lab[1], lab[2], lab[3]);
    } else {
#pragma unroll
      for (int x = 0; x < 4; ++x)
        if (xh * 4 + x < be[0]) out[x] = lab[x];
    }
  }
  if (__any_sync(0xffffffffu, nun > 0)) {  // K3: compaction of unresolved voxels
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
    for (int i = 0; i < nun; ++i)
      if (off + i < unres_cap) unres[off + i] = ulins[i];
  }
  __syncwarp();
  if (hist) {
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      const int j = lane + 32 * h2;
      if (((keepmask >> j) & 1ull) && ws.cnt[j] > 0)
        atomicAdd(&hist[ws.Widx[j]], (unsigned long long)ws.cnt[j]);
    }
  }
  if (lane == 0) {
    const unsigned long long ev =
        (unsigned long long)__popcll(keepmask) * (unsigned long long)(be[0] * be[1] * be[2]);
    if (ev) atomicAdd(&eval_slots[(brick * 13) & 63], ev);
    if (!ok) atomicAdd(&ctr->overflow_bricks, 1ull);
  }
}

}  // namespace v7

__global__ void ball7_publish_kernel(const unsigned long long* slots, DevCounters* ctr) {
  unsigned long long s = 0;
  for (int i = threadIdx.x; i < 64; i += 32) s += slots[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (threadIdx.x == 0) ctr->ball_evals += s;
}

template <int KIND, bool PER>
static void launch7(const Geo& g, const Bins& bins, const DevParams* prm, int* labels,
                    double* dist, unsigned long long* hist, long long* unres, long long cap,
                    DevCounters* ctr, unsigned long long* slots, cudaStream_t st) {
  static bool attr = false;
  const size_t sh = sizeof(v7::WarpS) * v7::kWarps;
  if (!attr) {
    cudaFuncSetAttribute(v7::ball7_kernel<KIND, PER>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sh);
    attr = true;
  }
  const long long nbricks = g.nbx * g.nby * g.nbz;
  const unsigned blocks = (unsigned)((nbricks + v7::kWarps - 1) / v7::kWarps);
  v7::ball7_kernel<KIND, PER><<<blocks, v7::kWarps * 32, sh, st>>>(g, bins, prm, labels, dist, hist,
                                                                  unres, cap, ctr, slots);
}

int launch_ball7(const Geo& g, const Bins& bins, const DevParams* prm, int* labels, double* dist,
                 unsigned long long* hist, long long* unres, long long unres_cap,
                 DevCounters* ctr, unsigned long long* slots, cudaStream_t st) {
  if (g.z_end <= g.z_begin) return 0;
  cudaMemsetAsync(slots, 0, 64 * sizeof(unsigned long long), st);
  switch (g.kind * 2 + (g.periodic ? 1 : 0)) {
    case 0: launch7<kVoronoi, false>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, slots, st); break;
    case 1: launch7<kVoronoi, true>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, slots, st); break;
    case 2: launch7<kJohnsonMehl, false>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, slots, st); break;
    case 3: launch7<kJohnsonMehl, true>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, slots, st); break;
    case 4: launch7<kLaguerre, false>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, slots, st); break;
    default: launch7<kLaguerre, true>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, slots, st); break;
  }
  ball7_publish_kernel<<<1, 32, 0, st>>>(slots, ctr);
  return 2;
}

}  // namespace vxb
