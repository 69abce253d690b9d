// K2 (v6): the ball phase in gather form -- one independent warp per 8^3 brick,
// lane-regular culling into per-sub-box candidate bitmasks.
//
// Same contract as ball.cu: labels and values are bit-identical to the
// reference because every culled site loses strictly (by far more than f64
// rounding) at every voxel of the box it was culled for, and the survivors
// are evaluated with the reference's exact f64 fold (ball_scan.hpp:89-96
// hoisting, geometry.hpp:106-123 order) in ascending site index with a strict
// < (tessellate.cpp:65,132).  No block-level barrier.
//
// Per warp (brick 8^3 = eight 4^3 sub-boxes b = (x-half, y-half, z-half)):
//   1 rows   : cell rows within R of the brick -> the brick's gathered list G
//              (binned positions, warp scan of per-lane counts).
//   2 tau_b  : W = {s in G : lb_brick(s) <= min ub_brick} (f32, widened).
//   3 sort   : W sorted by site index (<= 64 entries, 2 slots per lane).
//   4 masks  : lane = site slot; for each sub-box b: tau_b via a packed
//              (ub, slot) warp min -> reference r_b; site kept for b iff
//              lb_b(s) <= tau_b and r_b does not beat it everywhere in b.
//              -> 64-bit candidate mask per sub-box, in index order.
//   5 tables : exact f64 w^2 of every W site for the brick's 8+8+8 voxel
//              centres (fast path u*u when the periodic image is fixed).
//   6 eval   : lane = 4x2x2 voxels of one sub-box; loop over the sub-box mask,
//              strict < in index order; resolve (prox <= cutoff); int4 stores;
//              unresolved push; histogram counts.
#include "vx_internal.cuh"

namespace vxb {
namespace v6 {

constexpr int kWarps = 4;
constexpr int kRowCap = 64;
constexpr int kGcap = 256;   // gathered sites per brick
constexpr int kWcap = 64;    // tau survivors per brick (2 slots per lane)
constexpr float kRel = 1e-5f;

__device__ __forceinline__ float lo_add(float a, float b) {
  return (a + b) - kRel * (fabsf(a) + fabsf(b));
}
__device__ __forceinline__ float hi_add(float a, float b) {
  return (a + b) + kRel * (fabsf(a) + fabsf(b));
}

constexpr int kTcap = 32;    // W slots that are a candidate of some sub-box

struct __align__(16) WarpS {
  double T[kTcap][24];        // exact w^2: x[8] | y[8] | z[8], rows by rank in the any-mask
  double Tt[kTcap];           // birth times (f64)
  double cx[8], cy[8], cz[8]; // exact voxel centres of the brick
  float4 Wv[kWcap];           // f32 coords relative to the brick centre, t
  int G[kGcap];               // gathered binned positions
  int Wp[kWcap];              // sorted W: binned position
  int Widx[kWcap];            // sorted W: site index
  int cnt[kWcap];             // histogram counts per W slot
  int rs0[kRowCap], rn0[kRowCap], rs1[kRowCap], rn1[kRowCap];
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

// nearest-image offset of a (brick-relative) coordinate from a sub-box centre
template <bool PER>
__device__ __forceinline__ float rewrap(float v, float o, float L, float invL) {
  float w = v - o;
  if (PER) w = w - L * rintf(w * invL);
  return w;
}

// per-axis distance bounds of offset v to the interval [o - h, o + h]
template <bool PER>
__device__ __forceinline__ void ax(float v, float o, float h, float halfL, float L, float invL,
                                   float& mn, float& mx) {
  const float av = fabsf(rewrap<PER>(v, o, L, invL));
  mn = fmaxf(av - h, 0.f);
  mx = av + h;
  if (PER) mx = fminf(mx, halfL);
}

// does r beat s strictly (by >> f64 rounding) everywhere in the box (o, h)?
template <int KIND, bool PER>
__device__ __forceinline__ bool dominated(const float* s, float ts, float lbs, float ubs,
                                          const float* r, float tr, float lbr, float ubr,
                                          const float* o, const float* h, const float* halfL,
                                          const float* L, const float* invL, float invG,
                                          float e_d) {
  float D = 0.f, mag = 0.f;
  bool wrap = false;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float sv = rewrap<PER>(s[a], o[a], L[a], invL[a]);
    const float rv = rewrap<PER>(r[a], o[a], L[a], invL[a]);
    if (PER) wrap |= fabsf(sv) + h[a] > halfL[a] * (1.f - 1e-5f) ||
                     fabsf(rv) + h[a] > halfL[a] * (1.f - 1e-5f);
    const float dv = fabsf(sv - rv);
    D += (sv - rv) * (sv + rv) - 2.f * h[a] * dv;
    mag += fabsf(sv) + fabsf(rv) + h[a];
  }
  if (PER && wrap) return false;  // image may change inside the box: keep (rare)
  const float Dlo = D - mag * (mag * 2.f * kRel + 4.f * e_d);
  if (KIND == kVoronoi) return Dlo > 0.f;
  const float dt = lo_add(ts - kRel * fabsf(ts), -(tr + kRel * fabsf(tr)));
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

__device__ __forceinline__ unsigned long long ballot64(bool a0, bool a1) {
  return (unsigned long long)__ballot_sync(0xffffffffu, a0) |
         ((unsigned long long)__ballot_sync(0xffffffffu, a1) << 32);
}

template <int KIND, bool PER>
__global__ void __launch_bounds__(kWarps * 32, 4)
    ball6_kernel(Geo g, Bins bins, const DevParams* __restrict__ prm, int* __restrict__ labels,
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
  double blo[3], bhi[3], bcc[3];
  float bc[3], bh[3], halfL[3], Lf[3], iLf[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    blo[a] = ctab[a][0];
    bhi[a] = ctab[a][be[a] - 1];
    bcc[a] = 0.5 * (blo[a] + bhi[a]);
  }
  const float e_d =
      (float)(1e-6 * (g.lmax + R + (bhi[0] - blo[0]) + (bhi[1] - blo[1]) + (bhi[2] - blo[2])));
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    bc[a] = (float)bcc[a];
    bh[a] = (float)(0.5 * (bhi[a] - blo[a])) * (1.f + kRel) + 2.f * e_d;
    halfL[a] = (float)g.halfL[a];
    Lf[a] = (float)g.L[a];
    iLf[a] = (float)g.invL[a];
  }
  const float invG = KIND == kVoronoi ? 1.f : (float)(1.0 / g.growth);

  // ---- 1. rows -> gathered list G ----
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
          const long long cx0 = (long long)floor((blo[0] - exr) * g.inv_cw[0] - 1e-6);
          const long long cx1 = (long long)floor((bhi[0] + exr) * g.inv_cw[0] + 1e-6);
          const int wy = PER ? wrapi(cy, g.m[1]) : cy, wz = PER ? wrapi(cz, g.m[2]) : cz;
          const long long base = (long long)g.m[0] * (wy + (long long)g.m[1] * wz);
          const int mx = g.m[0];
          long long a0 = 0, a1 = -1, c0 = 0, c1 = -1;
          if (PER) {
            if (cx1 - cx0 + 1 >= mx) {
              a0 = 0;
              a1 = mx - 1;
            } else {
              const long long w0 = ((cx0 % mx) + mx) % mx, len = cx1 - cx0 + 1;
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

  // ---- 2. brick-level tau cull -> W ----
  int nW = 0;
  if (ok) {
    float mu = __int_as_float(0x7f800000);
    for (int f = lane; f < T; f += 32) {
      const float4 s = bins.f4[ws.G[f]];
      const float u[3] = {s.x, s.y, s.z};
      float ub = 0.f;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        float mn, mx;
        ax<PER>(relc<PER>(u[a], bc[a], Lf[a], iLf[a]), 0.f, bh[a], halfL[a], Lf[a], iLf[a], mn, mx);
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
      if (f < T) {
        p = ws.G[f];
        const float4 s = bins.f4[p];
        const float u[3] = {s.x, s.y, s.z};
        float lb = 0.f;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          float mn, mx;
          ax<PER>(relc<PER>(u[a], bc[a], Lf[a], iLf[a]), 0.f, bh[a], halfL[a], Lf[a], iLf[a], mn, mx);
          lb = __fmaf_rn(mn, mn, lb);
        }
        keep = lbp_of<KIND>(lb * (1.f - kRel), s.w, invG) <= mu;
      }
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      const int pos = nW + __popc(m & ((1u << lane) - 1u));
      if (keep && pos < kWcap) ws.Wp[pos] = p;  // unsorted for now
      nW += __popc(m);
    }
    ok = nW <= kWcap;
  }
  __syncwarp();

  // ---- 3. sort W by site index (slots: lane, lane + 32) ----
  unsigned long long mask[8];
#pragma unroll
  for (int b = 0; b < 8; ++b) mask[b] = 0ull;
  float sv0[3], sv1[3], st0 = 0.f, st1 = 0.f;
  if (ok) {
    const int p0 = lane < nW ? ws.Wp[lane] : 0, p1 = lane + 32 < nW ? ws.Wp[lane + 32] : 0;
    const int i0 = lane < nW ? bins.idx[p0] : 0x7fffffff;
    const int i1 = lane + 32 < nW ? bins.idx[p1] : 0x7fffffff;
    int r0 = 0, r1 = 0;
    for (int k = 0; k < 32 && k < nW; ++k) {
      const int a = __shfl_sync(0xffffffffu, i0, k);
      r0 += a < i0;
      r1 += a < i1;
    }
    for (int k = 0; k < 32 && k + 32 < nW; ++k) {
      const int a = __shfl_sync(0xffffffffu, i1, k);
      r0 += a < i0;
      r1 += a < i1;
    }
    __syncwarp();
    if (lane < nW) {
      ws.Wp[r0] = p0;  // all reads of Wp happened before the shuffles
      ws.Widx[r0] = i0;
    }
    if (lane + 32 < nW) {
      ws.Wp[r1] = p1;
      ws.Widx[r1] = i1;
    }
    __syncwarp();
    // ---- 4. per sub-box candidate masks (lane = slot) ----
    const bool v0 = lane < nW, v1 = lane + 32 < nW;
    float4 s0 = make_float4(0.f, 0.f, 0.f, 0.f), s1 = s0;
    if (v0) s0 = bins.f4[ws.Wp[lane]];
    if (v1) s1 = bins.f4[ws.Wp[lane + 32]];
    {
      const float u0[3] = {s0.x, s0.y, s0.z}, u1[3] = {s1.x, s1.y, s1.z};
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        sv0[a] = relc<PER>(u0[a], bc[a], Lf[a], iLf[a]);
        sv1[a] = relc<PER>(u1[a], bc[a], Lf[a], iLf[a]);
      }
      st0 = s0.w;
      st1 = s1.w;
    }
    if (v0) ws.Wv[lane] = make_float4(sv0[0], sv0[1], sv0[2], st0);
    if (v1) ws.Wv[lane + 32] = make_float4(sv1[0], sv1[1], sv1[2], st1);
    // sub-box geometry: offset o (relative to the brick centre) and half extent
    float so[8][3], sh[3];
    {
      // sub-box halves: [0, m) and [m, be) with m = min(4, be)
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const int m = min(4, be[a]);
        const double l0 = ctab[a][0], h0 = ctab[a][m - 1];
        const double l1 = ctab[a][m < be[a] ? m : m - 1], h1 = ctab[a][be[a] - 1];
        const float o0 = (float)(0.5 * (l0 + h0) - bcc[a]), o1 = (float)(0.5 * (l1 + h1) - bcc[a]);
        sh[a] = (float)fmax(0.5 * (h0 - l0), 0.5 * (h1 - l1)) * (1.f + kRel) + 2.f * e_d;
#pragma unroll
        for (int b = 0; b < 8; ++b) so[b][a] = ((b >> a) & 1) ? o1 : o0;
      }
    }
    __syncwarp();
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      float lb0 = 0.f, ub0 = 0.f, lb1 = 0.f, ub1 = 0.f;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        float mn, mx;
        ax<PER>(sv0[a], so[b][a], sh[a], halfL[a], Lf[a], iLf[a], mn, mx);
        lb0 = __fmaf_rn(mn, mn, lb0);
        ub0 = __fmaf_rn(mx, mx, ub0);
        ax<PER>(sv1[a], so[b][a], sh[a], halfL[a], Lf[a], iLf[a], mn, mx);
        lb1 = __fmaf_rn(mn, mn, lb1);
        ub1 = __fmaf_rn(mx, mx, ub1);
      }
      lb0 *= (1.f - kRel);
      lb1 *= (1.f - kRel);
      ub0 *= (1.f + kRel);
      ub1 *= (1.f + kRel);
      const float ubp0 = v0 ? ubp_of<KIND>(ub0, st0, invG) : __int_as_float(0x7f800000);
      const float ubp1 = v1 ? ubp_of<KIND>(ub1, st1, invG) : __int_as_float(0x7f800000);
      // packed (ub, slot) arg-min; tau rounded up past the truncated key bits
      auto key = [](float u, int slot) -> unsigned {
        unsigned k = __float_as_uint(u);
        return u >= 0.f ? ((k & ~63u) | (unsigned)slot) | 0x80000000u
                        : ((~k) & ~63u) | (unsigned)slot;
      };
      unsigned kmin = min(key(ubp0, lane), key(ubp1, lane + 32));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
      const int ref = (int)(kmin & 63u);
      // tau = the reference's own (exact f32) upper bound
      const float tauv = __shfl_sync(0xffffffffu, ref < 32 ? ubp0 : ubp1, ref & 31);
      const float4 rv = ws.Wv[ref];
      const float rvv[3] = {rv.x, rv.y, rv.z};
      float rlb = 0.f, rub = 0.f;
      if (KIND == kJohnsonMehl) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          float mn, mx;
          ax<PER>(rvv[a], so[b][a], sh[a], halfL[a], Lf[a], iLf[a], mn, mx);
          rlb = __fmaf_rn(mn, mn, rlb);
          rub = __fmaf_rn(mx, mx, rub);
        }
        rlb *= (1.f - kRel);
        rub *= (1.f + kRel);
      }
      bool k0 = v0 && lbp_of<KIND>(lb0, st0, invG) <= tauv;
      bool k1 = v1 && lbp_of<KIND>(lb1, st1, invG) <= tauv;
      if (k0 && lane != ref)
        k0 = !dominated<KIND, PER>(sv0, st0, lb0, ub0, rvv, rv.w, rlb, rub, so[b], sh, halfL, Lf, iLf, invG, e_d);
      if (k1 && lane + 32 != ref)
        k1 = !dominated<KIND, PER>(sv1, st1, lb1, ub1, rvv, rv.w, rlb, rub, so[b], sh, halfL, Lf, iLf, invG, e_d);
      mask[b] = ballot64(k0, k1);
    }
    // ---- 5. exact tables for every slot that is a candidate somewhere ----
    unsigned long long any = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b) any |= mask[b];
    if (__popcll(any) > kTcap) {  // too many candidates for the table space: fallback
      ok = false;
#pragma unroll
      for (int b = 0; b < 8; ++b) mask[b] = 0ull;
      any = 0ull;
    }
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      const int j0 = lane + 32 * h2;
      if (j0 < nW && ((any >> j0) & 1ull)) {
        const int j = __popcll(any & ((1ull << j0) - 1ull));  // table row
        const int p = ws.Wp[j0];
        const double sx[3] = {bins.x[p], bins.y[p], bins.z[p]};
        if (KIND != kVoronoi) ws.Tt[j] = bins.t[p];
        ws.cnt[j0] = 0;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const double* c = ctab[a];
          const double u0 = __dsub_rn(sx[a], c[0]), u7 = __dsub_rn(sx[a], c[be[a] - 1]);
          const bool fixed = !PER || (fabs(u0) < 0.49 * g.L[a] && fabs(u7) < 0.49 * g.L[a]);
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            double w2;
            if (fixed) {  // floor(u*invL + 0.5) == 0 exactly, so w == u
              const double u = __dsub_rn(sx[a], c[k]);
              w2 = __dmul_rn(u, u);
            } else {
              w2 = axis_sq<PER>(sx[a], c[k], g.L[a], g.invL[a]);
            }
            ws.T[j][8 * a + k] = w2;
          }
        }
      }
    }
  }
  __syncwarp();

  // ---- 6. exact evaluation: lane -> sub-box b = lane >> 2, 4 x 2 x 2 voxels ----
  const int b = lane >> 2, q = lane & 3;
  const int ox = (b & 1) * 4, oy = ((b >> 1) & 1) * 4 + (q & 1) * 2, oz = ((b >> 2) & 1) * 4 + (q >> 1) * 2;
  unsigned long long mb = 0ull;
#pragma unroll
  for (int bb = 0; bb < 8; ++bb)
    if (bb == b) mb = mask[bb];
  double best[2][2][4];
  int bj[2][2][4];
#pragma unroll
  for (int zz = 0; zz < 2; ++zz)
#pragma unroll
    for (int yy = 0; yy < 2; ++yy)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        best[zz][yy][k] = __longlong_as_double(0x7ff0000000000000ll);
        bj[zz][yy][k] = -1;
      }
  const bool g1 = g.g_is_one;
  unsigned long long anyw = 0;
#pragma unroll
  for (int bb = 0; bb < 8; ++bb) anyw |= mask[bb];
  unsigned long long mm = mb;
  while (mm) {
    const int j = __ffsll((long long)mm) - 1;  // W slot (ascending site index)
    mm &= mm - 1;
    const int tr = __popcll(anyw & ((1ull << j) - 1ull));
    const double* Tj = ws.T[tr];
    const double2 x01 = *reinterpret_cast<const double2*>(Tj + ox);
    const double2 x23 = *reinterpret_cast<const double2*>(Tj + ox + 2);
    const double2 yv = *reinterpret_cast<const double2*>(Tj + 8 + oy);
    const double2 zv = *reinterpret_cast<const double2*>(Tj + 16 + oz);
    const double tj = KIND == kVoronoi ? 0.0 : ws.Tt[tr];
#pragma unroll
    for (int zz = 0; zz < 2; ++zz)
#pragma unroll
      for (int yy = 0; yy < 2; ++yy) {
        const double a = __dadd_rn(zz ? zv.y : zv.x, yy ? yv.y : yv.x);  // 0 + wz^2 == wz^2
        const double d[4] = {__dadd_rn(a, x01.x), __dadd_rn(a, x01.y), __dadd_rn(a, x23.x),
                             __dadd_rn(a, x23.y)};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const double pr = prox_from_dsq<KIND>(d[k], g.growth, g1, tj);
          if (pr < best[zz][yy][k]) {
            best[zz][yy][k] = pr;
            bj[zz][yy][k] = j;
          }
        }
      }
  }
  // ---- resolve + store ----
  const long long slab_base = g.z_begin * g.n[0] * g.n[1];
  int nun = 0;
#pragma unroll
  for (int zz = 0; zz < 2; ++zz)
#pragma unroll
    for (int yy = 0; yy < 2; ++yy) {
      const bool rowvalid = oy + yy < be[1] && oz + zz < be[2];
      if (!rowvalid) continue;
      const long long lin0 =
          K0[0] + ox + g.n[0] * ((K0[1] + oy + yy) + g.n[1] * (K0[2] + oz + zz));
      int lab[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        lab[k] = -1;
        if (ox + k < be[0]) {
          if (bj[zz][yy][k] >= 0 && best[zz][yy][k] <= cutoff) {
            lab[k] = ws.Widx[bj[zz][yy][k]];
            if (hist) atomicAdd(&ws.cnt[bj[zz][yy][k]], 1);
          } else {
            ++nun;
          }
        }
      }
      int* out = labels + (lin0 - slab_base);
      if (ox + 4 <= be[0] && g.vec_store) {
        *reinterpret_cast<int4*>(out) = make_int4(lab[0], lab[1], lab[2], lab[3]);
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (ox + k < be[0]) out[k] = lab[k];
      }
      if (dist) {
        double* dout = dist + (lin0 - slab_base);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (ox + k < be[0] && lab[k] >= 0)
            dout[k] = KIND == kVoronoi ? __dsqrt_rn(best[zz][yy][k]) : best[zz][yy][k];
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
    long long off = (long long)base + inc - nun;
#pragma unroll
    for (int zz = 0; zz < 2; ++zz)
#pragma unroll
      for (int yy = 0; yy < 2; ++yy) {
        const bool rowvalid = oy + yy < be[1] && oz + zz < be[2];
        const long long lin0 =
            K0[0] + ox + g.n[0] * ((K0[1] + oy + yy) + g.n[1] * (K0[2] + oz + zz));
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (rowvalid && ox + k < be[0] && !(bj[zz][yy][k] >= 0 && best[zz][yy][k] <= cutoff)) {
            if (off < unres_cap) unres[off] = lin0 + k;
            ++off;
          }
      }
  }
  __syncwarp();
  if (hist && ok) {
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      const int j = lane + 32 * h2;
      if (j < nW && ws.cnt[j] > 0 && (((mask[0] | mask[1] | mask[2] | mask[3] | mask[4] | mask[5] |
                                        mask[6] | mask[7]) >> j) & 1ull))
        atomicAdd(&hist[ws.Widx[j]], (unsigned long long)ws.cnt[j]);
    }
  }
  // evaluation count: candidates x valid voxels per sub-box
  if (lane == 0) {
    unsigned long long ev = 0;
#pragma unroll
    for (int bb = 0; bb < 8; ++bb) {
      const int nx = min(4, be[0] - (bb & 1) * 4), ny = min(4, be[1] - ((bb >> 1) & 1) * 4),
                nz = min(4, be[2] - ((bb >> 2) & 1) * 4);
      if (nx > 0 && ny > 0 && nz > 0) ev += (unsigned long long)__popcll(mask[bb]) * (nx * ny * nz);
    }
    if (ev) atomicAdd(&eval_slots[(brick * 13) & 63], ev);
    if (!ok) atomicAdd(&ctr->overflow_bricks, 1ull);
  }
}

}  // namespace v6

__global__ void ball6_publish_kernel(const unsigned long long* slots, DevCounters* ctr) {
  unsigned long long s = 0;
  for (int i = threadIdx.x; i < 64; i += 32) s += slots[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (threadIdx.x == 0) ctr->ball_evals += s;
}

template <int KIND, bool PER>
static void launch6(const Geo& g, const Bins& bins, const DevParams* prm, int* labels,
                    double* dist, unsigned long long* hist, long long* unres, long long cap,
                    DevCounters* ctr, unsigned long long* slots, cudaStream_t st) {
  static bool attr = false;
  const size_t sh = sizeof(v6::WarpS) * v6::kWarps;
  if (!attr) {
    cudaFuncSetAttribute(v6::ball6_kernel<KIND, PER>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sh);
    attr = true;
  }
  const long long nbricks = g.nbx * g.nby * g.nbz;
  const unsigned blocks = (unsigned)((nbricks + v6::kWarps - 1) / v6::kWarps);
  v6::ball6_kernel<KIND, PER><<<blocks, v6::kWarps * 32, sh, st>>>(g, bins, prm, labels, dist, hist,
                                                                  unres, cap, ctr, slots);
}

int launch_ball6(const Geo& g, const Bins& bins, const DevParams* prm, int* labels, double* dist,
                 unsigned long long* hist, long long* unres, long long unres_cap,
                 DevCounters* ctr, unsigned long long* slots, cudaStream_t st) {
  if (g.z_end <= g.z_begin) return 0;
  cudaMemsetAsync(slots, 0, 64 * sizeof(unsigned long long), st);
  switch (g.kind * 2 + (g.periodic ? 1 : 0)) {
    case 0: launch6<kVoronoi, false>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, slots, st); break;
    case 1: launch6<kVoronoi, true>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, slots, st); break;
    case 2: launch6<kJohnsonMehl, false>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, slots, st); break;
    case 3: launch6<kJohnsonMehl, true>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, slots, st); break;
    case 4: launch6<kLaguerre, false>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, slots, st); break;
    default: launch6<kLaguerre, true>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, slots, st); break;
  }
  ball6_publish_kernel<<<1, 32, 0, st>>>(slots, ctr);
  return 2;
}

}  // namespace vxb
