// K2 (v5): the ball phase in gather form, one independent warp per 8^3 brick.
//
// Same contract as ball.cu: labels and values are bit-identical to the
// reference because every culled site loses strictly (by far more than f64
// rounding) at every voxel of the box it was culled for, and the survivors are
// evaluated with the reference's exact f64 fold (ball_scan.hpp:89-96 hoisting,
// geometry.hpp:106-123 order) in ascending site index with a strict <
// (tessellate.cpp:65,132).  There is no block-level barrier: every warp
// gathers, culls and evaluates its own brick.
//
//   rows    : x-rows of cells within R of the brick (lane = row) -> segments of
//             the cell-sorted site arrays (bin.cu).
//   tau_b   : lanes walk their rows' sites (compact f32 copies, bins.f4):
//             tau_b = min upper bound of prox over the brick; W = sites whose
//             lower bound is <= tau_b (ballot compaction).
//   per sub-brick (8 x SY x 4):
//     tau_s + multi-reference bisector cull of W (the kRefs smallest upper
//     bounds; strict dominance is transitive so a culled reference still
//     culls), survivors sorted by site index, exact f64 per-axis tables, exact
//     evaluation (4 voxels per lane), resolve (prox <= cutoff), int4 label
//     stores, warp-aggregated unresolved push, per-candidate histogram counts.
// f32 bounds are widened by kRel = 1e-5 of the magnitude of their terms plus
// an absolute coordinate slack e_d >> the f32 rounding of coordinates.
#include "vx_internal.cuh"

namespace vxb {
namespace v5 {

constexpr int kWarps = 4;
constexpr int kRowCap = 64;
constexpr int kWcap = 96;
constexpr int kFcap = 24;
constexpr int kRefs = 4;
constexpr float kRel = 1e-5f;

__device__ __forceinline__ float lo_add(float a, float b) {
  return (a + b) - kRel * (fabsf(a) + fabsf(b));
}
__device__ __forceinline__ float hi_add(float a, float b) {
  return (a + b) + kRel * (fabsf(a) + fabsf(b));
}

template <int SY>
struct __align__(16) WarpS {
  double T[kFcap][8 + SY + 4];  // exact w^2 for the sub-brick: x[8] | y[SY] | z[4]
  double Ft[kFcap];
  double cx[8], cy[8], cz[8];   // exact voxel centres of the brick (geometry.hpp:58-60)
  float4 Wv[kWcap];             // f32 coords relative to the sub-brick centre, t
  float Wlb[kWcap], Wub[kWcap], Wubp[kWcap];
  int W[kWcap];                 // binned position of each brick-level survivor
  int rs0[kRowCap], rn0[kRowCap], rs1[kRowCap], rn1[kRowCap];
  int refs[kRefs];
  int Fs[kFcap];
  int Fidx[kFcap];
  int cnt[kFcap];
  int Fu[kFcap];
  unsigned char Wfl[kWcap];     // bit a: near the antipode on axis a (bisector: wrap form)
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

struct Box {
  float c[3], h[3];      // centre (absolute, f32) and half extent (+ slack)
  float L[3], invL[3], halfL[3];
};

template <bool PER>
__device__ __forceinline__ float rel(float s, float c, float L, float invL) {
  float v = s - c;
  if (PER) v = v - L * rintf(v * invL);
  return v;
}

// squared-distance bounds of a site over the box; v = relative coordinates
template <bool PER>
__device__ __forceinline__ void bounds(const float4 s, const Box& B, float* v, float& lb,
                                       float& ub) {
  const float u[3] = {s.x, s.y, s.z};
  lb = 0.f;
  ub = 0.f;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    v[a] = rel<PER>(u[a], B.c[a], B.L[a], B.invL[a]);
    const float av = fabsf(v[a]);
    const float mn = fmaxf(av - B.h[a], 0.f);
    float mx = av + B.h[a];
    if (PER) mx = fminf(mx, B.halfL[a]);
    lb = __fmaf_rn(mn, mn, lb);
    ub = __fmaf_rn(mx, mx, ub);
  }
  lb *= (1.f - kRel);
  ub *= (1.f + kRel);
}

// true iff r beats s strictly (by >> f64 rounding) at every point of the box
template <int KIND, bool PER>
__device__ __forceinline__ bool dominated(const float4 s, unsigned fs, float lbs, float ubs,
                                          const float4 r, unsigned fr, float lbr, float ubr,
                                          const Box& B, float invG, float e_d) {
  const float sv[3] = {s.x, s.y, s.z}, rv[3] = {r.x, r.y, r.z};
  float D = 0.f, mag = 0.f;
  if (!PER || ((fs | fr) & 7u) == 0) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float dv = fabsf(sv[a] - rv[a]);
      const float hd = B.h[a] * dv;
      D += (sv[a] - rv[a]) * (sv[a] + rv[a]) - 2.f * hd;
      mag += fabsf(sv[a]) + fabsf(rv[a]) + B.h[a];
    }
    // |terms| <= 2 * (|s|+|r|+h)^2 per axis; coordinate slack e_d on s and r
    mag = mag * (mag * 2.f * kRel + 4.f * e_d);
  } else {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const bool wc = (((fs | fr) >> a) & 1u) != 0;
      float term, m;
      if (wc) {  // min w_s^2 - max w_r^2 along this axis
        const float mn = fmaxf(fabsf(sv[a]) - B.h[a], 0.f);
        const float mx = fminf(fabsf(rv[a]) + B.h[a], B.halfL[a]);
        term = mn * mn - mx * mx;
        m = mn * mn + mx * mx;
      } else {
        const float dv = fabsf(sv[a] - rv[a]);
        term = (sv[a] - rv[a]) * (sv[a] + rv[a]) - 2.f * B.h[a] * dv;
        m = sv[a] * sv[a] + rv[a] * rv[a] + 2.f * B.h[a] * dv;
      }
      D += term;
      mag += m * kRel + 4.f * e_d * (fabsf(sv[a]) + fabsf(rv[a]) + B.h[a] + e_d);
    }
  }
  const float Dlo = D - mag;  // lower bound over the box of d_s^2 - d_r^2
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

template <int KIND, bool PER, int SY>
__global__ void __launch_bounds__(kWarps * 32, 6)
    ball5_kernel(Geo g, Bins bins, const DevParams* __restrict__ prm, int* __restrict__ labels,
                 double* __restrict__ dist, unsigned long long* __restrict__ hist,
                 long long* __restrict__ unres, long long unres_cap, DevCounters* ctr,
                 unsigned long long* __restrict__ eval_slots) {
  constexpr int NT = 8 + SY + 4;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WarpS<SY>& ws = reinterpret_cast<WarpS<SY>*>(smem_raw)[wid];
  const long long brick = (long long)blockIdx.x * kWarps + wid;
  if (brick >= g.nbx * g.nby * g.nbz) return;
  const int bxi = (int)(brick % g.nbx);
  const long long rr = brick / g.nbx;
  const int byi = (int)(rr % g.nby), bzi = (int)(rr / g.nby);
  const long long K0[3] = {8ll * bxi, 8ll * byi, g.z_begin + 8ll * bzi};
  const int be[3] = {(int)min(8ll, g.n[0] - K0[0]), (int)min(8ll, g.n[1] - K0[1]),
                     (int)min(8ll, g.z_end - K0[2])};
  if (lane < 24) {  // exact voxel centres of the brick
    const int a = lane >> 3, k = lane & 7;
    (a == 0 ? ws.cx : a == 1 ? ws.cy : ws.cz)[k] = center(K0[a] + k, g.sp[a]);
  }
  __syncwarp();
  const double* ctab[3] = {ws.cx, ws.cy, ws.cz};
  const double R = prm->gather_r, cutoff = prm->cutoff;
  double blo[3], bhi[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    blo[a] = ctab[a][0];
    bhi[a] = ctab[a][be[a] - 1];
  }
  const float e_d = (float)(1e-6 * (g.lmax + R + (bhi[0] - blo[0]) + (bhi[1] - blo[1]) + (bhi[2] - blo[2])));
  Box B;  // brick box
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    B.c[a] = (float)(0.5 * (blo[a] + bhi[a]));
    B.h[a] = (float)(0.5 * (bhi[a] - blo[a])) * (1.f + kRel) + 2.f * e_d;
    B.L[a] = (float)g.L[a];
    B.invL[a] = (float)g.invL[a];
    B.halfL[a] = (float)g.halfL[a];
  }
  const float invG = KIND == kVoronoi ? 1.f : (float)(1.0 / g.growth);

  // ---- rows of cells within R of the brick ----
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
  if (ok) {
    const double R2 = R * R;
    for (int r = lane; r < nrows; r += 32) {
      const int cy = cl[1] + r % nry, cz = cl[2] + r / nry;
      double dy = 0.0, dz = 0.0;
      if (!full[1]) dy = fmax(0.0, fmax(cy * g.cw[1] - bhi[1], blo[1] - (cy + 1) * g.cw[1]));
      if (!full[2]) dz = fmax(0.0, fmax(cz * g.cw[2] - bhi[2], blo[2] - (cz + 1) * g.cw[2]));
      const double dyz = dy * dy + dz * dz;
      int st0 = 0, n0 = 0, st1 = 0, n1 = 0;
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
          st0 = bins.cell_start[base + a0];
          n0 = bins.cell_start[base + a1 + 1] - st0;
        }
        if (c1 >= c0) {
          st1 = bins.cell_start[base + c0];
          n1 = bins.cell_start[base + c1 + 1] - st1;
        }
      }
      ws.rs0[r] = st0;
      ws.rn0[r] = n0;
      ws.rs1[r] = st1;
      ws.rn1[r] = n1;
    }
  }
  __syncwarp();

  // ---- brick-level tau cull: lane walks the sites of rows lane, lane+32 ----
  int nW = 0;
  if (ok) {
    int sst[4], sn[4], cnt = 0;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int r = lane + 32 * k;
      const bool v = r < nrows;
      sst[2 * k] = v ? ws.rs0[r] : 0;
      sn[2 * k] = v ? ws.rn0[r] : 0;
      sst[2 * k + 1] = v ? ws.rs1[r] : 0;
      sn[2 * k + 1] = v ? ws.rn1[r] : 0;
      cnt += sn[2 * k] + sn[2 * k + 1];
    }
    float mu = __int_as_float(0x7f800000);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      for (int p = sst[q]; p < sst[q] + sn[q]; ++p) {
        const float4 s = bins.f4[p];
        float v[3], lb, ub;
        bounds<PER>(s, B, v, lb, ub);
        mu = fminf(mu, ubp_of<KIND>(ub, s.w, invG));
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mu = fminf(mu, __shfl_xor_sync(0xffffffffu, mu, o));
    int rounds = cnt;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rounds = max(rounds, __shfl_xor_sync(0xffffffffu, rounds, o));
    int q = 0, off = 0;
    for (int k = 0; k < rounds; ++k) {
      int p = -1;
      while (q < 4 && off >= sn[q]) {
        ++q;
        off = 0;
      }
      if (q < 4) {
        p = sst[q] + off;
        ++off;
      }
      bool keep = false;
      if (p >= 0) {
        const float4 s = bins.f4[p];
        float v[3], lb, ub;
        bounds<PER>(s, B, v, lb, ub);
        keep = lbp_of<KIND>(lb, s.w, invG) <= mu;
      }
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      const int pos = nW + __popc(m & ((1u << lane) - 1u));
      if (keep && pos < kWcap) ws.W[pos] = p;
      nW += __popc(m);
    }
    ok = nW <= kWcap;
  }
  __syncwarp();

  // ---- sub-bricks ----
  constexpr int NSY = 8 / SY;
  const long long slab_base = g.z_begin * g.n[0] * g.n[1];
  const bool g1 = g.g_is_one;
  unsigned long long evals = 0;
  for (int sb = 0; sb < 2 * NSY; ++sb) {
    const int so[3] = {0, (sb % NSY) * SY, (sb / NSY) * 4};
    const int se[3] = {be[0], min(SY, be[1] - so[1]), min(4, be[2] - so[2])};
    if (se[1] <= 0 || se[2] <= 0) continue;
    Box S = B;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double l = ctab[a][so[a]], h = ctab[a][so[a] + se[a] - 1];
      S.c[a] = (float)(0.5 * (l + h));
      S.h[a] = (float)(0.5 * (h - l)) * (1.f + kRel) + 2.f * e_d;
    }
    int nF = 0;
    bool sok = ok;
    if (sok) {
      float mu = __int_as_float(0x7f800000);
      for (int i = lane; i < nW; i += 32) {
        const int p = ws.W[i];
        const float4 s = bins.f4[p];
        float v[3], lb, ub;
        bounds<PER>(s, S, v, lb, ub);
        unsigned fl = 0;
        if (PER) {
#pragma unroll
          for (int a = 0; a < 3; ++a)
            if (fabsf(v[a]) + S.h[a] > S.halfL[a] * (1.f - 1e-5f)) fl |= 1u << a;
        }
        const float ubp = ubp_of<KIND>(ub, s.w, invG);
        ws.Wv[i] = make_float4(v[0], v[1], v[2], s.w);
        ws.Wlb[i] = lb;
        ws.Wub[i] = ub;
        ws.Wubp[i] = ubp;
        ws.Wfl[i] = (unsigned char)fl;
        mu = fminf(mu, ubp);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mu = fminf(mu, __shfl_xor_sync(0xffffffffu, mu, o));
      __syncwarp();
      // references: kRefs rounds of warp arg-min of the upper bound
      const int nref = min(kRefs, nW);
      unsigned taken = 0;  // bit k: entry lane + 32k already a reference
      for (int r = 0; r < nref; ++r) {
        float bv = __int_as_float(0x7f800000);
        int bi = 0x7fffffff;
        for (int k = 0; lane + 32 * k < nW; ++k) {
          const int i = lane + 32 * k;
          const float u = ws.Wubp[i];
          if (!((taken >> k) & 1u) && (u < bv || (u == bv && i < bi))) {
            bv = u;
            bi = i;
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ov < bv || (ov == bv && oi < bi)) {
            bv = ov;
            bi = oi;
          }
        }
        if ((bi & 31) == lane) taken |= 1u << (bi >> 5);
        if (lane == 0) ws.refs[r] = bi;
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
                                               ws.Wub[j], S, invG, e_d))
              keep = false;
          }
        }
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        const int pos = nF + __popc(m & ((1u << lane) - 1u));
        if (keep && pos < kFcap) ws.Fu[pos] = ws.W[i];
        nF += __popc(m);
      }
      sok = nF <= kFcap;
      if (!sok) nF = 0;
      __syncwarp();
      if (nF > 0) {
        const int myp = lane < nF ? ws.Fu[lane] : 0;
        const int me = lane < nF ? bins.idx[myp] : 0x7fffffff;
        int rank = 0;
        for (int k = 0; k < nF; ++k) rank += __shfl_sync(0xffffffffu, me, k) < me;
        if (lane < nF) {
          ws.Fs[rank] = myp;
          ws.Fidx[rank] = me;
          ws.cnt[rank] = 0;
        }
        __syncwarp();
        // exact per-axis tables: the reference's w^2 (geometry.hpp:82-89,109,119)
        for (int e = lane; e < nF * NT; e += 32) {
          const int j = e / NT, r = e - j * NT;
          const int p = ws.Fs[j];
          double w2;
          if (r < 8)
            w2 = axis_sq<PER>(bins.x[p], ws.cx[r], g.L[0], g.invL[0]);
          else if (r < 8 + SY)
            w2 = axis_sq<PER>(bins.y[p], ws.cy[so[1] + r - 8], g.L[1], g.invL[1]);
          else
            w2 = axis_sq<PER>(bins.z[p], ws.cz[so[2] + r - 8 - SY], g.L[2], g.invL[2]);
          ws.T[j][r] = w2;
          if (r == 0 && KIND != kVoronoi) ws.Ft[j] = bins.t[p];
        }
        __syncwarp();
      }
    }
    // ---- exact evaluation: lane -> 4 x-voxels of one (y, z) row ----
    constexpr int NPASS = SY == 8 ? 2 : 1;
#pragma unroll 1
    for (int pass = 0; pass < NPASS; ++pass) {
      const int qx = (lane & 1) * 4;
      const int vy = SY == 8 ? ((lane >> 1) & 7) : ((lane >> 1) & 3);
      const int vz = SY == 8 ? ((lane >> 4) * 2 + pass) : (lane >> 3);
      double best[4];
      int bj[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        best[k] = __longlong_as_double(0x7ff0000000000000ll);
        bj[k] = -1;
      }
      for (int j = 0; j < nF; ++j) {
        const double a = __dadd_rn(ws.T[j][8 + SY + vz], ws.T[j][8 + vy]);  // 0 + wz^2 == wz^2
        const double2 w01 = *reinterpret_cast<const double2*>(&ws.T[j][qx]);
        const double2 w23 = *reinterpret_cast<const double2*>(&ws.T[j][qx + 2]);
        const double tj = KIND == kVoronoi ? 0.0 : ws.Ft[j];
        const double d[4] = {__dadd_rn(a, w01.x), __dadd_rn(a, w01.y), __dadd_rn(a, w23.x),
                             __dadd_rn(a, w23.y)};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const double pr = prox_from_dsq<KIND>(d[k], g.growth, g1, tj);
          if (pr < best[k]) {
            best[k] = pr;
            bj[k] = j;
          }
        }
      }
      const bool rowvalid = vy < se[1] && vz < se[2];
      const long long ky = K0[1] + so[1] + vy, kz = K0[2] + so[2] + vz;
      const long long lin0 = K0[0] + qx + g.n[0] * (ky + g.n[1] * kz);
      int lab[4];
      int nun = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        lab[k] = -1;
        if (rowvalid && qx + k < se[0]) {
          if (bj[k] >= 0 && best[k] <= cutoff) lab[k] = ws.Fidx[bj[k]];
          else ++nun;
        }
      }
      if (rowvalid) {
        int* out = labels + (lin0 - slab_base);
        if (qx + 4 <= se[0] && g.vec_store) {
          *reinterpret_cast<int4*>(out) = make_int4(lab[0], lab[1], lab[2], lab[3]);
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (qx + k < se[0]) out[k] = lab[k];
        }
        if (dist) {
          double* dout = dist + (lin0 - slab_base);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (qx + k < se[0] && lab[k] >= 0)
              dout[k] = KIND == kVoronoi ? __dsqrt_rn(best[k]) : best[k];
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
        for (int k = 0; k < 4; ++k)
          if (rowvalid && qx + k < se[0] && lab[k] < 0) {
            if (off < unres_cap) unres[off] = lin0 + k;
            ++off;
          }
      }
      if (hist && nF > 0) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (lab[k] >= 0) atomicAdd(&ws.cnt[bj[k]], 1);
      }
    }
    if (hist && nF > 0) {
      __syncwarp();
      if (lane < nF && ws.cnt[lane]) atomicAdd(&hist[ws.Fidx[lane]], (unsigned long long)ws.cnt[lane]);
    }
    evals += (unsigned long long)nF * (se[0] * se[1] * se[2]);
    if (lane == 0 && !sok) atomicAdd(&ctr->overflow_bricks, 1ull);
    __syncwarp();
  }
  if (lane == 0 && evals) atomicAdd(&eval_slots[(brick * 13) & 63], evals);
}

}  // namespace v5

__global__ void ball5_publish_kernel(const unsigned long long* slots, DevCounters* ctr) {
  unsigned long long s = 0;
  for (int i = threadIdx.x; i < 64; i += 32) s += slots[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (threadIdx.x == 0) ctr->ball_evals += s;
}

template <int KIND, bool PER, int SY>
static void launch5(const Geo& g, const Bins& bins, const DevParams* prm, int* labels,
                    double* dist, unsigned long long* hist, long long* unres, long long cap,
                    DevCounters* ctr, unsigned long long* slots, cudaStream_t st) {
  static bool attr = false;
  const size_t sh = sizeof(v5::WarpS<SY>) * v5::kWarps;
  if (!attr) {
    cudaFuncSetAttribute(v5::ball5_kernel<KIND, PER, SY>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh);
    attr = true;
  }
  const long long nbricks = g.nbx * g.nby * g.nbz;
  const unsigned blocks = (unsigned)((nbricks + v5::kWarps - 1) / v5::kWarps);
  v5::ball5_kernel<KIND, PER, SY><<<blocks, v5::kWarps * 32, sh, st>>>(g, bins, prm, labels, dist,
                                                                     hist, unres, cap, ctr, slots);
}

template <int SY>
static void dispatch5(const Geo& g, const Bins& bins, const DevParams* prm, int* labels,
                      double* dist, unsigned long long* hist, long long* unres, long long cap,
                      DevCounters* ctr, unsigned long long* slots, cudaStream_t st) {
  switch (g.kind * 2 + (g.periodic ? 1 : 0)) {
    case 0: launch5<kVoronoi, false, SY>(g, bins, prm, labels, dist, hist, unres, cap, ctr, slots, st); break;
    case 1: launch5<kVoronoi, true, SY>(g, bins, prm, labels, dist, hist, unres, cap, ctr, slots, st); break;
    case 2: launch5<kJohnsonMehl, false, SY>(g, bins, prm, labels, dist, hist, unres, cap, ctr, slots, st); break;
    case 3: launch5<kJohnsonMehl, true, SY>(g, bins, prm, labels, dist, hist, unres, cap, ctr, slots, st); break;
    case 4: launch5<kLaguerre, false, SY>(g, bins, prm, labels, dist, hist, unres, cap, ctr, slots, st); break;
    default: launch5<kLaguerre, true, SY>(g, bins, prm, labels, dist, hist, unres, cap, ctr, slots, st); break;
  }
}

int launch_ball5(const Geo& g, const Bins& bins, const DevParams* prm, int* labels, double* dist,
                 unsigned long long* hist, long long* unres, long long unres_cap,
                 DevCounters* ctr, unsigned long long* slots, int sy, cudaStream_t st) {
  if (g.z_end <= g.z_begin) return 0;
  cudaMemsetAsync(slots, 0, 64 * sizeof(unsigned long long), st);
  if (sy == 8) dispatch5<8>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, slots, st);
  else dispatch5<4>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, slots, st);
  ball5_publish_kernel<<<1, 32, 0, st>>>(slots, ctr);
  return 2;
}

}  // namespace vxb
