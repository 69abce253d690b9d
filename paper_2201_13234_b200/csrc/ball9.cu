// K2 (v9): the ball phase in gather form -- CTA gather, warp bricks, lane-parallel
// sub-brick culling into candidate bitmasks.
//
// Contract (as ball.cu): labels and values bit-identical to the reference.
// Every culled site loses strictly -- by far more than f64 rounding -- at every
// voxel of the box it was culled for (f32 bounds widened by kRel = 1e-5 of the
// magnitude of their terms plus an absolute coordinate slack e_d), and the
// survivors are evaluated with the reference's exact f64 fold
// (ball_scan.hpp:89-96 hoisting, geometry.hpp:106-123 order) in ascending site
// index with a strict < (tessellate.cpp:65,132).
//
// One CTA (8 warps) = a 16^3 super-brick; warp w = the 8^3 brick
// (w&1, (w>>1)&1, w>>2) = four 8x4x4 sub-bricks.
//   G (CTA)   : cell rows within R of the super-brick; sites whose prox exceeds
//               the cutoff at every voxel of the super-brick are dropped (they
//               cannot decide a resolved voxel); f32 relative coordinates in smem.
//   W (warp)  : tau_brick cull -> W (<= 64 sites), sorted by site index.
//   M (warp)  : lane = W slot; for each sub-brick: bounds of my site, packed
//               (ubp, slot) warp arg-min -> reference r and tau, keep iff
//               lb <= tau and r does not beat me everywhere (bisector bound)
//               -> one 64-bit candidate mask per sub-brick, in index order.
//   T (warp)  : exact f64 w^2 tables of every candidate site for the brick's
//               8+8+8 voxel centres (u*u when the periodic image is fixed).
//   E (warp)  : per sub-brick (all lanes together, no divergence): lane = 4
//               x-voxels; strict-< fold over the mask; resolve (prox <= cutoff);
//               int4 stores; warp-aggregated unresolved push; histogram counts.
#include "vx_internal.cuh"

namespace vxb {
namespace v9 {

constexpr int kSB = 16;
constexpr int kB2Threads = 256;
constexpr int kTcap = 768;
constexpr int kRows2 = 256;
constexpr float kRel = 1e-5f;

struct __align__(16) WarpS9 {
  double T[32][24];   // exact w^2: x[8] | y[8] | z[8], rows = rank in the candidate union
  double Tt[32];
  int Wu[64];         // unsorted W (gather slots)
  int Ws[64];         // sorted W (gather slots)
  int Tidx[64];       // site index per W slot
  int cnt[64];
};

struct __align__(16) Smem9 {
  WarpS9 w[kB2Threads / 32];
  float4 rel[kTcap];  // (ux, uy, uz, t) relative to the super-brick centre (nearest image)
  int p[kTcap];
  int idx[kTcap];
  unsigned char flag[kTcap];  // bit a: periodic image ambiguous over the super-brick
  double cx[kSB], cy[kSB], cz[kSB];
  int seg_start[2 * kRows2];
  int seg_off[2 * kRows2 + 1];
  int warp_tot[kB2Threads / 32];
  int n_total;
  int n_kept;
};

__device__ __forceinline__ float lo_add9(float a, float b) {
  return (a + b) - kRel * (fabsf(a) + fabsf(b));
}
__device__ __forceinline__ float hi_add9(float a, float b) {
  return (a + b) + kRel * (fabsf(a) + fabsf(b));
}
template <int KIND>
__device__ __forceinline__ float lbp_of9(float lb, float t, float invG) {
  if (KIND == kVoronoi) return lb;
  const float dl = KIND == kJohnsonMehl ? sqrtf(lb) : lb;
  return lo_add9(dl * invG * (1.f - kRel), t - kRel * fabsf(t));
}
template <int KIND>
__device__ __forceinline__ float ubp_of9(float ub, float t, float invG) {
  if (KIND == kVoronoi) return ub;
  const float dh = KIND == kJohnsonMehl ? sqrtf(ub) : ub;
  return hi_add9(dh * invG * (1.f + kRel), t + kRel * fabsf(t));
}
__device__ __forceinline__ unsigned okey9(float v) {
  const unsigned b = __float_as_uint(v);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

struct Sub9 {
  float v[3];       // nearest-image offset from the sub-brick centre
  float t, lb, ub, lbp, ubp;
  unsigned near;    // bit a: the periodic image may change inside the sub-brick
};

// bounds of a site (brick-relative coords s) over the sub-brick (offset o, half h)
template <int KIND, bool PER>
__device__ __forceinline__ void sub_bounds9(const float4 s, unsigned fl, const float* o,
                                            const float* h, const float* halfL, float invG,
                                            Sub9& R) {
  const float u[3] = {s.x, s.y, s.z};
  float lb = 0.f, ub = 0.f;
  unsigned near = 0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    float v = u[a] - o[a];
    if (PER) v = v - 2.f * halfL[a] * rintf(v / (2.f * halfL[a]));
    const float av = fabsf(v);
    float mn = fmaxf(av - h[a], 0.f), mx = av + h[a];
    if (PER) {
      mx = fminf(mx, halfL[a]);
      if (av + h[a] > halfL[a] * (1.f - 1e-5f)) near |= 1u << a;
    }
    R.v[a] = v;
    lb = __fmaf_rn(mn, mn, lb);
    ub = __fmaf_rn(mx, mx, ub);
  }
  (void)fl;
  R.lb = lb * (1.f - kRel);
  R.ub = ub * (1.f + kRel);
  R.t = s.w;
  R.near = near;
  R.lbp = lbp_of9<KIND>(R.lb, s.w, invG);
  R.ubp = ubp_of9<KIND>(R.ub, s.w, invG);
}

// true iff r beats s strictly (by >> f64 rounding) everywhere in the sub-brick
template <int KIND>
__device__ __forceinline__ bool dominated9(const Sub9& s, const Sub9& r, const float* h, float invG,
                                           float e_d) {
  if (s.near | r.near) return false;  // image may change inside the box: keep
  float D = 0.f, mag = 0.f;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float dv = fabsf(s.v[a] - r.v[a]);
    D += (s.v[a] - r.v[a]) * (s.v[a] + r.v[a]) - 2.f * h[a] * dv;
    mag += fabsf(s.v[a]) + fabsf(r.v[a]) + h[a];
  }
  // |terms| <= 2 (|s|+|r|+h)^2 per axis; coordinate slack e_d on s and r
  const float Dlo = D - mag * (mag * 2.f * kRel + 4.f * e_d);
  if (KIND == kVoronoi) return Dlo > 0.f;
  const float dt = lo_add9(s.t - kRel * fabsf(s.t), -(r.t + kRel * fabsf(r.t)));
  float q;
  if (KIND == kLaguerre) {
    q = Dlo >= 0.f ? Dlo * invG * (1.f - kRel) : Dlo * invG * (1.f + kRel);
  } else {  // |x-s| - |x-r| = N / (|x-s| + |x-r|)
    if (Dlo >= 0.f) {
      q = Dlo / ((sqrtf(s.ub) + sqrtf(r.ub)) * (1.f + kRel)) * (1.f - kRel);
    } else {
      const float dlo = (sqrtf(s.lb) + sqrtf(r.lb)) * (1.f - kRel);
      if (!(dlo > 0.f)) return false;
      q = Dlo / dlo * (1.f + kRel);
    }
    q = q >= 0.f ? q * invG * (1.f - kRel) : q * invG * (1.f + kRel);
  }
  return lo_add9(q, dt) > 0.f;
}

__device__ __forceinline__ long long wrapi9(long long c, long long m) {
  const long long r = c % m;
  return r < 0 ? r + m : r;
}

template <int KIND, bool PER>
__global__ void __launch_bounds__(kB2Threads, 3)
    ball9_kernel(Geo g, Bins bins, const DevParams* __restrict__ prm, int* __restrict__ labels,
                 double* __restrict__ dist, unsigned long long* __restrict__ hist,
                 long long* __restrict__ unres, long long unres_cap, DevCounters* ctr,
                 unsigned long long* __restrict__ eval_slots) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem9& S = *reinterpret_cast<Smem9*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

  const long long K0[3] = {(long long)blockIdx.x * kSB, (long long)blockIdx.y * kSB,
                           g.z_begin + (long long)blockIdx.z * kSB};
  int ext[3];
  ext[0] = (int)min((long long)kSB, g.n[0] - K0[0]);
  ext[1] = (int)min((long long)kSB, g.n[1] - K0[1]);
  ext[2] = (int)min((long long)kSB, g.z_end - K0[2]);
  double blo[3], bhi[3], cc[3], hs[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    blo[a] = center(K0[a], g.sp[a]);
    bhi[a] = center(K0[a] + ext[a] - 1, g.sp[a]);
    cc[a] = 0.5 * (blo[a] + bhi[a]);
    hs[a] = 0.5 * (bhi[a] - blo[a]);
  }
  const double R = prm->gather_r;
  const double cutoff = prm->cutoff;
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
        const long long wy = PER ? wrapi9(cy, g.m[1]) : cy, wz = PER ? wrapi9(cz, g.m[2]) : cz;
        const long long base = (long long)g.m[0] * (wy + (long long)g.m[1] * wz);
        const int mx = g.m[0];
        long long a0 = 0, a1 = -1, c0 = 0, c1 = -1;
        if (PER) {
          if (cx1 - cx0 + 1 >= mx) {
            a0 = 0;
            a1 = mx - 1;
          } else {
            const long long w0 = wrapi9(cx0, mx), len = cx1 - cx0 + 1;
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
  if (tid < 3 * kSB) {  // exact voxel centres (geometry.hpp:58-60)
    const int a = tid / kSB, k = tid % kSB;
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
        S.rel[pos] = make_float4(uf[0], uf[1], uf[2], (float)tv);
        S.p[pos] = p;
        S.idx[pos] = bins.idx[p];
        S.flag[pos] = (unsigned char)fl;
      }
    }
  }
  __syncthreads();
  const int T = S.n_kept;
  cta_ok = cta_ok && T > 0 && T <= kTcap;

  // ---------------- per warp: 8^3 brick ----------------
  WarpS9& ws = S.w[wid];
  const int bxo = (wid & 1) * 8, byo = ((wid >> 1) & 1) * 8, bzo = (wid >> 2) * 8;
  const int bext[3] = {min(8, ext[0] - bxo), min(8, ext[1] - byo), min(8, ext[2] - bzo)};
  if (bext[0] <= 0 || bext[1] <= 0 || bext[2] <= 0) return;  // no barrier follows
  // brick box relative to the super-brick centre
  float bc[3], bh[3];
  {
    const double* ct[3] = {S.cx, S.cy, S.cz};
    const int bo[3] = {bxo, byo, bzo};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double l = ct[a][bo[a]], h = ct[a][bo[a] + bext[a] - 1];
      bc[a] = (float)(0.5 * (l + h) - cc[a]);
      bh[a] = (float)(0.5 * (h - l)) * (1.f + kRel) + 2.f * e_d;
    }
  }
  // ---- brick-level tau cull -> W (f32, conservative) ----
  int nW = 0;
  bool ok = cta_ok;
  if (ok) {
    float mu = __int_as_float(0x7f800000);
    for (int f = lane; f < T; f += 32) {
      const float4 s = S.rel[f];
      const unsigned fl = S.flag[f];
      const float u[3] = {s.x, s.y, s.z};
      float ub = 0.f;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        float mx = fabsf(u[a] - bc[a]) + bh[a];
        if (PER) mx = ((fl >> a) & 1u) ? halfLf[a] : fminf(mx, halfLf[a]);
        ub = __fmaf_rn(mx, mx, ub);
      }
      mu = fminf(mu, ubp_of9<KIND>(ub * (1.f + kRel), s.w, invG));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mu = fminf(mu, __shfl_xor_sync(0xffffffffu, mu, o));
    for (int f0 = 0; f0 < T; f0 += 32) {
      const int f = f0 + lane;
      bool keep = false;
      if (f < T) {
        const float4 s = S.rel[f];
        const unsigned fl = S.flag[f];
        const float u[3] = {s.x, s.y, s.z};
        float lb = 0.f;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          float mn = fmaxf(fabsf(u[a] - bc[a]) - bh[a], 0.f);
          if (PER && ((fl >> a) & 1u)) mn = 0.f;
          lb = __fmaf_rn(mn, mn, lb);
        }
        keep = lbp_of9<KIND>(lb * (1.f - kRel), s.w, invG) <= mu;
      }
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      const int pos = nW + __popc(m & ((1u << lane) - 1u));
      if (keep && pos < 64) ws.Wu[pos] = f;
      nW += __popc(m);
    }
    ok = nW <= 64;
  }
  __syncwarp();
  // ---- sort W by site index (slots lane, lane + 32) ----
  const bool va = ok && lane < nW, vb = ok && lane + 32 < nW;
  int fa = 0, fb = 0;
  if (ok) {
    const int ua = va ? ws.Wu[lane] : 0, ub_ = vb ? ws.Wu[lane + 32] : 0;
    const int ia = va ? S.idx[ua] : 0x7fffffff, ib = vb ? S.idx[ub_] : 0x7fffffff;
    int ra = 0, rb = 0;
    for (int k = 0; k < min(nW, 32); ++k) {
      const int x = __shfl_sync(0xffffffffu, ia, k);
      ra += x < ia;
      rb += x < ib;
    }
    for (int k = 0; k + 32 < nW; ++k) {
      const int x = __shfl_sync(0xffffffffu, ib, k);
      ra += x < ia;
      rb += x < ib;
    }
    __syncwarp();
    if (va) ws.Ws[ra] = ua;
    if (vb) ws.Ws[rb] = ub_;
    __syncwarp();
    fa = va ? ws.Ws[lane] : 0;  // slot lane now holds the lane-th smallest site index
    fb = vb ? ws.Ws[lane + 32] : 0;
  }
  // site data of my slots, relative to the brick centre
  float4 sa = make_float4(0.f, 0.f, 0.f, 0.f), sb = sa;
  unsigned fla = 0, flb = 0;
  if (va) {
    sa = S.rel[fa];
    fla = S.flag[fa];
    sa.x -= bc[0];
    sa.y -= bc[1];
    sa.z -= bc[2];
  }
  if (vb) {
    sb = S.rel[fb];
    flb = S.flag[fb];
    sb.x -= bc[0];
    sb.y -= bc[1];
    sb.z -= bc[2];
  }
  // ---- per sub-brick (8 x 4 x 4) candidate masks, lane = slot ----
  unsigned long long mask[4] = {0ull, 0ull, 0ull, 0ull};
  if (ok) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int sy = byo + (q & 1) * 4, sz = bzo + (q >> 1) * 4;
      const int ey = min(4, ext[1] - sy), ez = min(4, ext[2] - sz);
      if (ey <= 0 || ez <= 0) continue;
      // sub-brick box relative to the brick centre
      float o[3], h[3];
      {
        const double lx = S.cx[bxo], hx = S.cx[bxo + bext[0] - 1];
        const double ly = S.cy[sy], hy = S.cy[sy + ey - 1];
        const double lz = S.cz[sz], hz = S.cz[sz + ez - 1];
        o[0] = (float)(0.5 * (lx + hx) - cc[0]) - bc[0];
        o[1] = (float)(0.5 * (ly + hy) - cc[1]) - bc[1];
        o[2] = (float)(0.5 * (lz + hz) - cc[2]) - bc[2];
        h[0] = (float)(0.5 * (hx - lx)) * (1.f + kRel) + 3.f * e_d;
        h[1] = (float)(0.5 * (hy - ly)) * (1.f + kRel) + 3.f * e_d;
        h[2] = (float)(0.5 * (hz - lz)) * (1.f + kRel) + 3.f * e_d;
      }
      Sub9 A, B2;
      sub_bounds9<KIND, PER>(sa, fla, o, h, halfLf, invG, A);
      sub_bounds9<KIND, PER>(sb, flb, o, h, halfLf, invG, B2);
      // packed (ubp, slot) arg-min -> reference r, tau = its ubp
      unsigned km = min(va ? ((okey9(A.ubp) & ~63u) | (unsigned)lane) : 0xffffffffu,
                        vb ? ((okey9(B2.ubp) & ~63u) | (unsigned)(lane + 32)) : 0xffffffffu);
#pragma unroll
      for (int s = 16; s > 0; s >>= 1) km = min(km, __shfl_xor_sync(0xffffffffu, km, s));
      const int r = (int)(km & 63u), rl = r & 31;
      const bool rhi = r >= 32;
      Sub9 Z;
      Z.v[0] = __shfl_sync(0xffffffffu, rhi ? B2.v[0] : A.v[0], rl);
      Z.v[1] = __shfl_sync(0xffffffffu, rhi ? B2.v[1] : A.v[1], rl);
      Z.v[2] = __shfl_sync(0xffffffffu, rhi ? B2.v[2] : A.v[2], rl);
      Z.t = __shfl_sync(0xffffffffu, rhi ? B2.t : A.t, rl);
      Z.lb = __shfl_sync(0xffffffffu, rhi ? B2.lb : A.lb, rl);
      Z.ub = __shfl_sync(0xffffffffu, rhi ? B2.ub : A.ub, rl);
      Z.near = __shfl_sync(0xffffffffu, rhi ? B2.near : A.near, rl);
      const float tau = __shfl_sync(0xffffffffu, rhi ? B2.ubp : A.ubp, rl);
      const bool ka = va && (lane == r || (A.lbp <= tau && !dominated9<KIND>(A, Z, h, invG, e_d)));
      const bool kb = vb && (lane + 32 == r || (B2.lbp <= tau && !dominated9<KIND>(B2, Z, h, invG, e_d)));
      mask[q] = (unsigned long long)__ballot_sync(0xffffffffu, ka) |
                ((unsigned long long)__ballot_sync(0xffffffffu, kb) << 32);
    }
  }
  unsigned long long anym = mask[0] | mask[1] | mask[2] | mask[3];
  if (__popcll(anym) > 32) {  // table space exhausted: the brick goes to the shell search
    ok = false;
    anym = 0ull;
#pragma unroll
    for (int q = 0; q < 4; ++q) mask[q] = 0ull;
  }
  // ---- exact tables (the reference's w^2) for every slot that is a candidate ----
#pragma unroll
  for (int h2 = 0; h2 < 2; ++h2) {
    const int j = lane + 32 * h2;
    if ((anym >> j) & 1ull) {
      const int p = S.p[h2 ? fb : fa];
      const double sx[3] = {bins.x[p], bins.y[p], bins.z[p]};
      ws.Tidx[j] = S.idx[h2 ? fb : fa];
      ws.cnt[j] = 0;
      const int tr = __popcll(anym & ((1ull << j) - 1ull));  // table row
      if (KIND != kVoronoi) ws.Tt[tr] = bins.t[p];
      const double* ct[3] = {S.cx + bxo, S.cy + byo, S.cz + bzo};
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double u0 = __dsub_rn(sx[a], ct[a][0]), u7 = __dsub_rn(sx[a], ct[a][7]);
        const bool fixed = !PER || (fabs(u0) < 0.49 * g.L[a] && fabs(u7) < 0.49 * g.L[a]);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          double w = __dsub_rn(sx[a], ct[a][k]);
          if (!fixed) w = wrap_delta(w, g.L[a], g.invL[a]);  // else floor(u*invL+0.5) == 0: w == u
          ws.T[tr][8 * a + k] = __dmul_rn(w, w);
        }
      }
    }
  }
  __syncwarp();
  // ---- exact evaluation per sub-brick: lane -> 4 x-voxels of one (y, z) row ----
  unsigned long long evals = 0;
  const long long slab_base = g.z_begin * g.n[0] * g.n[1];
  const int qx = (lane & 1) * 4, vy = (lane >> 1) & 3, vz = lane >> 3;
  const bool g1 = g.g_is_one;
#pragma unroll 1
  for (int q = 0; q < 4; ++q) {
    const int sy = byo + (q & 1) * 4, sz = bzo + (q >> 1) * 4;
    const int ey = min(4, ext[1] - sy), ez = min(4, ext[2] - sz);
    if (ey <= 0 || ez <= 0) continue;
    unsigned long long mq = 0ull;
#pragma unroll
    for (int qq = 0; qq < 4; ++qq)
      if (qq == q) mq = mask[qq];
    const int ny = (sy - byo) + vy, nz = (sz - bzo) + vz;  // row within the brick
    double best[4];
    int bj[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      best[k] = __longlong_as_double(0x7ff0000000000000ll);
      bj[k] = -1;
    }
    unsigned long long mm = mq;
    while (mm) {
      const int j = __ffsll((long long)mm) - 1;  // ascending site index
      mm &= mm - 1;
      const int tr = __popcll(anym & ((1ull << j) - 1ull));
      const double* Tj = ws.T[tr];
      const double a = __dadd_rn(Tj[16 + nz], Tj[8 + ny]);  // 0 + wz^2 == wz^2 exactly
      const double2 w01 = *reinterpret_cast<const double2*>(Tj + qx);
      const double2 w23 = *reinterpret_cast<const double2*>(Tj + qx + 2);
      const double tj = KIND == kVoronoi ? 0.0 : ws.Tt[tr];
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
    // resolve + store + compaction of unresolved voxels
    const bool rowvalid = vy < ey && vz < ez;
    const long long lin0 = K0[0] + bxo + qx + g.n[0] * ((K0[1] + sy + vy) + g.n[1] * (K0[2] + sz + vz));
    int lab[4];
    long long mylins[4];
    int nun = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      lab[k] = -1;
      if (rowvalid && qx + k < bext[0]) {
        if (bj[k] >= 0 && best[k] <= cutoff) {
          lab[k] = ws.Tidx[bj[k]];
          if (hist) atomicAdd(&ws.cnt[bj[k]], 1);
        } else {
          mylins[nun++] = lin0 + k;
        }
      }
    }
    if (rowvalid) {
      int* out = labels + (lin0 - slab_base);
      if (qx + 4 <= bext[0] && g.vec_store) {
        *reinterpret_cast<int4*>(out) = make_int4(lab[0], lab[1], lab[2], lab[3]);
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (qx + k < bext[0]) out[k] = lab[k];
      }
      if (dist) {
        double* dout = dist + (lin0 - slab_base);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (qx + k < bext[0] && lab[k] >= 0)
            dout[k] = KIND == kVoronoi ? __dsqrt_rn(best[k]) : best[k];
      }
    }
    if (__any_sync(0xffffffffu, nun > 0)) {  // K3: compaction of unresolved voxels
      int inc = nun;
#pragma unroll
      for (int s = 1; s < 32; s <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, s);
        if (lane >= s) inc += y;
      }
      const int wtot = __shfl_sync(0xffffffffu, inc, 31);
      unsigned long long base = 0;
      if (lane == 31) base = atomicAdd(&ctr->n_unres, (unsigned long long)wtot);
      base = __shfl_sync(0xffffffffu, base, 31);
      const long long off = (long long)base + inc - nun;
      for (int i = 0; i < nun; ++i)
        if (off + i < unres_cap) unres[off + i] = mylins[i];
    }
    if (lane == 0) evals += (unsigned long long)__popcll(mq) * (bext[0] * ey * ez);
  }
  __syncwarp();
  if (hist) {
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      const int j = lane + 32 * h2;
      if (((anym >> j) & 1ull) && ws.cnt[j] > 0)
        atomicAdd(&hist[ws.Tidx[j]], (unsigned long long)ws.cnt[j]);
    }
  }
  if (lane == 0 && evals)
    atomicAdd(&eval_slots[(blockIdx.x + 7 * blockIdx.y + 13 * blockIdx.z + wid) & 63], evals);
  if (lane == 0 && !ok) atomicAdd(&ctr->overflow_bricks, 1ull);
}

}  // namespace v9

__global__ void ball9_publish_kernel(const unsigned long long* slots, DevCounters* ctr) {
  unsigned long long s = 0;
  for (int i = threadIdx.x; i < 64; i += 32) s += slots[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (threadIdx.x == 0) ctr->ball_evals += s;
}

template <int KIND, bool PER>
static void launch9(const Geo& g, const Bins& bins, const DevParams* prm, int* labels,
                    double* dist, unsigned long long* hist, long long* unres, long long cap,
                    DevCounters* ctr, unsigned long long* slots, cudaStream_t st) {
  static bool attr = false;
  const size_t sh = sizeof(v9::Smem9);
  if (!attr) {
    cudaFuncSetAttribute(v9::ball9_kernel<KIND, PER>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sh);
    attr = true;
  }
  const dim3 grid((unsigned)((g.n[0] + v9::kSB - 1) / v9::kSB), (unsigned)((g.n[1] + v9::kSB - 1) / v9::kSB),
                  (unsigned)((g.z_end - g.z_begin + v9::kSB - 1) / v9::kSB));
  v9::ball9_kernel<KIND, PER><<<grid, v9::kB2Threads, sh, st>>>(g, bins, prm, labels, dist, hist, unres,
                                                               cap, ctr, slots);
}

int launch_ball9(const Geo& g, const Bins& bins, const DevParams* prm, int* labels, double* dist,
                 unsigned long long* hist, long long* unres, long long unres_cap,
                 DevCounters* ctr, unsigned long long* slots, cudaStream_t st) {
  if (g.z_end <= g.z_begin) return 0;
  cudaMemsetAsync(slots, 0, 128 * sizeof(unsigned long long), st);
  switch (g.kind * 2 + (g.periodic ? 1 : 0)) {
    case 0: launch9<kVoronoi, false>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, slots, st); break;
    case 1: launch9<kVoronoi, true>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, slots, st); break;
    case 2: launch9<kJohnsonMehl, false>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, slots, st); break;
    case 3: launch9<kJohnsonMehl, true>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, slots, st); break;
    case 4: launch9<kLaguerre, false>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, slots, st); break;
    default: launch9<kLaguerre, true>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, slots, st); break;
  }
  ball9_publish_kernel<<<1, 32, 0, st>>>(slots, ctr);
  return 2;
}

}  // namespace vxb
