// The fast engine for d != 3 (d = 1, 2 and 4..16): the same two-step labelling
// as the 3-D ball kernels (reference tessellate_fast, tessellate.cpp:195-282,
// step 1 generic in d through ball_scan.hpp:27-45,55-124), written for a
// d-dimensional cell grid and d-dimensional voxel blocks.
//
//   binning : sites sorted by the id of a uniform d-dimensional cell grid (about
//             one site per cell, axis 0 fastest), stable, so each x-row of cells
//             is a contiguous ascending-index range of the SoA coordinate arrays.
//   block   : one warp per block of 256 voxels -- 256 along x (d = 1), 16 x 16
//             (d = 2), 4 x 4 x (16 over the higher axes) (d >= 4).  The warp
//             walks the cell rows within the gather radius R of its block (rows
//             indexed by axes 1..d-1, one lane per row, 32 rows per pass), loads
//             every gathered site once with exact f64 residuals to the block
//             centre, keeps the sites whose prox lower bound over the block is
//             <= min(cutoff, least upper bound) (every possible winner of a
//             resolved voxel), rank-sorts them by site index (the reference's
//             strict-< scan order, tessellate.cpp:65,132), then evaluates them
//             exactly -- per-axis f64 tables of w^2 folded from the last axis to
//             axis 0 (geometry.hpp:95-135) -- 8 voxels per lane, in chunks of 32
//             candidates with the running minimum carried over.
//   step 2  : voxels whose best prox exceeds the cutoff (outside every ball), and
//             the voxels of blocks whose gather overflows a cap, are labelled by
//             an all-sites scan (the reference's resolve_voxels_impl,
//             tessellate.cpp:36-75), keeping the lexicographic (prox, index)
//             minimum.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <atomic>
#include <cmath>

#include "vx_internal.cuh"

namespace vxb {
namespace vnd {

constexpr int kRowPass = 32;     // cell rows per gather pass (one per lane)
constexpr int kRowCap = 1 << 14; // rows a block may gather
constexpr int kGCap = 256;       // gathered sites within the cutoff per block
constexpr int kChunk = 16;       // candidates per exact-table pass
constexpr int kTW = 32;          // table width (doubles per candidate row)

struct __align__(16) BlockSmem {
  union {
    struct {                         // phase A: gather + list
      int kp[kGCap];                 // kept: binned position
      int kidx[kGCap];               // kept: original site index (sort key)
      float klbp[kGCap];             // kept: prox lower bound over the block (rounded down)
      alignas(16) int lkey[kGCap + 4];  // candidate list: original index, INT_MAX padded
      int lslot[kGCap];              // candidate list: kept slot
    } a;
    struct {                         // phase B: exact tables of one chunk
      alignas(16) double T[kChunk][kTW];
      double Ft[kChunk];
    } b;
  } u;
  int seg_start[2 * kRowPass];
  int seg_off[2 * kRowPass + 1];
  int sp[kGCap];        // sorted candidates: binned position
  int sidx[kGCap];      // sorted candidates: original index
  int cnt[kGCap];       // sorted candidates: resolved voxels (histogram)
  double C[kTW];        // the block's voxel centres per table column
};

__device__ __forceinline__ long long wrapm(long long c, long long m) {
  const long long r = c % m;
  return r < 0 ? r + m : r;
}

__device__ __forceinline__ long long slab_voxels(const GeoN& g, int D) {
  long long n = g.ze - g.zb;
  for (int a = 0; a < D - 1; ++a) n *= g.n[a];
  return n;
}

// table column layout of a block: axis 0 (d = 1: none, d = 2: 16 columns,
// d >= 4: 4), axis 1 (16 | 4), axes >= 2: E[a] columns each
struct Layout {
  int off[kMaxDim];
  int ext[kMaxDim];
  int ncol;
};

__device__ __forceinline__ Layout layout_of(const GeoN& g, int D) {
  Layout l;
  int o = 0;
  for (int a = 0; a < D; ++a) {
    l.off[a] = o;
    l.ext[a] = D == 1 ? 0 : g.E[a];
    o += l.ext[a];
  }
  l.ncol = o;
  return l;
}

// DT: the dimension at compile time (1, 2, 4), 0 = any (runtime g.dim, 5..16)
template <int DT, int KIND, bool PER, bool FA>
__global__ void __launch_bounds__(32, 20)
    ballnd_kernel(GeoN g, BinsN bins, const DevParams* __restrict__ prm, int* __restrict__ labels,
                  double* __restrict__ dist, unsigned long long* __restrict__ hist, long long* __restrict__ unres,
                  long long unres_cap, DevCounters* ctr, long long n_blocks) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  BlockSmem& ws = *reinterpret_cast<BlockSmem*>(smem_raw);
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  const int D = DT > 0 ? DT : g.dim;
  const long long blk = blockIdx.x + (long long)gridDim.x * blockIdx.y;
  if (blk >= n_blocks) return;
  // block coordinates (mixed radix, axis 0 fastest; the last axis counts from the slab start)
  long long o[kMaxDim];
  int ext[kMaxDim];
  {
    long long r = blk;
    for (int a = 0; a < D; ++a) {
      const long long b = r % g.nb[a];
      r /= g.nb[a];
      o[a] = b * g.E[a] + (a == D - 1 ? g.zb : 0);
      const long long hi = a == D - 1 ? g.ze : g.n[a];
      ext[a] = (int)min((long long)g.E[a], hi - o[a]);
    }
  }
  double blo[kMaxDim], bhi[kMaxDim], cc[kMaxDim], hs[kMaxDim];
  for (int a = 0; a < D; ++a) {
    blo[a] = center(o[a], g.sp[a]);
    bhi[a] = center(o[a] + ext[a] - 1, g.sp[a]);
    cc[a] = 0.5 * (blo[a] + bhi[a]);
    hs[a] = 0.5 * (bhi[a] - blo[a]);
  }
  const double R = prm->gather_r;
  const double R2 = R * R;
  const double cutoff = prm->cutoff;
  const double tc = cutoff + 1e-9 * fabs(cutoff);
  bool ok = true;

  // ---------------- gather ----------------
  long long cl[kMaxDim], cr[kMaxDim];
  bool full[kMaxDim];
  long long nrows = 1;
  for (int a = 0; a < D; ++a) {
    cl[a] = (long long)floor((blo[a] - R) * g.inv_cw[a] - 1e-6);
    const long long ch = (long long)floor((bhi[a] + R) * g.inv_cw[a] + 1e-6);
    full[a] = false;
    if (PER) {
      if (ch - cl[a] + 1 >= g.m[a]) {
        cl[a] = 0;
        cr[a] = g.m[a];
        full[a] = true;
      } else {
        cr[a] = ch - cl[a] + 1;
      }
    } else {
      cl[a] = max(cl[a], 0ll);
      cr[a] = max(0ll, min(ch, (long long)g.m[a] - 1) - cl[a] + 1);
    }
    if (a >= 1) nrows *= cr[a];
  }
  if (nrows > kRowCap) ok = false;
  int nk = 0;
  double taud = __longlong_as_double(0x7ff0000000000000ll);
  for (long long r0 = 0; ok && r0 < nrows; r0 += kRowPass) {
    // lane -> row r0 + lane: cells (c_1 .. c_{D-1}); up to 2 x-segments
    int st[2] = {0, 0}, cn[2] = {0, 0};
    const long long r = r0 + lane;
    if (r < nrows) {
      long long rr = r, base = 0;
      double d2 = 0.0;
      for (int a = 1; a < D; ++a) {
        const long long c = cl[a] + rr % cr[a];
        rr /= cr[a];
        if (!full[a]) {
          const double gap = fmax(0.0, fmax(c * g.cw[a] - bhi[a], blo[a] - (c + 1) * g.cw[a]));
          d2 += gap * gap;
        }
        base += (PER ? wrapm(c, g.m[a]) : c) * g.cstride[a];
      }
      if (d2 <= R2 * (1.0 + 1e-9)) {
        const double exr = sqrt(fmax(R2 - d2, 0.0)) * (1.0 + 1e-9) + 1e-12 * g.lmax;
        const long long cx0 = (long long)floor((blo[0] - exr) * g.inv_cw[0] - 1e-6);
        const long long cx1 = (long long)floor((bhi[0] + exr) * g.inv_cw[0] + 1e-6);
        const long long mx = g.m[0];
        long long a0 = 0, a1 = -1, c0 = 0, c1 = -1;
        if (PER) {
          if (cx1 - cx0 + 1 >= mx) {
            a1 = mx - 1;
          } else {
            const long long w0 = wrapm(cx0, mx), len = cx1 - cx0 + 1;
            a0 = w0;
            if (w0 + len <= mx) {
              a1 = w0 + len - 1;
            } else {
              a1 = mx - 1;
              c1 = len - (mx - w0) - 1;
            }
          }
        } else {
          a0 = max(cx0, 0ll);
          a1 = min(cx1, mx - 1);
        }
        VXCHK(base >= 0 && base + a1 + 1 <= g.n_cells && (c1 < c0 || base + c1 + 1 <= g.n_cells), "row cells");
        if (a1 >= a0) {
          st[0] = bins.cell_start[base + a0];
          cn[0] = bins.cell_start[base + a1 + 1] - st[0];
        }
        if (c1 >= c0) {
          st[1] = bins.cell_start[base + c0];
          cn[1] = bins.cell_start[base + c1 + 1] - st[1];
        }
      }
    }
    int inc = cn[0] + cn[1];
    const int mine = inc;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, s);
      if (lane >= s) inc += y;
    }
    const int ptot = __shfl_sync(0xffffffffu, inc, 31);
    __syncwarp();
    ws.seg_start[2 * lane] = st[0];
    ws.seg_start[2 * lane + 1] = st[1];
    ws.seg_off[2 * lane] = inc - mine;
    ws.seg_off[2 * lane + 1] = inc - mine + cn[0];
    __syncwarp();
    for (int f0 = 0; f0 < ptot; f0 += 32) {
      const int f = f0 + lane;
      bool keep = false;
      int p = 0;
      double lbp = 0.0;
      if (f < ptot) {
        int lo = 0, hi = 31;  // the last lane whose first offset is <= f
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (ws.seg_off[2 * mid] <= f) lo = mid;
          else hi = mid - 1;
        }
        const int sg = ws.seg_off[2 * lo + 1] <= f ? 2 * lo + 1 : 2 * lo;
        p = ws.seg_start[sg] + (f - ws.seg_off[sg]);
        VXCHK(p >= 0 && p < g.n_sites, "gathered position %d", p);
        double lb = 0.0, ub = 0.0;
        for (int a = 0; a < D; ++a) {
          double u = bins.x[p + a * bins.stride] - cc[a];
          bool amb = false;
          if (PER) {
            u = u - floor(u * g.invL[a] + 0.5) * g.L[a];
            amb = fabs(u) + hs[a] >= g.halfL[a] * (1.0 - 1e-7);
          }
          const double au = fabs(u);
          const double mn = amb ? 0.0 : fmax(au - hs[a], 0.0);
          const double mx = amb ? g.halfL[a] : (PER ? fmin(au + hs[a], g.halfL[a]) : au + hs[a]);
          lb += mn * mn;
          ub += mx * mx;
        }
        lb *= 1.0 - 1e-9;
        ub *= 1.0 + 1e-9;
        lbp = lb;
        double ubp = ub;
        if (KIND != kVoronoi) {
          const double tv = bins.t[p];
          const double A = (KIND == kJohnsonMehl ? sqrt(lb) : lb) / g.growth * (1.0 - 1e-9);
          const double B = (KIND == kJohnsonMehl ? sqrt(ub) : ub) / g.growth * (1.0 + 1e-9);
          lbp = A + tv - 1e-9 * (fabs(tv) + A);
          ubp = B + tv + 1e-9 * (fabs(tv) + B);
        }
        keep = lbp <= tc;
        taud = fmin(taud, ubp);
      }
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      const int pos = nk + __popc(m & lt_mask);
      if (keep && pos < kGCap) {
        ws.u.a.kp[pos] = p;
        ws.u.a.kidx[pos] = bins.idx[p];
        ws.u.a.klbp[pos] = __double2float_rd(lbp);
      }
      nk += __popc(m);
    }
    if (nk > kGCap) ok = false;
    __syncwarp();
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) taud = fmin(taud, __shfl_xor_sync(0xffffffffu, taud, s));
  const float tau = fminf(__double2float_ru(tc), __double2float_ru(taud));

  // ---------------- candidate list: lbp <= tau, sorted by site index ----------------
  int nl = 0;
  if (ok) {
    for (int k0 = 0; k0 < nk; k0 += 32) {
      const int k = k0 + lane;
      const bool keep = k < nk && ws.u.a.klbp[k] <= tau;
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      const int pos = nl + __popc(m & lt_mask);
      if (keep) {
        ws.u.a.lkey[pos] = ws.u.a.kidx[k];
        ws.u.a.lslot[pos] = k;
      }
      nl += __popc(m);
    }
    __syncwarp();
    if (lane < 4) ws.u.a.lkey[nl + lane] = 0x7fffffff;
    __syncwarp();
    const int4* key4 = reinterpret_cast<const int4*>(ws.u.a.lkey);
    for (int k = lane; k < nl; k += 32) {
      const int me = ws.u.a.lkey[k];
      int rank = 0;
      for (int i = 0; i < (nl + 3) >> 2; ++i) {
        const int4 v = key4[i];
        rank += (v.x < me) + (v.y < me) + (v.z < me) + (v.w < me);
      }
      VXCHK(rank >= 0 && rank < nl && ws.u.a.lslot[k] < nk, "rank %d nl %d", rank, nl);
      ws.sp[rank] = ws.u.a.kp[ws.u.a.lslot[k]];
      ws.sidx[rank] = me;
      ws.cnt[rank] = 0;
    }
  }
  __syncwarp();

  // ---------------- the lane's 8 voxels ----------------
  const Layout Ly = layout_of(g, D);
  // column of each table axis for this lane; voxel k = (xk, row h) within the lane
  int colx = 0, coly = 0, hcol[kMaxDim];
  int lx0 = 0, ly0 = 0;  // lane's first voxel offset in the block along x and y
  long long hi_off = 0;  // linear offset of the lane's higher-axis coordinates
  bool hvalid = true;
  if (D == 1) {
    lx0 = lane * 8;
  } else if (D == 2) {
    lx0 = (lane & 3) * 4;
    ly0 = lane >> 2;  // rows ly0 and ly0 + 8
    colx = Ly.off[0] + lx0;
    coly = Ly.off[1] + ly0;
  } else {
    lx0 = 0;
    ly0 = 2 * (lane & 1);  // rows ly0 and ly0 + 1
    colx = Ly.off[0];
    coly = Ly.off[1] + ly0;
    int hh = lane >> 1;
    long long stride = g.n[0] * g.n[1];
    for (int a = 2; a < D; ++a) {
      const int c = hh % g.E[a];
      hh /= g.E[a];
      hcol[a] = Ly.off[a] + c;
      hvalid = hvalid && c < ext[a];
      hi_off += (o[a] + c - (a == D - 1 ? g.zb : 0)) * stride;
      stride *= g.n[a];
    }
  }
  // table centres: lanes fill C[col] for every column
  for (int col = lane; col < Ly.ncol; col += 32) {
    int a = 0;
    while (a + 1 < D && Ly.off[a + 1] <= col) ++a;
    const int k = min(col - Ly.off[a], ext[a] - 1);  // beyond the grid: the last centre (never stored)
    ws.C[col] = center(o[a] + k, g.sp[a]);
  }
  double cx1[8];  // d = 1: the lane's own voxel centres
  if (D == 1) {
#pragma unroll
    for (int k = 0; k < 8; ++k) cx1[k] = center(o[0] + min(lx0 + k, ext[0] - 1), g.sp[0]);
  }
  __syncwarp();

  double best[8];
  int bj[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    best[k] = __longlong_as_double(0x7ff0000000000000ll);
    bj[k] = 0;
  }
  const bool g1 = g.g_is_one;
  const int nlist = ok ? nl : 0;
  for (int c0 = 0; c0 < nlist; c0 += kChunk) {
    const int m = min(kChunk, nlist - c0);
    if (D == 1) {
      // direct: each lane its own 8 residuals per candidate
      for (int j = 0; j < m; ++j) {
        const int p = ws.sp[c0 + j];
        const double sv = bins.x[p];
        const double tj = KIND == kVoronoi ? 0.0 : bins.t[p];
        double u[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) u[k] = __dsub_rn(sv, cx1[k]);
        if (PER) {
          const double lim = 0.49 * g.L[0];
          if (!(fabs(u[0]) < lim) || !(fabs(u[7]) < lim)) {
#pragma unroll
            for (int k = 0; k < 8; ++k)
              if (!(fabs(u[k]) < lim)) u[k] = wrap_delta(u[k], g.L[0], g.invL[0]);
          }
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const double d = __dmul_rn(u[k], u[k]);
          const double pr = FA ? prox_from_dsq_nc<KIND>(d, g.growth, g1, tj, g.inv_growth_rn)
                               : prox_from_dsq<KIND>(d, g.growth, g1, tj);
          if (pr < best[k]) {
            best[k] = pr;
            bj[k] = c0 + j;
          }
        }
      }
      continue;
    }
    // exact tables: one lane per (candidate, axis)
    for (int e = lane; e < D * m; e += 32) {
      const int a = e / m, j = e - a * m;
      VXCHK(Ly.off[a] + Ly.ext[a] <= kTW && j < kChunk, "table column %d", Ly.off[a] + Ly.ext[a]);
      const int p = ws.sp[c0 + j];
      const double sv = bins.x[p + a * bins.stride];
      const int ne = Ly.ext[a], col0 = Ly.off[a];
      const double lim = 0.49 * g.L[a];
      bool far = false;
      for (int r = 0; r < ne; ++r) {
        double u = __dsub_rn(sv, ws.C[col0 + r]);
        if (PER && !(fabs(u) < lim)) {
          u = wrap_delta(u, g.L[a], g.invL[a]);
          far = true;
        }
        ws.u.b.T[j][col0 + r] = __dmul_rn(u, u);
      }
      (void)far;
      if (KIND != kVoronoi && a == 0) ws.u.b.Ft[j] = bins.t[p];
    }
    __syncwarp();
    for (int j = 0; j < m; ++j) {
      const double* Tj = ws.u.b.T[j];
      double a0, a1;
      if (D == 2) {
        a0 = Tj[coly];      // 0 + w_1^2 == w_1^2
        a1 = Tj[coly + 8];
      } else {
        double hi = Tj[hcol[D - 1]];
        for (int a = D - 2; a >= 2; --a) hi = __dadd_rn(hi, Tj[hcol[a]]);  // fold from the last axis
        a0 = __dadd_rn(hi, Tj[coly]);
        a1 = __dadd_rn(hi, Tj[coly + 1]);
      }
      const double2 w01 = *reinterpret_cast<const double2*>(&Tj[colx]);
      const double2 w23 = *reinterpret_cast<const double2*>(&Tj[colx + 2]);
      const double tj = KIND == kVoronoi ? 0.0 : ws.u.b.Ft[j];
      const double d[8] = {__dadd_rn(a0, w01.x), __dadd_rn(a0, w01.y), __dadd_rn(a0, w23.x), __dadd_rn(a0, w23.y),
                           __dadd_rn(a1, w01.x), __dadd_rn(a1, w01.y), __dadd_rn(a1, w23.x), __dadd_rn(a1, w23.y)};
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
    __syncwarp();  // the next chunk rewrites the tables
  }

  // ---------------- resolve + store + compaction of unresolved voxels ----------------
  // voxel k of the lane: d = 1: x = lx0 + k; else x = lx0 + (k & 3), row h = k >> 2
  const long long rowstep = D == 2 ? 8 * g.n[0] : g.n[0];  // row h = 1
  long long lbase;  // linear index (slab-relative) of the lane's voxel 0
  unsigned vmask = 0;
  if (D == 1) {
    lbase = o[0] - g.zb + lx0;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (lx0 + k < ext[0]) vmask |= 1u << k;
  } else {
    const long long y0 = o[1] + ly0;
    const long long zrow = D == 2 ? o[1] - g.zb + ly0 : y0;
    lbase = (D == 2 ? zrow * g.n[0] : hi_off + y0 * g.n[0]) + o[0] + lx0;
    const int xr = ext[0] - lx0;
    const unsigned xm = xr >= 4 ? 0xFu : (xr > 0 ? (1u << xr) - 1u : 0u);
    const int r1 = D == 2 ? ly0 + 8 : ly0 + 1;
    if (hvalid) vmask = (ly0 < ext[1] ? xm : 0u) | (r1 < ext[1] ? xm << 4 : 0u);
  }
  int lab[8];
  unsigned umask = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    lab[k] = -1;
    if ((vmask >> k) & 1u) {
      if (best[k] <= cutoff) {
        lab[k] = ws.sidx[bj[k]];
        if (hist) atomicAdd(&ws.cnt[bj[k]], 1);
      } else {
        umask |= 1u << k;
      }
    }
  }
  auto vox = [&](int k) -> long long {
    return D == 1 ? lbase + k : lbase + (k >> 2) * rowstep + (k & 3);
  };
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    if (!((vmask >> k) & 1u)) continue;
    const long long v = vox(k);
    VXCHK(v >= 0 && v < slab_voxels(g, D), "voxel %lld", v);
    labels[v] = lab[k];
    if (dist && lab[k] >= 0) dist[v] = KIND == kVoronoi ? __dsqrt_rn(best[k]) : best[k];
  }
  if (__any_sync(0xffffffffu, umask != 0)) {
    const int nun = __popc(umask);
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
    unsigned mm = umask;
    for (int i = 0; i < nun; ++i) {
      const int k = __ffs(mm) - 1;
      mm &= mm - 1;
      if (off + i < unres_cap) unres[off + i] = vox(k);  // slab-relative
    }
  }
  __syncwarp();
  if (hist)
    for (int k = lane; k < nlist; k += 32)
      if (ws.cnt[k]) atomicAdd(&hist[ws.sidx[k]], (unsigned long long)ws.cnt[k]);
  if (lane == 0 && !ok) atomicAdd(&ctr->overflow_bricks, 1ull);
  unsigned long long ev = (unsigned long long)nlist * __popc(vmask);
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) ev += __shfl_xor_sync(0xffffffffu, ev, s);
  if (lane == 0 && ev) atomicAdd(&ctr->ball_evals, ev);
}

// Step 2: the unresolved voxels (outside every ball) -- one warp per voxel,
// widening gathers: all sites in the cell rows within radius rho of the voxel
// (rho = 2 R, 4 R, ...), exact prox, lexicographic (prox, index) minimum (the
// order-independent form of the reference's ascending strict-< all-sites scan,
// tessellate.cpp:36-75).  The search stops once a conservative lower bound of
// prox beyond rho exceeds the best (ties with a lower-index site further out
// are still found) or rho covers the whole domain.  The list holds
// slab-relative voxel indices; past its capacity the label image itself
// (-1 = unresolved) is scanned.
constexpr int kUT = 128;

template <int KIND, bool PER>
__global__ void __launch_bounds__(kUT)
    unres_nd_kernel(GeoN g, BinsN bins, const DevParams* __restrict__ prm, const long long* __restrict__ unres,
                    long long unres_cap, int* labels, double* __restrict__ dist, unsigned long long* __restrict__ hist,
                    DevCounters* ctr, long long nvs) {
  const int D = g.dim;
  const int lane = threadIdx.x & 31;
  const long long nlist = (long long)ctr->n_unres;
  const bool scan = nlist > unres_cap;
  const long long total = scan ? nvs : nlist;
  const bool g1 = g.g_is_one;
  const double t_min = prm->t_min;
  long long plane = 1;
  for (int a = 0; a < D - 1; ++a) plane *= g.n[a];
  double diag2 = 0.0;  // the largest possible distance^2 between a voxel and a site
  for (int a = 0; a < D; ++a) diag2 += PER ? g.halfL[a] * g.halfL[a] : g.L[a] * g.L[a];
  unsigned long long ne = 0;
  const long long nw = (long long)gridDim.x * (kUT / 32);
  for (long long i = blockIdx.x * (long long)(kUT / 32) + (threadIdx.x >> 5); i < total; i += nw) {
    const long long v = scan ? (labels[i] < 0 ? i : -1) : unres[i];
    if (v < 0) continue;  // uniform over the warp
    double x[kMaxDim];
    {
      long long r = v + g.zb * plane;  // absolute linear index
      for (int a = 0; a < D; ++a) {
        x[a] = center(r % g.n[a], g.sp[a]);
        r /= g.n[a];
      }
    }
    double best = __longlong_as_double(0x7ff0000000000000ll);
    int bi = 0x7fffffff;
    // an unresolved voxel's nearest site lies just beyond the gather radius:
    // start at 1.25 R and widen by 1.6
    double rho = 1.25 * prm->gather_r;
    if (!(rho > 0.0)) rho = g.lmax;
    for (int iter = 0; iter < 64; ++iter) {
      const bool last = rho * rho >= diag2;
      // cell box of [x - rho, x + rho] (whole axis when it wraps around)
      long long cl[kMaxDim], cr[kMaxDim], nrows = 1;
      unsigned fullm = 0;  // bit a: the box covers the whole (periodic) axis
      for (int a = 0; a < D; ++a) {
        long long lo = (long long)floor((x[a] - rho) * g.inv_cw[a]) - 1, hi = (long long)floor((x[a] + rho) * g.inv_cw[a]) + 1;
        if (last || (PER && hi - lo + 1 >= g.m[a])) {
          lo = 0;
          hi = g.m[a] - 1;
          fullm |= 1u << a;
        } else if (!PER) {
          lo = max(lo, 0ll);
          hi = min(hi, (long long)g.m[a] - 1);
        }
        cl[a] = lo;
        cr[a] = hi - lo + 1;
        nrows *= cr[a];  // cells, all axes
      }
      // every cell of the box, one lane per cell, its sites in turn
      for (long long c0 = 0; c0 < nrows; c0 += 32) {
        const long long c = c0 + lane;
        int s0 = 0, s1 = 0;
        if (c < nrows) {
          long long rr = c, key = 0;
          double d2 = 0.0;  // lower bound of the squared distance to the cell
          for (int a = 0; a < D; ++a) {
            long long cc = cl[a] + rr % cr[a];
            rr /= cr[a];
            if (!((fullm >> a) & 1u)) {  // unwrapped cell index: its distance along a (a full axis adds 0)
              const double gap = fmax(0.0, fmax(cc * g.cw[a] - x[a], x[a] - (cc + 1) * g.cw[a]));
              d2 += gap * gap;
            }
            if (PER) cc = wrapm(cc, g.m[a]);
            key += cc * g.cstride[a];
          }
          // every site of a cell farther than rho stays beyond the bound below
          if (last || d2 <= rho * rho * (1.0 + 1e-6)) {
            s0 = bins.cell_start[key];
            s1 = bins.cell_start[key + 1];
          }
        }
        for (int p = s0; p < s1; ++p) {
          double acc = 0.0;
          for (int a = D - 1; a >= 0; --a)  // fold from the last axis (geometry.hpp:106-123)
            acc = __dadd_rn(acc, axis_sq<PER>(bins.x[p + a * bins.stride], x[a], g.L[a], g.invL[a]));
          const double pr = prox_from_dsq<KIND>(acc, g.growth, g1, KIND == kVoronoi ? 0.0 : bins.t[p]);
          const int id = bins.idx[p];
          if (pr < best || (pr == best && id < bi)) {
            best = pr;
            bi = id;
          }
          ++ne;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob < best || (ob == best && oi < bi)) {
          best = ob;
          bi = oi;
        }
      }
      if (last) break;
      // every site outside the box is farther than rho (cell margins of one
      // cell on each side): its prox exceeds this bound
      const double r1 = rho * (1.0 - 1e-9);
      double bound = r1 * r1;
      if (KIND == kJohnsonMehl) bound = r1 / g.growth * (1.0 - 1e-9) + t_min - 1e-9 * fabs(t_min);
      if (KIND == kLaguerre) bound = r1 * r1 / g.growth * (1.0 - 1e-9) + t_min - 1e-9 * fabs(t_min);
      if (best < bound) break;  // strictly: a tie beyond rho could have a lower index
      rho *= 1.6;
    }
    if (lane == 0) {
      labels[v] = bi;
      if (dist) dist[v] = KIND == kVoronoi ? __dsqrt_rn(best) : best;
      if (hist) atomicAdd(&hist[bi], 1ull);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ne += __shfl_xor_sync(0xffffffffu, ne, o);
  if (lane == 0 && ne) atomicAdd(&ctr->shell_evals, ne);
}

// prune_ineffective_sites for d != 3 (sites.cpp:113-171; the predicate of
// prune.cu): each site against the sites of every cell within its reach --
// JM: d <= G (t_s - t_min); Laguerre: every axis_min_sq_diff term is
// <= -(wrapped delta)^2, so d <= sqrt(G (t_s - t_min)).  "Dropped" is an OR
// over o, so the enumeration order is irrelevant: identical survivors.
__device__ __forceinline__ double axis_min_sq_diff_nd(double a, double b, double L, double invL, bool periodic) {
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

template <bool PER>
__global__ void prune_nd_kernel(GeoN g, BinsN bins, const double* __restrict__ pos, const double* __restrict__ t,
                                const DevParams* __restrict__ prm, uint8_t* __restrict__ dropped) {
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= g.n_sites) return;
  const int D = g.dim;
  const double ts = t[s];
  const double t_min = dkey_inv(prm->tmin_key);
  const double dt = fmax(ts - t_min, 0.0);
  const double reach = (g.kind == kJohnsonMehl ? g.growth * dt : sqrt(g.growth * dt)) * (1.0 + 1e-9) + 1e-12 * g.lmax;
  double xs[kMaxDim];
  long long cl[kMaxDim], cr[kMaxDim], ncell = 1;
  for (int a = 0; a < D; ++a) {
    xs[a] = pos[s * D + a];
    long long lo = (long long)floor((xs[a] - reach) * g.inv_cw[a]) - 1, hi = (long long)floor((xs[a] + reach) * g.inv_cw[a]) + 1;
    if (PER && hi - lo + 1 >= g.m[a]) {
      lo = 0;
      hi = g.m[a] - 1;
    } else if (!PER) {
      lo = max(lo, 0ll);
      hi = min(hi, (long long)g.m[a] - 1);
    }
    cl[a] = lo;
    cr[a] = hi - lo + 1;
    ncell *= cr[a];
  }
  bool drop = false;
  for (long long c = 0; c < ncell && !drop; ++c) {
    long long rr = c, key = 0;
    for (int a = 0; a < D; ++a) {
      long long cc = cl[a] + rr % cr[a];
      rr /= cr[a];
      if (PER) cc = wrapm(cc, g.m[a]);
      key += cc * g.cstride[a];
    }
    const int p1 = bins.cell_start[key + 1];
    for (int p = bins.cell_start[key]; p < p1 && !drop; ++p) {
      const long long o = bins.idx[p];
      if (o == s) continue;
      if (g.kind == kJohnsonMehl) {
        double acc = 0.0;
        for (int a = D - 1; a >= 0; --a) acc = __dadd_rn(acc, axis_sq<PER>(bins.x[p + a * bins.stride], xs[a], g.L[a], g.invL[a]));
        double r = __dsqrt_rn(acc);
        if (!g.g_is_one) r = __ddiv_rn(r, g.growth);
        r = __dadd_rn(r, bins.t[p]);
        drop = r < ts || (r == ts && o < s);
      } else {
        double margin = __dmul_rn(g.growth, __dsub_rn(ts, bins.t[p]));
        for (int a = 0; a < D; ++a)
          margin = __dadd_rn(margin, axis_min_sq_diff_nd(xs[a], bins.x[p + a * bins.stride], g.L[a], g.invL[a], PER));
        drop = margin > 0.0 || (margin == 0.0 && o < s);
      }
    }
  }
  dropped[s] = drop ? 1 : 0;
}

// ---- binning ----
__global__ void keys_nd_kernel(GeoN g, const double* __restrict__ pos, const double* __restrict__ t,
                               const uint8_t* __restrict__ dropped, unsigned* __restrict__ keys,
                               int* __restrict__ vals, int* __restrict__ counts, DevParams* prm) {
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  bool alive = false;
  double tv = 0.0;
  if (s < g.n_sites) {
    alive = !(dropped && dropped[s]);
    unsigned key = (unsigned)g.n_cells;
    if (alive) {
      long long k = 0;
      for (int a = 0; a < g.dim; ++a) {
        int c = (int)(pos[s * g.dim + a] * g.inv_cw[a]);
        c = c < 0 ? 0 : (c >= g.m[a] ? g.m[a] - 1 : c);
        k += c * g.cstride[a];
      }
      key = (unsigned)k;
      if (t) tv = t[s];
      atomicAdd(&counts[key], 1);
    }
    keys[s] = key;
    vals[s] = (int)s;
  }
  if (t) {
    unsigned long long kmin = alive ? dkey(tv) : ~0ull, kmax = alive ? dkey(tv) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
      kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    }
    if ((threadIdx.x & 31) == 0) {
      if (kmin != ~0ull) atomicMin(&prm->tmin_key, kmin);
      if (kmax != 0ull) atomicMax(&prm->tmax_key, kmax);
    }
  }
}

__global__ void gather_nd_kernel(GeoN g, const int* __restrict__ vals, const double* __restrict__ pos,
                                 const double* __restrict__ t, double* __restrict__ bx, double* __restrict__ bt,
                                 int* __restrict__ bidx, const int* __restrict__ cell_start, DevCounters* ctr) {
  const long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (p == 0) ctr->n_alive = (unsigned long long)cell_start[g.n_cells];  // dropped sites sort last
  if (p >= g.n_sites) return;
  const int s = vals[p];
  for (int a = 0; a < g.dim; ++a) bx[p + a * g.n_sites] = pos[(long long)s * g.dim + a];
  if (t) bt[p] = t[s];
  bidx[p] = s;
}

static int key_bits_nd(long long n_cells) {
  int b = 1;
  while ((1ll << b) <= n_cells) ++b;
  return b;
}

}  // namespace vnd

void fill_geo_nd(GeoN& g, int kind, int dim, int periodic, const long long* counts, const double* lengths,
                 double growth, long long n_sites, long long zb, long long ze) {
  std::memset(&g, 0, sizeof(g));
  g.kind = kind;
  g.dim = dim;
  g.periodic = periodic;
  g.growth = kind == kVoronoi ? 0.0 : growth;
  g.g_is_one = g.growth == 1.0;
  g.inv_growth_rn = g.growth > 0.0 ? 1.0 / g.growth : 0.0;
  g.n_sites = n_sites;
  g.zb = zb;
  g.ze = ze;
  g.vol_true = 1.0;
  g.suml2_true = 0.0;
  g.lmax = 0.0;
  for (int a = 0; a < dim; ++a) {
    g.n[a] = counts[a];
    g.L[a] = lengths[a];
    g.invL[a] = 1.0 / lengths[a];        // geometry.cpp:52
    g.sp[a] = lengths[a] / (double)counts[a];  // geometry.cpp:69
    g.halfL[a] = 0.5 * lengths[a];
    g.vol_true *= lengths[a];
    g.suml2_true += lengths[a] * lengths[a];
    g.lmax = std::fmax(g.lmax, lengths[a]);
  }
  // cell grid: about one site per cell, <= 2^26 cells
  double cw = std::pow(g.vol_true / (double)std::max<long long>(n_sites, 1), 1.0 / dim);
  for (int it = 0; it < 256; ++it) {
    long long cells = 1;
    for (int a = 0; a < dim; ++a) {
      g.m[a] = (int)std::min(1048576.0, std::max(1.0, std::floor(lengths[a] / cw)));
      cells = std::min<long long>(cells * g.m[a], 1ll << 40);
    }
    g.n_cells = cells;
    if (cells <= (1ll << 26)) break;
    cw *= 1.25;
  }
  long long st = 1;
  for (int a = 0; a < dim; ++a) {
    g.cw[a] = lengths[a] / g.m[a];
    g.inv_cw[a] = g.m[a] / lengths[a];
    g.cstride[a] = st;
    st *= g.m[a];
  }
  // block extents: 256 voxels per warp
  if (dim == 1) {
    g.E[0] = 256;
  } else if (dim == 2) {
    g.E[0] = g.E[1] = 16;
  } else {
    g.E[0] = g.E[1] = 4;
    // 16 lane groups over the higher axes: extents 4 x 4 (d = 4), 4 x 2 x 2, 2 x 2 x 2 x 2, then 1
    static const int kHi[4][4] = {{4, 4, 1, 1}, {4, 2, 2, 1}, {2, 2, 2, 2}, {2, 2, 2, 2}};
    const int row = std::min(dim - 4, 3);
    for (int a = 2; a < dim; ++a) g.E[a] = a - 2 < 4 ? kHi[row][a - 2] : 1;
  }
  long long nb = 1;
  for (int a = 0; a < dim; ++a) {
    const long long n = a == dim - 1 ? ze - zb : counts[a];
    g.nb[a] = (n + g.E[a] - 1) / g.E[a];
    nb *= g.nb[a];
  }
  g.n_blocks = nb;
  bool ok = g.growth == 0.0 || (g.growth >= 0x1p-64 && g.growth <= 0x1p64);
  for (int a = 0; a < dim; ++a) ok = ok && g.L[a] >= 0x1p-100 && g.L[a] <= 0x1p100 && g.sp[a] >= 0x1p-120;
  g.fast_arith = ok && std::getenv("VX_EXACT_CALLS") == nullptr;
}

int launch_prune_nd(const GeoN& g, const BinsN& bins, const double* pos, const double* t, const DevParams* prm,
                    uint8_t* dropped, cudaStream_t st) {
  const int T = 128;
  const unsigned nb = (unsigned)((g.n_sites + T - 1) / T);
  if (g.periodic) vnd::prune_nd_kernel<true><<<nb, T, 0, st>>>(g, bins, pos, t, prm, dropped);
  else vnd::prune_nd_kernel<false><<<nb, T, 0, st>>>(g, bins, pos, t, prm, dropped);
  return 1;
}

size_t bin_nd_tmp_bytes(long long n_sites, long long n_cells) { return bin_tmp_bytes(n_sites, n_cells); }

int launch_bin_nd(const GeoN& g, const double* pos, const double* t, const uint8_t* dropped, void* cub_tmp,
                  size_t cub_tmp_bytes, unsigned* keys_a, unsigned* keys_b, int* vals_a, int* vals_b, double* bx,
                  double* bt, int* bidx, int* cell_start, DevParams* prm, DevCounters* ctr, cudaStream_t st) {
  const int T = 256;
  const unsigned nb = (unsigned)((g.n_sites + T - 1) / T);
  cudaError_t e = cudaMemsetAsync(cell_start, 0, sizeof(int) * (size_t)(g.n_cells + 1), st);
  if (e != cudaSuccess) return -1000 - (int)e;
  vnd::keys_nd_kernel<<<nb, T, 0, st>>>(g, pos, t, dropped, keys_a, vals_a, cell_start, prm);
  size_t bytes = cub_tmp_bytes;
  e = cub::DeviceRadixSort::SortPairs(cub_tmp, bytes, keys_a, keys_b, vals_a, vals_b, (int)g.n_sites, 0,
                                      vnd::key_bits_nd(g.n_cells), st);
  if (e != cudaSuccess) return -1000 - (int)e;
  bytes = cub_tmp_bytes;
  e = cub::DeviceScan::ExclusiveSum(cub_tmp, bytes, cell_start, cell_start, (int)(g.n_cells + 1), st);
  if (e != cudaSuccess) return -1000 - (int)e;
  vnd::gather_nd_kernel<<<nb, T, 0, st>>>(g, vals_b, pos, t, bx, bt, bidx, cell_start, ctr);
  return 4 + 2 * ((vnd::key_bits_nd(g.n_cells) + 7) / 8);
}

int launch_ball_nd(const GeoN& g, const BinsN& bins, const DevParams* prm, int* labels, double* dist,
                   unsigned long long* hist, long long* unres, long long unres_cap, DevCounters* ctr,
                   long long nvs, cudaStream_t st) {
  const size_t sh = sizeof(vnd::BlockSmem);
  static std::atomic<unsigned long long> attr_done{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  const bool fa = g.kind != kVoronoi && g.fast_arith;
  const long long nbk = g.n_blocks;
  const unsigned gx = (unsigned)std::min<long long>(nbk, 1ll << 30);
  const dim3 grid(gx, (unsigned)((nbk + gx - 1) / gx));
#define VX_LND1(DT, K, P, F)                                                                                      \
  do {                                                                                                            \
    if (!(attr_done.load() & bit))                                                                                \
      cudaFuncSetAttribute(vnd::ballnd_kernel<DT, K, P, F>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh); \
    vnd::ballnd_kernel<DT, K, P, F><<<grid, 32, sh, st>>>(g, bins, prm, labels, dist, hist, unres, unres_cap, ctr, \
                                                          nbk);                                                   \
  } while (0)
#define VX_LND(K, P, F)                                                                                           \
  do {                                                                                                            \
    if (g.dim == 1) VX_LND1(1, K, P, F);                                                                          \
    else if (g.dim == 2) VX_LND1(2, K, P, F);                                                                     \
    else if (g.dim == 4) VX_LND1(4, K, P, F);                                                                     \
    else VX_LND1(0, K, P, F);                                                                                     \
  } while (0)
  switch (g.kind * 2 + (g.periodic ? 1 : 0)) {
    case 0: VX_LND(kVoronoi, false, false); break;
    case 1: VX_LND(kVoronoi, true, false); break;
    case 2: if (fa) VX_LND(kJohnsonMehl, false, true); else VX_LND(kJohnsonMehl, false, false); break;
    case 3: if (fa) VX_LND(kJohnsonMehl, true, true); else VX_LND(kJohnsonMehl, true, false); break;
    case 4: if (fa) VX_LND(kLaguerre, false, true); else VX_LND(kLaguerre, false, false); break;
    default: if (fa) VX_LND(kLaguerre, true, true); else VX_LND(kLaguerre, true, false); break;
  }
#undef VX_LND
#undef VX_LND1
  attr_done.fetch_or(bit);
  return 1;
}

int launch_unres_nd(const GeoN& g, const BinsN& bins, const DevParams* prm, long long* unres, long long unres_cap,
                    int* labels, double* dist, unsigned long long* hist, DevCounters* ctr, long long nvs,
                    cudaStream_t st) {
  const unsigned ub = (unsigned)sm_count() * 8;
#define VX_UND(K, P) \
  vnd::unres_nd_kernel<K, P><<<ub, vnd::kUT, 0, st>>>(g, bins, prm, unres, unres_cap, labels, dist, hist, ctr, nvs)
  switch (g.kind * 2 + (g.periodic ? 1 : 0)) {
    case 0: VX_UND(kVoronoi, false); break;
    case 1: VX_UND(kVoronoi, true); break;
    case 2: VX_UND(kJohnsonMehl, false); break;
    case 3: VX_UND(kJohnsonMehl, true); break;
    case 4: VX_UND(kLaguerre, false); break;
    default: VX_UND(kLaguerre, true); break;
  }
#undef VX_UND
  return 1;
}

}  // namespace vxb
