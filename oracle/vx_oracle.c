/* TEST INFRASTRUCTURE ONLY -- see vx_oracle.h.  Plain-C restatement of the
 * reference arithmetic.  Compiled with -ffp-contract=off and no -march so that,
 * like the reference build, no FMA is contracted.       */
#include "vx_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- std::mt19937_64 (C++ [rand.eng.mers], parameters of mt19937_64) ---- */
#define NN 312
#define MM 156
#define MATRIX_A 0xB5026F5AA96619E9ULL
#define UM 0xFFFFFFFF80000000ULL
#define LM 0x7FFFFFFFULL

void vxo_mt64_seed(vxo_mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < NN; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->mti = NN;
}

uint64_t vxo_mt64_next(vxo_mt64* g) {
  static const uint64_t mag01[2] = {0ULL, MATRIX_A};
  uint64_t x;
  if (g->mti >= NN) {
    int i;
    for (i = 0; i < NN - MM; ++i) {
      x = (g->mt[i] & UM) | (g->mt[i + 1] & LM);
      g->mt[i] = g->mt[i + MM] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    }
    for (; i < NN - 1; ++i) {
      x = (g->mt[i] & UM) | (g->mt[i + 1] & LM);
      g->mt[i] = g->mt[i + (MM - NN)] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    }
    x = (g->mt[NN - 1] & UM) | (g->mt[0] & LM);
    g->mt[NN - 1] = g->mt[MM - 1] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    g->mti = 0;
  }
  x = g->mt[g->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* uniform01, sites.cpp:20-22 */
static double u01(vxo_mt64* g) { return (double)(vxo_mt64_next(g) >> 11) * 0x1.0p-53; }

/* sites.cpp:61-85: per site d coordinates (exact 0 redrawn), then a time. */
void vxo_generate_uniform_sites(int dim, const double* lengths, int64_t n_sites, int kind,
                                double horizon, uint64_t seed, double* pos, double* times) {
  vxo_mt64 g;
  vxo_mt64_seed(&g, seed);
  for (int64_t s = 0; s < n_sites; ++s) {
    for (int i = 0; i < dim; ++i) {
      double u = u01(&g);
      while (u == 0.0) u = u01(&g);
      pos[s * dim + i] = u * lengths[i];
    }
    if (kind != 0) times[s] = u01(&g) * horizon;
  }
}

/* x,y,z = u01 (0 redrawn); a = u01 (0 redrawn), b = u01;
 * z = sqrt(-2 ln a) cos(2 pi b); r = m exp(sigma z - sigma^2/2).        */
void vxo_generate_lognormal_spheres(int64_t n, double m, double sigma, uint64_t seed,
                                    double* pos, double* radii) {
  vxo_mt64 g;
  vxo_mt64_seed(&g, seed);
  const double two_pi = 2.0 * 3.14159265358979323846;
  for (int64_t s = 0; s < n; ++s) {
    for (int i = 0; i < 3; ++i) {
      double u = u01(&g);
      while (u == 0.0) u = u01(&g);
      pos[s * 3 + i] = u;
    }
    double a = u01(&g);
    while (a == 0.0) a = u01(&g);
    const double b = u01(&g);
    const double z = sqrt(-2.0 * log(a)) * cos(two_pi * b);
    radii[s] = m * exp(sigma * z - 0.5 * sigma * sigma);
  }
}

/* sites.cpp:98-102 */
void vxo_spheres_to_timed(int64_t n, const double* radii, double growth, double* times) {
  for (int64_t s = 0; s < n; ++s) times[s] = -(radii[s] * radii[s]) / growth;
}

/* geometry.hpp:80-89: N(x) = floor(x + 1/2); wrap = u - N(u * invL) * L */
static inline double wrap_delta(double u, double L, double invL) {
  return u - floor(u * invL + 0.5) * L;
}

/* geometry.hpp:128-135 */
static inline double proximity(int kind, double dsq, double growth, double ts) {
  if (kind == 1) return sqrt(dsq) / growth + ts;
  if (kind == 2) return dsq / growth + ts;
  return dsq;
}

void vxo_brute(int kind, int dim, int periodic, const int64_t* counts, const double* lengths,
               int64_t n_sites, const double* pos, const double* times, double growth,
               int64_t lin_begin, int64_t lin_end, uint32_t* labels_out, double* dist_out) {
  double spacing[16], invL[16];
  for (int i = 0; i < dim; ++i) {
    spacing[i] = lengths[i] / (double)counts[i]; /* geometry.cpp:69 */
    invL[i] = 1.0 / lengths[i];                  /* geometry.cpp:52 */
  }
#pragma omp parallel for schedule(static)
  for (int64_t lin = lin_begin; lin < lin_end; ++lin) {
    double x[16];
    int64_t rem = lin;
    for (int i = 0; i < dim; ++i) { /* VoxelGrid::decompose + center, geometry.hpp:58-77 */
      const int64_t k = rem % counts[i];
      rem /= counts[i];
      x[i] = ((double)k + 0.5) * spacing[i];
    }
    double best = INFINITY;
    uint32_t best_label = 0xFFFFFFFFu;
    for (int64_t s = 0; s < n_sites; ++s) {
      const double* b = pos + s * dim;
      double acc = 0.0; /* fold from the last axis down, geometry.hpp:106-123 */
      for (int i = dim - 1; i >= 0; --i) {
        double w = b[i] - x[i];
        if (periodic) w = wrap_delta(w, lengths[i], invL[i]);
        acc += w * w;
      }
      const double prox = proximity(kind, acc, growth, kind ? times[s] : 0.0);
      if (prox < best) { /* strict <, ascending s: lowest index wins ties */
        best = prox;
        best_label = (uint32_t)s;
      }
    }
    labels_out[lin - lin_begin] = best_label;
    if (dist_out) dist_out[lin - lin_begin] = kind == 0 ? sqrt(best) : best;
  }
}

/* sites.cpp:27-37 */
static double axis_min_sq_diff(double a, double b, double length, int periodic) {
  if (periodic) {
    const double half = 0.5 * length;
    const double w = wrap_delta((b - a) + half, length, 1.0 / length);
    return w * w - half * half;
  }
  const double delta = b - a;
  const double at0 = delta * (-a - b);
  const double atL = delta * (2.0 * length - a - b);
  return at0 < atL ? at0 : atL;
}

int64_t vxo_prune(int kind, int dim, int periodic, const double* lengths, int64_t n,
                  const double* pos, const double* times, double growth, uint8_t* dropped) {
  double invL[16];
  for (int i = 0; i < dim; ++i) invL[i] = 1.0 / lengths[i];
  memset(dropped, 0, (size_t)n);
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t s = 0; s < n; ++s) {
    const double* xs = pos + s * dim;
    const double ts = times[s];
    for (int64_t o = 0; o < n; ++o) {
      if (o == s) continue;
      const double* xo = pos + o * dim;
      if (kind == 1) {
        double acc = 0.0; /* l_periodic_distance_sq(xs, xo): a = xs, b = xo */
        for (int i = dim - 1; i >= 0; --i) {
          double w = xo[i] - xs[i];
          if (periodic) w = wrap_delta(w, lengths[i], invL[i]);
          acc += w * w;
        }
        const double reach = sqrt(acc) / growth + times[o];
        if (reach < ts || (reach == ts && o < s)) {
          dropped[s] = 1;
          break;
        }
      } else {
        double margin = growth * (ts - times[o]);
        for (int i = 0; i < dim; ++i) margin += axis_min_sq_diff(xs[i], xo[i], lengths[i], periodic);
        if (margin > 0.0 || (margin == 0.0 && o < s)) {
          dropped[s] = 1;
          break;
        }
      }
    }
  }
  int64_t removed = 0;
  for (int64_t s = 0; s < n; ++s) removed += dropped[s];
  return removed;
}

/* cost.cpp:15-39 */
double vxo_optimal_r0(int64_t n_sites, int dim, const double* lengths) {
  double V = 1.0;
  for (int i = 0; i < dim; ++i) V *= lengths[i];
  const double ns = (double)n_sites;
  const double v0 = V * (-expm1(-log(ns) / (ns - 1.0)));
  const double unit = pow(M_PI, 0.5 * dim) / tgamma(0.5 * dim + 1.0);
  return pow(v0 / unit, 1.0 / dim);
}

uint64_t vxo_fingerprint_u32(const uint32_t* labels, int64_t n) {
  uint64_t h = 1469598103934665603ULL;
  for (int64_t i = 0; i < n; ++i) {
    h ^= labels[i];
    h *= 1099511628211ULL;
  }
  return h;
}

/* libstdc++ 13 uniform_int_distribution::operator() for a 64-bit URBG:
 * Lemire's nearly-divisionless draw in 128-bit (uniform_int_dist.h:257-281). */
void vxo_sample_indices(int64_t nv, int64_t sample, uint64_t seed, int64_t* out) {
  vxo_mt64 g;
  vxo_mt64_seed(&g, seed);
  const uint64_t range = (uint64_t)(nv - 1) + 1; /* __uerange */
  for (int64_t i = 0; i < sample; ++i) {
    unsigned __int128 product = (unsigned __int128)vxo_mt64_next(&g) * range;
    uint64_t low = (uint64_t)product;
    if (low < range) {
      const uint64_t threshold = (0 - range) % range;
      while (low < threshold) {
        product = (unsigned __int128)vxo_mt64_next(&g) * range;
        low = (uint64_t)product;
      }
    }
    out[i] = (int64_t)(product >> 64);
  }
}
