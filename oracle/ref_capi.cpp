// TEST INFRASTRUCTURE ONLY -- a C wrapper over the *reference* library
// (/root/reference/proj, compiled from its own sources by oracle/Makefile into
// oracle/_ref/).  Used by tests/ (golden fixtures, parity), by
// __graft_entry__.smoke() as a checker, and by bench.py's cpu_baseline /
// --impl reference arm.  Never linked into or called by the product path.
//
// Every entry point forwards to the reference's public C++ API:
//   tessellate_fast / tessellate_brute   include/voxellate/tessellate.hpp:47,59-60
//   prune_ineffective_sites              include/voxellate/sites.hpp:69
//   generate_uniform_sites               include/voxellate/sites.hpp:48-49
//   optimal_v0 / radius_from_volume      include/voxellate/cost.hpp:13,28
//   search_optimal_t0                    include/voxellate/cost.hpp:51
//   validate_partition                   include/voxellate/tessellate.hpp:81-84
//   write/read_label_image, write/read_distance_image
//                                        include/voxellate/image_io.hpp:24-29
//                                        (only when built with VXREF_IMAGE_IO)
// vxref_slab_sample() re-drives the reference's own step-1 window scan
// (detail::for_each_window_voxel, ball_scan.hpp:55-124) and step-2 full scan
// for one z-slab, with the reference's param choice, so that bench.py can
// time a bounded sample of a 10^9-voxel run.
#include <omp.h>

#include <cstdint>
#include <cstring>
#include <exception>
#include <limits>
#include <string>
#include <vector>

#include "voxellate/cost.hpp"
#include "voxellate/detail/ball_scan.hpp"
#include "voxellate/geometry.hpp"
#include "voxellate/sites.hpp"
#include "voxellate/tessellate.hpp"
#ifdef VXREF_IMAGE_IO
#include "voxellate/image_io.hpp"
#endif

using namespace voxellate;

namespace {

thread_local std::string g_err;

Domain make_domain(int dim, int periodic, const double* lengths) {
  return Domain(std::vector<double>(lengths, lengths + dim),
                periodic ? Boundary::Periodic : Boundary::NonPeriodic);
}

VoxelGrid make_grid(int dim, int periodic, const int64_t* counts, const double* lengths) {
  return VoxelGrid(std::vector<std::int64_t>(counts, counts + dim),
                   make_domain(dim, periodic, lengths));
}

SiteSet make_sites(int kind, int dim, int64_t n, const double* pos, const double* times,
                   double growth) {
  SiteSet s;
  s.kind = static_cast<Kind>(kind);
  s.dim = dim;
  s.positions.assign(pos, pos + n * dim);
  if (s.kind != Kind::Voronoi) s.times.assign(times, times + n);
  s.growth = s.kind == Kind::Voronoi ? 0.0 : growth;
  return s;
}

template <class Fn>
int guarded(Fn fn) {
  try {
    fn();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

}  // namespace

extern "C" {

const char* vxref_last_error(void) { return g_err.c_str(); }

int vxref_max_threads(void) { return omp_get_max_threads(); }

// engine: 0 = tessellate_fast, 1 = tessellate_brute.  threads <= 0 keeps the
// OpenMP default.  distances_out / evals_out / param_out may be NULL.
int vxref_tessellate(int engine, int kind, int dim, int periodic, const int64_t* counts,
                     const double* lengths, int64_t n_sites, const double* positions,
                     const double* times, double growth, int prune, int has_override,
                     double override_param, int threads, uint32_t* labels_out,
                     double* distances_out, double* param_out, uint64_t* evals_out) {
  return guarded([&] {
    if (threads > 0) omp_set_num_threads(threads);
    const VoxelGrid grid = make_grid(dim, periodic, counts, lengths);
    const SiteSet sites = make_sites(kind, dim, n_sites, positions, times, growth);
    TessResult r;
    if (engine == 1) {
      r = tessellate_brute(sites, grid);
    } else {
      FastOptions opt;
      opt.prune = prune != 0;
      if (has_override) opt.override_param = override_param;
      r = tessellate_fast(sites, grid, opt);
    }
    std::memcpy(labels_out, r.labels.labels.data(), r.labels.labels.size() * sizeof(uint32_t));
    if (distances_out)
      std::memcpy(distances_out, r.distances.values.data(),
                  r.distances.values.size() * sizeof(double));
    if (param_out) *param_out = r.param;
    if (evals_out) {
      evals_out[0] = r.counters.step1_evals;
      evals_out[1] = r.counters.step2_evals;
    }
  });
}

// Returns the number of removed sites (>= 0) or -1 on error; dropped_out[s]=1
// for removed sites.
int64_t vxref_prune(int kind, int dim, int periodic, const double* lengths, int64_t n_sites,
                    const double* positions, const double* times, double growth,
                    uint8_t* dropped_out) {
  int64_t removed = -1;
  const int rc = guarded([&] {
    const Domain box = make_domain(dim, periodic, lengths);
    const SiteSet sites = make_sites(kind, dim, n_sites, positions, times, growth);
    const PruneResult pr = prune_ineffective_sites(sites, box);
    std::memset(dropped_out, 0, static_cast<size_t>(n_sites));
    for (int64_t s : pr.removed) dropped_out[s] = 1;
    removed = static_cast<int64_t>(pr.removed.size());
  });
  return rc == 0 ? removed : -1;
}

int vxref_generate_uniform_sites(int dim, const double* lengths, int64_t n_sites, int kind,
                                 double growth, double horizon, uint64_t seed,
                                 double* positions_out, double* times_out) {
  return guarded([&] {
    const Domain box = make_domain(dim, 1, lengths);
    const SiteSet s =
        generate_uniform_sites(box, n_sites, static_cast<Kind>(kind), growth, horizon, seed);
    std::memcpy(positions_out, s.positions.data(), s.positions.size() * sizeof(double));
    if (times_out && !s.times.empty())
      std::memcpy(times_out, s.times.data(), s.times.size() * sizeof(double));
  });
}

int vxref_spheres_to_timed(int dim, int64_t n, const double* positions, const double* radii,
                           double growth, double* times_out) {
  return guarded([&] {
    LaguerreSpheres sp;
    sp.dim = dim;
    sp.positions.assign(positions, positions + n * dim);
    sp.radii.assign(radii, radii + n);
    const SiteSet s = spheres_to_timed_sites(sp, growth);
    std::memcpy(times_out, s.times.data(), s.times.size() * sizeof(double));
  });
}

double vxref_optimal_r0(int64_t n_sites, int dim, const double* lengths, int periodic) {
  const Domain box = make_domain(dim, periodic, lengths);
  return radius_from_volume(optimal_v0(n_sites, box.volume()), dim);
}

double vxref_search_optimal_t0(int kind, int dim, int periodic, const int64_t* counts,
                               const double* lengths, int64_t n_sites, const double* positions,
                               const double* times, double growth) {
  double t0 = std::numeric_limits<double>::quiet_NaN();
  guarded([&] {
    const VoxelGrid grid = make_grid(dim, periodic, counts, lengths);
    const SiteSet sites = make_sites(kind, dim, n_sites, positions, times, growth);
    t0 = search_optimal_t0(sites, grid);
  });
  return t0;
}

// report_out: [checked, label_mismatches, value_mismatches, n_examples, ex0..ex15]
int vxref_validate_partition(int kind, int dim, int periodic, const int64_t* counts,
                             const double* lengths, int64_t n_sites, const double* positions,
                             const double* times, double growth, const uint32_t* labels,
                             const double* distances, int64_t sample, uint64_t seed,
                             int64_t* report_out) {
  return guarded([&] {
    const VoxelGrid grid = make_grid(dim, periodic, counts, lengths);
    const SiteSet sites = make_sites(kind, dim, n_sites, positions, times, growth);
    LabelImage li;
    li.grid = grid;
    li.labels.assign(labels, labels + grid.voxel_count());
    DistanceImage di;
    if (distances) {
      di.grid = grid;
      di.values.assign(distances, distances + grid.voxel_count());
    }
    const ValidationReport rep =
        validate_partition(li, distances ? &di : nullptr, sites, sample, seed);
    report_out[0] = rep.voxels_checked;
    report_out[1] = rep.label_mismatches;
    report_out[2] = rep.value_mismatches;
    report_out[3] = static_cast<int64_t>(rep.examples.size());
    for (size_t i = 0; i < rep.examples.size() && i < 16; ++i) report_out[4 + i] = rep.examples[i];
  });
}

// Bounded CPU sample for bench.py: the reference's tessellate_fast work for
// the voxels of last-axis slab [z0, z1) only.  Same parameter choice
// (tessellate.cpp:217-260, incl. prune for timed kinds), same step-1 window
// scan with slab bounds (tessellate.cpp:103-144 / ball_scan.hpp), same
// unassigned-voxel full scan (tessellate.cpp:36-75) and Voronoi sqrt pass.
// labels_out holds nx*ny*(z1-z0) entries; labels are original site indices.
int vxref_slab_sample(int kind, int dim, int periodic, const int64_t* counts,
                      const double* lengths, int64_t n_sites, const double* positions,
                      const double* times, double growth, int64_t z0, int64_t z1, int threads,
                      uint32_t* labels_out, double* param_out) {
  return guarded([&] {
    if (threads > 0) omp_set_num_threads(threads);
    const VoxelGrid grid = make_grid(dim, periodic, counts, lengths);
    const SiteSet all = make_sites(kind, dim, n_sites, positions, times, growth);
    all.validate(grid.domain);
    const SiteSet* work = &all;
    SiteSet pruned;
    std::vector<int64_t> kept;
    if (all.timed()) {
      PruneResult pr = prune_ineffective_sites(all, grid.domain);
      if (!pr.removed.empty()) {
        pruned = std::move(pr.sites);
        kept = std::move(pr.kept);
        work = &pruned;
      }
    }
    const int64_t ns = work->count();
    double param, cutoff;
    std::vector<double> radii(static_cast<size_t>(ns));
    if (all.kind == Kind::Voronoi) {
      if (ns == 1) {  // cover_radius, tessellate.cpp:25-30
        double s = 0.0;
        for (double L : grid.domain.lengths) s += L * L;
        param = grid.domain.periodic() ? 0.5 * std::sqrt(s) : std::sqrt(s);
      } else {
        param = radius_from_volume(optimal_v0(ns, grid.domain.volume()), grid.dim());
      }
      cutoff = param * param;
      std::fill(radii.begin(), radii.end(), param);
    } else {
      param = ns == 1 ? t0_bracket(*work, grid.domain).hi : search_optimal_t0(*work, grid);
      cutoff = param;
      for (int64_t s = 0; s < ns; ++s) {
        const double dt = param - work->times[s];
        radii[s] = dt < 0.0 ? -1.0
                            : (all.kind == Kind::JohnsonMehl ? work->growth * dt
                                                             : std::sqrt(work->growth * dt));
      }
    }
    if (param_out) *param_out = param;

    const int d = grid.dim();
    const int64_t plane = grid.voxel_count() / grid.counts[d - 1];
    const int64_t base = z0 * plane;
    const int64_t nvs = (z1 - z0) * plane;
    std::vector<uint32_t> lab(static_cast<size_t>(nvs), kUnassignedLabel);
    std::vector<double> val(static_cast<size_t>(nvs), std::numeric_limits<double>::infinity());
    const double G = work->growth;
    const Kind K = all.kind;

#pragma omp parallel
    {
      const int tid = omp_get_thread_num();
      const int nth = omp_get_num_threads();
      const int64_t lo = z0 + (z1 - z0) * tid / nth;
      const int64_t hi = z0 + (z1 - z0) * (tid + 1) / nth;
      if (lo < hi) {
        detail::ScanScratch scratch;
        for (int64_t s = 0; s < ns; ++s) {
          if (radii[s] < 0.0) continue;
          const double ts = K == Kind::Voronoi ? 0.0 : work->times[s];
          const uint32_t l = static_cast<uint32_t>(s);
          detail::for_each_window_voxel(work->pos(s), radii[s], grid, lo, hi, scratch,
                                        [&](int64_t lin, double dsq) {
                                          const double prox = proximity_from_dsq(K, dsq, G, ts);
                                          if (prox <= cutoff && prox < val[lin - base]) {
                                            val[lin - base] = prox;
                                            lab[lin - base] = l;
                                          }
                                        });
        }
      }
    }
    const double* L = grid.domain.lengths.data();
    const double* iL = grid.domain.inv_lengths.data();
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nvs; ++i) {
      if (lab[i] != kUnassignedLabel) continue;
      int64_t idx[kMaxDim];
      double x[kMaxDim];
      grid.decompose(base + i, idx);
      grid.center(idx, x);
      double best = std::numeric_limits<double>::infinity();
      uint32_t bl = kUnassignedLabel;
      for (int64_t s = 0; s < ns; ++s) {
        const double dsq = grid.domain.periodic() ? l_periodic_distance_sq(x, work->pos(s), d, L, iL)
                                                  : euclidean_distance_sq(x, work->pos(s), d);
        const double prox = proximity_from_dsq(K, dsq, G, K == Kind::Voronoi ? 0.0 : work->times[s]);
        if (prox < best) {
          best = prox;
          bl = static_cast<uint32_t>(s);
        }
      }
      lab[i] = bl;
      val[i] = best;
    }
    if (K == Kind::Voronoi) {
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < nvs; ++i) val[i] = std::sqrt(val[i]);
    }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nvs; ++i)
      labels_out[i] = kept.empty() ? lab[i] : static_cast<uint32_t>(kept[lab[i]]);
  });
}

#ifdef VXREF_IMAGE_IO
int vxref_have_image_io(void) { return 1; }

// type 0: labels (u32 payload), 1: distances (f64 payload)
int vxref_write_image(const char* path, int type, int dim, int periodic, const int64_t* counts,
                      const double* lengths, int kind, int64_t n_sites, int64_t seed,
                      const void* data) {
  return guarded([&] {
    ImageMeta meta;
    meta.kind = static_cast<Kind>(kind);
    meta.n_sites = n_sites;
    meta.seed = seed;
    const VoxelGrid grid = make_grid(dim, periodic, counts, lengths);
    const int64_t nv = grid.voxel_count();
    if (type == 0) {
      LabelImage im;
      im.grid = grid;
      const auto* u = static_cast<const std::uint32_t*>(data);
      im.labels.assign(u, u + nv);
      write_label_image(path, im, meta);
    } else {
      DistanceImage im;
      im.grid = grid;
      const auto* v = static_cast<const double*>(data);
      im.values.assign(v, v + nv);
      write_distance_image(path, im, meta);
    }
  });
}

// header_out: [dim, periodic, kind, n_sites, seed, format_version], dims_out /
// lengths_out: dim entries each (cap 16); data_out: voxel_count elements
int vxref_read_image(const char* path, int type, int64_t* header_out, int64_t* dims_out,
                     double* lengths_out, void* data_out, int64_t cap_voxels) {
  return guarded([&] {
    ImageMeta meta;
    const VoxelGrid* g = nullptr;
    LabelImage li;
    DistanceImage di;
    if (type == 0) {
      li = read_label_image(path, &meta);
      g = &li.grid;
    } else {
      di = read_distance_image(path, &meta);
      g = &di.grid;
    }
    header_out[0] = g->dim();
    header_out[1] = g->domain.boundary == Boundary::Periodic;
    header_out[2] = static_cast<int64_t>(meta.kind);
    header_out[3] = meta.n_sites;
    header_out[4] = meta.seed;
    header_out[5] = meta.format_version;
    for (int i = 0; i < g->dim() && i < 16; ++i) {
      dims_out[i] = g->counts[i];
      lengths_out[i] = g->domain.lengths[i];
    }
    const int64_t nv = g->voxel_count();
    if (data_out && nv <= cap_voxels) {
      if (type == 0) std::memcpy(data_out, li.labels.data(), sizeof(std::uint32_t) * nv);
      else std::memcpy(data_out, di.values.data(), sizeof(double) * nv);
    }
  });
}
#else
int vxref_have_image_io(void) { return 0; }
#endif

}  // extern "C"
