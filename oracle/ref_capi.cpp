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
// vxref_tessellate_timed() is the stock tessellate_fast with default options,
// timed around the call alone: bench.py's reference arm and cpu_baseline.
#include <omp.h>

#include <chrono>

#include <cstdint>
#include <cstring>
#include <exception>
#include <limits>
#include <string>
#include <vector>

#include "voxellate/cost.hpp"
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

// bench.py --impl reference / cpu_baseline: one stock tessellate_fast call
// (default FastOptions: prune on, model-optimal r0 / t0) timed around the call
// alone (steady_clock), so neither the input copies into the reference's
// SiteSet nor the output copies below are charged to it.  labels_out may be
// NULL; fingerprint_out (may be NULL) receives the SURVEY.md App. B label
// fingerprint of the result.
int vxref_tessellate_timed(int kind, int dim, int periodic, const int64_t* counts,
                           const double* lengths, int64_t n_sites, const double* positions,
                           const double* times, double growth, int threads, uint32_t* labels_out,
                           double* seconds_out, uint64_t* fingerprint_out, double* param_out) {
  return guarded([&] {
    if (threads > 0) omp_set_num_threads(threads);
    const VoxelGrid grid = make_grid(dim, periodic, counts, lengths);
    const SiteSet sites = make_sites(kind, dim, n_sites, positions, times, growth);
    const auto t0 = std::chrono::steady_clock::now();
    TessResult r = tessellate_fast(sites, grid, FastOptions{});
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds_out) *seconds_out = std::chrono::duration<double>(t1 - t0).count();
    if (param_out) *param_out = r.param;
    const std::vector<uint32_t>& lab = r.labels.labels;
    if (labels_out) std::memcpy(labels_out, lab.data(), lab.size() * sizeof(uint32_t));
    if (fingerprint_out) {
      uint64_t h = 1469598103934665603ull;
      for (uint32_t l : lab) {
        h ^= l;
        h *= 1099511628211ull;
      }
      *fingerprint_out = h;
    }
  });
}

// scan_ball / ball_voxels (tessellate.hpp:62-68): writes up to cap voxel
// indices in visit order; returns the count (>= 0) or -1 on error.
int64_t vxref_ball_voxels(int dim, int periodic, const int64_t* counts, const double* lengths,
                          const double* center, double radius, int64_t* out, int64_t cap) {
  int64_t n = -1;
  guarded([&] {
    const VoxelGrid grid = make_grid(dim, periodic, counts, lengths);
    const std::vector<int64_t> v = ball_voxels(Point(center, center + dim), radius, grid);
    for (size_t i = 0; i < v.size() && (int64_t)i < cap; ++i) out[i] = v[i];
    n = (int64_t)v.size();
  });
  return n;
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
