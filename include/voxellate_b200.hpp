// voxellate_b200.hpp -- the reference's C++ engine API over the C-ABI.
//
// Header-only shim with the signatures of the reference's
//   voxellate::tessellate_fast / tessellate_brute   (include/voxellate/tessellate.hpp:47,59-60)
//   voxellate::prune_ineffective_sites              (include/voxellate/sites.hpp:69)
//   voxellate::validate_partition                   (include/voxellate/tessellate.hpp:81-84)
//   voxellate::generate_uniform_sites               (include/voxellate/sites.hpp:48-49)
//   voxellate::spheres_to_timed_sites               (include/voxellate/sites.hpp:52)
//   voxellate::scan_ball / ball_voxels              (include/voxellate/tessellate.hpp:62-68)
// and value types with the same fields (Domain, VoxelGrid, SiteSet, FastOptions,
// TessResult, ...), in namespace vxb200 so it can coexist with the reference in
// one program.  Errors become the reference's exceptions: VX_EINVAL ->
// std::invalid_argument (same message), anything else -> std::runtime_error.
//
// A caller of the reference switches with
//     namespace voxellate = vxb200;   // and link libvoxellate_b200.so
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "voxellate_b200.h"

namespace vxb200 {

enum class Boundary { Periodic, NonPeriodic };
enum class Kind { Voronoi, JohnsonMehl, Laguerre };
inline constexpr int kMaxDim = VX_MAX_DIM;
inline constexpr std::uint32_t kUnassignedLabel = 0xFFFFFFFFu;

namespace detail {
inline void check(int rc) {
  if (rc == VX_OK) return;
  const std::string msg = vx_last_error();
  if (rc == VX_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}
}  // namespace detail

struct Domain {
  std::vector<double> lengths;
  std::vector<double> inv_lengths;
  Boundary boundary = Boundary::Periodic;
  Domain() = default;
  Domain(std::vector<double> l, Boundary b) : lengths(std::move(l)), boundary(b) {
    if (lengths.empty()) throw std::invalid_argument("domain must have at least one axis");
    if ((int)lengths.size() > kMaxDim)
      throw std::invalid_argument("domain dimension exceeds supported maximum (16)");
    for (double L : lengths) {
      if (!(std::isfinite(L) && L > 0.0)) throw std::invalid_argument("domain lengths must be positive");
      inv_lengths.push_back(1.0 / L);
    }
  }
  int dim() const { return (int)lengths.size(); }
  double volume() const {
    double v = 1.0;
    for (double L : lengths) v *= L;
    return v;
  }
  bool periodic() const { return boundary == Boundary::Periodic; }
};

struct VoxelGrid {
  std::vector<std::int64_t> counts;
  Domain domain;
  std::vector<double> spacing;
  VoxelGrid() = default;
  VoxelGrid(std::vector<std::int64_t> c, Domain d) : counts(std::move(c)), domain(std::move(d)) {
    if ((int)counts.size() != domain.dim())
      throw std::invalid_argument("grid counts must match domain dimension");
    for (auto n : counts)
      if (n < 1) throw std::invalid_argument("voxel counts must be positive");
    for (int i = 0; i < dim(); ++i) spacing.push_back(domain.lengths[i] / (double)counts[i]);
  }
  int dim() const { return (int)counts.size(); }
  std::int64_t voxel_count() const {
    std::int64_t n = 1;
    for (auto c : counts) n *= c;
    return n;
  }
  double center_coord(int axis, std::int64_t k) const { return ((double)k + 0.5) * spacing[axis]; }
};

struct SiteSet {
  Kind kind = Kind::Voronoi;
  int dim = 0;
  std::vector<double> positions;
  std::vector<double> times;
  double growth = 0.0;
  std::int64_t count() const { return dim == 0 ? 0 : (std::int64_t)positions.size() / dim; }
  bool timed() const { return kind != Kind::Voronoi; }
  const double* pos(std::int64_t s) const { return positions.data() + s * dim; }
};

struct LabelImage {
  VoxelGrid grid;
  std::vector<std::uint32_t> labels;
};
struct DistanceImage {
  VoxelGrid grid;
  std::vector<double> values;
};
// Boundary note -- two TessResult fields report THIS engine's numbers, not
// the reference's (labels and distances never depend on them):
//  * counters: step1_evals = exact evaluations of the ball phase (per voxel,
//    the candidates of its octant / sub-brick list), step2_evals = those of
//    the unresolved-voxel search; the reference counts its window scan and
//    all-sites step 2 (tessellate.cpp:264-270);
//  * param: for Voronoi the reference's r0 bit for bit; for the timed kinds
//    the t0 this engine's device cost scan chose (the reference reports its
//    golden-section search_optimal_t0, cost.cpp:98-146).  An explicit
//    FastOptions::override_param is used and reported as given by both.
struct EvalCounters {  // this engine's counts: ball phase / shell phase evaluations
  std::uint64_t step1_evals = 0;
  std::uint64_t step2_evals = 0;
  std::uint64_t total() const { return step1_evals + step2_evals; }
};
struct TessResult {
  LabelImage labels;
  DistanceImage distances;
  EvalCounters counters;
  double param = std::numeric_limits<double>::quiet_NaN();
};
struct FastOptions {
  std::optional<double> override_param;
  bool prune = true;
  int n_gpus = 1;  // extension: split the call over this many devices
};
struct LaguerreSpheres {  // sites.hpp:34-45
  int dim = 0;
  std::vector<double> positions;  // count() * dim
  std::vector<double> radii;
  std::int64_t count() const { return dim == 0 ? 0 : (std::int64_t)positions.size() / dim; }
};
struct PruneResult {
  SiteSet sites;
  std::vector<std::int64_t> removed;
  std::vector<std::int64_t> kept;
};
struct ValidationReport {
  std::int64_t voxels_checked = 0;
  std::int64_t label_mismatches = 0;
  std::int64_t value_mismatches = 0;
  std::vector<std::int64_t> examples;
  bool ok() const { return label_mismatches == 0 && value_mismatches == 0; }
};

namespace detail {
inline vx_problem problem(const SiteSet& s, const VoxelGrid& g) {
  if (s.dim != g.dim()) throw std::invalid_argument("site dimension does not match the domain");
  if (s.count() < 1) throw std::invalid_argument("site set must contain at least one site");
  if ((std::int64_t)s.positions.size() != s.count() * s.dim)
    throw std::invalid_argument("site position array has inconsistent size");
  if (s.timed() && (std::int64_t)s.times.size() != s.count())
    throw std::invalid_argument("timed site set must carry one birth time per site");
  vx_problem P{};
  P.kind = (int)s.kind;
  P.dim = g.dim();
  P.periodic = g.domain.periodic() ? 1 : 0;
  for (int i = 0; i < g.dim(); ++i) {
    P.counts[i] = g.counts[i];
    P.lengths[i] = g.domain.lengths[i];
  }
  P.n_sites = s.count();
  P.positions = s.positions.data();
  P.times = s.timed() ? s.times.data() : nullptr;
  P.growth = s.timed() ? s.growth : 0.0;
  return P;
}

inline TessResult run(const SiteSet& s, const VoxelGrid& g, const FastOptions* o, bool brute) {
  const vx_problem P = problem(s, g);
  vx_options O;
  vx_options_init(&O);
  if (o) {
    O.prune = o->prune ? 1 : 0;
    O.n_gpus = o->n_gpus;
    if (o->override_param) {
      O.has_override = 1;
      O.override_param = *o->override_param;
    }
  }
  TessResult r;
  r.labels.grid = g;
  r.distances.grid = g;
  r.labels.labels.resize((size_t)g.voxel_count());
  r.distances.values.resize((size_t)g.voxel_count());
  O.distances_out = r.distances.values.data();
  vx_stats st{};
  int32_t* out = reinterpret_cast<int32_t*>(r.labels.labels.data());
  check(brute ? vx_tessellate_brute(nullptr, &P, &O, out, &st) : vx_tessellate(nullptr, &P, &O, out, &st));
  r.counters.step1_evals = st.ball_evals;
  r.counters.step2_evals = st.shell_evals;
  if (!brute) r.param = st.param;
  return r;
}
}  // namespace detail

// tessellate.hpp:59-60
inline TessResult tessellate_fast(const SiteSet& sites, const VoxelGrid& grid,
                                  const FastOptions& options = {}) {
  return detail::run(sites, grid, &options, false);
}
// tessellate.hpp:47
inline TessResult tessellate_brute(const SiteSet& sites, const VoxelGrid& grid) {
  return detail::run(sites, grid, nullptr, true);
}

// sites.hpp:69
inline PruneResult prune_ineffective_sites(const SiteSet& sites, const Domain& domain) {
  if (!sites.timed()) throw std::invalid_argument("pruning applies to timed tessellations only");
  VoxelGrid g(std::vector<std::int64_t>(domain.dim(), 1), domain);
  const vx_problem P = detail::problem(sites, g);
  std::vector<std::uint8_t> dropped((size_t)sites.count());
  std::int64_t removed = 0;
  detail::check(vx_prune(nullptr, &P, dropped.data(), &removed));
  PruneResult out;
  out.sites.kind = sites.kind;
  out.sites.dim = sites.dim;
  out.sites.growth = sites.growth;
  for (std::int64_t s = 0; s < sites.count(); ++s) {
    if (dropped[s]) {
      out.removed.push_back(s);
      continue;
    }
    out.kept.push_back(s);
    out.sites.positions.insert(out.sites.positions.end(), sites.pos(s), sites.pos(s) + sites.dim);
    out.sites.times.push_back(sites.times[s]);
  }
  return out;
}

// tessellate.hpp:81-84
inline ValidationReport validate_partition(const LabelImage& labels, const DistanceImage* distances,
                                           const SiteSet& sites, std::int64_t sample = 0,
                                           std::uint64_t seed = 0) {
  const vx_problem P = detail::problem(sites, labels.grid);
  if ((std::int64_t)labels.labels.size() != labels.grid.voxel_count())
    throw std::invalid_argument("label image size does not match its grid");
  vx_validation rep{};
  detail::check(vx_validate_partition(nullptr, &P, reinterpret_cast<const int32_t*>(labels.labels.data()),
                                      distances ? distances->values.data() : nullptr, sample, seed, &rep));
  ValidationReport r;
  r.voxels_checked = rep.voxels_checked;
  r.label_mismatches = rep.label_mismatches;
  r.value_mismatches = rep.value_mismatches;
  r.examples.assign(rep.examples, rep.examples + rep.n_examples);
  return r;
}

// sites.hpp:48-49
// t_s = -(r_s * r_s) / G, same checks and messages as sites.cpp:87-104
inline SiteSet spheres_to_timed_sites(const LaguerreSpheres& spheres, double growth) {
  if (!(growth > 0.0)) throw std::invalid_argument("growth rate G must be positive");
  if (spheres.count() < 1) throw std::invalid_argument("sphere set must contain at least one sphere");
  if ((std::int64_t)spheres.radii.size() != spheres.count())
    throw std::invalid_argument("sphere set must carry one radius per center");
  SiteSet out;
  out.kind = Kind::Laguerre;
  out.dim = spheres.dim;
  out.growth = growth;
  out.positions = spheres.positions;
  out.times.reserve(spheres.radii.size());
  for (double r : spheres.radii) {
    if (!(r >= 0.0)) throw std::invalid_argument("sphere radii must be nonnegative");
    out.times.push_back(-(r * r) / growth);
  }
  return out;
}

using Point = std::vector<double>;

// Visits every voxel whose centre lies within `radius` of `center`, once
// (tessellate.hpp:62-68): per axis the candidate indices of a conservative
// window ((c -/+ r(1 + 1e-9)) / h - 0.5, rounded outwards with a relative
// slack) and their squared residuals (periodic: wrapped), then an odometer
// over the axes -- last axis outermost, axis 0 innermost, i.e. ascending
// window order -- accumulating the squared terms from the last axis down to
// axis 0 (the reference's fold, geometry.hpp:106-123) and pruning partial
// sums beyond the inflated radius; a voxel is visited iff dsq <= radius^2.
// Host code: this is the reference's investigation-ball enumeration, not a
// step of the GPU pipeline (which gathers per voxel block instead).
template <class Visit>
inline void scan_ball(const Point& center, double radius, const VoxelGrid& grid, Visit&& visit) {
  const int d = grid.dim();
  if ((int)center.size() != d) throw std::invalid_argument("ball center dimension does not match the grid");
  if (!(std::isfinite(radius) && radius >= 0.0)) throw std::invalid_argument("ball radius must be nonnegative");
  const double rp = radius * (1.0 + 1e-9), r2p = rp * rp, r2 = radius * radius;
  const bool per = grid.domain.periodic();
  std::vector<std::vector<std::int64_t>> idx(d);
  std::vector<std::vector<double>> sq(d);
  std::vector<std::int64_t> stride(d);
  std::int64_t st = 1;
  for (int a = 0; a < d; ++a) {
    stride[a] = st;
    st *= grid.counts[a];
    const std::int64_t n = grid.counts[a];
    const double h = grid.spacing[a], L = grid.domain.lengths[a], iL = grid.domain.inv_lengths[a];
    const double lo_t = (center[a] - rp) / h - 0.5, hi_t = (center[a] + rp) / h - 0.5;
    const double slack = 1e-9 * (std::fabs(lo_t) + std::fabs(hi_t) + 1.0);
    const double klo = std::ceil(lo_t - slack), khi = std::floor(hi_t + slack);
    if (khi < klo) return;
    // separately rounded products (volatile: no FMA contraction whatever the
    // caller's compiler flags), as the reference build computes them
    auto mul = [](double x, double y) {
      volatile double r = x * y;
      return (double)r;
    };
    auto add = [&](std::int64_t k) {
      double w = center[a] - mul((double)k + 0.5, h);                      // geometry.hpp:58-60
      if (per) w = w - mul(std::floor(mul(w, iL) + 0.5), L);                // geometry.hpp:80-89
      idx[a].push_back(k);
      sq[a].push_back(mul(w, w));
    };
    if (per) {
      if (khi - klo + 1.0 >= (double)n) {
        for (std::int64_t k = 0; k < n; ++k) add(k);
      } else {
        for (std::int64_t k = (std::int64_t)klo; k <= (std::int64_t)khi; ++k) add(((k % n) + n) % n);
      }
    } else {
      const std::int64_t a0 = klo <= 0.0 ? 0 : (std::int64_t)std::min(klo, (double)n);
      const std::int64_t a1 = khi >= (double)(n - 1) ? n - 1 : (std::int64_t)std::max(khi, -1.0);
      for (std::int64_t k = a0; k <= a1; ++k) add(k);
    }
    if (idx[a].empty()) return;
  }
  // odometer: pos[a] walks idx[a]; acc[a] = sum of the terms of axes >= a
  std::vector<std::size_t> pos(d, 0);
  std::vector<double> acc(d + 1, 0.0);
  std::vector<std::int64_t> lin(d + 1, 0);
  int a = d - 1;
  while (true) {
    if (pos[a] < idx[a].size()) {
      const double s = acc[a + 1] + sq[a][pos[a]];
      const std::int64_t l = lin[a + 1] + idx[a][pos[a]] * stride[a];
      ++pos[a];
      if (!(s <= r2p)) continue;
      if (a == 0) {
        if (s <= r2) visit(l);
      } else {
        acc[a] = s;
        lin[a] = l;
        --a;
        pos[a] = 0;
      }
    } else {
      if (++a == d) return;
    }
  }
}

inline std::vector<std::int64_t> ball_voxels(const Point& center, double radius, const VoxelGrid& grid) {
  std::vector<std::int64_t> out;
  scan_ball(center, radius, grid, [&](std::int64_t l) { out.push_back(l); });
  return out;
}

inline SiteSet generate_uniform_sites(const Domain& domain, std::int64_t n_sites, Kind kind,
                                      double growth, double time_horizon, std::uint64_t seed) {
  SiteSet s;
  s.kind = kind;
  s.dim = domain.dim();
  s.growth = kind == Kind::Voronoi ? 0.0 : growth;
  s.positions.resize((size_t)(n_sites * s.dim));
  if (kind != Kind::Voronoi) s.times.resize((size_t)n_sites);
  detail::check(vx_generate_uniform_sites(s.dim, domain.lengths.data(), n_sites, (int)kind, growth,
                                          time_horizon, seed, s.positions.data(),
                                          kind == Kind::Voronoi ? nullptr : s.times.data()));
  return s;
}

// ---- on-disk images (row f2; reference include/voxellate/image_io.hpp) ----
struct ImageMeta {  // image_io.hpp:13-19
  int format_version = 1;
  std::string type;
  Kind kind = Kind::Voronoi;
  std::int64_t n_sites = 0;
  std::int64_t seed = -1;
};

namespace detail {
inline void write_image(const std::string& path, int type, const VoxelGrid& g, const ImageMeta& meta,
                        const void* data, std::size_t n) {
  if ((std::int64_t)n != g.voxel_count()) throw std::invalid_argument("image payload size disagrees with its grid");
  detail::check(vx_write_image(path.c_str(), type, g.dim(), g.counts.data(), g.domain.lengths.data(),
                               g.domain.periodic() ? 1 : 0, (int)meta.kind, meta.n_sites, meta.seed, data));
}
template <class T>
inline VoxelGrid read_image(const std::string& path, int type, std::vector<T>& data, ImageMeta* meta) {
  std::int64_t hdr[6], counts[kMaxDim];
  double lengths[kMaxDim];
  detail::check(vx_read_image(path.c_str(), type, hdr, counts, lengths, nullptr, 0));
  const int d = (int)hdr[0];
  VoxelGrid g(std::vector<std::int64_t>(counts, counts + d),
              Domain(std::vector<double>(lengths, lengths + d), hdr[1] ? Boundary::Periodic : Boundary::NonPeriodic));
  data.resize((std::size_t)g.voxel_count());
  detail::check(vx_read_image(path.c_str(), type, hdr, counts, lengths, data.data(), g.voxel_count()));
  if (meta) {
    meta->format_version = (int)hdr[5];
    meta->type = type == 0 ? "labels" : "distances";
    meta->kind = (Kind)hdr[2];
    meta->n_sites = hdr[3];
    meta->seed = hdr[4];
  }
  return g;
}
}  // namespace detail

inline void write_label_image(const std::string& path, const LabelImage& image, const ImageMeta& meta) {
  detail::write_image(path, 0, image.grid, meta, image.labels.data(), image.labels.size());
}
inline void write_distance_image(const std::string& path, const DistanceImage& image, const ImageMeta& meta) {
  detail::write_image(path, 1, image.grid, meta, image.values.data(), image.values.size());
}
inline LabelImage read_label_image(const std::string& path, ImageMeta* meta = nullptr) {
  LabelImage im;
  im.grid = detail::read_image(path, 0, im.labels, meta);
  return im;
}
inline DistanceImage read_distance_image(const std::string& path, ImageMeta* meta = nullptr) {
  DistanceImage im;
  im.grid = detail::read_image(path, 1, im.values, meta);
  return im;
}
// tessellate_fast straight to the reference's files, the image streamed out of
// device memory chunk by chunk (run.cpp:121-150 computes, then writes)
inline void tessellate_to_files(const SiteSet& sites, const VoxelGrid& grid, const std::string& label_path,
                                const std::string* distance_path = nullptr,
                                const FastOptions& options = FastOptions(), std::int64_t seed = -1) {
  vx_problem P = detail::problem(sites, grid);
  vx_options O;
  vx_options_init(&O);
  O.prune = options.prune ? 1 : 0;
  if (options.override_param) {
    O.has_override = 1;
    O.override_param = *options.override_param;
  }
  vx_stats st;
  detail::check(vx_tessellate_to_files(nullptr, &P, &O, label_path.c_str(),
                                       distance_path ? distance_path->c_str() : nullptr, seed, &st));
}

}  // namespace vxb200
