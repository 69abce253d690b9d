// TEST PROGRAM (infrastructure): the C++ shim (include/voxellate_b200.hpp, CUDA
// engine) against the reference library itself (oracle/_ref, compiled from
// /root/reference/proj/src), in one process, through their identical APIs.
// Restates test_tessellate.cpp:178-216 (fast == brute bit for bit), :271-290
// (override validation), :312-341 (validate_partition) and the prune tests of
// test_sites.cpp:173-194.  Exit code 0 == all checks passed.
#include <cstdio>
#include <cstring>
#include <random>
#include <stdexcept>

#include "voxellate/sites.hpp"
#include "voxellate/tessellate.hpp"
#ifdef VXREF_IMAGE_IO
#include "voxellate/image_io.hpp"
#endif
#include "voxellate_b200.hpp"

namespace R = voxellate;
namespace G = vxb200;

static int failures = 0;
#define CHECK(c)                                                         \
  do {                                                                   \
    if (!(c)) {                                                          \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);            \
      ++failures;                                                        \
    }                                                                    \
  } while (0)

static double uni(std::mt19937_64& e, double lo, double hi) {
  return lo + (hi - lo) * ((double)(e() >> 11) * 0x1.0p-53);
}

int main() {
  std::mt19937_64 eng(2024);
  int instances = 0;
  for (int trial = 0; trial < 120; ++trial) {
    const int d = trial % 9 == 8 ? 4 : 1 + trial % 3;
    const int kind = trial % 3;
    const bool periodic = (trial / 3) % 2;
    std::vector<double> L(d);
    for (auto& x : L) x = uni(eng, 0.5, 2.0);
    const std::int64_t cap = d == 1 ? 200 : (d == 2 ? 24 : (d == 3 ? 12 : 6));
    std::vector<std::int64_t> counts(d);
    for (auto& n : counts) n = 2 + (std::int64_t)(eng() % (cap - 1));
    const std::int64_t ns = 1 + (std::int64_t)(eng() % 60);
    const double growth = kind ? std::exp(uni(eng, std::log(0.1), std::log(10.0))) : 1.0;
    const double horizon = uni(eng, 0.5, 2.0);
    const std::uint64_t seed = eng();

    R::Domain rbox(L, periodic ? R::Boundary::Periodic : R::Boundary::NonPeriodic);
    R::VoxelGrid rgrid(counts, rbox);
    R::SiteSet rs = R::generate_uniform_sites(rbox, ns, (R::Kind)kind, growth, horizon, seed);
    G::Domain gbox(L, periodic ? G::Boundary::Periodic : G::Boundary::NonPeriodic);
    G::VoxelGrid ggrid(counts, gbox);
    G::SiteSet gs = G::generate_uniform_sites(gbox, ns, (G::Kind)kind, growth, horizon, seed);
    CHECK(gs.positions == rs.positions && gs.times == rs.times);

    R::FastOptions ro;
    G::FastOptions go;
    ro.prune = go.prune = (trial % 5) != 0;
    if (trial % 4 == 0) {
      const double v = kind == 0 ? uni(eng, 0.02, 2.0)
                                 : *std::min_element(rs.times.begin(), rs.times.end()) + uni(eng, 0.0, 1.0);
      ro.override_param = go.override_param = v;
    }
    const R::TessResult rf = R::tessellate_fast(rs, rgrid, ro);
    const G::TessResult gf = G::tessellate_fast(gs, ggrid, go);
    CHECK(gf.labels.labels == rf.labels.labels);
    CHECK(std::memcmp(gf.distances.values.data(), rf.distances.values.data(),
                      rf.distances.values.size() * sizeof(double)) == 0);
    if (kind == 0 && !ro.override_param) CHECK(gf.param == rf.param);
    const G::TessResult gb = G::tessellate_brute(gs, ggrid);
    const R::TessResult rb = R::tessellate_brute(rs, rgrid);
    CHECK(gb.labels.labels == rb.labels.labels);
    CHECK(std::memcmp(gb.distances.values.data(), rb.distances.values.data(),
                      rb.distances.values.size() * sizeof(double)) == 0);
    if (kind != 0) {
      const R::PruneResult rp = R::prune_ineffective_sites(rs, rbox);
      const G::PruneResult gp = G::prune_ineffective_sites(gs, gbox);
      CHECK(gp.removed == rp.removed && gp.kept == rp.kept);
    }
    ++instances;
  }
  // override validation throws std::invalid_argument (test_tessellate.cpp:271-290)
  {
    G::Domain box({1.0, 1.0}, G::Boundary::Periodic);
    G::VoxelGrid grid({8, 8}, box);
    G::SiteSet s = G::generate_uniform_sites(box, 4, G::Kind::Voronoi, 0.0, 1.0, 1);
    G::FastOptions bad;
    bad.override_param = 0.0;
    bool threw = false;
    try {
      G::tessellate_fast(s, grid, bad);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
  }
  // validate_partition reports agree with the reference on a tampered image
  {
    std::mt19937_64 e(123);
    R::Domain rbox({1.0, 1.3}, R::Boundary::Periodic);
    R::VoxelGrid rgrid({24, 20}, rbox);
    R::SiteSet rs = R::generate_uniform_sites(rbox, 30, R::Kind::Laguerre, 1.3, 1.0, 77);
    G::Domain gbox({1.0, 1.3}, G::Boundary::Periodic);
    G::VoxelGrid ggrid({24, 20}, gbox);
    G::SiteSet gs = G::generate_uniform_sites(gbox, 30, G::Kind::Laguerre, 1.3, 1.0, 77);
    R::TessResult rr = R::tessellate_fast(rs, rgrid);
    G::TessResult gr = G::tessellate_fast(gs, ggrid);
    rr.labels.labels[173] = (rr.labels.labels[173] + 1) % 30;
    gr.labels.labels[173] = (gr.labels.labels[173] + 1) % 30;
    for (std::int64_t sample : {0, 100}) {
      const R::ValidationReport a = R::validate_partition(rr.labels, &rr.distances, rs, sample, 9);
      const G::ValidationReport b = G::validate_partition(gr.labels, &gr.distances, gs, sample, 9);
      CHECK(a.voxels_checked == b.voxels_checked && a.label_mismatches == b.label_mismatches &&
            a.value_mismatches == b.value_mismatches && a.examples == b.examples);
    }
  }
#ifdef VXREF_IMAGE_IO
  // on-disk images: the shim writes, the reference reads (and the other way);
  // payload and sidecar bytes are identical
  {
    R::Domain rbox({1.5, 0.75, 2.0}, R::Boundary::NonPeriodic);
    R::VoxelGrid rgrid({5, 4, 3}, rbox);
    R::SiteSet rs = R::generate_uniform_sites(rbox, 9, R::Kind::JohnsonMehl, 0.8, 1.0, 5);
    R::TessResult rr = R::tessellate_fast(rs, rgrid);
    G::Domain gbox({1.5, 0.75, 2.0}, G::Boundary::NonPeriodic);
    G::VoxelGrid ggrid({5, 4, 3}, gbox);
    G::SiteSet gs = G::generate_uniform_sites(gbox, 9, G::Kind::JohnsonMehl, 0.8, 1.0, 5);
    G::TessResult gr = G::tessellate_fast(gs, ggrid);
    R::ImageMeta rm;
    rm.kind = R::Kind::JohnsonMehl;
    rm.n_sites = 9;
    rm.seed = 5;
    G::ImageMeta gm;
    gm.kind = G::Kind::JohnsonMehl;
    gm.n_sites = 9;
    gm.seed = 5;
    R::write_label_image("/tmp/vx_shim_r.lab", rr.labels, rm);
    R::write_distance_image("/tmp/vx_shim_r.dist", rr.distances, rm);
    G::write_label_image("/tmp/vx_shim_g.lab", gr.labels, gm);
    G::write_distance_image("/tmp/vx_shim_g.dist", gr.distances, gm);
    auto slurp = [](const char* p) {
      std::string out;
      if (FILE* f = std::fopen(p, "rb")) {
        char b[4096];
        size_t n;
        while ((n = std::fread(b, 1, sizeof(b), f)) > 0) out.append(b, n);
        std::fclose(f);
      }
      return out;
    };
    for (const char* sfx : {".lab", ".lab.json", ".dist", ".dist.json"}) {
      const std::string a = slurp((std::string("/tmp/vx_shim_r") + sfx).c_str());
      const std::string b = slurp((std::string("/tmp/vx_shim_g") + sfx).c_str());
      CHECK(!a.empty() && a == b);
    }
    R::ImageMeta m1;
    const R::LabelImage back_r = R::read_label_image("/tmp/vx_shim_g.lab", &m1);
    CHECK(back_r.labels == rr.labels.labels && m1.seed == 5 && m1.n_sites == 9);
    G::ImageMeta m2;
    const G::DistanceImage back_g = G::read_distance_image("/tmp/vx_shim_r.dist", &m2);
    CHECK(std::memcmp(back_g.values.data(), rr.distances.values.data(), sizeof(double) * back_g.values.size()) == 0);
    bool threw = false;
    try {
      G::read_distance_image("/tmp/vx_shim_r.lab");
    } catch (const std::runtime_error& e) {
      threw = std::string(e.what()) == "image /tmp/vx_shim_r.lab has type 'labels', expected 'distances'";
    }
    CHECK(threw);
    for (const char* p : {"/tmp/vx_shim_r.lab", "/tmp/vx_shim_r.dist", "/tmp/vx_shim_g.lab", "/tmp/vx_shim_g.dist"}) {
      std::remove(p);
      std::remove((std::string(p) + ".json").c_str());
    }
  }
#endif
  {  // ball_voxels / scan_ball (tessellate.hpp:62-68), spheres_to_timed_sites (sites.hpp:52)
    std::mt19937_64 e2(77);
    for (int it = 0; it < 200; ++it) {
      const int d = 1 + it % 4;
      const bool per = it % 2;
      std::vector<double> L(d), c(d);
      std::vector<std::int64_t> counts(d);
      for (int a = 0; a < d; ++a) {
        L[a] = uni(e2, 0.5, 2.0);
        counts[a] = 1 + (std::int64_t)(e2() % (d == 1 ? 300 : (d == 2 ? 60 : (d == 3 ? 20 : 10))));
        c[a] = uni(e2, -0.2, 1.2) * L[a];
      }
      double diag = 0.0;
      for (double x : L) diag += x * x;
      double r = uni(e2, 0.0, 1.2) * std::sqrt(diag);
      R::VoxelGrid rg(counts, R::Domain(L, per ? R::Boundary::Periodic : R::Boundary::NonPeriodic));
      G::VoxelGrid gg(counts, G::Domain(L, per ? G::Boundary::Periodic : G::Boundary::NonPeriodic));
      if (it % 5 == 0) {  // a voxel centre exactly on the sphere
        double s2 = 0.0;
        for (int a = 0; a < d; ++a) {
          const double x = rg.center_coord(a, (std::int64_t)(e2() % counts[a]));
          s2 += (c[a] - x) * (c[a] - x);
        }
        r = std::sqrt(s2);
      }
      CHECK(G::ball_voxels(c, r, gg) == R::ball_voxels(c, r, rg));
      std::int64_t visits = 0;
      G::scan_ball(c, r, gg, [&](std::int64_t) { ++visits; });
      CHECK(visits == (std::int64_t)R::ball_voxels(c, r, rg).size());
    }
    bool t1 = false, t2 = false;
    try { G::ball_voxels({0.5}, -1.0, G::VoxelGrid({4}, G::Domain({1.0}, G::Boundary::Periodic))); }
    catch (const std::invalid_argument& e) { t1 = std::string(e.what()) == "ball radius must be nonnegative"; }
    try { G::ball_voxels({0.5, 0.5}, 0.1, G::VoxelGrid({4}, G::Domain({1.0}, G::Boundary::Periodic))); }
    catch (const std::invalid_argument& e) { t2 = std::string(e.what()) == "ball center dimension does not match the grid"; }
    CHECK(t1 && t2);
    R::LaguerreSpheres rs;
    G::LaguerreSpheres gs;
    rs.dim = gs.dim = 3;
    for (int i = 0; i < 30; ++i) {
      for (int a = 0; a < 3; ++a) {
        const double x = uni(e2, 0.01, 0.99);
        rs.positions.push_back(x);
        gs.positions.push_back(x);
      }
      const double rad = uni(e2, 0.0, 0.2);
      rs.radii.push_back(rad);
      gs.radii.push_back(rad);
    }
    const R::SiteSet a = R::spheres_to_timed_sites(rs, 1.7);
    const G::SiteSet b = G::spheres_to_timed_sites(gs, 1.7);
    CHECK(a.times == b.times && a.positions == b.positions && b.kind == G::Kind::Laguerre && b.growth == 1.7);
    gs.radii[3] = -1.0;
    bool t3 = false;
    try { G::spheres_to_timed_sites(gs, 1.0); }
    catch (const std::invalid_argument& e) { t3 = std::string(e.what()) == "sphere radii must be nonnegative"; }
    CHECK(t3);
  }
  std::printf("%d instances, %d failures\n", instances, failures);
  if (failures == 0) std::printf("ALL OK\n");
  return failures == 0 ? 0 : 1;
}
