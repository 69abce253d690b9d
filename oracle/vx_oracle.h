/* TEST INFRASTRUCTURE ONLY -- plain-C restatement of the reference's voxel
 * labelling arithmetic (the parity oracle).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it; the product never does.
 *
 * Pinned against: the reference library itself built from its sources
 * (oracle/_ref, see tests/test_oracle.py) and the golden fixtures in
 * tests/golden/ generated from it (tests/golden/make_golden.py).          */
#ifndef VX_ORACLE_H
#define VX_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* kind: 0 Voronoi, 1 Johnson-Mehl, 2 Laguerre (geometry.hpp:12). */

/* std::mt19937_64 + uniform01 (sites.cpp:20-22) */
typedef struct { uint64_t mt[312]; int mti; } vxo_mt64;
void vxo_mt64_seed(vxo_mt64* g, uint64_t seed);
uint64_t vxo_mt64_next(vxo_mt64* g);

/* generate_uniform_sites, sites.cpp:61-85 */
void vxo_generate_uniform_sites(int dim, const double* lengths, int64_t n_sites, int kind,
                                double horizon, uint64_t seed, double* positions_out,
                                double* times_out);
/* SURVEY.md App. C Laguerre recipe (cfg3): lognormal radii, then
 * spheres_to_timed_sites (sites.cpp:87-104): t = -(r*r)/G.           */
void vxo_generate_lognormal_spheres(int64_t n_sites, double mean_r, double sigma,
                                    uint64_t seed, double* positions_out, double* radii_out);
void vxo_spheres_to_timed(int64_t n, const double* radii, double growth, double* times_out);

/* tessellate_brute restated (tessellate.cpp:36-75,160-164,184-193) over the
 * linear voxel range [lin_begin, lin_end).  labels_out / distances_out hold
 * lin_end-lin_begin entries; distances_out may be NULL.                 */
void vxo_brute(int kind, int dim, int periodic, const int64_t* counts, const double* lengths,
               int64_t n_sites, const double* positions, const double* times, double growth,
               int64_t lin_begin, int64_t lin_end, uint32_t* labels_out, double* distances_out);

/* prune_ineffective_sites restated (sites.cpp:27-37,113-171).
 * Returns the number of removed sites; dropped_out[s] = 1 when removed. */
int64_t vxo_prune(int kind, int dim, int periodic, const double* lengths, int64_t n_sites,
                  const double* positions, const double* times, double growth,
                  uint8_t* dropped_out);

/* radius_from_volume(optimal_v0(n, V), d), cost.cpp:15-39 */
double vxo_optimal_r0(int64_t n_sites, int dim, const double* lengths);

/* SURVEY.md App. B label fingerprint. */
uint64_t vxo_fingerprint_u32(const uint32_t* labels, int64_t n);

/* validate_partition's sample draw (tessellate.cpp:325-330): mt19937_64(seed)
 * + libstdc++ uniform_int_distribution<int64_t>(0, nv-1) (Lemire, 128-bit). */
void vxo_sample_indices(int64_t nv, int64_t sample, uint64_t seed, int64_t* out);

#ifdef __cplusplus
}
#endif
#endif
