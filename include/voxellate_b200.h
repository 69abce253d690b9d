/* voxellate_b200 -- C-ABI of the B200-native voxel labeller.
 *
 * Drop-in boundary for the reference's hot path (arXiv 2201.13234 artifact,
 * `voxellate`), whose operator API is the C++ function
 *     TessResult tessellate_fast(const SiteSet&, const VoxelGrid&,
 *                                const FastOptions& = {});
 * (/root/reference/proj/include/voxellate/tessellate.hpp:59-60).  The reference
 * has no plugin registry or FFI: the boundary *is* that function.  This header
 * exports it as plain C (no exceptions, no torch or STL types), and
 * include/voxellate_b200.hpp wraps it back into the reference's C++ signature.
 *
 * Conventions (mirroring the reference):
 *  - kind: 0 Voronoi, 1 Johnson-Mehl, 2 Laguerre      (geometry.hpp:12)
 *  - positions are xyz-interleaved f64, n_sites * dim (sites.hpp:18)
 *  - voxel linear order is axis 0 fastest               (geometry.hpp:41-43)
 *  - label = argmin over sites of (ranking value, site index), i.e. the
 *    lowest index wins exact ties                       (tessellate.cpp:65,132)
 *  - labels are int32 (bit-identical to the reference's u32 for N_s < 2^31)
 *  - return codes: VX_EINVAL where the reference throws std::invalid_argument
 *    (same message text), VX_ECUDA/VX_ENOMEM for device failures.
 *  - every call blocks unless vx_options.asynchronous is set; inputs are read
 *    only, outputs are caller-allocated.  Calls on distinct contexts may run
 *    concurrently.  Calls on ONE context share its device workspaces: they
 *    are serialized on the host (a mutex) and on the device (a call on a
 *    different stream than the context's previous call first waits for that
 *    stream), so asynchronous calls on one context never overlap; a CUDA
 *    graph captured from a context must not be replayed concurrently with
 *    other work on that context.
 *  - TessResult.param / EvalCounters of the C++ shim are this engine's: the
 *    r0 is the reference's bit for bit, the timed t0 is this engine's own
 *    device cost scan (labels never depend on it), and the counters count
 *    this engine's ball-phase / unresolved-phase exact evaluations.
 */
#ifndef VOXELLATE_B200_H
#define VOXELLATE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VX_ABI_VERSION 2
#define VX_MAX_DIM 16 /* kMaxDim, geometry.hpp:16 */

enum vx_kind { VX_VORONOI = 0, VX_JOHNSON_MEHL = 1, VX_LAGUERRE = 2 };

enum vx_status {
  VX_OK = 0,
  VX_EINVAL = 1,       /* reference: std::invalid_argument */
  VX_ECUDA = 2,        /* CUDA runtime / launch failure */
  VX_ENOMEM = 3,       /* device allocation failed */
  VX_EUNSUPPORTED = 4, /* outside this engine's domain (e.g. N_s >= 2^31) */
  VX_EIO = 5,          /* reference: std::runtime_error from image I/O */
};

/* SiteSet + VoxelGrid of the reference (sites.hpp:15-31, geometry.hpp:27-78). */
typedef struct vx_problem {
  int32_t kind;     /* vx_kind */
  int32_t dim;      /* 1..16; d <= 3 runs the ball/shell engine, d >= 4 the brute engine */
  int32_t periodic; /* Boundary::Periodic = 1, NonPeriodic = 0 */
  int32_t reserved0;
  int64_t counts[VX_MAX_DIM];  /* voxels per axis, >= 1 */
  double lengths[VX_MAX_DIM];  /* domain edge lengths, finite > 0 */
  int64_t n_sites;             /* >= 1 */
  const double* positions;     /* n_sites*dim, strictly inside (0, L_i) */
  const double* times;         /* JM / Laguerre birth times t_s, or NULL */
  const double* weights;       /* Laguerre alternative to times: w_s = r_s^2,
                                  converted as t_s = -(w_s)/G (sites.cpp:101) */
  double growth;               /* G > 0 for timed kinds (ignored for Voronoi) */
} vx_problem;

/* FastOptions (tessellate.hpp:49-54) plus device-side controls. */
typedef struct vx_options {
  int32_t prune;          /* timed kinds: drop never-winning sites first (default 1) */
  int32_t has_override;   /* use override_param as r0 (Voronoi) / t0 (timed) */
  double override_param;
  int32_t device;         /* CUDA ordinal; -1 = the context's device */
  int32_t device_pointers;/* 1: positions/times/weights and all outputs are device pointers */
  void* stream;           /* cudaStream_t to run on; NULL = the context's stream (pass cudaStreamLegacy, 0x1, for the legacy default stream) */
  int32_t asynchronous;   /* 1: return after enqueueing (device_pointers only; stats
                             then carry no device-side counts) */
  int32_t profile_stages; /* 1: record CUDA events around each stage -> stats.stage_ms */
  double* distances_out;  /* optional: ranking value image (Voronoi: Euclidean distance) */
  uint64_t* histogram_out;/* optional: n_sites voxel counts per label (grain volumes) */
  int64_t slab_begin;     /* last-axis slab [slab_begin, slab_end) to label;      */
  int64_t slab_end;       /* 0,0 = whole grid.  Outputs then hold only the slab.  */
  double ball_scale;      /* gather radius = ball_scale * r0 (default 0 -> 1.0) */
  int32_t n_gpus;         /* > 1: split the slab over devices device..device+n_gpus-1 (wrapping
                             onto the devices present), one host thread each; host
                             buffers only (one process per GPU for device-resident data) */
  int32_t reserved;
} vx_options;

/* EvalCounters / param of TessResult (tessellate.hpp:31-43) for this engine. */
typedef struct vx_stats {
  double param;            /* r0 (Voronoi) or t0 (timed) used for the ball phase */
  int64_t n_voxels;        /* voxels labelled by this call */
  int64_t n_sites_kept;    /* sites left after prune */
  int64_t n_unresolved;    /* voxels handed to the widening-shell search */
  uint64_t ball_evals;     /* exact ranking evaluations, ball phase */
  uint64_t shell_evals;    /* exact ranking evaluations, shell phase */
  int32_t engine;          /* 0 = ball/shell engine, 1 = brute engine */
  int32_t kernel_launches; /* kernels this call enqueued */
  uint64_t overflow_bricks;/* bricks that fell back to the shell search */
  /* with options.profile_stages (synchronous calls): device ms per stage, timed
   * by CUDA events on the call's stream:
   * [0] H2D+ingest [1] bin+prune [2] params [3] ball [4] shell [5] D2H */
  float stage_ms[8];
} vx_stats;

#define VX_STAGE_INGEST 0
#define VX_STAGE_BIN 1
#define VX_STAGE_PARAMS 2
#define VX_STAGE_BALL 3
#define VX_STAGE_SHELL 4
#define VX_STAGE_D2H 5

/* ValidationReport (tessellate.hpp:70-76). */
typedef struct vx_validation {
  int64_t voxels_checked;
  int64_t label_mismatches;
  int64_t value_mismatches;
  int64_t n_examples;
  int64_t examples[16];
} vx_validation;

typedef struct vx_context vx_context;

/* ---- library ---- */
uint32_t vx_abi_version(void);
const char* vx_version_string(void);
/* thread-local message of the last failing call on this thread */
const char* vx_last_error(void);
/* Bytes the calling thread's last vx_tessellate call moved device -> host
 * (host-buffer calls: label image, distances, histogram).  Synchronous 3-D
 * host-buffer calls without distances move the label image as runs of equal
 * labels along x (per x-row an 8-byte record, per run one 32-bit word
 * `label << xbits | first x` when the site indices fit beside the x bits,
 * else an int32 label and a uint16 first x) and expand them into labels_out
 * on host threads; chunks
 * whose runs average < 4 voxels are copied raw.  labels_out is identical
 * either way.  VX_D2H_RAW=1 forces the raw copy. */
uint64_t vx_last_d2h_bytes(void);
void vx_options_init(vx_options* opt);

/* ---- contexts: own a device, a stream and cached workspaces ---- */
int vx_context_create(int device, vx_context** out);
void vx_context_destroy(vx_context* ctx);
/* device workspace bytes currently held by the context */
int64_t vx_context_workspace_bytes(const vx_context* ctx);
/* stage times (ms, the vx_stats.stage_ms layout) of the context's last call
 * with options.profile_stages -- also asynchronous calls and CUDA-graph
 * replays of a captured call; waits for that work to finish */
int vx_context_stage_ms(vx_context* ctx, float* stage_ms);

/* ---- engines ---- */
/* tessellate_fast (tessellate.cpp:195-282): labels_out holds N_v (or slab) int32.
 * ctx may be NULL (a per-thread default context on options->device). */
int vx_tessellate(vx_context* ctx, const vx_problem* problem, const vx_options* options,
                  int32_t* labels_out, vx_stats* stats_out);

/* tessellate_brute (tessellate.cpp:184-193): every voxel scans every site. */
int vx_tessellate_brute(vx_context* ctx, const vx_problem* problem, const vx_options* options,
                        int32_t* labels_out, vx_stats* stats_out);

/* prune_ineffective_sites (sites.cpp:113-171): dropped_out[s] = 1 for removed
 * sites (host pointer); *n_removed_out = number removed. Timed kinds only. */
int vx_prune(vx_context* ctx, const vx_problem* problem, uint8_t* dropped_out,
             int64_t* n_removed_out);

/* validate_partition (tessellate.cpp:304-367): sample == 0 checks every voxel,
 * else `sample` voxels drawn by mt19937_64(seed) exactly as the reference.
 * labels/distances are host pointers over the whole grid; distances may be NULL. */
int vx_validate_partition(vx_context* ctx, const vx_problem* problem, const int32_t* labels,
                          const double* distances, int64_t sample, uint64_t seed,
                          vx_validation* report_out);

/* ---- host helpers (reference API, no device work) ---- */
/* radius_from_volume(optimal_v0(n_sites, V), d) (cost.cpp:28-39) */
int vx_optimal_r0(int64_t n_sites, int dim, const double* lengths, double* r0_out);
/* generate_uniform_sites (sites.cpp:61-85); times_out may be NULL for Voronoi */
int vx_generate_uniform_sites(int dim, const double* lengths, int64_t n_sites, int kind,
                              double growth, double horizon, uint64_t seed,
                              double* positions_out, double* times_out);
/* the slab of the last axis owned by rank `rank` of `world` (tessellate.cpp:120-121) */
void vx_slab_bounds(int64_t n_last, int rank, int world, int64_t* begin_out, int64_t* end_out);
/* FNV-style label fingerprint: h ^= label; h *= 1099511628211 */
uint64_t vx_label_fingerprint(const int32_t* labels, int64_t n);

/* ---- on-disk images (row f2; reference include/voxellate/image_io.hpp:17-29) ----
 * Payload: raw little-endian labels (u32) or distances (f64), axis 0 fastest;
 * sidecar `<path>.json`: format_version, type, d, dims, lengths, boundary,
 * kind, n_sites, seed, payload_bytes.  type: 0 = "labels", 1 = "distances".
 * Errors: VX_EIO (the reference's std::runtime_error) / VX_EINVAL, with the
 * reference's message in vx_last_error(). */

/* tessellate_fast + write_label_image (+ write_distance_image when
 * distance_path != NULL) of the reference's run() (src/run.cpp:121-140,
 * image_io.cpp:164-175): positions are host pointers; the image is computed in
 * z-chunks and each chunk is copied out of device memory and appended to the
 * file while later chunks are computed.  options->distances_out,
 * histogram_out and device_pointers are ignored; seed goes to the sidecar
 * (-1: sites not from a seeded generator). */
int vx_tessellate_to_files(vx_context* ctx, const vx_problem* problem, const vx_options* options,
                           const char* label_path, const char* distance_path, int64_t seed,
                           vx_stats* stats);
/* write_label_image / write_distance_image of a host image (image_io.cpp:164-175) */
int vx_write_image(const char* path, int type, int dim, const int64_t* counts, const double* lengths,
                   int periodic, int kind, int64_t n_sites, int64_t seed, const void* data);
/* read_label_image / read_distance_image (image_io.cpp:177-202) with the
 * reference's checks.  header_out[6] = {dim, periodic, kind, n_sites, seed,
 * format_version}; counts_out / lengths_out hold VX_MAX_DIM entries; data may
 * be NULL (header only) and is filled when cap_voxels >= the voxel count. */
int vx_read_image(const char* path, int type, int64_t* header_out, int64_t* counts_out,
                  double* lengths_out, void* data, int64_t cap_voxels);
/* the sidecar alone: <path>.json, or its text into buf (returns its length) */
int vx_write_image_sidecar(const char* path, const char* type, int dim, const int64_t* counts,
                           const double* lengths, int periodic, int kind, int64_t n_sites,
                           int64_t seed, uint64_t payload_bytes);
int vx_image_sidecar_text(const char* type, int dim, const int64_t* counts, const double* lengths,
                          int periodic, int kind, int64_t n_sites, int64_t seed,
                          uint64_t payload_bytes, char* buf, int64_t cap);

/* ---- measurement ---- */
/* sustained f64 DADD and f32 FADD issue rates (adds/s) of `device`; the
 * roofline denominator for the per-voxel evaluation kernels */
int vx_probe_pipe_rates(int device, double* dadd_per_s, double* fadd_per_s);
/* Checks the eval kernel's call-free correctly rounded sqrt / division against
 * __dsqrt_rn / __ddiv_rn on n seeded random inputs (division by growth);
 * writes the number of bitwise mismatches of each. */
int vx_probe_exact_arith(int device, uint64_t n, uint64_t seed, double growth,
                         uint64_t* sqrt_mismatches, uint64_t* div_mismatches);
/* Best-of-3 device time (ms) of one host->device copy of `bytes` from `host`
 * through this library's runtime (diagnostics of the end-to-end number). */
int vx_probe_h2d(int device, const void* host, uint64_t bytes, int use_null_stream, float* ms_out);

#ifdef __cplusplus
}
#endif
#endif /* VOXELLATE_B200_H */
