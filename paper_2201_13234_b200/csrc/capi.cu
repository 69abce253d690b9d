// The C-ABI (include/voxellate_b200.h) and the host-side orchestration of the
// device pipeline:
//
//   H2D sites -> K0 ingest/validate -> [timed+prune: K1 bin, K6 prune] -> K1 bin
//   -> param (r0 closed form | device t0 scan) -> K2 ball (+K3 compaction,
//   +histogram) -> K4 shell search -> D2H labels / distances / histogram.
//
// Mirrors tessellate_fast (tessellate.cpp:195-282): the same input checks and
// messages (check_inputs / SiteSet::validate, tessellate.cpp:176-180,
// sites.cpp:41-59; override checks tessellate.cpp:221,231-232), and the same
// output semantics (labels = original site indices after prune, Voronoi
// distances = sqrt of the best squared distance, tessellate.cpp:160-164,272-280).
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <string>
#include <thread>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <vector>

#include "voxellate_b200.h"
#include "vx_internal.cuh"

using namespace vxb;

namespace {

thread_local std::string g_err;
thread_local uint64_t g_d2h_bytes = 0;  // vx_last_d2h_bytes

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

}  // namespace

void vxb::set_last_error(const std::string& msg) { g_err = msg; }

int vxb::sm_count() {
  static std::atomic<int> cache[64];
  int dev = 0;
  cudaGetDevice(&dev);
  std::atomic<int>& c = cache[dev & 63];
  int n = c.load();
  if (n <= 0) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = 148;
    }
    c.store(n);
  }
  return n;
}

namespace {

struct Buf {
  void* p = nullptr;
  size_t n = 0;
};

}  // namespace

constexpr int kMaxChunks = 16;
constexpr int64_t kMaxZPlanes = 4095 * 64;  // gridDim.z limit x the deepest ball super-brick

struct vx_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::mutex mu;
  Buf pos_raw, t_raw, w_raw, p3, t, dropped, keys_a, keys_b, vals_a, vals_b, bx, by, bz, bt, bidx,
      cell_start, cub, labels, dist, hist, unres, params, counters, scratch, vsample, vlab, vdist,
      vbad, slots, f4, sb_info, sb_list, sb_count, sb_slots, sb_ovf, ctab, nd_x, nd_t, nd_idx, nd_cells, cell_fill,
      rc_rows, rc_lab, rc_x, rc_cnt;
  DevParams* h_prm = nullptr;
  DevCounters* h_ctr = nullptr;
  cudaEvent_t ev[8] = {};  // stage markers (options.profile_stages)
  bool ev_marked[8] = {};  // which markers the last profiled call recorded
  cudaStream_t copy_stream = nullptr;  // chunked D2H of host-buffer calls
  cudaStream_t last_stream = nullptr;  // the stream of the context's previous call
  cudaEvent_t handoff_ev = nullptr;    // orders a call after the previous one on another stream
  cudaEvent_t chunk_ev[16] = {};
  std::vector<cudaEvent_t> sink_ev;    // vx_tessellate_to_files: one per chunk
  cudaEvent_t done_ev[2] = {};
  void* pin[2] = {};                   // pinned double buffer of the file writer
  size_t pin_bytes = 0;
  void* rc_pin = nullptr;              // pinned landing area of the run-coded label transport
  size_t rc_pin_bytes = 0;

  vx_context() = default;
  vx_context(const vx_context&) = delete;
  vx_context& operator=(const vx_context&) = delete;
  // Frees every device / pinned resource: vx_context_destroy, the per-thread
  // default contexts when their thread exits, and a failed create_context.
  ~vx_context();

  Buf* all[45] = {&pos_raw, &t_raw,   &w_raw, &p3,    &t,      &dropped, &keys_a,   &keys_b,
                  &vals_a,  &vals_b,  &bx,    &by,    &bz,     &bt,      &bidx,     &cell_start,
                  &cub,     &labels,  &dist,  &hist,  &unres,  &params,  &counters, &scratch,
                  &vsample, &vlab,    &vdist, &vbad,  &slots,  &f4,      &sb_info,  &sb_list,
                  &sb_count, &sb_slots, &sb_ovf, &ctab, &nd_x,  &nd_t,   &nd_idx,   &nd_cells, &cell_fill,
                  &rc_rows, &rc_lab, &rc_x, &rc_cnt};
};

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace

vx_context::~vx_context() {
  // at process exit the CUDA runtime may already be unloading: then there is
  // nothing left to free
  int cur = -1;
  if (cudaGetDevice(&cur) == cudaErrorCudartUnloading) return;
  cudaGetLastError();
  DeviceGuard guard(device);
  if (stream) cudaStreamSynchronize(stream);
  for (Buf* b : all)
    if (b->p) {
      cudaFree(b->p);
      b->p = nullptr;
      b->n = 0;
    }
  if (h_prm) cudaFreeHost(h_prm);
  if (h_ctr) cudaFreeHost(h_ctr);
  if (stream) cudaStreamDestroy(stream);
  if (copy_stream) {
    cudaStreamSynchronize(copy_stream);
    cudaStreamDestroy(copy_stream);
  }
  for (auto e : chunk_ev)
    if (e) cudaEventDestroy(e);
  for (auto e : sink_ev) cudaEventDestroy(e);
  for (auto e : done_ev)
    if (e) cudaEventDestroy(e);
  for (auto b : pin)
    if (b) cudaFreeHost(b);
  if (rc_pin) cudaFreeHost(rc_pin);
  for (auto e : ev)
    if (e) cudaEventDestroy(e);
  if (handoff_ev) cudaEventDestroy(handoff_ev);
  cudaGetLastError();
}

namespace {

struct CudaFail {
  int code;
  std::string msg;
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw CudaFail{e == cudaErrorMemoryAllocation ? VX_ENOMEM : VX_ECUDA,
                   std::string(what) + ": " + cudaGetErrorString(e)};
  }
}

// CUDA-event stage markers on the call's stream (options.profile_stages).
struct StageTimer {
  bool on = false;
  cudaStream_t st = nullptr;
  cudaEvent_t* ev = nullptr;
  bool marked[8] = {};
  void mark(int i) {
    if (on) {
      // under stream capture an External record becomes an event-record node
      // of the graph (a plain record would only order the capture); the flag
      // is invalid outside a capture
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      cudaStreamIsCapturing(st, &cs);
      if (cs == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(ev[i], st, cudaEventRecordExternal);
      else cudaEventRecord(ev[i], st);
      marked[i] = true;
    }
  }
  void fill(float* ms) const {
    for (int i = 0; i < 7; ++i) {
      float v = 0.f;
      if (on && marked[i] && marked[i + 1]) cudaEventElapsedTime(&v, ev[i], ev[i + 1]);
      if (i < 8) ms[i] = v;
    }
  }
};

// VX_SYNC_DEBUG=1: synchronize after every stage and name the one that faulted.
void dbg(cudaStream_t st, const char* stage) {
  static const bool on = std::getenv("VX_SYNC_DEBUG") != nullptr;
  if (!on) return;
  ck(cudaStreamSynchronize(st), stage);
  ck(cudaGetLastError(), stage);
}

template <class... A>
int bin_checked(A&&... a) {
  const int n = launch_bin(std::forward<A>(a)...);
  if (n < 0) ck(static_cast<cudaError_t>(-1000 - n), "radix sort");
  return n;
}

template <class T>
T* ensure(Buf& b, size_t count) {
  const size_t bytes = count * sizeof(T) + 16;
  if (b.n < bytes) {
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.n = 0;
    ck(cudaMalloc(&b.p, bytes), "cudaMalloc");
    b.n = bytes;
  }
  return static_cast<T*>(b.p);
}

bool timed(const vx_problem* P) { return P->kind != VX_VORONOI; }

// unit-ball volume, cost.cpp:15-22
double unit_ball_volume(int d) { return std::pow(M_PI, 0.5 * d) / std::tgamma(0.5 * d + 1.0); }

// radius_from_volume(optimal_v0(n, V), d), cost.cpp:28-39
double optimal_r0(int64_t n_sites, int d, const double* L) {
  double V = 1.0;
  for (int i = 0; i < d; ++i) V *= L[i];
  const double ns = static_cast<double>(n_sites);
  const double v0 = V * (-std::expm1(-std::log(ns) / (ns - 1.0)));
  return std::pow(v0 / unit_ball_volume(d), 1.0 / d);
}

// cover_radius, tessellate.cpp:25-30
double cover_radius(int d, const double* L, bool periodic) {
  double s = 0.0;
  for (int i = 0; i < d; ++i) s += L[i] * L[i];
  const double diag = std::sqrt(s);
  return periodic ? 0.5 * diag : diag;
}

// Scalar input checks in the reference's order and wording.
int check_problem(const vx_problem* P) {
  if (!P) return fail(VX_EINVAL, "problem must not be NULL");
  if (P->kind < 0 || P->kind > 2) return fail(VX_EINVAL, "unknown tessellation kind");
  if (P->dim < 1) return fail(VX_EINVAL, "domain must have at least one axis");
  if (P->dim > VX_MAX_DIM) return fail(VX_EINVAL, "domain dimension exceeds supported maximum (16)");
  for (int i = 0; i < P->dim; ++i)
    if (!(std::isfinite(P->lengths[i]) && P->lengths[i] > 0.0))
      return fail(VX_EINVAL, "domain lengths must be positive");
  for (int i = 0; i < P->dim; ++i)
    if (P->counts[i] < 1) return fail(VX_EINVAL, "voxel counts must be positive");
  if (P->n_sites < 1) return fail(VX_EINVAL, "site set must contain at least one site");
  if (!P->positions) return fail(VX_EINVAL, "site position array has inconsistent size");
  if (timed(P)) {
    if (!P->times && !P->weights)
      return fail(VX_EINVAL, "timed site set must carry one birth time per site");
    if (!(std::isfinite(P->growth) && P->growth > 0.0))
      return fail(VX_EINVAL, "growth rate G must be positive for timed tessellations");
  }
  if (P->n_sites >= 0xFFFFFFFFll) return fail(VX_EINVAL, "site count exceeds the 32-bit label range");
  if (P->n_sites > 0x7FFFFFFFll)
    return fail(VX_EUNSUPPORTED, "int32 labels need fewer than 2^31 sites");
  double nv = 1.0;
  for (int i = 0; i < P->dim; ++i) nv *= (double)P->counts[i];
  if (nv > 9.0e18) return fail(VX_EINVAL, "voxel count overflows int64");
  return VX_OK;
}

// SiteSet::validate position rule, sites.cpp:54-57 (host pointers only)
int check_positions_host(const vx_problem* P) {
  const int d = P->dim;
  auto bad_in = [&](int64_t s0, int64_t s1) {
    for (int64_t s = s0; s < s1; ++s)
      for (int i = 0; i < d; ++i) {
        const double v = P->positions[s * d + i];
        if (!(std::isfinite(v) && v > 0.0 && v < P->lengths[i])) return true;
      }
    return false;
  };
  // a 24 MB scan at 10^6 sites: split over host threads (it precedes all GPU work)
  const int64_t n = P->n_sites;
  const int nt = n >= (1 << 18) ? (int)std::min<unsigned>(16, std::max(1u, std::thread::hardware_concurrency())) : 1;
  bool bad = false;
  if (nt == 1) {
    bad = bad_in(0, n);
  } else {
    std::vector<char> flags(nt, 0);
    std::vector<std::thread> th;
    for (int t = 1; t < nt; ++t) th.emplace_back([&, t] { flags[t] = bad_in(n * t / nt, n * (t + 1) / nt); });
    flags[0] = bad_in(0, n / nt);
    for (auto& x : th) x.join();
    for (char f : flags) bad |= f != 0;
  }
  if (bad) return fail(VX_EINVAL, "site positions must lie strictly inside the domain");
  return VX_OK;
}

double host_time(const vx_problem* P, int64_t s) {
  return P->times ? P->times[s] : -(P->weights[s]) / P->growth;
}

void fill_geo(Geo& g, const vx_problem* P, int64_t zb, int64_t ze, int64_t n_for_cells, bool xy2d = false) {
  std::memset(&g, 0, sizeof(g));
  g.kind = P->kind;
  g.periodic = P->periodic ? 1 : 0;
  g.dim = P->dim;
  g.has_times = timed(P);
  g.growth = timed(P) ? P->growth : 0.0;
  g.g_is_one = g.growth == 1.0;
  g.inv_growth_rn = g.growth > 0.0 ? 1.0 / g.growth : 0.0;
  g.lmax = 0.0;
  // true axis a -> embedded axis; the last true axis is always z (see Geo)
  static const int kEmb[4][3] = {{0, 1, 2}, {2, 0, 0}, {0, 2, 0}, {0, 1, 2}};
  // xy2d: a whole 2-D image maps to embedded (x, y) with a one-voxel z, so an
  // 8 x 8 x 4 sub-brick holds 64 voxels instead of 32 (the slab axis z is then
  // the padded one: callers pass zb = 0, ze = 1)
  static const int kEmb2xy[3] = {0, 1, 2};
  const int dd = P->dim <= 3 ? P->dim : 3;
  bool real[3] = {false, false, false};
  for (int a = 0; a < 3; ++a) {
    g.emb[a] = xy2d ? kEmb2xy[a] : kEmb[dd][a];
    g.n[a] = 1;
    g.L[a] = 1.0;
  }
  for (int a = 0; a < dd; ++a) {
    g.n[g.emb[a]] = P->counts[a];
    g.L[g.emb[a]] = P->lengths[a];
    real[g.emb[a]] = true;
  }
  g.vol_true = 1.0;
  g.suml2_true = 0.0;
  for (int a = 0; a < P->dim; ++a) {
    g.vol_true *= P->lengths[a];
    g.suml2_true += P->lengths[a] * P->lengths[a];
  }
  for (int a = 0; a < 3; ++a) {
    g.invL[a] = 1.0 / g.L[a];                   // geometry.cpp:52
    g.sp[a] = g.L[a] / (double)g.n[a];          // geometry.cpp:69
    g.halfL[a] = 0.5 * g.L[a];
    if (real[a]) g.lmax = std::fmax(g.lmax, g.L[a]);
  }
  // cell grid: about one site per cell, true axes only
  const double V = g.vol_true;
  double occ = 1.0;
  if (const char* e = std::getenv("VX_CELL_OCC")) occ = std::atof(e);
  double cw = std::pow(V * occ / (double)std::max<int64_t>(n_for_cells, 1), 1.0 / P->dim);
  for (int iter = 0; iter < 64; ++iter) {
    long long cells = 1;
    for (int a = 0; a < 3; ++a) {
      g.m[a] = real[a] ? (int)std::min(4096.0, std::max(1.0, std::floor(g.L[a] / cw))) : 1;
      cells *= g.m[a];
    }
    g.n_cells = cells;
    if (cells <= (1ll << 26)) break;
    cw *= 1.25;
  }
  for (int a = 0; a < 3; ++a) {
    g.cw[a] = g.L[a] / g.m[a];
    g.inv_cw[a] = g.m[a] / g.L[a];
  }
  g.z_begin = zb;
  g.z_end = ze;
  g.plane = g.n[0] * g.n[1];
  {  // range of the call-free exact sqrt / division (vx_internal.cuh)
    bool ok = g.growth == 0.0 || (g.growth >= 0x1p-64 && g.growth <= 0x1p64);
    for (int a = 0; a < 3; ++a) ok = ok && g.L[a] >= 0x1p-100 && g.L[a] <= 0x1p100 && g.sp[a] >= 0x1p-120;
    g.fast_arith = ok && std::getenv("VX_EXACT_CALLS") == nullptr;
  }
  g.nsbx = (unsigned)((g.n[0] + 7) / 8);
  g.nsby = (unsigned)((g.n[1] + 7) / 8);
  g.nbx = (g.n[0] + BX - 1) / BX;
  g.nby = (g.n[1] + BY - 1) / BY;
  g.nbz = (ze - zb + BZ - 1) / BZ;
  g.n_sites = P->n_sites;
  g.stats_on = std::getenv("VX_STATS") != nullptr;
}

std::map<int, std::unique_ptr<vx_context>>& thread_contexts() {
  thread_local std::map<int, std::unique_ptr<vx_context>> m;
  return m;
}

int create_context(int device, vx_context** out) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(VX_ECUDA, "no CUDA device available");
  }
  if (device < 0 || device >= ndev) return fail(VX_EINVAL, "invalid CUDA device ordinal");
  DeviceGuard guard(device);
  std::unique_ptr<vx_context> c(new vx_context);
  c->device = device;
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMallocHost(&c->h_prm, sizeof(DevParams)) != cudaSuccess ||
      cudaMallocHost(&c->h_ctr, sizeof(DevCounters)) != cudaSuccess) {
    const std::string m = cudaGetErrorString(cudaGetLastError());
    return fail(VX_ECUDA, "context creation failed: " + m);
  }
  *out = c.release();
  return VX_OK;
}

vx_context* resolve_context(vx_context* ctx, const vx_options* O, int* rc) {
  *rc = VX_OK;
  if (ctx) return ctx;
  int dev = O && O->device >= 0 ? O->device : -1;
  if (dev < 0) {
    if (cudaGetDevice(&dev) != cudaSuccess) {
      cudaGetLastError();
      *rc = fail(VX_ECUDA, "no CUDA device available");
      return nullptr;
    }
  }
  auto& m = thread_contexts();
  auto it = m.find(dev);
  if (it != m.end()) return it->second.get();
  vx_context* c = nullptr;
  *rc = create_context(dev, &c);
  if (*rc != VX_OK) return nullptr;
  m[dev].reset(c);
  return c;
}

// bytes per streamed piece of vx_tessellate_to_files (VX_SINK_CHUNK_BYTES overrides, for tests)
int64_t sink_chunk_bytes() {
  const char* e = std::getenv("VX_SINK_CHUNK_BYTES");
  return e ? std::max<int64_t>(4096, std::atoll(e)) : (256ll << 20);
}

struct SinkChunk {
  int64_t z0, z1;
  cudaEvent_t ev;  // recorded on the call's stream once the chunk is labelled
};

cudaEvent_t sink_event(vx_context* ctx, size_t i, cudaStream_t st) {
  while (ctx->sink_ev.size() <= i) {
    cudaEvent_t e;
    ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    ctx->sink_ev.push_back(e);
  }
  ck(cudaEventRecord(ctx->sink_ev[i], st), "chunk event");
  return ctx->sink_ev[i];
}

// ---- run-coded label transport (labelrun.cu) ----
// One z-chunk of a host-buffer call: its x-rows [r0, r0 + rows) of the slab,
// its run region [b0, b0 + cap) of the run arrays.
struct RunChunk {
  long long r0, rows, b0, cap;
};

struct RunPlan {
  int2* rows = nullptr;  // device
  int* lab = nullptr;
  unsigned short* x = nullptr;
  unsigned long long* cnt = nullptr;
  int2* p_rows = nullptr;  // pinned mirrors
  int* p_lab = nullptr;
  unsigned short* p_x = nullptr;
  unsigned long long* p_cnt = nullptr;  // mapped: written by launch_run_publish
  unsigned long long* d_pcnt = nullptr;  // its device address
  int xbits = 0;  // > 0: packed runs, label << xbits | x (labelrun.cu)
  std::vector<RunChunk> chunks;
  std::vector<cudaEvent_t> enc, d2h;  // encoded (call stream), copied (copy stream)
  ~RunPlan() {
    for (auto e : enc) cudaEventDestroy(e);
    for (auto e : d2h) cudaEventDestroy(e);
  }
};

// Device and pinned buffers for a slab of nvs voxels in rows of n0, nck chunks.
void run_plan_init(vx_context* ctx, RunPlan& rp, int64_t nvs, int64_t n0, int nck) {
  const size_t nrows = (size_t)(nvs / n0), cap = (size_t)(nvs / 4);
  rp.rows = ensure<int2>(ctx->rc_rows, nrows);
  rp.lab = ensure<int>(ctx->rc_lab, cap);
  rp.x = ensure<unsigned short>(ctx->rc_x, cap);
  rp.cnt = ensure<unsigned long long>(ctx->rc_cnt, (size_t)nck);
  auto up = [](size_t b) { return (b + 63) / 64 * 64; };
  const size_t o_lab = up(nrows * sizeof(int2)), o_x = o_lab + up(cap * 4), o_cnt = o_x + up(cap * 2);
  const size_t bytes = o_cnt + up((size_t)nck * 8);
  if (ctx->rc_pin_bytes < bytes) {
    if (ctx->rc_pin) cudaFreeHost(ctx->rc_pin);
    ctx->rc_pin = nullptr;
    ctx->rc_pin_bytes = 0;
    ck(cudaHostAlloc(&ctx->rc_pin, bytes, cudaHostAllocMapped), "cudaHostAlloc (label runs)");
    ctx->rc_pin_bytes = bytes;
  }
  char* b = static_cast<char*>(ctx->rc_pin);
  rp.p_rows = reinterpret_cast<int2*>(b);
  rp.p_lab = reinterpret_cast<int*>(b + o_lab);
  rp.p_x = reinterpret_cast<unsigned short*>(b + o_x);
  rp.p_cnt = reinterpret_cast<unsigned long long*>(b + o_cnt);
  ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(&rp.d_pcnt), rp.p_cnt, 0), "mapped run counts");
  for (int i = 0; i < nck; ++i) {
    cudaEvent_t e1, e2;
    ck(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming | cudaEventBlockingSync), "event");
    rp.enc.push_back(e1);
    ck(cudaEventCreateWithFlags(&e2, cudaEventDisableTiming | cudaEventBlockingSync), "event");
    rp.d2h.push_back(e2);
  }
}

// Host side of the transport: as each chunk's runs are coded, copy them (or,
// when they exceed the chunk's cap, its raw labels) to the host on the copy
// stream; T host threads expand every copied chunk into `out` while the next
// one is in flight.  Returns the bytes moved device -> host.
uint64_t run_drain(vx_context* ctx, RunPlan& rp, const int32_t* d_labels, int32_t* out, int n0) {
  const int nck = (int)rp.chunks.size();
  // one hardware thread stays free for this (issuing) thread: it must wake
  // promptly when a chunk is coded, and busy expanders would delay it by a
  // scheduler slice
  // concurrent drains (one per device of an n_gpus call) share the cores
  static std::atomic<int> active{0};
  struct Active {
    int n;
    Active() : n(++active) {}
    ~Active() { --active; }
  } act;
  int T = ((int)std::thread::hardware_concurrency() - act.n) / act.n;
  if (const char* e = std::getenv("VX_D2H_THREADS")) T = std::atoi(e);
  T = std::max(1, std::min(T, 64));
  std::vector<int> mode(nck, 0);  // 1: raw copy, 2: runs
  // VX_RUN_TRACE=1: per chunk, ms since the drain started when its runs were
  // coded, copied and (thread 0's share) expanded
  const bool rtrace = std::getenv("VX_RUN_TRACE") != nullptr;
  const auto t_start = std::chrono::steady_clock::now();
  auto ms_now = [&] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count(); };
  std::vector<double> t_enc(nck), t_cp(nck), t_dec(nck);
  std::mutex mu;
  std::condition_variable cv;
  int issued = 0;
  bool failed = false;
  const long long kRowBlock = std::max<long long>(16, (1 << 18) / std::max(1, n0));  // ~1 MB of image
  const bool run_static = std::getenv("VX_RUN_STATIC") != nullptr;  // A/B: the fixed row split
  std::vector<std::atomic<long long>> next_row(nck);
  for (auto& a : next_row) a.store(0, std::memory_order_relaxed);
  auto worker = [&](int t) {
    std::vector<int> buf;
    for (int c = 0; c < nck; ++c) {
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return issued > c || failed; });
        if (failed) return;
      }
      if (mode[c] != 2) continue;
      if (cudaEventSynchronize(rp.d2h[c]) != cudaSuccess) {
        std::lock_guard<std::mutex> lk(mu);
        failed = true;
        cv.notify_all();
        return;
      }
      if (rtrace && t == 0) t_cp[c] = ms_now();
      const RunChunk& k = rp.chunks[c];
      // blocks of rows claimed from the chunk's counter: no thread waits for a
      // slower one, and the issuing thread joins once every chunk is issued
      if (run_static) {
        if (t < T)
          run_decode_rows(reinterpret_cast<const int*>(rp.p_rows + k.r0), rp.p_lab + k.b0, rp.p_x + k.b0,
                          k.rows * t / T, k.rows * (t + 1) / T, n0, rp.xbits, out + k.r0 * n0, buf);
      } else for (;;) {
        const long long r = next_row[c].fetch_add(kRowBlock, std::memory_order_relaxed);
        if (r >= k.rows) break;
        run_decode_rows(reinterpret_cast<const int*>(rp.p_rows + k.r0), rp.p_lab + k.b0, rp.p_x + k.b0, r,
                        std::min<long long>(k.rows, r + kRowBlock), n0, rp.xbits, out + k.r0 * n0, buf);
      }
      if (rtrace && t == 0) t_dec[c] = ms_now();
    }
  };
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t) th.emplace_back(worker, t);
  uint64_t bytes = 0;
  auto stop = [&] {
    {
      std::lock_guard<std::mutex> lk(mu);
      failed = true;
    }
    cv.notify_all();
    for (auto& x : th) x.join();
  };
  try {
    for (int c = 0; c < nck; ++c) {
      const RunChunk& k = rp.chunks[c];
      ck(cudaEventSynchronize(rp.enc[c]), "label runs");
      if (rtrace) t_enc[c] = ms_now();
      const unsigned long long n = reinterpret_cast<volatile unsigned long long*>(rp.p_cnt)[c];
      int m = 2;
      if (n <= (unsigned long long)k.cap) {
        ck(cudaMemcpyAsync(rp.p_rows + k.r0, rp.rows + k.r0, sizeof(int2) * k.rows, cudaMemcpyDeviceToHost,
                           ctx->copy_stream), "D2H label runs");
        ck(cudaMemcpyAsync(rp.p_lab + k.b0, rp.lab + k.b0, sizeof(int) * n, cudaMemcpyDeviceToHost, ctx->copy_stream),
           "D2H label runs");
        if (rp.xbits == 0)
          ck(cudaMemcpyAsync(rp.p_x + k.b0, rp.x + k.b0, sizeof(unsigned short) * n, cudaMemcpyDeviceToHost,
                             ctx->copy_stream), "D2H label runs");
        bytes += sizeof(int2) * k.rows + (rp.xbits ? 4 : 6) * n + 8;
      } else {  // short runs: the chunk's labels as they are
        m = 1;
        ck(cudaMemcpyAsync(out + k.r0 * n0, d_labels + k.r0 * n0, sizeof(int32_t) * k.rows * n0,
                           cudaMemcpyDeviceToHost, ctx->copy_stream), "D2H labels");
        bytes += sizeof(int32_t) * k.rows * n0 + 8;
      }
      ck(cudaEventRecord(rp.d2h[c], ctx->copy_stream), "copy event");
      {
        std::lock_guard<std::mutex> lk(mu);
        mode[c] = m;
        issued = c + 1;
      }
      cv.notify_all();
    }
    worker(T);  // every chunk is issued: expand with the others
    for (auto& x : th) x.join();
    th.clear();
    bool bad = false;
    {
      std::lock_guard<std::mutex> lk(mu);
      bad = failed;
    }
    ck(cudaStreamSynchronize(ctx->copy_stream), "D2H labels");
    if (bad) ck(cudaErrorUnknown, "label runs");
    if (rtrace) {
      fprintf(stderr, "VX_RUN_TRACE %d threads, %d chunks, %.1f ms:", T, nck, ms_now());
      for (int c = 0; c < nck; ++c) fprintf(stderr, " [%d %s enc %.1f cp %.1f dec %.1f]", c, mode[c] == 2 ? "runs" : "raw", t_enc[c], t_cp[c], t_dec[c]);
      fprintf(stderr, "\n");
    }
  } catch (...) {
    if (!th.empty()) stop();
    throw;
  }
  return bytes;
}

struct FileSink;
int write_sink(vx_context* ctx, const vx_problem* P, const FileSink& sink, const std::vector<SinkChunk>& chunks,
               const int32_t* lab, const double* dist, int64_t zb, int64_t plane);

// Where a streamed image goes: files (vx_tessellate_to_files) or, for a
// host-buffer call whose output is pageable memory, the caller's buffers
// (staged through pinned memory: the driver's own pageable copies run at a
// few GB/s).
struct FileSink {
  const char* lab_path;
  const char* dist_path;  // NULL: labels only
  int64_t seed;
  char* mem[2] = {nullptr, nullptr};  // memory mode: labels, distances
  bool to_memory() const { return mem[0] != nullptr; }
};

// Double-buffered device -> pinned -> file streaming of the labelled chunks:
// the copy of piece i+1 overlaps the file write of piece i, and every piece
// waits only for the chunk that produced it (later chunks keep computing).
int write_sink(vx_context* ctx, const vx_problem* P, const FileSink& sink, const std::vector<SinkChunk>& chunks,
               const int32_t* lab, const double* dist, int64_t zb, int64_t plane) {
  struct Piece {
    int64_t z0, z1;
    cudaEvent_t ev;
    int which;  // 0 labels, 1 distances
  };
  std::vector<Piece> pieces;
  size_t max_bytes = 0;
  for (const SinkChunk& c : chunks) {
    const int64_t step = std::max<int64_t>(1, sink_chunk_bytes() / (plane * (dist ? 8 : 4)));
    for (int64_t a = c.z0; a < c.z1; a += step) {
      const int64_t b = std::min(c.z1, a + step);
      pieces.push_back({a, b, c.ev, 0});
      if (dist) pieces.push_back({a, b, c.ev, 1});
      max_bytes = std::max(max_bytes, (size_t)((b - a) * plane * (dist ? 8 : 4)));
    }
  }
  if (!ctx->copy_stream) {
    ck(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking), "copy stream");
    for (auto& e : ctx->chunk_ev) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  }
  for (auto& e : ctx->done_ev)
    if (!e) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  if (ctx->pin_bytes < max_bytes) {
    for (auto& b : ctx->pin)
      if (b) {
        cudaFreeHost(b);
        b = nullptr;
      }
    ctx->pin_bytes = 0;
    for (auto& b : ctx->pin) ck(cudaMallocHost(&b, max_bytes), "pinned staging buffer");
    ctx->pin_bytes = max_bytes;
  }
  int f[2] = {-1, -1};
  int64_t off[2] = {0, 0};
  const char* path[2] = {sink.lab_path, sink.dist_path};
  int rc = VX_OK;
  if (!sink.to_memory()) {
    rc = io_open_payload(path[0], &f[0]);
    if (!rc && dist) rc = io_open_payload(path[1], &f[1]);
  }
  auto issue = [&](size_t i) {
    const Piece& q = pieces[i];
    const size_t el = q.which ? 8 : 4;
    const char* src = q.which ? reinterpret_cast<const char*>(dist) : reinterpret_cast<const char*>(lab);
    ck(cudaStreamWaitEvent(ctx->copy_stream, q.ev, 0), "chunk wait");
    ck(cudaMemcpyAsync(ctx->pin[i & 1], src + (size_t)(q.z0 - zb) * plane * el, (size_t)(q.z1 - q.z0) * plane * el,
                       cudaMemcpyDeviceToHost, ctx->copy_stream),
       "D2H image chunk");
    ck(cudaEventRecord(ctx->done_ev[i & 1], ctx->copy_stream), "copy event");
  };
  try {
    if (!rc && !pieces.empty()) issue(0);
    for (size_t i = 0; !rc && i < pieces.size(); ++i) {
      ck(cudaEventSynchronize(ctx->done_ev[i & 1]), "D2H image chunk");
      if (i + 1 < pieces.size()) issue(i + 1);  // into the other buffer, already written out
      const Piece& q = pieces[i];
      const size_t nb = (size_t)(q.z1 - q.z0) * plane * (q.which ? 8 : 4);
      if (sink.to_memory()) io_copy_parallel(sink.mem[q.which] + off[q.which], ctx->pin[i & 1], nb);
      else rc = io_write_payload_at(f[q.which], path[q.which], ctx->pin[i & 1], nb, off[q.which]);
      off[q.which] += (int64_t)nb;
    }
  } catch (...) {
    for (int x : f)
      if (x >= 0) ::close(x);
    cudaStreamSynchronize(ctx->copy_stream);
    throw;
  }
  cudaStreamSynchronize(ctx->copy_stream);
  for (int k = 0; k < 2; ++k)
    if (f[k] >= 0) {
      const int rc2 = io_close_payload(f[k], path[k]);
      if (!rc) rc = rc2;
    }
  if (rc || sink.to_memory()) return rc;
  int64_t nv_total = 1;  // the files hold the whole image
  for (int a = 0; a < P->dim; ++a) nv_total *= P->counts[a];
  rc = vx_write_image_sidecar(sink.lab_path, "labels", P->dim, P->counts, P->lengths, P->periodic, P->kind,
                              P->n_sites, sink.seed, (uint64_t)nv_total * 4u);
  if (!rc && dist)
    rc = vx_write_image_sidecar(sink.dist_path, "distances", P->dim, P->counts, P->lengths, P->periodic, P->kind,
                                P->n_sites, sink.seed, (uint64_t)nv_total * 8u);
  return rc;
}

bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// VX_TRACE=1: host timestamps of a call's phases and device timing of the
// chunk pipeline on stderr (diagnostics for the end-to-end number).
struct CallTrace {
  bool on = std::getenv("VX_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  // start, first chunk computed, all computed, copies done, inputs copied, binned
  cudaEvent_t ev[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  double host_ms() const {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  void note(const char* what) const {
    if (on) fprintf(stderr, "VX_TRACE %-22s %8.3f ms (host)\n", what, host_ms());
  }
  void rec(int i, cudaStream_t s) {
    if (!on) return;
    if (!ev[i]) cudaEventCreate(&ev[i]);
    cudaEventRecord(ev[i], s);
  }
  void report() {
    if (!on || !ev[0]) return;
    const char* names[6] = {"", "first chunk computed", "all chunks computed", "copies done", "inputs copied",
                            "binned + params"};
    for (int i = 1; i < 6; ++i) {
      float ms = 0.f;
      if (ev[i] && cudaEventElapsedTime(&ms, ev[0], ev[i]) == cudaSuccess)
        fprintf(stderr, "VX_TRACE %-22s %8.3f ms (device, from H2D start)\n", names[i], ms);
    }
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
  }
};

int run(vx_context* ctx_in, const vx_problem* P, const vx_options* O_in, int32_t* labels_out,
        vx_stats* stats, bool brute_engine, const FileSink* sink = nullptr) {
  CallTrace trace;
  vx_options O;
  if (O_in) O = *O_in;
  else vx_options_init(&O);
  int rc = check_problem(P);
  if (rc) return rc;
  if (!labels_out && !sink) return fail(VX_EINVAL, "labels_out must not be NULL");
  const int d = P->dim;
  const int64_t n_last = P->counts[d - 1];
  int64_t zb = O.slab_begin, ze = O.slab_end;
  if (zb == 0 && ze == 0) ze = n_last;
  if (!(zb >= 0 && zb < ze && ze <= n_last))
    return fail(VX_EINVAL, "slab must satisfy 0 <= slab_begin < slab_end <= counts[dim-1]");
  // a whole 2-D image: (x, y) embedding, one "plane" of n0 n1 voxels
  // (embedded y rides in gridDim.y of the ball kernels: <= 65535 super-brick
  // rows); a whole 1-D image likewise maps to embedded x
  // d != 3: the d-dimensional engine (ballnd.cu); VX_ND_OFF=1 keeps the
  // older routes (d = 1, 2 embedded into the 3-D kernels, d >= 4 brute force)
  const bool use_nd = !brute_engine && d != 3 && !std::getenv("VX_ND_OFF");
  const bool xy2d = !use_nd && (d == 2 || d == 1) && !brute_engine && zb == 0 && ze == n_last &&
                    (d == 1 || n_last <= 1000000) && !std::getenv("VX_2D_XZ");
  if (O.asynchronous && !O.device_pointers)
    return fail(VX_EINVAL, "asynchronous calls need device pointers");
  const bool host_io = !O.device_pointers;
  const bool do_prune = !brute_engine && timed(P) && O.prune;
  const bool use_brute = brute_engine || (d > 3 && !use_nd);
  double t_min_host = std::numeric_limits<double>::quiet_NaN();
  // Host buffers: the positions are validated on the device during ingest
  // (the same predicate, sites.cpp:54-57) and the call fails right after it,
  // before any labelling work.  A host-side scan over worker threads would
  // leave the buffer's cache lines spread over other cores and make the DMA
  // read that follows ~8x slower (3.8 ms for 10^6 sites, VX_TRACE=1).
  if (host_io && timed(P) && O.has_override) {
    t_min_host = host_time(P, 0);
    for (int64_t s = 1; s < P->n_sites; ++s) t_min_host = std::fmin(t_min_host, host_time(P, s));
  }
  if (!brute_engine && O.has_override) {
    const double v = O.override_param;
    const char* bad = nullptr;
    if (!timed(P)) {
      if (!(std::isfinite(v) && v > 0.0)) bad = "override r0 must be positive";
    } else if (!std::isfinite(v) || (host_io && !(v >= t_min_host))) {
      bad = "override t0 must not precede the earliest birth time";
    }
    if (bad) {  // the reference validates the sites first (tessellate.cpp check_inputs)
      if (host_io && (rc = check_positions_host(P))) return rc;
      return fail(VX_EINVAL, bad);
    }
  }
  double ball_scale = O.ball_scale > 0.0 ? O.ball_scale : 1.0;

  trace.note("validated");
  vx_context* ctx = resolve_context(ctx_in, &O, &rc);
  if (!ctx) {  // no device: still report invalid sites with the reference's message
    if (host_io && check_positions_host(P)) return VX_EINVAL;
    return rc;
  }
  std::lock_guard<std::mutex> lock(ctx->mu);
  DeviceGuard guard(ctx->device);
  cudaStream_t st = O.stream ? static_cast<cudaStream_t>(O.stream) : ctx->stream;
  {
    // Calls on one context share its workspaces (bins, lists, counters): a
    // call on another stream than the previous one first waits for that
    // stream, so asynchronous calls on one context never overlap.  (Inside a
    // stream capture the caller orders the replays.)
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    if (cs == cudaStreamCaptureStatusNone && ctx->last_stream && ctx->last_stream != st) {
      if (!ctx->handoff_ev && cudaEventCreateWithFlags(&ctx->handoff_ev, cudaEventDisableTiming) != cudaSuccess)
        return fail(VX_ECUDA, "context handoff event: " + std::string(cudaGetErrorString(cudaGetLastError())));
      if (cudaEventRecord(ctx->handoff_ev, ctx->last_stream) != cudaSuccess ||
          cudaStreamWaitEvent(st, ctx->handoff_ev, 0) != cudaSuccess)
        cudaGetLastError();  // the previous stream was destroyed: nothing left to wait for
    }
    if (cs == cudaStreamCaptureStatusNone) ctx->last_stream = st;
  }
  int launches = 0;
  int64_t plane = 1;
  for (int i = 0; i < d - 1; ++i) plane *= P->counts[i];
  if (xy2d) {
    plane *= n_last;
    zb = 0;
    ze = 1;
  }
  const int64_t nvs = plane * (ze - zb);
  const int64_t ns = P->n_sites;
  StageTimer tm;
  bool labels_copied = false;  // chunked D2H already issued
  RunPlan rp;                  // run-coded label transport of this call
  bool run_pending = false;    // its chunks still to be copied and expanded
  std::vector<SinkChunk> sink_chunks;
  try {
    // asynchronous calls (and CUDA-graph captures of them) record the stage
    // markers too; vx_context_stage_ms reads them once the work has run
    tm.on = O.profile_stages != 0;
    tm.st = st;
    tm.ev = ctx->ev;
    if (tm.on && !ctx->ev[0])
      for (auto& e : ctx->ev) ck(cudaEventCreate(&e), "event");
    tm.mark(0);
    // ---- inputs ----
    const double* pos = P->positions;
    const double* times = P->times;
    const double* weights = P->times ? nullptr : P->weights;
    trace.note("context ready");
    if (trace.on && host_io)
      fprintf(stderr, "VX_TRACE positions pinned %d, labels pinned %d\n", (int)is_pinned(P->positions),
              (int)is_pinned(labels_out));
    trace.rec(0, st);
    if (host_io) {
      double* dp = ensure<double>(ctx->pos_raw, (size_t)ns * d);
      ck(cudaMemcpyAsync(dp, pos, sizeof(double) * ns * d, cudaMemcpyHostToDevice, st), "H2D positions");
      pos = dp;
      if (timed(P)) {
        const double* src = times ? times : weights;
        double* dt = ensure<double>(times ? ctx->t_raw : ctx->w_raw, (size_t)ns);
        ck(cudaMemcpyAsync(dt, src, sizeof(double) * ns, cudaMemcpyHostToDevice, st), "H2D times");
        if (times) times = dt;
        else weights = dt;
      }
    }
    Geo g;
    fill_geo(g, P, zb, ze, ns, xy2d);
    int32_t* lab = host_io ? ensure<int32_t>(ctx->labels, (size_t)nvs) : labels_out;
    double* dist = nullptr;
    // host-buffer call into pageable memory: stage through pinned buffers
    FileSink mem_sink{nullptr, nullptr, -1};
    if (host_io && !sink && !tm.on && (size_t)nvs * 4 >= (16u << 20) && !is_pinned(labels_out)) {
      mem_sink.mem[0] = reinterpret_cast<char*>(labels_out);
      mem_sink.mem[1] = reinterpret_cast<char*>(O.distances_out);
      sink = &mem_sink;
    }
    const bool want_dist = sink ? (sink->dist_path != nullptr || sink->mem[1] != nullptr) : O.distances_out != nullptr;
    if (want_dist) dist = host_io ? ensure<double>(ctx->dist, (size_t)nvs) : O.distances_out;
    unsigned long long* hist = nullptr;
    if (O.histogram_out) {
      hist = host_io ? ensure<unsigned long long>(ctx->hist, (size_t)ns)
                     : reinterpret_cast<unsigned long long*>(O.histogram_out);
      ck(cudaMemsetAsync(hist, 0, sizeof(unsigned long long) * ns, st), "memset histogram");
    }
    g.vec_store = (g.n[0] % 4 == 0) && ((reinterpret_cast<uintptr_t>(lab) & 15) == 0);
    DevParams* prm = ensure<DevParams>(ctx->params, 1);
    DevCounters* ctr = ensure<DevCounters>(ctx->counters, 1);
    // 3-D positions already are the internal xyz AoS, and given birth times
    // the time array: the ingest kernel then only validates (no copies)
    const bool p3_alias = !use_brute && d == 3 && g.emb[0] == 0 && g.emb[1] == 1 && g.emb[2] == 2;
    const bool t_alias = timed(P) && times != nullptr;
    double* t_copy = timed(P) && !t_alias ? ensure<double>(ctx->t, (size_t)ns) : nullptr;
    // the embedded 3-D copy of the 3-D engine
    const bool want_p3 = !use_brute && !p3_alias && !use_nd;
    double* p3_copy = want_p3 ? ensure<double>(ctx->p3, (size_t)ns * 3) : nullptr;
    const double* tdev = t_alias ? times : t_copy;
    const double* p3 = p3_alias ? pos : p3_copy;
    Len16 len;
    for (int i = 0; i < 16; ++i) len.L[i] = i < d ? P->lengths[i] : 1.0;
    trace.rec(4, st);
    launches += launch_init(prm, ctr, st);
    // device-pointer Voronoi calls in 3-D: the positions need no copy, so the
    // binning pass itself checks them (one launch and one read of the sites
    // fewer per call); host-buffer calls validate first (fail before any work)
    const bool fuse_validation = !host_io && !use_brute && !use_nd && p3_alias && !timed(P);
    if (fuse_validation) g.validate_in_keys = 1;
    else launches += launch_ingest(g, len, d, pos, times, weights, p3_copy, t_copy, ctr, st);
    dbg(st, "ingest");
    if (host_io) {  // fail before any labelling work (SiteSet::validate)
      ck(cudaMemcpyAsync(&ctx->h_ctr->bad_site, &ctr->bad_site, sizeof(unsigned), cudaMemcpyDeviceToHost, st),
         "D2H validation");
      ck(cudaStreamSynchronize(st), "validation");
      if (ctx->h_ctr->bad_site) return fail(VX_EINVAL, "site positions must lie strictly inside the domain");
    }
    tm.mark(1);

    double r0 = std::numeric_limits<double>::quiet_NaN();
    if (use_nd) {
      unsigned* ka = ensure<unsigned>(ctx->keys_a, (size_t)ns);
      unsigned* kb = ensure<unsigned>(ctx->keys_b, (size_t)ns);
      int* va = ensure<int>(ctx->vals_a, (size_t)ns);
      int* vb = ensure<int>(ctx->vals_b, (size_t)ns);
      GeoN gn;
      fill_geo_nd(gn, P->kind, d, P->periodic, reinterpret_cast<const long long*>(P->counts), P->lengths, g.growth,
                  ns, zb, ze);
      const size_t cub_bytes = bin_tmp_bytes(ns, std::max<long long>(gn.n_cells, g.n_cells));
      void* cub = ensure<char>(ctx->cub, cub_bytes);
      uint8_t* dropped = nullptr;
      double* nx = ensure<double>(ctx->nd_x, (size_t)ns * d);
      double* nt = timed(P) ? ensure<double>(ctx->nd_t, (size_t)ns) : nullptr;
      int* nidx = ensure<int>(ctx->nd_idx, (size_t)ns);
      int* ncs = ensure<int>(ctx->nd_cells, (size_t)gn.n_cells + 1);
      const BinsN bins{nx, ns, nt, nidx, ncs};
      if (do_prune) {  // bin every site, prune against the cells, re-bin the survivors
        dropped = ensure<uint8_t>(ctx->dropped, (size_t)ns);
        const int nb0 = launch_bin_nd(gn, pos, tdev, nullptr, cub, cub_bytes, ka, kb, va, vb, nx, nt, nidx, ncs, prm,
                                      ctr, st);
        if (nb0 < 0) ck(static_cast<cudaError_t>(-1000 - nb0), "radix sort");
        launches += nb0;
        launches += launch_prune_nd(gn, bins, pos, tdev, prm, dropped, st);
        dbg(st, "prune");
      }
      const int nbin = launch_bin_nd(gn, pos, tdev, dropped, cub, cub_bytes, ka, kb, va, vb, nx, nt, nidx, ncs, prm,
                                     ctr, st);
      if (nbin < 0) ck(static_cast<cudaError_t>(-1000 - nbin), "radix sort");
      launches += nbin;
      dbg(st, "bin");
      tm.mark(2);
      if (!timed(P)) r0 = ns == 1 ? cover_radius(d, P->lengths, P->periodic) : optimal_r0(ns, d, P->lengths);
      Geo gp = g;  // the cost model reads kind, dim, growth, volume, lengths
      gp.lmax = gn.lmax;
      double* scratch = ensure<double>(ctx->scratch, 1024);
      launches += launch_params(gp, tdev, dropped, prm, ctr, O.has_override, O.override_param, r0, ball_scale,
                                scratch, st);
      dbg(st, "params");
      tm.mark(3);
      const long long cap = (long long)std::min<int64_t>(nvs, 1ll << 26);
      long long* unres = ensure<long long>(ctx->unres, (size_t)cap);
      launches += launch_ball_nd(gn, bins, prm, lab, dist, hist, unres, cap, ctr, nvs, st);
      dbg(st, "ball nd");
      tm.mark(4);
      launches += launch_unres_nd(gn, bins, prm, unres, cap, lab, dist, hist, ctr, nvs, st);
      dbg(st, "unresolved nd");
      tm.mark(5);
      if (sink) sink_chunks.push_back({zb, ze, sink_event(ctx, 0, st)});
    } else if (use_brute) {
      uint8_t* dropped = nullptr;
      if (do_prune) {
        dropped = ensure<uint8_t>(ctx->dropped, (size_t)ns);
        launches += launch_prune_generic(P->kind, P->periodic, d, P->lengths, g.growth, pos, tdev, ns,
                                         dropped, st);
      }
      tm.mark(2);
      tm.mark(3);
      launches += launch_brute(P->kind, P->periodic, d, reinterpret_cast<const long long*>(P->counts),
                               P->lengths, g.growth, pos, tdev, dropped, ns, zb * plane, ze * plane,
                               lab, dist, hist, st);
      tm.mark(4);
      tm.mark(5);
      if (sink) sink_chunks.push_back({zb, ze, sink_event(ctx, 0, st)});
    } else {
      Bins bins;
      // binned x, y, z in one allocation (the eval kernels index x + a * ns)
      double* bx = ensure<double>(ctx->bx, (size_t)ns * 3);
      double* by = bx + ns;
      double* bz = bx + 2 * ns;
      double* bt = timed(P) ? ensure<double>(ctx->bt, (size_t)ns) : nullptr;
      int* bidx = ensure<int>(ctx->bidx, (size_t)ns);
      int* cs = ensure<int>(ctx->cell_start, (size_t)g.n_cells + 1);
      unsigned* ka = ensure<unsigned>(ctx->keys_a, (size_t)ns);
      unsigned* kb = ensure<unsigned>(ctx->keys_b, (size_t)ns);
      int* va = ensure<int>(ctx->vals_a, (size_t)ns);
      int* vb = ensure<int>(ctx->vals_b, (size_t)ns);
      const size_t cub_bytes = bin_tmp_bytes(ns, g.n_cells);
      void* cub = ensure<char>(ctx->cub, cub_bytes);
      double* scratch = ensure<double>(ctx->scratch, 1024);
      const long long cap = (long long)std::min<int64_t>(nvs, 1ll << 22);
      long long* unres = ensure<long long>(ctx->unres, (size_t)cap);
      uint8_t* dropped = do_prune ? ensure<uint8_t>(ctx->dropped, (size_t)ns) : nullptr;
      bins.x = bx;
      bins.y = by;
      bins.z = bz;
      bins.stride = ns;
      bins.t = bt;
      bins.idx = bidx;
      bins.cell_start = cs;
      float4* f4 = ensure<float4>(ctx->f4, (size_t)ns);
      bins.f4 = f4;
      bins.win_r2 = 0.0;
      bins.all_p3 = p3;
      bins.n_all = ns;
      // Slab window (a rank's z-slab of a multi-GPU run, Voronoi): bin only the
      // sites within M = 2 R + 2 cells + 2 voxels of the slab along z.  The ball
      // phase gathers within R < M; a shell search whose best distance reaches
      // M is redone over all sites (shell.cu / subshell.cu), so labels stay exact.
      if (!timed(P) && d == 3 && (ze - zb) < n_last && !std::getenv("VX_NO_WINDOW")) {
        const double R = (O.has_override ? O.override_param
                                         : (ns == 1 ? cover_radius(d, P->lengths, P->periodic)
                                                    : optimal_r0(ns, d, P->lengths) * ball_scale)) *
                             (1.0 + 1e-9) + 1e-12 * g.lmax;
        const double M = 2.0 * R + 2.0 * g.cw[2] + 2.0 * g.sp[2];
        const double zlo = ((double)zb + 0.5) * g.sp[2], zhi = ((double)(ze - 1) + 0.5) * g.sp[2];
        const double half = 0.5 * (zhi - zlo) + M;
        if (2.0 * half < 0.9 * g.L[2]) {
          g.win_on = 1;
          g.win_c = 0.5 * (zlo + zhi);
          g.win_half = half;
          const double m1 = M * (1.0 - 1e-9);
          bins.win_r2 = m1 * m1 * (1.0 - 1e-9);
        }
      }
      if (do_prune) {
        launches += bin_checked(g, p3, tdev, nullptr, cub, cub_bytes, ka, kb, va, vb, bx, by, bz, bt,
                                bidx, f4, cs, ensure<int>(ctx->cell_fill, (size_t)g.n_cells + 1), prm, ctr, st);
        dbg(st, "bin0");
        launches += launch_prune(g, bins, p3, tdev, prm, dropped, st);
        dbg(st, "prune");
      }
      launches += bin_checked(g, p3, tdev, dropped, cub, cub_bytes, ka, kb, va, vb, bx, by, bz, bt,
                              bidx, f4, cs, ensure<int>(ctx->cell_fill, (size_t)g.n_cells + 1), prm, ctr, st);
      dbg(st, "bin");
      tm.mark(2);
      if (!timed(P))
        r0 = ns == 1 ? cover_radius(d, P->lengths, P->periodic) : optimal_r0(ns, d, P->lengths);
      launches += launch_params(g, tdev, dropped, prm, ctr, O.has_override, O.override_param, r0,
                                ball_scale, scratch, st);
      trace.rec(5, st);
      dbg(st, "params");
      tm.mark(3);
      auto ball_and_shell = [&](const Geo& gg, int32_t* lb, double* ds) {
        unsigned long long* slots = ensure<unsigned long long>(ctx->slots, 128);
        const long long nsb = ball12_subbricks(gg);
        int2* info = ensure<int2>(ctx->sb_info, (size_t)nsb);
        int* slots16 = ensure<int>(ctx->sb_slots, (size_t)nsb * 16);
        const long long lcap =  // lists > 16 only (dense mode: most of them)
            std::min<long long>(nsb * (ball12_dense(gg) ? 48 : 4) + (1 << 20), (1ll << 31) - 1);
        int* list = ensure<int>(ctx->sb_list, (size_t)lcap);
        unsigned long long* lcount = ensure<unsigned long long>(ctx->sb_count, 1);
        int* ovf = ensure<int>(ctx->sb_ovf, (size_t)nsb);
        launches += launch_ball12(gg, bins, prm, lb, ds, hist, unres, cap, ctr, slots, info, slots16, list, lcap,
                                  lcount, ovf, st);
        dbg(st, "ball");
        tm.mark(4);
        launches += launch_shell(gg, bins, prm, lb, ds, hist, unres, cap, ctr, st);
        dbg(st, "shell");
        tm.mark(5);
      };
      // Host-buffer calls: the slab is computed in z-chunks and each chunk's
      // labels go to the host on a second stream while the next chunk is
      // computed (the PCIe copy of the label image is the larger cost of such a
      // call).  Chunks are whole super-bricks of the ball kernel (64 planes).
      const int64_t nz = ze - zb;
      // run-coded label transport (labelrun.cu): synchronous host-buffer
      // calls of 3-D images, labels only, rows of 64..65535 voxels
      bool rle = host_io && !tm.on && (sink == nullptr || sink == &mem_sink) && !want_dist && !O.asynchronous &&
                 d == 3 && !xy2d && g.n[0] >= 64 && g.n[0] <= 65535 && (size_t)nvs * 4 >= (16u << 20) &&
                 nvs / 4 < (1ll << 31) && std::getenv("VX_D2H_RAW") == nullptr;
      if (rle) sink = nullptr;  // pageable output: the decode threads write it directly
      int nchunk = 1;
      if (host_io && !tm.on && !sink) {
        const char* e = std::getenv("VX_CHUNKS");
        nchunk = e ? std::max(1, std::min(kMaxChunks, std::atoi(e))) : (nz >= 256 ? (rle ? 16 : 8) : 1);
      }
      int64_t cz = nchunk > 1 ? ((nz + nchunk - 1) / nchunk + 63) / 64 * 64 : nz;
      const bool pipelined = nchunk > 1;  // chunk D2H overlaps the next chunk's compute
      if (sink) {  // file output: chunks of <= sink_chunk_bytes() per array, whole super-bricks
        cz = std::max<int64_t>(1, sink_chunk_bytes() / (plane * (dist ? 8 : 4)));
        if (cz >= 64) cz = cz / 64 * 64;
        cz = std::min<int64_t>(cz, nz);
      }
      // the ball kernels put the last axis in gridDim.z (<= 65535 of 4..64
      // planes each): longer slabs are labelled in several launches
      cz = std::min<int64_t>(cz, kMaxZPlanes);
      if (rle) {
        run_plan_init(ctx, rp, nvs, g.n[0], (int)((nz + cz - 1) / cz));
        // label and first x in one word when every label (an original site
        // index) fits beside the x bits
        int xb = 1;
        while ((1ll << xb) < g.n[0]) ++xb;
        if ((long long)P->n_sites <= (1ll << (32 - xb)) && std::getenv("VX_RUN_UNPACKED") == nullptr) rp.xbits = xb;
      }
      if ((pipelined || rle) && !ctx->copy_stream) {
        ck(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking), "copy stream");
        for (auto& e : ctx->chunk_ev) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
      }
      int ci = 0;
      for (int64_t c0 = zb; c0 < ze; c0 += cz, ++ci) {
        const int64_t c1 = std::min<int64_t>(ze, c0 + cz);
        Geo gc = g;
        gc.z_begin = c0;
        gc.z_end = c1;
        gc.nbz = (c1 - c0 + BZ - 1) / BZ;
        int32_t* lb = lab + (c0 - zb) * plane;
        double* ds = dist ? dist + (c0 - zb) * plane : nullptr;
        gc.vec_store = (gc.n[0] % 4 == 0) && ((reinterpret_cast<uintptr_t>(lb) & 15) == 0);
        if (ci > 0) launches += launch_chunk_roll(ctr, st);
        ball_and_shell(gc, lb, ds);
        if (sink) sink_chunks.push_back({c0, c1, sink_event(ctx, ci, st)});
        if (ci == 0) trace.rec(1, st);
        if (rle) {
          const RunChunk k{(c0 - zb) * plane / g.n[0], (c1 - c0) * plane / g.n[0], (c0 - zb) * plane / 4,
                           (c1 - c0) * plane / 4};
          launches += launch_run_encode(lb, k.rows, (int)g.n[0], rp.rows + k.r0, rp.lab + k.b0, rp.x + k.b0, k.cap,
                                        rp.cnt + ci, rp.xbits, st);
          launches += launch_run_publish(rp.cnt + ci, rp.d_pcnt + ci, st);
          ck(cudaEventRecord(rp.enc[ci], st), "run event");
          rp.chunks.push_back(k);
        } else if (pipelined) {
          cudaEvent_t ev = ctx->chunk_ev[ci % kMaxChunks];
          ck(cudaEventRecord(ev, st), "chunk event");
          ck(cudaStreamWaitEvent(ctx->copy_stream, ev, 0), "chunk wait");
          ck(cudaMemcpyAsync(labels_out + (c0 - zb) * plane, lb, sizeof(int32_t) * (c1 - c0) * plane,
                             cudaMemcpyDeviceToHost, ctx->copy_stream),
             "D2H labels");
          if (ds)
            ck(cudaMemcpyAsync(O.distances_out + (c0 - zb) * plane, ds, sizeof(double) * (c1 - c0) * plane,
                               cudaMemcpyDeviceToHost, ctx->copy_stream),
               "D2H distances");
        }
      }
      trace.rec(2, st);
      if (rle) {
        labels_copied = true;
        run_pending = true;
      } else if (pipelined) {  // the call's stream waits for the last copy
        trace.rec(3, ctx->copy_stream);
        ck(cudaEventRecord(ctx->chunk_ev[ci % kMaxChunks], ctx->copy_stream), "copy event");
        ck(cudaStreamWaitEvent(st, ctx->chunk_ev[ci % kMaxChunks], 0), "copy wait");
        labels_copied = true;
      }
    }
    ck(cudaGetLastError(), "kernel launch");
    if (sink) {
      rc = write_sink(ctx, P, *sink, sink_chunks, lab, dist, zb, plane);
      if (rc) return rc;
      labels_copied = true;
    }
    if (host_io) {
      if (!labels_copied) {
        ck(cudaMemcpyAsync(labels_out, lab, sizeof(int32_t) * nvs, cudaMemcpyDeviceToHost, st), "D2H labels");
        if (dist)
          ck(cudaMemcpyAsync(O.distances_out, dist, sizeof(double) * nvs, cudaMemcpyDeviceToHost, st),
             "D2H distances");
      }
      if (hist)
        ck(cudaMemcpyAsync(O.histogram_out, hist, sizeof(unsigned long long) * ns,
                           cudaMemcpyDeviceToHost, st),
           "D2H histogram");
      g_d2h_bytes = (uint64_t)(hist ? 8 * ns : 0) +
                    (run_pending ? run_drain(ctx, rp, lab, labels_out, (int)P->counts[0])
                                 : (uint64_t)nvs * (dist ? 12 : 4));
    }
    tm.mark(6);
    if (stats) {
      std::memset(stats, 0, sizeof(*stats));
      stats->engine = use_brute ? 1 : 0;
      stats->kernel_launches = launches;
      stats->n_voxels = nvs;
      stats->param = std::numeric_limits<double>::quiet_NaN();
    }
    if (tm.on)
      for (int i = 0; i < 8; ++i) ctx->ev_marked[i] = tm.marked[i];
    if (O.asynchronous) return VX_OK;
    ck(cudaMemcpyAsync(ctx->h_prm, prm, sizeof(DevParams), cudaMemcpyDeviceToHost, st), "D2H params");
    ck(cudaMemcpyAsync(ctx->h_ctr, ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, st), "D2H counters");
    trace.note("enqueued");
    ck(cudaStreamSynchronize(st), "pipeline");
    trace.note("synchronized");
    trace.report();
    if (g.stats_on && ctx->slots.p) {  // VX_STATS diagnostics (ball kernel v8)
      unsigned long long h[128];
      ck(cudaMemcpy(h, ctx->slots.p, sizeof(h), cudaMemcpyDeviceToHost), "stats");
      const double nc = h[66] ? (double)h[66] : 1.0, nb = h[68] ? (double)h[68] : 1.0,
                   ns2 = h[70] ? (double)h[70] : 1.0;
      fprintf(stderr,
              "VX_STATS gathered/CTA raw %.1f kept %.1f | brick list %.1f | sub-brick list %.2f "
              "(%llu CTAs, %llu bricks, %llu sub-bricks)\n",
              h[64] / nc, h[65] / nc, h[67] / nb, h[69] / ns2, h[66], h[68], h[70]);
      fprintf(stderr, "VX_STATS max kept/CTA %llu, max brick list %llu, max sub-brick list %llu\n", h[71], h[72],
              h[73]);
    }
    if (stats) tm.fill(stats->stage_ms);
    if (ctx->h_ctr->bad_site) return fail(VX_EINVAL, "site positions must lie strictly inside the domain");
    if (!brute_engine && O.has_override && timed(P) && !use_brute &&
        !(O.override_param >= dkey_inv(ctx->h_prm->tmin_key)))
      return fail(VX_EINVAL, "override t0 must not precede the earliest birth time");
    if (stats) {
      if (!use_brute) {
        stats->param = ctx->h_prm->param;
        stats->n_sites_kept = (int64_t)ctx->h_ctr->n_alive;
        stats->n_unresolved = (int64_t)(ctx->h_ctr->n_unres + ctx->h_ctr->n_unres_done);
        stats->ball_evals = ctx->h_ctr->ball_evals;
        stats->shell_evals = ctx->h_ctr->shell_evals;
        stats->overflow_bricks = ctx->h_ctr->overflow_bricks;
      } else {
        stats->n_sites_kept = ns;
        stats->shell_evals = (uint64_t)nvs * (uint64_t)ns;
        if (!brute_engine && !timed(P))
          stats->param = ns == 1 ? cover_radius(d, P->lengths, P->periodic) : optimal_r0(ns, d, P->lengths);
      }
    }
  } catch (const CudaFail& f) {
    return fail(f.code, f.msg);
  }
  return VX_OK;
}

// Contexts of the multi-GPU host-buffer path, one per device, kept for the
// process (single-device calls use per-thread contexts).
vx_context* pool_context(int dev, int* rc) {
  static std::mutex mu;
  static std::map<int, std::unique_ptr<vx_context>> pool;
  std::lock_guard<std::mutex> lock(mu);
  auto it = pool.find(dev);
  if (it != pool.end()) return it->second.get();
  vx_context* c = nullptr;
  *rc = create_context(dev, &c);
  if (*rc) return nullptr;
  pool[dev].reset(c);
  return c;
}

// options->n_gpus > 1 (host buffers): rank r of G labels the last-axis slab of
// the reference's per-thread formula (tessellate.cpp:120-121) on device
// (device + r) mod (devices present), from its own host thread, straight into
// its part of the caller's buffers; the partial histograms are summed here.
// Results are bit-identical to a one-device call.
int run_multi(const vx_problem* P, const vx_options& O, int32_t* labels_out, vx_stats* stats, bool brute) {
  int rc = check_problem(P);
  if (rc) return rc;
  if (O.device_pointers || O.asynchronous)
    return fail(VX_EUNSUPPORTED,
                "n_gpus > 1 needs host buffers (device-resident data: one process per GPU with slabs)");
  if (!labels_out) return fail(VX_EINVAL, "labels_out must not be NULL");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(VX_ECUDA, "no CUDA device available");
  }
  int dev0 = O.device;
  if (dev0 < 0 && cudaGetDevice(&dev0) != cudaSuccess) dev0 = 0;
  const int d = P->dim;
  const int64_t n_last = P->counts[d - 1];
  int64_t zb = O.slab_begin, ze = O.slab_end;
  if (zb == 0 && ze == 0) ze = n_last;
  if (!(zb >= 0 && zb < ze && ze <= n_last))
    return fail(VX_EINVAL, "slab must satisfy 0 <= slab_begin < slab_end <= counts[dim-1]");
  int64_t plane = 1;
  for (int i = 0; i < d - 1; ++i) plane *= P->counts[i];
  const int G = O.n_gpus;
  const int64_t ns = P->n_sites;
  std::vector<std::vector<uint64_t>> hist(O.histogram_out ? G : 0);
  std::vector<vx_stats> st(G);
  std::vector<int> rcs(G, VX_OK);
  std::vector<std::string> errs(G);
  std::vector<std::thread> th;
  for (int r = 0; r < G; ++r) {
    int64_t a = 0, b = 0;
    vx_slab_bounds(ze - zb, r, G, &a, &b);
    if (b <= a) continue;
    a += zb;
    b += zb;
    th.emplace_back([&, r, a, b] {
      const int dev = (dev0 + r) % ndev;
      int rr = VX_OK;
      vx_context* ctx = pool_context(dev, &rr);
      if (!ctx) {
        rcs[r] = rr;
        errs[r] = vx_last_error();
        return;
      }
      vx_options o = O;
      o.n_gpus = 1;
      o.device = dev;
      o.stream = nullptr;  // a caller's stream belongs to one device: each rank uses its context's
      o.slab_begin = a;
      o.slab_end = b;
      o.distances_out = O.distances_out ? O.distances_out + (a - zb) * plane : nullptr;
      if (O.histogram_out) {
        hist[r].assign((size_t)ns, 0);
        o.histogram_out = hist[r].data();
      }
      std::memset(&st[r], 0, sizeof(vx_stats));
      rcs[r] = run(ctx, P, &o, labels_out + (a - zb) * plane, &st[r], brute);
      if (rcs[r]) errs[r] = vx_last_error();
    });
  }
  for (auto& t : th) t.join();
  for (int r = 0; r < G; ++r)
    if (rcs[r]) return fail(rcs[r], errs[r]);
  if (O.histogram_out) {
    std::memset(O.histogram_out, 0, sizeof(uint64_t) * ns);
    for (const auto& h : hist)
      for (size_t i = 0; i < h.size(); ++i) O.histogram_out[i] += h[i];
  }
  if (stats) {
    // seed from the first rank that labelled a slab (ranks past the last
    // plane get none and leave their stats zero)
    int r0 = 0;
    while (r0 < G - 1 && st[r0].n_voxels == 0) ++r0;
    *stats = st[r0];
    for (int r = r0 + 1; r < G; ++r) {
      stats->n_voxels += st[r].n_voxels;
      stats->n_unresolved += st[r].n_unresolved;
      stats->ball_evals += st[r].ball_evals;
      stats->shell_evals += st[r].shell_evals;
      stats->kernel_launches += st[r].kernel_launches;
      stats->overflow_bricks += st[r].overflow_bricks;
      for (int k = 0; k < 8; ++k) stats->stage_ms[k] = std::max(stats->stage_ms[k], st[r].stage_ms[k]);
    }
  }
  return VX_OK;
}

}  // namespace

extern "C" {

uint32_t vx_abi_version(void) { return VX_ABI_VERSION; }

const char* vx_version_string(void) {
  return "voxellate_b200 1.0 (sm_100a; ball/shell gather engine, exact f64 labels)";
}

const char* vx_last_error(void) { return g_err.c_str(); }
uint64_t vx_last_d2h_bytes(void) { return g_d2h_bytes; }

void vx_options_init(vx_options* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->prune = 1;
  o->device = -1;
  o->ball_scale = 1.0;
}

int vx_context_create(int device, vx_context** out) {
  if (!out) return fail(VX_EINVAL, "out must not be NULL");
  return create_context(device, out);
}

void vx_context_destroy(vx_context* ctx) { delete ctx; }

int vx_context_stage_ms(vx_context* ctx, float* stage_ms) {
  if (!ctx || !stage_ms) return fail(VX_EINVAL, "context and stage_ms must not be NULL");
  std::lock_guard<std::mutex> lock(ctx->mu);
  DeviceGuard guard(ctx->device);
  for (int i = 0; i < 8; ++i) stage_ms[i] = 0.f;
  int last = -1;
  for (int i = 0; i < 8; ++i)
    if (ctx->ev_marked[i]) last = i;
  if (last < 0) return VX_OK;
  cudaError_t e = cudaEventSynchronize(ctx->ev[last]);
  if (e != cudaSuccess) return fail(VX_ECUDA, std::string("stage events: ") + cudaGetErrorString(e));
  for (int i = 0; i < 7; ++i)
    if (ctx->ev_marked[i] && ctx->ev_marked[i + 1]) {
      e = cudaEventElapsedTime(&stage_ms[i], ctx->ev[i], ctx->ev[i + 1]);
      if (e != cudaSuccess) return fail(VX_ECUDA, std::string("stage events: ") + cudaGetErrorString(e));
    }
  return VX_OK;
}

int64_t vx_context_workspace_bytes(const vx_context* ctx) {
  if (!ctx) return 0;
  int64_t s = 0;
  for (const Buf* b : ctx->all) s += (int64_t)b->n;
  return s;
}

int vx_tessellate(vx_context* ctx, const vx_problem* problem, const vx_options* options,
                  int32_t* labels_out, vx_stats* stats_out) {
  g_d2h_bytes = 0;
  if (options && options->n_gpus > 1) return run_multi(problem, *options, labels_out, stats_out, false);
  return run(ctx, problem, options, labels_out, stats_out, false);
}

int vx_tessellate_brute(vx_context* ctx, const vx_problem* problem, const vx_options* options,
                        int32_t* labels_out, vx_stats* stats_out) {
  if (options && options->n_gpus > 1) return run_multi(problem, *options, labels_out, stats_out, true);
  return run(ctx, problem, options, labels_out, stats_out, true);
}

int vx_tessellate_to_files(vx_context* ctx, const vx_problem* problem, const vx_options* options,
                           const char* label_path, const char* distance_path, int64_t seed,
                           vx_stats* stats) {
  if (!label_path) return fail(VX_EINVAL, "label_path must not be NULL");
  vx_options o;
  if (options) o = *options;
  else vx_options_init(&o);
  o.device_pointers = 0;  // positions are host pointers; the image goes to the files
  o.asynchronous = 0;
  o.distances_out = nullptr;
  o.histogram_out = nullptr;
  o.slab_begin = o.slab_end = 0;  // the files hold the whole image
  o.profile_stages = 0;
  const FileSink sink{label_path, distance_path, seed};
  return run(ctx, problem, &o, nullptr, stats, false, &sink);
}

int vx_prune(vx_context* ctx_in, const vx_problem* P, uint8_t* dropped_out, int64_t* n_removed) {
  int rc = check_problem(P);
  if (rc) return rc;
  if (!timed(P)) return fail(VX_EINVAL, "pruning applies to timed tessellations only");
  if (!dropped_out) return fail(VX_EINVAL, "dropped_out must not be NULL");
  if ((rc = check_positions_host(P))) return rc;
  vx_context* ctx = resolve_context(ctx_in, nullptr, &rc);
  if (!ctx) return rc;
  std::lock_guard<std::mutex> lock(ctx->mu);
  DeviceGuard guard(ctx->device);
  cudaStream_t st = ctx->stream;
  const int d = P->dim;
  const int64_t ns = P->n_sites;
  try {
    double* pos = ensure<double>(ctx->pos_raw, (size_t)ns * d);
    ck(cudaMemcpyAsync(pos, P->positions, sizeof(double) * ns * d, cudaMemcpyHostToDevice, st), "H2D");
    double* src = ensure<double>(ctx->t_raw, (size_t)ns);
    ck(cudaMemcpyAsync(src, P->times ? P->times : P->weights, sizeof(double) * ns,
                       cudaMemcpyHostToDevice, st), "H2D");
    Geo g;
    fill_geo(g, P, 0, P->counts[d - 1], ns);
    double* tdev = ensure<double>(ctx->t, (size_t)ns);
    double* p3 = d <= 3 ? ensure<double>(ctx->p3, (size_t)ns * 3) : nullptr;
    DevParams* prm = ensure<DevParams>(ctx->params, 1);
    DevCounters* ctr = ensure<DevCounters>(ctx->counters, 1);
    uint8_t* dropped = ensure<uint8_t>(ctx->dropped, (size_t)ns);
    Len16 len;
    for (int i = 0; i < 16; ++i) len.L[i] = i < d ? P->lengths[i] : 1.0;
    launch_init(prm, ctr, st);
    launch_ingest(g, len, d, pos, P->times ? src : nullptr, P->times ? nullptr : src, p3, tdev, ctr, st);
    if (d <= 3) {
      Bins bins;
      double* bx = ensure<double>(ctx->bx, (size_t)ns * 3);
      double* by = bx + ns;
      double* bz = bx + 2 * ns;
      double* bt = ensure<double>(ctx->bt, (size_t)ns);
      int* bidx = ensure<int>(ctx->bidx, (size_t)ns);
      int* cs = ensure<int>(ctx->cell_start, (size_t)g.n_cells + 1);
      unsigned* ka = ensure<unsigned>(ctx->keys_a, (size_t)ns);
      unsigned* kb = ensure<unsigned>(ctx->keys_b, (size_t)ns);
      int* va = ensure<int>(ctx->vals_a, (size_t)ns);
      int* vb = ensure<int>(ctx->vals_b, (size_t)ns);
      const size_t cub_bytes = bin_tmp_bytes(ns, g.n_cells);
      void* cub = ensure<char>(ctx->cub, cub_bytes);
      bins.x = bx; bins.y = by; bins.z = bz; bins.t = bt; bins.idx = bidx; bins.cell_start = cs;
      bins.stride = ns;
      bins.f4 = nullptr;
      bin_checked(g, p3, tdev, nullptr, cub, cub_bytes, ka, kb, va, vb, bx, by, bz, bt, bidx,
                  (float4*)nullptr, cs, nullptr, prm, ctr, st);
      launch_prune(g, bins, p3, tdev, prm, dropped, st);
    } else {
      launch_prune_generic(P->kind, P->periodic, d, P->lengths, P->growth, pos, tdev, ns, dropped, st);
    }
    ck(cudaGetLastError(), "kernel launch");
    ck(cudaMemcpyAsync(dropped_out, dropped, (size_t)ns, cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "prune");
  } catch (const CudaFail& f) {
    return fail(f.code, f.msg);
  }
  int64_t removed = 0;
  for (int64_t s = 0; s < ns; ++s) removed += dropped_out[s] ? 1 : 0;
  if (n_removed) *n_removed = removed;
  return VX_OK;
}

int vx_validate_partition(vx_context* ctx_in, const vx_problem* P, const int32_t* labels,
                          const double* distances, int64_t sample, uint64_t seed,
                          vx_validation* report) {
  int rc = check_problem(P);
  if (rc) return rc;
  if (!labels || !report) return fail(VX_EINVAL, "labels and report must not be NULL");
  if ((rc = check_positions_host(P))) return rc;
  const int d = P->dim;
  int64_t nv = 1;
  for (int i = 0; i < d; ++i) nv *= P->counts[i];
  // tessellate.cpp:321-330: every voxel in order, or `sample` mt19937_64 draws
  const bool all = sample <= 0 || sample >= nv;
  std::vector<long long> chosen;
  if (!all) {
    std::mt19937_64 eng(seed);
    std::uniform_int_distribution<std::int64_t> pick(0, nv - 1);
    chosen.resize((size_t)sample);
    for (auto& c : chosen) c = pick(eng);
  }
  const int64_t n = all ? nv : (int64_t)chosen.size();
  vx_context* ctx = resolve_context(ctx_in, nullptr, &rc);
  if (!ctx) return rc;
  std::lock_guard<std::mutex> lock(ctx->mu);
  DeviceGuard guard(ctx->device);
  cudaStream_t st = ctx->stream;
  const int64_t ns = P->n_sites;
  std::memset(report, 0, sizeof(*report));
  try {
    double* pos = ensure<double>(ctx->pos_raw, (size_t)ns * d);
    ck(cudaMemcpyAsync(pos, P->positions, sizeof(double) * ns * d, cudaMemcpyHostToDevice, st), "H2D");
    double* tdev = nullptr;
    if (timed(P)) {
      double* src = ensure<double>(ctx->t_raw, (size_t)ns);
      ck(cudaMemcpyAsync(src, P->times ? P->times : P->weights, sizeof(double) * ns,
                         cudaMemcpyHostToDevice, st), "H2D");
      tdev = ensure<double>(ctx->t, (size_t)ns);
      Geo g;
      fill_geo(g, P, 0, P->counts[d - 1], ns);
      Len16 len;
      for (int i = 0; i < 16; ++i) len.L[i] = i < d ? P->lengths[i] : 1.0;
      DevCounters* ctr = ensure<DevCounters>(ctx->counters, 1);
      launch_ingest(g, len, d, pos, P->times ? src : nullptr, P->times ? nullptr : src, nullptr, tdev,
                    ctr, st);
    }
    // pieces of <= 2^24 voxels: device and host memory stay bounded whatever
    // the image size (a full audit of a 10^9-voxel image never materialises
    // grid-sized index arrays)
    const int64_t piece = std::min<int64_t>(n, 1 << 24);
    long long* ds = all ? nullptr : ensure<long long>(ctx->vsample, (size_t)piece);
    int* dl = ensure<int>(ctx->vlab, (size_t)piece);
    double* dd = distances ? ensure<double>(ctx->vdist, (size_t)piece) : nullptr;
    int* bad = ensure<int>(ctx->vbad, (size_t)(2 * piece));
    std::vector<int> lab_at(all ? 0 : (size_t)piece), bad_h((size_t)(2 * piece));
    std::vector<double> dist_at(all || !distances ? 0 : (size_t)piece);
    for (int64_t c0 = 0; c0 < n; c0 += piece) {
      const int64_t m = std::min(piece, n - c0);
      if (all) {  // the caller's contiguous range goes straight to the device
        ck(cudaMemcpyAsync(dl, labels + c0, sizeof(int) * m, cudaMemcpyHostToDevice, st), "H2D");
        if (dd) ck(cudaMemcpyAsync(dd, distances + c0, sizeof(double) * m, cudaMemcpyHostToDevice, st), "H2D");
      } else {
        for (int64_t i = 0; i < m; ++i) {
          lab_at[i] = labels[chosen[c0 + i]];
          if (distances) dist_at[i] = distances[chosen[c0 + i]];
        }
        ck(cudaMemcpyAsync(ds, chosen.data() + c0, sizeof(long long) * m, cudaMemcpyHostToDevice, st), "H2D");
        ck(cudaMemcpyAsync(dl, lab_at.data(), sizeof(int) * m, cudaMemcpyHostToDevice, st), "H2D");
        if (dd) ck(cudaMemcpyAsync(dd, dist_at.data(), sizeof(double) * m, cudaMemcpyHostToDevice, st), "H2D");
      }
      ck(cudaMemsetAsync(bad, 0, sizeof(int) * 2 * m, st), "memset");
      launch_validate(P->kind, P->periodic, d, reinterpret_cast<const long long*>(P->counts), P->lengths,
                      timed(P) ? P->growth : 0.0, pos, tdev, ns, ds, all ? c0 : 0, m, dl, dd, bad, bad + m, st);
      ck(cudaGetLastError(), "kernel launch");
      ck(cudaMemcpyAsync(bad_h.data(), bad, sizeof(int) * 2 * m, cudaMemcpyDeviceToHost, st), "D2H");
      ck(cudaStreamSynchronize(st), "validate");
      for (int64_t i = 0; i < m; ++i) {
        ++report->voxels_checked;
        const bool bl = bad_h[i] != 0, bv = distances && bad_h[m + i] != 0;
        report->label_mismatches += bl;
        report->value_mismatches += bv;
        if ((bl || bv) && report->n_examples < 16)
          report->examples[report->n_examples++] = all ? c0 + i : chosen[c0 + i];
      }
    }
  } catch (const CudaFail& f) {
    return fail(f.code, f.msg);
  }
  return VX_OK;
}

int vx_optimal_r0(int64_t n_sites, int dim, const double* lengths, double* r0_out) {
  if (n_sites < 2) return fail(VX_EINVAL, "optimal ball volume needs at least 2 sites");
  if (dim < 1 || dim > VX_MAX_DIM || !lengths || !r0_out) return fail(VX_EINVAL, "bad arguments");
  *r0_out = optimal_r0(n_sites, dim, lengths);
  return VX_OK;
}

// sites.cpp:61-85 with std::mt19937_64 (the sequence is fixed by the standard)
int vx_generate_uniform_sites(int dim, const double* lengths, int64_t n_sites, int kind,
                              double growth, double horizon, uint64_t seed, double* positions_out,
                              double* times_out) {
  if (n_sites < 1) return fail(VX_EINVAL, "number of sites must be at least 1");
  if (dim < 1 || dim > VX_MAX_DIM || !lengths || !positions_out) return fail(VX_EINVAL, "bad arguments");
  if (kind != VX_VORONOI) {
    if (!(growth > 0.0)) return fail(VX_EINVAL, "growth rate G must be positive for timed tessellations");
    if (!(horizon > 0.0)) return fail(VX_EINVAL, "time horizon T must be positive");
    if (!times_out) return fail(VX_EINVAL, "times_out must not be NULL for timed kinds");
  }
  std::mt19937_64 eng(seed);
  auto u01 = [&eng] { return static_cast<double>(eng() >> 11) * 0x1.0p-53; };
  for (int64_t s = 0; s < n_sites; ++s) {
    for (int i = 0; i < dim; ++i) {
      double u = u01();
      while (u == 0.0) u = u01();
      positions_out[s * dim + i] = u * lengths[i];
    }
    if (kind != VX_VORONOI) times_out[s] = u01() * horizon;
  }
  return VX_OK;
}

void vx_slab_bounds(int64_t n_last, int rank, int world, int64_t* begin_out, int64_t* end_out) {
  if (world < 1) world = 1;
  if (begin_out) *begin_out = n_last * rank / world;
  if (end_out) *end_out = n_last * (rank + 1) / world;
}

}  // extern "C"
