// Brute engine: tessellate_brute (reference: tessellate.cpp:184-193 ->
// resolve_voxels_impl<K,P>(only_unassigned=false), tessellate.cpp:36-75) and
// the validate_partition re-check (tessellate.cpp:304-367).
//
// One thread per voxel, sites streamed through shared memory in ascending
// index order, strict-< update: the reference's tie rule.  Any dimension
// 1..16 (this is also the engine vx_tessellate uses for d >= 4).
#include "vx_internal.cuh"

namespace vxb {

struct BruteGeo {
  int dim, kind, periodic, g_is_one;
  double growth;
  long long counts[16];
  double L[16], invL[16], sp[16];
  const uint8_t* dropped;  // pruned sites never compete (nullptr = none)
};

constexpr int kBruteThreads = 128;
constexpr int kTile = 128;

template <int KIND, bool PER>
__device__ __forceinline__ void brute_voxel(const BruteGeo& g, const double* x, const double* s_pos,
                                            const double* s_t, int ntile, int tile_base,
                                            double& best, int& bl) {
  for (int j = 0; j < ntile; ++j) {
    const double* sp = s_pos + j * g.dim;
    double acc = 0.0;
    for (int i = g.dim - 1; i >= 0; --i)
      acc = __dadd_rn(acc, axis_sq<PER>(sp[i], x[i], g.L[i], g.invL[i]));
    const double pr = prox_from_dsq<KIND>(acc, g.growth, g.g_is_one, KIND == kVoronoi ? 0.0 : s_t[j]);
    if (pr < best) {
      best = pr;
      bl = tile_base + j;
    }
  }
}

// lin_list == nullptr: voxels lin_begin + [0, count); else lin_list[0, count)
template <int KIND, bool PER>
__global__ void __launch_bounds__(kBruteThreads)
    brute_kernel(BruteGeo g, const double* __restrict__ pos, const double* __restrict__ t,
                 long long n_sites, long long lin_begin, long long count,
                 const long long* __restrict__ lin_list, int* __restrict__ labels,
                 double* __restrict__ dist, unsigned long long* __restrict__ hist,
                 const int* __restrict__ chk_label, const double* __restrict__ chk_dist,
                 int* __restrict__ bad_label, int* __restrict__ bad_value) {
  extern __shared__ double smem[];
  double* s_pos = smem;                 // kTile * dim
  double* s_t = smem + kTile * g.dim;   // kTile
  const long long i = blockIdx.x * (long long)kBruteThreads + threadIdx.x;
  const bool active = i < count;
  const long long lin = active ? (lin_list ? lin_list[i] : lin_begin + i) : 0;
  double x[16];
  long long rem = lin;
  for (int a = 0; a < g.dim; ++a) {
    const long long k = rem % g.counts[a];
    rem /= g.counts[a];
    x[a] = center(k, g.sp[a]);
  }
  double best = __longlong_as_double(0x7ff0000000000000ll);
  int bl = -1;
  for (long long base = 0; base < n_sites; base += kTile) {
    const int nt = (int)min((long long)kTile, n_sites - base);
    __syncthreads();
    for (int e = threadIdx.x; e < nt * g.dim; e += kBruteThreads) s_pos[e] = pos[base * g.dim + e];
    if (KIND != kVoronoi)
      for (int e = threadIdx.x; e < nt; e += kBruteThreads)
        s_t[e] = (g.dropped && g.dropped[base + e]) ? __longlong_as_double(0x7ff0000000000000ll)
                                                    : t[base + e];
    __syncthreads();
    if (active) brute_voxel<KIND, PER>(g, x, s_pos, s_t, nt, (int)base, best, bl);
  }
  if (!active) return;
  const double val = KIND == kVoronoi ? __dsqrt_rn(best) : best;
  if (chk_label) {  // validate_partition
    bad_label[i] = chk_label[i] != bl;
    if (chk_dist) bad_value[i] = !(chk_dist[i] == val);
    return;
  }
  labels[i] = bl;
  if (dist) dist[i] = val;
  if (hist) atomicAdd(&hist[bl], 1ull);
}

static BruteGeo make_bgeo(int kind, int periodic, int dim, const long long* counts,
                          const double* lengths, double growth) {
  BruteGeo g{};
  g.dim = dim;
  g.kind = kind;
  g.periodic = periodic;
  g.growth = growth;
  g.g_is_one = growth == 1.0;
  for (int a = 0; a < dim; ++a) {
    g.counts[a] = counts[a];
    g.L[a] = lengths[a];
    g.invL[a] = 1.0 / lengths[a];                   // geometry.cpp:52
    g.sp[a] = lengths[a] / (double)counts[a];       // geometry.cpp:69
  }
  return g;
}

template <int KIND>
static void go(const BruteGeo& g, const double* pos, const double* t, long long ns, long long lb,
               long long count, const long long* list, int* labels, double* dist,
               unsigned long long* hist, const int* cl, const double* cd, int* bl, int* bv,
               cudaStream_t st) {
  const unsigned nb = (unsigned)((count + kBruteThreads - 1) / kBruteThreads);
  const size_t sh = (size_t)kTile * (g.dim + 1) * sizeof(double);
  if (g.periodic)
    brute_kernel<KIND, true><<<nb, kBruteThreads, sh, st>>>(g, pos, t, ns, lb, count, list, labels,
                                                            dist, hist, cl, cd, bl, bv);
  else
    brute_kernel<KIND, false><<<nb, kBruteThreads, sh, st>>>(g, pos, t, ns, lb, count, list, labels,
                                                             dist, hist, cl, cd, bl, bv);
}

static void dispatch(const BruteGeo& g, const double* pos, const double* t, long long ns,
                     long long lb, long long count, const long long* list, int* labels,
                     double* dist, unsigned long long* hist, const int* cl, const double* cd,
                     int* bl, int* bv, cudaStream_t st) {
  if (count <= 0) return;
  switch (g.kind) {
    case kVoronoi: go<kVoronoi>(g, pos, t, ns, lb, count, list, labels, dist, hist, cl, cd, bl, bv, st); break;
    case kJohnsonMehl: go<kJohnsonMehl>(g, pos, t, ns, lb, count, list, labels, dist, hist, cl, cd, bl, bv, st); break;
    default: go<kLaguerre>(g, pos, t, ns, lb, count, list, labels, dist, hist, cl, cd, bl, bv, st); break;
  }
}

int launch_brute(int kind, int periodic, int dim, const long long* counts, const double* lengths,
                 double growth, const double* pos, const double* t, const uint8_t* dropped,
                 long long n_sites, long long lin_begin, long long lin_end, int* labels,
                 double* dist, unsigned long long* hist, cudaStream_t st) {
  BruteGeo g = make_bgeo(kind, periodic, dim, counts, lengths, growth);
  g.dropped = dropped;
  dispatch(g, pos, t, n_sites, lin_begin, lin_end - lin_begin, nullptr, labels, dist, hist,
           nullptr, nullptr, nullptr, nullptr, st);
  return 1;
}

int launch_validate(int kind, int periodic, int dim, const long long* counts,
                    const double* lengths, double growth, const double* pos, const double* t,
                    long long n_sites, const long long* sample, long long lin_begin, long long n_sample,
                    const int* labels_at, const double* dist_at, int* bad_label, int* bad_value,
                    cudaStream_t st) {
  const BruteGeo g = make_bgeo(kind, periodic, dim, counts, lengths, growth);
  // sample == nullptr: the contiguous voxel range [lin_begin, lin_begin + n_sample)
  dispatch(g, pos, t, n_sites, lin_begin, n_sample, sample, nullptr, nullptr, nullptr, labels_at, dist_at,
           bad_label, bad_value, st);
  return 1;
}

}  // namespace vxb
