// lms_exact.cu -- exact per-vertex anchored-window evaluation and the
// lexicographic argmin.
//
// One CTA evaluates one arrangement vertex (i, j, u) exactly as the
// reference's `_evaluate_pairs` does for one row (backend.py:140-171):
//   v0      = a_i*u - b_i                              (backend.py:144)
//   x_k     = u*a_k - b_k, x_i = x_j = v0              (backend.py:145-148)
//   k_lo    = #(x < v0), k_hi = #(x <= v0) - 1          (backend.py:149-150)
//   down    = k_hi - (q-1), up = k_lo + (q-1)           (backend.py:152-153)
//   h_down  = v0 - vs[down] | inf, h_up = vs[up] - v0 | inf, up wins ties
//                                                       (backend.py:154-161)
// where vs is the sorted cut.  Instead of sorting (the reference's
// O(n log n) per vertex), the two order statistics vs[up] and vs[down] are
// selected by an MSD radix select over order-preserving uint64 keys:
// 8-bit digits, a shared-memory histogram per target, the prefix narrowed
// each pass, finishing early once the target bucket holds one element.
// Every pass recomputes the cut from the lines (16 B/line, L2-resident), so
// the per-vertex state is O(1) and any n fits.
//
// The argmin is the strict lexicographic (height, i, j) minimum of
// _merge / the chunk tie-break (backend.py:165-167, 182-187).

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cmath>
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "lms_common.cuh"
#include "lms_exact_warp.cuh"
#include "lms_kernels.cuh"

namespace lmsb {

namespace {

#ifndef LMSB_EXACT_THREADS
#define LMSB_EXACT_THREADS 256
#endif
constexpr int kExactThreads = LMSB_EXACT_THREADS;
constexpr int kExactWarps = kExactThreads / kWarp;

template <int kW>
struct SelectSharedT {
  unsigned hist[2][256];
  unsigned long long prefix[2];
  long long rank[2];
  unsigned long long result[2];
  int state[2];  // -1 inactive, 0 searching, 1 unique element pending, 2 done
  unsigned red_lt[kW];
  unsigned red_le[kW];
  unsigned red_up[kW];
  unsigned red_dn[kW];
};
using SelectShared = SelectSharedT<kExactWarps>;



// Warp `t` picks the digit bucket containing rank[t] from hist[t].
template <class SM>
__device__ void pick_digit(SM& sm, int t, int level) {
  const int lane = threadIdx.x & 31;
  unsigned h[8];
  unsigned sum = 0;
#pragma unroll
  for (int d = 0; d < 8; ++d) {
    h[d] = sm.hist[t][lane * 8 + d];
    sum += h[d];
  }
  unsigned incl = sum;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    unsigned o = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += o;
  }
  const unsigned excl = incl - sum;
  const long long r = sm.rank[t];
  const bool mine = r >= (long long)excl && r < (long long)incl;
  if (mine) {
    unsigned c = excl;
    int digit = 0;
    unsigned cnt = 0;
#pragma unroll
    for (int d = 0; d < 8; ++d) {
      if (r >= (long long)c && r < (long long)(c + h[d])) {
        digit = lane * 8 + d;
        cnt = h[d];
        break;
      }
      c += h[d];
    }
    sm.prefix[t] = (sm.prefix[t] << 8) | (unsigned long long)digit;
    sm.rank[t] = r - (long long)c;
    if (level == 7) {
      sm.result[t] = sm.prefix[t];
      sm.state[t] = 2;
    } else if (cnt == 1) {
      sm.state[t] = 1;
    }
  }
}

// Exact anchored window at (i, j, u) with anchors snapped to v0.  Must be
// called by all threads of the CTA; thread 0's return value is meaningful.
// When `bound` is finite the vertex is evaluated only if one of its windows
// can reach height <= bound; pass 0 counts, with the reference's own
// arithmetic, the lines x >= v0 with fl(x - v0) <= bound (resp. x <= v0 with
// fl(v0 - x) <= bound).  h_up <= bound iff that count reaches q, because
// fl(x - v0) is monotone in x and vs[up] is the q-th smallest x >= v0
// (backend.py:153,159); otherwise no select is needed and the vertex is
// reported as not found (it cannot win against a record of height bound).
// kCached: pass 0 keeps the order-preserving keys of the cut in shared
// memory (n <= kExactCacheN) and the select passes read them from there
// instead of recomputing the cut from the L2-resident lines.
template <int kT, bool kCached, class SM>
__device__ lms_candidate exact_vertex_t(const double* __restrict__ a,
                                        const double* __restrict__ b, int64_t n, int64_t q,
                                        int64_t i, int64_t j, double u, double v0, double bound,
                                        SM& sm, unsigned long long* cache) {
  constexpr int kW = kT / kWarp;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;

  if (bound < 0.0) return cand_none();  // (uniform) no height can reach it

  // Pass 0: rank counts of v0 in the snapped cut (+ window counts vs bound).
  unsigned lt = 0, le = 0, wu = 0, wd = 0;
  for (int64_t k = tid; k < n; k += kT) {
    double x = snapped_cut(a, b, k, i, j, u, v0);
    if (kCached) cache[k] = key_of(x);
    lt += x < v0;
    le += x <= v0;
    wu += x >= v0 && __dsub_rn(x, v0) <= bound;
    wd += x <= v0 && __dsub_rn(v0, x) <= bound;
  }
  lt = __reduce_add_sync(0xffffffffu, lt);
  le = __reduce_add_sync(0xffffffffu, le);
  wu = __reduce_add_sync(0xffffffffu, wu);
  wd = __reduce_add_sync(0xffffffffu, wd);
  if (lane == 0) {
    sm.red_lt[warp] = lt;
    sm.red_le[warp] = le;
    sm.red_up[warp] = wu;
    sm.red_dn[warp] = wd;
  }
  __syncthreads();
  int64_t c_lt = 0, c_le = 0, c_up = 0, c_dn = 0;
#pragma unroll
  for (int w = 0; w < kW; ++w) {
    c_lt += sm.red_lt[w];
    c_le += sm.red_le[w];
    c_up += sm.red_up[w];
    c_dn += sm.red_dn[w];
  }
  if (isfinite(bound) && c_up < q && c_dn < q) {
    __syncthreads();
    lms_candidate none = cand_none();
    return none;
  }
  const int64_t down = c_le - q;        // k_hi - (q - 1)
  const int64_t up = c_lt + q - 1;      // k_lo + (q - 1)
  const bool ok_down = down >= 0;
  const bool ok_up = up <= n - 1;

  lms_candidate c = cand_none();
  c.i = i;
  c.j = j;
  c.u = u;

  // Both windows inside the class of values equal to v0: vs[up] == vs[down]
  // == v0, so h_up = h_down = 0 and the upward window wins.
  if (c_le - c_lt >= q && isfinite(v0)) {
    c.height = 0.0;
    c.v_low = v0;
    c.v_high = v0;
    c.found = 1;
    __syncthreads();
    return c;
  }

  if (tid < 2) {
    const bool active = tid == 0 ? ok_up : ok_down;
    sm.prefix[tid] = 0ULL;
    sm.rank[tid] = tid == 0 ? up : down;
    sm.result[tid] = 0ULL;
    sm.state[tid] = active ? 0 : -1;
  }
  __syncthreads();

  for (int level = 0; level < 8; ++level) {
    const int shift = 56 - 8 * level;
    const int s0 = sm.state[0];
    const int s1 = sm.state[1];
    if ((s0 == 2 || s0 == -1) && (s1 == 2 || s1 == -1)) break;
    const unsigned long long p0 = sm.prefix[0];
    const unsigned long long p1 = sm.prefix[1];
    for (int e = tid; e < 512; e += kT) (&sm.hist[0][0])[e] = 0u;
    __syncthreads();
    for (int64_t k = tid; k < n; k += kT) {
      const unsigned long long key = kCached ? cache[k] : key_of(snapped_cut(a, b, k, i, j, u, v0));
      const unsigned long long hi = level == 0 ? 0ULL : (key >> (shift + 8));
      const unsigned digit = (unsigned)(key >> shift) & 255u;
      if (s0 == 0 && hi == p0) atomicAdd(&sm.hist[0][digit], 1u);
      if (s1 == 0 && hi == p1) atomicAdd(&sm.hist[1][digit], 1u);
      if (s0 == 1 && hi == p0) sm.result[0] = key;
      if (s1 == 1 && hi == p1) sm.result[1] = key;
    }
    __syncthreads();
    if (warp < 2) {
      const int t = warp;
      const int st = t == 0 ? s0 : s1;
      if (st == 0) pick_digit(sm, t, level);
      else if (st == 1 && lane == 0) sm.state[t] = 2;
    }
    __syncthreads();
  }

  const double v_up = ok_up ? value_of(sm.result[0]) : 0.0;
  const double v_down = ok_down ? value_of(sm.result[1]) : 0.0;
  const double h_down = ok_down ? __dsub_rn(v0, v_down) : INFINITY;
  const double h_up = ok_up ? __dsub_rn(v_up, v0) : INFINITY;
  const bool use_up = h_up <= h_down;
  const double h = use_up ? h_up : h_down;
  if (isfinite(h)) {
    c.height = h;
    c.v_low = use_up ? v0 : v_down;
    c.v_high = use_up ? v_up : v0;
    c.found = 1;
  }
  __syncthreads();
  return c;
}

__device__ __forceinline__ lms_candidate exact_vertex(const double* __restrict__ a,
                                                     const double* __restrict__ b, int64_t n,
                                                     int64_t q, int64_t i, int64_t j, double u,
                                                     double v0, double bound, SelectShared& sm) {
  return exact_vertex_t<kExactThreads, false>(a, b, n, q, i, j, u, v0, bound, sm, nullptr);
}

// Running minimum height of a single-fit exact launch (bits of a
// non-negative double order like its value).  A vertex whose windows all
// exceed it cannot win (a vertex of that height exists), so it is tested
// against it; ties stay (<=), the reduce settles them by (i, j).  The bound
// is uniform across the CTA: one read by thread 0, broadcast.
__device__ __forceinline__ double live_bound(const unsigned long long* live_h) {
  __shared__ double lb;
  __syncthreads();
  if (threadIdx.x == 0) lb = __longlong_as_double((long long)*(volatile const unsigned long long*)live_h);
  __syncthreads();
  return lb;
}

__device__ __forceinline__ void live_lower(unsigned long long* live_h, double h) {
  atomicMin(live_h, (unsigned long long)__double_as_longlong(h + 0.0));
}

// Bound for vertex (i, j) against the fit's record bc: a vertex after bc in
// (i, j) order wins only with a strictly smaller height (backend.py:182-187),
// so its bound drops to the next double below (a negative bound: nothing to
// evaluate, heights are >= 0 -- the many exact ties of collinear inputs).
__device__ __forceinline__ double vertex_bound(const lms_candidate& bc, int64_t i, int64_t j) {
  if (!bc.found) return INFINITY;
  const bool after = i > bc.i || (i == bc.i && j > bc.j);
  return after ? nextafter(bc.height, -INFINITY) : bc.height;
}

__device__ __forceinline__ bool item_vertex(const ExactArgs& args, int64_t s, int32_t& f,
                                            FitDesc& fd, int64_t& i, int64_t& j, double& u,
                                            double& v0, double& bound) {
  f = args.mode == kSrcList ? args.fit_of[s] : 0;
  fd = args.fits[f];
  const double* a = args.a + fd.off;
  const double* b = args.b + fd.off;
  bound = INFINITY;
  if (args.mode == kSrcExplicit) {
    i = args.ii[s];
    j = args.jj[s];
    u = args.uu[s];
    v0 = args.vv ? args.vv[s] : cut_value(u, a[i], b[i]);
    if (args.bound) bound = vertex_bound(args.bound[f], i, j);
    return true;
  }
  decode_rank(fd.n, args.ranks[s], &i, &j);
  if (args.bound) bound = vertex_bound(args.bound[f], i, j);
  const double ai = a[i], aj = a[j];
  // _scan_rank_range drops parallel duals and forms u unfused (backend.py:200-204).
  u = __ddiv_rn(__dsub_rn(b[i], b[j]), __dsub_rn(ai, aj));
  v0 = cut_value(u, ai, b[i]);
  return __dsub_rn(ai, aj) != 0.0;
}

constexpr int kWarpExactWarps = 8;

__global__ void __launch_bounds__(kWarpExactWarps * 32) exact_warp_kernel(ExactArgs args) {
  __shared__ SelectWarp sw[kWarpExactWarps];
  int64_t count = args.d_count ? (int64_t)*args.d_count : args.count;
  if (count > args.capacity) count = args.capacity;
  const int wib = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * kWarpExactWarps + wib;
  const int64_t nw = (int64_t)gridDim.x * kWarpExactWarps;
  for (int64_t s = gw; s < count; s += nw) {
    int32_t f;
    FitDesc fd;
    int64_t i, j;
    double u, v0, bound;
    const bool valid = item_vertex(args, s, f, fd, i, j, u, v0, bound);
    lms_candidate c = cand_none();
    if (valid)
      c = exact_vertex_warp(args.a + fd.off, args.b + fd.off, fd.n, fd.q, i, j, u, v0, bound,
                            sw[wib]);
    c.reserved = f;
    if ((threadIdx.x & 31) == 0) args.out[s] = c;
  }
}

__global__ void __launch_bounds__(kExactThreads) exact_kernel(ExactArgs args) {
  __shared__ SelectShared sm;
  int64_t count = args.d_count ? (int64_t)*args.d_count : args.count;
  if (count > args.capacity) count = args.capacity;
  for (int64_t s = args.begin + blockIdx.x; s < count; s += gridDim.x) {
    const int32_t f = args.mode == kSrcList ? args.fit_of[s] : 0;
    const FitDesc fd = args.fits[f];
    const double* a = args.a + fd.off;
    const double* b = args.b + fd.off;
    double bound = INFINITY;
    int64_t i, j;
    double u, v0;
    bool valid = true;
    if (args.mode == kSrcExplicit) {
      i = args.ii[s];
      j = args.jj[s];
      u = args.uu[s];
      v0 = args.vv ? args.vv[s] : cut_value(u, a[i], b[i]);
      if (args.bound) bound = vertex_bound(args.bound[f], i, j);
    } else {
      decode_rank(fd.n, args.ranks[s], &i, &j);
      if (args.bound) bound = vertex_bound(args.bound[f], i, j);
      const double ai = a[i], aj = a[j];
      // _scan_rank_range drops parallel duals and forms u unfused
      // (backend.py:200-204).
      valid = __dsub_rn(ai, aj) != 0.0;
      u = __ddiv_rn(__dsub_rn(b[i], b[j]), __dsub_rn(ai, aj));
      v0 = cut_value(u, ai, b[i]);
    }
    if (args.live_h) bound = fmin(bound, live_bound(args.live_h));
    lms_candidate c = cand_none();
    if (valid) c = exact_vertex(a, b, fd.n, fd.q, i, j, u, v0, bound, sm);
    c.reserved = f;
    if (threadIdx.x == 0) {
      args.out[s] = c;
      if (args.live_h && c.found) live_lower(args.live_h, c.height);
    }
  }
}

constexpr int kCachedThreads = 1024;

// One vertex per CTA with its cut's keys cached in shared memory: few
// vertices (seeds, band survivors) finish in a fraction of the time the
// L2-streaming exact_kernel needs per vertex.
__global__ void __launch_bounds__(kCachedThreads, 1) exact_cached_kernel(ExactArgs args) {
  using SM = SelectSharedT<kCachedThreads / kWarp>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(smem_raw);
  unsigned long long* cache = reinterpret_cast<unsigned long long*>(smem_raw + ((sizeof(SM) + 15) & ~size_t(15)));
  int64_t count = args.d_count ? (int64_t)*args.d_count : args.count;
  if (count > args.capacity) count = args.capacity;
  if (args.cluster_max > 0 && count <= args.cluster_max) return;  // (the cluster kernel's list)
  if (args.cached_end > 0 && count > args.cached_end) count = args.cached_end;
  for (int64_t s = blockIdx.x; s < count; s += gridDim.x) {
    int32_t f;
    FitDesc fd;
    int64_t i, j;
    double u, v0, bound;
    const bool valid = item_vertex(args, s, f, fd, i, j, u, v0, bound);
    if (args.live_h) bound = fmin(bound, live_bound(args.live_h));
    lms_candidate c = cand_none();
    if (valid)
      c = exact_vertex_t<kCachedThreads, true>(args.a + fd.off, args.b + fd.off, fd.n, fd.q, i, j,
                                               u, v0, bound, sm, cache);
    c.reserved = f;
    if (threadIdx.x == 0) {
      args.out[s] = c;
      if (args.live_h && c.found) live_lower(args.live_h, c.height);
    }
    __syncthreads();
  }
}

// ---- one vertex per 8-CTA cluster (n in (kExactCacheN, 8 kExactCacheN]):
// the cut of a large fit split over the cluster, every CTA caching the keys
// of its eighth in shared memory; the pass-0 counts and every select level's
// digit histograms are summed over distributed shared memory, so all CTAs
// hold the same select state and take the same branches.  A few vertices
// (seeds, survivors) of a 65,536-line fit finish ~8x sooner than with one
// CTA streaming the whole cut from L2 per pass (exact_kernel).
constexpr int kClusterCtas = 8;
constexpr int kClusterThreads = 512;

struct ClusterSelect {
  unsigned hist[2][256];   // the cluster's histogram (pick_digit reads it)
  unsigned local[2][256];  // this CTA's histogram (read by the cluster)
  unsigned long long prefix[2];
  long long rank[2];
  unsigned long long result[2];
  int state[2];
  unsigned long long found_key[2];  // the unique pending element, if in this CTA's slice
  int found[2];
  unsigned red[4][kClusterThreads / kWarp];
  unsigned long long cnt[4];  // this CTA's pass-0 counts (read by the cluster)
  long long tot[4];
  double live;  // rank 0: the fit's running minimum height
};

__device__ lms_candidate exact_vertex_cluster(const double* __restrict__ a,
                                              const double* __restrict__ b, int64_t n, int64_t q,
                                              int64_t i, int64_t j, double u, double v0,
                                              double bound, ClusterSelect& sm,
                                              unsigned long long* cache) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int r = (int)cl.block_rank();
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  if (bound < 0.0) return cand_none();  // (uniform)
  const int64_t m = (n + kClusterCtas - 1) / kClusterCtas;
  const int64_t k0 = min(n, (int64_t)r * m), k1 = min(n, k0 + m);
  const int mine = (int)(k1 - k0);

  unsigned lt = 0, le = 0, wu = 0, wd = 0;
  for (int kk = tid; kk < mine; kk += kClusterThreads) {
    const double x = snapped_cut(a, b, k0 + kk, i, j, u, v0);
    cache[kk] = key_of(x);
    lt += x < v0;
    le += x <= v0;
    wu += x >= v0 && __dsub_rn(x, v0) <= bound;
    wd += x <= v0 && __dsub_rn(v0, x) <= bound;
  }
  lt = __reduce_add_sync(0xffffffffu, lt);
  le = __reduce_add_sync(0xffffffffu, le);
  wu = __reduce_add_sync(0xffffffffu, wu);
  wd = __reduce_add_sync(0xffffffffu, wd);
  if (lane == 0) {
    sm.red[0][warp] = lt;
    sm.red[1][warp] = le;
    sm.red[2][warp] = wu;
    sm.red[3][warp] = wd;
  }
  __syncthreads();
  if (tid < 4) {
    unsigned long long t = 0;
    for (int w = 0; w < kClusterThreads / kWarp; ++w) t += sm.red[tid][w];
    sm.cnt[tid] = t;
  }
  cl.sync();
  if (tid < 4) {
    long long t = 0;
    for (int rr = 0; rr < kClusterCtas; ++rr) t += (long long)cl.map_shared_rank(&sm, rr)->cnt[tid];
    sm.tot[tid] = t;
  }
  __syncthreads();
  const int64_t c_lt = sm.tot[0], c_le = sm.tot[1], c_up = sm.tot[2], c_dn = sm.tot[3];
  // (every CTA read the counts: the next writes of cnt come after the
  // select's cluster barriers or the caller's)
  if (isfinite(bound) && c_up < q && c_dn < q) return cand_none();
  const int64_t down = c_le - q;
  const int64_t up = c_lt + q - 1;
  const bool ok_down = down >= 0;
  const bool ok_up = up <= n - 1;
  lms_candidate c = cand_none();
  c.i = i;
  c.j = j;
  c.u = u;
  if (c_le - c_lt >= q && isfinite(v0)) {
    c.height = 0.0;
    c.v_low = v0;
    c.v_high = v0;
    c.found = 1;
    return c;
  }
  if (tid < 2) {
    const bool active = tid == 0 ? ok_up : ok_down;
    sm.prefix[tid] = 0ULL;
    sm.rank[tid] = tid == 0 ? up : down;
    sm.result[tid] = 0ULL;
    sm.state[tid] = active ? 0 : -1;
  }
  __syncthreads();
  for (int level = 0; level < 8; ++level) {
    const int shift = 56 - 8 * level;
    const int s0 = sm.state[0];
    const int s1 = sm.state[1];
    if ((s0 == 2 || s0 == -1) && (s1 == 2 || s1 == -1)) break;  // (same in every CTA)
    const unsigned long long p0 = sm.prefix[0];
    const unsigned long long p1 = sm.prefix[1];
    for (int e = tid; e < 512; e += kClusterThreads) (&sm.local[0][0])[e] = 0u;
    if (tid < 2) sm.found[tid] = 0;
    __syncthreads();
    for (int kk = tid; kk < mine; kk += kClusterThreads) {
      const unsigned long long key = cache[kk];
      const unsigned long long hi = level == 0 ? 0ULL : (key >> (shift + 8));
      const unsigned digit = (unsigned)(key >> shift) & 255u;
      if (s0 == 0 && hi == p0) atomicAdd(&sm.local[0][digit], 1u);
      if (s1 == 0 && hi == p1) atomicAdd(&sm.local[1][digit], 1u);
      if (s0 == 1 && hi == p0) { sm.found_key[0] = key; sm.found[0] = 1; }
      if (s1 == 1 && hi == p1) { sm.found_key[1] = key; sm.found[1] = 1; }
    }
    cl.sync();
    for (int e = tid; e < 512; e += kClusterThreads) {
      unsigned t = 0;
      for (int rr = 0; rr < kClusterCtas; ++rr) t += (&cl.map_shared_rank(&sm, rr)->local[0][0])[e];
      (&sm.hist[0][0])[e] = t;
    }
    if (tid < 2) {  // (after its share of the histogram sum)
      const int t = tid;
      if ((t == 0 ? s0 : s1) == 1)
        for (int rr = 0; rr < kClusterCtas; ++rr) {
          const ClusterSelect* o = cl.map_shared_rank(&sm, rr);
          if (o->found[t]) sm.result[t] = o->found_key[t];
        }
    }
    __syncthreads();
    if (warp < 2) {
      const int t = warp;
      const int st = t == 0 ? s0 : s1;
      if (st == 0) pick_digit(sm, t, level);
      else if (st == 1 && lane == 0) sm.state[t] = 2;
    }
    cl.sync();  // the histograms were read; the state is settled in every CTA
  }
  const double v_up = ok_up ? value_of(sm.result[0]) : 0.0;
  const double v_down = ok_down ? value_of(sm.result[1]) : 0.0;
  const double h_down = ok_down ? __dsub_rn(v0, v_down) : INFINITY;
  const double h_up = ok_up ? __dsub_rn(v_up, v0) : INFINITY;
  const bool use_up = h_up <= h_down;
  const double h = use_up ? h_up : h_down;
  if (isfinite(h)) {
    c.height = h;
    c.v_low = use_up ? v0 : v_down;
    c.v_high = use_up ? v_up : v0;
    c.found = 1;
  }
  return c;
}

__global__ void __cluster_dims__(kClusterCtas, 1, 1) __launch_bounds__(kClusterThreads, 1)
    exact_cluster_kernel(ExactArgs args) {
  namespace cg = cooperative_groups;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ClusterSelect& sm = *reinterpret_cast<ClusterSelect*>(smem_raw);
  unsigned long long* cache =
      reinterpret_cast<unsigned long long*>(smem_raw + ((sizeof(ClusterSelect) + 15) & ~size_t(15)));
  cg::cluster_group cl = cg::this_cluster();
  const int r = (int)cl.block_rank();
  int64_t count = args.d_count ? (int64_t)*args.d_count : args.count;
  if (count > args.capacity) count = args.capacity;
  if (args.cluster_max > 0 && count > args.cluster_max) return;  // (the cached kernel's list)
  if (args.cached_end > 0 && count > args.cached_end) count = args.cached_end;
  const int64_t nclusters = gridDim.x / kClusterCtas;
  for (int64_t s = blockIdx.x / kClusterCtas; s < count; s += nclusters) {
    int32_t f;
    FitDesc fd;
    int64_t i, j;
    double u, v0, bound;
    const bool valid = item_vertex(args, s, f, fd, i, j, u, v0, bound);
    if (args.live_h) {  // one read for the whole cluster (uniform branches)
      if (r == 0 && threadIdx.x == 0)
        sm.live = __longlong_as_double((long long)*(volatile const unsigned long long*)args.live_h);
      cl.sync();
      bound = fmin(bound, cl.map_shared_rank(&sm, 0)->live);
    }
    lms_candidate c = cand_none();
    if (valid)
      c = exact_vertex_cluster(args.a + fd.off, args.b + fd.off, fd.n, fd.q, i, j, u, v0, bound,
                               sm, cache);
    c.reserved = f;
    if (r == 0 && threadIdx.x == 0) {
      args.out[s] = c;
      if (args.live_h && c.found) live_lower(args.live_h, c.height);
    }
    cl.sync();  // every remote read of this vertex is done
  }
}

// K1 of the materialised two-kernel flow (_materialized_inputs,
// backend.py:210-219; the paper's intersection kernel): every pair of ranks
// [r0, r0 + count) with a_i != a_j becomes an explicit (i, j, u) triple,
// u = (b_i - b_j) / (a_i - a_j) unfused; compacted in any order (the
// lexicographic reduce does not depend on it).
__global__ void materialize_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                   int64_t n, int64_t r0, int64_t count, int64_t* __restrict__ ii,
                                   int64_t* __restrict__ jj, double* __restrict__ uu,
                                   unsigned long long* __restrict__ nout) {
  const int lane = threadIdx.x & 31;
  const int64_t cend = ((count + 31) / 32) * 32;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < cend;
       t += (int64_t)gridDim.x * blockDim.x) {
    bool keep = false;
    int64_t i = 0, j = 0;
    double u = 0.0;
    if (t < count) {
      decode_rank(n, r0 + t, &i, &j);
      const double da = __dsub_rn(a[i], a[j]);
      keep = da != 0.0;
      u = __ddiv_rn(__dsub_rn(b[i], b[j]), da);
    }
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (m) {
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(nout, (unsigned long long)__popc(m));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (keep) {
        const unsigned long long pos = base + __popc(m & ((1u << lane) - 1u));
        ii[pos] = i;
        jj[pos] = j;
        uu[pos] = u;
      }
    }
  }
}

// 128-bit CAS on a BestKey (atom.global.cas.b128, sm_90+).
__device__ __forceinline__ BestKey cas_key(BestKey* addr, BestKey expect, BestKey desired) {
  BestKey old;
  asm volatile(
      "{\n .reg .b128 e, d, o;\n mov.b128 e, {%2, %3};\n mov.b128 d, {%4, %5};\n"
      " atom.global.cas.b128 o, [%6], e, d;\n mov.b128 {%0, %1}, o;\n}"
      : "=l"(old.lo), "=l"(old.hi)
      : "l"(expect.lo), "l"(expect.hi), "l"(desired.lo), "l"(desired.hi), "l"(addr)
      : "memory");
  return old;
}

__device__ __forceinline__ bool key_less(const BestKey& x, const BestKey& y) {
  return x.hi < y.hi || (x.hi == y.hi && x.lo < y.lo);
}

// (height, i, j) -> 128-bit key: heights are finite and >= 0 (or -0.0, which
// ties +0.0), so the bits of h + 0.0 order like the values; the pair rank
// orders like (i, j) (row-major triangle).
__device__ __forceinline__ BestKey record_key(const lms_candidate& c, int64_t n) {
  BestKey k;
  k.hi = (unsigned long long)__double_as_longlong(c.height + 0.0);
  k.lo = (unsigned long long)(row_offset(n, c.i) + (c.j - c.i - 1));
  return k;
}

__global__ void reduce_cas_kernel(const lms_candidate* __restrict__ recs,
                                  const unsigned long long* d_count, int64_t count,
                                  int64_t capacity, const FitDesc* __restrict__ fits,
                                  BestKey* keys) {
  if (d_count) count = (int64_t)*d_count;
  if (count > capacity) count = capacity;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < count;
       s += (int64_t)gridDim.x * blockDim.x) {
    const lms_candidate c = recs[s];
    if (!c.found) continue;
    const BestKey k = record_key(c, fits[c.reserved].n);
    BestKey* addr = keys + c.reserved;
    BestKey cur = *addr;  // a torn read only costs one failed CAS
    while (key_less(k, cur)) {
      const BestKey prev = cas_key(addr, cur, k);
      if (prev.lo == cur.lo && prev.hi == cur.hi) break;
      cur = prev;
    }
  }
}

__global__ void publish_kernel(const lms_candidate* __restrict__ recs,
                               const unsigned long long* d_count, int64_t count, int64_t capacity,
                               const FitDesc* __restrict__ fits, const BestKey* __restrict__ keys,
                               lms_candidate* __restrict__ best) {
  if (d_count) count = (int64_t)*d_count;
  if (count > capacity) count = capacity;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < count;
       s += (int64_t)gridDim.x * blockDim.x) {
    lms_candidate c = recs[s];
    if (!c.found) continue;
    const int32_t f = c.reserved;
    const BestKey k = record_key(c, fits[f].n);
    const BestKey w = keys[f];
    if (k.lo == w.lo && k.hi == w.hi) {  // duplicates of one vertex are identical
      c.reserved = 0;
      best[f] = c;
    }
  }
}

__global__ void reset_best_kernel(BestKey* keys, lms_candidate* best, int64_t nfits) {
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < nfits;
       f += (int64_t)gridDim.x * blockDim.x) {
    keys[f].lo = ~0ULL;
    keys[f].hi = ~0ULL;
    best[f] = cand_none();
  }
}

__global__ void gen_seeds_kernel(const FitDesc* __restrict__ fits,
                                 const int64_t* __restrict__ seed_prefix, int64_t nfits,
                                 int64_t* __restrict__ ranks, int32_t* __restrict__ fit_of) {
  const int64_t total = seed_prefix[nfits];
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < total;
       s += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = nfits - 1;  // largest f with seed_prefix[f] <= s
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (seed_prefix[mid] <= s) lo = mid;
      else hi = mid - 1;
    }
    const FitDesc fd = fits[lo];
    const int64_t k = s - seed_prefix[lo];
    const int64_t cnt = seed_prefix[lo + 1] - seed_prefix[lo];
    const int64_t span = fd.rank_hi - fd.rank_lo;
    ranks[s] = fd.rank_lo + ((2 * k + 1) * span) / (2 * cnt);
    fit_of[s] = (int32_t)lo;
  }
}

}  // namespace

// LMSB_EXACT_CLUSTER=0 keeps one streaming CTA per vertex for n > kExactCacheN
bool exact_cluster_enabled() {
  const char* e = getenv("LMSB_EXACT_CLUSTER");
  return !(e && e[0] == '0');
}

// short lists of a fit with n <= kExactCacheN: the cluster kernel when the
// list has at most this many vertices (LMSB_EXACT_CLUSTER_MAX; 0: never)
int64_t exact_cluster_max() {
  const char* e = getenv("LMSB_EXACT_CLUSTER_MAX");
  return e ? atoll(e) : 36;
}

template <class Kern>
void launch_cluster_exact(Kern kern, const ExactArgs& args, int64_t max_n, int64_t cluster_max,
                          cudaStream_t stream) {
  const int64_t m = (max_n + kClusterCtas - 1) / kClusterCtas;
  const size_t smem = ((sizeof(ClusterSelect) + 15) & ~size_t(15)) + sizeof(unsigned long long) * m;
  static DeviceOnce done;
  set_max_smem(kern,
               ((sizeof(ClusterSelect) + 15) & ~size_t(15)) +
                   sizeof(unsigned long long) * kExactCacheN,
               done);
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int clusters = std::max(1, sms / kClusterCtas);
  ExactArgs head = args;
  head.cluster_max = cluster_max;
  if (head.cached_end <= 0 || head.cached_end > (int64_t)clusters * 8)
    head.cached_end = (int64_t)clusters * 8;
  kern<<<clusters * kClusterCtas, kClusterThreads, smem, stream>>>(head);
}

void launch_exact(const ExactArgs& args, int grid, cudaStream_t stream, int64_t max_n) {
  if (grid <= 0) return;
  const int64_t cmax = exact_cluster_max();
  if (args.cached && max_n <= kExactCacheN && max_n > kWarpExactMaxN && cmax > 0 &&
      exact_cluster_enabled()) {
    // a short list by clusters, a long one by the per-SM cached kernel (each
    // kernel reads the device count and returns when the list is the other's)
    launch_cluster_exact(exact_cluster_kernel, args, max_n, cmax, stream);
    ExactArgs longl = args;
    longl.cluster_max = cmax;
    using SM = SelectSharedT<kCachedThreads / kWarp>;
    const size_t smem = ((sizeof(SM) + 15) & ~size_t(15)) + sizeof(unsigned long long) * max_n;
    static DeviceOnce done2;
    set_max_smem(exact_cached_kernel,
                 ((sizeof(SM) + 15) & ~size_t(15)) + sizeof(unsigned long long) * kExactCacheN,
                 done2);
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    exact_cached_kernel<<<sms, kCachedThreads, smem, stream>>>(longl);
    if (args.cached_end <= 0) return;
    ExactArgs rest = args;
    rest.begin = args.cached_end;
    rest.cached = 0;
    exact_kernel<<<grid, kExactThreads, 0, stream>>>(rest);
    return;
  }
  if (args.cached && max_n <= kExactCacheN && max_n > kWarpExactMaxN) {
    using SM = SelectSharedT<kCachedThreads / kWarp>;
    const size_t smem = ((sizeof(SM) + 15) & ~size_t(15)) + sizeof(unsigned long long) * max_n;
    static DeviceOnce done;
    set_max_smem(exact_cached_kernel,
                 ((sizeof(SM) + 15) & ~size_t(15)) + sizeof(unsigned long long) * kExactCacheN,
                 done);
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    exact_cached_kernel<<<sms, kCachedThreads, smem, stream>>>(args);
    if (args.cached_end <= 0) return;
    // the rest of a long list (beyond cached_end) streams
    ExactArgs rest = args;
    rest.begin = args.cached_end;
    rest.cached = 0;
    exact_kernel<<<grid, kExactThreads, 0, stream>>>(rest);
    return;
  }
  if (args.cached && max_n > kExactCacheN && max_n <= kClusterCtas * kExactCacheN &&
      exact_cluster_enabled()) {
    // the first 8 vertices per cluster here, the rest of a long list streams
    launch_cluster_exact(exact_cluster_kernel, args, max_n, 0, stream);
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    ExactArgs rest = args;
    rest.begin = std::min<int64_t>(args.cached_end > 0 ? args.cached_end : INT64_MAX,
                                   (int64_t)std::max(1, sms / kClusterCtas) * 8);
    rest.cached = 0;
    exact_kernel<<<grid, kExactThreads, 0, stream>>>(rest);
    return;
  }
  if (max_n <= kWarpExactMaxN) {
    exact_warp_kernel<<<grid, kWarpExactWarps * 32, 0, stream>>>(args);
  } else {
    exact_kernel<<<grid, kExactThreads, 0, stream>>>(args);
  }
}

void launch_reduce(const lms_candidate* recs, const unsigned long long* d_count, int64_t count,
                   int64_t capacity, const FitDesc* fits, BestKey* keys, lms_candidate* best,
                   int grid, cudaStream_t stream) {
  if (grid <= 0) return;
  reduce_cas_kernel<<<grid, 256, 0, stream>>>(recs, d_count, count, capacity, fits, keys);
  publish_kernel<<<grid, 256, 0, stream>>>(recs, d_count, count, capacity, fits, keys, best);
}

void launch_reset_best(BestKey* keys, lms_candidate* best, int64_t nfits, cudaStream_t stream) {
  const int grid = (int)((nfits + 255) / 256);
  reset_best_kernel<<<grid > 0 ? grid : 1, 256, 0, stream>>>(keys, best, nfits);
}

void launch_materialize(const double* a, const double* b, int64_t n, int64_t r0, int64_t count,
                        int64_t* ii, int64_t* jj, double* uu, unsigned long long* nout, int sms,
                        cudaStream_t stream) {
  if (count <= 0) return;
  materialize_kernel<<<sms * 8, 256, 0, stream>>>(a, b, n, r0, count, ii, jj, uu, nout);
}

void launch_gen_seeds(const FitDesc* fits, const int64_t* seed_prefix, int64_t nfits,
                      int64_t* ranks, int32_t* fit_of, cudaStream_t stream) {
  gen_seeds_kernel<<<512, 256, 0, stream>>>(fits, seed_prefix, nfits, ranks, fit_of);
}

// ---------------------------------------------------------------- contacts
// solve_lms tail (solver.py:122-140): cut_k = x_k u - y_k (numpy's unfused
// product and difference), the anchor pair snapped to x_i u - y_i;
// tol = GEOM_EPS * max(1, max_k |cut_k|); k touches when |cut_k - v_low| <= tol
// or |cut_k - v_high| <= tol.
namespace {
__device__ __forceinline__ double contact_cut(const double* a, const double* b, int64_t k,
                                              int64_t i, int64_t j, double u) {
  const int64_t kk = (k == j) ? i : k;
  return cut_value(u, a[kk], b[kk]);
}

__global__ void contacts_max_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                    int64_t n, int64_t i, int64_t j, double u,
                                    unsigned long long* __restrict__ maxbits) {
  unsigned long long m = 0;  // bits of non-negative doubles order like their values
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long v = (unsigned long long)__double_as_longlong(fabs(contact_cut(a, b, k, i, j, u)));
    m = v > m ? v : m;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const unsigned long long o = __shfl_xor_sync(0xffffffffu, m, off);
    m = o > m ? o : m;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(maxbits, m);
}

__global__ void contacts_collect_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                        int64_t n, int64_t i, int64_t j, double u, double v_low,
                                        double v_high, const unsigned long long* __restrict__ maxbits,
                                        int64_t* __restrict__ out, int64_t cap,
                                        unsigned long long* __restrict__ count) {
  const double tol = 1e-9 * fmax(1.0, __longlong_as_double((long long)*maxbits));
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const double x = contact_cut(a, b, k, i, j, u);
    if (fabs(__dsub_rn(x, v_low)) <= tol || fabs(__dsub_rn(x, v_high)) <= tol) {
      const unsigned long long pos = atomicAdd(count, 1ull);
      if ((int64_t)pos < cap) out[pos] = k;
    }
  }
}
}  // namespace

// Batched contact sets: one CTA per fit (grid-stride over fits), the fit's
// max |cut| by a block reduction, then a flag per point (fit-local anchors
// snapped as in contact_cut).
__global__ void __launch_bounds__(256) contacts_batch_kernel(const double* __restrict__ a,
                                                             const double* __restrict__ b,
                                                             const int64_t* __restrict__ offs,
                                                             const lms_candidate* __restrict__ recs,
                                                             int64_t nfits,
                                                             uint8_t* __restrict__ flags) {
  __shared__ unsigned long long red[8];
  for (int64_t f = blockIdx.x; f < nfits; f += gridDim.x) {
    const int64_t o = offs[f], n = offs[f + 1] - o;
    const lms_candidate r = recs[f];
    if (!r.found) {
      for (int64_t k = threadIdx.x; k < n; k += blockDim.x) flags[o + k] = 0;
      continue;
    }
    unsigned long long m = 0;
    for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
      const unsigned long long v =
          (unsigned long long)__double_as_longlong(fabs(contact_cut(a + o, b + o, k, r.i, r.j, r.u)));
      m = v > m ? v : m;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const unsigned long long x = __shfl_xor_sync(0xffffffffu, m, off);
      m = x > m ? x : m;
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    m = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = red[w] > m ? red[w] : m;
    const double tol = 1e-9 * fmax(1.0, __longlong_as_double((long long)m));
    for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
      const double x = contact_cut(a + o, b + o, k, r.i, r.j, r.u);
      flags[o + k] = (fabs(__dsub_rn(x, r.v_low)) <= tol || fabs(__dsub_rn(x, r.v_high)) <= tol);
    }
    __syncthreads();  // red reused by the next fit
  }
}

void launch_contacts_batch(const double* a, const double* b, const int64_t* offs,
                           const lms_candidate* recs, int64_t nfits, uint8_t* flags, int sms,
                           cudaStream_t st) {
  if (nfits <= 0) return;
  const int grid = (int)std::min<int64_t>(nfits, (int64_t)sms * 8);
  contacts_batch_kernel<<<grid, 256, 0, st>>>(a, b, offs, recs, nfits, flags);
}

void launch_contacts(const double* a, const double* b, int64_t n, const lms_candidate& rec,
                     unsigned long long* scratch, int64_t* out, int64_t cap, int sms,
                     cudaStream_t st) {
  cudaMemsetAsync(scratch, 0, 2 * sizeof(unsigned long long), st);
  const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)sms * 8);
  contacts_max_kernel<<<grid, 256, 0, st>>>(a, b, n, rec.i, rec.j, rec.u, scratch);
  contacts_collect_kernel<<<grid, 256, 0, st>>>(a, b, n, rec.i, rec.j, rec.u, rec.v_low,
                                                rec.v_high, scratch, out, cap, scratch + 1);
}

}  // namespace lmsb
