// lms_band.cu -- slope-band pruning of the exact LMS search.
//
// The reference evaluates every arrangement vertex against every line
// (backend.py:125-179, O(n) per vertex after an O(n log n) sort).  The count
// filter (lms_filter32m.cu) needs > n - q line tests before it can reject a
// vertex.  This stage rejects whole groups of vertices at once and the rest
// in O(log n) each, by grouping vertices of similar slope into bands that
// share one sorted view of the lines.
//
// Geometry.  Re-centre the dual lines on c (the middle of the a-range):
// y'_k(u) = (a_k - c) u - b_k differs from the cut value u a_k - b_k by the
// same c u for every k, so window membership is unchanged.  For a band of
// vertices with slopes in [uL, uR] and centre uM, every line satisfies
//   |y'_k(u) - m_k| <= dev * |u - uM| =: D_v,   m_k = (a_k - c) uM - b_k,
// with dev = max_k |a_k - c|.  Vertex v = (i, j, u) with anchor ordinate
// v0 = a_i u - b_i and z = v0 - c u has h_up <= H only if at least q lines
// have y'_k - z in [0, H] (backend.py:153,159; anchors and ties included),
// hence only if at least q of the band's sorted keys m_k lie in
// [z - D_v - E_v, z + H + D_v + E_v] (and symmetrically for h_down).  Binary
// searches in the band's sorted keys (shared memory) count that.
//
// Band lower bound.  If v has height h, q keys lie in an interval of width
// h + 2 D_v + 2 E_v, so h >= W_q - 2 D_max - 2 E_max with W_q the narrowest
// q-window of the sorted keys.  Bands whose bound exceeds H are never
// touched again; the lowest bounds point at the bands where the optimum
// lives, and the sampled vertices of those bands seed H.
//
// Error budget (amax = max|a|, bmax = max|b|): the reference's roundings of
// u a_k - b_k, v0 and fl(x - v0) <= H move membership by at most
// 2^-49 (|u| amax + bmax + H); z = fl(v0 - fl(c u)) adds 2^-50 (2|u| amax +
// bmax); keys are fp64-formed and rounded to fp32 once: <= 2^-23 (|uM| dev +
// bmax).  E_v = 2^-20 (|u| amax + bmax + H + |uM| dev) + 1e-300 covers the
// sum with a wide margin; dev and the band half-width are padded upward and
// window ends are rounded outward to fp32.  Survivors are re-evaluated
// bit-exactly (lms_exact.cu), so this stage only has to return a superset.
//
// Pipeline per fit (pair ranks [R0, R0 + span)):
//   sample   S stratified vertex slopes -> CUB sort -> K-1 boundaries: the
//            sample minimum, quantiles, just above the sample maximum (so the
//            two outer bands hold only the extremes)
//   bound    per inner band: slope extent from its boundaries, sorted keys,
//            W_q, lower bound (one CTA per band, no vertex touched)
//   seeds    the samples that fall in the lowest-bound bands (exact stage)
//   collect  one pass over all vertices: those in bands whose bound admits
//            H (and any beyond the fp32 key range) are appended, then
//            grouped by band (CUB radix sort on the band id)
//   filter   per collected band: window counts of every member; survivors
//            go to the exact stage

#include <cub/block/block_radix_sort.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_segmented_radix_sort.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "lms_band.cuh"
#include "lms_band_dev.cuh"
#include "lms_common.cuh"

namespace lmsb {

namespace {

#ifndef LMSB_RADIX_BITS
#define LMSB_RADIX_BITS 6  // 6 bits: config 2 0.811 -> 0.797 ms (4: 8 passes, 5 or 6: 6 or 7)
#endif
constexpr int kCollectThreads = 512;
#ifndef LMSB_COLLECT_STEP
#define LMSB_COLLECT_STEP 4
#endif
constexpr int kCollectStep = LMSB_COLLECT_STEP;  // vertices per lane per collect step
constexpr int kCollectQueue = 32 * (kCollectStep + 1);  // per-warp queue: < 32 waiting + a step
constexpr unsigned kSeedPerBand = 16;  // sampled vertices per seed band (safety net)
#ifndef LMSB_COLLECT_RUN
#define LMSB_COLLECT_RUN 64
#endif
constexpr int kRun = LMSB_COLLECT_RUN;  // ranks per lane per warp segment (lane-interleaved)
static_assert(kRun % kCollectStep == 0, "whole collect steps per segment");

__device__ __forceinline__ float rcp_approx_ftz(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__global__ void band_interleave_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                       int64_t n, double2* __restrict__ ab) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    ab[k] = make_double2(a[k], b[k]);
}

// Members per filter chunk of a group of `cnt` members: `chunk`, or (adaptive,
// when that gives fewer) an even split into min(kMinChunks, cnt / kMinChunkMembers) chunks,
// so a group with few members (one rank's share of a band in a sharded
// search) still gets chunks of a narrow slope range.
constexpr int64_t kMinChunks = 4;
constexpr int64_t kMinChunkMembers = 2048;
__host__ __device__ __forceinline__ int64_t chunk_size(int64_t cnt, int64_t chunk, bool adaptive) {
  if (!adaptive || cnt <= 0) return chunk;
  const int64_t nc = (cnt + chunk - 1) / chunk;
  int64_t want = (cnt + kMinChunkMembers - 1) / kMinChunkMembers;
  want = want < kMinChunks ? want : kMinChunks;
  return nc >= want ? chunk : (cnt + want - 1) / want;
}

__device__ __forceinline__ int64_t sample_rank(const BandFit& bf, int64_t S, int64_t s) {
  return bf.P0 + ((2 * s + 1) * bf.pspan) / (2 * S);
}

__global__ void band_sample_kernel(BandFit bf, int64_t S, float* __restrict__ keys,
                                   unsigned long long* __restrict__ nvalid) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < S;
       s += (int64_t)gridDim.x * blockDim.x) {
    int64_t i, j;
    decode_rank(bf.n, sample_rank(bf, S, s), &i, &j);
    double u = 0.0;
    const bool ok = classify(bf, bf.a[i], bf.b[i], bf.a[j], bf.b[j], &u) == 1;
    keys[s] = ok ? band_key(u) : INFINITY;
    if (ok) atomicAdd(nvalid, 1ull);
  }
}

// K >= 3 bands from the sorted valid samples s[0 .. sv): boundary 0 = s[0],
// boundary K-2 = just above s[sv-1], boundaries 1..K-3 = quantiles.
__global__ void band_bounds_kernel(const float* __restrict__ sorted,
                                   const unsigned long long* __restrict__ nvalid, int K,
                                   float* __restrict__ bounds) {
  const int64_t sv = (int64_t)*nvalid;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < K - 1; k += gridDim.x * blockDim.x) {
    float v = INFINITY;
    if (sv > 0) {
      if (k == 0) v = sorted[0];
      else if (k == K - 2) v = nextafterf(sorted[sv - 1], INFINITY);
      else v = sorted[(k * sv) / (K - 2)];
    }
    bounds[k] = v;
  }
}

// ------------------------------------------------------------------ per band
template <int kThreads, int kItems>
struct BandShared {
  using Sort = cub::BlockRadixSort<float, kThreads, kItems, cub::NullType, LMSB_RADIX_BITS>;
  union {
    typename Sort::TempStorage sort;
    float keys[kThreads * kItems];
  };
  double red[2][kThreads / 32];
  int kstar;
};

// Two branch-free binary searches in lockstep (independent loads in flight):
// *lo = first index with k >= xl, *up = first index with k > xu (n >= 1).
__device__ __forceinline__ void lower_upper(const float* __restrict__ k, int n, float xl, float xu,
                                            int* lo, int* up) {
  int bl = 0, bu = 0, len = n;
  while (len > 1) {
    const int half = len >> 1;
    bl = k[bl + half] < xl ? bl + half : bl;
    bu = k[bu + half] <= xu ? bu + half : bu;
    len -= half;
  }
  *lo = bl + (k[bl] < xl);
  *up = bu + (k[bu] <= xu);
}

template <int kThreads>
__device__ __forceinline__ double block_min(double v, double* red) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, off));
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  if (kThreads <= 32) return red[0];
  // every warp reduces the partials with shuffles (no serial smem loop)
  const int lane = threadIdx.x & 31;
  double r = lane < kThreads / 32 ? red[lane] : INFINITY;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) r = fmin(r, __shfl_xor_sync(0xffffffffu, r, off));
  return r;
}

__device__ __forceinline__ double slack_base(const BandFit& bf, double umag, double uM) {
  return 0x1p-20 * (umag * bf.amax + bf.bmax + fabs(uM) * bf.dev);
}

// Slope extent of an inner band from its boundaries: members satisfy
// b_{k-1} <= fl32(u) < b_k, so prev(b_{k-1}) < u < b_k.  false for the outer
// bands (their extent comes from the members).
__device__ __forceinline__ bool boundary_extent(const float* __restrict__ bounds, int K, int band,
                                                double* uL, double* uR) {
  if (band <= 0 || band >= K - 1) return false;
  const float lo = bounds[band - 1], hi = bounds[band];
  *uL = (double)nextafterf(lo, -INFINITY);
  *uR = (double)hi;
  return isfinite(*uL) && isfinite(*uR) && *uL <= *uR;
}

__device__ __forceinline__ bool keys_in_range(const BandFit& bf, double uL, double uR) {
  return fmax(fabs(uL), fabs(uR)) * bf.dev + bf.bmax < 1e37;
}

// Slope bound of a band: at slope u the line values v_k = a_k u - b_k lie
// within bmax of a_k u, so any window holding q of them is at least
// |u| W_q(a) - 2 bmax wide, and a vertex's height is at least that window
// (h_up, h_down each span q values at u; backend.py:153-159).  The
// reference's roundings move it by <= 2^-48 (|u| amax + bmax); margins of
// 2^-40 here.  Linear in |u|, so the band's smallest |u| bounds all of it
// (fl32(u) in [b_{k-1}, b_k): |u| >= that end less 2^-20).  -inf when the
// band reaches u = 0 or no W_q(a) bound is known.
__device__ __forceinline__ double slope_lb(const BandFit& bf, const BandArgs& ba, int band) {
  if (!ba.wqa) return -INFINITY;
  const double wqa = *ba.wqa;
  const double lo = band > 0 ? (double)ba.bounds[band - 1] : -INFINITY;
  const double hi = band < ba.K - 1 ? (double)ba.bounds[band] : INFINITY;
  double umin;
  if (lo > 0.0) umin = lo;
  else if (hi < 0.0) umin = -hi;
  else return -INFINITY;
  umin *= 1.0 - 0x1p-20;
  const double slope = wqa * (1.0 - 0x1p-40) - 0x1p-40 * bf.amax;
  if (!(slope > 0.0) || !isfinite(umin)) return -INFINITY;
  return umin * slope * (1.0 - 0x1p-40) - 2.0 * bf.bmax * (1.0 + 0x1p-38) - 1e-300;
}

// sorted keys m_k = (a_k - c) uM - b_k of the band into sh.keys (the input
// arrangement is irrelevant to a sort, so lines are loaded striped, i.e.
// coalesced, and the result is written striped, i.e. bank-conflict free)
template <int kThreads, int kItems>
__device__ __forceinline__ void band_keys(const BandFit& bf, double uM,
                                          BandShared<kThreads, kItems>& sh) {
  const int tid = threadIdx.x;
  const int n = (int)bf.n;
  float keys[kItems];
#pragma unroll
  for (int e = 0; e < kItems; ++e) {
    const int k = e * kThreads + tid;
    keys[e] = k < n ? (float)__dsub_rn(__dmul_rn(__dsub_rn(__ldg(bf.a + k), bf.c), uM), __ldg(bf.b + k))
                    : INFINITY;
  }
  typename BandShared<kThreads, kItems>::Sort(sh.sort).SortBlockedToStriped(keys);
  __syncthreads();
#pragma unroll
  for (int e = 0; e < kItems; ++e) sh.keys[e * kThreads + tid] = keys[e];
  __syncthreads();
}

// keys around the narrowest q-window [K[k*], K[k*+q-1]] of a band: the lines
// there bound the best window at the band's centre slope; pairs among them
// seed H (band_edge_seed_kernel)
__device__ __forceinline__ void write_edges(const float* K, int n, int q, int ks, float* e) {
#pragma unroll
  for (int t = 0; t < kEdge; ++t) {
    const int lo = min(max(ks + t - kEdge / 2, 0), n - 1);
    const int hi = min(max(ks + q - 1 + t - kEdge / 2, 0), n - 1);
    e[t] = K[lo];
    e[kEdge + t] = K[hi];
  }
}

// mode 0: lower bound of every inner band (grid = K)
template <int kThreads, int kItems>
__global__ void __launch_bounds__(kThreads, 1) band_bound_kernel(BandFit bf, BandArgs ba) {
  using SH = BandShared<kThreads, kItems>;
  extern __shared__ __align__(16) unsigned char band_smem[];
  SH& sh = *reinterpret_cast<SH*>(band_smem);
  const int band = ba.band_ids ? ba.band_ids[ba.band0 + (int)blockIdx.x] : ba.band0 + (int)blockIdx.x;
  if (band < 0) return;
  double uL, uR;
  if (!boundary_extent(ba.bounds, ba.K, band, &uL, &uR) || !keys_in_range(bf, uL, uR)) {
    if (threadIdx.x == 0) {
      ba.lb[band] = slope_lb(bf, ba, band);  // outer / unbounded: only the slope bound
      ba.wq[band] = INFINITY;
    }
    return;
  }
  if (ba.defer) {  // (uniform per CTA)
    const double slb = slope_lb(bf, ba, band);
    const bool deferred = slb > 0.0;
    if (ba.defer == 1 && deferred) {
      if (threadIdx.x == 0) {
        ba.lb[band] = slb;
        ba.wq[band] = INFINITY;
      }
      return;
    }
    if (ba.defer == 2) {
      if (!deferred) return;
      const lms_candidate best = *ba.best;
      // a band whose slope bound exceeds the seeds' H keeps it: dismissed
      if (best.found && slb > best.height * (1.0 + 0x1p-19)) return;
    }
  }
  const double uM = 0.5 * uL + 0.5 * uR;
  const double dmax = bf.dev * fmax(uR - uM, uM - uL) * (1.0 + 0x1p-40);
  band_keys<kThreads, kItems>(bf, uM, sh);
  const int n = (int)bf.n, q = (int)bf.q;
  if (ba.bkeys) {  // kept for the filter (row padded to a multiple of 4 keys)
    float* row = ba.bkeys + (int64_t)band * ba.bkeys_ld;
    for (int k = threadIdx.x; k < ba.bkeys_ld; k += kThreads) row[k] = k < n ? sh.keys[k] : INFINITY;
  }
  double w = INFINITY;
  for (int k = threadIdx.x; k + q - 1 < n; k += kThreads)
    w = fmin(w, (double)sh.keys[k + q - 1] - (double)sh.keys[k]);
  if (threadIdx.x == 0) sh.kstar = n;
  w = block_min<kThreads>(w, sh.red[0]);
  for (int k = threadIdx.x; k + q - 1 < n; k += kThreads)
    if ((double)sh.keys[k + q - 1] - (double)sh.keys[k] == w) {
      atomicMin(&sh.kstar, k);
      break;
    }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (ba.edge && sh.kstar < n) write_edges(sh.keys, n, q, sh.kstar, ba.edge + (int64_t)band * 2 * kEdge);
    const double e = slack_base(bf, fmax(fabs(uL), fabs(uR)), uM) + 1e-300;
    ba.lb[band] = fmax((w - 2.0 * dmax - 2.0 * e) * (1.0 - 0x1p-40), slope_lb(bf, ba, band));
    ba.wq[band] = w;
  }
}

// Coarse lower bound of every band without sorting: the band's keys binned
// linearly between their extremes (kCoarseBins bins of width res); with
// P = prefix counts, a q-window starting in bin b1 ends in a bin >= b2*(b1),
// the first bin where P[b2 + 1] - P[b1] >= q, so
//   W_q >= min_b1 (b2*(b1) - b1 - 3) res
// (one bin width, plus one either side for the roundings of the binning).
// lb = (that - 2 D_max - 2 E) as in band_bound_kernel; wq = the same
// estimate (ranks bands for seeding only).  The exact bound (sorted keys)
// is computed afterwards only for the bands this one cannot dismiss.
constexpr int kCoarseBins = 49152;
constexpr int kCoarseThreads = 1024;

__global__ void __launch_bounds__(kCoarseThreads, 1) band_coarse_kernel(BandFit bf, BandArgs ba) {
  extern __shared__ __align__(16) unsigned char band_smem[];
  unsigned* P = reinterpret_cast<unsigned*>(band_smem);  // kCoarseBins + 1
  __shared__ double red[2][kCoarseThreads / 32];
  __shared__ unsigned wsum[kCoarseThreads / 32];
  const int band = ba.band_ids ? ba.band_ids[ba.band0 + (int)blockIdx.x] : ba.band0 + (int)blockIdx.x;
  if (band < 0) return;
  const int tid = threadIdx.x;
  double uL, uR;
  if (!boundary_extent(ba.bounds, ba.K, band, &uL, &uR) || !keys_in_range(bf, uL, uR)) {
    if (tid == 0) {
      ba.lb[band] = slope_lb(bf, ba, band);
      ba.wq[band] = INFINITY;
    }
    return;
  }
  const double uM = 0.5 * uL + 0.5 * uR;
  const double dmax = bf.dev * fmax(uR - uM, uM - uL) * (1.0 + 0x1p-40);
  const int n = (int)bf.n, q = (int)bf.q;
  auto key = [&](int k) {
    return (float)__dsub_rn(__dmul_rn(__dsub_rn(__ldg(bf.a + k), bf.c), uM), __ldg(bf.b + k));
  };
  double lo = INFINITY, hi = -INFINITY;
  for (int k = tid; k < n; k += kCoarseThreads) {
    const double v = (double)key(k);
    lo = fmin(lo, v);
    hi = fmax(hi, v);
  }
  for (int b = tid; b <= kCoarseBins; b += kCoarseThreads) P[b] = 0;
  lo = block_min<kCoarseThreads>(lo, red[0]);
  hi = -block_min<kCoarseThreads>(-hi, red[1]);
  const double res = fmax((hi - lo) / kCoarseBins, 1e-300) * (1.0 + 0x1p-30);
  __syncthreads();
  for (int k = tid; k < n; k += kCoarseThreads) {
    const int b = (int)fmin(fmax(floor(((double)key(k) - lo) / res), 0.0), kCoarseBins - 1.0);
    atomicAdd(P + b, 1u);
  }
  __syncthreads();
  // exclusive prefix in place: P[b] = keys in bins < b, P[kCoarseBins] = n
  constexpr int kPer = kCoarseBins / kCoarseThreads;
  unsigned mine[kPer];
  unsigned sum = 0;
#pragma unroll
  for (int e = 0; e < kPer; ++e) {
    mine[e] = P[tid * kPer + e];
    sum += mine[e];
  }
  unsigned incl = sum;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned o = __shfl_up_sync(0xffffffffu, incl, off);
    if ((tid & 31) >= off) incl += o;
  }
  if ((tid & 31) == 31) wsum[tid >> 5] = incl;
  __syncthreads();
  unsigned base = incl - sum;
  for (int w = 0; w < (tid >> 5); ++w) base += wsum[w];
#pragma unroll
  for (int e = 0; e < kPer; ++e) {
    P[tid * kPer + e] = base;
    base += mine[e];
  }
  if (tid == kCoarseThreads - 1) P[kCoarseBins] = base;
  __syncthreads();
  // narrowest window in bins, over the non-empty start bins; `est` is the
  // same window with the keys spread evenly inside each bin (interpolated
  // end position; ranks bands for seeding, which whole bins cannot)
  double best = INFINITY, est = INFINITY;
  for (int b1 = tid; b1 < kCoarseBins; b1 += kCoarseThreads) {
    const unsigned p1 = P[b1];
    if (P[b1 + 1] == p1) continue;  // empty bin
    if (P[kCoarseBins] - p1 < (unsigned)q) continue;
    int a = b1, z = kCoarseBins - 1;  // first b2 with P[b2 + 1] - p1 >= q
    while (a < z) {
      const int mid = (a + z) >> 1;
      if (P[mid + 1] - p1 >= (unsigned)q) z = mid;
      else a = mid + 1;
    }
    best = fmin(best, (double)(a - b1));
    const double inb = (double)(p1 + (unsigned)q - P[a]) / (double)(P[a + 1] - P[a]);
    est = fmin(est, (double)(a - b1) + inb);
  }
  best = block_min<kCoarseThreads>(best, red[0]);
  est = block_min<kCoarseThreads>(est, red[1]);
  if (tid == 0) {
    const double w = fmax(best - 3.0, 0.0) * res;
    const double e = slack_base(bf, fmax(fabs(uL), fabs(uR)), uM) + 1e-300;
    ba.lb[band] = fmax((w - 2.0 * dmax - 2.0 * e) * (1.0 - 0x1p-40), slope_lb(bf, ba, band));
    ba.wq[band] = est < INFINITY ? est * res : INFINITY;
  }
}

// mode 1: window counts of the collected members, one CTA per chunk of up to
// kChunk members of a listed band (members are slope-ordered within their
// band, so a chunk spans a narrow slope range and gets its own centre uM,
// sorted keys, padding D and lower bound)
template <int kThreads, int kItems>
__device__ __forceinline__ void filter_chunk(const BandFit& bf, const BandArgs& ba,
                                             BandShared<kThreads, kItems>& sh, int band, int64_t m0,
                                             int64_t m1);

template <int kThreads, int kItems>
__global__ void __launch_bounds__(kThreads, 1) band_filter_kernel(BandFit bf, BandArgs ba) {
  using SH = BandShared<kThreads, kItems>;
  extern __shared__ __align__(16) unsigned char band_smem[];
  SH& sh = *reinterpret_cast<SH*>(band_smem);
  // chunk -> (band, member range): the explicit chunk table (persistent CTAs
  // taking chunks from a ticket counter: the table's length is known only on
  // the device), or (listed group, chunk index) from the groups' chunk prefix
  if (ba.ctab) {
    __shared__ int64_t s_ticket;
    const int64_t nct = (int64_t)*ba.nctab;
    for (;;) {
      __syncthreads();
      if (threadIdx.x == 0)
        s_ticket = ba.ticket ? (int64_t)atomicAdd(ba.ticket, 1ull) : (int64_t)blockIdx.x;
      __syncthreads();
      const int64_t c = s_ticket;
      if (c >= nct) return;
      filter_chunk<kThreads, kItems>(bf, ba, sh, ba.cband[c], ba.ctab[2 * c], ba.ctab[2 * c + 1]);
      if (!ba.ticket) return;
    }
  }
  const int64_t cidx = blockIdx.x;
  int band;
  int64_t m0, m1;
  {
    if (cidx >= ba.chunk_prefix[ba.nlist]) return;
    int lo = 0, hi = ba.nlist - 1;  // largest e with chunk_prefix[e] <= cidx
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (ba.chunk_prefix[mid] <= cidx) lo = mid;
      else hi = mid - 1;
    }
    const int grp = ba.list[lo];
    band = ba.group_band ? ba.group_band[grp] : grp;
    const int64_t cs = chunk_size(ba.end[grp] - ba.start[grp], ba.chunk, !ba.chunk_fixed);
    m0 = ba.start[grp] + (cidx - ba.chunk_prefix[lo]) * cs;
    m1 = min(ba.end[grp], m0 + cs);
  }
  filter_chunk<kThreads, kItems>(bf, ba, sh, band, m0, m1);
}

// window counts of members [m0, m1) of `band` (band_filter_kernel)
template <int kThreads, int kItems>
__device__ __forceinline__ void filter_chunk(const BandFit& bf, const BandArgs& ba,
                                             BandShared<kThreads, kItems>& sh, int band, int64_t m0,
                                             int64_t m1) {
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  if (m1 <= m0) return;
  double H = INFINITY;
  {
    const lms_candidate best = *ba.best;
    if (best.found) H = best.height;
  }
  bool all = band >= ba.K;  // the beyond-range pseudo band: every member survives
  if (!all && ba.lb[band] > H * (1.0 + 0x1p-19)) return;  // H tightened since collection
  double uL = 0.0, uR = 0.0;
  const float* K = sh.keys;
  const int n = (int)bf.n, q = (int)bf.q;
  double uM = 0.0;
  // inner band with stored keys: its sorted keys at the band centre (the
  // padding D = dev |u - uM| is valid for any uM; the chunk's own centre
  // measured no fewer survivors), no sort and no chunk bound here
  bool stored = false;
  if (!all && ba.bkeys && boundary_extent(ba.bounds, ba.K, band, &uL, &uR) &&
      keys_in_range(bf, uL, uR) && bf.dev * (uR - uL) <= ba.bkeys_tau * H) {
    stored = true;
    uM = 0.5 * uL + 0.5 * uR;
    const float4* src = reinterpret_cast<const float4*>(ba.bkeys + (int64_t)band * ba.bkeys_ld);
    float4* dst = reinterpret_cast<float4*>(sh.keys);
    for (int k = tid; k < (int)(ba.bkeys_ld >> 2); k += kThreads) dst[k] = __ldg(src + k);
    __syncthreads();
  }
  if (!all && !stored) {
    double l = INFINITY, h = -INFINITY;
    for (int64_t s = m0 + tid; s < m1; s += kThreads) {
      const uint32_t p = ba.members[s];
      const int64_t i = p >> 16, j = p & 0xFFFF;
      const double u = __ddiv_rn(__dsub_rn(bf.b[i], bf.b[j]), __dsub_rn(bf.a[i], bf.a[j]));
      l = fmin(l, u);
      h = fmax(h, u);
    }
    uL = block_min<kThreads>(l, sh.red[0]);
    uR = -block_min<kThreads>(-h, sh.red[1]);
    all = !(isfinite(uL) && isfinite(uR)) || !keys_in_range(bf, uL, uR);
  }
  if (!all && !stored) {
    uM = 0.5 * uL + 0.5 * uR;
    band_keys<kThreads, kItems>(bf, uM, sh);
    // the chunk's own lower bound (as band_bound_kernel, with its narrower extent)
    double w = INFINITY;
    for (int k = tid; k + q - 1 < n; k += kThreads) w = fmin(w, (double)K[k + q - 1] - (double)K[k]);
    w = block_min<kThreads>(w, sh.red[0]);
    const double dmax = bf.dev * fmax(uR - uM, uM - uL) * (1.0 + 0x1p-40);
    const double e = slack_base(bf, fmax(fabs(uL), fabs(uR)), uM) + 0x1p-20 * H + 1e-300;
    if ((w - 2.0 * dmax - 2.0 * e) * (1.0 - 0x1p-40) > H) return;
  }
  for (int64_t s0 = m0; s0 < m1; s0 += kThreads) {
    const int64_t s = s0 + tid;
    bool keep = false;
    int64_t rank = 0;
    if (s < m1) {
      const uint32_t p = ba.members[s];
      const int64_t i = p >> 16, j = p & 0xFFFF;
      rank = row_offset(bf.n, i) + (j - i - 1);
      keep = all;
      if (!all) {
        const double ai = bf.a[i], bi = bf.b[i];
        const double u = __ddiv_rn(__dsub_rn(bi, bf.b[j]), __dsub_rn(ai, bf.a[j]));
        const double v0 = cut_value(u, ai, bi);
        const double z = __dsub_rn(v0, __dmul_rn(bf.c, u));
        const double D = bf.dev * fabs(u - uM) * (1.0 + 0x1p-40);
        const double E = slack_base(bf, fabs(u), uM) + 0x1p-20 * H + 1e-300;
        const double pad = D + E;
        int top, bot;
        lower_upper(K, n, __double2float_rd(z - H - pad), __double2float_ru(z + H + pad), &bot, &top);
        if (top - bot >= q) {
          int up_lo, dn_hi;
          lower_upper(K, n, __double2float_rd(z - pad), __double2float_ru(z + pad), &up_lo, &dn_hi);
          keep = (top - up_lo >= q) || (dn_hi - bot >= q);
        }
      }
    }
    const unsigned mask = __ballot_sync(0xffffffffu, keep);
    if (mask) {
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(ba.out_count, (unsigned long long)__popc(mask));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (keep) {
        const unsigned slot = __popc(mask & ((1u << lane) - 1u));
        ba.out_ranks[base + slot] = rank;
        ba.out_fits[base + slot] = ba.fit;
      }
    }
  }
}

// chunk_prefix[e] = first chunk of listed band e (single block; nlist small)
// one warp: exclusive prefix of the listed groups' chunk counts, 32 groups
// per step (independent loads, shuffle scan, running carry)
__global__ void band_chunks_kernel(const int32_t* __restrict__ list, int nlist,
                                   const int64_t* __restrict__ start,
                                   const int64_t* __restrict__ end, int64_t chunk, bool adaptive,
                                   int64_t* __restrict__ prefix) {
  const int lane = threadIdx.x & 31;
  if (threadIdx.x >= 32) return;
  int64_t carry = 0;
  for (int e0 = 0; e0 < nlist; e0 += 32) {
    const int e = e0 + lane;
    int64_t c = 0;
    if (e < nlist) {
      const int64_t sz = end[list[e]] - start[list[e]];
      const int64_t cs = chunk_size(sz, chunk, adaptive);
      c = (sz + cs - 1) / cs;
    }
    int64_t incl = c;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int64_t o = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += o;
    }
    if (e < nlist) prefix[e] = carry + incl - c;
    carry += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (lane == 0) prefix[nlist] = carry;
}

// seeds: the sampled vertices of the flagged (lowest-bound) bands; also the
// sample count of every band (collection size estimate)
__global__ void band_seed_kernel(BandFit bf, int64_t S, const float* __restrict__ keys,
                                 const float* __restrict__ bounds, int K,
                                 const uint8_t* __restrict__ flag,
                                 unsigned* __restrict__ sample_counts, int64_t* __restrict__ ranks,
                                 int32_t* __restrict__ fits, int32_t fit, int64_t cap,
                                 unsigned long long* __restrict__ count) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < S;
       s += (int64_t)gridDim.x * blockDim.x) {
    const float key = keys[s];
    if (!(key <= FLT_MAX)) continue;  // not a banded sample
    const int band = band_of(bounds, K - 1, key);
    const unsigned seen = atomicAdd(sample_counts + band, 1u);
    if (flag[band] && seen < kSeedPerBand) {
      const unsigned long long pos = atomicAdd(count, 1ull);
      if ((int64_t)pos < cap) {
        ranks[pos] = sample_rank(bf, S, s);
        fits[pos] = fit;
      }
    }
  }
}

// one pass over all vertices: append (band, i << 16 | j) of every vertex in
// a flagged band, and (K, ...) of every vertex beyond the fp32 key range.
//
// Pre-test: the flagged bands form a few slope runs; a vertex is tested
// against them with an fp32 slope u32 = fl32(num) / fl32(da) (num = b_i - b_j,
// da = a_i - a_j, the reference's own fp64 differences), whose relative
// error is below 3 * 2^-24, against runs widened by 2^-18 relative (host
// side, BandRuns).  Vertices with tiny differences (fp32 underflow) or a
// non-finite u32 always pass.  Passing vertices are queued per warp and
// processed 32 at a time (no divergence): the fp64 slope exactly as the
// reference forms it, the band by binary search, the flag.
//
// Enumeration: a warp walks a segment of 32 * kRun consecutive ranks, lane l
// owning ranks base + l + 32 e; (i, j) is decoded once per segment and
// advanced along the row-major triangle (backend.py:111-122).
__device__ __forceinline__ void advance_pair(int n, int step, int& i, int& j) {
  j += step;
  while (j >= n && i < n - 2) {
    const int over = j - n;
    ++i;
    j = i + 1 + over;
  }
}

#ifndef LMSB_COLLECT_MINB
#define LMSB_COLLECT_MINB 2
#endif
template <int kR>
__global__ void __launch_bounds__(kCollectThreads, LMSB_COLLECT_MINB) band_collect_kernel(
    BandFit bf, const float* __restrict__ bounds, int K, const int16_t* __restrict__ slot,
    BandRuns runs, uint32_t* __restrict__ out_keys, uint32_t* __restrict__ out_vals, int64_t cap,
    unsigned long long* __restrict__ count) {
  float rlo[kR], rhi[kR];
#pragma unroll
  for (int k = 0; k < kR; ++k) {
    rlo[k] = runs.lo[k];
    rhi[k] = runs.hi[k];
  }
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int kWarps = kCollectThreads / 32;
  uint32_t* queue = reinterpret_cast<uint32_t*>(smem_raw);  // [kWarps][kCollectQueue]
  float* bnd = reinterpret_cast<float*>(queue + kWarps * kCollectQueue);
  int16_t* sl16 = reinterpret_cast<int16_t*>(bnd + K);
  for (int k = threadIdx.x; k <= K; k += blockDim.x) {
    if (k < K - 1) bnd[k] = bounds[k];
    sl16[k] = slot[k];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  uint32_t* q = queue + (threadIdx.x >> 5) * kCollectQueue;
  int qn = 0;
  const int n = (int)bf.n;
  const int64_t seg = 32 * kRun;
  const int64_t nseg = (bf.span + seg - 1) / seg;
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;

  // exact band lookup of 32 queued vertices (lanes >= cnt idle), append
  auto drain = [&](int cnt) {
    bool take = false;
    uint32_t key = 0, val = 0;
    if (lane < cnt) {
      val = q[lane];
      const int i = val >> 16, j = val & 0xFFFF;
      double u = 0.0;
      const int cls = classify(bf, __ldg(bf.a + i), __ldg(bf.b + i), __ldg(bf.a + j),
                               __ldg(bf.b + j), &u);
      if (cls == 1) {
        const float bk = band_key(u);
        const int band = band_of(bnd, K - 1, bk);
        const int sb = sl16[band];
        take = sb >= 0;
        // members of a band ordered by slope: kSlopeBits of fixed-point position
        // between the band's boundaries (monotone in u; 0 in the outer bands)
        uint32_t t = 0;
        if (band > 0 && band < K - 1) {
          const float lo = bnd[band - 1], w = bnd[band] - lo;
          const float f = w > 0.f ? (bk - lo) / w * (float)(1 << kSlopeBits) : 0.f;
          t = (uint32_t)fminf(fmaxf(f, 0.f), (float)((1 << kSlopeBits) - 1));
        }
        // grouped by collection slot (few bits: fewer radix passes), then slope
        key = ((uint32_t)max(sb, 0) << kSlopeBits) | t;
      } else if (cls == 2) {
        take = true;
        key = (uint32_t)sl16[K] << kSlopeBits;
      }
    }
    const unsigned mask = __ballot_sync(0xffffffffu, take);
    if (mask) {
      const int leader = __ffs(mask) - 1;
      unsigned long long b0 = 0;
      if (lane == leader) b0 = atomicAdd(count, (unsigned long long)__popc(mask));
      b0 = __shfl_sync(0xffffffffu, b0, leader);
      if (take) {
        const unsigned long long pos = b0 + __popc(mask & ((1u << lane) - 1u));
        if ((int64_t)pos < cap) {
          out_keys[pos] = key;
          out_vals[pos] = val;
        }
      }
    }
  };

  const double2* __restrict__ ab = bf.ab;
  // fp32 slope pre-test of vertex (i, j) against the runs
  auto pretest = [&](const double2& li, const double2& lj) {
    const double da = __dsub_rn(li.x, lj.x);
    const double num = __dsub_rn(li.y, lj.y);
    const float da32 = (float)da, num32 = (float)num;
    // rcp.approx.ftz: |da32| below FLT_MIN (ftz) gives an infinite or NaN
    // u32 (always passes); |da| <= 2e30 here (band path magnitudes < 1e30),
    // so the reciprocal stays normal.  Error of u32 <= ~5 * 2^-24 relative
    // unless num32 is subnormal (passes below) or u32 underflows (absolute
    // error < 1.2e-38, inside the runs' 1e-37 absolute widening).
    const float u32 = num32 * rcp_approx_ftz(da32);
    // (|num32| < 1e-30 includes num == 0 exactly: horizontal pairs go to the
    // exact band lookup, which is correct and rare outside integer data)
    bool cand = !(fabsf(u32) <= FLT_MAX) | (fabsf(num32) < 1e-30f);
#pragma unroll
    for (int k = 0; k < kR; ++k) cand |= (u32 >= rlo[k]) & (u32 <= rhi[k]);
    return cand & (da != 0.0);
  };
  for (int64_t g = warp0; g < nseg; g += nwarps) {
    const int64_t base = g * seg;
    int i0 = 0, j0 = 0;
    if (lane == 0) {
      int64_t i64, j64;
      decode_rank(bf.n, bf.R0 + base, &i64, &j64);
      i0 = (int)i64;
      j0 = (int)j64;
    }
    int i = __shfl_sync(0xffffffffu, i0, 0);
    int j = __shfl_sync(0xffffffffu, j0, 0);
    advance_pair(n, lane, i, j);
    double2 li = ab[i];
    // ranks of this lane still inside the span (all kRun in every full segment)
    const int64_t left = bf.span - base - lane;
    const int valid = left <= 0 ? 0 : (left >= (int64_t)32 * kRun ? kRun : (int)((left + 31) / 32));
    // kCollectStep vertices per lane per step (ranks r, r + 32, ...):
    // independent load -> test chains in flight, one drain check per step
#pragma unroll 1
    for (int e = 0; e < kRun; e += kCollectStep) {
      int vi[kCollectStep], vj[kCollectStep];
      double2 vli[kCollectStep];
      bool vc[kCollectStep];
      vi[0] = i;
      vj[0] = j;
      vli[0] = li;
#pragma unroll
      for (int t = 1; t < kCollectStep; ++t) {
        vi[t] = vi[t - 1];
        vj[t] = vj[t - 1];
        advance_pair(n, 32, vi[t], vj[t]);
      }
#pragma unroll
      for (int t = 0; t < kCollectStep; ++t) {
        // j runs past n only beyond the triangle's end
        const double2 lj = ab[min(vj[t], n - 1)];
        if (t > 0) vli[t] = vi[t] != vi[t - 1] ? ab[vi[t]] : vli[t - 1];
        vc[t] = pretest(vli[t], lj) & (e + t < valid);
      }
      const unsigned below = (1u << lane) - 1u;
#pragma unroll
      for (int t = 0; t < kCollectStep; ++t) {
        const unsigned m = __ballot_sync(0xffffffffu, vc[t]);
        if (vc[t]) q[qn + __popc(m & below)] = ((uint32_t)vi[t] << 16) | (uint32_t)vj[t];
        qn += __popc(m);
      }
      __syncwarp();
      while (qn >= 32) {
        drain(32);
        __syncwarp();
        for (int t = lane; t < qn - 32; t += 32) q[t] = q[32 + t];
        __syncwarp();
        qn -= 32;
      }
      i = vi[kCollectStep - 1];
      j = vj[kCollectStep - 1];
      li = vli[kCollectStep - 1];
      const int i_last = i;
      advance_pair(n, 32, i, j);
      if (i != i_last) li = ab[i];
    }
  }
  if (qn > 0) drain(qn);
}

// Exact-slope window counts of the band filter's survivors, in fp32: with
// A_k = fl32(a_k - c), B_k = fl32(b_k) and t_k = fma(A_k, fl32(u), -B_k), a
// line in the reference's upward window satisfies t_k in [z - E, z + H + E]
// (downward: [z - H - E, z + E]) where E = 2^-20 (3 amax |u| + 2 bmax + H)
// + 1e-37 covers the fp32 roundings of A, B, u and the FMA (<= 2^-22 (dev |u|
// + bmax) + subnormal steps) and the reference's own (see the file header).
// Removes the band padding D_v, so only vertices whose windows really can
// reach H go on to the exact select.
constexpr int kCountThreads = 512;
constexpr int kCountWarps = kCountThreads / 32;

// Line pairs (A_k, A_k+1, -B_k, -B_k+1) with A = fl32(a - c), B = fl32(b), as
// float4 (the operand pairs of FFMA2); an odd n gets a pad line (0, NaN) at
// index n, whose t is NaN and never counts
__global__ void band_lines32_kernel(BandFit bf, float2* __restrict__ lines) {
  float4* l4 = reinterpret_cast<float4*>(lines);
  const int64_t np = (bf.n + 1) / 2;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < np;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = 2 * p;
    float4 r = make_float4(0.f, 0.f, __int_as_float(0x7fc00000), __int_as_float(0x7fc00000));
    r.x = (float)__dsub_rn(bf.a[k], bf.c);
    r.z = -(float)bf.b[k];
    if (k + 1 < bf.n) {
      r.y = (float)__dsub_rn(bf.a[k + 1], bf.c);
      r.w = -(float)bf.b[k + 1];
    }
    l4[p] = r;
  }
}

// cnt += (x <= w), unsigned: one compare and one predicated add
__device__ __forceinline__ void count_le(unsigned& cnt, uint32_t x, uint32_t w) {
  asm("{\n .reg .pred p;\n setp.le.u32 p, %1, %2;\n @p add.u32 %0, %0, 1;\n}\n"
      : "+r"(cnt)
      : "r"(x), "r"(w));
}

// Persistent: all n lines staged once per CTA in shared memory; a tile is 32
// survivors (one per lane), every warp counts its slice of the lines for all
// 32, and the slices' counts are summed in shared memory.
__global__ void __launch_bounds__(kCountThreads) band_count_kernel(
    BandFit bf, const float2* __restrict__ lines, const lms_candidate* __restrict__ best,
    const int64_t* __restrict__ in_ranks, const unsigned long long* __restrict__ in_count,
    int64_t* __restrict__ out_ranks, int32_t* __restrict__ out_fits, int32_t fit,
    unsigned long long* __restrict__ out_count) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* sl = reinterpret_cast<float2*>(smem_raw);
  const int nst = (int)min(bf.n + (bf.n & 1), (int64_t)kBandMaxN);  // lines staged at once (even)
  unsigned* cnt = reinterpret_cast<unsigned*>(sl + nst);  // [2][32]
  const int64_t total = (int64_t)*in_count;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int n = (int)bf.n;
  const int q = (int)bf.q;
  if ((int64_t)blockIdx.x * 32 >= total) return;
  const bool resident = n <= nst;
  const int ne = n + (n & 1);  // lines incl. the pad line, an even count
  if (resident) {
    // TMA bulk copy of the whole line set (8 ne bytes)
    __shared__ __align__(8) uint64_t bar;
    if (tid == 0) mbar_init(&bar, 1);
    __syncthreads();
    bulk_stage(sl, lines, (uint32_t)ne * (uint32_t)sizeof(float2), &bar, 0);
  }
  double H = INFINITY;
  {
    const lms_candidate b0 = *best;
    if (b0.found) H = b0.height;
  }
  const float4* sl4 = reinterpret_cast<const float4*>(sl);  // two lines per entry
  const int pairs = nst / 2;
  const int per = (pairs + kCountWarps - 1) / kCountWarps;
  const int p0 = warp * per, p1 = min(pairs, p0 + per);
  for (int64_t t0 = (int64_t)blockIdx.x * 32; t0 < total; t0 += (int64_t)gridDim.x * 32) {
    const int64_t s = t0 + lane;
    const bool live = s < total;
    int64_t rank = 0;
    bool force = !isfinite(H) || (bf.amax > 0.0 && bf.amax < 1e-30) ||
                 (bf.bmax > 0.0 && bf.bmax < 1e-30);
    float u32 = 0.f, upLo = 1.f, upHi = 0.f, dnLo = 1.f, dnHi = 0.f;
    if (live) {
      rank = in_ranks[s];
      int64_t i, j;
      decode_rank(bf.n, rank, &i, &j);
      const double ai = bf.a[i], bi = bf.b[i];
      const double u = __ddiv_rn(__dsub_rn(bi, bf.b[j]), __dsub_rn(ai, bf.a[j]));
      const double v0 = cut_value(u, ai, bi);
      const double z = __dsub_rn(v0, __dmul_rn(bf.c, u));
      const double mag = fabs(u) * bf.amax;
      force = force || !(mag + bf.bmax + H < 1e36);
      const double E = 0x1p-20 * (3.0 * mag + 2.0 * bf.bmax + H) + 1e-37;
      u32 = (float)u;
      upLo = __double2float_rd(z - E);
      upHi = __double2float_ru(z + H + E);
      dnLo = __double2float_rd(z - H - E);
      dnHi = __double2float_ru(z + E);
    }
    // lo <= t <= hi implies fl(t - lo) in [+0, fl_ru(hi - lo)] (monotone
    // rounding): one unsigned compare of the bits per window (negatives and
    // NaN fail).  A lower end of +0 becomes -0 so that t = -0 gives +0.
    if (upLo == 0.f) upLo = -0.f;
    if (dnLo == 0.f) dnLo = -0.f;
    const uint32_t wu = live ? __float_as_uint(__fsub_ru(upHi, upLo)) : 0u;
    const uint32_t wd = live ? __float_as_uint(__fsub_ru(dnHi, dnLo)) : 0u;
    const float2 u2 = make_float2(u32, u32);
    const float2 nlu = make_float2(-upLo, -upLo), nld = make_float2(-dnLo, -dnLo);
    if (tid < 64) cnt[tid] = 0u;
    __syncthreads();  // also orders the line staging before first use
    unsigned cu = 0, cd = 0;
    for (int c0 = 0; c0 < ne; c0 += nst) {
      const int cn = min(nst, ne - c0);  // even
      if (!resident) {
        __syncthreads();
        for (int k = tid; k < cn; k += kCountThreads) sl[k] = lines[c0 + k];
        __syncthreads();
      }
      const int e1 = min(p1, cn / 2);
#pragma unroll 8
      for (int p = p0; p < e1; ++p) {
        const float4 L = sl4[p];
        const float2 t = __ffma2_rn(make_float2(L.x, L.y), u2, make_float2(L.z, L.w));
        const float2 du = __fadd2_rn(t, nlu);
        const float2 dd = __fadd2_rn(t, nld);
        count_le(cu, __float_as_uint(du.x), wu);
        count_le(cu, __float_as_uint(du.y), wu);
        count_le(cd, __float_as_uint(dd.x), wd);
        count_le(cd, __float_as_uint(dd.y), wd);
      }
    }
    atomicAdd(cnt + lane, cu);
    atomicAdd(cnt + 32 + lane, cd);
    __syncthreads();
    if (warp == 0) {
      const int tu = (int)cnt[lane], td = (int)cnt[32 + lane];
      const bool keep = live && (force || tu >= q || td >= q);
      const unsigned mask = __ballot_sync(0xffffffffu, keep);
      if (mask) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(out_count, (unsigned long long)__popc(mask));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (keep) {
          const unsigned slot = __popc(mask & ((1u << lane) - 1u));
          out_ranks[base + slot] = rank;
          out_fits[base + slot] = fit;
        }
      }
    }
    __syncthreads();
  }
}

// Exact pass-0 screen of the count kernel's survivors (the first pass of
// exact_vertex_t, lms_exact.cu, with the reference's fp64 arithmetic): lane
// per vertex, the lines staged in shared memory once per CTA chunk and shared
// by 32 vertices, instead of one CTA streaming the lines per vertex.  A
// vertex survives when at least q lines x (anchors snapped to v0) satisfy
// x >= v0 and fl(x - v0) <= bound, or x <= v0 and fl(v0 - x) <= bound, with
// bound = the record's height (its next double below for vertices after the
// record in (i, j) order) -- exactly the exact stage's own pruning test, so
// only vertices the exact select would fully evaluate reach it.
constexpr int kPreThreads = 512;
constexpr int kPreWarps = kPreThreads / 32;
#ifndef LMSB_PRE_LINES
#define LMSB_PRE_LINES 4096
#endif
#ifndef LMSB_PRE_CTAS
#define LMSB_PRE_CTAS 3
#endif
constexpr int kPreLines = LMSB_PRE_LINES;  // lines staged at once (16 B each)

__global__ void __launch_bounds__(kPreThreads) band_exact_prepass_kernel(
    BandFit bf, const lms_candidate* __restrict__ best, const int64_t* __restrict__ in_ranks,
    const unsigned long long* __restrict__ in_count, int64_t* __restrict__ out_ranks,
    int32_t* __restrict__ out_fits, int32_t fit, unsigned long long* __restrict__ out_count) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* sl = reinterpret_cast<double2*>(smem_raw);
  unsigned* cnt = reinterpret_cast<unsigned*>(sl + kPreLines);  // [2][32]
  const int64_t total = (int64_t)*in_count;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = (int)bf.n, q = (int)bf.q;
  if ((int64_t)blockIdx.x * 32 >= total) return;
  const lms_candidate rec = *best;
  const int nst = min(n, kPreLines);
  const int per = (nst + kPreWarps - 1) / kPreWarps;
  const int k0 = warp * per, k1 = min(nst, k0 + per);
  for (int64_t t0 = (int64_t)blockIdx.x * 32; t0 < total; t0 += (int64_t)gridDim.x * 32) {
    const int64_t s = t0 + lane;
    bool live = s < total;
    int64_t rank = 0, i = 0, j = 0;
    double u = 0.0, v0 = 0.0, bound = INFINITY;
    if (live) {
      rank = in_ranks[s];
      decode_rank(bf.n, rank, &i, &j);
      const double ai = bf.a[i], bi = bf.b[i];
      const double da = __dsub_rn(ai, bf.a[j]);
      u = __ddiv_rn(__dsub_rn(bi, bf.b[j]), da);
      v0 = cut_value(u, ai, bi);
      if (rec.found) {
        const bool after = i > rec.i || (i == rec.i && j > rec.j);
        bound = after ? nextafter(rec.height, -INFINITY) : rec.height;
      }
      live = da != 0.0 && bound >= 0.0;
    }
    if (tid < 64) cnt[tid] = 0u;
    unsigned cu = 0, cd = 0;
    for (int c0 = 0; c0 < n; c0 += nst) {
      const int cn = min(nst, n - c0);
      __syncthreads();
      for (int k = tid; k < cn; k += kPreThreads) sl[k] = bf.ab[c0 + k];
      __syncthreads();
      const int e1 = min(k1, cn);
#pragma unroll 4
      for (int k = k0; k < e1; ++k) {
        const double2 L = sl[k];
        const double x = cut_value(u, L.x, L.y);
        const double dx = __dsub_rn(x, v0), dv = __dsub_rn(v0, x);
        cu += (x >= v0) & (dx <= bound);
        cd += (x <= v0) & (dv <= bound);
      }
    }
    atomicAdd(cnt + lane, cu);
    atomicAdd(cnt + 32 + lane, cd);
    __syncthreads();
    if (warp == 0) {
      bool keep = false;
      if (live) {
        int tu = (int)cnt[lane], td = (int)cnt[32 + lane];
        // line j counted unsnapped; snapped it is v0 (counts in both windows;
        // line i's cut is v0 already)
        const double xj = cut_value(u, bf.a[j], bf.b[j]);
        tu += 1 - (int)((xj >= v0) & (__dsub_rn(xj, v0) <= bound));
        td += 1 - (int)((xj <= v0) & (__dsub_rn(v0, xj) <= bound));
        keep = !isfinite(bound) || tu >= q || td >= q;
#ifdef LMSB_PREPASS_TRACE
        if (i == LMSB_PREPASS_TRACE_I && j == LMSB_PREPASS_TRACE_J)
          printf("prepass (%lld,%lld) tu %d td %d q %d bound %.17g u %.17g v0 %.17g cnt %u %u\n",
                 (long long)i, (long long)j, tu, td, q, bound, u, v0, cnt[lane], cnt[32 + lane]);
#endif
      }
      const unsigned mask = __ballot_sync(0xffffffffu, keep);
      if (mask) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(out_count, (unsigned long long)__popc(mask));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (keep) {
          const unsigned slot = __popc(mask & ((1u << lane) - 1u));
          out_ranks[base + slot] = rank;
          out_fits[base + slot] = fit;
        }
      }
    }
    __syncthreads();  // warp 0 has read the counts before the next tile clears them
  }
}

// Seeds from the narrowest q-window of each listed band: the lines whose
// keys (recomputed exactly as the bound kernel formed them) lie among the
// kEdge keys around either end of the window, paired within each end.
__global__ void __launch_bounds__(1024) band_edge_seed_kernel(BandFit bf, BandArgs ba,
                                                            const int32_t* __restrict__ bands,
                                                            int64_t* __restrict__ ranks,
                                                            int32_t* __restrict__ fits,
                                                            int64_t cap,
                                                            unsigned long long* __restrict__ count,
                                                            int T, uint8_t* __restrict__ flag) {
  constexpr int kGroup = 16;
  __shared__ int grp[2][kGroup];
  __shared__ int ng[2];
  __shared__ int s_rank;
  int band;
  if (bands) {
    band = bands[blockIdx.x];
  } else {
    // self-selecting (grid = K): a band seeds when fewer than T bands have a
    // narrower window (ties: the lower index) -- band_top_kernel's choice
    // without its launch
    band = blockIdx.x;
    const double wb = ba.wq[band];
    if (!(wb < INFINITY)) return;
    if (threadIdx.x == 0) s_rank = 0;
    __syncthreads();
    int c = 0;
    for (int k = threadIdx.x; k < ba.K; k += blockDim.x) {
      const double wk = ba.wq[k];
      c += (wk < wb) || (wk == wb && k < band);
    }
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(&s_rank, c);
    __syncthreads();
    if (s_rank >= T) return;
    if (threadIdx.x == 0 && flag) flag[band] = 1;
  }
  double uL, uR;
  if (band < 0 || !boundary_extent(ba.bounds, ba.K, band, &uL, &uR) || !keys_in_range(bf, uL, uR))
    return;
  const double uM = 0.5 * uL + 0.5 * uR;
  const float* e = ba.edge + (int64_t)band * 2 * kEdge;
  if (threadIdx.x < 2) ng[threadIdx.x] = 0;
  __syncthreads();
  const int n = (int)bf.n;
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const float key = (float)__dsub_rn(__dmul_rn(__dsub_rn(__ldg(bf.a + k), bf.c), uM), __ldg(bf.b + k));
#pragma unroll
    for (int g = 0; g < 2; ++g)
      if (key >= e[g * kEdge] && key <= e[g * kEdge + kEdge - 1]) {
        const int slot = atomicAdd(&ng[g], 1);
        if (slot < kGroup) grp[g][slot] = k;
      }
  }
  __syncthreads();
  for (int g = 0; g < 2; ++g) {
    const int m = min(ng[g], kGroup);
    for (int t = threadIdx.x; t < m * m; t += blockDim.x) {
      int x = grp[g][t / m], y = grp[g][t % m];
      if (x >= y) continue;
      const int64_t r = row_offset(bf.n, x) + (y - x - 1);
      if (r < bf.P0 || r >= bf.P0 + bf.pspan) continue;
      const unsigned long long pos = atomicAdd(count, 1ull);
      if ((int64_t)pos < cap) {
        ranks[pos] = r;
        fits[pos] = ba.fit;
      }
    }
  }
}

// ---------------------------------------------------------- direct grouping
// Instead of appending (band, slope position, pair) and radix-sorting, the
// collect pass can write every collected vertex straight into a region of
// its sub-band: each admitted band is split into S_e sub-bands at quantiles
// of its sampled slopes (band_subbounds_kernel), each sub-band gets a region
// sized from the sample counts, and a vertex lands in its sub-band's region
// (atomic cursor).  A region overflow is reported; the host then falls back
// to the sorting path.  Sub-bands are narrow slope ranges, so they serve as
// the filter's chunks directly.

// inner sub-band boundaries of admitted band entry e: S_e - 1 quantiles of its
// samples, stored from sub[sb_first[e] - e]
__global__ void band_subbounds_kernel(const float* __restrict__ sorted,
                                      const unsigned long long* __restrict__ nvalid,
                                      const float* __restrict__ bounds, int K,
                                      const int32_t* __restrict__ list,
                                      const int32_t* __restrict__ sb_first, int nadm,
                                      float* __restrict__ sub, const int* __restrict__ dnadm) {
  if (dnadm) nadm = *dnadm;
  const int e = blockIdx.x;
  if (e >= nadm) return;
  const int k = list[e];
  const int S = sb_first[e + 1] - sb_first[e];
  if (S <= 1 || k >= K) return;
  const int sv = (int)*nvalid;
  auto lower = [&](float x) {
    int a = 0, b = sv;
    while (a < b) {
      const int mid = (a + b) >> 1;
      if (sorted[mid] < x) a = mid + 1;
      else b = mid;
    }
    return a;
  };
  const int lo = k > 0 ? lower(bounds[k - 1]) : 0;
  const int hi = k < K - 1 ? lower(bounds[k]) : sv;
  for (int t = threadIdx.x + 1; t < S; t += blockDim.x)
    sub[sb_first[e] - e + t - 1] = hi > lo ? sorted[lo + ((int64_t)t * (hi - lo)) / S] : INFINITY;
}

template <int kR>
__global__ void __launch_bounds__(kCollectThreads) band_collect_direct_kernel(
    BandFit bf, const float* __restrict__ bounds, int K, BandRuns runs, BandDirect dg) {
  float rlo[kR], rhi[kR];
#pragma unroll
  for (int k = 0; k < kR; ++k) {
    rlo[k] = runs.lo[k];
    rhi[k] = runs.hi[k];
  }
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int kWarps = kCollectThreads / 32;
  uint32_t* queue = reinterpret_cast<uint32_t*>(smem_raw);  // [kWarps][64]
  float* bnd = reinterpret_cast<float*>(queue + kWarps * 64);
  float* sub = bnd + K;
  int32_t* sbf = reinterpret_cast<int32_t*>(sub + dg.nsub);
  int16_t* slot = reinterpret_cast<int16_t*>(sbf + dg.nadm + 1);
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    if (k < K - 1) bnd[k] = bounds[k];
    slot[k] = dg.slot[k];
  }
  for (int t = threadIdx.x; t < dg.nsub; t += blockDim.x) sub[t] = dg.sub[t];
  for (int t = threadIdx.x; t <= dg.nadm; t += blockDim.x) sbf[t] = dg.sb_first[t];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  uint32_t* q = queue + (threadIdx.x >> 5) * 64;
  int qn = 0;
  const int n = (int)bf.n;
  const int64_t seg = 32 * kRun;
  const int64_t nseg = (bf.span + seg - 1) / seg;
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;

  auto drain = [&](int cnt) {
    int g = -1;
    uint32_t val = 0;
    if (lane < cnt) {
      val = q[lane];
      const int i = val >> 16, j = val & 0xFFFF;
      double u = 0.0;
      const int cls = classify(bf, __ldg(bf.a + i), __ldg(bf.b + i), __ldg(bf.a + j),
                               __ldg(bf.b + j), &u);
      if (cls == 1) {
        const float bk = band_key(u);
        const int e = slot[band_of(bnd, K - 1, bk)];
        if (e >= 0) {
          const int f0 = sbf[e], S = sbf[e + 1] - f0;
          g = f0 + (S > 1 ? band_of(sub + f0 - e, S - 1, bk) : 0);
        }
      } else if (cls == 2) {
        g = dg.force_group;
      }
    }
    const unsigned peers = __match_any_sync(0xffffffffu, g);
    const int leader = __ffs(peers) - 1;
    unsigned long long b0 = 0;
    if (g >= 0 && lane == leader) b0 = atomicAdd(dg.cursor + g, (unsigned long long)__popc(peers));
    b0 = __shfl_sync(0xffffffffu, b0, leader);
    if (g >= 0) {
      const unsigned long long pos = b0 + __popc(peers & ((1u << lane) - 1u));
      if ((int64_t)pos < dg.cap[g]) dg.members[dg.rstart[g] + pos] = val;
    }
  };

  for (int64_t gi = warp0; gi < nseg; gi += nwarps) {
    const int64_t base = gi * seg;
    int i0 = 0, j0 = 0;
    if (lane == 0) {
      int64_t i64, j64;
      decode_rank(bf.n, bf.R0 + base, &i64, &j64);
      i0 = (int)i64;
      j0 = (int)j64;
    }
    int i = __shfl_sync(0xffffffffu, i0, 0);
    int j = __shfl_sync(0xffffffffu, j0, 0);
    advance_pair(n, lane, i, j);
    double ai = __ldg(bf.a + i), bi = __ldg(bf.b + i);
    int64_t r = base + lane;
#pragma unroll 1
    for (int e = 0; e < kRun; ++e, r += 32) {
      bool cand = false;
      if (r < bf.span) {
        const double da = __dsub_rn(ai, __ldg(bf.a + j));
        const double num = __dsub_rn(bi, __ldg(bf.b + j));
        if (da != 0.0) {
          const float u32 = __fdividef((float)num, (float)da);
          cand = !(fabsf(u32) <= FLT_MAX) || fabs(da) < 1e-30 || (num != 0.0 && fabs(num) < 1e-30);
#pragma unroll
          for (int k = 0; k < kR; ++k) cand |= (u32 >= rlo[k]) & (u32 <= rhi[k]);
        }
      }
      const unsigned cm = __ballot_sync(0xffffffffu, cand);
      if (cand) q[qn + __popc(cm & ((1u << lane) - 1u))] = ((uint32_t)i << 16) | (uint32_t)j;
      qn += __popc(cm);
      __syncwarp();
      if (qn >= 32) {
        drain(32);
        __syncwarp();
        if (lane < qn - 32) q[lane] = q[32 + lane];
        __syncwarp();
        qn -= 32;
      }
      const int i_old = i;
      advance_pair(n, 32, i, j);
      if (i != i_old) {
        ai = __ldg(bf.a + i);
        bi = __ldg(bf.b + i);
      }
    }
  }
  if (qn > 0) drain(qn);
}

// ------------------------------------------------------------------ n > kBandMaxN
// The n keys of a band no longer fit shared memory.  Bounds: the keys of a
// batch of bands are written to global memory, sorted by a CUB segmented
// radix sort and scanned for W_q (band_wq_kernel).  Filter: every chunk CTA
// reads its band's sorted keys back and quantises them to 16 bits between the
// band's extreme keys (sorted order is preserved; a window [lo, hi] is
// widened to whole quantisation steps, so counts stay a superset), and
// counts with the band's own centre (no per-chunk sort).

__global__ void band_keys_global_kernel(BandFit bf, const float* __restrict__ bounds, int K,
                                        int band0, const int32_t* __restrict__ ids, int nb,
                                        float* __restrict__ keys) {
  const int n = (int)bf.n;
  for (int e = blockIdx.y; e < nb; e += gridDim.y) {
    const int band = ids ? ids[band0 + e] : band0 + e;
    double uL, uR;
    const bool ok = boundary_extent(bounds, K, band, &uL, &uR) && keys_in_range(bf, uL, uR);
    const double uM = 0.5 * uL + 0.5 * uR;
    float* dst = keys + (int64_t)e * n;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
      dst[k] = ok ? (float)__dsub_rn(__dmul_rn(__dsub_rn(__ldg(bf.a + k), bf.c), uM), __ldg(bf.b + k))
                  : 0.f;
  }
}

__global__ void __launch_bounds__(1024) band_wq_kernel(BandFit bf, BandArgs ba, int band0,
                                                      const int32_t* __restrict__ ids,
                                                      const float* __restrict__ sorted,
                                                      float* __restrict__ store) {
  __shared__ double red[32];
  __shared__ int kstar;
  const int band = ids ? ids[band0 + blockIdx.x] : band0 + (int)blockIdx.x;
  if (band < 0) return;
  const int n = (int)bf.n, q = (int)bf.q;
  double uL, uR;
  if (!boundary_extent(ba.bounds, ba.K, band, &uL, &uR) || !keys_in_range(bf, uL, uR)) {
    if (threadIdx.x == 0) {
      ba.lb[band] = slope_lb(bf, ba, band);
      ba.wq[band] = INFINITY;
    }
    return;
  }
  const float* K = sorted + (int64_t)blockIdx.x * n;
  double w = INFINITY;
  for (int k = threadIdx.x; k + q - 1 < n; k += blockDim.x) w = fmin(w, (double)K[k + q - 1] - (double)K[k]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) w = fmin(w, __shfl_xor_sync(0xffffffffu, w, off));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = w;
  if (threadIdx.x == 0) kstar = n;
  __syncthreads();
  w = red[0];
  for (int t = 1; t < (int)(blockDim.x >> 5); ++t) w = fmin(w, red[t]);
  for (int k = threadIdx.x; k + q - 1 < n; k += blockDim.x)
    if ((double)K[k + q - 1] - (double)K[k] == w) {
      atomicMin(&kstar, k);
      break;
    }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (ba.edge && kstar < n) write_edges(K, n, q, kstar, ba.edge + (int64_t)band * 2 * kEdge);
    const double uM = 0.5 * uL + 0.5 * uR;
    const double dmax = bf.dev * fmax(uR - uM, uM - uL) * (1.0 + 0x1p-40);
    const double e = slack_base(bf, fmax(fabs(uL), fabs(uR)), uM) + 1e-300;
    ba.lb[band] = fmax((w - 2.0 * dmax - 2.0 * e) * (1.0 - 0x1p-40), slope_lb(bf, ba, band));
    ba.wq[band] = w;
  }
  // keep the sorted keys of the band for the filter (admitted bands only use them)
  if (store) {
    float* dst = store + (int64_t)band * n;
    for (int k = threadIdx.x; k < n; k += blockDim.x) dst[k] = K[k];
  }
}

// members per slice of a group of `cnt` members: at least kMinSlices slices
// when the group has that many chunks (a rank of a sharded search holds few
// members per band), at most `smax` members each, whole chunks
constexpr int kMinSlices = 8;
__host__ __device__ __forceinline__ int64_t group_slice(int64_t cnt, int64_t chunk, int64_t smax) {
  int64_t s = (cnt + kMinSlices - 1) / kMinSlices;
  s = (s + chunk - 1) / chunk * chunk;
  return s < chunk ? chunk : (s > smax ? smax : s);
}

// slice size of listed group grp: a narrow band (BandArgs::narrow: its
// centre keys serve every member, dev * width <= tau * H) is one slice --
// one key sort for the whole band; otherwise group_slice
__device__ __forceinline__ int64_t slice_of(const BandArgs& ba, int grp) {
  const int64_t cnt = ba.end[grp] - ba.start[grp];
  const int band = ba.group_band ? ba.group_band[grp] : grp;
  if (ba.narrow && band < ba.K && ba.narrow[band]) {
    const int64_t s = (cnt + ba.chunk - 1) / ba.chunk * ba.chunk;
    return s < ba.chunk ? ba.chunk : s;
  }
  return group_slice(cnt, ba.chunk, ba.slice);
}

// per-slice bin table of the large-n filter: kSliceBins linear bins between
// the slice's extreme keys, P[0 .. kSliceBins] first key index of each bin
// (rows padded to a 16-byte multiple for the bulk copy)
constexpr int kSliceBins = 32768;
constexpr int64_t kSliceRow = kSliceBins + 4;
static_assert(kSliceRow == kSliceTableRow, "slice table row (lms_band.cuh)");
constexpr int kBigThreads = 1024;

__global__ void __launch_bounds__(kBigThreads, 1) band_filter_big_kernel(BandFit bf, BandArgs ba,
                                                                        const float* __restrict__ keys) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned* P = reinterpret_cast<unsigned*>(smem_raw);  // the slice's bin table
  __shared__ __align__(8) uint64_t pbar;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int64_t cidx = blockIdx.x;
  if (cidx >= ba.chunk_prefix[ba.nlist]) return;
  int lo = 0, hi = ba.nlist - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (ba.chunk_prefix[mid] <= cidx) lo = mid;
    else hi = mid - 1;
  }
  const int grp = ba.list[lo];
  const int band = ba.group_band ? ba.group_band[grp] : grp;
  const int64_t m0 = ba.start[grp] + (cidx - ba.chunk_prefix[lo]) * ba.chunk;
  const int64_t m1 = min(ba.end[grp], m0 + ba.chunk);
  if (m1 <= m0) return;
  double H = INFINITY;
  {
    const lms_candidate best = *ba.best;
    if (best.found) H = best.height;
  }
  const int n = (int)bf.n, q = (int)bf.q;
  bool all = band >= ba.K;
  double uL = 0.0, uR = 0.0;
  if (!all) {
    if (ba.lb[band] > H * (1.0 + 0x1p-19)) return;
    all = !boundary_extent(ba.bounds, ba.K, band, &uL, &uR) || !keys_in_range(bf, uL, uR);
  }
  // the chunk's slice: its sorted keys and their centre slope
  int64_t sl = 0;
  double uM = 0.0;
  if (!all) {
    sl = ba.slice_prefix[lo] + (m0 - ba.start[grp]) / slice_of(ba, grp);
    uM = ba.slice_u[sl];
  }
  if (!all) {
    // the chunk's own lower bound from its slice's narrowest q-window, with
    // the chunk's slope extent (members are slope-ordered, so a chunk is a
    // narrow part of its slice)
    __shared__ double cred[2][kBigThreads / 32];
    double l = INFINITY, h = -INFINITY;
    for (int64_t s = m0 + tid; s < m1; s += kBigThreads) {
      const uint32_t p = ba.members[s];
      const int64_t i = p >> 16, j = p & 0xFFFF;
      const double u = __ddiv_rn(__dsub_rn(bf.b[i], bf.b[j]), __dsub_rn(bf.a[i], bf.a[j]));
      l = fmin(l, u);
      h = fmax(h, u);
    }
    const double cl = block_min<kBigThreads>(l, cred[0]);
    const double ch = -block_min<kBigThreads>(-h, cred[1]);
    if (isfinite(cl) && isfinite(ch)) {
      const double dmax = bf.dev * fmax(ch - uM, uM - cl) * (1.0 + 0x1p-40);
      const double e = slack_base(bf, fmax(fabs(cl), fabs(ch)), uM) + 0x1p-20 * H + 1e-300;
      if ((ba.slice_wq[sl] - 2.0 * dmax - 2.0 * e) * (1.0 - 0x1p-40) > H) return;
    }
  }
  // the slice's bin table (launch_band_slices): P[b] = first key index whose
  // bin is >= b, bins of width res from the slice's smallest key; staged by a
  // bulk copy
  double kmin = 0.0, res = 1.0;
  if (!all) {
    kmin = ba.slice_kmin[sl];
    res = ba.slice_res[sl];
    if (tid == 0) mbar_init(&pbar, 1);
    __syncthreads();
    bulk_stage(P, ba.slice_ptab + sl * kSliceRow, kSliceRow * sizeof(unsigned), &pbar, 0);
  }
  auto q16 = [&](double x, bool up) -> int {
    // whole bins around x, one extra either side for rounding
    const double t = floor((x - kmin) / res);
    const double v = up ? t + 1.0 : t - 1.0;
    return (int)fmin(fmax(v, -1.0), (double)kSliceBins);
  };
  auto lower16 = [&](int x) {  // first index whose bin is >= x
    return (int)P[min(max(x, 0), kSliceBins)];
  };
  auto upper16 = [&](int x) {  // first index whose bin is > x
    return (int)P[min(max(x + 1, 0), kSliceBins)];
  };
  // Exact fp32 positions from the band's sorted keys in global memory (L2:
  // the admitted bands' rows), searched only inside the bracket the 16-bit
  // keys give: every key of index < lower16(t - 1) lies below x, every key of
  // index >= upper16(t + 1) above it (t = x's quantisation step; the one-step
  // margins absorb the roundings of the quantisation).
  const float* __restrict__ Kg = keys + sl * n;
  auto upper_f = [&](double x) {  // first index with key > x (x rounded up to fp32)
    float xf = (float)x;
    if ((double)xf < x) xf = nextafterf(xf, INFINITY);
    int a = lower16(q16((double)xf, false)), b = upper16(q16((double)xf, true));
    while (a < b) {
      const int mid = (a + b) >> 1;
      if (__ldg(Kg + mid) <= xf) a = mid + 1;
      else b = mid;
    }
    return a;
  };
  auto lower_f = [&](double x) {  // first index with key >= x (x rounded down to fp32)
    float xf = (float)x;
    if ((double)xf > x) xf = nextafterf(xf, -INFINITY);
    int a = lower16(q16((double)xf, false)), b = upper16(q16((double)xf, true));
    while (a < b) {
      const int mid = (a + b) >> 1;
      if (__ldg(Kg + mid) < xf) a = mid + 1;
      else b = mid;
    }
    return a;
  };
  for (int64_t s0 = m0; s0 < m1; s0 += kBigThreads) {
    const int64_t s = s0 + tid;
    bool keep = false;
    int64_t rank = 0;
    if (s < m1) {
      const uint32_t p = ba.members[s];
      const int64_t i = p >> 16, j = p & 0xFFFF;
      rank = row_offset(bf.n, i) + (j - i - 1);
      keep = all;
      if (!all) {
        const double ai = bf.a[i], bi = bf.b[i];
        const double u = __ddiv_rn(__dsub_rn(bi, bf.b[j]), __dsub_rn(ai, bf.a[j]));
        const double v0 = cut_value(u, ai, bi);
        const double z = __dsub_rn(v0, __dmul_rn(bf.c, u));
        const double D = bf.dev * fabs(u - uM) * (1.0 + 0x1p-40);
        const double E = slack_base(bf, fabs(u), uM) + 0x1p-20 * H + 1e-300;
        const double pad = D + E;
        // coarse: 16-bit keys in shared memory (a superset)
        int top = upper16(q16(z + H + pad, true));
        int bot = lower16(q16(z - H - pad, false));
        if (top - bot >= q) {
          // exact fp32 ends (the survivors' count kernel and exact select
          // follow, so this only has to stay a superset)
          top = upper_f(z + H + pad);
          bot = lower_f(z - H - pad);
          if (top - bot >= q) {
            const int up_lo = lower_f(z - pad);
            const int dn_hi = upper_f(z + pad);
            keep = (top - up_lo >= q) || (dn_hi - bot >= q);
          }
        }
      }
    }
    const unsigned mask = __ballot_sync(0xffffffffu, keep);
    if (mask) {
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(ba.out_count, (unsigned long long)__popc(mask));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (keep) {
        const unsigned slot = __popc(mask & ((1u << lane) - 1u));
        ba.out_ranks[base + slot] = rank;
        ba.out_fits[base + slot] = ba.fit;
      }
    }
  }
}

template <typename Kern>
void set_smem(Kern kern, size_t smem, DeviceOnce* done) {
  set_max_smem(kern, smem, *done);
}

template <int kThreads, int kItems>
void launch_band_t(const BandFit& bf, const BandArgs& ba, int mode, int grid, cudaStream_t st) {
  constexpr size_t smem = sizeof(BandShared<kThreads, kItems>);
  static DeviceOnce c0, c1;
  if (mode == 0) {
    set_smem(band_bound_kernel<kThreads, kItems>, smem, &c0);
    band_bound_kernel<kThreads, kItems><<<grid, kThreads, smem, st>>>(bf, ba);
  } else {
    set_smem(band_filter_kernel<kThreads, kItems>, smem, &c1);
    band_filter_kernel<kThreads, kItems><<<grid, kThreads, smem, st>>>(bf, ba);
  }
}



}  // namespace

size_t band_sample_temp_bytes(int64_t S) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, bytes, (const float*)nullptr, (float*)nullptr, (int)S);
  return std::max(bytes, sample_sort_scratch_bytes(S));
}

// the hand-written bucket sort of the sample (default) or CUB's (LMSB_SAMPLE_SORT=0)
bool use_sample_sort() {
  const char* e = getenv("LMSB_SAMPLE_SORT");
  return !(e && e[0] == '0');
}

// grouping buckets: (slot, top slope bits), at most kGroupBuckets
constexpr int kGroupBuckets = 1 << 14;  // scatter CTA: 12 bytes of shared memory per bucket
constexpr int kGroupTile = 4096;  // collected vertices per CTA of the bucket passes

size_t band_group_temp_bytes(int64_t m) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)m);
  return std::max(bytes, (size_t)3 * (kGroupBuckets + 1) * sizeof(int64_t));
}

int bits_for(int64_t v) {
  int b = 1;
  while (b < 32 && ((int64_t)1 << b) <= v) ++b;
  return b;
}

__global__ void band_runs_kernel(const uint32_t* __restrict__ keys, int64_t m,
                                 int64_t* __restrict__ start, int64_t* __restrict__ end) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m;
       p += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k = keys[p] >> kSlopeBits;
    if (p == 0 || (keys[p - 1] >> kSlopeBits) != k) start[k] = p;
    if (p == m - 1 || (keys[p + 1] >> kSlopeBits) != k) end[k] = p + 1;
  }
}

size_t band_collect_smem(int K) {
  return (size_t)(kCollectThreads / 32) * kCollectQueue * sizeof(uint32_t) +
         (size_t)K * sizeof(float) + (size_t)(K + 1) * sizeof(int16_t) + 16;
}

// The cluster sort (one 8-CTA cluster per segment, ~60 us for 65,536 keys,
// ~16 clusters resident) against the CUB sorts (one CTA per segment over
// several global passes: high latency, high throughput): the cluster sort
// wins for a few segments (the exact bounds of a shard plan's pool and
// refine lists), CUB for many (config 3's ~800 slices: 2.4 vs 3.1 ms) and
// for the single sample sort (config 2: 0.80 vs 0.82 ms).
// LMSB_SEG_SORT: 0 never, 1 always, 2 (default) segmented sorts of at most
// LMSB_SEG_SORT_MAX (default 32) segments.
bool use_seg_sort(int64_t max_len, int64_t nseg) {
  const char* e = getenv("LMSB_SEG_SORT");
  const int mode = e ? atoi(e) : 2;
  if (!seg_sort_fits(max_len) || mode == 0) return false;
  if (mode == 1) return true;
  const char* m = getenv("LMSB_SEG_SORT_MAX");
  const int64_t cap = m ? atoll(m) : 32;
  return nseg > 1 && nseg <= cap;
}

int launch_band_sample(const BandFit& bf, const BandWork& w, int sms, cudaStream_t st) {
  cudaMemsetAsync(w.nvalid, 0, sizeof(unsigned long long), st);
  band_sample_kernel<<<sms * 4, 256, 0, st>>>(bf, w.S, w.sample, w.nvalid);
  if (use_sample_sort()) {
    if (launch_sample_sort(w.sample, w.sample_sorted, w.S, w.temp, w.temp_bytes, st) != 0)
      return -1;
  } else if (use_seg_sort(w.S, 1)) {
    if (launch_seg_sort(w.sample, w.sample_sorted, w.S, 1, nullptr, nullptr, st) != 0) return -1;
  } else {
    size_t bytes = w.temp_bytes;
    if (cub::DeviceRadixSort::SortKeys(w.temp, bytes, w.sample, w.sample_sorted, (int)w.S, 0, 32,
                                       st) != cudaSuccess)
      return -1;
  }
  band_bounds_kernel<<<(w.K + 255) / 256, 256, 0, st>>>(w.sample_sorted, w.nvalid, w.K, w.bounds);
  return 0;
}

void launch_band(const BandFit& bf, const BandArgs& ba, int mode, int grid, cudaStream_t st) {
  if (grid <= 0) return;
  if (mode == 1 && !ba.ctab)
    band_chunks_kernel<<<1, 32, 0, st>>>(ba.list, ba.nlist, ba.start, ba.end, ba.chunk,
                                         !ba.chunk_fixed,
                                         ba.chunk_prefix);
  if (bf.n <= 1024) launch_band_t<256, 4>(bf, ba, mode, grid, st);
  else if (bf.n <= 4096) launch_band_t<512, 8>(bf, ba, mode, grid, st);
  // (the bounds run 512 threads x 32 keys: 10 % faster than 1024 x 16 for the
  // per-band sort; the filter keeps 1024 x 16 for its member loop)
  else if (mode == 0) launch_band_t<512, 32>(bf, ba, mode, grid, st);
  else launch_band_t<1024, 16>(bf, ba, mode, grid, st);
}

size_t band_big_sort_temp_bytes(int nb, int64_t n) {
  size_t bytes = 0;
  cub::DeviceSegmentedRadixSort::SortKeys(nullptr, bytes, (const float*)nullptr, (float*)nullptr,
                                          (int)(nb * n), nb, (const int64_t*)nullptr,
                                          (const int64_t*)nullptr);
  return std::max(bytes, seg_bucket_sort_scratch_bytes((int64_t)nb * n, nb, n));
}

// Opt-in (LMSB_SEG_BUCKET=1): the sample sort's bucket scheme per segment
// measured slower than the cluster / CUB sorts on every large-n path (config
// 3 7.65 -> 7.94 ms, n = 20,000 1.98 -> 2.45 ms: 256 buckets of ~78-256 keys
// per segment leave its per-bucket CTAs mostly idle)
bool use_seg_bucket() {
  const char* e = getenv("LMSB_SEG_BUCKET");
  return e && e[0] == '1';
}

__global__ void seg_offsets_kernel(int64_t* off, int nb, int64_t n) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e <= nb; e += gridDim.x * blockDim.x)
    off[e] = (int64_t)e * n;
}

int launch_band_bound_big(const BandFit& bf, const BandArgs& ba, const BandBig& bg, int k0,
                          int k1, const int32_t* ids, cudaStream_t st) {
  const int64_t n = bf.n;
  seg_offsets_kernel<<<(bg.batch + 256) / 256, 256, 0, st>>>(bg.seg, bg.batch, n);
  for (int b0 = k0; b0 < k1; b0 += bg.batch) {
    const int nb = std::min(bg.batch, k1 - b0);
    dim3 grid((unsigned)std::min<int64_t>((n + 255) / 256, 64), (unsigned)std::min(nb, 65535));
    band_keys_global_kernel<<<grid, 256, 0, st>>>(bf, ba.bounds, ba.K, b0, ids, nb, bg.keys);
    if (use_seg_bucket()) {
      if (launch_seg_bucket_sort(bg.keys, bg.keys_alt, (int64_t)nb * n, nb, n, nullptr, nullptr,
                                 bg.temp, bg.temp_bytes, st) != 0)
        return -1;
    } else if (use_seg_sort(n, nb)) {
      if (launch_seg_sort(bg.keys, bg.keys_alt, n, nb, nullptr, nullptr, st) != 0) return -1;
    } else {
      size_t bytes = bg.temp_bytes;
      if (cub::DeviceSegmentedRadixSort::SortKeys(bg.temp, bytes, bg.keys, bg.keys_alt,
                                                  (int)(nb * n), nb, bg.seg, bg.seg + 1, 0, 32,
                                                  st) != cudaSuccess)
        return -1;
    }
    band_wq_kernel<<<nb, 1024, 0, st>>>(bf, ba, b0, ids, bg.keys_alt, bg.store);
  }
  return 0;
}

__global__ void band_slice_prefix_kernel(BandArgs ba) {
  const int lane = threadIdx.x & 31;
  if (threadIdx.x >= 32) return;
  const int nlist = ba.nlist;
  int64_t* prefix = ba.slice_prefix;
  int64_t carry = 0;
  for (int e0 = 0; e0 < nlist; e0 += 32) {
    const int e = e0 + lane;
    int64_t c = 0;
    if (e < nlist) {
      const int grp = ba.list[e];
      const int64_t sz = ba.end[grp] - ba.start[grp];
      const int64_t sb = slice_of(ba, grp);
      c = (sz + sb - 1) / sb;
    }
    int64_t incl = c;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int64_t o = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += o;
    }
    if (e < nlist) prefix[e] = carry + incl - c;
    carry += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (lane == 0) prefix[nlist] = carry;
}

// exact slope of member pair p, or NaN when it is not a banded vertex
__device__ __forceinline__ double member_slope(const BandFit& bf, uint32_t p) {
  const int i = p >> 16, j = p & 0xFFFF;
  double u = 0.0;
  return classify(bf, bf.a[i], bf.b[i], bf.a[j], bf.b[j], &u) == 1 ? u : __longlong_as_double(
                                                                            0x7FF8000000000000LL);
}

__global__ void band_slice_keys_kernel(BandFit bf, BandArgs ba, int64_t nslices_max,
                                       float* __restrict__ keys, int64_t* __restrict__ seg_b,
                                       int64_t* __restrict__ seg_e) {
  const int n = (int)bf.n;
  const int64_t total = ba.slice_prefix[ba.nlist];
  for (int64_t s = blockIdx.y; s < nslices_max; s += gridDim.y) {
    bool live = s < total;
    double uC = 0.0;
    if (live) {
      int lo = 0, hi = ba.nlist - 1;  // listed group of slice s
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (ba.slice_prefix[mid] <= s) lo = mid;
        else hi = mid - 1;
      }
      const int grp = ba.list[lo];
      const int band = ba.group_band ? ba.group_band[grp] : grp;
      const int64_t sb = slice_of(ba, grp);
      const int64_t m0 = ba.start[grp] + (s - ba.slice_prefix[lo]) * sb;
      const int64_t m1 = min(ba.end[grp], m0 + sb);
      double uL, uR;
      live = band < ba.K && m1 > m0 && boundary_extent(ba.bounds, ba.K, band, &uL, &uR) &&
             keys_in_range(bf, uL, uR);  // else the filter keeps every member
      if (live) {
        const double uf = member_slope(bf, ba.members[m0]);
        const double ul = member_slope(bf, ba.members[m1 - 1]);
        // members of an inner band are banded vertices inside its extent
        uC = fmin(fmax(0.5 * uf + 0.5 * ul, uL), uR);
        if (!(uC == uC)) uC = 0.5 * uL + 0.5 * uR;
      }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      seg_b[s] = s * n;
      seg_e[s] = live ? s * n + n : s * n;
      ba.slice_u[s] = uC;
    }
    if (!live) continue;
    float* dst = keys + s * n;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
      dst[k] = (float)__dsub_rn(__dmul_rn(__dsub_rn(__ldg(bf.a + k), bf.c), uC), __ldg(bf.b + k));
  }
}

// narrowest q-window of every live slice's sorted keys (chunk lower bounds)
__global__ void __launch_bounds__(1024) band_slice_wq_kernel(BandFit bf, BandArgs ba,
                                                            int64_t nslices_max,
                                                            const float* __restrict__ store,
                                                            const int64_t* __restrict__ seg_b,
                                                            const int64_t* __restrict__ seg_e) {
  __shared__ double red[32];
  const int n = (int)bf.n, q = (int)bf.q;
  for (int64_t s = blockIdx.x; s < nslices_max; s += gridDim.x) {
    double w = INFINITY;
    if (seg_e[s] > seg_b[s]) {
      const float* K = store + s * n;
      for (int k = threadIdx.x; k + q - 1 < n; k += blockDim.x)
        w = fmin(w, (double)K[k + q - 1] - (double)K[k]);
    }
    w = block_min<1024>(w, red);
    if (threadIdx.x == 0) ba.slice_wq[s] = w;
    __syncthreads();
  }
}

// bin table of every live slice (band_filter_big_kernel): keys are sorted,
// so bins are non-decreasing in the key index and P[b] is where bin b starts
__global__ void __launch_bounds__(1024) band_slice_table_kernel(BandFit bf, BandArgs ba,
                                                               int64_t nslices_max,
                                                               const float* __restrict__ store,
                                                               const int64_t* __restrict__ seg_b,
                                                               const int64_t* __restrict__ seg_e) {
  const int n = (int)bf.n;
  for (int64_t s = blockIdx.x; s < nslices_max; s += gridDim.x) {
    if (seg_e[s] <= seg_b[s]) continue;
    const float* K = store + s * n;
    unsigned* P = ba.slice_ptab + s * kSliceRow;
    const double kmin = (double)K[0], kmax = (double)K[n - 1];
    const double res = fmax((kmax - kmin) / kSliceBins, 1e-300) * (1.0 + 0x1p-30);
    if (threadIdx.x == 0) {
      ba.slice_kmin[s] = kmin;
      ba.slice_res[s] = res;
    }
    auto bin = [&](int k) {
      return (int)fmin(fmax(floor(((double)K[k] - kmin) / res), 0.0), kSliceBins - 1.0);
    };
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
      const int bk = bin(k);
      const int bp = k > 0 ? bin(k - 1) : -1;
      for (int b = bp + 1; b <= bk; ++b) P[b] = (unsigned)k;
      if (k == n - 1)
        for (int b = bk + 1; b <= kSliceBins; ++b) P[b] = (unsigned)n;
    }
  }
}

size_t band_slice_sort_temp_bytes(int64_t nslices_max, int64_t n) {
  size_t bytes = 0;
  cub::DeviceSegmentedRadixSort::SortKeys(nullptr, bytes, (const float*)nullptr, (float*)nullptr,
                                          (int)(nslices_max * n), (int)nslices_max,
                                          (const int64_t*)nullptr, (const int64_t*)nullptr);
  return std::max(bytes,
                  seg_bucket_sort_scratch_bytes(nslices_max * n, (int)nslices_max, n));
}

int launch_band_slices(const BandFit& bf, const BandArgs& ba, int64_t nslices_max, float* keys,
                       float* store, int64_t* seg_begin, int64_t* seg_end, void* temp,
                       size_t temp_bytes, cudaStream_t st) {
  if (nslices_max <= 0) return 0;
  band_slice_prefix_kernel<<<1, 32, 0, st>>>(ba);
  dim3 grid((unsigned)std::min<int64_t>((bf.n + 255) / 256, 64),
            (unsigned)std::min<int64_t>(nslices_max, 65535));
  band_slice_keys_kernel<<<grid, 256, 0, st>>>(bf, ba, nslices_max, keys, seg_begin, seg_end);
  if (use_seg_bucket() && nslices_max <= 65535) {
    if (launch_seg_bucket_sort(keys, store, nslices_max * bf.n, (int)nslices_max, bf.n, seg_begin,
                               seg_end, temp, temp_bytes, st) != 0)
      return -1;
  } else if (use_seg_sort(bf.n, nslices_max)) {
    if (launch_seg_sort(keys, store, bf.n, (int)nslices_max, seg_begin, seg_end, st) != 0)
      return -1;
  } else {
    size_t bytes = temp_bytes;
    if (cub::DeviceSegmentedRadixSort::SortKeys(temp, bytes, keys, store,
                                                (int)(nslices_max * bf.n), (int)nslices_max,
                                                seg_begin, seg_end, 0, 32, st) != cudaSuccess)
      return -1;
  }
  band_slice_wq_kernel<<<(int)std::min<int64_t>(nslices_max, 4096), 1024, 0, st>>>(
      bf, ba, nslices_max, store, seg_begin, seg_end);
  band_slice_table_kernel<<<(int)std::min<int64_t>(nslices_max, 4096), 1024, 0, st>>>(
      bf, ba, nslices_max, store, seg_begin, seg_end);
  return 0;
}

void launch_band_filter_big(const BandFit& bf, const BandArgs& ba, const float* store, int grid,
                            cudaStream_t st) {
  if (grid <= 0) return;
  band_chunks_kernel<<<1, 32, 0, st>>>(ba.list, ba.nlist, ba.start, ba.end, ba.chunk, false,
                                       ba.chunk_prefix);
  const size_t smem = kSliceRow * sizeof(unsigned);
  static DeviceOnce done;
  set_smem(band_filter_big_kernel, smem, &done);
  band_filter_big_kernel<<<grid, kBigThreads, smem, st>>>(bf, ba, store);
}

// T rounds of a block-wide (wq, index) argmin; every thread holds its share
// of the candidates (at most 16) in registers and marks the ones taken.
constexpr int kTopThreads = 1024;
constexpr int kTopItems = 16;  // candidates per thread: K <= 16,384

__global__ void __launch_bounds__(kTopThreads) band_top_kernel(const double* __restrict__ wq, int k0,
                                                              int k1, const int32_t* __restrict__ ids,
                                                              int K, int T, int32_t* __restrict__ list,
                                                              uint8_t* __restrict__ flag) {
  __shared__ double rv[32];
  __shared__ int rk[32];
  __shared__ int pick_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double cv[kTopItems];
  int ck[kTopItems];
#pragma unroll
  for (int e = 0; e < kTopItems; ++e) {
    const int x0 = k0 + e * kTopThreads + tid;
    const int k = x0 < k1 ? (ids ? ids[x0] : x0) : -1;
    ck[e] = k;
    cv[e] = k >= 0 ? wq[k] : INFINITY;
  }
  for (int k = tid; k < K; k += kTopThreads) flag[k] = 0;
  __syncthreads();
  for (int t = 0; t < T; ++t) {
    double v = INFINITY;
    int bk = INT_MAX;
#pragma unroll
    for (int e = 0; e < kTopItems; ++e)
      if (ck[e] >= 0 && (cv[e] < v || (cv[e] == v && ck[e] < bk))) {
        v = cv[e];
        bk = ck[e];
      }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v, off);
      const int ok = __shfl_xor_sync(0xffffffffu, bk, off);
      if (ov < v || (ov == v && ok < bk)) {
        v = ov;
        bk = ok;
      }
    }
    if (lane == 0) {
      rv[warp] = v;
      rk[warp] = bk;
    }
    __syncthreads();
    if (warp == 0) {
      v = rv[lane];
      bk = rk[lane];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, off);
        const int ok = __shfl_xor_sync(0xffffffffu, bk, off);
        if (ov < v || (ov == v && ok < bk)) {
          v = ov;
          bk = ok;
        }
      }
      if (lane == 0) {
        const int pick = v < INFINITY ? bk : -1;
        pick_s = pick;
        list[t] = pick;
        if (pick >= 0) flag[pick] = 1;
      }
    }
    __syncthreads();
    const int pick = pick_s;
#pragma unroll
    for (int e = 0; e < kTopItems; ++e)
      if (ck[e] == pick) ck[e] = -1;  // taken
  }
}

void launch_band_coarse(const BandFit& bf, const BandArgs& ba, int grid, cudaStream_t st) {
  if (grid <= 0) return;
  constexpr size_t smem = (kCoarseBins + 1) * sizeof(unsigned);
  static DeviceOnce done;
  set_smem(band_coarse_kernel, smem, &done);
  band_coarse_kernel<<<grid, kCoarseThreads, smem, st>>>(bf, ba);
}

void launch_band_interleave(const double* a, const double* b, int64_t n, double2* ab,
                            cudaStream_t st) {
  band_interleave_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 1024), 256, 0, st>>>(a, b, n, ab);
}

void launch_band_top(const double* wq, int k0, int k1, int K, int T, int32_t* list, uint8_t* flag,
                     cudaStream_t st, const int32_t* ids) {
  band_top_kernel<<<1, kTopThreads, 0, st>>>(wq, k0, k1, ids, K, T < 64 ? T : 64, list, flag);
}

void launch_band_edge_seeds(const BandFit& bf, const BandArgs& ba, const int32_t* bands, int nb,
                            int64_t* ranks, int32_t* fits, int64_t cap,
                            unsigned long long* count, cudaStream_t st) {
  if (nb > 0 && ba.edge)
    band_edge_seed_kernel<<<nb, 1024, 0, st>>>(bf, ba, bands, ranks, fits, cap, count, 0, nullptr);
}

void launch_band_edge_seeds_top(const BandFit& bf, const BandArgs& ba, int T, uint8_t* flag,
                                int64_t* ranks, int32_t* fits, int64_t cap,
                                unsigned long long* count, cudaStream_t st) {
  cudaMemsetAsync(flag, 0, (size_t)ba.K, st);
  if (ba.K > 0 && ba.edge)
    band_edge_seed_kernel<<<ba.K, 1024, 0, st>>>(bf, ba, nullptr, ranks, fits, cap, count, T, flag);
}

void launch_band_seeds(const BandFit& bf, const BandWork& w, int64_t* ranks, int32_t* fits,
                       int32_t fit, int64_t cap, unsigned long long* count, cudaStream_t st) {
  cudaMemsetAsync(w.sample_counts, 0, sizeof(unsigned) * w.K, st);  // appends after *count
  const int grid = (int)std::min<int64_t>((w.S + 255) / 256, 1184);
  band_seed_kernel<<<grid, 256, 0, st>>>(bf, w.S, w.sample, w.bounds, w.K, w.flag,
                                         w.sample_counts, ranks, fits, fit, cap, count);
}

void launch_band_collect(const BandFit& bf, const BandWork& w, const BandRuns& runs, int64_t cap,
                         int sms, cudaStream_t st) {
  cudaMemsetAsync(w.ncollect, 0, sizeof(unsigned long long), st);
  switch (runs.count) {
#define LMSB_COLLECT(R)                                                                       \
  case R: {                                                                                   \
    static DeviceOnce done;                                                                 \
    set_smem(band_collect_kernel<R>, band_collect_smem(kBandMaxK), &done);                    \
    band_collect_kernel<R><<<sms * 4, kCollectThreads, band_collect_smem(w.K), st>>>(         \
        bf, w.bounds, w.K, w.slot, runs, w.ckeys, w.cvals, cap, w.ncollect);                  \
    break;                                                                                    \
  }
    LMSB_COLLECT(1)
    LMSB_COLLECT(2)
    LMSB_COLLECT(3)
    LMSB_COLLECT(4)
    LMSB_COLLECT(5)
    LMSB_COLLECT(6)
    LMSB_COLLECT(7)
    default:
    LMSB_COLLECT(8)
#undef LMSB_COLLECT
  }
}

// Split form of the pass-0 screen for few survivors: (tile of 32 vertices,
// slice of the lines) work items over the whole GPU, partial window counts
// added into per-vertex global counters; a second kernel applies the test
// and clears the counters for the next use.
__global__ void __launch_bounds__(kPreThreads) band_prepass_count_kernel(
    BandFit bf, const lms_candidate* __restrict__ best, const int64_t* __restrict__ in_ranks,
    const unsigned long long* __restrict__ in_count, unsigned* __restrict__ gcnt) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* sl = reinterpret_cast<double2*>(smem_raw);
  unsigned* cnt = reinterpret_cast<unsigned*>(sl + kPreLines);  // [2][32]
  const int64_t total = (int64_t)*in_count;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = (int)bf.n;
  const int64_t ntiles = (total + 31) / 32;
  if (ntiles == 0) return;
  const lms_candidate rec = *best;
  const int64_t want = ((int64_t)gridDim.x + ntiles - 1) / ntiles;
  const int nsplit = (int)max((int64_t)1, min(want, (int64_t)((n + 1023) / 1024)));
  const int64_t nwork = ntiles * nsplit;
  for (int64_t wk = blockIdx.x; wk < nwork; wk += gridDim.x) {
    const int64_t tile = wk / nsplit;
    const int sp = (int)(wk % nsplit);
    const int L0 = (int)((int64_t)n * sp / nsplit), L1 = (int)((int64_t)n * (sp + 1) / nsplit);
    const int64_t s = tile * 32 + lane;
    bool live = s < total;
    double u = 0.0, v0 = 0.0, bound = INFINITY;
    if (live) {
      int64_t i, j;
      decode_rank(bf.n, in_ranks[s], &i, &j);
      const double ai = bf.a[i], bi = bf.b[i];
      const double da = __dsub_rn(ai, bf.a[j]);
      u = __ddiv_rn(__dsub_rn(bi, bf.b[j]), da);
      v0 = cut_value(u, ai, bi);
      if (rec.found) {
        const bool after = i > rec.i || (i == rec.i && j > rec.j);
        bound = after ? nextafter(rec.height, -INFINITY) : rec.height;
      }
    }
    if (tid < 64) cnt[tid] = 0u;
    unsigned cu = 0, cd = 0;
    for (int c0 = L0; c0 < L1; c0 += kPreLines) {
      const int cn = min(kPreLines, L1 - c0);
      __syncthreads();
      for (int k = tid; k < cn; k += kPreThreads) sl[k] = bf.ab[c0 + k];
      __syncthreads();
      const int per = (cn + kPreWarps - 1) / kPreWarps;
      const int k0 = warp * per, k1 = min(cn, k0 + per);
#pragma unroll 4
      for (int k = k0; k < k1; ++k) {
        const double2 L = sl[k];
        const double x = cut_value(u, L.x, L.y);
        const double dx = __dsub_rn(x, v0), dv = __dsub_rn(v0, x);
        cu += (x >= v0) & (dx <= bound);
        cd += (x <= v0) & (dv <= bound);
      }
    }
    atomicAdd(cnt + lane, cu);
    atomicAdd(cnt + 32 + lane, cd);
    __syncthreads();
    if (warp == 0 && live) {
      atomicAdd(gcnt + 2 * s, cnt[lane]);
      atomicAdd(gcnt + 2 * s + 1, cnt[32 + lane]);
    }
    __syncthreads();
  }
}

__global__ void band_prepass_select_kernel(BandFit bf, const lms_candidate* __restrict__ best,
                                           const int64_t* __restrict__ in_ranks,
                                           const unsigned long long* __restrict__ in_count,
                                           unsigned* __restrict__ gcnt,
                                           int64_t* __restrict__ out_ranks,
                                           int32_t* __restrict__ out_fits, int32_t fit,
                                           unsigned long long* __restrict__ out_count) {
  const int64_t total = (int64_t)*in_count;
  const int lane = threadIdx.x & 31;
  const lms_candidate rec = *best;
  const int q = (int)bf.q;
  for (int64_t s0 = (int64_t)blockIdx.x * blockDim.x; s0 < total; s0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = s0 + threadIdx.x;
    bool keep = false;
    int64_t rank = 0;
    if (s < total) {
      int64_t i, j;
      rank = in_ranks[s];
      decode_rank(bf.n, rank, &i, &j);
      const double ai = bf.a[i], bi = bf.b[i];
      const double da = __dsub_rn(ai, bf.a[j]);
      const double u = __ddiv_rn(__dsub_rn(bi, bf.b[j]), da);
      const double v0 = cut_value(u, ai, bi);
      double bound = INFINITY;
      if (rec.found) {
        const bool after = i > rec.i || (i == rec.i && j > rec.j);
        bound = after ? nextafter(rec.height, -INFINITY) : rec.height;
      }
      int tu = (int)gcnt[2 * s], td = (int)gcnt[2 * s + 1];
      gcnt[2 * s] = 0u;  // cleared for the next use
      gcnt[2 * s + 1] = 0u;
      const double xj = cut_value(u, bf.a[j], bf.b[j]);
      tu += 1 - (int)((xj >= v0) & (__dsub_rn(xj, v0) <= bound));
      td += 1 - (int)((xj <= v0) & (__dsub_rn(v0, xj) <= bound));
      keep = da != 0.0 && bound >= 0.0 && (!isfinite(bound) || tu >= q || td >= q);
    }
    const unsigned mask = __ballot_sync(0xffffffffu, keep);
    if (mask) {
      unsigned long long base = 0;
      const int leader = __ffs(mask) - 1;
      if (lane == leader) base = atomicAdd(out_count, (unsigned long long)__popc(mask));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (keep) {
        const unsigned slot = __popc(mask & ((1u << lane) - 1u));
        out_ranks[base + slot] = rank;
        out_fits[base + slot] = fit;
      }
    }
  }
}

void launch_band_prepass_split(const BandFit& bf, const BandCount& bc, unsigned* gcnt, int sms,
                               cudaStream_t st) {
  cudaMemsetAsync(bc.out_count, 0, sizeof(unsigned long long), st);
  const size_t smem = (size_t)kPreLines * sizeof(double2) + 64 * sizeof(unsigned);
  static DeviceOnce done;
  set_smem(band_prepass_count_kernel, smem, &done);
  band_prepass_count_kernel<<<sms * LMSB_PRE_CTAS, kPreThreads, smem, st>>>(bf, bc.best, bc.in_ranks, bc.in_count,
                                                            gcnt);
  band_prepass_select_kernel<<<sms * 2, 256, 0, st>>>(bf, bc.best, bc.in_ranks, bc.in_count, gcnt,
                                                      bc.out_ranks, bc.out_fits, bc.fit,
                                                      bc.out_count);
}

void launch_band_exact_prepass(const BandFit& bf, const BandCount& bc, int sms, cudaStream_t st) {
  cudaMemsetAsync(bc.out_count, 0, sizeof(unsigned long long), st);
  const size_t smem = (size_t)kPreLines * sizeof(double2) + 64 * sizeof(unsigned);
  static DeviceOnce done;
  set_smem(band_exact_prepass_kernel, smem, &done);
  band_exact_prepass_kernel<<<sms, kPreThreads, smem, st>>>(bf, bc.best, bc.in_ranks, bc.in_count,
                                                            bc.out_ranks, bc.out_fits, bc.fit,
                                                            bc.out_count);
}

void launch_band_count(const BandFit& bf, const BandCount& bc, int sms, cudaStream_t st) {
  if (bc.make_lines) band_lines32_kernel<<<(int)((bf.n + 256) / 256), 256, 0, st>>>(bf, bc.lines);
  cudaMemsetAsync(bc.out_count, 0, sizeof(unsigned long long), st);
  const size_t smem = (size_t)std::min<int64_t>(bf.n + (bf.n & 1), kBandMaxN) * sizeof(float2) +
                      64 * sizeof(unsigned);
  static DeviceOnce done;
  set_smem(band_count_kernel, (size_t)kBandMaxN * sizeof(float2) + 64 * sizeof(unsigned), &done);
  band_count_kernel<<<sms, kCountThreads, smem, st>>>(bf, bc.lines, bc.best, bc.in_ranks,
                                                      bc.in_count, bc.out_ranks, bc.out_fits,
                                                      bc.fit, bc.out_count);
}


size_t band_direct_smem(int K, int nsub, int nadm) {
  return (size_t)(kCollectThreads / 32) * 64 * sizeof(uint32_t) + (size_t)K * sizeof(float) +
         (size_t)nsub * sizeof(float) + (size_t)(nadm + 1) * sizeof(int32_t) +
         (size_t)K * sizeof(int16_t) + 16;
}

void launch_band_collect_direct(const BandFit& bf, const BandWork& w, const BandRuns& runs,
                                const BandDirect& dg, int sms, cudaStream_t st) {
  band_subbounds_kernel<<<std::max(dg.nadm, 1), 128, 0, st>>>(w.sample_sorted, w.nvalid, w.bounds,
                                                              w.K, dg.list, dg.sb_first, dg.nadm,
                                                              dg.sub, nullptr);
  const size_t smem = band_direct_smem(w.K, dg.nsub, dg.nadm);
  switch (runs.count) {
#define LMSB_DIRECT(R)                                                                        \
  case R: {                                                                                   \
    cudaFuncSetAttribute(band_collect_direct_kernel<R>,                                       \
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);             \
    band_collect_direct_kernel<R><<<sms * 4, kCollectThreads, smem, st>>>(bf, w.bounds, w.K,  \
                                                                          runs, dg);          \
    break;                                                                                    \
  }
    LMSB_DIRECT(1)
    LMSB_DIRECT(2)
    LMSB_DIRECT(3)
    LMSB_DIRECT(4)
    LMSB_DIRECT(5)
    LMSB_DIRECT(6)
    LMSB_DIRECT(7)
    default:
    LMSB_DIRECT(8)
#undef LMSB_DIRECT
  }
}

// Grouping of the collected vertices by (slot, top slope bits): one bucket
// (counting) sort instead of a full radix sort of the keys -- the filter only
// needs every group contiguous and its chunks slope-local (each chunk takes
// its own slope extent from its members), not the order inside a bucket.
// Pass 1: per-CTA shared-memory histograms added into global counts; one CTA
// scans them (and writes each slot's [start, end)); pass 2: per-CTA
// histograms again, one global reservation per (CTA, bucket), members
// scattered to their reserved ranges.
__global__ void __launch_bounds__(1024) group_hist_kernel(const uint32_t* __restrict__ keys, int64_t m,
                                                          int shift, int nb,
                                                          unsigned long long* __restrict__ counts) {
  extern __shared__ unsigned int gh[];
  for (int e = threadIdx.x; e < nb; e += blockDim.x) gh[e] = 0u;
  __syncthreads();
  for (int64_t p = (int64_t)blockIdx.x * kGroupTile + threadIdx.x;
       p < m && p < (int64_t)(blockIdx.x + 1) * kGroupTile; p += blockDim.x)
    atomicAdd(&gh[keys[p] >> shift], 1u);
  __syncthreads();
  for (int e = threadIdx.x; e < nb; e += blockDim.x)
    if (gh[e]) atomicAdd(&counts[e], (unsigned long long)gh[e]);
}

__global__ void __launch_bounds__(1024) group_scan_kernel(const unsigned long long* __restrict__ counts,
                                                          int nb, int per_slot, int nslot,
                                                          unsigned long long* __restrict__ cursor,
                                                          int64_t* __restrict__ start,
                                                          int64_t* __restrict__ end) {
  __shared__ int64_t part[1024];
  const int per = (nb + 1023) / 1024;
  const int b0 = threadIdx.x * per, b1 = b0 + per < nb ? b0 + per : nb;
  int64_t sum = 0;
  for (int b = b0; b < b1; ++b) sum += (int64_t)counts[b];
  part[threadIdx.x] = sum;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    const int64_t v = threadIdx.x >= off ? part[threadIdx.x - off] : 0;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  int64_t run = threadIdx.x ? part[threadIdx.x - 1] : 0;
  for (int b = b0; b < b1; ++b) {
    cursor[b] = (unsigned long long)run;
    if (b % per_slot == 0) start[b / per_slot] = run;
    run += (int64_t)counts[b];
    if ((b + 1) % per_slot == 0) end[b / per_slot] = run;
  }
  (void)nslot;
}

__global__ void __launch_bounds__(1024) group_scatter_kernel(const uint32_t* __restrict__ keys,
                                                             const uint32_t* __restrict__ vals, int64_t m,
                                                             int shift, int nb,
                                                             unsigned long long* __restrict__ cursor,
                                                             uint32_t* __restrict__ out) {
  extern __shared__ unsigned int gh[];  // [nb] counts, then [nb] bases (64-bit)
  unsigned long long* base = reinterpret_cast<unsigned long long*>(gh + ((nb + 1) & ~1));
  for (int e = threadIdx.x; e < nb; e += blockDim.x) gh[e] = 0u;
  __syncthreads();
  const int64_t t0 = (int64_t)blockIdx.x * kGroupTile;
  const int64_t t1 = t0 + kGroupTile < m ? t0 + kGroupTile : m;
  for (int64_t p = t0 + threadIdx.x; p < t1; p += blockDim.x) atomicAdd(&gh[keys[p] >> shift], 1u);
  __syncthreads();
  for (int e = threadIdx.x; e < nb; e += blockDim.x) {
    base[e] = gh[e] ? atomicAdd(&cursor[e], (unsigned long long)gh[e]) : 0ull;
    gh[e] = 0u;
  }
  __syncthreads();
  for (int64_t p = t0 + threadIdx.x; p < t1; p += blockDim.x) {
    const int b = (int)(keys[p] >> shift);
    out[base[b] + atomicAdd(&gh[b], 1u)] = vals[p];
  }
}

int launch_band_group(const BandWork& w, int64_t m, bool full_order, cudaStream_t st) {
  cudaMemsetAsync(w.start, 0, sizeof(int64_t) * w.nslot, st);
  cudaMemsetAsync(w.end, 0, sizeof(int64_t) * w.nslot, st);
  if (m <= 0) return 0;
  if (full_order) {
    // n <= kBandMaxN: the filter's chunks are cut from the members in full
    // slope order (17 bits within the band) -- inside a band the members
    // crowd near the optimum slope, where coarser buckets would give chunks
    // 10x wider extents (12x the survivors measured)
    size_t bytes = w.temp_bytes;
    if (cub::DeviceRadixSort::SortPairs(w.temp, bytes, w.ckeys, w.ckeys_alt, w.cvals, w.members,
                                        (int)m, 0, kSlopeBits + bits_for(w.nslot - 1), st) !=
        cudaSuccess)
      return -1;
    band_runs_kernel<<<(int)std::min<int64_t>((m + 255) / 256, 4096), 256, 0, st>>>(
        w.ckeys_alt, m, w.start, w.end);
    return 0;
  }
  // slope bits kept per slot: as many as fit kGroupBuckets buckets (<= 8)
  int sb = 8;
  while (sb > 0 && ((int64_t)w.nslot << sb) > kGroupBuckets) --sb;
  const int shift = kSlopeBits - sb;
  const int per_slot = 1 << sb;
  const int nb = w.nslot * per_slot;
  if ((size_t)3 * (nb + 1) * sizeof(int64_t) > w.temp_bytes) return -1;
  unsigned long long* counts = reinterpret_cast<unsigned long long*>(w.temp);
  unsigned long long* cursor = counts + (nb + 1);
  cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * nb, st);
  const int tiles = (int)((m + kGroupTile - 1) / kGroupTile);
  static DeviceOnce d1, d2;
  const size_t smem1 = (size_t)nb * sizeof(unsigned);
  const size_t smem2 = (size_t)((nb + 1) & ~1) * sizeof(unsigned) + (size_t)nb * sizeof(unsigned long long);
  if (smem2 > 200 * 1024) return -1;
  set_max_smem(group_hist_kernel, 200 * 1024, d1);
  set_max_smem(group_scatter_kernel, 200 * 1024, d2);
  group_hist_kernel<<<tiles, 1024, smem1, st>>>(w.ckeys, m, shift, nb, counts);
  group_scan_kernel<<<1, 1024, 0, st>>>(counts, nb, per_slot, w.nslot, cursor, w.start, w.end);
  group_scatter_kernel<<<tiles, 1024, smem2, st>>>(w.ckeys, w.cvals, m, shift, nb, cursor, w.members);
  return 0;
}

// ---- sub-band grouping: counting sort of the collected members by group
// key, the member count read on the device (no host round trip for it).
// Pass 1 (sub_hist_kernel): per-CTA shared-memory histograms over a
// grid-stride range, added into the global counts once per CTA; one CTA
// scans them into group ranges and cursors (and clears the counts); pass 2
// (sub_scatter_kernel): per tile a shared-memory histogram, one global
// reservation per (tile, group), members scattered into the reservations.
constexpr int kSubTile = 4096;

__device__ __forceinline__ int64_t sub_count(const unsigned long long* m, int64_t cap) {
  const int64_t v = (int64_t)*m;
  return v < cap ? v : cap;
}

__global__ void __launch_bounds__(1024) sub_hist_kernel(const uint32_t* __restrict__ keys,
                                                        const unsigned long long* __restrict__ dm,
                                                        int64_t cap, int nb,
                                                        unsigned long long* __restrict__ counts,
                                                        const int* __restrict__ dnb) {
  if (dnb) nb = *dnb;
  extern __shared__ unsigned int sh_hist[];
  for (int e = threadIdx.x; e < nb; e += blockDim.x) sh_hist[e] = 0u;
  __syncthreads();
  const int64_t m = sub_count(dm, cap);
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m;
       p += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&sh_hist[min(keys[p], (uint32_t)(nb - 1))], 1u);
  __syncthreads();
  for (int e = threadIdx.x; e < nb; e += blockDim.x)
    if (sh_hist[e]) atomicAdd(&counts[e], (unsigned long long)sh_hist[e]);
}

__global__ void __launch_bounds__(1024) sub_scan_kernel(unsigned long long* __restrict__ counts,
                                                        int nb,
                                                        unsigned long long* __restrict__ cursor,
                                                        int64_t* __restrict__ start,
                                                        int64_t* __restrict__ end,
                                                        const int* __restrict__ dnb) {
  if (dnb) nb = *dnb;
  __shared__ unsigned long long part[1024];
  const int per = (nb + 1023) / 1024;
  const int b0 = min((int)threadIdx.x * per, nb), b1 = min(b0 + per, nb);
  unsigned long long sum = 0;
  for (int b = b0; b < b1; ++b) sum += counts[b];
  part[threadIdx.x] = sum;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    const unsigned long long v = threadIdx.x >= off ? part[threadIdx.x - off] : 0ull;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  unsigned long long run = threadIdx.x ? part[threadIdx.x - 1] : 0ull;
  for (int b = b0; b < b1; ++b) {
    cursor[b] = run;
    start[b] = (int64_t)run;
    run += counts[b];
    end[b] = (int64_t)run;
    counts[b] = 0ull;  // left zero for the next grouping
  }
}

__global__ void __launch_bounds__(1024) sub_scatter_kernel(const uint32_t* __restrict__ keys,
                                                           const uint32_t* __restrict__ vals,
                                                           const unsigned long long* __restrict__ dm,
                                                           int64_t cap, int nb,
                                                           unsigned long long* __restrict__ cursor,
                                                           uint32_t* __restrict__ out,
                                                           const int* __restrict__ dnb) {
  extern __shared__ unsigned int sh_hist[];  // [nb] counts, then [nb] bases (64-bit)
  // (the base array sits after the launch-time maximum of nb)
  unsigned long long* base = reinterpret_cast<unsigned long long*>(sh_hist + ((nb + 1) & ~1));
  if (dnb) nb = *dnb;
  const int64_t m = sub_count(dm, cap);
  constexpr int kPer = kSubTile / 1024;
  for (int64_t t0 = (int64_t)blockIdx.x * kSubTile; t0 < m; t0 += (int64_t)gridDim.x * kSubTile) {
    const int64_t t1 = t0 + kSubTile < m ? t0 + kSubTile : m;
    for (int e = threadIdx.x; e < nb; e += blockDim.x) sh_hist[e] = 0u;
    __syncthreads();
    uint32_t k[kPer], v[kPer];
#pragma unroll
    for (int r = 0; r < kPer; ++r) {
      const int64_t p = t0 + r * 1024 + threadIdx.x;
      k[r] = 0u;
      v[r] = 0u;
      if (p < t1) {
        k[r] = min(keys[p], (uint32_t)(nb - 1));
        v[r] = vals[p];
        atomicAdd(&sh_hist[k[r]], 1u);
      }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nb; e += blockDim.x) {
      base[e] = sh_hist[e] ? atomicAdd(&cursor[e], (unsigned long long)sh_hist[e]) : 0ull;
      sh_hist[e] = 0u;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kPer; ++r) {
      const int64_t p = t0 + r * 1024 + threadIdx.x;
      if (p < t1) out[base[k[r]] + atomicAdd(&sh_hist[k[r]], 1u)] = v[r];
    }
    __syncthreads();
  }
}

void launch_band_subbounds(const BandWork& w, const int32_t* list, const int32_t* sb_first,
                           int nadm, float* sub, cudaStream_t st, const int* dnadm) {
  band_subbounds_kernel<<<std::max(nadm, 1), 128, 0, st>>>(w.sample_sorted, w.nvalid, w.bounds,
                                                           w.K, list, sb_first, nadm, sub, dnadm);
}

int launch_band_group_sub(const uint32_t* keys, const uint32_t* vals,
                          const unsigned long long* m, int64_t cap, int ngroups,
                          unsigned long long* counts, unsigned long long* cursor, int64_t* start,
                          int64_t* end, uint32_t* members, cudaStream_t st, const int* dngroups) {
  if (ngroups <= 0 || ngroups > kSubMaxGroups) return -1;
  static DeviceOnce d1, d2;
  const size_t smem1 = (size_t)ngroups * sizeof(unsigned);
  const size_t smem2 = (size_t)((ngroups + 1) & ~1) * sizeof(unsigned) +
                       (size_t)ngroups * sizeof(unsigned long long);
  set_max_smem(sub_hist_kernel, 200 * 1024, d1);
  set_max_smem(sub_scatter_kernel, 200 * 1024, d2);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = (std::max<int64_t>(cap, 1) + kSubTile - 1) / kSubTile;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)sms * 2));
  sub_hist_kernel<<<grid, 1024, smem1, st>>>(keys, m, cap, ngroups, counts, dngroups);
  sub_scan_kernel<<<1, 1024, 0, st>>>(counts, ngroups, cursor, start, end, dngroups);
  sub_scatter_kernel<<<grid, 1024, smem2, st>>>(keys, vals, m, cap, ngroups, cursor, members,
                                                dngroups);
  return 0;
}


// Filter chunks of a slot's consecutive groups [g0, g1): greedy packing into
// chunks of <= chunk members (a group larger than chunk alone, split
// evenly).  One warp per slot: the group sizes are loaded 32 at a time and
// lane 0 walks them from registers (shuffles); run twice, counting first,
// then writing at the reserved position.
template <typename Emit>
__device__ __forceinline__ void pack_groups_warp(int g0, int g1, const int64_t* __restrict__ gstart,
                                                 const int64_t* __restrict__ gend, int64_t chunk,
                                                 Emit emit) {
  const int lane = threadIdx.x & 31;
  int64_t c0 = 0, cur = 0;
  for (int b = g0; b < g1; b += 32) {
    const int g = b + lane;
    int64_t s0 = 0, cnt = 0;
    if (g < g1) {
      s0 = gstart[g];
      cnt = gend[g] - s0;
    }
    const int nb = min(32, g1 - b);
    for (int t = 0; t < nb; ++t) {
      const int64_t ts = __shfl_sync(0xffffffffu, s0, t);
      const int64_t tc = __shfl_sync(0xffffffffu, cnt, t);
      if (lane != 0 || tc <= 0) continue;
      if (cur > 0 && cur + tc > chunk) {  // close the open chunk before this group
        emit(c0, c0 + cur);
        cur = 0;
      }
      if (tc > chunk) {
        const int64_t pieces = (tc + chunk - 1) / chunk, cs = (tc + pieces - 1) / pieces;
        for (int64_t p = ts; p < ts + tc; p += cs) emit(p, min(p + cs, ts + tc));
        continue;
      }
      if (cur == 0) c0 = ts;
      cur += tc;
    }
  }
  if (lane == 0 && cur > 0) emit(c0, c0 + cur);
}

#ifndef LMSB_PACK_FIXED
#define LMSB_PACK_FIXED 1
#endif
constexpr bool kPackFixed = LMSB_PACK_FIXED != 0;

__global__ void band_pack_chunks_kernel(const int32_t* __restrict__ sbf, int nslot,
                                        const int64_t* __restrict__ gstart,
                                        const int64_t* __restrict__ gend,
                                        const int32_t* __restrict__ gband, int64_t chunk,
                                        int64_t chunk_one, int64_t* __restrict__ ctab,
                                        int32_t* __restrict__ cband,
                                        unsigned long long* __restrict__ nct,
                                        const int* __restrict__ dnslot, int which) {
  if (dnslot) nslot = *dnslot;
  const int e = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (e >= nslot) return;
  const int g0 = sbf[e], g1 = sbf[e + 1];
  if (g1 <= g0) return;
  // which: 1 the multi-group (wide) slots, 2 the one-group slots
  if ((which == 1) != (g1 - g0 > 1)) return;
  const int band = gband[g0];
  // a one-group slot (a narrow band read with its stored keys): chunk_one
  if (g1 - g0 == 1) chunk = chunk_one;
  if (kPackFixed) {
    // fixed-size chunks over the slot's member range (its groups are slope
    // ordered, so a chunk spans at most a few adjacent groups)
    const int lane = threadIdx.x & 31;
    const int64_t s0 = gstart[g0], s1 = gend[g1 - 1];
    const int64_t ncs = s1 > s0 ? (s1 - s0 + chunk - 1) / chunk : 0;
    if (ncs == 0) return;
    unsigned long long at = 0;
    if (lane == 0) at = atomicAdd(nct, (unsigned long long)ncs);
    at = __shfl_sync(0xffffffffu, at, 0);
    for (int64_t c = lane; c < ncs; c += 32) {
      ctab[2 * (at + c)] = s0 + c * chunk;
      ctab[2 * (at + c) + 1] = min(s1, s0 + (c + 1) * chunk);
      cband[at + c] = band;
    }
    return;
  }
  unsigned long long nc = 0;
  pack_groups_warp(g0, g1, gstart, gend, chunk, [&](int64_t, int64_t) { ++nc; });
  unsigned long long at = 0;
  if ((threadIdx.x & 31) == 0 && nc) at = atomicAdd(nct, nc);
  if (__shfl_sync(0xffffffffu, nc, 0) == 0) return;
  pack_groups_warp(g0, g1, gstart, gend, chunk, [&](int64_t a, int64_t b) {
    ctab[2 * at] = a;
    ctab[2 * at + 1] = b;
    cband[at] = band;
    ++at;
  });
}

void launch_band_pack_chunks(const int32_t* sb_first, int nslot, const int64_t* gstart,
                             const int64_t* gend, const int32_t* gband, int64_t chunk,
                             int64_t chunk_one, int64_t* ctab, int32_t* cband,
                             unsigned long long* nctab, cudaStream_t st, const int* dnslot) {
  cudaMemsetAsync(nctab, 0, sizeof(unsigned long long), st);
  if (nslot <= 0) return;
  // wide bands' chunks (each sorts its keys: the heavy ones) first in the
  // table, so the filter's persistent CTAs do not end on them
  for (int which = 1; which <= 2; ++which)
    band_pack_chunks_kernel<<<(nslot + 3) / 4, 128, 0, st>>>(sb_first, nslot, gstart, gend, gband,
                                                              chunk, chunk_one, ctab, cband,
                                                              nctab, dnslot, which);
}

// ---- device-side plan of a band search (DevPlan, lms_band.cuh): the host
// planning of band_solve after the seeds, on one CTA, so the search needs no
// readback.  Same decisions as the host: admitted bands lb <= H (1 + 2^-19);
// sweep runs of the admitted and outer bands merged across the smallest gaps
// (ties: the earliest first) down to kPlanMaxRuns; run ends with the
// clearance and near-parallel threshold of band_solve; narrow bands one
// group, wide bands one sub-band per sorted sample.  Slots follow the band
// index (the host orders them by lb; only the member layout differs).
constexpr int kPlanThreads = 1024;
constexpr int kPlanPer = kPlanMaxK / kPlanThreads;  // bands per thread

// exclusive block scan of one int per thread; *total the sum
__device__ __forceinline__ int plan_scan(int v, int* wtot, int* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  __syncthreads();
  if (lane == 31) wtot[w] = incl;
  __syncthreads();
  if (w == 0) {
    const int t = wtot[lane];
    int ti = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, ti, o);
      if (lane >= o) ti += y;
    }
    wtot[lane] = ti - t;
    if (lane == 31) wtot[32] = ti;
  }
  __syncthreads();
  *total = wtot[32];
  return wtot[w] + incl - v;
}

__global__ void __launch_bounds__(kPlanThreads) band_plan_kernel(
    BandFit bf, const float* __restrict__ bnd, const unsigned* __restrict__ scnt,
    const double* __restrict__ lb, const lms_candidate* __restrict__ best, int K, int sub_samples,
    double bkeys_tau, DevPlan dp) {
  __shared__ int wtot[33];
  __shared__ int rk0[kPlanMaxK / 2 + 2], rk1[kPlanMaxK / 2 + 2];
  __shared__ int fk0[kPlanMaxRuns], fk1[kPlanMaxRuns];
  __shared__ unsigned char act[kPlanMaxK];
  __shared__ int s_bail;
  __shared__ double s_tau;
  __shared__ unsigned long long s_est;
  const int tid = threadIdx.x;
  const lms_candidate rec = *best;
  const double H = rec.found ? rec.height : INFINITY;
  const double thr = H * (1.0 + 0x1p-19);
  if (tid == 0) {
    s_bail = K > kPlanMaxK ? 1 : 0;
    s_tau = 0.0;
    s_est = 0ull;
  }
  __syncthreads();
  if (s_bail) {
    if (tid == 0) dp.hdr->bail = 1;
    return;
  }
  const int kb = tid * kPlanPer, ke = min(K, kb + kPlanPer);
  // (a) admitted bands -> slots; the sample estimate; sweep eligibility
  bool adm[kPlanPer];
  int cnt = 0;
  unsigned long long est = 0;
  bool bad = false;
#pragma unroll
  for (int t = 0; t < kPlanPer; ++t) {
    const int k = kb + t;
    adm[t] = k < ke && lb[k] <= thr;
    cnt += adm[t];
    if (adm[t]) est += (unsigned long long)scnt[k] + 2ull;
    if (k < ke && k < K - 1) bad |= !(isfinite(bnd[k]) && fabs((double)bnd[k]) * bf.amax < 1e29);
  }
  if (bad) atomicOr(&s_bail, 1);
  if (est) atomicAdd(&s_est, est);
  int nadm = 0;
  int base = plan_scan(cnt, wtot, &nadm);
#pragma unroll
  for (int t = 0; t < kPlanPer; ++t) {
    const int k = kb + t;
    if (k >= ke) break;
    if (adm[t]) {
      dp.slot[k] = (int16_t)base;
      dp.list[base] = k;
      ++base;
    } else {
      dp.slot[k] = -1;
    }
    act[k] = adm[t];  // (the outer bands only when admitted: see (d))
  }
  for (int e = tid; e <= nadm; e += kPlanThreads) dp.ident[e] = e;
  if (tid == 0) {
    dp.slot[K] = (int16_t)nadm;
    dp.list[nadm] = K;
  }
  __syncthreads();
  // (b) maximal runs of active bands (the j-th start pairs with the j-th end)
  int ns = 0;
#pragma unroll
  for (int t = 0; t < kPlanPer; ++t) {
    const int k = kb + t;
    if (k < ke && act[k] && (k == 0 || !act[k - 1])) ++ns;
  }
  int R0 = 0;
  int rb = plan_scan(ns, wtot, &R0);
#pragma unroll
  for (int t = 0; t < kPlanPer; ++t) {
    const int k = kb + t;
    if (k >= ke || !act[k]) continue;
    if (k == 0 || !act[k - 1]) rk0[rb++] = k;  // rb: runs started at or before k
    if (k == K - 1 || !act[k + 1]) rk1[rb - 1] = k;
  }
  __syncthreads();
  // (c) merge across the smallest gaps down to kPlanMaxRuns: gap j (between
  // runs j and j + 1) is kept when fewer than kPlanMaxRuns - 1 gaps rank
  // above it in (width desc, index desc) -- the host's greedy merging of
  // the smallest, earliest gap first
  int nr = R0;
  if (R0 > kPlanMaxRuns) {
    for (int j0 = 0; j0 < R0 - 1; j0 += kPlanThreads) {
      const int j = j0 + tid;
      bool keep = false;
      if (j < R0 - 1) {
        const int gj = rk0[j + 1] - rk1[j];
        int above = 0;
        for (int i = 0; i < R0 - 1 && above < kPlanMaxRuns - 1; ++i) {
          const int gi = rk0[i + 1] - rk1[i];
          above += (gi > gj) || (gi == gj && i > j);
        }
        keep = above < kPlanMaxRuns - 1;
      }
      if (j < R0 - 1) act[j] = keep;  // (act is free after (b): the kept gaps)
    }
    __syncthreads();
    if (tid == 0) {
      int r = 0;
      fk0[0] = rk0[0];
      for (int j = 0; j < R0 - 1; ++j)
        if (act[j]) {
          fk1[r++] = rk1[j];
          fk0[r] = rk0[j + 1];
        }
      fk1[r] = rk1[R0 - 1];
      nr = r + 1;
      wtot[0] = nr;
    }
    __syncthreads();
    nr = wtot[0];
  } else if (tid < R0) {
    fk0[tid] = rk0[tid];
    fk1[tid] = rk1[tid];
  }
  __syncthreads();
  if (nr == 0 || nadm == 0) atomicOr(&s_bail, 1);
  // (d) run ends, as band_solve: the bands' fp32 extents widened 2^-18, sort
  // ends a clearance m outside, tau = 4 e / m
  if (tid < nr) {
    const int k0 = fk0[tid], k1 = fk1[tid];
    double lo = -INFINITY, hi = INFINITY;
    if (k0 > 0) {
      lo = (double)nextafterf(bnd[k0 - 1], -INFINITY);
      lo -= 0x1p-18 * fabs(lo) + 1e-37;
    }
    if (k1 < K - 1) {
      hi = (double)bnd[k1];
      hi += 0x1p-18 * fabs(hi) + 1e-37;
    }
    double m;
    if (isfinite(lo) && isfinite(hi))
      m = 0x1p-20 * (fmax(fabs(lo), fabs(hi)) + (hi - lo)) + 1e-300;
    else
      m = 0x1p-20 * (isfinite(lo) ? fabs(lo) : isfinite(hi) ? fabs(hi) : 0.0) + 1e-300;
    const double s0 = lo - m, s1 = hi + m;
    double smax = 0.0;
    if (isfinite(s0)) smax = fabs(s0);
    if (isfinite(s1)) smax = fmax(smax, fabs(s1));
    const double err = 0x1p-52 * (bf.amax * smax + bf.bmax) + 1e-300;
    if (isfinite(s0) || isfinite(s1)) {
      const double tr = 4.0 * err / m;  // tau >= 0: integer-ordered atomicMax on the bits
      atomicMax(reinterpret_cast<unsigned long long*>(&s_tau),
                (unsigned long long)__double_as_longlong(tr));
    }
    const double fin = isfinite(s0) ? s0 : isfinite(s1) ? s1 : 0.0;
    dp.ends[2 * tid] = SweepEnd{isfinite(s0) ? s0 : 0.0, fin, isfinite(s0) ? 0 : 1, 0};
    dp.ends[2 * tid + 1] = SweepEnd{isfinite(s1) ? s1 : 0.0, fin, isfinite(s1) ? 0 : 2, 0};
    dp.rk[tid] = k0;
    dp.rk[kPlanMaxRuns + tid] = k1;
  }
  if (tid == 0) dp.ends[2 * kPlanMaxRuns] = SweepEnd{0.0, 0.0, 3, 0};
  // runs at the infinite ends are left out: the near-parallel pass owns
  // every class-2 pair when 2 bmax amax / 1e30 <= tau (band_solve's rule);
  // otherwise the host plans this fit (with the outer runs)
  __syncthreads();
  if (tid == 0 && !(2.0 * bf.bmax * bf.amax * (1.0 + 0x1p-20) <= 1e30 * s_tau)) s_bail = 1;
  // (e) sub-band groups: a narrow band one group, a wide one a group per
  // sub_samples sorted samples (<= 1,024); all bands one group each when
  // that would exceed kSubMaxGroups
  int se[kPlanPer];
  int scnt_local = 0;
#pragma unroll
  for (int t = 0; t < kPlanPer; ++t) {
    const int e = kb + t;
    se[t] = 0;
    if (e >= nadm) continue;
    const int k = dp.list[e];
    bool narrow = false;
    if (k > 0 && k < K - 1) {
      const double uL = (double)nextafterf(bnd[k - 1], -INFINITY), uR = (double)bnd[k];
      narrow = isfinite(uL) && isfinite(uR) && bf.dev * (uR - uL) <= bkeys_tau * H;
    }
    se[t] = narrow ? 1 : max(1, min(1024, (int)(scnt[k] / (unsigned)sub_samples)));
    scnt_local += se[t];
  }
  int G = 0;
  int gb = plan_scan(scnt_local, wtot, &G);
  const bool flat = G + 1 > kSubMaxGroups;
  if (flat) {
    G = nadm;
    gb = min(kb, nadm);
  }
#pragma unroll
  for (int t = 0; t < kPlanPer; ++t) {
    const int e = kb + t;
    if (e >= nadm) continue;
    const int k = dp.list[e];
    const int s_e = flat ? 1 : se[t];
    dp.sbf[e] = gb;
    for (int g = 0; g < s_e; ++g) dp.gband[gb + g] = k;
    gb += s_e;
  }
  __syncthreads();
  if (tid == 0) {
    dp.sbf[nadm] = G;
    dp.sbf[nadm + 1] = G + 1;
    dp.gband[G] = K;
    DevPlanHdr h{};
    h.nadm = nadm;
    h.nslot = nadm + 1;
    h.nr = nr;
    h.ngroups = G + 1;
    h.bail = s_bail;
    h.H = H;
    h.tau = s_tau;
    h.est = s_est;
    *dp.hdr = h;
  }
}

void launch_band_plan(const BandFit& bf, const BandWork& w, const double* lb,
                      const lms_candidate* best, int K, int sub_samples, double bkeys_tau,
                      const DevPlan& dp, cudaStream_t st) {
  band_plan_kernel<<<1, kPlanThreads, 0, st>>>(bf, w.bounds, w.sample_counts, lb, best, K,
                                               sub_samples, bkeys_tau, dp);
}

// Lower bound of the narrowest window holding q of the slopes a_k: the a_k
// binned linearly over [c - dev, c + dev] (which holds them all); a window
// whose first slope falls in bin i ends in a bin >= j*(i), the first where
// the counts from bin i reach q, so it is >= (j*(i) - i - 3) bin widths wide
// (one bin, plus one either side for the binning's roundings).
constexpr int kWqaBins = 8192;
__global__ void __launch_bounds__(1024) line_wqa_kernel(BandFit bf, double* __restrict__ out) {
  __shared__ unsigned P[kWqaBins + 1];
  __shared__ unsigned wsum[32];
  __shared__ double red[32];
  const int tid = threadIdx.x, lane = tid & 31;
  const int n = (int)bf.n, q = (int)bf.q;
  const double lo = bf.c - bf.dev;
  const double res = fmax(2.0 * bf.dev / kWqaBins, 1e-300) * (1.0 + 0x1p-30);
  for (int b = tid; b <= kWqaBins; b += 1024) P[b] = 0;
  __syncthreads();
  for (int k0 = 0; k0 < n; k0 += 16 * 1024) {  // 16 independent loads in flight per thread
    double av[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int k = k0 + e * 1024 + tid;
      av[e] = k < n ? __ldg(bf.a + k) : 0.0;
    }
#pragma unroll
    for (int e = 0; e < 16; ++e)
      if (k0 + e * 1024 + tid < n)
        atomicAdd(P + (int)fmin(fmax(floor((av[e] - lo) / res), 0.0), kWqaBins - 1.0), 1u);
  }
  __syncthreads();
  constexpr int kPer = kWqaBins / 1024;
  unsigned mine[kPer], sum = 0;
#pragma unroll
  for (int e = 0; e < kPer; ++e) {
    mine[e] = P[tid * kPer + e];
    sum += mine[e];
  }
  unsigned incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[tid >> 5] = incl;
  __syncthreads();
  unsigned base = incl - sum;
  for (int w = 0; w < (tid >> 5); ++w) base += wsum[w];
  __syncthreads();
#pragma unroll
  for (int e = 0; e < kPer; ++e) {
    P[tid * kPer + e] = base;  // keys in bins < tid * kPer + e
    base += mine[e];
  }
  if (tid == 1023) P[kWqaBins] = base;
  __syncthreads();
  // each thread walks its kPer consecutive start bins: one binary search for
  // the first end bin, then the end advances monotonically
  double best = INFINITY;
  {
    const int b0 = tid * kPer;
    int z = -1;
    for (int b1 = b0; b1 < b0 + kPer; ++b1) {
      const unsigned p1 = P[b1];
      if (P[kWqaBins] - p1 < (unsigned)q) break;  // (and for every later start)
      if (z < 0) {  // first b2 with P[b2 + 1] - p1 >= q
        int a = b1, hi = kWqaBins - 1;
        while (a < hi) {
          const int mid = (a + hi) >> 1;
          if (P[mid + 1] - p1 >= (unsigned)q) hi = mid;
          else a = mid + 1;
        }
        z = a;
      } else {
        if (z < b1) z = b1;
        while (P[z + 1] - p1 < (unsigned)q) ++z;
      }
      if (P[b1 + 1] != p1) best = fmin(best, (double)(z - b1));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = fmin(best, __shfl_xor_sync(0xffffffffu, best, o));
  if (lane == 0) red[tid >> 5] = best;
  __syncthreads();
  if (tid == 0) {
    double m = red[0];
    for (int w = 1; w < 32; ++w) m = fmin(m, red[w]);
    *out = isfinite(m) ? fmax(m - 3.0, 0.0) * res : 0.0;
  }
}

void launch_line_wqa(const BandFit& bf, double* out, cudaStream_t st) {
  line_wqa_kernel<<<1, 1024, 0, st>>>(bf, out);
}

}  // namespace lmsb
