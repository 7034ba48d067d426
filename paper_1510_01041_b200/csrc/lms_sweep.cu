// lms_sweep.cu -- output-sensitive collect of the band stage.
//
// The band stage must hand the filter every vertex (i, j) whose slope
// u = (b_i - b_j) / (a_i - a_j) (formed as _scan_rank_range does,
// backend.py:200-205) falls in a band whose lower bound admits H.  The
// admitted bands form a few slope runs [s0, s1].  Testing every one of the
// n(n-1)/2 vertices against the runs is O(n^2); this file enumerates the
// vertices of each run directly, in O(n log n + K) for K vertices in the run:
//
//   Two dual lines v = a u - b cross inside (s0', s1') exactly when their
//   order by value at s0' differs from their order at s1'.  Sort the lines
//   by value at both ends; with P[t] = position at s1' of the line at
//   position t at s0', the crossings are the inversions t < t', P[t'] < P[t].
//   A warp per t walks t' with per-32 block minima of P (skipping blocks
//   without a smaller value) and a suffix minimum (stopping when no smaller
//   value is left), so the work is proportional to the inversions found.
//
// Exactness (superset contract, as the pre-test it replaces): the runs are
// the admitted bands' fp32 extents widened by 2^-18 relative + 1e-37
// (lms_engine.cu); the sort ends s0' = lo - m and s1' = hi + m add a margin m
// so every vertex whose fp64 slope lies in the run has its real crossing u*
// at least m inside (s0', s1').  Keys are fma(a, s, -b) (one rounding,
// error <= 2^-53 |a s - b|), so two keys' errors sum to at most
// e = 2^-52 (amax |s| + bmax) + 1e-300; a crossing pair's true values differ
// at each end by |a_i - a_j| m, so for |a_i - a_j| > tau = 4 e / m the sorted
// orders are right at both ends and the pair is an inversion.  Pairs with
// 0 < |a_i - a_j| <= tau (nearly parallel lines) are skipped by the inversion
// pass and enumerated by a separate pass over the lines sorted by a.  An
// infinite end (the outer bands) sorts by slope exactly (a descending at
// -inf, ascending at +inf; equal slopes by their value at the finite end).
// Every enumerated pair is then classified with the reference's fp64 slope
// and kept only if its band is an admitted band of this run (or, beyond the
// fp32 key range, if the run is the outer one on that side), so each member
// is emitted once and the output is exactly the pre-test collect's member
// set: same (slot, slope position) keys, same packed i<<16|j values.

#include <cuda_runtime.h>

#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdint>

#include "lms_band.cuh"
#include "lms_band_dev.cuh"
#include "lms_common.cuh"

namespace lmsb {

namespace {

constexpr int kChunk = 2048;        // items per CTA-local bitonic sort (shared memory)
constexpr int kChunkThreads = 512;
constexpr int kMergeItems = 8;      // outputs per thread of a global merge round
constexpr int kMergeThreads = 256;
constexpr int kEnumThreads = 256;
constexpr int kEnumWarps = kEnumThreads / 32;
constexpr int kEnumQueue = 64;
constexpr int kOutBuf = 512;  // per-warp raw-pair buffer (one global atomic per ~480 pairs)
constexpr int kOutFlush = kOutBuf - 32;
constexpr int kClsBuf = 4096;  // per-CTA member buffer of the classification
constexpr int kClsUnroll = 4;  // pairs per thread per step of the classification
constexpr int kHitBatch = 4;

__device__ __forceinline__ int64_t i64min(int64_t x, int64_t y) { return x < y ? x : y; }
__device__ __forceinline__ int64_t i64max(int64_t x, int64_t y) { return x > y ? x : y; }

// items are (key, line id): keys unique with the id as the tie-break
__device__ __forceinline__ bool item_less(uint64_t ak, uint32_t ai, uint64_t bk, uint32_t bi) {
  return ak < bk || (ak == bk && ai < bi);
}

// Sort keys of every (segment, line): kind 0 finite end s (fma(a, s, -b)),
// 1 at -inf (a descending), 2 at +inf (a ascending), 3 by slope a (the
// near-parallel pass); equal keys in line order.
// a segment of a device-planned sweep that no run uses (SweepSort::dnr)
__device__ __forceinline__ bool seg_dead(int seg, const int32_t* dnr, int nr_max) {
  return dnr && seg < 2 * nr_max && seg >= 2 * *dnr;
}

__global__ void sweep_keys_kernel(const double2* __restrict__ ab, int n, const SweepEnd* __restrict__ ends,
                                  int nseg, uint64_t* __restrict__ k1, uint32_t* __restrict__ idx,
                                  const int32_t* __restrict__ dnr, int nr_max) {
  const int64_t total = (int64_t)nseg * n;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int s = (int)(g / n);
    const int k = (int)(g - (int64_t)s * n);
    if (seg_dead(s, dnr, nr_max)) continue;
    const SweepEnd e = ends[s];
    const double2 l = ab[k];
    uint64_t p;
    if (e.kind == 0) p = key_of(fma(l.x, e.s, -l.y));
    else if (e.kind == 1) p = key_of(-l.x);
    else p = key_of(l.x);
    k1[g] = p;
    idx[g] = (uint32_t)k;
  }
}

// One CTA sorts one chunk of kChunk items of one segment in shared memory
// (bitonic network over (key, line id); unique keys, deterministic order).
__global__ void __launch_bounds__(kChunkThreads) sweep_chunk_sort_kernel(
    int n, int chunks_per_seg, uint64_t* __restrict__ k1, uint32_t* __restrict__ idx,
    const int32_t* __restrict__ dnr, int nr_max) {
  __shared__ uint64_t sk[kChunk];
  __shared__ uint32_t si[kChunk];
  const int seg = blockIdx.x / chunks_per_seg;
  if (seg_dead(seg, dnr, nr_max)) return;
  const int c = blockIdx.x - seg * chunks_per_seg;
  const int64_t base = (int64_t)seg * n + (int64_t)c * kChunk;
  const int cnt = min(kChunk, n - c * kChunk);
  for (int t = threadIdx.x; t < kChunk; t += kChunkThreads) {
    sk[t] = t < cnt ? k1[base + t] : ~0ull;
    si[t] = t < cnt ? idx[base + t] : 0xFFFFFFFFu;
  }
  __syncthreads();
  for (int k = 2; k <= kChunk; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll
      for (int t = threadIdx.x; t < kChunk / 2; t += kChunkThreads) {
        const int lo = 2 * t - (t & (j - 1));
        const int hi = lo + j;
        const uint64_t a = sk[lo], b = sk[hi];
        const uint32_t ia = si[lo], ib = si[hi];
        if (item_less(b, ib, a, ia) == ((lo & k) == 0)) {
          sk[lo] = b;
          sk[hi] = a;
          si[lo] = ib;
          si[hi] = ia;
        }
      }
      __syncthreads();
    }
  }
  for (int t = threadIdx.x; t < cnt; t += kChunkThreads) {
    k1[base + t] = sk[t];
    idx[base + t] = si[t];
  }
}

// One global merge round: sorted runs of width w (per segment) pairwise into
// runs of 2w; merge path per thread (kMergeItems outputs).
__global__ void __launch_bounds__(kMergeThreads) sweep_merge_kernel(
    int n, int64_t w, int blocks_per_seg, const uint64_t* __restrict__ x1,
    const uint32_t* __restrict__ xi, uint64_t* __restrict__ y1, uint32_t* __restrict__ yi,
    const int32_t* __restrict__ dnr, int nr_max) {
  const int seg = blockIdx.x / blocks_per_seg;
  if (seg_dead(seg, dnr, nr_max)) return;
  const int64_t d0 =
      ((int64_t)(blockIdx.x - seg * blocks_per_seg) * kMergeThreads + threadIdx.x) * kMergeItems;
  if (d0 >= n) return;
  const int64_t sb = (int64_t)seg * n;
  const int64_t pbase = (d0 / (2 * w)) * (2 * w);
  const int64_t la = i64min(w, n - pbase);
  const int64_t lb = i64max(0, i64min(w, n - pbase - w));
  const int64_t a0 = sb + pbase, b0 = a0 + la;
  const int64_t dd = d0 - pbase;
  int64_t lo = i64max(0, dd - lb), hi = i64min(dd, la);
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    const int64_t jb = dd - mid - 1;
    if (item_less(x1[b0 + jb], xi[b0 + jb], x1[a0 + mid], xi[a0 + mid])) hi = mid;
    else lo = mid + 1;
  }
  int64_t ia = lo, ib = dd - lo;
  const int64_t end = i64min(d0 + kMergeItems, pbase + la + lb);
  for (int64_t d = d0; d < end; ++d) {
    bool takeA;
    if (ia >= la) takeA = false;
    else if (ib >= lb) takeA = true;
    else takeA = !item_less(x1[b0 + ib], xi[b0 + ib], x1[a0 + ia], xi[a0 + ia]);
    const int64_t src = takeA ? a0 + ia : b0 + ib;
    y1[sb + d] = x1[src];
    yi[sb + d] = xi[src];
    if (takeA) ++ia;
    else ++ib;
  }
}

// pos[run][line] = position of the line in the run's s1' order
__global__ void sweep_pos_kernel(int n, int nruns, const uint32_t* __restrict__ idx,
                                 int32_t* __restrict__ pos, const int32_t* __restrict__ dnr) {
  if (dnr) nruns = *dnr;
  const int64_t total = (int64_t)nruns * n;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(g / n);
    const int p = (int)(g - (int64_t)r * n);
    pos[(int64_t)r * n + idx[(int64_t)(2 * r + 1) * n + p]] = p;
  }
}

// P[run][t] = s1' position of the line at s0' position t, and per 32-block minima
__global__ void sweep_p_kernel(int n, int nruns, const uint32_t* __restrict__ idx,
                               const int32_t* __restrict__ pos, int32_t* __restrict__ P,
                               int32_t* __restrict__ bmin, const int32_t* __restrict__ dnr) {
  if (dnr) nruns = *dnr;
  const int nb = (n + 31) / 32;
  const int64_t total = (int64_t)nruns * nb * 32;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(g / ((int64_t)nb * 32));
    const int t = (int)(g - (int64_t)r * nb * 32);
    int v = INT_MAX;
    if (t < n) {
      v = pos[(int64_t)r * n + idx[(int64_t)(2 * r) * n + t]];
      P[(int64_t)r * n + t] = v;
    }
    int m = v;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, off));
    if ((threadIdx.x & 31) == 0) bmin[(int64_t)r * nb + (t >> 5)] = m;
  }
}

// suffix minima of the block minima, one CTA per run
__global__ void __launch_bounds__(1024) sweep_suffix_kernel(int n, const int32_t* __restrict__ bmin,
                                                            int32_t* __restrict__ suf,
                                                            const int32_t* __restrict__ dnr) {
  __shared__ int32_t part[1024];
  const int nb = (n + 31) / 32;
  const int r = blockIdx.x;
  if (dnr && r >= *dnr) return;
  const int per = (nb + 1023) / 1024;
  const int b0 = threadIdx.x * per;
  const int b1 = min(nb, b0 + per);
  const int32_t* bm = bmin + (int64_t)r * nb;
  int32_t* sf = suf + (int64_t)r * nb;
  int m = INT_MAX;
  for (int b = b1 - 1; b >= b0; --b) m = min(m, bm[b]);
  part[threadIdx.x] = m;
  __syncthreads();
  // inclusive suffix minimum over the thread totals (Hillis-Steele)
  for (int off = 1; off < 1024; off <<= 1) {
    const int v = threadIdx.x + off < 1024 ? part[threadIdx.x + off] : INT_MAX;
    __syncthreads();
    part[threadIdx.x] = min(part[threadIdx.x], v);
    __syncthreads();
  }
  m = threadIdx.x + 1 < 1024 ? part[threadIdx.x + 1] : INT_MAX;
  for (int b = b1 - 1; b >= b0; --b) {
    m = min(m, bm[b]);
    sf[b] = m;
  }
}

// Band of slope key bk if it lies in bands [k0, k1] of the K bands, else -1.
__device__ __forceinline__ int band_in_run(const float* bnd, int K, int k0, int k1, float bk) {
  if (k0 > 0 && !(bnd[k0 - 1] <= bk)) return -1;
  if (k1 < K - 1 && !(bk < bnd[k1])) return -1;
  int lo = k0, hi = k1;  // band = number of boundaries <= bk, in [k0, k1]
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;  // boundary mid separates bands mid and mid + 1
    if (bnd[mid] <= bk) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// (slot, slope position) key of a member of band `band` (lms_band.cu collect)
__device__ __forceinline__ uint32_t member_key(const float* bnd, int K, int band, float bk, int sb) {
  uint32_t t = 0;
  if (band > 0 && band < K - 1) {
    const float lo = bnd[band - 1], w = bnd[band] - lo;
    const float f = w > 0.f ? (bk - lo) / w * (float)(1 << kSlopeBits) : 0.f;
    t = (uint32_t)fminf(fmaxf(f, 0.f), (float)((1 << kSlopeBits) - 1));
  }
  return ((uint32_t)max(sb, 0) << kSlopeBits) | t;
}

// sub-band group of a member of slot sb (SweepArgs::sub_first): the slot's
// first group plus the number of its inner sub-band boundaries <= bk (the
// same convention as band_of)
__device__ __forceinline__ uint32_t sub_group(const SweepArgs& sa, int sb, float bk) {
  const int g0 = __ldg(sa.sub_first + sb);
  const float* s = sa.sub + (g0 - sb);
  int lo = 0, hi = __ldg(sa.sub_first + sb + 1) - g0 - 1;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(s + mid) <= bk) lo = mid + 1;
    else hi = mid;
  }
  return (uint32_t)(g0 + lo);
}

// Classify enumerated pair (k, l) and decide whether run (k0, k1) emits it
// (k0 < 0: the near-parallel pass, which owns every admitted band).
__device__ __forceinline__ bool sweep_take(const BandFit& bf, const SweepArgs& sa, const float* bnd,
                                           const int16_t* slot, int k0, int k1, bool parallel_pass,
                                           int k, int l, uint32_t* key, uint32_t* val) {
  const int i = min(k, l), j = max(k, l);
  if (i == j) return false;
  const int64_t r = row_offset(bf.n, i) + (j - i - 1);
  if (r < bf.R0 || r >= bf.R0 + bf.span) return false;
  const double2 li = bf.ab[i], lj = bf.ab[j];
  const double da = fabs(__dsub_rn(li.x, lj.x));
  if (!parallel_pass && da <= (sa.dtau ? __ldg(sa.dtau) : sa.tau))
    return false;  // the near-parallel pass owns it
  double u = 0.0;
  const int cls = classify(bf, li.x, li.y, lj.x, lj.y, &u);
  *val = ((uint32_t)i << 16) | (uint32_t)j;
  if (cls == 1) {
    const float bk = band_key(u);
    const int band = parallel_pass ? band_of(bnd, sa.K - 1, bk) : band_in_run(bnd, sa.K, k0, k1, bk);
    if (band < 0) return false;
    const int sb = slot[band];
    if (sb < 0) return false;
    *key = sa.sub_first ? sub_group(sa, sb, bk) : member_key(bnd, sa.K, band, bk, sb);
    return true;
  }
  if (cls == 2) {
    const bool own = parallel_pass || (u < 0.0 ? k0 == 0 : k1 == sa.K - 1);
    if (!own) return false;
    *key = sa.sub_first ? (uint32_t)sa.sub_first[slot[sa.K]] : (uint32_t)slot[sa.K] << kSlopeBits;
    return true;
  }
  return false;
}

__global__ void __launch_bounds__(kEnumThreads, 4) sweep_enum_kernel(BandFit bf, SweepArgs sa) {
  __shared__ uint32_t queue[kEnumWarps][kEnumQueue];
  __shared__ uint32_t okey[kEnumWarps][kOutBuf];
  __shared__ uint32_t oval[kEnumWarps][kOutBuf];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  uint32_t* q = queue[wib];
  uint32_t* ok = okey[wib];
  uint32_t* ov = oval[wib];
  int qn = 0, on = 0;
  // band boundaries and grouping slots in shared memory when they fit
  extern __shared__ __align__(16) unsigned char sw_dyn[];
  const float* bnd = sa.bounds;
  const int16_t* slot = sa.slot;
  if (sa.smem_tables) {
    float* sb = reinterpret_cast<float*>(sw_dyn);
    int16_t* ss = reinterpret_cast<int16_t*>(sb + sa.K);
    for (int e = threadIdx.x; e <= sa.K; e += blockDim.x) {
      if (e < sa.K - 1) sb[e] = sa.bounds[e];
      ss[e] = sa.slot[e];
    }
    __syncthreads();
    bnd = sb;
    slot = ss;
  }
  const int n = (int)bf.n;
  const int nb = (n + 31) / 32;
  const int64_t nitems = (int64_t)(sa.dnr ? *sa.dnr : sa.nruns) * n;
  const int64_t gw0 = (int64_t)blockIdx.x * kEnumWarps + wib;
  const int64_t nw = (int64_t)gridDim.x * kEnumWarps;
  int cur_run = -1, k0 = 0, k1 = 0;

  // members are buffered per warp and appended with one atomic per ~kOutFlush
  auto flush_out = [&]() {
    if (on == 0) return;
    unsigned long long b0 = 0;
    if (lane == 0) b0 = atomicAdd(sa.raw_count, (unsigned long long)on);
    b0 = __shfl_sync(0xffffffffu, b0, 0);
    for (int e = lane; e < on; e += 32) {
      const unsigned long long pos = b0 + e;
      if ((int64_t)pos < sa.raw_cap) sa.raw[pos] = ((unsigned long long)ov[e] << 32) | ok[e];
    }
    __syncwarp();
    on = 0;
  };
  // the enumerated pairs go out raw (run, pair) -- classified by
  // sweep_classify_kernel, a thread per pair with all its loads in flight
  auto drain = [&](int cnt) {
    if (lane < cnt) {
      ok[on + lane] = q[lane];
      ov[on + lane] = (uint32_t)cur_run;
    }
    on += cnt;
    __syncwarp();
    if (on >= kOutFlush) flush_out();
  };
  auto flush = [&]() {
    __syncwarp();
    while (qn >= 32) {
      drain(32);
      __syncwarp();
      if (lane < qn - 32) q[lane] = q[32 + lane];
      __syncwarp();
      qn -= 32;
    }
  };

  // items ordered run-major: a warp's consecutive items share the run
  for (int64_t it = gw0; it < nitems; it += nw) {
    const int r = (int)(it / n);
    const int t = (int)(it - (int64_t)r * n);
    if (r != cur_run) {
      if (qn > 0) {  // the queue holds pairs of the previous run
        __syncwarp();
        drain(qn);
        qn = 0;
        __syncwarp();
      }
      cur_run = r;
      k0 = sa.run_k0[r];
      k1 = sa.run_k1[r];
    }
    const int32_t* P = sa.P + (int64_t)r * n;
    const int32_t* bm = sa.bmin + (int64_t)r * nb;
    const int32_t* sf = sa.suf + (int64_t)r * nb;
    const uint32_t* line0 = sa.idx + (int64_t)(2 * r) * n;
    const int p = P[t];
    const uint32_t me = line0[t] << 16;
    int b = (t + 1) >> 5;
    while (b < nb && sf[b] < p) {
      const int bb = b + lane;
      const bool hit = bb < nb && bm[bb] < p;
      unsigned hits = __ballot_sync(0xffffffffu, hit);
      while (hits) {
        // up to kHitBatch hit blocks at a time: all their loads in flight at once
        int tp[kHitBatch];
        int32_t pv[kHitBatch];
        uint32_t lv[kHitBatch];
#pragma unroll
        for (int e = 0; e < kHitBatch; ++e) {
          tp[e] = -1;
          if (hits) {
            const int h = __ffs(hits) - 1;
            hits &= hits - 1;
            tp[e] = ((b + h) << 5) + lane;
          }
          const int tq = min(max(tp[e], 0), n - 1);
          pv[e] = P[tq];
          lv[e] = line0[tq];
        }
#pragma unroll
        for (int e = 0; e < kHitBatch; ++e) {
          if (tp[e] < 0 && e > 0) break;  // (warp-uniform: the same hits on every lane)
          const bool c = tp[e] > t && tp[e] < n && pv[e] < p;
          const unsigned m = __ballot_sync(0xffffffffu, c);
          if (sa.dbg && lane == 0) atomicAdd(sa.dbg + r, (unsigned long long)__popc(m));
          if (c) q[qn + __popc(m & ((1u << lane) - 1u))] = me | lv[e];
          qn += __popc(m);
          if (qn >= 32) flush();
        }
      }
      b += 32;
    }
  }
  __syncwarp();
  if (qn > 0) drain(qn);
  flush_out();
}

// Classification of the enumerated pairs: the reference's slope, the band,
// ownership by the pair's run (sweep_take); members appended per warp.
__global__ void __launch_bounds__(256) sweep_classify_kernel(BandFit bf, SweepArgs sa) {
  extern __shared__ __align__(16) unsigned char cl_dyn[];
  const float* bnd = sa.bounds;
  const int16_t* slot = sa.slot;
  if (sa.smem_tables) {
    float* sb = reinterpret_cast<float*>(cl_dyn);
    int16_t* ss = reinterpret_cast<int16_t*>(sb + sa.K);
    for (int e = threadIdx.x; e <= sa.K; e += blockDim.x) {
      if (e < sa.K - 1) sb[e] = sa.bounds[e];
      ss[e] = sa.slot[e];
    }
    __syncthreads();
    bnd = sb;
    slot = ss;
  }
  // members staged per CTA, appended with one global atomic per flush
  __shared__ uint32_t bkey[kClsBuf], bval[kClsBuf];
  __shared__ unsigned bn;
  __shared__ unsigned long long bbase;
  if (threadIdx.x == 0) bn = 0;
  __syncthreads();
  auto flush = [&]() {
    __syncthreads();
    const unsigned m = bn;
    if (threadIdx.x == 0 && m) bbase = atomicAdd(sa.count, (unsigned long long)m);
    __syncthreads();
    for (unsigned e = threadIdx.x; e < m; e += blockDim.x) {
      const unsigned long long pos = bbase + e;
      if ((int64_t)pos < sa.cap) {
        sa.out_keys[pos] = bkey[e];
        sa.out_vals[pos] = bval[e];
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) bn = 0;
    __syncthreads();
  };
  int64_t cnt = (int64_t)*sa.raw_count;
  if (cnt > sa.raw_cap) cnt = sa.raw_cap;
  // kClsUnroll pairs per thread per step (their loads and divisions
  // interleaved), appended to the CTA buffer with one shared atomic per warp
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t step = (int64_t)gridDim.x * blockDim.x * kClsUnroll;
  for (int64_t p0 = (int64_t)blockIdx.x * blockDim.x * kClsUnroll; p0 < cnt; p0 += step) {
    uint32_t key[kClsUnroll], val[kClsUnroll];
    bool take[kClsUnroll];
    unsigned long long e[kClsUnroll];
#pragma unroll
    for (int u = 0; u < kClsUnroll; ++u) {
      const int64_t p = p0 + (int64_t)u * blockDim.x + threadIdx.x;
      e[u] = p < cnt ? sa.raw[p] : ~0ull;
    }
#pragma unroll
    for (int u = 0; u < kClsUnroll; ++u) {
      take[u] = false;
      key[u] = val[u] = 0;
      if (e[u] != ~0ull) {
        const int r = (int)(e[u] >> 32);
        const uint32_t pr = (uint32_t)e[u];
        take[u] = sweep_take(bf, sa, bnd, slot, sa.run_k0[r], sa.run_k1[r], false, (int)(pr >> 16),
                             (int)(pr & 0xFFFF), &key[u], &val[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < kClsUnroll; ++u) {
      const unsigned m = __ballot_sync(0xffffffffu, take[u]);
      unsigned at = 0;
      if (lane == 0 && m) at = atomicAdd(&bn, (unsigned)__popc(m));
      at = __shfl_sync(0xffffffffu, at, 0) + __popc(m & lt);
      if (take[u]) {
        bkey[at] = key[u];
        bval[at] = val[u];
      }
    }
    __syncthreads();
    if (bn > kClsBuf - kClsUnroll * 256) flush();  // (uniform: bn read after the barrier)
  }
  flush();
}

// a raw-buffer overflow makes the member count exceed its capacity (the
// caller grows both and enumerates again)
__global__ void sweep_overflow_kernel(SweepArgs sa) {
  const unsigned long long raw = *sa.raw_count;
  if ((int64_t)raw <= sa.raw_cap) return;
  if (sa.raw_overflow) *sa.raw_overflow = raw;
  else if (*sa.count < raw) *sa.count = raw;
}

// Nearly parallel pairs (0 < |a_i - a_j| <= tau): lines sorted by a, each
// against the following lines with a larger slope within tau.
__global__ void sweep_parallel_kernel(BandFit bf, SweepArgs sa) {
  const double tau = sa.dtau ? *sa.dtau : sa.tau;
  if (!(tau > 0.0)) return;
  const int n = (int)bf.n;
  const uint64_t* ka = sa.k1a;
  const uint32_t* ia = sa.idxa;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int k = (int)ia[t];
    const double ak = bf.ab[k].x;
    // first position with a strictly larger slope
    int lo = t + 1, hi = n;
    const uint64_t kk = ka[t];
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (ka[mid] <= kk) lo = mid + 1;
      else hi = mid;
    }
    for (int tp = lo; tp < n; ++tp) {
      const int l = (int)ia[tp];
      if (__dsub_rn(bf.ab[l].x, ak) > tau) break;
      uint32_t key, val;
      if (sweep_take(bf, sa, sa.bounds, sa.slot, -1, -1, true, k, l, &key, &val)) {
        const unsigned long long pos = atomicAdd(sa.count, 1ull);
        if ((int64_t)pos < sa.cap) {
          sa.out_keys[pos] = key;
          sa.out_vals[pos] = val;
        }
      }
    }
  }
}

}  // namespace

size_t sweep_chunk_smem() { return 0; }  // static shared memory

int launch_sweep_sort(const double2* ab, int n, const SweepEnd* ends, int nseg, SweepSort& ss,
                      int sms, cudaStream_t st) {
  if (n <= 0 || nseg <= 0) return 0;
  sweep_keys_kernel<<<sms * 4, 256, 0, st>>>(ab, n, ends, nseg, ss.k1[0], ss.idx[0], ss.dnr,
                                             ss.nr_max);
  const int cps = (n + kChunk - 1) / kChunk;
  sweep_chunk_sort_kernel<<<nseg * cps, kChunkThreads, 0, st>>>(n, cps, ss.k1[0], ss.idx[0], ss.dnr,
                                                                ss.nr_max);
  int cur = 0, launches = 2;
  const int bps = (n + kMergeThreads * kMergeItems - 1) / (kMergeThreads * kMergeItems);
  for (int64_t w = kChunk; w < n; w *= 2) {
    sweep_merge_kernel<<<nseg * bps, kMergeThreads, 0, st>>>(n, w, bps, ss.k1[cur], ss.idx[cur],
                                                              ss.k1[cur ^ 1], ss.idx[cur ^ 1],
                                                              ss.dnr, ss.nr_max);
    cur ^= 1;
    ++launches;
  }
  ss.cur = cur;
  return launches;
}

void launch_sweep_prepare(int n, int nruns, const SweepSort& ss, int32_t* pos, int32_t* P,
                          int32_t* bmin, int32_t* suf, int sms, cudaStream_t st) {
  if (nruns <= 0) return;
  sweep_pos_kernel<<<sms * 4, 256, 0, st>>>(n, nruns, ss.idx[ss.cur], pos, ss.dnr);
  sweep_p_kernel<<<sms * 4, 256, 0, st>>>(n, nruns, ss.idx[ss.cur], pos, P, bmin, ss.dnr);
  sweep_suffix_kernel<<<nruns, 1024, 0, st>>>(n, bmin, suf, ss.dnr);
}

void launch_sweep_emit(const BandFit& bf, const SweepArgs& sa, int sms, cudaStream_t st) {
  cudaMemsetAsync(sa.count, 0, sizeof(unsigned long long), st);
  cudaMemsetAsync(sa.raw_count, 0, sizeof(unsigned long long), st);
  if (sa.nruns > 0) {
    const size_t tab = (size_t)sa.K * sizeof(float) + (size_t)(sa.K + 1) * sizeof(int16_t) + 16;
    SweepArgs a2 = sa;
    a2.smem_tables = tab <= 24 * 1024;
    SweepArgs ae = a2;
    ae.smem_tables = 0;  // the enumeration does not classify
    sweep_enum_kernel<<<sms * 8, kEnumThreads, 0, st>>>(bf, ae);
    sweep_classify_kernel<<<sms * 4, 256, a2.smem_tables ? tab : 0, st>>>(bf, a2);
    sweep_overflow_kernel<<<1, 1, 0, st>>>(a2);
  }
  if ((sa.tau > 0.0 || sa.dtau) && sa.k1a)
    sweep_parallel_kernel<<<(int)((bf.n + 255) / 256), 256, 0, st>>>(bf, sa);
}

}  // namespace lmsb
