// lms_band.cu -- slope-band pruning of the exact LMS search.
//
// The reference evaluates every arrangement vertex against every line
// (backend.py:125-179, O(n) per vertex after an O(n log n) sort).  The count
// filter (lms_filter32m.cu) needs > n - q line tests before it can reject a
// vertex.  This stage rejects almost every vertex in O(log n) instead, by
// grouping vertices of similar slope into bands that share one sorted view
// of the lines.
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
// [z - D_v - E_v, z + H + D_v + E_v] (and symmetrically for h_down).  Two
// binary searches in the band's sorted keys (shared memory) count that.
//
// Band lower bound.  If v has height h, q keys lie in an interval of width
// h + 2 D_v + 2 E_v, so h >= W_q - 2 D_max - 2 E_max with W_q the narrowest
// q-window of the sorted keys.  Bands whose bound exceeds the current H are
// skipped without touching their vertices; the lowest bounds also point at
// the bands where the optimum lives (their vertices seed H).
//
// Error budget (eps = 2^-53, amax = max|a|, bmax = max|b|): the reference's
// roundings of u a_k - b_k, v0 and fl(x - v0) <= H move membership by at
// most 2^-49 (|u| amax + bmax + H); the fp64 z = fl(v0 - fl(c u)) adds
// 2^-50 (2 |u| amax + bmax); keys are fp64-formed and rounded to fp32 once:
// <= 2^-23 (|uM| dev + bmax).  E_v = 2^-20 (|u| amax + bmax + H + |uM| dev)
// + 1e-300 covers the sum with a wide margin; D is computed from an
// upward-padded dev, window ends are rounded outward to fp32.  Survivors are
// re-evaluated bit-exactly (lms_exact.cu), so the band stage only has to
// return a superset.
//
// Pipeline per fit (rank range [R0, R0 + span)):
//   sample   stratified vertex slopes -> CUB sort -> K-1 quantile boundaries
//   hist     every vertex: u, band id (binary search of the boundaries)
//   scatter  vertices (packed i << 16 | j) grouped by band
//   bound    per band: sort the n keys, W_q, lower bound, slope extent
//   filter   per band in bound order (skip if bound > H): count windows of
//            every vertex, emit survivors for the exact stage

#include <cub/block/block_radix_sort.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include <cfloat>
#include <cmath>
#include <cstdint>

#include "lms_band.cuh"
#include "lms_common.cuh"

namespace lmsb {

namespace {

constexpr uint16_t kBidDrop = 0xFFFF;   // a_i == a_j or non-finite slope (never a window)
constexpr uint16_t kBidForce = 0xFFFE;  // magnitudes beyond the fp32 key range
constexpr int kRun = 16;                // consecutive ranks per thread in hist / scatter

__device__ __forceinline__ float band_key(double u) {
  // monotone non-decreasing map of the slope to fp32 (clamped, so ordered)
  const float f = (float)u;
  return fminf(fmaxf(f, -FLT_MAX), FLT_MAX);
}

// slope and class of vertex (i, j), exactly as _scan_rank_range (backend.py:203-205)
__device__ __forceinline__ int classify(const BandFit& bf, int64_t i, int64_t j, double* pu) {
  const double da = __dsub_rn(bf.a[i], bf.a[j]);
  if (da == 0.0) return 0;
  const double u = __ddiv_rn(__dsub_rn(bf.b[i], bf.b[j]), da);
  if (!isfinite(u)) return 0;
  *pu = u;
  if (!(fabs(u) * bf.amax < 1e30) || !(bf.bmax < 1e30) || !(bf.amax < 1e30)) return 2;
  return 1;
}

// first rank of a thread's run and its (i, j)
__device__ __forceinline__ void run_start(const BandFit& bf, int64_t r, int64_t* i, int64_t* j) {
  decode_rank(bf.n, r, i, j);
}

__device__ __forceinline__ void step_pair(int64_t n, int64_t* i, int64_t* j) {
  if (++*j >= n) {
    ++*i;
    *j = *i + 1;
  }
}

__global__ void band_sample_kernel(BandFit bf, int64_t S, float* __restrict__ keys,
                                   unsigned long long* __restrict__ nvalid) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < S;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = bf.R0 + ((2 * s + 1) * bf.span) / (2 * S);
    int64_t i, j;
    decode_rank(bf.n, r, &i, &j);
    double u = 0.0;
    const int cls = classify(bf, i, j, &u);
    const bool ok = cls == 1;
    keys[s] = ok ? band_key(u) : INFINITY;
    const unsigned m = __ballot_sync(__activemask(), ok);
    if ((threadIdx.x & 31) == __ffs(__activemask()) - 1 && m)
      atomicAdd(nvalid, (unsigned long long)__popc(m));
  }
}

__global__ void band_bounds_kernel(const float* __restrict__ sorted,
                                   const unsigned long long* __restrict__ nvalid, int K,
                                   float* __restrict__ bounds) {
  const int64_t sv = (int64_t)*nvalid;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x + 1; k < K; k += gridDim.x * blockDim.x)
    bounds[k - 1] = sv > 0 ? sorted[(k * sv) / K] : INFINITY;
}

// number of boundaries <= key (upper bound), i.e. the band index
__device__ __forceinline__ int band_of(const float* __restrict__ bnd, int nb, float key) {
  int lo = 0, hi = nb;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (bnd[mid] <= key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(512) band_hist_kernel(BandFit bf, int K,
                                                        const float* __restrict__ bounds,
                                                        uint16_t* __restrict__ bid,
                                                        unsigned long long* __restrict__ counts,
                                                        unsigned long long* __restrict__ nforce) {
  extern __shared__ unsigned char smem_raw[];
  float* bnd = reinterpret_cast<float*>(smem_raw);
  unsigned* hist = reinterpret_cast<unsigned*>(bnd + K);
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    if (k < K - 1) bnd[k] = bounds[k];
    hist[k] = 0;
  }
  __syncthreads();
  const int64_t runs = (bf.span + kRun - 1) / kRun;
  unsigned forced = 0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < runs;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r0 = t * kRun;
    const int64_t cnt = bf.span - r0 < kRun ? bf.span - r0 : kRun;
    int64_t i, j;
    run_start(bf, bf.R0 + r0, &i, &j);
    uint32_t w[kRun / 2];
#pragma unroll
    for (int e = 0; e < kRun; ++e) {
      uint16_t id = kBidDrop;
      if (e < cnt) {
        double u = 0.0;
        const int cls = classify(bf, i, j, &u);
        if (cls == 1) {
          const int k = band_of(bnd, K - 1, band_key(u));
          id = (uint16_t)k;
          atomicAdd(hist + k, 1u);
        } else if (cls == 2) {
          id = kBidForce;
          ++forced;
        }
        step_pair(bf.n, &i, &j);
      }
      if (e & 1) w[e >> 1] |= (uint32_t)id << 16;
      else w[e >> 1] = id;
    }
    if (cnt == kRun) {
      uint4* dst = reinterpret_cast<uint4*>(bid + r0);
      dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
      dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
    } else {
      for (int e = 0; e < cnt; ++e) bid[r0 + e] = (uint16_t)(w[e >> 1] >> (16 * (e & 1)));
    }
  }
  if (forced) atomicAdd(nforce, (unsigned long long)forced);
  __syncthreads();
  for (int k = threadIdx.x; k < K; k += blockDim.x)
    if (hist[k]) atomicAdd(counts + k, (unsigned long long)hist[k]);
}

__global__ void __launch_bounds__(512) band_scatter_kernel(BandFit bf,
                                                           const uint16_t* __restrict__ bid,
                                                           unsigned long long* __restrict__ cursor,
                                                           uint32_t* __restrict__ members) {
  const int64_t runs = (bf.span + kRun - 1) / kRun;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < runs;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r0 = t * kRun;
    const int64_t cnt = bf.span - r0 < kRun ? bf.span - r0 : kRun;
    int64_t i, j;
    run_start(bf, bf.R0 + r0, &i, &j);
    for (int e = 0; e < cnt; ++e) {
      const uint16_t id = bid[r0 + e];
      if (id < kBidForce) {
        const unsigned long long pos = atomicAdd(cursor + id, 1ull);
        members[pos] = ((uint32_t)i << 16) | (uint32_t)j;
      }
      step_pair(bf.n, &i, &j);
    }
  }
}

// ------------------------------------------------------------------ per band
template <int kThreads, int kItems>
struct BandShared {
  using Sort = cub::BlockRadixSort<float, kThreads, kItems>;
  union {
    typename Sort::TempStorage sort;
    float keys[kThreads * kItems];
  };
  double red[2][kThreads / 32];
  unsigned long long base;
};

__device__ __forceinline__ int lower_idx(const float* __restrict__ k, int n, float x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (k[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ int upper_idx(const float* __restrict__ k, int n, float x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (k[mid] <= x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

template <int kThreads>
__device__ __forceinline__ double block_min(double v, double* red) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, off));
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  double r = red[0];
#pragma unroll 1
  for (int k = 1; k < kThreads / 32; ++k) r = fmin(r, red[k]);
  return r;
}

__device__ __forceinline__ double slack_base(const BandFit& bf, double umag, double uM) {
  return 0x1p-20 * (umag * bf.amax + bf.bmax + fabs(uM) * bf.dev);
}

// mode 0: slope extent + lower bound of every band; mode 1: count windows
template <int kThreads, int kItems, int kMode>
__global__ void __launch_bounds__(kThreads, 1) band_kernel(BandFit bf, BandArgs ba) {
  using SH = BandShared<kThreads, kItems>;
  extern __shared__ __align__(16) unsigned char band_smem[];
  SH& sh = *reinterpret_cast<SH*>(band_smem);
  const int band = kMode == 0 ? (int)blockIdx.x : ba.list[blockIdx.x];
  const int64_t m0 = (int64_t)ba.offsets[band];
  const int64_t m1 = (int64_t)ba.offsets[band + 1];
  const int n = (int)bf.n;
  const int tid = threadIdx.x;
  if (m1 <= m0) {
    if (kMode == 0 && tid == 0) {
      ba.lb[band] = INFINITY;
      ba.ulo[band] = 0.0;
      ba.uhi[band] = 0.0;
    }
    return;
  }
  double uL, uR, H = INFINITY;
  if (kMode == 0) {
    double lo = INFINITY, hi = -INFINITY;
    for (int64_t s = m0 + tid; s < m1; s += kThreads) {
      const uint32_t p = ba.members[s];
      const int64_t i = p >> 16, j = p & 0xFFFF;
      const double u = __ddiv_rn(__dsub_rn(bf.b[i], bf.b[j]), __dsub_rn(bf.a[i], bf.a[j]));
      lo = fmin(lo, u);
      hi = fmax(hi, u);
    }
    uL = block_min<kThreads>(lo, sh.red[0]);
    uR = -block_min<kThreads>(-hi, sh.red[1]);
  } else {
    uL = ba.ulo[band];
    uR = ba.uhi[band];
    const lms_candidate best = *ba.best;
    if (best.found) H = best.height;
    if (ba.lb[band] > H * (1.0 + 0x1p-19)) return;  // no vertex of the band can reach H
  }
  const double uM = 0.5 * uL + 0.5 * uR;
  const double half_w = fmax(uR - uM, uM - uL) * (1.0 + 0x1p-40);
  const double dmax = bf.dev * half_w;

  // the band's keys m_k = (a_k - c) uM - b_k, sorted
  float keys[kItems];
#pragma unroll
  for (int e = 0; e < kItems; ++e) {
    const int k = tid * kItems + e;
    keys[e] = k < n ? (float)__dsub_rn(__dmul_rn(__dsub_rn(bf.a[k], bf.c), uM), bf.b[k]) : INFINITY;
  }
  typename SH::Sort(sh.sort).Sort(keys);
  __syncthreads();
#pragma unroll
  for (int e = 0; e < kItems; ++e) sh.keys[tid * kItems + e] = keys[e];
  __syncthreads();
  const float* K = sh.keys;
  const int q = (int)bf.q;

  if constexpr (kMode == 0) {
    double w = INFINITY;
    for (int k = tid; k + q - 1 < n; k += kThreads)
      w = fmin(w, (double)K[k + q - 1] - (double)K[k]);
    w = block_min<kThreads>(w, sh.red[0]);
    if (tid == 0) {
      const double umag = fmax(fabs(uL), fabs(uR));
      const double e = slack_base(bf, umag, uM) + 1e-300;
      ba.lb[band] = (w - 2.0 * dmax - 2.0 * e) * (1.0 - 0x1p-40);
      ba.ulo[band] = uL;
      ba.uhi[band] = uR;
    }
  } else {
  // mode 1: every vertex of the band
  for (int64_t s0 = m0; s0 < m1; s0 += kThreads) {
    const int64_t s = s0 + tid;
    bool keep = false;
    int64_t rank = 0;
    if (s < m1) {
      const uint32_t p = ba.members[s];
      const int64_t i = p >> 16, j = p & 0xFFFF;
      const double ai = bf.a[i], bi = bf.b[i];
      const double u = __ddiv_rn(__dsub_rn(bi, bf.b[j]), __dsub_rn(ai, bf.a[j]));
      const double v0 = cut_value(u, ai, bi);
      const double z = __dsub_rn(v0, __dmul_rn(bf.c, u));
      const double D = bf.dev * fabs(u - uM) * (1.0 + 0x1p-40);
      const double E = slack_base(bf, fabs(u), uM) + 0x1p-20 * H + 1e-300;
      const double pad = D + E;
      const int top = upper_idx(K, n, __double2float_ru(z + H + pad));
      const int bot = lower_idx(K, n, __double2float_rd(z - H - pad));
      if (top - bot >= q) {
        const int up_lo = lower_idx(K, n, __double2float_rd(z - pad));
        const int dn_hi = upper_idx(K, n, __double2float_ru(z + pad));
        keep = (top - up_lo >= q) || (dn_hi - bot >= q);
      }
      rank = row_offset(bf.n, i) + (j - i - 1);
    }
    const unsigned mask = __ballot_sync(0xffffffffu, keep);
    if (mask) {
      unsigned long long base = 0;
      const int lane = tid & 31;
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
}

template <int kThreads, int kItems, int kMode>
void launch_band_m(const BandFit& bf, const BandArgs& ba, int grid, cudaStream_t st) {
  constexpr size_t smem = sizeof(BandShared<kThreads, kItems>);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(band_kernel<kThreads, kItems, kMode>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = true;
  }
  band_kernel<kThreads, kItems, kMode><<<grid, kThreads, smem, st>>>(bf, ba);
}

template <int kThreads, int kItems>
void launch_band_t(const BandFit& bf, const BandArgs& ba, int mode, int grid, cudaStream_t st) {
  if (mode == 0) launch_band_m<kThreads, kItems, 0>(bf, ba, grid, st);
  else launch_band_m<kThreads, kItems, 1>(bf, ba, grid, st);
}

__global__ void band_seed_kernel(BandFit bf, const unsigned long long* __restrict__ offsets,
                                 const uint32_t* __restrict__ members,
                                 const int32_t* __restrict__ list, int nb, int per_band,
                                 int64_t* __restrict__ ranks, int32_t* __restrict__ fits,
                                 int32_t fit, unsigned long long* __restrict__ count) {
  const int e = blockIdx.x;
  if (e >= nb) return;
  const int band = list[e];
  const int64_t m0 = (int64_t)offsets[band], cnt = (int64_t)offsets[band + 1] - m0;
  const int64_t take = cnt < per_band ? cnt : per_band;
  for (int64_t t = threadIdx.x; t < take; t += blockDim.x) {
    const uint32_t p = members[m0 + (t * cnt) / take];
    const int64_t i = p >> 16, j = p & 0xFFFF;
    const unsigned long long pos = atomicAdd(count, 1ull);
    ranks[pos] = row_offset(bf.n, i) + (j - i - 1);
    fits[pos] = fit;
  }
}

}  // namespace

int band_max_n() { return kBandMaxN; }

size_t band_hist_smem(int K) { return (size_t)K * (sizeof(float) + sizeof(unsigned)); }

size_t band_sample_temp_bytes(int64_t S) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, bytes, (const float*)nullptr, (float*)nullptr, (int)S);
  return bytes;
}

size_t band_scan_temp_bytes(int K) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const unsigned long long*)nullptr,
                                (unsigned long long*)nullptr, K + 1);
  return bytes;
}

int launch_band_partition(const BandFit& bf, const BandPartition& bp, int sms, cudaStream_t st) {
  // 1. quantile boundaries from a stratified sample of slopes
  cudaMemsetAsync(bp.nvalid, 0, sizeof(unsigned long long), st);
  band_sample_kernel<<<sms * 4, 256, 0, st>>>(bf, bp.S, bp.sample, bp.nvalid);
  size_t bytes = bp.temp_bytes;
  if (cub::DeviceRadixSort::SortKeys(bp.temp, bytes, bp.sample, bp.sample_sorted, (int)bp.S, 0,
                                     32, st) != cudaSuccess)
    return -1;
  if (bp.K > 1) band_bounds_kernel<<<(bp.K + 255) / 256, 256, 0, st>>>(bp.sample_sorted, bp.nvalid,
                                                                        bp.K, bp.bounds);
  // 2. band of every vertex + histogram
  cudaMemsetAsync(bp.counts, 0, sizeof(unsigned long long) * (bp.K + 1), st);
  cudaMemsetAsync(bp.nforce, 0, sizeof(unsigned long long), st);
  const size_t smem = band_hist_smem(bp.K);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(band_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)band_hist_smem(kBandMaxK));
    configured = true;
  }
  band_hist_kernel<<<sms * 2, 512, smem, st>>>(bf, bp.K, bp.bounds, bp.bid, bp.counts, bp.nforce);
  // 3. offsets, then group the vertices by band
  bytes = bp.temp_bytes;
  if (cub::DeviceScan::ExclusiveSum(bp.temp, bytes, bp.counts, bp.offsets, bp.K + 1, st) !=
      cudaSuccess)
    return -1;
  cudaMemcpyAsync(bp.cursor, bp.offsets, sizeof(unsigned long long) * bp.K,
                  cudaMemcpyDeviceToDevice, st);
  band_scatter_kernel<<<sms * 4, 512, 0, st>>>(bf, bp.bid, bp.cursor, bp.members);
  return 0;
}

void launch_band(const BandFit& bf, const BandArgs& ba, int mode, int grid, cudaStream_t st) {
  if (grid <= 0) return;
  if (bf.n <= 1024) launch_band_t<256, 4>(bf, ba, mode, grid, st);
  else if (bf.n <= 4096) launch_band_t<512, 8>(bf, ba, mode, grid, st);
  else launch_band_t<1024, 16>(bf, ba, mode, grid, st);
}

void launch_band_seeds(const BandFit& bf, const unsigned long long* offsets,
                       const uint32_t* members, const int32_t* list, int nb, int per_band,
                       int64_t* ranks, int32_t* fits, int32_t fit, unsigned long long* count,
                       cudaStream_t st) {
  if (nb <= 0) return;
  band_seed_kernel<<<nb, 256, 0, st>>>(bf, offsets, members, list, nb, per_band, ranks, fits, fit,
                                       count);
}

}  // namespace lmsb
