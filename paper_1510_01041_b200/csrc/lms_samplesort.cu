// lms_samplesort.cu -- the band stage's slope-sample sort over the whole GPU
// (replaces a CUB device radix sort: six dependent launches of a decoupled
// look-back sort, ~47 us for config 2's 65,536 keys).
//
// The sorted sample gives the band boundaries (its quantiles) and the
// sub-band cuts of wide bands -- the reference has no counterpart (its scan
// visits every vertex, backend.py:190-207); only the order matters here.
//
// Bucket sort with regular-sample splitters, four short kernels:
//   split   one CTA: 512 regular samples as (ordered key, position)
//           composites, bitonic-sorted in shared memory; 255 splitters
//   count   one CTA per 1,024 keys: each key's bucket (binary search of the
//           composite among the splitters) and the tile's bucket histogram
//   scatter one CTA per tile: its write offsets from all tiles' histograms,
//           then keys to their buckets (order inside a bucket is free: the
//           bucket is sorted next)
//   bucket  one CTA per bucket: a block radix sort of <= 4,096 keys in
//           registers; a larger bucket (composites keep equal keys apart, so
//           only an input whose every 128th sample differs from the rest gets
//           one) is sorted in 4,096-key chunks and merged in global memory;
//           only the bits in which a bucket's keys differ are sorted.
// The output is the ascending order of the unsigned ordered keys -- the
// order CUB's radix sort produces (-0.0 before +0.0 aside, which no caller
// distinguishes).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include <cub/block/block_radix_sort.cuh>

#include "../../include/lms_b200.h"
#include "lms_band.cuh"

namespace lmsb {
namespace {

constexpr int kSsB = 256;      // buckets
constexpr int kSsR = 512;      // regular samples (2 per bucket)
constexpr int kSsTile = 1024;  // keys per CTA of count / scatter
constexpr int kSsT = 256;      // threads of count / scan / scatter / bucket
constexpr int kSsItems = 16;   // keys per thread of a bucket sort
constexpr int kSsCap = kSsT * kSsItems;

using BucketSort = cub::BlockRadixSort<uint32_t, kSsT, kSsItems>;
constexpr int kSsSmallItems = 2;  // buckets of <= 512 keys (most: ~256 on average)
using SmallSort = cub::BlockRadixSort<uint32_t, kSsT, kSsSmallItems>;

__device__ __forceinline__ uint32_t ss_key(float f) {
  const uint32_t u = __float_as_uint(f);
  return u ^ ((u >> 31) ? 0xFFFFFFFFu : 0x80000000u);
}
__device__ __forceinline__ float ss_float(uint32_t k) {
  return __uint_as_float(k ^ ((k >> 31) ? 0x80000000u : 0xFFFFFFFFu));
}
// segment y: keys[base, base + L) (seg_b / seg_e, or [y * stride, (y + 1) * stride))
struct SsSeg {
  const int64_t* seg_b;
  const int64_t* seg_e;
  int64_t stride;
};
__device__ __forceinline__ void ss_segment(const SsSeg& sg, int y, int64_t* base, int64_t* L) {
  if (sg.seg_b) {
    *base = sg.seg_b[y];
    *L = sg.seg_e[y] - *base;
  } else {
    *base = (int64_t)y * sg.stride;
    *L = sg.stride;
  }
}
// (ordered key, position in the segment): distinct for equal keys
__device__ __forceinline__ unsigned long long ss_comp(const float* keys, int64_t base, int64_t s) {
  return ((unsigned long long)ss_key(keys[base + s]) << 32) | (unsigned long long)(uint32_t)s;
}

__global__ void __launch_bounds__(kSsR) ss_split_kernel(const float* __restrict__ keys, SsSeg sg,
                                                        unsigned long long* __restrict__ spl) {
  __shared__ unsigned long long v[kSsR];
  int64_t base, S;
  ss_segment(sg, blockIdx.x, &base, &S);
  if (S <= 0) return;
  const int t = threadIdx.x;
  const int64_t pos = (t * S) / kSsR + (S / kSsR) / 2;
  v[t] = ss_comp(keys, base, pos < S ? pos : S - 1);
  for (int k = 2; k <= kSsR; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      __syncthreads();
      const int p = t ^ j;
      if (p > t) {
        const unsigned long long a = v[t], b = v[p];
        if ((a > b) == ((t & k) == 0)) {
          v[t] = b;
          v[p] = a;
        }
      }
    }
  }
  __syncthreads();
  if (t < kSsB - 1) spl[(int64_t)blockIdx.x * kSsB + t] = v[(t + 1) * (kSsR / kSsB) - 1];
}

// grid (tiles, segments); hist[(y * G + g) * 256 + b]
__global__ void __launch_bounds__(kSsT) ss_count_kernel(const float* __restrict__ keys, SsSeg sg,
                                                        int G,
                                                        const unsigned long long* __restrict__ spl,
                                                        uint8_t* __restrict__ bkt,
                                                        unsigned* __restrict__ hist) {
  __shared__ unsigned long long sp[kSsB];
  __shared__ unsigned h[kSsB];
  int64_t base, S;
  ss_segment(sg, blockIdx.y, &base, &S);
  const int64_t s0 = (int64_t)blockIdx.x * kSsTile;
  if (S <= 0 || s0 >= S) return;
  const int t = threadIdx.x;
  sp[t] = t < kSsB - 1 ? spl[(int64_t)blockIdx.y * kSsB + t] : ~0ull;
  h[t] = 0;
  __syncthreads();
  const int64_t s1 = s0 + kSsTile < S ? s0 + kSsTile : S;
  for (int64_t s = s0 + t; s < s1; s += kSsT) {
    const unsigned long long c = ss_comp(keys, base, s);
    int lo = 0, hi = kSsB - 1;  // first splitter >= c (sp[255] = max)
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (sp[mid] < c) lo = mid + 1;
      else hi = mid;
    }
    bkt[base + s] = (uint8_t)lo;
    atomicAdd(&h[lo], 1u);
  }
  __syncthreads();
  hist[((int64_t)blockIdx.y * G + blockIdx.x) * kSsB + t] = h[t];
}

// keys to their buckets; every CTA forms its own write offsets from the
// tiles' histograms (bucket start + the bucket's keys in earlier tiles), CTA
// 0 also publishes the bucket starts
// one CTA per segment: bucket starts and every tile's write offsets (in
// place of its histogram) -- many segments; one segment's tiles form their
// own offsets in ss_scatter_kernel (fused: one launch less)
__global__ void __launch_bounds__(kSsT) ss_scan_kernel(SsSeg sg, int G, unsigned* __restrict__ hist,
                                                       unsigned* __restrict__ bstart) {
  __shared__ unsigned wsum[kSsT / 32];
  int64_t base, S;
  ss_segment(sg, blockIdx.x, &base, &S);
  if (S <= 0) return;
  const int Gs = (int)((S + kSsTile - 1) / kSsTile);
  unsigned* hs = hist + (int64_t)blockIdx.x * G * kSsB;
  const int t = threadIdx.x;
  unsigned tot = 0;
  for (int g = 0; g < Gs; ++g) tot += hs[(int64_t)g * kSsB + t];
  unsigned incl = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned x = __shfl_up_sync(0xffffffffu, incl, o);
    if ((t & 31) >= o) incl += x;
  }
  if ((t & 31) == 31) wsum[t >> 5] = incl;
  __syncthreads();
  unsigned b = incl - tot;
  for (int w = 0; w < (t >> 5); ++w) b += wsum[w];
  bstart[(int64_t)blockIdx.x * (kSsB + 1) + t] = b;
  if (t == kSsB - 1) bstart[(int64_t)blockIdx.x * (kSsB + 1) + kSsB] = (unsigned)S;
  for (int g = 0; g < Gs; ++g) {
    const unsigned c = hs[(int64_t)g * kSsB + t];
    hs[(int64_t)g * kSsB + t] = b;
    b += c;
  }
}

__global__ void __launch_bounds__(kSsT) ss_scatter_kernel(const float* __restrict__ keys, SsSeg sg,
                                                          int G, bool fused,
                                                          const uint8_t* __restrict__ bkt,
                                                          const unsigned* __restrict__ hist,
                                                          unsigned* __restrict__ bstart,
                                                          uint32_t* __restrict__ tmp) {
  __shared__ unsigned cur[kSsB];
  __shared__ unsigned wsum[kSsT / 32];
  int64_t base, S;
  ss_segment(sg, blockIdx.y, &base, &S);
  const int g0 = blockIdx.x;
  const int64_t s0 = (int64_t)g0 * kSsTile;
  if (S <= 0 || s0 >= S) return;
  const int Gs = (int)((S + kSsTile - 1) / kSsTile);  // this segment's tiles
  const unsigned* hs = hist + (int64_t)blockIdx.y * G * kSsB;
  const int t = threadIdx.x;  // = bucket
  if (!fused) {  // offsets from ss_scan_kernel
    cur[t] = hs[(int64_t)g0 * kSsB + t];
    __syncthreads();
    const int64_t s1 = s0 + kSsTile < S ? s0 + kSsTile : S;
    for (int64_t s = s0 + t; s < s1; s += kSsT) {
      const unsigned p = atomicAdd(&cur[bkt[base + s]], 1u);
      tmp[base + p] = ss_key(keys[base + s]);
    }
    return;
  }
  unsigned tot = 0, pre = 0;
  for (int g = 0; g < Gs; ++g) {
    const unsigned c = hs[(int64_t)g * kSsB + t];
    tot += c;
    pre += g < g0 ? c : 0u;
  }
  unsigned incl = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned x = __shfl_up_sync(0xffffffffu, incl, o);
    if ((t & 31) >= o) incl += x;
  }
  if ((t & 31) == 31) wsum[t >> 5] = incl;
  __syncthreads();
  unsigned b = incl - tot;
  for (int w = 0; w < (t >> 5); ++w) b += wsum[w];
  if (g0 == 0) {
    bstart[(int64_t)blockIdx.y * (kSsB + 1) + t] = b;
    if (t == kSsB - 1) bstart[(int64_t)blockIdx.y * (kSsB + 1) + kSsB] = (unsigned)S;
  }
  cur[t] = b + pre;
  __syncthreads();
  const int64_t s1 = s0 + kSsTile < S ? s0 + kSsTile : S;
  for (int64_t s = s0 + t; s < s1; s += kSsT) {
    const unsigned p = atomicAdd(&cur[bkt[base + s]], 1u);
    tmp[base + p] = ss_key(keys[base + s]);
  }
}

// buckets of at most 512 keys (almost all): 2 keys per thread, few
// registers, so many CTAs per SM; larger buckets are left to ss_bucket_kernel
__global__ void __launch_bounds__(kSsT) ss_small_bucket_kernel(SsSeg sg,
                                                               const uint32_t* __restrict__ tmp,
                                                               const unsigned* __restrict__ bstart,
                                                               float* __restrict__ out) {
  __shared__ typename SmallSort::TempStorage sort;
  __shared__ uint32_t red[2][kSsT / 32];
  const int t = threadIdx.x;
  int64_t base, S;
  ss_segment(sg, blockIdx.y, &base, &S);
  if (S <= 0) return;
  const unsigned* bs = bstart + (int64_t)blockIdx.y * (kSsB + 1);
  const int64_t b0 = base + bs[blockIdx.x], b1 = base + bs[blockIdx.x + 1];
  const int64_t m = b1 - b0;
  if (m <= 0 || m > kSsT * kSsSmallItems) return;
  uint32_t k[kSsSmallItems];
  uint32_t lo = 0xFFFFFFFFu, hi = 0u;
#pragma unroll
  for (int i = 0; i < kSsSmallItems; ++i) {
    const int64_t e = (int64_t)i * kSsT + t;
    k[i] = e < m ? tmp[b0 + e] : 0u;
    if (e < m) {
      lo = min(lo, k[i]);
      hi = max(hi, k[i]);
    }
  }
  lo = __reduce_min_sync(0xffffffffu, lo);
  hi = __reduce_max_sync(0xffffffffu, hi);
  if ((t & 31) == 0) {
    red[0][t >> 5] = lo;
    red[1][t >> 5] = hi;
  }
  __syncthreads();
  lo = red[0][0];
  hi = red[1][0];
#pragma unroll
  for (int w = 1; w < kSsT / 32; ++w) {
    lo = min(lo, red[0][w]);
    hi = max(hi, red[1][w]);
  }
  if (lo == hi) {
    for (int64_t e = t; e < m; e += kSsT) out[b0 + e] = ss_float(lo);
    return;
  }
  const int end_bit = 32 - __clz(lo ^ hi);
#pragma unroll
  for (int i = 0; i < kSsSmallItems; ++i)
    if ((int64_t)i * kSsT + t >= m) k[i] = hi;  // padding = the largest key
  SmallSort(sort).SortBlockedToStriped(k, 0, end_bit);
#pragma unroll
  for (int i = 0; i < kSsSmallItems; ++i) {
    const int64_t e = (int64_t)i * kSsT + t;
    if (e < m) out[b0 + e] = ss_float(k[i]);
  }
}

// one merge-path round over global memory: sorted runs of w keys of src[0, m)
// merged pairwise into dst
__device__ void ss_merge_round(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst,
                               int64_t m, int64_t w) {
  const int64_t per = (m + kSsT - 1) / kSsT;
  int64_t x = (int64_t)threadIdx.x * per;
  const int64_t x1 = x + per < m ? x + per : m;
  while (x < x1) {
    const int64_t p0 = (x / (2 * w)) * (2 * w);
    const int64_t la = w < m - p0 ? w : m - p0;
    const int64_t lb = m - p0 - la < w ? (m - p0 - la > 0 ? m - p0 - la : 0) : w;
    const uint32_t* A = src + p0;
    const uint32_t* B = A + la;
    const int64_t d = x - p0;
    int64_t lo = d - lb > 0 ? d - lb : 0, hi = d < la ? d : la;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (A[mid] <= B[d - 1 - mid]) lo = mid + 1;
      else hi = mid;
    }
    int64_t i = lo, j = d - lo;
    const int64_t xe = x1 < p0 + la + lb ? x1 : p0 + la + lb;
    for (; x < xe; ++x) {
      const bool ta = j >= lb || (i < la && A[i] <= B[j]);
      dst[x] = ta ? A[i++] : B[j++];
    }
  }
}

__global__ void __launch_bounds__(kSsT) ss_bucket_kernel(SsSeg sg, int nseg, int64_t small_max,
                                                         uint32_t* __restrict__ tmp,
                                                         uint32_t* __restrict__ tmp2,
                                                         const unsigned* __restrict__ bstart,
                                                         float* __restrict__ out) {
  __shared__ union {
    typename BucketSort::TempStorage big;
    typename SmallSort::TempStorage small;
  } sort;
  __shared__ uint32_t red[2][kSsT / 32];
  const int t = threadIdx.x;
  // persistent over (segment, bucket): almost every bucket is small and
  // belongs to ss_small_bucket_kernel
  for (int64_t item = blockIdx.x; item < (int64_t)nseg * kSsB; item += gridDim.x) {
  const int y = (int)(item / kSsB), bb = (int)(item % kSsB);
  int64_t base, S;
  ss_segment(sg, y, &base, &S);
  if (S <= 0) continue;
  const unsigned* bs = bstart + (int64_t)y * (kSsB + 1);
  const int64_t b0 = base + bs[bb], b1 = base + bs[bb + 1];
  const int64_t m = b1 - b0;
  if (m <= small_max) continue;  // (ss_small_bucket_kernel's)
  if (m <= 0) continue;
  if (m <= kSsCap) {
    uint32_t k[kSsItems];
    uint32_t lo = 0xFFFFFFFFu, hi = 0u;
#pragma unroll
    for (int i = 0; i < kSsItems; ++i) {
      const int64_t e = (int64_t)i * kSsT + t;
      k[i] = e < m ? tmp[b0 + e] : 0xFFFFFFFFu;
      if (e < m) {
        lo = min(lo, k[i]);
        hi = max(hi, k[i]);
      }
    }
    // only the bits in which the bucket's keys differ are sorted (they share
    // every higher bit: a common prefix of the smallest and largest key)
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    if ((t & 31) == 0) {
      red[0][t >> 5] = lo;
      red[1][t >> 5] = hi;
    }
    __syncthreads();
    lo = red[0][0];
    hi = red[1][0];
#pragma unroll
    for (int w = 1; w < kSsT / 32; ++w) {
      lo = min(lo, red[0][w]);
      hi = max(hi, red[1][w]);
    }
    if (lo == hi) {  // one value
      for (int64_t e = t; e < m; e += kSsT) out[b0 + e] = ss_float(lo);
      __syncthreads();  // (red is reused by the next bucket)
      continue;
    }
    const int end_bit = 32 - __clz(lo ^ hi);
    // padding = the largest key: ties with it are equal values, so the first
    // m sorted keys are the bucket's whatever the tie order
#pragma unroll
    for (int i = 0; i < kSsItems; ++i)
      if ((int64_t)i * kSsT + t >= m) k[i] = hi;
    if (m <= kSsT * kSsSmallItems) {  // (a small bucket of the single-segment sort)
      uint32_t ks[kSsSmallItems];
#pragma unroll
      for (int i = 0; i < kSsSmallItems; ++i) ks[i] = k[i];
      SmallSort(sort.small).SortBlockedToStriped(ks, 0, end_bit);
#pragma unroll
      for (int i = 0; i < kSsSmallItems; ++i) {
        const int64_t e = (int64_t)i * kSsT + t;
        if (e < m) out[b0 + e] = ss_float(ks[i]);
      }
      __syncthreads();
      continue;
    }
    BucketSort(sort.big).SortBlockedToStriped(k, 0, end_bit);
#pragma unroll
    for (int i = 0; i < kSsItems; ++i) {
      const int64_t e = (int64_t)i * kSsT + t;
      if (e < m) out[b0 + e] = ss_float(k[i]);
    }
    __syncthreads();
    continue;
  }
  // oversize bucket: sorted 4,096-key chunks, then merge rounds (ping-pong)
  uint32_t* src = tmp + b0;
  uint32_t* dst = tmp2 + b0;
  for (int64_t c0 = 0; c0 < m; c0 += kSsCap) {
    uint32_t k[kSsItems];
#pragma unroll
    for (int i = 0; i < kSsItems; ++i) {
      const int64_t e = c0 + (int64_t)i * kSsT + t;
      k[i] = e < m ? src[e] : 0xFFFFFFFFu;
    }
    BucketSort(sort.big).SortBlockedToStriped(k);
#pragma unroll
    for (int i = 0; i < kSsItems; ++i) {
      const int64_t e = c0 + (int64_t)i * kSsT + t;
      if (e < m) src[e] = k[i];
    }
    __syncthreads();
  }
  for (int64_t w = kSsCap; w < m; w <<= 1) {
    ss_merge_round(src, dst, m, w);
    __syncthreads();
    uint32_t* x = src;
    src = dst;
    dst = x;
  }
  for (int64_t e = t; e < m; e += kSsT) out[b0 + e] = ss_float(src[e]);
  __syncthreads();
  }
}

}  // namespace

// scratch of a segmented sort: per segment 255 splitters, 257 bucket starts
// and max_len / 1,024 tile histograms; per key of keys[0, total) a bucket id
// and two staging words
size_t seg_bucket_sort_scratch_bytes(int64_t total, int nseg, int64_t max_len) {
  const int64_t G = (max_len + kSsTile - 1) / kSsTile;
  return (size_t)nseg * (kSsB * 8 + (kSsB + 1) * 4 + (size_t)G * kSsB * 4) + (size_t)total * 9 +
         256;
}

int launch_seg_bucket_sort(const float* keys, float* out, int64_t total, int nseg,
                           int64_t max_len, const int64_t* seg_b, const int64_t* seg_e,
                           void* scratch, size_t bytes, cudaStream_t st) {
  if (nseg <= 0 || max_len <= 0) return 0;
  if (max_len > ((int64_t)1 << 31) - 1 || nseg > 65535 ||
      bytes < seg_bucket_sort_scratch_bytes(total, nseg, max_len))
    return -1;
  const int G = (int)((max_len + kSsTile - 1) / kSsTile);
  auto align = [](uintptr_t p) { return (p + 15) & ~(uintptr_t)15; };
  uintptr_t p = align((uintptr_t)scratch);
  auto* spl = reinterpret_cast<unsigned long long*>(p);
  p = align(p + (size_t)nseg * kSsB * 8);
  auto* bstart = reinterpret_cast<unsigned*>(p);
  p = align(p + (size_t)nseg * (kSsB + 1) * 4);
  auto* hist = reinterpret_cast<unsigned*>(p);
  p = align(p + (size_t)nseg * G * kSsB * 4);
  auto* tmp = reinterpret_cast<uint32_t*>(p);
  p = align(p + (size_t)total * 4);
  auto* tmp2 = reinterpret_cast<uint32_t*>(p);
  p = align(p + (size_t)total * 4);
  auto* bkt = reinterpret_cast<uint8_t*>(p);
  SsSeg sg{seg_b, seg_e, seg_b ? 0 : max_len};
  ss_split_kernel<<<nseg, kSsR, 0, st>>>(keys, sg, spl);
  ss_count_kernel<<<dim3(G, nseg), kSsT, 0, st>>>(keys, sg, G, spl, bkt, hist);
  const bool fused = nseg == 1;
  if (!fused) ss_scan_kernel<<<nseg, kSsT, 0, st>>>(sg, G, hist, bstart);
  ss_scatter_kernel<<<dim3(G, nseg), kSsT, 0, st>>>(keys, sg, G, fused, bkt, hist, bstart, tmp);
  if (nseg == 1) {  // one CTA per bucket, every size (the sample sort)
    ss_bucket_kernel<<<kSsB, kSsT, 0, st>>>(sg, 1, 0, tmp, tmp2, bstart, out);
  } else {  // small buckets by the light kernel, the rest by persistent CTAs
    ss_small_bucket_kernel<<<dim3(kSsB, nseg), kSsT, 0, st>>>(sg, tmp, bstart, out);
    ss_bucket_kernel<<<(unsigned)std::min<int64_t>((int64_t)nseg * kSsB, 296), kSsT, 0, st>>>(
        sg, nseg, kSsT * kSsSmallItems, tmp, tmp2, bstart, out);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

size_t sample_sort_scratch_bytes(int64_t S) { return seg_bucket_sort_scratch_bytes(S, 1, S); }

int launch_sample_sort(const float* keys, float* out, int64_t S, void* scratch, size_t bytes,
                       cudaStream_t st) {
  if (S <= 0) return 0;
  return launch_seg_bucket_sort(keys, out, S, 1, S, nullptr, nullptr, scratch, bytes, st);
}

}  // namespace lmsb

extern "C" int lms_debug_sample_sort(int device, const float* keys, float* out, int64_t n) {
  if (!keys || !out || n < 0) return LMS_ERR_INVALID;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
    return LMS_ERR_NODEVICE;
  if (cudaSetDevice(device) != cudaSuccess) return LMS_ERR_CUDA;
  if (n == 0) return LMS_OK;
  float *d_in = nullptr, *d_out = nullptr;
  void* scratch = nullptr;
  const size_t sb = lmsb::sample_sort_scratch_bytes(n);
  int rc = LMS_OK;
  if (cudaMalloc(&d_in, n * sizeof(float)) != cudaSuccess ||
      cudaMalloc(&d_out, n * sizeof(float)) != cudaSuccess ||
      cudaMalloc(&scratch, sb) != cudaSuccess) {
    rc = LMS_ERR_NOMEM;
  } else if (cudaMemcpy(d_in, keys, n * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess ||
             lmsb::launch_sample_sort(d_in, d_out, n, scratch, sb, 0) != 0 ||
             cudaDeviceSynchronize() != cudaSuccess ||
             cudaMemcpy(out, d_out, n * sizeof(float), cudaMemcpyDeviceToHost) != cudaSuccess) {
    rc = LMS_ERR_CUDA;
  }
  cudaFree(d_in);
  cudaFree(d_out);
  cudaFree(scratch);
  return rc;
}
