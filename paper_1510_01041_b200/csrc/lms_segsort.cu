// lms_segsort.cu -- segmented ascending sort of fp32 keys, one thread-block
// cluster per segment (segments of at most 65,536 keys).
//
// Replaces the CUB device sorts of the band stage: the slope-sample sort
// behind the band boundaries (band_sample_kernel's keys, 65,536 at config 2)
// and, for n > 16,384, the per-band and per-slice key sorts of n keys each
// (launch_band_bound_big, launch_band_slices).  The reference sorts the same
// quantities row by row with numpy (backend.py:190-207: np.sort of the cut
// values of every vertex); here a segment is one band's or slice's keys.
//
// Parallel sorting by regular sampling inside a cluster of 8 CTAs:
//   1. each CTA sorts its eighth of the segment (8 keys per thread by a
//      sorting network in registers, then ten merge-path rounds in shared
//      memory) and keeps the sorted run in shared memory;
//   2. 8 regular samples per run (64 in all) are read over distributed shared
//      memory, ranked by one warp, and 7 pivots picked at ranks 8k + 3;
//   3. keys are totally ordered by (value, run, position), so every run
//      splits at each pivot by one binary search and bucket k of the
//      segment gathers 8 sorted sub-runs; regular sampling bounds a bucket by
//      twice a run (16,384 keys), the capacity of the merge buffers;
//   4. CTA k copies its bucket's 8 sub-runs out of the cluster's shared
//      memory, merges them in three merge-path rounds and writes the bucket
//      at its offset (the keys of all lower buckets).
// A bucket above capacity (not reachable under the bound; kept so the sort
// is correct for any input) places each key by its rank over the 8 sub-runs.
// The output is bit-identical to a radix sort of the same keys (same order of
// the unsigned ordered keys).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "../../include/lms_b200.h"
#include "lms_band.cuh"

namespace cg = cooperative_groups;

namespace lmsb {
namespace {

constexpr int kP = 8;                    // CTAs per cluster = runs per segment
constexpr int kT = 1024;                 // threads per CTA
constexpr int kRunItems = 8;             // keys per thread of the run sort
constexpr int kRun = kT * kRunItems;     // keys per run
constexpr int kCap = 2 * kRun;           // bucket capacity of the merge buffers
constexpr int kMaxLen = kP * kRun;       // longest segment

struct __align__(16) SegSortShared {
  uint32_t run[kRun];  // this CTA's sorted run (read by the whole cluster)
  uint32_t buf[2][kCap];  // merge ping-pong (the run sort uses buf[0] with run)
  uint32_t piv_v[kP - 1];
  int piv_r[kP - 1], piv_p[kP - 1];
  int bnd[kP + 1];     // this run's bucket boundaries
  int lo[kP], off[kP + 1];  // this CTA's bucket: sub-run starts, offsets in the bucket
  int loff[kP + 1];    // merge-round list offsets
  long long base_off;  // keys of all lower buckets
  int count;           // keys in this run
};

__device__ __forceinline__ uint32_t ord_key(float f) {
  const uint32_t u = __float_as_uint(f);
  return u ^ ((u >> 31) ? 0xFFFFFFFFu : 0x80000000u);
}
__device__ __forceinline__ float key_float(uint32_t k) {
  return __uint_as_float(k ^ ((k >> 31) ? 0x80000000u : 0xFFFFFFFFu));
}

// first index of run[0 .. c) with run[i] > v (upper) or >= v (lower)
__device__ __forceinline__ int bound_in(const uint32_t* run, int c, uint32_t v, bool upper) {
  int lo = 0, hi = c;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const uint32_t x = run[mid];
    if (upper ? x <= v : x < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// one merge-path round: lists [loff[e], loff[e+1]) of src, merged in pairs into
// dst at the same offsets; returns the new list count (in shared loff)
__device__ void merge_round(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst,
                            const int* loff, int nl, int tot) {
  const int per = (tot + kT - 1) / kT;
  int x = threadIdx.x * per;
  const int x1 = min(tot, x + per);
  if (x >= x1) return;
  int p = 0;  // pair holding x
  while (2 * p + 2 < nl && loff[2 * p + 2] <= x) ++p;
  while (x < x1) {
    const int a0 = loff[2 * p];
    const int a1 = loff[2 * p + 1];  // (= loff[nl] for an unpaired last list)
    const int b1 = 2 * p + 1 < nl ? loff[2 * p + 2] : a1;
    const uint32_t* A = src + a0;
    const uint32_t* B = src + a1;
    const int la = a1 - a0, lb = b1 - a1;
    const int d = x - a0;
    int lo = max(0, d - lb), hi = min(d, la);
    while (lo < hi) {  // co-rank: A elements among the first d outputs (A first on ties)
      const int mid = (lo + hi) >> 1;
      if (A[mid] <= B[d - 1 - mid]) lo = mid + 1;
      else hi = mid;
    }
    int i = lo, j = d - lo;
    const int xe = min(x1, b1);
    for (; x < xe; ++x) {
      const bool take_a = j >= lb || (i < la && A[i] <= B[j]);
      dst[x] = take_a ? A[i++] : B[j++];
    }
    ++p;
  }
}

__device__ __forceinline__ void cas(uint32_t& x, uint32_t& y) {
  const uint32_t lo = min(x, y), hi = max(x, y);
  x = lo;
  y = hi;
}

// 8 keys in registers: Batcher's odd-even merge network (19 compare-exchanges)
__device__ __forceinline__ void sort8(uint32_t (&k)[8]) {
  cas(k[0], k[1]); cas(k[2], k[3]); cas(k[4], k[5]); cas(k[6], k[7]);
  cas(k[0], k[2]); cas(k[1], k[3]); cas(k[4], k[6]); cas(k[5], k[7]);
  cas(k[1], k[2]); cas(k[5], k[6]);
  cas(k[0], k[4]); cas(k[1], k[5]); cas(k[2], k[6]); cas(k[3], k[7]);
  cas(k[2], k[4]); cas(k[3], k[5]);
  cas(k[1], k[2]); cas(k[3], k[4]); cas(k[5], k[6]);
}

// the run sort: sorted runs of w keys merged pairwise (w = 8 .. kRun / 2); a
// thread's 8 outputs never cross a pair.  Ten rounds: the result ends in src.
__device__ void run_sort(uint32_t* __restrict__ src, uint32_t* __restrict__ tmp) {
  const int x0 = threadIdx.x * kRunItems;
  uint32_t* s = src;
  uint32_t* d = tmp;
  for (int w = kRunItems; w < kRun; w <<= 1) {
    const int pb = x0 & ~(2 * w - 1);
    const uint32_t* A = s + pb;
    const uint32_t* B = A + w;
    const int dd = x0 - pb;
    int lo = dd > w ? dd - w : 0, hi = dd < w ? dd : w;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (A[mid] <= B[dd - 1 - mid]) lo = mid + 1;
      else hi = mid;
    }
    int i = lo, j = dd - lo;
    uint32_t av = i < w ? A[i] : 0xFFFFFFFFu, bv = j < w ? B[j] : 0xFFFFFFFFu;
#pragma unroll
    for (int e = 0; e < kRunItems; ++e) {
      const bool ta = j >= w || (i < w && av <= bv);
      if (ta) {
        d[x0 + e] = av;
        ++i;
        av = i < w ? A[i] : 0xFFFFFFFFu;
      } else {
        d[x0 + e] = bv;
        ++j;
        bv = j < w ? B[j] : 0xFFFFFFFFu;
      }
    }
    __syncthreads();
    uint32_t* t = s;
    s = d;
    d = t;
  }
}

__global__ void __cluster_dims__(kP, 1, 1) __launch_bounds__(kT, 1)
    seg_sort_kernel(const float* __restrict__ in, float* __restrict__ out, int64_t stride,
                    int nseg, const int64_t* __restrict__ seg_b, const int64_t* __restrict__ seg_e) {
  extern __shared__ __align__(16) unsigned char seg_smem[];
  SegSortShared& sh = *reinterpret_cast<SegSortShared*>(seg_smem);
  cg::cluster_group cl = cg::this_cluster();
  const int r = (int)cl.block_rank();
  const int tid = threadIdx.x;
  const int clusters = gridDim.x / kP;
  for (int s = blockIdx.x / kP; s < nseg; s += clusters) {
    int64_t base = (int64_t)s * stride, L = stride;
    if (seg_b) {
      base = seg_b[s];
      L = seg_e[s] - base;
    }
    if (L <= 0) continue;  // same decision in every CTA of the cluster
    const int m = (int)((L + kP - 1) / kP);
    const int64_t e0 = (int64_t)r * m, e1 = (int64_t)(r + 1) * m;
    const int r0 = (int)(e0 < L ? e0 : L);
    const int c = (int)(e1 < L ? e1 : L) - r0;

    // 1. the run: this CTA's keys, sorted
    {
      uint32_t k[kRunItems];
#pragma unroll
      for (int i = 0; i < kRunItems; ++i) {  // coalesced loads, staged in buf[0]
        const int idx = i * kT + tid;
        sh.buf[0][idx] = idx < c ? ord_key(__ldg(in + base + r0 + idx)) : 0xFFFFFFFFu;
      }
      __syncthreads();
      const uint4* kv = reinterpret_cast<const uint4*>(sh.buf[0] + tid * kRunItems);
      const uint4 k0 = kv[0], k1 = kv[1];
      k[0] = k0.x; k[1] = k0.y; k[2] = k0.z; k[3] = k0.w;
      k[4] = k1.x; k[5] = k1.y; k[6] = k1.z; k[7] = k1.w;
      sort8(k);
      uint4* rv = reinterpret_cast<uint4*>(sh.run + tid * kRunItems);
      rv[0] = make_uint4(k[0], k[1], k[2], k[3]);
      rv[1] = make_uint4(k[4], k[5], k[6], k[7]);
      if (tid == 0) sh.count = c;
      __syncthreads();
      run_sort(sh.run, sh.buf[0]);
    }
    cl.sync();

    // 2. pivots from 8 regular samples of every run, ranked by one warp
    if (tid < 32) {
      uint32_t v[2];
      int rr[2], pp[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int smp = tid + 32 * h;
        rr[h] = smp / kP;
        const int kk = smp % kP;
        const SegSortShared* rs = cl.map_shared_rank(&sh, rr[h]);
        const int cq = rs->count;
        pp[h] = cq > 0 ? (kk * cq) / kP : kk;
        v[h] = cq > 0 ? rs->run[pp[h]] : 0xFFFFFFFFu;
      }
      int rank[2] = {0, 0};
      for (int o = 0; o < 32; ++o) {
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          const uint32_t ov = __shfl_sync(0xffffffffu, v[g], o);
          const int orr = __shfl_sync(0xffffffffu, rr[g], o);
          const int op = __shfl_sync(0xffffffffu, pp[g], o);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            // (value, run, position), then the sample index: ranks are 0..63
            const bool less =
                ov < v[h] ||
                (ov == v[h] && (orr < rr[h] || (orr == rr[h] && (op < pp[h] || (op == pp[h] &&
                                                                            o + 32 * g < tid + 32 * h)))));
            rank[h] += less;
          }
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int k = rank[h] - (kP / 2 - 1);
        if (k > 0 && k % kP == 0 && k / kP <= kP - 1) {
          sh.piv_v[k / kP - 1] = v[h];
          sh.piv_r[k / kP - 1] = rr[h];
          sh.piv_p[k / kP - 1] = pp[h];
        }
      }
    }
    __syncthreads();
    // 3. this run's split at every pivot
    if (tid < kP + 1) {
      int b;
      if (tid == 0) b = 0;
      else if (tid == kP) b = c;
      else {
        const uint32_t v = sh.piv_v[tid - 1];
        const int rs = sh.piv_r[tid - 1];
        b = r < rs ? bound_in(sh.run, c, v, true)
                   : r > rs ? bound_in(sh.run, c, v, false) : min(sh.piv_p[tid - 1], c);
      }
      sh.bnd[tid] = b;
    }
    cl.sync();

    // 4. bucket r: sub-run j is [bnd_j[r], bnd_j[r + 1]) of run j
    if (tid < 32) {
      int lo = 0, len = 0, below = 0;
      if (tid < kP) {
        const SegSortShared* rs = cl.map_shared_rank(&sh, tid);
        lo = rs->bnd[r];
        len = rs->bnd[r + 1] - lo;
        below = lo;
      }
      int incl = len;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (tid >= o) incl += t;
      }
      int bsum = below;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) bsum += __shfl_xor_sync(0xffffffffu, bsum, o);
      if (tid < kP) {
        sh.lo[tid] = lo;
        sh.off[tid] = incl - len;
      }
      if (tid == kP - 1) sh.off[kP] = incl;
      if (tid == 0) sh.base_off = bsum;
    }
    __syncthreads();
    const int tot = sh.off[kP];
    float* dst_g = out + base + sh.base_off;
    if (tot <= kCap) {
      uint32_t* a = sh.buf[0];
      for (int x = tid; x < tot; x += kT) {
        int j = 0;
        while (j + 1 < kP && sh.off[j + 1] <= x) ++j;
        const SegSortShared* rs = cl.map_shared_rank(&sh, j);
        a[x] = rs->run[sh.lo[j] + x - sh.off[j]];
      }
    } else {
      // rank of every key over the 8 sub-runs (ties by run, then position)
      for (int x = tid; x < tot; x += kT) {
        int j = 0;
        while (j + 1 < kP && sh.off[j + 1] <= x) ++j;
        const uint32_t v = cl.map_shared_rank(&sh, j)->run[sh.lo[j] + x - sh.off[j]];
        int64_t pos = x - sh.off[j];
        for (int jj = 0; jj < kP; ++jj) {
          if (jj == j) continue;
          const uint32_t* rj = cl.map_shared_rank(&sh, jj)->run + sh.lo[jj];
          pos += bound_in(rj, sh.off[jj + 1] - sh.off[jj], v, jj < j);
        }
        dst_g[pos] = key_float(v);
      }
    }
    cl.sync();  // every remote read of this segment is done
    if (tot <= kCap) {
      if (tid <= kP) sh.loff[tid] = sh.off[tid];
      __syncthreads();
      int nl = kP, src = 0;
      while (nl > 1) {
        merge_round(sh.buf[src], sh.buf[src ^ 1], sh.loff, nl, tot);
        __syncthreads();
        const int nn = (nl + 1) / 2;
        if (tid == 0) {
          for (int e = 1; e <= nn; ++e) sh.loff[e] = sh.loff[min(2 * e, nl)];
        }
        __syncthreads();
        nl = nn;
        src ^= 1;
      }
      const uint32_t* fin = sh.buf[src];
      for (int x = tid; x < tot; x += kT) dst_g[x] = key_float(fin[x]);
    }
    __syncthreads();
  }
}

}  // namespace

bool seg_sort_fits(int64_t max_len) { return max_len <= kMaxLen; }

int launch_seg_sort(const float* in, float* out, int64_t stride, int nseg, const int64_t* seg_b,
                    const int64_t* seg_e, cudaStream_t st) {
  if (nseg <= 0) return 0;
  static int attr_device = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_device != dev) {
    if (cudaFuncSetAttribute(seg_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(SegSortShared)) != cudaSuccess)
      return -1;
    attr_device = dev;
  }
  const int clusters = nseg < 512 ? nseg : 512;
  seg_sort_kernel<<<clusters * kP, kT, sizeof(SegSortShared), st>>>(in, out, stride, nseg, seg_b,
                                                                    seg_e);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace lmsb

namespace {
// the cluster sort (default) or, with LMSB_SEG_BUCKET=1, the segmented bucket sort
bool sort_segments(const float* d_in, float* d_out, int64_t total, int32_t nseg,
                   const int64_t* h_b, const int64_t* h_e, const int64_t* d_seg) {
  if (!lmsb::use_seg_bucket()) return lmsb::launch_seg_sort(d_in, d_out, 0, nseg, d_seg, d_seg + nseg, 0) == 0;
  int64_t max_len = 0;
  for (int32_t s = 0; s < nseg; ++s) max_len = std::max<int64_t>(max_len, h_e[s] - h_b[s]);
  if (max_len <= 0) return true;
  const size_t sb = lmsb::seg_bucket_sort_scratch_bytes(total, nseg, max_len);
  void* scratch = nullptr;
  if (cudaMalloc(&scratch, sb) != cudaSuccess) return false;
  const bool ok = lmsb::launch_seg_bucket_sort(d_in, d_out, total, nseg, max_len, d_seg, d_seg + nseg,
                                               scratch, sb, 0) == 0 &&
                  cudaDeviceSynchronize() == cudaSuccess;
  cudaFree(scratch);
  return ok;
}
}  // namespace

extern "C" int lms_debug_seg_sort(int device, const float* keys, float* out, int64_t total,
                                  int32_t nseg, const int64_t* seg_begin, const int64_t* seg_end) {
  if (!keys || !out || total < 0 || nseg < 0 || (nseg > 0 && (!seg_begin || !seg_end)))
    return LMS_ERR_INVALID;
  for (int32_t s = 0; s < nseg; ++s)
    if (seg_begin[s] < 0 || seg_end[s] > total ||
        (seg_end[s] > seg_begin[s] && !lmsb::seg_sort_fits(seg_end[s] - seg_begin[s])))
      return LMS_ERR_INVALID;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
    return LMS_ERR_NODEVICE;
  if (cudaSetDevice(device) != cudaSuccess) return LMS_ERR_CUDA;
  float *d_in = nullptr, *d_out = nullptr;
  int64_t* d_seg = nullptr;
  const size_t kb = (size_t)(total > 0 ? total : 1) * sizeof(float);
  int rc = LMS_OK;
  if (cudaMalloc(&d_in, kb) != cudaSuccess || cudaMalloc(&d_out, kb) != cudaSuccess ||
      cudaMalloc(&d_seg, 2 * (size_t)(nseg > 0 ? nseg : 1) * sizeof(int64_t)) != cudaSuccess) {
    rc = LMS_ERR_NOMEM;
  } else if (cudaMemcpy(d_in, keys, total * sizeof(float), cudaMemcpyHostToDevice) !=
                 cudaSuccess ||
             cudaMemcpy(d_out, keys, total * sizeof(float), cudaMemcpyHostToDevice) !=
                 cudaSuccess ||
             cudaMemcpy(d_seg, seg_begin, nseg * sizeof(int64_t), cudaMemcpyHostToDevice) !=
                 cudaSuccess ||
             cudaMemcpy(d_seg + nseg, seg_end, nseg * sizeof(int64_t), cudaMemcpyHostToDevice) !=
                 cudaSuccess) {
    rc = LMS_ERR_CUDA;
  } else if (!sort_segments(d_in, d_out, total, nseg, seg_begin, seg_end, d_seg) ||
             cudaDeviceSynchronize() != cudaSuccess ||
             cudaMemcpy(out, d_out, total * sizeof(float), cudaMemcpyDeviceToHost) !=
                 cudaSuccess) {
    rc = LMS_ERR_CUDA;
  }
  cudaFree(d_in);
  cudaFree(d_out);
  cudaFree(d_seg);
  return rc;
}
