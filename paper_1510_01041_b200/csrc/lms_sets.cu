// lms_sets.cu -- device side of solve_lms_batch over a list of point sets
// (solver.py:83-140 per set; the reference's per-peak loop, detect.py:184-213):
// the sets arrive interleaved (x, y) as one staged upload, are split into
// the solver's dual lines, checked per set (solver.py:67-80: finite, at
// least two distinct x), and after the batched solve each set's contact set
// (solver.py:122-140, flagged per point by contacts_batch_kernel) is
// compacted into ascending point indices on the device.

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "lms_sets.cuh"

namespace lmsb {

namespace {

__global__ void split_xy_kernel(const double2* __restrict__ xy, int64_t n, double* __restrict__ a,
                                double* __restrict__ b) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const double2 p = xy[k];
    a[k] = p.x;
    b[k] = p.y;
  }
}

// per set: [0] all finite, [1] min x, [2] max x (one CTA per set)
__global__ void __launch_bounds__(256) set_stats_kernel(const double* __restrict__ a,
                                                        const double* __restrict__ b,
                                                        const int64_t* __restrict__ offs,
                                                        int64_t nsets, double* __restrict__ stats) {
  __shared__ double smin[8], smax[8];
  __shared__ int sbad[8];
  for (int64_t f = blockIdx.x; f < nsets; f += gridDim.x) {
    const int64_t o = offs[f], n = offs[f + 1] - o;
    double lo = INFINITY, hi = -INFINITY;
    int bad = 0;
    for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
      const double x = a[o + k], y = b[o + k];
      bad |= !(isfinite(x) && isfinite(y));
      lo = fmin(lo, x);
      hi = fmax(hi, x);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, off));
      hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, off));
      bad |= __shfl_xor_sync(0xffffffffu, bad, off);
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
      smin[w] = lo;
      smax[w] = hi;
      sbad[w] = bad;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int e = 1; e < 8; ++e) {
        lo = fmin(lo, smin[e]);
        hi = fmax(hi, smax[e]);
        bad |= sbad[e];
      }
      stats[3 * f] = bad ? 0.0 : 1.0;
      stats[3 * f + 1] = lo;
      stats[3 * f + 2] = hi;
    }
    __syncthreads();
  }
}

// contacts per set (count), then an exclusive scan over the sets (one CTA)
__global__ void __launch_bounds__(256) contact_count_kernel(const uint8_t* __restrict__ flags,
                                                            const int64_t* __restrict__ offs,
                                                            int64_t nsets, int64_t* __restrict__ cnt) {
  __shared__ int part[8];
  for (int64_t f = blockIdx.x; f < nsets; f += gridDim.x) {
    const int64_t o = offs[f], n = offs[f + 1] - o;
    int c = 0;
    for (int64_t k = threadIdx.x; k < n; k += blockDim.x) c += flags[o + k] != 0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
      for (int e = 0; e < 8; ++e) t += part[e];
      cnt[f] = t;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(1024) exclusive_scan_kernel(const int64_t* __restrict__ in, int64_t m,
                                                              int64_t* __restrict__ out) {
  __shared__ int64_t part[1024];
  const int64_t per = (m + 1023) / 1024;
  const int64_t b0 = threadIdx.x * per, b1 = b0 + per < m ? b0 + per : m;
  int64_t sum = 0;
  for (int64_t k = b0; k < b1; ++k) sum += in[k];
  part[threadIdx.x] = sum;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    const int64_t v = threadIdx.x >= off ? part[threadIdx.x - off] : 0;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  int64_t run = threadIdx.x ? part[threadIdx.x - 1] : 0;
  for (int64_t k = b0; k < b1; ++k) {
    out[k] = run;
    run += in[k];
  }
  if (threadIdx.x == 1023) out[m] = part[1023];
}

// each set's flagged points, ascending, as set-local int32 indices
__global__ void __launch_bounds__(256) contact_write_kernel(const uint8_t* __restrict__ flags,
                                                            const int64_t* __restrict__ offs,
                                                            int64_t nsets,
                                                            const int64_t* __restrict__ coff,
                                                            int32_t* __restrict__ out) {
  __shared__ int warp_tot[8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t f = blockIdx.x; f < nsets; f += gridDim.x) {
    const int64_t o = offs[f], n = offs[f + 1] - o;
    int64_t base = coff[f];
    for (int64_t k0 = 0; k0 < n; k0 += blockDim.x) {
      const int64_t k = k0 + threadIdx.x;
      const bool fl = k < n && flags[o + k] != 0;
      const unsigned bal = __ballot_sync(0xffffffffu, fl);
      if (lane == 0) warp_tot[w] = __popc(bal);
      __syncthreads();
      int before = 0, tot = 0;
      for (int e = 0; e < 8; ++e) {
        before += e < w ? warp_tot[e] : 0;
        tot += warp_tot[e];
      }
      if (fl) out[base + before + __popc(bal & ((1u << lane) - 1u))] = (int32_t)k;
      base += tot;
      __syncthreads();
    }
  }
}

}  // namespace

void launch_split_xy(const double* xy, int64_t n, double* a, double* b, int sms, cudaStream_t st) {
  if (n <= 0) return;
  const int grid = (int)((n + 255) / 256 < (int64_t)sms * 8 ? (n + 255) / 256 : (int64_t)sms * 8);
  split_xy_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const double2*>(xy), n, a, b);
}

void launch_set_stats(const double* a, const double* b, const int64_t* offs, int64_t nsets,
                      double* stats, int sms, cudaStream_t st) {
  if (nsets <= 0) return;
  const int grid = (int)(nsets < (int64_t)sms * 16 ? nsets : (int64_t)sms * 16);
  set_stats_kernel<<<grid, 256, 0, st>>>(a, b, offs, nsets, stats);
}

void launch_contact_compact(const uint8_t* flags, const int64_t* offs, int64_t nsets, int64_t* cnt,
                            int64_t* coff, int32_t* out, int sms, cudaStream_t st) {
  if (nsets <= 0) return;
  const int grid = (int)(nsets < (int64_t)sms * 16 ? nsets : (int64_t)sms * 16);
  contact_count_kernel<<<grid, 256, 0, st>>>(flags, offs, nsets, cnt);
  exclusive_scan_kernel<<<1, 1024, 0, st>>>(cnt, nsets, coff);
  contact_write_kernel<<<grid, 256, 0, st>>>(flags, offs, nsets, coff, out);
}

}  // namespace lmsb
