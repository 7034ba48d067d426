// lms_order.cu -- line streaming order for the count filter.
//
// The filter drops a vertex as soon as more than n - q lines have been seen
// outside both of its windows (it can no longer reach q).  Lines far from
// the best line found so far sit outside the windows of every near-optimal
// vertex, so streaming them first lets those (expensive, late-exiting)
// vertices exit after ~n - q lines instead of ~0.7n (measured on config 2:
// warp-task exit point 0.70n in input order, 0.51n far-first).  The order
// only changes when the filter stops counting, never what it counts, so the
// result is independent of it.
//
// key_k = |(u* a_k - b_k) - (v_low* + v_high*)/2|, the vertical distance of
// point k from its fit's current best LMS line; each fit's lines are sorted
// by descending key (CUB segmented radix sort, one segment per fit) and
// gathered into a permuted copy that the filter streams.  A fit without a
// best record keeps its input order.

#include <cub/device/device_segmented_radix_sort.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>

#include "lms_common.cuh"
#include "lms_kernels.cuh"

namespace lmsb {

namespace {

__global__ void order_keys_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                  int64_t nlines, const int32_t* __restrict__ line_fit,
                                  const lms_candidate* __restrict__ best,
                                  float* __restrict__ keys, int* __restrict__ idx) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nlines;
       k += (int64_t)gridDim.x * blockDim.x) {
    const lms_candidate bc = best[line_fit[k]];
    float key = 0.f;
    if (bc.found) {
      const double mid = 0.5 * (bc.v_low + bc.v_high);
      const double d = fabs(fma(bc.u, a[k], -b[k]) - mid);
      key = isfinite(d) ? (float)d : 3.0e38f;
    }
    keys[k] = key;
    idx[k] = (int)k;
  }
}

__global__ void gather_lines_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                    int64_t nlines, const int* __restrict__ perm,
                                    double* __restrict__ pa, double* __restrict__ pb) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nlines;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int s = perm[k];
    pa[k] = a[s];
    pb[k] = b[s];
  }
}

}  // namespace

size_t order_temp_bytes(int64_t nlines, int64_t nfits) {
  size_t bytes = 0;
  cub::DeviceSegmentedRadixSort::SortPairsDescending(
      nullptr, bytes, (const float*)nullptr, (float*)nullptr, (const int*)nullptr, (int*)nullptr,
      (int)nlines, (int)nfits, (const int64_t*)nullptr, (const int64_t*)nullptr);
  return bytes;
}

int launch_line_order(const OrderArgs& o, cudaStream_t stream) {
  const int threads = 256;
  const int blocks = (int)std::min<int64_t>((o.nlines + threads - 1) / threads, 148 * 16);
  order_keys_kernel<<<blocks, threads, 0, stream>>>(o.a, o.b, o.nlines, o.line_fit, o.best,
                                                    o.keys_in, o.idx_in);
  size_t bytes = o.temp_bytes;
  cudaError_t e = cub::DeviceSegmentedRadixSort::SortPairsDescending(
      o.temp, bytes, o.keys_in, o.keys_out, o.idx_in, o.idx_out, (int)o.nlines, (int)o.nfits,
      o.seg_begin, o.seg_begin + 1, 0, (int)(8 * sizeof(float)), stream);
  if (e != cudaSuccess) return -1;
  gather_lines_kernel<<<blocks, threads, 0, stream>>>(o.a, o.b, o.nlines, o.idx_out, o.pa, o.pb);
  return 0;
}

}  // namespace lmsb
