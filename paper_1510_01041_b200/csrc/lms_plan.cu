// lms_plan.cu -- device-side work plan of the count filter.
//
// The filter's unit of work is a warp task: up to 32*V consecutive vertex
// ranks of one triangle row of one fit.  Rows are ordered in two phases:
// phase A holds every kPhaseStride-th row of every fit, phase B the rest, so
// that after phase A each fit's bound H and line order already come from a
// spread sample of its vertices.  The plan is
//   row_fit[g], row_i[g]  fit and triangle row of global row g
//   row_task_prefix[g]    first task of row g (exclusive scan of task counts)
//   task_row[t]           global row of task t
// built on the device (one map/count kernel, a CUB scan, one expand kernel),
// so an 8,192-fit batch needs no host loop over its 4 M rows.

#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include <cstdint>

#include "lms_common.cuh"
#include "lms_kernels.cuh"
#include "lms_plan.cuh"

namespace lmsb {

namespace {

// phase prefix arrays: prefA[f] / prefB[f] = first global row of fit f in
// phase A / B (prefB already offset by the phase-A row total).
__device__ __forceinline__ int64_t fit_of_row(const int64_t* pref, int64_t nfits, int64_t g) {
  int64_t lo = 0, hi = nfits - 1;  // largest f with pref[f] <= g
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (pref[mid] <= g) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__global__ void row_counts_kernel(const FitDesc* __restrict__ fits,
                                  const int64_t* __restrict__ prefA,
                                  const int64_t* __restrict__ prefB, int64_t nfits,
                                  int64_t rowsA, int64_t nrows, int64_t tv,
                                  int64_t* __restrict__ counts, int32_t* __restrict__ row_fit,
                                  int32_t* __restrict__ row_i) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g <= nrows;
       g += (int64_t)gridDim.x * blockDim.x) {
    if (g == nrows) {
      counts[g] = 0;  // the scan's last element becomes the task total
      continue;
    }
    const bool phase_a = g < rowsA;
    const int64_t f = fit_of_row(phase_a ? prefA : prefB, nfits, g);
    const FitDesc fd = fits[f];
    const int64_t m = g - (phase_a ? prefA[f] : prefB[f]);
    // phase A: k = stride*m; phase B: the m-th k in [0, nrows) with k % stride != 0
    const int64_t k = phase_a ? kPhaseStride * m
                              : kPhaseStride * (m / (kPhaseStride - 1)) + (m % (kPhaseStride - 1)) + 1;
    const int64_t i = fd.row0 + k;
    const int64_t rlo = row_offset(fd.n, i);
    const int64_t rhi = rlo + (fd.n - 1 - i);
    const int64_t rs = rlo > fd.rank_lo ? rlo : fd.rank_lo;
    const int64_t re = rhi < fd.rank_hi ? rhi : fd.rank_hi;
    counts[g] = re > rs ? (re - rs + tv - 1) / tv : 0;
    row_fit[g] = (int32_t)f;
    row_i[g] = (int32_t)i;
  }
}

__global__ void expand_tasks_kernel(const int64_t* __restrict__ prefix, int64_t nrows,
                                    int32_t* __restrict__ task_row) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < nrows;
       g += (int64_t)gridDim.x * blockDim.x) {
    for (int64_t t = prefix[g]; t < prefix[g + 1]; ++t) task_row[t] = (int32_t)g;
  }
}

__global__ void line_fit_kernel(const int64_t* __restrict__ seg, int64_t nfits,
                                int32_t* __restrict__ line_fit) {
  for (int64_t f = blockIdx.x; f < nfits; f += gridDim.x) {
    for (int64_t k = seg[f] + threadIdx.x; k < seg[f + 1]; k += blockDim.x)
      line_fit[k] = (int32_t)f;
  }
}

}  // namespace

// Sum_{m=1..M} ceil(m / tv).
int64_t ceil_sum(int64_t M, int64_t tv) {
  if (M <= 0) return 0;
  const int64_t k = M / tv, r = M % tv;
  return tv * k * (k + 1) / 2 + (k + 1) * r;
}

int64_t row_tasks(int64_t n, int64_t R0, int64_t R1, int64_t i, int64_t tv) {
  const int64_t lo = row_offset(n, i), hi = lo + (n - 1 - i);
  const int64_t rs = lo > R0 ? lo : R0, re = hi < R1 ? hi : R1;
  return re > rs ? (re - rs + tv - 1) / tv : 0;
}

int64_t fit_tasks(int64_t n, int64_t R0, int64_t R1, int64_t tv, int64_t* row0, int64_t* nrows) {
  if (R1 <= R0) {
    *row0 = 0;
    *nrows = 0;
    return 0;
  }
  int64_t i0, j0, i1, j1;
  decode_rank(n, R0, &i0, &j0);
  decode_rank(n, R1 - 1, &i1, &j1);
  *row0 = i0;
  *nrows = i1 - i0 + 1;
  auto row_len = [&](int64_t i) {
    const int64_t lo = row_offset(n, i), hi = lo + (n - 1 - i);
    const int64_t rs = lo > R0 ? lo : R0, re = hi < R1 ? hi : R1;
    return re > rs ? re - rs : 0;
  };
  if (i0 == i1) return (row_len(i0) + tv - 1) / tv;
  int64_t t = (row_len(i0) + tv - 1) / tv + (row_len(i1) + tv - 1) / tv;
  // full middle rows i0+1 .. i1-1 have lengths n-2-i0 down to n-i1
  t += ceil_sum(n - 2 - i0, tv) - ceil_sum(n - i1 - 1, tv);
  return t;
}

int launch_plan(const PlanArgs& p, cudaStream_t stream) {
  const int threads = 256;
  const int blocks = (int)((p.nrows + 1 + threads - 1) / threads < 4096
                               ? (p.nrows + 1 + threads - 1) / threads
                               : 4096);
  row_counts_kernel<<<blocks, threads, 0, stream>>>(p.fits, p.prefA, p.prefB, p.nfits, p.rowsA,
                                                    p.nrows, p.task_vertices, p.counts, p.row_fit,
                                                    p.row_i);
  size_t bytes = p.temp_bytes;
  if (cub::DeviceScan::ExclusiveSum(p.temp, bytes, p.counts, p.row_task_prefix, p.nrows + 1,
                                    stream) != cudaSuccess)
    return -1;
  expand_tasks_kernel<<<blocks, threads, 0, stream>>>(p.row_task_prefix, p.nrows, p.task_row);
  return 0;
}

size_t plan_temp_bytes(int64_t nrows) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const int64_t*)nullptr, (int64_t*)nullptr,
                                nrows + 1);
  return bytes;
}

void launch_line_fit(const int64_t* seg, int64_t nfits, int32_t* line_fit, cudaStream_t stream) {
  const int blocks = (int)(nfits < 65535 ? nfits : 65535);
  line_fit_kernel<<<blocks > 0 ? blocks : 1, 128, 0, stream>>>(seg, nfits, line_fit);
}

}  // namespace lmsb
