// lms_band_dev.cuh -- device helpers shared by the band-stage kernels
// (lms_band.cu) and the sweep collect (lms_sweep.cu).
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdint>

#include "lms_band.cuh"

namespace lmsb {

#ifndef LMSB_SLOPE_BITS
#define LMSB_SLOPE_BITS 17
#endif
constexpr int kSlopeBits = LMSB_SLOPE_BITS;  // within-band slope order bits of a collected key

__device__ __forceinline__ float band_key(double u) {
  // monotone non-decreasing map of the slope to fp32 (clamped, so ordered)
  const float f = (float)u;
  return fminf(fmaxf(f, -FLT_MAX), FLT_MAX);
}

// slope and class of vertex (i, j) exactly as _scan_rank_range forms it
// (backend.py:200-205): 0 never a window (a_i == a_j or non-finite u),
// 1 banded, 2 beyond the fp32 key range (always passed to the exact stage)
__device__ __forceinline__ int classify(const BandFit& bf, double ai, double bi, double aj,
                                        double bj, double* pu) {
  const double da = __dsub_rn(ai, aj);
  if (da == 0.0) return 0;
  const double u = __ddiv_rn(__dsub_rn(bi, bj), da);
  if (!isfinite(u)) return 0;
  *pu = u;
  return fabs(u) * bf.amax < 1e30 ? 1 : 2;
}

// number of boundaries <= key, i.e. the band index
__device__ __forceinline__ int band_of(const float* __restrict__ bnd, int nb, float key) {
  int lo = 0, hi = nb;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (bnd[mid] <= key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

}  // namespace lmsb
