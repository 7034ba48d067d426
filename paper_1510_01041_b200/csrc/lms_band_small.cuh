// lms_band_small.cuh -- fused slope-band search of small fits (lms_band_small.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "lms_kernels.cuh"

namespace lmsb {

// Fits this small (lines) and this large (pairs) take the fused kernel.
constexpr int64_t kSmallMaxN = 1024;
constexpr int64_t kSmallMinPairs = 4097;

struct SmallArgs {
  const double* a;  // concatenated lines of the batch
  const double* b;
  const FitDesc* fits;
  const int32_t* list;  // fits handled, one CTA each
  lms_candidate* out;   // out[fit]: the fit's exact record (found == 0: none)
  unsigned long long* counters;  // optional [12]: admitted bands, queued, exact, sweeps, cycles
  int timing;                    // also accumulate per-stage clock64 cycles (LMSB_SMALL_DEBUG)
};

void launch_small_fits(const SmallArgs& args, int64_t count, int64_t max_n, int sms, cudaStream_t st);

}  // namespace lmsb
