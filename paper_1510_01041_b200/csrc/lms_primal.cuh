// lms_primal.cuh -- primal brute force (lms_primal.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/lms_b200.h"

namespace lmsb {

constexpr int64_t kPrimalMaxN = 16384;  // intercepts sorted in shared memory (128 KiB)

size_t primal_smem_bytes(int64_t n);
// One record per pair rank (height = narrowest q-span, u = slope,
// v_low / v_high = the window's intercepts).
int launch_primal(const double* x, const double* y, int64_t n, int64_t q, lms_candidate* recs,
                  int grid, cudaStream_t stream);

}  // namespace lmsb
