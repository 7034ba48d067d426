// lms_sets.cuh -- batches of point sets (lms_sets.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace lmsb {

// (x, y) pairs -> a = x, b = y
void launch_split_xy(const double* xy, int64_t n, double* a, double* b, int sms, cudaStream_t st);
// stats[3f .. 3f+2] = (all finite, min x, max x) of set f = [offs[f], offs[f+1])
void launch_set_stats(const double* a, const double* b, const int64_t* offs, int64_t nsets,
                      double* stats, int sms, cudaStream_t st);
// flagged points per set -> cnt (nsets), coff (nsets + 1 offsets), out (set-local ids)
void launch_contact_compact(const uint8_t* flags, const int64_t* offs, int64_t nsets, int64_t* cnt,
                            int64_t* coff, int32_t* out, int sms, cudaStream_t st);

}  // namespace lmsb
