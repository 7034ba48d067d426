// lms_band.cuh -- slope-band pruning stage (lms_band.cu), host interface.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "lms_kernels.cuh"

namespace lmsb {

// Lines per fit the band stage handles (its sorted keys live in shared memory).
constexpr int kBandMaxN = 16384;
// Most bands per fit (band ids are 16-bit; the hist kernel keeps K boundaries
// and K counters in shared memory).
constexpr int kBandMaxK = 16384;

struct BandFit {
  const double* a;  // the fit's lines (input order)
  const double* b;
  int64_t n, q;
  int64_t R0, span;  // pair ranks [R0, R0 + span)
  double c;          // centre of the a-range
  double dev;        // >= max_k |a_k - c|
  double amax, bmax;
};

struct BandPartition {
  int64_t S;  // slope samples
  int K;      // bands
  float* sample;
  float* sample_sorted;
  unsigned long long* nvalid;
  float* bounds;                 // K - 1
  uint16_t* bid;                 // span
  unsigned long long* counts;    // K + 1
  unsigned long long* offsets;   // K + 1
  unsigned long long* cursor;    // K
  unsigned long long* nforce;
  uint32_t* members;             // span: packed (i << 16 | j), grouped by band
  void* temp;
  size_t temp_bytes;
};

struct BandArgs {
  const unsigned long long* offsets;
  const uint32_t* members;
  const int32_t* list;  // mode 1: bands to filter (blockIdx -> band)
  double* lb;           // per band lower bound of any vertex height
  double* ulo;          // per band slope extent
  double* uhi;
  const lms_candidate* best;  // the fit's current best record (H)
  int64_t* out_ranks;
  int32_t* out_fits;
  int32_t fit;
  unsigned long long* out_count;
};

int band_max_n();
size_t band_sample_temp_bytes(int64_t S);
size_t band_scan_temp_bytes(int K);
size_t band_hist_smem(int K);
int launch_band_partition(const BandFit& bf, const BandPartition& bp, int sms, cudaStream_t st);
// mode 0: grid = K (bounds of every band); mode 1: grid = bands in `list`
void launch_band(const BandFit& bf, const BandArgs& ba, int mode, int grid, cudaStream_t st);
void launch_band_seeds(const BandFit& bf, const unsigned long long* offsets,
                       const uint32_t* members, const int32_t* list, int nb, int per_band,
                       int64_t* ranks, int32_t* fits, int32_t fit, unsigned long long* count,
                       cudaStream_t st);

}  // namespace lmsb
