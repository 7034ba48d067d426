// lms_detect.cuh -- detect_lines on the device straight from the image
// (lms_detect.cu): vote, peaks, supports, thinned LMS designs.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "lms_common.cuh"

namespace lmsb {

// accumulators up to this many bins go through the device peak finder
// (one CTA sorts their keys in shared memory)
constexpr int kDetectMaxBins = 16384;
// widest image the row-bitmask vote handles (bitmask words per CTA)
constexpr int64_t kDetectMaxWidth = 4096 * 32;

struct DetectImage {
  const uint8_t* img;
  int64_t npix, width;
  int threshold;
};

struct HoughGrid {
  int n_rho, n_theta;
  double rho_max, drho;
};

// wedge: n_rho bin-edge table (filled); bits: the image's lit bitmask,
// rows of ceil(width / 32) words (filled, read by the support passes)
void launch_detect_vote(const DetectImage& im, const HoughGrid& g, const double* cos_t,
                        const double* sin_t, double* wedge, uint32_t* bits, unsigned long long* acc,
                        unsigned long long* nlit, int sms, cudaStream_t st);
// peaks[3k .. 3k+2] = (rho bin, theta bin, votes), *npeaks of them (device)
void launch_detect_peaks(const unsigned long long* acc, const HoughGrid& g, int64_t min_votes,
                         int max_peaks, int64_t* peaks, int64_t* npeaks, cudaStream_t st);
// rows of the image (the support passes count per (peak, row))
int64_t detect_support_rows(int64_t npix, int64_t width);

// fp32 + fp64 trig of one theta bin centre
struct Trig {
  float c32, s32;
  double c, s;
  double ic;  // 1 / c (0 when c == 0): predictions only, never a decision
};
// The peaks grouped by their support trig (one slot per distinct theta bin;
// slot s holds peak[first[s] .. first[s + 1]) with their rho bins), built on
// the host from the peak list and passed by value.
struct SupportTable {
  int npeaks, nslot;
  Trig trig[64];
  int first[65];
  int peak[64];
  int rbin[64];
};
// counts: npeaks * rows scratch; soffs: npeaks + 1 support starts (prefix
// of the votes); offs: npeaks * rows positions; out: the members' pixel
// ids; *bad counts supports whose size differs from the votes
void launch_detect_support(const DetectImage& im, const HoughGrid& g, const SupportTable& tb,
                           const double* wedge, const uint32_t* bits, const int64_t* soffs,
                           unsigned* counts, int64_t* offs, int32_t* out, unsigned long long* bad,
                           int sms, cudaStream_t st);
// per peak: the thinned design (doffs) in the axis-swapped frame and the
// abscissa range lim[2q], lim[2q + 1]
void launch_detect_design(const int64_t* peaks, const int64_t* npeaks_d, int npeaks,
                          const int64_t* soffs, const int32_t* ids, int64_t width, int64_t cap,
                          const uint8_t* swap_t, const int64_t* doffs, double* da, double* db,
                          double* lim, cudaStream_t st);

}  // namespace lmsb
