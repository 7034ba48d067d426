// lms_hough.cuh -- launch interfaces of lms_hough.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace lmsb {

// Lit-pixel indices (row-major) of the image; *d_count receives their number.
int hough_extract(const uint8_t* d_img, int64_t npix, int threshold, int64_t* d_pix,
                  int64_t* d_count, void* temp, size_t* temp_bytes, cudaStream_t stream);
size_t extract_temp_bytes(int64_t npix);

// Votes of npts points (pixel indices, or explicit x/y when d_x != nullptr)
// into acc[n_rho * n_theta] (rho-major, as HoughAccumulator.bins).
void hough_vote(const int64_t* d_pix, const double* d_x, const double* d_y, int64_t npts,
                int64_t width, const double* d_cos, const double* d_sin, int n_theta,
                double rho_max, double drho, int64_t n_rho, unsigned long long* d_acc, int sms,
                cudaStream_t stream);

// Supports of up to 64 peaks in scan order; peak q's members are written to
// d_out[offsets[q*nb] .. offsets[(q+1)*nb]) with nb = support_blocks(npts);
// the total is offsets[npeaks*nb].  Ids are pixel indices (image points) or
// point ordinals (explicit points).
int64_t support_blocks(int64_t npts);
int hough_support(const int64_t* d_pix, const double* d_x, const double* d_y, int64_t npts,
                  int64_t width, const double* d_cos, const double* d_sin, const int64_t* d_rbin,
                  int npeaks, double rho_max, double drho, int64_t n_rho,
                  unsigned long long* d_masks, int64_t* d_counts, int64_t* d_offsets, void* temp,
                  size_t temp_bytes, int64_t* d_out, int64_t out_cap, cudaStream_t stream);
size_t support_scan_temp_bytes(int64_t m);

// out[k] = (int32) in[k], k < m (support ids narrowed for the download)
void launch_narrow_i32(const int64_t* in, int32_t* out, int64_t m, cudaStream_t st);

}  // namespace lmsb
