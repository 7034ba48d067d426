// lms_hough.cu -- Hough vote and per-peak support gather (HBM-bound stages
// that feed the batched LMS refits of detect_lines).
//
//   extract   lit pixels (value >= threshold) of the uint8 image, in
//             row-major scan order (extract_points, hough.py:93-103):
//             order-preserving compaction of pixel indices (CUB select)
//   vote      one vote per (point, theta bin) at the bin centre:
//             rho = x*cos(t) + y*sin(t) with two rounded products and a
//             rounded sum, bin = clip(floor((rho + rho_max) / d_rho))
//             (hough.py:112-129, HoughParams.rho_bin :60-63); per-CTA
//             shared-memory histograms merged with 64-bit global atomics
//   support   for up to 64 peaks at once, the points whose re-vote at the
//             peak's theta lands in the peak's rho bin, in scan order
//             (supporting_points, hough.py:171-184): pass 1 builds one
//             64-bit membership mask per point and per-(peak, block)
//             counts, a CUB scan turns the counts into output positions,
//             pass 2 writes each block's members in order with warp
//             ballots.
// cos/sin of the bin centres are computed on the host exactly as the
// reference computes them (np.cos/np.sin of np.radians for the vote,
// math.cos/math.sin of math.radians for the support) and passed in, so the
// device arithmetic reproduces the reference's bins bit for bit.

#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <cuda_runtime.h>

#include <cmath>
#include <algorithm>
#include <cstdint>

#include "lms_hough.cuh"

namespace lmsb {

namespace {

struct LitPixel {
  const uint8_t* img;
  int threshold;
  __host__ __device__ __forceinline__ bool operator()(const int64_t& k) const {
    return (int)img[k] >= threshold;
  }
};

// HoughParams.rho_bin (hough.py:60-63): floor((rho + rho_max) / d_rho) cast
// to int64 then clipped to [0, n_rho - 1].  numpy's float->int64 cast of a
// value outside the int64 range (or NaN) yields INT64_MIN on x86, which the
// clip maps to 0; the same is done here.
__device__ __forceinline__ int64_t rho_bin(double x, double y, double c, double s, double rho_max,
                                           double drho, int64_t n_rho) {
  const double rho = __dadd_rn(__dmul_rn(x, c), __dmul_rn(y, s));
  const double f = floor(__ddiv_rn(__dadd_rn(rho, rho_max), drho));
  if (!(f >= -9.2233720368547758e18 && f < 9.2233720368547758e18)) return 0;
  int64_t r = (int64_t)f;
  if (r < 0) r = 0;
  if (r > n_rho - 1) r = n_rho - 1;
  return r;
}

// rho_bin through an fp32 estimate: rho32 = x c + y s with every operand
// rounded to fp32 is within E = 2^-19 (|x c| + |y s| + |rho32| + rho_max) +
// 1e-30 of the reference's fp64 rho (fp32 operand / product / sum roundings
// <= 4 * 2^-24 of the magnitudes), and the fp32 bin coordinates of rho32 -+ E
// bracket the fp64 one (their own roundings add 2^-23 relative, inside E's
// slack).  When both ends floor to the same bin that bin is exact; otherwise
// (within E of a bin edge, or non-finite) the fp64 path decides.
__device__ __forceinline__ int64_t rho_bin_fast(double x, double y, const double* c, const double* s,
                                                float c32, float s32, double rho_max,
                                                float rho_max32, double drho, float inv_drho32,
                                                int64_t n_rho) {
  const float x32 = (float)x, y32 = (float)y;
  const float xc = x32 * c32, ys = y32 * s32;
  const float rho32 = xc + ys;
  const float E = 0x1p-19f * (fabsf(xc) + fabsf(ys) + fabsf(rho32) + rho_max32) + 1e-30f;
  const float glo = floorf((rho32 - E + rho_max32) * inv_drho32);
  const float ghi = floorf((rho32 + E + rho_max32) * inv_drho32);
  if (glo == ghi && fabsf(glo) < 0x1p22f) {
    int64_t r = (int64_t)glo;
    if (r < 0) r = 0;
    if (r > n_rho - 1) r = n_rho - 1;
    return r;
  }
  return rho_bin(x, y, *c, *s, rho_max, drho, n_rho);
}

// A point is either a pixel index (x = p % width, y = p / width) or an
// explicit (x, y) pair (xs != nullptr).
struct PointSrc {
  const int64_t* pix;
  const double* xs;
  const double* ys;
  int64_t width;
  __device__ __forceinline__ void get(int64_t k, double& x, double& y) const {
    if (xs) {
      x = xs[k];
      y = ys[k];
    } else {
      const int64_t p = pix[k];
      x = (double)(p % width);
      y = (double)(p / width);
    }
  }
  __device__ __forceinline__ int64_t id(int64_t k) const { return xs ? k : pix[k]; }
};

constexpr int kVoteThreads = 256;
constexpr int kMaxTheta = 512;  // theta bins with fp32 trig staged in shared memory

__global__ void __launch_bounds__(kVoteThreads)
    vote_kernel(PointSrc src, int64_t npts, const double* __restrict__ cos_t,
                const double* __restrict__ sin_t, int n_theta,
                double rho_max, double drho, int64_t n_rho, int use_smem,
                unsigned long long* __restrict__ acc) {
  extern __shared__ unsigned int hist[];
  __shared__ float2 cs32[kMaxTheta];
  const int64_t nbins = n_rho * n_theta;
  const float rho_max32 = (float)rho_max;
  const float inv_drho32 = (float)(1.0 / drho);
  for (int t = threadIdx.x; t < n_theta && t < kMaxTheta; t += blockDim.x)
    cs32[t] = make_float2((float)cos_t[t], (float)sin_t[t]);
  __syncthreads();
  if (use_smem) {
    for (int64_t e = threadIdx.x; e < nbins; e += blockDim.x) hist[e] = 0u;
    __syncthreads();
  }
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < npts;
       k += (int64_t)gridDim.x * blockDim.x) {
    double x, y;
    src.get(k, x, y);
    for (int t = 0; t < n_theta; ++t) {
      const float2 cs = t < kMaxTheta ? cs32[t] : make_float2((float)cos_t[t], (float)sin_t[t]);
      const int64_t r = rho_bin_fast(x, y, cos_t + t, sin_t + t, cs.x, cs.y, rho_max, rho_max32,
                                     drho, inv_drho32, n_rho);
      const int64_t bin = r * n_theta + t;
      if (use_smem) atomicAdd(&hist[bin], 1u);
      else atomicAdd(&acc[bin], 1ULL);
    }
  }
  if (use_smem) {
    __syncthreads();
    for (int64_t e = threadIdx.x; e < nbins; e += blockDim.x)
      if (hist[e]) atomicAdd(&acc[e], (unsigned long long)hist[e]);
  }
}

constexpr int kSupThreads = 256;
constexpr int kSupItems = 16;  // points per thread per block chunk
constexpr int64_t kSupChunk = (int64_t)kSupThreads * kSupItems;

struct PeakArgs {
  const double* cos_p;
  const double* sin_p;
  const int64_t* rbin_p;
  int npeaks;
  double rho_max;
  double drho;
  int64_t n_rho;
};

// Peaks sharing a theta bin share their support trig (support_trig of the
// bin, hough.py:181-182): one rho bin per distinct (cos, sin) slot, then one
// compare per peak.
__device__ __forceinline__ unsigned long long member_mask(double x, double y, const PeakArgs& pk,
                                                         const float2* __restrict__ cs32,
                                                         const int* __restrict__ slot_peak,
                                                         int nslot,
                                                         const int* __restrict__ peak_slot,
                                                         const int* __restrict__ rb) {
  const float rho_max32 = (float)pk.rho_max;
  const float inv_drho32 = (float)(1.0 / pk.drho);
  int bins[64];
#pragma unroll 4
  for (int t = 0; t < nslot; ++t) {
    const int q = slot_peak[t];
    bins[t] = (int)rho_bin_fast(x, y, pk.cos_p + q, pk.sin_p + q, cs32[t].x, cs32[t].y,
                                pk.rho_max, rho_max32, pk.drho, inv_drho32, pk.n_rho);
  }
  unsigned long long m = 0ULL;
  for (int q = 0; q < pk.npeaks; ++q)
    if (bins[peak_slot[q]] == rb[q]) m |= 1ULL << q;
  return m;
}

// Pass 1: membership masks and per-(peak, block) member counts
// (counts laid out peak-major: counts[q * nblocks + block]).
__global__ void __launch_bounds__(kSupThreads)
    support_count_kernel(PointSrc src, int64_t npts, PeakArgs pk,
                         unsigned long long* __restrict__ masks,
                         int64_t* __restrict__ counts, int64_t nblocks) {
  __shared__ unsigned int cnt[64];
  __shared__ float2 cs32[64];
  __shared__ int rb[64], peak_slot[64], slot_peak[64];
  __shared__ int nslot;
  if (threadIdx.x < 64) {
    cnt[threadIdx.x] = 0u;
    if (threadIdx.x < pk.npeaks) rb[threadIdx.x] = (int)pk.rbin_p[threadIdx.x];
  }
  if (threadIdx.x == 0) {
    int ns = 0;
    for (int q = 0; q < pk.npeaks; ++q) {
      int t = 0;
      while (t < ns && !(pk.cos_p[slot_peak[t]] == pk.cos_p[q] && pk.sin_p[slot_peak[t]] == pk.sin_p[q])) ++t;
      if (t == ns) {
        slot_peak[ns] = q;
        cs32[ns] = make_float2((float)pk.cos_p[q], (float)pk.sin_p[q]);
        ++ns;
      }
      peak_slot[q] = t;
    }
    nslot = ns;
  }
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kSupChunk;
  for (int it = 0; it < kSupItems; ++it) {
    const int64_t k = base + (int64_t)it * kSupThreads + threadIdx.x;
    unsigned long long m = 0ULL;
    if (k < npts) {
      double x, y;
      src.get(k, x, y);
      m = member_mask(x, y, pk, cs32, slot_peak, nslot, peak_slot, rb);
      masks[k] = m;
    }
    while (m) {
      const int q = __ffsll((long long)m) - 1;
      atomicAdd(&cnt[q], 1u);
      m &= m - 1;
    }
  }
  __syncthreads();
  if (threadIdx.x < pk.npeaks) counts[(int64_t)threadIdx.x * nblocks + blockIdx.x] = cnt[threadIdx.x];
}

// Pass 2: ordered write of each block's members; offsets = exclusive scan of
// counts, so peak q's block b writes from offsets[q * nblocks + b].  The
// block's masks are staged in shared memory and each warp walks them in scan
// order for its share of the peaks (ballot + popc positions, no block-wide
// barriers per peak).
__global__ void __launch_bounds__(kSupThreads)
    support_write_kernel(PointSrc src, int64_t npts, const unsigned long long* __restrict__ masks,
                         const int64_t* __restrict__ offsets, int64_t nblocks, int npeaks,
                         int64_t* __restrict__ out, int64_t cap) {
  __shared__ unsigned long long sm[kSupChunk];
  __shared__ unsigned long long tile_or;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t base = (int64_t)blockIdx.x * kSupChunk;
  if (threadIdx.x == 0) tile_or = 0ULL;
  __syncthreads();
  unsigned long long orv = 0ULL;
  for (int e = threadIdx.x; e < kSupChunk; e += kSupThreads) {
    const int64_t k = base + e;
    const unsigned long long m = k < npts ? masks[k] : 0ULL;
    sm[e] = m;
    orv |= m;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) orv |= __shfl_xor_sync(0xffffffffu, orv, off);
  if (lane == 0 && orv) atomicOr(&tile_or, orv);
  __syncthreads();
  const unsigned long long todo = tile_or;
  const int64_t nvalid = npts - base < kSupChunk ? npts - base : kSupChunk;
  for (int q = warp; q < npeaks; q += kSupThreads / 32) {
    if (!((todo >> q) & 1ULL)) continue;
    int64_t pos = offsets[(int64_t)q * nblocks + blockIdx.x];
    for (int e0 = 0; e0 < nvalid; e0 += 32) {
      const int e = e0 + lane;
      const bool mine = e < nvalid && ((sm[e] >> q) & 1ULL);
      const unsigned bal = __ballot_sync(0xffffffffu, mine);
      const int64_t at = pos + __popc(bal & ((1u << lane) - 1u));
      if (mine && at < cap) out[at] = src.id(base + e);  // beyond cap: the host regrows and reruns
      pos += __popc(bal);
    }
  }
}

}  // namespace

int hough_extract(const uint8_t* d_img, int64_t npix, int threshold, int64_t* d_pix,
                  int64_t* d_count, void* temp, size_t* temp_bytes, cudaStream_t stream) {
  thrust::counting_iterator<int64_t> it(0);
  LitPixel pred{d_img, threshold};
  return cub::DeviceSelect::If(temp, *temp_bytes, it, d_pix, d_count, npix, pred, stream) ==
                 cudaSuccess
             ? 0
             : -1;
}

void hough_vote(const int64_t* d_pix, const double* d_x, const double* d_y, int64_t npts,
                int64_t width, const double* d_cos, const double* d_sin, int n_theta,
                double rho_max, double drho, int64_t n_rho, unsigned long long* d_acc, int sms,
                cudaStream_t stream) {
  const PointSrc src{d_pix, d_x, d_y, width};
  const int64_t nbins = n_rho * n_theta;
  const size_t smem = (size_t)nbins * sizeof(unsigned int);
  const int use_smem = smem <= 96 * 1024;
  if (use_smem && smem + kMaxTheta * sizeof(float2) > 40 * 1024)
    cudaFuncSetAttribute(vote_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int64_t blocks = (npts + kVoteThreads - 1) / kVoteThreads;
  if (blocks > (int64_t)sms * 4) blocks = (int64_t)sms * 4;
  if (blocks < 1) blocks = 1;
  vote_kernel<<<(unsigned)blocks, kVoteThreads, use_smem ? smem : 0, stream>>>(
      src, npts, d_cos, d_sin, n_theta, rho_max, drho, n_rho, use_smem, d_acc);
}

int64_t support_blocks(int64_t npts) { return (npts + kSupChunk - 1) / kSupChunk; }

int hough_support(const int64_t* d_pix, const double* d_x, const double* d_y, int64_t npts,
                  int64_t width, const double* d_cos, const double* d_sin, const int64_t* d_rbin,
                  int npeaks, double rho_max, double drho, int64_t n_rho,
                  unsigned long long* d_masks, int64_t* d_counts, int64_t* d_offsets, void* temp,
                  size_t temp_bytes, int64_t* d_out, int64_t out_cap, cudaStream_t stream) {
  const int64_t nb = support_blocks(npts);
  if (nb == 0 || npeaks == 0) return 0;
  const PointSrc src{d_pix, d_x, d_y, width};
  PeakArgs pk{d_cos, d_sin, d_rbin, npeaks, rho_max, drho, n_rho};
  support_count_kernel<<<(unsigned)nb, kSupThreads, 0, stream>>>(src, npts, pk, d_masks, d_counts,
                                                                 nb);
  // exclusive scan over npeaks * nb counts (+1 slot for the total)
  const int64_t m = (int64_t)npeaks * nb + 1;
  size_t bytes = temp_bytes;
  if (cub::DeviceScan::ExclusiveSum(temp, bytes, d_counts, d_offsets, m, stream) != cudaSuccess)
    return -1;
  support_write_kernel<<<(unsigned)nb, kSupThreads, 0, stream>>>(src, npts, d_masks, d_offsets,
                                                                 nb, npeaks, d_out, out_cap);
  return 0;
}

size_t support_scan_temp_bytes(int64_t m) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const int64_t*)nullptr, (int64_t*)nullptr, m);
  return bytes;
}

size_t extract_temp_bytes(int64_t npix) {
  size_t bytes = 0;
  thrust::counting_iterator<int64_t> it(0);
  LitPixel pred{nullptr, 0};
  cub::DeviceSelect::If(nullptr, bytes, it, (int64_t*)nullptr, (int64_t*)nullptr, npix, pred);
  return bytes;
}

__global__ void narrow_i32_kernel(const int64_t* __restrict__ in, int32_t* __restrict__ out,
                                  int64_t m) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m;
       k += (int64_t)gridDim.x * blockDim.x)
    out[k] = (int32_t)in[k];
}

void launch_narrow_i32(const int64_t* in, int32_t* out, int64_t m, cudaStream_t st) {
  if (m <= 0) return;
  narrow_i32_kernel<<<(int)std::min<int64_t>((m + 255) / 256, 4096), 256, 0, st>>>(in, out, m);
}

}  // namespace lmsb
