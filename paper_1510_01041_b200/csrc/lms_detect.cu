// lms_detect.cu -- detect_lines on the device, straight from the image.
//
// The reference (detect.py:156-214) extracts the lit pixels as Point2
// objects (hough.py:93-103), votes (hough.py:112-129), finds the peaks of
// the accumulator (hough.py:132-168), gathers each peak's supporting points
// in scan order (hough.py:171-184), thins each support by a stride
// (detect.py:118-131) and refits it with exact LMS (detect.py:134-153).
// Here the lit pixels are never materialised: the uint8 image (1 byte per
// pixel, read three times -- vote, support count, support write -- instead
// of a point list of 8 bytes per lit pixel written and read back) is the
// point set, a pixel's id is its row-major index, and scan order is index
// order.
//
//   vote     every lit pixel votes at each theta bin centre (rho with the
//            reference's fp64 roundings, decided through a rigorously
//            bracketed fp32 estimate -- lms_hough.cu rho_bin_fast); per-CTA
//            shared-memory histogram with warp-aggregated adds
//            (__match_any_sync: neighbouring pixels share rho bins)
//   peaks    one CTA: 8-neighbour maxima >= min_votes of the accumulator
//            (edges padded with -1), keys (-votes, rho bin, theta bin)
//            bitonic-sorted in shared memory, the first max_peaks kept
//   support  pass 1 counts each (peak, pixel chunk)'s members, one CTA
//            scans the counts into output positions, pass 2 recomputes the
//            memberships and writes every member's pixel id in scan order
//            (a lane per pixel; lanes with the same peak grouped by
//            __match_any_sync, ranked by popc) -- no per-pixel mask in HBM
//   design   per peak, the stride-thinned support (k m) // cap in the
//            axis-swapped frame, as the LMS solver's dual lines, with its
//            abscissa range (the degenerate-support check)
//
// cos/sin of the bin centres come from the host exactly as the reference
// computes them (np.cos/np.sin for the vote, math.cos/math.sin for the
// support), so the bins and supports are the reference's bit for bit.

#include <cuda_runtime.h>

#include <climits>
#include <cmath>
#include <cstdint>

#include "lms_detect.cuh"
#include "lms_hough.cuh"

namespace lmsb {

namespace {

constexpr int kVoteThreads = 256;
constexpr int kMaxTheta = 512;
constexpr int kPeakThreads = 1024;
constexpr int kSupWarps = 8;
constexpr int kSupThreads = kSupWarps * 32;

// HoughParams.rho_bin in the reference's fp64 arithmetic (hough.py:60-63,
// 124-128): two rounded products, a rounded sum, floor of the rounded
// quotient, int64 cast (out of range / NaN -> INT64_MIN -> clipped to 0).
__device__ __forceinline__ int rho_bin64(double x, double y, double c, double s, double rho_max,
                                         double drho, int n_rho) {
  const double rho = __dadd_rn(__dmul_rn(x, c), __dmul_rn(y, s));
  const double f = floor(__ddiv_rn(__dadd_rn(rho, rho_max), drho));
  if (!(f >= -9.2233720368547758e18 && f < 9.2233720368547758e18)) return 0;
  const int64_t r = (int64_t)f;
  return (int)(r < 0 ? 0 : (r > n_rho - 1 ? n_rho - 1 : r));
}

// The same bin through an fp32 estimate bracketed by its error bound; the
// fp64 form decides only within the bound of a bin edge (see lms_hough.cu).
__device__ __forceinline__ int rho_bin(double x, double y, const Trig& t, double rho_max,
                                       float rho_max32, double drho, float inv_drho32, int n_rho) {
  const float x32 = (float)x, y32 = (float)y;
  const float xc = x32 * t.c32, ys = y32 * t.s32;
  const float rho32 = xc + ys;
  const float E = 0x1p-19f * (fabsf(xc) + fabsf(ys) + fabsf(rho32) + rho_max32) + 1e-30f;
  const float glo = floorf((rho32 - E + rho_max32) * inv_drho32);
  const float ghi = floorf((rho32 + E + rho_max32) * inv_drho32);
  if (glo == ghi && fabsf(glo) < 0x1p22f) {
    const int r = (int)glo;
    return r < 0 ? 0 : (r > n_rho - 1 ? n_rho - 1 : r);
  }
  return rho_bin64(x, y, t.c, t.s, rho_max, drho, n_rho);
}

// Lit pixels of [p0, p1) appended in scan order to the warp's queue (one
// 4-byte load per lane, 128 pixels per step; a warp scan of the per-lane
// counts gives each lane its slots), and handed to `work` 32 at a time (one
// per lane, lanes >= cnt idle) -- every lane busy whatever the pixel density.
template <typename Work>
__device__ __forceinline__ void walk_lit(const DetectImage& im, int64_t p0, int64_t p1,
                                         uint32_t* q, Work&& work) {
  const int lane = threadIdx.x & 31;
  int qn = 0;
  for (int64_t base = p0; base < p1; base += 128) {
    const int64_t pl = base + 4 * lane;
    uint32_t px = 0;
    if (pl + 3 < p1 && ((pl & 3) == 0)) {
      px = *reinterpret_cast<const uint32_t*>(im.img + pl);
    } else {
      for (int e = 0; e < 4; ++e)
        if (pl + e < p1) px |= (uint32_t)im.img[pl + e] << (8 * e);
    }
    unsigned bits = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (pl + e < p1 && (int)((px >> (8 * e)) & 0xFF) >= im.threshold) bits |= 1u << e;
    const int mine = __popc(bits);
    int incl = mine;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += v;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    int at = qn + incl - mine;
    for (int e = 0; e < 4; ++e)
      if (bits & (1u << e)) q[at++] = (uint32_t)(pl + e);
    qn += total;
    __syncwarp();
    while (qn >= 32) {
      work(q[lane], 32);
      __syncwarp();
      for (int e = lane; e < qn - 32; e += 32) q[e] = q[32 + e];
      __syncwarp();
      qn -= 32;
    }
  }
  if (qn > 0) work(lane < qn ? q[lane] : 0u, qn);
  __syncwarp();
}

constexpr int kQueue = 32 + 128;  // < 32 waiting + one step's 128 pixels

__global__ void __launch_bounds__(kVoteThreads) img_vote_kernel(DetectImage im, HoughGrid g,
                                                                const double* __restrict__ cos_t,
                                                                const double* __restrict__ sin_t,
                                                                unsigned long long* __restrict__ acc,
                                                                unsigned long long* __restrict__ nlit) {
  extern __shared__ unsigned int hist[];
  __shared__ Trig trig[kMaxTheta];
  __shared__ uint32_t queue[kVoteThreads / 32][kQueue];
  const int nbins = g.n_rho * g.n_theta;
  for (int t = threadIdx.x; t < g.n_theta; t += blockDim.x)
    trig[t] = Trig{(float)cos_t[t], (float)sin_t[t], cos_t[t], sin_t[t]};
  for (int e = threadIdx.x; e < nbins; e += blockDim.x) hist[e] = 0u;
  __syncthreads();
  const float rho_max32 = (float)g.rho_max;
  const float inv_drho32 = (float)(1.0 / g.drho);
  const int lane = threadIdx.x & 31;
  const int64_t chunk = (int64_t)kSupChunkPix;
  const int64_t nchunks = (im.npix + chunk - 1) / chunk;
  unsigned lit_count = 0;
  for (int64_t ch = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; ch < nchunks;
       ch += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t p0 = ch * chunk, p1 = p0 + chunk < im.npix ? p0 + chunk : im.npix;
    walk_lit(im, p0, p1, queue[threadIdx.x >> 5], [&](uint32_t p, int cnt) {
      if (lane >= cnt) return;
      ++lit_count;
      const double x = (double)(p % im.width), y = (double)(p / im.width);
      for (int t = 0; t < g.n_theta; ++t) {
        const int r = rho_bin(x, y, trig[t], g.rho_max, rho_max32, g.drho, inv_drho32, g.n_rho);
        atomicAdd(&hist[r * g.n_theta + t], 1u);
      }
    });
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nbins; e += blockDim.x)
    if (hist[e]) atomicAdd(&acc[e], (unsigned long long)hist[e]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) lit_count += __shfl_xor_sync(0xffffffffu, lit_count, off);
  if (lane == 0 && lit_count) atomicAdd(nlit, (unsigned long long)lit_count);
}

// find_peaks (hough.py:132-168) in one CTA; keys (2^32 - 1 - votes, r, t)
// ascending = (-votes, rho bin, theta bin); bins with key ~0 are not peaks.
__global__ void __launch_bounds__(kPeakThreads) peaks_kernel(const unsigned long long* __restrict__ acc,
                                                             HoughGrid g, int64_t min_votes,
                                                             int max_peaks, int pow2,
                                                             int64_t* __restrict__ peaks,
                                                             int64_t* __restrict__ npeaks) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* key = reinterpret_cast<uint64_t*>(smem_raw);
  const int nr = g.n_rho, nt = g.n_theta, nbins = nr * nt;
  auto at = [&](int r, int t) -> long long {
    return (r < 0 || r >= nr || t < 0 || t >= nt) ? -1LL : (long long)acc[r * nt + t];
  };
  for (int b = threadIdx.x; b < pow2; b += blockDim.x) {
    uint64_t k = ~0ull;
    if (b < nbins) {
      const int r = b / nt, t = b - r * nt;
      const long long v = (long long)acc[b];
      bool keep = v >= min_votes;
      for (int dr = -1; dr <= 1 && keep; ++dr)
        for (int dt = -1; dt <= 1; ++dt)
          if ((dr || dt) && v < at(r + dr, t + dt)) keep = false;
      if (keep) k = ((uint64_t)(0xFFFFFFFFull - (uint64_t)v) << 32) | ((uint64_t)r << 16) | (uint64_t)t;
    }
    key[b] = k;
  }
  __syncthreads();
  for (int k = 2; k <= pow2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < pow2 / 2; t += blockDim.x) {
        const int lo = 2 * t - (t & (j - 1)), hi = lo + j;
        const uint64_t a = key[lo], b = key[hi];
        if ((b < a) == ((lo & k) == 0)) {
          key[lo] = b;
          key[hi] = a;
        }
      }
      __syncthreads();
    }
  }
  for (int e = threadIdx.x; e < max_peaks; e += blockDim.x) {
    const uint64_t k = e < pow2 ? key[e] : ~0ull;
    if (k != ~0ull) {
      peaks[3 * e] = (int64_t)((k >> 16) & 0xFFFF);
      peaks[3 * e + 1] = (int64_t)(k & 0xFFFF);
      peaks[3 * e + 2] = (int64_t)(0xFFFFFFFFull - (k >> 32));
    }
  }
  if (threadIdx.x == 0) {
    int m = 0;
    while (m < max_peaks && m < pow2 && key[m] != ~0ull) ++m;
    *npeaks = m;
  }
}

// Pass 1: members per (peak, chunk of kSupChunkPix pixels), peak-major.
__global__ void __launch_bounds__(kSupThreads) support_count_img_kernel(DetectImage im, HoughGrid g,
                                                                        SupportTable tb,
                                                                        int64_t nchunks,
                                                                        unsigned* __restrict__ counts) {
  __shared__ unsigned cnt[kSupWarps][64];
  __shared__ uint32_t queue[kSupWarps][kQueue];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const float rho_max32 = (float)g.rho_max;
  const float inv_drho32 = (float)(1.0 / g.drho);
  for (int64_t ch = (int64_t)blockIdx.x * kSupWarps + w; ch < nchunks;
       ch += (int64_t)gridDim.x * kSupWarps) {
    for (int q = lane; q < 64; q += 32) cnt[w][q] = 0u;
    __syncwarp();
    const int64_t p0 = ch * kSupChunkPix, p1 = p0 + kSupChunkPix < im.npix ? p0 + kSupChunkPix : im.npix;
    walk_lit(im, p0, p1, queue[w], [&](uint32_t p, int n) {
      if (lane >= n) return;
      const double x = (double)(p % im.width), y = (double)(p / im.width);
      for (int s = 0; s < tb.nslot; ++s) {
        const int r = rho_bin(x, y, tb.trig[s], g.rho_max, rho_max32, g.drho, inv_drho32, g.n_rho);
        for (int e = tb.first[s]; e < tb.first[s + 1]; ++e)
          if (tb.rbin[e] == r) atomicAdd(&cnt[w][tb.peak[e]], 1u);
      }
    });
    __syncwarp();
    for (int q = lane; q < tb.npeaks; q += 32) counts[(int64_t)q * nchunks + ch] = cnt[w][q];
    __syncwarp();
  }
}

// Positions: one CTA per peak scans its chunk counts from the peak's start
// (soffs, the prefix of the votes).
__global__ void __launch_bounds__(1024) support_scan_kernel(const unsigned* __restrict__ counts,
                                                            int64_t nch,
                                                            const int64_t* __restrict__ soffs,
                                                            int64_t* __restrict__ offs,
                                                            unsigned long long* __restrict__ bad) {
  __shared__ int64_t part[1024];
  const int q = blockIdx.x;
  const unsigned* cq = counts + (int64_t)q * nch;
  int64_t* oq = offs + (int64_t)q * nch;
  const int64_t per = (nch + 1023) / 1024;
  const int64_t b0 = threadIdx.x * per, b1 = b0 + per < nch ? b0 + per : nch;
  int64_t sum = 0;
  for (int64_t k = b0; k < b1; ++k) sum += cq[k];
  part[threadIdx.x] = sum;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    const int64_t v = threadIdx.x >= off ? part[threadIdx.x - off] : 0;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  int64_t run = soffs[q] + (threadIdx.x ? part[threadIdx.x - 1] : 0);
  for (int64_t k = b0; k < b1; ++k) {
    oq[k] = run;
    run += cq[k];
  }
  // the support of a peak is its bin's voters: sizes must equal the votes
  if (threadIdx.x == 1023 && soffs[q] + part[1023] != soffs[q + 1]) atomicAdd(bad, 1ull);
}

// Pass 2: each member's pixel id at its position, in scan order.
__global__ void __launch_bounds__(kSupThreads) support_write_img_kernel(
    DetectImage im, HoughGrid g, SupportTable tb, int64_t nchunks, const int64_t* __restrict__ offs,
    int32_t* __restrict__ out) {
  __shared__ int64_t run[kSupWarps][64];
  __shared__ uint32_t queue[kSupWarps][kQueue];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned below = (1u << lane) - 1u;
  const float rho_max32 = (float)g.rho_max;
  const float inv_drho32 = (float)(1.0 / g.drho);
  for (int64_t ch = (int64_t)blockIdx.x * kSupWarps + w; ch < nchunks;
       ch += (int64_t)gridDim.x * kSupWarps) {
    for (int q = lane; q < tb.npeaks; q += 32) run[w][q] = offs[(int64_t)q * nchunks + ch];
    __syncwarp();
    const int64_t p0 = ch * kSupChunkPix, p1 = p0 + kSupChunkPix < im.npix ? p0 + kSupChunkPix : im.npix;
    walk_lit(im, p0, p1, queue[w], [&](uint32_t p, int n) {
      const bool live = lane < n;
      const double x = (double)(p % im.width), y = (double)(p / im.width);
      for (int s = 0; s < tb.nslot; ++s) {
        int q = -1;
        if (live) {
          const int r = rho_bin(x, y, tb.trig[s], g.rho_max, rho_max32, g.drho, inv_drho32, g.n_rho);
          for (int e = tb.first[s]; e < tb.first[s + 1]; ++e)
            if (tb.rbin[e] == r) q = tb.peak[e];
        }
        if (!__any_sync(0xffffffffu, q >= 0)) continue;
        const unsigned same = __match_any_sync(0xffffffffu, q);
        int64_t base = 0;
        if (q >= 0) base = run[w][q];
        __syncwarp();
        if (q >= 0) {
          out[base + __popc(same & below)] = (int32_t)p;
          if (lane == __ffs(same) - 1) run[w][q] = base + __popc(same);
        }
        __syncwarp();
      }
    });
  }
}

// Per peak (one CTA each): the stride-thinned support as dual lines in the
// axis-swapped frame (detect.py:91-95, 118-131) and its abscissa range.
__global__ void design_kernel(const int64_t* __restrict__ peaks, const int64_t* __restrict__ npeaks_d,
                              const int64_t* __restrict__ soffs, const int32_t* __restrict__ ids,
                              int64_t width, int64_t cap, const uint8_t* __restrict__ swap_t,
                              const int64_t* __restrict__ doffs, double* __restrict__ da,
                              double* __restrict__ db, double* __restrict__ lim) {
  __shared__ double smin[32], smax[32];
  const int q = blockIdx.x;
  if (q >= (int)*npeaks_d) return;
  const int64_t m = soffs[q + 1] - soffs[q];
  const bool thin = cap > 0 && m > cap;
  const int64_t keep = thin ? cap : m;
  const bool sw = swap_t[peaks[3 * q + 1]] != 0;
  double lo = INFINITY, hi = -INFINITY;
  for (int64_t k = threadIdx.x; k < keep; k += blockDim.x) {
    const int64_t src = thin ? (k * m) / cap : k;
    const int64_t id = ids[soffs[q] + src];
    const double x = (double)(id % width), y = (double)(id / width);
    const double t = sw ? y : x, z = sw ? x : y;
    da[doffs[q] + k] = t;
    db[doffs[q] + k] = z;
    lo = fmin(lo, t);
    hi = fmax(hi, t);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, off));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, off));
  }
  if ((threadIdx.x & 31) == 0) {
    smin[threadIdx.x >> 5] = lo;
    smax[threadIdx.x >> 5] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int e = 1; e < (int)(blockDim.x >> 5); ++e) {
      lo = fmin(lo, smin[e]);
      hi = fmax(hi, smax[e]);
    }
    lim[2 * q] = lo;
    lim[2 * q + 1] = hi;
  }
}

}  // namespace

void launch_detect_vote(const DetectImage& im, const HoughGrid& g, const double* cos_t,
                        const double* sin_t, unsigned long long* acc, unsigned long long* nlit,
                        int sms, cudaStream_t st) {
  const size_t smem = (size_t)g.n_rho * g.n_theta * sizeof(unsigned);
  static DeviceOnce done;
  set_max_smem(img_vote_kernel, kDetectMaxBins * sizeof(unsigned), done);
  const int64_t nch = (im.npix + kSupChunkPix - 1) / kSupChunkPix;
  int64_t blocks = (nch + kVoteThreads / 32 - 1) / (kVoteThreads / 32);
  if (blocks > (int64_t)sms * 4) blocks = (int64_t)sms * 4;
  if (blocks < 1) blocks = 1;
  img_vote_kernel<<<(unsigned)blocks, kVoteThreads, smem, st>>>(im, g, cos_t, sin_t, acc, nlit);
}

void launch_detect_peaks(const unsigned long long* acc, const HoughGrid& g, int64_t min_votes,
                         int max_peaks, int64_t* peaks, int64_t* npeaks, cudaStream_t st) {
  int pow2 = 1;
  while (pow2 < g.n_rho * g.n_theta) pow2 <<= 1;
  static DeviceOnce done;
  set_max_smem(peaks_kernel, kDetectMaxBins * sizeof(uint64_t), done);
  peaks_kernel<<<1, kPeakThreads, (size_t)pow2 * sizeof(uint64_t), st>>>(acc, g, min_votes,
                                                                       max_peaks, pow2, peaks,
                                                                       npeaks);
}

int64_t detect_support_chunks(int64_t npix) { return (npix + kSupChunkPix - 1) / kSupChunkPix; }

void launch_detect_support(const DetectImage& im, const HoughGrid& g, const SupportTable& tb,
                           const int64_t* soffs, unsigned* counts, int64_t* offs, int32_t* out,
                           unsigned long long* bad, int sms, cudaStream_t st) {
  const int64_t nch = detect_support_chunks(im.npix);
  if (nch == 0 || tb.npeaks == 0) return;
  int64_t blocks = (nch + kSupWarps - 1) / kSupWarps;
  if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
  support_count_img_kernel<<<(unsigned)blocks, kSupThreads, 0, st>>>(im, g, tb, nch, counts);
  support_scan_kernel<<<tb.npeaks, 1024, 0, st>>>(counts, nch, soffs, offs, bad);
  support_write_img_kernel<<<(unsigned)blocks, kSupThreads, 0, st>>>(im, g, tb, nch, offs, out);
}

void launch_detect_design(const int64_t* peaks, const int64_t* npeaks_d, int npeaks,
                          const int64_t* soffs, const int32_t* ids, int64_t width, int64_t cap,
                          const uint8_t* swap_t, const int64_t* doffs, double* da, double* db,
                          double* lim, cudaStream_t st) {
  if (npeaks <= 0) return;
  design_kernel<<<npeaks, 256, 0, st>>>(peaks, npeaks_d, soffs, ids, width, cap, swap_t, doffs, da,
                                        db, lim);
}

}  // namespace lmsb
