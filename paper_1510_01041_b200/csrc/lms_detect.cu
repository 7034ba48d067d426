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

#include <algorithm>

#include "lms_detect.cuh"
#include "lms_hough.cuh"

namespace lmsb {

namespace {

constexpr int kVoteThreads = 512;
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

// Vote by row segments.  Along one image row y the reference's bin of a
// pixel at theta t, floor((fl(fl(x c) + fl(y s)) + rho_max) / d_rho) clipped,
// is monotone in x (every rounding is monotone, c and the row's y s are
// fixed), so each bin holds one contiguous x-segment of the row.  A thread
// per (row, theta) finds the segment ends -- the predicted crossing of each
// bin edge, confirmed by the exact bin of the pixels around it (a bisection
// of the remaining range when the prediction is off) -- and adds the
// segment's lit-pixel count, a popcount over the row's lit bitmask in shared
// memory.  Work per row and theta is the number of bins the row crosses, not
// the number of lit pixels; the image is read once, 1 byte per pixel.
constexpr int kVoteRows = 16;          // rows per CTA pass
constexpr int kMaxRhoEdges = 4096;     // rho bins of the row-segment vote (edge table)
constexpr int kVoteMaxWords = 4096;    // row bitmask words per CTA (width * rows / 32)

__device__ __forceinline__ int exact_bin(int64_t x, int64_t y, const Trig& t, double rho_max,
                                         float rho_max32, double drho, float inv_drho32, int n_rho) {
  return rho_bin((double)x, (double)y, t, rho_max, rho_max32, drho, inv_drho32, n_rho);
}

// lit pixels of row bitmask `bits` in [x0, x1)
__device__ __forceinline__ int lit_between(const uint32_t* bits, int64_t x0, int64_t x1) {
  if (x1 <= x0) return 0;
  int64_t w0 = x0 >> 5, w1 = (x1 - 1) >> 5;
  const uint32_t m0 = 0xFFFFFFFFu << (x0 & 31);
  const uint32_t m1 = 0xFFFFFFFFu >> (31 - ((x1 - 1) & 31));
  if (w0 == w1) return __popc(bits[w0] & m0 & m1);
  int c = __popc(bits[w0] & m0) + __popc(bits[w1] & m1);
  for (int64_t w = w0 + 1; w < w1; ++w) c += __popc(bits[w]);
  return c;
}

// wedge[b] (1 <= b <= n_rho - 1): the smallest double w with fl(w / d_rho) >=
// b, so floor(fl(w / d_rho)) >= b -- a pixel's bin is >= b exactly when its
// w = fl(fl(fl(x c) + fl(y s)) + rho_max) reaches wedge[b] (the clip to
// [0, n_rho - 1] agrees for every such b); wedge[0] = -inf.
__global__ void wedge_kernel(HoughGrid g, double* __restrict__ wedge) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < g.n_rho; b += gridDim.x * blockDim.x) {
    if (b == 0) {
      wedge[0] = -INFINITY;
      continue;
    }
    double w = __dmul_rn((double)b, g.drho);
    while (!(__ddiv_rn(w, g.drho) >= (double)b)) w = nextafter(w, INFINITY);
    for (;;) {
      const double wp = nextafter(w, -INFINITY);
      if (__ddiv_rn(wp, g.drho) >= (double)b) w = wp;
      else break;
    }
    wedge[b] = w;
  }
}

__global__ void __launch_bounds__(kVoteThreads) img_vote_kernel(DetectImage im, HoughGrid g,
                                                                const double* __restrict__ cos_t,
                                                                const double* __restrict__ sin_t,
                                                                const double* __restrict__ wedge_g,
                                                                uint32_t* __restrict__ bits_g,
                                                                unsigned long long* __restrict__ acc,
                                                                unsigned long long* __restrict__ nlit) {
  extern __shared__ unsigned int hist[];
  __shared__ Trig trig[kMaxTheta];
  __shared__ uint32_t rowbits[kVoteMaxWords];
  const int nbins = g.n_rho * g.n_theta;
  double* wedge = reinterpret_cast<double*>(hist + ((nbins + 1) & ~1));  // after the histogram
  for (int b = threadIdx.x; b < g.n_rho; b += blockDim.x) wedge[b] = wedge_g[b];
  for (int t = threadIdx.x; t < g.n_theta; t += blockDim.x)
    trig[t] = Trig{(float)cos_t[t], (float)sin_t[t], cos_t[t], sin_t[t],
                   cos_t[t] != 0.0 ? 1.0 / cos_t[t] : 0.0};
  for (int e = threadIdx.x; e < nbins; e += blockDim.x) hist[e] = 0u;
  const float rho_max32 = (float)g.rho_max;
  const float inv_drho32 = (float)(1.0 / g.drho);
  const int64_t W = im.width, H = im.npix / im.width;
  const int wpr = (int)((W + 31) >> 5);  // bitmask words per row
  const int rows = kVoteMaxWords / wpr < kVoteRows ? kVoteMaxWords / wpr : kVoteRows;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned lit_count = 0;
  for (int64_t y0 = (int64_t)blockIdx.x * rows; y0 < H; y0 += (int64_t)gridDim.x * rows) {
    const int nr = (int)(H - y0 < rows ? H - y0 : rows);
    __syncthreads();  // (also orders the histogram clear before the first adds)
    // lit bitmasks of the rows
    if ((W & 15) == 0) {
      // 16 pixels per lane (one 16-byte load), 512 per warp step; two lanes per word
      const int spr = (int)(W / 512 + ((W & 511) ? 1 : 0));  // warp steps per row
      for (int wi = warp; wi < nr * spr; wi += kVoteThreads / 32) {
        const int r = wi / spr, st = wi - r * spr;
        const int64_t x = (int64_t)st * 512 + 16 * lane;
        uint32_t m16 = 0;
        if (x < W) {
          const uint4 v = *reinterpret_cast<const uint4*>(im.img + (y0 + r) * W + x);
          const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int e = 0; e < 16; ++e)
            if ((int)((w4[e >> 2] >> (8 * (e & 3))) & 0xFF) >= im.threshold) m16 |= 1u << e;
        }
        const uint32_t hi = __shfl_down_sync(0xffffffffu, m16, 1);
        if (!(lane & 1) && x < W) {
          const uint32_t word = m16 | (hi << 16);
          rowbits[r * wpr + (int)(x >> 5)] = word;
          bits_g[(y0 + r) * wpr + (x >> 5)] = word;
          lit_count += __popc(word);
        }
      }
    } else {
      // a warp ballots 32 consecutive pixels per word
      for (int wi = warp; wi < nr * wpr; wi += kVoteThreads / 32) {
        const int r = wi / wpr, w = wi - r * wpr;
        const int64_t x = (int64_t)w * 32 + lane;
        const bool lit = x < W && (int)im.img[(y0 + r) * W + x] >= im.threshold;
        const uint32_t word = __ballot_sync(0xffffffffu, lit);
        if (lane == 0) {
          rowbits[wi] = word;
          bits_g[(y0 + r) * wpr + w] = word;
          lit_count += __popc(word);
        }
      }
    }
    __syncthreads();
    // a warp per (row, theta): lane k finds the k-th bin change of the row
    for (int task = warp; task < nr * g.n_theta; task += kVoteThreads / 32) {
      const int r = task / g.n_theta, t = task - r * g.n_theta;
      const int64_t y = y0 + r;
      const uint32_t* bits = rowbits + r * wpr;
      const Trig& tr = trig[t];
      auto bin_at = [&](int64_t x) {
        return exact_bin(x, y, tr, g.rho_max, rho_max32, g.drho, inv_drho32, g.n_rho);
      };
      const int b0 = bin_at(0), b1 = bin_at(W - 1);
      const int dir = b1 >= b0 ? 1 : -1;
      const int T = (b1 - b0) * dir;  // bin changes along the row
      const double ys = __dmul_rn((double)y, tr.s);
      const int Wi = (int)W;
      // w(x) = fl(fl(fl(x c) + fl(y s)) + rho_max): bin(x) >= b  <=>  w(x) >= wedge[b]
      auto wof = [&](int x) { return __dadd_rn(__dadd_rn(__dmul_rn((double)x, tr.c), ys), g.rho_max); };
      int64_t carry = 0;  // start of the segment of bin b0 + dir * k0 (k0 = first k of this round)
      for (int k0 = 0; k0 <= T; k0 += 32) {
        const int k = k0 + lane;  // this lane: the segment of bin b0 + dir * k, [x_k, x_{k+1})
        // x_{k+1}: smallest x whose bin is beyond b0 + dir * k (W when k == T)
        int64_t xe = W;
        if (k < T) {
          const int target = b0 + dir * (k + 1);
          // up: bin >= target <=> w >= wedge[target]; down: bin <= target <=> w < wedge[target + 1]
          const double wt = dir > 0 ? wedge[target] : wedge[target + 1];
          auto beyond = [&](int x) { return dir > 0 ? wof(x) >= wt : wof(x) < wt; };
          // predicted crossing (real arithmetic), then the exact test walks to
          // it: beyond(W - 1) holds, beyond(0) does not
          const double xp = (wt - g.rho_max - ys) * tr.ic;
          int x = (xp == xp && fabs(xp) < 1.0e9) ? (int)fmin(fmax(ceil(xp), 1.0), (double)(Wi - 1))
                                                 : Wi / 2;
          int steps = 0;
          if (beyond(x)) {
            while (x > 1 && steps < 4 && beyond(x - 1)) {
              --x;
              ++steps;
            }
          } else {
            while (steps < 4 && !beyond(x)) {
              ++x;
              ++steps;
            }
          }
          if (steps == 4) {  // prediction off: bisection over the row
            int lo = 1, hi = Wi - 1;
            while (lo < hi) {
              const int mid = (lo + hi) >> 1;
              if (beyond(mid)) hi = mid;
              else lo = mid + 1;
            }
            x = lo;
          }
          xe = x;
        }
        int64_t xs = __shfl_up_sync(0xffffffffu, xe, 1);
        if (lane == 0) xs = carry;
        carry = __shfl_sync(0xffffffffu, xe, 31);
        if (k <= T) {
          const int cnt = lit_between(bits, xs, xe);
          if (cnt) atomicAdd(&hist[(b0 + dir * k) * g.n_theta + t], (unsigned)cnt);
        }
      }
    }
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
  // local maxima >= min_votes appended (any order), then only they are sorted
  __shared__ int ncand;
  if (threadIdx.x == 0) ncand = 0;
  __syncthreads();
  for (int b = threadIdx.x; b < nbins; b += blockDim.x) {
    const int r = b / nt, t = b - r * nt;
    const long long v = (long long)acc[b];
    bool keep = v >= min_votes;
    for (int dr = -1; dr <= 1 && keep; ++dr)
      for (int dt = -1; dt <= 1; ++dt)
        if ((dr || dt) && v < at(r + dr, t + dt)) keep = false;
    if (keep)
      key[atomicAdd(&ncand, 1)] =
          ((uint64_t)(0xFFFFFFFFull - (uint64_t)v) << 32) | ((uint64_t)r << 16) | (uint64_t)t;
  }
  __syncthreads();
  const int m = ncand;
  int p2 = 1;
  while (p2 < m) p2 <<= 1;
  for (int e = m + threadIdx.x; e < p2; e += blockDim.x) key[e] = ~0ull;
  __syncthreads();
  for (int k = 2; k <= p2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < p2 / 2; t += blockDim.x) {
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
    const uint64_t k = e < m ? key[e] : ~0ull;
    if (k != ~0ull) {
      peaks[3 * e] = (int64_t)((k >> 16) & 0xFFFF);
      peaks[3 * e + 1] = (int64_t)(k & 0xFFFF);
      peaks[3 * e + 2] = (int64_t)(0xFFFFFFFFull - (k >> 32));
    }
  }
  if (threadIdx.x == 0) *npeaks = m < max_peaks ? m : max_peaks;
}

// Support by row segments.  On row y a peak's members are the lit pixels
// whose exact bin at the peak's theta (support trig) is the peak's rho bin;
// the bin is monotone in x, so they form one x-segment [xa, xb) of the row,
// whose ends are found exactly from the bin-edge table (the predicted
// crossing, confirmed by the pixels around it; bisection otherwise), and
// the members are the set bits of the row's lit bitmask (written by the
// vote) in that segment.  A lane per (peak, row): no per-pixel arithmetic,
// the image is not read again.  Rows in order, bits in order: scan order.
struct StripArgs {
  int64_t W, H, wpr;
  HoughGrid g;
  SupportTable tb;
  const double* wedge;
  const uint32_t* bits;
};

// first x in [0, W] with pred(x) (pred monotone false -> true; W: none)
template <typename Pred>
__device__ __forceinline__ int64_t first_true(int64_t W, double xp, Pred pred) {
  if (pred(0)) return 0;
  if (!pred(W - 1)) return W;
  if (xp == xp && fabs(xp) < 4.0e18) {
    const int64_t xg = (int64_t)fmin(fmax(ceil(xp), 1.0), (double)(W - 1));
    for (int d = 0; d <= 2; ++d) {
      const int64_t c0 = xg - d, c1 = xg + d;
      if (c0 >= 1 && c0 <= W - 1 && pred(c0) && !pred(c0 - 1)) return c0;
      if (d && c1 >= 1 && c1 <= W - 1 && pred(c1) && !pred(c1 - 1)) return c1;
    }
  }
  int64_t lo = 1, hi = W - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (pred(mid)) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

// the member segment [xa, xb) of table entry e on row y
__device__ __forceinline__ void member_segment(const StripArgs& sa, int slot, int e, int64_t y,
                                               int64_t* xa, int64_t* xb) {
  const Trig& tr = sa.tb.trig[slot];
  const int rb = sa.tb.rbin[e];
  const double ys = __dmul_rn((double)y, tr.s);
  auto w_at = [&](int64_t x) { return __dadd_rn(__dadd_rn(__dmul_rn((double)x, tr.c), ys), sa.g.rho_max); };
  const bool top = rb + 1 >= sa.g.n_rho;
  const double wlo = sa.wedge[rb];                      // bin >= rb  <=>  w >= wlo (rb >= 1)
  const double whi = top ? INFINITY : sa.wedge[rb + 1];  // bin >= rb + 1  <=>  w >= whi
  const double inv_c = tr.ic;
  if (tr.c >= 0.0) {  // bins non-decreasing in x
    *xa = rb == 0 ? 0 : first_true(sa.W, (wlo - sa.g.rho_max - ys) * inv_c, [&](int64_t x) { return w_at(x) >= wlo; });
    *xb = top ? sa.W : first_true(sa.W, (whi - sa.g.rho_max - ys) * inv_c, [&](int64_t x) { return w_at(x) >= whi; });
  } else {  // bins non-increasing in x
    *xa = top ? 0 : first_true(sa.W, (whi - sa.g.rho_max - ys) * inv_c, [&](int64_t x) { return w_at(x) < whi; });
    *xb = rb == 0 ? sa.W : first_true(sa.W, (wlo - sa.g.rho_max - ys) * inv_c, [&](int64_t x) { return w_at(x) < wlo; });
  }
  if (*xb < *xa) *xb = *xa;
}

// Pass 1: members per (peak, row), peak-major (counts[q * H + y]); table
// entry e = blockIdx.y, a lane per row.
__global__ void __launch_bounds__(kSupThreads) support_count_img_kernel(StripArgs sa,
                                                                        unsigned* __restrict__ counts) {
  const int e = blockIdx.y;
  int slot = 0;
  while (sa.tb.first[slot + 1] <= e) ++slot;
  for (int64_t y = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; y < sa.H;
       y += (int64_t)gridDim.x * blockDim.x) {
    int64_t xa, xb;
    member_segment(sa, slot, e, y, &xa, &xb);
    counts[(int64_t)sa.tb.peak[e] * sa.H + y] = (unsigned)lit_between(sa.bits + y * sa.wpr, xa, xb);
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
__global__ void __launch_bounds__(kSupThreads) support_write_img_kernel(StripArgs sa,
                                                                        const int64_t* __restrict__ offs,
                                                                        int32_t* __restrict__ out) {
  const int e = blockIdx.y;
  int slot = 0;
  while (sa.tb.first[slot + 1] <= e) ++slot;
  for (int64_t y = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; y < sa.H;
       y += (int64_t)gridDim.x * blockDim.x) {
    int64_t xa, xb;
    member_segment(sa, slot, e, y, &xa, &xb);
    int64_t pos = offs[(int64_t)sa.tb.peak[e] * sa.H + y];
    const uint32_t* bits = sa.bits + y * sa.wpr;
    for (int64_t w = xa >> 5; w < xb && (w << 5) < xb; ++w) {
      uint32_t m = bits[w];
      const int64_t base = w << 5;
      if (base < xa) m &= 0xFFFFFFFFu << (xa - base);
      if (base + 32 > xb) m &= 0xFFFFFFFFu >> (base + 32 - xb);
      while (m) {
        const int bit = __ffs(m) - 1;
        m &= m - 1;
        out[pos++] = (int32_t)(y * sa.W + base + bit);
      }
    }
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
                        const double* sin_t, double* wedge, uint32_t* bits, unsigned long long* acc,
                        unsigned long long* nlit, int sms, cudaStream_t st) {
  wedge_kernel<<<(g.n_rho + 255) / 256, 256, 0, st>>>(g, wedge);
  const size_t smem = (size_t)((g.n_rho * g.n_theta + 1) & ~1) * sizeof(unsigned) +
                      (size_t)g.n_rho * sizeof(double);
  static DeviceOnce done;
  set_max_smem(img_vote_kernel, kDetectMaxBins * sizeof(unsigned) + kMaxRhoEdges * sizeof(double), done);
  const int64_t H = im.width > 0 ? im.npix / im.width : 0;
  const int64_t wpr = (im.width + 31) / 32;
  const int64_t rows = std::max<int64_t>(1, std::min<int64_t>(kVoteRows, kVoteMaxWords / wpr));
  int64_t blocks = (H + rows - 1) / rows;
  if (blocks > (int64_t)sms * 4) blocks = (int64_t)sms * 4;
  if (blocks < 1) blocks = 1;
  img_vote_kernel<<<(unsigned)blocks, kVoteThreads, smem, st>>>(im, g, cos_t, sin_t, wedge, bits, acc,
                                                                nlit);
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

int64_t detect_support_rows(int64_t npix, int64_t width) { return width > 0 ? npix / width : 0; }

void launch_detect_support(const DetectImage& im, const HoughGrid& g, const SupportTable& tb,
                           const double* wedge, const uint32_t* bits, const int64_t* soffs,
                           unsigned* counts, int64_t* offs, int32_t* out, unsigned long long* bad,
                           int sms, cudaStream_t st) {
  const int64_t H = im.width > 0 ? im.npix / im.width : 0;
  if (H == 0 || tb.npeaks == 0) return;
  const StripArgs sa{im.width, H, (im.width + 31) / 32, g, tb, wedge, bits};
  const dim3 grid((unsigned)((H + kSupThreads - 1) / kSupThreads), (unsigned)tb.npeaks);
  support_count_img_kernel<<<grid, kSupThreads, 0, st>>>(sa, counts);
  support_scan_kernel<<<tb.npeaks, 1024, 0, st>>>(counts, H, soffs, offs, bad);
  support_write_img_kernel<<<grid, kSupThreads, 0, st>>>(sa, offs, out);
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
