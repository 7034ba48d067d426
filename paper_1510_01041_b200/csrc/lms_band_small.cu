// lms_band_small.cu -- the slope-band search fused into one CTA per fit, for
// batches of small fits (n <= 1,024: the Hough-peak refinement workload,
// detect.py:118-153 / the per-peak loop of detect.py:184-213, config 4).
//
// Same mathematics as lms_band.cu (read its header for the geometry and the
// error budget); everything of one fit lives in the CTA's shared memory:
//   lines     fp64 (a, b) and fp32 (a - c, b)
//   bands     K slope bands (64 or 128) from 16 K stratified slope samples;
//             per inner band the keys m_k = fl32((a_k - c) uM - b_k) sorted
//             by one warp (bitonic network in registers, 8-32 keys per lane)
//             and the lower bound W_q - 2 D_max - 2 E_max
//   seeds     the samples of the two bands with the narrowest W_q, exact
//             (warp per vertex, lms_exact_warp.cuh) -> H
//   sweep     the admitted bands (bound <= H) get shared-memory key slots;
//             every vertex of the fit is visited once per slot group: an fp32
//             slope from the reference's fp64 differences picks its band
//             (vertices within 2^-18 of a band boundary are admitted without
//             the band bound, the padded test itself holds for any slope);
//             padded window counts by binary search in the band's keys;
//             passing vertices are queued per warp and counted 32 at a time
//             in fp32 at their own slope; those still passing are evaluated
//             exactly by the warp, tightening H (shared atomicMin)
//   reduce    lexicographic (height, i, j) minimum of the warps' records.
// Vertices of the outer bands (beyond the sample range) and fits whose
// magnitudes leave the fp32 range skip the band tests (straight to the fp32
// counts / the exact select).  No global scratch; one launch per batch.
//
// Extra error terms of the fp32 slope (|u32 - u| <= 2^-21 |u| from the fp32
// division of the rounded fp64 differences): z and the keys are formed from
// u32, which moves every line's offset by <= dev * 2^-21 |u|; E below adds
// 2^-19 (dev + amax) |u| for it.

#include <cub/block/block_radix_sort.cuh>
#include <cuda_runtime.h>

#include <cfloat>
#include <cmath>
#include <cstdint>

#include "lms_band_small.cuh"
#include "lms_common.cuh"
#include "lms_exact_warp.cuh"

namespace lmsb {

namespace {

#ifndef LMSB_SMALL_AB
#define LMSB_SMALL_AB 1
#endif
#ifndef LMSB_SMALL_BAND_VERTS
#define LMSB_SMALL_BAND_VERTS 512
#endif
#ifndef LMSB_SMALL_MINB
#define LMSB_SMALL_MINB 2
#endif
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
#ifndef LMSB_SMALL_MAX_BANDS
#define LMSB_SMALL_MAX_BANDS 128
#endif
constexpr int kMaxBands = LMSB_SMALL_MAX_BANDS;
constexpr int kSamplesPerBand = 16;
constexpr int kSamples = kMaxBands * kSamplesPerBand;  // 2,048
constexpr int kSampleItems = kSamples / kThreads;
constexpr int kSeedsPerBand = 16;
constexpr int kSeedBands = 2;
constexpr int kEdge = 5;  // keys kept around each end of a band's narrowest q-window
#ifndef LMSB_SMALL_SLOTS
#define LMSB_SMALL_SLOTS 16
#endif
constexpr int kSlots = LMSB_SMALL_SLOTS;  // admitted bands whose keys are resident at once
constexpr int kSegRun = 16;   // ranks per lane per warp segment
#ifndef LMSB_SMALL_STEP
#define LMSB_SMALL_STEP 4
#endif
constexpr int kSweepStep = LMSB_SMALL_STEP; // vertices per lane per sweep step
constexpr int kQueue = 32 * (kSweepStep + 1);  // per-warp queues: < 32 waiting + a step
static_assert(kSegRun % kSweepStep == 0, "whole sweep steps per segment");
constexpr int kMaxRuns = 8;   // slope runs tested before a band lookup (a 3-step search)
static_assert(kMaxRuns == 8, "the sweep's run search takes 3 steps");

template <int kItems, int kT = kThreads>
struct SmallShared {
  static constexpr int kNP = 32 * kItems;  // padded lines (one warp sorts a band)
  static constexpr int kWarps = kT / 32;
  static constexpr int kSampleItems = kSamples / kT;
  using SampleSort = cub::BlockRadixSort<float, kT, kSampleItems, int>;
  alignas(16) double a[kNP];
  alignas(16) double b[kNP];
#if LMSB_SMALL_AB
  double2 ab[kNP];            // (a_k, b_k) interleaved for the sweeps
#endif
  float4 l2[kNP / 2];         // (A_k, A_k+1, -B_k, -B_k+1) for the packed counts
  float rlo[kMaxRuns], rhi[kMaxRuns];  // slope runs of the current sweep (widened)
  int nruns;
  // phase-disjoint storage: the bound phase sorts into wkeys, the seeds and
  // sweeps select with sw; the samples live until the seeds, the admitted
  // bands' keys (slots) only in the sweeps
  union {
    float wkeys[kWarps][kNP];   // per-warp sort output (bound phase)
    SelectWarp sw[kWarps];      // exact select state (seeds, sweeps)
  };
  union {
    struct {
      union {
        typename SampleSort::TempStorage ssort;
        struct {
          float skey[kSamples];
          int sidx[kSamples];
        } s;
      };
    };
    float slot[kSlots][kNP];    // resident keys of admitted bands (sweeps)
  };
  float bounds[kMaxBands - 1];
  double lb[kMaxBands], um[kMaxBands], wq[kMaxBands];
  double slb[kMaxBands];  // slope bound of every band (keyless ones: dismissal test)
  double wqa;             // lower bound of the narrowest q-window of the slopes a_k
  float edge[kMaxBands][2 * 5];  // keys around the ends of each band's narrowest q-window
  int egrp[2][16];               // edge-seed line groups
  int negrp[2];
  int16_t band_slot[kMaxBands];
  int admitted[kMaxBands];
  int nadmitted;
  int seed_band[kSeedBands];
  uint32_t queue[kWarps][kQueue];   // fp32-count queue
  uint32_t squeue[kWarps][kQueue];  // in-run vertices awaiting band lookup + padded counts
  lms_candidate wbest[kWarps];
  double red[2][kWarps];
  unsigned long long hbits;  // current bound H (bits of a non-negative double)
  uint64_t bar;              // mbarrier of the line bulk copies
  int nvalid;
  unsigned long long cnt[12];  // admitted bands, queued, exact, sweeps; phase cycles (stats)
};

// cnt += (x <= w), unsigned: one compare and one predicated add
__device__ __forceinline__ void count_le(unsigned& cnt, uint32_t x, uint32_t w) {
  asm("{\n .reg .pred p;\n setp.le.u32 p, %1, %2;\n @p add.u32 %0, %0, 1;\n}\n"
      : "+r"(cnt)
      : "r"(x), "r"(w));
}

__device__ __forceinline__ float rcp_approx_ftz(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ float band_key(double u) {
  const float f = (float)u;
  return fminf(fmaxf(f, -FLT_MAX), FLT_MAX);
}

__device__ __forceinline__ int band_of(const float* __restrict__ bnd, int nb, float key) {
  int lo = 0, hi = nb;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (bnd[mid] <= key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ int lower_idx(const float* __restrict__ k, int n, float x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (k[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ int upper_idx(const float* __restrict__ k, int n, float x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (k[mid] <= x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ void advance_pair(int n, int step, int& i, int& j) {
  j += step;
  while (j >= n && i < n - 2) {
    const int over = j - n;
    ++i;
    j = i + 1 + over;
  }
}

template <int kItems, int kT>
__device__ __forceinline__ double block_min(double v, SmallShared<kItems, kT>& sh, int slot) {
  constexpr int kWarps = kT / 32;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, off));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh.red[slot][threadIdx.x >> 5] = v;
  __syncthreads();
  double r = sh.red[slot][0];
#pragma unroll
  for (int w = 1; w < kWarps; ++w) r = fmin(r, sh.red[slot][w]);
  return r;
}

__device__ __forceinline__ double current_h(const volatile unsigned long long* hb) {
  return __longlong_as_double((long long)*hb);
}

// Ascending bitonic sort of 32 * kItems keys held blocked by one warp (lane l
// owns elements [l * kItems, (l + 1) * kItems)).
template <int kItems>
__device__ __forceinline__ void warp_bitonic_sort(float (&x)[kItems]) {
  const int lane = threadIdx.x & 31;
  constexpr int kN = 32 * kItems;
#pragma unroll
  for (int k = 2; k <= kN; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= kItems) {
        const int lm = j / kItems;
        const bool lower = (lane & lm) == 0;
#pragma unroll
        for (int e = 0; e < kItems; ++e) {
          const int i = lane * kItems + e;
          const float y = __shfl_xor_sync(0xffffffffu, x[e], lm);
          const bool asc = (i & k) == 0;
          x[e] = (lower == asc) ? fminf(x[e], y) : fmaxf(x[e], y);
        }
      } else {
#pragma unroll
        for (int e = 0; e < kItems; ++e) {
          const int p = e ^ j;
          if (p > e) {
            const int i = lane * kItems + e;
            const bool asc = (i & k) == 0;
            const float lo = fminf(x[e], x[p]), hi = fmaxf(x[e], x[p]);
            x[e] = asc ? lo : hi;
            x[p] = asc ? hi : lo;
          }
        }
      }
    }
  }
}

// keys of band `band` at its centre uM, sorted by the calling warp into dst
template <int kItems, int kT>
__device__ __forceinline__ void band_keys_warp(const SmallShared<kItems, kT>& sh, int n, double c,
                                               double uM, float* dst) {
  const int lane = threadIdx.x & 31;
  float x[kItems];
#pragma unroll
  for (int e = 0; e < kItems; ++e) {
    const int l = lane * kItems + e;
    x[e] = l < n ? (float)__dsub_rn(__dmul_rn(__dsub_rn(sh.a[l], c), uM), sh.b[l]) : INFINITY;
  }
  warp_bitonic_sort<kItems>(x);
#pragma unroll
  for (int e = 0; e < kItems; ++e) dst[lane * kItems + e] = x[e];
  __syncwarp();
}

template <int kItems, int kT>
__global__ void __launch_bounds__(kT, kT == kThreads ? LMSB_SMALL_MINB : 1) small_fit_kernel(SmallArgs args) {
  using SH = SmallShared<kItems, kT>;
  constexpr int kThreads = kT;  // this instance's CTA size (the file-scope default is 256)
  constexpr int kWarps = kT / 32;
  constexpr int kSampleItems = kSamples / kT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SH& sh = *reinterpret_cast<SH*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int fit = args.list[blockIdx.x];
  const FitDesc fd = args.fits[fit];
  const int n = (int)fd.n, q = (int)fd.q;
  const double* ga = args.a + fd.off;
  const double* gb = args.b + fd.off;
  const int64_t P = (int64_t)n * (n - 1) / 2;
  const int K = (int)min((int64_t)kMaxBands, max((int64_t)16, P / LMSB_SMALL_BAND_VERTS));

  // ---- lines, centre, magnitudes
  double alo = INFINITY, ahi = -INFINITY, am = 0.0, bm = 0.0;
  // the fit's lines: TMA bulk copies when 16-byte aligned (even n, aligned
  // offset), element loads otherwise
  const bool bulk = ((reinterpret_cast<uintptr_t>(ga) | reinterpret_cast<uintptr_t>(gb)) & 15) == 0 &&
                    (n & 1) == 0;
  if (bulk) {
    if (tid == 0) mbar_init(&sh.bar, 1);
    __syncthreads();
    if (tid == 0) {
      mbar_expect_tx(&sh.bar, 2u * 8u * (uint32_t)n);
      bulk_g2s(sh.a, ga, 8u * (uint32_t)n, &sh.bar);
      bulk_g2s(sh.b, gb, 8u * (uint32_t)n, &sh.bar);
    }
    mbar_wait(&sh.bar, 0);
  }
  for (int k = tid; k < n; k += kThreads) {
    const double ak = bulk ? sh.a[k] : ga[k], bk = bulk ? sh.b[k] : gb[k];
    if (!bulk) {
      sh.a[k] = ak;
      sh.b[k] = bk;
    }
#if LMSB_SMALL_AB
    sh.ab[k] = make_double2(ak, bk);
#endif
    alo = fmin(alo, ak);
    ahi = fmax(ahi, ak);
    am = fmax(am, fabs(ak));
    bm = fmax(bm, fabs(bk));
  }
  alo = block_min<kItems>(alo, sh, 0);
  ahi = -block_min<kItems>(-ahi, sh, 1);
  am = -block_min<kItems>(-am, sh, 0);
  bm = -block_min<kItems>(-bm, sh, 1);
  const double c = 0.5 * alo + 0.5 * ahi;
  const double dev = fmax(ahi - c, c - alo) * (1.0 + 0x1p-40) + 1e-300;
  for (int p2 = tid; p2 < SH::kNP / 2; p2 += kThreads) {
    const int k = 2 * p2;
    float4 r = make_float4(0.f, 0.f, __int_as_float(0x7fc00000), __int_as_float(0x7fc00000));
    if (k < n) {
      r.x = (float)__dsub_rn(sh.a[k], c);
      r.z = -(float)sh.b[k];
    }
    if (k + 1 < n) {
      r.y = (float)__dsub_rn(sh.a[k + 1], c);
      r.w = -(float)sh.b[k + 1];
    }
    sh.l2[p2] = r;
  }
  if (tid == 0) {
    sh.hbits = (unsigned long long)__double_as_longlong(INFINITY);
    sh.nvalid = 0;
    sh.nadmitted = 0;
    for (int t = 0; t < 12; ++t) sh.cnt[t] = 0;
  }
  lms_candidate mybest = cand_none();
  __syncthreads();
  // magnitudes the fp32 stages cannot represent: every vertex goes exact
  const bool huge = !(am < 1e30) || !(bm < 1e30) || (am > 0.0 && am < 1e-30) ||
                    (bm > 0.0 && bm < 1e-30);

  // ---- slope samples -> K - 1 band boundaries
  const int64_t S = P < K * kSamplesPerBand ? P : K * kSamplesPerBand;
  {
    float k_[kSampleItems];
    int s_[kSampleItems];
    int nv = 0;
#pragma unroll
    for (int e = 0; e < kSampleItems; ++e) {
      const int s = e * kThreads + tid;
      float key = INFINITY;
      if (s < S) {
        int64_t i, j;
        decode_rank(n, ((2 * (int64_t)s + 1) * P) / (2 * S), &i, &j);
        const double da = __dsub_rn(sh.a[i], sh.a[j]);
        if (da != 0.0) {
          const double u = __ddiv_rn(__dsub_rn(sh.b[i], sh.b[j]), da);
          if (isfinite(u) && fabs(u) * am < 1e30) {
            key = band_key(u);
            ++nv;
          }
        }
      }
      k_[e] = key;
      s_[e] = s;
    }
    nv = __reduce_add_sync(0xffffffffu, nv);
    if (lane == 0) atomicAdd(&sh.nvalid, nv);
    typename SH::SampleSort(sh.ssort).Sort(k_, s_);
    __syncthreads();
#pragma unroll
    for (int e = 0; e < kSampleItems; ++e) {
      sh.s.skey[tid * kSampleItems + e] = k_[e];
      sh.s.sidx[tid * kSampleItems + e] = s_[e];
    }
    __syncthreads();
    const int sv = sh.nvalid;
    for (int t = tid; t < K - 1; t += kThreads) {
      float v = INFINITY;
      if (sv > 0) {
        if (t == 0) v = sh.s.skey[0];
        else if (t == K - 2) v = nextafterf(sh.s.skey[sv - 1], INFINITY);
        else v = sh.s.skey[(t * sv) / (K - 2)];
      }
      sh.bounds[t] = v;
    }
    __syncthreads();
  }

  // W_q of the slopes a_k (one warp sorts the centred slopes in fp32; each
  // rounding moves a slope by <= 2^-24 dev): the slope bound |u| W_q(a) -
  // 2 bmax of every band (lms_band.cu slope_lb)
  if (warp == 0) {
    float x[kItems];
#pragma unroll
    for (int e = 0; e < kItems; ++e) {
      const int l = lane * kItems + e;
      x[e] = l < n ? (float)__dsub_rn(sh.a[l], c) : INFINITY;
    }
    warp_bitonic_sort<kItems>(x);
#pragma unroll
    for (int e = 0; e < kItems; ++e) sh.wkeys[0][lane * kItems + e] = x[e];
    __syncwarp();
    double w = INFINITY;
    for (int l = lane; l + q - 1 < n; l += 32)
      w = fmin(w, (double)sh.wkeys[0][l + q - 1] - (double)sh.wkeys[0][l]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) w = fmin(w, __shfl_xor_sync(0xffffffffu, w, off));
    if (lane == 0) sh.wqa = isfinite(w) ? fmax(w - 0x1p-22 * dev, 0.0) : 0.0;
  }
  __syncthreads();
  auto slope_bound = [&](int k) -> double {
    const double lo = k > 0 ? (double)sh.bounds[k - 1] : -INFINITY;
    const double hi = k < K - 1 ? (double)sh.bounds[k] : INFINITY;
    double umin;
    if (lo > 0.0) umin = lo;
    else if (hi < 0.0) umin = -hi;
    else return -INFINITY;
    umin *= 1.0 - 0x1p-20;
    const double slope = sh.wqa * (1.0 - 0x1p-40) - 0x1p-40 * am;
    if (!(slope > 0.0) || !isfinite(umin) || huge) return -INFINITY;
    return umin * slope * (1.0 - 0x1p-40) - 2.0 * bm * (1.0 + 0x1p-38) - 1e-300;
  };

  long long t_mark = clock64();
  if (tid == 0) sh.cnt[4] = 0;
  // ---- per inner band (one warp each): sorted keys at the centre, lower bound
  for (int k = warp; k < K; k += kWarps) {
    double uL = 0.0, uR = 0.0;
    bool ok = !huge && k > 0 && k < K - 1;
    if (ok) {
      uL = (double)nextafterf(sh.bounds[k - 1], -INFINITY);
      uR = (double)sh.bounds[k];
      ok = isfinite(uL) && isfinite(uR) && uL <= uR &&
           fmax(fabs(uL), fabs(uR)) * dev + bm < 1e37;
    }
    if (!ok) {
      if (lane == 0) {
        sh.lb[k] = -INFINITY;  // no keys: members go straight to the fp32 counts
        sh.wq[k] = INFINITY;
        sh.um[k] = NAN;
        sh.slb[k] = slope_bound(k);  // (unless the slope bound dismisses the band)
      }
      continue;
    }
    const double uM = 0.5 * uL + 0.5 * uR;
    band_keys_warp<kItems>(sh, n, c, uM, sh.wkeys[warp]);
    const float* ks = sh.wkeys[warp];
    double w = INFINITY;
    for (int l = lane; l + q - 1 < n; l += 32) w = fmin(w, (double)ks[l + q - 1] - (double)ks[l]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) w = fmin(w, __shfl_xor_sync(0xffffffffu, w, off));
    {  // the narrowest window's position, its end keys for the edge seeds
      int ks_ = n;
      for (int l = lane; l + q - 1 < n; l += 32)
        if ((double)ks[l + q - 1] - (double)ks[l] == w) {
          ks_ = l;
          break;
        }
      ks_ = __reduce_min_sync(0xffffffffu, (unsigned)ks_);
      if (lane < 2 * kEdge && ks_ < n) {
        const int t = lane % kEdge;
        const int at = (lane < kEdge ? ks_ : ks_ + q - 1) + t - kEdge / 2;
        sh.edge[k][lane] = ks[min(max(at, 0), n - 1)];
      }
    }
    if (lane == 0) {
      const double dmax = dev * fmax(uR - uM, uM - uL) * (1.0 + 0x1p-40);
      const double e = 0x1p-20 * (fmax(fabs(uL), fabs(uR)) * am + bm + fabs(uM) * dev) + 1e-300;
      sh.slb[k] = slope_bound(k);
      sh.lb[k] = fmax((w - 2.0 * dmax - 2.0 * e) * (1.0 - 0x1p-40), sh.slb[k]);
      sh.wq[k] = w;
      sh.um[k] = uM;
    }
    __syncwarp();
  }
  __syncthreads();

  // exact record of vertex (i, j) by this warp, against the current H
  auto exact_one = [&](int i, int j) {
    const double ai = sh.a[i], bi = sh.b[i];
    const double da = __dsub_rn(ai, sh.a[j]);
    if (da == 0.0) return;
    const double u = __ddiv_rn(__dsub_rn(bi, sh.b[j]), da);
    const double v0 = cut_value(u, ai, bi);
    const double H = current_h(&sh.hbits);
    if (lane == 0) atomicAdd(&sh.cnt[2], 1ull);
    const long long te = args.timing ? clock64() : 0;
    lms_candidate r = exact_vertex_warp(ga, gb, n, q, i, j, u, v0, H, sh.sw[warp]);
    if (args.timing && lane == 0) atomicAdd(&sh.cnt[8], (unsigned long long)(clock64() - te));
    if (r.found) {
      if (cand_less(r, mybest)) mybest = r;
      if (lane == 0)
        atomicMin(&sh.hbits, (unsigned long long)__double_as_longlong(r.height + 0.0));
    }
  };

  if (tid == 0) {
    const long long t1 = clock64();
    sh.cnt[5] = (unsigned long long)(t1 - t_mark);
    t_mark = t1;
  }
  // ---- seeds: samples of the bands with the narrowest q-windows
  if (tid == 0) {
    for (int t = 0; t < kSeedBands; ++t) {
      int best = -1;
      for (int k = 1; k < K - 1; ++k) {
        bool used = false;
        for (int u2 = 0; u2 < t; ++u2) used |= sh.seed_band[u2] == k;
        if (!used && isfinite(sh.wq[k]) && (best < 0 || sh.wq[k] < sh.wq[best])) best = k;
      }
      sh.seed_band[t] = best;
    }
  }
  __syncthreads();
  // window-edge pairs of the seed bands first: lines whose keys sit among the
  // kEdge keys around either end of the band's narrowest q-window, paired
  // within each end (the optimum's anchors are window-end lines)
  for (int t = 0; t < kSeedBands; ++t) {
    const int band = sh.seed_band[t];
    if (band < 0) continue;  // uniform
    if (tid < 2) sh.negrp[tid] = 0;
    __syncthreads();
    const double uM = sh.um[band];
    for (int l = tid; l < n; l += kThreads) {
      const float key = (float)__dsub_rn(__dmul_rn(__dsub_rn(sh.a[l], c), uM), sh.b[l]);
#pragma unroll
      for (int g = 0; g < 2; ++g)
        if (key >= sh.edge[band][g * kEdge] && key <= sh.edge[band][g * kEdge + kEdge - 1]) {
          const int slot = atomicAdd(&sh.negrp[g], 1);
          if (slot < 16) sh.egrp[g][slot] = l;
        }
    }
    __syncthreads();
    for (int g = 0; g < 2; ++g) {
      const int m = min(sh.negrp[g], 16);
      for (int pr = warp; pr < m * m; pr += kWarps) {
        const int x = sh.egrp[g][pr / m], y = sh.egrp[g][pr % m];
        if (x < y) exact_one(x, y);
      }
    }
    __syncthreads();
  }
  {
    const int sv = sh.nvalid;
    for (int t = warp; t < kSeedBands * kSeedsPerBand; t += kWarps) {
      const int band = sh.seed_band[t / kSeedsPerBand];
      if (band < 0) continue;
      // the band's samples are a contiguous run of the sorted samples
      const int lo = lower_idx(sh.s.skey, sv, sh.bounds[band - 1]);
      const int hi = lower_idx(sh.s.skey, sv, sh.bounds[band]);
      const int cnt = hi - lo;
      const int e = t % kSeedsPerBand;
      if (e >= cnt) continue;
      const int pos = lo + (int)(((int64_t)e * cnt) / (cnt < kSeedsPerBand ? cnt : kSeedsPerBand));
      int64_t i, j;
      decode_rank(n, ((2 * (int64_t)sh.s.sidx[pos] + 1) * P) / (2 * S), &i, &j);
      exact_one((int)i, (int)j);
    }
  }
  __syncthreads();

  if (tid == 0) {
    const long long t1 = clock64();
    sh.cnt[6] = (unsigned long long)(t1 - t_mark);
    t_mark = t1;
  }
  // ---- admitted bands (bound <= H), in bound order is not needed: slots
  if (tid == 0) {
    const double H = current_h(&sh.hbits);
    int na = 0;
    for (int k = 0; k < K; ++k) {
      sh.band_slot[k] = -1;
      // a keyless band the slope bound dismisses: neither keyless nor admitted
      if (!(sh.lb[k] > -INFINITY) && sh.slb[k] > H * (1.0 + 0x1p-19)) sh.lb[k] = INFINITY;
      if (sh.lb[k] > -INFINITY && sh.lb[k] <= H * (1.0 + 0x1p-19)) sh.admitted[na++] = k;
    }
    sh.nadmitted = na;
    sh.cnt[0] = na;
  }
  __syncthreads();
  const int na = sh.nadmitted;

  uint32_t* qw = sh.queue[warp];
  int qn = 0;
  uint32_t* sq = sh.squeue[warp];
  int sn = 0;
  // fp32 exact-slope counts of queued vertices (lane per vertex), then the
  // exact select of every vertex that still passes
  auto drain = [&](int cnt) {
    if (lane == 0) atomicAdd(&sh.cnt[1], (unsigned long long)cnt);
    const long long td = args.timing ? clock64() : 0;
    const double H = current_h(&sh.hbits);
    bool pass = false;
    int vi = 0, vj = 0;
    if (lane < cnt) {
      const uint32_t p = qw[lane];
      vi = (int)(p >> 16);
      vj = (int)(p & 0xFFFF);
      const double ai = sh.a[vi], bi = sh.b[vi];
      const double u = __ddiv_rn(__dsub_rn(bi, sh.b[vj]), __dsub_rn(ai, sh.a[vj]));
      const double v0 = cut_value(u, ai, bi);
      const double z = __dsub_rn(v0, __dmul_rn(c, u));
      const double mag = fabs(u) * am;
      if (huge || !isfinite(H) || !(mag + bm + H < 1e36)) {
        pass = true;
      } else {
        const double E = 0x1p-20 * (3.0 * mag + 2.0 * bm + H) + 1e-37;
        const float u32 = (float)u;
        float upLo = __double2float_rd(z - E), upHi = __double2float_ru(z + H + E);
        float dnLo = __double2float_rd(z - H - E), dnHi = __double2float_ru(z + E);
        if (upLo == 0.f) upLo = -0.f;  // so that t = -0 gives fl(t - lo) = +0
        if (dnLo == 0.f) dnLo = -0.f;
        // lo <= t <= hi implies fl(t - lo) in [+0, fl(hi - lo)] (monotone rounding),
        // tested as one unsigned compare of the bits (negatives and NaN fail)
        const uint32_t wu = __float_as_uint(__fsub_ru(upHi, upLo));
        const uint32_t wd = __float_as_uint(__fsub_ru(dnHi, dnLo));
        const float2 u2 = make_float2(u32, u32);
        const float2 nlu = make_float2(-upLo, -upLo), nld = make_float2(-dnLo, -dnLo);
        unsigned cu = 0, cd = 0;
#pragma unroll 4
        for (int p2 = 0; p2 < (n + 1) / 2; ++p2) {
          const float4 R = sh.l2[p2];
          const float2 t = __ffma2_rn(make_float2(R.x, R.y), u2, make_float2(R.z, R.w));
          const float2 du = __fadd2_rn(t, nlu);
          const float2 dd = __fadd2_rn(t, nld);
          count_le(cu, __float_as_uint(du.x), wu);
          count_le(cu, __float_as_uint(du.y), wu);
          count_le(cd, __float_as_uint(dd.x), wd);
          count_le(cd, __float_as_uint(dd.y), wd);
        }
        pass = (int)cu >= q || (int)cd >= q;
      }
    }
    if (args.timing && lane == 0) atomicAdd(&sh.cnt[9], (unsigned long long)(clock64() - td));
    unsigned m = __ballot_sync(0xffffffffu, pass);
    while (m) {
      const int src = __ffs(m) - 1;
      m &= m - 1;
      exact_one(__shfl_sync(0xffffffffu, vi, src), __shfl_sync(0xffffffffu, vj, src));
    }
  };

  // ---- sweeps: slot groups of admitted bands (the first also takes the
  // outer bands and the fits that skip the band tests)
  const int ngroups = na == 0 ? 1 : (na + kSlots - 1) / kSlots;
  if (tid == 0) sh.cnt[3] = ngroups;
  for (int grp = 0; grp < ngroups; ++grp) {
    const int g0 = grp * kSlots, g1 = min(na, g0 + kSlots);
    for (int e = g0 + warp; e < g1; e += kWarps) {
      const int band = sh.admitted[e];
      band_keys_warp<kItems>(sh, n, c, sh.um[band], sh.slot[e - g0]);
      if (lane == 0) sh.band_slot[band] = (int16_t)(e - g0);
    }
    __syncthreads();
    const bool first = grp == 0;
    if (tid == 0) {
      // runs of bands that can act in this sweep: resident ones, and in the
      // first sweep the keyless ones; widened by the edge tolerance below
      int nr = 0;
      int k = 0;
      while (k < K) {
        const bool act = sh.band_slot[k] >= 0 || (first && !(sh.lb[k] > -INFINITY));
        if (!act) {
          ++k;
          continue;
        }
        int k1 = k;
        while (k1 + 1 < K &&
               (sh.band_slot[k1 + 1] >= 0 || (first && !(sh.lb[k1 + 1] > -INFINITY))))
          ++k1;
        float lo = k == 0 ? -INFINITY : sh.bounds[k - 1];
        float hi = k1 == K - 1 ? INFINITY : sh.bounds[k1];
        lo = lo - (0x1p-17f * fabsf(lo) + 1e-36f);
        hi = hi + (0x1p-17f * fabsf(hi) + 1e-36f);
        if (nr < kMaxRuns) {
          sh.rlo[nr] = lo;
          sh.rhi[nr] = hi;
          ++nr;
        } else {  // merge into the last run (superset)
          sh.rhi[nr - 1] = hi;
        }
        k = k1 + 1;
      }
      sh.nruns = nr;
      for (int w = nr; w < kMaxRuns; ++w) sh.rlo[w] = INFINITY;  // (the run search below)
    }
    __syncthreads();
    const float amf = (float)am;
    // band lookup and padded window counts of queued in-run vertices, lane per
    // vertex; vertices of keyless bands go straight to the fp32 counts
    auto search = [&](int cnt) {
      const long long ts = args.timing ? clock64() : 0;
      const double H = current_h(&sh.hbits);
      bool pass = false;
      uint32_t p = 0;
      if (lane < cnt) {
        p = sq[lane];
        const int vi = (int)(p >> 16), vj = (int)(p & 0xFFFF);
        const double ai = sh.a[vi], bi = sh.b[vi];
        const double da = __dsub_rn(ai, sh.a[vj]);
        const double num = __dsub_rn(bi, sh.b[vj]);
        const float u32 = (float)num * rcp_approx_ftz((float)da);  // as the sweep formed it
        const int band = band_of(sh.bounds, K - 1, u32);
        int slot_id = sh.band_slot[band];
        if (slot_id < 0) {
          if (first && !(sh.lb[band] > -INFINITY)) {
            pass = true;  // outer / keyless band
          } else {
            // within the tolerance of a boundary the true band may be the
            // neighbour: test with its keys (valid for any slope), or send the
            // vertex to the counts when the neighbour is keyless
            const float tol = 0x1p-18f * fabsf(u32) + 1e-37f;
            if (band > 0 && (u32 - sh.bounds[band - 1]) <= tol) {
              if (sh.band_slot[band - 1] >= 0) slot_id = sh.band_slot[band - 1];
              else if (first && !(sh.lb[band - 1] > -INFINITY)) pass = true;
            }
            if (slot_id < 0 && !pass && band < K - 1 && (sh.bounds[band] - u32) <= tol) {
              if (sh.band_slot[band + 1] >= 0) slot_id = sh.band_slot[band + 1];
              else if (first && !(sh.lb[band + 1] > -INFINITY)) pass = true;
            }
          }
        }
        if (slot_id >= 0) {
          const double u = (double)u32;
          const double uM = sh.um[sh.admitted[g0 + slot_id]];
          const double v0 = __dsub_rn(__dmul_rn(ai, u), bi);
          const double z = __dsub_rn(v0, __dmul_rn(c, u));
          const double D = dev * fabs(u - uM) * (1.0 + 0x1p-40);
          const double E = 0x1p-20 * (fabs(u) * am + bm + fabs(uM) * dev + H) +
                           0x1p-19 * (dev + am) * fabs(u) + dev * 1e-43 + 1e-300;
          const double pad = D + E;
          const float* Ks = sh.slot[slot_id];
          const int top = upper_idx(Ks, n, __double2float_ru(z + H + pad));
          const int bot = lower_idx(Ks, n, __double2float_rd(z - H - pad));
          if (top - bot >= q) {
            const int up_lo = lower_idx(Ks, n, __double2float_rd(z - pad));
            const int dn_hi = upper_idx(Ks, n, __double2float_ru(z + pad));
            pass = (top - up_lo >= q) || (dn_hi - bot >= q);
          }
        }
      }
      if (args.timing && lane == 0) atomicAdd(&sh.cnt[10], (unsigned long long)(clock64() - ts));
      const unsigned pm = __ballot_sync(0xffffffffu, pass);
      if (pass) qw[qn + __popc(pm & ((1u << lane) - 1u))] = p;
      qn += __popc(pm);
      __syncwarp();
      if (qn >= 32) {
        drain(32);
        __syncwarp();
        if (lane < qn - 32) qw[lane] = qw[32 + lane];
        __syncwarp();
        qn -= 32;
      }
    };
    const int64_t seg = 32 * kSegRun;
    const int64_t nseg = (P + seg - 1) / seg;
    for (int64_t g = warp; g < nseg; g += kWarps) {
      const int64_t base = g * seg;
      int i = 0, j = 0;
      {
        int64_t i64 = 0, j64 = 0;
        if (lane == 0) decode_rank(n, base, &i64, &j64);
        i = __shfl_sync(0xffffffffu, (int)i64, 0);
        j = __shfl_sync(0xffffffffu, (int)j64, 0);
        advance_pair(n, lane, i, j);
      }
      // ranks of this lane inside the fit (all kSegRun except in the last segment)
      const int64_t left = P - base - lane;
      const int valid = left <= 0 ? 0 : (left >= (int64_t)32 * kSegRun ? kSegRun : (int)((left + 31) / 32));
      // kSweepStep vertices per lane per step (ranks r, r + 32, ...): independent
      // load -> test chains, one queue update and drain check per step
#pragma unroll 1
      for (int e0 = 0; e0 < kSegRun; e0 += kSweepStep) {
        int vi[kSweepStep], vj[kSweepStep];
        bool cand[kSweepStep];  // straight to the fp32 counts
        bool inr[kSweepStep];   // padded window counts against a resident band
        vi[0] = i;
        vj[0] = j;
#pragma unroll
        for (int t = 1; t < kSweepStep; ++t) {
          vi[t] = vi[t - 1];
          vj[t] = vj[t - 1];
          advance_pair(n, 32, vi[t], vj[t]);
        }
#pragma unroll
        for (int t = 0; t < kSweepStep; ++t) {
          // j runs past n only beyond the triangle's end
#if LMSB_SMALL_AB
          const double2 li = sh.ab[vi[t]], lj = sh.ab[min(vj[t], n - 1)];
#else
          const int jj = min(vj[t], n - 1);
          const double2 li = make_double2(sh.a[vi[t]], sh.b[vi[t]]);
          const double2 lj = make_double2(sh.a[jj], sh.b[jj]);
#endif
          const double da = __dsub_rn(li.x, lj.x);
          const double num = __dsub_rn(li.y, lj.y);
          const float da32 = (float)da, num32 = (float)num;
          // rcp.approx.ftz: a subnormal da32 gives an infinite / NaN u32,
          // caught by the magnitude test below (the band path of lms_band.cu
          // uses the same pre-test)
          const float u32 = num32 * rcp_approx_ftz(da32);
          const bool live = (da != 0.0) & (e0 + t < valid);
          const bool beyond = huge | !(fabsf(u32) * amf < 1e29f) |
                              ((fabsf(num32) < 1e-30f) & (num != 0.0));
          // the last run starting at or below u32 (runs ascend, unused
          // entries start at +inf), then its end: 3 steps instead of a test
          // per run
          int w = (sh.rlo[4] <= u32) ? 4 : 0;
          w += (sh.rlo[w + 2] <= u32) ? 2 : 0;
          w += (sh.rlo[w + 1] <= u32) ? 1 : 0;
          const bool inrun = (sh.rlo[w] <= u32) & (u32 <= sh.rhi[w]);
          cand[t] = live & beyond & first;  // beyond the fp32 tests (first sweep only)
          inr[t] = live & !beyond & inrun;  // band lookup deferred to search()
        }
        const unsigned below = (1u << lane) - 1u;
#pragma unroll
        for (int t = 0; t < kSweepStep; ++t) {
          const uint32_t packed = ((uint32_t)vi[t] << 16) | (uint32_t)vj[t];
          const unsigned sm_ = __ballot_sync(0xffffffffu, inr[t]);
          if (inr[t]) sq[sn + __popc(sm_ & below)] = packed;
          sn += __popc(sm_);
          const unsigned cm = __ballot_sync(0xffffffffu, cand[t]);
          if (cand[t]) qw[qn + __popc(cm & below)] = packed;
          qn += __popc(cm);
        }
        __syncwarp();
        while (qn >= 32) {
          drain(32);
          __syncwarp();
          for (int t = lane; t < qn - 32; t += 32) qw[t] = qw[32 + t];
          __syncwarp();
          qn -= 32;
        }
        while (sn >= 32) {
          search(32);  // may append to qw (and drain it)
          __syncwarp();
          for (int t = lane; t < sn - 32; t += 32) sq[t] = sq[32 + t];
          __syncwarp();
          sn -= 32;
        }
        i = vi[kSweepStep - 1];
        j = vj[kSweepStep - 1];
        advance_pair(n, 32, i, j);
      }
    }
    if (sn > 0) {
      search(sn);
      sn = 0;
    }
    if (qn > 0) {
      drain(qn);
      qn = 0;
    }
    __syncthreads();
    for (int e = g0 + tid; e < g1; e += kThreads) sh.band_slot[sh.admitted[e]] = -1;
    __syncthreads();
  }

  // ---- lexicographic minimum of the warps' records
  if (lane == 0) sh.wbest[warp] = mybest;
  __syncthreads();
  if (tid == 0) sh.cnt[7] = (unsigned long long)(clock64() - t_mark);
  if (tid == 0) {
    lms_candidate b = sh.wbest[0];
    for (int w = 1; w < kWarps; ++w)
      if (cand_less(sh.wbest[w], b)) b = sh.wbest[w];
    b.reserved = 0;
    args.out[fit] = b;
    if (args.counters)
      for (int t = 0; t < 12; ++t) atomicAdd(args.counters + t, sh.cnt[t]);
  }
}

template <int kItems, int kT>
void launch_small_t(const SmallArgs& args, int grid, cudaStream_t st) {
  constexpr size_t smem = sizeof(SmallShared<kItems, kT>);
  static DeviceOnce done;
  set_max_smem(small_fit_kernel<kItems, kT>, smem, done);
  small_fit_kernel<kItems, kT><<<grid, kT, smem, st>>>(args);
}

}  // namespace

void launch_small_fits(const SmallArgs& args, int64_t count, int64_t max_n, int sms, cudaStream_t st) {
  if (count <= 0) return;
  // fewer fits than SMs (the 64 peaks of a detect_lines call): one CTA per
  // fit is the latency, so 512 threads a fit; otherwise 256 (2 CTAs/SM)
  const bool wide = count <= sms;
  if (max_n <= 256) {
    if (wide) launch_small_t<8, 512>(args, (int)count, st);
    else launch_small_t<8, 256>(args, (int)count, st);
  } else if (max_n <= 512) {
    if (wide) launch_small_t<16, 512>(args, (int)count, st);
    else launch_small_t<16, 256>(args, (int)count, st);
  } else {
    launch_small_t<32, 256>(args, (int)count, st);
  }
}

}  // namespace lmsb
