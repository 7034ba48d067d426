// lms_exact_warp.cuh -- exact anchored window of one vertex, evaluated by one
// warp (radix select over order-preserving uint64 keys of the snapped cut),
// shared by the exact stage (lms_exact.cu) and the fused small-fit kernel
// (lms_band_small.cu).  Same arithmetic as the reference's _evaluate_pairs
// (backend.py:140-171): see lms_exact.cu for the derivation.
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "lms_common.cuh"

namespace lmsb {

__device__ __forceinline__ double snapped_cut(const double* __restrict__ a,
                                              const double* __restrict__ b, int64_t k, int64_t i,
                                              int64_t j, double u, double v0) {
  return (k == i || k == j) ? v0 : cut_value(u, __ldg(a + k), __ldg(b + k));
}

// ---------------------------------------------------------------------------
// Warp-per-vertex variant for small fits (n <= kWarpExactMaxN): the same
// passes as exact_vertex with warp-synchronous reductions, so a 512-line
// vertex does not idle a 256-thread CTA.  Per-warp shared state: two
// 256-bin digit histograms.
constexpr int kWarpExactMaxN = 4096;

struct SelectWarp {
  unsigned hist[2][256];
};

// Bucket of rank r in hist (warp-wide): digit, count below it, its count.
__device__ __forceinline__ void pick_digit_warp(const unsigned* hist, long long r, int& digit,
                                                long long& below, unsigned& cnt) {
  const int lane = threadIdx.x & 31;
  unsigned h[8];
  unsigned sum = 0;
#pragma unroll
  for (int d = 0; d < 8; ++d) {
    h[d] = hist[lane * 8 + d];
    sum += h[d];
  }
  unsigned incl = sum;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned o = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += o;
  }
  const unsigned excl = incl - sum;
  const bool mine = r >= (long long)excl && r < (long long)incl;
  int dg = 0;
  unsigned c = excl, ct = 0;
  if (mine) {
#pragma unroll
    for (int d = 0; d < 8; ++d) {
      if (r >= (long long)c && r < (long long)(c + h[d])) {
        dg = lane * 8 + d;
        ct = h[d];
        break;
      }
      c += h[d];
    }
  }
  const unsigned ballot = __ballot_sync(0xffffffffu, mine);
  const int src = __ffs(ballot) - 1;
  digit = __shfl_sync(0xffffffffu, dg, src);
  below = (long long)__shfl_sync(0xffffffffu, c, src);
  cnt = __shfl_sync(0xffffffffu, ct, src);
}

static __device__ __noinline__ lms_candidate exact_vertex_warp(const double* __restrict__ a,
                                           const double* __restrict__ b, int64_t n, int64_t q,
                                           int64_t i, int64_t j, double u, double v0,
                                           double bound, SelectWarp& sw) {
  const int lane = threadIdx.x & 31;
  if (bound < 0.0) return cand_none();  // (warp-uniform) no height can reach it
  unsigned lt = 0, le = 0, wu = 0, wd = 0;
  for (int64_t k = lane; k < n; k += 32) {
    const double x = snapped_cut(a, b, k, i, j, u, v0);
    lt += x < v0;
    le += x <= v0;
    wu += x >= v0 && __dsub_rn(x, v0) <= bound;
    wd += x <= v0 && __dsub_rn(v0, x) <= bound;
  }
  const int64_t c_lt = __reduce_add_sync(0xffffffffu, lt);
  const int64_t c_le = __reduce_add_sync(0xffffffffu, le);
  const int64_t c_up = __reduce_add_sync(0xffffffffu, wu);
  const int64_t c_dn = __reduce_add_sync(0xffffffffu, wd);
  lms_candidate c = cand_none();
  if (isfinite(bound) && c_up < q && c_dn < q) return c;
  const int64_t down = c_le - q;
  const int64_t up = c_lt + q - 1;
  const bool ok_down = down >= 0;
  const bool ok_up = up <= n - 1;
  c.i = i;
  c.j = j;
  c.u = u;
  if (c_le - c_lt >= q && isfinite(v0)) {
    c.height = 0.0;
    c.v_low = v0;
    c.v_high = v0;
    c.found = 1;
    return c;
  }
  unsigned long long prefix[2] = {0ULL, 0ULL}, result[2] = {0ULL, 0ULL};
  long long rank[2] = {up, down};
  int state[2] = {ok_up ? 0 : -1, ok_down ? 0 : -1};
  for (int level = 0; level < 8; ++level) {
    if ((state[0] == 2 || state[0] == -1) && (state[1] == 2 || state[1] == -1)) break;
    const int shift = 56 - 8 * level;
#pragma unroll
    for (int e = lane; e < 512; e += 32) (&sw.hist[0][0])[e] = 0u;
    __syncwarp();
    unsigned long long found0 = 0ULL, found1 = 0ULL;
    bool has0 = false, has1 = false;
    for (int64_t k = lane; k < n; k += 32) {
      const unsigned long long key = key_of(snapped_cut(a, b, k, i, j, u, v0));
      const unsigned long long hi = level == 0 ? 0ULL : (key >> (shift + 8));
      const unsigned digit = (unsigned)(key >> shift) & 255u;
      if (state[0] == 0 && hi == prefix[0]) atomicAdd(&sw.hist[0][digit], 1u);
      if (state[1] == 0 && hi == prefix[1]) atomicAdd(&sw.hist[1][digit], 1u);
      if (state[0] == 1 && hi == prefix[0]) {
        found0 = key;
        has0 = true;
      }
      if (state[1] == 1 && hi == prefix[1]) {
        found1 = key;
        has1 = true;
      }
    }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      if (state[t] == 1) {  // the unique element with this prefix, found this pass
        const unsigned bal = __ballot_sync(0xffffffffu, t == 0 ? has0 : has1);
        result[t] = __shfl_sync(0xffffffffu, t == 0 ? found0 : found1, __ffs(bal) - 1);
        state[t] = 2;
      } else if (state[t] == 0) {
        int digit;
        long long below;
        unsigned cnt;
        pick_digit_warp(sw.hist[t], rank[t], digit, below, cnt);
        prefix[t] = (prefix[t] << 8) | (unsigned long long)digit;
        rank[t] -= below;
        if (level == 7) {
          result[t] = prefix[t];
          state[t] = 2;
        } else if (cnt == 1) {
          state[t] = 1;
        }
      }
    }
    __syncwarp();
  }
  const double v_up = ok_up ? value_of(result[0]) : 0.0;
  const double v_down = ok_down ? value_of(result[1]) : 0.0;
  const double h_down = ok_down ? __dsub_rn(v0, v_down) : INFINITY;
  const double h_up = ok_up ? __dsub_rn(v_up, v0) : INFINITY;
  const bool use_up = h_up <= h_down;
  const double h = use_up ? h_up : h_down;
  if (isfinite(h)) {
    c.height = h;
    c.v_low = use_up ? v0 : v_down;
    c.v_high = use_up ? v_up : v0;
    c.found = 1;
  }
  return c;
}

}  // namespace lmsb
