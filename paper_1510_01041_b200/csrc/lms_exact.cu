// lms_exact.cu -- exact per-vertex anchored-window evaluation and the
// lexicographic argmin.
//
// One CTA evaluates one arrangement vertex (i, j, u) exactly as the
// reference's `_evaluate_pairs` does for one row (backend.py:140-171):
//   v0      = a_i*u - b_i                              (backend.py:144)
//   x_k     = u*a_k - b_k, x_i = x_j = v0              (backend.py:145-148)
//   k_lo    = #(x < v0), k_hi = #(x <= v0) - 1          (backend.py:149-150)
//   down    = k_hi - (q-1), up = k_lo + (q-1)           (backend.py:152-153)
//   h_down  = v0 - vs[down] | inf, h_up = vs[up] - v0 | inf, up wins ties
//                                                       (backend.py:154-161)
// where vs is the sorted cut.  Instead of sorting (the reference's
// O(n log n) per vertex), the two order statistics vs[up] and vs[down] are
// selected by an MSD radix select over order-preserving uint64 keys:
// 8-bit digits, a shared-memory histogram per target, the prefix narrowed
// each pass, finishing early once the target bucket holds one element.
// Every pass recomputes the cut from the lines (16 B/line, L2-resident), so
// the per-vertex state is O(1) and any n fits.
//
// The argmin is the strict lexicographic (height, i, j) minimum of
// _merge / the chunk tie-break (backend.py:165-167, 182-187).

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "lms_common.cuh"
#include "lms_kernels.cuh"

namespace lmsb {

namespace {

constexpr int kExactThreads = 256;
constexpr int kExactWarps = kExactThreads / kWarp;

struct SelectShared {
  unsigned hist[2][256];
  unsigned long long prefix[2];
  long long rank[2];
  unsigned long long result[2];
  int state[2];  // -1 inactive, 0 searching, 1 unique element pending, 2 done
  unsigned red_lt[kExactWarps];
  unsigned red_le[kExactWarps];
  unsigned red_up[kExactWarps];
  unsigned red_dn[kExactWarps];
};

__device__ __forceinline__ double snapped_cut(const double* __restrict__ a,
                                              const double* __restrict__ b, int64_t k, int64_t i,
                                              int64_t j, double u, double v0) {
  return (k == i || k == j) ? v0 : cut_value(u, __ldg(a + k), __ldg(b + k));
}

// Warp `t` picks the digit bucket containing rank[t] from hist[t].
__device__ void pick_digit(SelectShared& sm, int t, int level) {
  const int lane = threadIdx.x & 31;
  unsigned h[8];
  unsigned sum = 0;
#pragma unroll
  for (int d = 0; d < 8; ++d) {
    h[d] = sm.hist[t][lane * 8 + d];
    sum += h[d];
  }
  unsigned incl = sum;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    unsigned o = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += o;
  }
  const unsigned excl = incl - sum;
  const long long r = sm.rank[t];
  const bool mine = r >= (long long)excl && r < (long long)incl;
  if (mine) {
    unsigned c = excl;
    int digit = 0;
    unsigned cnt = 0;
#pragma unroll
    for (int d = 0; d < 8; ++d) {
      if (r >= (long long)c && r < (long long)(c + h[d])) {
        digit = lane * 8 + d;
        cnt = h[d];
        break;
      }
      c += h[d];
    }
    sm.prefix[t] = (sm.prefix[t] << 8) | (unsigned long long)digit;
    sm.rank[t] = r - (long long)c;
    if (level == 7) {
      sm.result[t] = sm.prefix[t];
      sm.state[t] = 2;
    } else if (cnt == 1) {
      sm.state[t] = 1;
    }
  }
}

// Exact anchored window at (i, j, u) with anchors snapped to v0.  Must be
// called by all threads of the CTA; thread 0's return value is meaningful.
// When `bound` is finite the vertex is evaluated only if one of its windows
// can reach height <= bound; pass 0 counts, with the reference's own
// arithmetic, the lines x >= v0 with fl(x - v0) <= bound (resp. x <= v0 with
// fl(v0 - x) <= bound).  h_up <= bound iff that count reaches q, because
// fl(x - v0) is monotone in x and vs[up] is the q-th smallest x >= v0
// (backend.py:153,159); otherwise no select is needed and the vertex is
// reported as not found (it cannot win against a record of height bound).
__device__ lms_candidate exact_vertex(const double* __restrict__ a, const double* __restrict__ b,
                                      int64_t n, int64_t q, int64_t i, int64_t j, double u,
                                      double v0, double bound, SelectShared& sm) {
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;

  // Pass 0: rank counts of v0 in the snapped cut (+ window counts vs bound).
  unsigned lt = 0, le = 0, wu = 0, wd = 0;
  for (int64_t k = tid; k < n; k += kExactThreads) {
    double x = snapped_cut(a, b, k, i, j, u, v0);
    lt += x < v0;
    le += x <= v0;
    wu += x >= v0 && __dsub_rn(x, v0) <= bound;
    wd += x <= v0 && __dsub_rn(v0, x) <= bound;
  }
  lt = __reduce_add_sync(0xffffffffu, lt);
  le = __reduce_add_sync(0xffffffffu, le);
  wu = __reduce_add_sync(0xffffffffu, wu);
  wd = __reduce_add_sync(0xffffffffu, wd);
  if (lane == 0) {
    sm.red_lt[warp] = lt;
    sm.red_le[warp] = le;
    sm.red_up[warp] = wu;
    sm.red_dn[warp] = wd;
  }
  __syncthreads();
  int64_t c_lt = 0, c_le = 0, c_up = 0, c_dn = 0;
#pragma unroll
  for (int w = 0; w < kExactWarps; ++w) {
    c_lt += sm.red_lt[w];
    c_le += sm.red_le[w];
    c_up += sm.red_up[w];
    c_dn += sm.red_dn[w];
  }
  if (isfinite(bound) && c_up < q && c_dn < q) {
    __syncthreads();
    lms_candidate none = cand_none();
    return none;
  }
  const int64_t down = c_le - q;        // k_hi - (q - 1)
  const int64_t up = c_lt + q - 1;      // k_lo + (q - 1)
  const bool ok_down = down >= 0;
  const bool ok_up = up <= n - 1;

  lms_candidate c = cand_none();
  c.i = i;
  c.j = j;
  c.u = u;

  // Both windows inside the class of values equal to v0: vs[up] == vs[down]
  // == v0, so h_up = h_down = 0 and the upward window wins.
  if (c_le - c_lt >= q && isfinite(v0)) {
    c.height = 0.0;
    c.v_low = v0;
    c.v_high = v0;
    c.found = 1;
    __syncthreads();
    return c;
  }

  if (tid < 2) {
    const bool active = tid == 0 ? ok_up : ok_down;
    sm.prefix[tid] = 0ULL;
    sm.rank[tid] = tid == 0 ? up : down;
    sm.result[tid] = 0ULL;
    sm.state[tid] = active ? 0 : -1;
  }
  __syncthreads();

  for (int level = 0; level < 8; ++level) {
    const int shift = 56 - 8 * level;
    const int s0 = sm.state[0];
    const int s1 = sm.state[1];
    if ((s0 == 2 || s0 == -1) && (s1 == 2 || s1 == -1)) break;
    const unsigned long long p0 = sm.prefix[0];
    const unsigned long long p1 = sm.prefix[1];
    for (int e = tid; e < 512; e += kExactThreads) (&sm.hist[0][0])[e] = 0u;
    __syncthreads();
    for (int64_t k = tid; k < n; k += kExactThreads) {
      const unsigned long long key = key_of(snapped_cut(a, b, k, i, j, u, v0));
      const unsigned long long hi = level == 0 ? 0ULL : (key >> (shift + 8));
      const unsigned digit = (unsigned)(key >> shift) & 255u;
      if (s0 == 0 && hi == p0) atomicAdd(&sm.hist[0][digit], 1u);
      if (s1 == 0 && hi == p1) atomicAdd(&sm.hist[1][digit], 1u);
      if (s0 == 1 && hi == p0) sm.result[0] = key;
      if (s1 == 1 && hi == p1) sm.result[1] = key;
    }
    __syncthreads();
    if (warp < 2) {
      const int t = warp;
      const int st = t == 0 ? s0 : s1;
      if (st == 0) pick_digit(sm, t, level);
      else if (st == 1 && lane == 0) sm.state[t] = 2;
    }
    __syncthreads();
  }

  const double v_up = ok_up ? value_of(sm.result[0]) : 0.0;
  const double v_down = ok_down ? value_of(sm.result[1]) : 0.0;
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
  __syncthreads();
  return c;
}

__global__ void __launch_bounds__(kExactThreads) exact_kernel(ExactArgs args) {
  __shared__ SelectShared sm;
  int64_t count = args.count;
  if (args.mode == kSrcRanks) count = (int64_t)*args.d_count;
  if (count > args.capacity) count = args.capacity;
  const int64_t n = args.n;
  double bound = INFINITY;
  if (args.bound) {
    const lms_candidate bc = *args.bound;
    if (bc.found) bound = bc.height;
  }
  for (int64_t s = blockIdx.x; s < count; s += gridDim.x) {
    int64_t i, j;
    double u, v0;
    bool valid = true;
    if (args.mode == kSrcExplicit) {
      i = args.ii[s];
      j = args.jj[s];
      u = args.uu[s];
      v0 = args.vv ? args.vv[s] : cut_value(u, args.a[i], args.b[i]);
    } else {
      int64_t r;
      if (args.mode == kSrcRanks) {
        r = args.ranks[s];
      } else {  // stratified sample of [rank_lo, rank_hi)
        const int64_t span = args.rank_hi - args.rank_lo;
        r = args.rank_lo + ((2 * s + 1) * span) / (2 * count);
      }
      decode_rank(n, r, &i, &j);
      const double ai = args.a[i], aj = args.a[j];
      // _scan_rank_range drops parallel duals and forms u unfused
      // (backend.py:200-204).
      valid = __dsub_rn(ai, aj) != 0.0;
      u = __ddiv_rn(__dsub_rn(args.b[i], args.b[j]), __dsub_rn(ai, aj));
      v0 = cut_value(u, ai, args.b[i]);
    }
    lms_candidate c = cand_none();
    if (valid) c = exact_vertex(args.a, args.b, n, args.q, i, j, u, v0, bound, sm);
    if (threadIdx.x == 0) args.out[s] = c;
  }
}

constexpr int kReduceThreads = 256;

__global__ void __launch_bounds__(kReduceThreads)
    reduce_partial_kernel(const lms_candidate* __restrict__ recs, const unsigned long long* d_count,
                          int64_t count, int64_t capacity, lms_candidate* __restrict__ partials) {
  if (d_count) count = (int64_t)*d_count;
  if (count > capacity) count = capacity;
  lms_candidate best = cand_none();
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < count;
       s += (int64_t)gridDim.x * blockDim.x) {
    lms_candidate c = recs[s];
    if (cand_less(c, best)) best = c;
  }
  best = warp_min_cand(best);
  __shared__ lms_candidate sh[kReduceThreads / kWarp];
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x < 32) {
    best = threadIdx.x < kReduceThreads / kWarp ? sh[threadIdx.x] : cand_none();
    best = warp_min_cand(best);
    if (threadIdx.x == 0) partials[blockIdx.x] = best;
  }
}

__global__ void __launch_bounds__(32)
    reduce_final_kernel(const lms_candidate* __restrict__ partials, int np,
                        lms_candidate* __restrict__ best_io) {
  lms_candidate best = threadIdx.x == 0 ? *best_io : cand_none();
  for (int s = threadIdx.x; s < np; s += 32) {
    lms_candidate c = partials[s];
    if (cand_less(c, best)) best = c;
  }
  best = warp_min_cand(best);
  if (threadIdx.x == 0) *best_io = best;
}

}  // namespace

void launch_exact(const ExactArgs& args, int grid, cudaStream_t stream) {
  if (grid <= 0) return;
  exact_kernel<<<grid, kExactThreads, 0, stream>>>(args);
}

void launch_reduce(const lms_candidate* recs, const unsigned long long* d_count, int64_t count,
                   int64_t capacity, lms_candidate* partials, int npartials,
                   lms_candidate* best_io, cudaStream_t stream) {
  reduce_partial_kernel<<<npartials, kReduceThreads, 0, stream>>>(recs, d_count, count, capacity,
                                                                  partials);
  reduce_final_kernel<<<1, 32, 0, stream>>>(partials, npartials, best_io);
}

}  // namespace lmsb
