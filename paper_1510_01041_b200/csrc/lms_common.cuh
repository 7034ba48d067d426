// lms_common.cuh -- device helpers shared by the exact-LMS kernels.
//
// Arithmetic contract: every cut value is formed exactly as the reference's
// numpy expression `u * a_k - b_k` (backend.py:145): one rounded product,
// then one rounded difference.  The intrinsics __dmul_rn / __dsub_rn are
// never contracted into an FMA, so the exact path is bit-identical to numpy
// regardless of -fmad.  Only the conservative count filter (lms_filter.cu)
// uses FMA, and it carries an explicit error margin.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "../../include/lms_b200.h"

namespace lmsb {

constexpr int kWarp = 32;

// Order-preserving uint64 key of a double: key(x) < key(y) iff x sorts before
// y.  NaN is canonicalised to the positive quiet NaN so it sorts after +inf,
// as np.sort places NaNs last; -0.0 sorts just before +0.0 (they compare
// equal, so either order reproduces np.sort's values).
__device__ __forceinline__ uint64_t key_of(double x) {
  if (x != x) x = __longlong_as_double(0x7FF8000000000000LL);
  uint64_t bits = static_cast<uint64_t>(__double_as_longlong(x));
  return (bits >> 63) ? ~bits : (bits | 0x8000000000000000ULL);
}

__device__ __forceinline__ double value_of(uint64_t key) {
  uint64_t bits = (key >> 63) ? (key & 0x7FFFFFFFFFFFFFFFULL) : ~key;
  return __longlong_as_double(static_cast<long long>(bits));
}

// Cut value of line k at abscissa u: numpy's `u * a_k - b_k`, unfused.
__device__ __forceinline__ double cut_value(double u, double ak, double bk) {
  return __dsub_rn(__dmul_rn(u, ak), bk);
}

// Row-major upper-triangle pair ranks (backend.py:111-122):
// offsets[i] = rank of (i, i+1) = i*(n-1) - i*(i-1)/2.
__host__ __device__ __forceinline__ int64_t row_offset(int64_t n, int64_t i) {
  return i * (n - 1) - i * (i - 1) / 2;
}

// searchsorted(offsets, r, side="right") - 1, then j = r - offsets[i] + i + 1.
__host__ __device__ __forceinline__ void decode_rank(int64_t n, int64_t r, int64_t* pi,
                                                     int64_t* pj) {
  int64_t lo = 0, hi = n - 2;
  while (lo < hi) {
    int64_t mid = (lo + hi + 1) >> 1;
    if (row_offset(n, mid) <= r) lo = mid;
    else hi = mid - 1;
  }
  *pi = lo;
  *pj = r - row_offset(n, lo) + lo + 1;
}

// Strict lexicographic (height, i, j) order with IEEE equality on height
// (so -0.0 ties +0.0), as Python's tuple compare in _merge (backend.py:185)
// and the chunk tie-break on i*n + j (backend.py:165-167).  Not-found
// records sort last.
__host__ __device__ __forceinline__ bool cand_less(const lms_candidate& x,
                                                   const lms_candidate& y) {
  if (!x.found) return false;
  if (!y.found) return true;
  if (x.height < y.height) return true;
  if (x.height > y.height) return false;
  if (x.i != y.i) return x.i < y.i;
  return x.j < y.j;
}

__device__ __forceinline__ lms_candidate cand_none() {
  lms_candidate c;
  c.height = 0.0;
  c.u = 0.0;
  c.v_low = 0.0;
  c.v_high = 0.0;
  c.i = -1;
  c.j = -1;
  c.found = 0;
  c.reserved = 0;
  return c;
}

__device__ __forceinline__ lms_candidate shfl_cand(const lms_candidate& c, int src) {
  lms_candidate o;
  o.height = __shfl_sync(0xffffffffu, c.height, src);
  o.u = __shfl_sync(0xffffffffu, c.u, src);
  o.v_low = __shfl_sync(0xffffffffu, c.v_low, src);
  o.v_high = __shfl_sync(0xffffffffu, c.v_high, src);
  o.i = __shfl_sync(0xffffffffu, c.i, src);
  o.j = __shfl_sync(0xffffffffu, c.j, src);
  o.found = __shfl_sync(0xffffffffu, c.found, src);
  o.reserved = 0;
  return o;
}

// Warp-wide lexicographic minimum (result valid in every lane).
__device__ __forceinline__ lms_candidate warp_min_cand(lms_candidate c) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    lms_candidate o = shfl_cand(c, (threadIdx.x & 31) ^ off);
    if (cand_less(o, c)) c = o;
  }
  return c;
}

// cudaFuncSetAttribute applies to the current device: remember it per device
// (bit d of the mask), so a process driving several GPUs (the `par` backend)
// sets every kernel's shared-memory limit on each of them.
struct DeviceOnce {
  std::atomic<unsigned long long> mask{0};
};

template <typename Kern>
inline void set_max_smem(Kern kern, size_t smem, DeviceOnce& once) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (once.mask.load(std::memory_order_relaxed) & bit) return;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  once.mask.fetch_or(bit);
}

// ---------------------------------------------------------------- bulk copy
// 1-D TMA bulk copies global -> shared (cp.async.bulk, completion counted on
// an mbarrier in transaction bytes).  Sizes and both addresses must be
// multiples of 16 bytes.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// One thread stages `bytes` (multiple of 16, both pointers 16-byte aligned)
// into shared memory with bulk copies of <= 64 KB; every thread of the CTA
// then waits for the transaction count.  `bar` must be initialised (count 1)
// and visible to the CTA; `phase` alternates per use.
__device__ __forceinline__ void bulk_stage(void* dst, const void* src, uint32_t bytes,
                                           uint64_t* bar, uint32_t phase) {
  if (threadIdx.x == 0) {
    mbar_expect_tx(bar, bytes);
    for (uint32_t off = 0; off < bytes; off += 65536u) {
      const uint32_t len = bytes - off < 65536u ? bytes - off : 65536u;
      bulk_g2s(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off, len, bar);
    }
  }
  mbar_wait(bar, phase);
}

}  // namespace lmsb
