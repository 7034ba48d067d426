// lms_primal.cu -- the reference's independent primal brute force
// (oracle_lms, solver.py:143-196) on the GPU.
//
// For every pair i < j with x_i != x_j: slope s = (y_j - y_i)/(x_j - x_i),
// intercepts c_k = y_k - s*x_k (one rounded product, one rounded
// difference, as numpy's `y[None, :] - s[:, None] * x[None, :]`), sorted;
// the narrowest contiguous q-window c[w + q - 1] - c[w] with the first
// minimal w.  The global winner is the lexicographic (span, i, j) minimum
// (solver.py:170-179), reduced with the same 128-bit CAS key as the dual
// search.  One CTA per pair sorts the n intercepts in shared memory
// (bitonic, n padded to a power of two with +inf), so n is limited to
// kPrimalMaxN; the routine is a cross-check for moderate n, as in the
// reference.

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "lms_common.cuh"
#include "lms_kernels.cuh"
#include "lms_primal.cuh"

namespace lmsb {

namespace {

constexpr int kPrimalThreads = 256;

__global__ void __launch_bounds__(kPrimalThreads)
    primal_kernel(const double* __restrict__ x, const double* __restrict__ y, int64_t n, int64_t q,
                  int64_t npow2, lms_candidate* __restrict__ recs) {
  extern __shared__ double cs[];
  __shared__ double red_span[kPrimalThreads / 32];
  __shared__ int64_t red_w[kPrimalThreads / 32];
  const int64_t total = n * (n - 1) / 2;
  const int tid = threadIdx.x;
  for (int64_t r = blockIdx.x; r < total; r += gridDim.x) {
    int64_t i, j;
    decode_rank(n, r, &i, &j);
    lms_candidate c = cand_none();
    c.i = i;
    c.j = j;
    const double dx = __dsub_rn(x[j], x[i]);
    if (dx != 0.0) {  // uniform across the CTA
      const double s = __ddiv_rn(__dsub_rn(y[j], y[i]), dx);
      for (int64_t k = tid; k < npow2; k += kPrimalThreads)
        cs[k] = k < n ? __dsub_rn(y[k], __dmul_rn(s, x[k])) : INFINITY;
      __syncthreads();
      // bitonic sort (ascending) of npow2 values
      for (int64_t size = 2; size <= npow2; size <<= 1) {
        for (int64_t stride = size >> 1; stride > 0; stride >>= 1) {
          for (int64_t k = tid; k < npow2; k += kPrimalThreads) {
            const int64_t p = k ^ stride;
            if (p > k) {
              const bool up = (k & size) == 0;
              const double a = cs[k], b = cs[p];
              if ((a > b) == up) {
                cs[k] = b;
                cs[p] = a;
              }
            }
          }
          __syncthreads();
        }
      }
      // first minimal window: lexicographic min of (span, w)
      double best = INFINITY;
      int64_t bw = -1;
      for (int64_t w = tid; w + q - 1 < n; w += kPrimalThreads) {
        const double span = __dsub_rn(cs[w + q - 1], cs[w]);
        if (span < best || (span == best && (bw < 0 || w < bw))) {
          best = span;
          bw = w;
        }
      }
      for (int off = 16; off > 0; off >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, off);
        const int64_t ow = __shfl_xor_sync(0xffffffffu, bw, off);
        if (ow >= 0 && (bw < 0 || ob < best || (ob == best && ow < bw))) {
          best = ob;
          bw = ow;
        }
      }
      if ((tid & 31) == 0) {
        red_span[tid >> 5] = best;
        red_w[tid >> 5] = bw;
      }
      __syncthreads();
      if (tid == 0) {
        for (int k = 1; k < kPrimalThreads / 32; ++k) {
          const double ob = red_span[k];
          const int64_t ow = red_w[k];
          if (ow >= 0 && (bw < 0 || ob < best || (ob == best && ow < bw))) {
            best = ob;
            bw = ow;
          }
        }
        if (bw >= 0 && isfinite(best)) {
          c.height = best;
          c.u = s;
          c.v_low = cs[bw];
          c.v_high = cs[bw + q - 1];
          c.found = 1;
        }
      }
      __syncthreads();
    }
    if (tid == 0) recs[r] = c;
  }
}

}  // namespace

size_t primal_smem_bytes(int64_t n) {
  int64_t p = 1;
  while (p < n) p <<= 1;
  return (size_t)p * sizeof(double);
}

int launch_primal(const double* x, const double* y, int64_t n, int64_t q, lms_candidate* recs,
                  int grid, cudaStream_t stream) {
  int64_t p = 1;
  while (p < n) p <<= 1;
  const size_t smem = (size_t)p * sizeof(double);
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(primal_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
          cudaSuccess)
    return -1;
  primal_kernel<<<grid, kPrimalThreads, smem, stream>>>(x, y, n, q, p, recs);
  return 0;
}

}  // namespace lmsb
