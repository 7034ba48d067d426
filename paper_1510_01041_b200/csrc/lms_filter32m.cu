// lms_filter32m.cu -- the count filter (the O(n^3) stage of the exact search).
//
// For the bound H (the height of an exactly evaluated vertex, so H >= the
// optimum) a vertex can only matter if one of its anchored windows has
// height <= H.  With d_k = x_k - v0 the vertical offset of line k from the
// anchor, the reference's upward window (backend.py:153,159) has h_up <= H
// iff at least q lines satisfy 0 <= d_k <= H (anchors and ties included),
// and symmetrically h_down <= H iff at least q lines satisfy -H <= d_k <= 0.
// This kernel counts both windows for every vertex, widened by a rigorous
// rounding margin, and keeps the vertex when either count reaches q.
// Survivors are re-evaluated bit-exactly in FP64 (lms_exact.cu), so the
// filter only has to return a superset; its arithmetic may be approximate as
// long as the margin covers the error.
//
// Warp task: up to 32*V consecutive vertices of one triangle row i of one
// fit.  Lines are re-expressed relative to the row's anchor line,
// A_k = (a_k - a_i)/S and Bu_k = ((b_k - b_i) + H/2)/S, formed in FP64 and
// rounded to FP32 once per line and warp (S = power of two >= the warp's
// largest window, so the scaling is exact), and staged per warp in 64-line
// chunks of shared memory (16-byte (A_k, A_k+1, -Bu_k, -Bu_k+1) records,
// broadcast to all lanes).  Lane l owns vertices l + 32*s.  Per vertex and
// line pair:
//
//   t    = fma2(u, (A_k, A_k+1), -(Bu_k, Bu_k+1))   FFMA2 (packed fp32x2)
//   hu   = half2(t)                                  F2FP
//   hd   = hu + (H/S, H/S)                           HADD2 (down window)
//   mu   = |hu| <= w_v  as 0xFFFF masks per half     HSET2 (mask form)
//   md   = |hd| <= w_v                               HSET2
//   cu  += mu, cd += md                              IADD3 (ptxas merges two)
//
// A 32-bit sum of such masks encodes two independent counts: with U_e, U_o
// the hits in the low / high halves, sum = (U_e - U_o)*2^16 - U_e (mod
// 2^32), so U_e = -lo16(sum) mod 2^16 and U_o = U_e - hi16(sum + U_e)
// (mod 2^16) are recovered exactly while both stay below 2^16 (n <= 131070
// lines).  (Tensor-core counting with legacy mma.sync was measured slower:
// on B200 HMMA.16816 issues at ~0.1/clk/SMSP and throttles the other pipes;
// see DESIGN.md.)
//
// Early exit: once max(count_up, count_dn) + lines left < q for every vertex
// of the warp, none can reach q and the warp stops.  Lines stream far-first
// (lms_order.cu), so this happens after ~n - q lines.
//
// Error budget (unnormalised units; eps32 = 2^-24):
//   u -> fp32, A, Bu -> fp32 and the FFMA rounding: <= 3*eps32*(|u|*|A|max
//   + |B|max + H); the FP64 line shifts and the reference's own roundings of
//   x_k, v0 and fl(x - v0) <= H: <= 2^-50*(|u|*amax + bmax + H).  Margin
//   E_v = 2^-20*(|u|*amax + bmax + H) + 1e-300 covers both with >= 2x to
//   spare (|A|max <= 2*amax, |B|max <= 2*bmax).  In units of S, FP16
//   rounding of t (|t| < 4 where it matters) is <= 2^-10, of H/S <= 2^-11
//   and of the HADD2 <= 2^-11; thresholds add 2^-8 and round up.  t beyond
//   the FP16 range becomes inf and never counts, which is correct because
//   such lines are far outside every window (|t|/S > 65504 >> 2).  Vertices
//   whose magnitudes could overflow FP32 are passed to the exact stage
//   unconditionally.

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "lms_common.cuh"
#include "lms_kernels.cuh"

namespace lmsb {

namespace {

struct __align__(16) LinePair {
  float2 A;   // (A_k, A_k+1)
  float2 Bn;  // (-Bu_k, -Bu_k+1)
};

__device__ __forceinline__ uint32_t mask_total(uint32_t sum) {
  const uint32_t ue = (0x10000u - (sum & 0xFFFFu)) & 0xFFFFu;
  const uint32_t uo = (ue - ((sum + ue) >> 16)) & 0xFFFFu;
  return ue + uo;
}

template <int kV>
__global__ void __launch_bounds__(kFilterWarpsPerBlock * 32, kV >= 4 ? 3 : 4)
    filter32m_kernel(FilterArgs args) {
  constexpr int64_t kTaskVertices = 32 * kV;
  __shared__ LinePair slab[kFilterWarpsPerBlock][32];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t task = args.task_begin + (int64_t)blockIdx.x * kFilterWarpsPerBlock + wib;
  if (task >= args.task_end) return;

  // task -> global row -> (fit, triangle row i, first vertex rank)
  const int64_t grow = args.task_row[task];
  const int32_t fit = args.row_fit[grow];
  const FitDesc fd = args.fits[fit];
  const int64_t n = fd.n;
  const int64_t i = args.row_i[grow];
  const int64_t row_lo = row_offset(n, i);
  const int64_t row_hi = row_lo + (n - 1 - i);
  const int64_t rs = row_lo > fd.rank_lo ? row_lo : fd.rank_lo;
  const int64_t re = row_hi < fd.rank_hi ? row_hi : fd.rank_hi;
  const int64_t r_first = rs + (task - args.row_task_prefix[grow]) * kTaskVertices;
  const double* a = args.a + fd.off;
  const double* b = args.b + fd.off;
  const double* la = args.la + fd.off;
  const double* lb = args.lb + fd.off;

  const double ai = a[i];
  const double bi = b[i];
  const lms_candidate best = args.best[fit];
  const double H = best.found ? best.height : INFINITY;
  const double half = 0.5 * H;

  double w64[kV];
  float u32[kV];
  bool valid[kV], force[kV];
  double wmax = 0.0;
#pragma unroll
  for (int s = 0; s < kV; ++s) {
    const int64_t r = r_first + lane + 32 * s;
    valid[s] = r < re;
    force[s] = false;
    u32[s] = 0.f;
    w64[s] = 0.0;
    if (valid[s]) {
      const int64_t j = r - row_lo + i + 1;
      const double aj = a[j];
      const double da = __dsub_rn(ai, aj);
      const double uv = __ddiv_rn(__dsub_rn(bi, b[j]), da);
      valid[s] = da != 0.0 && isfinite(uv);
      if (valid[s]) {
        const double mag = fabs(uv) * fd.amax;
        const double w = half + (0x1p-20 * (mag + fd.bmax + H) + 1e-300);
        force[s] = !(mag < 1e30) || !(fd.bmax < 1e30) || !(w < 1e30);
        u32[s] = (float)uv;
        w64[s] = w;
        if (!force[s]) wmax = fmax(wmax, w);
      }
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) wmax = fmax(wmax, __shfl_xor_sync(0xffffffffu, wmax, off));
  int e = 0;
  if (wmax > 0.0) frexp(wmax, &e);
  const double invS = ldexp(1.0, -e);
  const __half hnh = __float2half_rn((float)(H * invS));
  const __half2 hn2 = __halves2half2(hnh, hnh);
  __half2 w2[kV];
#pragma unroll
  for (int s = 0; s < kV; ++s) {
    const float wn = (float)(w64[s] * invS) + 0x1p-8f;
    const bool live = valid[s] && !force[s];
    const __half wh = __float2half_ru(live ? wn : -1.0f);
    w2[s] = __halves2half2(wh, wh);
  }

  uint32_t cu[kV], cd[kV];
#pragma unroll
  for (int s = 0; s < kV; ++s) cu[s] = cd[s] = 0u;

  LinePair* my = slab[wib];
  double2 ak2 = make_double2(0.0, 0.0), bk2 = make_double2(0.0, 0.0);
  auto load_pair = [&](int64_t k) {
    if (k + 1 < n) {
      ak2 = make_double2(__ldg(la + k), __ldg(la + k + 1));
      bk2 = make_double2(__ldg(lb + k), __ldg(lb + k + 1));
    } else if (k < n) {
      ak2 = make_double2(__ldg(la + k), 0.0);
      bk2 = make_double2(__ldg(lb + k), 0.0);
    }
  };
  load_pair(2 * lane);
  int64_t evals = 0;
  for (int64_t k0 = 0; k0 < n; k0 += 64) {
    const int64_t k = k0 + 2 * lane;
    LinePair P;
    if (k < n) {
      P.A.x = (float)(__dsub_rn(ak2.x, ai) * invS);
      P.Bn.x = -(float)(__dadd_rn(__dsub_rn(bk2.x, bi), half) * invS);
    } else {
      P.A.x = 0.f;
      P.Bn.x = __int_as_float(0x7fc00000);
    }
    if (k + 1 < n) {
      P.A.y = (float)(__dsub_rn(ak2.y, ai) * invS);
      P.Bn.y = -(float)(__dadd_rn(__dsub_rn(bk2.y, bi), half) * invS);
    } else {
      P.A.y = 0.f;
      P.Bn.y = __int_as_float(0x7fc00000);
    }
    load_pair(k + 64);
    __syncwarp();
    my[lane] = P;
    __syncwarp();
#pragma unroll 8
    for (int p = 0; p < 32; ++p) {
      const LinePair L = my[p];
#pragma unroll
      for (int s = 0; s < kV; ++s) {
        const float2 t = __ffma2_rn(L.A, make_float2(u32[s], u32[s]), L.Bn);
        const __half2 hu = __floats2half2_rn(t.x, t.y);
        const __half2 hd = __hadd2(hu, hn2);
        cu[s] += __hle2_mask(__habs2(hu), w2[s]);
        cd[s] += __hle2_mask(__habs2(hd), w2[s]);
      }
    }
    evals += (n - k0) < 64 ? (n - k0) : 64;
    if (args.early_exit) {
      const int64_t rem = n - (k0 + 64);
      const uint32_t left = rem > 0 ? (uint32_t)rem : 0u;
      bool alive = false;
#pragma unroll
      for (int s = 0; s < kV; ++s) {
        const uint32_t m = max(mask_total(cu[s]), mask_total(cd[s]));
        alive |= valid[s] && !force[s] && (m + left >= (uint32_t)fd.q);
      }
      if (!__any_sync(0xffffffffu, alive)) break;
    }
  }

#pragma unroll
  for (int s = 0; s < kV; ++s) {
    const uint32_t q = (uint32_t)fd.q;
    const bool keep = valid[s] && (force[s] || mask_total(cu[s]) >= q || mask_total(cd[s]) >= q);
    const unsigned mask = __ballot_sync(0xffffffffu, keep);
    if (mask) {
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(args.out_count, (unsigned long long)__popc(mask));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (keep) {
        const unsigned slot = __popc(mask & ((1u << lane) - 1u));
        args.out_ranks[base + slot] = r_first + lane + 32 * s;
        args.out_fits[base + slot] = fit;
      }
    }
  }
  if (args.line_evals && lane == 0) {
    const int64_t left_in_task = re - r_first;
    const int nv = left_in_task < kTaskVertices ? (int)left_in_task : (int)kTaskVertices;
    atomicAdd(args.line_evals, (unsigned long long)(evals * nv));
  }
}

}  // namespace

void launch_filter(const FilterArgs& args, int v, cudaStream_t stream) {
  const int64_t tasks = args.task_end - args.task_begin;
  if (tasks <= 0) return;
  const unsigned blocks = (unsigned)((tasks + kFilterWarpsPerBlock - 1) / kFilterWarpsPerBlock);
  const unsigned threads = kFilterWarpsPerBlock * 32;
  switch (v) {
    case 1: filter32m_kernel<1><<<blocks, threads, 0, stream>>>(args); break;
    case 2: filter32m_kernel<2><<<blocks, threads, 0, stream>>>(args); break;
    default: filter32m_kernel<4><<<blocks, threads, 0, stream>>>(args); break;
  }
}

}  // namespace lmsb
