// lms_filter32m.cu -- count filter with packed-FP16 compares and integer
// mask accumulation (no tensor core).  Same contract, margins and line
// staging as lms_filter32.cu; only the counting differs:
//
//   t    = fma2(u, (A_k, A_k+1), -(Bu_k, Bu_k+1))   FFMA2
//   hu   = half2(t)                                  F2FP
//   hd   = hu + (H/S, H/S)                           HADD2
//   mu   = |hu| <= w_v  as 0xFFFF masks per half     HSET2 (mask form)
//   md   = |hd| <= w_v                               HSET2
//   cu  += mu, cd += md                              2x IADD (32-bit)
//
// A 32-bit sum of such masks encodes two independent counts: with U_e, U_o
// the hits in the low / high halves, sum = (U_e - U_o)*2^16 - U_e (mod
// 2^32), so U_e = -lo16(sum) mod 2^16 and U_o = U_e - hi16(sum + U_e)
// (mod 2^16) are recovered exactly while both stay below 2^16 (n <= 131070
// lines).  Thread-per-vertex layout: lane l owns vertices l + 32*s of the
// warp task; every lane streams the same line pairs (shared-memory
// broadcast).

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "lms_common.cuh"
#include "lms_kernels.cuh"

namespace lmsb {

namespace {

constexpr int kV = kFilter32mV;  // vertices per lane

struct __align__(16) LinePair {
  float2 A;   // (A_k, A_k+1)
  float2 Bn;  // (-Bu_k, -Bu_k+1)
};

// Accumulation of a half2 mask word.  IMAD (mad.lo c, m, 1, c) issues on the
// FMA pipe, IADD3 on the ALU pipe that F2FP and HSET2 already load; the
// LMSB_F32M_ACC policy picks the split (0: both IADD3, 1: up IMAD / down
// IADD3, 2: both IMAD).
#ifndef LMSB_F32M_ACC
#define LMSB_F32M_ACC 1
#endif
__device__ __forceinline__ void acc_imad(uint32_t& c, uint32_t m) {
  asm volatile("mad.lo.u32 %0, %1, 1, %0;" : "+r"(c) : "r"(m));
}
__device__ __forceinline__ void acc_up(uint32_t& c, uint32_t m) {
  if (LMSB_F32M_ACC >= 1) acc_imad(c, m);
  else c += m;
}
__device__ __forceinline__ void acc_dn(uint32_t& c, uint32_t m) {
  if (LMSB_F32M_ACC >= 2) acc_imad(c, m);
  else c += m;
}

__device__ __forceinline__ uint32_t mask_total(uint32_t sum) {
  const uint32_t ue = (0x10000u - (sum & 0xFFFFu)) & 0xFFFFu;
  const uint32_t uo = (ue - ((sum + ue) >> 16)) & 0xFFFFu;
  return ue + uo;
}

__global__ void __launch_bounds__(kFilterWarpsPerBlock * 32, kFilter32mMinBlocks)
    filter32m_kernel(FilterArgs args) {
  __shared__ LinePair slab[kFilterWarpsPerBlock][32];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t task = args.task_begin + (int64_t)blockIdx.x * kFilterWarpsPerBlock + wib;
  if (task >= args.task_end) return;

  int64_t lo = 0, hi = args.nrows - 1;
  while (lo < hi) {
    int64_t mid = (lo + hi + 1) >> 1;
    if (args.task_prefix[mid] <= task) lo = mid;
    else hi = mid - 1;
  }
  const int64_t n = args.n;
  const int64_t i = args.row0 + lo;
  const int64_t row_lo = row_offset(n, i);
  const int64_t row_hi = row_lo + (n - 1 - i);
  const int64_t rs = row_lo > args.rank_lo ? row_lo : args.rank_lo;
  const int64_t re = row_hi < args.rank_hi ? row_hi : args.rank_hi;
  const int64_t r_first = rs + (task - args.task_prefix[lo]) * kFilter32mTaskVertices;

  const double ai = args.a[i];
  const double bi = args.b[i];
  const lms_candidate best = *args.best;
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
      const double aj = args.a[j];
      const double da = __dsub_rn(ai, aj);
      const double uv = __ddiv_rn(__dsub_rn(bi, args.b[j]), da);
      valid[s] = da != 0.0 && isfinite(uv);
      if (valid[s]) {
        const double mag = fabs(uv) * args.amax;
        const double w = half + (0x1p-20 * (mag + args.bmax + H) + 1e-300);
        force[s] = !(mag < 1e30) || !(args.bmax < 1e30) || !(w < 1e30);
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
      ak2 = __ldg(reinterpret_cast<const double2*>(args.la + k));
      bk2 = __ldg(reinterpret_cast<const double2*>(args.lb + k));
    } else if (k < n) {
      ak2 = make_double2(__ldg(args.la + k), 0.0);
      bk2 = make_double2(__ldg(args.lb + k), 0.0);
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
        acc_up(cu[s], __hle2_mask(__habs2(hu), w2[s]));
        acc_dn(cd[s], __hle2_mask(__habs2(hd), w2[s]));
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
        alive |= valid[s] && !force[s] && (m + left >= (uint32_t)args.q);
      }
      if (!__any_sync(0xffffffffu, alive)) break;
    }
  }

#pragma unroll
  for (int s = 0; s < kV; ++s) {
    const uint32_t q = (uint32_t)args.q;
    const bool keep = valid[s] && (force[s] || mask_total(cu[s]) >= q || mask_total(cd[s]) >= q);
    const unsigned mask = __ballot_sync(0xffffffffu, keep);
    if (mask) {
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(args.out_count, (unsigned long long)__popc(mask));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (keep) {
        const unsigned slot = __popc(mask & ((1u << lane) - 1u));
        args.out_ranks[base + slot] = r_first + lane + 32 * s;
      }
    }
  }
  if (args.line_evals && lane == 0) {
    const int64_t left_in_task = re - r_first;
    const int nv =
        left_in_task < kFilter32mTaskVertices ? (int)left_in_task : kFilter32mTaskVertices;
    atomicAdd(args.line_evals, (unsigned long long)(evals * nv));
  }
}

}  // namespace

void launch_filter32m(const FilterArgs& args, cudaStream_t stream) {
  const int64_t tasks = args.task_end - args.task_begin;
  if (tasks <= 0) return;
  const int64_t blocks = (tasks + kFilterWarpsPerBlock - 1) / kFilterWarpsPerBlock;
  filter32m_kernel<<<(unsigned)blocks, kFilterWarpsPerBlock * 32, 0, stream>>>(args);
}

}  // namespace lmsb
