// lms_filter32.cu -- the count filter on FP32 FMA + FP16 compare + tensor-core
// counting (default filter; lms_filter.cu is the all-FP64 variant).
//
// Same contract as lms_filter.cu: for the bound H, keep every vertex whose
// upward or downward anchored window could have height <= H, i.e. whose
// count of lines with offset d_k = x_k - v0 in [0, H] (resp. [-H, 0]),
// widened by a rigorous rounding margin, reaches q.  Survivors are then
// re-evaluated bit-exactly in FP64 (lms_exact.cu), so this stage only has to
// return a superset; its arithmetic may be approximate as long as the
// margin covers the error.
//
// Per vertex and PAIR of lines (k, k+1), 5 instructions = 2.5 per
// vertex-line evaluation:
//   t_k   = fma(u, A_k, -Bu_k)        FFMA2: Blackwell's packed fp32x2 FMA,
//                                      both lines in one instruction (the 2
//                                      algorithmic flops u*a_k - b_k per eval)
//   hu    = half2(t_k, t_k+1)         F2FP pack
//   hd    = hu + (H/S, H/S)           HADD2   (down window = up window
//                                              shifted by H)
//   up    = |hu| <= w_v               HSET2   -> half2 of 1.0 / 0.0
//   dn    = sat(C_v - K*|hd|)         HFMA2.SAT (1.0 inside the window,
//                                              [0,1] in a 1/K band outside)
// where, for the warp's row i, A_k = (a_k - a_i)/S and Bu_k = ((b_k - b_i)
// + H/2)/S are formed in FP64 and rounded to FP32 once per line and warp
// (S = power of two >= the warp's largest window, so scaling is exact).
// The indicator half2s are (row, k-pair) elements of the A operand of
// mma.sync.m16n8k16 (f16 x f16 -> f32): rows are 16 vertices, columns 0-7
// the up indicators and 8-15 the down indicators of 8 lines, and the
// constant B operand routes columns 0-7 to output column 0 and 8-15 to
// column 1.  The tensor core accumulates both window counts of 16 vertices
// over 8 lines per instruction (counts < 2^24, exact in fp32; the
// fractional band values only ever ADD to a count, keeping the superset).
// The compare is split across the ALU (HSET2) and FMA (HFMA2) pipes so
// neither saturates before the issue slot does.
//
// Warp task: 64 consecutive vertices (4 MMA row tiles) of one row of the
// triangle; lane (g = lane/4, c = lane%4) evaluates vertices {16t+g,
// 16t+g+8} against lines {2c, 2c+1} of every 8-line group, the fragment
// layout of mma.m16n8k16.  Lines are staged per warp in 64-line chunks in
// shared memory as 16-byte (A_k, A_k+1, -Bu_k, -Bu_k+1) records.
//
// Error budget (unnormalised units; eps32 = 2^-24):
//   u -> fp32, A, Bu -> fp32 and the FFMA rounding: <= 3*eps32*(|u|*|A|max
//   + |B|max + H); the FP64 line shifts and the reference's own roundings of
//   x_k, v0 and fl(x - v0) <= H: <= 2^-50*(|u|*amax + bmax + H).  Margin
//   E_v = 2^-20*(|u|*amax + bmax + H) + 1e-300 covers both with >= 2x to
//   spare (|A|max <= 2*amax, |B|max <= 2*bmax).  In units of S, FP16
//   rounding of t_up (|t| < 4 where it matters) is <= 2^-10, of H/S <= 2^-11
//   and of the HADD2 <= 2^-11; thresholds add 2^-8 and round up, and the
//   ramp constant C_v = K*w_v + 1 is rounded up.  t beyond the FP16 range
//   becomes inf and never counts, which is correct because such lines are
//   far outside every window (|t|/S > 65504 >> 2).  Vertices whose scaled
//   magnitudes could overflow FP32 are passed to the exact stage
//   unconditionally.

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "lms_common.cuh"
#include "lms_kernels.cuh"

namespace lmsb {

namespace {

constexpr int kTiles = kFilter32Tiles;  // 16-vertex MMA row tiles per warp
#ifndef LMSB_F32_MIN_BLOCKS
#define LMSB_F32_MIN_BLOCKS 3
#endif
constexpr int kFilter32MinBlocks = LMSB_F32_MIN_BLOCKS;  // resident CTAs per SM (register cap)
constexpr int kSlots = 2 * kTiles;      // vertices per lane

struct __align__(16) LinePair {
  float2 A;   // (A_k, A_k+1)
  float2 Bn;  // (-Bu_k, -Bu_k+1)
};

constexpr float kRampK = 1024.0f;  // HFMA2 ramp slope (power of two: exact product)

// Up/down indicator half2s of one vertex against one line pair.
__device__ __forceinline__ void indicators(float u, const LinePair& L, uint32_t hn2, uint32_t w2,
                                           uint32_t c2, uint32_t& up, uint32_t& dn) {
  const float2 t = __ffma2_rn(L.A, make_float2(u, u), L.Bn);  // FFMA2: both lines at once
  const __half2 hu = __floats2half2_rn(t.x, t.y);
  const __half2 hd = __hadd2(hu, *reinterpret_cast<const __half2*>(&hn2));
  const __half2 iu = __hle2(__habs2(hu), *reinterpret_cast<const __half2*>(&w2));
  const __half2 mk = __float2half2_rn(-kRampK);
  const __half2 id = __hfma2_sat(__habs2(hd), mk, *reinterpret_cast<const __half2*>(&c2));
  up = *reinterpret_cast<const uint32_t*>(&iu);
  dn = *reinterpret_cast<const uint32_t*>(&id);
}

__device__ __forceinline__ void mma_count(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                          uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 "
      "{%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, {%0, %1, %2, %3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__global__ void __launch_bounds__(kFilterWarpsPerBlock * 32, kFilter32MinBlocks)
    filter32_kernel(FilterArgs args) {
  __shared__ LinePair slab[kFilterWarpsPerBlock][32];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int g = lane >> 2;
  const int c = lane & 3;
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
  const int64_t r_first = rs + (task - args.task_prefix[lo]) * kFilter32TaskVertices;

  const double ai = args.a[i];
  const double bi = args.b[i];
  const lms_candidate best = *args.best;
  const double H = best.found ? best.height : INFINITY;
  const double half = 0.5 * H;

  // Per-slot vertex parameters; slot s = 2t + h is vertex 16t + g + 8h.
  double w64[kSlots];
  float u32[kSlots];
  bool valid[kSlots], force[kSlots];
  double wmax = 0.0;
#pragma unroll
  for (int s = 0; s < kSlots; ++s) {
    const int vi = 16 * (s >> 1) + g + 8 * (s & 1);
    const int64_t r = r_first + vi;
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
        // FP32 range guard: |u|*|A|/S and |B|/S must stay far below FLT_MAX,
        // and an unbounded H (no seed found) cannot be scaled.
        force[s] = !(mag < 1e30) || !(args.bmax < 1e30) || !(w < 1e30);
        u32[s] = (float)uv;
        w64[s] = w;
        if (!force[s]) wmax = fmax(wmax, w);
      }
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) wmax = fmax(wmax, __shfl_xor_sync(0xffffffffu, wmax, off));
  // S = 2^e >= wmax (exact scaling); an all-forced / empty warp uses S = 1.
  int e = 0;
  if (wmax > 0.0) frexp(wmax, &e);
  const double invS = ldexp(1.0, -e);
  const __half hnh = __float2half_rn((float)(H * invS));
  const __half2 hn2h = __halves2half2(hnh, hnh);
  const uint32_t hn2 = *reinterpret_cast<const uint32_t*>(&hn2h);
  uint32_t w2[kSlots], c2[kSlots];
#pragma unroll
  for (int s = 0; s < kSlots; ++s) {
    const float wn = (float)(w64[s] * invS) + 0x1p-8f;
    const bool live = valid[s] && !force[s];
    const __half wh = __float2half_ru(live ? wn : -1.0f);
    const __half ch = __float2half_ru(live ? fmaf(kRampK, wn, 1.0f) : -1.0f);
    const __half2 w = __halves2half2(wh, wh);
    const __half2 cc = __halves2half2(ch, ch);
    w2[s] = *reinterpret_cast<const uint32_t*>(&w);
    c2[s] = *reinterpret_cast<const uint32_t*>(&cc);
  }

  // B operand: k-rows 0-7 (up) -> column 0, k-rows 8-15 (down) -> column 1.
  const __half2 onesh = __float2half2_rn(1.0f), zerosh = __float2half2_rn(0.0f);
  const __half2 b0h = g == 0 ? onesh : zerosh;
  const __half2 b1h = g == 1 ? onesh : zerosh;
  const uint32_t b0 = *reinterpret_cast<const uint32_t*>(&b0h);
  const uint32_t b1 = *reinterpret_cast<const uint32_t*>(&b1h);

  float d[kTiles][4];
#pragma unroll
  for (int t = 0; t < kTiles; ++t) d[t][0] = d[t][1] = d[t][2] = d[t][3] = 0.f;

  // 64-line chunks: lane p stages the line pair (k0 + 2p, k0 + 2p + 1) as one
  // 16-byte record (A0, A1, -Bu0, -Bu1); the next chunk's a/b are prefetched
  // (one coalesced double2 load each) while this chunk is consumed.
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
    } else {  // padding line: NaN never counts
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
#pragma unroll
    for (int grp = 0; grp < 8; ++grp) {
      const LinePair L = my[grp * 4 + c];
#pragma unroll
      for (int t = 0; t < kTiles; ++t) {
        uint32_t a0, a1, a2, a3;
        indicators(u32[2 * t], L, hn2, w2[2 * t], c2[2 * t], a0, a2);
        indicators(u32[2 * t + 1], L, hn2, w2[2 * t + 1], c2[2 * t + 1], a1, a3);
        mma_count(d[t], a0, a1, a2, a3, b0, b1);
      }
    }
    evals += (n - k0) < 64 ? (n - k0) : 64;
    if (args.early_exit) {
      const float left = (float)(n - (k0 + 64));
      const float qf = (float)args.q;
      bool alive = false;
      if (c == 0) {
#pragma unroll
        for (int t = 0; t < kTiles; ++t) {
          alive |= valid[2 * t] && !force[2 * t] && (fmaxf(d[t][0], d[t][1]) + left >= qf);
          alive |= valid[2 * t + 1] && !force[2 * t + 1] && (fmaxf(d[t][2], d[t][3]) + left >= qf);
        }
      }
      if (!__any_sync(0xffffffffu, alive)) break;
    }
  }

  // Survivors: lanes with c == 0 hold both counts of rows g and g+8.
  const float qf = (float)args.q;
#pragma unroll
  for (int s = 0; s < kSlots; ++s) {
    const int t = s >> 1;
    const float up = (s & 1) ? d[t][2] : d[t][0];
    const float dn = (s & 1) ? d[t][3] : d[t][1];
    const bool keep = c == 0 && valid[s] && (force[s] || up >= qf || dn >= qf);
    const unsigned mask = __ballot_sync(0xffffffffu, keep);
    if (mask) {
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(args.out_count, (unsigned long long)__popc(mask));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (keep) {
        const unsigned slot = __popc(mask & ((1u << lane) - 1u));
        args.out_ranks[base + slot] = r_first + 16 * t + g + 8 * (s & 1);
      }
    }
  }
  if (args.line_evals && lane == 0) {
    const int64_t left_in_task = re - r_first;
    const int nv = left_in_task < kFilter32TaskVertices ? (int)left_in_task : kFilter32TaskVertices;
    atomicAdd(args.line_evals, (unsigned long long)(evals * nv));
  }
}

}  // namespace

void launch_filter32(const FilterArgs& args, cudaStream_t stream) {
  const int64_t tasks = args.task_end - args.task_begin;
  if (tasks <= 0) return;
  const int64_t blocks = (tasks + kFilterWarpsPerBlock - 1) / kFilterWarpsPerBlock;
  filter32_kernel<<<(unsigned)blocks, kFilterWarpsPerBlock * 32, 0, stream>>>(args);
}

}  // namespace lmsb
