// lms_filter.cu -- conservative per-vertex count filter (the O(n^3) stage).
//
// For a bound H (the height of some exactly evaluated vertex, so H >= the
// optimum) a vertex can only matter if one of its anchored windows has
// height <= H.  With d_k = x_k - v0 the vertical offset of line k from the
// anchor, the reference's upward window (backend.py:153,159) has
// h_up <= H  iff  at least q lines satisfy 0 <= d_k <= H (the anchors and
// lines equal to v0 included), and symmetrically h_down <= H iff at least q
// lines satisfy -H <= d_k <= 0.  This kernel counts, for every vertex, the
// lines in both windows widened by a rigorous rounding margin E_v, and keeps
// the vertex when either count reaches q.  The kept vertices ("survivors")
// are re-evaluated bit-exactly by lms_exact.cu, so the filter never decides
// a result; it only has to be a superset.
//
// Work layout (one warp task = up to 256 consecutive vertices of one row i
// of the triangle, 8 per lane):
//   * lines are re-expressed relative to the row's anchor line i,
//     A_k = a_k - a_i, B_k = b_k - b_i, so d_k = u*A_k - B_k, and pre-shifted
//     by -/+ H/2 so both windows become |t| <= H/2 + E_v:
//         t_up = fma(u, A_k, -(B_k + H/2)),  t_dn = fma(u, A_k, -(B_k - H/2))
//     (2 DFMA + 2 DSETP per vertex-line);
//   * each lane stages one line of every 32-line chunk into the warp's
//     shared-memory slab, the warp then streams the chunk from shared memory
//     (broadcast loads) while the next chunk's a/b are already in flight;
//   * a vertex is dropped early once max(count_up, count_dn) + lines left
//     < q (it can no longer reach q); the warp stops when all its vertices
//     are dropped.
// Error bound: with eps = 2^-53 the reference's x_k, v0 and the rounding of
// fl(x - v0) <= H, plus this kernel's rounded A, B, B -/+ H/2 and the FMA,
// differ from exact arithmetic by at most 8*eps*(|u|*amax + bmax + H/2)
// (see DESIGN.md); E_v uses 2^-46*(|u|*amax + bmax + H), a 16x cushion.
// Vertices whose magnitudes could overflow (|u|*amax or bmax > 1e300) are
// passed through unconditionally.

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "lms_common.cuh"
#include "lms_kernels.cuh"

namespace lmsb {

namespace {

struct alignas(32) ShiftedLine {
  double A;
  double Bu;
  double Bd;
  double pad;
};

__global__ void __launch_bounds__(kFilterWarpsPerBlock * 32)
    filter_kernel(FilterArgs args) {
  __shared__ ShiftedLine slab[kFilterWarpsPerBlock][32];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t task = args.task_begin + (int64_t)blockIdx.x * kFilterWarpsPerBlock + wib;
  if (task >= args.task_end) return;

  // Locate the task's row: largest r with task_prefix[r] <= task.
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
  const int64_t r_first = rs + (task - args.task_prefix[lo]) * kFilterTaskVertices;

  const double ai = args.a[i];
  const double bi = args.b[i];
  const lms_candidate best = *args.best;
  const double H = best.found ? best.height : INFINITY;
  const double half = 0.5 * H;

  double u[kFilterV], w[kFilterV];
  int cu[kFilterV], cd[kFilterV];
  bool valid[kFilterV], force[kFilterV];
#pragma unroll
  for (int v = 0; v < kFilterV; ++v) {
    const int64_t r = r_first + lane + 32 * v;
    valid[v] = r < re;
    force[v] = false;
    u[v] = 0.0;
    w[v] = -1.0;  // never counts
    cu[v] = 0;
    cd[v] = 0;
    if (valid[v]) {
      const int64_t j = r - row_lo + i + 1;
      const double aj = args.a[j];
      const double da = __dsub_rn(ai, aj);
      valid[v] = da != 0.0;
      const double uv = __ddiv_rn(__dsub_rn(bi, args.b[j]), da);
      valid[v] = valid[v] && isfinite(uv);
      if (valid[v]) {
        const double mag = fabs(uv) * args.amax;
        force[v] = !(mag < 1e300) || !(args.bmax < 1e300) || (isfinite(H) && !(H < 1e300));
        const double E = 0x1p-46 * (mag + args.bmax + H) + 1e-300;
        u[v] = uv;
        w[v] = half + E;
      }
    }
  }

  ShiftedLine* my = slab[wib];
  int64_t k0 = 0;
  double ak = lane < n ? __ldg(args.la + lane) : 0.0;
  double bk = lane < n ? __ldg(args.lb + lane) : 0.0;
  int64_t evals = 0;
  for (; k0 < n; k0 += 32) {
    // Stage this chunk's shifted lines; padding lines are NaN (never count).
    ShiftedLine s;
    if (k0 + lane < n) {
      s.A = __dsub_rn(ak, ai);
      const double B = __dsub_rn(bk, bi);
      s.Bu = __dadd_rn(B, half);
      s.Bd = __dsub_rn(B, half);
    } else {
      s.A = 0.0;
      s.Bu = NAN;
      s.Bd = NAN;
    }
    s.pad = 0.0;
    // Prefetch the next chunk while this one is consumed.
    const int64_t kn = k0 + 32 + lane;
    if (kn < n) {
      ak = __ldg(args.la + kn);
      bk = __ldg(args.lb + kn);
    }
    __syncwarp();
    my[lane] = s;
    __syncwarp();
#pragma unroll 4
    for (int kk = 0; kk < 32; ++kk) {
      const double2 ab = *reinterpret_cast<const double2*>(&my[kk].A);
      const double Bd = my[kk].Bd;
#pragma unroll
      for (int v = 0; v < kFilterV; ++v) {
        const double t1 = fma(u[v], ab.x, -ab.y);
        const double t2 = fma(u[v], ab.x, -Bd);
        cu[v] += fabs(t1) <= w[v];
        cd[v] += fabs(t2) <= w[v];
      }
    }
    evals += (n - k0) < 32 ? (n - k0) : 32;
    if (args.early_exit) {
      const int64_t left = n - (k0 + 32);
      bool alive = false;
#pragma unroll
      for (int v = 0; v < kFilterV; ++v) {
        const int64_t m = cu[v] > cd[v] ? cu[v] : cd[v];
        alive |= valid[v] && !force[v] && (m + left >= args.q);
      }
      if (!__any_sync(0xffffffffu, alive)) break;
    }
  }

  // Append survivors (warp-aggregated).
#pragma unroll
  for (int v = 0; v < kFilterV; ++v) {
    const bool keep = valid[v] && (force[v] || cu[v] >= args.q || cd[v] >= args.q);
    const unsigned mask = __ballot_sync(0xffffffffu, keep);
    if (mask) {
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(args.out_count, (unsigned long long)__popc(mask));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (keep) {
        const unsigned slot = __popc(mask & ((1u << lane) - 1u));
        args.out_ranks[base + slot] = r_first + lane + 32 * v;
      }
    }
  }
  if (args.line_evals && lane == 0) {
    const int64_t left_in_task = re - r_first;
    const int nv = left_in_task < kFilterTaskVertices ? (int)left_in_task : kFilterTaskVertices;
    atomicAdd(args.line_evals, (unsigned long long)(evals * nv));
  }
}

}  // namespace

void launch_filter(const FilterArgs& args, cudaStream_t stream) {
  const int64_t tasks = args.task_end - args.task_begin;
  if (tasks <= 0) return;
  const int64_t blocks = (tasks + kFilterWarpsPerBlock - 1) / kFilterWarpsPerBlock;
  filter_kernel<<<(unsigned)blocks, kFilterWarpsPerBlock * 32, 0, stream>>>(args);
}

}  // namespace lmsb
