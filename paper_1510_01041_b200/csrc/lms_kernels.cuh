// lms_kernels.cuh -- device data model and launch interfaces of the
// exact-LMS kernels (host side).
//
// A solve is a batch of F independent fits (F = 1 for one large fit, F =
// 8,192 for the Hough-refinement workload).  Fit f owns lines
// [off, off + n) of the concatenated fp64 arrays a[] (x) and b[] (y) and the
// pair-rank range [rank_lo, rank_hi) of its own row-major upper triangle
// (backend.py:111-122).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/lms_b200.h"

namespace lmsb {

struct FitDesc {
  int64_t off;       // first line of the fit in a[] / b[]
  int64_t n;
  int64_t q;
  int64_t rank_lo;   // vertex ranks of this fit handled by the solve
  int64_t rank_hi;
  int64_t row0;      // first triangle row of [rank_lo, rank_hi)
  int64_t nrows;     // rows in the filter task list (0: fit solved exhaustively)
  double amax;       // max |a|, max |b| over the fit's lines (filter margins)
  double bmax;
};

// 128-bit lexicographic key (height bits, pair rank) of a fit's best record,
// updated with 128-bit atomic CAS; hi = canonical bits of the height, lo = rank.
struct __align__(16) BestKey {
  unsigned long long lo;
  unsigned long long hi;
};

// ---------------------------------------------------------------- exact stage
enum ExactSource : int {
  kSrcList = 0,      // (ranks[s], fit_of[s]), s < *d_count or count
  kSrcExplicit = 1,  // explicit (i, j, u[, v]) of fit 0, s < count
};

struct ExactArgs {
  const double* a;
  const double* b;
  const FitDesc* fits;
  int mode;
  int64_t count;                      // used when d_count == nullptr
  const unsigned long long* d_count;  // device-side item count (survivors)
  int64_t capacity;
  const int64_t* ranks;
  const int32_t* fit_of;
  const int64_t* ii;
  const int64_t* jj;
  const double* uu;
  const double* vv;
  const lms_candidate* bound;  // optional per-fit bound (skip vertices that cannot win)
  lms_candidate* out;          // out[s].reserved = fit id
  unsigned long long* live_h;  // optional (single fit): bits of the lowest height found so far;
                               // vertices are tested against it and lower it as they finish
  int cached;                  // few vertices: one CTA each, cut keys cached in shared memory
  int64_t cached_end;          // cached: items beyond this go to the streaming kernel (0: none)
  int64_t begin;               // streaming kernel: first item
  int64_t cluster_max;         // > 0: lists of at most this many items go to the cluster
                               // kernel, longer ones to the cached kernel (n <= kExactCacheN)
};

// Largest fit whose cut keys the cached exact kernel keeps in shared memory.
constexpr int64_t kExactCacheN = 16384;

// One CTA per vertex for large fits, one warp per vertex when every fit has
// at most 4,096 lines (max_n).
void launch_exact(const ExactArgs& args, int grid, cudaStream_t stream, int64_t max_n);

// Lexicographic (height, i, j) minimum per fit (backend.py:165-167,182-187)
// over records [0, count): CAS into keys[fit], then publish into best[fit].
void launch_reduce(const lms_candidate* recs, const unsigned long long* d_count, int64_t count,
                   int64_t capacity, const FitDesc* fits, BestKey* keys, lms_candidate* best,
                   int grid, cudaStream_t stream);
void launch_reset_best(BestKey* keys, lms_candidate* best, int64_t nfits, cudaStream_t stream);

// K1 of the materialised flow: explicit (i, j, u) of the non-parallel pairs
// of ranks [r0, r0 + count), compacted; *nout counts them (zeroed by caller).
void launch_materialize(const double* a, const double* b, int64_t n, int64_t r0, int64_t count,
                        int64_t* ii, int64_t* jj, double* uu, unsigned long long* nout, int sms,
                        cudaStream_t stream);

// Contact set of a fit's record (solve_lms tail, solver.py:122-140): indices
// appended in any order to out (at most cap); scratch[1] = total count.
void launch_contacts(const double* a, const double* b, int64_t n, const lms_candidate& rec,
                     unsigned long long* scratch, int64_t* out, int64_t cap, int sms,
                     cudaStream_t st);

// Contact flags of every point of a batch (offs: F + 1 device offsets, recs:
// the fits' records on the device, fit-local i / j).
void launch_contacts_batch(const double* a, const double* b, const int64_t* offs,
                           const lms_candidate* recs, int64_t nfits, uint8_t* flags, int sms,
                           cudaStream_t st);

// Seeds: stratified vertex samples per fit; seed_prefix[f] = first seed of fit f.
void launch_gen_seeds(const FitDesc* fits, const int64_t* seed_prefix, int64_t nfits,
                      int64_t* ranks, int32_t* fit_of, cudaStream_t stream);

// ---------------------------------------------------------------- filter
constexpr int kFilterWarpsPerBlock = 8;

struct FilterArgs {
  const double* a;   // lines in input order (anchors i, j)
  const double* b;
  const double* la;  // lines in streaming order (lms_order.cu); may alias a / b
  const double* lb;
  const FitDesc* fits;
  const int32_t* task_row;         // global row of every warp task
  const int64_t* row_task_prefix;  // first task of every global row
  const int32_t* row_fit;          // fit of every global row
  const int32_t* row_i;            // triangle row of every global row
  int64_t task_begin;
  int64_t task_end;
  const lms_candidate* best;       // per-fit best record (its height bounds the search)
  int64_t* out_ranks;              // survivors
  int32_t* out_fits;
  unsigned long long* out_count;
  unsigned long long* line_evals;  // executed vertex-line evaluations (stats)
  int early_exit;
};

// Vertices per warp task for lanes owning V vertices each.
inline int64_t filter_task_vertices(int v) { return 32 * (int64_t)v; }
void launch_filter(const FilterArgs& args, int v, cudaStream_t stream);

// ---------------------------------------------------------------- line order
struct OrderArgs {
  const double* a;
  const double* b;
  int64_t nlines;
  const int64_t* seg_begin;  // per-fit line offsets (F + 1 entries)
  int64_t nfits;
  const int32_t* line_fit;   // fit of every line
  const lms_candidate* best;
  float* keys_in;
  float* keys_out;
  int* idx_in;
  int* idx_out;
  void* temp;
  size_t temp_bytes;
  double* pa;
  double* pb;
};
size_t order_temp_bytes(int64_t nlines, int64_t nfits);
int launch_line_order(const OrderArgs& o, cudaStream_t stream);

}  // namespace lmsb
