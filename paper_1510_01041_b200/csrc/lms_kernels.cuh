// lms_kernels.cuh -- launch interfaces of the exact-LMS kernels (host side).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/lms_b200.h"

namespace lmsb {

enum ExactSource : int {
  kSrcRanks = 0,     // ranks[s], s < *d_count (filter survivors)
  kSrcStrided = 1,   // stratified sample of [rank_lo, rank_hi), s < count
  kSrcExplicit = 2,  // explicit (i, j, u[, v]) lists, s < count
};

struct ExactArgs {
  const double* a;
  const double* b;
  int64_t n;
  int64_t q;
  int mode;
  int64_t count;
  const unsigned long long* d_count;
  int64_t capacity;
  const int64_t* ranks;
  int64_t rank_lo;
  int64_t rank_hi;
  const int64_t* ii;
  const int64_t* jj;
  const double* uu;
  const double* vv;
  const lms_candidate* bound;  // optional: skip vertices that cannot beat bound->height
  lms_candidate* out;
};

void launch_exact(const ExactArgs& args, int grid, cudaStream_t stream);
void launch_reduce(const lms_candidate* recs, const unsigned long long* d_count, int64_t count,
                   int64_t capacity, lms_candidate* partials, int npartials,
                   lms_candidate* best_io, cudaStream_t stream);

// Count filter over warp tasks [task_begin, task_end).  A warp task is up to
// kFilterTaskVertices consecutive pair ranks of one row of the triangle.
constexpr int kFilterV = 8;                          // vertices per lane
constexpr int kFilterTaskVertices = 32 * kFilterV;   // vertices per warp task
constexpr int kFilterWarpsPerBlock = 8;

struct FilterArgs {
  const double* a;   // lines in input order (anchors i, j)
  const double* b;
  const double* la;  // lines in streaming order (lms_order.cu); may alias a/b
  const double* lb;
  int64_t n;
  int64_t q;
  const int64_t* task_prefix;  // task_prefix[r] = first task of row row0 + r
  int64_t row0;
  int64_t nrows;
  int64_t rank_lo;
  int64_t rank_hi;
  int64_t task_begin;
  int64_t task_end;
  double amax;
  double bmax;
  const lms_candidate* best;        // current best (its height bounds the search)
  int64_t* out_ranks;               // survivors
  unsigned long long* out_count;
  unsigned long long* line_evals;   // executed vertex-line evaluations (stats)
  int early_exit;
};

void launch_filter(const FilterArgs& args, cudaStream_t stream);

// FP32-FMA / FP16-compare / mma.sync-count variant (lms_filter32.cu).
#ifndef LMSB_F32_TILES
#define LMSB_F32_TILES 4
#endif
constexpr int kFilter32Tiles = LMSB_F32_TILES;             // 16-vertex MMA row tiles per warp
constexpr int kFilter32TaskVertices = 16 * kFilter32Tiles; // vertices per warp task

void launch_filter32(const FilterArgs& args, cudaStream_t stream);

// Packed-FP16 compare / integer-mask counting variant (lms_filter32m.cu).
#ifndef LMSB_F32M_V
#define LMSB_F32M_V 4
#endif
#ifndef LMSB_F32M_MIN_BLOCKS
#define LMSB_F32M_MIN_BLOCKS 3
#endif
constexpr int kFilter32mV = LMSB_F32M_V;                    // vertices per lane
constexpr int kFilter32mMinBlocks = LMSB_F32M_MIN_BLOCKS;
constexpr int kFilter32mTaskVertices = 32 * kFilter32mV;    // vertices per warp task

void launch_filter32m(const FilterArgs& args, cudaStream_t stream);

// Far-first line streaming order (lms_order.cu).
struct OrderArgs {
  const double* a;
  const double* b;
  int64_t n;
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
size_t order_temp_bytes(int64_t n);
int launch_line_order(const OrderArgs& o, cudaStream_t stream);

}  // namespace lmsb
