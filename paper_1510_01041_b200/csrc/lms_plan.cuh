// lms_plan.cuh -- filter work plan (lms_plan.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "lms_kernels.cuh"

namespace lmsb {

// Phase A rows: every kPhaseStride-th row of each fit (see lms_plan.cu).
constexpr int64_t kPhaseStride = 8;

struct PlanArgs {
  const FitDesc* fits;
  const int64_t* prefA;         // F + 1: first phase-A global row of every fit
  const int64_t* prefB;         // F + 1: first phase-B global row of every fit
  int64_t nfits;
  int64_t rowsA;                // phase-A rows (they come first)
  int64_t nrows;                // total global rows
  int64_t task_vertices;
  int64_t* counts;              // nrows + 1 scratch
  int32_t* row_fit;             // nrows
  int32_t* row_i;               // nrows: triangle row of every global row
  int64_t* row_task_prefix;     // nrows + 1
  int32_t* task_row;            // total tasks
  void* temp;
  size_t temp_bytes;
};

// Sum_{m=1..M} ceil(m / tv) (tasks of M consecutive full-row lengths).
int64_t ceil_sum(int64_t M, int64_t tv);
// Warp tasks of row i of one fit restricted to ranks [R0, R1).
int64_t row_tasks(int64_t n, int64_t R0, int64_t R1, int64_t i, int64_t tv);
// Warp tasks of ranks [R0, R1) of one fit; also returns its first row and row count.
int64_t fit_tasks(int64_t n, int64_t R0, int64_t R1, int64_t tv, int64_t* row0, int64_t* nrows);
int launch_plan(const PlanArgs& p, cudaStream_t stream);
size_t plan_temp_bytes(int64_t nrows);
void launch_line_fit(const int64_t* seg, int64_t nfits, int32_t* line_fit, cudaStream_t stream);

}  // namespace lmsb
