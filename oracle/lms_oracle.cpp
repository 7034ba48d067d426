/*
 * lms_oracle.c -- CPU restatement of the reference's exact-LMS search.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links or calls
 * this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg load it, and only as the checker or
 * the timed CPU baseline.
 *
 * What it restates (reference = /root/reference/pkg/src/lmsline):
 *   - backend.py:111-122  _row_offsets / _decode_pair_ranks (row-major
 *                         upper-triangle pair ranks; walked directly here)
 *   - backend.py:190-207  _scan_rank_range: drop a_i == a_j pairs,
 *                         u = (b_i - b_j) / (a_i - a_j)
 *   - backend.py:125-179  _evaluate_pairs: cut values u*a_k - b_k with the
 *                         anchor copies snapped to v0 = a_i*u - b_i, k_lo /
 *                         k_hi rank counts, a FULL sort of the cut, down/up
 *                         q-windows, upward window wins ties, per-chunk
 *                         argmin by (h, i*n + j)
 *   - backend.py:182-187  _merge: strict lexicographic (h, i, j) minimum
 *   - backend.py:250-289  ParallelBackend: contiguous rank partitions over
 *                         worker threads, merged in partition order
 *   - geometry.py:182-218 bracelet_at (oracle_eval_vertex: explicit u, v)
 *
 * Arithmetic is IEEE fp64 with contraction disabled (build with
 * -ffp-contract=off): every product and difference is rounded separately,
 * exactly as numpy's elementwise ufuncs do.  The reference sorts the whole
 * cut (backend.py:151) and then reads two entries, vs[down] and vs[up]
 * (backend.py:156-157); this restatement obtains exactly those two order
 * statistics with std::nth_element over order-preserving uint64 keys (NaN
 * canonicalised to sort last, as np.sort does).  The selected values equal
 * the sorted array's entries at those indices (up to the sign of a zero,
 * and -0.0 == +0.0), and selection is O(n) instead of O(n log n), so the
 * timed CPU baseline is, if anything, faster than the reference's sort.
 *
 * Parity pinning: tests/test_oracle.py checks this file against the golden
 * vectors in tests/golden/ (generated from the reference itself by
 * tests/golden/make_golden.py).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>

extern "C" {

typedef struct oracle_candidate {
  double height;
  double u;
  double v_low;
  double v_high;
  int64_t i;
  int64_t j;
  int32_t found;
  int32_t pad;
} oracle_candidate;

static inline uint64_t key_of(double x) {
  uint64_t bits;
  if (x != x) x = NAN; /* canonical positive quiet NaN: sorts after +inf */
  memcpy(&bits, &x, 8);
  return (bits >> 63) ? ~bits : (bits | 0x8000000000000000ULL);
}

static inline double value_of(uint64_t key) {
  uint64_t bits = (key >> 63) ? (key & 0x7FFFFFFFFFFFFFFFULL) : ~key;
  double x;
  memcpy(&x, &bits, 8);
  return x;
}

/* keys[0..n) <- order-preserving keys of vals; returns the value at sorted
 * index k1 and k2 (k1 <= k2 not required; both in [0, n)). */
static void select_two(const double* vals, int64_t n, uint64_t* keys, int64_t k1, int64_t k2,
                       double* v1, double* v2) {
  for (int64_t k = 0; k < n; ++k) keys[k] = key_of(vals[k]);
  std::nth_element(keys, keys + k1, keys + n);
  *v1 = value_of(keys[k1]);
  if (k2 == k1) {
    *v2 = *v1;
  } else if (k2 < k1) {
    std::nth_element(keys, keys + k2, keys + k1);
    *v2 = value_of(keys[k2]);
  } else {
    std::nth_element(keys + k1 + 1, keys + k2, keys + n);
    *v2 = value_of(keys[k2]);
  }
}

/* One anchored-window evaluation (backend.py:144-171 for one row, or
 * geometry.py:557-572 with the given snapped ordinate v0).  Returns 1 and
 * fills *out when the height is finite, else 0. */
static int eval_vertex(const double* a, const double* b, int64_t n, int64_t q, int64_t i,
                       int64_t j, double u, double v0, double* vals, uint64_t* keys,
                       uint64_t* tmp, oracle_candidate* out) {
  for (int64_t k = 0; k < n; ++k) {
    double p = u * a[k];
    vals[k] = p - b[k];
  }
  vals[i] = v0;
  vals[j] = v0;
  int64_t k_lo = 0, k_le = 0;
  for (int64_t k = 0; k < n; ++k) {
    k_lo += vals[k] < v0;
    k_le += vals[k] <= v0;
  }
  int64_t k_hi = k_le - 1;
  int64_t down = k_hi - (q - 1);
  int64_t up = k_lo + (q - 1);
  double v_down, v_up;
  (void)tmp;
  select_two(vals, n, keys, down >= 0 ? down : 0, up <= n - 1 ? up : n - 1, &v_down, &v_up);
  double h_down = down >= 0 ? v0 - v_down : INFINITY;
  double h_up = up <= n - 1 ? v_up - v0 : INFINITY;
  int use_up = h_up <= h_down;
  double h = use_up ? h_up : h_down;
  if (!isfinite(h)) return 0;
  out->height = h;
  out->u = u;
  out->i = i;
  out->j = j;
  out->v_low = use_up ? v0 : v_down;
  out->v_high = use_up ? v_up : v0;
  out->found = 1;
  out->pad = 0;
  return 1;
}

/* (h, i, j) strict lexicographic less-than, IEEE equality on h (so -0.0 and
 * +0.0 tie), as Python's tuple comparison in backend.py:185. */
static inline int cand_less(const oracle_candidate* x, const oracle_candidate* y) {
  if (x->height < y->height) return 1;
  if (x->height > y->height) return 0;
  if (x->i != y->i) return x->i < y->i;
  return x->j < y->j;
}

static void merge_into(oracle_candidate* best, const oracle_candidate* cand) {
  if (!cand->found) return;
  if (!best->found || cand_less(cand, best)) *best = *cand;
}

/* Row of pair rank r: offsets[i] = i*(n-1) - i*(i-1)/2 (backend.py:111-116). */
static inline int64_t row_offset(int64_t n, int64_t i) { return i * (n - 1) - i * (i - 1) / 2; }

static void decode_rank(int64_t n, int64_t r, int64_t* pi, int64_t* pj) {
  /* binary search the row offsets, as np.searchsorted(side="right") - 1 */
  int64_t lo = 0, hi = n - 2;
  while (lo < hi) {
    int64_t mid = (lo + hi + 1) / 2;
    if (row_offset(n, mid) <= r) lo = mid;
    else hi = mid - 1;
  }
  *pi = lo;
  *pj = r - row_offset(n, lo) + lo + 1;
}

/* _scan_rank_range (backend.py:190-207) over [r0, r1). */
static void scan_ranks(const double* a, const double* b, int64_t n, int64_t q, int64_t r0,
                       int64_t r1, oracle_candidate* best) {
  memset(best, 0, sizeof(*best));
  if (r0 >= r1) return;
  double* vals = (double*)malloc(sizeof(double) * n);
  uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * n);
  uint64_t* tmp = (uint64_t*)malloc(sizeof(uint64_t) * n);
  int64_t i, j;
  decode_rank(n, r0, &i, &j);
  for (int64_t r = r0; r < r1; ++r) {
    double da = a[i] - a[j];
    if (da != 0.0) {
      double u = (b[i] - b[j]) / (a[i] - a[j]);
      double p = a[i] * u;
      double v0 = p - b[i];
      oracle_candidate c;
      if (eval_vertex(a, b, n, q, i, j, u, v0, vals, keys, tmp, &c)) merge_into(best, &c);
    }
    if (++j == n) {
      ++i;
      j = i + 1;
    }
  }
  free(vals);
  free(keys);
  free(tmp);
}

typedef struct scan_job {
  const double* a;
  const double* b;
  int64_t n, q, r0, r1;
  oracle_candidate best;
} scan_job;

static void* scan_job_run(void* p) {
  scan_job* job = (scan_job*)p;
  scan_ranks(job->a, job->b, job->n, job->q, job->r0, job->r1, &job->best);
  return NULL;
}

/* minimum_bracelet over pair ranks [r0, r1) with `threads` contiguous
 * partitions (ParallelBackend, backend.py:264-289).  Returns 0 on success,
 * -1 on invalid arguments. */
int oracle_min_bracelet(const double* a, const double* b, int64_t n, int64_t q, int64_t r0,
                        int64_t r1, int threads, oracle_candidate* out) {
  memset(out, 0, sizeof(*out));
  int64_t total = n * (n - 1) / 2;
  if (n < 2 || q < 1 || r0 < 0 || r1 > total || r0 > r1 || threads < 1) return -1;
  int64_t span = r1 - r0;
  if (span == 0) return 0;
  if (threads > span) threads = (int)span;
  int64_t size = (span + threads - 1) / threads;
  scan_job* jobs = (scan_job*)calloc((size_t)threads, sizeof(scan_job));
  pthread_t* tids = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  int started = 0;
  for (int t = 0; t < threads; ++t) {
    int64_t s = r0 + t * size;
    if (s >= r1) break;
    jobs[t].a = a;
    jobs[t].b = b;
    jobs[t].n = n;
    jobs[t].q = q;
    jobs[t].r0 = s;
    jobs[t].r1 = s + size < r1 ? s + size : r1;
    if (threads == 1) {
      scan_job_run(&jobs[t]);
    } else {
      pthread_create(&tids[t], NULL, scan_job_run, &jobs[t]);
    }
    started++;
  }
  for (int t = 0; t < started; ++t) {
    if (threads != 1) pthread_join(tids[t], NULL);
    merge_into(out, &jobs[t].best);
  }
  free(jobs);
  free(tids);
  return 0;
}

/* Per-vertex anchored windows at explicit (i, j, u, v): bracelet_at
 * (geometry.py:182-218) when v is given, _evaluate_pairs' row semantics
 * (v0 = a_i*u - b_i, backend.py:144) when v == NULL.  out[k].found = 0 when
 * no window fits. */
int oracle_eval_vertices(const double* a, const double* b, int64_t n, int64_t q,
                         const int64_t* ii, const int64_t* jj, const double* uu,
                         const double* vv, int64_t m, oracle_candidate* out) {
  if (n < 2 || q < 1) return -1;
  double* vals = (double*)malloc(sizeof(double) * n);
  uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * n);
  uint64_t* tmp = (uint64_t*)malloc(sizeof(uint64_t) * n);
  for (int64_t s = 0; s < m; ++s) {
    double u = uu[s];
    double v0;
    if (vv) {
      v0 = vv[s];
    } else {
      double p = a[ii[s]] * u;
      v0 = p - b[ii[s]];
    }
    memset(&out[s], 0, sizeof(out[s]));
    eval_vertex(a, b, n, q, ii[s], jj[s], u, v0, vals, keys, tmp, &out[s]);
  }
  free(vals);
  free(keys);
  free(tmp);
  return 0;
}

/* Per-vertex h for EVERY pair rank in [r0, r1) (NaN-free: +inf when no
 * finite window or when a_i == a_j).  Test helper for distribution checks. */
int oracle_all_heights(const double* a, const double* b, int64_t n, int64_t q, int64_t r0,
                       int64_t r1, double* h_out) {
  double* vals = (double*)malloc(sizeof(double) * n);
  uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * n);
  uint64_t* tmp = (uint64_t*)malloc(sizeof(uint64_t) * n);
  int64_t i, j;
  decode_rank(n, r0, &i, &j);
  for (int64_t r = r0; r < r1; ++r) {
    h_out[r - r0] = INFINITY;
    if (a[i] - a[j] != 0.0) {
      double u = (b[i] - b[j]) / (a[i] - a[j]);
      double p = a[i] * u;
      double v0 = p - b[i];
      oracle_candidate c;
      if (eval_vertex(a, b, n, q, i, j, u, v0, vals, keys, tmp, &c)) h_out[r - r0] = c.height;
    }
    if (++j == n) {
      ++i;
      j = i + 1;
    }
  }
  free(vals);
  free(keys);
  free(tmp);
  return 0;
}

}  // extern "C"
