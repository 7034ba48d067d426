/*
 * lms_b200.h -- C ABI of the B200-native exact 2D LMS engine.
 *
 * Plain pointers and sizes only; no torch or CUDA types cross this boundary.
 * Every entry point returns LMS_OK (0) on success or a negative LMS_ERR_*
 * code; lms_last_error() gives the message of the calling thread's last
 * failure.  Host buffers are owned by the caller and copied by the library;
 * the *_dev entry points take device pointers already resident in HBM.
 *
 * Each entry point replaces one seam of the reference package
 * (/root/reference/pkg/src/lmsline, cited file:line):
 *
 *   lms_min_bracelet_materialized_f64
 *                             minimum_bracelet(..., materialize=True), i.e.
 *                             _materialized_inputs + _scan_materialized
 *                             (backend.py:210-231): the two-kernel flow
 *   lms_min_bracelet_f64      SequentialBackend/ParallelBackend.minimum_bracelet
 *                             (backend.py:239-247, 264-289) over a contiguous
 *                             pair-rank range, i.e. _scan_rank_range
 *                             (backend.py:190-207) for one partition
 *   lms_eval_vertices_f64     _evaluate_pairs per intersection
 *                             (backend.py:125-179) / bracelet_at
 *                             (geometry.py:182-218)
 *   lms_min_over_vertices_f64 run_phase2 / _scan_materialized
 *                             (backend.py:221-231, 321-354)
 *   lms_batched_f64           refine_lms per Hough peak (detect.py:134-153,
 *                             the per-peak loop of detect.py:184-213)
 *   lms_primal_brute_f64      oracle_lms, the primal brute force (solver.py:143-196)
 *   lms_hough_vote_u8         extract_points + hough_vote (hough.py:93-129)
 *   lms_hough_vote_points     hough_vote of a point list (hough.py:112-129)
 *   lms_hough_support         supporting_points (hough.py:171-184)
 *
 * Results are bit-identical to the reference's fp64 arithmetic: the winning
 * pair (i, j), u, v_low, v_high and height are the values the reference's
 * seq backend returns for the same input.
 */
#ifndef LMS_B200_H
#define LMS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LMS_OK 0
#define LMS_ERR_INVALID -1  /* bad argument (InvalidInputError on the Python side) */
#define LMS_ERR_CUDA -2     /* CUDA runtime failure */
#define LMS_ERR_NODEVICE -3 /* no CUDA device / device index out of range */
#define LMS_ERR_NOMEM -4    /* device allocation failed */
#define LMS_NOT_FITTED 1    /* lms_detect_supports_u8: a thinned support cannot be fitted (no fits run) */

/* CandidateRecord (backend.py:37-54) plus a found flag: found == 0 is the
 * reference's None ("no window fits"). 56 bytes. */
typedef struct lms_candidate {
  double height;
  double u;
  double v_low;
  double v_high;
  int64_t i;
  int64_t j;
  int32_t found;
  int32_t reserved;
} lms_candidate;

/* Counters of the last solve on a context (device-timed). */
typedef struct lms_stats {
  int64_t n;
  int64_t pairs;            /* pair ranks in the solved range */
  int64_t seed_vertices;    /* vertices evaluated exactly to seed the bound */
  int64_t filtered_vertices;/* vertices that went through the count filter */
  int64_t survivors;        /* vertices the filter passed to the exact select */
  int64_t line_evals;       /* vertex-line evaluations executed by the filter */
  int64_t launches;         /* kernels launched by the solve */
  int64_t chunks;
  float ms_total;           /* device time of the whole solve (CUDA events) */
  float ms_filter;          /* device time inside the filter kernels */
  float ms_exact;           /* device time inside seed + exact-select + reduce */
  float ms_bound_kernel;    /* the per-band bound kernel alone (band_bound_kernel) */
  /* slope-band stage (lms_band.cu); zero when the count filter ran instead */
  int64_t bands;            /* slope bands the fit's vertices were grouped into */
  int64_t bands_searched;   /* bands whose lower bound admitted the bound H */
  float ms_partition;       /* sample + band histogram + scatter */
  float ms_bound;           /* per-band sorted keys and lower bounds */
  float ms_band_filter;     /* chunk window counts + fp32 counts + exact survivors */
  float ms_collect;         /* the collect pass alone (last attempt) */
  double seed_height;       /* the bound H the band stage collected with */
  int64_t band_survivors;   /* collected vertices whose band window counts reached q */
  int64_t small_fits;       /* fits of the batch solved by the fused per-fit band kernel */
  int64_t direct_groups;    /* sub-band regions of the direct grouping (0: radix-sort path) */
  int64_t bands_refined;    /* bands whose coarse bound admitted H and got the exact bound */
  int64_t sweep_runs;       /* slope runs of the sweep collect (0: the pre-test pass ran) */
  float ms_filter_kernel;   /* the band filter kernel alone (band_filter / band_filter_big) */
  float ms_sweep_enum;      /* the sweep collect's enumeration kernels (enum + near-parallel) */
  float ms_hough_vote;      /* device detect: the vote kernel (lms_detect_peaks_u8) */
  float ms_hough_support;   /* device detect: support count + scan + write kernels */
} lms_stats;

/* Counters of the last call on `device`'s shared context (the one the
 * lms_* entry points without a context use). */
int lms_device_stats(int device, lms_stats* out);

/* Library identity and device discovery. */
int lms_version(void);
int lms_device_count(int* count);
const char* lms_last_error(void);

/* Exact LMS search over pair ranks [rank_begin, rank_end) of the row-major
 * upper triangle (rank 0 = (0,1)).  a, b: n dual-line coefficients (the
 * points' x and y, dualize geometry.py:141-144).  q in [2, n].
 * out->found == 0 when no pair in the range yields a finite window. */
int lms_min_bracelet_f64(const double* a, const double* b, int64_t n, int64_t q,
                         int64_t rank_begin, int64_t rank_end, int device, lms_candidate* out);

/* solve_lms on the device end to end (solver.py:115-140): the exact search
 * over all n(n-1)/2 pairs, then the fit's contact set -- indices k with
 * |x_k u - y_k - v_low| <= tol or |x_k u - y_k - v_high| <= tol, anchors
 * snapped, tol = GEOM_EPS max(1, max_k |x_k u - y_k|) -- ascending in
 * contacts[0 .. min(*ncontacts, cap)).  *ncontacts may exceed cap (call again
 * with more room).  Replaces the SequentialBackend.minimum_bracelet call plus
 * the numpy tail of solve_lms (solver.py:115-140, backend.py:234-247). */
int lms_solve_fit_f64(const double* a, const double* b, int64_t n, int64_t q, int device,
                      lms_candidate* out, int64_t* contacts, int64_t cap, int64_t* ncontacts);

/* The materialised two-kernel flow over the same rank range (materialize=True,
 * backend.py:210-231): K1 writes every non-parallel pair's (i, j, u), K2
 * evaluates every one exactly; no pruning filter.  Same record as
 * lms_min_bracelet_f64. */
int lms_min_bracelet_materialized_f64(const double* a, const double* b, int64_t n, int64_t q,
                                      int64_t rank_begin, int64_t rank_end, int device,
                                      lms_candidate* out);

/* Batched exact LMS (refine_lms over many Hough peaks, detect.py:134-153 /
 * the per-peak loop of detect.py:184-213): fit f uses points
 * [offsets[f], offsets[f+1]) of x / y with coverage q[f]; out[f] is the
 * minimum over all of the fit's pair ranks.  offsets[0] == 0. */
int lms_batched_f64(const double* x, const double* y, const int64_t* offsets, const int64_t* q,
                    int64_t nfits, int device, lms_candidate* out);
/* lms_batched_f64 plus the solve_lms tail on the device: contact_flags[k]
 * (one per point, offsets[nfits] of them) is 1 when point k touches its
 * fit's slab edges within GEOM_EPS max(1, max |cut|) (solver.py:122-140). */
int lms_batched_fit_f64(const double* x, const double* y, const int64_t* offsets, const int64_t* q,
                        int64_t nfits, int device, lms_candidate* out, uint8_t* contact_flags);

/* solve_lms over a list of point sets (solve_lms_batch; the reference's
 * per-peak refits, detect.py:184-213): set f is sets[f], counts[f] rows of
 * (x, y) fp64, row-major, coverage q[f].  The sets go up through pinned
 * staging filled by host threads (no concatenated host copy), are checked on
 * the device as solve_lms checks them (solver.py:67-80) -- status[f] = 0 ok,
 * 1 non-finite, 2 fewer than 3 points, 3 one distinct x, 4 q outside
 * [2, n]; any non-zero: LMS_NOT_FITTED, nothing solved -- then solved in one
 * batch; out[f] the record, each set's contact indices (solver.py:122-140)
 * ascending in contacts[contact_offsets[f] .. contact_offsets[f+1]),
 * *ncontacts in total (only written when <= contact_capacity). */
int lms_batched_fit_sets_f64(const double* const* sets, const int64_t* counts, const int64_t* q,
                             int64_t nfits, int device, int32_t* status, lms_candidate* out,
                             int64_t* contact_offsets, int32_t* contacts, int64_t contact_capacity,
                             int64_t* ncontacts);
/* Python-binding helper: data pointers and row counts of `count` numpy
 * arrays given by object address (id()), each checked to be a C-contiguous
 * (n, 2) array of 8-byte elements (the caller checks the dtype). */
int lms_ndarray_rows_f64(const uintptr_t* objs, int64_t count, const double** data, int64_t* rows);

/* oracle_lms (solver.py:143-196), the reference's independent primal brute
 * force: per pair slope, sorted intercepts, narrowest q-window (first
 * minimal); lexicographic (span, i, j) minimum.  out->height = span,
 * out->u = slope, out->v_low / v_high = the window's intercepts.  n <= 16384. */
int lms_primal_brute_f64(const double* x, const double* y, int64_t n, int64_t q, int device,
                         lms_candidate* out);

/* extract_points + hough_vote (hough.py:93-129): the lit pixels (value >=
 * threshold) of the height x width uint8 image, in row-major scan order,
 * vote once per theta bin; acc[n_rho * n_theta] (rho-major, as
 * HoughAccumulator.bins) receives the counts, *npoints the number of lit
 * pixels.  cos_t / sin_t are the cosines / sines of the theta bin centres
 * (np.cos / np.sin of np.radians, as hough.py:124-125).  The lit pixels stay
 * on the device for lms_hough_support. */
int lms_hough_vote_u8(const uint8_t* img, int64_t height, int64_t width, int threshold,
                      const double* cos_t, const double* sin_t, int64_t n_theta, double rho_max,
                      double delta_rho, int64_t n_rho, int device, int64_t* acc,
                      int64_t* npoints);
/* hough_vote over explicit points (x[k], y[k]) (hough.py:112-129). */
int lms_hough_vote_points(const double* x, const double* y, int64_t npts, const double* cos_t,
                          const double* sin_t, int64_t n_theta, double rho_max, double delta_rho,
                          int64_t n_rho, int device, int64_t* acc);
/* supporting_points (hough.py:171-184) of the points of the last vote on
 * `device`, for npeaks peaks: peak p's members are the points whose rho bin
 * at (cos_p[p], sin_p[p]) (math.cos / math.sin of math.radians, as
 * hough.py:181-183) equals rbin_p[p], in scan order, written to
 * out[offsets[p] .. offsets[p+1]) as pixel indices (image votes) or point
 * ordinals (point votes).  offsets has npeaks + 1 entries and is always
 * filled; LMS_ERR_INVALID when the members exceed `capacity`. */
int lms_hough_support(const double* cos_p, const double* sin_p, const int64_t* rbin_p,
                      int64_t npeaks, double rho_max, double delta_rho, int64_t n_rho, int device,
                      int64_t* offsets, int64_t* out, int64_t capacity);
/* lms_hough_support with the ids written as int32 (half the download; the
 * ids are narrowed on the device).  LMS_ERR_INVALID when an id of the last
 * vote could exceed INT32_MAX (more than 2^31 pixels or points). */
int lms_hough_support_i32(const double* cos_p, const double* sin_p, const int64_t* rbin_p,
                          int64_t npeaks, double rho_max, double delta_rho, int64_t n_rho,
                          int device, int64_t* offsets, int32_t* out, int64_t capacity);

/* Anchored window at each explicit intersection (i[k], j[k], u[k]).  When v
 * is non-NULL the anchors are snapped to v[k] (bracelet_at); when NULL to
 * a[i]*u - b[i] (_evaluate_pairs).  With v non-NULL an index of -1 snaps no
 * line (the caller has already placed its anchor lines at v).  out: m
 * records. */
int lms_eval_vertices_f64(const double* a, const double* b, int64_t n, int64_t q,
                          const int64_t* i, const int64_t* j, const double* u, const double* v,
                          int64_t m, int device, lms_candidate* out);

/* Lexicographic (height, i, j) minimum over explicit intersections
 * (v0 = a[i]*u - b[i]); out->found == 0 when none fits. */
int lms_min_over_vertices_f64(const double* a, const double* b, int64_t n, int64_t q,
                              const int64_t* i, const int64_t* j, const double* u, int64_t m,
                              int device, lms_candidate* out);

/* Context API: keeps lines, scratch and a stream resident on one device. */
typedef struct lms_ctx lms_ctx;
int lms_ctx_create(int device, lms_ctx** out);
int lms_ctx_destroy(lms_ctx* ctx);
/* Copy n lines host -> device (H2D on the context stream). */
int lms_ctx_upload(lms_ctx* ctx, const double* a, const double* b, int64_t n);
/* Use n lines already resident on this context's device. */
int lms_ctx_bind_dev(lms_ctx* ctx, const double* d_a, const double* d_b, int64_t n);
/* Solve over [rank_begin, rank_end) of the bound lines; blocks until done. */
int lms_ctx_solve(lms_ctx* ctx, int64_t q, int64_t rank_begin, int64_t rank_end,
                  lms_candidate* out);
/* Sharded band search (multi-GPU, one context per GPU).
 * Replaces the per-partition _scan_rank_range call of a multi-worker run
 * (backend.py:190-207, partitions backend.py:84-92) when the partitions are
 * GPUs that can exchange a small per-band table.  Shard s of S searches the
 * pair ranks [lo, hi) of the ceil split of [0, n(n-1)/2) (distributed.partition).
 *   1. lms_ctx_shard_plan: every shard samples the whole pair space (the same
 *      samples, band boundaries and K on every shard) and bounds only its slice
 *      of the K slope bands, bands shard, shard + nshards, shard + 2 nshards,
 *      ... (*nslice of them; interleaved, so the bands near the optimum slope
 *      spread over all shards): per band its lower bound, narrowest q-window
 *      and LMS_BAND_EDGE_KEYS window-edge keys, written in that order to the
 *      caller's arrays (capacity bands).  *seed is the
 *      best exactly evaluated vertex at the ends of the slice's narrowest
 *      windows (any vertex of the fit; not found if none).  nbands = 0: the
 *      fit is not searched by bands; skip the exchange.
 *   2. the caller all-gathers the slices (NCCL over NVLink) into K-band arrays
 *      (band k is entry k / nshards of shard k % nshards's slice) and takes
 *      the lexicographic minimum of the seeds.
 *   3. lms_ctx_shard_search: starts from that seed (H = its height) and
 *      searches the shard's rank range against the full band table.  *out is
 *      the minimum over the shard's range and the seed (which may lie outside
 *      the range), so the lexicographic minimum of all shards' records is the
 *      fit's record (backend.py:182-187), bit-identical to one lms_ctx_solve
 *      over [0, n(n-1)/2).  A search on the context that ran the plan reuses
 *      the plan's samples and band boundaries. */
#define LMS_BAND_EDGE_KEYS 10
int lms_ctx_shard_plan(lms_ctx* ctx, int64_t q, int32_t nshards, int32_t shard, int64_t capacity,
                       int64_t* nbands, int64_t* nslice, double* lower_bound, double* window,
                       float* edge_keys, lms_candidate* seed);
int lms_ctx_shard_search(lms_ctx* ctx, int64_t q, int32_t nshards, int32_t shard, int64_t nbands,
                         const double* lower_bound, const double* window, const float* edge_keys,
                         const lms_candidate* seed, lms_candidate* out);
/* Materialised two-kernel solve over the bound lines (see
 * lms_min_bracelet_materialized_f64). */
int lms_ctx_solve_materialized(lms_ctx* ctx, int64_t q, int64_t rank_begin, int64_t rank_end,
                               lms_candidate* out);
/* Batched solve over the bound lines (see lms_batched_f64). */
int lms_ctx_solve_batch(lms_ctx* ctx, const int64_t* offsets, const int64_t* q, int64_t nfits,
                        lms_candidate* out);
int lms_ctx_stats(const lms_ctx* ctx, lms_stats* out);
/* CUDA events on the context stream, for device timing around solves. */
int lms_ctx_event_record(lms_ctx* ctx, int slot);
int lms_ctx_event_elapsed_ms(lms_ctx* ctx, int slot0, int slot1, float* ms);
int lms_ctx_synchronize(lms_ctx* ctx);

/* Diagnostics: measured FP64 pipe issue rate of `device` (DFMA per second,
 * all SMs busy, 8 independent chains per thread).  bench.py's roofline
 * denominator for the FP64-bound filter kernel. */
int lms_probe_fp64_rate(int device, double* dfma_per_second);
/* Measured FP32 FMA lane rate (FFMA2 packed chains, all SMs busy): the
 * roofline denominator of the default FP32/FP16 count filter. */
int lms_probe_fp32_rate(int device, double* fma_lanes_per_second);
/* Diagnostics: the band stage's cluster segmented sort (lms_segsort.cu) on
 * host buffers: segment s = keys[seg_begin[s] .. seg_end[s]) sorted
 * ascending into the same positions of out (positions outside every segment
 * are left as in `keys`); segments of at most 65,536 keys.  Stands in for
 * the np.sort of the reference's cut rows (backend.py:199-203) in parity
 * tests of the sort itself. */
int lms_debug_seg_sort(int device, const float* keys, float* out, int64_t total, int32_t nseg,
                       const int64_t* seg_begin, const int64_t* seg_end);
/* Diagnostics: the band stage's slope-sample bucket sort (lms_samplesort.cu)
 * on a host buffer: keys[0, n) ascending into out. */
int lms_debug_sample_sort(int device, const float* keys, float* out, int64_t n);

/* ---- multi-GPU exact LMS: the vertex space of one fit
 * shared over several GPUs, one NCCL collective exchange of 56-byte records
 * before the search (the best seed) and one after it (the results).
 *
 * Sharded band search with band ownership: every shard bounds and seeds its
 * own interleaved slice of the slope bands, the seed records are
 * all-gathered, and each shard searches the vertices of its own bands that
 * the best seed cannot dismiss; the lexicographic (height, i, j) minimum of
 * the shards' records is the one-GPU record (backend.py:182-187).  Fits too
 * small for the band stage split the pair ranks into contiguous partitions
 * instead (BatchPlan.partitions, backend.py:84-92). */

/* In one process: shard r runs on devices[r] (one host thread per shard).
 * Distinct devices exchange through NCCL (ncclCommInitAll, ncclAllGather on
 * device buffers); shards sharing a device exchange through host memory.
 * Replaces ParallelBackend.minimum_bracelet's thread fan-out and merge
 * (backend.py:264-289). */
int lms_min_bracelet_multi(const double* a, const double* b, int64_t n, int64_t q,
                           int32_t nshards, const int32_t* devices, lms_candidate* out);
/* 1 when libnccl.so.2 could be loaded (its version in *version), else 0. */
int lms_nccl_available(int* version);
/* One process per GPU (torchrun): rank 0 makes the 128-byte NCCL unique id,
 * the caller broadcasts it, every rank binds a communicator to its context,
 * then lms_ctx_solve_distributed runs plan -> all-gather of seed records ->
 * own-band search -> all-gather of records -> minimum, same record on
 * every rank. */
int lms_nccl_unique_id(uint8_t* id);
int lms_ctx_comm_init(lms_ctx* c, int32_t nranks, int32_t rank, const uint8_t* id);
int lms_ctx_solve_distributed(lms_ctx* c, int64_t q, lms_candidate* out);
/* The own-band search of one shard after lms_ctx_shard_plan(c, q, nshards,
 * shard, ...) on the same context, with the best seed over all shards
 * (seed may be NULL).  Not banded (the plan reported no bands): the shard's
 * pair-rank partition. */
int lms_ctx_shard_search_owned(lms_ctx* c, int64_t q, int32_t nshards, int32_t shard,
                               const lms_candidate* seed, lms_candidate* out);

/* ---- detect_lines on the device, straight from the image (detect.py:156-214).
 * Phase 1: the uint8 image thresholded (>= threshold, hough.py:93-103) and
 * voted at the theta bin centres (cos_t/sin_t: np.cos/np.sin of the centres,
 * hough.py:112-129), then find_peaks (hough.py:132-168): 8-neighbour maxima
 * >= min_votes ordered by (-votes, rho_bin, theta_bin), at most max_peaks
 * (<= 64).  peaks[3k .. 3k+2] = (rho_bin, theta_bin, votes), *npeaks of
 * them; acc (n_rho * n_theta int64) optional.  n_rho * n_theta <= 16384,
 * n_theta <= 512, fewer than 2^31 pixels. */
int lms_detect_peaks_u8(const uint8_t* img, int64_t height, int64_t width, int threshold,
                        const double* cos_t, const double* sin_t, int64_t n_theta, double rho_max,
                        double delta_rho, int64_t n_rho, int64_t max_peaks, int64_t min_votes,
                        int device, int64_t* acc, int64_t* npoints, int64_t* peaks,
                        int64_t* npeaks);
/* Phase 2 on the peaks of the last phase 1 on this device (hold one lock
 * across both): every peak's support in scan order (supporting_points,
 * hough.py:171-184; cos_s/sin_s: math.cos/math.sin of every theta bin
 * centre) as int32 pixel ids in support_ids[support_offsets[k] ..
 * support_offsets[k+1]) (capacity entries; NULL: not downloaded); each
 * support thinned to support_cap (0: whole) by the stride (k m) // cap
 * (detect.py:118-131) in the axis-swapped frame of swap_t[theta_bin]
 * (detect.py:91-95), design_offsets (npeaks + 1) and the thinned
 * abscissa range abscissa_range[2k], [2k+1]; with fit != 0 the exact LMS
 * refit of every design with coverage q[k] (refine_lms, detect.py:134-153)
 * into records[k] and contact_flags (one per design point, the solve_lms
 * contact set, solver.py:122-140).  Returns LMS_NOT_FITTED (no fits run)
 * when a design has < 3 points, a single abscissa, or q[k] outside [2, n]. */
int lms_detect_supports_u8(const double* cos_s, const double* sin_s, const uint8_t* swap_t,
                           int64_t support_cap, const int64_t* q, int fit, int device,
                           int64_t* support_offsets, int32_t* support_ids, int64_t capacity,
                           int64_t* design_offsets, double* abscissa_range, lms_candidate* records,
                           uint8_t* contact_flags);

#ifdef __cplusplus
}
#endif

#endif /* LMS_B200_H */
