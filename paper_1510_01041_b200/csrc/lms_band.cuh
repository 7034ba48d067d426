// lms_band.cuh -- slope-band pruning stage (lms_band.cu), host interface.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "lms_kernels.cuh"

namespace lmsb {

// Lines per fit the band stage handles (the sorted keys of a band live in
// shared memory; member vertices pack (i, j) into 16 + 16 bits).
constexpr int kBandMaxN = 16384;
// Lines per fit of the large-n band path (global segmented sorts for the
// bounds, 16-bit quantised keys in the filter; pair indices pack 16 + 16 bits).
constexpr int kBandMaxBigN = 65536;
// Most bands per fit (the collect kernel keeps K boundaries in shared memory).
constexpr int kBandMaxK = 16384;

struct BandFit {
  const double* a;  // the fit's lines (input order)
  const double* b;
  int64_t n, q;
  int64_t R0, span;  // pair ranks [R0, R0 + span) searched
  int64_t P0, pspan; // plan range [P0, P0 + pspan): slope samples, band boundaries and seed
                     // pairs (the search range, unless one shard of a sharded solve)
  double c;          // centre of the a-range
  double dev;        // >= max_k |a_k - c|
  double amax, bmax;
  const double2* ab;  // the lines interleaved (a_k, b_k): one 16-byte load per line
};

// Device scratch of one banded solve.
struct BandWork {
  int64_t S;  // slope samples
  int K;      // bands (>= 3)
  float* sample;          // S keys in sample order
  float* sample_sorted;   // S
  unsigned long long* nvalid;
  float* bounds;          // K - 1
  unsigned* sample_counts;// K
  uint8_t* flag;          // K: band selected (seeds)
  const int16_t* slot;    // K + 1: grouping slot of every collected band (-1: not
                          // collected; entry K: the beyond-range vertices)
  int nslot;              // slots (collected bands + 1)
  uint32_t* ckeys;        // collected (band, packed i<<16|j), capacity cap
  uint32_t* cvals;
  uint32_t* ckeys_alt;    // grouped copies
  uint32_t* members;
  unsigned long long* ncollect;
  int64_t* start;         // K + 1: members of band k are [start[k], end[k]); band K =
  int64_t* end;           //        vertices beyond the fp32 key range
  void* temp;
  size_t temp_bytes;
};

// keys kept around each end of a band's narrowest q-window (2 * kEdge per band)
constexpr int kEdge = 5;

// Slope runs of the flagged bands (collect pre-test), at most kMaxRuns: fp32
// bounds widened by 2^-18 relative + 1e-37 and rounded outward (-inf / +inf:
// open end).
constexpr int kMaxRuns = 8;
struct BandRuns {
  int count;
  float lo[kMaxRuns], hi[kMaxRuns];
};

// Direct grouping of the collected vertices into sub-band regions.
struct BandDirect {
  int nadm;                   // admitted band entries
  const int32_t* list;        // nadm: their bands
  const int32_t* sb_first;    // nadm + 1: first sub-band of each entry
  int nsub;                   // inner sub-boundaries (sum of S_e - 1)
  float* sub;                 // nsub, filled by the collect launcher
  const int16_t* slot;        // K: admitted entry of a band, or -1
  int force_group;            // sub-band id of the beyond-range vertices
  unsigned long long* cursor; // groups: members written (may exceed cap)
  const int64_t* cap;         // groups: region capacity
  const int64_t* rstart;      // groups: region start in members
  uint32_t* members;
};

struct BandArgs {
  int K;
  int band0;                  // bound launch (mode 0): first band, block b bounds band0 + b
  const int32_t* band_ids;    // optional: block b bounds band_ids[band0 + b] (< 0: none)
  const float* bounds;
  const int64_t* start;
  const int64_t* end;
  const uint32_t* members;
  const int32_t* list;        // filter: groups to process (bands, or sub-bands with group_band)
  const int32_t* group_band;  // optional: band of every group
  int nlist;
  int64_t chunk;              // filter: members per CTA
  // sorted keys of every inner band at its centre slope, row b at
  // bkeys + b * bkeys_ld: written by the bound kernel when non-null, read by
  // the filter (no per-chunk sort) when non-null
  float* bkeys;
  int64_t bkeys_ld;
  double bkeys_tau;  // filter: stored keys for bands with dev * (width) <= bkeys_tau * H
  int chunk_fixed;            // filter: 1 = groups are cut into `chunk`-member pieces only;
                              // 0 = adaptive (>= kMinChunks per group)
  // optional explicit chunk table (sub-band grouping, launch_band_pack_chunks):
  // chunk c = members [ctab[2c], ctab[2c + 1]) of band cband[c], *nctab chunks
  const int64_t* ctab;
  const int32_t* cband;
  const unsigned long long* nctab;
  unsigned long long* ticket;  // optional: chunk tickets of persistent filter CTAs (zeroed)
  int64_t* chunk_prefix;      // nlist + 1 scratch: first chunk of every listed band
  double* lb;                 // per band lower bound of any vertex height (-inf: unknown)
  double* wq;                 // per band narrowest q-window of the keys at the band centre
  float* edge;                // per band 2 * 5 keys around the ends of that window (optional)
  // large n (filter): slices of up to `slice` consecutive members of each
  // listed group, each with its own sorted keys at its own centre slope
  int64_t slice;              // members per slice (a multiple of chunk)
  int64_t* slice_prefix;      // nlist + 1: first slice of every listed group
  double* slice_u;            // per slice: centre slope of its keys
  double* slice_wq;           // per slice: narrowest q-window of its sorted keys
  double* slice_kmin;         // per slice: smallest key and bin width of its bin table
  double* slice_res;
  unsigned* slice_ptab;       // per slice: bin table (band_slice_table_kernel)
  const uint8_t* narrow;      // optional, per band: 1 = one slice for the whole band
  // optional: lower bound of the narrowest q-window of the lines' slopes a_k
  // (line_wqa_kernel); every band bound is raised to the slope bound
  // min |u| * W_q(a) - 2 bmax (slope_lb)
  const double* wqa;
  const lms_candidate* best;  // the fit's current best record (H)
  // bounds (mode 0) in two phases: 1 = bands whose slope bound is positive
  // only get it (lb = slope bound, wq = inf: no seeds from them); 2 = after
  // the seeds, exactly those bands, bounded fully unless the slope bound
  // already exceeds H; 0 = one phase
  int defer;
  int64_t* out_ranks;
  int32_t* out_fits;
  int32_t fit;
  unsigned long long* out_count;
};

// fp32 exact-slope window counts of the band filter's survivors
struct BandCount {
  float2* lines;  // n scratch: (fl32(a_k - c), fl32(b_k))
  const lms_candidate* best;
  const int64_t* in_ranks;
  const unsigned long long* in_count;
  int64_t* out_ranks;
  int32_t* out_fits;
  int32_t fit;
  unsigned long long* out_count;
  bool make_lines;      // fill `lines` first
};

// large-n bounds: keys of `batch` bands at a time in global memory
struct BandBig {
  int batch;
  float* keys;      // batch * n
  float* keys_alt;  // batch * n
  float* store;     // K * n: every band's sorted keys, kept for the filter
  int64_t* seg;     // batch + 1
  void* temp;
  size_t temp_bytes;
};
size_t band_big_sort_temp_bytes(int nb, int64_t n);
// bounds (and stored sorted keys) of bands [k0, k1), or of bands ids[k0 .. k1)
// when ids (device) is given
int launch_band_bound_big(const BandFit& bf, const BandArgs& ba, const BandBig& bg, int k0,
                          int k1, const int32_t* ids, cudaStream_t st);
// large n: sorted keys (store, nslices_max * n) of every slice of the listed
// groups at the slice's centre slope (midpoint of its first and last member's
// slopes); slices past the real count are empty segments
size_t band_slice_sort_temp_bytes(int64_t nslices_max, int64_t n);
constexpr int64_t kSliceTableRow = 32768 + 4;  // unsigned entries per slice (kSliceRow)
int launch_band_slices(const BandFit& bf, const BandArgs& ba, int64_t nslices_max, float* keys,
                       float* store, int64_t* seg_begin, int64_t* seg_end, void* temp,
                       size_t temp_bytes, cudaStream_t st);
void launch_band_filter_big(const BandFit& bf, const BandArgs& ba, const float* store, int grid,
                            cudaStream_t st);

size_t band_sample_temp_bytes(int64_t S);
// The slope-sample sort over the whole GPU (lms_samplesort.cu): keys[0, S)
// ascending into out; scratch of sample_sort_scratch_bytes(S).  Used by
// launch_band_sample unless LMSB_SAMPLE_SORT=0 (CUB's device radix sort).
size_t sample_sort_scratch_bytes(int64_t S);
// The same bucket sort per segment (segments keys[seg_b[y], seg_e[y]) or
// [y * max_len, (y + 1) * max_len)), all segments in the same launches.
size_t seg_bucket_sort_scratch_bytes(int64_t total, int nseg, int64_t max_len);
int launch_seg_bucket_sort(const float* keys, float* out, int64_t total, int nseg,
                           int64_t max_len, const int64_t* seg_b, const int64_t* seg_e,
                           void* scratch, size_t bytes, cudaStream_t st);
// the bucket sort for the large-n segmented sorts when LMSB_SEG_BUCKET=1 (opt-in)
bool use_seg_bucket();
int launch_sample_sort(const float* keys, float* out, int64_t S, void* scratch, size_t bytes,
                       cudaStream_t st);
// Segmented ascending sort of fp32 keys, one 8-CTA cluster per segment
// (lms_segsort.cu): segment s is in[seg_b[s] .. seg_e[s]) (or [s * stride,
// (s + 1) * stride) without seg_b), written to the same positions of out.
// seg_sort_fits(L): segments of L keys are supported (L <= 65,536).
bool seg_sort_fits(int64_t max_len);
int launch_seg_sort(const float* in, float* out, int64_t stride, int nseg, const int64_t* seg_b,
                    const int64_t* seg_e, cudaStream_t st);
// the cluster sort or the CUB device sorts for `nseg` segments of at most
// max_len keys (LMSB_SEG_SORT, lms_band.cu)
bool use_seg_sort(int64_t max_len, int64_t nseg);
size_t band_group_temp_bytes(int64_t m);
size_t band_collect_smem(int K);
int launch_band_sample(const BandFit& bf, const BandWork& w, int sms, cudaStream_t st);
// *out = a lower bound of the narrowest window of q of the lines' slopes a_k
// (binned, one CTA)
void launch_line_wqa(const BandFit& bf, double* out, cudaStream_t st);
// mode 0: grid = bands [ba.band0, ba.band0 + grid) (their lower bounds); mode 1: grid >=
// chunks of the listed bands
void launch_band(const BandFit& bf, const BandArgs& ba, int mode, int grid, cudaStream_t st);
// coarse (sort-free) lower bounds of bands [ba.band0, ba.band0 + grid): binned keys
void launch_band_coarse(const BandFit& bf, const BandArgs& ba, int grid, cudaStream_t st);
// ab[k] = (a[k], b[k]), k < n (BandFit::ab)
void launch_band_interleave(const double* a, const double* b, int64_t n, double2* ab,
                            cudaStream_t st);
// the T bands of [k0, k1) (or of ids[k0 .. k1) when ids is given; entries < 0
// skipped) with the narrowest finite q-windows into list[0 .. T) (-1: none),
// flagged in flag[0 .. K) (cleared first); T <= 64
void launch_band_top(const double* wq, int k0, int k1, int K, int T, int32_t* list, uint8_t* flag,
                     cudaStream_t st, const int32_t* ids = nullptr);
// pairs of lines at the ends of the listed bands' narrowest q-windows
void launch_band_edge_seeds(const BandFit& bf, const BandArgs& ba, const int32_t* bands, int nb,
                            int64_t* ranks, int32_t* fits, int64_t cap,
                            unsigned long long* count, cudaStream_t st);
// the same for the T bands with the narrowest windows, each CTA of a K grid
// deciding whether its band is one of them (flag[] zeroed, then set for them)
void launch_band_edge_seeds_top(const BandFit& bf, const BandArgs& ba, int T, uint8_t* flag,
                                int64_t* ranks, int32_t* fits, int64_t cap,
                                unsigned long long* count, cudaStream_t st);
void launch_band_seeds(const BandFit& bf, const BandWork& w, int64_t* ranks, int32_t* fits,
                       int32_t fit, int64_t cap, unsigned long long* count, cudaStream_t st);
void launch_band_collect(const BandFit& bf, const BandWork& w, const BandRuns& runs, int64_t cap,
                         int sms, cudaStream_t st);
// group the collected vertices by slot: full_order sorts by (slot, slope
// position) (radix sort), else buckets of (slot, top 8 slope bits)
int launch_band_group(const BandWork& w, int64_t m, bool full_order, cudaStream_t st);
constexpr int kSubMaxGroups = 1 << 14;  // groups of launch_band_group_sub


// Sub-band grouping (the default for the sweep collect at n <= kBandMaxN):
// inner sub-band boundaries of every admitted band from its sorted samples
// (band_subbounds_kernel), then a counting sort of the collected members by
// their group key (SweepArgs::sub_first): members of a group are contiguous,
// unordered inside it.  m: the device member count (clamped to cap); counts,
// cursor: ngroups scratch each; start / end: ngroups group ranges.
void launch_band_subbounds(const BandWork& w, const int32_t* list, const int32_t* sb_first,
                           int nadm, float* sub, cudaStream_t st, const int* dnadm = nullptr);
int launch_band_group_sub(const uint32_t* keys, const uint32_t* vals,
                          const unsigned long long* m, int64_t cap, int ngroups,
                          unsigned long long* counts, unsigned long long* cursor, int64_t* start,
                          int64_t* end, uint32_t* members, cudaStream_t st,
                          const int* dngroups = nullptr);
// filter chunks of the sub-band groups: per admitted slot e (groups
// sb_first[e] .. sb_first[e + 1] - 1, contiguous in slope and in memory)
// consecutive groups packed greedily into chunks of <= chunk members, a
// larger group split evenly (chunk_one members for a one-group slot); ctab /
// cband / nctab as BandArgs
void launch_band_pack_chunks(const int32_t* sb_first, int nslot, const int64_t* gstart,
                             const int64_t* gend, const int32_t* gband, int64_t chunk,
                             int64_t chunk_one, int64_t* ctab, int32_t* cband,
                             unsigned long long* nctab, cudaStream_t st,
                             const int* dnslot = nullptr);
size_t band_direct_smem(int K, int nsub, int nadm);
void launch_band_collect_direct(const BandFit& bf, const BandWork& w, const BandRuns& runs,
                                const BandDirect& dg, int sms, cudaStream_t st);
void launch_band_count(const BandFit& bf, const BandCount& bc, int sms, cudaStream_t st);
// exact pass-0 screen (fp64, the reference's arithmetic) of bc.in_ranks[0 ..
// *bc.in_count) against the record bc.best: the vertices the exact select
// would not prune go to bc.out_*; lines from bf.ab
void launch_band_exact_prepass(const BandFit& bf, const BandCount& bc, int sms, cudaStream_t st);
// the same screen with the lines split over several CTAs per 32-vertex tile
// (few survivors: the whole GPU busy); gcnt: 2 counters per survivor, zero
// on entry and left zero
void launch_band_prepass_split(const BandFit& bf, const BandCount& bc, unsigned* gcnt, int sms,
                               cudaStream_t st);

// ---- output-sensitive collect (lms_sweep.cu): the vertices of each admitted
// slope run as the inversions between the lines' orders at its two ends
struct SweepEnd {
  double s;    // kind 0: abscissa of the sort
  double fin;  // (unused: equal slopes at an infinite end tie-break by line id)
  int kind;    // 0 finite, 1 -inf, 2 +inf, 3 sort by slope a
  int pad;
};
struct SweepSort {  // ping-pong (key, line id) buffers, nseg * n each
  uint64_t* k1[2];
  uint32_t* idx[2];
  int cur;  // buffer holding the sorted segments
  // device-planned sweep (band_plan_kernel): the run count is read on the
  // device; segments 2r, 2r + 1 for runs r < *dnr of nr_max, the slope
  // segment at 2 * nr_max, the rest skipped (null: every segment is live)
  const int32_t* dnr;
  int nr_max;
};
struct SweepArgs {
  const float* bounds;   // K - 1 band boundaries
  int K;
  const int16_t* slot;   // K + 1 grouping slots (-1: not collected)
  int nruns;
  const int32_t* run_k0;  // per run: first and last band
  const int32_t* run_k1;
  const int32_t* P;       // nruns * n
  const int32_t* bmin;    // nruns * ceil(n / 32)
  const int32_t* suf;
  const uint32_t* idx;    // sorted segments (run r: 2r at s0', 2r + 1 at s1')
  const uint64_t* k1a;    // the slope-sorted segment (near-parallel pass), or null
  const uint32_t* idxa;
  double tau;             // pairs with 0 < |a_i - a_j| <= tau: near-parallel pass
  uint32_t* out_keys;
  uint32_t* out_vals;
  int64_t cap;
  unsigned long long* count;
  int smem_tables;        // (launcher) boundaries and slots staged in shared memory
  unsigned long long* dbg;  // optional: per run, pairs enumerated (LMSB_SWEEP_DEBUG)
  unsigned long long* raw;  // enumerated (run << 32 | pair) entries, raw_cap of them
  int64_t raw_cap;
  unsigned long long* raw_count;
  // optional sub-band grouping (launch_band_group_sub): the key of a member of
  // slot e is its sub-band group sub_first[e] + (number of the slot's inner
  // sub-band boundaries sub[sub_first[e] - e ...] <= fl32(u)); the
  // beyond-range pseudo slot gets group sub_first[nslot - 1].  null: the
  // (slot, slope position) key.
  const int32_t* sub_first;
  const float* sub;
  // device-planned sweep: run count and near-parallel threshold on the
  // device (nruns / tau are then the maxima / unused)
  const int32_t* dnr;
  const double* dtau;
  // deferred member count (no readback before the grouping): a raw-buffer
  // overflow is flagged here instead of raising `count` past the members
  // actually written (the grouping reads min(count, cap) of them)
  unsigned long long* raw_overflow;
};
size_t sweep_chunk_smem();
// sort nseg segments of the n lines by their end keys; returns launches
int launch_sweep_sort(const double2* ab, int n, const SweepEnd* ends, int nseg, SweepSort& ss,
                      int sms, cudaStream_t st);
// P, block minima and suffix minima of every run (pos: nruns * n scratch)
void launch_sweep_prepare(int n, int nruns, const SweepSort& ss, int32_t* pos, int32_t* P,
                          int32_t* bmin, int32_t* suf, int sms, cudaStream_t st);
// enumerate and classify; members appended to out_keys / out_vals (count may exceed cap)
void launch_sweep_emit(const BandFit& bf, const SweepArgs& sa, int sms, cudaStream_t st);

// Device-side plan of a band search after the seeds (band_plan_kernel): the
// admitted bands, grouping slots, sweep runs and ends, sub-band groups --
// what band_solve's host planning computes from the readback, without the
// round trip.  Counts live in DevPlanHdr; arrays in the pointers below.
constexpr int kPlanMaxRuns = 16;  // = kSweepMaxRuns (lms_engine.cu)
struct DevPlanHdr {
  int nadm;      // admitted bands (the outer bands included when admitted)
  int nslot;     // nadm + 1 (the beyond-range pseudo band last)
  int nr;        // sweep runs (<= kPlanMaxRuns)
  int ngroups;   // sub-band groups (nadm .. kSubMaxGroups)
  int bail;      // 1: the plan cannot run on the device (the host plans instead)
  int pad;
  double H;      // the seed height the bands were admitted against
  double tau;    // near-parallel threshold of the sweep
  unsigned long long est;  // sampled members of the admitted bands (+2 each)
};
struct DevPlan {
  DevPlanHdr* hdr;
  int32_t* list;    // K + 1: slot -> band (pseudo band K last)
  int16_t* slot;    // K + 1: band -> slot (-1)
  int32_t* ident;   // K + 1: 0, 1, 2, ...
  SweepEnd* ends;   // 2 * kPlanMaxRuns + 1 (slope segment last)
  int32_t* rk;      // 2 * kPlanMaxRuns: run_k0 [0, 16), run_k1 [16, 32)
  int32_t* sbf;     // K + 2: first group of every slot
  int32_t* gband;   // kSubMaxGroups: band of every group
};
// one CTA; K <= kPlanMaxK
constexpr int kPlanMaxK = 4096;
void launch_band_plan(const BandFit& bf, const BandWork& w, const double* lb,
                      const lms_candidate* best, int K, int sub_samples, double bkeys_tau,
                      const DevPlan& dp, cudaStream_t st);

}  // namespace lmsb
