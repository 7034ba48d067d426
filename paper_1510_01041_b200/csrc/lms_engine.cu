// lms_engine.cu -- host orchestration of the exact-LMS search and the C ABI.
//
// A solve is a batch of fits (one large fit, or thousands of Hough-peak
// refits).  For every fit f with pair ranks [R0, R1) (a contiguous partition
// as BatchPlan.partitions, backend.py:84-92):
//   1. seed     exact-evaluate a stratified sample of its vertices and reduce
//               them to the fit's best record (its height is the bound H);
//               fits with at most kExhaustive pairs evaluate every vertex here
//   2. order    stream its lines far-first from the best line (lms_order.cu)
//   3. filter   all remaining fits' warp tasks in chunks through the count
//               filter (lms_filter32m.cu), H read per fit from device memory
//   4. exact    re-evaluate each chunk's survivors bit-exactly (lms_exact.cu)
//   5. reduce   per-fit lexicographic (height, i, j) minimum by 128-bit CAS,
//               tightening every fit's H for the next chunk.
// All launches are asynchronous on the context stream; the host
// synchronises once, when it reads the best records back.

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <condition_variable>
#include <atomic>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <string>
#include <vector>

#include "lms_band.cuh"
#include "lms_band_small.cuh"
#include "lms_common.cuh"
#include "lms_detect.cuh"
#include "lms_hough.cuh"
#include "lms_kernels.cuh"
#include "lms_nccl.cuh"
#include "lms_plan.cuh"
#include "lms_sets.cuh"
#include "lms_primal.cuh"

#define LMS_VERSION 2

namespace {

thread_local std::string g_last_error;

int set_error(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

#define CUDA_TRY(expr)                                                                   \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess) {                                                             \
      return set_error(_e == cudaErrorMemoryAllocation ? LMS_ERR_NOMEM : LMS_ERR_CUDA,   \
                       "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, \
                       __LINE__);                                                        \
    }                                                                                    \
  } while (0)

#define RC_TRY(expr)     \
  do {                   \
    int _rc = (expr);    \
    if (_rc) return _rc; \
  } while (0)

constexpr int64_t kSeedsMax = 2048;          // exact seed vertices per large fit
constexpr int64_t kSeedsMin = 64;            // ... per small fit
constexpr int64_t kSeedDivisor = 2048;       // seeds = span / kSeedDivisor, clamped
constexpr int64_t kExhaustive = 4096;        // fits this small skip the filter
constexpr int64_t kChunkVertices = 1 << 24;  // filter chunk (and survivor capacity)
constexpr int64_t kBandMinSpan = 3 << 19;    // smaller fits: seeds + count filter are faster
                                              // (measured crossover n ~ 1,800: 1.6 M pairs)
constexpr int kNumEvents = 16;

// bumped by every device allocation: a captured CUDA graph holds buffer
// addresses, so it is valid only while the epoch it was captured at lasts
std::atomic<uint64_t> g_buf_epoch{0};

template <typename T>
int grow(T** ptr, int64_t* cap, int64_t need) {
  if (need <= *cap) return LMS_OK;
  g_buf_epoch.fetch_add(1);
  if (*ptr) cudaFree(*ptr);
  *ptr = nullptr;
  *cap = 0;
  int64_t c = std::max<int64_t>(need, 64);
  CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(ptr), sizeof(T) * c));
  *cap = c;
  return LMS_OK;
}

// Vertices per band: smaller bands for small fits, where the per-band sort
// is cheap and the tighter bounds prune more (n = 2,048-3,000: 196,608 ->
// 65,536 is 5-9 % faster; n = 4,096: 98,304 is 11 % faster; n = 8,192:
// 131,072 is 3-7 % faster).
int64_t band_size(int64_t knob, int64_t n) {
  if (knob > 0) return knob;
  return n <= 3072 ? 65536 : n <= 5120 ? 98304 : n <= 12288 ? 131072 : 196608;
}

// Most slope runs of the sweep collect (two sorts of the n lines each).
constexpr int kSweepMaxRuns = 16;
// Auto mode: sweep collect from this many lines.  With the hybrid grouping
// (no radix sort of the members) the sweep wins from the band stage's
// threshold up (fit times, sweep vs pre-test: n = 2,500 0.62 vs 0.63 ms,
// 5,000 0.62 vs 0.67, 8,192 0.71 vs 0.84, 11,000 0.84 vs 0.98).
constexpr int64_t kSweepMinN = 2048;

// Large-n band size (vertices per band = mult * n): fewer, wider bands pay
// once n > ~36 k (config 3, n = 65,536: 8 -> 18.6 ms, 16 -> 17.9, 32 ->
// 16.5; n = 40,000: 8 -> 7.35, 16 -> 6.98; n = 20,000-32,768: 8 best).
int64_t big_band_mult(int64_t knob, int64_t n) {
  if (knob > 0) return knob;
  return n >= 57344 ? 32 : n > 36864 ? 16 : 8;
}

template <typename T>
struct DevBuf {
  T* p = nullptr;
  int64_t cap = 0;
  int need(int64_t n) { return grow(&p, &cap, n); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

struct HostFit {
  int64_t off, n, q, r0, r1;
};

// One shard of a sharded band search (lms_ctx_shard_plan / _search): the
// band plan (samples, boundaries, seeds) covers the whole pair space
// [P0, P1); the shard bounds only its slice of the bands (plan: bands
// shard, shard + nshards, ...) or
// takes every band's bound from the caller (search) and searches its own
// rank range.
struct ShardSpec {
  int mode = 0;          // 1 plan, 2 search (rank range), 3 search (own bands)
  int64_t P0 = 0, P1 = 0;
  int nshards = 1, shard = 0;
  int64_t K = 0, k0 = 0, k1 = 0;  // plan: set by band_solve (k0 = k1 = bands in the slice)
  int64_t cap = 0;                // plan: capacity of the output slice
  double* lb_out = nullptr;
  double* wq_out = nullptr;
  float* edge_out = nullptr;
  lms_candidate seed_out{};       // plan: best seed of the slice's narrowest windows
  int64_t K_in = 0;               // search: bands of the caller's arrays
  const double* lb_in = nullptr;
  const double* wq_in = nullptr;
  const float* edge_in = nullptr;
  lms_candidate seed_in{};        // search: best seed over all shards
};

// Host side of the last shard plan run on a context (its device keeps the
// samples and boundaries), reused by a search of the same fit.
struct ShardPlanState {
  bool valid = false;
  uint64_t gen = 0;
  int64_t n = 0, q = 0, K = 0, S = 0, P0 = 0, pspan = 0;
  std::vector<float> h_bnd;
  std::vector<unsigned> h_scnt;
  std::vector<double> h_lb;  // the plan's bounds of its own slice (+inf elsewhere)
  int nshards = 0, shard = -1;
};

// contiguous share `s` of `total` items over `parts` (ceil split, as
// distributed.partition / BatchPlan.partitions, backend.py:84-92)
inline void share_of(int64_t total, int64_t parts, int64_t s, int64_t* lo, int64_t* hi) {
  const int64_t size = std::max<int64_t>(1, (total + parts - 1) / parts);
  *lo = std::min(total, s * size);
  *hi = std::min(total, *lo + size);
}

}  // namespace

// Page-locked host memory for std::vector (cudaMallocHost / cudaFreeHost).
template <class T>
struct PinnedAlloc {
  using value_type = T;
  PinnedAlloc() = default;
  template <class U>
  PinnedAlloc(const PinnedAlloc<U>&) {}
  T* allocate(size_t n) {
    void* p = nullptr;
    if (cudaMallocHost(&p, n * sizeof(T)) != cudaSuccess) throw std::bad_alloc();
    return static_cast<T*>(p);
  }
  void deallocate(T* p, size_t) { cudaFreeHost(p); }
  template <class U>
  bool operator==(const PinnedAlloc<U>&) const { return true; }
  template <class U>
  bool operator!=(const PinnedAlloc<U>&) const { return false; }
};

struct lms_ctx {
  int device = 0;
  int sms = 148;
  cudaStream_t stream = nullptr;
  cudaEvent_t user_ev[kNumEvents] = {};
  cudaEvent_t ev_begin = nullptr, ev_end = nullptr;
  std::vector<cudaEvent_t> ev_chunk;
  // LMSB_TRACE=1: an event after every stage of a band solve, the stage
  // times printed to stderr (one JSON line per solve)
  bool trace = false;
  bool sync_check = false;  // LMSB_SYNC_CHECK=1: synchronise after every traced stage
  std::vector<cudaEvent_t> tr_ev;
  std::vector<const char*> tr_lab;
  int tr_n = 0;
  bool line_order = true;  // far-first streaming order (LMSB_ORDER=0 disables, for A/B runs)
  // lines (concatenated over fits)
  DevBuf<double> a_own, b_own;
  const double* a = nullptr;
  const double* b = nullptr;
  int64_t nlines = 0;
  // host copy (pinned: the upload's DMA reads it asynchronously): per-fit
  // max |a|, max |b| for the filter margins
  std::vector<double, PinnedAlloc<double>> h_a, h_b;
  // or, for lines that stay on the device (lms_batched_fit_sets_f64), the
  // per-fit statistics computed there: fit offsets and (alo, ahi, am, bm)
  std::vector<int64_t> ext_off;
  std::vector<double> ext_st;
  DevBuf<double> set_xy, set_stats;
  DevBuf<int64_t> set_cnt, set_coff;
  DevBuf<int32_t> set_contacts;
  double s_alo = 0, s_ahi = 0, s_am = 0, s_bm = 0;  // range / magnitudes of all bound lines
  // fits
  DevBuf<lmsb::FitDesc> fits;
  DevBuf<int64_t> prefA, prefB, seed_prefix, seg;
  DevBuf<lmsb::BestKey> keys;
  DevBuf<lms_candidate> best;
  // plan
  DevBuf<int64_t> counts, row_task_prefix;
  DevBuf<int32_t> row_fit, row_i, task_row;
  DevBuf<unsigned char> plan_tmp;
  // order
  DevBuf<float> sort_keys;
  DevBuf<int> sort_idx;
  DevBuf<double> pa, pb;
  DevBuf<int32_t> line_fit;
  DevBuf<unsigned char> sort_tmp;
  // items (seeds, survivors) and their records
  DevBuf<int64_t> ranks;
  DevBuf<int32_t> item_fit;
  DevBuf<lms_candidate> recs;
  DevBuf<unsigned long long> counters;
  // explicit vertices
  DevBuf<int64_t> ii, jj;
  DevBuf<double> uu, vv;
  lms_candidate* h_best = nullptr;  // pinned
  unsigned char* pin = nullptr;      // pinned staging of the band stage's small readbacks
  unsigned char* stage = nullptr;    // 2 x 4 MB pinned chunks for large transfers
  cudaEvent_t ev_stage[2] = {};
  size_t cap_pin = 0;
  int64_t cap_h_best = 0;
  // Hough: the points of the last vote (image pixels or explicit x/y)
  DevBuf<uint8_t> img;
  DevBuf<int64_t> pix, pcount;
  DevBuf<double> pxs, pys;
  DevBuf<unsigned char> ext_tmp, scan_tmp;
  DevBuf<unsigned long long> acc, masks;
  // device detect_lines (lms_detect.cu): the image of the last
  // lms_detect_peaks_u8 call, its grid and peaks, supports and designs
  DevBuf<int64_t> dt_peaks, dt_offs, dt_soffs, dt_doffs;
  DevBuf<unsigned> dt_counts;
  DevBuf<int32_t> dt_ids;
  DevBuf<double> dt_a, dt_b, dt_lim, dt_strig, dt_wedge;
  DevBuf<uint32_t> dt_bits;
  DevBuf<uint8_t> dt_swap;
  DevBuf<unsigned long long> dt_nlit;
  int64_t dt_npix = 0, dt_width = 0, dt_npeaks = -1;
  int dt_threshold = 0;
  lmsb::HoughGrid dt_grid{};
  DevBuf<double> tcos, tsin;
  DevBuf<int64_t> rbin, scounts, soffsets, sout;
  DevBuf<int32_t> sout32;
  // slope bands (lms_band.cu)
  int band_mode = 1;  // LMSB_BAND: 0 count-filter path only, 1 auto (large fits), 2 always
  int64_t band_vertices = 0;      // target vertices per band (LMSB_BAND_VERTICES; 0: by n,
                                  // see band_size)
  int64_t band_chunk = 12288;    // collected members per filter CTA (LMSB_BAND_CHUNK)
  int64_t big_mult = 0;          // n > 16,384: vertices per band >= big_mult * n (LMSB_BIG_MULT;
                                 // 0: by n, see big_band_mult)
  DevBuf<float> bsample, bbounds;
  DevBuf<unsigned> bscnt;
  DevBuf<uint8_t> bflag;
  DevBuf<uint32_t> bck, bcv, bcka, bmem;
  DevBuf<unsigned long long> bscal;
  DevBuf<int64_t> bstart, bend;
  DevBuf<unsigned char> btemp;
  DevBuf<double> blb, bwq;
  DevBuf<float> bedge;
  DevBuf<int32_t> blist;
  DevBuf<int64_t> branks2;
  DevBuf<unsigned> pcnt;  // split prepass counters (2 per survivor), kept zero
  DevBuf<int32_t> bfits2;
  DevBuf<int64_t> bchunks;
  DevBuf<float> bbig_keys, bbig_store;
  DevBuf<float> bslice_keys, bslice_store;
  DevBuf<int64_t> bslice_seg, bslice_prefix;
  DevBuf<double> bslice_u;
  DevBuf<int32_t> bslice_ids;  // a shard plan's interleaved bands
  DevBuf<int16_t> bslot;       // grouping slot of every band
  DevBuf<int64_t> boffs;       // batched contacts: fit offsets
  DevBuf<uint8_t> bcflags;     // batched contacts: one flag per point
  DevBuf<int32_t> bident;      // 0 .. nslot - 1
  DevBuf<unsigned> bslice_ptab;
  int64_t big_slice = 393216;    // n > 16,384: members per filter slice (LMSB_BIG_SLICE; 65,536
                                 // -> 393,216: config 3 9.28 -> 7.85 ms, flat from 196,608 up)
  // sort-free band bounds first, exact ones where they cannot dismiss a band
  // (LMSB_BAND_COARSE: 0 never, 1 always, 2 large n only -- for n <= 16,384
  // one shared-memory sort per band is cheaper than binning plus a refine)
  int band_coarse = 2;
  int prepass_split = 1;         // pass-0 screen with lines split over CTAs (LMSB_PREPASS_SPLIT)
  int seed_bands = 3;            // bands whose window-edge pairs seed H (LMSB_SEED_BANDS; 8 -> 3:
                                 // config 2 0.762 -> 0.750 ms, n = 20,000 2.03 -> 1.98 ms, same
                                 // survivors: the seeds fit one round of the cached exact kernel)
  int defer_bounds = 1;          // bands with a positive slope bound bounded after the seeds
                                 // (LMSB_DEFER)
  int plan_pool = 0;             // large-n shard plan: coarse-window pool given exact bounds
                                 // (LMSB_PLAN_POOL; 0: 64 / shards, at least 4 T)
  DevBuf<int64_t> bbig_seg;
  DevBuf<int32_t> small_list, dg_i32;
  DevBuf<int64_t> dg_i64;
  DevBuf<unsigned long long> dg_cursor;
  DevBuf<float> dg_sub;
  DevBuf<int16_t> dg_slot;
  // LMSB_BAND_DIRECT=1: collect straight into sub-band regions (no radix sort);
  // slower on config 2 (sub-bands are wider than slope-sorted chunks), kept
  // for A/B runs
  int band_direct = 0;
  // LMSB_GROUP_MODE: grouping of the swept members for n <= kBandMaxN:
  // 3 (default) = hybrid: a band narrow enough that its centre keys serve
  // every member (dev * width <= bkeys_tau * H: the filter reads the keys the
  // bound kernel stored, no sort) is one group; a wide band is cut into
  // sub-bands at every `sub_samples`-th sorted sample; the groups are
  // counting-sorted on the device and packed into filter chunks;
  // 1 = a radix sort by (slot, 17-bit slope position), keys sorted per chunk
  int group_mode = 3;
  int sub_samples = 1;     // LMSB_SUB_SAMPLES
  int filter_keys = 1;     // LMSB_FILTER_KEYS: store the bands' sorted keys (group_mode 3)
  double bkeys_tau = 0.1;  // LMSB_BKEYS_TAU
  // LMSB_SLOPE_BOUND (default 1): band bounds raised to |u|min W_q(a) - 2 bmax
  int slope_bound = 1;
  // LMSB_COUNT (default 0): 1 runs the fp32 exact-slope window counts
  // between the band filter and the exact pass-0 screen; with the slope bound
  // they pass 93 % of the band survivors (config 2: 1,717 -> 1,605) and cost
  // more than they save (config 2 0.869 vs 0.845 ms, config 3 0.27 ms)
  int band_count = 0;
  DevBuf<double> bwqa;
  uint64_t wqa_gen = ~0ull;
  int64_t wqa_off = -1, wqa_n = -1, wqa_q = -1;
  int64_t collect_floor = 0;    // smallest member capacity (grown after a deferred overflow)
  int64_t raw_floor = 0;        // smallest raw-enumeration capacity (grown after a raw overflow)
  bool cap_test = false;        // LMSB_CAP_TEST=1: first collect capacity 4,096 (overflow path)
  int64_t wide_chunk = 3072;    // LMSB_WIDE_CHUNK: members per filter chunk of a wide band
  int64_t narrow_chunk = 8192;  // LMSB_NARROW_CHUNK: ... of a narrow band (stored keys)
  DevBuf<float> bkeys;
  DevBuf<uint8_t> bnarrow;
  // LMSB_BIG_NARROW=1: n > kBandMaxN cuts a narrow band into one filter slice
  // (one key sort instead of >= 8); measured no faster at config 3 (more
  // survivors offset the saved sorts), so off by default
  int big_narrow = 0;
  DevBuf<int64_t> bctab;
  DevBuf<unsigned long long> bticket;
  DevBuf<int32_t> bcband;
  // LMSB_SWEEP: output-sensitive collect (lms_sweep.cu): 0 never (the
  // pre-test pass over every vertex), 1 always, 2 auto (n >= kSweepMinN, where
  // its fixed sort cost is below the pre-test pass's O(n^2))
  int band_sweep = 2;
  DevBuf<uint64_t> sw_k1;
  DevBuf<uint32_t> sw_idx;
  DevBuf<int32_t> sw_pos, sw_P, sw_bmin, sw_suf, sw_rk;
  DevBuf<lmsb::SweepEnd> sw_ends;
  // LMSB_DEVICE_PLAN (default 1): one-fit band searches plan their sweep and
  // groups on the device (band_plan_kernel) once a host-planned fit of the
  // same n has sized the member buffers (plan_cap); a plan the device cannot
  // make, or a member overflow, re-solves with the host plan
  int device_plan = 1;
  // LMSB_GRAPH (default 1): a device-planned search is captured into a CUDA
  // graph on its second identical run (same shape, line statistics, buffer
  // addresses) and replayed from then on -- one launch instead of ~45
  int use_graph = 1;
  cudaGraphExec_t gexec = nullptr;
  unsigned char gkey[160] = {0}, gseen[160] = {0};
  int64_t g_launches = 0;
  bool capturing = false;  // a band search is being captured on `stream`
  int64_t plan_cap = 0, plan_cap_n = -1;
  bool force_host_plan = false;
  DevBuf<lmsb::DevPlanHdr> dp_hdr;
  DevBuf<int32_t> dp_list, dp_ident, dp_rk, dp_sbf, dp_gband;
  DevBuf<int16_t> dp_slot;
  DevBuf<lmsb::SweepEnd> dp_ends;
  DevBuf<unsigned long long> sw_dbg, sw_raw, sw_rawcnt;
  DevBuf<unsigned long long> small_cnt;
  int small_mode = 1;  // LMSB_SMALL: 0 off, 1 batches, 2 also single fits
  DevBuf<float2> blines32;
  std::vector<double> h_blb;
  ShardSpec* shard = nullptr;  // set for the duration of a shard plan / search call
  ShardPlanState splan;
  DevBuf<double2> bab;         // interleaved lines of the last banded fit
  uint64_t ab_gen = ~0ull;
  int64_t ab_off = -1, ab_n = -1;
  const double2* ab_ptr = nullptr;
  uint64_t gen = 0;            // bumped whenever the bound lines change
  int hough_mode = 0;  // 0 none, 1 image pixels, 2 explicit points
  int64_t hough_npts = 0, hough_width = 1;
  int64_t hough_maxid = 0;  // bound of the support ids of the last vote
  lms_stats stats{};
  // multi-GPU: this context's NCCL communicator (lms_ctx_comm_init) and the
  // device buffers of its two record exchanges
  // the last shard plan run on this context (gen of its lines, shard, bands)
  uint64_t plan_gen = ~0ull;
  int plan_nshards = 0, plan_shard = -1;
  int64_t plan_K = 0;
  ncclComm_t comm = nullptr;
  bool comm_owned = false;
  int comm_ranks = 0, comm_rank = -1;
  DevBuf<lms_candidate> xsend, xrecv;
  std::mutex mu;
};

namespace {

int ctx_init(lms_ctx* c, int device) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    return set_error(LMS_ERR_NODEVICE, "no CUDA device available");
  if (device < 0 || device >= count)
    return set_error(LMS_ERR_NODEVICE, "device %d out of range (%d devices)", device, count);
  c->device = device;
  const char* ov = getenv("LMSB_ORDER");
  c->line_order = !(ov && std::strcmp(ov, "0") == 0);
  const char* bm = getenv("LMSB_BAND");
  c->band_mode = bm ? std::max(0, std::min(2, atoi(bm))) : 1;
  const char* bv = getenv("LMSB_BAND_VERTICES");
  if (bv && atoll(bv) >= 256) c->band_vertices = atoll(bv);
  const char* bd = getenv("LMSB_BAND_DIRECT");
  c->band_direct = (bd && std::strcmp(bd, "1") == 0) ? 1 : 0;
  if (const char* sw = getenv("LMSB_SWEEP")) c->band_sweep = std::max(0, std::min(2, atoi(sw)));
  if (const char* fk = getenv("LMSB_FILTER_KEYS")) c->filter_keys = atoi(fk) != 0 ? 1 : 0;
  if (const char* bt = getenv("LMSB_BKEYS_TAU")) c->bkeys_tau = atof(bt);
  if (const char* bn = getenv("LMSB_BIG_NARROW")) c->big_narrow = atoi(bn) != 0;
  if (const char* ct = getenv("LMSB_CAP_TEST")) c->cap_test = atoi(ct) != 0;
  if (const char* dpl = getenv("LMSB_DEVICE_PLAN")) c->device_plan = atoi(dpl) != 0;
  if (const char* gr = getenv("LMSB_GRAPH")) c->use_graph = atoi(gr) != 0;
  if (const char* sb = getenv("LMSB_SLOPE_BOUND")) c->slope_bound = atoi(sb) != 0;
  if (const char* bc = getenv("LMSB_COUNT")) c->band_count = atoi(bc) != 0;
  if (const char* wc = getenv("LMSB_WIDE_CHUNK"); wc && atoll(wc) >= 256) c->wide_chunk = atoll(wc);
  if (const char* nc = getenv("LMSB_NARROW_CHUNK"); nc && atoll(nc) >= 256)
    c->narrow_chunk = atoll(nc);
  if (const char* gm = getenv("LMSB_GROUP_MODE")) c->group_mode = atoi(gm) == 1 ? 1 : 3;
  if (const char* ss = getenv("LMSB_SUB_SAMPLES"); ss && atoi(ss) >= 1)
    c->sub_samples = std::min(64, atoi(ss));
  const char* bmul = getenv("LMSB_BIG_MULT");
  if (bmul && atoll(bmul) >= 1) c->big_mult = atoll(bmul);
  if (const char* bs = getenv("LMSB_BIG_SLICE"); bs && atoll(bs) >= 1) c->big_slice = atoll(bs);
  if (const char* sb = getenv("LMSB_SEED_BANDS"); sb && atoi(sb) >= 1)
    c->seed_bands = std::min(48, atoi(sb));
  if (const char* df = getenv("LMSB_DEFER")) c->defer_bounds = atoi(df) != 0;
  if (const char* pp = getenv("LMSB_PLAN_POOL"); pp && atoi(pp) >= 1)
    c->plan_pool = std::min(64, atoi(pp));
  if (const char* ps = getenv("LMSB_PREPASS_SPLIT")) c->prepass_split = atoi(ps) != 0;
  if (const char* bc0 = getenv("LMSB_BAND_COARSE")) c->band_coarse = std::max(0, std::min(2, atoi(bc0)));
  const char* sm = getenv("LMSB_SMALL");
  c->small_mode = sm ? std::max(0, std::min(2, atoi(sm))) : 1;
  const char* bc = getenv("LMSB_BAND_CHUNK");
  if (bc && atoll(bc) >= 32) c->band_chunk = atoll(bc);
  if (const char* tr = getenv("LMSB_TRACE")) c->trace = atoi(tr) != 0;
  if (const char* sc = getenv("LMSB_SYNC_CHECK")) c->sync_check = atoi(sc) != 0;
  CUDA_TRY(cudaSetDevice(device));
  CUDA_TRY(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device));
  CUDA_TRY(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  for (auto& e : c->user_ev) CUDA_TRY(cudaEventCreate(&e));
  CUDA_TRY(cudaEventCreate(&c->ev_begin));
  CUDA_TRY(cudaEventCreate(&c->ev_end));
  return LMS_OK;
}

void ctx_release(lms_ctx* c) {
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto& e : c->user_ev)
    if (e) cudaEventDestroy(e);
  for (auto e : c->ev_chunk) cudaEventDestroy(e);
  for (auto& e : c->ev_stage)
    if (e) cudaEventDestroy(e);
  if (c->stage) cudaFreeHost(c->stage);
  c->stage = nullptr;
  if (c->ev_begin) cudaEventDestroy(c->ev_begin);
  if (c->ev_end) cudaEventDestroy(c->ev_end);
  c->a_own.release();
  c->b_own.release();
  c->fits.release();
  c->prefA.release();
  c->prefB.release();
  c->seed_prefix.release();
  c->seg.release();
  c->keys.release();
  c->best.release();
  c->counts.release();
  c->row_task_prefix.release();
  c->row_fit.release();
  c->row_i.release();
  c->task_row.release();
  c->plan_tmp.release();
  c->sort_keys.release();
  c->sort_idx.release();
  c->pa.release();
  c->pb.release();
  c->line_fit.release();
  c->sort_tmp.release();
  c->ranks.release();
  c->item_fit.release();
  c->recs.release();
  c->counters.release();
  c->ii.release();
  c->jj.release();
  c->uu.release();
  c->vv.release();
  c->img.release();
  c->pix.release();
  c->pcount.release();
  c->pxs.release();
  c->pys.release();
  c->ext_tmp.release();
  c->scan_tmp.release();
  c->acc.release();
  c->masks.release();
  c->tcos.release();
  c->tsin.release();
  c->rbin.release();
  c->scounts.release();
  c->soffsets.release();
  c->sout.release();
  c->bsample.release();
  c->bbounds.release();
  c->bscnt.release();
  c->bflag.release();
  c->bck.release();
  c->bcv.release();
  c->bcka.release();
  c->bmem.release();
  c->bscal.release();
  c->bstart.release();
  c->bend.release();
  c->btemp.release();
  c->blb.release();
  c->bwq.release();
  c->bedge.release();
  c->blist.release();
  c->branks2.release();
  c->pcnt.release();
  c->bfits2.release();
  c->bchunks.release();
  c->bbig_keys.release();
  c->bbig_store.release();
  c->bslice_keys.release();
  c->bslice_store.release();
  c->bslice_seg.release();
  c->bslice_prefix.release();
  c->bslice_u.release();
  c->bslice_ids.release();
  c->bslot.release();
  c->boffs.release();
  c->bcflags.release();
  c->bident.release();
  c->bslice_ptab.release();
  c->bab.release();
  c->bbig_seg.release();
  c->small_list.release();
  c->dg_i32.release();
  c->dg_i64.release();
  c->dg_cursor.release();
  c->dg_sub.release();
  c->bctab.release();
  c->bticket.release();
  c->bwqa.release();
  c->bkeys.release();
  c->bnarrow.release();
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  c->gexec = nullptr;
  c->dp_hdr.release();
  c->dp_list.release();
  c->dp_ident.release();
  c->dp_rk.release();
  c->dp_sbf.release();
  c->dp_gband.release();
  c->dp_slot.release();
  c->dp_ends.release();
  c->bcband.release();
  c->dg_slot.release();
  c->small_cnt.release();
  c->blines32.release();
  c->sw_k1.release();
  c->sw_idx.release();
  c->sw_pos.release();
  c->sw_P.release();
  c->sw_bmin.release();
  c->sw_suf.release();
  c->sw_rk.release();
  c->sw_ends.release();
  c->sw_dbg.release();
  c->sw_raw.release();
  c->sw_rawcnt.release();
  c->dt_peaks.release();
  c->dt_offs.release();
  c->dt_soffs.release();
  c->dt_doffs.release();
  c->dt_counts.release();
  c->dt_ids.release();
  c->dt_a.release();
  c->dt_b.release();
  c->dt_lim.release();
  c->dt_strig.release();
  c->dt_wedge.release();
  c->dt_bits.release();
  c->dt_swap.release();
  c->dt_nlit.release();
  c->set_xy.release();
  c->set_stats.release();
  c->set_cnt.release();
  c->set_coff.release();
  c->set_contacts.release();
  c->xsend.release();
  c->xrecv.release();
  if (c->comm && c->comm_owned && lmsb::nccl().ok) lmsb::nccl().CommDestroy(c->comm);
  c->comm = nullptr;
  if (c->h_best) cudaFreeHost(c->h_best);
  if (c->pin) cudaFreeHost(c->pin);
  if (c->stream) cudaStreamDestroy(c->stream);
}

// Range and magnitudes of lines [off, off + n) (the whole bound set is cached
// at upload).
void line_stats(const lms_ctx* c, int64_t off, int64_t n, double* alo, double* ahi, double* am,
                double* bm) {
  if (!c->ext_off.empty()) {
    const auto it = std::lower_bound(c->ext_off.begin(), c->ext_off.end(), off);
    if (it != c->ext_off.end() && *it == off) {
      const size_t k = (size_t)(it - c->ext_off.begin());
      *alo = c->ext_st[4 * k];
      *ahi = c->ext_st[4 * k + 1];
      *am = c->ext_st[4 * k + 2];
      *bm = c->ext_st[4 * k + 3];
      return;
    }
  }
  if (off == 0 && n == c->nlines) {
    *alo = c->s_alo;
    *ahi = c->s_ahi;
    *am = c->s_am;
    *bm = c->s_bm;
    return;
  }
  double lo = INFINITY, hi = -INFINITY, ma = 0.0, mb = 0.0;
  for (int64_t k = off; k < off + n; ++k) {
    lo = std::min(lo, c->h_a[k]);
    hi = std::max(hi, c->h_a[k]);
    ma = std::max(ma, std::fabs(c->h_a[k]));
    mb = std::max(mb, std::fabs(c->h_b[k]));
  }
  *alo = lo;
  *ahi = hi;
  *am = ma;
  *bm = mb;
}

void cache_line_stats(lms_ctx* c) {
  ++c->gen;
  double alo = INFINITY, ahi = -INFINITY, am = 0.0, bm = 0.0;
  const double* a = c->h_a.data();
  const double* b = c->h_b.data();
  const int64_t n = c->nlines;
#pragma omp simd reduction(min : alo) reduction(max : ahi, am, bm)
  for (int64_t k = 0; k < n; ++k) {
    alo = a[k] < alo ? a[k] : alo;
    ahi = a[k] > ahi ? a[k] : ahi;
    am = std::fabs(a[k]) > am ? std::fabs(a[k]) : am;
    bm = std::fabs(b[k]) > bm ? std::fabs(b[k]) : bm;
  }
  c->s_alo = alo;
  c->s_ahi = ahi;
  c->s_am = am;
  c->s_bm = bm;
}

int ctx_upload(lms_ctx* c, const double* a, const double* b, int64_t n) {
  if (!a || !b || n < 1)
    return set_error(LMS_ERR_INVALID, "need at least 1 line, got %lld", (long long)n);
  CUDA_TRY(cudaSetDevice(c->device));
  RC_TRY(c->a_own.need(n));
  RC_TRY(c->b_own.need(n));
  // the host copy (pinned) and the line statistics in one pass, then two
  // asynchronous DMAs from it (a pageable source would be staged by the
  // driver synchronously)
  try {
    c->h_a.resize(n);
    c->h_b.resize(n);
  } catch (const std::bad_alloc&) {
    return set_error(LMS_ERR_NOMEM, "pinned host copy of %lld lines", (long long)n);
  }
  double* ha = c->h_a.data();
  double* hb = c->h_b.data();
  double alo = INFINITY, ahi = -INFINITY, am = 0.0, bm = 0.0;
#pragma omp simd reduction(min : alo) reduction(max : ahi, am, bm)
  for (int64_t k = 0; k < n; ++k) {
    const double x = a[k], y = b[k];
    ha[k] = x;
    hb[k] = y;
    alo = x < alo ? x : alo;
    ahi = x > ahi ? x : ahi;
    am = std::fabs(x) > am ? std::fabs(x) : am;
    bm = std::fabs(y) > bm ? std::fabs(y) : bm;
  }
  CUDA_TRY(cudaMemcpyAsync(c->a_own.p, ha, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->b_own.p, hb, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  c->ext_off.clear();
  c->a = c->a_own.p;
  c->b = c->b_own.p;
  c->nlines = n;
  ++c->gen;  // (cache_line_stats, fused into the copy)
  c->s_alo = alo;
  c->s_ahi = ahi;
  c->s_am = am;
  c->s_bm = bm;
  return LMS_OK;
}

// Host memcpy split over threads (the large pageable <-> pinned copies of
// the Hough image and supports).
void par_memcpy(void* dst, const void* src, size_t n) {
  if (n < ((size_t)1 << 20)) {
    std::memcpy(dst, src, n);
    return;
  }
  constexpr int kThreadsCopy = 8;
  const size_t part = ((n + kThreadsCopy - 1) / kThreadsCopy + 63) & ~(size_t)63;
#pragma omp parallel for num_threads(kThreadsCopy) schedule(static)
  for (int t = 0; t < kThreadsCopy; ++t) {
    const size_t o = (size_t)t * part;
    if (o < n) std::memcpy(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o,
                           std::min(part, n - o));
  }
}

constexpr size_t kStageChunk = (size_t)4 << 20;

int ensure_stage(lms_ctx* c) {
  if (c->stage) return LMS_OK;
  CUDA_TRY(cudaMallocHost(&c->stage, 2 * kStageChunk));
  for (auto& e : c->ev_stage) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return LMS_OK;
}

// H2D of a large pageable buffer: threaded copies into two pinned chunks,
// each DMA overlapping the next chunk's copy (stream-ordered; returns once
// the last chunk is queued).
int upload_staged(lms_ctx* c, void* d_dst, const void* h_src, size_t bytes) {
  if (bytes < 2 * kStageChunk) {
    CUDA_TRY(cudaMemcpyAsync(d_dst, h_src, bytes, cudaMemcpyHostToDevice, c->stream));
    return LMS_OK;
  }
  RC_TRY(ensure_stage(c));
  bool used[2] = {false, false};
  int slot = 0;
  for (size_t off = 0; off < bytes; off += kStageChunk, slot ^= 1) {
    const size_t len = std::min(kStageChunk, bytes - off);
    unsigned char* buf = c->stage + slot * kStageChunk;
    if (used[slot]) CUDA_TRY(cudaEventSynchronize(c->ev_stage[slot]));
    par_memcpy(buf, static_cast<const char*>(h_src) + off, len);
    CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(d_dst) + off, buf, len, cudaMemcpyHostToDevice,
                             c->stream));
    CUDA_TRY(cudaEventRecord(c->ev_stage[slot], c->stream));
    used[slot] = true;
  }
  return LMS_OK;
}

// D2H into a large pageable buffer: chunk k + 1's DMA overlaps chunk k's
// threaded copy out of pinned memory.  Synchronous.
int download_staged(lms_ctx* c, void* h_dst, const void* d_src, size_t bytes) {
  if (bytes < 2 * kStageChunk) {
    CUDA_TRY(cudaMemcpyAsync(h_dst, d_src, bytes, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return LMS_OK;
  }
  RC_TRY(ensure_stage(c));
  const size_t nchunks = (bytes + kStageChunk - 1) / kStageChunk;
  auto issue = [&](size_t k) -> int {
    const size_t off = k * kStageChunk, len = std::min(kStageChunk, bytes - off);
    unsigned char* buf = c->stage + (k & 1) * kStageChunk;
    CUDA_TRY(cudaMemcpyAsync(buf, static_cast<const char*>(d_src) + off, len,
                             cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaEventRecord(c->ev_stage[k & 1], c->stream));
    return LMS_OK;
  };
  RC_TRY(issue(0));
  for (size_t k = 0; k < nchunks; ++k) {
    if (k + 1 < nchunks) RC_TRY(issue(k + 1));
    CUDA_TRY(cudaEventSynchronize(c->ev_stage[k & 1]));
    const size_t off = k * kStageChunk, len = std::min(kStageChunk, bytes - off);
    par_memcpy(static_cast<char*>(h_dst) + off, c->stage + (k & 1) * kStageChunk, len);
  }
  return LMS_OK;
}

int ensure_pinned(lms_ctx* c, size_t bytes) {
  if (bytes <= c->cap_pin) return LMS_OK;
  if (c->pin) cudaFreeHost(c->pin);
  c->pin = nullptr;
  c->cap_pin = 0;
  CUDA_TRY(cudaMallocHost(&c->pin, bytes));
  c->cap_pin = bytes;
  return LMS_OK;
}

int ensure_host_best(lms_ctx* c, int64_t nfits) {
  if (nfits <= c->cap_h_best) return LMS_OK;
  if (c->h_best) cudaFreeHost(c->h_best);
  c->h_best = nullptr;
  c->cap_h_best = 0;
  CUDA_TRY(cudaMallocHost(&c->h_best, sizeof(lms_candidate) * nfits));
  c->cap_h_best = nfits;
  return LMS_OK;
}

// stage events: inside a CUDA-graph capture recorded as external event
// nodes (their times stay readable after each replay)
cudaError_t ev_rec(lms_ctx* c, cudaEvent_t e) {
  return c->capturing ? cudaEventRecordWithFlags(e, c->stream, cudaEventRecordExternal)
                      : cudaEventRecord(e, c->stream);
}

void trace_mark(lms_ctx* c, const char* label) {
  if (c->sync_check) {  // (debugging) the first stage whose kernels fault
    const cudaError_t e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) fprintf(stderr, "LMSB_SYNC_CHECK: stage %s: %s\n", label, cudaGetErrorString(e));
  }
  if (!c->trace) return;
  if (c->tr_n >= (int)c->tr_ev.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    c->tr_ev.push_back(e);
    c->tr_lab.push_back(nullptr);
  }
  c->tr_lab[c->tr_n] = label;
  cudaEventRecord(c->tr_ev[c->tr_n++], c->stream);
}

void trace_dump(lms_ctx* c) {
  if (!c->trace || c->tr_n < 2) {
    c->tr_n = 0;
    return;
  }
  cudaEventSynchronize(c->tr_ev[c->tr_n - 1]);
  std::string out = "{\"trace_us\": [";
  for (int e = 1; e < c->tr_n; ++e) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->tr_ev[e - 1], c->tr_ev[e]);
    char buf[160];
    snprintf(buf, sizeof(buf), "%s[\"%s\", %.1f]", e > 1 ? ", " : "", c->tr_lab[e], ms * 1e3f);
    out += buf;
  }
  float tot = 0.f;
  cudaEventElapsedTime(&tot, c->tr_ev[0], c->tr_ev[c->tr_n - 1]);
  char buf[64];
  snprintf(buf, sizeof(buf), "], \"total_us\": %.1f}", tot * 1e3f);
  out += buf;
  fprintf(stderr, "%s\n", out.c_str());
  c->tr_n = 0;
}

int persistent_grid(const lms_ctx* c, int64_t count) {
  int64_t g = (int64_t)c->sms * 8;
  if (count >= 0) g = std::min<int64_t>(g, std::max<int64_t>(count, 1));
  return (int)g;
}

int reduce_grid(const lms_ctx* c, int64_t count) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)c->sms * 4, (count + 255) / 256));
}

// Far-first streaming order of every fit's lines (lms_order.cu); returns the
// permuted line arrays through la / lb.
int order_lines(lms_ctx* c, const std::vector<int64_t>& seg, int64_t F, const double** la,
                const double** lb, lms_stats* st) {
  const int64_t o = seg[0];
  const int64_t nl = seg[F] - o;
  RC_TRY(c->sort_keys.need(2 * nl));
  RC_TRY(c->sort_idx.need(2 * nl));
  RC_TRY(c->pa.need(c->nlines));
  RC_TRY(c->pb.need(c->nlines));
  RC_TRY(c->line_fit.need(nl));
  RC_TRY(c->sort_tmp.need((int64_t)lmsb::order_temp_bytes(nl, F)));
  // the sort works on [o, o + nl): segment offsets relative to o
  std::vector<int64_t> rel(F + 1);
  for (int64_t f = 0; f <= F; ++f) rel[f] = seg[f] - o;
  CUDA_TRY(cudaMemcpyAsync(c->seg.p, rel.data(), sizeof(int64_t) * (F + 1), cudaMemcpyHostToDevice,
                           c->stream));
  lmsb::launch_line_fit(c->seg.p, F, c->line_fit.p, c->stream);
  lmsb::OrderArgs oa{};
  oa.a = c->a + o;
  oa.b = c->b + o;
  oa.nlines = nl;
  oa.seg_begin = c->seg.p;
  oa.nfits = F;
  oa.line_fit = c->line_fit.p;
  oa.best = c->best.p;
  oa.keys_in = c->sort_keys.p;
  oa.keys_out = c->sort_keys.p + nl;
  oa.idx_in = c->sort_idx.p;
  oa.idx_out = c->sort_idx.p + nl;
  oa.temp = c->sort_tmp.p;
  oa.temp_bytes = (size_t)c->sort_tmp.cap;
  oa.pa = c->pa.p + o;
  oa.pb = c->pb.p + o;
  if (lmsb::launch_line_order(oa, c->stream) != 0)
    return set_error(LMS_ERR_CUDA, "line order sort failed");
  CUDA_TRY(cudaGetLastError());
  st->launches += 4;
  *la = c->pa.p;
  *lb = c->pb.p;
  return LMS_OK;
}

// Slope-band search of one large fit (lms_band.cu): bound every slope band,
// seed H from the samples of the lowest-bound bands, collect the vertices of
// the bands whose bound admits H, count their windows, and re-evaluate the
// survivors exactly.  best[0] must be reset; the caller checked that the
// fit's magnitudes are finite and n <= kBandMaxBigN.
// The band search after the seeds with the plan made on the device
// (band_plan_kernel): sweep collect over the planned runs (device run count,
// kPlanMaxRuns segments reserved), sub-band grouping and chunking with
// device counts.  Members are collected into c->plan_cap slots; *m = that
// capacity (the real count is checked by the final readback).
int devplan_search(lms_ctx* c, const HostFit& h, lms_stats* st, const lmsb::BandFit& bf,
                   lmsb::BandArgs& ba, lmsb::BandWork& w, int K, int64_t S, unsigned long long* sc,
                   unsigned long long* m, int64_t* nchunk_max) {
  (void)S;
  const int64_t n = h.n;
  constexpr int R = lmsb::kPlanMaxRuns;
  const int nseg = 2 * R + 1;
  RC_TRY(c->dp_hdr.need(1));
  RC_TRY(c->dp_list.need(K + 1));
  RC_TRY(c->dp_ident.need(K + 1));
  RC_TRY(c->dp_slot.need(K + 1));
  RC_TRY(c->dp_rk.need(2 * R));
  RC_TRY(c->dp_sbf.need(K + 2));
  RC_TRY(c->dp_gband.need(lmsb::kSubMaxGroups));
  RC_TRY(c->dp_ends.need(nseg));
  lmsb::DevPlan dp{};
  dp.hdr = c->dp_hdr.p;
  dp.list = c->dp_list.p;
  dp.slot = c->dp_slot.p;
  dp.ident = c->dp_ident.p;
  dp.ends = c->dp_ends.p;
  dp.rk = c->dp_rk.p;
  dp.sbf = c->dp_sbf.p;
  dp.gband = c->dp_gband.p;
  lmsb::launch_band_plan(bf, w, c->blb.p, c->best.p, K, c->sub_samples, c->bkeys_tau, dp,
                         c->stream);
  st->launches += 1;
  trace_mark(c, "plan");
  const int* d_nadm = &c->dp_hdr.p->nadm;
  const int* d_nslot = &c->dp_hdr.p->nslot;
  const int32_t* d_nr = &c->dp_hdr.p->nr;
  const int* d_ng = &c->dp_hdr.p->ngroups;
  const double* d_tau = &c->dp_hdr.p->tau;
  // sweep sorts at the planned run ends
  const int64_t nbk = (n + 31) / 32;
  RC_TRY(c->sw_k1.need(2 * nseg * n));
  RC_TRY(c->sw_idx.need(2 * nseg * n));
  RC_TRY(c->sw_pos.need(R * n));
  RC_TRY(c->sw_P.need(R * n));
  RC_TRY(c->sw_bmin.need(R * nbk));
  RC_TRY(c->sw_suf.need(R * nbk));
  lmsb::SweepSort ss{};
  for (int b = 0; b < 2; ++b) {
    ss.k1[b] = c->sw_k1.p + b * nseg * n;
    ss.idx[b] = c->sw_idx.p + b * nseg * n;
  }
  ss.dnr = d_nr;
  ss.nr_max = R;
  st->launches += lmsb::launch_sweep_sort(bf.ab, (int)n, c->dp_ends.p, nseg, ss, c->sms, c->stream);
  trace_mark(c, "sweep_sort");
  lmsb::launch_sweep_prepare((int)n, R, ss, c->sw_pos.p, c->sw_P.p, c->sw_bmin.p, c->sw_suf.p,
                             c->sms, c->stream);
  st->launches += 3;
  trace_mark(c, "sweep_prep");
  // sub-band boundaries of the admitted bands
  RC_TRY(c->dg_sub.need(lmsb::kSubMaxGroups));
  lmsb::launch_band_subbounds(w, c->dp_list.p, c->dp_sbf.p, K, c->dg_sub.p, c->stream, d_nadm);
  st->launches += 1;
  trace_mark(c, "subbounds");
  // collect
  const int64_t cap = c->plan_cap;
  RC_TRY(c->bck.need(cap));
  RC_TRY(c->bcv.need(cap));
  const int64_t raw_cap = std::max(cap, c->raw_floor);
  RC_TRY(c->sw_raw.need(raw_cap));
  RC_TRY(c->sw_rawcnt.need(1));
  w.ckeys = c->bck.p;
  w.cvals = c->bcv.p;
  lmsb::SweepArgs sa{};
  sa.bounds = c->bbounds.p;
  sa.K = K;
  sa.slot = c->dp_slot.p;
  sa.nruns = R;
  sa.run_k0 = c->dp_rk.p;
  sa.run_k1 = c->dp_rk.p + R;
  sa.P = c->sw_P.p;
  sa.bmin = c->sw_bmin.p;
  sa.suf = c->sw_suf.p;
  sa.idx = ss.idx[ss.cur];
  sa.k1a = ss.k1[ss.cur] + (int64_t)(2 * R) * n;
  sa.idxa = ss.idx[ss.cur] + (int64_t)(2 * R) * n;
  sa.tau = 0.0;
  sa.dtau = d_tau;
  sa.dnr = d_nr;
  sa.count = sc + 1;
  sa.out_keys = w.ckeys;
  sa.out_vals = w.cvals;
  sa.cap = cap;
  sa.raw = c->sw_raw.p;
  sa.raw_cap = raw_cap;
  sa.raw_count = c->sw_rawcnt.p;
  sa.raw_overflow = sc + 8;
  sa.sub_first = c->dp_sbf.p;
  sa.sub = c->dg_sub.p;
  CUDA_TRY(ev_rec(c, c->ev_chunk[2]));
  CUDA_TRY(ev_rec(c, c->ev_chunk[5]));
  CUDA_TRY(ev_rec(c, c->ev_chunk[10]));
  lmsb::launch_sweep_emit(bf, sa, c->sms, c->stream);
  CUDA_TRY(ev_rec(c, c->ev_chunk[11]));
  CUDA_TRY(ev_rec(c, c->ev_chunk[6]));
  st->launches += 3;
  trace_mark(c, "sweep_emit");
  // grouping with device counts, then the chunk table
  const int G = lmsb::kSubMaxGroups;
  const int64_t cmin = std::max<int64_t>(1, std::min(c->wide_chunk, c->narrow_chunk));
  *nchunk_max = 2 * ((cap + cmin - 1) / cmin) + G + K + 2;
  RC_TRY(c->bmem.need(std::max<int64_t>(cap, 1)));
  RC_TRY(c->dg_cursor.need(2 * (int64_t)G));
  RC_TRY(c->bstart.need(std::max<int64_t>(G, K + 1)));
  RC_TRY(c->bend.need(std::max<int64_t>(G, K + 1)));
  RC_TRY(c->bctab.need(2 * *nchunk_max));
  RC_TRY(c->bcband.need(*nchunk_max));
  w.start = c->bstart.p;
  w.end = c->bend.p;
  ba.start = c->bstart.p;
  ba.end = c->bend.p;
  CUDA_TRY(cudaMemsetAsync(c->dg_cursor.p, 0, sizeof(unsigned long long) * G, c->stream));
  if (lmsb::launch_band_group_sub(w.ckeys, w.cvals, sc + 1, cap, G, c->dg_cursor.p,
                                  c->dg_cursor.p + G, c->bstart.p, c->bend.p, c->bmem.p, c->stream,
                                  d_ng) != 0)
    return set_error(LMS_ERR_CUDA, "sub-band grouping failed");
  trace_mark(c, "group");
  lmsb::launch_band_pack_chunks(c->dp_sbf.p, K + 1, c->bstart.p, c->bend.p, c->dp_gband.p,
                                c->wide_chunk, c->narrow_chunk, c->bctab.p, c->bcband.p, sc + 7,
                                c->stream, d_nslot);
  CUDA_TRY(cudaGetLastError());
  st->launches += 4;
  trace_mark(c, "pack");
  st->bands = K;
  *m = (unsigned long long)cap;
  return LMS_OK;
}

struct BandTail {
  unsigned long long m;  // member capacity the search ran with (or the exact count)
  bool direct, dplan, filter_timed, bound_timed, sweep_timed;
};

// The end of a band search: the one readback (counts, the device plan's
// header), the overflow / bail re-solves, the stage times.
int band_solve(lms_ctx* c, const HostFit& h, lms_stats* st);

int band_finish(lms_ctx* c, const HostFit& h, lms_stats* st, BandTail t) {
  unsigned long long* sc = c->bscal.p;
  unsigned long long m = t.m;
  const bool direct = t.direct, dplan = t.dplan;
  const bool filter_timed = t.filter_timed, bound_timed = t.bound_timed,
             sweep_timed = t.sweep_timed;
  unsigned long long* cnts = reinterpret_cast<unsigned long long*>(c->pin);  // readbacks done
  CUDA_TRY(cudaMemcpyAsync(cnts, sc + 1, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                           c->stream));
  lmsb::DevPlanHdr* ph = reinterpret_cast<lmsb::DevPlanHdr*>(c->pin + 128);
  if (dplan)
    CUDA_TRY(cudaMemcpyAsync(ph, c->dp_hdr.p, sizeof(lmsb::DevPlanHdr), cudaMemcpyDeviceToHost,
                             c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  // members classified; a raw-enumeration overflow (cnts[7]: the raw count;
  // then not every member was seen) grows the raw capacity to it
  const unsigned long long m_dev = cnts[0];
  const unsigned long long raw_over = cnts[7];
  if (raw_over > 0) c->raw_floor = std::max<int64_t>(c->raw_floor, (int64_t)raw_over);
  cnts += 2;  // [0] band survivors .. [3] exact-stage inputs, as before
  if (dplan) {
    const lmsb::DevPlanHdr hd = *ph;
    if (hd.bail || m_dev > m || raw_over > 0) {
      // the device could not plan this fit, or the members outgrew the
      // capacity: solve again with the host plan (which also resizes)
      if (m_dev > m) c->plan_cap = std::max<int64_t>(c->plan_cap, (int64_t)m_dev + m_dev / 4);
      trace_dump(c);
      c->force_host_plan = true;
      const int rc = band_solve(c, h, st);
      c->force_host_plan = false;
      return rc;
    }
    st->bands_searched = hd.nadm;
    st->seed_height = hd.H;
    st->sweep_runs = hd.nr;
  }
  if ((m_dev > m || raw_over > 0) && !direct) {
    // deferred member count above the capacity (or raw entries dropped):
    // members were lost, so solve again with room for all of them (the
    // record found so far stays installed; it is a real vertex).  Both
    // floors are exact counts, so this happens at most twice.
    if (m_dev > m) c->collect_floor = std::max<int64_t>(c->collect_floor, (int64_t)m_dev);
    trace_dump(c);
    return band_solve(c, h, st);
  }
  m = m_dev;
  st->survivors = (int64_t)cnts[3];
  if (getenv("LMSB_BAND_DEBUG"))
    fprintf(stderr, "band: members %llu band survivors %llu count survivors %llu exact inputs %llu\n",
            m_dev, cnts[0], cnts[1], cnts[3]);
  trace_mark(c, "readback3");
  trace_dump(c);  // evaluated by the exact select (cnts[2]: running height)
  st->band_survivors = (int64_t)cnts[0];
  st->filtered_vertices = (int64_t)m;
  st->chunks = 1;
  float ms = 0.f;
  CUDA_TRY(cudaEventElapsedTime(&ms, c->ev_chunk[0], c->ev_chunk[1]));
  st->ms_bound = ms;
  CUDA_TRY(cudaEventElapsedTime(&ms, c->ev_chunk[2], c->ev_chunk[3]));
  st->ms_partition = ms;
  CUDA_TRY(cudaEventElapsedTime(&ms, c->ev_chunk[3], c->ev_chunk[4]));
  st->ms_band_filter = ms;
  CUDA_TRY(cudaEventElapsedTime(&ms, c->ev_chunk[5], c->ev_chunk[6]));
  st->ms_collect = ms;
  st->ms_filter_kernel = 0.f;
  if (filter_timed) {
    CUDA_TRY(cudaEventElapsedTime(&ms, c->ev_chunk[8], c->ev_chunk[9]));
    st->ms_filter_kernel = ms;
  }
  st->ms_bound_kernel = 0.f;
  if (bound_timed) {
    CUDA_TRY(cudaEventElapsedTime(&ms, c->ev_chunk[12], c->ev_chunk[13]));
    st->ms_bound_kernel = ms;
  }
  st->ms_sweep_enum = 0.f;
  if (sweep_timed) {
    CUDA_TRY(cudaEventElapsedTime(&ms, c->ev_chunk[10], c->ev_chunk[11]));
    st->ms_sweep_enum = ms;
  }
  if (getenv("LMSB_BAND_DEBUG")) {
    float t[6];
    cudaEventElapsedTime(&t[0], c->ev_chunk[0], c->ev_chunk[1]);
    cudaEventElapsedTime(&t[1], c->ev_chunk[1], c->ev_chunk[7]);
    cudaEventElapsedTime(&t[2], c->ev_chunk[7], c->ev_chunk[2]);
    cudaEventElapsedTime(&t[3], c->ev_chunk[2], c->ev_chunk[3]);
    cudaEventElapsedTime(&t[4], c->ev_chunk[3], c->ev_chunk[4]);
    cudaEventElapsedTime(&t[5], c->ev_begin, c->ev_chunk[0]);
    fprintf(stderr,
            "band: pre %.3f bound %.3f seeds %.3f gap %.3f collect+group %.3f filter+count+exact %.3f ms\n",
            t[5], t[0], t[1], t[2], t[3], t[4]);
  }
  return LMS_OK;
}

int band_solve(lms_ctx* c, const HostFit& h, lms_stats* st) {
  if (c->capturing) {  // a capture an error path left open: drop it, no graphs
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(c->stream, &g);
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
    c->capturing = false;
    c->use_graph = 0;
  }
  const int64_t span = h.r1 - h.r0;
  bool filter_timed = false, sweep_timed = false, bound_timed = false;
  bool defer_bounds = false;  // two-phase bounds (LMSB_DEFER)
  ShardSpec* sh = c->shard;
  const int64_t P0 = sh ? sh->P0 : h.r0;
  const int64_t pspan = sh ? sh->P1 - sh->P0 : span;
  // large n: bands of >= 32 n vertices (their keys are sorted in global memory)
  const bool big = h.n > lmsb::kBandMaxN;
  const bool coarse = c->band_coarse == 1 || (c->band_coarse == 2 && big);
  const int64_t bv0 = band_size(c->band_vertices, h.n);
  const int64_t bv = big ? std::max<int64_t>(bv0, big_band_mult(c->big_mult, h.n) * h.n) : bv0;
  const int K = (int)std::max<int64_t>(3, std::min<int64_t>(lmsb::kBandMaxK, (pspan + bv - 1) / bv));
  const int64_t S =
      std::min<int64_t>(pspan, std::min<int64_t>(1 << 20, std::max<int64_t>(64 * K, 1 << 16)));
  // bands bounded here: all, or the shard's slice (plan), or none (search:
  // every band's bound comes from the caller)
  int64_t k0 = 0, k1 = K;
  // plan: the shard's bands are interleaved (k = shard + t * nshards), so the
  // bands near the optimum slope -- the ones that need exact bounds -- are
  // spread over all shards
  std::vector<int32_t> slice_ids;
  if (sh && sh->mode == 1) {
    for (int64_t k = sh->shard; k < K; k += sh->nshards) slice_ids.push_back((int32_t)k);
    k0 = k1 = 0;
  }
  if (sh && sh->mode == 2) {
    if (sh->K_in != K)
      return set_error(LMS_ERR_INVALID, "shard search: %lld bands given, the plan has %d",
                       (long long)sh->K_in, K);
    k0 = k1 = 0;
  }
  if (sh && sh->mode == 3) k0 = k1 = 0;  // own bands' bounds come from this context's plan
  const int kSeedBands = c->seed_bands;
  const int64_t seed_cap = S;
  RC_TRY(c->bsample.need(2 * S));
  RC_TRY(c->bbounds.need(K));
  RC_TRY(c->bscnt.need(K));
  RC_TRY(c->bflag.need(K + 1));
  RC_TRY(c->bscal.need(9));  // [5]: running best height bits of the exact launches, [6]: prepass,
                             // [7]: filter chunks of the sub-band grouping
  RC_TRY(c->bstart.need(K + 1));
  RC_TRY(c->bend.need(K + 1));
  RC_TRY(c->blb.need(K));
  RC_TRY(c->bwq.need(K));
  RC_TRY(c->blist.need(std::max(K + 1, 128)));
  RC_TRY(c->btemp.need((int64_t)lmsb::band_sample_temp_bytes(S)));
  RC_TRY(c->ranks.need(seed_cap));
  RC_TRY(c->item_fit.need(seed_cap));
  RC_TRY(c->recs.need(seed_cap));

  lmsb::BandFit bf{};
  bf.a = c->a + h.off;
  bf.b = c->b + h.off;
  bf.n = h.n;
  bf.q = h.q;
  bf.R0 = h.r0;
  bf.span = span;
  bf.P0 = P0;
  bf.pspan = pspan;
  double alo, ahi, am, bmx;
  line_stats(c, h.off, h.n, &alo, &ahi, &am, &bmx);
  bf.c = 0.5 * alo + 0.5 * ahi;
  bf.dev = std::max(ahi - bf.c, bf.c - alo) * (1.0 + 0x1p-40) + 1e-300;
  bf.amax = am;
  bf.bmax = bmx;
  // ---- CUDA graph: a device-planned search (no host step between its
  // launches) is captured on the second fit with the same key -- shape, line
  // statistics (the kernels' by-value arguments), member capacity, buffer
  // epoch -- and replayed from then on; the replay recomputes everything from
  // the lines in the context's buffers
  const bool sweep_n = (c->band_sweep == 1 || (c->band_sweep == 2 && h.n >= kSweepMinN)) &&
                       h.n <= lmsb::kBandMaxBigN;
  const bool dplan_pre = c->device_plan && !sh && !big && !coarse && c->filter_keys &&
                         c->group_mode == 3 && !c->band_direct && sweep_n &&
                         K <= lmsb::kPlanMaxK && c->plan_cap_n == h.n && c->plan_cap > 0 &&
                         !c->force_host_plan;
  const bool graph_ok = c->use_graph && dplan_pre && !c->trace && !c->sync_check;
  unsigned char gk[sizeof(c->gkey)];
  std::memset(gk, 0, sizeof(gk));
  const uint64_t epoch0 = g_buf_epoch.load();
  {
    struct GraphKey {
      int64_t n, q, off, r0, span, P0, pspan, K, S, cap, wide, narrow, sub;
      uint64_t epoch;
      double c, dev, amax, bmax, tau;
    } key;
    std::memset(&key, 0, sizeof(key));
    key.n = h.n;
    key.q = h.q;
    key.off = h.off;
    key.r0 = h.r0;
    key.span = span;
    key.P0 = P0;
    key.pspan = pspan;
    key.K = K;
    key.S = S;
    key.cap = c->plan_cap;
    key.wide = c->wide_chunk;
    key.narrow = c->narrow_chunk;
    key.sub = c->sub_samples;
    key.epoch = epoch0;
    key.c = bf.c;
    key.dev = bf.dev;
    key.amax = bf.amax;
    key.bmax = bf.bmax;
    key.tau = c->bkeys_tau;
    static_assert(sizeof(key) <= sizeof(gk), "graph key size");
    std::memcpy(gk, &key, sizeof(key));
  }
  if (graph_ok && c->gexec && std::memcmp(gk, c->gkey, sizeof(gk)) == 0) {
    CUDA_TRY(cudaGraphLaunch(c->gexec, c->stream));
    st->launches += c->g_launches;
    st->bands = K;
    return band_finish(c, h, st,
                       BandTail{(unsigned long long)c->plan_cap, false, true, true, true, true});
  }
  bool capturing = false;
  int64_t launches0 = st->launches;
  if (graph_ok) {
    if (std::memcmp(gk, c->gseen, sizeof(gk)) == 0) {
      CUDA_TRY(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeRelaxed));
      capturing = true;
      c->capturing = true;
    }
    std::memcpy(c->gseen, gk, sizeof(gk));
  }
  trace_mark(c, "begin");
  // interleaved copy of the fit's lines for the collect pass (kept while the
  // bound lines and the fit's offset are unchanged)
  RC_TRY(c->bab.need(h.n));
  if (capturing || c->ab_gen != c->gen || c->ab_off != h.off || c->ab_n != h.n ||
      c->ab_ptr != c->bab.p) {
    lmsb::launch_band_interleave(bf.a, bf.b, h.n, c->bab.p, c->stream);
    st->launches += 1;
    c->ab_gen = c->gen;
    c->ab_off = h.off;
    c->ab_n = h.n;
    c->ab_ptr = c->bab.p;
  }
  trace_mark(c, "interleave");
  bf.ab = c->bab.p;
  // W_q of the slopes a_k (the slope bound of every band, slope_lb), kept
  // while the lines, the fit and q are unchanged
  RC_TRY(c->bwqa.need(1));
  if (capturing || c->wqa_gen != c->gen || c->wqa_off != h.off || c->wqa_n != h.n ||
      c->wqa_q != h.q || !c->slope_bound) {
    lmsb::launch_line_wqa(bf, c->bwqa.p, c->stream);
    st->launches += 1;
    c->wqa_gen = c->gen;
    c->wqa_off = h.off;
    c->wqa_n = h.n;
    c->wqa_q = h.q;
  }

  // [0] valid samples [1] collected [2] seeds [3] band survivors [4] count survivors
  unsigned long long* sc = c->bscal.p;
  CUDA_TRY(cudaMemsetAsync(sc + 5, 0xFF, sizeof(unsigned long long), c->stream));  // no height yet
  CUDA_TRY(cudaMemsetAsync(sc + 8, 0, sizeof(unsigned long long), c->stream));  // raw overflow
  lmsb::BandWork w{};
  w.S = S;
  w.K = K;
  w.sample = c->bsample.p;
  w.sample_sorted = c->bsample.p + S;
  w.nvalid = sc;
  w.bounds = c->bbounds.p;
  w.sample_counts = c->bscnt.p;
  w.flag = c->bflag.p;
  w.ncollect = sc + 1;
  w.start = c->bstart.p;
  w.end = c->bend.p;
  w.temp = c->btemp.p;
  w.temp_bytes = (size_t)c->btemp.cap;
  while (c->ev_chunk.size() < 14) {
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreate(&e));
    c->ev_chunk.push_back(e);
  }
  // exact select + reduce of a survivor list: d_count on the device, or the
  // first `cap` entries when d_count is null
  auto exact_list = [&](unsigned long long* d_count, int64_t cap, const int64_t* ranks,
                        const int32_t* fits) -> int {
    lmsb::ExactArgs xa{};
    xa.a = c->a;
    xa.b = c->b;
    xa.fits = c->fits.p;
    xa.mode = lmsb::kSrcList;
    xa.d_count = d_count;
    xa.count = cap;
    xa.capacity = cap;
    xa.ranks = ranks;
    xa.fit_of = fits;
    xa.bound = c->best.p;
    xa.out = c->recs.p;
    // few vertices (seeds, band survivors): latency-bound, one CTA per vertex
    // with its cut cached; a long list (degenerate q, loose bounds) streams
    // everything beyond the first 8 per SM
    xa.cached = 1;
    xa.cached_end = (int64_t)c->sms * 8;
    xa.live_h = sc + 5;
    lmsb::launch_exact(xa, persistent_grid(c, -1), c->stream, h.n);
    lmsb::launch_reduce(c->recs.p, d_count, d_count ? 0 : cap, cap, c->fits.p, c->keys.p,
                        c->best.p, (int)c->sms * 4, c->stream);
    CUDA_TRY(cudaGetLastError());
    st->launches += 3;
    return LMS_OK;
  };

  // ---- sample, boundaries, per-band lower bounds
  CUDA_TRY(ev_rec(c, c->ev_chunk[0]));
  // a shard search reuses its context's plan (samples, boundaries, counts)
  // when the same fit was planned on it last
  ShardPlanState& sp = c->splan;
  const bool reuse = sh && (sh->mode == 2 || sh->mode == 3) && sp.valid && sp.gen == c->gen &&
                     sp.n == h.n && sp.q == h.q && sp.K == K && sp.S == S && sp.P0 == P0 &&
                     sp.pspan == pspan;
  if (sh && sh->mode == 3 &&
      !(reuse && sp.nshards == sh->nshards && sp.shard == sh->shard))
    return set_error(LMS_ERR_INVALID,
                     "own-band shard search needs the shard's plan on this context first");
  if (!reuse) {
    sp.valid = false;
    if (lmsb::launch_band_sample(bf, w, c->sms, c->stream) != 0)
      return set_error(LMS_ERR_CUDA, "band sample sort failed");
    st->launches += 4;
  }
  trace_mark(c, "sample");
  lmsb::BandArgs ba{};
  ba.K = K;
  ba.band0 = (int)k0;
  ba.bounds = c->bbounds.p;
  ba.start = c->bstart.p;
  ba.end = c->bend.p;
  ba.lb = c->blb.p;
  ba.wq = c->bwq.p;
  RC_TRY(c->bedge.need((int64_t)K * 2 * lmsb::kEdge));
  ba.edge = c->bedge.p;
  ba.best = c->best.p;
  ba.fit = 0;
  ba.wqa = c->slope_bound ? c->bwqa.p : nullptr;
  // stored band keys: bounds computed here (or by this context's own plan
  // for an own-band search), not taken from a caller
  const bool use_bkeys = !big && c->filter_keys && c->group_mode == 3 &&
                         (!sh || sh->mode == 1 || sh->mode == 3);
  if (use_bkeys) {
    ba.bkeys_ld = (h.n + 3) & ~(int64_t)3;
    RC_TRY(c->bkeys.need((int64_t)K * ba.bkeys_ld));
    ba.bkeys = c->bkeys.p;
    ba.bkeys_tau = c->bkeys_tau;
  }
  lmsb::BandBig bg{};
  if (big) {
    constexpr int kBatch = 256;
    RC_TRY(c->bbig_keys.need((int64_t)kBatch * h.n * 2));
    RC_TRY(c->bbig_seg.need(kBatch + 1));
    RC_TRY(c->btemp.need((int64_t)std::max(lmsb::band_sample_temp_bytes(S),
                                           lmsb::band_big_sort_temp_bytes(kBatch, h.n))));
    bg.batch = kBatch;
    bg.keys = c->bbig_keys.p;
    bg.keys_alt = c->bbig_keys.p + (int64_t)kBatch * h.n;
    bg.store = nullptr;  // the filter sorts its own slices (launch_band_slices)
    bg.seg = c->bbig_seg.p;
    bg.temp = c->btemp.p;
    bg.temp_bytes = (size_t)c->btemp.cap;
    if (k1 > k0 && !coarse) {
      if (lmsb::launch_band_bound_big(bf, ba, bg, (int)k0, (int)k1, nullptr, c->stream) != 0)
        return set_error(LMS_ERR_CUDA, "large-n band bound sort failed");
      st->launches += 4 * ((k1 - k0 + kBatch - 1) / kBatch);
    }
  } else if (k1 > k0 && !coarse) {
    CUDA_TRY(ev_rec(c, c->ev_chunk[12]));
    // bands whose slope bound is positive are bounded after the seeds, and
    // only while that bound does not already exceed H (LMSB_DEFER)
    defer_bounds = c->defer_bounds && !sh && ba.wqa;
    lmsb::BandArgs bd = ba;
    bd.defer = defer_bounds ? 1 : 0;
    lmsb::launch_band(bf, bd, 0, (int)(k1 - k0), c->stream);
    CUDA_TRY(ev_rec(c, c->ev_chunk[13]));
    bound_timed = true;
    st->launches += 1;
  }
  if (k1 > k0 && coarse) {  // sort-free bounds; exact ones only where needed
    lmsb::launch_band_coarse(bf, ba, (int)(k1 - k0), c->stream);
    st->launches += 1;
  }
  trace_mark(c, "bound");
  // exact (sorted-key) bounds, window widths and edge keys of `nb` listed bands
  // (device list; entries < 0 are skipped)
  auto exact_bounds = [&](const int32_t* d_ids, int nb) -> int {
    if (nb <= 0) return LMS_OK;
    lmsb::BandArgs bx = ba;
    bx.band0 = 0;
    bx.band_ids = d_ids;
    if (big) {
      if (lmsb::launch_band_bound_big(bf, bx, bg, 0, nb, d_ids, c->stream) != 0)
        return set_error(LMS_ERR_CUDA, "large-n band bound sort failed");
      st->launches += 4 * ((nb + bg.batch - 1) / bg.batch);
    } else {
      lmsb::launch_band(bf, bx, 0, nb, c->stream);
      st->launches += 1;
    }
    CUDA_TRY(cudaGetLastError());
    return LMS_OK;
  };
  CUDA_TRY(cudaGetLastError());
  // small readbacks through pinned staging (truly asynchronous copies)
  const size_t pin_rb = ((size_t)K * (2 * sizeof(double) + sizeof(float) + sizeof(unsigned)) +
                        sizeof(lms_candidate) + 64 + 255) & ~(size_t)255;
  // upload staging: collected bands (or a shard's slice), grouping slots, slot identity
  const size_t pin_up = (size_t)(K + 1) * (2 * sizeof(int32_t) + sizeof(int16_t)) + 1024;
  // a search's band table goes up through pinned staging as well
  const size_t pin_tab = (sh && sh->mode == 2) ? (size_t)K * (2 * sizeof(double) +
                                                              2 * lmsb::kEdge * sizeof(float)) : 0;
  // sweep collect: run ends and band ranges (lms_sweep.cu)
  const size_t pin_sw = (size_t)kSweepMaxRuns * (2 * sizeof(lmsb::SweepEnd) + 2 * sizeof(int32_t)) +
                        sizeof(lmsb::SweepEnd) + 64;
  // sub-band grouping: group firsts and bands
  const size_t pin_sub = (size_t)(K + 3 + lmsb::kSubMaxGroups) * sizeof(int32_t) + 64;
  RC_TRY(ensure_pinned(c, pin_rb + pin_up + pin_tab + pin_sw + pin_sub));
  int32_t* u_sub = reinterpret_cast<int32_t*>(
      ((uintptr_t)(c->pin + pin_rb + pin_up + pin_tab + pin_sw) + 15) & ~(uintptr_t)15);
  unsigned char* u_sweep = reinterpret_cast<unsigned char*>(
      ((uintptr_t)(c->pin + pin_rb + pin_up + pin_tab) + 15) & ~(uintptr_t)15);
  // upload staging after the readbacks
  int32_t* u_list = reinterpret_cast<int32_t*>(((uintptr_t)(c->pin + pin_rb) + 15) & ~(uintptr_t)15);
  double* p_lb = reinterpret_cast<double*>(c->pin);
  double* p_wq = p_lb + K;
  lms_candidate* p_hb = reinterpret_cast<lms_candidate*>(p_wq + K);
  float* p_bnd = reinterpret_cast<float*>(p_hb + 1);
  unsigned* p_scnt = reinterpret_cast<unsigned*>(p_bnd + K);
  const int nsl = (int)slice_ids.size();
  if (nsl > 0) {  // plan: bounds of the shard's interleaved slice
    RC_TRY(c->bslice_ids.need(nsl));
    std::memcpy(u_list, slice_ids.data(), sizeof(int32_t) * nsl);  // staging (K + 1 entries)
    CUDA_TRY(cudaMemcpyAsync(c->bslice_ids.p, u_list, sizeof(int32_t) * nsl,
                             cudaMemcpyHostToDevice, c->stream));
    if (coarse) {
      lmsb::BandArgs bx = ba;
      bx.band0 = 0;
      bx.band_ids = c->bslice_ids.p;
      lmsb::launch_band_coarse(bf, bx, nsl, c->stream);
      st->launches += 1;
    } else {
      RC_TRY(exact_bounds(c->bslice_ids.p, nsl));
    }
    trace_mark(c, "plan_bounds");
  }

  if (sh && sh->mode == 1) {
    // ---- plan: seeds from the slice's narrowest windows (picked on the
    // device), exact bounds of the slice's bands this shard's seed height
    // cannot dismiss, then one readback of the slice's table, the seed
    // record, the boundaries and the sample counts
    const int T = std::max(2, (kSeedBands + sh->nshards - 1) / sh->nshards);
    const int32_t* d_sl = c->bslice_ids.p;
    const int32_t* d_seed = c->blist.p;
    if (nsl > 0) {
      if (coarse) {
        // a pool of the narrowest coarse windows gets exact bounds (and edge
        // keys); the T narrowest exact windows among them seed
        // (the pools of all shards together cover the one-GPU pool: each
        // shard's share of the narrowest windows shrinks as 1 / shards)
        const int kPool = c->plan_pool > 0
                              ? c->plan_pool
                              : std::max(4 * T, (64 + sh->nshards - 1) / sh->nshards);
        lmsb::launch_band_top(c->bwq.p, 0, nsl, K, kPool, c->blist.p, c->bflag.p, c->stream, d_sl);
        RC_TRY(exact_bounds(c->blist.p, kPool));
        lmsb::launch_band_top(c->bwq.p, 0, kPool, K, T, c->blist.p + kPool, c->bflag.p, c->stream,
                              c->blist.p);
        d_seed = c->blist.p + kPool;
        st->launches += 2;
        trace_mark(c, "plan_pool");
      } else {
        lmsb::launch_band_top(c->bwq.p, 0, nsl, K, T, c->blist.p, c->bflag.p, c->stream, d_sl);
      }
      CUDA_TRY(cudaMemsetAsync(sc + 2, 0, sizeof(unsigned long long), c->stream));
      lmsb::launch_band_edge_seeds(bf, ba, d_seed, T, c->ranks.p, c->item_fit.p, seed_cap, sc + 2,
                                   c->stream);
      lmsb::launch_band_seeds(bf, w, c->ranks.p, c->item_fit.p, 0, seed_cap, sc + 2, c->stream);
      RC_TRY(exact_list(sc + 2, seed_cap, c->ranks.p, c->item_fit.p));
      st->launches += 3;
      trace_mark(c, "plan_seeds");
    } else {  // no bands here: only the sample counts
      CUDA_TRY(cudaMemsetAsync(c->bflag.p, 0, K, c->stream));
      CUDA_TRY(cudaMemsetAsync(sc + 2, 0, sizeof(unsigned long long), c->stream));
      lmsb::launch_band_seeds(bf, w, c->ranks.p, c->item_fit.p, 0, 0, sc + 2, c->stream);
    }
    if (sh->lb_out && nsl > sh->cap)
      return set_error(LMS_ERR_INVALID, "shard plan: %d bands exceed the capacity %lld", nsl,
                       (long long)sh->cap);
    if (coarse && nsl > 0) {
      // the global seed height is never above this shard's, so bands it
      // cannot dismiss are all the search could need exactly
      CUDA_TRY(cudaMemcpyAsync(p_hb, c->best.p, sizeof(lms_candidate), cudaMemcpyDeviceToHost,
                               c->stream));
      CUDA_TRY(cudaMemcpyAsync(p_lb, c->blb.p, sizeof(double) * K, cudaMemcpyDeviceToHost,
                               c->stream));
      CUDA_TRY(cudaStreamSynchronize(c->stream));
      const double Hs = p_hb->found ? p_hb->height : INFINITY;
      std::vector<int32_t> cand;
      for (int32_t k : slice_ids)
        if (p_lb[k] <= Hs * (1.0 + 0x1p-19) && std::isfinite(p_lb[k])) cand.push_back(k);
      if (!cand.empty()) {
        std::copy(cand.begin(), cand.end(), u_list);
        CUDA_TRY(cudaMemcpyAsync(c->blist.p, u_list, sizeof(int32_t) * cand.size(),
                                 cudaMemcpyHostToDevice, c->stream));
        RC_TRY(exact_bounds(c->blist.p, (int)cand.size()));
      }
      st->bands_refined = (int64_t)cand.size();
      trace_mark(c, "plan_refine");
    }
    std::vector<float> h_edge((size_t)K * 2 * lmsb::kEdge);
    CUDA_TRY(cudaMemcpyAsync(p_lb, c->blb.p, sizeof(double) * K, cudaMemcpyDeviceToHost,
                             c->stream));
    CUDA_TRY(cudaMemcpyAsync(p_wq, c->bwq.p, sizeof(double) * K, cudaMemcpyDeviceToHost,
                             c->stream));
    CUDA_TRY(cudaMemcpyAsync(p_hb, c->best.p, sizeof(lms_candidate), cudaMemcpyDeviceToHost,
                             c->stream));
    CUDA_TRY(cudaMemcpyAsync(p_bnd, c->bbounds.p, sizeof(float) * (K - 1), cudaMemcpyDeviceToHost,
                             c->stream));
    CUDA_TRY(cudaMemcpyAsync(p_scnt, c->bscnt.p, sizeof(unsigned) * K, cudaMemcpyDeviceToHost,
                             c->stream));
    CUDA_TRY(cudaMemcpyAsync(h_edge.data(), c->bedge.p, sizeof(float) * h_edge.size(),
                             cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    for (int t = 0; t < nsl && sh->lb_out; ++t) {
      const int32_t k = slice_ids[t];
      sh->lb_out[t] = p_lb[k];
      sh->wq_out[t] = p_wq[k];
      std::memcpy(sh->edge_out + (size_t)t * 2 * lmsb::kEdge,
                  h_edge.data() + (size_t)k * 2 * lmsb::kEdge, sizeof(float) * 2 * lmsb::kEdge);
    }
    trace_mark(c, "plan_readback");
    sh->seed_out = nsl > 0 ? *p_hb : lms_candidate{};
    sh->K = K;
    sh->k0 = nsl;  // bands in the slice (shard, shard + nshards, ...)
    sh->k1 = nsl;
    sp.h_bnd.assign(p_bnd, p_bnd + (K - 1));
    sp.h_scnt.assign(p_scnt, p_scnt + K);
    sp.h_lb.assign(K, INFINITY);
    for (int32_t k : slice_ids) sp.h_lb[k] = p_lb[k];
    sp.nshards = sh->nshards;
    sp.shard = sh->shard;
    sp.valid = true;
    sp.gen = c->gen;
    sp.n = h.n;
    sp.q = h.q;
    sp.K = K;
    sp.S = S;
    sp.P0 = P0;
    sp.pspan = pspan;
    st->bands = K;
    st->seed_height = sh->seed_out.found ? sh->seed_out.height : INFINITY;
    CUDA_TRY(ev_rec(c, c->ev_chunk[1]));
    return LMS_OK;
  }

  // device-side plan (no readback after the seeds): the one-fit default path
  // once this context has a member capacity for n (a host-planned fit sets it)
  const bool dplan = c->device_plan && !sh && !big && !coarse && use_bkeys && !c->band_direct &&
                     (c->band_sweep == 1 || (c->band_sweep == 2 && h.n >= kSweepMinN)) &&
                     K <= lmsb::kPlanMaxK && c->plan_cap_n == h.n && c->plan_cap > 0 &&
                     !c->force_host_plan;
  std::vector<double>& lb = c->h_blb;
  std::vector<float> hbnd;
  std::vector<double> wq;
  std::vector<unsigned> scnt;
  double H = INFINITY;
  std::vector<uint8_t> flag(K + 1, 0);
  if (sh && sh->mode == 3) {
    // ---- own-band search: this shard's bands (shard, shard + nshards, ...)
    // with the bounds its own plan computed, every other band dismissed, the
    // global seed record (exchanged) installed; the whole pair space searched
    if (sh->seed_in.found) {
      lms_candidate* p_seed = p_hb;
      *p_seed = sh->seed_in;
      p_seed->reserved = 0;
      CUDA_TRY(cudaMemcpyAsync(c->recs.p, p_seed, sizeof(lms_candidate), cudaMemcpyHostToDevice,
                               c->stream));
      lmsb::launch_reduce(c->recs.p, nullptr, 1, 1, c->fits.p, c->keys.p, c->best.p, 1,
                          c->stream);
      st->launches += 2;
      H = sh->seed_in.height;
    }
    hbnd = sp.h_bnd;
    scnt = sp.h_scnt;
    lb = sp.h_lb;
    wq.assign(K, INFINITY);
    CUDA_TRY(ev_rec(c, c->ev_chunk[1]));
    CUDA_TRY(ev_rec(c, c->ev_chunk[7]));
  } else if (sh && sh->mode == 2) {
    // ---- search: every band's bound and the global seed record from the
    // caller (the exchanged plan); boundaries and counts from this context's
    // plan, or recomputed
    double* t_lb = reinterpret_cast<double*>(c->pin + pin_rb + pin_up);
    double* t_wq = t_lb + K;
    float* t_edge = reinterpret_cast<float*>(t_wq + K);
    std::memcpy(t_lb, sh->lb_in, sizeof(double) * K);
    std::memcpy(t_wq, sh->wq_in, sizeof(double) * K);
    std::memcpy(t_edge, sh->edge_in, sizeof(float) * K * 2 * lmsb::kEdge);
    CUDA_TRY(cudaMemcpyAsync(c->blb.p, t_lb, sizeof(double) * K, cudaMemcpyHostToDevice,
                             c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->bwq.p, t_wq, sizeof(double) * K, cudaMemcpyHostToDevice,
                             c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->bedge.p, t_edge, sizeof(float) * K * 2 * lmsb::kEdge,
                             cudaMemcpyHostToDevice, c->stream));
    if (sh->seed_in.found) {
      lms_candidate* p_seed = p_hb;
      *p_seed = sh->seed_in;
      p_seed->reserved = 0;
      CUDA_TRY(cudaMemcpyAsync(c->recs.p, p_seed, sizeof(lms_candidate), cudaMemcpyHostToDevice,
                               c->stream));
      lmsb::launch_reduce(c->recs.p, nullptr, 1, 1, c->fits.p, c->keys.p, c->best.p, 1,
                          c->stream);
      st->launches += 2;
      H = sh->seed_in.height;
    }
    if (reuse) {
      hbnd = sp.h_bnd;
      scnt = sp.h_scnt;
    } else {
      CUDA_TRY(cudaMemsetAsync(c->bflag.p, 0, K, c->stream));
      CUDA_TRY(cudaMemsetAsync(sc + 2, 0, sizeof(unsigned long long), c->stream));
      lmsb::launch_band_seeds(bf, w, c->ranks.p, c->item_fit.p, 0, 0, sc + 2, c->stream);  // counts
      st->launches += 1;
      CUDA_TRY(cudaMemcpyAsync(p_bnd, c->bbounds.p, sizeof(float) * (K - 1),
                               cudaMemcpyDeviceToHost, c->stream));
      CUDA_TRY(cudaMemcpyAsync(p_scnt, c->bscnt.p, sizeof(unsigned) * K, cudaMemcpyDeviceToHost,
                               c->stream));
      CUDA_TRY(cudaStreamSynchronize(c->stream));
      hbnd.assign(p_bnd, p_bnd + (K - 1));
      scnt.assign(p_scnt, p_scnt + K);
    }
    lb.assign(sh->lb_in, sh->lb_in + K);
    wq.assign(sh->wq_in, sh->wq_in + K);
    CUDA_TRY(ev_rec(c, c->ev_chunk[1]));
    CUDA_TRY(ev_rec(c, c->ev_chunk[7]));
  } else {
    CUDA_TRY(ev_rec(c, c->ev_chunk[1]));
    // ---- seeds, picked on the device (no round trip after the bounds): the
    // bands with the narrowest q-windows at their centre slope (the bands an
    // LMS line of that slope would come from); with coarse bounds a pool of
    // the kSeedPool narrowest coarse windows gets exact bounds first and the
    // kSeedBands narrowest exact windows among them seed
    constexpr int kSeedPool = 64;
    const int32_t* d_seed = c->blist.p;
    if (coarse) {
      lmsb::launch_band_top(c->bwq.p, 0, K, K, kSeedPool, c->blist.p, c->bflag.p, c->stream);
      RC_TRY(exact_bounds(c->blist.p, kSeedPool));
      lmsb::launch_band_top(c->bwq.p, 0, kSeedPool, K, kSeedBands, c->blist.p + kSeedPool,
                            c->bflag.p, c->stream, c->blist.p);
      d_seed = c->blist.p + kSeedPool;
      st->launches += 2;
    }
    trace_mark(c, "top");
    // the window-edge pairs (usually the optimum itself) and, as a safety net,
    // up to 16 sampled vertices of each of the same bands, in one exact launch
    CUDA_TRY(cudaMemsetAsync(sc + 2, 0, sizeof(unsigned long long), c->stream));
    if (coarse)
      lmsb::launch_band_edge_seeds(bf, ba, d_seed, kSeedBands, c->ranks.p, c->item_fit.p, seed_cap,
                                   sc + 2, c->stream);
    else  // the kSeedBands narrowest windows pick themselves (no top-k launch)
      lmsb::launch_band_edge_seeds_top(bf, ba, kSeedBands, c->bflag.p, c->ranks.p, c->item_fit.p,
                                       seed_cap, sc + 2, c->stream);
    lmsb::launch_band_seeds(bf, w, c->ranks.p, c->item_fit.p, 0, seed_cap, sc + 2, c->stream);
    RC_TRY(exact_list(sc + 2, seed_cap, c->ranks.p, c->item_fit.p));
    if (defer_bounds) {
      lmsb::BandArgs bd = ba;
      bd.defer = 2;
      lmsb::launch_band(bf, bd, 0, (int)(k1 - k0), c->stream);
      st->launches += 1;
    }
    CUDA_TRY(ev_rec(c, c->ev_chunk[7]));
    trace_mark(c, "seeds");
    if (!dplan) {
    // one readback: bounds, window widths, boundaries, the seed record, counts
    CUDA_TRY(cudaMemcpyAsync(p_wq, c->bwq.p, sizeof(double) * K, cudaMemcpyDeviceToHost,
                             c->stream));
    CUDA_TRY(cudaMemcpyAsync(p_lb, c->blb.p, sizeof(double) * K, cudaMemcpyDeviceToHost,
                             c->stream));
    CUDA_TRY(cudaMemcpyAsync(p_bnd, c->bbounds.p, sizeof(float) * (K - 1), cudaMemcpyDeviceToHost,
                             c->stream));
    CUDA_TRY(cudaMemcpyAsync(p_hb, c->best.p, sizeof(lms_candidate), cudaMemcpyDeviceToHost,
                             c->stream));
    CUDA_TRY(cudaMemcpyAsync(p_scnt, c->bscnt.p, sizeof(unsigned) * K, cudaMemcpyDeviceToHost,
                             c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    lb.assign(p_lb, p_lb + K);
    hbnd.assign(p_bnd, p_bnd + (K - 1));
    wq.assign(p_wq, p_wq + K);
    const lms_candidate hb = *p_hb;
    scnt.assign(p_scnt, p_scnt + K);
    H = hb.found ? hb.height : INFINITY;
    trace_mark(c, "readback1");
    }
  }
  if (capturing && !dplan) {  // (cannot happen: the key's conditions are dplan's)
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(c->stream, &g);
    c->capturing = false;
    if (g) cudaGraphDestroy(g);
    c->use_graph = 0;
    c->ab_gen = ~0ull;
    c->wqa_gen = ~0ull;
    return band_solve(c, h, st);
  }
  // (set by the host plan below, or by the device plan)
  std::vector<int32_t> list;
  int nslot = 0;
  unsigned long long m = 0;
  int64_t nchunk_max = 0;  // > 0: filter chunks from the sub-band grouping's table
  bool direct = false;
  int ngroups = 0;
  if (dplan) {
    RC_TRY(devplan_search(c, h, st, bf, ba, w, K, S, sc, &m, &nchunk_max));
    sweep_timed = true;
  } else {
  if (coarse && !(sh && (sh->mode == 2 || sh->mode == 3))) {  // (a shard's plan refined its own slice)
    // the bands the coarse bounds cannot dismiss get their exact bound
    std::vector<int32_t> cand;
    for (int k = 0; k < K; ++k)
      if (lb[k] <= H * (1.0 + 0x1p-19) && std::isfinite(lb[k])) cand.push_back(k);
    if (!cand.empty()) {
      std::copy(cand.begin(), cand.end(), u_list);
      CUDA_TRY(cudaMemcpyAsync(c->blist.p, u_list, sizeof(int32_t) * cand.size(),
                               cudaMemcpyHostToDevice, c->stream));
      RC_TRY(exact_bounds(c->blist.p, (int)cand.size()));
      CUDA_TRY(cudaMemcpyAsync(p_lb, c->blb.p, sizeof(double) * K, cudaMemcpyDeviceToHost,
                               c->stream));
      CUDA_TRY(cudaStreamSynchronize(c->stream));
      for (int32_t k : cand) lb[k] = p_lb[k];
    }
    st->bands_refined = (int64_t)cand.size();
  }
  std::vector<int32_t> order(K);
  for (int k = 0; k < K; ++k) order[k] = k;
  std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) { return lb[x] < lb[y]; });
  st->bands = K;
  st->seed_height = H;

  // ---- collect the vertices of the bands whose bound admits H
  double est = 0.0;
  for (int e = 0; e < K; ++e) {
    const int32_t k = order[e];
    if (!(lb[k] <= H * (1.0 + 0x1p-19))) break;  // ascending: the rest cannot reach H
    list.push_back(k);
    est += (double)scnt[k] + 2.0;
  }
  st->bands_searched = (int64_t)list.size();
  if (getenv("LMSB_DEBUG_BANDS")) {
    for (int32_t k : list) {
      double uL = -INFINITY, uR = INFINITY;
      if (k > 0 && k < K) uL = (double)std::nextafter(hbnd[k - 1], -INFINITY);
      if (k < K - 1) uR = (double)hbnd[k];
      fprintf(stderr, "band %d lb %.4g wq %.4g uL %.6g uR %.6g devw/H %.4g scnt %u\n", k,
              k < K ? lb[k] : 0.0, k < K ? wq[k] : 0.0, uL, uR, bf.dev * (uR - uL) / H,
              k < K ? scnt[k] : 0u);
    }
  }
  std::fill(flag.begin(), flag.end(), 0);
  for (int32_t k : list) flag[k] = 1;
  list.push_back(K);  // vertices beyond the key range
  int64_t cap = std::min<int64_t>(span, (int64_t)(2.0 * est * (double)span / (double)S) + 65536);
  cap = std::max(cap, std::min<int64_t>(span, c->collect_floor));
  if (c->cap_test && c->collect_floor == 0) cap = std::min<int64_t>(cap, 4096);  // (tests)
  if (!sh && !big) {  // member capacity for later device-planned fits of this n
    if (c->plan_cap_n != h.n) c->plan_cap = 0;
    c->plan_cap = std::max(c->plan_cap, cap);
    c->plan_cap_n = h.n;
  }
  std::copy(list.begin(), list.end(), u_list);
  CUDA_TRY(cudaMemcpyAsync(c->blist.p, u_list, sizeof(int32_t) * list.size(),
                           cudaMemcpyHostToDevice, c->stream));
  // grouping slot of every band (its index in `list`, -1 when not collected;
  // the beyond-range pseudo band last): the grouping sort keys on the slot
  nslot = (int)list.size();
  {
    int16_t* u_slot = reinterpret_cast<int16_t*>(u_list + (K + 1));
    int32_t* u_ident =
        reinterpret_cast<int32_t*>(((uintptr_t)(u_slot + (K + 1)) + 15) & ~(uintptr_t)15);
    for (int k = 0; k <= K; ++k) u_slot[k] = -1;
    for (int e = 0; e < nslot; ++e) {
      u_slot[list[e]] = (int16_t)e;
      u_ident[e] = e;
    }
    RC_TRY(c->bslot.need(K + 1));
    RC_TRY(c->bident.need(K + 1));
    CUDA_TRY(cudaMemcpyAsync(c->bslot.p, u_slot, sizeof(int16_t) * (K + 1), cudaMemcpyHostToDevice,
                             c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->bident.p, u_ident, sizeof(int32_t) * nslot,
                             cudaMemcpyHostToDevice, c->stream));
    w.slot = c->bslot.p;
    w.nslot = nslot;
  }
  // slope runs of the flagged bands for the collect pre-test, merged across the
  // smallest gaps down to kMaxRuns
  std::vector<std::pair<int, int>> rr;
  for (int k = 0; k < K; ++k) {
    if (!flag[k]) continue;
    if (!rr.empty() && rr.back().second == k - 1) rr.back().second = k;
    else rr.push_back({k, k});
  }
  while ((int)rr.size() > lmsb::kMaxRuns) {
    size_t best = 0;
    for (size_t e = 1; e + 1 < rr.size(); ++e)
      if (rr[e + 1].first - rr[e].second < rr[best + 1].first - rr[best].second) best = e;
    rr[best].second = rr[best + 1].second;
    rr.erase(rr.begin() + best + 1);
  }
  lmsb::BandRuns runs{};
  runs.count = (int)rr.size();
  if (runs.count == 0) {  // nothing flagged: an empty run (only beyond-range vertices)
    runs.count = 1;
    runs.lo[0] = INFINITY;
    runs.hi[0] = -INFINITY;
  }
  for (int e = 0; e < (int)rr.size(); ++e) {  // (no run: the empty run set above)
    const int k0 = rr[e].first, k1 = rr[e].second;
    const double lo = k0 == 0 ? -INFINITY : (double)std::nextafter(hbnd[k0 - 1], -INFINITY);
    const double hi = k1 == K - 1 ? INFINITY : (double)hbnd[k1];
    runs.lo[e] = -INFINITY;
    runs.hi[e] = INFINITY;
    if (std::isfinite(lo)) {
      const double w = lo - (0x1p-18 * std::fabs(lo) + 1e-37);
      float f = (float)w;
      if ((double)f > w) f = std::nextafter(f, -INFINITY);
      runs.lo[e] = f;
    }
    if (std::isfinite(hi)) {
      const double w = hi + (0x1p-18 * std::fabs(hi) + 1e-37);
      float f = (float)w;
      if ((double)f < w) f = std::nextafter(f, INFINITY);
      runs.hi[e] = f;
    }
  }
  trace_mark(c, "plan_upload");
  CUDA_TRY(ev_rec(c, c->ev_chunk[2]));
  // direct grouping into sub-band regions (falls back to the sorting path on a
  // region overflow)
  std::vector<int64_t> gstart, gend;
  if (c->band_direct) {
    const int nadm = (int)list.size() - 1;  // the last entry is the beyond-range pseudo band
    std::vector<int32_t> sbf(nadm + 1, 0);
    std::vector<int64_t> gcap;
    std::vector<int32_t> gband;
    std::vector<int16_t> slot(K, -1);
    const double per_sample = (double)span / (double)S;
    for (int e = 0; e < nadm; ++e) {
      const int32_t k = list[e];
      slot[k] = (int16_t)e;
      const double est = (double)scnt[k] * per_sample;
      int Se = (int)std::ceil(est / (double)c->band_chunk);
      Se = std::max(1, std::min({Se, 64, (int)(scnt[k] / 4)}));
      sbf[e + 1] = sbf[e] + Se;
      // sub-band quantiles rest on ~16-32 samples each: room for 4x the mean
      const int64_t cap_g = (int64_t)std::min(est + 1.0, 4.0 * est / Se) + 4096;
      for (int t = 0; t < Se; ++t) {
        gcap.push_back(cap_g);
        gband.push_back(k);
      }
    }
    const int G = sbf[nadm];
    gcap.push_back(65536);  // beyond-range vertices
    gband.push_back(K);
    ngroups = G + 1;
    std::vector<int64_t> rstart(ngroups + 1, 0);
    for (int g = 0; g < ngroups; ++g) rstart[g + 1] = rstart[g] + gcap[g];
    const int64_t total_cap = rstart[ngroups];
    const int nsub = G - nadm;
    if (nadm < 32767 && total_cap < ((int64_t)1 << 31) &&
        lmsb::band_direct_smem(K, nsub, nadm) <= 200 * 1024) {
      RC_TRY(c->bmem.need(total_cap));
      RC_TRY(c->dg_i32.need((int64_t)(nadm + 1) + 2 * (int64_t)ngroups + 1));
      RC_TRY(c->dg_i64.need(2 * (int64_t)ngroups + 2));
      RC_TRY(c->dg_cursor.need(ngroups));
      RC_TRY(c->dg_sub.need(std::max(nsub, 1)));
      RC_TRY(c->dg_slot.need(K));
      RC_TRY(c->bstart.need(std::max<int64_t>(ngroups, K + 1)));
      RC_TRY(c->bend.need(std::max<int64_t>(ngroups, K + 1)));
      w.start = c->bstart.p;
      w.end = c->bend.p;
      ba.start = c->bstart.p;
      ba.end = c->bend.p;
      int32_t* d_list = c->blist.p;  // list[0..nadm) already uploaded
      int32_t* d_sbf = c->dg_i32.p;
      int32_t* d_gband = d_sbf + (nadm + 1);
      int32_t* d_glist = d_gband + ngroups;
      int64_t* d_cap = c->dg_i64.p;
      int64_t* d_rstart = d_cap + ngroups;
      std::vector<int32_t> glist(ngroups);
      for (int g = 0; g < ngroups; ++g) glist[g] = g;
      CUDA_TRY(cudaMemcpyAsync(d_sbf, sbf.data(), sizeof(int32_t) * (nadm + 1),
                               cudaMemcpyHostToDevice, c->stream));
      CUDA_TRY(cudaMemcpyAsync(d_gband, gband.data(), sizeof(int32_t) * ngroups,
                               cudaMemcpyHostToDevice, c->stream));
      CUDA_TRY(cudaMemcpyAsync(d_glist, glist.data(), sizeof(int32_t) * ngroups,
                               cudaMemcpyHostToDevice, c->stream));
      CUDA_TRY(cudaMemcpyAsync(d_cap, gcap.data(), sizeof(int64_t) * ngroups,
                               cudaMemcpyHostToDevice, c->stream));
      CUDA_TRY(cudaMemcpyAsync(d_rstart, rstart.data(), sizeof(int64_t) * ngroups,
                               cudaMemcpyHostToDevice, c->stream));
      CUDA_TRY(cudaMemcpyAsync(c->dg_slot.p, slot.data(), sizeof(int16_t) * K,
                               cudaMemcpyHostToDevice, c->stream));
      CUDA_TRY(cudaMemsetAsync(c->dg_cursor.p, 0, sizeof(unsigned long long) * ngroups, c->stream));
      lmsb::BandDirect dg{};
      dg.nadm = nadm;
      dg.list = d_list;
      dg.sb_first = d_sbf;
      dg.nsub = nsub;
      dg.sub = c->dg_sub.p;
      dg.slot = c->dg_slot.p;
      dg.force_group = G;
      dg.cursor = c->dg_cursor.p;
      dg.cap = d_cap;
      dg.rstart = d_rstart;
      dg.members = c->bmem.p;
      CUDA_TRY(ev_rec(c, c->ev_chunk[5]));
      lmsb::launch_band_collect_direct(bf, w, runs, dg, c->sms, c->stream);
      CUDA_TRY(ev_rec(c, c->ev_chunk[6]));
      CUDA_TRY(cudaGetLastError());
      st->launches += 2;
      std::vector<unsigned long long> cur(ngroups);
      CUDA_TRY(cudaMemcpyAsync(cur.data(), c->dg_cursor.p, sizeof(unsigned long long) * ngroups,
                               cudaMemcpyDeviceToHost, c->stream));
      CUDA_TRY(cudaStreamSynchronize(c->stream));
      bool overflow = false;
      gstart.assign(ngroups, 0);
      gend.assign(ngroups, 0);
      for (int g = 0; g < ngroups; ++g) {
        overflow |= (int64_t)cur[g] > gcap[g];
        m += cur[g];
        gstart[g] = rstart[g];
        gend[g] = rstart[g] + std::min<int64_t>((int64_t)cur[g], gcap[g]);
      }
      if (overflow && getenv("LMSB_BAND_DEBUG")) {
        for (int g = 0; g < ngroups; ++g)
          if ((int64_t)cur[g] > gcap[g])
            fprintf(stderr, "band direct: group %d (band %d) %llu > cap %lld\n", g, gband[g],
                    (unsigned long long)cur[g], (long long)gcap[g]);
      }
      if (!overflow) {
        direct = true;
        CUDA_TRY(cudaMemcpyAsync(c->bstart.p, gstart.data(), sizeof(int64_t) * ngroups,
                                 cudaMemcpyHostToDevice, c->stream));
        CUDA_TRY(cudaMemcpyAsync(c->bend.p, gend.data(), sizeof(int64_t) * ngroups,
                                 cudaMemcpyHostToDevice, c->stream));
        ba.list = d_glist;
        ba.group_band = d_gband;
        ba.nlist = ngroups;
        st->direct_groups = ngroups;
      } else {
        m = 0;
      }
    }
  }
  if (!direct) {
  // output-sensitive collect: the vertices of each admitted slope run as the
  // inversions between the lines' orders at its ends (lms_sweep.cu).  Needs
  // every inner boundary inside the fp32-key range, so that vertices beyond
  // it (class 2) can only lie in the two outer bands.
  // an own-band search covers the whole pair space for few bands: always swept
  const bool own_bands = sh && sh->mode == 3;
  bool sweep = (c->band_sweep == 1 || (c->band_sweep == 2 && (h.n >= kSweepMinN || own_bands))) &&
               h.n >= 3 && h.n <= lmsb::kBandMaxBigN;
  // (an own-band search with no admitted band still owns the outer bands'
  // class-2 vertices; otherwise a search needs a run)
  if (rr.empty() && !own_bands) sweep = false;
  for (int k = 0; sweep && k < K - 1; ++k)
    sweep = std::isfinite(hbnd[k]) && std::fabs((double)hbnd[k]) * bf.amax < 1e29;
  lmsb::SweepArgs sa{};
  if (sweep) {
    // runs of flagged bands, merged across the smallest gaps down to
    // kSweepMaxRuns.  The outer bands join for their class-2 vertices (|u|
    // beyond the fp32 key range) unless the near-parallel pass already owns
    // every such pair: |u| amax >= 1e30 needs |da| <= 2 bmax amax / 1e30,
    // so when that is <= tau (and the outer bands' class-1 vertices are
    // dismissed) a one-fit search sorts no lines at the infinite ends
    std::vector<std::pair<int, int>> sr;
    int nr = 0, nseg = 0;
    lmsb::SweepEnd* ends = reinterpret_cast<lmsb::SweepEnd*>(u_sweep);
    int32_t* rk = nullptr;
    double tau = 0.0;
    for (int with_outer = sh ? 1 : 0; with_outer < 2; ++with_outer) {
    sr.clear();
    for (int k = 0; k < K; ++k) {
      const bool outer = with_outer && (k == 0 || k == K - 1) &&
                         (!own_bands || k % sh->nshards == sh->shard);
      if (!(flag[k] || outer)) continue;
      if (!sr.empty() && sr.back().second == k - 1) sr.back().second = k;
      else sr.push_back({k, k});
    }
    while ((int)sr.size() > kSweepMaxRuns) {
      size_t best = 0;
      for (size_t e = 1; e + 1 < sr.size(); ++e)
        if (sr[e + 1].first - sr[e].second < sr[best + 1].first - sr[best].second) best = e;
      sr[best].second = sr[best + 1].second;
      sr.erase(sr.begin() + best + 1);
    }
    nr = (int)sr.size();
    nseg = 2 * nr + 1;
    rk = reinterpret_cast<int32_t*>(ends + nseg);
    tau = 0.0;
    for (int e = 0; e < nr; ++e) {
      const int k0 = sr[e].first, k1 = sr[e].second;
      double lo = -INFINITY, hi = INFINITY;
      if (k0 > 0) {
        lo = (double)std::nextafter(hbnd[k0 - 1], -INFINITY);
        lo -= 0x1p-18 * std::fabs(lo) + 1e-37;
      }
      if (k1 < K - 1) {
        hi = (double)hbnd[k1];
        hi += 0x1p-18 * std::fabs(hi) + 1e-37;
      }
      // clearance of the sort ends: relative to the run's magnitude and width
      // (not more: a wide sparse run next to a dense slope region must not
      // reach into it)
      double m;
      if (std::isfinite(lo) && std::isfinite(hi))
        m = 0x1p-20 * (std::max(std::fabs(lo), std::fabs(hi)) + (hi - lo)) + 1e-300;
      else
        m = 0x1p-20 * (std::isfinite(lo) ? std::fabs(lo) : std::isfinite(hi) ? std::fabs(hi) : 0.0) +
            1e-300;
      const double s0 = lo - m, s1 = hi + m;
      double smax = 0.0;
      if (std::isfinite(s0)) smax = std::fabs(s0);
      if (std::isfinite(s1)) smax = std::max(smax, std::fabs(s1));
      const double err = 0x1p-52 * (bf.amax * smax + bf.bmax) + 1e-300;
      if (std::isfinite(s0) || std::isfinite(s1)) tau = std::max(tau, 4.0 * err / m);
      const double fin = std::isfinite(s0) ? s0 : std::isfinite(s1) ? s1 : 0.0;
      ends[2 * e] = lmsb::SweepEnd{std::isfinite(s0) ? s0 : 0.0, fin, std::isfinite(s0) ? 0 : 1, 0};
      ends[2 * e + 1] = lmsb::SweepEnd{std::isfinite(s1) ? s1 : 0.0, fin, std::isfinite(s1) ? 0 : 2, 0};
      rk[e] = k0;
      rk[nr + e] = k1;
    }
    if (with_outer) break;
    if (nr > 0 && 2.0 * bf.bmax * bf.amax * (1.0 + 0x1p-20) <= 1e30 * tau) break;
    }
    ends[2 * nr] = lmsb::SweepEnd{0.0, 0.0, 3, 0};
    const int64_t nn = h.n;
    const int64_t nbk = (nn + 31) / 32;
    RC_TRY(c->sw_k1.need(2 * nseg * nn));
    RC_TRY(c->sw_idx.need(2 * nseg * nn));
    RC_TRY(c->sw_pos.need(nr * nn));
    RC_TRY(c->sw_P.need(nr * nn));
    RC_TRY(c->sw_bmin.need(nr * nbk));
    RC_TRY(c->sw_suf.need(nr * nbk));
    RC_TRY(c->sw_rk.need(2 * nr));
    RC_TRY(c->sw_ends.need(nseg));
    CUDA_TRY(cudaMemcpyAsync(c->sw_ends.p, ends, sizeof(lmsb::SweepEnd) * nseg,
                             cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->sw_rk.p, rk, sizeof(int32_t) * 2 * nr, cudaMemcpyHostToDevice,
                             c->stream));
    lmsb::SweepSort ss{};
    for (int b = 0; b < 2; ++b) {
      ss.k1[b] = c->sw_k1.p + b * nseg * nn;
      ss.idx[b] = c->sw_idx.p + b * nseg * nn;
    }
    CUDA_TRY(ev_rec(c, c->ev_chunk[5]));
    st->launches += lmsb::launch_sweep_sort(bf.ab, (int)nn, c->sw_ends.p, nseg, ss, c->sms,
                                            c->stream);
    trace_mark(c, "sweep_sort");
    lmsb::launch_sweep_prepare((int)nn, nr, ss, c->sw_pos.p, c->sw_P.p, c->sw_bmin.p, c->sw_suf.p,
                               c->sms, c->stream);
    trace_mark(c, "sweep_prep");
    CUDA_TRY(cudaGetLastError());
    st->launches += 3;
    sa.bounds = c->bbounds.p;
    sa.K = K;
    sa.slot = w.slot;
    sa.nruns = nr;
    sa.run_k0 = c->sw_rk.p;
    sa.run_k1 = c->sw_rk.p + nr;
    sa.P = c->sw_P.p;
    sa.bmin = c->sw_bmin.p;
    sa.suf = c->sw_suf.p;
    sa.idx = ss.idx[ss.cur];
    sa.k1a = ss.k1[ss.cur] + (int64_t)(2 * nr) * nn;
    sa.idxa = ss.idx[ss.cur] + (int64_t)(2 * nr) * nn;
    sa.tau = tau;
    sa.count = w.ncollect;
    st->sweep_runs = nr;
    if (getenv("LMSB_SWEEP_DEBUG")) {
      RC_TRY(c->sw_dbg.need(nr + 1));
      CUDA_TRY(cudaMemsetAsync(c->sw_dbg.p, 0, sizeof(unsigned long long) * (nr + 1), c->stream));
      sa.dbg = c->sw_dbg.p;
      for (int e = 0; e < nr; ++e)
        fprintf(stderr, "sweep run %d: bands [%d, %d] s0 %.17g s1 %.17g kinds %d/%d\n", e, rk[e],
                rk[nr + e], ends[2 * e].s, ends[2 * e + 1].s, ends[2 * e].kind, ends[2 * e + 1].kind);
      fprintf(stderr, "sweep tau %.6g\n", tau);
    }
  }
  // sub-band groups of the admitted bands (boundaries at every sub_samples-th
  // sorted sample of the band, computed on the device): the collected keys
  // are group ids, counting-sorted after the collect and packed into chunks
  bool subgrp = false;
  int ngroups_sub = 0, nadm_sub = 0;
  int32_t* d_sbf = nullptr;
  int32_t* d_gband = nullptr;
  if (sweep && use_bkeys) {
    nadm_sub = nslot - 1;  // the last slot is the beyond-range pseudo band
    int32_t* sbf = u_sub;  // nadm + 2
    int32_t* gb = u_sub + (nadm_sub + 2);
    sbf[0] = 0;
    int G = 0;
    bool fits = true;
    for (int e = 0; e < nadm_sub && fits; ++e) {
      const int32_t k = list[e];
      // narrow inner band: one group (its stored keys serve every member);
      // wide (or outer) band: sub-bands at the samples
      bool narrow = false;
      if (k > 0 && k < K - 1) {
        const double uL = (double)std::nextafter(hbnd[k - 1], -INFINITY), uR = (double)hbnd[k];
        narrow = std::isfinite(uL) && std::isfinite(uR) && bf.dev * (uR - uL) <= c->bkeys_tau * H;
      }
      const int Se =
          narrow ? 1 : std::max(1, std::min(1024, (int)(scnt[k] / (unsigned)c->sub_samples)));
      if (G + Se + 1 > lmsb::kSubMaxGroups) fits = false;
      for (int t = 0; t < Se && fits; ++t) gb[G + t] = k;
      G += Se;
      sbf[e + 1] = G;
    }
    if (fits) {
      sbf[nadm_sub + 1] = G + 1;
      gb[G] = K;
      ngroups_sub = G + 1;
      RC_TRY(c->dg_i32.need((int64_t)(nadm_sub + 2) + ngroups_sub));
      RC_TRY(c->dg_sub.need(std::max(G - nadm_sub, 1)));
      d_sbf = c->dg_i32.p;
      d_gband = d_sbf + (nadm_sub + 2);
      CUDA_TRY(cudaMemcpyAsync(d_sbf, u_sub, sizeof(int32_t) * ((nadm_sub + 2) + ngroups_sub),
                               cudaMemcpyHostToDevice, c->stream));
      lmsb::launch_band_subbounds(w, c->blist.p, d_sbf, nadm_sub, c->dg_sub.p, c->stream);
      sa.sub_first = d_sbf;
      sa.sub = c->dg_sub.p;
      subgrp = true;
      st->launches += 1;
      trace_mark(c, "subbounds");
    }
  }
  for (int attempt = 0; attempt < 2; ++attempt) {
    RC_TRY(c->bck.need(cap));
    RC_TRY(c->bcv.need(cap));
    w.ckeys = c->bck.p;
    w.cvals = c->bcv.p;
    if (sweep) {
      sa.out_keys = w.ckeys;
      sa.out_vals = w.cvals;
      sa.cap = cap;
      // (raw entries: inversions, not members -- their own capacity)
      const int64_t raw_cap = std::max(cap, c->raw_floor);
      RC_TRY(c->sw_raw.need(raw_cap));
      RC_TRY(c->sw_rawcnt.need(1));
      sa.raw = c->sw_raw.p;
      sa.raw_cap = raw_cap;
      sa.raw_count = c->sw_rawcnt.p;
      sa.raw_overflow = subgrp ? sc + 8 : nullptr;  // (deferred count: flagged, not counted)
      CUDA_TRY(ev_rec(c, c->ev_chunk[10]));
      lmsb::launch_sweep_emit(bf, sa, c->sms, c->stream);
      trace_mark(c, "sweep_emit");
      CUDA_TRY(ev_rec(c, c->ev_chunk[11]));
      sweep_timed = true;
      st->launches += 2;
    } else {
      CUDA_TRY(ev_rec(c, c->ev_chunk[5]));
      lmsb::launch_band_collect(bf, w, runs, cap, c->sms, c->stream);
      st->launches += 1;
    }
    CUDA_TRY(ev_rec(c, c->ev_chunk[6]));
    CUDA_TRY(cudaGetLastError());
    if (sweep && sa.dbg) {
      std::vector<unsigned long long> d(sa.nruns);
      CUDA_TRY(cudaMemcpyAsync(d.data(), sa.dbg, sizeof(unsigned long long) * sa.nruns,
                               cudaMemcpyDeviceToHost, c->stream));
      CUDA_TRY(cudaStreamSynchronize(c->stream));
      for (int e = 0; e < sa.nruns; ++e) fprintf(stderr, "sweep run %d: %llu pairs\n", e, d[e]);
    }
    if (subgrp) {
      // the member count stays on the device (the grouping reads it there);
      // buffers are sized for `cap` and an overflow is caught by the final
      // readback (the fit is then solved again with the exact capacity)
      m = (unsigned long long)cap;
      break;
    }
    unsigned long long* p_m = reinterpret_cast<unsigned long long*>(c->pin);
    CUDA_TRY(cudaMemcpyAsync(p_m, sc + 1, sizeof(m), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    m = *p_m;
    trace_mark(c, "readback2");
    if ((int64_t)m <= cap) break;
    cap = (int64_t)m;  // estimate too small: collect again with the exact size
  }
  if (subgrp) {
    // counting sort by group, then the groups packed into filter chunks
    const int64_t cmin = std::max<int64_t>(1, std::min(c->wide_chunk, c->narrow_chunk));
    nchunk_max = 2 * (((int64_t)m + cmin - 1) / cmin) + ngroups_sub + nslot + 1;
    RC_TRY(c->bmem.need(std::max<int64_t>((int64_t)m, 1)));
    RC_TRY(c->dg_cursor.need(2 * (int64_t)ngroups_sub));
    RC_TRY(c->bstart.need(std::max<int64_t>(ngroups_sub, K + 1)));
    RC_TRY(c->bend.need(std::max<int64_t>(ngroups_sub, K + 1)));
    RC_TRY(c->bctab.need(2 * nchunk_max));
    RC_TRY(c->bcband.need(nchunk_max));
    w.start = c->bstart.p;
    w.end = c->bend.p;
    ba.start = c->bstart.p;
    ba.end = c->bend.p;
    CUDA_TRY(cudaMemsetAsync(c->dg_cursor.p, 0, sizeof(unsigned long long) * ngroups_sub,
                             c->stream));
    if (lmsb::launch_band_group_sub(w.ckeys, w.cvals, sc + 1, (int64_t)m, ngroups_sub,
                                    c->dg_cursor.p, c->dg_cursor.p + ngroups_sub, c->bstart.p,
                                    c->bend.p, c->bmem.p, c->stream) != 0)
      return set_error(LMS_ERR_CUDA, "sub-band grouping failed");
    trace_mark(c, "group");
    lmsb::launch_band_pack_chunks(d_sbf, nadm_sub + 1, c->bstart.p, c->bend.p, d_gband,
                                  c->wide_chunk, c->narrow_chunk, c->bctab.p, c->bcband.p, sc + 7,
                                  c->stream);
    trace_mark(c, "pack");
    CUDA_TRY(cudaGetLastError());
    st->launches += 4;
  } else {
  RC_TRY(c->bcka.need((int64_t)m));
  RC_TRY(c->bmem.need((int64_t)m));
  RC_TRY(c->btemp.need((int64_t)std::max(lmsb::band_sample_temp_bytes(S),
                                         lmsb::band_group_temp_bytes((int64_t)m))));
  w.ckeys_alt = c->bcka.p;
  w.members = c->bmem.p;
  w.temp = c->btemp.p;
  w.temp_bytes = (size_t)c->btemp.cap;
  if (lmsb::launch_band_group(w, (int64_t)m, !big, c->stream) != 0)
    return set_error(LMS_ERR_CUDA, "band grouping sort failed");
  trace_mark(c, "group");
  CUDA_TRY(cudaGetLastError());
  st->launches += 3;
  }
  }
  }
  CUDA_TRY(ev_rec(c, c->ev_chunk[3]));

  // ---- window counts of the collected vertices; fp32 counts at each
  // survivor's own slope; exact select of the most promising few (tightens H),
  // counts again against the tightened H, exact select of the rest
  const int64_t scap = std::max<int64_t>((int64_t)m, 1);
  RC_TRY(c->ranks.need(scap));
  RC_TRY(c->item_fit.need(scap));
  RC_TRY(c->recs.need(scap));
  RC_TRY(c->branks2.need(scap));
  RC_TRY(c->bfits2.need(scap));
  RC_TRY(c->blines32.need(h.n + 2));
  RC_TRY(c->bchunks.need((int64_t)std::max<size_t>(list.size(), (size_t)ngroups) + 1));
  ba.members = c->bmem.p;
  if (!direct) {
    ba.list = c->bident.p;       // groups are the slots 0 .. nslot - 1
    ba.group_band = c->blist.p;  // slot -> band
    ba.nlist = nslot;
  }
  if (nchunk_max > 0) {  // sub-band grouping: the packed chunk table
    ba.ctab = c->bctab.p;
    ba.cband = c->bcband.p;
    ba.nctab = sc + 7;
    RC_TRY(c->bticket.need(1));
    CUDA_TRY(cudaMemsetAsync(c->bticket.p, 0, sizeof(unsigned long long), c->stream));
    ba.ticket = c->bticket.p;
  }
  ba.chunk = c->band_chunk;
  ba.chunk_prefix = c->bchunks.p;
  ba.out_ranks = c->ranks.p;
  ba.out_fits = c->item_fit.p;
  ba.out_count = sc + 3;
  // [3] band survivors, [4] count survivors ([5] is the running best height;
  // [6] the prepass output, cleared by its launcher)
  CUDA_TRY(cudaMemsetAsync(sc + 3, 0, 2 * sizeof(unsigned long long), c->stream));
  CUDA_TRY(cudaMemsetAsync(sc + 6, 0, sizeof(unsigned long long), c->stream));
  if (m > 0) {
    // (small path: up to kMinChunks = 4 chunks per group beyond m / chunk)
    // (the chunk table: persistent CTAs, one per SM, taking chunk tickets)
    const int fgrid = nchunk_max > 0
                          ? (int)std::min<int64_t>(nchunk_max, c->sms)
                          : (int)(((int64_t)m + ba.chunk - 1) / ba.chunk + 5 * (int64_t)ba.nlist);
    if (big) {
      // sorted keys per slice of `big_slice` members at the slice's own
      // centre slope (padding D shrinks with the slice's slope range)
      const int64_t SB = std::max<int64_t>(ba.chunk, (c->big_slice / ba.chunk) * ba.chunk);
      // per group at most ceil(cnt / SB) or kMinSlices + 1 slices (group_slice)
      const int64_t nsl = (int64_t)m / SB + 9 * (int64_t)ba.nlist + 1;
      RC_TRY(c->bslice_keys.need(nsl * h.n));
      RC_TRY(c->bslice_store.need(nsl * h.n));
      RC_TRY(c->bslice_seg.need(2 * nsl));
      RC_TRY(c->bslice_prefix.need(ba.nlist + 1));
      RC_TRY(c->bslice_u.need(4 * nsl));
      RC_TRY(c->bslice_ptab.need(nsl * lmsb::kSliceTableRow));
      RC_TRY(c->btemp.need((int64_t)std::max<size_t>((size_t)c->btemp.cap,
                                                     lmsb::band_slice_sort_temp_bytes(nsl, h.n))));
      ba.slice = SB;
      if (c->big_narrow) {  // narrow bands: one slice (one key sort) per band
        RC_TRY(c->bnarrow.need(K + 1));
        uint8_t* u_nar = reinterpret_cast<uint8_t*>(u_sub);  // (sub-band staging unused here)
        for (int k = 0; k <= K; ++k) u_nar[k] = 0;
        for (int e = 0; e + 1 < nslot; ++e) {
          const int32_t k = list[e];
          if (k <= 0 || k >= K - 1) continue;
          const double uL = (double)std::nextafter(hbnd[k - 1], -INFINITY), uR = (double)hbnd[k];
          u_nar[k] = std::isfinite(uL) && std::isfinite(uR) && bf.dev * (uR - uL) <= c->bkeys_tau * H;
        }
        CUDA_TRY(cudaMemcpyAsync(c->bnarrow.p, u_nar, K + 1, cudaMemcpyHostToDevice, c->stream));
        ba.narrow = c->bnarrow.p;
      }
      ba.slice_prefix = c->bslice_prefix.p;
      ba.slice_u = c->bslice_u.p;
      ba.slice_wq = c->bslice_u.p + nsl;
      ba.slice_kmin = c->bslice_u.p + 2 * nsl;
      ba.slice_res = c->bslice_u.p + 3 * nsl;
      ba.slice_ptab = c->bslice_ptab.p;
      if (lmsb::launch_band_slices(bf, ba, nsl, c->bslice_keys.p, c->bslice_store.p,
                                   c->bslice_seg.p, c->bslice_seg.p + nsl, c->btemp.p,
                                   (size_t)c->btemp.cap, c->stream) != 0)
        return set_error(LMS_ERR_CUDA, "large-n slice sort failed");
      trace_mark(c, "slices");
      st->launches += 4;
      CUDA_TRY(ev_rec(c, c->ev_chunk[8]));
      lmsb::launch_band_filter_big(bf, ba, c->bslice_store.p, fgrid, c->stream);
      trace_mark(c, "filter_big");
      CUDA_TRY(ev_rec(c, c->ev_chunk[9]));
    } else {
      CUDA_TRY(ev_rec(c, c->ev_chunk[8]));
      lmsb::launch_band(bf, ba, 1, fgrid, c->stream);
      trace_mark(c, "filter");
      CUDA_TRY(ev_rec(c, c->ev_chunk[9]));
    }
    filter_timed = true;
    lmsb::BandCount bc{};
    bc.lines = c->blines32.p;
    bc.best = c->best.p;
    bc.in_ranks = c->ranks.p;
    bc.in_count = sc + 3;
    bc.out_ranks = c->branks2.p;
    bc.out_fits = c->bfits2.p;
    bc.fit = 0;
    bc.out_count = sc + 4;
    bc.make_lines = true;
    const bool counted = c->band_count != 0;
    if (counted) {
      lmsb::launch_band_count(bf, bc, c->sms, c->stream);
      trace_mark(c, "count");
      CUDA_TRY(cudaGetLastError());
      st->launches += 4;
    }
    // the window-edge seeds put H at (or within a few ulps of) the optimum, so
    // the exact stage's pass 0 prunes every survivor that cannot tie it
    // exact pass-0 screen, lane per vertex with shared-memory lines; only the
    // vertices the exact select would not prune go on to it
    lmsb::BandCount bp = bc;
    // (without the fp32 counts the screen reads the band survivors and
    // writes into the count stage's buffers)
    bp.in_ranks = counted ? c->branks2.p : c->ranks.p;
    bp.in_count = counted ? sc + 4 : sc + 3;
    bp.out_ranks = counted ? c->ranks.p : c->branks2.p;
    bp.out_fits = counted ? c->item_fit.p : c->bfits2.p;
    bp.out_count = sc + 6;
    if (c->prepass_split) {
      if (c->pcnt.cap < 2 * scap) {
        RC_TRY(c->pcnt.need(2 * scap));
        CUDA_TRY(cudaMemsetAsync(c->pcnt.p, 0, (size_t)c->pcnt.cap * sizeof(unsigned), c->stream));
      }
      lmsb::launch_band_prepass_split(bf, bp, c->pcnt.p, c->sms, c->stream);
      st->launches += 2;
    } else {
      lmsb::launch_band_exact_prepass(bf, bp, c->sms, c->stream);
      st->launches += 1;
    }
    trace_mark(c, "prepass");
    RC_TRY(exact_list(sc + 6, scap, bp.out_ranks, bp.out_fits));
    trace_mark(c, "exact");
  }
  CUDA_TRY(ev_rec(c, c->ev_chunk[4]));
  if (capturing) {
    // the whole search captured: instantiate and run it (replayed by the
    // next identical fit)
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(c->stream, &graph);
    c->capturing = false;
    cudaGraphExec_t ex = nullptr;
    bool ok = ce == cudaSuccess && graph &&
              cudaGraphInstantiate(&ex, graph, 0) == cudaSuccess &&
              g_buf_epoch.load() == epoch0;
    if (graph) cudaGraphDestroy(graph);
    if (!ok) {
      // nothing of the captured search ran: solve again with direct launches
      // (and without the caches the capture marked as filled)
      if (ex) cudaGraphExecDestroy(ex);
      cudaGetLastError();
      c->use_graph = 0;
      c->ab_gen = ~0ull;
      c->wqa_gen = ~0ull;
      return band_solve(c, h, st);
    }
    if (c->gexec) cudaGraphExecDestroy(c->gexec);
    c->gexec = ex;
    std::memcpy(c->gkey, gk, sizeof(gk));
    c->g_launches = st->launches - launches0;
    CUDA_TRY(cudaGraphLaunch(c->gexec, c->stream));
  }
  return band_finish(c, h, st, BandTail{m, direct, dplan, filter_timed, bound_timed, sweep_timed});
}

// Exact LMS search over a batch of fits; out[f] receives fit f's record.
int ctx_solve_fits(lms_ctx* c, const std::vector<HostFit>& hf, lms_candidate* out) {
  const int64_t F = (int64_t)hf.size();
  std::memset(out, 0, sizeof(lms_candidate) * F);
  if (F == 0) return LMS_OK;
  CUDA_TRY(cudaSetDevice(c->device));
  lms_stats st{};

  // ---- host plan: fit descriptors, seeds, task counts (closed form)
  int64_t maxn = 0;
  for (const auto& f : hf) maxn = std::max(maxn, f.n);
  const int V = maxn >= 4096 ? 4 : 2;
  const int64_t tv = lmsb::filter_task_vertices(V);
  std::vector<lmsb::FitDesc> fd(F);
  std::vector<int64_t> prefA(F + 1), prefB(F + 1), seed_pref(F + 1), seg(F + 1);
  int64_t rowsA = 0, rows = 0, tasks = 0, tasksA = 0, seeds = 0;
  bool disjoint = true;
  bool banded = false;
  std::vector<int32_t> small_list;
  int64_t small_maxn = 0;
  for (int64_t f = 0; f < F; ++f) {
    const HostFit& h = hf[f];
    const int64_t span = h.r1 - h.r0;
    // a shard of a sharded search decides on the whole pair space, as its plan did
    const int64_t bspan = c->shard ? c->shard->P1 - c->shard->P0 : span;
    bool exhaustive = bspan <= kExhaustive;
    // small fits of a batch: the fused per-fit band kernel (lms_band_small.cu),
    // which derives its own magnitudes on the device
    const bool small = c->small_mode != 0 && (F > 1 || c->small_mode == 2) &&
                       h.n <= lmsb::kSmallMaxN && span >= lmsb::kSmallMinPairs &&
                       h.r0 == 0 && h.r1 == h.n * (h.n - 1) / 2;
    if (small) {
      small_list.push_back((int32_t)f);
      small_maxn = std::max(small_maxn, h.n);
    }
    double am = 0.0, bm = 0.0;
    if (!small) {
      double alo_, ahi_;
      line_stats(c, h.off, h.n, &alo_, &ahi_, &am, &bm);
    }
    if (F == 1 && !exhaustive && !small && h.n <= lmsb::kBandMaxBigN && am < 1e30 && bm < 1e30 &&
        (c->band_mode == 2 || (c->band_mode == 1 && bspan >= kBandMinSpan)))
      banded = true;  // slope-band stage instead of seeds + count filter
    exhaustive = !banded && span <= kExhaustive;
    int64_t s = exhaustive ? span : std::min(kSeedsMax, std::max(kSeedsMin, span / kSeedDivisor));
    s = (banded || small) ? 0 : std::min(s, span);
    lmsb::FitDesc& d = fd[f];
    d.off = h.off;
    d.n = h.n;
    d.q = h.q;
    d.rank_lo = h.r0;
    d.rank_hi = h.r1;
    d.row0 = 0;
    d.nrows = 0;
    if (!exhaustive && !banded && !small) {
      tasks += lmsb::fit_tasks(h.n, h.r0, h.r1, tv, &d.row0, &d.nrows);
      for (int64_t k = 0; k < d.nrows; k += lmsb::kPhaseStride)
        tasksA += lmsb::row_tasks(h.n, h.r0, h.r1, d.row0 + k, tv);
    }
    prefA[f] = rowsA;
    rowsA += (d.nrows + lmsb::kPhaseStride - 1) / lmsb::kPhaseStride;
    rows += d.nrows;
    d.amax = am;
    d.bmax = bm;
    seed_pref[f] = seeds;
    seeds += s;
    seg[f] = h.off;
    if (f > 0 && h.off < hf[f - 1].off + hf[f - 1].n) disjoint = false;
    st.pairs += span;
    st.n = std::max(st.n, h.n);
  }
  prefA[F] = rowsA;
  {
    int64_t rb = rowsA;
    for (int64_t f = 0; f < F; ++f) {
      prefB[f] = rb;
      rb += fd[f].nrows - (prefA[f + 1] - prefA[f]);
    }
    prefB[F] = rb;
  }
  if (c->shard && c->shard->mode == 1 && !banded) return LMS_OK;  // plan: no bands
  seed_pref[F] = seeds;
  seg[F] = hf[F - 1].off + hf[F - 1].n;
  st.seed_vertices = seeds;

  RC_TRY(c->fits.need(F));
  RC_TRY(c->prefA.need(F + 1));
  RC_TRY(c->prefB.need(F + 1));
  RC_TRY(c->seed_prefix.need(F + 1));
  RC_TRY(c->seg.need(F + 1));
  RC_TRY(c->keys.need(F));
  RC_TRY(c->best.need(F));
  RC_TRY(ensure_host_best(c, F));
  const int64_t cap = tasks > 0 ? std::min(kChunkVertices, tasks * tv) : 0;
  const int64_t cap_items = std::max<int64_t>(seeds, cap);
  RC_TRY(c->ranks.need(cap_items));
  RC_TRY(c->item_fit.need(cap_items));
  RC_TRY(c->recs.need(cap_items));

  CUDA_TRY(cudaEventRecord(c->ev_begin, c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->fits.p, fd.data(), sizeof(lmsb::FitDesc) * F,
                           cudaMemcpyHostToDevice, c->stream));
  if (tasks > 0) {  // the count filter's task plan
    CUDA_TRY(cudaMemcpyAsync(c->prefA.p, prefA.data(), sizeof(int64_t) * (F + 1),
                             cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->prefB.p, prefB.data(), sizeof(int64_t) * (F + 1),
                             cudaMemcpyHostToDevice, c->stream));
  }
  if (seeds > 0)
    CUDA_TRY(cudaMemcpyAsync(c->seed_prefix.p, seed_pref.data(), sizeof(int64_t) * (F + 1),
                             cudaMemcpyHostToDevice, c->stream));
  lmsb::launch_reset_best(c->keys.p, c->best.p, F, c->stream);
  st.launches += 1;

  // ---- 1. seeds (every vertex of the exhaustive fits)
  if (seeds > 0) {
    lmsb::launch_gen_seeds(c->fits.p, c->seed_prefix.p, F, c->ranks.p, c->item_fit.p, c->stream);
    lmsb::ExactArgs ea{};
    ea.a = c->a;
    ea.b = c->b;
    ea.fits = c->fits.p;
    ea.mode = lmsb::kSrcList;
    ea.count = seeds;
    ea.capacity = seeds;
    ea.ranks = c->ranks.p;
    ea.fit_of = c->item_fit.p;
    ea.out = c->recs.p;
    lmsb::launch_exact(ea, persistent_grid(c, seeds), c->stream, maxn);
    lmsb::launch_reduce(c->recs.p, nullptr, seeds, seeds, c->fits.p, c->keys.p, c->best.p,
                        reduce_grid(c, seeds), c->stream);
    CUDA_TRY(cudaGetLastError());
    st.launches += 4;
  }

  // ---- band path: one large fit with lines in shared-memory range
  if (banded) {
    RC_TRY(band_solve(c, hf[0], &st));
    if (c->shard && c->shard->mode == 1) {
      c->stats = st;
      return LMS_OK;  // plan: the slice's bounds are with the caller
    }
  }

  // ---- fused band search of the batch's small fits, one CTA each
  if (!small_list.empty()) {
    RC_TRY(c->small_list.need((int64_t)small_list.size()));
    CUDA_TRY(cudaMemcpyAsync(c->small_list.p, small_list.data(),
                             sizeof(int32_t) * small_list.size(), cudaMemcpyHostToDevice,
                             c->stream));
    lmsb::SmallArgs sa{};
    sa.a = c->a;
    sa.b = c->b;
    sa.fits = c->fits.p;
    sa.list = c->small_list.p;
    sa.out = c->best.p;
    RC_TRY(c->small_cnt.need(12));
    CUDA_TRY(cudaMemsetAsync(c->small_cnt.p, 0, 12 * sizeof(unsigned long long), c->stream));
    sa.counters = c->small_cnt.p;
    sa.timing = getenv("LMSB_SMALL_DEBUG") != nullptr;
    lmsb::launch_small_fits(sa, (int64_t)small_list.size(), small_maxn, c->sms, c->stream);
    CUDA_TRY(cudaGetLastError());
    st.launches += 1;
    st.small_fits = (int64_t)small_list.size();
  }

  // ---- 2.-5. filter the non-exhaustive fits: phase A (every kPhaseStride-th
  // row), re-order, phase B (the rest)
  int64_t nchunks = 0;
  if (tasks > 0 && !banded) {
    RC_TRY(c->counts.need(rows + 1));
    RC_TRY(c->row_task_prefix.need(rows + 1));
    RC_TRY(c->row_fit.need(rows));
    RC_TRY(c->row_i.need(rows));
    RC_TRY(c->task_row.need(tasks));
    RC_TRY(c->plan_tmp.need((int64_t)lmsb::plan_temp_bytes(rows)));
    lmsb::PlanArgs pa{};
    pa.fits = c->fits.p;
    pa.prefA = c->prefA.p;
    pa.prefB = c->prefB.p;
    pa.nfits = F;
    pa.rowsA = rowsA;
    pa.nrows = rows;
    pa.task_vertices = tv;
    pa.counts = c->counts.p;
    pa.row_fit = c->row_fit.p;
    pa.row_i = c->row_i.p;
    pa.row_task_prefix = c->row_task_prefix.p;
    pa.task_row = c->task_row.p;
    pa.temp = c->plan_tmp.p;
    pa.temp_bytes = (size_t)c->plan_tmp.cap;
    if (lmsb::launch_plan(pa, c->stream) != 0) return set_error(LMS_ERR_CUDA, "plan scan failed");
    CUDA_TRY(cudaGetLastError());
    st.launches += 3;

    const int64_t chunk_tasks = kChunkVertices / tv;
    std::vector<std::pair<int64_t, int64_t>> chunks;
    for (int64_t t0 = 0; t0 < tasksA; t0 += chunk_tasks)
      chunks.push_back({t0, std::min(tasksA, t0 + chunk_tasks)});
    const int64_t first_b = (int64_t)chunks.size();
    for (int64_t t0 = tasksA; t0 < tasks; t0 += chunk_tasks)
      chunks.push_back({t0, std::min(tasks, t0 + chunk_tasks)});
    nchunks = (int64_t)chunks.size();
    RC_TRY(c->counters.need(2 + nchunks));
    CUDA_TRY(cudaMemsetAsync(c->counters.p, 0, sizeof(unsigned long long) * (2 + nchunks),
                             c->stream));
    while ((int64_t)c->ev_chunk.size() < 2 * nchunks) {
      cudaEvent_t e;
      CUDA_TRY(cudaEventCreate(&e));
      c->ev_chunk.push_back(e);
    }
    const double* la = c->a;
    const double* lb = c->b;
    for (int64_t ch = 0; ch < nchunks; ++ch) {
      if ((ch == 0 || ch == first_b) && c->line_order && disjoint)
        RC_TRY(order_lines(c, seg, F, &la, &lb, &st));  // from the current best lines
      lmsb::FilterArgs fa{};
      fa.a = c->a;
      fa.b = c->b;
      fa.la = la;
      fa.lb = lb;
      fa.fits = c->fits.p;
      fa.task_row = c->task_row.p;
      fa.row_task_prefix = c->row_task_prefix.p;
      fa.row_fit = c->row_fit.p;
      fa.row_i = c->row_i.p;
      fa.task_begin = chunks[ch].first;
      fa.task_end = chunks[ch].second;
      fa.best = c->best.p;
      fa.out_ranks = c->ranks.p;
      fa.out_fits = c->item_fit.p;
      fa.out_count = c->counters.p + 2 + ch;
      fa.line_evals = c->counters.p + 1;
      fa.early_exit = 1;
      CUDA_TRY(cudaEventRecord(c->ev_chunk[2 * ch], c->stream));
      lmsb::launch_filter(fa, V, c->stream);
      CUDA_TRY(cudaEventRecord(c->ev_chunk[2 * ch + 1], c->stream));
      lmsb::ExactArgs xa{};
      xa.a = c->a;
      xa.b = c->b;
      xa.fits = c->fits.p;
      xa.mode = lmsb::kSrcList;
      xa.d_count = c->counters.p + 2 + ch;
      xa.capacity = cap;
      xa.ranks = c->ranks.p;
      xa.fit_of = c->item_fit.p;
      xa.bound = c->best.p;
      xa.out = c->recs.p;
      lmsb::launch_exact(xa, persistent_grid(c, -1), c->stream, maxn);
      lmsb::launch_reduce(c->recs.p, c->counters.p + 2 + ch, 0, cap, c->fits.p, c->keys.p,
                          c->best.p, (int)c->sms * 4, c->stream);
      CUDA_TRY(cudaGetLastError());
      st.launches += 4;
      st.filtered_vertices += (fa.task_end - fa.task_begin) * tv;
    }
  }
  CUDA_TRY(cudaMemcpyAsync(c->h_best, c->best.p, sizeof(lms_candidate) * F,
                           cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaEventRecord(c->ev_end, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  std::memcpy(out, c->h_best, sizeof(lms_candidate) * F);
  if (!banded) st.chunks = nchunks;
  if (!small_list.empty()) {
    unsigned long long sc4[12];
    CUDA_TRY(cudaMemcpy(sc4, c->small_cnt.p, sizeof(sc4), cudaMemcpyDeviceToHost));
    if (getenv("LMSB_SMALL_DEBUG")) {
      const double F = (double)small_list.size();
      fprintf(stderr,
              "small: bounds %.3g seeds %.3g sweeps %.3g cycles/fit; warp-cycles/fit: exact %.3g "
              "counts %.3g searches %.3g\n",
              sc4[5] / F, sc4[6] / F, sc4[7] / F, sc4[8] / F, sc4[9] / F, sc4[10] / F);
    }
    st.bands_searched = (int64_t)sc4[0];
    st.band_survivors = (int64_t)sc4[1];
    st.survivors = (int64_t)sc4[2];
    st.chunks = (int64_t)sc4[3];
  }
  if (nchunks > 0) {
    std::vector<unsigned long long> cnt(2 + nchunks);
    CUDA_TRY(cudaMemcpy(cnt.data(), c->counters.p, sizeof(unsigned long long) * (2 + nchunks),
                        cudaMemcpyDeviceToHost));
    st.line_evals = (int64_t)cnt[1];
    for (int64_t ch = 0; ch < nchunks; ++ch) {
      st.survivors += (int64_t)cnt[2 + ch];
      float ms = 0.f;
      CUDA_TRY(cudaEventElapsedTime(&ms, c->ev_chunk[2 * ch], c->ev_chunk[2 * ch + 1]));
      st.ms_filter += ms;
    }
  }
  st.filtered_vertices = std::min(st.filtered_vertices, st.pairs);
  CUDA_TRY(cudaEventElapsedTime(&st.ms_total, c->ev_begin, c->ev_end));
  st.ms_exact = st.ms_total - st.ms_filter - st.ms_partition - st.ms_bound - st.ms_band_filter;
  c->stats = st;
  return LMS_OK;
}

int check_fit(lms_ctx* c, int64_t off, int64_t n, int64_t q) {
  if (n < 2) return set_error(LMS_ERR_INVALID, "a fit needs at least 2 lines, got %lld", (long long)n);
  if (q < 1) return set_error(LMS_ERR_INVALID, "coverage must be positive, got %lld", (long long)q);
  if (off < 0 || off + n > c->nlines)
    return set_error(LMS_ERR_INVALID, "fit lines [%lld, %lld) outside the %lld bound lines",
                     (long long)off, (long long)(off + n), (long long)c->nlines);
  return LMS_OK;
}

int ctx_solve(lms_ctx* c, int64_t q, int64_t R0, int64_t R1, lms_candidate* out) {
  std::memset(out, 0, sizeof(*out));
  if (!c->a) return set_error(LMS_ERR_INVALID, "no lines bound to the context");
  const int64_t n = c->nlines;
  RC_TRY(check_fit(c, 0, n, q));
  const int64_t total = n * (n - 1) / 2;
  if (R0 < 0 || R1 > total || R0 > R1)
    return set_error(LMS_ERR_INVALID, "rank range [%lld, %lld) outside [0, %lld)", (long long)R0,
                     (long long)R1, (long long)total);
  std::vector<HostFit> hf{{0, n, q, R0, R1}};
  return ctx_solve_fits(c, hf, out);
}

// The materialised two-kernel flow (_scan_materialized, backend.py:221-231;
// the paper's K1 -> K2): chunks of 2^22 pair ranks are materialised as
// explicit (i, j, u) triples (K1) and every triple is evaluated exactly (K2,
// exact stage in explicit mode with the running best as its bound), then
// reduced.  No band or count filter: every vertex is counted exactly, so it
// doubles as an independent cross-check of the pruned search.
int ctx_solve_materialized(lms_ctx* c, int64_t q, int64_t R0, int64_t R1, lms_candidate* out) {
  std::memset(out, 0, sizeof(*out));
  if (!c->a) return set_error(LMS_ERR_INVALID, "no lines bound to the context");
  const int64_t n = c->nlines;
  RC_TRY(check_fit(c, 0, n, q));
  const int64_t total = n * (n - 1) / 2;
  if (R0 < 0 || R1 > total || R0 > R1)
    return set_error(LMS_ERR_INVALID, "rank range [%lld, %lld) outside [0, %lld)", (long long)R0,
                     (long long)R1, (long long)total);
  CUDA_TRY(cudaSetDevice(c->device));
  constexpr int64_t kMatChunk = 1 << 22;
  const int64_t cap = std::min<int64_t>(kMatChunk, std::max<int64_t>(R1 - R0, 1));
  RC_TRY(c->ii.need(cap));
  RC_TRY(c->jj.need(cap));
  RC_TRY(c->uu.need(cap));
  RC_TRY(c->recs.need(cap));
  RC_TRY(c->fits.need(1));
  RC_TRY(c->keys.need(1));
  RC_TRY(c->best.need(1));
  RC_TRY(c->counters.need(1));
  lmsb::FitDesc fd{};
  fd.n = n;
  fd.q = q;
  fd.rank_lo = R0;
  fd.rank_hi = R1;
  lms_stats st{};
  st.n = n;
  st.pairs = R1 - R0;
  CUDA_TRY(cudaEventRecord(c->ev_begin, c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->fits.p, &fd, sizeof(fd), cudaMemcpyHostToDevice, c->stream));
  lmsb::launch_reset_best(c->keys.p, c->best.p, 1, c->stream);
  for (int64_t r = R0; r < R1; r += cap) {
    const int64_t cnt = std::min<int64_t>(cap, R1 - r);
    CUDA_TRY(cudaMemsetAsync(c->counters.p, 0, sizeof(unsigned long long), c->stream));
    lmsb::launch_materialize(c->a, c->b, n, r, cnt, c->ii.p, c->jj.p, c->uu.p, c->counters.p,
                             c->sms, c->stream);
    lmsb::ExactArgs ea{};
    ea.a = c->a;
    ea.b = c->b;
    ea.fits = c->fits.p;
    ea.mode = lmsb::kSrcExplicit;
    ea.d_count = c->counters.p;
    ea.capacity = cap;
    ea.ii = c->ii.p;
    ea.jj = c->jj.p;
    ea.uu = c->uu.p;
    ea.bound = c->best.p;
    ea.out = c->recs.p;
    lmsb::launch_exact(ea, persistent_grid(c, -1), c->stream, n);
    lmsb::launch_reduce(c->recs.p, c->counters.p, 0, cap, c->fits.p, c->keys.p, c->best.p,
                        (int)c->sms * 4, c->stream);
    CUDA_TRY(cudaGetLastError());
    st.launches += 5;
    st.chunks += 1;
  }
  CUDA_TRY(cudaMemcpyAsync(out, c->best.p, sizeof(lms_candidate), cudaMemcpyDeviceToHost,
                           c->stream));
  CUDA_TRY(cudaEventRecord(c->ev_end, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  CUDA_TRY(cudaEventElapsedTime(&st.ms_total, c->ev_begin, c->ev_end));
  st.ms_exact = st.ms_total;
  st.filtered_vertices = 0;
  c->stats = st;
  return LMS_OK;
}

int ctx_solve_batch(lms_ctx* c, const int64_t* offsets, const int64_t* q, int64_t nfits,
                    lms_candidate* out) {
  if (nfits < 0 || (nfits > 0 && (!offsets || !q))) return set_error(LMS_ERR_INVALID, "bad batch");
  if (nfits > 0 && !c->a) return set_error(LMS_ERR_INVALID, "no lines bound to the context");
  std::vector<HostFit> hf(nfits);
  for (int64_t f = 0; f < nfits; ++f) {
    const int64_t off = offsets[f], n = offsets[f + 1] - offsets[f];
    if (f > 0 && off < offsets[f - 1])
      return set_error(LMS_ERR_INVALID, "batch offsets must be non-decreasing");
    RC_TRY(check_fit(c, off, n, q[f]));
    hf[f] = {off, n, q[f], 0, n * (n - 1) / 2};
  }
  return ctx_solve_fits(c, hf, out);
}

int ctx_eval_explicit(lms_ctx* c, int64_t q, const int64_t* i, const int64_t* j, const double* u,
                      const double* v, int64_t m, lms_candidate* out, bool reduce) {
  if (m < 0) return set_error(LMS_ERR_INVALID, "negative vertex count");
  const int64_t n = c->nlines;
  RC_TRY(check_fit(c, 0, n, q));
  for (int64_t s = 0; s < m; ++s) {
    // with explicit anchor ordinates (v) an index of -1 snaps no line
    const int64_t lo = (v && !reduce) ? -1 : 0;
    if (i[s] < lo || i[s] >= n || j[s] < lo || j[s] >= n)
      return set_error(LMS_ERR_INVALID, "vertex %lld has a line index out of range", (long long)s);
    if (reduce && i[s] >= j[s])
      return set_error(LMS_ERR_INVALID, "vertex %lld must have i < j", (long long)s);
  }
  if (m == 0) {
    if (reduce) std::memset(out, 0, sizeof(*out));
    return LMS_OK;
  }
  CUDA_TRY(cudaSetDevice(c->device));
  RC_TRY(c->ii.need(m));
  RC_TRY(c->jj.need(m));
  RC_TRY(c->uu.need(m));
  RC_TRY(c->vv.need(m));
  RC_TRY(c->recs.need(m));
  RC_TRY(c->fits.need(1));
  RC_TRY(c->keys.need(1));
  RC_TRY(c->best.need(1));
  lmsb::FitDesc fd{};
  fd.off = 0;
  fd.n = n;
  fd.q = q;
  CUDA_TRY(cudaMemcpyAsync(c->fits.p, &fd, sizeof(fd), cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->ii.p, i, sizeof(int64_t) * m, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->jj.p, j, sizeof(int64_t) * m, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->uu.p, u, sizeof(double) * m, cudaMemcpyHostToDevice, c->stream));
  if (v)
    CUDA_TRY(cudaMemcpyAsync(c->vv.p, v, sizeof(double) * m, cudaMemcpyHostToDevice, c->stream));
  lmsb::ExactArgs ea{};
  ea.a = c->a;
  ea.b = c->b;
  ea.fits = c->fits.p;
  ea.mode = lmsb::kSrcExplicit;
  ea.count = m;
  ea.capacity = m;
  ea.ii = c->ii.p;
  ea.jj = c->jj.p;
  ea.uu = c->uu.p;
  ea.vv = v ? c->vv.p : nullptr;
  ea.out = c->recs.p;
  lmsb::launch_exact(ea, persistent_grid(c, m), c->stream, n);
  if (reduce) {
    lmsb::launch_reset_best(c->keys.p, c->best.p, 1, c->stream);
    lmsb::launch_reduce(c->recs.p, nullptr, m, m, c->fits.p, c->keys.p, c->best.p,
                        reduce_grid(c, m), c->stream);
    CUDA_TRY(cudaMemcpyAsync(out, c->best.p, sizeof(lms_candidate), cudaMemcpyDeviceToHost,
                             c->stream));
  } else {
    CUDA_TRY(cudaMemcpyAsync(out, c->recs.p, sizeof(lms_candidate) * m, cudaMemcpyDeviceToHost,
                             c->stream));
  }
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (!reduce)
    for (int64_t s = 0; s < m; ++s) out[s].reserved = 0;
  return LMS_OK;
}


// ---------------------------------------------------------------- primal brute force

int ctx_primal(lms_ctx* c, int64_t q, lms_candidate* out) {
  std::memset(out, 0, sizeof(*out));
  const int64_t n = c->nlines;
  RC_TRY(check_fit(c, 0, n, q));
  if (n > lmsb::kPrimalMaxN)
    return set_error(LMS_ERR_INVALID, "the primal brute force is limited to n <= %lld, got %lld",
                     (long long)lmsb::kPrimalMaxN, (long long)n);
  CUDA_TRY(cudaSetDevice(c->device));
  const int64_t P = n * (n - 1) / 2;
  RC_TRY(c->recs.need(P));
  RC_TRY(c->fits.need(1));
  RC_TRY(c->keys.need(1));
  RC_TRY(c->best.need(1));
  lmsb::FitDesc fd{};
  fd.n = n;
  fd.q = q;
  CUDA_TRY(cudaMemcpyAsync(c->fits.p, &fd, sizeof(fd), cudaMemcpyHostToDevice, c->stream));
  if (lmsb::launch_primal(c->a, c->b, n, q, c->recs.p, persistent_grid(c, P), c->stream) != 0)
    return set_error(LMS_ERR_CUDA, "primal kernel shared memory configuration failed");
  lmsb::launch_reset_best(c->keys.p, c->best.p, 1, c->stream);
  lmsb::launch_reduce(c->recs.p, nullptr, P, P, c->fits.p, c->keys.p, c->best.p, reduce_grid(c, P),
                      c->stream);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(out, c->best.p, sizeof(lms_candidate), cudaMemcpyDeviceToHost,
                           c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return LMS_OK;
}


// ---------------------------------------------------------------- Hough

int check_hough(int64_t n_theta, double rho_max, double drho, int64_t n_rho) {
  if (n_theta < 1 || n_rho < 1 || !(drho > 0.0) || !(rho_max > 0.0))
    return set_error(LMS_ERR_INVALID, "Hough bin widths and rho range must be positive");
  if (n_theta * n_rho > (int64_t)1 << 31)
    return set_error(LMS_ERR_INVALID, "Hough accumulator too large");
  return LMS_OK;
}

int ctx_vote(lms_ctx* c, const double* cos_t, const double* sin_t, int64_t n_theta,
             double rho_max, double drho, int64_t n_rho, int64_t* acc_out) {
  const int64_t nb = n_theta * n_rho;
  RC_TRY(c->acc.need(nb));
  RC_TRY(c->tcos.need(n_theta));
  RC_TRY(c->tsin.need(n_theta));
  CUDA_TRY(cudaMemcpyAsync(c->tcos.p, cos_t, sizeof(double) * n_theta, cudaMemcpyHostToDevice,
                           c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->tsin.p, sin_t, sizeof(double) * n_theta, cudaMemcpyHostToDevice,
                           c->stream));
  CUDA_TRY(cudaMemsetAsync(c->acc.p, 0, sizeof(unsigned long long) * nb, c->stream));
  if (c->hough_npts > 0)
    lmsb::hough_vote(c->hough_mode == 1 ? c->pix.p : nullptr, c->hough_mode == 2 ? c->pxs.p : nullptr,
                     c->hough_mode == 2 ? c->pys.p : nullptr, c->hough_npts, c->hough_width,
                     c->tcos.p, c->tsin.p, (int)n_theta, rho_max, drho, n_rho, c->acc.p, c->sms,
                     c->stream);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(acc_out, c->acc.p, sizeof(int64_t) * nb, cudaMemcpyDeviceToHost,
                           c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return LMS_OK;
}

int ctx_vote_image(lms_ctx* c, const uint8_t* img, int64_t height, int64_t width, int threshold,
                   const double* cos_t, const double* sin_t, int64_t n_theta, double rho_max,
                   double drho, int64_t n_rho, int64_t* acc_out, int64_t* npoints) {
  if (!img || height < 0 || width < 0) return set_error(LMS_ERR_INVALID, "bad image");
  RC_TRY(check_hough(n_theta, rho_max, drho, n_rho));
  CUDA_TRY(cudaSetDevice(c->device));
  const int64_t npix = height * width;
  RC_TRY(c->img.need(std::max<int64_t>(npix, 1)));
  RC_TRY(c->pix.need(std::max<int64_t>(npix, 1)));
  RC_TRY(c->pcount.need(1));
  RC_TRY(c->ext_tmp.need((int64_t)lmsb::extract_temp_bytes(std::max<int64_t>(npix, 1))));
  int64_t npts = 0;
  if (npix > 0) {
    RC_TRY(upload_staged(c, c->img.p, img, (size_t)npix));
    size_t tb = (size_t)c->ext_tmp.cap;
    if (lmsb::hough_extract(c->img.p, npix, threshold, c->pix.p, c->pcount.p, c->ext_tmp.p, &tb,
                            c->stream) != 0)
      return set_error(LMS_ERR_CUDA, "pixel compaction failed");
    CUDA_TRY(cudaMemcpyAsync(&npts, c->pcount.p, sizeof(int64_t), cudaMemcpyDeviceToHost,
                             c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
  }
  c->hough_mode = 1;
  c->hough_npts = npts;
  c->hough_width = std::max<int64_t>(width, 1);
  c->hough_maxid = npix;  // pixel indices < width * height
  *npoints = npts;
  return ctx_vote(c, cos_t, sin_t, n_theta, rho_max, drho, n_rho, acc_out);
}

int ctx_vote_points(lms_ctx* c, const double* x, const double* y, int64_t npts,
                    const double* cos_t, const double* sin_t, int64_t n_theta, double rho_max,
                    double drho, int64_t n_rho, int64_t* acc_out) {
  if (npts < 0 || (npts > 0 && (!x || !y))) return set_error(LMS_ERR_INVALID, "bad points");
  RC_TRY(check_hough(n_theta, rho_max, drho, n_rho));
  CUDA_TRY(cudaSetDevice(c->device));
  RC_TRY(c->pxs.need(std::max<int64_t>(npts, 1)));
  RC_TRY(c->pys.need(std::max<int64_t>(npts, 1)));
  if (npts > 0) {
    CUDA_TRY(cudaMemcpyAsync(c->pxs.p, x, sizeof(double) * npts, cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->pys.p, y, sizeof(double) * npts, cudaMemcpyHostToDevice, c->stream));
  }
  c->hough_mode = 2;
  c->hough_npts = npts;
  c->hough_width = 1;
  c->hough_maxid = npts;
  return ctx_vote(c, cos_t, sin_t, n_theta, rho_max, drho, n_rho, acc_out);
}

int ctx_support(lms_ctx* c, const double* cos_p, const double* sin_p, const int64_t* rbin_p,
                int64_t npeaks, double rho_max, double drho, int64_t n_rho, int64_t* offsets,
                int64_t* out, int64_t capacity, int32_t* out32 = nullptr) {
  if (npeaks < 0 || !offsets || (npeaks > 0 && (!cos_p || !sin_p || !rbin_p)))
    return set_error(LMS_ERR_INVALID, "bad peaks");
  if (c->hough_mode == 0) return set_error(LMS_ERR_INVALID, "no points: call a vote first");
  RC_TRY(check_hough(1, rho_max, drho, n_rho));
  CUDA_TRY(cudaSetDevice(c->device));
  const int64_t npts = c->hough_npts;
  const int64_t nb = lmsb::support_blocks(npts);
  offsets[0] = 0;
  if (npts == 0 || npeaks == 0) {
    for (int64_t p = 0; p < npeaks; ++p) offsets[p + 1] = 0;
    return LMS_OK;
  }
  RC_TRY(c->masks.need(npts));
  RC_TRY(c->scounts.need(64 * nb + 1));
  RC_TRY(c->soffsets.need(64 * nb + 1));
  RC_TRY(c->rbin.need(64));
  RC_TRY(c->tcos.need(64));
  RC_TRY(c->tsin.need(64));
  RC_TRY(c->scan_tmp.need((int64_t)lmsb::support_scan_temp_bytes(64 * nb + 1)));
  std::vector<int64_t> goff(64 * nb + 1);
  int64_t total = 0;
  for (int64_t g0 = 0; g0 < npeaks; g0 += 64) {
    const int np = (int)std::min<int64_t>(64, npeaks - g0);
    CUDA_TRY(cudaMemcpyAsync(c->tcos.p, cos_p + g0, sizeof(double) * np, cudaMemcpyHostToDevice,
                             c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->tsin.p, sin_p + g0, sizeof(double) * np, cudaMemcpyHostToDevice,
                             c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->rbin.p, rbin_p + g0, sizeof(int64_t) * np, cudaMemcpyHostToDevice,
                             c->stream));
    CUDA_TRY(cudaMemsetAsync(c->scounts.p, 0, sizeof(int64_t) * (np * nb + 1), c->stream));
    RC_TRY(c->sout.need(std::max<int64_t>(1, capacity - total)));
    // pass 1 + scan + pass 2 into a device buffer sized by the caller's
    // capacity; rerun once with a grown buffer if the members did not fit
    const int64_t m = (int64_t)np * nb + 1;
    int64_t group_total = 0;
    for (int attempt = 0; attempt < 2; ++attempt) {
      if (lmsb::hough_support(c->hough_mode == 1 ? c->pix.p : nullptr,
                              c->hough_mode == 2 ? c->pxs.p : nullptr,
                              c->hough_mode == 2 ? c->pys.p : nullptr, npts, c->hough_width,
                              c->tcos.p, c->tsin.p, c->rbin.p, np, rho_max, drho, n_rho,
                              c->masks.p, c->scounts.p, c->soffsets.p, c->scan_tmp.p,
                              (size_t)c->scan_tmp.cap, c->sout.p, c->sout.cap, c->stream) != 0)
        return set_error(LMS_ERR_CUDA, "support scan failed");
      CUDA_TRY(cudaGetLastError());
      CUDA_TRY(cudaMemcpyAsync(goff.data(), c->soffsets.p, sizeof(int64_t) * m,
                               cudaMemcpyDeviceToHost, c->stream));
      CUDA_TRY(cudaStreamSynchronize(c->stream));
      group_total = goff[m - 1];
      if (group_total <= c->sout.cap) break;
      RC_TRY(c->sout.need(group_total));  // grown: write again
    }
    for (int q = 0; q < np; ++q) offsets[g0 + q + 1] = total + goff[(int64_t)(q + 1) * nb];
    if (out && total + group_total <= capacity && group_total > 0)
      RC_TRY(download_staged(c, out + total, c->sout.p, sizeof(int64_t) * group_total));
    if (out32 && total + group_total <= capacity && group_total > 0) {
      // half the download: indices narrowed on the device
      RC_TRY(c->sout32.need(group_total));
      lmsb::launch_narrow_i32(c->sout.p, c->sout32.p, group_total, c->stream);
      RC_TRY(download_staged(c, out32 + total, c->sout32.p, sizeof(int32_t) * group_total));
    }
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    total += group_total;
  }
  if (total > capacity)
    return set_error(LMS_ERR_INVALID, "support output capacity %lld < %lld members",
                     (long long)capacity, (long long)total);
  return LMS_OK;
}

// One cached context per device for the one-shot entry points.
std::mutex g_ctx_mu;
std::vector<lms_ctx*> g_ctx;

int shared_ctx(int device, lms_ctx** out) {
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    return set_error(LMS_ERR_NODEVICE, "no CUDA device available");
  if (device < 0 || device >= count)
    return set_error(LMS_ERR_NODEVICE, "device %d out of range (%d devices)", device, count);
  if ((int)g_ctx.size() < count) g_ctx.resize(count, nullptr);
  if (!g_ctx[device]) {
    lms_ctx* c = new lms_ctx();
    int rc = ctx_init(c, device);
    if (rc) {
      ctx_release(c);
      delete c;
      return rc;
    }
    g_ctx[device] = c;
  }
  *out = g_ctx[device];
  return LMS_OK;
}

// ---------------------------------------------------------------- multi-GPU
// Sharded band search with band ownership: every shard samples the whole
// pair space (the same slope bands everywhere), bounds and seeds its own
// interleaved slice of the bands (shard, shard + nshards, ...), the seed
// records are exchanged (one all-gather of 56-byte records), and each shard
// searches the vertices of its own bands that the best seed cannot dismiss,
// over the whole pair space; a second all-gather of the records and the
// lexicographic (height, i, j) minimum (backend.py:182-187) finish the fit.
// Every vertex lies in exactly one band and the global seed is a real
// vertex, so the minimum is the one-GPU record for any shard count.  Fits
// too small for the band stage (the plan reports no bands) split the pair
// ranks instead (BatchPlan.partitions, backend.py:84-92).

// plan of shard `shard` (no band-table output); *nbands = 0: not banded
int owned_plan(lms_ctx* c, int64_t q, int nshards, int shard, lms_candidate* seed,
               int64_t* nbands) {
  const int64_t n = c->nlines;
  RC_TRY(check_fit(c, 0, n, q));
  const int64_t total = n * (n - 1) / 2;
  ShardSpec sp;
  sp.mode = 1;
  sp.P0 = 0;
  sp.P1 = total;
  sp.nshards = nshards;
  sp.shard = shard;
  c->shard = &sp;
  lms_candidate dummy;
  std::vector<HostFit> hf{{0, n, q, 0, total}};
  const int rc = ctx_solve_fits(c, hf, &dummy);
  c->shard = nullptr;
  if (rc != LMS_OK) return rc;
  *seed = sp.seed_out;
  *nbands = sp.K;
  c->plan_gen = c->gen;
  c->plan_nshards = nshards;
  c->plan_shard = shard;
  c->plan_K = sp.K;
  return LMS_OK;
}

// search of shard `shard` after its plan: own bands (banded) or its pair-rank
// partition (not banded), with the exchanged best seed installed
int owned_search(lms_ctx* c, int64_t q, int nshards, int shard, int64_t nbands,
                 const lms_candidate& seed, lms_candidate* out) {
  const int64_t n = c->nlines;
  RC_TRY(check_fit(c, 0, n, q));
  const int64_t total = n * (n - 1) / 2;
  std::memset(out, 0, sizeof(*out));
  if (nbands <= 0) {
    int64_t r0, r1;
    share_of(total, nshards, shard, &r0, &r1);
    if (r1 <= r0) return LMS_OK;
    std::vector<HostFit> hf{{0, n, q, r0, r1}};
    return ctx_solve_fits(c, hf, out);
  }
  ShardSpec sp;
  sp.mode = 3;
  sp.P0 = 0;
  sp.P1 = total;
  sp.nshards = nshards;
  sp.shard = shard;
  sp.seed_in = seed;
  c->shard = &sp;
  std::vector<HostFit> hf{{0, n, q, 0, total}};
  const int rc = ctx_solve_fits(c, hf, out);
  c->shard = nullptr;
  return rc;
}

lms_candidate cand_min(const lms_candidate* recs, int m) {
  lms_candidate best{};
  for (int r = 0; r < m; ++r)
    if (lmsb::cand_less(recs[r], best)) best = recs[r];
  return best;
}

#define NCCL_TRY(expr)                                                                     \
  do {                                                                                     \
    const ncclResult_t nr_ = (expr);                                                       \
    if (nr_ != ncclSuccess)                                                                \
      return set_error(LMS_ERR_CUDA, "%s: %s", #expr, lmsb::nccl().GetErrorString(nr_)); \
  } while (0)

// All-gather of one record per rank over the context's NCCL communicator, on
// device buffers (the context's stream); all[0 .. comm_ranks) on the host.
int nccl_gather_records(lms_ctx* c, const lms_candidate& mine, lms_candidate* all) {
  const int R = c->comm_ranks;
  RC_TRY(c->xsend.need(1));
  RC_TRY(c->xrecv.need(R));
  RC_TRY(ensure_pinned(c, sizeof(lms_candidate) * (R + 1)));
  lms_candidate* pin = reinterpret_cast<lms_candidate*>(c->pin);
  pin[0] = mine;
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaMemcpyAsync(c->xsend.p, pin, sizeof(lms_candidate), cudaMemcpyHostToDevice,
                           c->stream));
  NCCL_TRY(lmsb::nccl().AllGather(c->xsend.p, c->xrecv.p, sizeof(lms_candidate), ncclUint8,
                                  c->comm, c->stream));
  CUDA_TRY(cudaMemcpyAsync(pin + 1, c->xrecv.p, sizeof(lms_candidate) * R, cudaMemcpyDeviceToHost,
                           c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  std::memcpy(all, pin + 1, sizeof(lms_candidate) * R);
  return LMS_OK;
}

// In-process exchange between the shard threads of one lms_min_bracelet_multi
// call: a host barrier (shards that share a GPU cannot form an NCCL clique).
struct HostExchange {
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0, phase = 0, parties = 0;
  std::vector<lms_candidate> slots;
  bool failed = false;
  // publish `mine` at `rank`, wait for everyone, copy all records out
  bool gather(int rank, const lms_candidate& mine, lms_candidate* all, bool ok) {
    std::unique_lock<std::mutex> lk(mu);
    slots[rank] = mine;
    failed |= !ok;
    const int ph = phase;
    if (++arrived == parties) {
      arrived = 0;
      ++phase;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return phase != ph; });
    }
    std::copy(slots.begin(), slots.end(), all);
    return !failed;
  }
};

struct MultiCtx {
  std::vector<int> devices;
  std::vector<lms_ctx*> ctxs;
  bool nccl = false;
};
std::mutex g_multi_mu;
MultiCtx g_multi;

void multi_release() {
  for (lms_ctx* c : g_multi.ctxs) {
    ctx_release(c);
    delete c;
  }
  g_multi.ctxs.clear();
  g_multi.devices.clear();
  g_multi.nccl = false;
}

// contexts (and, with NCCL, a communicator clique) for this shard-to-device map
int multi_setup(const int32_t* devices, int nshards, bool use_nccl) {
  std::vector<int> dv(devices, devices + nshards);
  if (g_multi.devices == dv && g_multi.nccl == use_nccl && (int)g_multi.ctxs.size() == nshards)
    return LMS_OK;
  multi_release();
  for (int r = 0; r < nshards; ++r) {
    lms_ctx* c = new lms_ctx();
    const int rc = ctx_init(c, dv[r]);
    if (rc) {
      ctx_release(c);
      delete c;
      multi_release();
      return rc;
    }
    g_multi.ctxs.push_back(c);
  }
  if (use_nccl) {
    std::vector<ncclComm_t> comms(nshards);
    const ncclResult_t nr = lmsb::nccl().CommInitAll(comms.data(), nshards, dv.data());
    if (nr != ncclSuccess) {
      multi_release();
      return set_error(LMS_ERR_CUDA, "ncclCommInitAll: %s", lmsb::nccl().GetErrorString(nr));
    }
    for (int r = 0; r < nshards; ++r) {
      g_multi.ctxs[r]->comm = comms[r];
      g_multi.ctxs[r]->comm_owned = true;
      g_multi.ctxs[r]->comm_ranks = nshards;
      g_multi.ctxs[r]->comm_rank = r;
    }
  }
  g_multi.devices = dv;
  g_multi.nccl = use_nccl;
  return LMS_OK;
}

}  // namespace

extern "C" {

int lms_version(void) { return LMS_VERSION; }

int lms_device_count(int* count) {
  if (!count) return set_error(LMS_ERR_INVALID, "null count");
  *count = 0;
  cudaError_t e = cudaGetDeviceCount(count);
  if (e != cudaSuccess) {
    *count = 0;
    cudaGetLastError();
  }
  return LMS_OK;
}

const char* lms_last_error(void) { return g_last_error.c_str(); }

int lms_min_bracelet_f64(const double* a, const double* b, int64_t n, int64_t q,
                         int64_t rank_begin, int64_t rank_end, int device, lms_candidate* out) {
  if (!out) return set_error(LMS_ERR_INVALID, "null output");
  lms_ctx* c = nullptr;
  RC_TRY(shared_ctx(device, &c));
  std::lock_guard<std::mutex> lk(c->mu);
  RC_TRY(ctx_upload(c, a, b, n));
  return ctx_solve(c, q, rank_begin, rank_end, out);
}

int lms_solve_fit_f64(const double* a, const double* b, int64_t n, int64_t q, int device,
                      lms_candidate* out, int64_t* contacts, int64_t cap, int64_t* ncontacts) {
  if (!out || !ncontacts || (cap > 0 && !contacts)) return set_error(LMS_ERR_INVALID, "null output");
  *ncontacts = 0;
  lms_ctx* c = nullptr;
  RC_TRY(shared_ctx(device, &c));
  std::lock_guard<std::mutex> lk(c->mu);
  RC_TRY(ctx_upload(c, a, b, n));
  RC_TRY(ctx_solve(c, q, 0, n * (n - 1) / 2, out));
  if (!out->found) return LMS_OK;
  RC_TRY(c->ii.need(std::max<int64_t>(n, 1)));
  RC_TRY(c->counters.need(2));
  lmsb::launch_contacts(c->a, c->b, n, *out, c->counters.p, c->ii.p, n, c->sms, c->stream);
  CUDA_TRY(cudaGetLastError());
  // one round trip for the usual few contacts: the count and the first
  // kPrefetch indices come back together
  constexpr int64_t kPrefetch = 1024;
  RC_TRY(ensure_pinned(c, (kPrefetch + 1) * sizeof(int64_t)));
  unsigned long long* p_cnt = reinterpret_cast<unsigned long long*>(c->pin);
  int64_t* p_idx = reinterpret_cast<int64_t*>(c->pin) + 1;
  const int64_t pre = std::min<int64_t>(kPrefetch, n);
  CUDA_TRY(cudaMemcpyAsync(p_cnt, c->counters.p + 1, sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaMemcpyAsync(p_idx, c->ii.p, sizeof(int64_t) * pre, cudaMemcpyDeviceToHost,
                           c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  const unsigned long long cnt = *p_cnt;
  const int64_t m = std::min<int64_t>((int64_t)cnt, cap);
  if (m > 0) {
    std::vector<int64_t> h((size_t)cnt);
    if ((int64_t)cnt <= pre) std::copy(p_idx, p_idx + cnt, h.begin());
    else CUDA_TRY(cudaMemcpy(h.data(), c->ii.p, sizeof(int64_t) * cnt, cudaMemcpyDeviceToHost));
    std::sort(h.begin(), h.end());
    std::copy(h.begin(), h.begin() + m, contacts);
  }
  *ncontacts = (int64_t)cnt;
  return LMS_OK;
}

int lms_min_bracelet_materialized_f64(const double* a, const double* b, int64_t n, int64_t q,
                                      int64_t rank_begin, int64_t rank_end, int device,
                                      lms_candidate* out) {
  if (!out) return set_error(LMS_ERR_INVALID, "null output");
  lms_ctx* c = nullptr;
  RC_TRY(shared_ctx(device, &c));
  std::lock_guard<std::mutex> lk(c->mu);
  RC_TRY(ctx_upload(c, a, b, n));
  return ctx_solve_materialized(c, q, rank_begin, rank_end, out);
}

int lms_ctx_solve_materialized(lms_ctx* c, int64_t q, int64_t rank_begin, int64_t rank_end,
                               lms_candidate* out) {
  if (!c || !out) return set_error(LMS_ERR_INVALID, "null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  return ctx_solve_materialized(c, q, rank_begin, rank_end, out);
}

int lms_batched_f64(const double* x, const double* y, const int64_t* offsets, const int64_t* q,
                    int64_t nfits, int device, lms_candidate* out) {
  if (!offsets || nfits < 0 || (nfits > 0 && (!out || !x || !y || !q)))
    return set_error(LMS_ERR_INVALID, "null argument");
  if (nfits == 0) return LMS_OK;
  if (offsets[0] != 0) return set_error(LMS_ERR_INVALID, "offsets[0] must be 0");
  lms_ctx* c = nullptr;
  RC_TRY(shared_ctx(device, &c));
  std::lock_guard<std::mutex> lk(c->mu);
  RC_TRY(ctx_upload(c, x, y, offsets[nfits]));
  return ctx_solve_batch(c, offsets, q, nfits, out);
}

int lms_batched_fit_f64(const double* x, const double* y, const int64_t* offsets, const int64_t* q,
                        int64_t nfits, int device, lms_candidate* out, uint8_t* contact_flags) {
  if (!offsets || nfits < 0 || (nfits > 0 && (!out || !x || !y || !q || !contact_flags)))
    return set_error(LMS_ERR_INVALID, "null argument");
  if (nfits == 0) return LMS_OK;
  if (offsets[0] != 0) return set_error(LMS_ERR_INVALID, "offsets[0] must be 0");
  lms_ctx* c = nullptr;
  RC_TRY(shared_ctx(device, &c));
  std::lock_guard<std::mutex> lk(c->mu);
  const int64_t N = offsets[nfits];
  RC_TRY(ctx_upload(c, x, y, N));
  RC_TRY(ctx_solve_batch(c, offsets, q, nfits, out));
  // the fits' records are in c->best (fit-local anchors)
  RC_TRY(c->boffs.need(nfits + 1));
  RC_TRY(c->bcflags.need(std::max<int64_t>(N, 1)));
  CUDA_TRY(cudaMemcpyAsync(c->boffs.p, offsets, sizeof(int64_t) * (nfits + 1),
                           cudaMemcpyHostToDevice, c->stream));
  lmsb::launch_contacts_batch(c->a, c->b, c->boffs.p, c->best.p, nfits, c->bcflags.p, c->sms,
                              c->stream);
  CUDA_TRY(cudaGetLastError());
  RC_TRY(download_staged(c, contact_flags, c->bcflags.p, (size_t)N));
  return LMS_OK;
}

int lms_primal_brute_f64(const double* x, const double* y, int64_t n, int64_t q, int device,
                         lms_candidate* out) {
  if (!out) return set_error(LMS_ERR_INVALID, "null output");
  lms_ctx* c = nullptr;
  RC_TRY(shared_ctx(device, &c));
  std::lock_guard<std::mutex> lk(c->mu);
  RC_TRY(ctx_upload(c, x, y, n));
  return ctx_primal(c, q, out);
}

int lms_hough_vote_u8(const uint8_t* img, int64_t height, int64_t width, int threshold,
                      const double* cos_t, const double* sin_t, int64_t n_theta, double rho_max,
                      double delta_rho, int64_t n_rho, int device, int64_t* acc,
                      int64_t* npoints) {
  if (!acc || !npoints || !cos_t || !sin_t) return set_error(LMS_ERR_INVALID, "null argument");
  lms_ctx* c = nullptr;
  RC_TRY(shared_ctx(device, &c));
  std::lock_guard<std::mutex> lk(c->mu);
  return ctx_vote_image(c, img, height, width, threshold, cos_t, sin_t, n_theta, rho_max,
                        delta_rho, n_rho, acc, npoints);
}

int lms_hough_vote_points(const double* x, const double* y, int64_t npts, const double* cos_t,
                          const double* sin_t, int64_t n_theta, double rho_max, double delta_rho,
                          int64_t n_rho, int device, int64_t* acc) {
  if (!acc || !cos_t || !sin_t) return set_error(LMS_ERR_INVALID, "null argument");
  lms_ctx* c = nullptr;
  RC_TRY(shared_ctx(device, &c));
  std::lock_guard<std::mutex> lk(c->mu);
  return ctx_vote_points(c, x, y, npts, cos_t, sin_t, n_theta, rho_max, delta_rho, n_rho, acc);
}

int lms_hough_support(const double* cos_p, const double* sin_p, const int64_t* rbin_p,
                      int64_t npeaks, double rho_max, double delta_rho, int64_t n_rho, int device,
                      int64_t* offsets, int64_t* out, int64_t capacity) {
  lms_ctx* c = nullptr;
  RC_TRY(shared_ctx(device, &c));
  std::lock_guard<std::mutex> lk(c->mu);
  return ctx_support(c, cos_p, sin_p, rbin_p, npeaks, rho_max, delta_rho, n_rho, offsets, out,
                     capacity);
}

int lms_hough_support_i32(const double* cos_p, const double* sin_p, const int64_t* rbin_p,
                          int64_t npeaks, double rho_max, double delta_rho, int64_t n_rho,
                          int device, int64_t* offsets, int32_t* out, int64_t capacity) {
  lms_ctx* c = nullptr;
  RC_TRY(shared_ctx(device, &c));
  std::lock_guard<std::mutex> lk(c->mu);
  if (std::max(c->hough_npts, c->hough_maxid) > INT32_MAX)
    return set_error(LMS_ERR_INVALID, "support ids exceed int32: use lms_hough_support");
  return ctx_support(c, cos_p, sin_p, rbin_p, npeaks, rho_max, delta_rho, n_rho, offsets, nullptr,
                     capacity, out);
}

int lms_eval_vertices_f64(const double* a, const double* b, int64_t n, int64_t q, const int64_t* i,
                          const int64_t* j, const double* u, const double* v, int64_t m, int device,
                          lms_candidate* out) {
  if (!out || (m > 0 && (!i || !j || !u))) return set_error(LMS_ERR_INVALID, "null argument");
  lms_ctx* c = nullptr;
  RC_TRY(shared_ctx(device, &c));
  std::lock_guard<std::mutex> lk(c->mu);
  RC_TRY(ctx_upload(c, a, b, n));
  return ctx_eval_explicit(c, q, i, j, u, v, m, out, false);
}

int lms_min_over_vertices_f64(const double* a, const double* b, int64_t n, int64_t q,
                              const int64_t* i, const int64_t* j, const double* u, int64_t m,
                              int device, lms_candidate* out) {
  if (!out || (m > 0 && (!i || !j || !u))) return set_error(LMS_ERR_INVALID, "null argument");
  lms_ctx* c = nullptr;
  RC_TRY(shared_ctx(device, &c));
  std::lock_guard<std::mutex> lk(c->mu);
  RC_TRY(ctx_upload(c, a, b, n));
  return ctx_eval_explicit(c, q, i, j, u, nullptr, m, out, true);
}

int lms_ctx_create(int device, lms_ctx** out) {
  if (!out) return set_error(LMS_ERR_INVALID, "null output");
  *out = nullptr;
  lms_ctx* c = new lms_ctx();
  int rc = ctx_init(c, device);
  if (rc) {
    ctx_release(c);
    delete c;
    return rc;
  }
  *out = c;
  return LMS_OK;
}

int lms_ctx_destroy(lms_ctx* c) {
  if (!c) return LMS_OK;
  ctx_release(c);
  delete c;
  return LMS_OK;
}

int lms_ctx_upload(lms_ctx* c, const double* a, const double* b, int64_t n) {
  if (!c) return set_error(LMS_ERR_INVALID, "null context");
  std::lock_guard<std::mutex> lk(c->mu);
  return ctx_upload(c, a, b, n);
}

int lms_ctx_bind_dev(lms_ctx* c, const double* d_a, const double* d_b, int64_t n) {
  if (!c || !d_a || !d_b || n < 1) return set_error(LMS_ERR_INVALID, "bad arguments");
  std::lock_guard<std::mutex> lk(c->mu);
  CUDA_TRY(cudaSetDevice(c->device));
  c->ext_off.clear();
  c->h_a.resize(n);
  c->h_b.resize(n);
  CUDA_TRY(cudaMemcpy(c->h_a.data(), d_a, sizeof(double) * n, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(c->h_b.data(), d_b, sizeof(double) * n, cudaMemcpyDeviceToHost));
  c->a = d_a;
  c->b = d_b;
  c->nlines = n;
  cache_line_stats(c);
  return LMS_OK;
}

int lms_ctx_solve(lms_ctx* c, int64_t q, int64_t rank_begin, int64_t rank_end,
                  lms_candidate* out) {
  if (!c || !out) return set_error(LMS_ERR_INVALID, "null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  return ctx_solve(c, q, rank_begin, rank_end, out);
}

int lms_ctx_shard_plan(lms_ctx* c, int64_t q, int32_t nshards, int32_t shard, int64_t capacity,
                       int64_t* nbands, int64_t* nslice, double* lower_bound,
                       double* window, float* edge_keys, lms_candidate* seed) {
  if (!c || !nbands || !nslice || !seed)
    return set_error(LMS_ERR_INVALID, "null argument");
  std::memset(seed, 0, sizeof(*seed));
  if (nshards < 1 || shard < 0 || shard >= nshards)
    return set_error(LMS_ERR_INVALID, "bad shard %d of %d", shard, nshards);
  if (capacity > 0 && (!lower_bound || !window || !edge_keys))
    return set_error(LMS_ERR_INVALID, "null band buffers");
  std::lock_guard<std::mutex> lk(c->mu);
  *nbands = *nslice = 0;
  if (!c->a) return set_error(LMS_ERR_INVALID, "no lines bound to the context");
  const int64_t n = c->nlines;
  RC_TRY(check_fit(c, 0, n, q));
  const int64_t total = n * (n - 1) / 2;
  ShardSpec sp;
  sp.mode = 1;
  sp.P0 = 0;
  sp.P1 = total;
  sp.nshards = nshards;
  sp.shard = shard;
  sp.cap = capacity;
  sp.lb_out = lower_bound;
  sp.wq_out = window;
  sp.edge_out = edge_keys;
  c->shard = &sp;
  lms_candidate dummy;
  std::vector<HostFit> hf{{0, n, q, 0, total}};
  const int rc = ctx_solve_fits(c, hf, &dummy);
  c->shard = nullptr;
  if (rc != LMS_OK) return rc;
  *nbands = sp.K;
  *nslice = sp.k0;
  *seed = sp.seed_out;
  c->plan_gen = c->gen;
  c->plan_nshards = nshards;
  c->plan_shard = shard;
  c->plan_K = sp.K;
  return LMS_OK;
}

int lms_ctx_shard_search(lms_ctx* c, int64_t q, int32_t nshards, int32_t shard, int64_t nbands,
                         const double* lower_bound, const double* window, const float* edge_keys,
                         const lms_candidate* seed, lms_candidate* out) {
  if (!c || !out) return set_error(LMS_ERR_INVALID, "null argument");
  if (nshards < 1 || shard < 0 || shard >= nshards)
    return set_error(LMS_ERR_INVALID, "bad shard %d of %d", shard, nshards);
  if (nbands < 0 || (nbands > 0 && (!lower_bound || !window || !edge_keys)))
    return set_error(LMS_ERR_INVALID, "null band arrays");
  std::lock_guard<std::mutex> lk(c->mu);
  std::memset(out, 0, sizeof(*out));
  if (!c->a) return set_error(LMS_ERR_INVALID, "no lines bound to the context");
  const int64_t n = c->nlines;
  RC_TRY(check_fit(c, 0, n, q));
  const int64_t total = n * (n - 1) / 2;
  ShardSpec sp;
  sp.mode = 2;
  sp.P0 = 0;
  sp.P1 = total;
  sp.nshards = nshards;
  sp.shard = shard;
  sp.K_in = nbands;
  sp.lb_in = lower_bound;
  sp.wq_in = window;
  sp.edge_in = edge_keys;
  if (seed) sp.seed_in = *seed;
  int64_t r0, r1;
  share_of(total, nshards, shard, &r0, &r1);
  c->shard = &sp;
  std::vector<HostFit> hf{{0, n, q, r0, r1}};
  const int rc = ctx_solve_fits(c, hf, out);
  c->shard = nullptr;
  return rc;
}

int lms_ctx_shard_search_owned(lms_ctx* c, int64_t q, int32_t nshards, int32_t shard,
                               const lms_candidate* seed, lms_candidate* out) {
  if (!c || !out) return set_error(LMS_ERR_INVALID, "null argument");
  if (nshards < 1 || shard < 0 || shard >= nshards)
    return set_error(LMS_ERR_INVALID, "bad shard %d of %d", shard, nshards);
  std::lock_guard<std::mutex> lk(c->mu);
  std::memset(out, 0, sizeof(*out));
  if (!c->a) return set_error(LMS_ERR_INVALID, "no lines bound to the context");
  if (!(c->plan_gen == c->gen && c->plan_nshards == nshards && c->plan_shard == shard))
    return set_error(LMS_ERR_INVALID,
                     "own-band search of shard %d/%d needs that shard's plan on this context first",
                     shard, nshards);
  lms_candidate none{};
  return owned_search(c, q, nshards, shard, c->plan_K, seed ? *seed : none, out);
}

int lms_nccl_available(int* version) {
  const lmsb::NcclApi& api = lmsb::nccl();
  if (version) {
    *version = 0;
    if (api.ok) api.GetVersion(version);
  }
  return api.ok ? 1 : 0;
}

int lms_nccl_unique_id(uint8_t* id) {
  if (!id) return set_error(LMS_ERR_INVALID, "null argument");
  if (!lmsb::nccl().ok) return set_error(LMS_ERR_INVALID, "NCCL (libnccl.so.2) not available");
  ncclUniqueId u;
  NCCL_TRY(lmsb::nccl().GetUniqueId(&u));
  std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
  return LMS_OK;
}

int lms_ctx_comm_init(lms_ctx* c, int32_t nranks, int32_t rank, const uint8_t* id) {
  if (!c || !id) return set_error(LMS_ERR_INVALID, "null argument");
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return set_error(LMS_ERR_INVALID, "bad rank %d of %d", rank, nranks);
  if (!lmsb::nccl().ok) return set_error(LMS_ERR_INVALID, "NCCL (libnccl.so.2) not available");
  std::lock_guard<std::mutex> lk(c->mu);
  if (c->comm && c->comm_owned) lmsb::nccl().CommDestroy(c->comm);
  c->comm = nullptr;
  ncclUniqueId u;
  std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
  CUDA_TRY(cudaSetDevice(c->device));
  ncclComm_t comm;
  NCCL_TRY(lmsb::nccl().CommInitRank(&comm, nranks, u, rank));
  c->comm = comm;
  c->comm_owned = true;
  c->comm_ranks = nranks;
  c->comm_rank = rank;
  return LMS_OK;
}

int lms_ctx_solve_distributed(lms_ctx* c, int64_t q, lms_candidate* out) {
  if (!c || !out) return set_error(LMS_ERR_INVALID, "null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  std::memset(out, 0, sizeof(*out));
  if (!c->comm) return set_error(LMS_ERR_INVALID, "no communicator (lms_ctx_comm_init first)");
  if (!c->a) return set_error(LMS_ERR_INVALID, "no lines bound to the context");
  const int R = c->comm_ranks, r = c->comm_rank;
  lms_candidate seed{}, mine{};
  int64_t nb = 0;
  // every rank joins both collectives whatever happens locally (a failed
  // rank sends a record with reserved = -1, so no peer waits forever and
  // every rank reports the failure)
  int rc = owned_plan(c, q, R, r, &seed, &nb);
  std::string err = rc != LMS_OK ? std::string(lms_last_error()) : std::string();
  std::vector<lms_candidate> all(R);
  if (rc != LMS_OK) {
    seed = lms_candidate{};
    seed.reserved = -1;
  }
  RC_TRY(nccl_gather_records(c, seed, all.data()));
  bool peer_failed = false;
  for (int k = 0; k < R; ++k) peer_failed |= all[k].reserved == -1;
  if (rc == LMS_OK && !peer_failed) {
    rc = owned_search(c, q, R, r, nb, cand_min(all.data(), R), &mine);
    if (rc != LMS_OK) err = lms_last_error();
  }
  if (rc != LMS_OK || peer_failed) {
    mine = lms_candidate{};
    mine.reserved = -1;
  }
  RC_TRY(nccl_gather_records(c, mine, all.data()));
  for (int k = 0; k < R; ++k) peer_failed |= all[k].reserved == -1;
  if (rc != LMS_OK) return set_error(rc, "%s", err.c_str());
  if (peer_failed) return set_error(LMS_ERR_CUDA, "a peer rank of the sharded search failed");
  for (auto& x : all) x.reserved = 0;
  *out = cand_min(all.data(), R);
  return LMS_OK;
}

int lms_min_bracelet_multi(const double* a, const double* b, int64_t n, int64_t q,
                           int32_t nshards, const int32_t* devices, lms_candidate* out) {
  if (!a || !b || !out || !devices) return set_error(LMS_ERR_INVALID, "null argument");
  if (nshards < 1 || nshards > 64) return set_error(LMS_ERR_INVALID, "bad shard count %d", nshards);
  std::memset(out, 0, sizeof(*out));
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    return set_error(LMS_ERR_NODEVICE, "no CUDA device available");
  std::vector<int> dv(devices, devices + nshards);
  bool distinct = true;
  for (int r = 0; r < nshards; ++r) {
    if (dv[r] < 0 || dv[r] >= count)
      return set_error(LMS_ERR_NODEVICE, "device %d out of range (%d devices)", dv[r], count);
    for (int t = 0; t < r; ++t) distinct &= dv[t] != dv[r];
  }
  // NCCL between distinct GPUs (LMSB_NCCL=0 disables, =1 also for one shard);
  // shards sharing a GPU exchange through host memory
  const char* env = getenv("LMSB_NCCL");
  const int nccl_knob = env ? atoi(env) : 2;
  const bool use_nccl = lmsb::nccl().ok && distinct && nccl_knob != 0 &&
                        (nshards > 1 || nccl_knob == 1);
  std::lock_guard<std::mutex> lk(g_multi_mu);
  RC_TRY(multi_setup(devices, nshards, use_nccl));
  HostExchange hx;
  hx.parties = nshards;
  hx.slots.assign(nshards, lms_candidate{});
  std::vector<int> rcs(nshards, LMS_OK);
  std::vector<std::string> errs(nshards);
  std::vector<lms_candidate> result(nshards);
  auto shard_main = [&](int r) {
    lms_ctx* c = g_multi.ctxs[r];
    std::lock_guard<std::mutex> ck(c->mu);
    std::vector<lms_candidate> all(nshards);
    lms_candidate seed{}, mine{};
    int64_t nb = 0;
    int rc = ctx_upload(c, a, b, n);
    if (rc == LMS_OK) rc = owned_plan(c, q, nshards, r, &seed, &nb);
    if (use_nccl) {
      // (a failed rank still joins both collectives with an empty record)
      int rc2 = nccl_gather_records(c, seed, all.data());
      if (rc == LMS_OK) rc = rc2;
      if (rc == LMS_OK) rc = owned_search(c, q, nshards, r, nb, cand_min(all.data(), nshards), &mine);
      rc2 = nccl_gather_records(c, rc == LMS_OK ? mine : lms_candidate{}, all.data());
      if (rc == LMS_OK) rc = rc2;
    } else {
      bool ok = hx.gather(r, seed, all.data(), rc == LMS_OK);
      if (rc == LMS_OK && ok) rc = owned_search(c, q, nshards, r, nb, cand_min(all.data(), nshards), &mine);
      ok = hx.gather(r, mine, all.data(), rc == LMS_OK && ok);
      if (rc == LMS_OK && !ok) rc = LMS_ERR_CUDA;
    }
    if (rc != LMS_OK) errs[r] = lms_last_error();
    rcs[r] = rc;
    result[r] = cand_min(all.data(), nshards);
  };
  if (nshards == 1) {
    shard_main(0);
  } else {
    std::vector<std::thread> th;
    for (int r = 0; r < nshards; ++r) th.emplace_back(shard_main, r);
    for (auto& t : th) t.join();
  }
  for (int r = 0; r < nshards; ++r)
    if (rcs[r] != LMS_OK) {
      const bool own = !errs[r].empty() && errs[r] != "ok";
      return set_error(rcs[r], "shard %d: %s", r, own ? errs[r].c_str() : "peer failure");
    }
  *out = result[0];
  return LMS_OK;
}

int lms_device_stats(int device, lms_stats* out) {
  if (!out) return set_error(LMS_ERR_INVALID, "null argument");
  lms_ctx* c = nullptr;
  RC_TRY(shared_ctx(device, &c));
  std::lock_guard<std::mutex> lk(c->mu);
  *out = c->stats;
  return LMS_OK;
}

int lms_detect_peaks_u8(const uint8_t* img, int64_t height, int64_t width, int threshold,
                        const double* cos_t, const double* sin_t, int64_t n_theta, double rho_max,
                        double delta_rho, int64_t n_rho, int64_t max_peaks, int64_t min_votes,
                        int device, int64_t* acc, int64_t* npoints, int64_t* peaks,
                        int64_t* npeaks) {
  if (!img || !cos_t || !sin_t || !npoints || !peaks || !npeaks)
    return set_error(LMS_ERR_INVALID, "null argument");
  if (height < 0 || width < 0) return set_error(LMS_ERR_INVALID, "bad image");
  if (max_peaks < 1 || max_peaks > 64) return set_error(LMS_ERR_INVALID, "max_peaks must be in [1, 64]");
  if (n_theta * n_rho > lmsb::kDetectMaxBins || n_theta > 512)
    return set_error(LMS_ERR_INVALID, "accumulator too large for the device peak finder");
  const int64_t npix = height * width;
  if (npix > INT32_MAX) return set_error(LMS_ERR_INVALID, "image too large for int32 pixel ids");
  if (width > lmsb::kDetectMaxWidth || n_rho > 4095)
    return set_error(LMS_ERR_INVALID, "image too wide or rho range too fine for the device vote");
  lms_ctx* c = nullptr;
  RC_TRY(shared_ctx(device, &c));
  std::lock_guard<std::mutex> lk(c->mu);
  RC_TRY(check_hough(n_theta, rho_max, delta_rho, n_rho));
  CUDA_TRY(cudaSetDevice(c->device));
  const int64_t nb = n_theta * n_rho;
  RC_TRY(c->img.need(std::max<int64_t>(npix, 4)));
  RC_TRY(c->acc.need(nb));
  RC_TRY(c->tcos.need(n_theta));
  RC_TRY(c->tsin.need(n_theta));
  RC_TRY(c->dt_peaks.need(3 * 64 + 1));
  RC_TRY(c->dt_nlit.need(1));
  RC_TRY(ensure_pinned(c, sizeof(int64_t) * (3 * 64 + 4) + sizeof(unsigned long long) * nb));
  if (npix > 0) RC_TRY(upload_staged(c, c->img.p, img, (size_t)npix));
  CUDA_TRY(cudaMemcpyAsync(c->tcos.p, cos_t, sizeof(double) * n_theta, cudaMemcpyHostToDevice,
                           c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->tsin.p, sin_t, sizeof(double) * n_theta, cudaMemcpyHostToDevice,
                           c->stream));
  CUDA_TRY(cudaMemsetAsync(c->acc.p, 0, sizeof(unsigned long long) * nb, c->stream));
  CUDA_TRY(cudaMemsetAsync(c->dt_nlit.p, 0, sizeof(unsigned long long), c->stream));
  lmsb::DetectImage im{c->img.p, npix, std::max<int64_t>(width, 1), threshold};
  lmsb::HoughGrid g{(int)n_rho, (int)n_theta, rho_max, delta_rho};
  while (c->ev_chunk.size() < 14) {
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreate(&e));
    c->ev_chunk.push_back(e);
  }
  CUDA_TRY(cudaEventRecord(c->ev_chunk[12], c->stream));
  RC_TRY(c->dt_wedge.need(n_rho));
  RC_TRY(c->dt_bits.need(std::max<int64_t>(1, height * ((width + 31) / 32))));
  if (npix > 0)
    lmsb::launch_detect_vote(im, g, c->tcos.p, c->tsin.p, c->dt_wedge.p, c->dt_bits.p, c->acc.p,
                             c->dt_nlit.p, c->sms, c->stream);
  CUDA_TRY(cudaEventRecord(c->ev_chunk[13], c->stream));
  int64_t* d_np = c->dt_peaks.p + 3 * 64;
  lmsb::launch_detect_peaks(c->acc.p, g, min_votes, (int)max_peaks, c->dt_peaks.p, d_np, c->stream);
  CUDA_TRY(cudaGetLastError());
  int64_t* pin = reinterpret_cast<int64_t*>(c->pin);
  CUDA_TRY(cudaMemcpyAsync(pin, c->dt_peaks.p, sizeof(int64_t) * (3 * 64 + 1), cudaMemcpyDeviceToHost,
                           c->stream));
  CUDA_TRY(cudaMemcpyAsync(pin + 3 * 64 + 1, c->dt_nlit.p, sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, c->stream));
  if (acc) CUDA_TRY(cudaMemcpyAsync(acc, c->acc.p, sizeof(int64_t) * nb, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  const int64_t m = pin[3 * 64];
  *npeaks = m;
  *npoints = pin[3 * 64 + 1];
  float vote_ms = 0.f;
  CUDA_TRY(cudaEventElapsedTime(&vote_ms, c->ev_chunk[12], c->ev_chunk[13]));
  c->stats.ms_hough_vote = vote_ms;
  std::memcpy(peaks, pin, sizeof(int64_t) * 3 * m);
  c->dt_npix = npix;
  c->dt_width = std::max<int64_t>(width, 1);
  c->dt_threshold = threshold;
  c->dt_grid = g;
  c->dt_npeaks = m;
  c->hough_mode = 0;  // the point-list Hough calls need their own vote
  return LMS_OK;
}

int lms_detect_supports_u8(const double* cos_s, const double* sin_s, const uint8_t* swap_t,
                           int64_t support_cap, const int64_t* q, int fit, int device,
                           int64_t* support_offsets, int32_t* support_ids, int64_t capacity,
                           int64_t* design_offsets, double* abscissa_range, lms_candidate* records,
                           uint8_t* contact_flags) {
  if (!cos_s || !sin_s || !swap_t || !support_offsets || !design_offsets || !abscissa_range)
    return set_error(LMS_ERR_INVALID, "null argument");
  lms_ctx* c = nullptr;
  RC_TRY(shared_ctx(device, &c));
  std::lock_guard<std::mutex> lk(c->mu);
  if (c->dt_npeaks < 0) return set_error(LMS_ERR_INVALID, "no peaks: call lms_detect_peaks_u8 first");
  const int P = (int)c->dt_npeaks;
  const int nt = c->dt_grid.n_theta;
  CUDA_TRY(cudaSetDevice(c->device));
  support_offsets[0] = 0;
  design_offsets[0] = 0;
  if (P == 0) return LMS_OK;
  const int64_t nch = lmsb::detect_support_rows(c->dt_npix, c->dt_width);
  RC_TRY(c->dt_counts.need(std::max<int64_t>((int64_t)P * nch, 1)));
  RC_TRY(c->dt_offs.need((int64_t)P * nch + 1));
  RC_TRY(c->dt_soffs.need(P + 1));
  RC_TRY(c->dt_doffs.need(P + 1));
  RC_TRY(c->dt_swap.need(nt));
  RC_TRY(c->dt_lim.need(2 * P));
  CUDA_TRY(cudaMemcpyAsync(c->dt_swap.p, swap_t, nt, cudaMemcpyHostToDevice, c->stream));
  // the supports' sizes are the peaks' votes (a support is the peak bin's
  // voters at the bin's own trig): the host sizes the outputs from them
  RC_TRY(ensure_pinned(c, sizeof(int64_t) * (3 * 64 + 4)));
  int64_t* pin = reinterpret_cast<int64_t*>(c->pin);
  CUDA_TRY(cudaMemcpyAsync(pin, c->dt_peaks.p, sizeof(int64_t) * 3 * P, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  int64_t total = 0;
  std::vector<int64_t> soff(P + 1, 0);
  for (int k = 0; k < P; ++k) {
    total += pin[3 * k + 2];
    soff[k + 1] = total;
  }
  // peaks grouped by theta bin (their support trig), in order of appearance
  lmsb::SupportTable tb{};
  tb.npeaks = P;
  {
    std::vector<int> slot_tb;
    for (int k = 0; k < P; ++k) {
      const int t = (int)pin[3 * k + 1];
      if (std::find(slot_tb.begin(), slot_tb.end(), t) == slot_tb.end()) slot_tb.push_back(t);
    }
    int m = 0;
    tb.nslot = (int)slot_tb.size();
    for (int sl = 0; sl < tb.nslot; ++sl) {
      const int t = slot_tb[sl];
      tb.trig[sl] = lmsb::Trig{(float)cos_s[t], (float)sin_s[t], cos_s[t], sin_s[t],
                               cos_s[t] != 0.0 ? 1.0 / cos_s[t] : 0.0};
      tb.first[sl] = m;
      for (int k = 0; k < P; ++k)
        if ((int)pin[3 * k + 1] == t) {
          tb.peak[m] = k;
          tb.rbin[m] = (int)pin[3 * k];
          ++m;
        }
    }
    tb.first[tb.nslot] = m;
  }
  std::vector<int64_t> doff(P + 1, 0);
  for (int k = 0; k < P; ++k) {
    const int64_t m = pin[3 * k + 2];
    doff[k + 1] = doff[k] + ((support_cap > 0 && m > support_cap) ? support_cap : m);
  }
  RC_TRY(c->dt_ids.need(std::max<int64_t>(total, 1)));
  RC_TRY(c->dt_a.need(std::max<int64_t>(doff[P], 1)));
  RC_TRY(c->dt_b.need(std::max<int64_t>(doff[P], 1)));
  CUDA_TRY(cudaMemcpyAsync(c->dt_doffs.p, doff.data(), sizeof(int64_t) * (P + 1), cudaMemcpyHostToDevice,
                           c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->dt_soffs.p, soff.data(), sizeof(int64_t) * (P + 1), cudaMemcpyHostToDevice,
                           c->stream));
  CUDA_TRY(cudaMemsetAsync(c->dt_nlit.p, 0, sizeof(unsigned long long), c->stream));
  lmsb::DetectImage im{c->img.p, c->dt_npix, c->dt_width, c->dt_threshold};
  const int64_t* d_np = c->dt_peaks.p + 3 * 64;
  CUDA_TRY(cudaEventRecord(c->ev_chunk[12], c->stream));
  lmsb::launch_detect_support(im, c->dt_grid, tb, c->dt_wedge.p, c->dt_bits.p, c->dt_soffs.p,
                              c->dt_counts.p, c->dt_offs.p, c->dt_ids.p, c->dt_nlit.p, c->sms,
                              c->stream);
  CUDA_TRY(cudaEventRecord(c->ev_chunk[13], c->stream));
  lmsb::launch_detect_design(c->dt_peaks.p, d_np, P, c->dt_soffs.p, c->dt_ids.p, c->dt_width,
                             support_cap, c->dt_swap.p, c->dt_doffs.p, c->dt_a.p, c->dt_b.p,
                             c->dt_lim.p, c->stream);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(abscissa_range, c->dt_lim.p, sizeof(double) * 2 * P,
                           cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaMemcpyAsync(pin, c->dt_nlit.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                           c->stream));
  std::memcpy(design_offsets, doff.data(), sizeof(int64_t) * (P + 1));
  std::memcpy(support_offsets, soff.data(), sizeof(int64_t) * (P + 1));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (pin[0] != 0)
    return set_error(LMS_ERR_CUDA, "%lld supports differ in size from their peaks' votes",
                     (long long)pin[0]);
  float sup_ms = 0.f;
  CUDA_TRY(cudaEventElapsedTime(&sup_ms, c->ev_chunk[12], c->ev_chunk[13]));
  const float vote_ms = c->stats.ms_hough_vote;
  if (total > capacity) return set_error(LMS_ERR_INVALID, "support capacity %lld < %lld",
                                         (long long)capacity, (long long)total);
  // the supports go down while the fits run: the designs are copied first
  // (the solver binds host copies of its lines for its line statistics)
  bool run_fit = fit != 0;
  for (int k = 0; k < P && run_fit; ++k) {
    const int64_t n = doff[k + 1] - doff[k];
    run_fit = n >= 3 && abscissa_range[2 * k] < abscissa_range[2 * k + 1] && q && q[k] >= 2 && q[k] <= n;
  }
  if (run_fit) {
    const int64_t N = doff[P];
    c->ext_off.clear();
    c->h_a.resize(N);
    c->h_b.resize(N);
    CUDA_TRY(cudaMemcpyAsync(c->h_a.data(), c->dt_a.p, sizeof(double) * N, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->h_b.data(), c->dt_b.p, sizeof(double) * N, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    c->a = c->dt_a.p;
    c->b = c->dt_b.p;
    c->nlines = N;
    cache_line_stats(c);
    RC_TRY(ctx_solve_batch(c, doff.data(), q, P, records));
    RC_TRY(c->boffs.need(P + 1));
    RC_TRY(c->bcflags.need(std::max<int64_t>(N, 1)));
    CUDA_TRY(cudaMemcpyAsync(c->boffs.p, doff.data(), sizeof(int64_t) * (P + 1), cudaMemcpyHostToDevice,
                             c->stream));
    lmsb::launch_contacts_batch(c->a, c->b, c->boffs.p, c->best.p, P, c->bcflags.p, c->sms, c->stream);
    CUDA_TRY(cudaGetLastError());
    if (contact_flags)
      CUDA_TRY(cudaMemcpyAsync(contact_flags, c->bcflags.p, (size_t)N, cudaMemcpyDeviceToHost, c->stream));
  }
  if (support_ids) RC_TRY(download_staged(c, support_ids, c->dt_ids.p, sizeof(int32_t) * total));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  c->stats.ms_hough_vote = vote_ms;  // (the fits' solve reset the counters)
  c->stats.ms_hough_support = sup_ms;
  return run_fit || fit == 0 ? LMS_OK : LMS_NOT_FITTED;
}

// H2D of many host pieces concatenated: each 4 MB pinned chunk is filled by
// host threads from the pieces it overlaps (the concatenation and the copy
// into pinned memory are one pass), its DMA overlapping the next chunk.
int upload_gather(lms_ctx* c, void* d_dst, const unsigned char* const* src, const int64_t* bytes,
                  int64_t count) {
  std::vector<int64_t> start(count + 1, 0);
  for (int64_t k = 0; k < count; ++k) start[k + 1] = start[k] + bytes[k];
  const int64_t total = start[count];
  if (total == 0) return LMS_OK;
  RC_TRY(ensure_stage(c));
  bool used[2] = {false, false};
  int slot = 0;
  int64_t first = 0;  // first piece overlapping the chunk
  for (int64_t off = 0; off < total; off += (int64_t)kStageChunk, slot ^= 1) {
    const int64_t len = std::min<int64_t>((int64_t)kStageChunk, total - off);
    unsigned char* buf = c->stage + slot * kStageChunk;
    if (used[slot]) CUDA_TRY(cudaEventSynchronize(c->ev_stage[slot]));
    while (start[first + 1] <= off) ++first;
    int64_t last = first;
    while (last + 1 < count && start[last + 1] < off + len) ++last;
#pragma omp parallel for num_threads(8) schedule(static)
    for (int64_t k = first; k <= last; ++k) {
      const int64_t s0 = std::max(start[k], off), s1 = std::min(start[k + 1], off + len);
      if (s1 > s0) std::memcpy(buf + (s0 - off), src[k] + (s0 - start[k]), (size_t)(s1 - s0));
    }
    CUDA_TRY(cudaMemcpyAsync(static_cast<unsigned char*>(d_dst) + off, buf, (size_t)len,
                             cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(cudaEventRecord(c->ev_stage[slot], c->stream));
    used[slot] = true;
  }
  return LMS_OK;
}

int lms_ndarray_rows_f64(const uintptr_t* objs, int64_t count, const double** data, int64_t* rows) {
  // numpy's PyArrayObject_fields (numpy/ndarraytypes.h): after PyObject_HEAD
  // (refcount, type: 16 bytes) come char* data, int nd, npy_intp* dimensions,
  // npy_intp* strides -- a stable part of numpy's C ABI
  if (count < 0 || (count > 0 && (!objs || !data || !rows))) return set_error(LMS_ERR_INVALID, "null argument");
  for (int64_t k = 0; k < count; ++k) {
    const unsigned char* o = reinterpret_cast<const unsigned char*>(objs[k]);
    const char* d = *reinterpret_cast<const char* const*>(o + 16);
    const int nd = *reinterpret_cast<const int*>(o + 24);
    const int64_t* dims = *reinterpret_cast<const int64_t* const*>(o + 32);
    const int64_t* strides = *reinterpret_cast<const int64_t* const*>(o + 40);
    if (nd != 2 || dims[1] != 2 || (dims[0] > 0 && strides[1] != 8) || (dims[0] > 1 && strides[0] != 16))
      return set_error(LMS_ERR_INVALID, "set %lld is not a C-contiguous (n, 2) float64 array", (long long)k);
    data[k] = reinterpret_cast<const double*>(d);
    rows[k] = dims[0];
  }
  return LMS_OK;
}

int lms_batched_fit_sets_f64(const double* const* sets, const int64_t* counts, const int64_t* q,
                             int64_t nfits, int device, int32_t* status, lms_candidate* out,
                             int64_t* contact_offsets, int32_t* contacts, int64_t contact_capacity,
                             int64_t* ncontacts) {
  if (nfits < 0 || (nfits > 0 && (!sets || !counts || !q || !status || !out || !contact_offsets ||
                                  !ncontacts)))
    return set_error(LMS_ERR_INVALID, "null argument");
  if (nfits == 0) {
    if (contact_offsets) contact_offsets[0] = 0;
    if (ncontacts) *ncontacts = 0;
    return LMS_OK;
  }
  lms_ctx* c = nullptr;
  RC_TRY(shared_ctx(device, &c));
  std::lock_guard<std::mutex> lk(c->mu);
  CUDA_TRY(cudaSetDevice(c->device));
  std::vector<int64_t> offs(nfits + 1, 0), bytes(nfits);
  for (int64_t f = 0; f < nfits; ++f) {
    if (counts[f] < 0 || (counts[f] > 0 && !sets[f])) return set_error(LMS_ERR_INVALID, "bad set %lld", (long long)f);
    offs[f + 1] = offs[f] + counts[f];
    bytes[f] = 16 * counts[f];
  }
  const int64_t N = offs[nfits];
  RC_TRY(c->set_xy.need(2 * std::max<int64_t>(N, 1)));
  RC_TRY(c->a_own.need(std::max<int64_t>(N, 1)));
  RC_TRY(c->b_own.need(std::max<int64_t>(N, 1)));
  RC_TRY(c->boffs.need(nfits + 1));
  RC_TRY(c->set_stats.need(3 * nfits));
  RC_TRY(upload_gather(c, c->set_xy.p, reinterpret_cast<const unsigned char* const*>(sets), bytes.data(),
                       nfits));
  CUDA_TRY(cudaMemcpyAsync(c->boffs.p, offs.data(), sizeof(int64_t) * (nfits + 1),
                           cudaMemcpyHostToDevice, c->stream));
  lmsb::launch_split_xy(c->set_xy.p, N, c->a_own.p, c->b_own.p, c->sms, c->stream);
  lmsb::launch_set_stats(c->a_own.p, c->b_own.p, c->boffs.p, nfits, c->set_stats.p, c->sms, c->stream);
  CUDA_TRY(cudaGetLastError());
  std::vector<double> stv(3 * nfits);
  CUDA_TRY(cudaMemcpyAsync(stv.data(), c->set_stats.p, sizeof(double) * 3 * nfits, cudaMemcpyDeviceToHost,
                           c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  // solve_lms's checks per set (solver.py:67-80): 1 non-finite, 2 fewer than
  // 3 points, 3 one distinct x, 4 q outside [2, n]; the caller raises the
  // first failing set's error
  bool all_ok = true;
  for (int64_t f = 0; f < nfits; ++f) {
    const int64_t n = counts[f];
    int32_t st = 0;
    if (n > 0 && stv[3 * f] == 0.0) st = 1;
    else if (n < 3) st = 2;
    else if (!(stv[3 * f + 1] < stv[3 * f + 2])) st = 3;
    else if (q[f] < 2 || q[f] > n) st = 4;
    status[f] = st;
    all_ok &= st == 0;
  }
  if (!all_ok) return LMS_NOT_FITTED;
  // bind the device lines; the solver's per-fit magnitudes come from a
  // second small reduction instead of a host copy of the lines
  c->a = c->a_own.p;
  c->b = c->b_own.p;
  c->nlines = N;
  c->h_a.clear();
  c->h_b.clear();
  ++c->gen;
  {
    // per-set max |a| = max(|min x|, |max x|); max |b| from y's range: the
    // stats kernel again with the arrays swapped (x's stats are on the host)
    lmsb::launch_set_stats(c->b_own.p, c->a_own.p, c->boffs.p, nfits, c->set_stats.p, c->sms, c->stream);
    std::vector<double> sty(3 * nfits);
    CUDA_TRY(cudaMemcpyAsync(sty.data(), c->set_stats.p, sizeof(double) * 3 * nfits, cudaMemcpyDeviceToHost,
                             c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    c->ext_off.assign(offs.begin(), offs.end() - 1);
    c->ext_st.resize(4 * nfits);
    double alo = INFINITY, ahi = -INFINITY, am = 0.0, bm = 0.0;
    for (int64_t f = 0; f < nfits; ++f) {
      const double lo = stv[3 * f + 1], hi = stv[3 * f + 2];
      const double bmx = std::max(std::fabs(sty[3 * f + 1]), std::fabs(sty[3 * f + 2]));
      c->ext_st[4 * f] = lo;
      c->ext_st[4 * f + 1] = hi;
      c->ext_st[4 * f + 2] = std::max(std::fabs(lo), std::fabs(hi));
      c->ext_st[4 * f + 3] = bmx;
      alo = std::min(alo, lo);
      ahi = std::max(ahi, hi);
      am = std::max(am, c->ext_st[4 * f + 2]);
      bm = std::max(bm, bmx);
    }
    c->s_alo = alo;
    c->s_ahi = ahi;
    c->s_am = am;
    c->s_bm = bm;
  }
  RC_TRY(ctx_solve_batch(c, offs.data(), q, nfits, out));
  RC_TRY(c->bcflags.need(std::max<int64_t>(N, 1)));
  RC_TRY(c->set_cnt.need(nfits));
  RC_TRY(c->set_coff.need(nfits + 1));
  RC_TRY(c->set_contacts.need(std::max<int64_t>(N, 1)));
  CUDA_TRY(cudaMemcpyAsync(c->boffs.p, offs.data(), sizeof(int64_t) * (nfits + 1),
                           cudaMemcpyHostToDevice, c->stream));
  lmsb::launch_contacts_batch(c->a, c->b, c->boffs.p, c->best.p, nfits, c->bcflags.p, c->sms, c->stream);
  lmsb::launch_contact_compact(c->bcflags.p, c->boffs.p, nfits, c->set_cnt.p, c->set_coff.p,
                               c->set_contacts.p, c->sms, c->stream);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(contact_offsets, c->set_coff.p, sizeof(int64_t) * (nfits + 1),
                           cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  const int64_t total = contact_offsets[nfits];
  *ncontacts = total;
  if (total > contact_capacity) return LMS_OK;  // the caller asks again with room (records kept)
  if (total > 0 && contacts)
    CUDA_TRY(cudaMemcpyAsync(contacts, c->set_contacts.p, sizeof(int32_t) * total, cudaMemcpyDeviceToHost,
                             c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return LMS_OK;
}

int lms_ctx_solve_batch(lms_ctx* c, const int64_t* offsets, const int64_t* q, int64_t nfits,
                        lms_candidate* out) {
  if (!c || (nfits > 0 && !out)) return set_error(LMS_ERR_INVALID, "null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  return ctx_solve_batch(c, offsets, q, nfits, out);
}

int lms_ctx_stats(const lms_ctx* c, lms_stats* out) {
  if (!c || !out) return set_error(LMS_ERR_INVALID, "null argument");
  *out = c->stats;
  return LMS_OK;
}

int lms_ctx_event_record(lms_ctx* c, int slot) {
  if (!c || slot < 0 || slot >= kNumEvents) return set_error(LMS_ERR_INVALID, "bad event slot");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaEventRecord(c->user_ev[slot], c->stream));
  return LMS_OK;
}

int lms_ctx_event_elapsed_ms(lms_ctx* c, int slot0, int slot1, float* ms) {
  if (!c || !ms || slot0 < 0 || slot1 < 0 || slot0 >= kNumEvents || slot1 >= kNumEvents)
    return set_error(LMS_ERR_INVALID, "bad event slot");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaEventSynchronize(c->user_ev[slot1]));
  CUDA_TRY(cudaEventElapsedTime(ms, c->user_ev[slot0], c->user_ev[slot1]));
  return LMS_OK;
}

int lms_ctx_synchronize(lms_ctx* c) {
  if (!c) return set_error(LMS_ERR_INVALID, "null context");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return LMS_OK;
}

}  // extern "C"
