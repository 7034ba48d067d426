// lms_engine.cu -- host orchestration of the exact-LMS search and the C ABI.
//
// One solve over pair ranks [R0, R1) (a contiguous partition, as
// BatchPlan.partitions, backend.py:84-92):
//   1. seed     exact-evaluate a stratified sample of S vertices and reduce
//               them to the current best record (its height is the bound H);
//   2. filter   stream the range in chunks of warp tasks through the count
//               filter (lms_filter.cu) with H read from device memory;
//   3. exact    re-evaluate the chunk's survivors bit-exactly (lms_exact.cu);
//   4. reduce   lexicographic (height, i, j) minimum into the best record,
//               tightening H for the next chunk.
// Every launch is asynchronous on the context stream; the host synchronises
// once, when it reads the 56-byte best record back.  Small ranges (fewer
// than kExhaustive pairs) skip the filter and evaluate every vertex exactly.

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "lms_common.cuh"
#include "lms_kernels.cuh"

#define LMS_VERSION 1

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

constexpr int64_t kSeeds = 2048;            // exact seed vertices per solve
constexpr int64_t kExhaustive = 4096;       // ranges this small skip the filter
constexpr int64_t kChunkVertices = 1 << 24; // filter chunk (and survivor capacity)
constexpr int kNumEvents = 16;

// Count-filter variants: all-FP64 (lms_filter.cu), FP16 compare + mma.sync
// counting (lms_filter32.cu), FP16 compare + integer-mask counting
// (lms_filter32m.cu).
constexpr int kFilterFp64 = 1;
constexpr int kFilterMma = 2;
constexpr int kFilterMask = 3;
constexpr int kDefaultFilter = kFilterMask;

template <typename T>
int grow(T** ptr, int64_t* cap, int64_t need) {
  if (need <= *cap) return LMS_OK;
  if (*ptr) cudaFree(*ptr);
  *ptr = nullptr;
  *cap = 0;
  int64_t c = std::max<int64_t>(need, 64);
  CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(ptr), sizeof(T) * c));
  *cap = c;
  return LMS_OK;
}

}  // namespace

struct lms_ctx {
  int device = 0;
  int sms = 148;
  cudaStream_t stream = nullptr;
  cudaEvent_t user_ev[kNumEvents] = {};
  cudaEvent_t ev_begin = nullptr, ev_seed = nullptr, ev_end = nullptr;
  std::vector<cudaEvent_t> ev_chunk;  // filter start / filter end per chunk
  // lines
  double* d_a = nullptr;
  double* d_b = nullptr;
  int64_t cap_a = 0, cap_b = 0;
  const double* a = nullptr;  // bound lines (owned or external)
  const double* b = nullptr;
  int64_t n = 0;
  double amax = 0.0, bmax = 0.0;
  // scratch
  int64_t* d_task_prefix = nullptr;
  int64_t cap_rows = 0;
  int64_t* d_ranks = nullptr;
  int64_t cap_ranks = 0;
  lms_candidate* d_recs = nullptr;
  int64_t cap_recs = 0;
  lms_candidate* d_partials = nullptr;
  int64_t cap_partials = 0;
  lms_candidate* d_best = nullptr;
  unsigned long long* d_counters = nullptr;  // [0] survivors (current chunk), [1] line evals, [2..] per-chunk survivors
  int64_t cap_counters = 0;
  int64_t* d_ii = nullptr;
  int64_t* d_jj = nullptr;
  int64_t cap_ii = 0, cap_jj = 0;
  double* d_uu = nullptr;
  double* d_vv = nullptr;
  int64_t cap_uu = 0, cap_vv = 0;
  lms_candidate* h_best = nullptr;  // pinned
  lms_stats stats{};
  int filter_variant = 0;  // LMSB_FILTER=fp64|mma|mask (A/B switch; see kDefaultFilter)
  bool line_order = true;  // far-first streaming order (LMSB_ORDER=0 disables)
  // far-first order buffers (lms_order.cu)
  float* d_keys = nullptr;
  int64_t cap_keys = 0;
  int* d_idx = nullptr;
  int64_t cap_idx = 0;
  double* d_pa = nullptr;
  double* d_pb = nullptr;
  int64_t cap_pa = 0, cap_pb = 0;
  unsigned char* d_sort_tmp = nullptr;
  int64_t cap_sort_tmp = 0;
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
  const char* fv = getenv("LMSB_FILTER");
  c->filter_variant = kDefaultFilter;
  if (fv && std::strcmp(fv, "fp64") == 0) c->filter_variant = kFilterFp64;
  if (fv && std::strcmp(fv, "mma") == 0) c->filter_variant = kFilterMma;
  if (fv && std::strcmp(fv, "mask") == 0) c->filter_variant = kFilterMask;
  const char* ov = getenv("LMSB_ORDER");
  c->line_order = !(ov && std::strcmp(ov, "0") == 0);
  CUDA_TRY(cudaSetDevice(device));
  CUDA_TRY(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device));
  CUDA_TRY(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  for (auto& e : c->user_ev) CUDA_TRY(cudaEventCreate(&e));
  CUDA_TRY(cudaEventCreate(&c->ev_begin));
  CUDA_TRY(cudaEventCreate(&c->ev_seed));
  CUDA_TRY(cudaEventCreate(&c->ev_end));
  CUDA_TRY(cudaMalloc(&c->d_best, sizeof(lms_candidate)));
  CUDA_TRY(cudaMallocHost(&c->h_best, sizeof(lms_candidate)));
  return LMS_OK;
}

void ctx_release(lms_ctx* c) {
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto& e : c->user_ev)
    if (e) cudaEventDestroy(e);
  for (auto e : c->ev_chunk) cudaEventDestroy(e);
  if (c->ev_begin) cudaEventDestroy(c->ev_begin);
  if (c->ev_seed) cudaEventDestroy(c->ev_seed);
  if (c->ev_end) cudaEventDestroy(c->ev_end);
  cudaFree(c->d_a);
  cudaFree(c->d_b);
  cudaFree(c->d_task_prefix);
  cudaFree(c->d_ranks);
  cudaFree(c->d_recs);
  cudaFree(c->d_partials);
  cudaFree(c->d_best);
  cudaFree(c->d_counters);
  cudaFree(c->d_ii);
  cudaFree(c->d_jj);
  cudaFree(c->d_uu);
  cudaFree(c->d_vv);
  cudaFree(c->d_keys);
  cudaFree(c->d_idx);
  cudaFree(c->d_pa);
  cudaFree(c->d_pb);
  cudaFree(c->d_sort_tmp);
  if (c->h_best) cudaFreeHost(c->h_best);
  if (c->stream) cudaStreamDestroy(c->stream);
}

int ctx_upload(lms_ctx* c, const double* a, const double* b, int64_t n) {
  if (!a || !b || n < 2) return set_error(LMS_ERR_INVALID, "need at least 2 lines, got %lld", (long long)n);
  CUDA_TRY(cudaSetDevice(c->device));
  int rc = grow(&c->d_a, &c->cap_a, n);
  if (rc) return rc;
  rc = grow(&c->d_b, &c->cap_b, n);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(c->d_a, a, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->d_b, b, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  double am = 0.0, bm = 0.0;
  for (int64_t k = 0; k < n; ++k) {
    am = std::max(am, std::fabs(a[k]));
    bm = std::max(bm, std::fabs(b[k]));
  }
  c->a = c->d_a;
  c->b = c->d_b;
  c->n = n;
  c->amax = am;
  c->bmax = bm;
  return LMS_OK;
}

int ensure_counters(lms_ctx* c, int64_t chunks) {
  return grow(&c->d_counters, &c->cap_counters, 2 + chunks);
}

int ensure_partials(lms_ctx* c) {
  return grow(&c->d_partials, &c->cap_partials, (int64_t)c->sms);
}

int exact_grid(const lms_ctx* c, int64_t count) {
  int64_t g = (int64_t)c->sms * 8;
  if (count >= 0) g = std::min<int64_t>(g, std::max<int64_t>(count, 1));
  return (int)g;
}

int ctx_solve(lms_ctx* c, int64_t q, int64_t R0, int64_t R1, lms_candidate* out) {
  std::memset(out, 0, sizeof(*out));
  const int64_t n = c->n;
  if (n < 2 || !c->a) return set_error(LMS_ERR_INVALID, "no lines bound to the context");
  const int64_t total = n * (n - 1) / 2;
  if (q < 1) return set_error(LMS_ERR_INVALID, "coverage must be positive, got %lld", (long long)q);
  if (R0 < 0 || R1 > total || R0 > R1)
    return set_error(LMS_ERR_INVALID, "rank range [%lld, %lld) outside [0, %lld)", (long long)R0,
                     (long long)R1, (long long)total);
  CUDA_TRY(cudaSetDevice(c->device));
  lms_stats st{};
  st.n = n;
  st.pairs = R1 - R0;
  const int64_t span = R1 - R0;
  int rc = ensure_partials(c);
  if (rc) return rc;
  CUDA_TRY(cudaEventRecord(c->ev_begin, c->stream));
  CUDA_TRY(cudaMemsetAsync(c->d_best, 0, sizeof(lms_candidate), c->stream));
  if (span == 0) {
    CUDA_TRY(cudaEventRecord(c->ev_seed, c->stream));
    CUDA_TRY(cudaEventRecord(c->ev_end, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    c->stats = st;
    return LMS_OK;
  }

  // 1. seed (or exhaustive evaluation of a small range)
  const bool exhaustive = span <= kExhaustive;
  const int64_t S = exhaustive ? span : std::min<int64_t>(kSeeds, span);
  rc = grow(&c->d_recs, &c->cap_recs, S);
  if (rc) return rc;
  lmsb::ExactArgs ea{};
  ea.a = c->a;
  ea.b = c->b;
  ea.n = n;
  ea.q = q;
  ea.mode = lmsb::kSrcStrided;
  ea.count = S;
  ea.capacity = S;
  ea.rank_lo = R0;
  ea.rank_hi = R1;
  ea.out = c->d_recs;
  lmsb::launch_exact(ea, exact_grid(c, S), c->stream);
  lmsb::launch_reduce(c->d_recs, nullptr, S, S, c->d_partials, c->sms, c->d_best, c->stream);
  CUDA_TRY(cudaGetLastError());
  st.launches += 3;
  st.seed_vertices = S;
  CUDA_TRY(cudaEventRecord(c->ev_seed, c->stream));

  int64_t nchunks = 0;
  const double* la = c->a;
  const double* lb = c->b;
  if (!exhaustive && c->line_order) {
    // Far-first streaming order from the seed's best line (lms_order.cu).
    const size_t tmp = lmsb::order_temp_bytes(n);
    if ((rc = grow(&c->d_keys, &c->cap_keys, 2 * n))) return rc;
    if ((rc = grow(&c->d_idx, &c->cap_idx, 2 * n))) return rc;
    if ((rc = grow(&c->d_pa, &c->cap_pa, n))) return rc;
    if ((rc = grow(&c->d_pb, &c->cap_pb, n))) return rc;
    if ((rc = grow(&c->d_sort_tmp, &c->cap_sort_tmp, (int64_t)tmp))) return rc;
    lmsb::OrderArgs oa{};
    oa.a = c->a;
    oa.b = c->b;
    oa.n = n;
    oa.best = c->d_best;
    oa.keys_in = c->d_keys;
    oa.keys_out = c->d_keys + n;
    oa.idx_in = c->d_idx;
    oa.idx_out = c->d_idx + n;
    oa.temp = c->d_sort_tmp;
    oa.temp_bytes = (size_t)c->cap_sort_tmp;
    oa.pa = c->d_pa;
    oa.pb = c->d_pb;
    if (lmsb::launch_line_order(oa, c->stream) != 0)
      return set_error(LMS_ERR_CUDA, "line order sort failed");
    CUDA_TRY(cudaGetLastError());
    st.launches += 3;
    la = c->d_pa;
    lb = c->d_pb;
  }
  if (!exhaustive) {
    const int variant = c->filter_variant;
    const int64_t task_vertices = variant == kFilterFp64   ? lmsb::kFilterTaskVertices
                                  : variant == kFilterMask ? lmsb::kFilter32mTaskVertices
                                                           : lmsb::kFilter32TaskVertices;
    // Warp tasks per row of the range.
    int64_t i0, j0, i1, j1;
    lmsb::decode_rank(n, R0, &i0, &j0);
    lmsb::decode_rank(n, R1 - 1, &i1, &j1);
    const int64_t nrows = i1 - i0 + 1;
    std::vector<int64_t> prefix(nrows + 1);
    int64_t acc = 0;
    for (int64_t r = 0; r < nrows; ++r) {
      const int64_t i = i0 + r;
      const int64_t lo = std::max(lmsb::row_offset(n, i), R0);
      const int64_t hi = std::min(lmsb::row_offset(n, i) + (n - 1 - i), R1);
      prefix[r] = acc;
      acc += (hi - lo + task_vertices - 1) / task_vertices;
    }
    prefix[nrows] = acc;
    const int64_t ntasks = acc;
    rc = grow(&c->d_task_prefix, &c->cap_rows, nrows + 1);
    if (rc) return rc;
    CUDA_TRY(cudaMemcpyAsync(c->d_task_prefix, prefix.data(), sizeof(int64_t) * (nrows + 1),
                             cudaMemcpyHostToDevice, c->stream));
    const int64_t chunk_tasks = kChunkVertices / task_vertices;
    nchunks = (ntasks + chunk_tasks - 1) / chunk_tasks;
    const int64_t cap = std::min<int64_t>(kChunkVertices, span);
    rc = grow(&c->d_ranks, &c->cap_ranks, cap);
    if (rc) return rc;
    rc = grow(&c->d_recs, &c->cap_recs, cap);
    if (rc) return rc;
    rc = ensure_counters(c, nchunks);
    if (rc) return rc;
    CUDA_TRY(cudaMemsetAsync(c->d_counters, 0, sizeof(unsigned long long) * (2 + nchunks),
                             c->stream));
    while ((int64_t)c->ev_chunk.size() < 2 * nchunks) {
      cudaEvent_t e;
      CUDA_TRY(cudaEventCreate(&e));
      c->ev_chunk.push_back(e);
    }
    for (int64_t ch = 0; ch < nchunks; ++ch) {
      lmsb::FilterArgs fa{};
      fa.a = c->a;
      fa.b = c->b;
      fa.la = la;
      fa.lb = lb;
      fa.n = n;
      fa.q = q;
      fa.task_prefix = c->d_task_prefix;
      fa.row0 = i0;
      fa.nrows = nrows;
      fa.rank_lo = R0;
      fa.rank_hi = R1;
      fa.task_begin = ch * chunk_tasks;
      fa.task_end = std::min(ntasks, (ch + 1) * chunk_tasks);
      fa.amax = c->amax;
      fa.bmax = c->bmax;
      fa.best = c->d_best;
      fa.out_ranks = c->d_ranks;
      fa.out_count = c->d_counters + 2 + ch;
      fa.line_evals = c->d_counters + 1;
      fa.early_exit = 1;
      CUDA_TRY(cudaEventRecord(c->ev_chunk[2 * ch], c->stream));
      if (variant == kFilterFp64) lmsb::launch_filter(fa, c->stream);
      else if (variant == kFilterMask) lmsb::launch_filter32m(fa, c->stream);
      else lmsb::launch_filter32(fa, c->stream);
      CUDA_TRY(cudaEventRecord(c->ev_chunk[2 * ch + 1], c->stream));
      lmsb::ExactArgs xa = ea;
      xa.mode = lmsb::kSrcRanks;
      xa.count = -1;
      xa.d_count = c->d_counters + 2 + ch;
      xa.capacity = cap;
      xa.ranks = c->d_ranks;
      xa.bound = c->d_best;
      xa.out = c->d_recs;
      lmsb::launch_exact(xa, exact_grid(c, -1), c->stream);
      lmsb::launch_reduce(c->d_recs, c->d_counters + 2 + ch, 0, cap, c->d_partials, c->sms,
                          c->d_best, c->stream);
      CUDA_TRY(cudaGetLastError());
      st.launches += 4;
      st.filtered_vertices += (fa.task_end - fa.task_begin) * task_vertices;
    }
    st.filtered_vertices = std::min(st.filtered_vertices, span);
  }
  CUDA_TRY(cudaMemcpyAsync(c->h_best, c->d_best, sizeof(lms_candidate), cudaMemcpyDeviceToHost,
                           c->stream));
  CUDA_TRY(cudaEventRecord(c->ev_end, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  *out = *c->h_best;
  st.chunks = nchunks;
  if (nchunks > 0) {
    std::vector<unsigned long long> cnt(2 + nchunks);
    CUDA_TRY(cudaMemcpy(cnt.data(), c->d_counters, sizeof(unsigned long long) * (2 + nchunks),
                        cudaMemcpyDeviceToHost));
    st.line_evals = (int64_t)cnt[1];
    for (int64_t ch = 0; ch < nchunks; ++ch) {
      st.survivors += (int64_t)cnt[2 + ch];
      float ms = 0.f;
      CUDA_TRY(cudaEventElapsedTime(&ms, c->ev_chunk[2 * ch], c->ev_chunk[2 * ch + 1]));
      st.ms_filter += ms;
    }
  }
  CUDA_TRY(cudaEventElapsedTime(&st.ms_total, c->ev_begin, c->ev_end));
  st.ms_exact = st.ms_total - st.ms_filter;
  c->stats = st;
  return LMS_OK;
}

int ctx_eval_explicit(lms_ctx* c, int64_t q, const int64_t* i, const int64_t* j, const double* u,
                      const double* v, int64_t m, lms_candidate* out, bool reduce) {
  if (m < 0) return set_error(LMS_ERR_INVALID, "negative vertex count");
  if (q < 1) return set_error(LMS_ERR_INVALID, "coverage must be positive, got %lld", (long long)q);
  const int64_t n = c->n;
  for (int64_t s = 0; s < m; ++s) {
    if (i[s] < 0 || i[s] >= n || j[s] < 0 || j[s] >= n)
      return set_error(LMS_ERR_INVALID, "vertex %lld has line index out of range", (long long)s);
  }
  if (m == 0) {
    if (reduce) std::memset(out, 0, sizeof(*out));
    return LMS_OK;
  }
  CUDA_TRY(cudaSetDevice(c->device));
  int rc = grow(&c->d_ii, &c->cap_ii, m);
  if (rc) return rc;
  rc = grow(&c->d_jj, &c->cap_jj, m);
  if (rc) return rc;
  rc = grow(&c->d_uu, &c->cap_uu, m);
  if (rc) return rc;
  rc = grow(&c->d_vv, &c->cap_vv, m);
  if (rc) return rc;
  rc = grow(&c->d_recs, &c->cap_recs, m);
  if (rc) return rc;
  rc = ensure_partials(c);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(c->d_ii, i, sizeof(int64_t) * m, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->d_jj, j, sizeof(int64_t) * m, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->d_uu, u, sizeof(double) * m, cudaMemcpyHostToDevice, c->stream));
  if (v) CUDA_TRY(cudaMemcpyAsync(c->d_vv, v, sizeof(double) * m, cudaMemcpyHostToDevice, c->stream));
  lmsb::ExactArgs ea{};
  ea.a = c->a;
  ea.b = c->b;
  ea.n = n;
  ea.q = q;
  ea.mode = lmsb::kSrcExplicit;
  ea.count = m;
  ea.capacity = m;
  ea.ii = c->d_ii;
  ea.jj = c->d_jj;
  ea.uu = c->d_uu;
  ea.vv = v ? c->d_vv : nullptr;
  ea.out = c->d_recs;
  lmsb::launch_exact(ea, exact_grid(c, m), c->stream);
  if (reduce) {
    CUDA_TRY(cudaMemsetAsync(c->d_best, 0, sizeof(lms_candidate), c->stream));
    lmsb::launch_reduce(c->d_recs, nullptr, m, m, c->d_partials, c->sms, c->d_best, c->stream);
    CUDA_TRY(cudaMemcpyAsync(out, c->d_best, sizeof(lms_candidate), cudaMemcpyDeviceToHost,
                             c->stream));
  } else {
    CUDA_TRY(cudaMemcpyAsync(out, c->d_recs, sizeof(lms_candidate) * m, cudaMemcpyDeviceToHost,
                             c->stream));
  }
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(c->stream));
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
  int rc = shared_ctx(device, &c);
  if (rc) return rc;
  std::lock_guard<std::mutex> lk(c->mu);
  rc = ctx_upload(c, a, b, n);
  if (rc) return rc;
  return ctx_solve(c, q, rank_begin, rank_end, out);
}

int lms_eval_vertices_f64(const double* a, const double* b, int64_t n, int64_t q, const int64_t* i,
                          const int64_t* j, const double* u, const double* v, int64_t m, int device,
                          lms_candidate* out) {
  if (!out || (m > 0 && (!i || !j || !u))) return set_error(LMS_ERR_INVALID, "null argument");
  lms_ctx* c = nullptr;
  int rc = shared_ctx(device, &c);
  if (rc) return rc;
  std::lock_guard<std::mutex> lk(c->mu);
  rc = ctx_upload(c, a, b, n);
  if (rc) return rc;
  return ctx_eval_explicit(c, q, i, j, u, v, m, out, false);
}

int lms_min_over_vertices_f64(const double* a, const double* b, int64_t n, int64_t q,
                              const int64_t* i, const int64_t* j, const double* u, int64_t m,
                              int device, lms_candidate* out) {
  if (!out || (m > 0 && (!i || !j || !u))) return set_error(LMS_ERR_INVALID, "null argument");
  lms_ctx* c = nullptr;
  int rc = shared_ctx(device, &c);
  if (rc) return rc;
  std::lock_guard<std::mutex> lk(c->mu);
  rc = ctx_upload(c, a, b, n);
  if (rc) return rc;
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
  if (!c || !d_a || !d_b || n < 2) return set_error(LMS_ERR_INVALID, "bad arguments");
  std::lock_guard<std::mutex> lk(c->mu);
  CUDA_TRY(cudaSetDevice(c->device));
  std::vector<double> ha(n), hb(n);
  CUDA_TRY(cudaMemcpy(ha.data(), d_a, sizeof(double) * n, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(hb.data(), d_b, sizeof(double) * n, cudaMemcpyDeviceToHost));
  double am = 0.0, bm = 0.0;
  for (int64_t k = 0; k < n; ++k) {
    am = std::max(am, std::fabs(ha[k]));
    bm = std::max(bm, std::fabs(hb[k]));
  }
  c->a = d_a;
  c->b = d_b;
  c->n = n;
  c->amax = am;
  c->bmax = bm;
  return LMS_OK;
}

int lms_ctx_solve(lms_ctx* c, int64_t q, int64_t rank_begin, int64_t rank_end,
                  lms_candidate* out) {
  if (!c || !out) return set_error(LMS_ERR_INVALID, "null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  return ctx_solve(c, q, rank_begin, rank_end, out);
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
