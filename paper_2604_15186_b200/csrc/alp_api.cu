// Host side of the C ABI declared in include/alp.h: validation, the static search plan (sort
// list, u-sorted b columns), per-search launch geometry, and the kernel launches.  All ALP
// arithmetic of the search path (option terms, objective sums, mins, counts, FP64 winner
// prediction) runs in the kernels (alp_kernels.cu, alp_search.cuh with alp_terms.cuh and
// alp_finalize.cuh); for the search this file only moves integers and pointers.  The two steps
// around the path, alp_workflow_stats (before alp_build) and alp_place (after the search), are
// small host computations here.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "alp_internal.h"
#include "nvtx3/nvToolsExt.h"  // header-only NVTX v3: ranges for nsys timelines (no-ops without a tool)

using namespace alp;

namespace {

thread_local std::string g_err = "no error";

// NVTX range for the duration of a scope (alp_build / search / finalize phases in nsys)
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
constexpr size_t kPinnedStageMax = 256 * 1024;  // larger arena uploads skip the pinned staging buffer
constexpr size_t kArenaWork = 64;  // work counters kept in the handle arena (phases of one search)
// fused-launch work counters: <= kInlineTargets targets x <= 16 b-chunks (b columns are split in
// chunks of >= 64 and K <= 1024)
constexpr size_t kFusedWork = (size_t)kInlineTargets * 16;

// Small pinned host buffer per host thread (allocated once, shared by all handles the thread uses)
// for the per-search H2D of targets and D2H of results: pageable copies cost a staging hop each.
// Two fixed halves: [0, 32 KB) feeds target H2D copies, [32 KB, 64 KB) receives result D2H copies
// (or, for the fused search, the kernel's own zero-copy result stores).
constexpr size_t kPinHalf = 32 * 1024;
void *pinned_scratch(size_t bytes) {
  struct Buf {
    void *p = nullptr;
    size_t n = 0;
    ~Buf() {
      if (p) cudaFreeHost(p);
    }
  };
  static thread_local Buf b;
  if (bytes > b.n) {
    if (b.p) cudaFreeHost(b.p);
    b.p = nullptr;
    b.n = 0;
    const size_t want = std::max<size_t>(bytes, 2 * kPinHalf);
    // mapped: the fused search kernel writes its results straight into the upper half (zero-copy)
    if (cudaHostAlloc(&b.p, want, cudaHostAllocPortable | cudaHostAllocMapped) != cudaSuccess) {
      b.p = nullptr;
      return nullptr;
    }
    b.n = want;
  }
  return b.p;
}

alp_status fail(alp_status st, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

#define CU(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) return fail(ALP_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

template <class T>
struct DBuf {
  T *p = nullptr;
  size_t n = 0;
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  cudaError_t ensure(size_t count) {
    if (count <= n && p) return cudaSuccess;
    release();
    n = count ? count : 1;
    return cudaMalloc(&p, n * sizeof(T));
  }
};

// One device allocation for every table a handle owns: the host stages the copied sections into
// one buffer (one cudaMalloc + one cudaMemcpy per alp_build); scratch sections follow, uncopied.
struct Arena {
  std::vector<unsigned char> host;
  size_t copied = 0, total = 0;
  std::vector<std::pair<size_t, void **>> fix;
  static size_t align(size_t x) { return (x + 255) & ~size_t(255); }
  template <class T>
  void add(const std::vector<T> &v, T **dptr) {
    const size_t off = align(total);
    total = off + v.size() * sizeof(T);
    host.resize(total);
    if (!v.empty()) memcpy(host.data() + off, v.data(), v.size() * sizeof(T));
    copied = total;
    fix.push_back({off, reinterpret_cast<void **>(dptr)});
  }
  // a trailing region of `bytes` whose first `zeros` bytes are uploaded as zeros (must come last)
  void region(size_t bytes, size_t zeros, unsigned char **dptr) {
    const size_t off = align(total);
    host.resize(off + zeros, 0);
    copied = off + zeros;
    total = off + bytes;
    fix.push_back({off, reinterpret_cast<void **>(dptr)});
  }
  template <class T>
  void scratch(size_t count, T **dptr) {
    const size_t off = align(total);
    total = off + count * sizeof(T);
    fix.push_back({off, reinterpret_cast<void **>(dptr)});
  }
  // H2D through a process-wide pinned staging buffer (one cudaMemcpyAsync, stream-ordered on `st`).
  cudaError_t commit(void **base, uint64_t &h2d, cudaStream_t st) {
    static std::mutex mu;
    static void *pinned = nullptr;
    static size_t pinned_bytes = 0;
    // stream-ordered allocation from the device's default memory pool (kept warm across handles)
    cudaError_t e = cudaMallocAsync(base, total ? total : 1, st);
    if (e != cudaSuccess) return e;
    if (copied > kPinnedStageMax) {
      // large, rare uploads (static plans): a pageable copy beats growing the pinned staging
      // buffer (page-locking megabytes costs more than the copy); the call returns once the
      // driver has staged the source, the DMA is ordered on st
      e = cudaMemcpyAsync(*base, host.data(), copied, cudaMemcpyHostToDevice, st);
    } else if (copied) {
      std::lock_guard<std::mutex> lock(mu);
      if (pinned_bytes < copied) {
        if (pinned) cudaFreeHost(pinned);
        pinned_bytes = std::max(copied, pinned_bytes * 2);
        e = cudaHostAlloc(&pinned, pinned_bytes, cudaHostAllocDefault);
        if (e != cudaSuccess) {
          pinned = nullptr;
          pinned_bytes = 0;
          return e;
        }
      }
      // the staging buffer may still feed a previous (async) upload on any device: wait for those
      // copies only.  One event per device (an event can only be recorded on a stream of the
      // device it was created on).
      static cudaEvent_t staged[kMaxDevices] = {};
      int dev = 0;
      e = cudaGetDevice(&dev);
      if (e != cudaSuccess) return e;
      if (dev >= kMaxDevices) return cudaErrorInvalidDevice;
      for (cudaEvent_t ev : staged)
        if (ev && (e = cudaEventSynchronize(ev)) != cudaSuccess) return e;
      if (!staged[dev] && (e = cudaEventCreateWithFlags(&staged[dev], cudaEventDisableTiming)) != cudaSuccess) return e;
      memcpy(pinned, host.data(), copied);
      e = cudaMemcpyAsync(*base, pinned, copied, cudaMemcpyHostToDevice, st);
      if (e == cudaSuccess) e = cudaEventRecord(staged[dev], st);
    }
    h2d += copied;
    for (auto &f : fix) *f.second = static_cast<unsigned char *>(*base) + f.first;
    return e;
  }
};

// ALP_TRACE=1 prints host-side phase times of alp_build (tracing aid for the e2e path).
struct Trace {
  bool on = getenv("ALP_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  void mark(const char *what) {
    if (!on) return;
    const auto t1 = std::chrono::steady_clock::now();
    fprintf(stderr, "[alp] %-12s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  }
};

// FastDiv (alp_internal.h): p = 31 + ceil(log2 d), mul = ceil(2^p / d), shift = p - 32; exact for n < 2^31
FastDiv make_fastdiv(uint32_t d) {
  FastDiv f{0u, 0u};
  if (d <= 1) return f;
  int s = 0;
  while ((1ull << s) < d) ++s;
  const int p = 31 + s;
  f.mul = (uint32_t)(((1ull << p) + d - 1) / d);
  f.shift = (uint32_t)(p - 32);
  return f;
}


}  // namespace

// Stream + events of a handle, pooled process-wide per device: alp_build / alp_destroy are on the
// end-to-end path, and creating a stream and six events costs more than the whole build otherwise.
struct StreamCtx {
  int device = -1;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, evs0 = nullptr, evs1 = nullptr;  // timing events
  cudaEvent_t ready = nullptr, last = nullptr;                              // ordering only
};
std::mutex g_ctx_mu;
std::vector<StreamCtx> g_ctx_pool;

cudaError_t ctx_acquire(int device, StreamCtx &c) {
  {
    std::lock_guard<std::mutex> lock(g_ctx_mu);
    for (size_t i = 0; i < g_ctx_pool.size(); ++i)
      if (g_ctx_pool[i].device == device) {
        c = g_ctx_pool[i];
        g_ctx_pool.erase(g_ctx_pool.begin() + i);
        return cudaSuccess;
      }
  }
  c.device = device;
  cudaError_t e = cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking);
  for (cudaEvent_t *ev : {&c.ev0, &c.ev1, &c.evs0, &c.evs1})
    if (e == cudaSuccess) e = cudaEventCreate(ev);
  for (cudaEvent_t *ev : {&c.ready, &c.last})
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
  return e;
}

void ctx_release(const StreamCtx &c) {
  if (!c.stream) return;
  std::lock_guard<std::mutex> lock(g_ctx_mu);
  g_ctx_pool.push_back(c);
}

// Per-search scratch: the option tables of the searched targets, the (key, count) accumulators, the
// work counters and the finalize inputs/outputs of one search.  It is either the handle's own (one
// target: inside the handle's arena; more: a grown buffer) or a caller workspace (alp_search_shard /
// alp_finalize with d_workspace, sized by alp_workspace_bytes).  Layout (ws_layout): a fixed-size
// section that the kernels leave zero after every call (fused accumulators: complemented keys,
// counts, work counters, ticket), then the per-target tables.
struct Scratch {
  unsigned long long *fzkeys = nullptr, *fzcounts = nullptr, *fzwork = nullptr;  // zero at rest
  unsigned *fzticket = nullptr;                                                 // zero at rest
  unsigned long long *fbest = nullptr;  // [n] finalize combine (zeroed by every search launch)
  unsigned *fdone = nullptr;            // [n]
  double *targets = nullptr, *term = nullptr, *b = nullptr;
  float *tau = nullptr;
  alp_result *res = nullptr;
  unsigned long long *keys = nullptr, *counts = nullptr, *work = nullptr;
  int *qb = nullptr;
  int cap = 0;        // targets the tables hold
  bool ws = false;    // a caller workspace (no cross-stream ordering through the handle)
};

// Device copy of a static search plan (sort-list tiles, u-sorted b columns, units).  The plan depends
// only on the grids (units table), rows per lane and the device, so handles with the same key share it.
struct PlanDev {
  void *mem = nullptr;
  int device = 0;
  ~PlanDev() {
    if (mem) {
      cudaSetDevice(device);
      cudaFree(mem);
    }
  }
};

struct alp_s {
  // problem
  int M = 0, F = 1, nS = 0, nT = 0, nR = 0, K = 0;
  bool from_terms = false;
  std::vector<double> n, p, rate, lat, tmax;
  std::vector<int> S, T, R, prof_off, min_units;
  std::vector<int> meas_off;               // measured per-share curves (R2), empty = none
  std::vector<double> mrate, mlat, mtmax;
  std::vector<int> u;  // [M*K] units s*t*d (integer grid product)
  std::vector<float> tau_fixed;
  std::vector<double> term_fixed, b_fixed;
  uint64_t N = 0;
  // static plan
  int a_llm = -1, b_llm = 0, Ka = 1, Kb = 1, g0 = 0, g1 = 0, ng = 0;
  uint32_t L = 1, n_chunks = 1, n_groups = 1, nQ = 1, A = 1;
  uint32_t pw[ALP_MAX_M] = {0};
  std::vector<int> tile_s, bperm, bu, dv, dcnt;
  // per warp group: the unit sum shared by its 32 lane tiles (uniform groups [0, n_groups_u)), or
  // the smallest tile sum of a mixed group (all its lanes are over budget when that one is)
  std::vector<int> gsum;
  uint32_t n_groups_u = 0;
  std::vector<uint32_t> tile_e;
  int rows_per_lane = 8;
  int nq_force = 0;    // ALP_NQ: a-ranges per row (tuning), 0 = automatic
  int min_blocks = 0;  // 0: per rows-per-lane default (T = 8: 3 blocks/SM, T = 16: 2); ALP_BLOCKS_PER_SM overrides
  int umax_a = 0, umax_b = 0;
  long long umax_total = 0;
  // device
  int device = 0, sm_count = 148;
  std::shared_ptr<PlanDev> plan_dev;  // shared static plan tables
  void *d_arena = nullptr;  // every static table + single-target scratch (one allocation)
  double *d_n = nullptr, *d_p = nullptr, *d_rate = nullptr, *d_lat = nullptr, *d_tmax = nullptr;
  int *d_S = nullptr, *d_T = nullptr, *d_R = nullptr, *d_off = nullptr, *d_minu = nullptr, *d_u = nullptr;
  int *d_moff = nullptr;
  double *d_mrate = nullptr, *d_mlat = nullptr, *d_mtmax = nullptr;
  int *d_tile_s = nullptr, *d_bperm = nullptr, *d_dv = nullptr, *d_dcnt = nullptr, *d_gsum = nullptr;
  uint32_t *d_tile_e = nullptr, *d_tile_off = nullptr;
  float *d_tau_fixed = nullptr;
  double *d_term_fixed = nullptr, *d_b_fixed = nullptr;
  // per-search scratch (Scratch / ws_layout): own1 = one target, inside the arena; g_ws = the
  // handle's own for more targets (capacity g_ws_cap); sc = the scratch of the current call
  Scratch own1, sc;
  DBuf<unsigned char> g_ws;
  int g_ws_cap = 0;
  DBuf<unsigned long long> g_dbg;
  DBuf<unsigned char> g_lv;  // one-pass budget sweep scratch (levels, level keys, histograms)
  cudaEvent_t evs0 = nullptr, evs1 = nullptr;  // step events: search start .. result D2H enqueued
  float last_step_ms = 0.f;
  int *s_qb = nullptr;  // per-query budgets (device) when the current search uses them, else nullptr
  DBuf<int> d_opts, d_pfeas;
  DBuf<double> d_plat, d_pthr;
  DBuf<long long> d_punits;
  StreamCtx ctx;                      // pooled stream + events (see ctx_acquire)
  cudaStream_t stream = nullptr;      // == ctx.stream
  cudaStream_t last_stream = nullptr; // last stream a search/finalize ran on (for alp_destroy)
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  bool ev_pending = false;
  float last_ms = 0.f;
  int last_launches = 0;
  bool last_ur = false;
  bool ws_used = false;  // a call ran on a caller workspace (its stream is not tracked: destroy syncs)  // the last search ran the uniform-register pair (k_uprep + k_search_u)
  uint64_t h2d = 0;
  SearchArgs last_args{};
  std::map<long long, int> occ_cache;  // (smem bytes, b width, T, MB) -> resident blocks per SM

  DevProfiles dprof() const {
    DevProfiles d;
    d.M = M; d.F = F; d.nS = nS; d.nT = nT; d.nR = nR; d.K = K;
    d.n = d_n; d.p = d_p; d.S = d_S; d.T = d_T; d.R = d_R; d.prof_off = d_off;
    d.rate = d_rate; d.lat = d_lat; d.tmax = d_tmax;
    d.min_units = min_units.empty() ? nullptr : d_minu;
    d.meas_off = meas_off.empty() ? nullptr : d_moff;
    d.mrate = d_mrate; d.mlat = d_mlat; d.mtmax = d_mtmax;
    d.n_mpts = (int)mrate.size();
    d.n_pts = (int)rate.size();
    return d;
  }

  ~alp_s() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (ctx.stream && cur != device) cudaSetDevice(device);
    for (auto *b : {&d_plat, &d_pthr}) b->release();
    for (auto *b : {&d_opts, &d_pfeas}) b->release();
    g_ws.release();
    g_dbg.release();
    g_lv.release();
    d_punits.release();
    // stream-ordered release: after the last work on the handle's stream and on the last caller
    // stream (alp_search_shard may run on a caller's stream), without a host synchronisation
    if (ws_used) cudaDeviceSynchronize();  // workspace calls may still run on untracked streams
    if (stream && last_stream && last_stream != stream) {
      cudaEventRecord(ctx.last, last_stream);
      cudaStreamWaitEvent(stream, ctx.last, 0);
    }
    if (d_arena) cudaFreeAsync(d_arena, stream);
    ctx_release(ctx);
    if (cur >= 0 && cur != device) cudaSetDevice(cur);
  }
};

namespace {

// ---------------------------------------------------------------- static plan (build time)
alp_status make_plan(alp_s *h) {
  const int M = h->M, K = h->K;
  h->N = 1;
  for (int m = 0; m < M; ++m) {
    if (h->N > (1ull << 62) / (uint64_t)K) return fail(ALP_EINVAL, "K^M exceeds 2^62 candidates (K=%d, M=%d)", K, M);
    h->N *= (uint64_t)K;
  }
  h->b_llm = M - 1;
  h->a_llm = M >= 2 ? M - 2 : -1;
  h->Kb = K;
  h->Ka = h->a_llm >= 0 ? K : 1;
  h->g1 = h->a_llm >= 0 ? h->a_llm : 0;
  int ng = 0;
  uint64_t L = 1;
  while (ng < std::min(4, h->g1) && L * (uint64_t)K <= (1ull << 18)) {
    ++ng;
    L *= (uint64_t)K;
  }
  h->ng = ng;
  h->g0 = h->g1 - ng;
  h->L = (uint32_t)L;
  uint64_t chunks = 1;
  for (int m = 0; m < h->g0; ++m) {
    chunks *= (uint64_t)K;
    if (chunks >= (1ull << 32)) return fail(ALP_EINVAL, "too many prefix chunks (K=%d, M=%d)", K, M);
  }
  h->n_chunks = (uint32_t)chunks;
  for (int m = 0; m < ALP_MAX_M; ++m) h->pw[m] = 0;
  for (int m = 0; m < h->g0; ++m) {
    uint32_t p = 1;
    for (int j = m + 1; j < h->g0; ++j) p *= (uint32_t)K;
    h->pw[m] = p;
  }
  auto U = [&](int m, int k) { return h->u[(size_t)m * K + k]; };
  // sort list: entries of the sort group ordered by unit sum (stable in canonical order), padded
  // so every lane tile holds T entries of one unit sum.
  // unit sum of every entry, built digit by digit (entry e = sum_j d_j K^(ng-1-j))
  // (odometer over the ng digits, last digit fastest: no divisions)
  std::vector<int> sum(L, 0);
  {
    int dg[4] = {0, 0, 0, 0}, cur = 0;
    for (int j = 0; j < ng; ++j) cur += U(h->g0 + j, 0);
    for (uint32_t e = 0; e < L; ++e) {
      sum[e] = cur;
      for (int j = ng - 1; j >= 0; --j) {
        cur -= U(h->g0 + j, dg[j]);
        if (++dg[j] < K) {
          cur += U(h->g0 + j, dg[j]);
          break;
        }
        dg[j] = 0;
        cur += U(h->g0 + j, 0);
      }
    }
  }
  int smax = 0;
  for (uint32_t e = 0; e < L; ++e) smax = std::max(smax, sum[e]);
  // stable counting sort by unit sum, written straight into the final tile layout: per sum s its
  // entries fill ceil(c_s / T) lane tiles (T rows, the last one padded with kDummy rows); the first
  // whole multiple of 32 of them go to the uniform warp groups (all sums in order), the leftover
  // tiles of every sum after them (mixed groups), padded to a multiple of 32 tiles
  const int T = h->rows_per_lane;
  std::vector<uint32_t> cnt(smax + 1, 0);
  for (uint32_t e = 0; e < L; ++e) ++cnt[sum[e]];
  std::vector<uint64_t> full(smax + 1), uoff(smax + 1), roff(smax + 1);
  uint64_t nfull = 0, nrest = 0;
  for (int v = 0; v <= smax; ++v) {
    const uint64_t tiles = (cnt[v] + T - 1) / T;
    full[v] = tiles / kWarpTiles * kWarpTiles;
    uoff[v] = nfull;
    nfull += full[v];
  }
  for (int v = 0; v <= smax; ++v) {
    const uint64_t tiles = (cnt[v] + T - 1) / T;
    roff[v] = nfull + nrest;
    nrest += tiles - full[v];
  }
  const uint64_t ntiles = (nfull + nrest + kWarpTiles - 1) / kWarpTiles * kWarpTiles;
  h->tile_s.assign(ntiles, 0);
  h->tile_e.assign(ntiles * T, kDummy);
  // per sum: its next slot (tile, row) — no divisions in the pass over the entries
  std::vector<uint64_t> nt(smax + 1), ntile(smax + 1);
  std::vector<int> nrow(smax + 1, 0);
  for (int v = 0; v <= smax; ++v) {
    nt[v] = 0;
    ntile[v] = full[v] > 0 ? uoff[v] : roff[v];
  }
  uint32_t *te = h->tile_e.data();
  int *tsum = h->tile_s.data();
  for (uint32_t e = 0; e < L; ++e) {
    const int v = sum[e];
    const uint64_t tile = ntile[v];
    te[tile * T + nrow[v]] = e;  // canonical within-group index (LLM g0 most significant)
    tsum[tile] = v;
    if (++nrow[v] == T) {
      nrow[v] = 0;
      ++nt[v];
      ntile[v] = nt[v] < full[v] ? uoff[v] + nt[v] : roff[v] + (nt[v] - full[v]);
    }
  }
  for (uint64_t t = nfull + nrest; t < ntiles; ++t) h->tile_s[t] = h->tile_s[nfull + nrest - 1];  // padding tiles
  h->n_groups_u = (uint32_t)(nfull / kWarpTiles);
  h->gsum.resize(ntiles / kWarpTiles);
  for (uint64_t g = 0; g < ntiles / kWarpTiles; ++g)  // uniform: the group's sum; mixed: its smallest tile sum
    h->gsum[g] = *std::min_element(h->tile_s.begin() + g * kWarpTiles, h->tile_s.begin() + (g + 1) * kWarpTiles);
  h->n_groups = (uint32_t)(h->tile_s.size() / kWarpTiles);
  // (the four shared-memory byte offsets of each row's sort-group terms, tile_off, are expanded from
  // tile_e on the device after the upload: launch_plan_offsets)
  // b columns sorted by units (stable): the feasible set for a remaining budget is a prefix.
  h->bperm.resize(K);
  std::iota(h->bperm.begin(), h->bperm.end(), 0);
  std::stable_sort(h->bperm.begin(), h->bperm.end(), [&](int a, int b) { return U(h->b_llm, a) < U(h->b_llm, b); });
  h->bu.resize(K);
  for (int j = 0; j < K; ++j) h->bu[j] = U(h->b_llm, h->bperm[j]);
  h->dv.clear();
  for (int j = 0; j < K; ++j)
    if (h->dv.empty() || h->dv.back() != h->bu[j]) h->dv.push_back(h->bu[j]);
  h->dcnt.assign(h->dv.size() + 1, 0);
  for (size_t i = 1; i <= h->dv.size(); ++i)
    h->dcnt[i] = (int)(std::upper_bound(h->bu.begin(), h->bu.end(), h->dv[i - 1]) - h->bu.begin());
  h->umax_b = h->bu.back();
  h->umax_a = 0;
  if (h->a_llm >= 0)
    for (int k = 0; k < K; ++k) h->umax_a = std::max(h->umax_a, U(h->a_llm, k));
  h->umax_total = 0;
  for (int m = 0; m < M; ++m) {
    int mx = 0;
    for (int k = 0; k < K; ++k) mx = std::max(mx, U(m, k));
    h->umax_total += mx;
  }
  // a-ranges: enough equal-cost work items for ~24 items per resident warp (load balance); a warp
  // keeps its lane tile across consecutive a-ranges, so small ranges cost little.
  const uint64_t want = (uint64_t)h->sm_count * 24 * 24;
  uint32_t nQ = 1;
  while ((uint64_t)h->n_chunks * h->n_groups * nQ < want && nQ < (uint32_t)h->Ka) ++nQ;
  if (h->nq_force > 0) nQ = (uint32_t)std::min(h->nq_force, h->Ka);  // ALP_NQ (tuning)
  h->A = (uint32_t)((h->Ka + nQ - 1) / nQ);
  h->nQ = (uint32_t)((h->Ka + h->A - 1) / h->A);
  while ((uint64_t)h->n_chunks * h->L * h->nQ >= (1ull << 32)) {
    if (h->nQ == 1) return fail(ALP_EINVAL, "problem too large: > 2^32 segments");
    h->A *= 2;
    h->nQ = (uint32_t)((h->Ka + h->A - 1) / h->A);
  }
  return ALP_OK;
}

// Snapshot of a built plan (everything make_plan produces that the searches need).
struct PlanSnap {
  uint64_t N;
  int a_llm, b_llm, Ka, Kb, g0, g1, ng, umax_a, umax_b;
  uint32_t L, n_chunks, n_groups, nQ, A;
  uint32_t pw[ALP_MAX_M];
  long long umax_total;
  std::vector<int> dv, dcnt, gsum;
  uint32_t n_groups_u;
  int *d_u, *d_tile_s, *d_bperm, *d_dv, *d_dcnt, *d_gsum;
  uint32_t *d_tile_e, *d_tile_off;
  std::shared_ptr<PlanDev> dev;
};

std::mutex g_plan_mu;
std::map<std::string, std::shared_ptr<PlanSnap>> g_plans;

std::string plan_key(const alp_s *h) {
  std::string k;
  auto put = [&](const void *p, size_t n) { k.append(static_cast<const char *>(p), n); };
  const int hdr[6] = {h->device, h->sm_count, h->M, h->K, h->rows_per_lane, h->nq_force};
  put(hdr, sizeof(hdr));
  put(h->u.data(), h->u.size() * sizeof(int));
  return k;
}

alp_status make_plan(alp_s *h);

// Build (or fetch from the process-wide cache) the static plan and its device tables.
alp_status get_plan(alp_s *h) {
  Trace tr;
  const std::string key = plan_key(h);
  std::lock_guard<std::mutex> lock(g_plan_mu);
  auto it = g_plans.find(key);
  std::shared_ptr<PlanSnap> P;
  if (it != g_plans.end()) {
    P = it->second;
  } else {
    alp_status s = make_plan(h);
    if (s != ALP_OK) return s;
    P = std::make_shared<PlanSnap>();
    P->dev = std::make_shared<PlanDev>();
    P->dev->device = h->device;
    Arena A;
    A.add(h->u, &P->d_u);
    A.add(h->tile_s, &P->d_tile_s);
    A.add(h->tile_e, &P->d_tile_e);
    A.add(h->bperm, &P->d_bperm);
    A.add(h->dv, &P->d_dv);
    A.add(h->dcnt, &P->d_dcnt);
    A.add(h->gsum, &P->d_gsum);
    A.scratch(h->tile_e.size() * 4, &P->d_tile_off);  // not uploaded: expanded on the device
    tr.mark("make_plan");
    CU(A.commit(&P->dev->mem, h->h2d, h->stream));
    tr.mark("plan upload");
    CU(launch_plan_offsets(P->d_tile_e, h->tile_e.size(), h->g0, h->g1, h->ng, h->K, P->d_tile_off, h->stream));
    CU(cudaStreamSynchronize(h->stream));  // shared by handles on other streams (cold path only)
    tr.mark("plan sync");
    P->N = h->N; P->a_llm = h->a_llm; P->b_llm = h->b_llm; P->Ka = h->Ka; P->Kb = h->Kb; P->g0 = h->g0;
    P->g1 = h->g1; P->ng = h->ng; P->umax_a = h->umax_a; P->umax_b = h->umax_b;
    P->L = h->L; P->n_chunks = h->n_chunks; P->n_groups = h->n_groups; P->nQ = h->nQ; P->A = h->A;
    memcpy(P->pw, h->pw, sizeof(P->pw));
    P->umax_total = h->umax_total;
    P->dv = h->dv;
    P->dcnt = h->dcnt;
    P->gsum = h->gsum;
    P->n_groups_u = h->n_groups_u;
    g_plans[key] = P;
    h->tile_s.clear(); h->tile_e.clear(); h->bperm.clear(); h->bu.clear();
  }
  h->N = P->N; h->a_llm = P->a_llm; h->b_llm = P->b_llm; h->Ka = P->Ka; h->Kb = P->Kb; h->g0 = P->g0;
  h->g1 = P->g1; h->ng = P->ng; h->umax_a = P->umax_a; h->umax_b = P->umax_b;
  h->L = P->L; h->n_chunks = P->n_chunks; h->n_groups = P->n_groups; h->nQ = P->nQ; h->A = P->A;
  memcpy(h->pw, P->pw, sizeof(h->pw));
  h->umax_total = P->umax_total;
  h->dv = P->dv;
  h->dcnt = P->dcnt;
  h->gsum = P->gsum;
  h->n_groups_u = P->n_groups_u;
  h->d_u = P->d_u; h->d_tile_s = P->d_tile_s; h->d_tile_e = P->d_tile_e; h->d_tile_off = P->d_tile_off;
  h->d_bperm = P->d_bperm; h->d_dv = P->d_dv; h->d_dcnt = P->d_dcnt; h->d_gsum = P->d_gsum;
  h->plan_dev = P->dev;
  return ALP_OK;
}

// Byte layout of a Scratch for n targets at `base` (nullptr: sizes only).  Returns the total bytes;
// *rest = the bytes of the leading section that must be zero before the first use (fixed size,
// independent of n, so one buffer serves calls with any n up to its capacity).
size_t ws_layout(const alp_s *h, int n, unsigned char *base, Scratch *sc, size_t *rest = nullptr) {
  const size_t MK = (size_t)h->M * h->K, nn = (size_t)std::max(n, 1);
  size_t off = 0;
  auto take = [&](size_t bytes) -> unsigned char * {
    const size_t o = (off + 255) & ~size_t(255);
    off = o + bytes;
    return base ? base + o : nullptr;
  };
  Scratch x;
  x.fzkeys = reinterpret_cast<unsigned long long *>(take(8 * kInlineTargets));
  x.fzcounts = reinterpret_cast<unsigned long long *>(take(8 * kInlineTargets));
  x.fzwork = reinterpret_cast<unsigned long long *>(take(8 * kFusedWork));
  x.fzticket = reinterpret_cast<unsigned *>(take(4));
  if (rest) *rest = off;
  x.fbest = reinterpret_cast<unsigned long long *>(take(8 * nn));
  x.fdone = reinterpret_cast<unsigned *>(take(4 * nn));
  x.targets = reinterpret_cast<double *>(take(8 * nn));
  x.tau = reinterpret_cast<float *>(take(4 * nn * MK));
  x.term = reinterpret_cast<double *>(take(8 * nn * MK));
  x.b = reinterpret_cast<double *>(take(8 * nn * MK));
  x.res = reinterpret_cast<alp_result *>(take(sizeof(alp_result) * nn));
  x.keys = reinterpret_cast<unsigned long long *>(take(8 * nn));
  x.counts = reinterpret_cast<unsigned long long *>(take(8 * nn));
  x.qb = reinterpret_cast<int *>(take(4 * nn));
  x.work = reinterpret_cast<unsigned long long *>(take(8 * std::max<size_t>(kArenaWork, 16 * nn)));
  x.cap = (int)nn;
  if (sc) *sc = x;
  return (off + 255) & ~size_t(255);
}

// Stage the handle's own tables (profiles or injected terms) + single-target scratch in one allocation.
alp_status upload_all(alp_s *h) {
  alp_status s = get_plan(h);
  if (s != ALP_OK) return s;
  Arena A;
  const size_t MK = (size_t)h->M * h->K;
  if (h->from_terms) {
    A.add(h->tau_fixed, &h->d_tau_fixed);
    A.add(h->term_fixed, &h->d_term_fixed);
    A.add(h->b_fixed, &h->d_b_fixed);
  } else {
    A.add(h->n, &h->d_n);
    A.add(h->p, &h->d_p);
    A.add(h->S, &h->d_S);
    A.add(h->prof_off, &h->d_off);
    A.add(h->rate, &h->d_rate);
    A.add(h->lat, &h->d_lat);
    A.add(h->tmax, &h->d_tmax);
    if (!h->min_units.empty()) A.add(h->min_units, &h->d_minu);
    if (!h->meas_off.empty()) {
      A.add(h->meas_off, &h->d_moff);
      A.add(h->mrate, &h->d_mrate);
      A.add(h->mlat, &h->d_mlat);
      A.add(h->mtmax, &h->d_mtmax);
    }
  }
  A.add(h->T, &h->d_T);
  A.add(h->R, &h->d_R);
  // the single-target scratch: its zero-at-rest section rides in the copied part (no memset)
  size_t rest = 0;
  const size_t own = ws_layout(h, 1, nullptr, nullptr, &rest);
  unsigned char *d_own = nullptr;
  A.region(own, rest, &d_own);
  CU(A.commit(&h->d_arena, h->h2d, h->stream));
  ws_layout(h, 1, d_own, &h->own1);
  CU(cudaEventRecord(h->ctx.ready, h->stream));  // searches on other streams wait for the upload
  return ALP_OK;
}

// Order a caller's stream after the handle's upload and after the handle's previous work on
// another stream (the per-handle scratch is reused by every call); remember it for alp_destroy.
alp_status use_stream(alp_s *h, cudaStream_t st, bool own_scratch = true) {
  if (st != h->stream) CU(cudaStreamWaitEvent(st, h->ctx.ready, 0));
  if (!own_scratch) return ALP_OK;  // caller workspace: calls on other streams may overlap
  if (h->last_stream && h->last_stream != st) {
    CU(cudaEventRecord(h->ctx.last, h->last_stream));
    CU(cudaStreamWaitEvent(st, h->ctx.last, 0));
  }
  h->last_stream = st;
  return ALP_OK;
}

alp_status init_device(alp_s *h) {
  // rows per lane: 12 at 2 blocks/SM (no register cap) beats 8 at 3 blocks/SM and 16 on both C4
  // and C3 (profiles/r01_rows_per_lane.txt); ALP_ROWS_PER_LANE (8 / 12 / 16) overrides.
  h->rows_per_lane = 12;
  if (const char *v = getenv("ALP_ROWS_PER_LANE")) {
    const int t = atoi(v);
    h->rows_per_lane = (t == 16 || t == 12) ? t : 8;
  }
  if (const char *v = getenv("ALP_BLOCKS_PER_SM")) h->min_blocks = std::min(4, std::max(2, atoi(v)));
  if (const char *v = getenv("ALP_NQ")) h->nq_force = std::max(0, atoi(v));
  CU(cudaGetDevice(&h->device));
  CU(cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, h->device));
  CU(ctx_acquire(h->device, h->ctx));
  h->stream = h->ctx.stream;
  h->ev0 = h->ctx.ev0; h->ev1 = h->ctx.ev1; h->evs0 = h->ctx.evs0; h->evs1 = h->ctx.evs1;
  if (h->device >= kMaxDevices) return fail(ALP_ECUDA, "device index %d >= %d", h->device, kMaxDevices);
  static std::once_flag pool_once[kMaxDevices];
  std::call_once(pool_once[h->device], [&] {
    // keep freed handle memory in the default pool so the next alp_build reuses it cheaply
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, h->device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  });
  return ALP_OK;
}

void compute_units(alp_s *h) {
  h->u.assign((size_t)h->M * h->K, 0);
  for (int m = 0; m < h->M; ++m)
    for (int k = 0; k < h->K; ++k) {
      const int r_i = k % h->nR, t_i = (k / h->nR) % h->nT, s_i = k / (h->nR * h->nT);
      h->u[(size_t)m * h->K + k] = h->S[s_i] * h->T[t_i] * h->R[r_i];
    }
}

bool ascending(const int32_t *v, int n, int lo) {
  for (int i = 0; i < n; ++i) {
    if (v[i] < lo) return false;
    if (i && v[i] <= v[i - 1]) return false;
  }
  return true;
}

// ---------------------------------------------------------------- per-search geometry
struct Geometry {
  SearchArgs a;
  int grid;
};

alp_status make_geometry(alp_s *h, int n_targets, int64_t budget, uint64_t lo, uint64_t hi, Geometry &g,
                         bool fused = false) {
  if (budget < 0) return fail(ALP_EINVAL, "budget_units < 0");
  const long long Reff = std::min<long long>(budget, h->umax_total);
  if (Reff > 16384) return fail(ALP_EINVAL, "budget_units (capped at the total max units) exceeds 16384");
  SearchArgs &a = g.a;
  memset(&a, 0, sizeof(a));
  a.M = h->M; a.K = h->K; a.g0 = h->g0; a.g1 = h->g1; a.a_llm = h->a_llm; a.b_llm = h->b_llm;
  a.Ka = h->Ka; a.Kb = h->Kb; a.ng = h->ng; a.L = h->L; a.n_chunks = h->n_chunks;
  a.n_groups = h->n_groups; a.nQ = h->nQ; a.A = h->A; a.item_lo = lo; a.item_hi = hi;
  a.fd_nQ = make_fastdiv(h->nQ);
  a.fd_ng = make_fastdiv(h->n_groups);
  const bool fine = (uint64_t)h->n_chunks * h->L * (uint64_t)h->Ka < 0xffffffffull;  // segment per a option
  a.seg_q = fine ? (uint32_t)h->Ka : h->nQ;
  a.seg_A = fine ? 1u : h->A;
  a.seg_mul = fine ? h->A : 1u;
  a.u_nbulk = 0xffffffffu;  // k_search_u: no tail split unless u_tail_split sets one
  a.u_S = 1;
  a.u_As = h->A;
  a.fd_S = make_fastdiv(1);
  a.budget = (int)Reff;
  a.n_targets = n_targets;
  a.D = (int)(std::upper_bound(h->dv.begin(), h->dv.end(), (int)Reff) - h->dv.begin());
  for (int m = 0; m < ALP_MAX_M; ++m) a.pw[m] = h->pw[m];
  const int rows = a.D + 1;
  a.rows_max = rows;
  auto align16 = [](int x) { return (x + 15) & ~15; };
  auto layout = [&](int W) {
    a.bchunk_w = W;
    a.n_bchunks = (h->Kb + W - 1) / W;
    a.bchunk_wpad = W <= 34 ? (W + 1) / 2 * 2 : (W + 3) / 4 * 4;
    a.row_stride = a.bchunk_wpad + 1;  // >= 1 padding column (holds the row's finite count)
    while (a.row_stride % 8 != 4) ++a.row_stride;
    int off = 0;
    a.off_tau = off; off = align16(off + (h->g1 * h->K + 2) * 4);  // must stay at offset 0
    a.off_u = off; off = align16(off + h->g0 * h->K * 4);
    a.off_a = off; off = align16(off + h->Ka * 8);
    a.off_lut = off; off = align16(off + (a.budget + 2) * 8);
    a.off_tmp = off; off = align16(off + (3 * h->Kb + 3 + h->Ka) * 4);  // dv, dcnt, bperm, ua
    a.off_btab = off; off = align16(off + rows * a.row_stride * 4);
    a.off_pfx = -1;
    if (h->g0 > 0 && h->n_chunks <= kPfxTableMax) {
      a.off_pfx = off;
      off = align16(off + (int)h->n_chunks * 8);
    }
    a.fz.off_opt = 0;
    if (fused) {
      a.fz.off_opt = off;
      off = align16(off + h->M * h->K * 4);
    }
    a.smem_bytes = off;
    return off;
  };
  int W = h->Kb;
  while (layout(W) > 72 * 1024 && W > 64) W = (W + 1) / 2;
  if (a.smem_bytes > 220 * 1024) return fail(ALP_EINVAL, "shared-memory tables too large (%d B)", a.smem_bytes);
  a.tau = nullptr;  // set by caller
  a.u = h->d_u; a.tile_s = h->d_tile_s; a.tile_e = h->d_tile_e; a.tile_off = h->d_tile_off; a.bperm = h->d_bperm;
  a.rows_per_lane = h->rows_per_lane;
  a.min_blocks = h->min_blocks;
  a.dv = h->d_dv; a.dcnt = h->d_dcnt;
  a.n_groups_u = h->n_groups_u; a.gsum = h->d_gsum;
  a.t_begin = 0; a.t_end = n_targets; a.c_begin = 0; a.c_end = a.n_bchunks;
  // occupancy per kernel variant and smem size (cached: the query costs microseconds per search)
  const long long okey = ((long long)a.smem_bytes << 24) | ((long long)a.bchunk_wpad << 8) |
                         ((long long)a.rows_per_lane << 3) | a.min_blocks;
  auto oit = h->occ_cache.find(okey);
  const int bps = (oit != h->occ_cache.end()) ? oit->second : (h->occ_cache[okey] = search_max_blocks_per_sm(a));
  if (bps < 1) return fail(ALP_ECUDA, "search kernel cannot be resident (smem %d B)", a.smem_bytes);
  g.grid = h->sm_count * bps;
  return ALP_OK;
}

// Select the handle's own scratch for n targets (grown on demand; a new buffer's zero-at-rest
// section is cleared on `st`).
alp_status ensure_scratch(alp_s *h, int n, cudaStream_t st) {
  if (n <= 1) {
    h->sc = h->own1;
    return ALP_OK;
  }
  if (h->g_ws_cap < n) {
    const int cap = std::max(n, 2 * h->g_ws_cap);
    size_t rest = 0;
    CU(h->g_ws.ensure(ws_layout(h, cap, nullptr, nullptr, &rest)));
    CU(cudaMemsetAsync(h->g_ws.p, 0, rest, st));
    h->g_ws_cap = cap;
  }
  ws_layout(h, h->g_ws_cap, h->g_ws.p, &h->sc);  // laid out for the capacity: any n <= cap
  return ALP_OK;
}

// Select a caller workspace (alp_workspace_bytes(h, n) bytes, zero-filled before its first use).
alp_status bind_workspace(alp_s *h, void *ws, int n) {
  if (reinterpret_cast<uintptr_t>(ws) & 255) return fail(ALP_EINVAL, "d_workspace must be 256-byte aligned");
  ws_layout(h, n, static_cast<unsigned char *>(ws), &h->sc);
  h->sc.ws = true;
  h->ws_used = true;
  return ALP_OK;
}

// Scratch of a call: the caller's workspace when given, else the handle's own.
alp_status select_scratch(alp_s *h, void *ws, int n, cudaStream_t st) {
  return ws ? bind_workspace(h, ws, n) : ensure_scratch(h, n, st);
}

// K1 for n targets into the scratch tables (profiles mode) or replicate the fixed terms.
alp_status option_tables(alp_s *h, const double *targets, int n, cudaStream_t st, unsigned long long *keys,
                         unsigned long long *counts, unsigned long long *work = nullptr, int n_work = 0) {
  const size_t MK = (size_t)h->M * h->K;
  double *pin = (n * sizeof(double) <= kPinHalf) ? static_cast<double *>(pinned_scratch(2 * kPinHalf)) : nullptr;
  const bool inline_t = !h->from_terms && n <= kInlineTargets;  // targets travel in K1's parameters
  if (inline_t) {
  } else if (pin) {
    // the pinned buffer may still feed an earlier copy (any stream, any device): wait for those
    // copies only (one event per device: events record only on their own device's streams)
    static thread_local cudaEvent_t pin_ev[kMaxDevices] = {};
    if (h->device >= kMaxDevices) return fail(ALP_ECUDA, "device index %d >= %d", h->device, kMaxDevices);
    for (cudaEvent_t ev : pin_ev)
      if (ev) CU(cudaEventSynchronize(ev));
    if (!pin_ev[h->device]) CU(cudaEventCreateWithFlags(&pin_ev[h->device], cudaEventDisableTiming));
    memcpy(pin, targets, n * sizeof(double));
    CU(cudaMemcpyAsync(h->sc.targets, pin, n * sizeof(double), cudaMemcpyHostToDevice, st));
    CU(cudaEventRecord(pin_ev[h->device], st));
  } else {
    CU(cudaMemcpyAsync(h->sc.targets, targets, n * sizeof(double), cudaMemcpyHostToDevice, st));
  }
  if (h->from_terms) {
    for (int t = 0; t < n; ++t) {
      CU(cudaMemcpyAsync(h->sc.tau + t * MK, h->d_tau_fixed, MK * sizeof(float), cudaMemcpyDeviceToDevice, st));
      CU(cudaMemcpyAsync(h->sc.term + t * MK, h->d_term_fixed, MK * sizeof(double), cudaMemcpyDeviceToDevice, st));
      CU(cudaMemcpyAsync(h->sc.b + t * MK, h->d_b_fixed, MK * sizeof(double), cudaMemcpyDeviceToDevice, st));
    }
    if (keys) CU(launch_init_keys(keys, counts, n, work, n_work, h->sc.fbest, h->sc.fdone, st));
    return ALP_OK;
  }
  OptionArgs o;
  o.prof = h->dprof();
  o.targets = inline_t ? nullptr : h->sc.targets;
  for (int i = 0; i < kInlineTargets; ++i) o.tgt[i] = (inline_t && i < n) ? targets[i] : 0.0;
  o.n_targets = n;
  o.tau = h->sc.tau;
  o.term = h->sc.term;
  o.b = h->sc.b;
  o.u = h->d_u;
  o.keys = keys;
  o.counts = counts;
  o.work = work;
  o.n_work = n_work;
  o.fbest = h->sc.fbest;  // finalize combine scratch, zeroed for the K3 after this search
  o.fdone = h->sc.fdone;
  CU(launch_option_table(o, st));
  return ALP_OK;
}

alp_status check_targets(const double *targets, int n) {
  if (!targets || n < 1) return fail(ALP_EINVAL, "targets: need n >= 1 targets");
  for (int i = 0; i < n; ++i)
    if (!(targets[i] > 0.0) || !std::isfinite(targets[i])) return fail(ALP_EINVAL, "targets[%d] must be finite and > 0", i);
  return ALP_OK;
}

// Per-query budgets: validated, capped at the total max units (never binding above it) and uploaded.
// Returns the largest (capped) budget, which sizes the shared-memory tables.
alp_status prepare_budgets(alp_s *h, const int64_t *budgets, int n, cudaStream_t st, int64_t *rmax) {
  h->s_qb = nullptr;
  if (!budgets) return ALP_OK;
  std::vector<int> qb(n);
  int64_t mx = 0;
  for (int i = 0; i < n; ++i) {
    if (budgets[i] < 0) return fail(ALP_EINVAL, "budgets[%d] < 0", i);
    qb[i] = (int)std::min<int64_t>(budgets[i], h->umax_total);
    mx = std::max<int64_t>(mx, budgets[i]);
  }
  h->s_qb = h->sc.qb;
  CU(cudaMemcpyAsync(h->s_qb, qb.data(), n * sizeof(int), cudaMemcpyHostToDevice, st));
  CU(cudaStreamSynchronize(st));  // qb is a host temporary
  *rmax = mx;
  return ALP_OK;
}

// Fused single launch (no K1 / K3): few targets, a common budget, and a small option table (every
// block recomputes it: cheaper than a K1 launch only while M*K is small) and a short finalize
// re-scan (one block, <= Ka*Kb candidates; larger ones use K3's multi-block re-scan).
// Injected terms (alp_build_from_terms) describe one target only.
bool use_fused(const alp_s *h, int n, const int64_t *budgets) {
  if (getenv("ALP_NO_FUSED")) return false;  // A/B switch for measurements
  return !budgets && n <= kInlineTargets && h->M * h->K <= kFusedMaxTerms &&
         (uint64_t)h->Ka * h->Kb <= kFusedMaxRescan && (!h->from_terms || n == 1);
}

// Finalize inputs of the handle's scratch (K3 and the fused last block).
void fill_finalize(alp_s *h, SearchArgs &a) {
  FinalizeExtra &f = a.fin;
  f.term = h->sc.term;
  f.b = h->sc.b;
  if (h->from_terms) {  // injected terms: the FP64 terms are the handle's fixed tables (any path)
    f.term = h->d_term_fixed;
    f.b = h->d_b_fixed;
  }
  f.S = h->from_terms ? nullptr : h->d_S;
  f.T = h->d_T;
  f.R = h->d_R;
  f.nS = h->nS; f.nT = h->nT; f.nR = h->nR;
  f.N = h->N;
  f.out = h->sc.res;
  f.best = h->sc.fbest;
  f.done = h->sc.fdone;
}

// Uniform-register path (alp_search_u.cu) for single-target searches with short b rows: the
// arguments with its shared-memory layout, lut geometry and grid; false when not applicable.
bool ur_path(alp_s *h, const SearchArgs &a, int n, uint64_t hi, SearchArgs &ua, int &grid) {
  if (getenv("ALP_NO_UR") || n < 1 || n > kInlineTargets || a.q_budget || h->from_terms ||
      h->rows_per_lane != search_u_rows() || hi >= (1ull << 31) || n * h->M * h->K > 8192)
    return false;
  const int R = a.budget, Kb = h->Kb;
  auto umax = [&](int m) {
    int x = 0;
    for (int k = 0; k < h->K; ++k) x = std::max(x, h->u[(size_t)m * h->K + k]);
    return x;
  };
  // lut span: the prefix, sort-group and a unit sums enter clamped at R + 1 (a clamped sum keeps
  // the remaining budget negative, i.e. the all-+inf row, exactly like the true sum)
  int up = 0, ug = 0;
  for (int m = 0; m < h->g0; ++m) up += umax(m);
  for (int m = h->g0; m < h->g1; ++m) ug += umax(m);
  const int lb = std::min(up, R + 1) + std::min(ug, R + 1) + (h->a_llm >= 0 ? std::min(umax(h->a_llm), R + 1) : 0);
  ua = a;
  ua.lut_base = lb;
  ua.lut_n = lb + 1;
  ua.u_amax = h->a_llm >= 0 ? std::min(umax(h->a_llm), R + 1) : 0;
  // b chunks: a short b row (<= 34 options) is one chunk with the k_search row layout; longer rows
  // are cut into chunks of kUChunkW u-sorted columns, each with its own lut and de-duplicated masked
  // rows (a chunk has a new row only where the budget threshold falls inside it)
  int W, wpad, cstride;
  if (Kb <= 34) {
    if (a.n_bchunks != 1) return false;
    W = Kb;
    wpad = a.bchunk_wpad;
    cstride = a.row_stride;
  } else {
    W = wpad = cstride = kUChunkW;
  }
  const int nch = (Kb + W - 1) / W;
  if (nch > kUMaxChunks) return false;
  ua.bchunk_w = W;
  ua.bchunk_wpad = wpad;
  ua.n_bchunks = nch;
  ua.u_nch = nch;
  ua.u_cstride = cstride;
  ua.row_stride = cstride;
  ua.u_smem_rows = (n == 1 && nch == 1) ? 1 : 0;
  auto a16 = [](int x) { return (x + 15) & ~15; };
  // constant-bank layout: gsum (every group), then one block per target: a-options, prefix chunks,
  // then per chunk its lut and rows
  ua.u_tbase = a16((int)h->n_groups * 4);
  ua.u_off_a = 0;
  ua.u_off_pfx = a16((h->Ka + 1) * 16);  // Ka + 1 a entries: .w holds the feasible-option prefix count
  int off = a16(ua.u_off_pfx + (int)h->n_chunks * 8), rows0 = 0;
  for (int c = 0; c < nch; ++c) {
    const int c0 = c * W, wc = std::min(W, Kb - c0);
    int rows = 1, prev = 0;  // row 0: all +inf
    for (int i = 1; i <= a.D; ++i) {
      const int len = std::min(std::max(std::min(h->dcnt[i], Kb) - c0, 0), wc);
      if (len > prev) ++rows;
      prev = len;
    }
    if (c == 0) rows0 = rows;
    ua.u_off_lut_c[c] = off;
    off = a16(off + ua.lut_n * 8);
    ua.u_off_btab_c[c] = off;
    off = a16(off + rows * cstride * 4);
  }
  ua.u_tstride = off;
  if ((long long)ua.u_tbase + (long long)n * ua.u_tstride > kUBytes) return false;
  if (uprep_smem_bytes(ua) > kUPrepSmemMax) return false;
  // shared memory: the option terms of LLMs 0..g1-1 (+ {0, +inf}) of every target; with u_smem_rows
  // also copies of the chunk's lut and masked rows (the mixed groups read them from there)
  off = a16(n * (h->g1 * h->K + 2) * 4);
  ua.off_lut = off;
  ua.off_btab = off;
  if (ua.u_smem_rows) {
    off = a16(off + ua.lut_n * 8);
    ua.off_btab = off;
    off = a16(off + rows0 * cstride * 4);
  }
  // room for the fused finalize's staged inputs (the epilogue reuses the search's shared memory;
  // up to 8 KB keeps 24 one-warp blocks per SM)
  const int stage = (int)finalize_stage_bytes(h->M, h->K, h->nS, h->nT, h->nR);
  ua.fin.stage = stage <= 8192 ? 1 : 0;
  if (ua.fin.stage && stage > off) off = a16(stage);
  ua.smem_bytes = off;
  const long long okey = (1ll << 60) | ((long long)ua.smem_bytes << 8) | ua.bchunk_wpad;
  auto oit = h->occ_cache.find(okey);
  const int bps = (oit != h->occ_cache.end()) ? oit->second : (h->occ_cache[okey] = search_u_max_blocks_per_sm(ua));
  if (bps < 1) return false;
  // 24 one-warp blocks per SM (6 per SMSP): more when ptxas allocates fewer registers was slower
  // (C4 0.4507 vs 0.4362 ms at 28 blocks/SM with 71 registers, tools/shard_timing.py)
  int use = std::min(bps, 24);
  if (const char *v = getenv("ALP_U_BPS")) use = std::max(1, std::min(bps, atoi(v)));  // tuning knob
  grid = h->sm_count * use;
  return true;
}

// k_search_u tail split: the last items of the rank's range are handed out as S sub-items of
// ceil(A / S) a options (needs single-option segments), so the warps' last tickets are short.
// Default: the last warps/2 items in 2 parts (3 parts before the full-row loop: C4 8-rank shard
// kernel 0.0758 -> 0.0737 ms; with the full-row kernel 2 parts measured 0.0973-0.0993 ms vs 0.0993
// for 3, profiles/r02_tail_split_fullrow.txt).  ALP_U_SPLIT="x,S": split the last x * warps items
// (x = 0: off).
void u_tail_split(SearchArgs &ua, uint64_t warps, uint64_t n_items) {
  static double xw = 0.5;
  static int S = 2;
  static bool once = [] {
    if (const char *v = getenv("ALP_U_SPLIT")) sscanf(v, "%lf,%d", &xw, &S);
    return true;
  }();
  (void)once;
  if (ua.seg_A != 1 || S < 2 || xw <= 0.0) return;
  const int As = ((int)ua.A + S - 1) / S;
  const int Sx = ((int)ua.A + As - 1) / As;
  const uint64_t x = std::min<uint64_t>(n_items, (uint64_t)(xw * (double)warps));
  if (x == 0 || Sx < 2 || n_items + x * (uint64_t)(Sx - 1) >= 0x7fffffffull) return;
  ua.u_nbulk = (uint32_t)(n_items - x);
  ua.u_S = (uint32_t)Sx;
  ua.u_As = (uint32_t)As;
  ua.fd_S = make_fastdiv((uint32_t)Sx);
}

// Targets per uniform-register launch for a large batch (0: the path does not apply): the most
// (<= kInlineTargets) whose tables fit the constant bank.
int ur_batch_group(alp_s *h, int64_t budget) {
  if (getenv("ALP_NO_UR") || getenv("ALP_NO_FUSED")) return 0;
  for (int g = kInlineTargets; g >= 1; g /= 2) {
    if (!use_fused(h, g, nullptr)) continue;
    Geometry geo;
    if (make_geometry(h, g, budget, 0, 0, geo, true) != ALP_OK) return 0;
    SearchArgs ua;
    int grid = 0;
    const uint64_t items = (uint64_t)h->n_chunks * h->n_groups * h->nQ;
    if (ur_path(h, geo.a, g, items, ua, grid)) return g;
  }
  return 0;
}

// K2 over work items [lo, hi) (classic: after K1; fused: alone, finalize optional).  Writes the
// per-target (key, count) of this shard to keys/counts; async on st.
alp_status search_shard_impl(alp_s *h, const double *targets, const int64_t *budgets, int n, int64_t budget,
                             uint64_t lo, uint64_t hi, cudaStream_t st, unsigned long long *keys,
                             unsigned long long *counts, bool fuse_finalize = false,
                             alp_result *fused_out = nullptr, bool first_of_batch = true, void *ws = nullptr,
                             const PeerArgs *peer = nullptr) {
  alp_status s = check_targets(targets, n);
  if (s != ALP_OK) return s;
  CU(cudaSetDevice(h->device));
  s = use_stream(h, st, ws == nullptr);
  if (s != ALP_OK) return s;
  if (first_of_batch) CU(cudaEventRecord(h->evs0, st));  // step start (a batch of launches: the first)
  s = select_scratch(h, ws, n, st);
  if (s != ALP_OK) return s;
  if (peer) {  // the rank's own (key, count) stay in the call's scratch
    keys = h->sc.keys;
    counts = h->sc.counts;
  }
  s = prepare_budgets(h, budgets, n, st, &budget);
  if (s != ALP_OK) return s;
  const bool fused = use_fused(h, n, budgets);
  Geometry g;
  s = make_geometry(h, n, budget, 0, 0, g, fused);
  if (s != ALP_OK) return s;
  const uint64_t items = (uint64_t)h->n_chunks * h->n_groups * h->nQ;
  if (lo > hi || hi > items) return fail(ALP_EINVAL, "item range [%llu, %llu) outside [0, %llu)",
                                         (unsigned long long)lo, (unsigned long long)hi, (unsigned long long)items);
  // The uniform-register pair (k_uprep + k_search_u) computes the option terms itself and
  // accumulates like the fused launch.  It shares one constant bank per device: a search on a
  // caller workspace whose bank is still in use by another stream's search takes k_search instead
  // (same keys and counts), so searches on distinct workspaces and streams overlap.
  SearchArgs ua;
  int ugrid = 0;
  // (a peer search never waits for the bank either: the search holding it may be another rank of
  // the same exchange on this device, which waits for this one)
  bool ur = !budgets && ur_path(h, g.a, n, hi, ua, ugrid);
  if (ur && peer) ur = search_u_claim();             // released by the launch (or below on an error)
  else if (ur && h->sc.ws) ur = !search_u_busy();
  struct Claim {
    bool on;
    ~Claim() {
      if (on) search_u_release();  // no-op after the launch
    }
  } claim{ur && peer};
  const bool accum = fused || ur;  // self-resetting accumulators + last-block epilogue (no K1)
  const size_t nctr = (size_t)n * (ur ? ua.u_nch : g.a.n_bchunks);
  int launches = 0;
  unsigned long long *work = h->sc.work;
  if (accum) {
    if (nctr > kFusedWork) return fail(ALP_EINTERNAL, "fused search: %zu work counters", nctr);
    FusedArgs &z = g.a.fz;
    z.on = 1;
    z.finalize = ((fuse_finalize || peer) && fused) ? 1 : 0;
    if (peer) {
      if (!fused) return fail(ALP_EINVAL, "peer exchange needs a fused search (<= %d targets, M*K <= %d, Ka*Kb <= %llu)",
                              kInlineTargets, kFusedMaxTerms, (unsigned long long)kFusedMaxRescan);
      z.peer = *peer;
    }
    if (!h->from_terms) z.prof = h->dprof();
    for (int i = 0; i < kInlineTargets; ++i) z.tgt[i] = i < n ? targets[i] : 0.0;
    z.tau_fixed = h->from_terms ? h->d_tau_fixed : nullptr;
    z.o_tau = h->sc.tau;
    z.o_term = h->sc.term;
    z.o_b = h->sc.b;
    z.acc_keys = h->sc.fzkeys;
    z.acc_counts = h->sc.fzcounts;
    z.work = h->sc.fzwork;
    z.ticket = h->sc.fzticket;
    work = h->sc.fzwork;
  } else {
    // work counters (one per phase, zeroed by K1; the scratch holds >= 16 per target)
    s = option_tables(h, targets, n, st, keys, counts, work, (int)nctr);
    if (s != ALP_OK) return s;
    launches = 1;  // K1
  }
  g.a.q_budget = h->s_qb;
  g.a.item_lo = lo;
  g.a.item_hi = hi;
  g.a.tau = h->sc.tau;
  g.a.keys = keys;
  g.a.counts = counts;
  fill_finalize(h, g.a);
  if (fused_out) g.a.fin.out = fused_out;
  if (first_of_batch) CU(cudaEventRecord(h->ev0, st));
  if (hi > lo || accum) {  // the fused / UR launch also computes the terms and writes keys/counts
    g.a.t_begin = 0; g.a.t_end = n; g.a.c_begin = 0; g.a.c_end = g.a.n_bchunks;
    g.a.work = work;
    // ~16 grabs per warp; the last ~1/8 of the items go in grabs a quarter that size (tail balance;
    // finer a-ranges balance the tail better but cost more in the bulk: measured)
    const uint64_t warps = (uint64_t)g.grid * (kThreads / 32);
    const uint64_t n_items = hi - lo;
    g.a.grab = (int)std::max<uint64_t>(1, std::min<uint64_t>(1u << 20, n_items / (warps * 16)));
    g.a.grab2 = std::max(1, g.a.grab / 4);
    g.a.grab_t1 = (n_items - n_items / 8) / (uint64_t)g.a.grab;
    static const bool dbg = getenv("ALP_DBG_TS") != nullptr;  // per-block timeline (diagnostics)
    if (ur && !ur_path(h, g.a, n, hi, ua, ugrid)) return fail(ALP_EINTERNAL, "uniform-register geometry changed");
    if (ur) u_tail_split(ua, (uint64_t)ugrid, n_items);
    const int dgrid = ur ? ugrid : g.grid;
    if (dbg) {
      CU(h->g_dbg.ensure((size_t)(dgrid + 2) * 8));  // + one row of epilogue stamps
      CU(cudaMemsetAsync(h->g_dbg.p, 0, (size_t)(dgrid + 2) * 8 * sizeof(unsigned long long), st));
      g.a.dbg_ts = ua.dbg_ts = h->g_dbg.p;
    }
    if (ur) {  // option terms + tables, then the UR search
      // the kernel-time events bracket the search kernel itself (ev0 re-recorded after the prep)
      CU(launch_search_u(ua, ugrid, st, first_of_batch ? h->ev0 : nullptr));
      claim.on = false;  // the launch ended the claim
      launches += 2;
      h->last_ur = true;
    } else {
      CU(launch_search(g.a, g.grid, st));
      launches += 1;
      h->last_ur = false;
    }
    if (dbg) {
      std::vector<unsigned long long> ts((size_t)(dgrid + 2) * 8);
      CU(cudaMemcpyAsync(ts.data(), h->g_dbg.p, ts.size() * 8, cudaMemcpyDeviceToHost, st));
      CU(cudaStreamSynchronize(st));
      unsigned long long t0 = ~0ull;
      for (int b = 0; b < dgrid; ++b) t0 = std::min(t0, ts[b * 8]);
      std::vector<double> v[5];
      for (int b = 0; b < dgrid; ++b)
        for (int i = 0; i < 5; ++i) v[i].push_back(ts[b * 8 + i] ? (ts[b * 8 + i] - t0) * 1e-3 : 0.0);
      for (auto &x : v) std::sort(x.begin(), x.end());
      auto q = [&](int i, double f) { return v[i][(size_t)(f * (v[i].size() - 1))]; };
      if (const char *dump = getenv("ALP_DBG_DUMP")) {  // raw stamps (tools/block_hist.py)
        if (FILE *f = fopen(dump, "ab")) {
          fwrite(ts.data(), 8, ts.size(), f);
          fclose(f);
        }
      }
      fprintf(stderr, "[alp dbg] grid %d us: start med %.1f max %.1f | terms med %.1f max %.1f | tables med %.1f "
              "max %.1f | loop-end min %.1f med %.1f max %.1f | end max %.1f\n", dgrid, q(0, .5), q(0, 1), q(4, .5),
              q(4, 1), q(1, .5), q(1, 1), q(2, 0), q(2, .5), q(2, 1), q(3, 1));
      if (ur && ts[5])  // k_uprep phases (us from its start; the search's t0 is later)
        fprintf(stderr, "[alp dbg] k_uprep us: staged %.2f | terms %.2f | plan tables landed %.2f | a/pfx/b-sorted %.2f | "
                "b rows + lut %.2f | end %.2f | search t0 %+.2f\n",
                (ts[15] - ts[5]) * 1e-3, (ts[6] - ts[5]) * 1e-3, (ts[7] - ts[5]) * 1e-3, (ts[21] - ts[5]) * 1e-3,
                (ts[23] - ts[5]) * 1e-3, (ts[13] - ts[5]) * 1e-3, ((double)t0 - (double)ts[5]) * 1e-3);
    }
  }
  CU(cudaEventRecord(h->ev1, st));
  h->ev_pending = true;
  h->last_args = g.a;
  h->last_launches = launches;
  return ALP_OK;
}

// D2H of the n results (pinned staging), step-end event, sync; status from the results.
// Device pointer into this thread's mapped pinned scratch (upper half) for n results, written by
// the finalizing kernel itself (zero-copy: no D2H copy op, whose start after a kernel costs
// ~5-10 us); nullptr when n results do not fit or mapping is unavailable.
alp_result *zero_copy_out(int n, alp_result **host) {
  *host = nullptr;
  struct Buf {
    alp_result *p = nullptr;
    size_t n = 0;
    ~Buf() {
      if (p) cudaFreeHost(p);
    }
  };
  static thread_local Buf b;  // mapped pinned results, grown on demand (per host thread)
  if ((size_t)n > b.n) {
    if (b.p) cudaFreeHost(b.p);
    b.p = nullptr;
    b.n = 0;
    const size_t want = std::max<size_t>((size_t)n, 128);
    if (cudaHostAlloc(reinterpret_cast<void **>(&b.p), want * sizeof(alp_result),
                      cudaHostAllocPortable | cudaHostAllocMapped) != cudaSuccess) {
      cudaGetLastError();
      b.p = nullptr;
      return nullptr;
    }
    b.n = want;
  }
  alp_result *dres = nullptr;
  if (cudaHostGetDevicePointer(reinterpret_cast<void **>(&dres), b.p, 0) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  *host = b.p;
  return dres;
}

// The n results on the host (zero-copy results already written by the kernel into host_zc, else a
// D2H copy through pinned staging), step-end event, sync; status from the results.
alp_status collect_results(alp_s *h, int n, cudaStream_t st, alp_result *out, const alp_result *host_zc = nullptr) {
  void *pin = (!host_zc && n * sizeof(alp_result) <= kPinHalf) ? pinned_scratch(2 * kPinHalf) : nullptr;
  if (host_zc) {
    CU(cudaEventRecord(h->evs1, st));
    CU(cudaStreamSynchronize(st));
    memcpy(out, host_zc, n * sizeof(alp_result));
  } else if (pin) {
    pin = static_cast<unsigned char *>(pin) + kPinHalf;
    CU(cudaMemcpyAsync(pin, h->sc.res, n * sizeof(alp_result), cudaMemcpyDeviceToHost, st));
    CU(cudaEventRecord(h->evs1, st));
    CU(cudaStreamSynchronize(st));
    memcpy(out, pin, n * sizeof(alp_result));
  } else {
    CU(cudaMemcpyAsync(out, h->sc.res, n * sizeof(alp_result), cudaMemcpyDeviceToHost, st));
    CU(cudaEventRecord(h->evs1, st));
    CU(cudaStreamSynchronize(st));
  }
  CU(cudaEventElapsedTime(&h->last_step_ms, h->evs0, h->evs1));
  if (h->ev_pending) {
    CU(cudaEventElapsedTime(&h->last_ms, h->ev0, h->ev1));
    h->ev_pending = false;
  }
  int any = 0;
  for (int i = 0; i < n; ++i) any |= out[i].found;
  return any ? ALP_OK : ALP_EINFEASIBLE;
}

alp_status finalize_impl(alp_s *h, const double *targets, const int64_t *budgets, int n, int64_t budget,
                         const unsigned long long *keys, const unsigned long long *counts, cudaStream_t st,
                         alp_result *out, int world = 0, void *ws = nullptr) {
  if (!out) return fail(ALP_EINVAL, "out is NULL");
  CU(cudaSetDevice(h->device));
  alp_status s = use_stream(h, st, ws == nullptr);
  if (s != ALP_OK) return s;
  s = select_scratch(h, ws, n, st);  // the scratch the shard search wrote (same n)
  if (s != ALP_OK) return s;
  if (budgets) {
    s = prepare_budgets(h, budgets, n, st, &budget);
    if (s != ALP_OK) return s;
  } else {
    h->s_qb = nullptr;
  }
  Geometry g;
  s = make_geometry(h, n, budget, 0, 0, g);
  if (s != ALP_OK) return s;
  // option tables must describe these targets (the shard call computed them on this handle)
  (void)targets;
  g.a.q_budget = h->s_qb;
  g.a.tau = h->sc.tau;
  fill_finalize(h, g.a);
  g.a.fin.keys = keys;
  g.a.fin.counts = counts;
  g.a.fin.world = world;
  alp_result *hzc = nullptr, *zc = zero_copy_out(n, &hzc);
  if (zc) g.a.fin.out = zc;
  CU(launch_finalize(g.a, st));
  h->last_launches += 1;
  return collect_results(h, n, st, out, hzc);
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

const char *alp_last_error(void) { return g_err.c_str(); }

alp_status alp_build(const alp_desc *d, alp_t **out) {
  NvtxRange nv("alp_build");
  if (!out) return fail(ALP_EINVAL, "out is NULL");
  *out = nullptr;
  if (!d) return fail(ALP_EINVAL, "desc is NULL");
  if (d->M < 1 || d->M > ALP_MAX_M) return fail(ALP_EINVAL, "M must be in 1..%d (got %d)", ALP_MAX_M, d->M);
  if (d->F < 1) return fail(ALP_EINVAL, "F must be >= 1");
  if (!d->n || !d->p) return fail(ALP_EINVAL, "n/p is NULL");
  for (int m = 0; m < d->M; ++m) {
    if (!(d->n[m] > 0) || !std::isfinite(d->n[m])) return fail(ALP_EINVAL, "n[%d] must be finite and > 0", m);
    if (!(d->p[m] >= 1) || !std::isfinite(d->p[m])) return fail(ALP_EINVAL, "p[%d] must be finite and >= 1", m);
  }
  if (d->nS < 1 || d->nT < 1 || d->nR < 1) return fail(ALP_EINVAL, "nS, nT, nR must be >= 1");
  const long long K = (long long)d->nS * d->nT * d->nR;
  if (K > ALP_MAX_K) return fail(ALP_EINVAL, "K = nS*nT*nR = %lld exceeds %d", K, ALP_MAX_K);
  if (!d->share_units || !ascending(d->share_units, d->nS, 1) || d->share_units[d->nS - 1] > d->F)
    return fail(ALP_EINVAL, "share_units must be strictly ascending within 1..F");
  if (!d->tp || !ascending(d->tp, d->nT, 1)) return fail(ALP_EINVAL, "tp must be strictly ascending and >= 1");
  if (!d->replicas || !ascending(d->replicas, d->nR, 1))
    return fail(ALP_EINVAL, "replicas must be strictly ascending and >= 1");
  if (d->pct < 0 || d->pct > 3) return fail(ALP_EINVAL, "pct must be 0..3");
  const double *lat = d->lat[d->pct];
  if (!lat) return fail(ALP_EINVAL, "lat[%d] (selected percentile column) is NULL", d->pct);
  if (!d->prof_off || !d->rate) return fail(ALP_EINVAL, "prof_off/rate is NULL");
  const int C = d->M * d->nT;
  if (d->prof_off[0] != 0) return fail(ALP_EINVAL, "prof_off[0] must be 0");
  double term_bound = 0.0;
  for (int c = 0; c < C; ++c) {
    const int a = d->prof_off[c], b = d->prof_off[c + 1];
    if (b <= a) return fail(ALP_EINVAL, "profile of LLM %d tp index %d has no points", c / d->nT, c % d->nT);
    for (int i = a; i < b; ++i) {
      if (!std::isfinite(d->rate[i]) || d->rate[i] < 0) return fail(ALP_EINVAL, "rate[%d] must be finite and >= 0", i);
      if (i > a && !(d->rate[i] > d->rate[i - 1]))
        return fail(ALP_EINVAL, "rates of LLM %d tp index %d not strictly increasing", c / d->nT, c % d->nT);
      if (!(lat[i] > 0) || !std::isfinite(lat[i])) return fail(ALP_EINVAL, "lat[%d] must be finite and > 0", i);
      if (i > a && lat[i] < lat[i - 1])
        return fail(ALP_EINVAL, "latencies of LLM %d tp index %d decrease", c / d->nT, c % d->nT);
    }
    if (d->tmax && (!std::isfinite(d->tmax[c]) || d->tmax[c] < d->rate[b - 1]))
      return fail(ALP_EINVAL, "tmax[%d] must be finite and >= the last profiled rate", c);
    if (d->min_units && d->min_units[c] < 0) return fail(ALP_EINVAL, "min_units[%d] < 0", c);
  }
  for (int m = 0; m < d->M; ++m) {
    double lmax = 0;
    for (int t = 0; t < d->nT; ++t) lmax = std::max(lmax, lat[d->prof_off[m * d->nT + t + 1] - 1]);
    term_bound += lmax * ((double)d->F / d->share_units[0]) * (d->n[m] / d->p[m]) * 1.0000001;
  }
  // measured per-share curves (R2): same validation as the base curves
  const int CM = C * d->nS;
  const double *mlat = nullptr;
  if (d->meas_off) {
    mlat = d->meas_lat[d->pct];
    if (d->meas_off[0] != 0) return fail(ALP_EINVAL, "meas_off[0] must be 0");
    if (d->meas_off[CM] > 0 && (!d->meas_rate || !mlat))
      return fail(ALP_EINVAL, "meas_rate / meas_lat[%d] (selected percentile column) is NULL", d->pct);
    for (int c = 0; c < CM; ++c) {
      const int a = d->meas_off[c], b = d->meas_off[c + 1];
      if (b < a) return fail(ALP_EINVAL, "meas_off not non-decreasing at %d", c);
      const int m = c / (d->nT * d->nS), ti = (c / d->nS) % d->nT, si = c % d->nS;
      for (int i = a; i < b; ++i) {
        if (!std::isfinite(d->meas_rate[i]) || d->meas_rate[i] < 0)
          return fail(ALP_EINVAL, "meas_rate[%d] must be finite and >= 0", i);
        if (i > a && !(d->meas_rate[i] > d->meas_rate[i - 1]))
          return fail(ALP_EINVAL, "measured rates of LLM %d tp index %d share index %d not strictly increasing", m, ti, si);
        if (!(mlat[i] > 0) || !std::isfinite(mlat[i])) return fail(ALP_EINVAL, "meas_lat[%d] must be finite and > 0", i);
        if (i > a && mlat[i] < mlat[i - 1])
          return fail(ALP_EINVAL, "measured latencies of LLM %d tp index %d share index %d decrease", m, ti, si);
      }
      if (b > a) {
        if (d->meas_tmax && (!std::isfinite(d->meas_tmax[c]) || d->meas_tmax[c] < d->meas_rate[b - 1]))
          return fail(ALP_EINVAL, "meas_tmax[%d] must be finite and >= the last measured rate", c);
        term_bound += mlat[b - 1] * (d->n[m] / d->p[m]) * 1.0000001;
      }
    }
  }
  if (!(term_bound < 1e37)) return fail(ALP_EINVAL, "latency terms could overflow binary32 (sum bound %g)", term_bound);

  alp_s *h = new alp_s();
  h->M = d->M; h->F = d->F; h->nS = d->nS; h->nT = d->nT; h->nR = d->nR; h->K = (int)K;
  h->n.assign(d->n, d->n + d->M);
  h->p.assign(d->p, d->p + d->M);
  h->S.assign(d->share_units, d->share_units + d->nS);
  h->T.assign(d->tp, d->tp + d->nT);
  h->R.assign(d->replicas, d->replicas + d->nR);
  h->prof_off.assign(d->prof_off, d->prof_off + C + 1);
  const int P = d->prof_off[C];
  h->rate.assign(d->rate, d->rate + P);
  h->lat.assign(lat, lat + P);
  h->tmax.resize(C);
  for (int c = 0; c < C; ++c) h->tmax[c] = d->tmax ? d->tmax[c] : d->rate[d->prof_off[c + 1] - 1];
  if (d->min_units) h->min_units.assign(d->min_units, d->min_units + C);
  if (d->meas_off && d->meas_off[CM] > 0) {
    h->meas_off.assign(d->meas_off, d->meas_off + CM + 1);
    const int PM = d->meas_off[CM];
    h->mrate.assign(d->meas_rate, d->meas_rate + PM);
    h->mlat.assign(mlat, mlat + PM);
    h->mtmax.assign(CM, 0.0);
    for (int c = 0; c < CM; ++c)
      if (d->meas_off[c + 1] > d->meas_off[c])
        h->mtmax[c] = d->meas_tmax ? d->meas_tmax[c] : d->meas_rate[d->meas_off[c + 1] - 1];
  }
  compute_units(h);
  Trace tr;
  tr.mark("validate");
  alp_status s = init_device(h);
  tr.mark("init_device");
  if (s == ALP_OK) s = upload_all(h);
  tr.mark("plan+upload");
  if (s != ALP_OK) {
    delete h;
    return s;
  }
  *out = h;
  return ALP_OK;
}

alp_status alp_build_from_terms(int32_t M, int32_t K, const float *tau, const int32_t *u, alp_t **out) {
  if (!out) return fail(ALP_EINVAL, "out is NULL");
  *out = nullptr;
  if (M < 1 || M > ALP_MAX_M) return fail(ALP_EINVAL, "M must be in 1..%d", ALP_MAX_M);
  if (K < 1 || K > ALP_MAX_K) return fail(ALP_EINVAL, "K must be in 1..%d", ALP_MAX_K);
  if (!tau || !u) return fail(ALP_EINVAL, "tau/u is NULL");
  double bound = 0;
  for (int m = 0; m < M; ++m) {
    double mx = 0;
    for (int k = 0; k < K; ++k) {
      const float t = tau[m * K + k];
      if (std::isnan(t) || t < 0) return fail(ALP_EINVAL, "tau[%d] must be >= 0 or +inf", m * K + k);
      if (u[m * K + k] < 0) return fail(ALP_EINVAL, "u[%d] < 0", m * K + k);
      if (std::isfinite(t)) mx = std::max(mx, (double)t);
    }
    bound += mx;
  }
  if (!(bound < 1e37)) return fail(ALP_EINVAL, "terms could overflow binary32");
  alp_s *h = new alp_s();
  h->from_terms = true;
  h->M = M; h->K = K; h->F = 1; h->nS = 1; h->nT = 1; h->nR = K;
  h->u.assign(u, u + (size_t)M * K);
  h->tau_fixed.assign(tau, tau + (size_t)M * K);
  h->term_fixed.resize((size_t)M * K);
  h->b_fixed.assign((size_t)M * K, INFINITY);
  for (size_t i = 0; i < h->tau_fixed.size(); ++i) h->term_fixed[i] = (double)h->tau_fixed[i];
  h->S = {1};
  h->T = {1};
  h->R.resize(K);
  std::iota(h->R.begin(), h->R.end(), 1);
  alp_status s = init_device(h);
  if (s == ALP_OK) s = upload_all(h);
  if (s != ALP_OK) {
    delete h;
    return s;
  }
  *out = h;
  return ALP_OK;
}

void alp_destroy(alp_t *h) { delete h; }

uint64_t alp_num_candidates(const alp_t *h) { return h ? h->N : 0; }

uint64_t alp_h2d_bytes(const alp_t *h) { return h ? h->h2d : 0; }

alp_status alp_decode(const alp_t *h, uint64_t index, int32_t *s, int32_t *t, int32_t *r) {
  if (!h) return fail(ALP_EINVAL, "handle is NULL");
  if (index >= h->N) return fail(ALP_EINVAL, "index %llu >= N", (unsigned long long)index);
  for (int m = h->M - 1; m >= 0; --m) {
    const int k = (int)(index % (uint64_t)h->K);
    index /= (uint64_t)h->K;
    const int r_i = k % h->nR, t_i = (k / h->nR) % h->nT, s_i = k / (h->nR * h->nT);
    if (s) s[m] = h->S[s_i];
    if (t) t[m] = h->T[t_i];
    if (r) r[m] = h->R[r_i];
  }
  return ALP_OK;
}

alp_status alp_option_table(alp_t *h, double lambda, float *tau, double *term, double *b, int32_t *u) {
  if (!h) return fail(ALP_EINVAL, "handle is NULL");
  alp_status s = check_targets(&lambda, 1);
  if (s != ALP_OK) return s;
  CU(cudaSetDevice(h->device));
  s = use_stream(h, h->stream);
  if (s != ALP_OK) return s;
  s = ensure_scratch(h, 1, h->stream);
  if (s != ALP_OK) return s;
  s = option_tables(h, &lambda, 1, h->stream, nullptr, nullptr);
  if (s != ALP_OK) return s;
  const size_t MK = (size_t)h->M * h->K;
  if (tau) CU(cudaMemcpyAsync(tau, h->sc.tau, MK * sizeof(float), cudaMemcpyDeviceToHost, h->stream));
  if (term) CU(cudaMemcpyAsync(term, h->sc.term, MK * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  if (b) CU(cudaMemcpyAsync(b, h->sc.b, MK * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  if (u) memcpy(u, h->u.data(), MK * sizeof(int32_t));
  return ALP_OK;
}

alp_status alp_predict(alp_t *h, const int32_t *opts, int32_t n, double lambda, int64_t budget, double *latency,
                       double *throughput, int64_t *units, int32_t *feasible) {
  if (!h) return fail(ALP_EINVAL, "handle is NULL");
  if (h->from_terms) return fail(ALP_EINVAL, "alp_predict needs a profile-built handle");
  if (!opts || n < 1) return fail(ALP_EINVAL, "opts: need n >= 1 allocations");
  alp_status s = check_targets(&lambda, 1);
  if (s != ALP_OK) return s;
  for (long long i = 0; i < (long long)n * h->M; ++i)
    if (opts[i] < 0 || opts[i] >= h->K) return fail(ALP_EINVAL, "opts[%lld] out of range 0..K-1", i);
  CU(cudaSetDevice(h->device));
  s = use_stream(h, h->stream);
  if (s != ALP_OK) return s;
  CU(h->d_opts.ensure((size_t)n * h->M));
  CU(h->d_plat.ensure(n));
  CU(h->d_pthr.ensure(n));
  CU(h->d_punits.ensure(n));
  CU(h->d_pfeas.ensure(n));
  CU(cudaMemcpyAsync(h->d_opts.p, opts, (size_t)n * h->M * sizeof(int), cudaMemcpyHostToDevice, h->stream));
  PredictArgs a;
  a.prof = h->dprof();
  a.opts = h->d_opts.p;
  a.n = n;
  a.lambda = lambda;
  a.budget = budget;
  a.latency = h->d_plat.p;
  a.throughput = h->d_pthr.p;
  a.units = h->d_punits.p;
  a.feasible = h->d_pfeas.p;
  CU(launch_predict(a, h->stream));
  if (latency) CU(cudaMemcpyAsync(latency, a.latency, n * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  if (throughput) CU(cudaMemcpyAsync(throughput, a.throughput, n * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  if (units) CU(cudaMemcpyAsync(units, a.units, n * sizeof(long long), cudaMemcpyDeviceToHost, h->stream));
  if (feasible) CU(cudaMemcpyAsync(feasible, a.feasible, n * sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  return ALP_OK;
}

uint64_t alp_num_items(const alp_t *h, int64_t budget_units) {
  (void)budget_units;
  return h ? (uint64_t)h->n_chunks * h->n_groups * h->nQ : 0;
}

alp_status alp_shard_range(const alp_t *h, int64_t budget_units, int32_t rank, int32_t world, uint64_t *lo,
                           uint64_t *hi) {
  if (!h) return fail(ALP_EINVAL, "handle is NULL");
  if (world < 1 || rank < 0 || rank >= world) return fail(ALP_EINVAL, "need 0 <= rank < world");
  if (!lo || !hi) return fail(ALP_EINVAL, "lo/hi is NULL");
  // contiguous ranges of whole rows of nQ items (a lane tile's a-ranges stay on one rank), balanced
  // by estimated cost rather than count: a row of a mixed warp group (lanes with different unit
  // sums: per-lane masked rows on the vector path) costs `wm` rows of a uniform group (x16 integer
  // weights; rows are chunk-major, uniform groups [0, n_groups_u) first in every chunk).
  // Measured on C3 at 8 ranks (slowest rank's step): w = 1.0 0.460, 1.2 0.439, 1.4 0.431, 1.7
  // 0.468 ms; C4 (mostly uniform groups) unchanged.  ALP_SHARD_MIXED=w overrides (1 = by count).
  static const int wm16 = [] {
    const char *v = getenv("ALP_SHARD_MIXED");
    return v ? std::max(1, (int)std::lround(16.0 * atof(v))) : 22;  // 1.375
  }();
  const uint64_t nq = h->nQ, rows = alp_num_items(h, budget_units) / nq;
  const uint64_t ng = h->n_groups, ngu = std::min<uint64_t>(h->n_groups_u, ng);
  // Short b rows (k_search_u's full-row loop, Kb <= 20): a uniform group's row is cheaper when even
  // the a option with the most units leaves it the widest masked row (1.05 vs 1.17 instructions per
  // candidate), which depends on the chunk's prefix units: per-chunk weights, rows of a uniform
  // partial group weigh `wp` (ALP_SHARD_PARTIAL, default 1.125).
  static const int wp16 = [] {
    const char *v = getenv("ALP_SHARD_PARTIAL");
    return v ? std::max(1, (int)std::lround(16.0 * atof(v))) : 18;
  }();
  if (h->Kb <= 20 && h->g0 >= 1 && ng > 0 && rows % ng == 0 && (uint64_t)h->n_chunks == rows / ng &&
      h->gsum.size() >= ng && wp16 != 16) {
    const long long R = std::min<long long>(budget_units, h->umax_total);
    int ubw = 0;  // widest row: every b option with u <= R
    for (int k = 0; k < h->K; ++k) {
      const int ub = h->u[(size_t)h->b_llm * h->K + k];
      if (ub <= R) ubw = std::max(ubw, ub);
    }
    const long long amax = h->a_llm >= 0 ? std::min<long long>(h->umax_a, R + 1) : 0;
    std::vector<int> gs_sorted(h->gsum.begin(), h->gsum.begin() + ngu);
    std::sort(gs_sorted.begin(), gs_sorted.end());
    const uint64_t nc = h->n_chunks;
    std::vector<long long> thr(nc);
    std::vector<uint64_t> wcum(nc + 1, 0);
    for (uint64_t c = 0; c < nc; ++c) {
      long long upfx = 0;
      for (int m = 0; m < h->g0; ++m) upfx += h->u[(size_t)m * h->K + (c / h->pw[m]) % (uint64_t)h->K];
      thr[c] = R - upfx - amax - ubw;  // a uniform group of unit sum gs is full-row iff gs <= thr
      const uint64_t nfull = thr[c] < 0 ? 0 : (uint64_t)(std::upper_bound(gs_sorted.begin(), gs_sorted.end(), (int)std::min<long long>(thr[c], INT32_MAX)) - gs_sorted.begin());
      wcum[c + 1] = wcum[c] + 16 * nfull + (uint64_t)wp16 * (ngu - nfull) + (uint64_t)wm16 * (ng - ngu);
    }
    auto bound = [&](uint64_t r) -> uint64_t {
      if (r == 0) return 0;
      if (r >= (uint64_t)world) return rows;
      const unsigned __int128 tgt = (unsigned __int128)wcum[nc] * r / (uint64_t)world;
      const uint64_t c = (uint64_t)(std::upper_bound(wcum.begin(), wcum.end(), (uint64_t)tgt) - wcum.begin()) - 1;
      if (c >= nc) return rows;
      uint64_t acc = wcum[c], g = 0;
      while (g < ng && acc < (uint64_t)tgt) {
        acc += g >= ngu ? (uint64_t)wm16 : (h->gsum[g] <= thr[c] ? 16u : (uint64_t)wp16);
        ++g;
      }
      return c * ng + g;
    };
    *lo = bound((uint64_t)rank) * nq;
    *hi = bound((uint64_t)rank + 1) * nq;
    return ALP_OK;
  }
  const uint64_t wchunk = 16 * ngu + (uint64_t)wm16 * (ng - ngu), total = wchunk * (rows / std::max<uint64_t>(ng, 1));
  auto bound = [&](uint64_t r) -> uint64_t {  // first row whose cumulative cost reaches r / world of the total
    if (r == 0 || ng == 0 || rows % ng != 0) return r * (rows / (uint64_t)world) + std::min<uint64_t>(r, rows % (uint64_t)world);
    if (r >= (uint64_t)world) return rows;
    const unsigned __int128 tgt = (unsigned __int128)total * r / (uint64_t)world;
    const uint64_t chunk = (uint64_t)(tgt / wchunk), rem = (uint64_t)(tgt % wchunk);
    const uint64_t g = rem <= 16 * ngu ? (rem + 15) / 16 : ngu + (rem - 16 * ngu + wm16 - 1) / wm16;
    return std::min<uint64_t>(rows, chunk * ng + g);
  };
  *lo = bound((uint64_t)rank) * nq;
  *hi = bound((uint64_t)rank + 1) * nq;
  return ALP_OK;
}

size_t alp_workspace_bytes(const alp_t *h, int32_t n_targets) {
  if (!h || n_targets < 1) return 0;
  return ws_layout(h, n_targets, nullptr, nullptr);
}

// every result of the call that found nothing gets the candidate with the maximal
// Eq. 2 T_w within its budget (k_max_throughput on the call's option table; once per budget).
static alp_status apply_fallbacks(alp_s *h, int n, const int64_t *budgets, int64_t budget, alp_result *out,
                                  cudaStream_t st, alp_status s) {
  if (s != ALP_OK && s != ALP_EINFEASIBLE) return s;
  if (h->from_terms) return s;
  std::map<long long, alp_result> memo;
  for (int i = 0; i < n; ++i) {
    if (out[i].found) continue;
    const long long B = budgets ? budgets[i] : budget;
    auto it = memo.find(B);
    if (it == memo.end()) {
      alp_result *host = nullptr, *dres = zero_copy_out(1, &host);
      if (!dres) return fail(ALP_ECUDA, "no mapped pinned memory for the fallback result");
      CU(launch_max_throughput(h->sc.b, h->d_u, h->dprof(), B, h->N, dres, st));
      CU(cudaStreamSynchronize(st));
      it = memo.emplace(B, *host).first;
    }
    const alp_result &f = it->second;
    out[i].fallback = f.fallback;
    if (f.fallback) {
      out[i].index = f.index;
      out[i].units = f.units;
      out[i].throughput = f.throughput;
      for (int m = 0; m < ALP_MAX_M; ++m) {
        out[i].share_units[m] = f.share_units[m];
        out[i].tp[m] = f.tp[m];
        out[i].replicas[m] = f.replicas[m];
      }
    }
  }
  return s;
}

alp_status alp_search_shard(alp_t *h, const double *targets, int32_t n, int64_t budget_units, uint64_t lo,
                            uint64_t hi, void *d_workspace, void *stream, int64_t *d_keys, int64_t *d_counts) {
  NvtxRange nv("alp_search_shard");
  if (!h) return fail(ALP_EINVAL, "handle is NULL");
  if (!d_keys || !d_counts) return fail(ALP_EINVAL, "d_keys/d_counts is NULL");
  return search_shard_impl(h, targets, nullptr, n, budget_units, lo, hi, stream ? (cudaStream_t)stream : h->stream,
                           reinterpret_cast<unsigned long long *>(d_keys),
                           reinterpret_cast<unsigned long long *>(d_counts), false, nullptr, true, d_workspace);
}

alp_status alp_finalize(alp_t *h, const double *targets, int32_t n, int64_t budget_units, const int64_t *d_keys,
                        const int64_t *d_counts, void *d_workspace, void *stream, alp_result *out) {
  NvtxRange nv("alp_finalize");
  if (!h) return fail(ALP_EINVAL, "handle is NULL");
  if (!d_keys || !d_counts) return fail(ALP_EINVAL, "d_keys/d_counts is NULL");
  alp_status s = check_targets(targets, n);
  if (s != ALP_OK) return s;
  cudaStream_t st = stream ? (cudaStream_t)stream : h->stream;
  s = finalize_impl(h, targets, nullptr, n, budget_units, reinterpret_cast<const unsigned long long *>(d_keys),
                    reinterpret_cast<const unsigned long long *>(d_counts), st, out, 0, d_workspace);
  return apply_fallbacks(h, n, nullptr, budget_units, out, st, s);
}

alp_status alp_finalize_gathered(alp_t *h, const double *targets, int32_t n, int64_t budget_units,
                                 const int64_t *d_gathered, int32_t world, void *d_workspace, void *stream,
                                 alp_result *out) {
  NvtxRange nv("alp_finalize_gathered");
  if (!h) return fail(ALP_EINVAL, "handle is NULL");
  if (!d_gathered) return fail(ALP_EINVAL, "d_gathered is NULL");
  if (world < 1) return fail(ALP_EINVAL, "world must be >= 1");
  alp_status s = check_targets(targets, n);
  if (s != ALP_OK) return s;
  cudaStream_t st = stream ? (cudaStream_t)stream : h->stream;
  s = finalize_impl(h, targets, nullptr, n, budget_units, reinterpret_cast<const unsigned long long *>(d_gathered),
                    nullptr, st, out, world, d_workspace);
  return apply_fallbacks(h, n, nullptr, budget_units, out, st, s);
}

size_t alp_peer_bytes(int32_t n_targets, int32_t world) {
  if (n_targets < 1 || world < 1) return 0;
  return kPeerHdr + 2 * (size_t)world * n_targets * sizeof(PeerRow);
}

alp_status alp_peer_alloc(size_t bytes, void **d_buf) {
  if (!d_buf || bytes < kPeerHdr) return fail(ALP_EINVAL, "d_buf is NULL or bytes < alp_peer_bytes");
  *d_buf = nullptr;
  void *p = nullptr;
  CU(cudaMalloc(&p, bytes));  // a whole allocation of its own: IPC handles name allocations
  cudaError_t e = cudaMemset(p, 0, bytes);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    cudaFree(p);
    return fail(ALP_ECUDA, "alp_peer_alloc: %s", cudaGetErrorString(e));
  }
  *d_buf = p;
  return ALP_OK;
}

alp_status alp_peer_free(void *d_buf) {
  if (d_buf) CU(cudaFree(d_buf));
  return ALP_OK;
}

alp_status alp_peer_ipc_handle(void *d_buf, void *handle) {
  if (!d_buf || !handle) return fail(ALP_EINVAL, "d_buf/handle is NULL");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "64-byte IPC handles");
  cudaIpcMemHandle_t hd;
  CU(cudaIpcGetMemHandle(&hd, d_buf));
  memcpy(handle, &hd, sizeof(hd));
  return ALP_OK;
}

alp_status alp_peer_open(const void *handle, void **d_peer) {
  if (!handle || !d_peer) return fail(ALP_EINVAL, "handle/d_peer is NULL");
  *d_peer = nullptr;
  cudaIpcMemHandle_t hd;
  memcpy(&hd, handle, sizeof(hd));
  CU(cudaIpcOpenMemHandle(d_peer, hd, cudaIpcMemLazyEnablePeerAccess));
  return ALP_OK;
}

alp_status alp_peer_close(void *d_peer) {
  if (d_peer) CU(cudaIpcCloseMemHandle(d_peer));
  return ALP_OK;
}

alp_status alp_search_peer(alp_t *h, const double *targets, int32_t n, int64_t budget_units, uint64_t lo,
                           uint64_t hi, int32_t rank, int32_t world, void *const *d_bufs, void *d_workspace,
                           void *stream, alp_result *out) {
  NvtxRange nv("alp_search_peer");
  if (!h) return fail(ALP_EINVAL, "handle is NULL");
  if (!out) return fail(ALP_EINVAL, "out is NULL");
  if (!d_bufs) return fail(ALP_EINVAL, "d_bufs is NULL");
  if (world < 1 || world > kMaxPeers) return fail(ALP_EINVAL, "world must be in [1, %d]", kMaxPeers);
  if (rank < 0 || rank >= world) return fail(ALP_EINVAL, "rank %d outside [0, %d)", rank, world);
  alp_status s = check_targets(targets, n);
  if (s != ALP_OK) return s;
  if (n > kInlineTargets) return fail(ALP_EINVAL, "peer exchange: at most %d targets per call", kInlineTargets);
  PeerArgs pa{};
  pa.on = 1;
  pa.rank = rank;
  pa.world = world;
  for (int j = 0; j < world; ++j) {
    if (!d_bufs[j]) return fail(ALP_EINVAL, "d_bufs[%d] is NULL", j);
    pa.buf[j] = static_cast<unsigned char *>(d_bufs[j]);
  }
  static const long long timeout_ms = getenv("ALP_PEER_TIMEOUT_MS") ? atoll(getenv("ALP_PEER_TIMEOUT_MS")) : 30000;
  pa.timeout_ns = timeout_ms * 1000000ll;
  alp_result *hzc = nullptr, *zc = zero_copy_out(n, &hzc);
  if (!zc) return fail(ALP_ECUDA, "no mapped pinned memory for %d results", n);
  pa.out = zc;
  cudaStream_t st = stream ? (cudaStream_t)stream : h->stream;
  s = search_shard_impl(h, targets, nullptr, n, budget_units, lo, hi, st, nullptr, nullptr, false, nullptr, true,
                        d_workspace, &pa);
  if (s != ALP_OK) return s;
  s = collect_results(h, n, st, out, hzc);
  for (int t = 0; t < n; ++t)
    if (out[t].found < 0) return fail(ALP_EINTERNAL, "peer exchange timed out (rank %d of %d)", rank, world);
  return apply_fallbacks(h, n, nullptr, budget_units, out, st, s);
}

// One target, n budgets: the one-pass budget-indexed search (alp_levels.cu) — every candidate with
// units <= the largest budget evaluated once (instead of one exhaustive pass per budget), then K3
// per budget.  Returns ALP_EINTERNAL + no error message when the plan does not allow it (the caller
// falls back to the per-query passes): non-default rows per lane, coarse segments, > 4096 distinct
// budgets or a largest budget above 16384 units.
static alp_status budget_sweep(alp_s *h, double target, const int64_t *budgets, int n, alp_result *out, bool *done) {
  *done = false;
  static const bool off = getenv("ALP_NO_LEVELS") != nullptr;  // A/B switch: per-query passes
  if (off || h->from_terms || h->rows_per_lane != 12 || n < 2 ||
      (uint64_t)h->n_chunks * h->L * (uint64_t)h->Ka >= 0xffffffffull)
    return ALP_OK;
  std::vector<int> lv;
  for (int i = 0; i < n; ++i) {
    if (budgets[i] < 0) return fail(ALP_EINVAL, "budgets[%d] < 0", i);
    lv.push_back((int)std::min<int64_t>(budgets[i], h->umax_total));
  }
  std::sort(lv.begin(), lv.end());
  lv.erase(std::unique(lv.begin(), lv.end()), lv.end());
  const int L = (int)lv.size(), bmax = lv.back();
  if (L > 4096 || bmax > 16384) return ALP_OK;
  std::vector<int> ql(n);
  for (int i = 0; i < n; ++i)
    ql[i] = (int)(std::lower_bound(lv.begin(), lv.end(), (int)std::min<int64_t>(budgets[i], h->umax_total)) - lv.begin());
  std::vector<double> tg(n, target);
  cudaStream_t st = h->stream;
  alp_status s = use_stream(h, st);
  if (s != ALP_OK) return s;
  CU(cudaEventRecord(h->evs0, st));
  s = ensure_scratch(h, n, st);
  if (s != ALP_OK) return s;
  h->s_qb = nullptr;
  s = option_tables(h, tg.data(), n, st, h->sc.keys, h->sc.counts);  // K1: the terms of every query (= target)
  if (s != ALP_OK) return s;
  Geometry g;
  s = make_geometry(h, 1, bmax, 0, 0, g);
  if (s != ALP_OK) return s;
  const uint64_t items = (uint64_t)h->n_chunks * h->n_groups * h->nQ;
  g.a.item_lo = 0;
  g.a.item_hi = items;
  g.a.tau = h->sc.tau;
  // scratch: level keys [L], ticket, histograms 2 x [bmax + 1], levels [L], query levels [n]
  const size_t nb = 8 * (size_t)L + 8 + 16 * (size_t)(bmax + 1) + 4 * (size_t)L + 4 * (size_t)n + 64;
  CU(h->g_lv.ensure(nb));
  unsigned char *p = h->g_lv.p;
  auto take = [&](size_t bytes) {
    unsigned char *r = p;
    p += (bytes + 7) & ~size_t(7);
    return r;
  };
  auto *lkeys = reinterpret_cast<unsigned long long *>(take(8 * (size_t)L));
  auto *ticket = reinterpret_cast<unsigned long long *>(take(8));
  auto *h0 = reinterpret_cast<unsigned long long *>(take(8 * (size_t)(bmax + 1)));
  auto *h1 = reinterpret_cast<unsigned long long *>(take(8 * (size_t)(bmax + 1)));
  auto *d_lv = reinterpret_cast<int *>(take(4 * (size_t)L));
  auto *d_ql = reinterpret_cast<int *>(take(4 * (size_t)n));
  CU(cudaMemcpyAsync(d_lv, lv.data(), 4 * (size_t)L, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(d_ql, ql.data(), 4 * (size_t)n, cudaMemcpyHostToDevice, st));
  CU(cudaEventRecord(h->ev0, st));
  CU(launch_levels(g.a, d_lv, L, bmax, lkeys, ticket, d_ql, n, h->sc.keys, h->sc.counts, h0, h1, h->sm_count, st));
  CU(cudaEventRecord(h->ev1, st));
  h->ev_pending = true;
  h->last_ur = false;
  s = finalize_impl(h, tg.data(), budgets, n, 0, h->sc.keys, h->sc.counts, st, out);
  h->last_launches = 4;  // K1, search, finish, K3
  if (s == ALP_OK || s == ALP_EINFEASIBLE) *done = true;
  return s;
}

static alp_status search_queries_core(alp_t *h, const double *targets, const int64_t *budgets, int32_t n,
                                      int64_t budget_units, alp_result *out);

static alp_status search_queries(alp_t *h, const double *targets, const int64_t *budgets, int32_t n,
                                 int64_t budget_units, alp_result *out) {
  alp_status s = search_queries_core(h, targets, budgets, n, budget_units, out);
  if (s != ALP_OK && s != ALP_EINFEASIBLE) return s;
  return apply_fallbacks(h, n, budgets, budget_units, out, h->stream, s);
}

static alp_status search_queries_core(alp_t *h, const double *targets, const int64_t *budgets, int32_t n,
                                      int64_t budget_units, alp_result *out) {
  NvtxRange nv("alp_search");
  if (!h) return fail(ALP_EINVAL, "handle is NULL");
  if (!out) return fail(ALP_EINVAL, "out is NULL");
  alp_status s = check_targets(targets, n);
  if (s != ALP_OK) return s;
  CU(cudaSetDevice(h->device));
  s = ensure_scratch(h, n, h->stream);
  if (s != ALP_OK) return s;
  if (budgets && n >= 2) {  // one target, several budgets: the one-pass budget-indexed search
    bool same = true;
    for (int i = 1; i < n; ++i) same &= targets[i] == targets[0];
    if (same) {
      bool done = false;
      s = budget_sweep(h, targets[0], budgets, n, out, &done);
      if (done || (s != ALP_OK && s != ALP_EINFEASIBLE)) return s;
    }
  }
  const uint64_t items = alp_num_items(h, budget_units);
  const int ug = budgets ? 0 : ur_batch_group(h, budget_units);
  if (n > kInlineTargets && ug > 0) {
    // large batches (C5) on the uniform-register path: groups of ug targets, each one k_uprep +
    // k_search_u pair with the finalize fused; the results land zero-copy, one sync at the end
    alp_result *hzc = nullptr, *zc = zero_copy_out(n, &hzc);
    if (!zc) return fail(ALP_ECUDA, "no mapped pinned memory for %d results", n);
    int launches = 0;
    for (int i = 0; i < n; i += ug) {
      const int g = std::min(ug, n - i);
      s = search_shard_impl(h, targets + i, nullptr, g, budget_units, 0, items, h->stream, h->sc.keys, h->sc.counts,
                            true, zc + i, i == 0);
      if (s != ALP_OK) return s;
      launches += h->last_launches;
    }
    h->last_launches = launches;
    return collect_results(h, n, h->stream, out, hzc);
  }
  if (use_fused(h, n, budgets)) {  // one launch: terms + search + finalize
    alp_result *hzc = nullptr, *zc = zero_copy_out(n, &hzc);  // the last block stores the results
    s = search_shard_impl(h, targets, nullptr, n, budget_units, 0, items, h->stream, h->sc.keys, h->sc.counts, true,
                          zc);
    if (s != ALP_OK) return s;
    return collect_results(h, n, h->stream, out, hzc);
  }
  s = search_shard_impl(h, targets, budgets, n, budget_units, 0, items, h->stream, h->sc.keys, h->sc.counts);
  if (s != ALP_OK) return s;
  return finalize_impl(h, targets, budgets, n, budget_units, h->sc.keys, h->sc.counts, h->stream, out);
}

alp_status alp_search_batch(alp_t *h, const double *targets, int32_t n, int64_t budget_units, alp_result *out) {
  return search_queries(h, targets, nullptr, n, budget_units, out);
}

alp_status alp_search_queries(alp_t *h, const double *targets, const int64_t *budgets, int32_t n, alp_result *out) {
  if (!budgets) return fail(ALP_EINVAL, "budgets is NULL");
  return search_queries(h, targets, budgets, n, 0, out);
}

alp_status alp_search(alp_t *h, double target, int64_t budget_units, alp_result *out) {
  return alp_search_batch(h, &target, 1, budget_units, out);
}

alp_status alp_schedule_egalitarian(alp_t *const *hs, const double *targets, int32_t W, int32_t gpus,
                                    int32_t units_per_gpu, int32_t *gpus_out, alp_result *results_out,
                                    double *min_utility, double *sum_utility) {
  if (!hs || !targets || !gpus_out || !results_out) return fail(ALP_EINVAL, "NULL argument");
  if (W < 1 || W > ALP_MAX_M) return fail(ALP_EINVAL, "W must be in 1..%d", ALP_MAX_M);
  if (gpus < 0 || gpus > 4096) return fail(ALP_EINVAL, "gpus must be in 0..4096");
  if (units_per_gpu < 1) return fail(ALP_EINVAL, "units_per_gpu must be >= 1");
  double splits = 1;
  for (int w = 0; w + 1 < W; ++w) splits *= (gpus + 1);
  if (splits > 1e8) return fail(ALP_EINVAL, "too many GPU splits (%.3g)", splits);
  for (int w = 0; w < W; ++w) {
    if (!hs[w]) return fail(ALP_EINVAL, "hs[%d] is NULL", w);
    if (hs[w]->device != hs[0]->device) return fail(ALP_EINVAL, "all handles must live on one device");
  }
  // budget-indexed search per workflow: the best allocation on g = 0..G GPUs
  const int G = gpus;
  std::vector<int64_t> budgets(G + 1);
  for (int g = 0; g <= G; ++g) budgets[g] = (int64_t)g * units_per_gpu;
  std::vector<double> lat((size_t)W * (G + 1));
  std::vector<std::vector<alp_result>> per(W, std::vector<alp_result>(G + 1));
  for (int w = 0; w < W; ++w) {
    std::vector<double> tg(G + 1, targets[w]);
    alp_status s = search_queries(hs[w], tg.data(), budgets.data(), G + 1, 0, per[w].data());
    if (s != ALP_OK && s != ALP_EINFEASIBLE) return s;
    for (int g = 0; g <= G; ++g) lat[(size_t)w * (G + 1) + g] = per[w][g].found ? per[w][g].latency : INFINITY;
  }
  alp_s *h0 = hs[0];
  CU(cudaSetDevice(h0->device));
  DBuf<double> d_lat, d_out;
  DBuf<long long> d_idx;
  CU(d_lat.ensure(lat.size()));
  CU(d_out.ensure(2));
  CU(d_idx.ensure(1));
  CU(cudaMemcpyAsync(d_lat.p, lat.data(), lat.size() * sizeof(double), cudaMemcpyHostToDevice, h0->stream));
  CU(launch_egalitarian(d_lat.p, W, G, d_idx.p, d_out.p, d_out.p + 1, h0->stream));
  long long idx = -1;
  double mm[2] = {0, 0};
  CU(cudaMemcpyAsync(&idx, d_idx.p, sizeof(idx), cudaMemcpyDeviceToHost, h0->stream));
  CU(cudaMemcpyAsync(mm, d_out.p, sizeof(mm), cudaMemcpyDeviceToHost, h0->stream));
  CU(cudaStreamSynchronize(h0->stream));
  d_lat.release();
  d_out.release();
  d_idx.release();
  if (idx < 0) return fail(ALP_EINTERNAL, "no split evaluated");
  int used = 0;
  for (int w = W - 2; w >= 0; --w) {
    gpus_out[w] = (int32_t)(idx % (G + 1));
    idx /= (G + 1);
    used += gpus_out[w];
  }
  gpus_out[W - 1] = G - used;
  bool all = true;
  for (int w = 0; w < W; ++w) {
    results_out[w] = per[w][gpus_out[w]];
    all &= results_out[w].found != 0;
  }
  if (min_utility) *min_utility = mm[0];
  if (sum_utility) *sum_utility = mm[1];
  return all ? ALP_OK : ALP_EINFEASIBLE;
}

alp_status alp_workflow_stats(int32_t n_req, int32_t M, int64_t n_inv, const int32_t *req, const int32_t *llm,
                              const double *start, const double *end, double *n_out, double *p_out) {
  if (n_req < 1) return fail(ALP_EINVAL, "n_req must be >= 1 (empty trace list)");
  if (M < 1 || M > ALP_MAX_M) return fail(ALP_EINVAL, "M must be in 1..%d", ALP_MAX_M);
  if (n_inv < 0 || (n_inv > 0 && (!req || !llm || !start || !end))) return fail(ALP_EINVAL, "NULL invocation arrays");
  if (!n_out || !p_out) return fail(ALP_EINVAL, "n_out/p_out is NULL");
  for (int64_t i = 0; i < n_inv; ++i) {
    if (req[i] < 0 || req[i] >= n_req) return fail(ALP_EINVAL, "req[%lld] out of range", (long long)i);
    if (llm[i] < 0 || llm[i] >= M) return fail(ALP_EINVAL, "llm[%lld] out of range", (long long)i);
    if (!std::isfinite(start[i]) || !std::isfinite(end[i]) || end[i] < start[i])
      return fail(ALP_EINVAL, "invocation %lld: need finite start <= end", (long long)i);
  }
  // group invocations by (request, LLM), sorted by start; per group: summed durations and the length
  // of the union of the intervals (busy time).  p_m = sum_r dur_rm / sum_r busy_rm, i.e. the
  // busy-time-weighted average over requests of the time-averaged concurrency.
  std::vector<int64_t> order(n_inv);
  std::iota(order.begin(), order.end(), (int64_t)0);
  std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
    if (req[a] != req[b]) return req[a] < req[b];
    if (llm[a] != llm[b]) return llm[a] < llm[b];
    if (start[a] != start[b]) return start[a] < start[b];
    return a < b;
  });
  std::vector<double> dur(M, 0.0), busy(M, 0.0);
  std::vector<int64_t> cnt(M, 0);
  for (int64_t i = 0; i < n_inv;) {
    const int r = req[order[i]], m = llm[order[i]];
    double lo = start[order[i]], hi = end[order[i]], d = 0.0, b = 0.0;
    int64_t j = i;
    for (; j < n_inv && req[order[j]] == r && llm[order[j]] == m; ++j) {
      const int64_t k = order[j];
      d += end[k] - start[k];
      if (start[k] > hi) {  // gap: close the current busy run
        b += hi - lo;
        lo = start[k];
        hi = end[k];
      } else if (end[k] > hi) {
        hi = end[k];
      }
    }
    b += hi - lo;
    dur[m] += d;
    busy[m] += b;
    cnt[m] += j - i;
    i = j;
  }
  for (int m = 0; m < M; ++m) {
    n_out[m] = (double)cnt[m] / (double)n_req;
    p_out[m] = busy[m] > 0.0 ? dur[m] / busy[m] : 1.0;  // never invoked / zero-length busy: 1
  }
  return ALP_OK;
}

// Topology-aware placement of a chosen allocation (PAPER.md:411-416
// "Hierarchical placement algorithm"; tie-breaks and the imbalance definition from).
//
// Host code (alp_place): the placement is a short sequential heuristic over a handful of shards (the paper
// calls the optimum NP-hard and uses this greedy; it runs once per chosen allocation).  Every replica of
// LLM m is a tensor group of tp_m shards demanding share_units_m units each.  Two stages (PAPER.md:413
// "first places LLMs into nodes while prioritizing larger instances (inter-node stage), and then assigns
// GPU fractions within a node (intra-node stage)"):
//  * inter-node: groups most-constrained-first (tensor-parallel groups before single shards, larger total
//    demand first, then (LLM, replica)).  A tensor group goes to one NVLink domain: among domains with tp
//    free GPUs of enough capacity keep those with the smallest imbalance (max - min free units over the
//    domain's GPUs), then the least total free capacity, then the lowest (node, domain) -- its node is
//    the domain's.  A single shard goes to the node with the least free units among the nodes that still
//    have a GPU it fits on (occupied nodes first), lowest node on ties;
//  * intra-node: each node re-places its own groups from scratch -- its tensor groups in the same order
//    and scoring restricted to its domains (the tp GPUs with the least sufficient free units), then its
//    single shards largest first onto already occupied GPUs first, best fit by free units, lowest GPU on
//    ties.  Should a node's re-placement fail, the node keeps its inter-node stage GPUs (always valid).
namespace {
struct PlaceGroup {
  int m, r, tp, units, first;  // first = index of the group's first shard in shard_gpu
};

// Domain choice + GPUs for a tensor group over the given domains (free_units updated); false if none fits.
bool place_tensor(const PlaceGroup &grp, const std::map<std::pair<int, int>, std::vector<int>> &domains, int node_only,
                  int F, std::vector<int> &free_units, std::vector<int> &gpus) {
  const std::vector<int> *best = nullptr;
  long long best_imb = 0, best_cap = 0;
  for (const auto &kv : domains) {
    if (node_only >= 0 && kv.first.first != node_only) continue;
    const std::vector<int> &gs = kv.second;
    int fit = 0, mx = 0, mn = F;
    long long cap = 0;
    for (int g : gs) {
      fit += free_units[g] >= grp.units;
      mx = std::max(mx, free_units[g]);
      mn = std::min(mn, free_units[g]);
      cap += free_units[g];
    }
    if (fit < grp.tp) continue;
    const long long imb = mx - mn;
    if (!best || imb < best_imb || (imb == best_imb && cap < best_cap)) {
      best = &gs;
      best_imb = imb;
      best_cap = cap;
    }
  }
  if (!best) return false;
  std::vector<int> cand;
  for (int g : *best)
    if (free_units[g] >= grp.units) cand.push_back(g);
  // the tp GPUs with the MOST free units (lowest index on ties): keeps the domain balanced, which is
  // what its score rewards; taking the least sufficient ones stacks groups on the same GPUs and
  // strands the rest (3 tp-2 groups on a 3-GPU domain of 2 units each: (0,1),(0,1) then nothing fits)
  std::stable_sort(cand.begin(), cand.end(), [&](int a, int b) { return free_units[a] > free_units[b]; });
  gpus.assign(cand.begin(), cand.begin() + grp.tp);
  std::sort(gpus.begin(), gpus.end());
  for (int g : gpus) free_units[g] -= grp.units;
  return true;
}

// Single shard onto one of `gs` (index order): occupied GPUs first, best fit by free units; -1 if none fits.
int place_single(int units, const std::vector<int> &gs, int F, std::vector<int> &free_units) {
  int pick = -1;
  for (int pass = 0; pass < 2 && pick < 0; ++pass)
    for (int g : gs) {
      const bool occupied = free_units[g] < F;
      if ((pass == 0) != occupied || free_units[g] < units) continue;
      if (pick < 0 || free_units[g] < free_units[pick]) pick = g;
    }
  if (pick >= 0) free_units[pick] -= units;
  return pick;
}
}  // namespace

alp_status alp_place(int32_t G, int32_t F, const int32_t *gpu_node, const int32_t *gpu_domain, int32_t M,
                     const int32_t *share_units, const int32_t *tp, const int32_t *replicas, int32_t *shard_gpu) {
  if (G < 1 || F < 1) return fail(ALP_EINVAL, "need G >= 1 GPUs and F >= 1 units per GPU");
  if (!gpu_node || !gpu_domain || !share_units || !tp || !replicas || !shard_gpu)
    return fail(ALP_EINVAL, "NULL argument");
  if (M < 1) return fail(ALP_EINVAL, "M must be >= 1");
  std::map<int, int> dom_node;
  for (int g = 0; g < G; ++g) {
    auto it = dom_node.find(gpu_domain[g]);
    if (it != dom_node.end() && it->second != gpu_node[g])
      return fail(ALP_EINVAL, "NVLink domain %d spans nodes", gpu_domain[g]);
    dom_node[gpu_domain[g]] = gpu_node[g];
  }
  std::vector<PlaceGroup> groups;
  int shards = 0;
  long long demand = 0;
  for (int m = 0; m < M; ++m) {
    if (share_units[m] < 1 || share_units[m] > F || tp[m] < 1 || replicas[m] < 1)
      return fail(ALP_EINVAL, "LLM %d: need 1 <= share_units <= F, tp >= 1, replicas >= 1", m);
    for (int r = 0; r < replicas[m]; ++r) {
      groups.push_back({m, r, tp[m], share_units[m], shards});
      shards += tp[m];
      demand += (long long)tp[m] * share_units[m];
    }
  }
  if (demand > (long long)G * F)
    return fail(ALP_EINFEASIBLE, "demand %lld units exceeds the cluster's %lld", demand, (long long)G * F);
  std::stable_sort(groups.begin(), groups.end(), [](const PlaceGroup &a, const PlaceGroup &b) {
    const bool ta = a.tp > 1, tb = b.tp > 1;
    if (ta != tb) return ta;
    const long long ua = (long long)a.tp * a.units, ub = (long long)b.tp * b.units;
    if (ua != ub) return ua > ub;
    return a.m != b.m ? a.m < b.m : a.r < b.r;
  });
  // domains in (node, domain id) order with their GPUs in index order; nodes with their GPUs
  std::map<std::pair<int, int>, std::vector<int>> domains;
  std::map<int, std::vector<int>> nodes;
  for (int g = 0; g < G; ++g) {
    domains[{gpu_node[g], gpu_domain[g]}].push_back(g);
    nodes[gpu_node[g]].push_back(g);
  }
  // ---- inter-node stage: a node for every group (GPUs tentatively, for the capacity accounting)
  std::vector<int> free_units(G, F), group_node(groups.size());
  std::vector<int> gpus;
  for (size_t i = 0; i < groups.size(); ++i) {
    const PlaceGroup &grp = groups[i];
    if (grp.tp > 1) {
      if (!place_tensor(grp, domains, -1, F, free_units, gpus))
        return fail(ALP_EINFEASIBLE, "no NVLink domain fits LLM %d replica %d (tp %d x %d units)", grp.m, grp.r,
                    grp.tp, grp.units);
      for (int s = 0; s < grp.tp; ++s) shard_gpu[grp.first + s] = gpus[s];
      group_node[i] = gpu_node[gpus[0]];
    } else {
      int best = -1;
      long long best_free = 0;
      for (const auto &kv : nodes) {
        long long fr = 0;
        bool fits = false;
        for (int g : kv.second) {
          fr += free_units[g];
          fits |= free_units[g] >= grp.units;
        }
        if (fits && (best < 0 || fr < best_free)) {
          best = kv.first;
          best_free = fr;
        }
      }
      const int g = best < 0 ? -1 : place_single(grp.units, nodes[best], F, free_units);
      if (g < 0) return fail(ALP_EINFEASIBLE, "no GPU fits LLM %d replica %d (%d units)", grp.m, grp.r, grp.units);
      shard_gpu[grp.first] = g;
      group_node[i] = best;
    }
  }
  // ---- intra-node stage: every node re-places its groups; kept when all of them fit
  for (const auto &kv : nodes) {
    const int n = kv.first;
    std::vector<int> fu(G, 0);
    for (int g : kv.second) fu[g] = F;
    std::vector<std::pair<size_t, std::vector<int>>> mine;  // (group, GPUs)
    bool ok = true;
    std::vector<size_t> singles;
    for (size_t i = 0; i < groups.size() && ok; ++i) {
      if (group_node[i] != n) continue;
      if (groups[i].tp > 1) {
        ok = place_tensor(groups[i], domains, n, F, fu, gpus);
        if (ok) mine.push_back({i, gpus});
      } else {
        singles.push_back(i);
      }
    }
    std::stable_sort(singles.begin(), singles.end(),
                     [&](size_t a, size_t b) { return groups[a].units > groups[b].units; });
    for (size_t i : singles) {
      if (!ok) break;
      const int g = place_single(groups[i].units, kv.second, F, fu);
      ok = g >= 0;
      if (ok) mine.push_back({i, {g}});
    }
    if (!ok) continue;  // keep the inter-node stage's GPUs for this node
    for (const auto &x : mine)
      for (int s = 0; s < (int)x.second.size(); ++s) shard_gpu[groups[x.first].first + s] = x.second[s];
  }
  return ALP_OK;
}


float alp_last_kernel_ms(const alp_t *h) {
  if (!h) return 0.f;
  alp_s *m = const_cast<alp_s *>(h);
  if (m->ev_pending && cudaEventSynchronize(m->ev1) == cudaSuccess) {
    cudaEventElapsedTime(&m->last_ms, m->ev0, m->ev1);
    m->ev_pending = false;
  }
  return m->last_ms;
}

int32_t alp_last_launches(const alp_t *h) { return h ? h->last_launches : 0; }

int32_t alp_last_path(const alp_t *h) { return h ? (h->last_ur ? 1 : 0) : -1; }

float alp_last_step_ms(const alp_t *h) { return h ? h->last_step_ms : 0.f; }

void alp_plan_cache_clear(void) {
  std::lock_guard<std::mutex> lock(g_plan_mu);
  g_plans.clear();
}

}  // extern "C"
