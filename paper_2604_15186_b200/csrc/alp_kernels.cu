// sm_100a kernels of the exhaustive ALP allocation search (Scepsy, arXiv 2604.15186).
//
//   K1 k_option_table  per (target, LLM, option): FP64 option terms of PAPER.md:355-359
//                      (Eq. 1 term, Eq. 2 term, feasibility) -> binary32 tau (reading R7).
//   K2 k_search        exhaustive evaluation of every candidate: canonical binary32 Eq. 1 sum,
//                      budget + target feasibility, argmin (lowest index on ties) and count.
//   K3 k_finalize      decodes the reduced 64-bit key into the lowest canonical index and the
//                      FP64 Eq. 1 / Eq. 2 prediction of the winner.
//   k_predict          FP64 prediction of given allocations (alp_predict).
//
// K2 is the hot path.  Its design:
//  * the candidate digits are split into  prefix LLMs [0,g0) | sort-group LLMs [g0,g1) |
//    a = LLM M-2 | b = LLM M-1.  A "row" is (prefix, sort-group) digits; its canonical partial
//    sum Q_row = ((0 + tau_0) + tau_1) + ... is computed once and reused for Ka*Kb candidates.
//  * the b options are sorted by units; for a remaining budget r the feasible b options are a
//    prefix of that order, so a shared-memory "masked row" (tau_b, or +inf when u_b > r) folds
//    the budget test into the value.  Sort-group entries are pre-sorted (static, at build) by
//    their unit sum so the T rows of a lane (T = 12 by default; 8 / 16 variants) share one remaining budget -> one masked row.
//  * per candidate the SASS is half an FADD2 (add.rn.f32x2, binary32 RNE, scalar broadcast of
//    Q_a) and half an FMNMX3 (3-input min): 1 issue slot per candidate, with the b values
//    streamed by LDS.128 (4 columns x T rows = 48 candidates per load at T = 12).
//  * argmin: per-row min over the item's (a,b) block, folded into the thread's (value, segment)
//    best with a lowest-segment tie-break; keys = bits(value)<<32 | segment; warp shuffle ->
//    block -> atomicMin.  K3 re-scans the single winning segment for the lowest index.
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include <algorithm>
#include <mutex>
#include <set>

#include "alp_internal.h"
#include "alp_terms.cuh"
#include "alp_finalize.cuh"

namespace alp {

__device__ __forceinline__ float finf() { return __int_as_float(0x7f800000); }

__global__ void k_option_table(const __grid_constant__ OptionArgs A) {
  pdl_trigger();  // let K2 launch and stage its static tables while the terms are computed
  const int MK = A.prof.M * A.prof.K;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < A.n_targets) {
    if (A.keys) A.keys[i] = kKeyNone;
    if (A.counts) A.counts[i] = 0ull;
    if (A.fbest) A.fbest[i] = 0ull;  // the finalize after this search combines into zeroed scratch
    if (A.fdone) A.fdone[i] = 0u;
  }
  if (i < A.n_work) A.work[i] = 0ull;
  if (i >= A.n_targets * MK) return;
  const int t = i / MK, mk = i % MK, m = mk / A.prof.K, k = mk % A.prof.K;
  float tau;
  double term, b;
  int u;
  option_terms(A.prof, A.targets ? A.targets[t] : A.tgt[t], m, k, &tau, &term, &b, &u);
  A.tau[i] = tau;
  A.term[i] = term;
  A.b[i] = b;
  if (t == 0) A.u[mk] = u;
}

// tau of LLM g0+j, option d lives at ((g0+j)*K + d)*4 in the search kernels' shared memory; slot
// g1*K holds 0.0f (unused digit), slot g1*K+1 holds +inf (padded row): four offsets per row, the
// row's sort-group digits most significant first.
__global__ void k_plan_offsets(const uint32_t *tile_e, size_t rows, int g0, int g1, int ng, int K, uint4 *tile_off) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const uint32_t zero_off = (uint32_t)(g1 * K) * 4u, inf_off = zero_off + 4u;
  uint32_t off[4] = {zero_off, zero_off, zero_off, zero_off};
  const uint32_t e = tile_e[i];
  if (e == kDummy) {
    off[0] = inf_off;
  } else {
    uint32_t rem = e;
    for (int j = ng - 1; j >= 0; --j) {
      off[j] = (uint32_t)((g0 + j) * K + (int)(rem % (uint32_t)K)) * 4u;
      rem /= (uint32_t)K;
    }
  }
  tile_off[i] = make_uint4(off[0], off[1], off[2], off[3]);
}

cudaError_t launch_plan_offsets(const uint32_t *tile_e, size_t rows, int g0, int g1, int ng, int K, uint32_t *tile_off,
                                cudaStream_t st) {
  if (!rows) return cudaSuccess;
  k_plan_offsets<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(tile_e, rows, g0, g1, ng, K,
                                                                 reinterpret_cast<uint4 *>(tile_off));
  return cudaGetLastError();
}

// SPEC.md:374 fallback (no candidate meets the target): the candidate with the maximal Eq. 2
// T_w = min_m b_m among those within the budget whose options clear their memory floors, lowest
// canonical index on ties.  The Eq. 2 terms b (FP64, from the option table of the search) do not
// depend on the target.  One block: every thread tests thresholds theta = b of one option (a
// candidate with T_w >= theta exists iff sum_m min{u : b >= theta, floor ok} <= B; the answer is
// the largest such theta, an atomicMax on the bits of the positive double), then thread 0 picks
// the digits from LLM 0 on, each the smallest option whose completion still fits.
__global__ void k_max_throughput(const double *b, const int *u, DevProfiles pr, long long B, uint64_t N,
                                 alp_result *out) {
  const int M = pr.M, K = pr.K, MK = M * K;
  __shared__ unsigned long long s_theta;
  __shared__ int s_minu[ALP_MAX_M];
  auto ok = [&](int m, int k) {
    if (!pr.min_units) return true;
    const int si = k / (pr.nT * pr.nR), ti = (k / pr.nR) % pr.nT;
    return pr.S[si] >= pr.min_units[m * pr.nT + ti];
  };
  auto minu = [&](int m, double th) {
    int mn = 0x7fffffff;
    for (int k = 0; k < K; ++k)
      if (ok(m, k) && b[m * K + k] >= th) mn = min(mn, u[m * K + k]);
    return mn;
  };
  if (threadIdx.x == 0) s_theta = 0ull;
  __syncthreads();
  for (int i = threadIdx.x; i < MK; i += blockDim.x) {
    if (!ok(i / K, i % K)) continue;
    const double th = b[i];
    long long tot = 0;
    for (int m = 0; m < M && tot <= B; ++m) {
      const int mn = minu(m, th);
      tot = (mn == 0x7fffffff) ? B + 1 : tot + mn;
    }
    if (tot <= B) atomicMax(&s_theta, (unsigned long long)__double_as_longlong(th));
  }
  __syncthreads();
  const double th = __longlong_as_double((long long)s_theta);
  const bool any = s_theta != 0ull;
  if (any && (int)threadIdx.x < M) s_minu[threadIdx.x] = minu(threadIdx.x, th);
  __syncthreads();
  if (threadIdx.x != 0) return;
  alp_result r;
  memset(&r, 0, sizeof(r));
  r.M = M;
  r.candidates = N;
  r.index = ~0ull;
  r.latency = CUDART_INF;
  r.latency_key = __int_as_float(0x7f800000);
  if (any) {
    long long used = 0, rest = 0;
    for (int m = 0; m < M; ++m) rest += s_minu[m];
    unsigned long long idx = 0;
    double tw = CUDART_INF;
    for (int m = 0; m < M; ++m) {
      rest -= s_minu[m];
      int kk = -1;
      for (int k = 0; k < K && kk < 0; ++k)
        if (ok(m, k) && b[m * K + k] >= th && used + u[m * K + k] + rest <= B) kk = k;
      used += u[m * K + kk];
      idx = idx * (unsigned long long)K + (unsigned long long)kk;
      tw = b[m * K + kk] < tw ? b[m * K + kk] : tw;
      r.share_units[m] = pr.S[kk / (pr.nT * pr.nR)];
      r.tp[m] = pr.T[(kk / pr.nR) % pr.nT];
      r.replicas[m] = pr.R[kk % pr.nR];
    }
    r.index = idx;
    r.units = used;
    r.throughput = tw;
    r.fallback = 1;
  }
  *out = r;
}

cudaError_t launch_max_throughput(const double *b, const int *u, const DevProfiles &pr, long long B, uint64_t N,
                                  alp_result *out, cudaStream_t st) {
  k_max_throughput<<<1, 256, 0, st>>>(b, u, pr, B, N, out);
  return cudaGetLastError();
}

__global__ void k_init_keys(unsigned long long *keys, unsigned long long *counts, int n, unsigned long long *work,
                            int n_work, unsigned long long *fbest, unsigned *fdone) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    keys[i] = kKeyNone;
    counts[i] = 0ull;
    if (fbest) fbest[i] = 0ull;
    if (fdone) fdone[i] = 0u;
  }
  if (i < n_work) work[i] = 0ull;
}

// ------------------------------------------------------------------ search kernel (K2) dispatch
// The kernel templates live in alp_search.cuh; each rows-per-lane value is its own translation unit.
cudaError_t launch_search_t8(const SearchArgs &a, int grid, cudaStream_t st);
cudaError_t launch_search_t16(const SearchArgs &a, int grid, cudaStream_t st);
cudaError_t launch_search_t12(const SearchArgs &a, int grid, cudaStream_t st);
int occ_search_t12(const SearchArgs &a);
int occ_search_t8(const SearchArgs &a);
int occ_search_t16(const SearchArgs &a);

cudaError_t launch_search(const SearchArgs &a, int grid, cudaStream_t st) {
  if (a.rows_per_lane == 16) return launch_search_t16(a, grid, st);
  if (a.rows_per_lane == 12) return launch_search_t12(a, grid, st);
  return launch_search_t8(a, grid, st);
}

int search_max_blocks_per_sm(const SearchArgs &a) {
  if (a.rows_per_lane == 16) return occ_search_t16(a);
  if (a.rows_per_lane == 12) return occ_search_t12(a);
  return occ_search_t8(a);
}

// ------------------------------------------------------------------ finalize (K3)
// grid (nb, n_targets): the nb blocks of a target split the re-scan of the winning segment.
__global__ void k_finalize(const __grid_constant__ SearchArgs P) {
  pdl_wait();  // keys/counts/terms come from K2 (or the all-reduce after it)
  const int t = blockIdx.y;
  unsigned long long key = 0, count = 0;
  if (P.fin.world > 0) {
    // per-rank (keys, counts) gathered as [world][2][n_t]: MIN of keys (lowest value, then lowest
    // global segment), SUM of counts
    const size_t stride = 2 * (size_t)P.n_targets;
    key = ~0ull;
    for (int r = 0; r < P.fin.world; ++r) {
      const unsigned long long k = P.fin.keys[r * stride + t];
      key = k < key ? k : key;
      count += P.fin.keys[r * stride + P.n_targets + t];
    }
  } else {
    key = P.fin.keys[t];
    count = P.fin.counts[t];
  }
  // one block per target: its inputs staged in dynamic shared memory in one wave of loads
  finalize_target(P, t, key, count, blockIdx.x, gridDim.x, nullptr, nullptr, P.fin.stage != 0 && gridDim.x == 1);
}

// ------------------------------------------------------------------ multi-workflow split (NEXT-1)
// Egalitarian welfare over whole-GPU splits: lat[w*(G+1)+g] = best FP64 latency
// of workflow w on g GPUs (+inf if infeasible).  u_w(g) = lat_w(G) / lat_w(g) (0 if infeasible);
// splits (g_0..g_{W-2}, g_{W-1} = G - sum) maximise min_w u_w, then sum_w u_w, then the lowest
// split index (g_0 most significant).  One block; out: best split index, min and sum utility.
__global__ void k_egalitarian(const double *lat, int W, int G, long long *best_idx, double *best_min, double *best_sum) {
  __shared__ double s_min[256], s_sum[256];
  __shared__ long long s_idx[256];
  long long total = 1;
  for (int w = 0; w + 1 < W; ++w) total *= (G + 1);
  double bmin = -1.0, bsum = -1.0;
  long long bidx = -1;
  for (long long i = threadIdx.x; i < total; i += blockDim.x) {
    long long rem = i;
    int g[ALP_MAX_M];
    int used = 0;
    for (int w = W - 2; w >= 0; --w) {
      g[w] = (int)(rem % (G + 1));
      rem /= (G + 1);
      used += g[w];
    }
    if (used > G) continue;
    g[W - 1] = G - used;
    double mn = CUDART_INF, sm = 0.0;
    for (int w = 0; w < W; ++w) {
      const double solo = lat[w * (G + 1) + G], l = lat[w * (G + 1) + g[w]];
      const double u = (l < CUDART_INF && solo < CUDART_INF) ? __ddiv_rn(solo, l) : 0.0;
      mn = u < mn ? u : mn;
      sm = __dadd_rn(sm, u);
    }
    if (mn > bmin || (mn == bmin && (sm > bsum || (sm == bsum && i < bidx)))) {
      bmin = mn;
      bsum = sm;
      bidx = i;
    }
  }
  s_min[threadIdx.x] = bmin;
  s_sum[threadIdx.x] = bsum;
  s_idx[threadIdx.x] = bidx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int j = 1; j < (int)blockDim.x; ++j) {
      if (s_idx[j] < 0) continue;
      if (bidx < 0 || s_min[j] > bmin || (s_min[j] == bmin && (s_sum[j] > bsum || (s_sum[j] == bsum && s_idx[j] < bidx)))) {
        bmin = s_min[j];
        bsum = s_sum[j];
        bidx = s_idx[j];
      }
    }
    *best_idx = bidx;
    *best_min = bmin;
    *best_sum = bsum;
  }
}

cudaError_t launch_egalitarian(const double *lat, int W, int G, long long *best_idx, double *best_min,
                               double *best_sum, cudaStream_t st) {
  k_egalitarian<<<1, 256, 0, st>>>(lat, W, G, best_idx, best_min, best_sum);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ predict
__global__ void k_predict(const PredictArgs A) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n) return;
  double L = 0.0, Tw = CUDART_INF;
  long long U = 0;
  int all_ok = 1;
  for (int m = 0; m < A.prof.M; ++m) {
    float tau;
    double term, b;
    int u;
    all_ok &= option_terms(A.prof, A.lambda, m, A.opts[i * A.prof.M + m], &tau, &term, &b, &u);
    L = (m == 0) ? term : __dadd_rn(L, term);
    Tw = b < Tw ? b : Tw;
    U += u;
  }
  const int feas = all_ok && U <= A.budget;
  A.latency[i] = all_ok ? L : CUDART_INF;
  A.throughput[i] = Tw;
  A.units[i] = U;
  A.feasible[i] = feas;
}

// ------------------------------------------------------------------ launchers
// Every kernel of a search prefers the maximum shared-memory carveout, like K2, so consecutive
// launches on a stream do not reconfigure the SMs' L1/shared split in between.
static void max_carveout(const void *fn) {
  static std::mutex mu;
  static std::set<std::pair<const void *, int>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  if (done.insert({fn, dev}).second)
    cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
}

cudaError_t launch_option_table(const OptionArgs &a, cudaStream_t st) {
  const int total = a.n_targets * a.prof.M * a.prof.K;
  const int n = max(max(total, a.n_targets), a.n_work);
  max_carveout(reinterpret_cast<const void *>(k_option_table));
  k_option_table<<<(n + 255) / 256, 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_init_keys(unsigned long long *keys, unsigned long long *counts, int n, unsigned long long *work,
                             int n_work, unsigned long long *fbest, unsigned *fdone, cudaStream_t st) {
  const int m = n > n_work ? n : n_work;
  max_carveout(reinterpret_cast<const void *>(k_init_keys));
  k_init_keys<<<(m + 255) / 256, 256, 0, st>>>(keys, counts, n, work, n_work, fbest, fdone);
  return cudaGetLastError();
}

cudaError_t launch_finalize(const SearchArgs &a, cudaStream_t st) {
  // blocks per target for the winning-segment re-scan (<= Ka*Kb candidates): ~16 per thread
  const long long cand = (long long)a.Ka * a.Kb;
  const int nb = (int)std::min<long long>(64, std::max<long long>(1, cand / (256 * 16)));
  max_carveout(reinterpret_cast<const void *>(k_finalize));
  // a one-block re-scan stages the finalize inputs (option terms, units, FP64 terms, grids) in
  // dynamic shared memory by one wave of cp.async: C4's K3 8.0 -> see profiles
  SearchArgs b = a;
  const size_t stage = finalize_stage_bytes(a.M, a.K, a.fin.nS, a.fin.nT, a.fin.nR);
  b.fin.stage = (nb == 1 && a.fin.S && stage <= 48 * 1024) ? 1 : 0;
  return launch_pdl(k_finalize, dim3(nb, a.n_targets), dim3(256), b.fin.stage ? stage : 0, st, b);
}

cudaError_t launch_predict(const PredictArgs &a, cudaStream_t st) {
  k_predict<<<(a.n + 127) / 128, 128, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace alp
