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
//    their unit sum so the 8 rows of a lane share one remaining budget -> one masked row.
//  * per candidate the SASS is half an FADD2 (add.rn.f32x2, binary32 RNE, scalar broadcast of
//    Q_a) and half an FMNMX3 (3-input min): 1 issue slot per candidate, with the b values
//    streamed by LDS.128 (4 columns x 8 rows = 32 candidates per load).
//  * argmin: per-row min over the item's (a,b) block, folded into the thread's (value, segment)
//    best with a lowest-segment tie-break; keys = bits(value)<<32 | segment; warp shuffle ->
//    block -> atomicMin.  K3 re-scans the single winning segment for the lowest index.
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include <algorithm>

#include "alp_internal.h"

namespace alp {

__device__ __forceinline__ float finf() { return __int_as_float(0x7f800000); }

// ------------------------------------------------------------------ option terms (FP64, no FMA)
// SURVEY.md §8(c) / DESIGN.md §3: every operation is an explicit IEEE RNE intrinsic, in the
// order written, so the result is bit-identical to the oracle's -ffp-contract=off C code.
__device__ double lookup_latency(const double *r, const double *l, int P, double x) {
  // R3: clamp below r_0; i = max{i : r_i <= x}; hold L_last at/after the last point.
  if (x <= r[0]) return l[0];
  int i = 0;
  for (int j = 0; j < P; ++j)
    if (r[j] <= x) i = j;
  if (i == P - 1) return l[P - 1];
  double dl = __dsub_rn(l[i + 1], l[i]);
  double dx = __dsub_rn(x, r[i]);
  double dr = __dsub_rn(r[i + 1], r[i]);
  double w = __ddiv_rn(dx, dr);
  return __dadd_rn(l[i], __dmul_rn(dl, w));
}

__device__ int option_terms(const DevProfiles &P, double lambda, int m, int k, float *tau, double *term,
                            double *b, int *u) {
  const int r_i = k % P.nR;
  const int t_i = (k / P.nR) % P.nT;
  const int s_i = k / (P.nR * P.nT);
  const int s_units = P.S[s_i], t = P.T[t_i], d = P.R[r_i];
  const int c = m * P.nT + t_i;
  const double T = P.tmax[c];
  const double lam_m = __dmul_rn(lambda, P.n[m]);              // lambda_m = lambda_W n_m
  const double rate = __ddiv_rn(lam_m, (double)d);            // per replica
  const double f = __ddiv_rn((double)s_units, (double)P.F);   // per-shard share
  const double x = __ddiv_rn(rate, f);                        // L'(l) = L(l/f)/f
  const double cap = __dmul_rn(f, T);
  const double bb = __ddiv_rn(__dmul_rn((double)d, cap), P.n[m]);  // Eq. 2 term
  int ok = (x <= T) && (bb >= lambda);                        // R4
  if (P.min_units && s_units < P.min_units[c]) ok = 0;        // memory floor
  *b = bb;
  *u = s_units * t * d;
  if (ok) {
    const int o = P.prof_off[c];
    const double L = lookup_latency(P.rate + o, P.lat + o, P.prof_off[c + 1] - o, x);
    const double tt = __dmul_rn(__ddiv_rn(L, f), __ddiv_rn(P.n[m], P.p[m]));  // Eq. 1 term
    *term = tt;
    *tau = __double2float_rn(tt);
  } else {
    *term = CUDART_INF;
    *tau = finf();
  }
  return ok;
}

__global__ void k_option_table(const OptionArgs A) {
  const int MK = A.prof.M * A.prof.K;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < A.n_targets) {
    if (A.keys) A.keys[i] = kKeyNone;
    if (A.counts) A.counts[i] = 0ull;
  }
  if (i < A.n_work) A.work[i] = 0ull;
  if (i >= A.n_targets * MK) return;
  const int t = i / MK, mk = i % MK, m = mk / A.prof.K, k = mk % A.prof.K;
  float tau;
  double term, b;
  int u;
  option_terms(A.prof, A.targets[t], m, k, &tau, &term, &b, &u);
  A.tau[i] = tau;
  A.term[i] = term;
  A.b[i] = b;
  if (t == 0) A.u[mk] = u;
}

__global__ void k_init_keys(unsigned long long *keys, unsigned long long *counts, int n, unsigned long long *work,
                            int n_work) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    keys[i] = kKeyNone;
    counts[i] = 0ull;
  }
  if (i < n_work) work[i] = 0ull;
}

// ------------------------------------------------------------------ search kernel (K2) dispatch
// The kernel templates live in alp_search.cuh; each rows-per-lane value is its own translation unit.
cudaError_t launch_search_t8(const SearchArgs &a, int grid, cudaStream_t st);
cudaError_t launch_search_t16(const SearchArgs &a, int grid, cudaStream_t st);
int occ_search_t8(const SearchArgs &a);
int occ_search_t16(const SearchArgs &a);

cudaError_t launch_search(const SearchArgs &a, int grid, cudaStream_t st) {
  return a.rows_per_lane == 16 ? launch_search_t16(a, grid, st) : launch_search_t8(a, grid, st);
}

int search_max_blocks_per_sm(const SearchArgs &a) {
  return a.rows_per_lane == 16 ? occ_search_t16(a) : occ_search_t8(a);
}

// ------------------------------------------------------------------ finalize (K3)
// grid (nb, n_targets): the nb blocks of a target split the re-scan of the winning segment; the
// last block to finish (ticket) assembles the result and resets the target's scratch.
__global__ void k_finalize(const FinalizeArgs F) {
  const SearchArgs &P = F.s;
  const int t = blockIdx.y;
  const unsigned long long key = F.keys[t];
  const unsigned long long count = F.counts[t];
  __shared__ unsigned long long s_best;
  const int K = P.K;
  const float *tau_t = P.tau + (size_t)t * P.M * K;
  const uint32_t seg = (uint32_t)(key & 0xffffffffull);
  const float val = __uint_as_float((uint32_t)(key >> 32));
  const bool found = key != kKeyNone && val < finf();
  uint32_t q = 0, chunk = 0, e = 0;
  float Qrow = 0.f;
  int Urow = 0;
  if (found) {
    q = seg % P.nQ;
    const uint32_t row = seg / P.nQ;
    chunk = row / P.L;
    e = row % P.L;
    // canonical partial sum over LLMs 0..g1-1 (digits of chunk then e, most significant first)
    int kd[ALP_MAX_M];
    uint32_t rem = chunk;
    for (int m = P.g0 - 1; m >= 0; --m) { kd[m] = (int)(rem % (uint32_t)K); rem /= (uint32_t)K; }
    rem = e;
    for (int j = P.ng - 1; j >= 0; --j) { kd[P.g0 + j] = (int)(rem % (uint32_t)K); rem /= (uint32_t)K; }
    for (int m = 0; m < P.g1; ++m) {
      Qrow = __fadd_rn(Qrow, tau_t[m * K + kd[m]]);
      Urow += P.u[m * K + kd[m]];
    }
  }
  if (threadIdx.x == 0) {
    s_best = ~0ull;
  }
  __syncthreads();
  if (found) {
    // the segment starts at a-range q and runs to the end of the row (see fold_rows)
    const int a0 = (int)(q * P.A), a1 = P.Ka;
    const unsigned long long n = (unsigned long long)(a1 - a0) * P.Kb;
    unsigned long long mine = ~0ull;
    for (unsigned long long li = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; li < n;
         li += (unsigned long long)gridDim.x * blockDim.x) {
      const int a = a0 + (int)(li / P.Kb), b = (int)(li % P.Kb);
      float ta = 0.f;
      int ua = 0;
      if (P.a_llm >= 0) {
        ta = tau_t[P.a_llm * K + a];
        ua = P.u[P.a_llm * K + a];
      }
      const float v = __fadd_rn(__fadd_rn(Qrow, ta), tau_t[P.b_llm * K + b]);
      const int units = Urow + ua + P.u[P.b_llm * K + b];
      if (v == val && units <= qbudget(P, t)) {
        mine = li;
        break;
      }
    }
    atomicMin(&s_best, mine);
  }
  __syncthreads();
  // combine the blocks of this target: global min, then only the last block continues
  __shared__ unsigned s_last;
  if (threadIdx.x == 0) {
    if (found) atomicMin(F.best + t, s_best);
    __threadfence();
    s_last = (atomicAdd(F.done + t, 1u) == gridDim.x - 1) ? 1u : 0u;
  }
  __syncthreads();
  if (!s_last) return;
  if (threadIdx.x == 0) {
    __threadfence();
    s_best = atomicAdd(F.best + t, 0ull);  // coherent read of the combined minimum
    F.best[t] = ~0ull;                    // reset for the next finalize on this scratch
    F.done[t] = 0u;
  }
  __syncthreads();
  // winner digits, then the per-LLM FP64 terms gathered in parallel (one thread per LLM)
  __shared__ int s_k[ALP_MAX_M];
  __shared__ double s_term[ALP_MAX_M], s_bterm[ALP_MAX_M];
  __shared__ int s_u[ALP_MAX_M], s_grid[3][ALP_MAX_M];
  const bool win = found && s_best != ~0ull;
  if (threadIdx.x == 0 && win) {
    const int a0 = (int)(q * P.A);
    const int a = a0 + (int)(s_best / P.Kb), b = (int)(s_best % P.Kb);
    uint32_t rem = chunk;
    for (int m = P.g0 - 1; m >= 0; --m) {
      s_k[m] = (int)(rem % (uint32_t)K);
      rem /= (uint32_t)K;
    }
    rem = e;
    for (int j = P.ng - 1; j >= 0; --j) {
      s_k[P.g0 + j] = (int)(rem % (uint32_t)K);
      rem /= (uint32_t)K;
    }
    if (P.a_llm >= 0) s_k[P.a_llm] = a;
    s_k[P.b_llm] = b;
  }
  __syncthreads();
  if (win && (int)threadIdx.x < P.M) {
    const int m = threadIdx.x, km = s_k[m];
    s_term[m] = F.term[((size_t)t * P.M + m) * K + km];
    s_bterm[m] = F.b[((size_t)t * P.M + m) * K + km];
    s_u[m] = P.u[m * K + km];
    if (F.S) {
      s_grid[0][m] = F.S[km / (F.nR * F.nT)];
      s_grid[1][m] = F.T[(km / F.nR) % F.nT];
      s_grid[2][m] = F.R[km % F.nR];
    }
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  alp_result r;
  memset(&r, 0, sizeof(r));
  r.M = P.M;
  r.feasible_count = count;
  r.candidates = F.N;
  r.index = ~0ull;
  r.latency_key = finf();
  if (win) {
    unsigned long long idx = 0;
    double L = 0.0, Tw = CUDART_INF;
    long long U = 0;
    for (int m = 0; m < P.M; ++m) {
      idx = idx * (unsigned long long)K + (unsigned long long)s_k[m];
      L = (m == 0) ? s_term[m] : __dadd_rn(L, s_term[m]);  // Eq. 1 in canonical order (FP64)
      Tw = s_bterm[m] < Tw ? s_bterm[m] : Tw;               // Eq. 2
      U += s_u[m];
      if (F.S) {
        r.share_units[m] = s_grid[0][m];
        r.tp[m] = s_grid[1][m];
        r.replicas[m] = s_grid[2][m];
      }
    }
    r.found = 1;
    r.index = idx;
    r.latency_key = val;
    r.latency = L;
    r.throughput = Tw;
    r.units = U;
  } else {
    r.latency = CUDART_INF;
    r.throughput = 0.0;
  }
  F.out[t] = r;
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
cudaError_t launch_option_table(const OptionArgs &a, cudaStream_t st) {
  const int total = a.n_targets * a.prof.M * a.prof.K;
  const int n = max(max(total, a.n_targets), a.n_work);
  k_option_table<<<(n + 255) / 256, 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_init_keys(unsigned long long *keys, unsigned long long *counts, int n, unsigned long long *work,
                             int n_work, cudaStream_t st) {
  const int m = n > n_work ? n : n_work;
  k_init_keys<<<(m + 255) / 256, 256, 0, st>>>(keys, counts, n, work, n_work);
  return cudaGetLastError();
}

cudaError_t launch_finalize(const FinalizeArgs &a, cudaStream_t st) {
  // blocks per target for the winning-segment re-scan (<= Ka*Kb candidates): ~16 per thread
  const long long cand = (long long)a.s.Ka * a.s.Kb;
  const int nb = (int)std::min<long long>(64, std::max<long long>(1, cand / (256 * 16)));
  k_finalize<<<dim3(nb, a.s.n_targets), 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_predict(const PredictArgs &a, cudaStream_t st) {
  k_predict<<<(a.n + 127) / 128, 128, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace alp
