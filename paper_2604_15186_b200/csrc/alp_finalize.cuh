// Finalize (K3) device code, shared by k_finalize (alp_kernels.cu) and the last block of the fused
// search kernel (alp_search.cuh).
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "alp_internal.h"

namespace alp {

// Finalize of target t from its reduced (key, count): the lowest canonical index inside the
// winning segment, the winner's (share, tp, replicas) and its FP64 Eq. 1 / Eq. 2 prediction.
// Blocks [part] of [nparts] split the re-scan of the segment; with nparts > 1 the last block to
// finish (ticket) assembles the result and resets the target's scratch.  Called by every thread
// of a block (K3, or the last block of the fused search).
__device__ inline void finalize_target(const SearchArgs &P, int t, unsigned long long key, unsigned long long count,
                                       int part, int nparts) {
  const FinalizeExtra &F = P.fin;
  __shared__ unsigned long long s_best;
  const int K = P.K;
  const float *tau_t = P.tau + (size_t)t * P.M * K;
  const uint32_t seg = (uint32_t)(key & 0xffffffffull);
  const float val = __uint_as_float((uint32_t)(key >> 32));
  const bool found = key != kKeyNone && val < __int_as_float(0x7f800000);
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
      Qrow = __fadd_rn(Qrow, __ldcg(tau_t + m * K + kd[m]));
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
    for (unsigned long long li = (unsigned long long)part * blockDim.x + threadIdx.x; li < n;
         li += (unsigned long long)nparts * blockDim.x) {
      const uint32_t l32 = (uint32_t)li;  // n <= Ka*Kb <= 2^20
      const int a = a0 + (int)(l32 / (uint32_t)P.Kb), b = (int)(l32 % (uint32_t)P.Kb);
      float ta = 0.f;
      int ua = 0;
      if (P.a_llm >= 0) {
        ta = __ldcg(tau_t + P.a_llm * K + a);
        ua = P.u[P.a_llm * K + a];
      }
      const float v = __fadd_rn(__fadd_rn(Qrow, ta), __ldcg(tau_t + P.b_llm * K + b));
      const int units = Urow + ua + P.u[P.b_llm * K + b];
      if (v == val && units <= qbudget(P, t)) {
        mine = li;
        break;
      }
    }
    atomicMin(&s_best, mine);
  }
  __syncthreads();
  if (nparts > 1) {
    // combine the blocks of this target: global min, then only the last block continues
    __shared__ unsigned s_last;
    if (threadIdx.x == 0) {
      if (found) atomicMin(F.best + t, s_best);
      __threadfence();
      s_last = (atomicAdd(F.done + t, 1u) == (unsigned)nparts - 1) ? 1u : 0u;
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
  }
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
    s_term[m] = __ldcg(F.term + ((size_t)t * P.M + m) * K + km);
    s_bterm[m] = __ldcg(F.b + ((size_t)t * P.M + m) * K + km);
    s_u[m] = P.u[m * K + km];
    if (F.S) {
      s_grid[0][m] = F.S[km / (F.nR * F.nT)];
      s_grid[1][m] = F.T[(km / F.nR) % F.nT];
      s_grid[2][m] = F.R[km % F.nR];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
  alp_result r;
  memset(&r, 0, sizeof(r));
  r.M = P.M;
  r.feasible_count = count;
  r.candidates = F.N;
  r.index = ~0ull;
  r.latency_key = __int_as_float(0x7f800000);
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
  __syncthreads();  // shared scratch reused by the next target
}

}  // namespace alp
