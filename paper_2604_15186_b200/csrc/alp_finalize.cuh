// Finalize (K3) device code, shared by k_finalize (alp_kernels.cu) and the last block of the fused
// search kernel (alp_search.cuh).
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "alp_internal.h"

namespace alp {

// asynchronous global -> shared copies (the staging wave: every load in flight at once)
__device__ __forceinline__ void fin_cp4(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void fin_cp8(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}

// Finalize of target t from its reduced (key, count): the lowest canonical index inside the
// winning segment, the winner's (share, tp, replicas) and its FP64 Eq. 1 / Eq. 2 prediction.
// Blocks [part] of [nparts] split the re-scan of the segment; with nparts > 1 the last block to
// finish (ticket) assembles the result and resets the target's scratch.  Called by every thread
// of a block (K3, or the last block of the fused search).  stage: the block's dynamic shared
// memory is free and holds finalize_stage_bytes — every input (option terms, units, FP64 terms,
// grids) is copied there in one wave of loads first, so the dependent steps (digits, re-scan,
// winner terms) read shared memory instead of waiting on L2 / DRAM one round trip each.
__device__ inline void finalize_target(const SearchArgs &P, int t, unsigned long long key, unsigned long long count,
                                       int part, int nparts, const float *tau_s = nullptr,
                                       alp_result *out_row = nullptr, bool stage = false) {
  const FinalizeExtra &F = P.fin;
  const int K = P.K, MK = P.M * K, nG = F.nS + F.nT + F.nR;
  auto stamp = [&](int i) {  // ALP_DBG_TS (fused epilogue only): phases in the second extra row
    if (P.dbg_ts && threadIdx.x == 0 && P.fz.on)  // SM clock cycles (same SM: exact phase deltas)
      P.dbg_ts[(size_t)gridDim.x * 8 + 8 + i] = (unsigned long long)clock64();
  };
  stamp(0);
  // option terms of target t: the caller's shared-memory copy (fused kernel) or the global tables
  const float *tau_g = P.tau + (size_t)t * MK;
  const double *term_g = F.term + (size_t)t * MK, *b_g = F.b + (size_t)t * MK;
  extern __shared__ __align__(16) unsigned char fin_stage[];  // the block's dynamic shared memory
  double *st_term = reinterpret_cast<double *>(fin_stage), *st_b = st_term + MK;
  float *st_tau = reinterpret_cast<float *>(st_b + MK);
  int *st_u = reinterpret_cast<int *>(st_tau + MK), *st_g = st_u + MK;
  auto tau = [&](int i) { return stage ? st_tau[i] : (tau_s ? tau_s[i] : __ldcg(tau_g + i)); };
  auto uni = [&](int i) { return stage ? st_u[i] : P.u[i]; };
  auto term = [&](int i) { return stage ? st_term[i] : __ldcg(term_g + i); };
  auto bterm = [&](int i) { return stage ? st_b[i] : __ldcg(b_g + i); };
  auto grid = [&](int i) { return stage ? st_g[i] : (i < F.nS ? F.S[i] : i < F.nS + F.nT ? F.T[i - F.nS] : F.R[i - F.nS - F.nT]); };
  __shared__ unsigned long long s_best;
  __shared__ int s_k[ALP_MAX_M], s_u[ALP_MAX_M], s_grid[3][ALP_MAX_M];
  __shared__ float s_tq[ALP_MAX_M];
  __shared__ double s_term[ALP_MAX_M], s_bterm[ALP_MAX_M];
  __shared__ float s_Q;
  __shared__ int s_U;
  __shared__ alp_result s_res;
  const uint32_t seg = (uint32_t)(key & 0xffffffffull);
  const float val = __uint_as_float((uint32_t)(key >> 32));
  const bool found = key != kKeyNone && val < __int_as_float(0x7f800000);
  if (found && stage) {  // cp.async: one wave of loads in flight, not one round trip per element
    for (int i = threadIdx.x; i < MK; i += blockDim.x) {
      fin_cp8(st_term + i, term_g + i);
      fin_cp8(st_b + i, b_g + i);
      if (tau_s)
        st_tau[i] = tau_s[i];
      else
        fin_cp4(st_tau + i, tau_g + i);
      fin_cp4(st_u + i, P.u + i);
    }
    if (F.S)
      for (int i = threadIdx.x; i < nG; i += blockDim.x)
        fin_cp4(st_g + i, i < F.nS ? F.S + i : i < F.nS + F.nT ? F.T + (i - F.nS) : F.R + (i - F.nS - F.nT));
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
  }
  uint32_t q = 0, chunk = 0, e = 0;
  if (found) {
    q = seg % P.seg_q;  // segment slot: first a option = q * seg_A
    const uint32_t row = seg / P.seg_q;
    chunk = row / P.L;
    e = row % P.L;
    // digits of the row's LLMs 0..g1-1 (chunk digits, then sort-group digits; LLM 0 most
    // significant), one thread per LLM, with their terms and units
    const int m = threadIdx.x;
    if (m < P.g1) {
      uint32_t d;
      if (m < P.g0) {
        d = (chunk / P.pw[m]) % (uint32_t)K;
      } else {
        uint32_t pw = 1;
        for (int j = m - P.g0 + 1; j < P.ng; ++j) pw *= (uint32_t)K;
        d = (e / pw) % (uint32_t)K;
      }
      s_k[m] = (int)d;
      s_tq[m] = tau(m * K + (int)d);
      s_u[m] = uni(m * K + (int)d);
    }
  }
  if (threadIdx.x == 0) s_best = ~0ull;
  __syncthreads();
  stamp(1);
  if (found && threadIdx.x == 0) {
    // canonical partial sum over LLMs 0..g1-1: ((0 + tau_0) + tau_1) + ...
    float Q = 0.f;
    int U = 0;
    for (int m = 0; m < P.g1; ++m) {
      Q = __fadd_rn(Q, s_tq[m]);
      U += s_u[m];
    }
    s_Q = Q;
    s_U = U;
  }
  __syncthreads();
  if (found) {
    // the segment starts at a option q * seg_A and runs to the end of the row (see fold_rows)
    const float Qrow = s_Q;
    const int Urow = s_U;
    const int a0 = (int)(q * P.seg_A), a1 = P.Ka;
    const unsigned long long n = (unsigned long long)(a1 - a0) * P.Kb;
    unsigned long long mine = ~0ull;
    for (unsigned long long li = (unsigned long long)part * blockDim.x + threadIdx.x; li < n;
         li += (unsigned long long)nparts * blockDim.x) {
      const uint32_t l32 = (uint32_t)li;  // n <= Ka*Kb <= 2^20
      const int a = a0 + (int)(l32 / (uint32_t)P.Kb), b = (int)(l32 % (uint32_t)P.Kb);
      float ta = 0.f;
      int ua = 0;
      if (P.a_llm >= 0) {
        ta = tau(P.a_llm * K + a);
        ua = uni(P.a_llm * K + a);
      }
      const float v = __fadd_rn(__fadd_rn(Qrow, ta), tau(P.b_llm * K + b));
      const int units = Urow + ua + uni(P.b_llm * K + b);
      if (v == val && units <= qbudget(P, t)) {
        mine = li;
        break;
      }
    }
    atomicMin(&s_best, mine);
  }
  __syncthreads();
  stamp(2);
  if (nparts > 1) {
    // combine the blocks of this target: global min, then only the last block continues
    __shared__ unsigned s_last;
    if (threadIdx.x == 0) {
      if (found) atomicMax(F.best + t, ~s_best);  // complemented minimum: zero at rest
      __threadfence();
      s_last = (atomicAdd(F.done + t, 1u) == (unsigned)nparts - 1) ? 1u : 0u;
    }
    __syncthreads();
    if (!s_last) return;
    if (threadIdx.x == 0) {
      __threadfence();
      s_best = ~atomicAdd(F.best + t, 0ull);  // coherent read of the combined minimum
      F.best[t] = 0ull;                      // rest state (zero) for the next finalize on this scratch
      F.done[t] = 0u;
    }
    __syncthreads();
  }
  // the winner's a and b digits, then its per-LLM FP64 terms gathered in parallel (one thread per LLM)
  const bool win = found && s_best != ~0ull;
  if (win && threadIdx.x == 0) {
    const int a = (int)(q * P.seg_A) + (int)(s_best / P.Kb), b = (int)(s_best % P.Kb);
    if (P.a_llm >= 0) s_k[P.a_llm] = a;
    s_k[P.b_llm] = b;
  }
  __syncthreads();
  if (win && (int)threadIdx.x < P.M) {
    const int m = threadIdx.x, km = s_k[m];
    s_term[m] = term(m * K + km);
    s_bterm[m] = bterm(m * K + km);
    s_u[m] = uni(m * K + km);
    if (F.S) {
      s_grid[0][m] = grid(km / (F.nR * F.nT));
      s_grid[1][m] = grid(F.nS + (km / F.nR) % F.nT);
      s_grid[2][m] = grid(F.nS + F.nT + km % F.nR);
    }
  }
  __syncthreads();
  stamp(3);
  if (threadIdx.x == 0) {
    alp_result &r = s_res;
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
  }
  __syncthreads();
  // one coalesced copy of the result (device memory, or mapped host memory for the fused search)
  static_assert(sizeof(alp_result) % 4 == 0, "alp_result is copied as 32-bit words");
  const uint32_t *src = reinterpret_cast<const uint32_t *>(&s_res);
  uint32_t *dst = reinterpret_cast<uint32_t *>(out_row ? out_row : F.out + t);
  for (int i = threadIdx.x; i < (int)(sizeof(alp_result) / 4); i += blockDim.x) dst[i] = src[i];
  __syncthreads();  // shared scratch reused by the next target
  stamp(4);
}

}  // namespace alp
