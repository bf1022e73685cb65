// Budget-indexed search in ONE pass ("searches for the
// per-workflow allocation independently" on every GPU count the multi-workflow split considers):
// for one target and budgets b_0 < ... < b_{L-1}, the best candidate under every budget from a
// single evaluation of the candidates with units <= b_{L-1}, instead of one exhaustive pass per
// budget.
//
// A candidate with units U belongs to level l(U) = min{l : b_l >= U}; it is feasible exactly for
// the budgets of levels >= l(U).  So best(b_g) = MIN over levels l <= g of the level's best key,
// and count(b_g) = #feasible candidates with U <= b_g.  The kernel walks the same rows, lane
// tiles and a options as k_search; per (lane tile, a) the u-sorted b columns split into runs of
// equal level (a unit value never decreases along the sorted columns), each run evaluated with the
// same binary32 additions as the definition ((Q_row + tau_a) + tau_b) and folded into the block's
// per-level best (value, segment) key.  Segments are single a options (row * Ka + a), so the
// finalize (K3, per budget) re-scans from the winner's exact (row, a) to the end of the row.
// Counts are exact integers from the per-LLM feasible-unit histograms (k_level_finish).
#include "alp_search.cuh"

namespace alp {

struct LevelArgs {
  SearchArgs s;             // plan geometry and tables; s.tau = option terms of the target (t = 0)
  const int *levels;        // [L] ascending distinct budgets (units, capped at the total max)
  int L, bmax;              // levels, b_{L-1}
  unsigned long long *lvl_keys;  // [L] min key per level (0xFF..FF = none at the start)
  unsigned long long *ticket;    // work counter, 0 at the start
  int off_lvl, off_ta, off_tb, off_best, smem_bytes;  // dynamic shared-memory layout (bytes)
  int off_runs;  // per ubase (row + a units) the equal-level runs of the u-sorted b columns, or -1
};

constexpr int kLvlThreads = 256;
constexpr int kLvlT = 12;  // rows per lane (the plan's lane tiles)

__global__ void __launch_bounds__(kLvlThreads, 2) k_search_levels(const __grid_constant__ LevelArgs A) {
  const SearchArgs &P = A.s;
  constexpr int T = kLvlT;
  extern __shared__ __align__(16) unsigned char smem[];
  float *s_tau = reinterpret_cast<float *>(smem);                        // [g1*K + 2] at offset 0 (tile_off)
  unsigned short *s_lvl = reinterpret_cast<unsigned short *>(smem + A.off_lvl);  // [bmax + 1] U -> level
  float2 *s_ta = reinterpret_cast<float2 *>(smem + A.off_ta);          // [Ka] {tau_a, bits(u_a)}
  float2 *s_tb = reinterpret_cast<float2 *>(smem + A.off_tb);          // [Kb] u-sorted {tau_b, bits(u_b)}
  unsigned long long *s_best = reinterpret_cast<unsigned long long *>(smem + A.off_best);  // [L]
  int *s_u = reinterpret_cast<int *>(smem + P.off_u);                  // [g0*K] prefix units
  float2 *s_pfx = reinterpret_cast<float2 *>(smem + (P.off_pfx >= 0 ? P.off_pfx : 0));
  const int tid = threadIdx.x, K = P.K;
  const float *tau = P.tau;  // target 0
  for (int i = tid; i < P.g1 * K; i += blockDim.x) s_tau[i] = tau[i];
  if (tid == 0) {
    s_tau[P.g1 * K] = 0.f;
    s_tau[P.g1 * K + 1] = finf();
  }
  for (int i = tid; i < P.g0 * K; i += blockDim.x) s_u[i] = P.u[i];
  for (int a = tid; a < P.Ka; a += blockDim.x) {
    const float ta = P.a_llm >= 0 ? tau[P.a_llm * K + a] : 0.f;
    const int ua = P.a_llm >= 0 ? P.u[P.a_llm * K + a] : 0;
    s_ta[a] = make_float2(ta, __int_as_float(ua));
  }
  for (int j = tid; j < P.Kb; j += blockDim.x) {
    const int b = P.bperm[j];
    s_tb[j] = make_float2(tau[P.b_llm * K + b], __int_as_float(P.u[P.b_llm * K + b]));
  }
  for (int U = tid; U <= A.bmax; U += blockDim.x) {
    int lo = 0, hi = A.L - 1;  // smallest level with budget >= U
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (A.levels[mid] >= U) hi = mid; else lo = mid + 1;
    }
    s_lvl[U] = (unsigned short)lo;
  }
  for (int l = tid; l < A.L; l += blockDim.x) s_best[l] = ~0ull;
  __syncthreads();
  // run table: for every ubase, the u-sorted b columns split where the budget level of ubase + u_b
  // changes, as (end column << 16 | level) entries ended by 0xffffffff — the boundaries depend only
  // on ubase, so the loop below walks runs instead of looking up every column's level
  uint32_t *s_runs = reinterpret_cast<uint32_t *>(smem + (A.off_runs >= 0 ? A.off_runs : 0));
  const int rw = P.Kb + 1;
  if (A.off_runs >= 0) {
    for (int ub = tid; ub <= A.bmax; ub += blockDim.x) {
      uint32_t *rt = s_runs + (size_t)ub * rw;
      int n = 0, cur = -1, j = 0;
      for (; j < P.Kb; ++j) {
        const int U = ub + __float_as_int(s_tb[j].y);
        if (U > A.bmax) break;
        const int l = s_lvl[U];
        if (l != cur) {
          if (cur >= 0) rt[n++] = ((uint32_t)j << 16) | (uint32_t)cur;
          cur = l;
        }
      }
      if (cur >= 0) rt[n++] = ((uint32_t)j << 16) | (uint32_t)cur;
      rt[n] = 0xffffffffu;
    }
    __syncthreads();
  }
  if (P.off_pfx >= 0) {
    Smem sm;
    sm.tau = s_tau;
    sm.u = s_u;
    for (uint32_t c = tid; c < P.n_chunks; c += blockDim.x) {
      float pa;
      int U;
      prefix_sum(P, sm, c, pa, U);
      s_pfx[c] = make_float2(pa, __int_as_float(U));
    }
    __syncthreads();
  }
  const int lane = tid & 31;
  const uint32_t n = (uint32_t)(P.item_hi - P.item_lo);
  const unsigned char *tau_b = smem;
  for (;;) {
    unsigned k = 0;
    if (lane == 0) k = (unsigned)atomicAdd(A.ticket, 1ull);
    k = __shfl_sync(0xffffffffu, k, 0);
    if (k >= n) break;
    const uint32_t it = (uint32_t)P.item_lo + k;
    const uint32_t tq = fdiv(it, P.fd_nQ);
    const uint32_t q = it - tq * P.nQ;
    const uint32_t chunk = fdiv(tq, P.fd_ng);
    const uint32_t grp = tq - chunk * P.n_groups;
    const uint32_t tile = grp * kWarpTiles + lane;
    float pfx;
    int upfx;
    if (P.off_pfx >= 0) {
      const float2 pf = s_pfx[chunk];
      pfx = pf.x;
      upfx = __float_as_int(pf.y);
    } else {
      Smem sm;
      sm.tau = s_tau;
      sm.u = s_u;
      prefix_sum(P, sm, chunk, pfx, upfx);
    }
    float Qr[T], acc[T];
    const unsigned nfin = load_tile<T>(P, tau_b, pfx, tile, Qr, acc);
    const int urow = upfx + __ldg(P.tile_s + tile);
    if (nfin == 0 || urow > A.bmax) continue;  // padded / infeasible rows, or over every budget
    const int a0 = (int)(q * P.A), a1 = min(a0 + (int)P.A, P.Ka);
    for (int a = a0; a < a1; ++a) {
      const float2 av = s_ta[a];
      if (!(av.x < finf())) continue;  // target-infeasible a option
      const int ubase = urow + __float_as_int(av.y);
      if (ubase > A.bmax) continue;
      float Qa[T];
#pragma unroll
      for (int i = 0; i < T; ++i) Qa[i] = __fadd_rn(Qr[i], av.x);
      int cur = -1;
      // fold the run's row minima into the block's best key of level `cur`
      // (the rows' canonical indices are read only when the run's minimum can still improve the
      // level's best: its value bits alone bound the key from below)
      auto fold = [&](bool reset) {
        float m = acc[0];
#pragma unroll
        for (int i = 1; i < T; ++i) m = fminf(m, acc[i]);
        if (m < finf()) {
          const unsigned long long hi = (unsigned long long)__float_as_uint(m) << 32;
          if (hi <= s_best[cur]) {
            uint32_t bs = 0xffffffffu;
#pragma unroll
            for (int i = 0; i < T; ++i)
              if (acc[i] == m) bs = min(bs, (chunk * P.L + __ldg(P.tile_e + (size_t)tile * T + i)) * (uint32_t)P.Ka + (uint32_t)a);
            const unsigned long long key = hi | bs;
            if (key < s_best[cur]) atomicMin(s_best + cur, key);
          }
        }
        if (reset) {
#pragma unroll
          for (int i = 0; i < T; ++i) acc[i] = finf();
        }
      };
      if (A.off_runs >= 0) {
        const uint32_t *rt = s_runs + (size_t)ubase * rw;
        int j = 0;
        for (int r = 0;; ++r) {
          const uint32_t e = rt[r];
          if (e == 0xffffffffu) break;
          const int jend = (int)(e >> 16);
          cur = (int)(e & 0xffffu);
          // the run's first column(s) initialise the row minima (no reset after the previous fold)
          if (j + 1 < jend) {
            const float2 bv = s_tb[j], bw = s_tb[j + 1];
#pragma unroll
            for (int i = 0; i < T; i += 2) {
              float x0, x1, y0, y1;
              add2b(x0, x1, Qa[i], Qa[i + 1], bv.x);
              add2b(y0, y1, Qa[i], Qa[i + 1], bw.x);
              acc[i] = fminf(x0, y0);
              acc[i + 1] = fminf(x1, y1);
            }
            j += 2;
          } else {
            const float bx = s_tb[j].x;
#pragma unroll
            for (int i = 0; i < T; ++i) acc[i] = __fadd_rn(Qa[i], bx);
            ++j;
          }
          for (; j + 1 < jend; j += 2) {  // two columns: FADD2 per row pair + FMNMX3
            const float2 bv = s_tb[j], bw = s_tb[j + 1];
#pragma unroll
            for (int i = 0; i < T; i += 2) {
              float x0, x1, y0, y1;
              add2b(x0, x1, Qa[i], Qa[i + 1], bv.x);
              add2b(y0, y1, Qa[i], Qa[i + 1], bw.x);
              acc[i] = min3(acc[i], x0, y0);
              acc[i + 1] = min3(acc[i + 1], x1, y1);
            }
          }
          if (j < jend) {
            const float bx = s_tb[j].x;
#pragma unroll
            for (int i = 0; i < T; ++i) acc[i] = fminf(acc[i], __fadd_rn(Qa[i], bx));
            ++j;
          }
          fold(false);
        }
        continue;  // (every run initialises the row minima itself: no reset between a options)
      }
      for (int j = 0; j < P.Kb;) {
        const float2 bv = s_tb[j];
        const int U = ubase + __float_as_int(bv.y);
        if (U > A.bmax) break;  // u-sorted: the rest is over every budget
        const int l = s_lvl[U];
        if (l != cur) {
          if (cur >= 0) fold(true);
          cur = l;
        }
        if (j + 1 < P.Kb) {  // two columns of the same level: FADD2 per row pair + FMNMX3
          const float2 bw = s_tb[j + 1];
          const int U2 = ubase + __float_as_int(bw.y);
          if (U2 <= A.bmax && s_lvl[U2] == cur) {
#pragma unroll
            for (int i = 0; i < T; i += 2) {
              float x0, x1, y0, y1;
              add2b(x0, x1, Qa[i], Qa[i + 1], bv.x);  // {Q_i + b_j, Q_i+1 + b_j}
              add2b(y0, y1, Qa[i], Qa[i + 1], bw.x);  // {Q_i + b_j+1, Q_i+1 + b_j+1}
              acc[i] = min3(acc[i], x0, y0);
              acc[i + 1] = min3(acc[i + 1], x1, y1);
            }
            j += 2;
            continue;
          }
        }
#pragma unroll
        for (int i = 0; i < T; ++i) acc[i] = fminf(acc[i], __fadd_rn(Qa[i], bv.x));
        ++j;
      }
      if (cur >= 0) fold(true);
    }
  }
  __syncthreads();
  for (int l = tid; l < A.L; l += blockDim.x)
    if (s_best[l] != ~0ull) atomicMin(A.lvl_keys + l, s_best[l]);
}

// Per-query keys and counts from the level keys: key(b_g) = MIN over levels <= level(b_g) (prefix
// minimum), count(b_g) = sum over U <= b_g of the exact number of feasible candidates with U units
// (convolution of the per-LLM histograms of feasible options' units; one block).
__global__ void k_level_finish(const float *tau, const int *u, int M, int K, const int *levels, int L, int bmax,
                               const unsigned long long *lvl_keys, const int *q_level, int n,
                               unsigned long long *keys, unsigned long long *counts, unsigned long long *h0,
                               unsigned long long *h1) {
  const int tid = threadIdx.x;
  for (int U = tid; U <= bmax; U += blockDim.x) h0[U] = (U == 0) ? 1ull : 0ull;
  __syncthreads();
  unsigned long long *src = h0, *dst = h1;
  for (int m = 0; m < M; ++m) {
    for (int U = tid; U <= bmax; U += blockDim.x) {
      unsigned long long c = 0;
      for (int k = 0; k < K; ++k) {
        const int uk = u[m * K + k];
        if (uk <= U && tau[m * K + k] < __int_as_float(0x7f800000)) c += src[U - uk];
      }
      dst[U] = c;
    }
    __syncthreads();
    unsigned long long *t = src;
    src = dst;
    dst = t;
  }
  // src[U] = #feasible candidates with exactly U units; per query the prefix up to its budget
  for (int i = tid; i < n; i += blockDim.x) {
    const int g = q_level[i];
    unsigned long long key = ~0ull, cnt = 0;
    for (int l = 0; l <= g; ++l) key = min(key, lvl_keys[l]);
    for (int U = 0; U <= levels[g]; ++U) cnt += src[U];
    keys[i] = key == ~0ull ? kKeyNone : key;
    counts[i] = cnt;
  }
}

size_t levels_smem_bytes(const SearchArgs &s, int L, int bmax, LevelArgs *A) {
  auto a16 = [](size_t x) { return (x + 15) & ~size_t(15); };
  size_t off = a16((size_t)(s.g1 * s.K + 2) * 4);
  const size_t off_u = off;
  off = a16(off + (size_t)s.g0 * s.K * 4);
  const size_t off_pfx = off;
  const bool pfx = s.g0 > 0 && s.n_chunks <= kPfxTableMax;
  if (pfx) off = a16(off + (size_t)s.n_chunks * 8);
  const size_t off_ta = off;
  off = a16(off + (size_t)s.Ka * 8);
  const size_t off_tb = off;
  off = a16(off + (size_t)s.Kb * 8);
  const size_t off_best = off;
  off = a16(off + (size_t)L * 8);
  const size_t off_lvl = off;
  off = a16(off + (size_t)(bmax + 1) * 2);
  const size_t runs_bytes = (size_t)(bmax + 1) * (size_t)(s.Kb + 1) * 4;
  const bool runs = runs_bytes <= 48 * 1024;  // (C4: 9.8 KB; long b rows keep the per-column walk)
  const size_t off_runs = off;
  if (runs) off = a16(off + runs_bytes);
  if (A) {
    A->s.off_u = (int)off_u;
    A->s.off_pfx = pfx ? (int)off_pfx : -1;
    A->off_ta = (int)off_ta;
    A->off_tb = (int)off_tb;
    A->off_best = (int)off_best;
    A->off_lvl = (int)off_lvl;
    A->off_runs = runs ? (int)off_runs : -1;
    A->smem_bytes = (int)off;
  }
  return off;
}

// Launch the one-pass search (after the option terms of the target are in s.tau) and the finish.
cudaError_t launch_levels(const SearchArgs &s, const int *d_levels, int L, int bmax, unsigned long long *lvl_keys,
                          unsigned long long *ticket, const int *d_q_level, int n, unsigned long long *keys,
                          unsigned long long *counts, unsigned long long *h0, unsigned long long *h1, int sm_count,
                          cudaStream_t st) {
  LevelArgs A;
  A.s = s;
  A.levels = d_levels;
  A.L = L;
  A.bmax = bmax;
  A.lvl_keys = lvl_keys;
  A.ticket = ticket;
  levels_smem_bytes(s, L, bmax, &A);
  cudaError_t e;
  if ((e = cudaMemsetAsync(lvl_keys, 0xff, (size_t)L * 8, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(ticket, 0, 8, st)) != cudaSuccess) return e;
  static std::once_flag f[kMaxDevices];
  int dev = 0;
  cudaGetDevice(&dev);
  std::call_once(f[dev & (kMaxDevices - 1)], [] {
    cudaFuncSetAttribute(k_search_levels, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_search_levels, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  });
  int bps = 0;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_search_levels, kLvlThreads, A.smem_bytes)) != cudaSuccess)
    return e;
  if (bps < 1) return cudaErrorInvalidConfiguration;
  k_search_levels<<<sm_count * bps, kLvlThreads, A.smem_bytes, st>>>(A);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  k_level_finish<<<1, 1024, 0, st>>>(s.tau, s.u, s.M, s.K, d_levels, L, bmax, lvl_keys, d_q_level, n, keys, counts,
                                     h0, h1);
  return cudaGetLastError();
}

}  // namespace alp
