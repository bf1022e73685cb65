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

#include "alp_internal.h"

#ifndef ALP_A_UNROLL
#define ALP_A_UNROLL 2  // a-loop unroll (tuned: 2 beats 1 on C3 and C4, profiles/r01_variant_sweep.txt)
#endif

namespace alp {

constexpr int kAUnroll = ALP_A_UNROLL;

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

__global__ void k_init_keys(unsigned long long *keys, unsigned long long *counts, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    keys[i] = kKeyNone;
    counts[i] = 0ull;
  }
}

// ------------------------------------------------------------------ search kernel (K2)
// add.rn.f32x2 {v0,v1} = {q,q} + {b0,b1}  (SASS: FADD2 with scalar-broadcast operand)
__device__ __forceinline__ void add2(float &v0, float &v1, float q, float b0, float b1) {
  asm("{.reg .b64 x,y,z;\n\tmov.b64 x,{%2,%2};\n\tmov.b64 y,{%3,%4};\n\tadd.rn.f32x2 z,x,y;\n\tmov.b64 {%0,%1},z;}"
      : "=f"(v0), "=f"(v1)
      : "f"(q), "f"(b0), "f"(b1));
}
// add.rn.f32x2 {v0,v1} = {q0,q1} + {b,b}
__device__ __forceinline__ void add2b(float &v0, float &v1, float q0, float q1, float b) {
  asm("{.reg .b64 x,y,z;\n\tmov.b64 x,{%2,%3};\n\tmov.b64 y,{%4,%4};\n\tadd.rn.f32x2 z,x,y;\n\tmov.b64 {%0,%1},z;}"
      : "=f"(v0), "=f"(v1)
      : "f"(q0), "f"(q1), "f"(b));
}
// 3-input min (SASS: FMNMX3)
__device__ __forceinline__ float min3(float a, float b, float c) {
  float d;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

struct Smem {
  float *tau;      // [g1*K + 2] tau of prefix + sort-group LLMs (current target), then {0, +inf}; offset 0
  int *u;          // [g0*K] units of prefix LLMs
  float2 *a;       // [Ka] {tau_a, bits(-u_a)}; u_a := kBigUnits when tau_a is +inf
  int2 *lut;       // [R+2] {shared address of the masked row, #finite entries in it} for r = -1..R
  int *dv;         // [D] distinct b unit values <= R, ascending
  int *dcnt;       // [D+1] #u-sorted columns with u <= dv[i-1]
  float *btab;     // [rows][row_stride] masked rows
};

constexpr int kBigUnits = 1 << 28;

// a-table entry for option a (infeasible a gets +inf units -> maps to the all-+inf row)
__device__ __forceinline__ float2 a_entry(const SearchArgs &P, const float *tau_t, int a) {
  if (P.a_llm < 0) return make_float2(0.f, __int_as_float(0));
  const float ta = tau_t[P.a_llm * P.K + a];
  return make_float2(ta, __int_as_float(ta < __int_as_float(0x7f800000) ? -P.u[P.a_llm * P.K + a] : -kBigUnits));
}
// masked-row element (row, j) of b-chunk [c0, c1): tau_b of the j-th u-sorted column if it fits
__device__ __forceinline__ float btab_entry(const SearchArgs &P, const float *tau_t, const int *dcnt, int row, int j,
                                            int c0, int c1) {
  const int len = min(max(dcnt[row], c0), c1) - c0;
  return (j < len) ? tau_t[P.b_llm * P.K + P.bperm[c0 + j]] : __int_as_float(0x7f800000);
}
// budget of query t (per-query budgets for budget sweeps, else the common budget)
__device__ __forceinline__ int qbudget(const SearchArgs &P, int t) { return P.q_budget ? P.q_budget[t] : P.budget; }

// masked-row index for remaining budget r: #{distinct b unit values <= r}
__device__ __forceinline__ int row_of(const int *dv, int D, int r) {
  int lo = 0, hi = D;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (dv[mid] <= r) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ Smem smem_layout(const SearchArgs &P, unsigned char *base) {
  Smem s;
  s.tau = reinterpret_cast<float *>(base + P.off_tau);
  s.u = reinterpret_cast<int *>(base + P.off_u);
  s.a = reinterpret_cast<float2 *>(base + P.off_a);
  s.lut = reinterpret_cast<int2 *>(base + P.off_lut);
  s.dv = reinterpret_cast<int *>(base + P.off_tmp);
  s.dcnt = s.dv + (P.Kb + 1);
  s.btab = reinterpret_cast<float *>(base + P.off_btab);
  return s;
}

// Build the per-(target, b-chunk) tables in shared memory.  All threads participate.
__device__ void build_tables(const SearchArgs &P, const Smem &s, int t, int c, int R) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int K = P.K, D = row_of(P.dv, P.D, R);
  const float *tau_t = P.tau + (size_t)t * P.M * K;
  const int c0 = c * P.bchunk_w;
  const int c1 = min(c0 + P.bchunk_w, P.Kb);
  for (int i = tid; i < P.g1 * K; i += nt) s.tau[i] = tau_t[i];
  if (tid == 0) {
    s.tau[P.g1 * K] = 0.f;         // unused sort-group digit slot: x + 0 = x exactly
    s.tau[P.g1 * K + 1] = finf();  // padded (dummy) row
  }
  for (int i = tid; i < P.g0 * K; i += nt) s.u[i] = P.u[i];
  for (int a = tid; a < P.Ka; a += nt) s.a[a] = a_entry(P, tau_t, a);
  for (int i = tid; i < D; i += nt) s.dv[i] = P.dv[i];
  for (int i = tid; i <= D; i += nt) s.dcnt[i] = P.dcnt[i];
  __syncthreads();
  // masked row i holds the u-sorted columns [c0, c1) with u <= dv[i-1] (row 0: none), +inf elsewhere
  const int rows = D + 1;
  for (int i = tid; i < rows * P.bchunk_wpad; i += nt) {
    const int row = i / P.bchunk_wpad, j = i % P.bchunk_wpad;
    s.btab[row * P.row_stride + j] = btab_entry(P, tau_t, s.dcnt, row, j, c0, c1);
  }
  __syncthreads();
  // finite entries per masked row (feasible b count), kept in the row's padding column
  const int warp = tid >> 5, lane = tid & 31, nwarp = nt >> 5;
  for (int row = warp; row < rows; row += nwarp) {
    unsigned n = 0;
    for (int j = lane; j < P.bchunk_wpad; j += 32) n += (s.btab[row * P.row_stride + j] < finf()) ? 1u : 0u;
    n = __reduce_add_sync(0xffffffffu, n);
    if (lane == 0) s.btab[row * P.row_stride + P.bchunk_wpad] = __int_as_float((int)n);
  }
  __syncthreads();
  // r -> masked row: index = #{distinct b unit values <= r}
  for (int r = tid - 1; r <= R; r += nt) {
    const int lo = row_of(s.dv, D, r);
    s.lut[r + 1] = make_int2((int)(uint32_t)__cvta_generic_to_shared(s.btab + lo * P.row_stride),
                             __float_as_int(s.btab[lo * P.row_stride + P.bchunk_wpad]));
  }
  __syncthreads();
}

__device__ __forceinline__ float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ float2 lds64(uint32_t addr) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
  return v;
}

// "candidate = Q_a + tau_b; acc = min(acc, candidate)" for 4 b values and T rows:
//   FADD2 {Q_i, Q_i+1} + {b, b} per (row pair, b)   (add.rn.f32x2; the b operand is a scalar broadcast)
//   FMNMX3 acc_i = min(acc_i, v_b0, v_b1)           (3-input min)
// = one issue slot per candidate.  The row-pair form lets the Q pair sit in the operand-reuse cache
// across the 4 b values (tools/microbench/pipes3: fastest of the encodings tried).
template <int T>
__device__ __forceinline__ void eval4(const float4 bv, const float (&Qa)[T], float (&acc)[T]) {
#pragma unroll
  for (int i = 0; i < T; i += 2) {
    float a0, b0, a1, b1, a2, b2, a3, b3;
    add2b(a0, b0, Qa[i], Qa[i + 1], bv.x);
    add2b(a1, b1, Qa[i], Qa[i + 1], bv.y);
    add2b(a2, b2, Qa[i], Qa[i + 1], bv.z);
    add2b(a3, b3, Qa[i], Qa[i + 1], bv.w);
    acc[i] = min3(acc[i], a0, a1);
    acc[i + 1] = min3(acc[i + 1], b0, b1);
    acc[i] = min3(acc[i], a2, a3);
    acc[i + 1] = min3(acc[i + 1], b2, b3);
  }
}

template <int T>
__device__ __forceinline__ void eval2(const float2 bv, const float (&Qa)[T], float (&acc)[T]) {
#pragma unroll
  for (int i = 0; i < T; i += 2) {
    float a0, b0, a1, b1;
    add2b(a0, b0, Qa[i], Qa[i + 1], bv.x);
    add2b(a1, b1, Qa[i], Qa[i + 1], bv.y);
    acc[i] = min3(acc[i], a0, a1);
    acc[i + 1] = min3(acc[i + 1], b0, b1);
  }
}

template <int T, int NB4, bool TAIL2>
__device__ __forceinline__ void eval_row(uint32_t rp, const float (&Qa)[T], float (&acc)[T], int ng4) {
  if constexpr (NB4 > 0) {
#pragma unroll
    for (int g = 0; g < NB4; ++g) eval4<T>(lds128(rp + 16 * g), Qa, acc);
  } else {
#pragma unroll 2
    for (int g = 0; g < ng4; ++g) eval4<T>(lds128(rp + 16 * g), Qa, acc);
  }
  if constexpr (TAIL2) eval2<T>(lds64(rp + (NB4 > 0 ? NB4 : ng4) * 16), Qa, acc);
}

// Fold a lane tile's per-row minima into the thread's best (value, segment).  Segment of a row =
// row * nQ + q0, q0 = first a-range this warp evaluated for the row; K3 re-scans from there.
// The tile's packed digits are read only when a row can improve the best (rare).
template <int T>
__device__ __forceinline__ void fold_rows(const SearchArgs &P, const float (&acc)[T], uint32_t tile, uint32_t chunk,
                                          uint32_t q0, float &best, uint32_t &best_seg) {
  bool any = false;
#pragma unroll
  for (int i = 0; i < T; ++i) any |= (acc[i] <= best) && (acc[i] < finf());
  if (!any) return;
  const uint32_t dmask = (1u << P.dig_bits) - 1u;
  for (int i = 0; i < T; ++i) {
    if (acc[i] <= best && acc[i] < finf()) {
      const uint32_t e = __ldg(P.tile_e + (size_t)tile * T + i);
      uint32_t ec = 0;  // canonical within-group index: LLM g0 most significant
      for (int j = 0; j < P.ng; ++j) ec = ec * (uint32_t)P.K + ((e >> (j * P.dig_bits)) & dmask);
      const uint32_t seg = (chunk * P.L + ec) * P.nQ + q0;
      if (acc[i] < best || seg < best_seg) {
        best = acc[i];
        best_seg = seg;
      }
    }
  }
}

template <int T, int NB4, bool TAIL2>
__device__ void process_items(const SearchArgs &P, const Smem &s, unsigned char *base, float &best,
                              uint32_t &best_seg, unsigned long long &cnt, int R) {
  const int lane = threadIdx.x & 31;
  const uint64_t nW = (uint64_t)gridDim.x * (blockDim.x >> 5);
  const uint64_t w = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const uint64_t n = P.item_hi - P.item_lo;
  uint64_t it = P.item_lo + n * w / nW;
  const uint64_t end = P.item_lo + n * (w + 1) / nW;
  if (it >= end) return;
  const int K = P.K;
  const int ng4 = P.bchunk_wpad >> 2;
  uint32_t q = (uint32_t)(it % P.nQ);
  const uint64_t tq = it / P.nQ;
  uint32_t grp = (uint32_t)(tq % P.n_groups);
  uint32_t chunk = (uint32_t)(tq / P.n_groups);
  // state of the lane tile currently loaded
  float Qr[T], acc[T];
  int r_tile = 0;
  unsigned nfin = 0;
  uint32_t q0 = q, tchunk = chunk, ttile = 0;
  bool loaded = false;
  float Pfx = 0.f;
  int Upfx = 0;
  uint32_t pchunk = 0xffffffffu;
  const unsigned char *tau_b = reinterpret_cast<const unsigned char *>(s.tau);
  for (; it < end; ++it) {
    if (!loaded) {
      if (chunk != pchunk) {
        // canonical partial sum over LLMs 0..g0-1 (LLM 0 most significant): ((0 + tau_0) + tau_1) + ...
        float pa = 0.f;
        int U = 0;
        for (int m = 0; m < P.g0; ++m) {
          const uint32_t d = (chunk / P.pw[m]) % (uint32_t)K;
          pa = __fadd_rn(pa, s.tau[m * K + d]);
          U += s.u[m * K + d];
        }
        Pfx = pa;
        Upfx = U;
        pchunk = chunk;
      }
      const uint32_t tile = grp * kWarpTiles + lane;
      const int stile = __ldg(P.tile_s + tile);
      // per row: 4 smem byte offsets (16 bits each) of the sort-group terms, in LLM order;
      // unused digits point at 0.0f, padded rows at +inf
      const uint4 *op = reinterpret_cast<const uint4 *>(P.tile_off) + (size_t)tile * (T / 2);
      nfin = 0;
#pragma unroll
      for (int v = 0; v < T / 2; ++v) {
        const uint4 o = __ldg(op + v);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t w0 = h ? o.z : o.x, w1 = h ? o.w : o.y;
          float qv = Pfx;
          qv = __fadd_rn(qv, *reinterpret_cast<const float *>(tau_b + (w0 & 0xffffu)));
          qv = __fadd_rn(qv, *reinterpret_cast<const float *>(tau_b + (w0 >> 16)));
          qv = __fadd_rn(qv, *reinterpret_cast<const float *>(tau_b + (w1 & 0xffffu)));
          qv = __fadd_rn(qv, *reinterpret_cast<const float *>(tau_b + (w1 >> 16)));
          Qr[2 * v + h] = qv;
          nfin += (qv < finf()) ? 1u : 0u;
          acc[2 * v + h] = finf();
        }
      }
      r_tile = R - Upfx - stile;
      q0 = q;
      tchunk = chunk;
      ttile = tile;
      loaded = true;
    }
    unsigned c32 = 0;
    const int a0 = (int)(q * P.A);
    const int a1 = min(a0 + (int)P.A, P.Ka);
    const float2 *ap = s.a + a0;
#pragma unroll(kAUnroll)
    for (int a = a0; a < a1; ++a, ++ap) {
      const float2 av = *ap;
      const int ra = max(r_tile + __float_as_int(av.y), -1);
      const int2 lu = s.lut[ra + 1];
      c32 += (unsigned)lu.y;
      float Qa[T];
#pragma unroll
      for (int i = 0; i < T; i += 2) add2b(Qa[i], Qa[i + 1], Qr[i], Qr[i + 1], av.x);
      eval_row<T, NB4, TAIL2>((uint32_t)lu.x, Qa, acc, ng4);
    }
    cnt += (unsigned long long)c32 * nfin;  // rows with a finite partial sum x feasible (a, b) pairs
    // advance to the next item (q fastest); fold when the lane tile changes
    if (++q == P.nQ) {
      q = 0;
      fold_rows<T>(P, acc, ttile, tchunk, q0, best, best_seg);
      loaded = false;
      if (++grp == P.n_groups) {
        grp = 0;
        ++chunk;
      }
    }
  }
  if (loaded) fold_rows<T>(P, acc, ttile, tchunk, q0, best, best_seg);
}

// T = rows per lane; MB = minimum resident blocks per SM (register cap 65536 / (256 * MB)).
template <int T, int NB4, bool TAIL2, int MB>
__global__ void __launch_bounds__(kThreads, MB)
    k_search(const __grid_constant__ SearchArgs P) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ unsigned long long red_key[kThreads / 32], red_cnt[kThreads / 32];
  const Smem s = smem_layout(P, smem);
  for (int t = P.t_begin; t < P.t_end; ++t) {
    float best = finf();
    uint32_t best_seg = 0xffffffffu;
    unsigned long long cnt = 0ull;
    for (int c = P.c_begin; c < P.c_end; ++c) {
      __syncthreads();
      const int R = qbudget(P, t);
      build_tables(P, s, t, c, R);
      process_items<T, NB4, TAIL2>(P, s, smem, best, best_seg, cnt, R);
    }
    unsigned long long key = (best < finf()) ? ((unsigned long long)__float_as_uint(best) << 32) | best_seg : kKeyNone;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long ok = __shfl_xor_sync(0xffffffffu, key, o);
      const unsigned long long oc = __shfl_xor_sync(0xffffffffu, cnt, o);
      key = ok < key ? ok : key;
      cnt += oc;
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
      red_key[warp] = key;
      red_cnt[warp] = cnt;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long k = red_key[0], n = red_cnt[0];
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
        k = red_key[w] < k ? red_key[w] : k;
        n += red_cnt[w];
      }
      if (k != kKeyNone) atomicMin(P.keys + t, k);
      if (n) atomicAdd(P.counts + t, n);
    }
  }
}

// Host-side dispatch over rows per lane (T) and the b-chunk width specialisations.
// Register-cap variants: T = 8 -> 3 (default) or 4 blocks/SM; T = 16 -> 2 (default) or 3.
template <int T, int NB4, bool TAIL2>
static auto pick(const SearchArgs &a) {
  constexpr int kLo = (T == 8) ? 3 : 2, kHi = (T == 8) ? 4 : 3;
  if (a.min_blocks == kHi) return k_search<T, NB4, TAIL2, kHi>;
  return k_search<T, NB4, TAIL2, kLo>;
}

template <int T, int NB4, bool TAIL2>
static cudaError_t launch_one(const SearchArgs &a, int grid, cudaStream_t st) {
  auto fn = pick<T, NB4, TAIL2>(a);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, a.smem_bytes);
  if (e != cudaSuccess) return e;
  fn<<<grid, kThreads, a.smem_bytes, st>>>(a);
  return cudaGetLastError();
}

template <int T, int NB4, bool TAIL2>
static int occ_one(const SearchArgs &a) {
  auto fn = pick<T, NB4, TAIL2>(a);
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, a.smem_bytes) != cudaSuccess) return 0;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, kThreads, a.smem_bytes) != cudaSuccess) return 0;
  return n;
}

// Fully unrolled b loop for chunk widths <= 34 columns: NB4 LDS.128 groups plus an optional LDS.64
// tail; wider chunks use the runtime loop (NB4 = 0).
#define ALP_DISPATCH_W(CALL, T)                                              \
  do {                                                                       \
    const int w = a.bchunk_wpad;                                             \
    const bool t2 = (w % 4) == 2;                                            \
    if (w > 34) {                                                            \
      if (t2) return CALL(T, 0, true);                                       \
      return CALL(T, 0, false);                                              \
    }                                                                        \
    switch (w) {                                                             \
      case 2: return CALL(T, 0, true);                                       \
      case 4: return CALL(T, 1, false); case 6: return CALL(T, 1, true);     \
      case 8: return CALL(T, 2, false); case 10: return CALL(T, 2, true);    \
      case 12: return CALL(T, 3, false); case 14: return CALL(T, 3, true);   \
      case 16: return CALL(T, 4, false); case 18: return CALL(T, 4, true);   \
      case 20: return CALL(T, 5, false); case 22: return CALL(T, 5, true);   \
      case 24: return CALL(T, 6, false); case 26: return CALL(T, 6, true);   \
      case 28: return CALL(T, 7, false); case 30: return CALL(T, 7, true);   \
      case 32: return CALL(T, 8, false); case 34: return CALL(T, 8, true);   \
      default: if (t2) return CALL(T, 0, true); return CALL(T, 0, false);    \
    }                                                                        \
  } while (0)

#define ALP_DISPATCH(CALL)                  \
  do {                                      \
    if (a.rows_per_lane == 16) ALP_DISPATCH_W(CALL, 16); \
    ALP_DISPATCH_W(CALL, 8);                \
  } while (0)

cudaError_t launch_search(const SearchArgs &a, int grid, cudaStream_t st) {
#define CALL(T, N, T2) launch_one<T, N, T2>(a, grid, st)
  ALP_DISPATCH(CALL);
#undef CALL
}

int search_max_blocks_per_sm(const SearchArgs &a) {
#define CALL(T, N, T2) occ_one<T, N, T2>(a)
  ALP_DISPATCH(CALL);
#undef CALL
}

// ------------------------------------------------------------------ finalize (K3)
__global__ void k_finalize(const FinalizeArgs F) {
  const SearchArgs &P = F.s;
  const int t = blockIdx.x;
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
    for (unsigned long long li = threadIdx.x; li < n; li += blockDim.x) {
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
  if (threadIdx.x != 0) return;
  alp_result r;
  memset(&r, 0, sizeof(r));
  r.M = P.M;
  r.feasible_count = count;
  r.candidates = F.N;
  r.index = ~0ull;
  r.latency_key = finf();
  if (found && s_best != ~0ull) {
    const int a0 = (int)(q * P.A);
    const int a = a0 + (int)(s_best / P.Kb), b = (int)(s_best % P.Kb);
    int k[ALP_MAX_M];
    uint32_t rem = chunk;
    for (int m = P.g0 - 1; m >= 0; --m) {
      k[m] = (int)(rem % (uint32_t)K);
      rem /= (uint32_t)K;
    }
    rem = e;
    for (int j = P.ng - 1; j >= 0; --j) {
      k[P.g0 + j] = (int)(rem % (uint32_t)K);
      rem /= (uint32_t)K;
    }
    if (P.a_llm >= 0) k[P.a_llm] = a;
    k[P.b_llm] = b;
    unsigned long long idx = 0;
    double L = 0.0, Tw = CUDART_INF;
    long long U = 0;
    const double *term_t = F.term + (size_t)t * P.M * K;
    const double *b_t = F.b + (size_t)t * P.M * K;
    for (int m = 0; m < P.M; ++m) {
      idx = idx * (unsigned long long)K + (unsigned long long)k[m];
      const double tm = term_t[m * K + k[m]];
      L = (m == 0) ? tm : __dadd_rn(L, tm);  // Eq. 1 in canonical order (FP64)
      const double bm = b_t[m * K + k[m]];
      Tw = bm < Tw ? bm : Tw;                // Eq. 2
      U += P.u[m * K + k[m]];
      if (F.S) {
        const int s_i = k[m] / (F.nR * F.nT), t_i = (k[m] / F.nR) % F.nT, r_i = k[m] % F.nR;
        r.share_units[m] = F.S[s_i];
        r.tp[m] = F.T[t_i];
        r.replicas[m] = F.R[r_i];
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
  const int n = total > a.n_targets ? total : a.n_targets;
  k_option_table<<<(n + 255) / 256, 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_init_keys(unsigned long long *keys, unsigned long long *counts, int n, cudaStream_t st) {
  k_init_keys<<<(n + 255) / 256, 256, 0, st>>>(keys, counts, n);
  return cudaGetLastError();
}

cudaError_t launch_finalize(const FinalizeArgs &a, cudaStream_t st) {
  k_finalize<<<a.s.n_targets, 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_predict(const PredictArgs &a, cudaStream_t st) {
  k_predict<<<(a.n + 127) / 128, 128, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace alp
