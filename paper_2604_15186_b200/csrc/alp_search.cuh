// Search kernel K2 (k_search) and its launch helpers, shared by the per-rows-per-lane translation
// units alp_search_t8.cu / alp_search_t16.cu (split so nvcc compiles them in parallel).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <mutex>

#include "alp_finalize.cuh"
#include "alp_internal.h"
#include "alp_terms.cuh"

#ifndef ALP_A_UNROLL
#define ALP_A_UNROLL 2  // a-loop unroll (tuned: 2 beats 1 on C3 and C4, profiles/r01_variant_sweep.txt)
#endif

namespace alp {

constexpr int kAUnroll = ALP_A_UNROLL;

__device__ __forceinline__ float finf() { return __int_as_float(0x7f800000); }

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
  int *bperm;      // [Kb] canonical b option of u-sorted column j
  int *ua;         // [Ka] units of the a options
  float *btab;     // [rows][row_stride] masked rows
  float2 *pfx;     // [n_chunks] {prefix partial sum, bits(prefix units)} when P.off_pfx >= 0
  float *opt;      // [M*K] option terms of the phase's target (fused mode)
};

constexpr int kBigUnits = 1 << 28;

// a-table entry for option a (infeasible a gets +inf units -> maps to the all-+inf row)
__device__ __forceinline__ float2 a_entry(const SearchArgs &P, const float *tau_t, const int *ua, int a) {
  if (P.a_llm < 0) return make_float2(0.f, __int_as_float(0));
  const float ta = tau_t[P.a_llm * P.K + a];
  return make_float2(ta, __int_as_float(ta < __int_as_float(0x7f800000) ? -ua[a] : -kBigUnits));
}
// masked-row element (row, j) of b-chunk [c0, c1): tau_b of the j-th u-sorted column if it fits
__device__ __forceinline__ float btab_entry(const SearchArgs &P, const float *tau_t, const int *dcnt,
                                            const int *bperm, int row, int j, int c0, int c1) {
  const int len = min(max(dcnt[row], c0), c1) - c0;
  return (j < len) ? tau_t[P.b_llm * P.K + bperm[c0 + j]] : __int_as_float(0x7f800000);
}
// masked-row index for remaining budget r: #{distinct b unit values <= r}
__device__ __forceinline__ int row_of(const int *dv, int D, int r) {
  int lo = 0, hi = D;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (dv[mid] <= r) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// n / d for n < 2^31 with a host-computed multiplier (FastDiv in alp_internal.h)
__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv &f) {
  return f.mul ? (__umulhi(n, f.mul) >> f.shift) : n;
}

// canonical partial sum over LLMs 0..g0-1 of a prefix chunk (LLM 0 most significant):
// ((0 + tau_0) + tau_1) + ..., and its units
__device__ __forceinline__ void prefix_sum(const SearchArgs &P, const Smem &s, uint32_t chunk, float &pa, int &U) {
  pa = 0.f;
  U = 0;
  for (int m = 0; m < P.g0; ++m) {
    const uint32_t d = (chunk / P.pw[m]) % (uint32_t)P.K;
    pa = __fadd_rn(pa, s.tau[m * P.K + d]);
    U += s.u[m * P.K + d];
  }
}

__device__ __forceinline__ Smem smem_layout(const SearchArgs &P, unsigned char *base) {
  Smem s;
  s.tau = reinterpret_cast<float *>(base + P.off_tau);
  s.u = reinterpret_cast<int *>(base + P.off_u);
  s.a = reinterpret_cast<float2 *>(base + P.off_a);
  s.lut = reinterpret_cast<int2 *>(base + P.off_lut);
  s.dv = reinterpret_cast<int *>(base + P.off_tmp);
  s.dcnt = s.dv + (P.Kb + 1);
  s.bperm = s.dcnt + (P.Kb + 2);
  s.ua = s.bperm + P.Kb;
  s.btab = reinterpret_cast<float *>(base + P.off_btab);
  s.pfx = reinterpret_cast<float2 *>(base + (P.off_pfx >= 0 ? P.off_pfx : 0));
  s.opt = reinterpret_cast<float *>(base + (P.fz.on ? P.fz.off_opt : 0));
  return s;
}

// Build the per-(target, b-chunk) tables in shared memory.  All threads participate.
// The target-independent tables (static plan) in shared memory, once per block, before the
// option terms exist: one wave of global loads (no dependency on K1 / the fused prologue).
// Asynchronous copies (cp.async, no register staging): the thread goes on to the option terms
// while they land; cp_async_wait() + a barrier make them visible.
__device__ __forceinline__ void cp_async4(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ inline void load_static(const SearchArgs &P, const Smem &s) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int i = tid; i < P.g0 * P.K; i += nt) cp_async4(s.u + i, P.u + i);
  for (int i = tid; i < P.D; i += nt) cp_async4(s.dv + i, P.dv + i);
  for (int i = tid; i <= P.D; i += nt) cp_async4(s.dcnt + i, P.dcnt + i);
  for (int i = tid; i < P.Kb; i += nt) cp_async4(s.bperm + i, P.bperm + i);
  if (P.a_llm >= 0)
    for (int i = tid; i < P.Ka; i += nt) cp_async4(s.ua + i, P.u + P.a_llm * P.K + i);
}

// Build the per-(target, b-chunk) tables in shared memory.  All threads participate; the static
// tables (load_static) are visible (a barrier separates them).
__device__ inline void build_tables(const SearchArgs &P, const Smem &s, const float *tau_t, int c, int R) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int K = P.K, D = row_of(s.dv, P.D, R);
  const int c0 = c * P.bchunk_w;
  const int c1 = min(c0 + P.bchunk_w, P.Kb);
  for (int i = tid; i < P.g1 * K; i += nt) s.tau[i] = tau_t[i];
  if (tid == 0) {
    s.tau[P.g1 * K] = 0.f;         // unused sort-group digit slot: x + 0 = x exactly
    s.tau[P.g1 * K + 1] = finf();  // padded (dummy) row
  }
  for (int a = tid; a < P.Ka; a += nt) s.a[a] = a_entry(P, tau_t, s.ua, a);
  // masked row i holds the u-sorted columns [c0, c1) with u <= dv[i-1] (row 0: none), +inf elsewhere
  const int rows = D + 1;
  for (int i = tid; i < rows * P.bchunk_wpad; i += nt) {
    const int row = i / P.bchunk_wpad, j = i % P.bchunk_wpad;
    s.btab[row * P.row_stride + j] = btab_entry(P, tau_t, s.dcnt, s.bperm, row, j, c0, c1);
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
  // prefix chunk table (small prefix spaces): one canonical partial sum per chunk
  if (P.off_pfx >= 0)
    for (uint32_t c = tid; c < P.n_chunks; c += nt) {
      float pa;
      int U;
      prefix_sum(P, s, c, pa, U);
      s.pfx[c] = make_float2(pa, __int_as_float(U));
    }
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
    // runtime b-chunk width (long rows, C3): unroll 8 (C3 3.148 -> 3.039 ms vs unroll 2)
#pragma unroll 8
    for (int g = 0; g < ng4; ++g) eval4<T>(lds128(rp + 16 * g), Qa, acc);
  }
  if constexpr (TAIL2) eval2<T>(lds64(rp + (NB4 > 0 ? NB4 : ng4) * 16), Qa, acc);
}

// Fold a lane tile's per-row minima into the thread's best (value, segment).  Segment of a row =
// row * seg_q + qs, qs = (first a option this warp evaluated for the row) / seg_A; K3 re-scans from
// there to the end of the row.
// The row's canonical within-group index is read only when the row can improve the best.
template <int T>
__device__ __forceinline__ void fold_rows(const SearchArgs &P, const float (&acc)[T], uint32_t tile, uint32_t chunk,
                                          uint32_t qs, float &best, uint32_t &best_seg) {
  // tile minimum first (FMNMX3 tree); the rows' canonical indices are read only when it can
  // improve the best (value, segment)
  float m = acc[0];
#pragma unroll
  for (int i = 1; i + 1 < T; i += 2) m = min3(m, acc[i], acc[i + 1]);
  if (T % 2 == 0) m = fminf(m, acc[T - 1]);
  if (!(m <= best) || !(m < finf())) return;
  uint32_t bs = 0xffffffffu;
#pragma unroll
  for (int i = 0; i < T; ++i) {
    if (acc[i] == m) {
      const uint32_t ec = __ldg(P.tile_e + (size_t)tile * T + i);  // canonical within-group index
      bs = min(bs, (chunk * P.L + ec) * P.seg_q + qs);
    }
  }
  if (m < best) {
    best = m;
    best_seg = bs;
  } else if (bs < best_seg) {  // m == best: lowest segment wins
    best_seg = bs;
  }
}

// Load a lane tile: the canonical partial sums Q_row = (((P + tau_g0) + ...) of its T rows from the
// chunk prefix P and the sort-group terms in shared memory (4 byte offsets per row, in LLM order;
// unused digits point at 0.0f, padded rows at +inf); resets the row minima.  Returns the number of
// rows with a finite partial sum.
template <int T>
__device__ __forceinline__ unsigned load_tile(const SearchArgs &P, const unsigned char *tau_b, float pfx,
                                              uint32_t tile, float (&Qr)[T], float (&acc)[T]) {
  const uint4 *op = reinterpret_cast<const uint4 *>(P.tile_off) + (size_t)tile * T;
  unsigned nfin = 0;
#pragma unroll
  for (int v = 0; v < T; ++v) {
    const uint4 o = __ldg(op + v);
    float qv = pfx;
    qv = __fadd_rn(qv, *reinterpret_cast<const float *>(tau_b + o.x));
    qv = __fadd_rn(qv, *reinterpret_cast<const float *>(tau_b + o.y));
    qv = __fadd_rn(qv, *reinterpret_cast<const float *>(tau_b + o.z));
    qv = __fadd_rn(qv, *reinterpret_cast<const float *>(tau_b + o.w));
    Qr[v] = qv;
    nfin += (qv < finf()) ? 1u : 0u;
    acc[v] = finf();
  }
  return nfin;
}

template <int T, int NB4, bool TAIL2>
__device__ void process_items(const SearchArgs &P, const Smem &s, unsigned char *base, float &best,
                              uint32_t &best_seg, unsigned long long &cnt, int R, int work_slot) {
  const int lane = threadIdx.x & 31;
  const uint64_t n = P.item_hi - P.item_lo;
  const int ng4 = P.bchunk_wpad >> 2;
  // Dynamic work distribution: warps take runs of P.grab consecutive items from this phase's
  // counter (the result is independent of who evaluates what: keys carry (value, segment) and the
  // counts are sums).  The next run is requested while the current one is evaluated.
  // Guided tickets: the first grab_t1 tickets cover P.grab items each, later ones P.grab2 (<= grab)
  // so the last grabs of the phase are short (tail balance).
  unsigned long long *ctr = P.work + work_slot;
  unsigned long long tk = 0;
  if (lane == 0) tk = atomicAdd(ctr, 1ull);
  tk = __shfl_sync(0xffffffffu, tk, 0);
  // state of the lane tile currently loaded
  float Qr[T], acc[T];
  int r_tile = 0;
  unsigned nfin = 0;
  uint32_t q0 = 0, tchunk = 0, ttile = 0;
  float Pfx = 0.f;
  int Upfx = 0;
  uint32_t pchunk = 0xffffffffu;
  const unsigned char *tau_b = reinterpret_cast<const unsigned char *>(s.tau);
  const bool small = P.item_hi < (1ull << 31);  // 32-bit item decode with host-computed fast divisors
  for (;;) {
  const uint64_t t1 = (uint64_t)P.grab_t1;
  const uint64_t nxt = tk < t1 ? tk * (uint64_t)P.grab : t1 * (uint64_t)P.grab + (tk - t1) * (uint64_t)P.grab2;
  if (nxt >= n) break;
  uint64_t it = P.item_lo + nxt;
  const uint64_t end = P.item_lo + min((unsigned long long)n,
                                       nxt + (unsigned long long)(tk < t1 ? P.grab : P.grab2));
  if (lane == 0) tk = atomicAdd(ctr, 1ull);
  uint32_t q, grp, chunk;
  if (small) {
    const uint32_t i32 = (uint32_t)it;
    const uint32_t tq = fdiv(i32, P.fd_nQ);
    q = i32 - tq * P.nQ;
    chunk = fdiv(tq, P.fd_ng);
    grp = tq - chunk * P.n_groups;
  } else {
    q = (uint32_t)(it % P.nQ);
    const uint64_t tq = it / P.nQ;
    grp = (uint32_t)(tq % P.n_groups);
    chunk = (uint32_t)(tq / P.n_groups);
  }
  bool loaded = false;
  for (; it < end; ++it) {
    if (!loaded) {
      if (chunk != pchunk) {
        if (P.off_pfx >= 0) {
          const float2 pf = s.pfx[chunk];  // table built per phase (build_tables)
          Pfx = pf.x;
          Upfx = __float_as_int(pf.y);
        } else {
          prefix_sum(P, s, chunk, Pfx, Upfx);
        }
        pchunk = chunk;
      }
      const uint32_t tile = grp * kWarpTiles + lane;
      const int stile = __ldg(P.tile_s + tile);
      nfin = load_tile<T>(P, tau_b, Pfx, tile, Qr, acc);
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
      fold_rows<T>(P, acc, ttile, tchunk, q0 * P.seg_mul, best, best_seg);
      loaded = false;
      if (++grp == P.n_groups) {
        grp = 0;
        ++chunk;
      }
    }
  }
  if (loaded) fold_rows<T>(P, acc, ttile, tchunk, q0 * P.seg_mul, best, best_seg);
  tk = __shfl_sync(0xffffffffu, tk, 0);
  }
}

// Fused prologue: the option terms of target t (K1's arithmetic, alp_terms.cuh) into shared memory;
// block 0 also publishes them (with the FP64 Eq. 1 / Eq. 2 terms) for the finalize.
__device__ inline void fused_terms(const SearchArgs &P, const Smem &s, int t, bool publish) {
  const int MK = P.M * P.K;
  const bool wr = publish && blockIdx.x == 0;
  const DevProfiles &sp = P.fz.prof;
  for (int i = threadIdx.x; i < MK; i += blockDim.x) {
    float tau;
    if (P.fz.tau_fixed) {
      tau = P.fz.tau_fixed[i];
    } else {
      double term, b;
      int u;
      option_terms(sp, P.fz.tgt[t], i / P.K, i % P.K, &tau, &term, &b, &u);
      if (wr) {
        P.fz.o_term[(size_t)t * MK + i] = term;
        P.fz.o_b[(size_t)t * MK + i] = b;
      }
    }
    s.opt[i] = tau;
    if (wr) P.fz.o_tau[(size_t)t * MK + i] = tau;
  }
  __syncthreads();
}

// ------------------------------------------------------------------ peer exchange (alp_search_peer)
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ long long globaltimer_ns() {
  unsigned long long g;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
  return (long long)g;
}

// The cross-GPU reduction inside the search kernel's last block, over peer
// memory instead of a collective + K3 launch.  The epilogue (inlined: kernel parameters come from
// the constant bank) finalizes this rank's own (key, count) into its row of slot p = epoch & 1 (its
// key's segment lies in its own shard, so the local re-scan is the global one if this key wins);
// then peer_exchange stores the (key, count, result) rows into slot p of every rank's buffer
// (NVLink stores), publishes them with one system-scope fence + a flag per destination, waits for
// all ranks' flags in the own buffer (acquire), and takes the MIN over the keys, the SUM over the
// counts and the winning rank's result.  Keys carry global segment ids and whole rows live on one
// rank, so equal keys never come from two ranks.  Buffer layout: PeerRow, kPeerHdr (alp_internal.h).
__device__ __forceinline__ PeerRow *peer_rows(unsigned char *b, unsigned long long e, int W, int n, int j) {
  return reinterpret_cast<PeerRow *>(b + kPeerHdr) + ((size_t)(e & 1) * W + j) * n;
}
__device__ __forceinline__ unsigned long long *peer_flag(unsigned char *b, unsigned long long e, int j) {
  return reinterpret_cast<unsigned long long *>(b + 64) + (size_t)(e & 1) * kMaxPeers + j;
}

// Not inlined (ptxas keeps the search loops' uniform datapath only while this code stays out of the
// kernel body); everything it needs comes in as scalars or from shared memory (a reference to the
// kernel parameters would turn every field access into a generic load).
static __device__ __noinline__ void peer_exchange(unsigned char *const *s_buf, int me, int W, int n,
                                                  unsigned long long e, alp_result *out, long long timeout_ns,
                                                  unsigned long long *dbg) {
  static_assert(sizeof(PeerRow) % 8 == 0 && sizeof(alp_result) % 8 == 0, "rows move as 64-bit words");
  auto stamp = [&](int i) {  // ALP_DBG_TS: the exchange's phases (SM clock cycles)
    if (dbg && threadIdx.x == 0) dbg[i] = (unsigned long long)clock64();
  };
  __shared__ int s_fail;
  unsigned char *own = s_buf[me];
  const PeerRow *mine = peer_rows(own, e, W, n, me);
  const int words = n * (int)(sizeof(PeerRow) / 8);
  const unsigned long long *src = reinterpret_cast<const unsigned long long *>(mine);
  for (int i = threadIdx.x; i < (W - 1) * words; i += blockDim.x) {
    int j = i / words;
    const int w = i - j * words;
    j += (j >= me) ? 1 : 0;
    reinterpret_cast<unsigned long long *>(peer_rows(s_buf[j], e, W, n, me))[w] = src[w];
  }
  if (threadIdx.x == 0) s_fail = 0;
  // publish: every thread's row stores precede thread 0's system-scope fence (bar.sync orders them),
  // then relaxed flag stores (the grid-barrier release pattern, at system scope)
  __syncthreads();
  stamp(2);
  if (threadIdx.x == 0) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    for (int j = 0; j < W; ++j)
      asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(peer_flag(s_buf[j], e, me)), "l"(e) : "memory");
  }
  stamp(3);
  for (int j = threadIdx.x; j < W; j += blockDim.x) {
    const unsigned long long *f = peer_flag(own, e, j);
    const long long t0 = globaltimer_ns();
    while (ld_acquire_sys(f) != e) {
      __nanosleep(64);
      if (globaltimer_ns() - t0 > timeout_ns) {
        s_fail = 1;
        break;
      }
    }
  }
  __syncthreads();
  stamp(4);
  // reduce, one warp per target: lane j reads rank j's (key, count) (one parallel round trip), MIN
  // (lowest rank on equal keys: only kKeyNone repeats) and SUM by shuffles; then the lanes copy the
  // winning row's result, one 64-bit word each, into the final (mapped host) results
  constexpr int kResW = (int)(sizeof(alp_result) / 8);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  for (int t = warp; t < n; t += nw) {
    unsigned long long k = ~0ull, c = 0ull;
    if (lane < W) {
      const PeerRow *r = peer_rows(own, e, W, n, lane) + t;
      k = ld_relaxed_sys(&r->key);
      c = ld_relaxed_sys(&r->count);
    }
    int jw = lane < W ? lane : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long ok = __shfl_xor_sync(0xffffffffu, k, o);
      const int oj = __shfl_xor_sync(0xffffffffu, jw, o);
      c += __shfl_xor_sync(0xffffffffu, c, o);
      if (ok < k || (ok == k && oj < jw)) {
        k = ok;
        jw = oj;
      }
    }
    const unsigned long long *rw = reinterpret_cast<const unsigned long long *>(&(peer_rows(own, e, W, n, jw) + t)->res);
    unsigned long long *dw = reinterpret_cast<unsigned long long *>(out + t);
    constexpr int kCnt = (int)(offsetof(alp_result, feasible_count) / 8), kFound = (int)(offsetof(alp_result, found) / 8);
    for (int w = lane; w < kResW; w += 32) {
      unsigned long long v = ld_relaxed_sys(rw + w);
      if (w == kCnt) v = c;
      if (w == kFound && s_fail) v = (v & ~0xffffffffull) | 0xffffffffull;  // found = -1: the host reports the timeout
      dw[w] = v;
    }
  }
  __syncthreads();
  stamp(5);
  if (threadIdx.x == 0) *reinterpret_cast<volatile unsigned long long *>(own) = e;
}

// The peer epilogue (not inlined, see peer_exchange): a shared-memory copy of the kernel
// parameters first (through the reference every field access would be a generic load, one
// dependent round trip each in the finalize), then this rank's finalize into its own row, then the
// exchange.
static __device__ __noinline__ void peer_epilogue(const SearchArgs &Pg, const unsigned long long *s_key,
                                                  const unsigned long long *s_cnt, const float *tau_last,
                                                  bool stage) {
  __shared__ __align__(16) unsigned char s_args[sizeof(SearchArgs)];
  __shared__ unsigned char *s_buf[kMaxPeers];
  __shared__ unsigned long long s_e;
  static_assert(sizeof(SearchArgs) % 8 == 0, "SearchArgs copied as 64-bit words");
  const unsigned long long *src = reinterpret_cast<const unsigned long long *>(&Pg);
  for (int i = threadIdx.x; i < (int)(sizeof(SearchArgs) / 8); i += blockDim.x)
    reinterpret_cast<unsigned long long *>(s_args)[i] = src[i];
  __syncthreads();
  const SearchArgs &P = *reinterpret_cast<const SearchArgs *>(s_args);
  const PeerArgs &X = P.fz.peer;
  const int n = P.n_targets, W = X.world, me = X.rank;
  unsigned long long *dbg = P.dbg_ts ? P.dbg_ts + (size_t)gridDim.x * 8 : nullptr;
  if (dbg && threadIdx.x == 0) dbg[0] = (unsigned long long)clock64();
  for (int j = threadIdx.x; j < W; j += blockDim.x) s_buf[j] = X.buf[j];
  if (threadIdx.x == 0) s_e = *reinterpret_cast<volatile unsigned long long *>(X.buf[me]) + 1;  // this epoch
  __syncthreads();
  const unsigned long long e = s_e;
  PeerRow *mine = peer_rows(X.buf[me], e, W, n, me);
  for (int t = 0; t < n; ++t)
    finalize_target(P, t, s_key[t], s_cnt[t], 0, 1, t + 1 == n ? tau_last : nullptr, &mine[t].res, stage);
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    mine[t].key = s_key[t];
    mine[t].count = s_cnt[t];
  }
  __syncthreads();
  if (dbg && threadIdx.x == 0) dbg[1] = (unsigned long long)clock64();
  peer_exchange(s_buf, me, W, n, e, X.out, X.timeout_ns, dbg);
}

// Fused epilogue: the last block to finish writes the reduced (key, count) of every target, resets
// the scratch to its rest state and (fz.finalize) finalizes every target, or (fz.peer.on) runs the
// cross-GPU exchange.  stage: the finalize may stage its re-scan rows at the start of the block's
// dynamic shared memory (the caller's search no longer uses it).
__device__ inline void fused_epilogue(const SearchArgs &P, const float *tau_last, bool stage = false) {
  __shared__ unsigned s_last;
  __shared__ unsigned long long s_key[kInlineTargets], s_cnt[kInlineTargets];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = (atomicAdd(P.fz.ticket, 1u) == gridDim.x - 1) ? 1u : 0u;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int t = threadIdx.x; t < P.n_targets; t += blockDim.x) {
    unsigned long long k = ~atomicExch(P.fz.acc_keys + t, 0ull);  // complemented keys, zero at rest
    const unsigned long long n = atomicExch(P.fz.acc_counts + t, 0ull);
    if (k == ~0ull) k = kKeyNone;
    P.keys[t] = k;
    P.counts[t] = n;
    s_key[t] = k;
    s_cnt[t] = n;
  }
  for (int i = threadIdx.x; i < P.n_targets * P.n_bchunks; i += blockDim.x) P.fz.work[i] = 0ull;
  if (threadIdx.x == 0) atomicExch(P.fz.ticket, 0u);
  // a K3 finalize after this (shard) search combines its blocks in zeroed scratch
  if (!P.fz.finalize && P.fin.best)
    for (int t = threadIdx.x; t < P.n_targets; t += blockDim.x) {
      P.fin.best[t] = 0ull;
      P.fin.done[t] = 0u;
    }
  __syncthreads();
  if (P.fz.peer.on) {
    peer_epilogue(P, s_key, s_cnt, tau_last, stage);
    return;
  }
  if (P.fz.finalize)  // the last target's option terms are still in shared memory (tau_last)
    for (int t = 0; t < P.n_targets; ++t)
      finalize_target(P, t, s_key[t], s_cnt[t], 0, 1, t + 1 == P.n_targets ? tau_last : nullptr, nullptr, stage);
}

// T = rows per lane; MB = minimum resident blocks per SM (register cap 65536 / (256 * MB)).
template <int T, int NB4, bool TAIL2, int MB>
__global__ void __launch_bounds__(kThreads, MB)
    k_search(const __grid_constant__ SearchArgs P) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ unsigned long long red_key[kThreads / 32], red_cnt[kThreads / 32];
  const Smem s = smem_layout(P, smem);
  auto stamp = [&](int i) {
    if (P.dbg_ts && threadIdx.x == 0) {
      unsigned long long g;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
      P.dbg_ts[blockIdx.x * 8 + i] = g;
    }
  };
  stamp(0);
  load_static(P, s);  // static plan tables: independent of K1, in flight during the option terms
  pdl_wait();         // option terms, zeroed work counters and keys come from K1
  for (int t = P.t_begin; t < P.t_end; ++t) {
    float best = finf();
    uint32_t best_seg = 0xffffffffu;
    unsigned long long cnt = 0ull;
    for (int c = P.c_begin; c < P.c_end; ++c) {
      const bool first = (t == P.t_begin && c == P.c_begin);
      if (!first) __syncthreads();  // the previous phase is done with the shared tables
      const int R = qbudget(P, t);
      const float *tau_t = P.tau + (size_t)t * P.M * P.K;
      if (P.fz.on && c == P.c_begin) fused_terms(P, s, t, true);  // kept in shared memory across b-chunks
      if (first) {
        cp_async_wait();
        __syncthreads();  // static tables (and the fused option terms) visible
        stamp(4);
      }
      if (P.fz.on) tau_t = s.opt;
      build_tables(P, s, tau_t, c, R);
      if (t == P.t_begin && c == P.c_begin) stamp(1);
      process_items<T, NB4, TAIL2>(P, s, smem, best, best_seg, cnt, R, t * P.n_bchunks + c);
    }
    if (t + 1 == P.t_end) stamp(2);
    if (t + 1 == P.t_end) pdl_trigger();  // K3 may launch; it waits for this grid to complete
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
      unsigned long long *cd = P.fz.on ? P.fz.acc_counts : P.counts;
      if (k != kKeyNone) {
        if (P.fz.on)
          atomicMax(P.fz.acc_keys + t, ~k);  // fused scratch holds complemented keys (zero at rest)
        else
          atomicMin(P.keys + t, k);
      }
      if (n) atomicAdd(cd + t, n);
    }
  }
  if (P.fz.on) fused_epilogue(P, s.opt);
  stamp(3);
}

// Host-side dispatch over rows per lane (T) and the b-chunk width specialisations.
// Register-cap variants: T = 8 -> 3 (default) or 4 blocks/SM; T = 12 and T = 16 -> 2 (default)
// or 3 (T = 12 under the 3-block cap spills and is 4 % slower on C4)
// (min_blocks 0 = the default).
template <int T, int NB4, bool TAIL2>
static auto pick(const SearchArgs &a) {
  constexpr int kLo = (T == 8) ? 3 : 2, kHi = (T == 8) ? 4 : 3;
  if (a.min_blocks == kHi) return k_search<T, NB4, TAIL2, kHi>;
  return k_search<T, NB4, TAIL2, kLo>;
}

// cudaFuncSetAttribute only when a kernel needs more dynamic smem than already granted (per device)
static cudaError_t ensure_smem(const void *fn, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void *, int>, int> granted;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  int &g = granted[{fn, dev}];
  if (bytes <= g) return cudaSuccess;
  if (g == 0) cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) g = bytes;
  return e;
}

template <int T, int NB4, bool TAIL2>
static cudaError_t launch_one(const SearchArgs &a, int grid, cudaStream_t st) {
  auto fn = pick<T, NB4, TAIL2>(a);
  cudaError_t e = ensure_smem(reinterpret_cast<const void *>(fn), a.smem_bytes);
  if (e != cudaSuccess) return e;
  return launch_pdl(fn, dim3(grid), dim3(kThreads), (size_t)a.smem_bytes, st, a);
}

template <int T, int NB4, bool TAIL2>
static int occ_one(const SearchArgs &a) {
  auto fn = pick<T, NB4, TAIL2>(a);
  if (ensure_smem(reinterpret_cast<const void *>(fn), a.smem_bytes) != cudaSuccess) return 0;
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

}  // namespace alp
