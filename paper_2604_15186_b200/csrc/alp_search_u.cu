// Uniform-register variant of the search (k_uprep + k_search_u), for searches with short b rows
// (C4-like) and up to 8 targets per launch.  The per-target tables — prefix-chunk partial sums,
// a-options, the remaining-budget -> masked-row lookup and the masked rows — live in the constant
// bank, and the search kernel runs one warp per block with item tickets broadcast by redux.sync, so
// for the warp groups whose 32 lane tiles share one unit sum the masked-row index is warp-uniform:
// ptxas loads the b values with LDCU into uniform registers and FADD2 reads them from there
// (tools/microbench/pipes6: 92 vs 80 candidates/clk/SM).  Mixed groups read their lanes' rows from
// shared-memory copies.  Same arithmetic, same keys and counts as k_search.
#include "alp_search.cuh"

#include <cstring>
#include <mutex>
#include <vector>

namespace alp {

__constant__ __align__(16) unsigned char cu_mem[kUBytes];  // tables (layout: SearchArgs u_*)
// the same bank as b pairs (masked rows start at even float offsets inside 16-byte aligned blocks)
#define cu_pairs (reinterpret_cast<const float2 *>(cu_mem))

// typed views of a target's block of the tables (constant bank or its global staging copy)
struct UView {
  const unsigned char *t;
  const SearchArgs &P;
  __device__ __forceinline__ const float4 &a(int i) const { return reinterpret_cast<const float4 *>(t + P.u_off_a)[i]; }
  __device__ __forceinline__ const float2 &pfx(uint32_t c) const {
    return reinterpret_cast<const float2 *>(t + P.u_off_pfx)[c];
  }
  // b chunk c: its lut (remaining budget -> {row offset in floats, #finite entries}) and masked rows
  __device__ __forceinline__ const int2 &lut(int c, int x) const {
    return reinterpret_cast<const int2 *>(t + P.u_off_lut_c[c])[x];
  }
  __device__ __forceinline__ const float *btab(int c) const { return reinterpret_cast<const float *>(t + P.u_off_btab_c[c]); }
};

__device__ __forceinline__ void cp_async8(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}

// ------------------------------------------------------------------ prep: one block
// Option terms of the (single) target into global (finalize inputs) and shared memory, then the
// constant-bank tables written through the symbol's global address (the constant cache is
// refilled at the next kernel launch).
__global__ void k_uprep(const __grid_constant__ SearchArgs P, unsigned char *T) {
  extern __shared__ __align__(16) float s_t[];  // [n_t][M*K] option terms, then the staged plan tables
  const int MK = P.M * P.K, K = P.K, tid = threadIdx.x, nt = blockDim.x, NT = P.n_targets;
  const int R = P.budget, D = P.D, Kb = P.Kb;
  float *s_bs = s_t + NT * MK;                              // [Kb] u-sorted b terms (per target, reused)
  int *s_dv = reinterpret_cast<int *>(s_bs + Kb);           // [D]
  int *s_len = s_dv + D;                                    // [D+1] masked-row lengths (dcnt)
  int *s_bp = s_len + (D + 1);                              // [Kb] bperm
  int *s_u = s_bp + Kb;                                     // [g0*K] prefix units
  int *s_ua = s_u + P.g0 * K;                               // [Ka] a units
  const int NC = P.u_nch, D1 = D + 1;
  int *s_crow = s_ua + P.Ka;                                // [NC][D+1] chunk row of each budget row
  int *s_clen = s_crow + NC * D1;                           // [NC][D+1] length of each chunk row
  int *s_cfin = s_clen + NC * D1;                           // [NC][D+1] finite entries of each chunk row
  int *s_pf = s_cfin + NC * D1;                             // [Kb+1] finite u-sorted b terms before j
  __shared__ int s_rows[kUMaxChunks];                       // rows per chunk
  auto stamp = [&](int slot) {  // ALP_DBG_TS: slots 5-7 of blocks 0-2 (k_search_u uses 0-4, and 6 of blocks > 0)
    if (P.dbg_ts && tid == 0) {
      unsigned long long g;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
      P.dbg_ts[slot] = g;
    }
  };
  stamp(5);
  // the profile tables in shared memory (one wave of cp.async; the lookups' dependent loads then hit
  // shared memory instead of L2/DRAM)
  const DevProfiles &gp = P.fz.prof;
  const int MT = gp.M * gp.nT;
  double *s_pd = reinterpret_cast<double *>((reinterpret_cast<uintptr_t>(s_pf + Kb + 1) + 15) & ~uintptr_t(15));
  DevProfiles sp = gp;
  {
    double *d = s_pd;
    // (8-byte copies: 16-byte cp.async measured slower here, 2.9 vs 2.6 us to the staged tables)
    auto stage_d = [&](const double *src, int n) {
      for (int i = tid; i < n; i += nt) cp_async8(d + i, src + i);
      const double *r = d;
      d += n;
      return r;
    };
    sp.n = stage_d(gp.n, gp.M);
    sp.p = stage_d(gp.p, gp.M);
    sp.tmax = stage_d(gp.tmax, MT);
    sp.rate = stage_d(gp.rate, gp.n_pts);
    sp.lat = stage_d(gp.lat, gp.n_pts);
    const int MTS = MT * gp.nS;
    if (gp.meas_off) {  // measured per-share curves (R2)
      sp.mrate = stage_d(gp.mrate, gp.n_mpts);
      sp.mlat = stage_d(gp.mlat, gp.n_mpts);
      sp.mtmax = stage_d(gp.mtmax, MTS);
    }
    int *w = reinterpret_cast<int *>(d);
    auto stage_i = [&](const int *src, int n) {
      for (int i = tid; i < n; i += nt) cp_async4(w + i, src + i);
      const int *r = w;
      w += n;
      return r;
    };
    sp.S = stage_i(gp.S, gp.nS);
    sp.T = stage_i(gp.T, gp.nT);
    sp.R = stage_i(gp.R, gp.nR);
    sp.prof_off = stage_i(gp.prof_off, MT + 1);
    if (gp.min_units) sp.min_units = stage_i(gp.min_units, MT);
    if (gp.meas_off) sp.meas_off = stage_i(gp.meas_off, MTS + 1);
  }
  // static plan tables (cp.async: in flight with the profile tables)
  for (int i = tid; i < D; i += nt) cp_async4(s_dv + i, P.dv + i);
  for (int i = tid; i <= D; i += nt) cp_async4(s_len + i, P.dcnt + i);
  for (int i = tid; i < Kb; i += nt) cp_async4(s_bp + i, P.bperm + i);
  for (int i = tid; i < P.g0 * K; i += nt) cp_async4(s_u + i, P.u + i);
  if (P.a_llm >= 0)
    for (int i = tid; i < P.Ka; i += nt) cp_async4(s_ua + i, P.u + P.a_llm * K + i);
  // group unit sums, clamped at R + 1 (an over-budget sum only has to keep r negative): the first
  // 4 per thread loaded now, in flight with the staging wave, and stored after the option terms (a
  // load -> store loop here put its DRAM round trips in front of the wait)
  int gv[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t g = tid + (uint32_t)(j * nt);
    gv[j] = g < P.n_groups ? __ldg(P.gsum + g) : 0;
  }
  cp_async_wait();
  __syncthreads();
  stamp(15);
  for (int i = tid; i < NT * MK; i += nt) {
    const int t = i / MK, j = i % MK;
    float tau;
    double term, b;
    int u;
    option_terms(sp, P.fz.tgt[t], j / K, j % K, &tau, &term, &b, &u);
    s_t[i] = tau;
    P.fz.o_tau[i] = tau;
    P.fz.o_term[i] = term;
    P.fz.o_b[i] = b;
  }
  stamp(6);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t g = tid + (uint32_t)(j * nt);
    if (g < P.n_groups) reinterpret_cast<int *>(T)[g] = min(gv[j], R + 1);
  }
  for (uint32_t g = tid + 4u * nt; g < P.n_groups; g += nt) reinterpret_cast<int *>(T)[g] = min(P.gsum[g], R + 1);
  for (int i = tid; i <= D; i += nt) s_len[i] = min(s_len[i], Kb);
  __syncthreads();
  stamp(7);
  for (int t = 0; t < NT; ++t) {
    const float *st = s_t + t * MK;
    unsigned char *tb = T + P.u_tbase + t * P.u_tstride;
    float2 *pfx = reinterpret_cast<float2 *>(tb + P.u_off_pfx);
    float4 *ta4 = reinterpret_cast<float4 *>(tb + P.u_off_a);
    // prefix chunks: canonical sum over LLMs 0..g0-1 (units clamped at R + 1)
    for (uint32_t c = tid; c < P.n_chunks; c += nt) {
      float pa = 0.f;
      int U = 0;
      for (int m = 0; m < P.g0; ++m) {
        const uint32_t d = (c / P.pw[m]) % (uint32_t)K;
        pa = __fadd_rn(pa, st[m * K + d]);
        U += s_u[m * K + d];
      }
      pfx[c] = make_float2(pa, __int_as_float(min(U, R + 1)));
    }
    // a options {tau_a, units (clamped), feasible, #feasible options before a}; entry Ka holds the
    // total in .w (k_search_u's full-row items count Ka ranges by two loads).  One warp, ballots.
    if (tid < 32) {
      int run = 0;
      for (int b0 = 0; b0 <= P.Ka; b0 += 32) {
        const int a = b0 + tid;
        float ta = 0.f;
        int ua = 0, feas = 0;
        if (a < P.Ka) {
          ta = P.a_llm >= 0 ? st[P.a_llm * K + a] : 0.f;
          ua = P.a_llm >= 0 ? min(s_ua[a], R + 1) : 0;
          feas = ta < __int_as_float(0x7f800000) ? 1 : 0;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, feas);
        const int pre = run + __popc(bal & ((1u << tid) - 1u));
        if (a <= P.Ka) ta4[a] = make_float4(ta, __int_as_float(feas ? ua : 0), __int_as_float(feas), __int_as_float(pre));
        run += __popc(bal);
      }
    }
    // u-sorted b terms
    for (int j = tid; j < Kb; j += nt) s_bs[j] = st[P.b_llm * K + s_bp[j]];
    __syncthreads();
    if (t == 0) stamp(21);
    // per b chunk: budget row i (the u-sorted columns with u <= dv[i-1]; row 0 none) restricted to
    // the chunk's columns; equal restrictions share one chunk row (the length is non-decreasing in
    // i).  All chunks at once: one thread per chunk de-duplicates, then every (chunk, row) pair,
    // row element and lut entry in parallel (three barriers in all, not three per chunk).
    // warp 0: s_pf[j] = finite terms among the first j u-sorted b columns (ballot scan), so a chunk
    // row's finite count is a difference of two entries; the other warps de-duplicate the rows
    if (tid < 32) {
      int run = 0;
      for (int j0 = 0; j0 <= Kb; j0 += 32) {
        const int j = j0 + tid;
        const int fin = j < Kb && s_bs[j] < __int_as_float(0x7f800000) ? 1 : 0;
        const unsigned bal = __ballot_sync(0xffffffffu, fin);
        if (j <= Kb) s_pf[j] = run + __popc(bal & ((1u << tid) - 1u));
        run += __popc(bal);
      }
    }
    for (int c = tid - 32; c >= 0 && c < NC; c += nt - 32) {
      const int c0 = c * P.bchunk_w, wc = min(P.bchunk_w, Kb - c0);
      int rows = 0, prev = -1;
      for (int i = 0; i <= D; ++i) {
        const int len = min(max(s_len[i] - c0, 0), wc);
        if (len > prev) {
          s_clen[c * D1 + rows] = len;
          ++rows;
        }
        s_crow[c * D1 + i] = rows - 1;
        prev = len;
      }
      s_rows[c] = rows;
    }
    __syncthreads();
    for (int c = 0; c < NC; ++c) {
      const int c0 = c * P.bchunk_w, rows = s_rows[c];
      float *btab = reinterpret_cast<float *>(tb + P.u_off_btab_c[c]);
      for (int i = tid; i < rows * P.u_cstride; i += nt) {
        const int row = i / P.u_cstride, j = i % P.u_cstride;
        btab[i] = (j < s_clen[c * D1 + row]) ? s_bs[c0 + j] : __int_as_float(0x7f800000);
      }
    }
    // lut: index x <-> remaining budget r = R - lut_base + x; budget row = #{distinct b unit values
    // <= r}, mapped to the chunk row
    for (int i = tid; i < NC * P.lut_n; i += nt) {
      const int c = i / P.lut_n, x = i % P.lut_n;
      const int r = R - P.lut_base + x;
      int lo = 0, hi = D;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (s_dv[mid] <= r) lo = mid + 1; else hi = mid;
      }
      const int row = s_crow[c * D1 + lo], c0 = c * P.bchunk_w;
      reinterpret_cast<int2 *>(tb + P.u_off_lut_c[c])[x] =
          make_int2(row * P.u_cstride, s_pf[c0 + s_clen[c * D1 + row]] - s_pf[c0]);
    }
    if (t == 0) stamp(23);
    __syncthreads();  // s_bs and the chunk tables are reused by the next target
  }
  stamp(8 + 5);
}

// "candidate = Q_a,i + tau_b; acc_i = min(acc_i, candidate)" over a uniform masked row: per b PAIR
// one LDCU.64 into a uniform register pair, then per row one FADD2 Q_a,i.F32 + {b_j, b_j+1} (the
// scalar vector operand broadcast by .F32; the b pair read from the uniform register file) and one
// FMNMX3 acc_i = min(acc_i, x, y): 1 issue slot per candidate and half the LDCU of the row-pair form
// (tools/microbench/pipes7: 96 vs 93 candidates/clk/SM at 18 b per row, 103 vs 98 at 64).
#ifndef ALP_FAST_ROWS
#define ALP_FAST_ROWS 1  // full-row items: b pairs held in uniform registers for the whole item
#endif
#ifndef ALP_FAST_UA
#define ALP_FAST_UA 1  // unroll of the full-row a loop
#endif
#ifndef ALP_U_ROWS
#define ALP_U_ROWS 12  // rows per lane of the uniform-register kernel (the plan's lane tiles)
#endif
// The same over b pairs already in uniform registers (a full-row item: one row for every a option).
template <int NP>
__device__ __forceinline__ void eval_pairs_u(const float2 (&bv)[NP], const float (&Qa)[ALP_U_ROWS], float (&acc)[ALP_U_ROWS]) {
#pragma unroll
  for (int j = 0; j < NP; ++j) {
#pragma unroll
    for (int i = 0; i < ALP_U_ROWS; ++i) {
      float x, y;
      add2(x, y, Qa[i], bv[j].x, bv[j].y);
      acc[i] = min3(acc[i], x, y);
    }
  }
}

template <int NB4, bool TAIL2>
__device__ __forceinline__ void eval_row_u(const float2 *rb, const float (&Qa)[ALP_U_ROWS], float (&acc)[ALP_U_ROWS]) {
#pragma unroll
  for (int j = 0; j < 2 * NB4 + (TAIL2 ? 1 : 0); ++j) {
    const float2 b = rb[j];
#pragma unroll
    for (int i = 0; i < ALP_U_ROWS; ++i) {
      float x, y;
      add2(x, y, Qa[i], b.x, b.y);
      acc[i] = min3(acc[i], x, y);
    }
  }
}

// The search's epilogue (fused_epilogue: last-block detection, finalize or peer exchange) out of
// line: inlined, the finalize's live values set the kernel's register count (84 -> 20 one-warp
// blocks per SM); out of line the search loops need 76 (24 blocks per SM): C4 kernel 0.425 ->
// 0.420 ms.  (A speculative finalize of the running minimum by the first block to finish was
// measured here too and not kept: on a busy SM it ran longer than the loop's tail, +1.7 us.)
static __device__ __noinline__ void epilogue_u(const SearchArgs &P) { fused_epilogue(P, nullptr, P.fin.stage != 0); }

// ALP_CHECK_BOUNDS builds (tests only: compute-sanitizer is unavailable on the GPU pool): every
// table index of the search loops asserted in range; an out-of-range index traps the kernel.
#ifdef ALP_CHECK_BOUNDS
#define ALP_BOUND(cond) do { if (!(cond)) __trap(); } while (0)
#else
#define ALP_BOUND(cond) do { } while (0)
#endif

// ------------------------------------------------------------------ search: one warp per block
template <int NB4, bool TAIL2>
__global__ void __launch_bounds__(32) k_search_u(const __grid_constant__ SearchArgs P, const unsigned char *ug) {
  constexpr int T = ALP_U_ROWS;
  extern __shared__ __align__(16) unsigned char smem[];
  // per target [g1*K + 2] terms of LLMs 0..g1-1 then {0, +inf}, all targets copied up front: any
  // lane-divergent code inside the target loop makes ptxas give up the uniform datapath there
  const int tw = P.g1 * P.K + 2;
  float *s_tau = reinterpret_cast<float *>(smem);
  const int lane = threadIdx.x;
  const uint32_t n = (uint32_t)(P.item_hi - P.item_lo);
  const int *gsum = reinterpret_cast<const int *>(cu_mem);
  auto stamp = [&](int i) {  // ALP_DBG_TS per-block timeline (outside the target loop only)
    if (P.dbg_ts && lane == 0) {
      unsigned long long g;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
      P.dbg_ts[blockIdx.x * 8 + i] = g;
    }
  };
  stamp(0);
  pdl_wait();
  // every block reads the same few lines at launch: L1-allocating loads (ld.global.ca) so one miss
  // per SM goes to L2 — L2-only loads from all 3552 warps cost ~7.5 us per block (ALP_DBG_TS).
  // (__ldg or cp.async here change the search loop's register allocation: 2 % slower, measured)
  for (int i = lane; i < P.n_targets * tw; i += 32) {
    const int t = i / tw, j = i % tw;
    s_tau[i] = j < tw - 2 ? __ldca(P.tau + (size_t)t * P.M * P.K + j) : (j == tw - 2 ? 0.f : __int_as_float(0x7f800000));
  }
  // single target: shared-memory copies of the lut and masked rows for the mixed groups
  int2 *s_lut = reinterpret_cast<int2 *>(smem + P.off_lut);
  float *s_btab = reinterpret_cast<float *>(smem + P.off_btab);
  const bool smem_rows = P.u_smem_rows;  // single target, single b chunk (its rows: D + 1)
  if (smem_rows) {
    const UView gv0{ug + P.u_tbase, P};
    const int *lut_w = reinterpret_cast<const int *>(&gv0.lut(0, 0));
    int *s_lut_w = reinterpret_cast<int *>(s_lut);
    for (int i = lane; i < 2 * P.lut_n; i += 32) s_lut_w[i] = __ldca(lut_w + i);
    for (int i = lane; i < (P.D + 1) * P.u_cstride; i += 32) s_btab[i] = __ldca(gv0.btab(0) + i);
  }
  const int R1 = P.budget + 1;  // unit sums enter the lut index clamped at R + 1
  cp_async_wait();
  __syncwarp();
  stamp(4);
  stamp(1);
  for (int t = 0; t < P.n_targets; ++t) {  // target phases: the warp moves on when the tickets run out
    const UView cv{cu_mem + P.u_tbase + t * P.u_tstride, P};
    const UView gv{ug + P.u_tbase + t * P.u_tstride, P};
    const unsigned char *tau_b = smem + (size_t)t * tw * 4;
    float best = __int_as_float(0x7f800000);
    uint32_t best_seg = 0xffffffffu;
    unsigned long long cnt = 0ull;
    float Qr[T], acc[T];
    for (int c = 0; c < P.u_nch; ++c) {  // b-chunk phases of the target (C4: one)
    // dynamic item tickets: lane 0 takes the next ticket while the current item is evaluated;
    // redux.sync broadcasts it into a uniform register (ptxas keeps the derived indices uniform)
    unsigned long long *ctr = P.work + t * P.u_nch + c;
    // the chunk's masked rows as b pairs: float2 indexing from the 16-byte aligned bank base makes
    // every address provably 8-byte aligned, so ptxas loads each pair with ONE LDCU.64 (a float* +
    // offset form is split into two scalar LDCU)
    const float2 *rows_u = cu_pairs + ((P.u_tbase + t * P.u_tstride + P.u_off_btab_c[c]) >> 3);
    unsigned tnext = 0xffffffffu;
    if (lane == 0) tnext = (unsigned)atomicAdd(ctr, 1ull);
    // tickets [0, nbulk) are whole items; the rank's last items are handed out as u_S sub-items of
    // u_As a options each (single-option segments), so the warps finish within a sub-item's time
    const uint32_t nbulk = min(P.u_nbulk, n);
    const uint32_t ntk = nbulk + (n - nbulk) * P.u_S;
    for (;;) {
      const uint32_t k = __reduce_min_sync(0xffffffffu, tnext);
      if (k >= ntk) break;
      if (P.dbg_ts && lane == 0 && blockIdx.x > 0) P.dbg_ts[blockIdx.x * 8 + 6] += 1;  // tickets taken (diagnostics)
      uint32_t kk = k, part = 0;
      if (k >= nbulk) {
        const uint32_t j = k - nbulk, ji = fdiv(j, P.fd_S);
        part = j - ji * P.u_S;
        kk = nbulk + ji;
      }
      const uint32_t it = (uint32_t)P.item_lo + kk;
      const uint32_t tq = fdiv(it, P.fd_nQ);
      const uint32_t q = it - tq * P.nQ;           // a-range of the row
      const uint32_t chunk = fdiv(tq, P.fd_ng);
      const uint32_t grp = tq - chunk * P.n_groups;
      const int q0 = (int)(q * P.A), q1 = min(q0 + (int)P.A, P.Ka);
      const int a0 = k >= nbulk ? min(q0 + (int)(part * P.u_As), q1) : q0;
      const int a1 = k >= nbulk ? min(a0 + (int)P.u_As, q1) : q1;
      const uint32_t qs = k >= nbulk ? (uint32_t)a0 : q * P.seg_mul;  // segment slot of a0
      const float2 pf = cv.pfx(chunk);
      const int upfx = __float_as_int(pf.y);       // clamped at R + 1
      const uint32_t tile = grp * kWarpTiles + lane;
      const unsigned nfin = load_tile<T>(P, tau_b, pf.x, tile, Qr, acc);
      unsigned c32 = 0;
      const int gs = gsum[grp];                     // clamped at R + 1
      // warp-uniform remaining budget (one unit sum, or a mixed group whose every lane is over budget,
      // where every row is the all-+inf row 0): uniform-register b operands
      const bool uni = grp < P.n_groups_u || gs + upfx >= R1;
      const int xg = P.lut_base - upfx - gs;
      // a-loop unrolled by 2 for short rows; long rows (64-column chunks: an ~800-instruction body)
      // stay rolled so the uniform and mixed loops together fit the 32 KB instruction cache
      constexpr int kUA = NB4 > 8 ? 1 : 2;
      // Full-row items (short rows): when even the a option with the most units leaves the widest
      // row (the lut is monotone), every a option of the item reads that one row — its b pairs are
      // loaded into uniform registers once per item, the count is fin x #feasible a options (two
      // prefix-count loads), and the a loop is tau_a + the row's FADD2/FMNMX3 only (C4: ~96 % of
      // the (prefix, a) pairs, 81 % of the items; 1.05 instead of 1.14 instructions per candidate).
      // The other uniform items then take the mixed-group loop (its per-a row test finds one row
      // for all lanes) instead of a loop of their own: hot code that fits the instruction cache.
      constexpr int kNP = 2 * NB4 + (TAIL2 ? 1 : 0);
      constexpr bool kFastRows = ALP_FAST_ROWS && kNP >= 1 && kNP <= 10;
      constexpr int kFUA = ALP_FAST_UA;
      // a mixed group's lanes: their own remaining budgets (uniform groups: the group's)
      const int xl = uni ? xg : P.lut_base - upfx - min(__ldg(P.tile_s + tile), R1);
      const int xq = uni ? xg : __reduce_min_sync(0xffffffffu, xl);  // the smallest of them
      if (kFastRows && cv.lut(c, xq - P.u_amax).x == cv.lut(c, P.lut_n - 1).x) {
        const int2 lf = cv.lut(c, xq - P.u_amax);
        ALP_BOUND(xq - P.u_amax >= 0 && xq - P.u_amax < P.lut_n && a0 >= 0 && a0 <= a1 && a1 <= P.Ka &&
                  P.u_off_btab_c[c] + 4 * (lf.x + 2 * kNP) <= (c + 1 < P.u_nch ? P.u_off_lut_c[c + 1] : P.u_tstride) &&
                  __float_as_int(cv.a(a1).w) - __float_as_int(cv.a(a0).w) >= 0);
        const float2 *rb = rows_u + (lf.x >> 1);
        float2 bv[kNP > 0 ? kNP : 1];
#pragma unroll
        for (int j = 0; j < kNP; ++j) bv[j] = rb[j];
        c32 = (unsigned)lf.y * (unsigned)(__float_as_int(cv.a(a1).w) - __float_as_int(cv.a(a0).w));
#pragma unroll(kFUA)
        for (int a = a0; a < a1; ++a) {
          const float ta = cv.a(a).x;
          float Qa[T];
#pragma unroll
          for (int i = 0; i < T; i += 2) add2b(Qa[i], Qa[i + 1], Qr[i], Qr[i + 1], ta);
          eval_pairs_u<(kNP > 0 ? kNP : 1)>(bv, Qa, acc);
        }
      } else if (!kFastRows && uni) {
#pragma unroll(kUA)
        for (int a = a0; a < a1; ++a) {
          const float4 av = cv.a(a);
          const int2 lu = cv.lut(c, xg - __float_as_int(av.y));
          c32 += (unsigned)(lu.y * __float_as_int(av.z));
          float Qa[T];
#pragma unroll
          for (int i = 0; i < T; i += 2) add2b(Qa[i], Qa[i + 1], Qr[i], Qr[i + 1], av.x);
          eval_row_u<NB4, TAIL2>(rows_u + (lu.x >> 1), Qa, acc);
        }
      } else {
        // mixed group: the lanes' own remaining budgets, rows from the global staging copy of the
        // tables (L1-resident; a different memory space keeps the compiler from merging this loop
        // with the uniform one into a single vector loop)
        if (smem_rows) {
          const uint32_t bbase = (uint32_t)__cvta_generic_to_shared(s_btab);
          // not unrolled: the smaller mixed-group code leaves the instruction cache to the uniform
          // loop (C4 0.4763 vs 0.4784 ms with unroll 2)
          // the lanes' lut indices span [xlo, xhi] (uniform, by redux); the lut is monotone in its
          // index, so where lut(xlo - u_a) and lut(xhi - u_a) name the same masked row every lane
          // uses that row: evaluated with uniform-register b operands like a uniform group
          const int xlo = xq, xhi = uni ? xg : __reduce_max_sync(0xffffffffu, xl);
#pragma unroll 1
          for (int a = a0; a < a1; ++a) {
            const float4 av = cv.a(a);
            ALP_BOUND(xlo - __float_as_int(av.y) >= 0 && xhi - __float_as_int(av.y) < P.lut_n &&
                      xl - __float_as_int(av.y) >= 0 && xl - __float_as_int(av.y) < P.lut_n);
            const int2 l0 = cv.lut(c, xlo - __float_as_int(av.y));
            const int2 l1 = cv.lut(c, xhi - __float_as_int(av.y));
            float Qa[T];
#pragma unroll
            for (int i = 0; i < T; i += 2) add2b(Qa[i], Qa[i + 1], Qr[i], Qr[i + 1], av.x);
            if (l0.x == l1.x) {
              c32 += (unsigned)(l0.y * __float_as_int(av.z));
              eval_row_u<NB4, TAIL2>(rows_u + (l0.x >> 1), Qa, acc);
            } else {
              const int2 lu = s_lut[xl - __float_as_int(av.y)];
              c32 += (unsigned)(lu.y * __float_as_int(av.z));
              eval_row<T, NB4, TAIL2>(bbase + 4u * (uint32_t)lu.x, Qa, acc, 0);
            }
          }
        } else
#pragma unroll 1
        for (int a = a0; a < a1; ++a) {
          const float4 av = cv.a(a);
          const int2 lu = __ldg(&gv.lut(c, xl - __float_as_int(av.y)));
          c32 += (unsigned)(lu.y * __float_as_int(av.z));
          float Qa[T];
#pragma unroll
          for (int i = 0; i < T; i += 2) add2b(Qa[i], Qa[i + 1], Qr[i], Qr[i + 1], av.x);
          const float *rb = gv.btab(c) + lu.x;
#pragma unroll
          for (int g = 0; g < NB4; ++g) eval4<T>(__ldg(reinterpret_cast<const float4 *>(rb) + g), Qa, acc);
          if constexpr (TAIL2) eval2<T>(__ldg(reinterpret_cast<const float2 *>(rb + 4 * NB4)), Qa, acc);
        }
      }
      // the next ticket only now, not prefetched at the item's start: the warp scheduler favours the
      // oldest warps, and a starved warp holding a prefetched ticket delays that item to the end of
      // the kernel (C4: 0.4709 -> 0.4669 ms; 8-rank shard 0.0819 -> 0.0778 ms, tools/shard_timing.py)
      if (lane == 0) tnext = (unsigned)atomicAdd(ctr, 1ull);
      cnt += (unsigned long long)c32 * nfin;
      fold_rows<T>(P, acc, tile, chunk, qs, best, best_seg);  // segment: from a option a0 to the row's end
    }
    }
    unsigned long long key = (best < __int_as_float(0x7f800000))
                                 ? ((unsigned long long)__float_as_uint(best) << 32) | best_seg : kKeyNone;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long ok = __shfl_xor_sync(0xffffffffu, key, o);
      const unsigned long long oc = __shfl_xor_sync(0xffffffffu, cnt, o);
      key = ok < key ? ok : key;
      cnt += oc;
    }
    if (lane == 0) {
      if (key != kKeyNone) atomicMax(P.fz.acc_keys + t, ~key);  // complemented: zero at rest
      if (cnt) atomicAdd(P.fz.acc_counts + t, cnt);
    }
  }
  stamp(2);
  pdl_trigger();
  // the search's shared memory is free now: the finalize stages its inputs in it
  // (rows of 12-34 options: out of line — the finalize's registers cost C4 4 one-warp blocks per
  // SM; long rows (C3) measured 5 % slower out of line, and the 2-option variant spills around the
  // call: both keep it inline)
  if constexpr (NB4 >= 3 && NB4 <= 8) epilogue_u(P);
  else fused_epilogue(P, nullptr, P.fin.stage);
  stamp(3);
}

// ------------------------------------------------------------------ launch
// Per-device staging copy of the tables (k_uprep writes it; one D2D copy moves it into the
// constant bank; the mixed groups' shared-memory copies read it) and the ordering event that keeps
// concurrent searches on other streams from overwriting the constant bank in use.
// The prep → constant-bank copy → search sequence is replayed as one CUDA graph (instantiated once
// per launch shape, kernel arguments updated in place when they change): one host submission
// instead of four, so the device runs the three nodes back to back instead of waiting for the
// host's launch calls (measured: tools/step_timeline.py; C4 step 0.505 -> 0.498 ms, 0.1-0.2 us
// between the nodes).
struct UGraph {
  const void *fn = nullptr;  // search kernel instantiation
  int grid = 0, threads = 0;
  size_t prep_smem = 0, used = 0;
  bool ev = false;  // has the kernel-time event record node
  cudaGraph_t g = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaGraphNode_t n_prep = nullptr, n_search = nullptr, n_ev = nullptr;
  cudaEvent_t ev_set = nullptr;  // event the record node currently targets
  SearchArgs last;               // arguments the kernel nodes currently hold
};
struct UState {
  unsigned char *staging = nullptr;
  cudaEvent_t done = nullptr;
  cudaStream_t cap = nullptr, cap2 = nullptr;  // capture streams (cap2: the event branch)
  cudaEvent_t fork = nullptr, join = nullptr;
  std::vector<UGraph> graphs;
  bool claimed = false;  // a peer search took the bank (search_u_claim) and has not launched yet
};
static std::mutex g_u_mu;
static UState &ustate() {
  static UState s[kMaxDevices];
  int dev = 0;
  cudaGetDevice(&dev);
  UState &u = s[dev & (kMaxDevices - 1)];
  if (!u.staging) {
    cudaMalloc(reinterpret_cast<void **>(&u.staging), kUBytes);
    cudaEventCreateWithFlags(&u.done, cudaEventDisableTiming);
  }
  return u;
}

template <int NB4, bool TAIL2>
static const void *fn_u() {
  return reinterpret_cast<const void *>(k_search_u<NB4, TAIL2>);
}

template <int NB4, bool TAIL2>
static cudaError_t launch_u(const SearchArgs &a, int grid, cudaStream_t st) {
  const int smem = a.smem_bytes;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(32);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = st;
  const unsigned char *ug = ustate().staging;
  return cudaLaunchKernelEx(&cfg, k_search_u<NB4, TAIL2>, a, ug);
}

template <int NB4, bool TAIL2>
static int occ_u(const SearchArgs &a) {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_search_u<NB4, TAIL2>, 32, a.smem_bytes) != cudaSuccess)
    return 0;
  return n;
}


// b-chunk widths of the uniform-register path: the short-row specialisations (<= 34) and kUChunkW
#define ALP_DISPATCH_U(CALL)                                 \
  do {                                                       \
    static_assert(kUChunkW == 64, "chunk width dispatch");   \
    if (a.bchunk_wpad == 64) return CALL(12, 16, false);     \
    ALP_DISPATCH_W(CALL, 12);                                \
  } while (0)

static cudaError_t launch_u_search(const SearchArgs &a, int grid, cudaStream_t st) {
#define CALL(T_, N, T2) launch_u<N, T2>(a, grid, st)
  ALP_DISPATCH_U(CALL);
#undef CALL
}

static const void *search_u_fn(const SearchArgs &a) {
#define CALL(T_, N, T2) fn_u<N, T2>()
  ALP_DISPATCH_U(CALL);
#undef CALL
}

// Kernel-node arguments of the cached graph, rewritten only when they differ from the last launch.
static cudaError_t set_node_args(UGraph &gr, const SearchArgs &a, unsigned char *staging, cudaEvent_t ev) {
  cudaError_t e;
  if (std::memcmp(&gr.last, &a, sizeof(SearchArgs)) != 0) {
    for (cudaGraphNode_t n : {gr.n_prep, gr.n_search}) {
      cudaKernelNodeParams kp;
      if ((e = cudaGraphKernelNodeGetParams(n, &kp)) != cudaSuccess) return e;
      void *args[2] = {const_cast<SearchArgs *>(&a), &staging};
      kp.kernelParams = args;
      kp.extra = nullptr;
      if (n == gr.n_search) kp.sharedMemBytes = (unsigned)a.smem_bytes;  // the search's layout may differ
      if ((e = cudaGraphExecKernelNodeSetParams(gr.exec, n, &kp)) != cudaSuccess) return e;
    }
    std::memcpy(&gr.last, &a, sizeof(SearchArgs));
  }
  if (gr.ev && ev != gr.ev_set) {
    if ((e = cudaGraphExecEventRecordNodeSetEvent(gr.exec, gr.n_ev, ev)) != cudaSuccess) return e;
    gr.ev_set = ev;
  }
  return cudaSuccess;
}

// Capture prep → copy → [event] → search once on the capture stream and instantiate it.
static cudaError_t build_graph(UGraph &gr, UState &u, const SearchArgs &a, int grid, cudaEvent_t ev) {
  cudaError_t e;
  if (!u.cap && (e = cudaStreamCreateWithFlags(&u.cap, cudaStreamNonBlocking)) != cudaSuccess) return e;
  if (!u.cap2 && (e = cudaStreamCreateWithFlags(&u.cap2, cudaStreamNonBlocking)) != cudaSuccess) return e;
  if (!u.fork && (e = cudaEventCreateWithFlags(&u.fork, cudaEventDisableTiming)) != cudaSuccess) return e;
  if (!u.join && (e = cudaEventCreateWithFlags(&u.join, cudaEventDisableTiming)) != cudaSuccess) return e;
  if ((e = cudaStreamBeginCapture(u.cap, cudaStreamCaptureModeThreadLocal)) != cudaSuccess) return e;
  k_uprep<<<1, gr.threads, gr.prep_smem, u.cap>>>(a, u.staging);
  cudaError_t ec = cudaGetLastError();
  // The kernel-time event hangs off a side branch that starts with the table copy, so the search
  // never waits for it: in series (copy -> event -> search) the event node alone left a ~5 us
  // bubble before the search. Recorded when the prep is done, it brackets the copy (1.4 us) and
  // the search: an upper bound of the search kernel's time, never an underestimate.
  if (ev) {
    if (ec == cudaSuccess) ec = cudaEventRecord(u.fork, u.cap);
    if (ec == cudaSuccess) ec = cudaStreamWaitEvent(u.cap2, u.fork, 0);
    if (ec == cudaSuccess) ec = cudaEventRecordWithFlags(ev, u.cap2, cudaEventRecordExternal);
    if (ec == cudaSuccess) ec = cudaEventRecord(u.join, u.cap2);
  }
  if (ec == cudaSuccess) ec = cudaMemcpyToSymbolAsync(cu_mem, u.staging, gr.used, 0, cudaMemcpyDeviceToDevice, u.cap);
  if (ec == cudaSuccess) ec = launch_u_search(a, grid, u.cap);
  if (ec == cudaSuccess && ev) ec = cudaStreamWaitEvent(u.cap, u.join, 0);
  cudaGraph_t g = nullptr;
  e = cudaStreamEndCapture(u.cap, &g);
  if (ec != cudaSuccess) {
    if (g) cudaGraphDestroy(g);
    return ec;
  }
  if (e != cudaSuccess) return e;
  size_t nn = 0;
  if ((e = cudaGraphGetNodes(g, nullptr, &nn)) != cudaSuccess) return e;
  std::vector<cudaGraphNode_t> nodes(nn);
  if ((e = cudaGraphGetNodes(g, nodes.data(), &nn)) != cudaSuccess) return e;
  for (cudaGraphNode_t n : nodes) {
    cudaGraphNodeType t;
    if ((e = cudaGraphNodeGetType(n, &t)) != cudaSuccess) return e;
    if (t == cudaGraphNodeTypeKernel) {
      cudaKernelNodeParams kp;
      if ((e = cudaGraphKernelNodeGetParams(n, &kp)) != cudaSuccess) return e;
      (kp.func == reinterpret_cast<void *>(k_uprep) ? gr.n_prep : gr.n_search) = n;
    } else if (t == cudaGraphNodeTypeEventRecord) {
      gr.n_ev = n;
    }
  }
  if (!gr.n_prep || !gr.n_search || (ev && !gr.n_ev)) {
    cudaGraphDestroy(g);
    return cudaErrorInvalidValue;
  }
  if ((e = cudaGraphInstantiate(&gr.exec, g, 0)) != cudaSuccess) {
    cudaGraphDestroy(g);
    return e;
  }
  gr.g = g;
  gr.ev_set = ev;
  std::memcpy(&gr.last, &a, sizeof(SearchArgs));
  return cudaSuccess;
}

size_t uprep_smem_bytes(const SearchArgs &a) {
  const DevProfiles &pr = a.fz.prof;
  const int MT = pr.M * pr.nT;
  return (size_t)(a.n_targets * a.M * a.K + a.Kb) * 4 + (size_t)(2 * a.D + 1 + 3 * a.u_nch * (a.D + 1) + a.Kb + a.g0 * a.K + a.Ka) * 4 +
         (size_t)(a.Kb + 1) * 4 + 16 + 16 * 16 +  // s_pf, 16-byte alignment, per-array padding of the staging

         (size_t)(2 * pr.M + MT + 2 * pr.n_pts) * 8 +
         (size_t)(pr.nS + pr.nT + pr.nR + MT + 1 + (pr.min_units ? MT : 0)) * 4 +
         (pr.meas_off ? (size_t)(2 * pr.n_mpts + MT * pr.nS) * 8 + (size_t)(MT * pr.nS + 1) * 4 : 0);
}

cudaError_t launch_search_u(const SearchArgs &a, int grid, cudaStream_t st, cudaEvent_t before_search) {
  std::lock_guard<std::mutex> lock(g_u_mu);
  UState &u = ustate();
  if (!u.staging) return cudaErrorMemoryAllocation;
  const int MK = a.M * a.K, NTM = a.n_targets * MK;
  // (more threads measured slower at C4: 1024 threads 7.8 vs 6.9 us, tools/uprep_ab.sh)
  int threads = NTM >= 512 ? 1024 : (NTM >= 256 ? 512 : 256);
  static const int thr_env = getenv("ALP_UPREP_THREADS") ? atoi(getenv("ALP_UPREP_THREADS")) : 0;  // tuning knob
  if (thr_env >= 64 && thr_env <= 1024) threads = thr_env & ~31;
  cudaError_t e = cudaStreamWaitEvent(st, u.done, 0);  // the previous search using the constant bank
  if (e != cudaSuccess) return e;
  const size_t prep_smem = uprep_smem_bytes(a);
  if (prep_smem > 48 * 1024) {  // function attributes are per device: one grant per device
    int dev = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    static std::once_flag f[kMaxDevices];
    std::call_once(f[dev & (kMaxDevices - 1)],
                   [] { cudaFuncSetAttribute(k_uprep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kUPrepSmemMax); });
  }
  const size_t used = (size_t)a.u_tbase + (size_t)a.n_targets * a.u_tstride;
  static const bool no_graph = getenv("ALP_U_NOGRAPH") != nullptr;  // per-call launches (comparison)
  if (!no_graph) {
    const void *fn = search_u_fn(a);
    const bool ev = before_search != nullptr;
    UGraph *gr = nullptr;
    for (UGraph &x : u.graphs)
      if (x.fn == fn && x.grid == grid && x.threads == threads && x.prep_smem == prep_smem && x.used == used &&
          x.ev == ev)
        gr = &x;
    if (!gr) {
      if (u.graphs.size() >= 16) {  // many launch shapes (tests, shard sweeps): start over
        for (UGraph &x : u.graphs) {
          cudaGraphExecDestroy(x.exec);
          cudaGraphDestroy(x.g);
        }
        u.graphs.clear();
      }
      UGraph x;
      x.fn = fn; x.grid = grid; x.threads = threads; x.prep_smem = prep_smem; x.used = used; x.ev = ev;
      if ((e = build_graph(x, u, a, grid, before_search)) != cudaSuccess) return e;
      u.graphs.push_back(x);
      gr = &u.graphs.back();
    }
    if ((e = set_node_args(*gr, a, u.staging, before_search)) != cudaSuccess) return e;
    if ((e = cudaGraphLaunch(gr->exec, st)) != cudaSuccess) return e;
    u.claimed = false;
    return cudaEventRecord(u.done, st);
  }
  k_uprep<<<1, threads, prep_smem, st>>>(a, u.staging);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if ((e = cudaMemcpyToSymbolAsync(cu_mem, u.staging, used, 0, cudaMemcpyDeviceToDevice, st)) != cudaSuccess) return e;
  if (before_search && (e = cudaEventRecord(before_search, st)) != cudaSuccess) return e;
  if ((e = launch_u_search(a, grid, st)) != cudaSuccess) return e;
  u.claimed = false;
  return cudaEventRecord(u.done, st);
}

// The bank for a peer search: taken only when free and not claimed, atomically with the check, so
// two ranks of one exchange sharing a device never both take it (the second would wait for the
// first, which waits for the second).  The claim ends at the launch (or search_u_release).
int search_u_rows() { return ALP_U_ROWS; }

bool search_u_claim() {
  std::lock_guard<std::mutex> lock(g_u_mu);
  UState &u = ustate();
  if (u.claimed) return false;
  const cudaError_t e = cudaEventQuery(u.done);
  if (e == cudaErrorNotReady) {
    cudaGetLastError();
    return false;
  }
  u.claimed = true;
  return true;
}

void search_u_release() {
  std::lock_guard<std::mutex> lock(g_u_mu);
  ustate().claimed = false;
}

bool search_u_busy() {
  std::lock_guard<std::mutex> lock(g_u_mu);
  UState &u = ustate();
  if (u.claimed) return true;
  const cudaError_t e = cudaEventQuery(u.done);
  if (e == cudaErrorNotReady) {
    cudaGetLastError();  // not an error: clear it
    return true;
  }
  return false;
}

int search_u_max_blocks_per_sm(const SearchArgs &a) {
#define CALL(T_, N, T2) occ_u<N, T2>(a)
  ALP_DISPATCH_U(CALL);
#undef CALL
}


}  // namespace alp
