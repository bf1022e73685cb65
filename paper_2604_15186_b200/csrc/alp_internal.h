// Internal declarations shared by the host library (alp_api.cu) and the kernels (alp_kernels.cu).
// Not part of the C ABI (include/alp.h is).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "../../include/alp.h"

namespace alp {

constexpr int kMaxDevices = 64;         // per-device state arrays (events, graphs, attributes)
constexpr int kWarpTiles = 32;           // lane tiles per warp group
constexpr int kThreads = 256;            // threads per search block
constexpr uint32_t kPfxTableMax = 4096;  // prefix chunks tabulated in shared memory (8 B each)
constexpr uint32_t kDummy = 0xFFFFFFFFu; // padded row marker in the tile list
constexpr unsigned long long kKeyNone = 0x7FFFFFFFFFFFFFFFull;  // INT64_MAX: nothing feasible
constexpr int kUMaxChunks = 16;          // b chunks of the uniform-register path (K <= 1024, 64 columns each)
constexpr int kUChunkW = 64;             // b chunk width of the uniform-register path for long b rows
constexpr int kInlineTargets = 8;        // targets passed in kernel parameters (no H2D copy)
constexpr int kFusedMaxTerms = 1024;     // max option terms (M*K) recomputed per block by the fused launch
constexpr uint64_t kFusedMaxRescan = 65536;  // max finalize re-scan (Ka*Kb) done by one block

// Programmatic dependent launch (sm_90+): a kernel launched with the programmatic-serialization
// attribute may start while its predecessor on the stream still runs; it waits here before
// touching anything the predecessor writes.  No-ops for ordinary launches.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Division by a fixed divisor d for dividends < 2^31: q = umulhi(n, mul) >> shift, with
// shift = ceil(log2 d), mul = ceil(2^(32+shift) / d); mul = 0 encodes d = 1.
struct FastDiv {
  uint32_t mul, shift;
};

// Device-resident profile description (uploaded by alp_build).
struct DevProfiles {
  int M, F, nS, nT, nR, K;
  const double *n, *p;
  const int *S, *T, *R;
  const int *prof_off;
  const double *rate, *lat, *tmax;
  const int *min_units;  // nullptr = no floor
  int n_pts;             // profile points (rate / lat length)
  // measured per-share curves (R2): curve (m*nT + t)*nS + s, points meas_off[c] .. meas_off[c+1]-1
  // (empty: capacity-scale the base curve); nullptr = none measured
  const int *meas_off;
  const double *mrate, *mlat, *mtmax;
  int n_mpts;            // measured points
};

// Option-term kernel (K1) arguments.
struct OptionArgs {
  DevProfiles prof;
  const double *targets;            // [n_targets] device, or nullptr when n_targets <= kInlineTargets
  double tgt[kInlineTargets];       // inline targets
  int n_targets;
  float *tau;      // [n_t][M][K]
  double *term;    // [n_t][M][K]
  double *b;       // [n_t][M][K]
  int *u;          // [M][K]
  unsigned long long *keys;    // [n_t] initialised to kKeyNone (may be null)
  unsigned long long *counts;  // [n_t] initialised to 0 (may be null)
  unsigned long long *work;    // [n_work] search work counters, zeroed (may be null)
  int n_work;
  unsigned long long *fbest;   // [n_targets] finalize combine scratch, zeroed (may be null)
  unsigned *fdone;             // [n_targets] zeroed (may be null)
};


// Finalize inputs/outputs (K3, or the fused search's last block).
struct FinalizeExtra {
  const double *term;    // [n_t][M][K] FP64 Eq. 1 terms
  const double *b;       // [n_t][M][K] FP64 Eq. 2 terms
  const int *S, *T, *R;  // grids (for the winner's (share, tp, replicas)); S == nullptr: injected terms
  int nS, nT, nR;
  uint64_t N;
  const unsigned long long *keys;    // [n_t] reduced keys (K3 input); world > 0: [world][2][n_t] gathered pairs
  const unsigned long long *counts;  // [n_t] reduced counts (K3 input; unused when world > 0)
  int world;                         // > 0: K3 reduces the gathered per-rank (keys, counts) itself
  alp_result *out;       // [n_t] device
  unsigned long long *best;  // [n_t] scratch: complemented minimum, 0 between calls (self-resetting)
  unsigned *done;            // [n_t] scratch: 0 between calls (self-resetting)
  int stage;                 // the fused epilogue may stage the finalize inputs in dynamic smem
};

// Peer exchange (alp_search_peer): the fused epilogue of every rank's search finalizes its own
// shard, writes the (key, count, local result) rows into every rank's exchange buffer over
// NVLink peer memory, and waits for all ranks' rows in its own buffer; then it reduces them (MIN
// key, SUM count) and stores the winner's result.  Exchange buffer of a rank (alp_peer_bytes):
//   [0, 8)    epoch of the last completed exchange (read / written by the owner only)
//   [64, ...) u64 flags[2][kMaxPeers]: flags[p][j] = epoch of rank j's rows in slot p
//   [kPeerHdr, ...) PeerRow rows[2][world][n]: slot p = epoch & 1 (double-buffered: a rank may
//   start epoch e + 1 while a slower rank still reads epoch e)
constexpr int kMaxPeers = 16;
constexpr size_t kPeerHdr = 512;
struct PeerRow {
  unsigned long long key, count;  // the rank's reduced key (kKeyNone: nothing feasible) and count
  alp_result res;                 // the rank's finalize of its key (its own shard)
};
struct PeerArgs {
  int on, rank, world;
  unsigned char *buf[kMaxPeers];  // every rank's exchange buffer as mapped in this process
  alp_result *out;                // [n] final results (mapped host memory)
  long long timeout_ns;           // give up waiting for the other ranks after this long
};

// Bytes of the finalize's optional shared-memory staging (see finalize_target): FP64 Eq. 1 and
// Eq. 2 terms, binary32 terms and units of every option, and the share / TP / replica grids.
__host__ __device__ inline size_t finalize_stage_bytes(int M, int K, int nS, int nT, int nR) {
  return (size_t)M * K * (8 + 8 + 4 + 4) + (size_t)(nS + nT + nR) * 4;
}

// Fused single-launch search (targets <= kInlineTargets): every block computes the option terms of
// the phase's target in its prologue (no K1), blocks accumulate into self-resetting scratch, and
// the last block to finish writes the (key, count) pairs, resets the scratch and (finalize = 1)
// runs the finalize (no K3).
struct FusedArgs {
  int on, finalize;
  DevProfiles prof;
  double tgt[kInlineTargets];
  const float *tau_fixed;     // injected terms (alp_build_from_terms) instead of prof, or nullptr
  float *o_tau;               // [n_t][M][K] written by block 0 (K3 / finalize inputs)
  double *o_term, *o_b;       // [n_t][M][K] written by block 0 (nullptr with injected terms)
  unsigned long long *acc_keys;    // [n_t] complemented keys (~key, atomicMax), 0 at rest
  unsigned long long *acc_counts;  // [n_t] 0 at rest
  unsigned long long *work;        // [n_t * n_bchunks] 0 at rest
  unsigned *ticket;                // 0 at rest
  int off_opt;                // smem offset of the phase's option terms [M*K] floats
  PeerArgs peer;              // peer exchange in the epilogue (peer.on)
};

// Search kernel (K2) arguments: the static plan + per-search values.
struct SearchArgs {
  int M, K;
  int g0, g1;            // prefix LLMs [0,g0), sort-group LLMs [g0,g1)
  int a_llm, b_llm;      // a = LLM M-2 (or -1: virtual single zero option), b = LLM M-1
  int Ka, Kb;
  int ng;                // sort group size (LLMs)
  uint32_t L;            // sort-list length K^ng
  uint32_t n_chunks;     // K^g0
  uint32_t n_groups;     // warp groups of 32 lane tiles
  uint32_t nQ, A;        // a-ranges: a in [q*A, min((q+1)*A, Ka))
  uint64_t item_lo, item_hi;
  unsigned long long *work;  // [n_targets * n_bchunks] work counters (zeroed before the launch)
  int grab, grab2;       // items per dynamic work grab: tickets [0, grab_t1) take grab, later ones grab2
  unsigned long long grab_t1;
  FastDiv fd_nQ, fd_ng;  // item -> (chunk, group, a-range) decode when item_hi < 2^31
  // segment ids (key low word): row * seg_q + (first a option evaluated) / seg_A, where seg_A = 1
  // (single-option granularity) when rows * Ka < 2^32, else seg_A = A; seg_mul = A / seg_A
  uint32_t seg_q, seg_A, seg_mul;
  // k_search_u tail split: tickets [0, u_nbulk) are whole items, then the rank's remaining items are
  // cut into u_S sub-items of u_As a options (ticket -> item nbulk + j / u_S, part j % u_S)
  uint32_t u_nbulk, u_S, u_As;
  FastDiv fd_S;
  int budget;            // R (capped at the total max units); max over queries when q_budget is set
  const int *q_budget;   // [n_targets] per-query budgets (capped) or nullptr (all = budget)
  int n_targets;
  int n_bchunks, bchunk_w, bchunk_wpad;  // b columns (u-sorted) split in chunks
  int row_stride;        // floats per masked row (== 4 mod 8)
  int rows_max;          // max distinct masked rows per chunk
  // device tables
  const float *tau;      // [n_t][M][K]
  const int *u;          // [M][K]
  const int *tile_s;     // [n_tiles] units of the lane tile's sort-group options
  const uint32_t *tile_e;// [n_tiles][T] canonical sort-group entry index (kDummy = padding)
  const uint32_t *tile_off;// [n_tiles][T][4] smem byte offsets of the row's sort-group terms
  int rows_per_lane;     // T (12 by default; 8 or 16 via ALP_ROWS_PER_LANE)
  int min_blocks;        // launch-bounds variant for T = 8 (3 or 4 blocks/SM)
  int t_begin, t_end, c_begin, c_end;  // phases (target, b-chunk) evaluated by this launch
  const int *bperm;      // [Kb] canonical option of u-sorted column j
  const int *dv;         // [Dall] distinct b unit values, ascending
  const int *dcnt;       // [Dall+1] dcnt[i] = #u-sorted columns with u <= dv[i-1] (dcnt[0] = 0)
  int D;                 // #distinct b unit values <= budget (masked rows = D + 1)
  uint32_t pw[ALP_MAX_M];// pw[m] = K^(g0-1-m): prefix digit m of a chunk index
  unsigned long long *keys;
  unsigned long long *counts;
  FusedArgs fz;
  FinalizeExtra fin;
  unsigned long long *dbg_ts;  // [grid][8] %globaltimer stamps per block (ALP_DBG_TS) or nullptr
  // uniform-register path (k_uprep + k_search_u): tables in the constant bank
  uint32_t n_groups_u;   // warp groups [0, n_groups_u) have one unit sum (uniform remaining budget)
  const int *gsum;       // [n_groups] their unit sums; mixed groups: their smallest tile sum (plan)
  int lut_base;          // lut index of remaining budget r = r + lut_base - R (>= 0 for every r reached;
                         // unit sums enter clamped at R + 1, which keeps an over-budget r negative)
  int lut_n;             // lut entries (lut_base + 1)
  // byte layout of the constant-bank tables: gsum at 0; target t's block at u_tbase + t*u_tstride
  // with the a-options and prefix chunks at these offsets inside it, then per b chunk c its lut and
  // its masked rows (u_off_lut_c[c], u_off_btab_c[c]; rows of u_cstride floats)
  int u_tbase, u_tstride, u_off_a, u_off_pfx;
  int u_off_lut_c[kUMaxChunks], u_off_btab_c[kUMaxChunks];
  int u_nch, u_cstride;  // b chunks (each bchunk_w u-sorted columns, padded to bchunk_wpad) and row stride
  int u_smem_rows;       // 1: the mixed groups read the (single) chunk's lut and rows from shared memory
  // shared memory layout (byte offsets)
  int off_tau, off_u, off_a, off_lut, off_btab, off_tmp, smem_bytes;
  int off_pfx;           // prefix-chunk table offset, -1 when the prefix space is too large for it
  // (last: ptxas' uniform-datapath choices in k_search_u change with the offsets of the fields above)
  int u_amax;            // largest a-option unit count (clamped at R + 1): lut(x - u_amax) is the
                         // widest row every a option of a warp-uniform budget x reaches
};

// budget of query t (per-query budgets for budget sweeps, else the common budget)
__device__ __forceinline__ int qbudget(const SearchArgs &P, int t) { return P.q_budget ? P.q_budget[t] : P.budget; }

struct PredictArgs {
  DevProfiles prof;
  const int *opts;       // [n][M]
  int n;
  double lambda;
  long long budget;
  double *latency, *throughput;
  long long *units;
  int *feasible;
};

// Launch with the programmatic-stream-serialization attribute (see pdl_wait).
template <typename Args>
inline cudaError_t launch_pdl(void (*fn)(Args), dim3 grid, dim3 block, size_t smem, cudaStream_t st, const Args &a) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  static const bool off = getenv("ALP_NO_PDL") != nullptr;  // A/B switch for measurements
  cfg.numAttrs = off ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, fn, a);
}

// Launchers (alp_kernels.cu). Return cudaError_t of the launch.
cudaError_t launch_option_table(const OptionArgs &a, cudaStream_t st);
cudaError_t launch_init_keys(unsigned long long *keys, unsigned long long *counts, int n, unsigned long long *work,
                             int n_work, unsigned long long *fbest, unsigned *fdone, cudaStream_t st);
cudaError_t launch_search(const SearchArgs &a, int grid, cudaStream_t st);
// uniform-register path: prep (option terms + constant-bank tables, one block) and search
// (before_search, if set, is recorded on st between the prep and the search kernel)
cudaError_t launch_search_u(const SearchArgs &a, int grid, cudaStream_t st, cudaEvent_t before_search);
int search_u_max_blocks_per_sm(const SearchArgs &a);
int search_u_rows();   // rows per lane the uniform-register kernel was compiled for (ALP_U_ROWS)
bool search_u_busy();  // a uniform-register search launched on this device has not completed yet
bool search_u_claim(); // take the bank for a peer search if it is free (see alp_search_u.cu)
void search_u_release();
size_t uprep_smem_bytes(const SearchArgs &a);  // k_uprep dynamic shared memory (<= kUPrepSmemMax)
constexpr size_t kUPrepSmemMax = 200 * 1024;
constexpr int kUBytes = 60 * 1024;      // constant-bank table space of the uniform-register path
cudaError_t launch_finalize(const SearchArgs &a, cudaStream_t st);
// SPEC.md:374 fallback: the max-T_w candidate within budget B into *out (device or mapped memory).
cudaError_t launch_max_throughput(const double *b, const int *u, const DevProfiles &pr, long long B, uint64_t N,
                                  alp_result *out, cudaStream_t st);
// Static plan: tile_off[4 * row] (shared-memory byte offsets of the row's sort-group terms) from
// tile_e (canonical within-group index or kDummy) on the device.
cudaError_t launch_plan_offsets(const uint32_t *tile_e, size_t rows, int g0, int g1, int ng, int K, uint32_t *tile_off,
                                cudaStream_t st);
// One-pass budget-indexed search (alp_levels.cu): per-level best keys over the candidates with
// units <= bmax, then per-query keys (prefix minimum over levels) and exact counts.
cudaError_t launch_levels(const SearchArgs &s, const int *d_levels, int L, int bmax, unsigned long long *lvl_keys,
                          unsigned long long *ticket, const int *d_q_level, int n, unsigned long long *keys,
                          unsigned long long *counts, unsigned long long *h0, unsigned long long *h1, int sm_count,
                          cudaStream_t st);
cudaError_t launch_predict(const PredictArgs &a, cudaStream_t st);
int search_max_blocks_per_sm(const SearchArgs &a);
cudaError_t launch_egalitarian(const double *lat, int W, int G, long long *best_idx, double *best_min,
                               double *best_sum, cudaStream_t st);

}  // namespace alp
