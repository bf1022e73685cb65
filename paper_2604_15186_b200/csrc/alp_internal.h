// Internal declarations shared by the host library (alp_api.cu) and the kernels (alp_kernels.cu).
// Not part of the C ABI (include/alp.h is).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/alp.h"

namespace alp {

constexpr int kWarpTiles = 32;           // lane tiles per warp group
constexpr int kThreads = 256;            // threads per search block
constexpr uint32_t kPfxTableMax = 4096;  // prefix chunks tabulated in shared memory (8 B each)
constexpr uint32_t kDummy = 0xFFFFFFFFu; // padded row marker in the tile list
constexpr unsigned long long kKeyNone = 0x7FFFFFFFFFFFFFFFull;  // INT64_MAX: nothing feasible

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
};

// Option-term kernel (K1) arguments.
struct OptionArgs {
  DevProfiles prof;
  const double *targets;
  int n_targets;
  float *tau;      // [n_t][M][K]
  double *term;    // [n_t][M][K]
  double *b;       // [n_t][M][K]
  int *u;          // [M][K]
  unsigned long long *keys;    // [n_t] initialised to kKeyNone (may be null)
  unsigned long long *counts;  // [n_t] initialised to 0 (may be null)
  unsigned long long *work;    // [n_work] search work counters, zeroed (may be null)
  int n_work;
};

// Search kernel (K2) arguments: the static plan + per-search values.
struct SearchArgs {
  int M, K;
  int g0, g1;            // prefix LLMs [0,g0), sort-group LLMs [g0,g1)
  int a_llm, b_llm;      // a = LLM M-2 (or -1: virtual single zero option), b = LLM M-1
  int Ka, Kb;
  int ng, dig_bits;      // sort group size, bits per packed digit
  uint32_t L;            // sort-list length K^ng
  uint32_t n_chunks;     // K^g0
  uint32_t n_groups;     // warp groups of 32 lane tiles
  uint32_t nQ, A;        // a-ranges: a in [q*A, min((q+1)*A, Ka))
  uint64_t item_lo, item_hi;
  unsigned long long *work;  // [n_targets * n_bchunks] work counters (zeroed before the launch)
  int grab, grab2;       // items per dynamic work grab: tickets [0, grab_t1) take grab, later ones grab2
  unsigned long long grab_t1;
  FastDiv fd_nQ, fd_ng;  // item -> (chunk, group, a-range) decode when item_hi < 2^31
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
  const uint32_t *tile_off;// [n_tiles][T][2] smem byte offsets of the row's sort-group terms (4 x 16 bit)
  int rows_per_lane;     // T (8 or 16)
  int min_blocks;        // launch-bounds variant for T = 8 (3 or 4 blocks/SM)
  int t_begin, t_end, c_begin, c_end;  // phases (target, b-chunk) evaluated by this launch
  const int *bperm;      // [Kb] canonical option of u-sorted column j
  const int *dv;         // [Dall] distinct b unit values, ascending
  const int *dcnt;       // [Dall+1] dcnt[i] = #u-sorted columns with u <= dv[i-1] (dcnt[0] = 0)
  int D;                 // #distinct b unit values <= budget (masked rows = D + 1)
  uint32_t pw[ALP_MAX_M];// pw[m] = K^(g0-1-m): prefix digit m of a chunk index
  unsigned long long *keys;
  unsigned long long *counts;
  // shared memory layout (byte offsets)
  int off_tau, off_u, off_a, off_lut, off_btab, off_tmp, smem_bytes;
  int off_pfx;           // prefix-chunk table offset, -1 when the prefix space is too large for it
};

// budget of query t (per-query budgets for budget sweeps, else the common budget)
__device__ __forceinline__ int qbudget(const SearchArgs &P, int t) { return P.q_budget ? P.q_budget[t] : P.budget; }

struct FinalizeArgs {
  SearchArgs s;
  const double *term;    // [n_t][M][K]
  const double *b;       // [n_t][M][K]
  const int *S, *T, *R;  // grids (for the winner's (share, tp, replicas))
  int nS, nT, nR;
  uint64_t N;
  const unsigned long long *keys;
  const unsigned long long *counts;
  alp_result *out;       // [n_t] device
  unsigned long long *best;  // [n_t] scratch: ~0 between calls (self-resetting)
  unsigned *done;            // [n_t] scratch: 0 between calls (self-resetting)
};

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

// Launchers (alp_kernels.cu). Return cudaError_t of the launch.
cudaError_t launch_option_table(const OptionArgs &a, cudaStream_t st);
cudaError_t launch_init_keys(unsigned long long *keys, unsigned long long *counts, int n, unsigned long long *work,
                             int n_work, cudaStream_t st);
cudaError_t launch_search(const SearchArgs &a, int grid, cudaStream_t st);
cudaError_t launch_finalize(const FinalizeArgs &a, cudaStream_t st);
cudaError_t launch_predict(const PredictArgs &a, cudaStream_t st);
int search_max_blocks_per_sm(const SearchArgs &a);
cudaError_t launch_egalitarian(const double *lat, int W, int G, long long *best_idx, double *best_min,
                               double *best_sum, cudaStream_t st);

}  // namespace alp
