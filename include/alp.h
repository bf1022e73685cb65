/*
 * alp.h — C ABI of the B200-native exhaustive ALP allocation search (Scepsy, arXiv 2604.15186).
 *
 * The operation ("Workflow Predictions", Eq. 1 at PAPER.md:340-343, Eq. 2 at
 * PAPER.md:346-349; scheduler goal "lowest latency within a target workflow-level arrival rate",
 * PAPER.md:293): for every candidate allocation — each LLM m gets a per-shard GPU share
 * f_m = share_units/F, a tensor-parallel degree tp_m and a replica count d_m — predict the
 * workflow latency L_w (Eq. 1) and throughput T_w (Eq. 2) from the per-LLM profiles and the
 * workflow statistics (n_m, p_m), reject candidates that exceed the GPU budget or
 * miss the throughput target, and return the minimum-latency candidate (lowest canonical index
 * on ties) plus the number of feasible candidates.  The exact arithmetic (FP64 option terms,
 * canonical binary32 objective) is fixed in DESIGN.md §3 (readings R1-R13 of SURVEY.md §8(c)).
 *
 * Candidate order: option index inside an LLM k = (s_i*nT + t_i)*nR + r_i
 * (share most significant, replicas least); candidate index idx = sum_m k_m * K^(M-1-m) (LLM 0
 * most significant), K = nS*nT*nR.
 *
 * Conventions
 *  - Every entry point returns alp_status; on error alp_last_error() names the offending field.
 *    No C++ exception crosses this boundary.
 *  - alp_build copies every input array; the caller may free them on return.  The handle owns
 *    host copies plus immutable device tables on the device current at build time.  A handle may
 *    be used by one host thread at a time.  Calls that use the handle's own scratch are ordered on
 *    the device even across streams (a call on another stream waits for the handle's previous
 *    work), and alp_destroy releases device memory stream-ordered after that work.  Calls given a
 *    caller workspace (alp_workspace_bytes; "predictions are pure and may run
 *    concurrently") are NOT ordered against each other: searches on distinct workspaces and
 *    streams overlap on the device; alp_destroy then synchronises the device first.
 *  - Budgets are integer GPU units (1 unit = 1/F GPU); targets are workflow requests/second.
 *  - All results are bit-identical for any rank count / grid shape (see alp_search_shard).
 */
#ifndef SCEPSY_ALP_H
#define SCEPSY_ALP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ALP_MAX_M 16        /* max LLMs per workflow */
#define ALP_MAX_K 1024      /* max options per LLM (nS*nT*nR) */

typedef struct alp_s alp_t; /* opaque, immutable after alp_build */

typedef enum {
  ALP_OK = 0,          /* success */
  ALP_EINVAL = 1,      /* invalid argument (field named by alp_last_error) */
  ALP_EINFEASIBLE = 2, /* search finished but no candidate is feasible (result.found = 0) */
  ALP_EINTERNAL = 3,   /* internal inconsistency */
  ALP_ECUDA = 4,       /* CUDA runtime error (message in alp_last_error) */
  ALP_ENCCL = 5        /* cross-GPU exchange failed (raised by the binding around torch.distributed's
                          NCCL collectives; the library itself never calls NCCL) */
} alp_status;

typedef enum { ALP_P_MEAN = 0, ALP_P50 = 1, ALP_P90 = 2, ALP_P99 = 3 } alp_percentile; /* PAPER.md:356 "percentile P" */

/* Workflow + profile description (host pointers, caller-owned, copied by alp_build).
 * Profiles: one piecewise-linear curve per (LLM m, tp index t), CSR over points:
 * curve c = m*nT + t has points prof_off[c] .. prof_off[c+1]-1 (>= 1 point), rates strictly
 * increasing, latencies > 0 and non-decreasing.  T_{m,t} = tmax[c] (>= last
 * rate) or the last rate when tmax == NULL.  Sub-GPU shares use capacity scaling
 * L'(x) = L(x/f)/f, T' = f*T (reading R2). */
typedef struct {
  int32_t M;                    /* number of LLMs, 1..ALP_MAX_M */
  int32_t F;                    /* GPU units per GPU (share grid denominator), >= 1 */
  const double *n;              /* [M] mean invocations per workflow request, > 0 */
  const double *p;              /* [M] mean request-level parallelism, >= 1 */
  int32_t nS, nT, nR;           /* grid sizes; K = nS*nT*nR <= ALP_MAX_K */
  const int32_t *share_units;   /* [nS] strictly ascending, 1..F */
  const int32_t *tp;            /* [nT] strictly ascending, >= 1 */
  const int32_t *replicas;      /* [nR] strictly ascending, >= 1 */
  const int32_t *prof_off;      /* [M*nT+1] CSR offsets, prof_off[0] = 0 */
  const double *rate;           /* [prof_off[M*nT]] requests/s */
  const double *lat[4];         /* per alp_percentile column, seconds; NULL = absent */
  const double *tmax;           /* [M*nT] saturation throughput or NULL */
  const int32_t *min_units;     /* [M*nT] memory floor in units per shard, or NULL */
  int32_t pct;                  /* alp_percentile used by this handle */
  /* Optional profiles MEASURED at a share (reading R2, "measured profiles always win"):
   * curve c = (m*nT + t)*nS + s (LLM m, tp index t, share index s) has points meas_off[c] ..
   * meas_off[c+1]-1; an empty curve means "not measured" (the base curve is capacity-scaled).  A
   * measured curve is used verbatim: lookup at the per-replica rate, capacity d*T_f, no 1/f factor.
   * Same rules as the base curves (rates strictly increasing, latencies > 0 non-decreasing,
   * meas_tmax[c] >= the last rate or NULL = the last rate).  meas_off == NULL: none measured. */
  const int32_t *meas_off;      /* [M*nT*nS+1] */
  const double *meas_rate;      /* [meas_off[M*nT*nS]] requests/s */
  const double *meas_lat[4];    /* per alp_percentile column; the selected one must be present */
  const double *meas_tmax;      /* [M*nT*nS] or NULL */
} alp_desc;

/* One search result (all fields host-side after the call returns). */
typedef struct {
  int32_t found;                /* 0 => no feasible candidate */
  int32_t M;
  uint64_t index;               /* canonical candidate index (UINT64_MAX if !found) */
  float latency_key;            /* canonical binary32 objective of the winner (R7) */
  double latency;               /* FP64 Eq. 1 L_w of the winner, seconds */
  double throughput;            /* FP64 Eq. 2 T_w of the winner, requests/s */
  int64_t units;                /* GPU units used by the winner */
  uint64_t feasible_count;      /* number of feasible candidates (R10) */
  uint64_t candidates;          /* candidates evaluated = N (exhaustive) */
  int32_t share_units[ALP_MAX_M], tp[ALP_MAX_M], replicas[ALP_MAX_M]; /* winner, per LLM */
  /* 1 when found = 0 but some candidate fits the budget: index, share_units / tp / replicas, units
   * and throughput then describe the candidate with the maximal Eq. 2 T_w among those within the
   * budget whose options clear their memory floors (lowest canonical index on ties; SPEC.md:374
   * "no feasible candidate -> returns the candidate with maximal T_w flagged INFEASIBLE-rate");
   * latency stays +inf.  0 otherwise. */
  int32_t fallback;
} alp_result;

/* Validate, copy and plan.  Uploads the profile tables and the static search plan to the
 * current CUDA device.  Errors: ALP_EINVAL naming the field; ALP_ECUDA. */
alp_status alp_build(const alp_desc *desc, alp_t **out);

/* Test-only constructor: search directly over given binary32 option terms tau[M*K] (+INF =
 * infeasible option) and units u[M*K], bypassing the profiles (same for every target).  Used to
 * inject exactly-representable terms and ties (SURVEY.md §8(c) "option-table injection"). */
alp_status alp_build_from_terms(int32_t M, int32_t K, const float *tau, const int32_t *u, alp_t **out);

void alp_destroy(alp_t *h);

/* N = K^M candidates. */
uint64_t alp_num_candidates(const alp_t *h);

/* Host bytes copied to the device by alp_build (for end-to-end accounting). */
uint64_t alp_h2d_bytes(const alp_t *h);

/* Canonical index -> per-LLM (share units, tp, replicas); out arrays [M]. */
alp_status alp_decode(const alp_t *h, uint64_t index, int32_t *share_units, int32_t *tp, int32_t *replicas);

/* Per-option table at target lambda, computed by the device option-term kernel and copied back:
 * tau[M*K] (binary32 Eq. 1 terms, +INF if infeasible), term[M*K] (FP64), b[M*K] (FP64 Eq. 2
 * terms d*f*T/n), u[M*K] units.  Any output pointer may be NULL. */
alp_status alp_option_table(alp_t *h, double lambda, float *tau, double *term, double *b, int32_t *u);

/* FP64 prediction of n allocations at target lambda (device kernel; synchronous).
 * opts[n*M] = option index k_m per LLM; outputs [n]: latency (INF if infeasible), throughput,
 * units, feasible (budget_units applied). */
alp_status alp_predict(alp_t *h, const int32_t *opts, int32_t n, double lambda, int64_t budget_units,
                       double *latency, double *throughput, int64_t *units, int32_t *feasible);

/* Single-device search on the current device (internal stream, synchronous).  Returns ALP_OK,
 * or ALP_EINFEASIBLE with out->found = 0. */
alp_status alp_search(alp_t *h, double target, int64_t budget_units, alp_result *out);

/* Batched targets (Pareto sweep): out[n]. Returns ALP_OK if at least one target is feasible. */
alp_status alp_search_batch(alp_t *h, const double *targets, int32_t n, int64_t budget_units, alp_result *out);

/* Independent (target, budget) queries in one pass, out[n] — e.g. the best allocation of one
 * workflow for every GPU count (the budget-indexed search behind multi-workflow scheduling,
 * PAPER.md:396-398).  budgets[i] >= 0 units.  Returns ALP_OK if at least one query is feasible. */
alp_status alp_search_queries(alp_t *h, const double *targets, const int64_t *budgets, int32_t n, alp_result *out);

/* Multi-workflow allocation ("egalitarian welfare"; utility per SPEC.md:383):
 * W workflows (handles hs[w], all built on one device, same units-per-GPU F) with targets[w]; the
 * cluster has `gpus` GPUs of `units_per_gpu` units.  For each workflow the budget-indexed search
 * gives L_w(g), the best FP64 latency on g = 0..gpus whole GPUs; utility u_w(g) = L_w(gpus)/L_w(g)
 * (0 if infeasible).  Chooses the split g_0..g_{W-1} (sum = gpus) maximising min_w u_w, then
 * sum_w u_w, then the lowest split index (g_0 most significant), in a device kernel.
 * gpus_out[W] = GPUs per workflow; results_out[W] = each workflow's best allocation on its share;
 * min/sum utility optional.  ALP_EINFEASIBLE if some workflow is infeasible on its share. */
alp_status alp_schedule_egalitarian(alp_t *const *hs, const double *targets, int32_t W, int32_t gpus,
                                    int32_t units_per_gpu, int32_t *gpus_out, alp_result *results_out,
                                    double *min_utility, double *sum_utility);

/* Workflow statistics from execution traces (the input side of alp_build):
 * n_m = invocations of LLM m per workflow request; p_m = request-level parallelism, the time
 * average of the number of concurrently running invocations of m over the intervals where it is
 * >= 1, averaged over requests weighted by each request's busy time for m
 * = sum_r (summed durations) / sum_r (length of the union of m's intervals in request r); 1 for an
 * LLM with no (or only zero-length) invocations.  Host computation (traces are small).
 * Invocation i: request req[i] in [0, n_req), LLM llm[i] in [0, M), start[i] <= end[i] (seconds). */
alp_status alp_workflow_stats(int32_t n_req, int32_t M, int64_t n_inv, const int32_t *req, const int32_t *llm,
                              const double *start, const double *end, double *n_out, double *p_out);

/* Topology-aware placement of an allocation ("hierarchical placement",
 * most-constrained-first, inter-node stage then intra-node stage; SPEC.md:440-445 tie-breaks).  Cluster: G GPUs of F units; gpu_node[g],
 * gpu_domain[g] = node and NVLink domain of GPU g (a domain never spans nodes).  Allocation: per LLM
 * share_units (per shard, 1..F), tp, replicas; every replica is a tensor group of tp shards.
 * Output shard_gpu[sum_m tp_m*replicas_m], ordered (LLM, replica, shard): the GPU of each shard.
 * Tensor groups use distinct GPUs of one NVLink domain.  ALP_EINFEASIBLE names the first shard
 * group that cannot be placed. */
alp_status alp_place(int32_t G, int32_t F, const int32_t *gpu_node, const int32_t *gpu_domain, int32_t M,
                     const int32_t *share_units, const int32_t *tp, const int32_t *replicas, int32_t *shard_gpu);

/* ---- multi-GPU building blocks (PyTorch owns memory, streams and the process group) ----
 * The candidate space is cut into equal-cost work items; rank r of world w gets the contiguous
 * item range [lo, hi).  Every rank calls alp_search_shard on its range (async on `stream`),
 * then all-reduces keys with MIN and counts with SUM as int64 (every key < 2^63), then calls
 * alp_finalize with the reduced arrays.  Keys encode (binary32 objective, global segment id),
 * so the reduced result does not depend on how items were split. */
uint64_t alp_num_items(const alp_t *h, int64_t budget_units);
alp_status alp_shard_range(const alp_t *h, int64_t budget_units, int32_t rank, int32_t world, uint64_t *lo,
                           uint64_t *hi);
/* Bytes of a caller-owned device workspace for searches of n_targets targets (0 on a NULL handle
 * or n_targets < 1).  A workspace holds one search's option tables, accumulators, work counters
 * and finalize scratch.  It must be 256-byte aligned and zero-filled before its first use (e.g.
 * torch.zeros); every call leaves its leading control section zero again, so it can be reused
 * without re-clearing.  Give alp_finalize the workspace (and n) the shard search used. */
size_t alp_workspace_bytes(const alp_t *h, int32_t n_targets);
/* d_keys/d_counts: device int64[n] (initialised by this call).  d_workspace: NULL (the handle's
 * own scratch; calls ordered across streams) or alp_workspace_bytes(h, n) caller-owned bytes (no
 * ordering against other calls: concurrent searches on distinct workspaces / streams).
 * stream: cudaStream_t or NULL (the handle's stream).  Asynchronous. */
alp_status alp_search_shard(alp_t *h, const double *targets, int32_t n, int64_t budget_units, uint64_t lo,
                            uint64_t hi, void *d_workspace, void *stream, int64_t *d_keys, int64_t *d_counts);
/* Decode reduced keys on the device (lowest index inside the winning segment, FP64 Eq. 1/Eq. 2
 * of the winner) and copy n results to the host (synchronises `stream`).  d_workspace: the one the
 * shard search used (NULL: the handle's own). */
alp_status alp_finalize(alp_t *h, const double *targets, int32_t n, int64_t budget_units,
                        const int64_t *d_keys, const int64_t *d_counts, void *d_workspace, void *stream,
                        alp_result *out);
/* Same, from the per-rank pairs gathered by ONE all-gather instead of two all-reduces: every rank
 * searches with d_keys = buf, d_counts = buf + n (a contiguous int64[2n] buffer), all-gathers buf
 * into d_gathered = int64[world][2][n], and the finalize kernel takes the MIN of the keys and the
 * SUM of the counts itself (the result equals alp_finalize's on the all-reduced pair). */
alp_status alp_finalize_gathered(alp_t *h, const double *targets, int32_t n, int64_t budget_units,
                                 const int64_t *d_gathered, int32_t world, void *d_workspace, void *stream,
                                 alp_result *out);

/* ---- fused peer exchange: the cross-GPU reduction inside the search kernel ----
 * Instead of a collective and a finalize launch, the last block of every rank's search kernel
 * finalizes its own shard (its key's segment lies in its shard), stores its (key, count, result)
 * rows into every rank's exchange buffer over NVLink peer memory (release flag per destination),
 * waits for all ranks' rows in its own buffer (acquire), and reduces them: MIN key, SUM count, the
 * winning rank's result — the same result as alp_finalize on the all-reduced pair, on every rank.
 * Each rank owns one exchange buffer of alp_peer_bytes(n, world) bytes from alp_peer_alloc on its
 * device; the ranks share them by IPC handles (alp_peer_ipc_handle / alp_peer_open, e.g. through
 * the process group) or, inside one process, by plain device pointers.  All ranks must call
 * alp_search_peer the same number of times with the same (targets, budget, world) and their own
 * buffer at d_bufs[rank]: the buffers count exchanges (epochs) and alternate two row slots. */
size_t alp_peer_bytes(int32_t n_targets, int32_t world);     /* 0 if n_targets < 1 or world < 1 */
/* Zero-filled device allocation of its own (IPC-shareable) on the current device. */
alp_status alp_peer_alloc(size_t bytes, void **d_buf);
alp_status alp_peer_free(void *d_buf);
/* 64-byte cudaIpcMemHandle_t of a buffer from alp_peer_alloc (written to handle). */
alp_status alp_peer_ipc_handle(void *d_buf, void *handle);
/* Map another process's buffer into this one (cudaIpcOpenMemHandle; not for this process's own). */
alp_status alp_peer_open(const void *handle, void **d_peer);
alp_status alp_peer_close(void *d_peer);
/* Search items [lo, hi) (alp_shard_range(rank, world) in a real run) and exchange with the other
 * world-1 ranks; n <= 8 targets, a fused-size problem (M*K <= 1024, Ka*Kb <= 65536: C1, C2, C4,
 * the hand case; others ALP_EINVAL — use alp_search_shard + a collective).  d_bufs[world]: every
 * rank's buffer as mapped in this process.  Synchronous: returns with out[n] (identical on every
 * rank) on the host.  ALP_EINTERNAL if the other ranks do not arrive within ALP_PEER_TIMEOUT_MS
 * (default 30000).  d_workspace / stream as in alp_search_shard. */
alp_status alp_search_peer(alp_t *h, const double *targets, int32_t n, int64_t budget_units, uint64_t lo,
                           uint64_t hi, int32_t rank, int32_t world, void *const *d_bufs, void *d_workspace,
                           void *stream, alp_result *out);

/* Device time (ms) of the last search kernel launched through this handle (CUDA events on the
 * launching stream), and the number of kernels the last search/finalize launched.  Searches with
 * short b rows and a common budget run the uniform-register pair (option terms + constant-bank
 * tables, then the search with the finalize fused; batches in groups of 8 targets); other searches
 * of at most 8 targets with a common budget run as ONE kernel (option terms, exhaustive search and
 * finalize fused); the rest run K1 + K2 + K3. */
float alp_last_kernel_ms(const alp_t *h);
int32_t alp_last_launches(const alp_t *h);
/* Device time (ms) of the last complete search step through this handle: CUDA events on the
 * search stream from the start of alp_search* / alp_search_shard to the completion of the
 * result D2H in alp_search* / alp_finalize (includes an all-reduce issued in between on that
 * stream; excludes the host's wake-up after the final synchronisation). */
float alp_last_step_ms(const alp_t *h);
/* Which search kernel the last search ran: 0 = k_search (shared-memory masked rows), 1 = the
 * uniform-register pair k_uprep + k_search_u (single target, short b rows; ALP_NO_UR disables). */
int32_t alp_last_path(const alp_t *h);

/* Static search plans (sort-list tiles, u-sorted columns; they depend only on the grids) are cached
 * process-wide and shared by handles built on the same device with the same grids.  This drops the
 * cache (plans still referenced by live handles stay alive until those handles are destroyed). */
void alp_plan_cache_clear(void);

/* Thread-local message for the last error (never NULL). */
const char *alp_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* SCEPSY_ALP_H */
