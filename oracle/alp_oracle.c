/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct CPU reference for the
 * Scepsy ALP allocation search (arXiv 2604.15186).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant with the CUDA path (paper_2604_15186_b200/), and never imports it.
 *
 * Build (done by oracle/__init__.py and __graft_entry__.build()):
 *   gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fPIC -shared -pthread alp_oracle.c -o liboracle.so
 * -ffp-contract=off: no FMA contraction, so every + - * / below is one IEEE-754 RNE operation.
 *
 * What it computes (SURVEY.md §8(c) "Definition"; readings R1-R13 listed in DESIGN.md §3):
 *
 *   For LLM m with option (s_units, t, d), f = s_units / F:              (R1, R2: SPEC.md:196-204)
 *     lam_m = lambda * n_m                      lambda_m = lambda_W * n_m
 *     rate  = lam_m / d                         per-replica rate
 *     x     = rate / f                          base-profile axis L'(l)=L(l/f)/f
 *     b     = ((double)d * (f * T_mt)) / n_m    Eq. 2 term T_m/n_m with capacity d*f*T
 *     ok    = x <= T_mt && b >= lambda && s_units >= minu_mt        (R4)
 *     L     = piecewise-linear lookup of the profile at x            (R3)
 *     term  = (L / f) * (n_m / p_m)             Eq. 1 contribution L_m(lambda n_m) n_m/p_m
 *     tau   = ok ? (float)term : +INF           RNE to binary32 (R7)
 *     u     = s_units * t * d                   GPU units
 *   A profile MEASURED at (m, t, share s) replaces the scaled one (R2: "exact pass-through
 *   when a directly measured profile at target_fraction exists in the store (measured profiles
 *   always win)"): the effective profile is that curve verbatim, so with its points and
 *   saturation throughput T_f:
 *     x     = rate                              lookup axis (no 1/f scaling)
 *     b     = ((double)d * T_f) / n_m           capacity d*T_f
 *     ok    = x <= T_f && b >= lambda && s_units >= minu_mt
 *     term  = L * (n_m / p_m)                   L = lookup of the measured curve at x
 *   Candidate (k_0..k_{M-1}), idx = sum_m k_m * stride_m, LLM 0 most significant,
 *   k = (s_i * nT + t_i) * nR + r_i:
 *     lat32    = tau_0; lat32 = lat32 + tau_m for m = 1..M-1   (binary32, left to right; R7)
 *     units    = sum_m u_m
 *     feasible = all ok_m && units <= B       (north star: reject over budget / under target; R10)
 *   best = argmin_{feasible} lat32, ties -> lowest idx (R6); count = #feasible.
 *   Reported latency = FP64 sum of term_m in the same order (Eq. 1), throughput = min_m b_m (Eq. 2).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int M, F, nS, nT, nR;
  const double *n, *p;       /* [M] */
  const int *S, *T, *R;      /* share units, tp degrees, replica counts */
  const int *prof_off;       /* [M*nT+1] CSR offsets: curve (m,t) = points prof_off[m*nT+t] .. */
  const double *rate, *lat;  /* [P_total] rate and latency at the chosen percentile */
  const double *tmax;        /* [M*nT] saturation throughput T_{m,t} */
  const int *min_units;      /* [M*nT] or NULL (= no floor) */
  /* measured per-share curves (R2), or meas_off == NULL: curve (m, t_i, s_i) = index
   * (m*nT + t_i)*nS + s_i has points meas_off[c] .. meas_off[c+1]-1 (none: scale the base curve) */
  const int *meas_off;       /* [M*nT*nS+1] */
  const double *mrate, *mlat;/* measured rates / latencies at the chosen percentile */
  const double *mtmax;       /* [M*nT*nS] saturation throughput of each measured curve */
} orc_inst;

/* R3: piecewise-linear, clamp below the first point, hold L_last on (r_last, T].
 * i = max{i : r_i <= x}; the interpolation is "3 subs, 1 div, 1 mul, 1 add, this order". */
double orc_lookup(const double *r, const double *l, int P, double x) {
  if (x <= r[0]) return l[0];
  int i = 0;
  for (int j = 0; j < P; ++j)
    if (r[j] <= x) i = j;
  if (i == P - 1) return l[P - 1];
  double dl = l[i + 1] - l[i];
  double dx = x - r[i];
  double dr = r[i + 1] - r[i];
  double w = dx / dr;
  return l[i] + dl * w;
}

/* One option of one LLM at target lambda.  Returns ok (0/1). */
int orc_option(const orc_inst *I, double lambda, int m, int k, float *tau, double *term, double *b,
               int *u) {
  int r_i = k % I->nR;
  int t_i = (k / I->nR) % I->nT;
  int s_i = k / (I->nR * I->nT);
  int s_units = I->S[s_i], t = I->T[t_i], d = I->R[r_i];
  int c = m * I->nT + t_i;
  const double *rr = I->rate + I->prof_off[c];
  const double *ll = I->lat + I->prof_off[c];
  int P = I->prof_off[c + 1] - I->prof_off[c];
  double T = I->tmax[c];

  double lam_m = lambda * I->n[m];
  double rate = lam_m / (double)d;
  double f = (double)s_units / (double)I->F;
  int mc = (m * I->nT + t_i) * I->nS + s_i; /* measured curve of this (LLM, tp, share), if any */
  int measured = I->meas_off && I->meas_off[mc + 1] > I->meas_off[mc];
  double x, bb;
  int ok;
  if (measured) { /* R2: the measured curve verbatim */
    double Tf = I->mtmax[mc];
    x = rate;
    bb = ((double)d * Tf) / I->n[m];
    ok = (x <= Tf) && (bb >= lambda);
  } else {        /* capacity scaling L'(l) = L(l/f)/f, T' = f*T */
    x = rate / f;
    double cap = f * T;
    bb = ((double)d * cap) / I->n[m];
    ok = (x <= T) && (bb >= lambda);
  }
  if (I->min_units && s_units < I->min_units[c]) ok = 0;
  *b = bb;
  *u = s_units * t * d;
  if (ok && measured) {
    int o = I->meas_off[mc];
    double L = orc_lookup(I->mrate + o, I->mlat + o, I->meas_off[mc + 1] - o, x);
    double tt = L * (I->n[m] / I->p[m]);
    *term = tt;
    *tau = (float)tt;
  } else if (ok) {
    double L = orc_lookup(rr, ll, P, x);
    double tt = (L / f) * (I->n[m] / I->p[m]);
    *term = tt;
    *tau = (float)tt;
  } else {
    *term = INFINITY;
    *tau = INFINITY;
  }
  return ok;
}

/* Per-(m,k) option table, M*K entries, row-major [m][k]. */
void orc_option_table(const orc_inst *I, double lambda, float *tau, double *term, double *b, int *u,
                      uint8_t *ok) {
  int K = I->nS * I->nT * I->nR;
  for (int m = 0; m < I->M; ++m)
    for (int k = 0; k < K; ++k)
      ok[m * K + k] = (uint8_t)orc_option(I, lambda, m, k, &tau[m * K + k], &term[m * K + k],
                                          &b[m * K + k], &u[m * K + k]);
}

/* FP64 prediction of one allocation (opt[m] = option index k_m).  Returns feasible (0/1). */
int orc_predict(const orc_inst *I, double lambda, int64_t budget, const int *opt, double *latency,
                double *throughput, int64_t *units, float *lat32) {
  double L = 0.0, Tw = INFINITY;
  float l32 = 0.0f;
  int64_t U = 0;
  int all_ok = 1;
  for (int m = 0; m < I->M; ++m) {
    float tau;
    double term, b;
    int u;
    int ok = orc_option(I, lambda, m, opt[m], &tau, &term, &b, &u);
    all_ok &= ok;
    L = (m == 0) ? term : L + term;
    l32 = (m == 0) ? tau : l32 + tau;
    if (b < Tw) Tw = b;
    U += u;
  }
  *latency = L;
  *throughput = Tw;
  *units = U;
  *lat32 = l32;
  return all_ok && U <= budget;
}

typedef struct {
  int M, K;
  const float *tau;
  const int *u;
  const uint8_t *ok;
  int64_t budget;
  uint64_t lo, hi;
  /* out */
  int found;
  float best;
  uint64_t best_idx;
  uint64_t count;
} orc_job;

/* Brute force over canonical indices [lo, hi) using the per-option table (every candidate's
 * objective, units and feasibility are evaluated literally; the odometer only replaces the
 * mixed-radix division with an increment). */
static void *orc_run(void *arg) {
  orc_job *J = (orc_job *)arg;
  int M = J->M, K = J->K;
  int digit[64];
  uint64_t rem = J->lo;
  for (int m = M - 1; m >= 0; --m) {
    digit[m] = (int)(rem % (uint64_t)K);
    rem /= (uint64_t)K;
  }
  J->found = 0;
  J->best = INFINITY;
  J->best_idx = UINT64_MAX;
  J->count = 0;
  for (uint64_t idx = J->lo; idx < J->hi; ++idx) {
    float lat32 = J->tau[digit[0]];
    int64_t units = J->u[digit[0]];
    int all_ok = J->ok[digit[0]];
    for (int m = 1; m < M; ++m) {
      int j = m * K + digit[m];
      lat32 = lat32 + J->tau[j];
      units += J->u[j];
      all_ok &= J->ok[j];
    }
    if (all_ok && units <= J->budget) {
      J->count++;
      if (!J->found || lat32 < J->best) {
        J->found = 1;
        J->best = lat32;
        J->best_idx = idx;
      }
    }
    for (int m = M - 1; m >= 0; --m) { /* odometer: next canonical index */
      if (++digit[m] < K) break;
      digit[m] = 0;
    }
  }
  return NULL;
}

/* Brute-force search of [lo, hi) at target lambda, budget B (units), with nthreads host threads
 * (static contiguous split, deterministic merge: min value, then min index).  Returns found. */
int orc_search(const orc_inst *I, double lambda, int64_t budget, uint64_t lo, uint64_t hi,
               int nthreads, float *best, uint64_t *best_idx, uint64_t *count) {
  int M = I->M, K = I->nS * I->nT * I->nR;
  float *tau = malloc(sizeof(float) * M * K);
  double *term = malloc(sizeof(double) * M * K);
  double *b = malloc(sizeof(double) * M * K);
  int *u = malloc(sizeof(int) * M * K);
  uint8_t *ok = malloc(M * K);
  orc_option_table(I, lambda, tau, term, b, u, ok);
  if (nthreads < 1) nthreads = 1;
  uint64_t n = hi > lo ? hi - lo : 0;
  if ((uint64_t)nthreads > n) nthreads = n ? (int)n : 1;
  orc_job *jobs = calloc(nthreads, sizeof(orc_job));
  pthread_t *th = calloc(nthreads, sizeof(pthread_t));
  for (int i = 0; i < nthreads; ++i) {
    jobs[i] = (orc_job){M, K, tau, u, ok, budget, lo + n * i / nthreads, lo + n * (i + 1) / nthreads,
                        0, 0, 0, 0};
    if (nthreads == 1)
      orc_run(&jobs[i]);
    else
      pthread_create(&th[i], NULL, orc_run, &jobs[i]);
  }
  int found = 0;
  float bv = INFINITY;
  uint64_t bi = UINT64_MAX, cnt = 0;
  for (int i = 0; i < nthreads; ++i) {
    if (nthreads > 1) pthread_join(th[i], NULL);
    cnt += jobs[i].count;
    if (jobs[i].found && (!found || jobs[i].best < bv || (jobs[i].best == bv && jobs[i].best_idx < bi))) {
      found = 1;
      bv = jobs[i].best;
      bi = jobs[i].best_idx;
    }
  }
  *best = bv;
  *best_idx = bi;
  *count = cnt;
  free(jobs);
  free(th);
  free(tau);
  free(term);
  free(b);
  free(u);
  free(ok);
  return found;
}

/* One candidate, recomputed from the profiles with no hoisting at all (for sampled checks). */
int orc_candidate(const orc_inst *I, double lambda, int64_t budget, uint64_t idx, float *lat32,
                  int64_t *units) {
  int K = I->nS * I->nT * I->nR;
  int opt[64];
  for (int m = I->M - 1; m >= 0; --m) {
    opt[m] = (int)(idx % (uint64_t)K);
    idx /= (uint64_t)K;
  }
  double L, Tw;
  return orc_predict(I, lambda, budget, opt, &L, &Tw, units, lat32);
}
