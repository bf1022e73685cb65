// FP64 option terms of PAPER.md:355-359 (K1's arithmetic), shared by the option-term kernel, the
// fused search prologue (alp_search.cuh) and k_predict.
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>

#include "alp_internal.h"

namespace alp {

// ------------------------------------------------------------------ option terms (FP64, no FMA)
// SURVEY.md §8(c) / DESIGN.md §3: every operation is an explicit IEEE RNE intrinsic, in the
// order written, so the result is bit-identical to the oracle's -ffp-contract=off C code.
__device__ __forceinline__ double lookup_latency(const double *r, const double *l, int P, double x) {
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

__device__ __forceinline__ int option_terms(const DevProfiles &P, double lambda, int m, int k, float *tau, double *term,
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
  const int mc = (m * P.nT + t_i) * P.nS + s_i;               // measured curve of (LLM, tp, share)
  const bool measured = P.meas_off && P.meas_off[mc + 1] > P.meas_off[mc];
  double x, bb;
  int ok;
  if (measured) {  // R2: the measured curve verbatim ("measured profiles always win")
    const double Tf = P.mtmax[mc];
    x = rate;
    bb = __ddiv_rn(__dmul_rn((double)d, Tf), P.n[m]);         // Eq. 2 term, capacity d*T_f
    ok = (x <= Tf) && (bb >= lambda);
  } else {         // capacity scaling L'(l) = L(l/f)/f, T' = f*T
    x = __ddiv_rn(rate, f);
    const double cap = __dmul_rn(f, T);
    bb = __ddiv_rn(__dmul_rn((double)d, cap), P.n[m]);        // Eq. 2 term
    ok = (x <= T) && (bb >= lambda);                          // R4
  }
  if (P.min_units && s_units < P.min_units[c]) ok = 0;        // memory floor
  *b = bb;
  *u = s_units * t * d;
  if (ok && measured) {
    const int o = P.meas_off[mc];
    const double L = lookup_latency(P.mrate + o, P.mlat + o, P.meas_off[mc + 1] - o, x);
    const double tt = __dmul_rn(L, __ddiv_rn(P.n[m], P.p[m]));  // Eq. 1 term of the measured profile
    *term = tt;
    *tau = __double2float_rn(tt);
  } else if (ok) {
    const int o = P.prof_off[c];
    const double L = lookup_latency(P.rate + o, P.lat + o, P.prof_off[c + 1] - o, x);
    const double tt = __dmul_rn(__ddiv_rn(L, f), __ddiv_rn(P.n[m], P.p[m]));  // Eq. 1 term
    *term = tt;
    *tau = __double2float_rn(tt);
  } else {
    *term = CUDART_INF;
    *tau = __int_as_float(0x7f800000);
  }
  return ok;
}

}  // namespace alp
