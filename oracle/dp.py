"""ORACLE O2 — test infrastructure only.  Exact search by dynamic programming (SURVEY.md §8(c)
"Special cases that reduce to textbook routines": the search is a multiple-choice knapsack with a
separable objective).

Input is the per-option table (tau: binary32 Eq. 1 terms with +inf for infeasible options, u: GPU
units) — the same quantities O1 enumerates — so O2 checks O1's *search* (enumeration order, sum
order, budget test, tie-break, count) with a different algorithm:

* value DP   V_m[U] = min over options of fl32(V_{m-1}[U - u] + tau)   (exact: binary32 RNE addition
  is monotone non-decreasing in each argument, so the minimal partial sum per (m, units) state
  dominates every completion; the canonical sum order ((tau_0 + tau_1) + tau_2) + ... is kept);
* lowest-index DFS  walks LLM 0..M-1 taking the smallest option from which the optimum is still
  reachable (re-running the value DP from the partial state), giving the lowest canonical index;
* counting DP  C_m[U] = sum over finite options of C_{m-1}[U - u] (exact integers).
"""
from __future__ import annotations

import numpy as np

INF32 = np.float32(np.inf)


def _step(V: np.ndarray, tau_m: np.ndarray, u_m: np.ndarray, B: int) -> np.ndarray:
    """One knapsack layer: W[U] = min_k fl32(V[U - u_k] + tau_k) over finite options."""
    W = np.full(B + 1, INF32, dtype=np.float32)
    for t, u in zip(tau_m, u_m):
        if not np.isfinite(t) or u > B:
            continue
        cand = (V[: B + 1 - u] + np.float32(t)).astype(np.float32)  # binary32 RNE
        np.minimum(W[u:], cand, out=W[u:])
    return W


def best_value(tau: np.ndarray, u: np.ndarray, B: int, start: float | None = None, start_units: int = 0,
               first: int = 0) -> np.float32:
    """Minimal canonical FP32 objective over LLMs first..M-1, from a partial sum `start` (None = empty)."""
    M = tau.shape[0]
    if start is None:
        V = np.full(B + 1, INF32, dtype=np.float32)
        m0 = first
        # first layer: the sum starts at tau_0 itself (no leading addition)
        for t, uu in zip(tau[m0], u[m0]):
            if np.isfinite(t) and uu <= B:
                V[uu] = min(V[uu], np.float32(t))
        m0 += 1
    else:
        V = np.full(B + 1, INF32, dtype=np.float32)
        if start_units > B:
            return INF32
        V[start_units] = np.float32(start)
        m0 = first
    for m in range(m0, M):
        V = _step(V, tau[m], u[m], B)
    return V.min()


def count(tau: np.ndarray, u: np.ndarray, B: int) -> int:
    """Exact number of candidates with every option finite and total units <= B."""
    C = np.zeros(B + 1, dtype=object)
    C[0] = 1
    for m in range(tau.shape[0]):
        D = np.zeros(B + 1, dtype=object)
        for t, uu in zip(tau[m], u[m]):
            if np.isfinite(t) and uu <= B:
                D[uu:] = D[uu:] + C[: B + 1 - uu]
        C = D
    return int(sum(C))


def search(tau: np.ndarray, u: np.ndarray, B: int):
    """Returns (found, value f32, lowest canonical index, feasible count)."""
    tau = np.asarray(tau, dtype=np.float32)
    u = np.asarray(u, dtype=np.int64)
    M, K = tau.shape
    cnt = count(tau, u, B)
    opt = best_value(tau, u, B)
    if not np.isfinite(opt):
        return False, float("inf"), -1, cnt
    digits = []
    S = None
    U = 0
    for m in range(M):
        chosen = None
        for k in range(K):
            t = tau[m, k]
            if not np.isfinite(t) or U + u[m, k] > B:
                continue
            S2 = np.float32(t) if S is None else np.float32(S + t)
            if S2 > opt:            # monotone: the final sum is >= every partial sum
                continue
            if m == M - 1:
                reach = S2
            else:
                reach = best_value(tau, u, B, start=S2, start_units=int(U + u[m, k]), first=m + 1)
            if reach == opt:
                chosen = k
                S, U = S2, int(U + u[m, k])
                break
        assert chosen is not None, "DFS lost the optimum"
        digits.append(chosen)
    idx = 0
    for k in digits:
        idx = idx * K + k
    return True, float(opt), idx, cnt
