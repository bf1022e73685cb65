"""The paper's own *pruned* GPU scheduler (§5 steps 1-3) as a comparator for the
exhaustive search: how many candidates it evaluates, how long it takes and
how far its optimum is from the exhaustive optimum over the same ALP.

Steps (prior art, re-implemented from the paper's text; details the paper leaves open follow
SPEC.md:343-378, listed in DESIGN.md §3 R16):
  1. latency ratios at the baseline allocation (tp=1, f=1, d=1), rate clamped to feasibility
     (SPEC.md:284-292, 397);
  2. enumerate GPU-fraction assignments: every LLM gets >= its minimum units, units non-increasing
     along the descending-ratio order, all units used;
  3. pack contiguously from GPU 0 in ratio order;
  4. resolve parallelism: whole-GPU spans take tp * d = #GPUs with tp <= the NVLink degree; other
     spans take tp = 1 with replicas that tile every per-GPU piece;
  5. evaluate every resulting allocation with the ALP and keep the lowest latency that meets the
     target (ties: fewer units, then enumeration order).
Predictions go through the product library (alp_predict, FP64 on the device); only allocations
that exist in the exhaustive grid (share, tp, replicas) can be evaluated and compared.
"""
from __future__ import annotations

import itertools
import math
import time
from dataclasses import dataclass, field



def count_unpruned(G: int, F: int, M: int) -> int:
    """Mappings of M LLMs to G*F GPU fractions: C(G*F + M - 1, M - 1)."""
    return math.comb(G * F + M - 1, M - 1)


def fraction_assignments(total: int, mins: list[int]):
    """Non-increasing compositions of `total` (LLMs already in descending-ratio order), part i >= mins[i].

    Ordering relaxation: when LLM i's memory minimum exceeds the previous
    (higher-ratio) LLM's part, the ordering constraint is waived for that pair (part i is then bounded
    only by the units left); the next LLM is still ordered against part i."""
    M = len(mins)

    def rec(i, left, cap):
        waived = mins[i] > cap
        if i == M - 1:
            if mins[i] <= left and (left <= cap or waived):
                yield (left,)
            return
        rest_min = sum(mins[i + 1:])
        us = range((left - rest_min) if waived else min(cap, left - rest_min), mins[i] - 1, -1)
        for u in us:
            for tail in rec(i + 1, left - u, u):
                yield (u,) + tail

    yield from rec(0, total, total)


def pack(units: tuple[int, ...], F: int):
    """Contiguous layout from GPU 0: per LLM the list of per-GPU unit pieces and whether the span
    consists of whole GPUs only."""
    out, off = [], 0
    for u in units:
        pieces, o, left = [], off, u
        while left > 0:
            take = min(left, F - o % F)
            pieces.append(take)
            o += take
            left -= take
        whole = (off % F == 0) and (u % F == 0)
        out.append((pieces, whole))
        off += u
    return out


def parallelism(pieces: list[int], whole: bool, F: int, tps, reps, shares, nvlink: int, minu: int = 1):
    """(share units, tp, d) options for one packed LLM (replica shares >= minu units)."""
    opts = []
    if whole and pieces:
        g = len(pieces)
        for tp in tps:
            if tp <= nvlink and g % tp == 0 and (g // tp) in reps and F in shares:
                opts.append((F, tp, g // tp))
    if not whole or not opts:
        tot = sum(pieces)
        for d in reps:
            if d >= 1 and tot % d == 0:
                q = tot // d
                if q >= minu and q in shares and all(p % q == 0 for p in pieces):
                    opts.append((q, 1, d))
    return sorted(set(opts))


@dataclass
class PrunedResult:
    found: bool
    latency: float
    throughput: float
    units: int
    allocation: list = field(default_factory=list)   # per LLM (share units, tp, d), input order
    assignments: int = 0
    candidates: int = 0          # allocations evaluated with the ALP
    off_grid: int = 0            # allocations the exhaustive grid cannot express (skipped)
    seconds: float = 0.0


def pruned_search(alp, d: dict, lam: float, gpus: int, nvlink: int = 8, batch: int = 1 << 16) -> PrunedResult:
    t0 = time.perf_counter()
    M, F = d["M"], d["F"]
    S, T, R = list(d["share_units"]), list(d["tp"]), list(d["replicas"])
    nT, nR = len(T), len(R)
    K = len(S) * nT * nR
    kidx = {(S[si], T[ti], R[ri]): (si * nT + ti) * nR + ri
            for si in range(len(S)) for ti in range(nT) for ri in range(nR)}
    # 1. latency ratios at the baseline allocation, rate clamped to feasibility
    tab = alp.option_table(lam, K)
    base = kidx.get((F, 1, 1))
    if base is None:
        raise ValueError("the grid needs the baseline option (share F, tp 1, d 1)")
    # (just below the smallest baseline Eq. 2 term: at b itself x may exceed T by one rounding)
    lam_ref = min(lam, 0.999999 * float(min(tab["b"][m][base] for m in range(M))))
    tref = alp.option_table(lam_ref, K)["term"][:, base]
    order = sorted(range(M), key=lambda m: (-tref[m], m))  # descending latency ratio
    mins = [1] * M
    mu = d.get("min_units")
    if mu is not None:
        mins = [max(1, int(mu[m][T.index(1)])) if 1 in T else 1 for m in order]
    res = PrunedResult(False, float("inf"), 0.0, 0)
    best_key = None
    pending, meta = [], []

    def flush():
        nonlocal best_key
        if not pending:
            return
        out = alp.predict(pending, lam, gpus * F)
        for i, (units, alloc) in enumerate(meta):
            if out["feasible"][i] and out["throughput"][i] >= lam:
                key = (out["latency"][i], units)
                if best_key is None or key < best_key:
                    best_key = key
                    res.found, res.latency, res.throughput, res.units = True, float(out["latency"][i]), \
                        float(out["throughput"][i]), int(out["units"][i])
                    res.allocation = alloc
        pending.clear()
        meta.clear()

    for assign in fraction_assignments(gpus * F, mins):
        res.assignments += 1
        layout = pack(assign, F)
        per = [parallelism(p, w, F, T, R, S, nvlink, mins[i]) for i, (p, w) in enumerate(layout)]
        for combo in itertools.product(*per):
            alloc = [None] * M
            for pos, m in enumerate(order):
                alloc[m] = combo[pos]
            ks = [kidx.get(a) for a in alloc]
            if any(k is None for k in ks):
                res.off_grid += 1
                continue
            res.candidates += 1
            pending.append(ks)
            meta.append((sum(a[0] * a[1] * a[2] for a in alloc), alloc))
            if len(pending) >= batch:
                flush()
    flush()
    res.seconds = time.perf_counter() - t0
    return res


def main():
    import argparse
    import json
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2604_15186_b200 as P
    from workloads import generate
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C3")
    args = ap.parse_args()
    for name in args.configs.split(","):
        d = generate.load(name)
        alp = P.Alp.from_instance(d)
        lam, B = d["targets"][0], d["budget_units"]
        t0 = time.perf_counter()
        ex = alp.search(lam, B)
        t_ex = time.perf_counter() - t0
        pr = pruned_search(alp, d, lam, B // d["F"])
        print(json.dumps({"config": name, "unpruned_fraction_mappings": count_unpruned(B // d["F"], d["F"], d["M"]),
                          "pruned_assignments": pr.assignments, "pruned_candidates": pr.candidates,
                          "pruned_off_grid": pr.off_grid, "pruned_seconds": pr.seconds,
                          "pruned_latency": pr.latency if pr.found else None,
                          "exhaustive_candidates": ex.candidates, "exhaustive_seconds": t_ex,
                          "exhaustive_latency": ex.latency,
                          "gap": (pr.latency / ex.latency - 1.0) if pr.found else None}))


if __name__ == "__main__":
    main()
