"""Randomised parity sweep of the CUDA path against the oracle (more cases than the test suite):
seeded random instances (2-8 LLMs, 1-48 options per LLM, random budgets, memory floors on a third
of them), three targets each plus one batch and one per-query-budget call of 2-19 targets, a
one-target budget sweep of 2-11 budgets (the one-pass k_search_levels; infeasible budgets also
check the SPEC.md:374 fallback against its brute-force definition on small spaces) and a
one-rank peer exchange; every result against the DP oracle (O2) and, for the single searches in
small spaces, the brute-force oracle (O1).  Run once per launch path:

    python tests/sweep_parity.py [n_instances] [seed0]            # default path choice
    ALP_NO_UR=1 python tests/sweep_parity.py ...                  # fused k_search
    ALP_NO_FUSED=1 python tests/sweep_parity.py ...               # K1 + K2 + K3
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (test infrastructure: this is a checking tool)
from oracle import dp  # noqa: E402
import paper_2604_15186_b200 as P  # noqa: E402
from workloads import generate  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 90000
    ok = bad = brute = 0
    paths = {}
    for s in range(seed0, seed0 + n):
        rng = np.random.default_rng(s)
        S = sorted(set(int(x) for x in rng.integers(1, 9, size=int(rng.integers(1, 5)))))
        T = [1, 2, 4, 8][: int(rng.integers(1, 5))]
        R = list(range(1, int(rng.integers(2, 5))))
        K = len(S) * len(T) * len(R)
        M = int(rng.integers(2, 9))
        while K ** M > 3e10:
            M -= 1
        if M < 2:
            continue
        budget = int(rng.integers(1, 8 * M * 4))
        d = generate.random_instance(s, M=M, F=8, S=S, T=T, R=R, budget=budget, points=int(rng.integers(2, 7)),
                                     min_units=bool(s % 3 == 0))
        I = oracle.from_json(d)
        alp = P.Alp.from_instance(d)
        for lam in (float(rng.uniform(0.01, 0.2)), float(rng.uniform(0.2, 1.0)), float(rng.uniform(1.0, 4.0))):
            r = alp.search(lam, budget)
            paths[alp.last_path] = paths.get(alp.last_path, 0) + 1
            tab = oracle.option_table(I, lam)
            f, v, idx, cnt = dp.search(tab["tau"], tab["u"], budget)
            good = (r.found == f and r.feasible_count == cnt and
                    (not f or (r.index == idx and np.float32(r.latency_key) == np.float32(v))))
            if I.N <= 2_000_000:
                o = oracle.search(I, lam, budget, threads=8)
                brute += 1
                good = good and o.found == r.found and o.count == r.feasible_count and (
                    not o.found or (o.index == r.index and o.latency_key == r.latency_key))
            if good:
                ok += 1
            else:
                bad += 1
                print("MISMATCH", s, lam, budget, r.index, idx, r.feasible_count, cnt, flush=True)
        # a batch (uniform-register groups of <= 8 targets) and per-query budgets, vs the DP oracle
        lams = [float(x) for x in rng.uniform(0.01, 4.0, size=int(rng.integers(2, 20)))]
        buds = [int(x) for x in rng.integers(0, 8 * M * 4, size=len(lams))]
        for kind, res in (("batch", alp.search_batch(lams, budget)), ("queries", alp.search_queries(lams, buds))):
            paths[kind] = paths.get(kind, 0) + len(lams)
            for j, (lam, r) in enumerate(zip(lams, res)):
                bj = budget if kind == "batch" else buds[j]
                tab = oracle.option_table(I, lam)
                f, v, idx, cnt = dp.search(tab["tau"], tab["u"], bj)
                good = (r.found == f and r.feasible_count == cnt and
                        (not f or (r.index == idx and np.float32(r.latency_key) == np.float32(v))))
                if good:
                    ok += 1
                else:
                    bad += 1
                    print("MISMATCH", kind, s, lam, bj, r.index, idx, r.feasible_count, cnt, flush=True)
        # one target, several budgets: the one-pass budget sweep (k_search_levels), vs the DP oracle
        lam = float(rng.uniform(0.05, 2.0))
        sweep = sorted(int(x) for x in rng.integers(0, 8 * M * 4, size=int(rng.integers(2, 12))))
        paths["sweep"] = paths.get("sweep", 0) + len(sweep)
        tab = oracle.option_table(I, lam)
        for bj, r in zip(sweep, alp.search_queries([lam] * len(sweep), sweep)):
            f, v, idx, cnt = dp.search(tab["tau"], tab["u"], bj)
            good = (r.found == f and r.feasible_count == cnt and
                    (not f or (r.index == idx and np.float32(r.latency_key) == np.float32(v))))
            if not f and I.N <= 2_000_000:  # the SPEC.md:374 fallback vs its brute-force definition
                fb = oracle.max_throughput(I, bj) if I.N <= 200_000 else None
                if fb is not None or I.N <= 200_000:
                    good = good and (r.fallback == (fb is not None)) and (
                        fb is None or (r.index == fb["index"] and r.throughput == fb["throughput"]))
            if good:
                ok += 1
            else:
                bad += 1
                print("MISMATCH sweep", s, lam, bj, r.index, idx, r.feasible_count, cnt, flush=True)
        # the fused peer exchange with one rank over the whole range (search + in-kernel reduction)
        if not hasattr(main, "_buf"):
            main._buf = P.PeerBuffer.alloc(1, 1)
        lo, hi = alp.shard_range(budget, 0, 1)
        try:
            r = alp.search_peer([lam], budget, lo, hi, 0, [main._buf.ptr])[0]
            f, v, idx, cnt = dp.search(tab["tau"], tab["u"], budget)
            good = (r.found == f and r.feasible_count == cnt and
                    (not f or (r.index == idx and np.float32(r.latency_key) == np.float32(v))))
            paths["peer"] = paths.get("peer", 0) + 1
            if good:
                ok += 1
            else:
                bad += 1
                print("MISMATCH peer", s, lam, budget, r.index, idx, r.feasible_count, cnt, flush=True)
        except P.AlpError:  # not a fused-size problem: the peer exchange does not apply
            paths["peer_n/a"] = paths.get("peer_n/a", 0) + 1
    print({"instances": n, "searches": ok + bad, "match": ok, "mismatch": bad, "also_brute_force": brute,
           "paths": paths, "env": {k: v for k, v in os.environ.items() if k.startswith("ALP_")}})


if __name__ == "__main__":
    main()
