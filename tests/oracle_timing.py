"""CPU oracle timings on the host this runs on (SURVEY.md §8(d) "oracle beside it"): O1 brute force
single-thread on full C1/C2 and on 10^8-candidate sub-ranges of C3/C4 (4 seeded offsets), O1 on all
host cores on a C4 sub-range, and O2 (DP + lowest-index DFS + counting DP) on full C3, C4 and the
C5 sweep.  Prints one JSON line per measurement."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from oracle import dp  # noqa: E402
from workloads import generate  # noqa: E402


def emit(**kw):
    print(json.dumps(kw), flush=True)


cores = os.cpu_count() or 1
for name in ("C1", "C2"):
    d = generate.load(name)
    I = oracle.from_json(d)
    t0 = time.perf_counter()
    oracle.search(I, d["targets"][0], I.budget, threads=1)
    dt = time.perf_counter() - t0
    emit(oracle="O1", workload=name, threads=1, candidates=I.N, seconds=dt, cand_per_s=I.N / dt)
for name in ("C3", "C4"):
    d = generate.load(name)
    I = oracle.from_json(d)
    n = 10 ** 8
    rates = []
    for seed in range(4):
        lo = int(np.random.default_rng(seed).integers(0, I.N - n))
        t0 = time.perf_counter()
        oracle.search(I, d["targets"][0], I.budget, lo=lo, hi=lo + n, threads=1)
        rates.append(n / (time.perf_counter() - t0))
    emit(oracle="O1", workload=name, threads=1, candidates=n, sample="4 seeded 1e8 sub-ranges",
         cand_per_s=float(np.median(rates)))
    t0 = time.perf_counter()
    oracle.search(I, d["targets"][0], I.budget, lo=0, hi=min(I.N, 4 * 10 ** 9), threads=cores)
    dt = time.perf_counter() - t0
    emit(oracle="O1", workload=name, threads=cores, candidates=min(I.N, 4 * 10 ** 9), seconds=dt,
         cand_per_s=min(I.N, 4 * 10 ** 9) / dt)
for name in ("C3", "C4", "C5"):
    d = generate.load(name)
    I = oracle.from_json(d)
    t0 = time.perf_counter()
    for lam in d["targets"]:
        tab = oracle.option_table(I, lam)
        dp.search(tab["tau"], tab["u"], I.budget)
    dt = time.perf_counter() - t0
    emit(oracle="O2", workload=name, targets=len(d["targets"]), candidates=I.N * len(d["targets"]), seconds=dt,
         cand_per_s_equivalent=I.N * len(d["targets"]) / dt)
