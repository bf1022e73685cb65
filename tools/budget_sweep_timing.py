"""One-pass budget-indexed search vs per-budget passes (NEXT-1): C4, one target, the best
allocation on 0..G whole GPUs (F = 2), device step time (alp_last_step_ms) and host time.

    python tools/budget_sweep_timing.py [G]        # ALP_NO_LEVELS=1 for the per-budget passes
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_15186_b200 as P  # noqa: E402
from workloads import generate  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 64
d = generate.load("C4")
alp = P.Alp.from_instance(d)
lam = d["targets"][0]
budgets = [2 * g for g in range(G + 1)]
alp.search_queries([lam] * len(budgets), budgets)
ts, hs = [], []
for _ in range(5):
    t0 = time.perf_counter()
    res = alp.search_queries([lam] * len(budgets), budgets)
    hs.append(1e3 * (time.perf_counter() - t0))
    ts.append(alp.last_step_ms)
print(json.dumps({"workload": "C4", "budgets": len(budgets), "mode": "per-budget" if os.environ.get("ALP_NO_LEVELS") else "one-pass",
                  "step_ms": sorted(ts)[2], "host_ms": sorted(hs)[2], "launches": alp.last_launches,
                  "best_64gpu_index": res[-1].index, "feasible_64gpu": res[-1].feasible_count}))
