"""Host wall time of the end-to-end pieces (median of 50 warm iterations): alp_build from host
arrays, the search (device work + result on the host), alp_destroy.

    python tools/e2e_breakdown.py [C4]
"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_15186_b200 as P  # noqa: E402
from workloads import generate  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
d = generate.load(name)
desc = P.Desc(d)
lam, B = d["targets"][0], d["budget_units"]
t = {"build": [], "search": [], "close": [], "search_warm_handle": []}
keep = P.Alp.build(desc)
for i in range(60):
    t0 = time.perf_counter()
    a = P.Alp.build(desc)
    t1 = time.perf_counter()
    a.search_batch([lam], B)
    t2 = time.perf_counter()
    a.close()
    t3 = time.perf_counter()
    keep.search_batch([lam], B)
    t4 = time.perf_counter()
    if i >= 10:
        t["build"].append(t1 - t0)
        t["search"].append(t2 - t1)
        t["close"].append(t3 - t2)
        t["search_warm_handle"].append(t4 - t3)
print(name, {k: round(statistics.median(v) * 1e3, 4) for k, v in t.items()}, "ms (median)",
      "device step", round(keep.last_step_ms, 4))
