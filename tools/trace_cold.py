"""Host-side phases of cold and warm end-to-end searches (ALP_TRACE=1 prints alp_build phases)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_15186_b200 as P  # noqa: E402
from workloads import generate  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
d = generate.load(name)
desc = P.Desc(d)
for i in range(6):
    if i in (0, 3):
        P.plan_cache_clear()
        print("-- plan cache cleared", file=sys.stderr)
    t0 = time.perf_counter()
    a = P.Alp.build(desc)
    t1 = time.perf_counter()
    r = a.search(d["targets"][0], d["budget_units"])
    t2 = time.perf_counter()
    a.close()
    t3 = time.perf_counter()
    print(f"build {1e3*(t1-t0):.3f} ms search {1e3*(t2-t1):.3f} ms destroy {1e3*(t3-t2):.3f} ms", file=sys.stderr)
