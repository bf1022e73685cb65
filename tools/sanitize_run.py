"""Small searches for compute-sanitizer (memcheck / racecheck / synccheck): hand case, C1, a
two-LLM slice of the C3 grid (K = 512: b-chunked masked tables, 16 rows per lane) and a target batch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json  # noqa: E402

import paper_2604_15186_b200 as P  # noqa: E402
from workloads import generate  # noqa: E402

for name in ("hand", "C1"):
    d = generate.load(name)
    r = P.Alp.from_instance(d).search(d["targets"][0], d["budget_units"])
    print(name, r.index, r.feasible_count)
d = json.loads(json.dumps(generate.load("C3")))
for k in ("n", "p", "profiles"):
    d[k] = d[k][:2]
d["M"] = 2
alp = P.Alp.from_instance(d)
print("C3x2", alp.search(d["targets"][0], 128).index, alp.search_batch([d["targets"][0], 1.0, 3.0], 64)[0].index)
print("queries", [r.index for r in alp.search_queries([d["targets"][0]] * 3, [0, 40, 128])])
