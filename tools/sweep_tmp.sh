ALP_DBG_TS=1 python - <<'PY' 2>&1 | grep "alp dbg" | tail -3
import sys; sys.path.insert(0, '.')
import paper_2604_15186_b200 as P
from workloads import generate
d = generate.load('C4'); a = P.Alp.from_instance(d)
for i in range(10): a.search(d['targets'][0], d['budget_units'])
PY
