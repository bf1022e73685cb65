"""Per-rank cost of a sharded C4 search, measured on ONE GPU: for world w = 1, 2, 4, 8 the rank-0
shard (1/w of the work items) is searched and finalized on its own (no all-reduce) — the device
work one B200 does in a w-GPU run.  NCCL all-reduce time (16 B per target) is not included."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_15186_b200 as P  # noqa: E402
from workloads import generate  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
d = generate.load(name)
alp = P.Alp.from_instance(d)
B, t = d["budget_units"], list(d["targets"])
keys = torch.empty(len(t), dtype=torch.int64, device="cuda")
cnts = torch.empty(len(t), dtype=torch.int64, device="cuda")
st = torch.cuda.Stream()
out = []
for world in (1, 2, 4, 8):
    lo, hi = alp.shard_range(B, 0, world)
    ks, ss = [], []
    for rep in range(23):
        with torch.cuda.stream(st):
            alp.search_shard(t, B, lo, hi, keys.data_ptr(), cnts.data_ptr(), st.cuda_stream)
            alp.finalize(t, B, keys.data_ptr(), cnts.data_ptr(), st.cuda_stream)
        torch.cuda.synchronize()
        if rep >= 3:
            ks.append(alp.last_kernel_ms)
            ss.append(alp.last_step_ms)  # library events: search start .. result D2H complete
    k, s = sorted(ks)[len(ks) // 2], sorted(ss)[len(ss) // 2]
    out.append({"workload": name, "world": world, "items": hi - lo, "kernel_ms": k, "step_ms_no_allreduce": s,
                "projected_cand_per_s": alp.num_candidates * len(t) / (s * 1e-3)})
    print(json.dumps(out[-1]))
