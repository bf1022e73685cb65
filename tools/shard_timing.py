"""Per-rank cost of a sharded search, measured on ONE GPU: for world w = 1, 2, 4, 8 every rank's
shard (1/w of the work items) is searched and finalized on its own (no collective) — the device
work one B200 does in a w-GPU run.  Reports the rank-0 and the slowest rank's step (a w-GPU step
waits for the slowest rank) and the projected whole-job rate N / max step.  The exchange between
ranks (NCCL all-gather + K3, or the peer exchange) is not included.

    python tools/shard_timing.py [C4|C3] [worlds, e.g. 1,8] [reps]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_15186_b200 as P  # noqa: E402
from workloads import generate  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
worlds = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 2, 4, 8]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
d = generate.load(name)
alp = P.Alp.from_instance(d)
B, t = d["budget_units"], list(d["targets"])
keys = torch.empty(len(t), dtype=torch.int64, device="cuda")
cnts = torch.empty(len(t), dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.Stream()
mode = os.environ.get("SHARD_MODE", "nccl")  # nccl: shard search + K3 finalize; peer: alp_search_peer (1-rank exchange)
buf = P.PeerBuffer.alloc(len(t), 1) if mode == "peer" else None
ref = alp.search_batch(t, B)[-1]
for world in worlds:
    per = []
    for rank in range(world):
        lo, hi = alp.shard_range(B, rank, world)
        ks, ss = [], []
        for rep in range(reps + 3):
            with torch.cuda.stream(st):
                if not os.environ.get("NO_FLUSH"):
                    flush.zero_()
                if mode == "peer":  # search + in-kernel exchange (with itself) over the rank's range
                    alp.search_peer(t, B, lo, hi, 0, [buf.ptr], st.cuda_stream)
                else:
                    alp.search_shard(t, B, lo, hi, keys.data_ptr(), cnts.data_ptr(), st.cuda_stream)
                    alp.finalize(t, B, keys.data_ptr(), cnts.data_ptr(), st.cuda_stream)
            torch.cuda.synchronize()
            if rep >= 3:
                ks.append(alp.last_kernel_ms)
                ss.append(alp.last_step_ms)  # library events: search start .. result on the host
        per.append((sorted(ks)[len(ks) // 2], sorted(ss)[len(ss) // 2], hi - lo))
    kmax = max(p[0] for p in per)
    smax = max(p[1] for p in per)
    out = {"workload": name, "world": world, "items_rank0": per[0][2], "kernel_ms_rank0": per[0][0],
           "step_ms_rank0": per[0][1], "kernel_ms_max": kmax, "step_ms_max": smax,
           "slowest_rank": max(range(world), key=lambda r: per[r][1]),
           "projected_cand_per_s": alp.num_candidates * len(t) / (smax * 1e-3),
           "mode": mode}
    print(json.dumps(out), flush=True)
