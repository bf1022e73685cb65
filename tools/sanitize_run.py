"""Small searches for compute-sanitizer (memcheck / racecheck / synccheck): hand case, C1 (fused
single launch and, with ALP_NO_FUSED, K1 + K2 + K3), a two-LLM slice of the C3 grid (K = 512:
b-chunked masked tables), a target batch, budget queries, a sharded search on a caller stream
with a device finalize, injected terms, the one-pass budget sweep, the infeasible fallback, a
peer exchange of 2 logical ranks (one host thread each) on the hand case, a cold plan build
(device tile_off expansion), and (SANITIZE_C4=1) the full C4 headline search."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_15186_b200 as P  # noqa: E402
from workloads import generate  # noqa: E402

for fused in (True, False):
    if not fused:
        os.environ["ALP_NO_FUSED"] = "1"
    for name in ("hand", "C1"):
        d = generate.load(name)
        r = P.Alp.from_instance(d).search(d["targets"][0], d["budget_units"])
        print(name, "fused" if fused else "classic", r.index, r.feasible_count)
    os.environ.pop("ALP_NO_FUSED", None)
d = json.loads(json.dumps(generate.load("C3")))
for k in ("n", "p", "profiles"):
    d[k] = d[k][:2]
d["M"] = 2
alp = P.Alp.from_instance(d)
print("C3x2", alp.search(d["targets"][0], 128).index, alp.search_batch([d["targets"][0], 1.0, 3.0], 64)[0].index)
print("queries", [r.index for r in alp.search_queries([d["targets"][0]] * 3, [0, 40, 128])])
# shard path on a caller stream: 3 shards, torch-side reduction, device finalize (PDL K3)
d = generate.load("C1")
alp = P.Alp.from_instance(d)
B, lam = d["budget_units"], [d["targets"][0]]
st = torch.cuda.Stream()
keys = torch.empty((3, 1), dtype=torch.int64, device="cuda")
cnts = torch.empty((3, 1), dtype=torch.int64, device="cuda")
for rank in range(3):
    lo, hi = alp.shard_range(B, rank, 3)
    alp.search_shard(lam, B, lo, hi, keys[rank].data_ptr(), cnts[rank].data_ptr(), st.cuda_stream)
st.synchronize()
k = keys.min(dim=0).values.contiguous()
c = cnts.sum(dim=0).contiguous()
print("shards", alp.finalize(lam, B, k.data_ptr(), c.data_ptr())[0].index)
# one-all-gather exchange layout: per-rank int64[2n] rows, reduced inside K3
g = torch.empty(3 * 2, dtype=torch.int64, device="cuda")
for rank in range(3):
    lo, hi = alp.shard_range(B, rank, 3)
    alp.search_shard(lam, B, lo, hi, g[2 * rank:].data_ptr(), g[2 * rank + 1:].data_ptr(), st.cuda_stream)
st.synchronize()
print("gathered", alp.finalize_gathered(lam, B, g.data_ptr(), 3)[0].index)
tau = (np.arange(24, dtype=np.float32).reshape(3, 8) % 5 + 1) / 8
u = (np.arange(24, dtype=np.int32).reshape(3, 8) % 3)
print("terms", P.Alp.from_terms(tau, u).search(1.0, 4).index)
# uniform-register path: a batch of 12 targets on the hand case (groups of 8 + 4)
d = generate.load("hand")
alp = P.Alp.from_instance(d)
print("ur batch", [r.index for r in alp.search_batch([0.125 * (i + 1) for i in range(12)], d["budget_units"])])
# one-pass budget sweep (levels kernel + finish + K3 per budget) and the fallback kernel
d = generate.load("C1")
alp = P.Alp.from_instance(d)
print("sweep", [r.index for r in alp.search_queries([d["targets"][0]] * 5, [0, 3, 8, 12, 16])])
print("fallback", alp.search(1e6, 16).index, alp.search_queries([1e6] * 2, [4, 16])[1].index)
# peer exchange: 2 logical ranks, a host thread each, own handle / workspace / stream / buffer
import threading  # noqa: E402
d = generate.load("hand")
alps = [P.Alp.from_instance(d) for _ in range(2)]
bufs = [P.PeerBuffer.alloc(1, 2) for _ in range(2)]
wss = [torch.zeros(a.workspace_bytes(1), dtype=torch.uint8, device="cuda") for a in alps]
sts = [torch.cuda.Stream() for _ in range(2)]
outp = [None, None]


def _rank(r):
    torch.cuda.set_device(0)
    lo, hi = alps[r].shard_range(d["budget_units"], r, 2)
    outp[r] = alps[r].search_peer(d["targets"][:1], d["budget_units"], lo, hi, r, [b.ptr for b in bufs],
                                  sts[r].cuda_stream, wss[r].data_ptr())[0].index


ths = [threading.Thread(target=_rank, args=(r,)) for r in range(2)]
for t in ths:
    t.start()
for t in ths:
    t.join()
print("peer", outp)
P.plan_cache_clear()
print("cold", P.Alp.from_instance(generate.load("C2")).search(generate.load("C2")["targets"][0], 64).index)
if os.environ.get("SANITIZE_C4"):
    d = generate.load("C4")
    r = P.Alp.from_instance(d).search(d["targets"][0], d["budget_units"])
    print("C4", r.index, r.feasible_count)
