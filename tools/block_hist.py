"""Per-warp timeline of k_search_u for one shard (ALP_DBG_TS=1 + ALP_DBG_DUMP): loop-end time
against the number of tickets each warp took, and the SM-level spread (blocks -> SM via
%smid is not recorded; blocks are grouped by index mod SM count, the launch order).

    python tools/block_hist.py C4 8 0      # workload, world, rank
"""
import collections
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
name, world, rank = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
dump = f"/tmp/alp_dbg_{os.getpid()}.bin"
os.environ["ALP_DBG_TS"] = "1"
os.environ["ALP_DBG_DUMP"] = dump
import torch  # noqa: E402

import paper_2604_15186_b200 as P  # noqa: E402
from workloads import generate  # noqa: E402

d = generate.load(name)
alp = P.Alp.from_instance(d)
B, t = d["budget_units"], list(d["targets"])
keys = torch.empty(len(t), dtype=torch.int64, device="cuda")
cnts = torch.empty(len(t), dtype=torch.int64, device="cuda")
lo, hi = alp.shard_range(B, rank, world)
mode = os.environ.get("SHARD_MODE", "nccl")
buf = P.PeerBuffer.alloc(len(t), 1) if mode == "peer" else None
for rep in range(4):
    if os.path.exists(dump):
        os.remove(dump)
    if mode == "peer":
        alp.search_peer(t, B, lo, hi, 0, [buf.ptr])
    else:
        alp.search_shard(t, B, lo, hi, keys.data_ptr(), cnts.data_ptr(), torch.cuda.current_stream().cuda_stream)
        alp.finalize(t, B, keys.data_ptr(), cnts.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
ts = np.fromfile(dump, dtype=np.uint64).reshape(-1, 8)
ep = ts[-2].astype(np.int64)  # peer epilogue phase stamps (extra rows)
fz = ts[-1].astype(np.int64)  # finalize phase stamps
ts = ts[:-2]
g = ts.shape[0]
t0 = ts[:, 0].min()
rel = lambda c: (ts[:, c].astype(np.int64) - int(t0)) / 1e3
start, tables, lend, end = rel(0), rel(1), rel(2), rel(3)
tk = ts[:, 6].astype(np.int64)
tk[0] = -1
print(f"[{mode}] {name} world {world} rank {rank}: grid {g}, items {hi - lo}, kernel span {end.max():.1f} us, "
      f"tables med {np.median(tables):.1f}, loop-end min/med/p90/max {lend.min():.1f}/{np.median(lend):.1f}/"
      f"{np.percentile(lend, 90):.1f}/{lend.max():.1f}")
by = collections.defaultdict(list)
for b in range(1, g):
    by[int(tk[b])].append(lend[b])
for k in sorted(by):
    v = np.array(by[k])
    print(f"  tickets {k:3d}: warps {len(v):5d}  loop-end min {v.min():6.1f} med {np.median(v):6.1f} max {v.max():6.1f}")
h = np.histogram(lend[1:], bins=20)
print("  loop-end histogram:", " ".join(f"{int(e):d}:{c}" for c, e in zip(h[0], h[1])))
CLK = 1.965e3  # SM cycles per us (clocks.max.sm; the epilogue stamps are clock64 on one SM)
if ep[0]:
    print("  peer epilogue phases (us):", " ".join(f"{(ep[i + 1] - ep[i]) / CLK:.2f}" for i in range(5)),
          "| local finalize, rows, fence + flags, wait for all flags, reduce + result")
if fz[0]:
    print("  finalize phases (us):", " ".join(f"{(fz[i + 1] - fz[i]) / CLK:.2f}" for i in range(4)),
          "| stage + digits + row terms, re-scan, winner terms, result stored")
