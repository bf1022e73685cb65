"""Worker for tests/test_peer_exchange.py (launched by torch.distributed.run, 127.0.0.1).

Every rank builds the handle on its GPU (LOCAL_RANK modulo the visible devices: both ranks share
one GPU on a one-GPU box), shares its exchange buffer with the other ranks by CUDA IPC handles
all-gathered over a gloo process group, and runs the fused peer exchange (alp_search_peer) for
several target sets in a row (the buffers alternate their two row slots); rank 0 prints the
results as one JSON line, every rank checks that it got the same results.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2604_15186_b200 as P  # noqa: E402
from paper_2604_15186_b200.dist import PeerExchange, search_distributed  # noqa: E402
from workloads import generate  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local % torch.cuda.device_count())
    dist.init_process_group("gloo")
    d = generate.load(sys.argv[1] if len(sys.argv) > 1 else "C4")
    alp = P.Alp.from_instance(d)
    lam = d["targets"][0]
    sets = [[lam], [lam, 2.0 * lam, 40.0 * lam], [0.5 * lam]]
    px = PeerExchange(3)
    out = []
    for targets in sets:
        res = search_distributed(alp, targets, d["budget_units"], exchange="peer", peer=px)
        out.append([[r.found, r.index, r.feasible_count, r.latency_key, r.latency, r.throughput] for r in res])
    allr = [None] * dist.get_world_size()
    dist.all_gather_object(allr, out)
    assert all(x == out for x in allr), "ranks disagree"
    if dist.get_rank() == 0:
        print(json.dumps({"world": dist.get_world_size(), "targets": sets, "results": out}))
    dist.barrier()
    px.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
