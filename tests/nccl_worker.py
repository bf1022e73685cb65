"""Worker for tests/test_gpu_parity.py::test_nccl_search_distributed (launched by torch.distributed.run).

Every rank builds the C4 handle on its GPU (LOCAL_RANK modulo the visible devices), runs
dist.search_distributed over an NCCL process group (one all-gather of the per-rank (key, count)
pairs, then the finalize kernel), and rank 0 prints the result as one JSON line.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2604_15186_b200 as P  # noqa: E402
from paper_2604_15186_b200.dist import search_distributed  # noqa: E402
from workloads import generate  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local % torch.cuda.device_count())
    dist.init_process_group("nccl", device_id=torch.device("cuda", local % torch.cuda.device_count()))
    d = generate.load(sys.argv[1] if len(sys.argv) > 1 else "C4")
    alp = P.Alp.from_instance(d)
    targets = [d["targets"][0], 2.0 * d["targets"][0], 40.0 * d["targets"][0]]
    res = search_distributed(alp, targets, d["budget_units"])
    if dist.get_rank() == 0:
        print(json.dumps({"world": dist.get_world_size(), "backend": dist.get_backend(),
                          "results": [[r.found, r.index, r.feasible_count, r.latency_key, r.latency] for r in res]}))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
