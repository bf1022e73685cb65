"""Multi-GPU search: the candidate work items are split into contiguous per-rank ranges
(alp_shard_range), every rank runs the search kernel on its range, and ONE grouped all-reduce
(MIN over int64 keys, SUM over int64 counts; every key < 2^63) combines them over NCCL /
NVLink.  PyTorch owns the device memory, the stream and the process group; the kernels are the
library's.  Keys carry the global segment id, so the result is independent of the split.
"""
from __future__ import annotations

from typing import Sequence

import torch
import torch.distributed as dist

from . import Alp, Result


def reduce_keys(keys: torch.Tensor, counts: torch.Tensor, group=None) -> None:
    """In-place cross-rank reduction of per-target (key, count) pairs (no-op for world size 1)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    dist.all_reduce(keys, op=dist.ReduceOp.MIN, group=group)
    dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)


def search_distributed(alp: Alp, targets: Sequence[float], budget: int, group=None,
                       stream: torch.cuda.Stream | None = None) -> list[Result]:
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    lo, hi = alp.shard_range(budget, rank, world)
    st = stream or torch.cuda.current_stream()
    n = len(targets)
    keys = torch.empty(n, dtype=torch.int64, device="cuda")
    counts = torch.empty(n, dtype=torch.int64, device="cuda")
    with torch.cuda.stream(st):
        alp.search_shard(targets, budget, lo, hi, keys.data_ptr(), counts.data_ptr(), st.cuda_stream)
        reduce_keys(keys, counts, group)
        return alp.finalize(targets, budget, keys.data_ptr(), counts.data_ptr(), st.cuda_stream)
