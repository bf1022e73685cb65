"""Multi-GPU search: the candidate work items are split into contiguous per-rank ranges
(alp_shard_range), every rank runs the search kernel on its range, and the per-rank results are
combined over NVLink:

* exchange="peer" (the fused path): the search kernel's last block on every rank writes its
  (key, count, local result) rows into every rank's exchange buffer through peer memory and reduces
  them itself (alp_search_peer) — no collective, no finalize launch.  The buffers are shared once
  per process group by CUDA IPC handles sent over the group (PeerExchange).
* exchange="nccl": ONE all-gather of the 16-byte (key, count) pairs (the finalize kernel takes MIN
  of the keys and SUM of the counts itself, alp_finalize_gathered), or two all-reduces (MIN over
  int64 keys, SUM over int64 counts; every key < 2^63) and alp_finalize.

PyTorch owns the device memory, the stream and the process group; the kernels are the library's.
Keys carry the global segment id, so the result is independent of the split.
"""
from __future__ import annotations

from typing import Sequence

import torch
import torch.distributed as dist

from . import ALP_ENCCL, Alp, AlpError, PeerBuffer, Result


def reduce_keys(keys: torch.Tensor, counts: torch.Tensor, group=None) -> None:
    """In-place cross-rank reduction of per-target (key, count) pairs (no-op for world size 1)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    try:
        dist.all_reduce(keys, op=dist.ReduceOp.MIN, group=group)
        dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    except (RuntimeError, dist.DistBackendError) as e:
        raise AlpError(ALP_ENCCL, f"all-reduce of the (key, count) pairs failed: {e}") from e


def gather_pairs(pairs: torch.Tensor, gathered: torch.Tensor, group=None) -> int:
    """One all-gather of this rank's int64[2n] (keys, counts) into int64[world][2n]; returns world.
    Without a process group (or world size 1) the pairs are copied through."""
    if not dist.is_available() or not dist.is_initialized():
        gathered[: pairs.numel()].copy_(pairs)
        return 1
    world = dist.get_world_size(group)  # world 1 still runs the collective (one code path)
    try:
        if dist.get_backend(group) == "nccl":
            dist.all_gather_into_tensor(gathered, pairs, group=group)
        else:  # gloo (CPU tests, several ranks on one GPU): list form
            dist.all_gather(list(gathered[: world * pairs.numel()].view(world, -1).unbind(0)), pairs, group=group)
    except (RuntimeError, dist.DistBackendError) as e:  # NCCL / gloo failure -> the library's status
        raise AlpError(ALP_ENCCL, f"all-gather of the (key, count) pairs failed: {e}") from e
    return world


class PeerExchange:
    """The exchange buffers of the fused peer exchange for one process group and up to n_targets
    targets per call: this rank's own buffer (alp_peer_alloc on the current device) and every other
    rank's, mapped through the CUDA IPC handles all-gathered over the group (any backend: gloo
    works, so the handles travel even where NCCL would not).  Every rank of the group must use it
    for the same sequence of searches (alp_search_peer counts exchanges)."""

    def __init__(self, n_targets: int, group=None):
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.n_targets = n_targets
        self.own = PeerBuffer.alloc(n_targets, self.world)
        self._mapped: list[PeerBuffer] = []
        ptrs = []
        if self.world > 1:
            handles: list = [None] * self.world
            dist.all_gather_object(handles, self.own.ipc_handle(), group=group)
            for j, h in enumerate(handles):
                if j == self.rank:
                    ptrs.append(self.own.ptr)
                else:
                    b = PeerBuffer.from_ipc(h)
                    self._mapped.append(b)
                    ptrs.append(b.ptr)
        else:
            ptrs.append(self.own.ptr)
        self.ptrs = ptrs

    def close(self):
        for b in self._mapped:
            b.close()
        self._mapped = []
        self.own.close()


def search_peer(alp: Alp, targets: Sequence[float], budget: int, px: PeerExchange,
                stream: torch.cuda.Stream | None = None) -> list[Result]:
    """Every rank searches its shard and the kernels reduce across ranks over peer memory
    (alp_search_peer); identical results on all ranks."""
    lo, hi = alp.shard_range(budget, px.rank, px.world)
    st = stream or torch.cuda.current_stream()
    ws = workspace(alp, len(targets))
    return alp.search_peer(targets, budget, lo, hi, px.rank, px.ptrs, st.cuda_stream, ws.data_ptr())


def search_distributed(alp: Alp, targets: Sequence[float], budget: int, group=None,
                       stream: torch.cuda.Stream | None = None, exchange: str = "nccl",
                       peer: PeerExchange | None = None) -> list[Result]:
    """Every rank searches its shard; the (key, count) pairs are combined by one all-gather and the
    finalize kernel (exchange="nccl"), or inside the search kernel over peer memory
    (exchange="peer", with `peer` or a PeerExchange created and cached on the handle).  Identical
    results on all ranks."""
    if exchange == "peer":
        if peer is None:
            cache = alp.__dict__.setdefault("_peer", {})
            peer = cache.get(len(targets))
            if peer is None:
                peer = cache[len(targets)] = PeerExchange(len(targets), group)
        return search_peer(alp, targets, budget, peer, stream)
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    lo, hi = alp.shard_range(budget, rank, world)
    st = stream or torch.cuda.current_stream()
    n = len(targets)
    pairs = torch.empty(2 * n, dtype=torch.int64, device="cuda")
    gathered = torch.empty(world * 2 * n, dtype=torch.int64, device="cuda")
    ws = workspace(alp, n)
    with torch.cuda.stream(st):
        alp.search_shard(targets, budget, lo, hi, pairs.data_ptr(), pairs.data_ptr() + 8 * n, st.cuda_stream,
                         ws.data_ptr())
        w = gather_pairs(pairs, gathered, group)
        return alp.finalize_gathered(targets, budget, gathered.data_ptr(), w, st.cuda_stream, ws.data_ptr())


def workspace(alp: Alp, n: int) -> torch.Tensor:
    """A torch-owned, zero-filled caller workspace for n targets (alp_workspace_bytes), cached on the
    handle: every call leaves its control section zero, so it is reused without clearing."""
    cache = alp.__dict__.setdefault("_workspaces", {})
    ws = cache.get(n)
    if ws is None:
        ws = torch.zeros(alp.workspace_bytes(n), dtype=torch.uint8, device="cuda")
        cache[n] = ws
    return ws
