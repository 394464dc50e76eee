"""Multi-GPU sweep sharding: one process per GPU (torch.distributed), NCCL over NVLink.

The metric pass is replicated on every rank (no exchange: SURVEY.md §8e,
"replicas only" for the class tables). The candidate sweep is split into
contiguous class ranges balanced by cost (`plan_shards`, the GPU analogue of
the reference's plan_partition, parallel.hpp:28-41). Because ranks own
ascending class ranges and each rank's records are already in
(origin, method, destination) order, concatenating the per-rank lists in rank
order IS suggest_all's ordered list (suggest.hpp:344-348). The exchange moves
exact counts, no padding: one all-gather of the per-rank record counts
(8 bytes each), then one broadcast per non-empty rank of exactly its records
straight into their slice of the assembled list (NCCL has no all-gather-v;
the same protocol mm_group_sweep runs in-process, include/mmgpu.h).
"""
from __future__ import annotations

from typing import List, Tuple

import torch
import torch.distributed as dist

RECORD_BYTES = 64


def shard_range(bounds, rank: int) -> Tuple[int, int]:
    return int(bounds[rank]), int(bounds[rank + 1])


def record_offsets(counts: List[int]) -> List[int]:
    """Exclusive prefix of the per-rank counts: where each rank's list starts."""
    out, acc = [], 0
    for c in counts:
        out.append(acc)
        acc += int(c)
    return out


def allgather_records(local: torch.Tensor, n_local: int, group=None, out: torch.Tensor = None
                      ) -> Tuple[torch.Tensor, List[int]]:
    """All-gather variable-size record lists (uint8 tensors of n*64 bytes) with
    exact counts: all-gather the counts, then every non-empty rank broadcasts
    exactly its records into their slice of the assembled buffer (no padding).

    Works for any backend with all_gather_into_tensor and broadcast on the
    tensor's device (NCCL on CUDA tensors, gloo on CPU tensors). Returns the
    rank-order concatenation and the per-rank counts."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = local.device
    cnt = torch.tensor([n_local], dtype=torch.int64, device=dev)
    cnts = torch.empty(world, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(cnts, cnt, group=group)
    counts = [int(c) for c in cnts.tolist()]
    offs = record_offsets(counts)
    total = sum(counts)
    if out is None or out.numel() < total * RECORD_BYTES:
        out = torch.empty(total * RECORD_BYTES, dtype=torch.uint8, device=dev)
    res = out[: total * RECORD_BYTES]
    if n_local:
        a = offs[rank] * RECORD_BYTES
        res[a: a + n_local * RECORD_BYTES].copy_(local[: n_local * RECORD_BYTES])
    works = []
    for r in range(world):
        if counts[r] == 0:
            continue
        a = offs[r] * RECORD_BYTES
        works.append(dist.broadcast(res[a: a + counts[r] * RECORD_BYTES],
                                    src=dist.get_global_rank(group, r) if group is not None else r,
                                    group=group, async_op=True))
    for w in works:
        w.wait()
    return res, counts


def device_records_tensor(ptr: int, n: int, device) -> torch.Tensor:
    """Zero-copy uint8 view of n mm_suggestion records in libmmgpu's device buffer."""

    class _View:
        __cuda_array_interface__ = {"shape": (n * RECORD_BYTES,), "typestr": "|u1", "data": (ptr, False),
                                    "version": 3, "strides": None}

    if n == 0:
        return torch.empty(0, dtype=torch.uint8, device=device)
    return torch.as_tensor(_View(), device=device)
