"""Multi-GPU sweep sharding: one process per GPU (torch.distributed), NCCL over NVLink.

The metric pass is replicated on every rank (no exchange: SURVEY.md §8e,
"replicas only" for the class tables). The candidate sweep is split into
contiguous class ranges balanced by cost (`plan_shards`, the GPU analogue of
the reference's plan_partition, parallel.hpp:28-41). Because ranks own
ascending class ranges and each rank's records are already in
(origin, method, destination) order, concatenating the per-rank lists in rank
order IS suggest_all's ordered list (suggest.hpp:344-348): one all-gather of
the counts, one all-gather of the count-padded 64-byte records — NCCL has no
all-gather-v — then a slice-and-concatenate.
"""
from __future__ import annotations

from typing import List, Tuple

import torch
import torch.distributed as dist

RECORD_BYTES = 64


def shard_range(bounds, rank: int) -> Tuple[int, int]:
    return int(bounds[rank]), int(bounds[rank + 1])


def allgather_records(local: torch.Tensor, n_local: int, group=None) -> Tuple[torch.Tensor, List[int]]:
    """All-gather variable-size record lists (uint8 tensors of n*64 bytes).

    Works for any backend whose all_gather_into_tensor supports the tensor's
    device (NCCL on CUDA tensors, gloo on CPU tensors). Returns the rank-order
    concatenation and the per-rank counts."""
    world = dist.get_world_size(group)
    dev = local.device
    cnt = torch.tensor([n_local], dtype=torch.int64, device=dev)
    cnts = torch.empty(world, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(cnts, cnt, group=group)
    counts = [int(c) for c in cnts.tolist()]
    mx = max(counts) if counts else 0
    if mx == 0:
        return torch.empty(0, dtype=torch.uint8, device=dev), counts
    send = torch.zeros(mx * RECORD_BYTES, dtype=torch.uint8, device=dev)
    if n_local:
        send[: n_local * RECORD_BYTES] = local[: n_local * RECORD_BYTES]
    recv = torch.empty(world * mx * RECORD_BYTES, dtype=torch.uint8, device=dev)
    dist.all_gather_into_tensor(recv, send, group=group)
    parts = [recv[r * mx * RECORD_BYTES:(r * mx + counts[r]) * RECORD_BYTES] for r in range(world)]
    return torch.cat(parts), counts


def device_records_tensor(ptr: int, n: int, device) -> torch.Tensor:
    """Zero-copy uint8 view of n mm_suggestion records in libmmgpu's device buffer."""

    class _View:
        __cuda_array_interface__ = {"shape": (n * RECORD_BYTES,), "typestr": "|u1", "data": (ptr, False),
                                    "version": 3, "strides": None}

    if n == 0:
        return torch.empty(0, dtype=torch.uint8, device=device)
    return torch.as_tensor(_View(), device=device)
