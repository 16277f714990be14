"""Sequence sharding for one process per GPU ("balanced workload ... across all
parallel workers").  Units (sequence, kv head) are independent, so rank r owns whole sequences and the
decode step needs no collective; torch.distributed (NCCL on GPUs, gloo in the CPU tests) is used only
to gather outputs / slots and to reduce statistics after the timed region."""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env():
    """(world_size, rank, local_rank) from the torchrun environment (1, 0, 0 when absent)."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard(batch: int, world: int, rank: int, scaling: str = "weak"):
    """Sequences of this rank: returns (B_local, b0, B_total).

    weak   -- every rank holds `batch` sequences (global batch = batch * world)
    strong -- the `batch` sequences are split evenly (batch % world == 0 required)"""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if scaling == "weak":
        return batch, rank * batch, batch * world
    if scaling != "strong":
        raise ValueError(f"unknown scaling {scaling!r}")
    if batch % world:
        raise ValueError(f"batch {batch} not divisible by {world} ranks")
    b = batch // world
    return b, rank * b, batch


def gather_rows(t: torch.Tensor) -> torch.Tensor:
    """All-gather equal shards along dim 0 (rank order) -> the full-batch tensor on every rank."""
    world = dist.get_world_size()
    if dist.get_backend() != "nccl":   # gloo (CPU tests): list form
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t.contiguous())
        return torch.cat(parts, dim=0)
    out = torch.empty((world * t.shape[0], *t.shape[1:]), dtype=t.dtype, device=t.device)
    dist.all_gather_into_tensor(out, t.contiguous())
    return out


def max_over_ranks(x: float, device=None) -> float:
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
