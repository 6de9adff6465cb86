"""Multi-GPU plumbing: environments shard by contiguous global env-id blocks;
the only collective is an element-wise SUM of the FP64 episode statistics (a15).

One process per GPU, torch.distributed for the process group (NCCL on GPUs, gloo in the CPU
tests).  Envs never interact and every per-env random stream is keyed by the global env id
(Q20), so a shard computes exactly what a single-GPU run computes for those ids.
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def world_info() -> tuple[int, int, int]:
    """(world_size, rank, local_rank) from the torchrun environment (1, 0, 0 when absent)."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard(rank: int, world: int, envs_per_rank: int) -> tuple[int, int]:
    """Weak scaling: rank r owns global env ids [r * n, (r + 1) * n).  Returns (offset, n)."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return rank * envs_per_rank, envs_per_rank


def shard_total(rank: int, world: int, total: int) -> tuple[int, int]:
    """Strong scaling: a fixed total split into contiguous near-equal blocks.  (offset, n)."""
    lo = total * rank // world
    hi = total * (rank + 1) // world
    return lo, hi - lo


def allreduce_stats(stats: torch.Tensor, group=None) -> torch.Tensor:
    """SUM of the [8] FP64 statistics over ranks, in place (no-op without a process group)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.SUM, group=group)
    return stats


def max_over_ranks(x: float, device) -> float:
    """Max of a per-rank scalar (device timings are reported as the max over ranks)."""
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
