"""Single-box multi-GPU plumbing for the α-entmax attention hot path.

Every (b, h) head is independent in the forward and the backward pass, so the path
shards by heads with no collective on the data path.  torch.distributed (NCCL on the GPUs, gloo
in the CPU tests) is used only for barriers, the max-over-ranks reduction of timings, and the
optional gather of results for checking.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_heads(n_heads: int, world: int, rank: int) -> range:
    """Contiguous slice of the flattened b·H + h head index owned by `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n_heads, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (timings are reported as the slowest rank)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_heads(local: torch.Tensor, n_heads: int, device=None) -> torch.Tensor | None:
    """Gather per-rank head slices [n_local, ...] into [n_heads, ...] on rank 0 (checking only)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return local
    world, rank = dist.get_world_size(), dist.get_rank()
    sizes = [len(shard_heads(n_heads, world, r)) for r in range(world)]
    parts = [torch.empty((s,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device) for s in sizes]
    dist.all_gather(parts, local.contiguous())
    return torch.cat(parts, 0) if rank == 0 else None


def imbalance(per_rank_ms) -> float:
    """max/mean of the per-rank step times (1.0 = perfectly balanced; heads of different block
    density make the ranks' work differ)."""
    t = [float(x) for x in per_rank_ms]
    return max(t) / (sum(t) / len(t))
