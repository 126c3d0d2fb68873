"""Multi-GPU driver pieces: one process per GPU, points sharded across ranks.

The batched HVP partitions into independent points (the paper's L0 level), so
there is no exchange step on the data path: each rank takes a contiguous range of the
global point index space (inputs are index-addressable, synth/), runs chessfad_hvp_batch on
its own GPU, and the only collectives are the max-over-ranks timing reduction and an
OPTIONAL result gather (NCCL over NVLink on GPUs; gloo in the CPU tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard(m_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous balanced shard of [0, m_total): (first, count); counts differ by <= 1."""
    if world < 1 or not 0 <= rank < world or m_total < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(m_total, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def all_shards(m_total: int, world: int) -> list[tuple[int, int]]:
    return [shard(m_total, r, world) for r in range(world)]


def max_over_ranks(x: float, device=None) -> float:
    """Max of a per-rank scalar (e.g. a CUDA-event time) over all ranks."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_rows(local: torch.Tensor, m_total: int) -> torch.Tensor:
    """All-gather row shards (shard() layout) into the full (m_total, ...) tensor on every
    rank.  Shards are padded to the largest count so that one all_gather suffices."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return local
    world = dist.get_world_size()
    shards = all_shards(m_total, world)
    cmax = max(c for _, c in shards)
    pad = torch.zeros((cmax,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    return torch.cat([p[:c] for p, (_, c) in zip(parts, shards)], dim=0)
