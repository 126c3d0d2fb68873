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


def _world_rank():
    if not dist.is_initialized():
        return 1, 0
    return dist.get_world_size(), dist.get_rank()


class GatherBuffer:
    """Preallocated result gather for the shard() layout.

    One (world * cmax, *row) buffer holds every rank's slot (cmax = largest shard); the
    kernel writes this rank's rows straight into its own slot (local()), and gather() is one
    in-place all_gather_into_tensor (no staging copy, no list of parts, no torch.cat).  When
    the shards are equal (m_total % world == 0, e.g. cfg5) the buffer IS the gathered
    result; otherwise result() compacts the padded slots once."""

    def __init__(self, m_total: int, row_shape=(), dtype=torch.float64, device=None):
        self.world, self.rank = _world_rank()
        self.m_total = m_total
        self.shards = all_shards(m_total, self.world)
        self.cmax = max(c for _, c in self.shards) if m_total else 0
        self.equal = all(c == self.cmax for _, c in self.shards)
        self.full = torch.empty((self.world * self.cmax,) + tuple(row_shape), dtype=dtype, device=device)
        self.kind = "all_gather_into_tensor in place" if self.world > 1 else "none (1 rank)"

    def slot(self, rank: int) -> torch.Tensor:
        return self.full[rank * self.cmax:(rank + 1) * self.cmax]

    def local(self, rank: int | None = None) -> torch.Tensor:
        """This rank's output rows (a view into the gather buffer)."""
        r = self.rank if rank is None else rank
        return self.slot(r)[: self.shards[r][1]]

    def gather(self) -> None:
        if self.world > 1:
            dist.all_gather_into_tensor(self.full, self.slot(self.rank))

    def result(self) -> torch.Tensor:
        if self.world == 1 or self.equal:
            return self.full[: self.m_total]
        return torch.cat([self.slot(r)[:c] for r, (_, c) in enumerate(self.shards)], dim=0)


def gather_rows(local: torch.Tensor, m_total: int) -> torch.Tensor:
    """All-gather row shards (shard() layout) into the full (m_total, ...) tensor on every
    rank.  Copies `local` into a GatherBuffer slot; write into GatherBuffer.local() directly
    to avoid that copy."""
    world, rank = _world_rank()
    if world == 1:
        return local
    gb = GatherBuffer(m_total, tuple(local.shape[1:]), local.dtype, local.device)
    gb.local(rank).copy_(local)
    gb.gather()
    return gb.result()
