"""Multi-process host logic of the multi-GPU driver on CPU: gloo backend, world_size 2.

The GPU kernels cannot run here, so the per-point work is stood in for by a row-local
function of the index-addressable inputs; what is tested is the sharding, the gather and
the max-over-ranks timing reduction that bench.py uses with NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from paper_2410_22575_b200.dist import GatherBuffer, all_shards, gather_rows, max_over_ranks, shard


def test_shard_cover():
    for m in (0, 1, 7, 1024, 1 << 20):
        for w in (1, 2, 3, 8):
            s = all_shards(m, w)
            assert sum(c for _, c in s) == m
            assert s[0][0] == 0
            for (f0, c0), (f1, _) in zip(s[:-1], s[1:]):
                assert f0 + c0 == f1
            assert max(c for _, c in s) - min(c for _, c in s) <= 1
    with pytest.raises(ValueError):
        shard(10, 2, 2)


def test_shard_inputs_independent_of_world():
    """A shard generated on its own equals the same rows of the full array (synth is
    index-addressable), so 1/2/4/8-GPU runs see identical data."""
    n, m = 16, 1000
    full = synth.points(0, n, m)
    for w in (2, 3, 8):
        for f, c in all_shards(m, w):
            assert np.array_equal(synth.points(0, n, c, f), full[f:f + c])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, m_total, n, q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    first, count = shard(m_total, rank, world)
    pts = torch.from_numpy(synth.points(0, n, count, first))
    local = pts * 2.0 + 1.0  # stand-in row-local result
    full = gather_rows(local, m_total)
    # preallocated in-place path: the "kernel" writes straight into this rank's slot
    gb = GatherBuffer(m_total, (n,), torch.float64)
    gb.local().copy_(local)
    gb.gather()
    full2 = gb.result()
    t = max_over_ranks(0.5 + rank)
    q.put((rank, full.numpy(), t, full2.numpy(), gb.kind))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("m_total", [37, 64])
def test_gloo_world2_gather_and_max(m_total):
    n, world = 4, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m_total, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = synth.points(0, n, m_total) * 2.0 + 1.0
    for rank, full, t, full2, kind in res:
        assert np.array_equal(full, want)
        assert np.array_equal(full2, want)
        assert t == 1.5 and "all_gather_into_tensor" in kind
