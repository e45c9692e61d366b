"""Multi-GPU host logic on CPU: row sharding and max-over-ranks timing (gloo, world 2).

The data path has no collective (every row is independent); the only
cross-rank operation is the MAX reduction of the per-rank device time that
bench.py reports.  Both are exercised here with the gloo backend.
"""

import os
import socket

import numpy as np
import pytest

from paper_2203_09384_b200 import ShapeError, shard_bounds


def test_shard_bounds_partition():
    for batch in (1, 2, 7, 64, 65536, 1000003):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_bounds(batch, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == batch
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and a <= b
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(s for s in sizes if s) <= -(-batch // world)
    with pytest.raises(ShapeError):
        shard_bounds(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, batch, n, q):
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2203_09384_b200 import max_over_ranks, shard_bounds

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    x = oracle.generate_batch(batch, n, seed=7)  # every rank sees the same global batch
    lo, hi = shard_bounds(batch, world, rank)
    # per-rank work: the rank's own row block only (no data exchange)
    y = oracle.reference_execute(x[lo:hi], "forward")
    t = max_over_ranks(10.0 + rank)  # rank-specific "device time"
    # gather only for the check
    parts = [None] * world
    dist.all_gather_object(parts, (lo, hi, y))
    dist.destroy_process_group()
    if rank == 0:
        full = np.empty((batch, n), np.complex64)
        for a, b, part in parts:
            full[a:b] = part
        q.put((t, np.array_equal(full, oracle.reference_execute(x, "forward"))))


def test_gloo_world2_sharded_rows_and_max_timing():
    torch = pytest.importorskip("torch")
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 33, 64, q)) for r in range(2)]
    for p in procs:
        p.start()
    t, same = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert t == 11.0  # max over ranks, not rank 0's own value
    assert same  # concatenated shards == the unsharded batch, bit for bit
    assert torch is not None


def test_max_over_ranks_without_group_is_identity():
    from paper_2203_09384_b200 import max_over_ranks

    assert max_over_ranks(3.5) == 3.5
