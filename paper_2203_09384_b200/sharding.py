"""Batch sharding across GPUs: independent per-device launches, no collective.

Every row of a batched C2C FFT is independent, so k GPUs split
the batch into contiguous row blocks, device d taking rows
[d*ceil(B/k), min(B, (d+1)*ceil(B/k))).  Each device gets its own native plan
replica (twiddles uploaded per device) and its own launches; nothing crosses
NVLink on the compute path.  Two ways in:

* one process, many devices: ``execute_sharded`` runs one host thread per
  device (ctypes drops the GIL inside the C ABI, so the per-device host
  pipelines run concurrently);
* one process per GPU (torchrun): each rank calls ``shard_bounds(B, world,
  rank)`` and executes its block; ``bench.py`` times it with a barrier on
  both sides and the max over ranks.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np

from .errors import ShapeError
from .executor import _execute_host, _prepare_host
from .planner import FftPlan


def shard_bounds(batch: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row block of ``rank`` out of ``world`` (ceil-sized blocks)."""
    if world < 1 or not 0 <= rank < world:
        raise ShapeError(f"rank {rank} outside world of size {world}")
    per = -(-batch // world)
    start = min(batch, rank * per)
    return start, min(batch, start + per)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (device time) over the process group.

    Multi-GPU numbers are timed on each device and reduced with MAX, never
    by wall clock; with no process group this is the identity.
    """
    try:
        import torch
        import torch.distributed as dist
    except ImportError:  # pragma: no cover
        return float(value)
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    if dist.get_backend() == "gloo":
        device = "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def execute_sharded(plan: FftPlan, signal, devices) -> np.ndarray:
    """Run a (B, N) host batch split across ``devices``; returns numpy (B, N)."""
    devices = [int(d) for d in devices]
    if not devices:
        raise ShapeError("execute_sharded needs at least one device")
    _, xc, rows, _ = _prepare_host(plan, signal, allow_real=True)
    x2 = xc.reshape(rows, plan.length)
    out = np.empty(x2.shape, dtype=plan.dtype)

    def run(rank: int) -> None:
        lo, hi = shard_bounds(rows, len(devices), rank)
        if hi > lo:  # each device writes its rows of `out` in place (no staging copy)
            _execute_host(_for_device(plan, devices[rank]), x2[lo:hi], out[lo:hi])

    with ThreadPoolExecutor(max_workers=len(devices)) as pool:
        list(pool.map(run, range(len(devices))))
    return out.reshape(xc.shape)


def _for_device(plan: FftPlan, device: int) -> FftPlan:
    """A view of ``plan`` pinned to ``device`` sharing its native handles."""
    import dataclasses

    view = dataclasses.replace(plan, device=device)
    object.__setattr__(view, "_handles", plan._handles)
    return view
