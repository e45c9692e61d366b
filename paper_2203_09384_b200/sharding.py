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
  both sides and the max over ranks;
* device-resident shards in one process: ``scatter_rows`` places the row
  blocks on their devices (peer copies over NVLink), ``execute_shards``
  launches every shard asynchronously on its own device and then waits on
  each, and ``gather_rows`` brings the results to one device (peer copies;
  the optional, untimed gather of SURVEY.md 8e).
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np

from .errors import DomainError, ShapeError
from .executor import _execute_host, _is_torch, _prepare_device, _prepare_host, launch
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


def scatter_rows(x, devices):
    """Contiguous row blocks of a (B, N) tensor (or array), one per device in
    ``devices`` (``shard_bounds``), each moved to its device -- peer copies
    between GPUs, H2D from host.  Empty blocks (B < len(devices)) are skipped."""
    import torch

    t = x if _is_torch(x) else torch.from_numpy(np.ascontiguousarray(x))
    if t.dim() != 2:
        raise ShapeError(f"scatter_rows needs a (batch, N) input, got shape {tuple(t.shape)}")
    blocks = []
    for rank, d in enumerate(devices):
        lo, hi = shard_bounds(t.shape[0], len(devices), rank)
        if hi > lo:
            blocks.append(t[lo:hi].to(torch.device("cuda", int(d)), non_blocking=True))
    return blocks


def execute_shards(plan: FftPlan, shards) -> list:
    """Transform device-resident shards (CUDA tensors, possibly on different
    GPUs): one asynchronous launch per shard on its device's current stream,
    issued for all shards before any wait, then one wait per shard (its
    NaN/Inf flag read).  Returns the outputs, each on its shard's device."""
    import torch

    cdt = torch.complex64 if plan.dtype == np.complex64 else torch.complex128
    outs, flags = [], []
    for x in shards:
        if not (_is_torch(x) and x.is_cuda):
            raise ShapeError("execute_shards takes CUDA tensors (scatter_rows places host rows)")
        xc, rows, _ = _prepare_device(plan, x)
        with torch.cuda.device(xc.device):
            out = torch.empty(xc.shape, dtype=cdt, device=xc.device)
            flag = torch.zeros(1, dtype=torch.int32, device=xc.device)
            launch(plan, xc, out, rows, flag=flag)
        outs.append(out)
        flags.append(flag)
    for flag in flags:  # .item() waits for that device's stream
        if int(flag.item()):
            raise DomainError("signal contains NaN or Inf values")
    return outs


def gather_rows(shards, device):
    """Concatenate row blocks on one device (peer copies over NVLink)."""
    import torch

    dev = torch.device("cuda", int(device)) if not isinstance(device, torch.device) else device
    return torch.cat([s.to(dev, non_blocking=True) for s in shards], dim=0)


def _for_device(plan: FftPlan, device: int) -> FftPlan:
    """A view of ``plan`` pinned to ``device`` sharing its native handles."""
    import dataclasses

    view = dataclasses.replace(plan, device=device)
    object.__setattr__(view, "_handles", plan._handles)
    return view
