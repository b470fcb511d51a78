"""Multi-GPU sharding of independent systems (one process per GPU).

The systems never interact (batch_driver.hpp:16-21), so a batch is split into
contiguous shards -- the reference's static partition (batch_driver.cpp:68-73)
applied across ranks -- each rank integrates its shard on its own device with
no data-path collective, and the final states and stats are gathered once
(SURVEY.md 8e). Shards are re-laid out as local SoA arrays so the device
kernels stay coalesced.

torch.distributed is only the plumbing for that final gather. With the NCCL
backend the shards travel as CUDA tensors (GPU to GPU over NVLink) and rank 0
assembles the global SoA on its device before one D2H copy; with gloo (the
CPU tests) they travel as host tensors. Either way the result is bitwise the
single-process one: only bytes move.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Tuple

import numpy as np


def shard_range(num: int, world: int, rank: int) -> Tuple[int, int]:
    """[begin, end) of rank's contiguous shard (batch_driver.cpp:68-73)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, rem = divmod(num, world)
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


def local_soa(y_soa: np.ndarray, num: int, dim: int, begin: int, end: int) -> np.ndarray:
    """Shard [begin, end) of a global SoA array as a local SoA array."""
    return np.ascontiguousarray(y_soa.reshape(dim, num)[:, begin:end]).reshape(-1)


def scatter_back(y_soa: np.ndarray, num: int, dim: int, begin: int, end: int,
                 local: np.ndarray) -> None:
    y_soa.reshape(dim, num)[:, begin:end] = local.reshape(dim, end - begin)


def _backend_device(torch, dist, group):
    """Where the gather payload must live for this group's backend."""
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def gather_bytes(torch, dist, payload, sizes: List[int], group=None) -> Optional[list]:
    """Gather one uint8 tensor per rank (rank r's has sizes[r] bytes) on the
    group's first rank. Returns the list of per-rank tensors there (on the
    backend's device), None elsewhere."""
    dev = _backend_device(torch, dist, group)
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    maxb = max(max(sizes), 1)
    buf = torch.zeros(maxb, dtype=torch.uint8, device=dev)
    if payload.numel():
        buf[: payload.numel()].copy_(payload.reshape(-1).view(torch.uint8), non_blocking=True)
    dst = dist.get_global_rank(group, 0) if group is not None else 0
    out = [torch.empty(maxb, dtype=torch.uint8, device=dev) for _ in range(world)] \
        if rank == 0 else None
    dist.gather(buf, out, dst=dst, group=group)
    if rank != 0:
        return None
    return [out[r][: sizes[r]] for r in range(world)]


def gather_soa_to_rank0(torch, dist, y_local, dim: int, num: int, y_global=None,
                        group=None):
    """The final result gather: every rank's local SoA shard
    (torch float64 tensor of dim x count_r, host or device) is assembled into
    the global SoA array y_global (dim x num) on the group's first rank. With
    NCCL the shards go GPU to GPU and rank 0 writes the global array with one
    D2H copy. Returns y_global on rank 0 (allocated if None), None elsewhere."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    ranges = [shard_range(num, world, r) for r in range(world)]
    sizes = [(hi - lo) * dim * 8 for lo, hi in ranges]
    parts = gather_bytes(torch, dist, y_local.reshape(-1).view(torch.uint8), sizes, group)
    if rank != 0:
        return None
    dev = parts[0].device
    full = torch.empty((dim, num), dtype=torch.float64, device=dev)
    for (lo, hi), p in zip(ranges, parts):
        if hi > lo:
            full[:, lo:hi].copy_(p.view(torch.float64).view(dim, hi - lo))
    if y_global is None:
        y_global = torch.empty(dim * num, dtype=torch.float64,
                               pin_memory=dev.type == "cuda")
    y_global.view(dim, num).copy_(full)  # one D2H copy on the NCCL path
    return y_global


def integrate_sharded(integrate_local: Callable[[np.ndarray, Optional[np.ndarray]],
                                                Tuple[np.ndarray, np.ndarray]],
                      y_soa: np.ndarray, g_soa: Optional[np.ndarray], num: int, dim: int,
                      param_dim: int, group=None) -> Tuple[Optional[np.ndarray],
                                                           Optional[np.ndarray]]:
    """Integrate this rank's shard with `integrate_local(y_local, g_local) ->
    (y_local, stats_local)` and gather every shard on the group's first rank.

    Returns (y_soa, stats) there and (None, None) elsewhere. With no process
    group the call is a single-rank pass-through. A rank whose shard is empty
    (world > num) skips the integration and contributes zero bytes.
    """
    import torch
    import torch.distributed as dist

    from . import _abi as A

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    b, e = shard_range(num, world, rank)
    if e > b:
        y_loc = local_soa(y_soa, num, dim, b, e)
        g_loc = local_soa(g_soa, num, param_dim, b, e) if param_dim else None
        y_loc, st_loc = integrate_local(y_loc, g_loc)
    else:
        y_loc, st_loc = np.empty(0), np.empty(0, dtype=A.STATS_DTYPE)
    if world == 1:
        return y_loc, st_loc
    # the only exchange on the path: one gather of the final shards
    sdt = A.STATS_DTYPE
    payload = torch.from_numpy(np.concatenate([y_loc.view(np.uint8),
                                               np.ascontiguousarray(st_loc).view(np.uint8)]))
    ranges = [shard_range(num, world, r) for r in range(world)]
    nbytes = [(hi - lo) * (dim * 8 + sdt.itemsize) for lo, hi in ranges]
    parts = gather_bytes(torch, dist, payload, nbytes, group)
    if rank != 0:
        return None, None
    y_out = np.empty(num * dim)
    st_out = np.empty(num, dtype=sdt)
    for (lo, hi), p in zip(ranges, parts):
        raw = p.cpu().numpy()
        ny = (hi - lo) * dim * 8
        scatter_back(y_out, num, dim, lo, hi, raw[:ny].view(np.float64))
        st_out[lo:hi] = raw[ny:].view(sdt)
    return y_out, st_out
