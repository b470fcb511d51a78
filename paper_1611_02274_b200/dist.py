"""Multi-GPU sharding of independent systems (one process per GPU).

The systems never interact (batch_driver.hpp:16-21), so a batch is split into
contiguous shards -- the reference's static partition (batch_driver.cpp:68-73)
applied across ranks -- each rank integrates its shard on its own device with
no data-path collective, and the final states and stats are gathered once
(SURVEY.md 8e). Shards are re-laid out as local SoA arrays so the device
kernels stay coalesced. torch.distributed (NCCL on GPUs, gloo in the CPU
tests) is only the plumbing for that final gather.
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple

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


def integrate_sharded(integrate_local: Callable[[np.ndarray, Optional[np.ndarray]],
                                                Tuple[np.ndarray, np.ndarray]],
                      y_soa: np.ndarray, g_soa: Optional[np.ndarray], num: int, dim: int,
                      param_dim: int, group=None) -> Tuple[Optional[np.ndarray],
                                                           Optional[np.ndarray]]:
    """Integrate this rank's shard with `integrate_local(y_local, g_local) ->
    (y_local, stats_local)` and gather every shard on rank 0.

    Returns (y_soa, stats) on rank 0 and (None, None) elsewhere. With no
    process group the call is a single-rank pass-through.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    b, e = shard_range(num, world, rank)
    y_loc = local_soa(y_soa, num, dim, b, e)
    g_loc = local_soa(g_soa, num, param_dim, b, e) if param_dim else None
    y_loc, st_loc = integrate_local(y_loc, g_loc)
    if world == 1:
        return y_loc, st_loc
    # the only exchange on the path: one gather of the final shards
    payload = torch.from_numpy(np.concatenate([y_loc.view(np.uint8), st_loc.view(np.uint8)]))
    sizes = [shard_range(num, world, r) for r in range(world)]
    nbytes = [(hi - lo) * (dim * 8 + st_loc.dtype.itemsize) for lo, hi in sizes]
    maxb = max(nbytes)
    buf = torch.zeros(maxb, dtype=torch.uint8)
    buf[: payload.numel()] = payload
    gathered = [torch.zeros(maxb, dtype=torch.uint8) for _ in range(world)] if rank == 0 else None
    dist.gather(buf, gathered, dst=0, group=group)
    if rank != 0:
        return None, None
    y_out = np.empty(num * dim)
    st_out = np.empty(num, dtype=st_loc.dtype)
    for r, ((lo, hi), nb) in enumerate(zip(sizes, nbytes)):
        raw = gathered[r][:nb].numpy()
        ny = (hi - lo) * dim * 8
        scatter_back(y_out, num, dim, lo, hi, raw[:ny].view(np.float64))
        st_out[lo:hi] = raw[ny:nb].view(st_loc.dtype)
    return y_out, st_out
