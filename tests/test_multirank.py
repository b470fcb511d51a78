"""World-size-2 sharding over gloo on CPU: the shard partition,
the SoA re-layout and the final gather reassemble exactly the single-process
result -- the distributed analogue of the reference's worker-invariance test
(test_batch.cpp:127-142). The per-shard integrator here is the C oracle
(test infrastructure); on GPUs bench.py runs the same plumbing over NCCL with
the CUDA kernels."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1611_02274_b200.dist import local_soa, scatter_back, shard_range


def test_shard_range_partition():
    for num in (1, 2, 7, 1000, 1 << 20):
        for world in (1, 2, 3, 8):
            ranges = [shard_range(num, world, r) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == num
            assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))
            sizes = [e - b for b, e in ranges]
            assert max(sizes) - min(sizes) <= 1


def test_soa_relayout_roundtrip():
    num, dim = 37, 5
    y = np.arange(num * dim, dtype=np.float64)
    out = np.zeros_like(y)
    for r in range(3):
        b, e = shard_range(num, 3, r)
        loc = local_soa(y, num, dim, b, e)
        assert loc.reshape(dim, e - b)[2, 0] == y.reshape(dim, num)[2, b]
        scatter_back(out, num, dim, b, e, loc)
    assert np.array_equal(out, y)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    import torch.distributed as dist
    from golden_cases import PLEIADES_IC, perturb
    from oracle_lib import Oracle
    from paper_1611_02274_b200 import _abi as A
    from paper_1611_02274_b200.dist import integrate_sharded

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    O = Oracle()
    prob = A.make_problem(A.PLEIADES)
    num = 301
    y0 = perturb(PLEIADES_IC, 0.01, 7, num)

    def local(y_loc, g_loc):
        rc, y, st, _ = O.outer_loop(prob, A.SOLVER_RKCK, 0.0, 0.3, 0.1, y_loc, threads=1)
        assert rc == 0
        return y, st

    y, st = integrate_sharded(local, y0, None, num, 28, 0)
    if rank == 0:
        q.put((y, st))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_matches_single_process(oracle):
    from golden_cases import PLEIADES_IC, perturb
    from paper_1611_02274_b200 import _abi as A
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    y, st = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    num = 301
    y0 = perturb(PLEIADES_IC, 0.01, 7, num)
    rc, y_ref, st_ref, _ = oracle.outer_loop(A.make_problem(A.PLEIADES), A.SOLVER_RKCK, 0.0, 0.3,
                                             0.1, y0)
    assert np.array_equal(y.view(np.uint64), y_ref.view(np.uint64))
    for k in ("steps_accepted", "steps_rejected", "rhs_evals", "h_min_seen", "h_max_seen"):
        assert np.array_equal(st[k], st_ref[k]), k


def _gather_worker(rank, world, port, num, dim, q):
    import torch
    import torch.distributed as dist
    from paper_1611_02274_b200.dist import gather_soa_to_rank0, shard_range

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    b, e = shard_range(num, world, rank)
    y = np.arange(num * dim, dtype=np.float64).reshape(dim, num)
    loc = torch.from_numpy(np.ascontiguousarray(y[:, b:e]).reshape(-1))
    out = gather_soa_to_rank0(torch, dist, loc, dim, num)
    if rank == 0:
        q.put(out.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


def _empty_shard_worker(rank, world, port, q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    import torch.distributed as dist
    from golden_cases import PLEIADES_IC, perturb
    from oracle_lib import Oracle
    from paper_1611_02274_b200 import _abi as A
    from paper_1611_02274_b200.dist import integrate_sharded

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    O = Oracle()
    prob = A.make_problem(A.PLEIADES)
    y0 = perturb(PLEIADES_IC, 0.01, 3, 2)
    calls = []

    def local(y_loc, g_loc):
        calls.append(y_loc.size)
        rc, y, st, _ = O.outer_loop(prob, A.SOLVER_RKCK, 0.0, 0.1, 0.1, y_loc, threads=1)
        assert rc == 0
        return y, st

    y, st = integrate_sharded(local, y0, None, 2, 28, 0)
    assert (rank < 2) == bool(calls)  # the empty shard never integrates
    if rank == 0:
        q.put((y, st))
    dist.barrier()
    dist.destroy_process_group()


def _spawn(target, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, *args, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    return out


@pytest.mark.parametrize("world,num", [(2, 301), (3, 2)])
def test_gather_soa_to_rank0_gloo(world, num):
    """The final result gather used by bench.py's multi-rank e2e: ragged and
    empty shards land in the global SoA layout byte for byte."""
    dim = 5
    out = _spawn(_gather_worker, world, num, dim)
    assert np.array_equal(out, np.arange(num * dim, dtype=np.float64))


def test_integrate_sharded_empty_shard_gloo(oracle):
    """world > num: the rank with no systems skips the integration."""
    from golden_cases import PLEIADES_IC, perturb
    from paper_1611_02274_b200 import _abi as A
    y, st = _spawn(_empty_shard_worker, 3)
    y0 = perturb(PLEIADES_IC, 0.01, 3, 2)
    rc, y_ref, st_ref, _ = oracle.outer_loop(A.make_problem(A.PLEIADES), A.SOLVER_RKCK, 0.0, 0.1,
                                             0.1, y0)
    assert np.array_equal(y.view(np.uint64), y_ref.view(np.uint64))
    assert np.array_equal(st["rhs_evals"], st_ref["rhs_evals"])
