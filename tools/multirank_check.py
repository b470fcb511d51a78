#!/usr/bin/env python3
"""Multi-rank correctness check of the config-5 sharding (run under torchrun).

Each rank builds its contiguous shard of a fixed Pleiades batch
(bode_perturb_initial_conditions_range), integrates it over [0, 1] in 10
windows through bode_outer_loop on its own device, and the shards are
gathered to rank 0 (paper_1611_02274_b200.dist.gather_soa_to_rank0: NCCL
between GPUs, gloo when BODE_BENCH_SHARE_GPU=1 puts every rank on cuda:0).
Rank 0 compares the gathered states and stats with one single-process run of
the whole batch, bitwise, and prints MULTIRANK_OK.
"""
import argparse
import ctypes
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--systems", type=int, default=1 << 20)
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    import paper_1611_02274_b200 as P
    from paper_1611_02274_b200 import _abi as A
    from paper_1611_02274_b200 import dist as D

    share = os.environ.get("BODE_BENCH_SHARE_GPU") == "1"
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = local % torch.cuda.device_count() if share else local
    torch.cuda.set_device(local)
    if share:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    L = P.lib()
    P.api.check(L.bode_use_device(local))
    num = args.systems
    b, e = D.shard_range(num, world, rank)
    base = np.array(P.problems.pleiades_initial_conditions())
    dp = ctypes.POINTER(ctypes.c_double)
    y = np.empty((e - b) * 28)
    P.api.check(L.bode_perturb_initial_conditions_range(base.ctypes.data_as(dp), 28, 0.01, 42,
                                                        b, e - b, y.ctypes.data_as(dp)))
    prob = A.make_problem(A.PLEIADES)
    st = A.empty_stats(e - b)
    steps = ctypes.c_int32(0)
    P.api.check(L.bode_outer_loop(ctypes.byref(prob), 0, 0, 0.0, 1.0, 0.1, e - b, None,
                                  y.ctypes.data_as(dp), ctypes.byref(A.default_tol()),
                                  A.vptr(st), 1, P.api.SINK(), None, ctypes.byref(steps)))
    yg = D.gather_soa_to_rank0(torch, dist, torch.from_numpy(y), 28, num)
    st_soa = np.ascontiguousarray(st.view(np.float64).reshape(-1, 8).T).reshape(-1)
    sg = D.gather_soa_to_rank0(torch, dist, torch.from_numpy(st_soa), 8, num)
    if rank == 0:
        full = P.problems.perturb_initial_conditions(base, 0.01, 42, num)
        r = P.outer_loop(P.problems.pleiades(), full, 0.0, 1.0, 0.1, solver="rkck")
        ok_y = np.array_equal(yg.numpy().view(np.uint64), r.states.values.view(np.uint64))
        # stats travel as 8 float64 rows of the AoS records: re-interleave
        st_all = np.ascontiguousarray(sg.numpy().reshape(8, num).T).view(A.STATS_DTYPE).reshape(-1)
        ok_s = all(np.array_equal(st_all[k], r.stats[k]) for k in
                   ("steps_accepted", "steps_rejected", "rhs_evals", "h_min_seen", "h_max_seen"))
        print(f"world={world} systems={num} states_bitwise={ok_y} stats_equal={ok_s}", flush=True)
        if ok_y and ok_s:
            print("MULTIRANK_OK", flush=True)
        else:
            sys.exit(1)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
