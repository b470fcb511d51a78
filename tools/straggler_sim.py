#!/usr/bin/env python3
"""What a straggler-compaction schedule would save (simulation on measured
per-system attempt counts of the FAST RKCK bench workload).

Static cost of a window = sum over warps of max(attempts). Two-pass cost with
threshold T: a warp stops once fewer than T of its lanes are live; its live
systems are compacted (original order) into dense warps that finish them.
Costs are in warp-attempts; the kernel time is proportional.
"""
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))


def two_pass(a, T):
    w = a.reshape(-1, 32)
    s = np.sort(w, axis=1)  # per warp, attempts ascending
    # the warp runs until live lanes < T, i.e. until the (32-T+1)-th smallest finishes
    stop = s[:, 32 - T] if T > 0 else s[:, -1]
    cost1 = stop.sum()
    rem = (w - stop[:, None]).reshape(-1)
    rem = rem[rem > 0]
    pad = (-rem.size) % 32
    rem = np.concatenate([rem, np.zeros(pad, rem.dtype)]).reshape(-1, 32)
    return cost1 + rem.max(axis=1).sum(), rem.shape[0] * 32


def main():
    import torch
    import paper_1611_02274_b200 as P
    from paper_1611_02274_b200 import _abi as A
    from golden_cases import PLEIADES_IC, perturb
    num = 1 << 20
    prob = P.OdeProblem(A.PLEIADES, 28, 0)
    y = torch.from_numpy(perturb(PLEIADES_IC, 0.01, 42, num)).cuda()
    st = torch.zeros(num * 8, dtype=torch.int64, device="cuda")
    tol = A.default_tol()
    s = torch.cuda.current_stream()
    tot = {"static": 0.0, "sorted_by_prev": 0.0}
    cum = np.zeros(num, np.int64)
    # adaptive policy: re-pack (sort by cumulative cost) after a window whose
    # cumulative-cost lockstep efficiency in the current order is below thr
    pol = {thr: {"order": np.arange(num), "cost": 0.0, "repacks": 0} for thr in (0.9, 0.95, 0.97)}
    for k in range(10):
        P.int_driver_device(prob, "rkck", "fast", 0.1 * k, 1.0 if k == 9 else 0.1 * (k + 1), num, 0,
                            y.data_ptr(), tol, st.data_ptr(), False, s.cuda_stream)
        torch.cuda.synchronize()
        stats = st.cpu().numpy().view(A.STATS_DTYPE)
        a = (stats["steps_accepted"] + stats["steps_rejected"]).astype(np.int64)
        static = a.reshape(-1, 32).max(axis=1).sum()
        row = {"window": k, "useful": int(a.sum()), "static": int(static) * 32}
        tot["static"] += static
        # order for this window = systems sorted by their cumulative cost so far
        # (what bode_repack_by_cost would have done after the previous window)
        order = np.argsort(cum, kind="stable") if k > 0 else np.arange(num)
        sp = a[order].reshape(-1, 32).max(axis=1).sum()
        row["sorted_by_prev"] = int(sp) * 32
        tot["sorted_by_prev"] += sp
        for thr, st_ in pol.items():
            st_["cost"] += a[st_["order"]].reshape(-1, 32).max(axis=1).sum()
        cum += a
        for thr, st_ in pol.items():
            cw = cum[st_["order"]].reshape(-1, 32)
            eff = cw.sum() / (cw.max(axis=1).sum() * 32)
            row[f"cum_eff_{thr}"] = float(eff)
            if k < 9 and eff < thr:
                st_["order"] = np.argsort(cum, kind="stable")
                st_["repacks"] += 1
        for T in (4, 8, 16, 24):
            c, n2 = two_pass(a, T)
            row[f"T{T}"] = int(c) * 32
            row[f"T{T}_stragglers"] = int(n2)
            tot[f"T{T}"] = tot.get(f"T{T}", 0.0) + c
        print(json.dumps(row), flush=True)
    # one launch for all 10 windows: a warp runs max over lanes of each lane's
    # total attempts, instead of the sum over windows of per-window maxima
    fused = cum.reshape(-1, 32).max(axis=1).sum()
    tot["fused_windows"] = float(fused)
    for thr, st_ in pol.items():
        tot[f"adaptive_{thr}"] = st_["cost"]
        tot[f"adaptive_{thr}_repacks"] = st_["repacks"] * tot["static"]
    print(json.dumps({k: v / tot["static"] for k, v in tot.items()}))


if __name__ == "__main__":
    main()
