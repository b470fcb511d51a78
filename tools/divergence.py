#!/usr/bin/env python3
"""Per-window kernel time and SIMT lockstep efficiency of the RKCK/RKC kernels.

Lockstep efficiency of a warp = mean(attempts) / max(attempts) over its 32
consecutive systems (one system per lane), i.e. the fraction of issue slots
doing useful attempts when every lane waits for the slowest system.
    python tools/divergence.py [--problem pleiades|heat|expdecay|expdecay_sorted] [--num N]
                               [--arith fast]
"""
import argparse
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--problem", default="pleiades")
    ap.add_argument("--num", type=int, default=1 << 20)
    ap.add_argument("--arith", default="fast")
    ap.add_argument("--mag", type=float, default=0.01)
    args = ap.parse_args()
    import torch
    import paper_1611_02274_b200 as P
    from paper_1611_02274_b200 import _abi as A
    from golden_cases import PLEIADES_IC, heat_ic, perturb

    from paper_1611_02274_b200.api import stiffness_params
    gh = None
    if args.problem == "pleiades":
        dim, solver, base, lanes = 28, "rkck", PLEIADES_IC, 1
    elif args.problem == "heat":
        dim, solver, base, lanes = 64, "rkc", heat_ic(64), 8
    else:  # config 4: expdecay (natural order) or expdecay_sorted (sorted by g0)
        dim, solver, base, lanes = 1, "rkc", np.array([1.0]), 1
        gh = stiffness_params(args.num)
    y0 = perturb(base, args.mag, 42, args.num)
    if args.problem == "expdecay_sorted":
        order = np.argsort(gh, kind="stable")
        gh, y0 = gh[order], y0[order]
    kind = "expdecay" if args.problem.startswith("expdecay") else args.problem
    prob = P.OdeProblem(A.PROBLEM_NAMES[kind], dim, 0 if gh is None else 1)
    y = torch.from_numpy(y0).cuda()
    g = torch.from_numpy(gh).cuda() if gh is not None else None
    st = torch.zeros(args.num * 8, dtype=torch.int64, device="cuda")
    tol = A.default_tol()
    s = torch.cuda.current_stream()
    out = []
    for k in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        P.int_driver_device(prob, solver, args.arith, 0.1 * k, 1.0 if k == 9 else 0.1 * (k + 1),
                            args.num, g.data_ptr() if g is not None else 0, y.data_ptr(), tol,
                            st.data_ptr(), False, s.cuda_stream)
        e1.record()
        torch.cuda.synchronize()
        stats = st.cpu().numpy().view(A.STATS_DTYPE)
        att = (stats["steps_accepted"] + stats["steps_rejected"]).astype(np.float64)
        work = stats["stages_total"].astype(np.float64) if solver == "rkc" else att
        per_warp = work.reshape(-1, 32 // lanes)
        eff = float(np.mean(per_warp.mean(axis=1) / per_warp.max(axis=1)))
        out.append({"window": k, "ms": e0.elapsed_time(e1), "attempts_mean": float(att.mean()),
                    "attempts_max": float(att.max()), "lockstep_eff": eff})
        print(json.dumps(out[-1]), flush=True)
    print(json.dumps({"problem": args.problem, "arith": args.arith, "num": args.num,
                      "mean_lockstep_eff": float(np.mean([o["lockstep_eff"] for o in out])),
                      "total_ms": float(sum(o["ms"] for o in out))}))


if __name__ == "__main__":
    main()
