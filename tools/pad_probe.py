#!/usr/bin/env python3
"""Throughput of heatEquation(n) on whichever kernel the library picks for n
(padded lane groups, or one system per block), one window [0, t1] of RKC on
HBM-resident state, wall time around bode_int_driver_device after a warm-up
window. Prints one JSON object per (n, arith) with a hash of the final state,
so two library builds (BODE_LIB_PATH) can be compared for speed and bitwise
agreement.

    python tools/pad_probe.py --dims 90,100,120 --num 262144 --t1 0.1
"""
import argparse
import hashlib
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [REPO, os.path.join(REPO, "tests")]

import torch  # noqa: E402

import paper_1611_02274_b200 as B  # noqa: E402
from paper_1611_02274_b200 import _abi as A  # noqa: E402
from golden_cases import heat_ic, perturb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", default="90,100,120")
    ap.add_argument("--arith", default="exact,fast")
    ap.add_argument("--num", type=int, default=1 << 18)
    ap.add_argument("--t1", type=float, default=0.1)
    ap.add_argument("--wide", type=int, default=0)
    ap.add_argument("--solver", default="rkc", choices=["rkc", "rkck"])
    a = ap.parse_args()
    L = B.lib()
    L.bode_set_wide(a.wide)
    for n in map(int, a.dims.split(",")):
        y0 = torch.from_numpy(perturb(heat_ic(n), 0.01, 42, a.num))
        for arith in a.arith.split(","):
            yd = y0.cuda()
            st = torch.zeros(a.num * 8, dtype=torch.int64, device="cuda")
            p = B.OdeProblem(A.HEAT, n, 0)

            def run():
                B.int_driver_device(p, a.solver, arith, 0.0, a.t1, a.num, 0, yd.data_ptr(),
                                    A.default_tol(), st.data_ptr(), 0, 0)

            run()
            yd.copy_(y0)
            torch.cuda.synchronize()
            t = time.perf_counter()
            run()
            torch.cuda.synchronize()
            dt = time.perf_counter() - t
            h = hashlib.sha1(yd.cpu().numpy().tobytes() + st.cpu().numpy().tobytes()).hexdigest()
            print(json.dumps({"n": n, "arith": arith, "solver": a.solver, "num": a.num, "t1": a.t1,
                              "system_windows_per_s": a.num / dt, "ms": dt * 1e3,
                              "state_hash": h[:16], "lib": os.environ.get("BODE_LIB_PATH", "")}),
                  flush=True)
    L.bode_set_wide(0)


if __name__ == "__main__":
    main()
