#!/usr/bin/env python3
"""Configs 2, 3 and 5 as a size sweep on one GPU: RKCK Pleiades
(FAST and EXACT) and RKC heat64 (EXACT) from 2^10 to 2^22 systems, plus the
2^24-system point of config 5, device-resident, the paper's [0, 1] protocol
(10 restart windows after one warm-up window). Prints one JSON line per point.

    python tools/sweep.py [--max-log2 24] [--rkc-max-log2 24]
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
    ap.add_argument("--max-log2", type=int, default=24)
    ap.add_argument("--rkc-max-log2", type=int, default=24)
    args = ap.parse_args()
    import ctypes
    import torch
    import paper_1611_02274_b200 as P
    from paper_1611_02274_b200 import _abi as A
    from golden_cases import PLEIADES_IC, heat_ic, perturb
    import bench

    L = P.lib()
    peak, psec = ctypes.c_double(), ctypes.c_double()
    P.api.check(L.bode_selftest_fp64_peak(ctypes.byref(peak), ctypes.byref(psec)))
    stream = torch.cuda.Stream()
    cases = [("pleiades", "rkck", "fast", 28, PLEIADES_IC, args.max_log2),
             ("pleiades", "rkck", "exact", 28, PLEIADES_IC, args.max_log2),
             ("heat", "rkc", "exact", 64, heat_ic(64), args.rkc_max_log2)]
    for problem, solver, arith, dim, base, top in cases:
        for lg in list(range(10, 23, 2)) + ([24] if top >= 24 else []):
            if lg > top:
                continue
            num = 1 << lg
            y0 = perturb(base, 0.01, 42, num)
            secs, per, stats, launches, _ = bench.measure_device(
                P, A, torch, problem, solver, arith, dim, y0, None, 10, 1, stream)
            flops = bench.algorithmic_flops(problem, solver, dim, stats, 10)
            print(json.dumps({"problem": problem, "solver": solver, "arith": arith, "num": num,
                              "ms_total": secs * 1e3,
                              "system_windows_per_s": num * 10 / secs,
                              "systems_per_s_full_protocol": num / secs,
                              "frac_of_fp64_peak": flops / secs / peak.value}), flush=True)
            del y0


if __name__ == "__main__":
    main()
