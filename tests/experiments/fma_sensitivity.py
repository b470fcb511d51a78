#!/usr/bin/env python3
"""How far does a legitimate re-compilation of the reference arithmetic move
the Pleiades results? Builds the oracle restatement (oracle/bode_oracle.c,
pinned bitwise to the reference) a second time with FMA contraction
(-ffp-contract=fast -mfma, what nvcc does by default) and compares the two
over [0, 1] in 10 windows, with the north_star metric (per-system max-norm
relative error <= 1e-13 = 1e-3*eps, equal accepted/rejected/RHS counts).

This is the yardstick for the FAST policy: at the 0.1 stress perturbation the
bar is out of reach for ANY non-bitwise arithmetic, the reference's own
source included (test infrastructure; CPU only).
"""
import ctypes
import os
import subprocess
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
from golden_cases import PLEIADES_IC, perturb  # noqa: E402
from oracle_lib import Oracle  # noqa: E402
from paper_1611_02274_b200 import _abi as A  # noqa: E402


def main(num=65536):
    so = "/tmp/liboracle_fma.so"
    subprocess.run(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=fast", "-mfma",
                    "-mavx2", "-o", so, os.path.join(REPO, "oracle", "bode_oracle.c"), "-lm",
                    "-lpthread"], check=True)
    O = Oracle()
    F = Oracle.__new__(Oracle)
    F.lib = ctypes.CDLL(so)
    F.lib.orc_outer_loop.restype = O.lib.orc_outer_loop.restype
    F.lib.orc_outer_loop.argtypes = O.lib.orc_outer_loop.argtypes
    prob = A.make_problem(A.PLEIADES)
    for mag in (0.01, 0.1):
        y0 = perturb(PLEIADES_IC, mag, 42, num)
        _, ya, sa, _ = O.outer_loop(prob, A.SOLVER_RKCK, 0.0, 1.0, 0.1, y0)
        _, yb, sb, _ = F.outer_loop(prob, A.SOLVER_RKCK, 0.0, 1.0, 0.1, y0)
        a, b = ya.reshape(28, num), yb.reshape(28, num)
        err = np.max(np.abs(a - b), axis=0) / np.max(np.abs(a), axis=0)
        same = np.ones(num, bool)
        for k in ("steps_accepted", "steps_rejected", "rhs_evals"):
            same &= sa[k] == sb[k]
        print(f"perturb {mag}, {num} systems: FMA-contracted reference arithmetic vs reference: "
              f"within 1e-13 {((err <= 1e-13) & same).mean():.4f}, max rel err {err.max():.3e}, "
              f"count mismatches {(~same).sum()}")


if __name__ == "__main__":
    main()
