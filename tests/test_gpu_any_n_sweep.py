"""heatEquation(n) for EVERY n in 2..1100 (RKC) and 2..800 (RKCK), EXACT,
bitwise against the oracle (states and every counter): the exact-size lane
kernels, every padded capacity (kernels_pad_a.cu / _b.cu, kernels.cu) at every
fill level, and the one-system-per-block kernels past 1024 (problems.cpp:94-115).
A few systems per n over one short window."""
import numpy as np
import pytest

import paper_1611_02274_b200 as B
from paper_1611_02274_b200 import _abi as A
from golden_cases import heat_ic, perturb

pytestmark = pytest.mark.gpu

COUNTS = ("steps_accepted", "steps_rejected", "rhs_evals", "spec_rad_evals", "underflow",
          "stages_total")


def _sweep(oracle, solver, nmax, window):
    bad, work = [], []
    for n in range(2, nmax + 1):
        num, t1 = 6, window(n)
        y0 = perturb(heat_ic(n), 0.01, 1000 + n, num)
        b = B.BatchStates(num, n, 0, y0.copy(), np.zeros(0))
        r = B.outer_loop(B.OdeProblem(A.HEAT, n, 0), b, 0.0, t1, t1, solver=solver,
                         arith="exact")
        rc, yo, so, _ = oracle.outer_loop(A.make_problem(A.HEAT, n), A.SOLVER_NAMES[solver],
                                          0.0, t1, t1, y0)
        ok = rc == 0 and np.array_equal(r.states.values.view(np.uint64), yo.view(np.uint64))
        ok = ok and all(np.array_equal(r.stats[k], so[k]) for k in COUNTS)
        if not ok:
            bad.append(n)
        work.append(int(r.stats["steps_accepted"].min()))
    assert not bad, f"{solver}: {len(bad)} dimensions differ, first {bad[:20]}"
    assert min(work) >= 2  # every window took several accepted steps


def test_rkc_every_n_to_1100(gpu, oracle):
    _sweep(oracle, "rkc", 1100, lambda n: 0.02 if n <= 128 else 0.004 if n <= 512 else 0.001)


def test_rkck_every_n_to_800(gpu, oracle):
    # RKCK on the stiff heat problem needs h ~ dx^2: a window of a few such steps
    _sweep(oracle, "rkck", 800, lambda n: min(0.01, 2.0 / (n + 1) ** 2))
