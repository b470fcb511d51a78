"""The opt-in per-window attempt budget (bode_set_attempt_budget, include/bode.h).

Not a reference feature: the reference's drivers run until tEnd or underflow
(rkck.cpp:131-157, rkc.cpp:223-279). With a budget B, a system that reaches
B attempts (accepted + rejected) in a window stops there, frozen at its last
accepted state with stats.budget_exhausted set; every other system is
bitwise the unbudgeted run. Default 0 (no budget) is the reference.
"""
import numpy as np
import pytest

import paper_1611_02274_b200 as B
from paper_1611_02274_b200 import _abi as A
from golden_cases import perturb, PLEIADES_IC, heat_ic
from test_gpu_parity import run_gpu

pytestmark = pytest.mark.gpu


def _window(prob, solver, y0, arith, budget, t1, wide=False):
    L = B.lib()
    assert L.bode_set_attempt_budget(budget) == 0
    L.bode_set_wide(1 if wide else 0)
    try:
        return run_gpu(prob, solver, y0, None, arith, t1=t1, hout=t1)
    finally:
        L.bode_set_attempt_budget(0)
        L.bode_set_wide(0)


@pytest.mark.parametrize("case", ["pleiades_fast", "pleiades_exact", "heat64_rkc", "heat100_wide"])
def test_budget_freezes_only_the_systems_that_reach_it(gpu, case):
    if case.startswith("pleiades"):
        prob, solver, n = A.make_problem(A.PLEIADES, 28), A.SOLVER_RKCK, 28
        y0 = perturb(PLEIADES_IC, 0.1, 9, 4096)
        arith, t1 = case.split("_")[1], 0.6
    elif case == "heat64_rkc":
        prob, solver, n = A.make_problem(A.HEAT, 64), A.SOLVER_RKC, 64
        y0 = perturb(heat_ic(64), 0.01, 9, 1024)
        arith, t1 = "exact", 0.2
    else:
        prob, solver, n = A.make_problem(A.HEAT, 100), A.SOLVER_RKC, 100
        y0 = perturb(heat_ic(100), 0.01, 9, 256)
        arith, t1 = "exact", 0.1
    num = y0.size // n
    wide = case == "heat100_wide"  # the one-system-per-block kernel (forced)
    y_free, st_free = _window(prob, solver, y0, arith, 0, t1, wide)
    att = st_free["steps_accepted"] + st_free["steps_rejected"]
    budget = int(np.percentile(att, 90))
    assert att.max() > budget  # some systems must hit it
    y_b, st_b = _window(prob, solver, y0, arith, budget, t1, wide)
    hit = st_b["budget_exhausted"] != 0
    assert not st_free["budget_exhausted"].any()
    # exactly the systems that needed more attempts than the budget
    assert np.array_equal(hit, att > budget)
    assert np.array_equal((st_b["steps_accepted"] + st_b["steps_rejected"])[hit],
                          np.full(hit.sum(), budget))
    # everyone else: bitwise the unbudgeted run
    ok = ~hit
    a, b = y_b.reshape(n, num), y_free.reshape(n, num)
    assert np.array_equal(a[:, ok].view(np.uint64), b[:, ok].view(np.uint64))
    for k in ("steps_accepted", "steps_rejected", "rhs_evals", "underflow"):
        assert np.array_equal(st_b[k][ok], st_free[k][ok]), k
    assert np.isfinite(a[:, hit]).all()
    assert (st_b["steps_accepted"][hit] <= st_free["steps_accepted"][hit]).all()


def test_budget_merges_across_outer_windows(gpu):
    """bode_outer_loop merges the flag like underflow (ode_problem.hpp:72-80)."""
    L = B.lib()
    prob = A.make_problem(A.PLEIADES, 28)
    y0 = perturb(PLEIADES_IC, 0.1, 4, 2048)
    assert L.bode_set_attempt_budget(12) == 0
    try:
        y, st = run_gpu(prob, A.SOLVER_RKCK, y0, None, "exact", t1=1.0, hout=0.1)
    finally:
        L.bode_set_attempt_budget(0)
    hit = st["budget_exhausted"] != 0
    assert hit.any() and not hit.all()
    # at most 12 attempts in each of the 10 windows
    assert ((st["steps_accepted"] + st["steps_rejected"]) <= 120).all()
