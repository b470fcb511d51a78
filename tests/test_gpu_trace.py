"""StepObserver on the device (bode_trace_steps; ode_problem.hpp:85-94, invoked
at rkck.cpp:142 and rkc.cpp:253): one system's window with every attempt
recorded as (t, h, stages, err, accepted). Under EXACT the records, the final
state and the stats are bitwise the oracle driver's with an observer; under
FAST the attempt sequence is the same length on the bench workload. The
batch kernels never record (the instrumented instances run only for a trace
or an attempt budget)."""
import numpy as np
import pytest

import paper_1611_02274_b200 as B
from paper_1611_02274_b200 import _abi as A
from golden_cases import PLEIADES_IC, heat_ic, perturb

pytestmark = pytest.mark.gpu


def oracle_records(oracle, prob, solver, t, t1, y, g=None):
    recs = []
    rc, yo, so = oracle.driver(prob, solver, t, t1, y, g,
                               observer=lambda tt, h, s, err, acc, u: recs.append(
                                   (tt, h, err, s, 1 if acc else 0)))
    assert rc == 0
    return yo, so, np.array(recs, dtype=A.STEP_DTYPE)


CASES = [
    ("pleiades-rkck", lambda: (A.make_problem(A.PLEIADES), A.SOLVER_RKCK,
                               perturb(PLEIADES_IC, 0.1, 9, 8)[3::8], None, 0.0, 0.6)),
    ("heat64-rkc", lambda: (A.make_problem(A.HEAT, 64), A.SOLVER_RKC,
                            perturb(heat_ic(64), 0.01, 9, 1), None, 0.0, 0.1)),
    ("heat100-rkc", lambda: (A.make_problem(A.HEAT, 100), A.SOLVER_RKC,
                             perturb(heat_ic(100), 0.01, 9, 1), None, 0.0, 0.05)),
    ("heat1000-rkc", lambda: (A.make_problem(A.HEAT, 1000), A.SOLVER_RKC,
                              perturb(heat_ic(1000), 0.01, 9, 1), None, 0.0, 1e-3)),
    ("heat17-rkck", lambda: (A.make_problem(A.HEAT, 17), A.SOLVER_RKCK,
                             perturb(heat_ic(17), 0.01, 9, 1), None, 0.0, 0.01)),
    ("expdecay-rkc", lambda: (A.make_problem(A.EXPDECAY), A.SOLVER_RKC, np.array([1.0]),
                              np.array([3.0e3]), 0.0, 1.0)),
    ("expdecay-rkck", lambda: (A.make_problem(A.EXPDECAY), A.SOLVER_RKCK, np.array([1.0]),
                               np.array([20.0]), 0.0, 1.0)),
]


@pytest.mark.parametrize("name,make", CASES, ids=[c[0] for c in CASES])
def test_trace_is_the_reference_observer(gpu, oracle, name, make):
    prob, solver, y0, g, t0, t1 = make()
    yo, so, ro = oracle_records(oracle, prob, solver, t0, t1, y0, g)
    y, st, rec = B.trace_steps(B.OdeProblem(prob.kind, prob.dim, prob.param_dim), y0, g, t0, t1,
                               solver=solver, arith="exact")
    assert len(rec) == len(ro) > 0
    assert np.array_equal(rec.view(np.uint8), ro.view(np.uint8))
    assert np.array_equal(y.view(np.uint64), yo.view(np.uint64))
    for k in ("steps_accepted", "steps_rejected", "rhs_evals", "spec_rad_evals"):
        assert st[k] == so[k], k
    # the records add up to the stats (acc + rej attempts, s stages each)
    assert rec["accepted"].sum() == st["steps_accepted"]
    assert (1 - rec["accepted"]).sum() == st["steps_rejected"]
    assert rec["stages"].sum() == st["stages_total"]


def test_trace_fast_and_capacity(gpu, oracle):
    prob = A.make_problem(A.PLEIADES)
    y0 = perturb(PLEIADES_IC, 0.01, 42, 1)
    yo, so, ro = oracle_records(oracle, prob, A.SOLVER_RKCK, 0.0, 0.1, y0)
    bp = B.OdeProblem(prob.kind, 28, 0)
    y, st, rec = B.trace_steps(bp, y0, None, 0.0, 0.1, solver="rkck", arith="fast")
    assert len(rec) == len(ro)
    assert np.array_equal(rec["accepted"], ro["accepted"])
    # FAST forms err from different (FMA, RKN) arithmetic: h follows err^-0.2
    assert np.max(np.abs(rec["h"] - ro["h"]) / ro["h"]) < 1e-5
    # a short buffer keeps the first records; the count still reports every attempt
    y2, st2, rec2 = B.trace_steps(bp, y0, None, 0.0, 0.1, solver="rkck", arith="exact",
                                  capacity=3)
    assert len(rec2) == 3 and np.array_equal(rec2.view(np.uint8), ro[:3].view(np.uint8))
    with pytest.raises(B.InvalidInterval):
        B.trace_steps(bp, y0, None, 1.0, 1.0)
