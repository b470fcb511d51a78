"""Fixed-step harnesses on the device: bitwise against
the oracle's rkck::integrateFixed / rkc::integrateFixed restatements, and the
reference's convergence-order acceptance criterion (acceptance.cpp:92-124:
RKCK slope 5 +- 0.3, RKC slope 2 +- 0.2) measured through the GPU."""
import ctypes
import math

import numpy as np
import pytest

import paper_1611_02274_b200 as B
from paper_1611_02274_b200 import _abi as A
from golden_cases import PLEIADES_IC, heat_ic, perturb

pytestmark = pytest.mark.gpu


def oracle_fixed(oracle, prob, solver, y0, g, num, t0, t1, nsteps, stages=5):
    out = []
    for i in range(num):
        y = np.ascontiguousarray(y0.reshape(prob.dim, num)[:, i])
        gi = None if g is None else np.ascontiguousarray(g.reshape(prob.param_dim, num)[:, i])
        if solver == "rkck":
            oracle.lib.orc_rkck_integrate_fixed(ctypes.byref(prob), t0, t1, nsteps, A.dptr(y),
                                                A.dptr(gi))
        else:
            oracle.lib.orc_rkc_integrate_fixed(ctypes.byref(prob), t0, t1, nsteps, stages,
                                               2.0 / 13.0, A.dptr(y), A.dptr(gi))
        out.append(y)
    return np.ascontiguousarray(np.array(out).T).reshape(-1)


@pytest.mark.parametrize("case", ["pleiades-rkck", "heat64-rkc", "decay-rkck", "decay-rkc",
                                  "harmonic-rkck"])
def test_fixed_bitwise_vs_oracle(gpu, oracle, case):
    num = 64
    name, solver = case.split("-")
    g = None
    if name == "pleiades":
        prob, y0 = A.make_problem(A.PLEIADES), perturb(PLEIADES_IC, 0.01, 3, num)
    elif name == "heat64":
        prob, y0 = A.make_problem(A.HEAT, 64), perturb(heat_ic(64), 0.01, 3, num)
    elif name == "decay":
        prob, y0 = A.make_problem(A.EXPDECAY), perturb(np.array([1.0]), 0.01, 3, num)
        g = np.linspace(0.5, 3.0, num)
    else:
        prob, y0 = A.make_problem(A.HARMONIC), perturb(np.array([1.0, 0.5]), 0.01, 3, num)
    batch = B.BatchStates(num, prob.dim, prob.param_dim, y0.copy(),
                          g.copy() if g is not None else np.zeros(0))
    out = B.integrate_fixed(B.OdeProblem(prob.kind, prob.dim, prob.param_dim), batch, 0.0, 0.5,
                            40, solver=solver, stages=7)
    ref = oracle_fixed(oracle, prob, solver, y0, g, num, 0.0, 0.5, 40, stages=7)
    assert np.array_equal(out.values.view(np.uint64), ref.view(np.uint64))


def test_convergence_orders(gpu):  # acceptance criterion 2 (acceptance.cpp:92-124)
    exact = math.exp(-1.0)
    decay = B.problems.exp_decay()
    batch = B.pack([[1.0]], [[1.0]])

    def slope(ns, solver, stages=0):
        hs, errs = [], []
        for n in ns:
            y = B.integrate_fixed(decay, batch, 0.0, 1.0, n, solver=solver, stages=stages)
            hs.append(1.0 / n)
            errs.append(abs(y.values[0] - exact))
        return np.polyfit(np.log(hs), np.log(errs), 1)[0]

    assert abs(slope((10, 20, 40, 80), "rkck") - 5.0) <= 0.3
    assert abs(slope((20, 40, 80, 160), "rkc", 5) - 2.0) <= 0.2


def test_fixed_validation(gpu):
    b = B.pack([[1.0]], [[1.0]])
    with pytest.raises(B.InvalidInterval):
        B.integrate_fixed(B.problems.exp_decay(), b, 1.0, 1.0, 10)
    with pytest.raises(B.InvalidStageCount):
        B.integrate_fixed(B.problems.exp_decay(), b, 0.0, 1.0, 10, solver="rkc", stages=1)
