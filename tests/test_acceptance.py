"""The reference's release criteria (proj/tests/acceptance.cpp) that exercise
the device path, at their stated tolerances: 1 (tableau identities, plus the
identities the FAST Runge-Kutta-Nystrom form relies on), 3 (Pleiades
self-consistency and conservation), 4 (RKC stability beyond the explicit Euler
limit). Criteria 2, 7 and 9 are in test_gpu_fixed.py / test_gpu_parity.py /
test_gpu_kats.py; 5, 6, 8 are controller/oracle properties (test_oracle_kats.py)."""
from fractions import Fraction as F

import numpy as np
import pytest

import paper_1611_02274_b200 as B
from paper_1611_02274_b200 import _abi as A
from golden_cases import PLEIADES_IC, heat_ic

# Cash-Karp tableau (rkck.cpp:8-27)
a = [None, F(0), F(1, 5), F(3, 10), F(3, 5), F(1), F(7, 8)]
b = {2: [F(1, 5)], 3: [F(3, 40), F(9, 40)], 4: [F(3, 10), F(-9, 10), F(6, 5)],
     5: [F(-11, 54), F(5, 2), F(-70, 27), F(35, 27)],
     6: [F(1631, 55296), F(175, 512), F(575, 13824), F(44275, 110592), F(253, 4096)]}
c = [None, F(37, 378), F(0), F(250, 621), F(125, 594), F(0), F(512, 1771)]
cs = [None, F(2825, 27648), F(0), F(18575, 48384), F(13525, 55296), F(277, 14336), F(1, 4)]


def test_criterion1_tableau_and_nystrom_identities():  # acceptance.cpp:60-90
    for j in range(2, 7):
        assert sum(b[j]) == a[j]                       # row sums are the nodes
    assert sum(c[1:]) == 1 and sum(cs[1:]) == 1
    d = [None] + [c[m] - cs[m] for m in range(1, 7)]
    assert sum(d[1:]) == 0                             # => yErr_q has no v term
    assert c[2] == 0 and cs[2] == 0                    # k6 may reuse k2's slot
    # the RKN coefficients are exact products of tableau entries (rkck_nystrom.cuh rkn)
    bb = {(j, l): sum(b[j][m - 1] * b[m][l - 1] for m in range(l + 1, j)) for j in range(3, 7)
          for l in range(1, j - 1)}
    assert bb[(3, 1)] == b[3][1] * b[2][0]
    assert bb[(6, 4)] == b[6][4] * b[5][3]


def _outer(y0, eps, arith):
    tol = A.default_tol(eps=eps)
    batch = B.BatchStates(1, 28, 0, np.array(y0, dtype=np.float64), np.zeros(0))
    return B.outer_loop(B.problems.pleiades(), batch, 0.0, 1.0, 0.1, solver="rkck", tol=tol,
                        arith=arith).states.values


def _energy(w):
    kin = sum(0.5 * (i + 1) * (w[14 + i] ** 2 + w[21 + i] ** 2) for i in range(7))
    pot = 0.0
    for i in range(7):
        for j in range(i + 1, 7):
            pot -= (i + 1) * (j + 1) / np.hypot(w[i] - w[j], w[7 + i] - w[7 + j])
    return kin + pot


@pytest.mark.gpu
@pytest.mark.parametrize("arith", ["exact", "fast"])
def test_criterion3_pleiades_self_consistency(gpu, arith):  # acceptance.cpp:137-166
    run10 = _outer(PLEIADES_IC, 1e-10, arith)
    run13 = _outer(PLEIADES_IC, 1e-13, arith)
    state_err = np.max(np.abs(run10 - run13)) / np.max(np.abs(run13))
    energy = abs(_energy(run10) - _energy(PLEIADES_IC)) / abs(_energy(PLEIADES_IC))
    m = np.arange(1, 8)
    px, py = np.sum(m * run10[14:21]), np.sum(m * run10[21:28])
    scale = np.sum(m * (np.abs(run10[14:21]) + np.abs(run10[21:28])))
    assert state_err <= 1e-6 and energy <= 1e-6 and np.hypot(px, py) / scale <= 1e-8


@pytest.mark.gpu
def test_criterion4_rkc_beyond_euler_limit(gpu):  # acceptance.cpp:168-203
    n = 64
    sigma = 4.0 * (n + 1.0) ** 2 * np.sin(n * np.pi / (2.0 * (n + 1.0))) ** 2
    tol = A.default_tol(abs_tol=1e-6, rel_tol=1e-3)
    batch = B.BatchStates(1, n, 0, heat_ic(n).copy(), np.zeros(0))
    r = B.integrate_batch(B.problems.heat_equation(n), batch, 0.0, 1.0, solver="rkc", tol=tol)
    assert r.stats["h_max_seen"][0] >= 100.0 * 2.0 / sigma   # 100x the explicit Euler limit
    # the criterion's StepObserver (acceptance.cpp:175-182) through the device
    # step trace: max accepted h and max accepted err <= 1, under both policies
    for arith in ("exact", "fast"):
        _, st, rec = B.trace_steps(B.problems.heat_equation(n), heat_ic(n).copy(), None, 0.0, 1.0,
                                   solver="rkc", arith=arith, tol=tol)
        acc = rec[rec["accepted"] == 1]
        assert len(acc) == st["steps_accepted"] > 0
        assert acc["h"].max() >= 100.0 * 2.0 / sigma and acc["err"].max() <= 1.0
    # max-norm monotone over 50 checkpointed restarts of the same run
    u, prev = heat_ic(n).copy(), 1.0
    for k in range(50):
        bk = B.BatchStates(1, n, 0, u, np.zeros(0))
        u = B.integrate_batch(B.problems.heat_equation(n), bk, k / 50.0, (k + 1) / 50.0,
                              solver="rkc", tol=tol).states.values
        norm = np.max(np.abs(u))
        assert norm <= prev + 1e-15
        prev = norm
