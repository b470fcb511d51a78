"""The reference test suites' behavioural KATs, run through the GPU path
(proj/tests/test_rkck.cpp, test_rkc.cpp, test_batch.cpp)."""
import math

import numpy as np
import pytest

import paper_1611_02274_b200 as B

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("solver", ["rkck", "rkc"])
@pytest.mark.parametrize("arith", ["exact", "fast"])
def test_zero_rhs_identity(gpu, solver, arith):  # test_batch.cpp:102-114
    b = B.pack([[1.0, -2.5], [3.25, 4.0], [0.0, 1e-8]])
    r = B.integrate_batch(B.problems.zero(2), b, 0.0, 1.0, solver=solver, arith=arith)
    assert np.array_equal(r.states.values, b.values)
    assert np.all(r.stats["steps_accepted"] >= 1)
    assert np.all(r.stats["rhs_evals"] >= r.stats["steps_accepted"])
    assert not r.stats["underflow"].any()


def test_zero_rhs_step_counts(gpu):  # test_rkck.cpp:178-194, test_rkc.cpp:363-375
    b = B.pack([[1.25, -7.0]])
    r = B.integrate_batch(B.problems.zero(2), b, 0.0, 3.0, solver="rkck")
    st = r.stats[0]
    assert st["steps_accepted"] == 2 and st["steps_rejected"] == 0
    assert st["h_min_seen"] == 1.5 and st["h_max_seen"] == 1.5
    r = B.integrate_batch(B.problems.zero(2), B.pack([[4.0, -0.5]]), 0.0, 2.0, solver="rkc")
    assert r.stats[0]["steps_accepted"] == 1 and r.stats[0]["steps_rejected"] == 0


@pytest.mark.parametrize("solver", ["rkck", "rkc"])
def test_linear_decay(gpu, solver):  # test_batch.cpp:116-125, test_rkc.cpp:377-385
    b = B.pack([[1.0], [2.0], [3.0], [4.0]], [[1.0]] * 4)
    r = B.integrate_batch(B.problems.exp_decay(), b, 0.0, 1.0, solver=solver)
    tolr = 1e-8 if solver == "rkck" else 1e-4
    for i in range(4):
        assert abs(r.states.at(i, 0) - (i + 1) * math.exp(-1.0)) <= tolr * (i + 1) * math.exp(-1.0)
    if solver == "rkc":
        assert np.all(r.stats["spec_rad_evals"] > 0)


def test_riccati_and_harmonic(gpu):  # test_rkck.cpp:202-206, :267-273
    r = B.integrate_batch(B.problems.riccati(), B.pack([[1.0]]), 0.0, 0.5)
    assert abs(r.states.at(0, 0) - 2.0) < 1e-7 * 2.0
    r = B.integrate_batch(B.problems.harmonic(), B.pack([[1.0, 0.0]]), 0.0, 2 * math.pi)
    q, p = r.states.at(0, 0), r.states.at(0, 1)
    assert abs(q * q + p * p - 1.0) < 1e-7


@pytest.mark.parametrize("solver", ["rkck", "rkc"])
def test_nan_system_freezes_neighbour_unaffected(gpu, solver):  # test_batch.cpp:241-258
    b = B.pack([[1.0], [1.0]], [[float("nan")], [1.0]])
    r = B.integrate_batch(B.problems.exp_decay(), b, 0.0, 1.0, solver=solver)
    assert r.stats[0]["underflow"] == 1 and r.states.at(0, 0) == 1.0
    assert r.stats[1]["underflow"] == 0
    assert abs(r.states.at(1, 0) - math.exp(-1.0)) < (1e-8 if solver == "rkck" else 1e-4)


def test_system_isolation(gpu):  # test_batch.cpp:154-169
    y0 = [1.0, 2.0, 3.0, 4.0, 5.0]
    mk = lambda ys: B.pack([[v] for v in ys], [[1.0]] * len(ys))
    base = B.integrate_batch(B.problems.exp_decay(), mk(y0), 0.0, 1.0)
    y0[2] += 1e-3
    bumped = B.integrate_batch(B.problems.exp_decay(), mk(y0), 0.0, 1.0)
    for i in range(5):
        same = bumped.states.at(i, 0) == base.states.at(i, 0)
        assert same != (i == 2)


def test_sink_cadence(gpu):  # test_batch.cpp:171-192
    b = B.pack([[1.0, 2.0]])
    for span, hout, n in ((1.0, 0.1, 10), (1.0, 1.0, 1), (1.05, 0.1, 11)):
        times = []
        r = B.outer_loop(B.problems.zero(2), b, 0.0, span, hout, sink=lambda t, s: times.append(t))
        assert len(times) == n and r.outer_steps == n and times[-1] == span


def test_restart_windows_agree_with_single_window(gpu):  # test_batch.cpp:194-205
    b = B.pack([[1.0]], [[1.0]])
    multi = B.outer_loop(B.problems.exp_decay(), b, 0.0, 1.0, 0.1)
    single = B.outer_loop(B.problems.exp_decay(), b, 0.0, 1.0, 1.0)
    e = math.exp(-1.0)
    assert abs(multi.states.at(0, 0) - e) < 1e-8 * e and abs(single.states.at(0, 0) - e) < 1e-8 * e
    assert multi.outer_steps == 10 and single.outer_steps == 1


def test_stats_sanity(gpu):  # test_batch.cpp:217-228
    b = B.pack([[1.0], [5.0]], [[1.0], [1.0]])
    r = B.integrate_batch(B.problems.exp_decay(), b, 0.0, 1.0, solver="rkc")
    for st in r.stats:
        assert st["steps_accepted"] > 0 and st["rhs_evals"] >= st["steps_accepted"]
        assert st["spec_rad_evals"] > 0 and 0 < st["h_min_seen"] <= st["h_max_seen"]


def test_launch_counter_advances(gpu):
    n0 = B.lib().bode_launch_count()
    B.integrate_batch(B.problems.zero(2), B.pack([[1.0, 2.0]]), 0.0, 1.0)
    assert B.lib().bode_launch_count() > n0


@pytest.mark.parametrize("arith", ["exact", "fast"])
@pytest.mark.parametrize("problem", ["pleiades", "expdecay"])
def test_nan_freeze_all_paths(gpu, arith, problem):
    """rkck.cpp:150-154 on every RKCK kernel path: the Nystrom/RKN Pleiades
    kernels (FAST, 1 lane), the lane-pair kernel (EXACT) and the generic one
    (expDecay). A NaN system freezes with the underflow flag; every other
    system is bitwise what it is without the NaN neighbour."""
    import numpy as np
    from paper_1611_02274_b200 import _abi as A
    from golden_cases import PLEIADES_IC, perturb
    num = 64
    if problem == "pleiades":
        prob, base, g = A.make_problem(A.PLEIADES), PLEIADES_IC, None
    else:
        prob, base = A.make_problem(A.EXPDECAY), np.array([1.0])
        g = np.linspace(0.5, 5.0, num)
    y0 = perturb(base, 0.01, 5, num)
    bad = y0.copy()
    bad[7 + num * min(3, prob.dim - 1)] = float("nan")  # one component of system 7

    def run(y):
        b = B.BatchStates(num, prob.dim, prob.param_dim, y.copy(),
                          g.copy() if g is not None else np.zeros(0))
        return B.integrate_batch(B.OdeProblem(prob.kind, prob.dim, prob.param_dim), b, 0.0, 0.1,
                                 solver="rkck", arith=arith)

    ref, got = run(y0), run(bad)
    assert got.stats["underflow"][7] == 1
    ys = got.states.values.reshape(prob.dim, num)
    assert np.array_equal(ys[:, 7].view(np.uint64), bad.reshape(prob.dim, num)[:, 7].view(np.uint64))
    others = np.arange(num) != 7
    assert np.array_equal(ys[:, others].view(np.uint64),
                          ref.states.values.reshape(prob.dim, num)[:, others].view(np.uint64))
    assert not got.stats["underflow"][others].any()
