"""Pin the C restatement (oracle/bode_oracle.c) to the reference test suites'
known-answer values, transcribed from proj/tests/*.cpp (file:line cited)."""
import ctypes
import math

import numpy as np
import pytest

from paper_1611_02274_b200 import _abi as A
from oracle_lib import OBS


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


P_DECAY = A.make_problem(A.DIAG, 1)  # y' = g0*y with g0 = -1
G_DECAY = np.array([-1.0])


def test_splitmix64_kats(oracle):  # test_problems.cpp:189-191
    assert oracle.lib.orc_splitmix64_at(0, 0) == 0xe220a8397b1dcdaf
    assert oracle.lib.orc_splitmix64_at(0, 1) == 0x6e789e6aa1b965f4
    assert oracle.lib.orc_splitmix64_at(0, 2) == 0x06c45d188009454f
    u = oracle.lib.orc_unit_symmetric_at(0, 0)
    assert -1.0 <= u < 1.0


def test_perturb_bounds_and_zero_components(oracle):  # test_problems.cpp:160-200
    base = np.array([3.0, -1.5, 0.0, 2.0e3])
    rc, b0 = oracle.perturb(base, 0.0, 9, 11)
    assert rc == 0 and np.all(b0.reshape(4, 11).T == base)
    rc, b = oracle.perturb(base, 0.01, 42, 1024)
    b = b.reshape(4, 1024).T
    assert np.all(b[:, 2] == 0.0)
    nz = base != 0
    assert np.all(np.abs(b[:, nz] / base[nz] - 1.0) <= 0.01)
    assert oracle.perturb(base, 0.5, 1, 4)[0] == A.E_INVALID_SHAPE
    assert oracle.perturb(base, 0.01, 1, 0)[0] == A.E_INVALID_SHAPE


def test_rkck_step_decay_kat(oracle):  # test_rkck.cpp:75-84
    y, f = np.array([1.0]), np.array([-1.0])
    yn, ye = np.empty(1), np.empty(1)
    oracle.lib.orc_rkck_step(ctypes.byref(P_DECAY), 0.0, A.dptr(y), A.dptr(G_DECAY), A.dptr(f),
                             0.1, A.dptr(yn), A.dptr(ye))
    assert rel(yn[0], 0.90483741791666672) < 1e-15
    assert abs(ye[0] - 2.4232991536458335e-09) < 1e-17


def test_rkck_zero_rhs_exact(oracle):  # test_rkck.cpp:62-66
    p = A.make_problem(A.ZERO, 1)
    y, f = np.array([3.5]), np.array([0.0])
    yn, ye = np.empty(1), np.empty(1)
    oracle.lib.orc_rkck_step(ctypes.byref(p), 0.0, A.dptr(y), None, A.dptr(f), 0.7, A.dptr(yn),
                             A.dptr(ye))
    assert yn[0] == 3.5 and ye[0] == 0.0


def test_rkck_adjust_step_kats(oracle):  # test_rkck.cpp:129-160
    tol = A.default_tol()
    acc, h = ctypes.c_int(), ctypes.c_double()

    def adj(hh, err, nan=0, hmin=1e-20, hmax=100.0):
        oracle.lib.orc_rkck_adjust_step(hh, err, nan, hmin, hmax, ctypes.byref(tol),
                                        ctypes.byref(acc), ctypes.byref(h))
        return acc.value, h.value

    a, hn = adj(0.1, 0.5)
    assert a and rel(hn, 0.10338285194973316) < 1e-14
    assert adj(0.1, 1e-6) == (1, 0.5)
    a, hn = adj(0.1, float("nan"))
    assert not a and rel(hn, 0.01) < 1e-14
    assert adj(0.1, 0.5, nan=1)[0] == 0
    a, hn = adj(0.1, 2.0)
    assert not a and rel(hn, 0.9 * 0.1 * 2.0 ** -0.25) < 1e-12
    assert rel(adj(0.1, 1e9)[1], 0.01) < 1e-12
    assert adj(0.1, 1e-6, hmax=0.3)[1] == 0.3


def test_rkck_driver_zero_rhs_two_steps(oracle):  # test_rkck.cpp:178-194
    rc, y, st = oracle.driver(A.make_problem(A.ZERO, 2), A.SOLVER_RKCK, 0.0, 3.0, [1.25, -7.0])
    assert rc == 0 and list(y) == [1.25, -7.0]
    assert st["steps_accepted"] == 2 and st["steps_rejected"] == 0
    assert st["h_min_seen"] == 1.5 and st["h_max_seen"] == 1.5


def test_rkck_driver_accuracy(oracle):  # test_rkck.cpp:196-206, :267-273
    _, y, _ = oracle.driver(P_DECAY, A.SOLVER_RKCK, 0.0, 1.0, [1.0], G_DECAY)
    assert rel(y[0], 0.36787944117144233) < 1e-8
    _, y, _ = oracle.driver(A.make_problem(A.RICCATI), A.SOLVER_RKCK, 0.0, 0.5, [1.0])
    assert rel(y[0], 2.0) < 1e-7
    _, y, _ = oracle.driver(A.make_problem(A.HARMONIC), A.SOLVER_RKCK, 0.0, 2 * math.pi, [1.0, 0.0])
    assert abs(y[0] ** 2 + y[1] ** 2 - 1.0) < 1e-7


def test_rkck_observer_accepted_steps_satisfy_bound(oracle):  # test_rkck.cpp:208-218
    recs = []
    oracle.driver(A.make_problem(A.RICCATI), A.SOLVER_RKCK, 0.0, 0.5, [1.0],
                  observer=lambda t, h, s, err, acc, u: recs.append((err, acc)))
    assert recs and all(err <= 1.0 for err, acc in recs if acc)


def test_rkck_empty_interval(oracle):  # test_rkck.cpp:237-242
    rc, _, _ = oracle.driver(P_DECAY, A.SOLVER_RKCK, 1.0, 1.0, [1.0], G_DECAY)
    assert rc == A.E_INVALID_INTERVAL


def test_rkck_order_five(oracle):  # test_rkck.cpp:244-254
    hs, errs = [], []
    for n in (10, 20, 40, 80):
        y = np.array([1.0])
        oracle.lib.orc_rkck_integrate_fixed(ctypes.byref(P_DECAY), 0.0, 1.0, n, A.dptr(y),
                                            A.dptr(G_DECAY))
        hs.append(1.0 / n)
        errs.append(abs(y[0] - 0.36787944117144233))
    slope = np.polyfit(np.log(hs), np.log(errs), 1)[0]
    assert abs(slope - 5.0) <= 0.3


def test_chebyshev_kats(oracle):  # test_rkc.cpp:60-75
    out = np.empty(3)
    oracle.lib.orc_chebyshev_eval(0, 2.7, A.dptr(out))
    assert list(out) == [1.0, 0.0, 0.0]
    oracle.lib.orc_chebyshev_eval(1, -1.3, A.dptr(out))
    assert list(out) == [-1.3, 1.0, 0.0]
    oracle.lib.orc_chebyshev_eval(2, 1.5, A.dptr(out))
    assert list(out) == [3.5, 6.0, 4.0]


def test_rkc_coefficient_identities(oracle):  # test_rkc.cpp:94-124
    cf = oracle.coefficients(2)
    assert rel(cf["omega0"], 27.0 / 26.0) < 1e-15
    assert oracle.coefficients(1)["rc"] == A.E_INVALID_STAGE_COUNT
    cf0 = oracle.coefficients(2, 0.0)
    assert cf0["omega0"] == 1.0 and cf0["b"][1] == 1.0 and cf0["c"][2] == 1.0
    assert rel(cf0["c"][1], 0.25) < 1e-15
    cf10 = oracle.coefficients(10)
    for j in range(2, 10):
        assert abs(cf10["c"][j] - (j * j - 1.0) / 99.0) <= 5e-3
    for s in range(2, 51):
        cf = oracle.coefficients(s)
        assert cf["c"][s] == 1.0 and cf["b"][0] == cf["b"][2] and cf["c"][1] > 0
        assert all(cf["c"][j] > cf["c"][j - 1] for j in range(2, s + 1))


def test_rkc_step_lambda_kat_and_zero_fixed_point(oracle):  # test_rkc.cpp:126-167
    p = A.make_problem(A.DIAG, 1)
    g = np.array([-10.0])
    y, f, out = np.array([1.0]), np.array([-10.0]), np.empty(1)
    oracle.lib.orc_rkc_step(ctypes.byref(p), 0.0, A.dptr(y), A.dptr(g), A.dptr(f), 0.1, 5,
                            2.0 / 13.0, A.dptr(out))
    assert rel(out[0], 0.41776078685534035) < 1e-12
    z = A.make_problem(A.ZERO, 3)
    y3 = np.array([1.2345, -6.789e3, 1e-12])
    f3 = np.zeros(3)
    o3 = np.empty(3)
    for s in range(2, 51):
        oracle.lib.orc_rkc_step(ctypes.byref(z), 0.0, A.dptr(y3), None, A.dptr(f3), 0.37, s,
                                2.0 / 13.0, A.dptr(o3))
        assert np.array_equal(o3, y3)


def test_rkc_stage_count_kats(oracle):  # test_rkc.cpp:240-282
    s, h = ctypes.c_int(), ctypes.c_double()
    u = 2.22e-16

    def sc(hh, sig, rt=1e-6):
        oracle.lib.orc_rkc_stage_count(hh, sig, rt, u, ctypes.byref(s), ctypes.byref(h))
        return s.value, h.value

    assert sc(1.0, 0.0) == (2, 1.0)
    assert sc(1.0, 100.0) == (13, 1.0)
    st, hh = sc(1.0, 3.0e8)
    assert st == 21224 and rel(hh, (21224.0 ** 2 - 1.0) / (1.54 * 3.0e8)) < 1e-12
    rt = 2500.0 * u
    h16 = (15.5 ** 2 - 1.0) / (1.54 * 1e4)
    assert sc(h16, 1e4, rt) == (16, h16)
    h17 = (16.5 ** 2 - 1.0) / (1.54 * 1e4)
    st, hh = sc(h17, 1e4, rt)
    assert st == 16 and rel(hh, (16.0 ** 2 - 1.0) / (1.54 * 1e4)) < 1e-12 and hh < h17


def test_rkc_initial_step_kat(oracle):  # test_rkc.cpp:284-325
    tol = A.default_tol()
    p = A.make_problem(A.DIAG, 1)
    y, f, g = np.array([1.0]), np.array([-1.0]), np.array([-1.0])
    h, e = ctypes.c_double(), ctypes.c_double()
    oracle.lib.orc_rkc_initial_step(ctypes.byref(p), 0.0, A.dptr(y), A.dptr(g), A.dptr(f), 1.0,
                                    10.0, 1e-20, ctypes.byref(tol), ctypes.byref(h), ctypes.byref(e))
    assert rel(e.value, 999900.00999900012) < 1e-12
    assert rel(h.value, 0.00010000499987500625) < 1e-12
    z = A.make_problem(A.ZERO, 1)
    oracle.lib.orc_rkc_initial_step(ctypes.byref(z), 0.0, A.dptr(y), None, A.dptr(np.zeros(1)),
                                    0.0, 5.0, 1e-20, ctypes.byref(tol), ctypes.byref(h),
                                    ctypes.byref(e))
    assert e.value == 0.0 and h.value == 5.0


def test_rkc_next_step_kats(oracle):  # test_rkc.cpp:327-342
    inf = float("inf")
    L = oracle.lib
    assert rel(L.orc_rkc_next_step_accepted(0.512, 0.0, 0.25, 0.0, 1, 0.0, inf), 0.25) < 1e-14
    a = L.orc_rkc_next_step_accepted(0.2, 0.2, 0.03, 0.03, 0, 0.0, inf)
    assert rel(a, 0.03 * min(10.0, 0.8 / 0.2 ** (1 / 3))) < 1e-13
    assert rel(L.orc_rkc_next_step_rejected(8.0, 0.5), 0.2) < 1e-14


def test_rkc_driver_kats(oracle):  # test_rkc.cpp:363-385, :465-477
    rc, y, st = oracle.driver(A.make_problem(A.ZERO, 2), A.SOLVER_RKC, 0.0, 2.0, [4.0, -0.5])
    assert list(y) == [4.0, -0.5] and st["steps_accepted"] == 1 and st["steps_rejected"] == 0
    rc, y, st = oracle.driver(P_DECAY, A.SOLVER_RKC, 0.0, 1.0, [1.0], G_DECAY)
    assert rel(y[0], 0.36787944117144233) < 1e-4 and st["spec_rad_evals"] > 0
    assert st["rhs_evals"] > st["steps_accepted"]
    nanp = A.make_problem(A.EXPDECAY)
    rc, y, st = oracle.driver(nanp, A.SOLVER_RKC, 0.0, 1.0, [1.0], np.array([np.nan]))
    assert st["underflow"] == 1 and y[0] == 1.0


def test_rkc_order_two(oracle):  # test_rkc.cpp:479-489
    hs, errs = [], []
    for n in (20, 40, 80, 160):
        y = np.array([1.0])
        oracle.lib.orc_rkc_integrate_fixed(ctypes.byref(P_DECAY), 0.0, 1.0, n, 5, 2.0 / 13.0,
                                           A.dptr(y), A.dptr(G_DECAY))
        hs.append(1.0 / n)
        errs.append(abs(y[0] - 0.36787944117144233))
    assert abs(np.polyfit(np.log(hs), np.log(errs), 1)[0] - 2.0) <= 0.2


def _power(oracle, p, y, v, hmax, g=None):
    f = oracle.rhs(p, y, g)
    sig, it, cv = ctypes.c_double(), ctypes.c_int(), ctypes.c_int()
    eig = np.empty(p.dim)
    y = np.ascontiguousarray(y, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    oracle.lib.orc_power_method(ctypes.byref(p), 0.0, A.dptr(y), A.dptr(g), A.dptr(f), hmax,
                                A.dptr(v), ctypes.byref(sig), A.dptr(eig), ctypes.byref(it),
                                ctypes.byref(cv))
    return sig.value, it.value, cv.value


def test_power_method_kats(oracle):  # test_specrad.cpp:35-69
    p = A.make_problem(A.DIAG, 3)
    s, it, cv = _power(oracle, p, [1.0, 1.0, 1.0], [1.0, 1.0, 1.0], 10.0, np.array([-1.0, -10.0, -100.0]))
    assert cv and 100.0 <= s <= 130.0 and it <= 50
    s, it, cv = _power(oracle, A.make_problem(A.ZERO, 4), [1.0, 2.0, 3.0, 4.0], [1.0, 0, 0, 0], 2.0)
    assert s == 0.0 and cv
    hp = A.make_problem(A.HEAT, 64)
    u0 = np.empty(64)
    oracle.lib.orc_heat_initial_condition(64, A.dptr(u0))
    f = oracle.rhs(hp, u0)
    star = oracle.lib.orc_heat_spectral_radius(64)
    assert rel(star, 16890.13232) < 1e-6
    s, _, _ = _power(oracle, hp, u0, f, 1.0)
    assert star <= s <= 1.35 * star


def test_heat_stencil_kats(oracle):  # test_problems.cpp:113-144
    p2 = A.make_problem(A.HEAT, 2)
    out = oracle.rhs(p2, [1.0, 0.0])
    assert rel(out[0], -18.0) < 1e-14 and rel(out[1], 9.0) < 1e-14
    n = 64
    dx = 1.0 / (n + 1)
    u = np.sin((np.arange(n) + 1) * math.pi * dx)
    lam1 = 4.0 / dx ** 2 * math.sin(math.pi * dx / 2) ** 2
    out = oracle.rhs(A.make_problem(A.HEAT, n), u)
    assert np.all(np.abs(out + lam1 * u) <= 1e-11 * np.abs(lam1 * u))


def test_pleiades_rhs_cases(oracle):  # test_problems.cpp:30-70
    p = A.make_problem(A.PLEIADES)
    w = np.zeros(28)
    w[1] = 1.0
    for i in range(2, 7):
        w[i] = 1.0e8 + 1.0e6 * i
        w[7 + i] = 1.0e8 - 1.0e6 * i
    out = oracle.rhs(p, w)
    assert np.all(out[:14] == 0.0)
    assert rel(out[14], 2.0) < 1e-12 and rel(out[15], -1.0) < 1e-12
    w = np.zeros(28)
    w[:7] = 3.0 * np.arange(7)
    assert np.all(oracle.rhs(p, w)[21:] == 0.0)


def test_pleiades_conservation(oracle):  # test_problems.cpp:96-111
    from paper_1611_02274_b200.api import problems  # host helper, no device needed
    ic = problems.pleiades_initial_conditions()
    _, w, _ = oracle.driver(A.make_problem(A.PLEIADES), A.SOLVER_RKCK, 0.0, 1.0, ic)
    e0 = oracle.lib.orc_pleiades_energy(A.dptr(ic))
    e1 = oracle.lib.orc_pleiades_energy(A.dptr(w))
    assert abs(e1 - e0) / abs(e0) < 1e-6


def test_outer_loop_window_count(oracle):  # test_batch.cpp:171-192
    z = A.make_problem(A.ZERO, 1)
    for span, hout, n in ((1.0, 0.1, 10), (1.0, 1.0, 1), (1.05, 0.1, 11)):
        rc, _, _, steps = oracle.outer_loop(z, A.SOLVER_RKCK, 0.0, span, hout, np.array([1.0]))
        assert rc == 0 and steps == n
    assert oracle.outer_loop(z, 0, 0.0, 1.0, 0.0, np.array([1.0]))[0] == A.E_INVALID_INTERVAL
    assert oracle.outer_loop(z, 0, 1.0, 0.5, 0.1, np.array([1.0]))[0] == A.E_INVALID_INTERVAL


def test_batch_nan_isolation(oracle):  # test_batch.cpp:241-258
    p = A.make_problem(A.EXPDECAY)
    rc, y, st = oracle.integrate_batch(p, A.SOLVER_RKCK, 0.0, 1.0, np.array([1.0, 1.0]),
                                       np.array([np.nan, 1.0]), threads=2)
    assert st[0]["underflow"] == 1 and y[0] == 1.0
    assert st[1]["underflow"] == 0 and rel(y[1], math.exp(-1.0)) < 1e-8


def test_batch_worker_invariance(oracle):  # test_batch.cpp:127-142
    from paper_1611_02274_b200.api import problems
    ic = problems.pleiades_initial_conditions()
    _, y0 = oracle.perturb(ic, 0.01, 20140609, 256)
    p = A.make_problem(A.PLEIADES)
    ref = oracle.integrate_batch(p, 0, 0.0, 0.1, y0, threads=1)[1]
    for w in (2, 4, 8):
        assert np.array_equal(oracle.integrate_batch(p, 0, 0.0, 0.1, y0, threads=w)[1], ref)
