"""heatEquation(n) for any n >= 2 (problems.cpp:94-115) against the oracle:
padded lane-group kernels (HeatPad, csrc/problems.cuh) for n <= 1024 without
an exact-size kernel, and the one-system-per-block kernels (csrc/wide.cuh)
beyond that (and for every n under bode_set_wide(1)).

Bars as in test_gpu_parity.py: EXACT bitwise (states and every counter),
RKCK FAST <= 1e-13 per system with identical counts, RKC FAST reported
against the reference within relTol (its step selection is chaotic at the
ulp level). The reference's own large-dimension smoke case is
test_rkc.cpp:491-512 (dim 1e6).
"""
import numpy as np
import pytest

import paper_1611_02274_b200 as B
from paper_1611_02274_b200 import _abi as A
from golden_cases import perturb, heat_ic
from test_gpu_parity import run_gpu, sysrel, COUNTS

pytestmark = pytest.mark.gpu


def _bitwise(y, st, yo, so):
    assert np.array_equal(y.view(np.uint64), yo.view(np.uint64))
    for k in COUNTS + ("stages_total",):
        assert np.array_equal(st[k], so[k]), k
    assert np.array_equal(st["h_min_seen"], so["h_min_seen"])
    assert np.array_equal(st["h_max_seen"], so["h_max_seen"])


class forced_wide:
    """bode_set_wide(1) for the block: the one-system-per-block kernels even
    where a (padded) lane-group kernel holds the dimension."""
    def __init__(self, on):
        self.on = on

    def __enter__(self):
        B.lib().bode_set_wide(1 if self.on else 0)

    def __exit__(self, *a):
        B.lib().bode_set_wide(0)


@pytest.mark.parametrize("wide", [False, True], ids=["lanes", "blocks"])
@pytest.mark.parametrize("n", [2, 3, 5, 17, 63, 100, 129, 300, 512, 513, 1000, 1025])
def test_heat_any_n_rkc_exact_bitwise(gpu, oracle, n, wide):
    """n <= 1024 runs on padded lane groups (HeatPad, problems.cuh), larger n
    on one system per block; forcing the block kernels checks those at small
    n too."""
    num = 96
    prob = A.make_problem(A.HEAT, n)
    assert B.lib().bode_problem_supported(prob, A.SOLVER_RKC, A.ARITH_EXACT) == 1
    y0 = perturb(heat_ic(n), 0.01, 7 + n, num)
    t1 = 0.2 if n <= 129 else 0.02
    with forced_wide(wide):
        y, st = run_gpu(prob, A.SOLVER_RKC, y0, None, "exact", t1=t1, hout=t1 / 2)
    rc, yo, so, _ = oracle.outer_loop(prob, A.SOLVER_RKC, 0.0, t1, t1 / 2, y0)
    assert rc == 0
    _bitwise(y, st, yo, so)


@pytest.mark.parametrize("n", [9, 12, 40, 70, 78, 90, 104, 110, 120, 140, 150, 180, 200, 210,
                               220, 250, 280, 310, 350, 400, 420, 440, 500])
def test_heat_every_padded_capacity_bitwise(gpu, oracle, n):
    """One n inside every padded RKC capacity (kernels_pad_a.cu / _b.cu: 1, 2,
    4, 8, 16 and 32 lanes, 6-16 components per lane), EXACT bitwise, and FAST
    within relTol of the reference."""
    num = 40
    prob = A.make_problem(A.HEAT, n)
    y0 = perturb(heat_ic(n), 0.01, 13 + n, num)
    t1 = 0.02 if n <= 128 else 0.005
    y, st = run_gpu(prob, A.SOLVER_RKC, y0, None, "exact", t1=t1, hout=t1)
    rc, yo, so, _ = oracle.outer_loop(prob, A.SOLVER_RKC, 0.0, t1, t1, y0)
    assert rc == 0
    _bitwise(y, st, yo, so)
    yf, _ = run_gpu(prob, A.SOLVER_RKC, y0, None, "fast", t1=t1, hout=t1)
    assert sysrel(yf, yo, num, n).max() <= 1e-6


@pytest.mark.parametrize("wide", [False, True], ids=["lanes", "blocks"])
@pytest.mark.parametrize("n,t1", [(2, 0.1), (5, 0.05), (17, 0.01), (40, 5e-3), (60, 2e-3),
                                  (100, 1e-3)])
def test_heat_any_n_rkck_exact_bitwise_and_fast(gpu, oracle, n, t1, wide):
    num = 64
    prob = A.make_problem(A.HEAT, n)
    y0 = perturb(heat_ic(n), 0.01, 3 + n, num)
    rc, yo, so, _ = oracle.outer_loop(prob, A.SOLVER_RKCK, 0.0, t1, t1, y0)
    assert rc == 0
    with forced_wide(wide):
        y, st = run_gpu(prob, A.SOLVER_RKCK, y0, None, "exact", t1=t1, hout=t1)
    _bitwise(y, st, yo, so)
    with forced_wide(wide):
        y, st = run_gpu(prob, A.SOLVER_RKCK, y0, None, "fast", t1=t1, hout=t1)
    assert sysrel(y, yo, num, n).max() <= 1e-13
    for k in ("steps_accepted", "steps_rejected", "rhs_evals"):
        assert np.array_equal(st[k], so[k]), k


@pytest.mark.parametrize("n", [37, 200, 1100, 1250])  # 1100, 1250: FAST-only capacities
def test_heat_any_n_rkc_fast_within_reltol(gpu, oracle, n):
    num = 64
    prob = A.make_problem(A.HEAT, n)
    y0 = perturb(heat_ic(n), 0.01, 11, num)
    y, st = run_gpu(prob, A.SOLVER_RKC, y0, None, "fast", t1=0.1, hout=0.1)
    rc, yo, so, _ = oracle.outer_loop(prob, A.SOLVER_RKC, 0.0, 0.1, 0.1, y0)
    assert sysrel(y, yo, num, n).max() <= 1e-6


@pytest.mark.parametrize("solver", [A.SOLVER_RKC, A.SOLVER_RKCK])
def test_forced_wide_equals_lane_kernels_at_n64(gpu, solver):
    """The block kernel and the 8-lane heat64 kernel are two schedules of the
    same arithmetic: bitwise equal under EXACT."""
    L = B.lib()
    num = 300
    prob = A.make_problem(A.HEAT, 64)
    y0 = perturb(heat_ic(64), 0.01, 5, num)
    t1 = 0.1 if solver == A.SOLVER_RKC else 1e-3
    y_lane, st_lane = run_gpu(prob, solver, y0, None, "exact", t1=t1, hout=t1)
    L.bode_set_wide(1)
    try:
        n0 = L.bode_launch_count()
        y_wide, st_wide = run_gpu(prob, solver, y0, None, "exact", t1=t1, hout=t1)
        assert L.bode_launch_count() > n0
    finally:
        L.bode_set_wide(0)
    _bitwise(y_wide, st_wide, y_lane, st_lane)


def test_heat_global_scratch_path_bitwise(gpu, oracle):
    """n = 4000: 8 n doubles exceed the shared-memory budget, so the vectors
    live in a per-block global scratch (stream-ordered allocation)."""
    n, num = 4000, 6
    prob = A.make_problem(A.HEAT, n)
    y0 = perturb(heat_ic(n), 0.01, 1, num)
    t1 = 1e-3
    y, st = run_gpu(prob, A.SOLVER_RKC, y0, None, "exact", t1=t1, hout=t1)
    rc, yo, so, _ = oracle.outer_loop(prob, A.SOLVER_RKC, 0.0, t1, t1, y0)
    _bitwise(y, st, yo, so)


def test_heat_dim_1e6_smoke(gpu, oracle):
    """One heat system of 10^6 interior points (test_rkc.cpp:491-512's size),
    one short RKC window: bitwise the oracle."""
    n = 1_000_000
    prob = A.make_problem(A.HEAT, n)
    y0 = heat_ic(n).astype(np.float64)
    t1 = 1e-8
    y, st = run_gpu(prob, A.SOLVER_RKC, y0, None, "exact", t1=t1, hout=t1)
    rc, yo, so, _ = oracle.outer_loop(prob, A.SOLVER_RKC, 0.0, t1, t1, y0)
    assert st["steps_accepted"][0] >= 5 and st["stages_total"][0] > 400
    _bitwise(y, st, yo, so)


@pytest.mark.parametrize("n,solver,t1,steps", [(5, "rkck", 0.05, 40), (100, "rkck", 1e-4, 20),
                                               (5, "rkc", 0.05, 10), (100, "rkc", 1e-3, 10),
                                               (4000, "rkc", 1e-7, 3)])
def test_heat_any_n_fixed_step_bitwise(gpu, oracle, n, solver, t1, steps):
    """integrateFixed (rkck.cpp:168-181, rkc.cpp:290-306) on the block kernels,
    including the global-scratch path (n = 4000)."""
    from test_gpu_fixed import oracle_fixed
    num = 12
    prob = A.make_problem(A.HEAT, n)
    y0 = perturb(heat_ic(n), 0.01, 5, num)
    batch = B.BatchStates(num, n, 0, y0.copy(), np.zeros(0))
    out = B.integrate_fixed(B.OdeProblem(prob.kind, n, 0), batch, 0.0, t1, steps, solver=solver,
                            stages=9)
    ref = oracle_fixed(oracle, prob, solver, y0, None, num, 0.0, t1, steps, stages=9)
    assert np.array_equal(out.values.view(np.uint64), ref.view(np.uint64))


@pytest.mark.parametrize("wide", [False, True], ids=["lanes", "blocks"])
@pytest.mark.parametrize("solver", ["rkc", "rkck"])
@pytest.mark.parametrize("n", [17, 100])
def test_heat_any_n_nan_system_freezes(gpu, n, solver, wide):
    """test_batch.cpp:241-258 on the padded and block kernels: a NaN system
    freezes at its initial state with the underflow flag; its neighbours are
    bitwise what they are without it."""
    num = 40
    prob = A.make_problem(A.HEAT, n)
    y0 = perturb(heat_ic(n), 0.01, 5, num)
    bad = y0.copy()
    bad[7 + num * 3] = float("nan")  # component 3 of system 7
    t1 = 1e-3 if solver == "rkck" else 0.05

    def run(y):
        b = B.BatchStates(num, n, 0, y.copy(), np.zeros(0))
        with forced_wide(wide):
            return B.integrate_batch(B.OdeProblem(prob.kind, n, 0), b, 0.0, t1, solver=solver,
                                     arith="exact")

    ref, got = run(y0), run(bad)
    assert got.stats["underflow"][7] == 1
    ys = got.states.values.reshape(n, num)
    assert np.array_equal(ys[:, 7].view(np.uint64), bad.reshape(n, num)[:, 7].view(np.uint64))
    others = np.arange(num) != 7
    assert np.array_equal(ys[:, others].view(np.uint64),
                          ref.states.values.reshape(n, num)[:, others].view(np.uint64))
    assert not got.stats["underflow"][others].any()


@pytest.mark.parametrize("n", [17, 100, 300])
def test_padded_heat_block_size_invariance(gpu, n):
    """The padded lane-group kernels are bitwise independent of the block size
    (batch_driver.hpp:16-21's partition independence, on the device)."""
    L = B.lib()
    num = 333
    prob = A.make_problem(A.HEAT, n)
    y0 = perturb(heat_ic(n), 0.01, 2, num)
    outs = []
    try:
        for block in (0, 64, 256):
            assert L.bode_set_block_size(block) == 0
            outs.append(run_gpu(prob, A.SOLVER_RKC, y0, None, "exact", t1=0.02, hout=0.02))
    finally:
        L.bode_set_block_size(0)
    for y, st in outs[1:]:
        _bitwise(y, st, outs[0][0], outs[0][1])
