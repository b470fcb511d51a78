"""Parity of problems registered through include/bode_problem.cuh: the
built-in extension (Brusselator, csrc/problems_ext.cu) and an out-of-tree
library (examples/user_problem.cu, Lorenz-96), against the REFERENCE drivers
(oracle/_ref) integrating the same right-hand side written as a reference
OdeProblem. EXACT: bitwise states and counters; FAST: the north_star bar."""
import ctypes
import os

import numpy as np
import pytest

import paper_1611_02274_b200 as B
from paper_1611_02274_b200 import _abi as A
from golden_cases import brusselator_ic, brusselator_params, perturb

pytestmark = pytest.mark.gpu

COUNTS = ("steps_accepted", "steps_rejected", "rhs_evals", "spec_rad_evals", "underflow")
USER_LIB = os.path.join(A.PKG_DIR, "lib", "libuser_problem.so")
LORENZ = A.USER_BASE + 96


def sysrel(y, yref, num, dim):
    a = y.reshape(dim, num)
    b = yref.reshape(dim, num)
    return np.max(np.abs(a - b), axis=0) / np.maximum(np.max(np.abs(b), axis=0), 1e-300)


def run(prob, solver, y0, g, arith, t1=1.0):
    num = y0.size // prob.dim
    batch = B.BatchStates(num, prob.dim, prob.param_dim, y0.copy(), g.copy())
    r = B.outer_loop(B.OdeProblem(prob.kind, prob.dim, prob.param_dim), batch, 0.0, t1, 0.1,
                     solver=solver, arith=arith)
    return r.states.values, r.stats


@pytest.mark.parametrize("solver,alpha", [(A.SOLVER_RKC, (0.02, 0.5)),
                                          (A.SOLVER_RKCK, (0.002, 0.02))])
def test_brusselator_exact_bitwise(gpu, ref, solver, alpha):
    num = 1024
    prob = A.make_problem(A.BRUSSELATOR)
    y0 = perturb(brusselator_ic(32), 0.01, 7, num)
    g = brusselator_params(num, *alpha)
    y, st = run(prob, solver, y0, g, "exact")
    rc, yo, so, _ = ref.outer_loop(prob, solver, 0.0, 1.0, 0.1, y0, g)
    assert rc == 0
    assert np.array_equal(y.view(np.uint64), yo.view(np.uint64))
    for k in COUNTS:
        assert np.array_equal(st[k], so[k]), k
    assert st["steps_accepted"].min() > 0


def test_brusselator_fast_within_bar(gpu, ref):
    num = 1024
    prob = A.make_problem(A.BRUSSELATOR)
    y0 = perturb(brusselator_ic(32), 0.01, 7, num)
    g = brusselator_params(num, 0.002, 0.02)
    y, st = run(prob, A.SOLVER_RKCK, y0, g, "fast")
    rc, yo, so, _ = ref.outer_loop(prob, A.SOLVER_RKCK, 0.0, 1.0, 0.1, y0, g)
    assert sysrel(y, yo, num, 64).max() <= 1e-13  # 1e-3 * eps
    for k in ("steps_accepted", "steps_rejected", "rhs_evals"):
        assert np.array_equal(st[k], so[k]), k


@pytest.fixture(scope="module")
def user_lib(gpu):
    return B.api.load_problem_library(USER_LIB)


def _lorenz_inputs(num):
    base = 8.0 + np.sin(np.arange(40))
    y0 = perturb(base, 0.01, 11, num)
    g = np.linspace(6.0, 10.0, num)
    return y0, g


@pytest.mark.parametrize("solver", [A.SOLVER_RKCK, A.SOLVER_RKC])
def test_out_of_tree_problem_exact_bitwise(user_lib, ref, solver):
    num = 512
    prob = A.Problem(kind=LORENZ, dim=40, param_dim=1, reserved=0)
    y0, g = _lorenz_inputs(num)
    y, st = run(prob, solver, y0, g, "exact", t1=0.5)
    rhs = ctypes.cast(user_lib.bode_example_lorenz96_rhs, ctypes.c_void_p).value
    rc, yo, so, _ = ref.outer_loop_fn(rhs, 40, 1, solver, 0.0, 0.5, 0.1, y0, g)
    assert rc == 0
    assert np.array_equal(y.view(np.uint64), yo.view(np.uint64))
    for k in COUNTS:
        assert np.array_equal(st[k], so[k]), k


def test_out_of_tree_problem_fast(user_lib, ref):
    num = 512
    prob = A.Problem(kind=LORENZ, dim=40, param_dim=1, reserved=0)
    y0, g = _lorenz_inputs(num)
    y, st = run(prob, A.SOLVER_RKCK, y0, g, "fast", t1=0.5)
    rhs = ctypes.cast(user_lib.bode_example_lorenz96_rhs, ctypes.c_void_p).value
    rc, yo, so, _ = ref.outer_loop_fn(rhs, 40, 1, A.SOLVER_RKCK, 0.0, 0.5, 0.1, y0, g)
    # chaotic flow: FMA-level differences grow, but stay far inside 1e-3 * eps
    assert sysrel(y, yo, num, 40).max() <= 1e-13


NBODY = A.USER_BASE + 97


def _nbody_inputs(num):
    nb = 5
    ang = 2 * np.pi * np.arange(nb) / nb
    pos = np.stack([1.5 * np.cos(ang), 1.5 * np.sin(ang), 0.2 * np.sin(2 * ang)], axis=1).reshape(-1)
    vel = np.stack([-0.9 * np.sin(ang), 0.9 * np.cos(ang), 0.05 * np.cos(ang)], axis=1).reshape(-1)
    y0 = perturb(np.concatenate([pos, vel]), 0.01, 13, num)
    m = 1.0 + 0.5 * np.sin(np.arange(num * nb) * 0.37).reshape(nb, num)  # SoA masses
    return y0, m.reshape(-1)


@pytest.mark.parametrize("solver", [A.SOLVER_RKCK, A.SOLVER_RKC])
def test_second_order_user_problem_exact_bitwise(user_lib, ref, solver):
    """An out-of-tree second-order problem (bode::SecondOrderProblem): RKCK runs
    the Nystrom kernel, RKC the generic one; both bitwise the reference drivers."""
    num = 512
    prob = A.Problem(kind=NBODY, dim=30, param_dim=5, reserved=0)
    y0, m = _nbody_inputs(num)
    y, st = run(prob, solver, y0, m, "exact", t1=0.5)
    rhs = ctypes.cast(user_lib.bode_example_nbody_rhs, ctypes.c_void_p).value
    rc, yo, so, _ = ref.outer_loop_fn(rhs, 30, 5, solver, 0.0, 0.5, 0.1, y0, m)
    assert rc == 0
    assert np.array_equal(y.view(np.uint64), yo.view(np.uint64))
    for k in COUNTS:
        assert np.array_equal(st[k], so[k]), k


def test_second_order_user_problem_fast_rkn(user_lib, ref):
    """FAST RKCK on it runs in Runge-Kutta-Nystrom form: within 1e-3 * eps of
    the reference with identical step counts."""
    num = 512
    prob = A.Problem(kind=NBODY, dim=30, param_dim=5, reserved=0)
    y0, m = _nbody_inputs(num)
    y, st = run(prob, A.SOLVER_RKCK, y0, m, "fast", t1=0.5)
    rhs = ctypes.cast(user_lib.bode_example_nbody_rhs, ctypes.c_void_p).value
    rc, yo, so, _ = ref.outer_loop_fn(rhs, 30, 5, A.SOLVER_RKCK, 0.0, 0.5, 0.1, y0, m)
    assert sysrel(y, yo, num, 30).max() <= 1e-13
    for k in ("steps_accepted", "steps_rejected", "rhs_evals"):
        assert np.array_equal(st[k], so[k]), k


@pytest.mark.parametrize("env", [("4", "255"), ("8", "128")])
def test_brusselator_rkc_lane_variants_bitwise(gpu, ref, env):
    """Both compiled RKC Brusselator shapes (4 lanes uncapped, the default, and
    8 lanes at 128 registers; BODE_LANES / BODE_MAXREG) give the reference's bits."""
    import os
    import subprocess
    import sys
    num = 512
    code = ("import sys; sys.path.insert(0, 'tests'); import numpy as np;"
            "from test_gpu_user_problems import run; from golden_cases import brusselator_ic,"
            " brusselator_params, perturb; from paper_1611_02274_b200 import _abi as A;"
            "p = A.make_problem(A.BRUSSELATOR); y0 = perturb(brusselator_ic(32), 0.01, 11, %d);"
            "g = brusselator_params(%d, 0.02, 0.5);"
            "y, st = run(p, A.SOLVER_RKC, y0, g, 'exact'); np.save(sys.argv[1], y)" % (num, num))
    out = os.path.join(os.environ.get("TMPDIR", "/tmp"), f"bru_variant_{env[0]}_{env[1]}.npy")
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code, out], cwd=repo, capture_output=True, text=True,
                       env=dict(os.environ, BODE_LANES=env[0], BODE_MAXREG=env[1]))
    assert r.returncode == 0, r.stderr[-2000:]
    prob = A.make_problem(A.BRUSSELATOR)
    y0 = perturb(brusselator_ic(32), 0.01, 11, num)
    g = brusselator_params(num, 0.02, 0.5)
    rc, yo, so, _ = ref.outer_loop(prob, A.SOLVER_RKC, 0.0, 1.0, 0.1, y0, g)
    assert rc == 0
    assert np.array_equal(np.load(out).view(np.uint64), yo.view(np.uint64))
