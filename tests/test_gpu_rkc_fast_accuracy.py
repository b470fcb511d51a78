"""RKC FAST against the exact solution (SURVEY.md 7.4 hard part 2).

RKC's step selection is chaotic at the ulp level, so the FAST policy (FMA
contraction, pairwise sums, libdevice cbrt) cannot match the reference
bitwise. Its claim is equal *accuracy*: both policies are
compared with the exact solution of the linear test problems, and FAST's
global error must be of the same size as EXACT's (= the reference's).

  heat n=64: u' = A u, A the (1,-2,1)/dx^2 stencil; u(1) = V exp(L) V^T u0
             with A = V L V^T (problems.cpp:94-115).
  expDecay:  y(1) = y0 exp(-g0)  (problems.cpp:134-144), g0 in [1, 1e4].
Error unit: max_j |y_j - y*_j| / (absTol + relTol |y*_j|), the RKC norm's
weight (rkc.cpp:122-127).
"""
import numpy as np
import pytest

import paper_1611_02274_b200 as B
from golden_cases import heat_ic

pytestmark = pytest.mark.gpu


def heat_exact(y0, n, num, t):
    dx = 1.0 / (n + 1)
    A = (np.diag(-2.0 * np.ones(n)) + np.diag(np.ones(n - 1), 1) + np.diag(np.ones(n - 1), -1)) \
        / (dx * dx)
    lam, V = np.linalg.eigh(A)
    E = V @ np.diag(np.exp(lam * t)) @ V.T
    return (E @ y0.reshape(n, num)).reshape(-1)


def weighted(y, ys, dim, num):
    w = np.abs(y - ys) / (1e-10 + 1e-6 * np.abs(ys))
    return w.reshape(dim, num).max(axis=0)


def run(prob, b, arith):
    r = B.outer_loop(prob, b, 0.0, 1.0, 0.1, solver="rkc", arith=arith)
    return r.states.values, r.stats


def test_heat64_fast_as_accurate_as_exact():
    n, num = 64, 1 << 14
    b = B.problems.perturb_initial_conditions(heat_ic(n), 0.01, 42, num)
    truth = heat_exact(b.values, n, num, 1.0)
    ye, se = run(B.problems.heat_equation(n), b, "exact")
    yf, sf = run(B.problems.heat_equation(n), b, "fast")
    ee, ef = weighted(ye, truth, n, num), weighted(yf, truth, n, num)
    print(f"heat64 error vs exact solution (tolerance units): EXACT median {np.median(ee):.3g} "
          f"p99 {np.percentile(ee, 99):.3g} max {ee.max():.3g}; FAST median {np.median(ef):.3g} "
          f"p99 {np.percentile(ef, 99):.3g} max {ef.max():.3g}; steps EXACT "
          f"{se['steps_accepted'].mean():.2f} FAST {sf['steps_accepted'].mean():.2f}")
    assert np.median(ef) <= 1.5 * np.median(ee) and ef.max() <= 1.5 * ee.max()


def test_expdecay_stiff_fast_as_accurate_as_exact():
    from paper_1611_02274_b200.api import stiffness_params
    num = 1 << 16
    b = B.problems.perturb_initial_conditions(np.array([1.0]), 0.01, 42, num)
    b.param_dim, b.params = 1, stiffness_params(num)
    truth = b.values * np.exp(-b.params)
    ye, _ = run(B.problems.exp_decay(), b, "exact")
    yf, _ = run(B.problems.exp_decay(), b, "fast")
    ee, ef = weighted(ye, truth, 1, num), weighted(yf, truth, 1, num)
    print(f"expDecay error vs exact solution (tolerance units): EXACT median {np.median(ee):.3g} "
          f"max {ee.max():.3g}; FAST median {np.median(ef):.3g} max {ef.max():.3g}")
    assert np.median(ef) <= 1.5 * np.median(ee) and ef.max() <= 1.5 * ee.max()
