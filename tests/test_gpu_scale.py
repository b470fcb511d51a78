"""Parity at BASELINE config 5's size (2^24 systems on one B200) and config 4
at 2^22, by deterministic stride samples (every 64th system):
the GPU integrates the whole batch, the reference re-integrates the sample
(systems are independent, batch_driver.hpp:16-21). The checker is the
reference library itself (oracle/_ref) where it was built, else the pinned
C restatement.

Bars: RKCK EXACT and RKC EXACT bitwise with every counter; RKCK FAST
<= 1e-13 (1e-3 * eps) per system with identical counts at the bench
perturbation (0.01). At the 0.1 stress perturbation the FAST bar is asserted
at the bound measured on B200 (regression guard): there, even the reference's
own source compiled with FMA contraction misses 1e-13 on 13% of the systems
(tests/experiments/fma_sensitivity.py, profiles/r02_fma_sensitivity.txt), so EXACT is
the parity policy for that config.
"""
import numpy as np
import pytest

import paper_1611_02274_b200 as B
from paper_1611_02274_b200 import _abi as A
from golden_cases import PLEIADES_IC, heat_ic

pytestmark = pytest.mark.gpu

# (stages_total is not kept by the reference's stats, ode_problem.hpp:57-81;
# the restatement's is compared in test_gpu_parity.py)
COUNTS = ("steps_accepted", "steps_rejected", "rhs_evals", "spec_rad_evals", "underflow")


@pytest.fixture(scope="module")
def checker():
    from oracle_lib import Oracle, RefLib, ref_available
    return RefLib() if ref_available() else Oracle()


def sysrel(y, yref, num, dim):
    a, b = y.reshape(dim, num), yref.reshape(dim, num)
    return np.max(np.abs(a - b), axis=0) / np.maximum(np.max(np.abs(b), axis=0), 1e-300)


def gpu_outer(prob, solver, y0, g, arith):
    num = y0.size // prob.dim
    batch = B.BatchStates(num, prob.dim, prob.param_dim, y0,
                          g if g is not None else np.zeros(0))
    r = B.outer_loop(B.OdeProblem(prob.kind, prob.dim, prob.param_dim), batch, 0.0, 1.0, 0.1,
                     solver=solver, arith=arith)
    return r.states.values, r.stats


def cols(a, dim, num, idx):
    return np.ascontiguousarray(a.reshape(dim, num)[:, idx]).reshape(-1)


def stride_case(checker, prob, solver, base, mag, num, stride, ariths, g=None):
    y0 = B.problems.perturb_initial_conditions(base, mag, 42, num).values
    idx = np.arange(0, num, stride)
    gs = cols(g, prob.param_dim, num, idx) if g is not None else None
    rc, yo, so, _ = checker.outer_loop(prob, solver, 0.0, 1.0, 0.1, cols(y0, prob.dim, num, idx),
                                       gs)
    assert rc == 0
    out = {}
    for arith in ariths:
        y, st = gpu_outer(prob, solver, y0, g, arith)
        out[arith] = (cols(y, prob.dim, num, idx), st[idx])
        del y, st
    return out, yo, so, idx


def test_rkck_pleiades_2_24_stride(gpu, checker):
    """Config 5 (RKCK leg): 2^24 systems, every 64th checked; EXACT bitwise,
    FAST within 1e-13 with identical counts."""
    prob = A.make_problem(A.PLEIADES)
    out, yo, so, idx = stride_case(checker, prob, A.SOLVER_RKCK, PLEIADES_IC, 0.01, 1 << 24, 64,
                                   ("exact", "fast"))
    ye, se = out["exact"]
    assert np.array_equal(ye.view(np.uint64), yo.view(np.uint64))
    for k in COUNTS + ("h_min_seen", "h_max_seen"):
        assert np.array_equal(se[k], so[k]), k
    yf, sf = out["fast"]
    err = sysrel(yf, yo, idx.size, 28)
    print(f"2^24 FAST: max rel err {err.max():.3e} over {idx.size} sampled systems")
    assert err.max() <= 1e-13
    for k in ("steps_accepted", "steps_rejected", "rhs_evals", "underflow"):
        assert np.array_equal(sf[k], so[k]), k


def test_rkc_heat64_2_24_stride(gpu, checker):
    """Config 5 (RKC leg): heat n = 64, 2^24 systems, every 256th checked;
    EXACT bitwise with every counter."""
    prob = A.make_problem(A.HEAT, 64)
    out, yo, so, idx = stride_case(checker, prob, A.SOLVER_RKC, heat_ic(64), 0.01, 1 << 24, 256,
                                   ("exact",))
    ye, se = out["exact"]
    assert np.array_equal(ye.view(np.uint64), yo.view(np.uint64))
    for k in COUNTS + ("h_min_seen", "h_max_seen"):
        assert np.array_equal(se[k], so[k]), k


def test_config4_stiffness_varied_2_22_stride(gpu, checker):
    """Config 4 at 2^22: expDecay with g0 log-uniform in [1, 1e4] in natural
    order (the outer loop sorts by g0 and re-packs by cost internally; results
    must not move), every 64th system checked, EXACT bitwise."""
    from paper_1611_02274_b200.api import stiffness_params
    num = 1 << 22
    prob = A.make_problem(A.EXPDECAY)
    g = stiffness_params(num)
    out, yo, so, idx = stride_case(checker, prob, A.SOLVER_RKC, np.array([1.0]), 0.01, num, 64,
                                   ("exact",), g=g)
    ye, se = out["exact"]
    assert np.array_equal(ye.view(np.uint64), yo.view(np.uint64))
    for k in COUNTS + ("h_min_seen", "h_max_seen"):
        assert np.array_equal(se[k], so[k]), k


def test_rkck_stress_policies(gpu, checker):
    """Config 2 stress (perturb 0.1), 65536 systems: EXACT bitwise; FAST at
    the bound measured on B200 (0.829 of systems within 1e-13, max 2.6e-9,
    no count mismatch), next to the FMA-compiled reference's own 0.868 /
    6.6e-10 / 2 mismatches on the same batch."""
    prob = A.make_problem(A.PLEIADES)
    num = 1 << 16
    out, yo, so, idx = stride_case(checker, prob, A.SOLVER_RKCK, PLEIADES_IC, 0.1, num, 1,
                                   ("exact", "fast"))
    ye, se = out["exact"]
    assert np.array_equal(ye.view(np.uint64), yo.view(np.uint64))
    for k in COUNTS:
        assert np.array_equal(se[k], so[k]), k
    yf, sf = out["fast"]
    err = sysrel(yf, yo, num, 28)
    same = np.ones(num, bool)
    for k in ("steps_accepted", "steps_rejected", "rhs_evals", "underflow"):
        same &= sf[k] == so[k]
    within = ((err <= 1e-13) & same).mean()
    print(f"stress FAST: within {within:.4f}, max {err.max():.3e}, mismatches {(~same).sum()}")
    assert within >= 0.825 and err.max() <= 3e-9 and (~same).sum() <= 1


@pytest.mark.parametrize("n", [100, 700])
def test_rkc_heat_any_n_stride(gpu, checker, n):
    """heatEquation(n) on the padded lane-group kernels at scale (2^17 systems,
    the paper's [0, 1] protocol): every 256th system bitwise the reference."""
    from golden_cases import heat_ic
    num = 1 << 17 if n <= 128 else 1 << 14
    prob = A.make_problem(A.HEAT, n)
    out, yo, so, idx = stride_case(checker, prob, A.SOLVER_RKC, heat_ic(n), 0.01, num,
                                   256 if n <= 128 else 64, ("exact",))
    y, st = out["exact"]
    assert np.array_equal(y.view(np.uint64), yo.view(np.uint64))
    for k in COUNTS:
        assert np.array_equal(st[k], so[k]), k
