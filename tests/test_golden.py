"""The C restatement reproduces the reference's own outputs bit for bit:
against committed golden fixtures (made by tests/golden/make_golden.py from
the unmodified reference) and, where oracle/_ref is built, against the
reference library directly on further inputs."""
import os

import numpy as np
import pytest

from paper_1611_02274_b200 import _abi as A
from golden_cases import CASES, build_inputs, perturb, PLEIADES_IC, heat_ic

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
COUNTS = ("steps_accepted", "steps_rejected", "rhs_evals", "spec_rad_evals", "underflow")


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_reproduces_golden(oracle, name):
    gold = load(name)
    prob, solver, y0, g = build_inputs(CASES[name])
    rc, y, st, steps = oracle.outer_loop(prob, solver, 0.0, 1.0, 0.1, y0, g)
    assert rc == 0 and steps == 10
    assert np.array_equal(y.view(np.uint64), gold["y"].view(np.uint64))
    for k in COUNTS:
        assert np.array_equal(st[k], gold[k]), k
    assert np.array_equal(st["h_min_seen"], gold["h_min_seen"])
    assert np.array_equal(st["h_max_seen"], gold["h_max_seen"])


EXTRA = [
    ("pleiades-stress", A.make_problem(A.PLEIADES), A.SOLVER_RKCK, PLEIADES_IC, 0.1, None),
    ("heat16-rkc", A.make_problem(A.HEAT, 16), A.SOLVER_RKC, heat_ic(16), 0.01, None),
    ("heat8-rkck", A.make_problem(A.HEAT, 8), A.SOLVER_RKCK, heat_ic(8), 0.01, None),
    ("harmonic-rkc", A.make_problem(A.HARMONIC), A.SOLVER_RKC, np.array([1.0, 0.0]), 0.1, None),
    ("expdecay-rkck", A.make_problem(A.EXPDECAY), A.SOLVER_RKCK, np.array([1.0]), 0.01, "stiff"),
]


@pytest.mark.parametrize("case", EXTRA, ids=[c[0] for c in EXTRA])
def test_oracle_matches_reference_library(oracle, ref, case):
    _, prob, solver, base, mag, g = case
    n = 512
    y0 = perturb(base, mag, 7, n)
    gg = 10.0 ** (2.0 + 2.0 * np.linspace(-1, 1, n)) if g else None
    a = oracle.outer_loop(prob, solver, 0.0, 1.0, 0.1, y0, gg)
    b = ref.outer_loop(prob, solver, 0.0, 1.0, 0.1, y0, gg)
    assert a[0] == b[0] == 0
    assert np.array_equal(a[1].view(np.uint64), b[1].view(np.uint64))
    for k in COUNTS:
        assert np.array_equal(a[2][k], b[2][k]), k


def test_reference_ic_asset_matches_embedded(ref):
    """data/pleiades_ic.txt (FNV-1a pinned at problems.hpp:29) == the embedded ICs."""
    path = b"/root/reference/proj/data/pleiades_ic.txt"
    assert ref.lib.ref_fnv1a(path) == 0x5583feb418028048
    out = np.empty(28)
    assert ref.lib.ref_load_pleiades_ic(path, A.dptr(out)) == 0
    assert np.array_equal(out, PLEIADES_IC)


@pytest.mark.parametrize("n,solver,t1", [(2, A.SOLVER_RKC, 0.2), (5, A.SOLVER_RKCK, 0.05),
                                         (100, A.SOLVER_RKC, 0.02), (513, A.SOLVER_RKC, 0.02),
                                         (17, A.SOLVER_RKCK, 0.01), (4000, A.SOLVER_RKC, 1e-3)])
def test_oracle_matches_reference_any_heat_dim(oracle, ref, n, solver, t1):
    """heatEquation(n) at the dimensions the GPU runs on one-system-per-block
    kernels (tests/test_gpu_wide.py checks those against this oracle)."""
    num = 24
    prob = A.make_problem(A.HEAT, n)
    y0 = perturb(heat_ic(n), 0.01, 3 + n, num)
    a = oracle.outer_loop(prob, solver, 0.0, t1, t1 / 2, y0)
    b = ref.outer_loop(prob, solver, 0.0, t1, t1 / 2, y0)
    assert a[0] == b[0] == 0
    assert np.array_equal(a[1].view(np.uint64), b[1].view(np.uint64))
    for k in COUNTS:
        assert np.array_equal(a[2][k], b[2][k]), k
