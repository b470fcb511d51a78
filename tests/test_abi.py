"""The C-ABI library loads and exports every symbol include/bode.h declares;
host-side logic (validation order, generators, window schedule) matches the
reference without touching a device."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

import paper_1611_02274_b200 as B
from paper_1611_02274_b200 import _abi as A
from golden_cases import PLEIADES_IC, perturb

HEADER = os.path.join(A.REPO_DIR, "include", "bode.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bode_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    names = declared_functions()
    assert len(names) >= 20
    lib = ctypes.CDLL(A.LIB_PATH)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_version_and_defaults():
    L = B.lib()
    assert b"sm_100a" in L.bode_version()
    t = A.Tol()
    L.bode_tol_default(ctypes.byref(t))
    d = A.default_tol()
    for name, _ in A.Tol._fields_:
        assert getattr(t, name) == getattr(d, name), name
    assert L.bode_tol_validate(ctypes.byref(t)) == 0


@pytest.mark.parametrize("field,value", [("eps", 0.0), ("abs_tol", -1.0), ("safety", 1.5),
                                         ("p1", 0.0), ("uround", 0.0), ("kappa", -1.0)])
def test_tolerance_validation(field, value):  # ode_problem.hpp:46-53, test_batch.cpp:230-239
    t = A.default_tol(**{field: value})
    assert B.lib().bode_tol_validate(ctypes.byref(t)) == A.E_INVALID_SHAPE
    b = B.pack([[1.0]])
    with pytest.raises(B.InvalidShape):
        B.integrate_batch(B.problems.zero(1), b, 0.0, 1.0, tol=t)


def test_generators_match_reference(oracle):
    L = B.lib()
    for k in range(5):
        assert L.bode_splitmix64_at(0, k) == oracle.lib.orc_splitmix64_at(0, k)
    assert L.bode_splitmix64_at(0, 0) == 0xe220a8397b1dcdaf
    b = B.problems.perturb_initial_conditions(PLEIADES_IC, 0.01, 42, 3000)
    assert np.array_equal(b.values.view(np.uint64), perturb(PLEIADES_IC, 0.01, 42, 3000).view(np.uint64))
    assert np.array_equal(B.problems.pleiades_initial_conditions(), PLEIADES_IC)
    u = np.empty(64)
    oracle.lib.orc_heat_initial_condition(64, A.dptr(u))
    assert np.array_equal(B.problems.heat_initial_condition(64), u)
    with pytest.raises(B.InvalidShape):
        B.problems.perturb_initial_conditions(PLEIADES_IC, 0.5, 1, 4)
    with pytest.raises(B.InvalidShape):
        B.problems.perturb_initial_conditions(PLEIADES_IC, 0.01, 1, 0)


def test_window_schedule():  # batch_driver.cpp:99-105, test_batch.cpp:171-192
    L = B.lib()
    assert L.bode_num_windows(0.0, 1.0, 0.1) == 10
    assert L.bode_num_windows(0.0, 1.0, 1.0) == 1
    assert L.bode_num_windows(0.0, 1.05, 0.1) == 11
    assert L.bode_window_end(0.0, 1.05, 0.1, 11) == 1.05
    assert L.bode_window_end(0.0, 1.0, 0.1, 3) == 0.0 + 3.0 * 0.1


def test_pack_unpack_roundtrip():  # test_batch.cpp:16-76
    b = B.pack([[1.0, 2.0], [3.0, 4.0]])
    assert list(b.values) == [1.0, 3.0, 2.0, 4.0]
    assert B.unpack(b) == [[1.0, 2.0], [3.0, 4.0]]
    with pytest.raises(B.InvalidShape):
        B.pack([[1.0, 2.0], [3.0]])
    with pytest.raises(B.InvalidShape):
        B.pack([])
    for n in range(1, 9):
        for d in range(1, 9):
            v = [[100.0 * i + j for j in range(d)] for i in range(n)]
            bb = B.pack(v)
            assert all(bb.values[i + n * j] == 100.0 * i + j for i in range(n) for j in range(d))
            assert B.unpack(bb) == v


def test_validation_precedes_device_use():
    b = B.pack([[1.0]])
    with pytest.raises(B.InvalidInterval):  # batch_driver.cpp:42
        B.integrate_batch(B.problems.zero(1), b, 1.0, 1.0)
    with pytest.raises(B.InvalidShape):  # dim mismatch, batch_driver.cpp:45-46
        B.integrate_batch(B.problems.zero(2), b, 0.0, 1.0)
    with pytest.raises(B.InvalidInterval):
        B.outer_loop(B.problems.zero(1), b, 0.0, 1.0, 0.0)
    with pytest.raises(B.Unsupported):  # no device kernel compiled for Pleiades with RKC
        B.integrate_batch(B.problems.pleiades(), B.pack([list(PLEIADES_IC)]), 0.0, 0.1, solver="rkc")


def test_no_cpu_fallback_without_device():
    if B.lib().bode_device_count() > 0:
        pytest.skip("a device is present")
    b = B.pack([[1.0, 2.0]])
    with pytest.raises(B.NoDevice):
        B.integrate_batch(B.problems.zero(2), b, 0.0, 1.0)


def test_supported_matrix():
    L = B.lib()
    for kind, dim, solver in [(A.PLEIADES, 28, 0), (A.HEAT, 64, 1), (A.EXPDECAY, 1, 1),
                              (A.EXPDECAY, 1, 0), (A.HARMONIC, 2, 1)]:
        for arith in (0, 1):
            p = A.make_problem(kind, dim)
            assert L.bode_problem_supported(ctypes.byref(p), solver, arith) == 1
    # heatEquation(n) for any n >= 2 (problems.cpp:94-115): lane-group kernels
    # for n in {8, 16, 32, 64}, one system per block (csrc/wide.cuh) otherwise
    for n in (2, 3, 63, 100, 4000, 1_000_000):
        for solver in (0, 1):
            for arith in (0, 1):
                p = A.make_problem(A.HEAT, n)
                assert L.bode_problem_supported(ctypes.byref(p), solver, arith) == 1
    assert L.bode_set_wide(1) == 0 and L.bode_set_wide(0) == 0


def test_scheduling_knob_validation():
    """Host-side setters reject out-of-range values before any device use, and
    the re-pack entry points validate their arguments (include/bode.h)."""
    L = B.lib()
    if L.bode_device_count() < 1:
        assert L.bode_use_device(0) == A.E_NO_DEVICE
    else:
        assert L.bode_use_device(-1) == A.E_INVALID_SHAPE
    assert L.bode_set_shard_layout(2) == A.E_INVALID_SHAPE
    assert L.bode_set_shard_layout(0) == 0
    assert L.bode_set_attempt_budget(-1) == A.E_INVALID_SHAPE
    assert L.bode_set_attempt_budget(0) == 0
    assert L.bode_set_repack_threshold(1.5) == A.E_INVALID_SHAPE
    assert L.bode_set_repack_threshold(-0.1) == A.E_INVALID_SHAPE
    assert L.bode_set_presort_param(-3) == A.E_INVALID_SHAPE
    assert L.bode_set_block_size(48) == A.E_INVALID_SHAPE
    for ok in (-2, -1, 0):
        assert L.bode_set_presort_param(ok) == 0
    assert L.bode_set_presort_param(-2) == 0  # the default
    assert L.bode_set_repack_threshold(0.7) == 0
    prob = A.make_problem(A.EXPDECAY)
    # param_row must name a parameter row; g and order must be given
    assert L.bode_repack_by_param(ctypes.byref(prob), 8, None, None, None, None, 0,
                                  None) == A.E_INVALID_SHAPE
    assert L.bode_repack_by_param(ctypes.byref(prob), 8, ctypes.c_void_p(8), ctypes.c_void_p(8),
                                  None, ctypes.c_void_p(8), 1, None) == A.E_INVALID_SHAPE


def test_stats_summary_straggler_report():
    """bode_stats_summary (host-side): the costliest system, totals, flag counts
    and the lockstep efficiency of consecutive 32-system warps."""
    st = np.zeros(40, dtype=A.STATS_DTYPE)
    st["steps_accepted"] = 8
    st["steps_rejected"] = 1
    st["rhs_evals"] = 50
    st["steps_accepted"][37] = 900  # a straggler in the second (partial) warp
    st["rhs_evals"][37] = 5000
    st["underflow"][3] = 1
    st["budget_exhausted"][37] = 1
    r = B.stats_summary(st)
    assert r["num"] == 40 and r["attempts_max"] == 901 and r["attempts_argmax"] == 37
    assert r["attempts_total"] == 39 * 9 + 901
    assert r["underflow_count"] == 1 and r["budget_exhausted_count"] == 1
    assert r["rhs_evals_max"] == 5000
    expect = (39 * 50 + 5000) / (32 * 50 + 8 * 5000)
    assert abs(r["lockstep_efficiency"] - expect) < 1e-15
    with pytest.raises(B.InvalidShape):
        B.stats_summary(st[:0])
