"""ctypes mirror of include/bode.h (structs, constants, library loader).

The structs mirror the reference types field for field:
  Tol      <- batchode::ToleranceSettings  (proj/include/batchode/ode_problem.hpp:32-54)
  Stats    <- batchode::IntegrationStats   (ode_problem.hpp:57-81) + stages_total
  Problem  <- batchode::OdeProblem shape   (ode_problem.hpp:23-28)
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

OK = 0
E_INVALID_INTERVAL = 1
E_INVALID_SHAPE = 2
E_INVALID_STAGE_COUNT = 3
E_UNSUPPORTED = 4
E_CUDA = 5
E_NO_DEVICE = 6

SOLVER_RKCK = 0
SOLVER_RKC = 1
ARITH_EXACT = 0
ARITH_FAST = 1

PLEIADES = 0
HEAT = 1
EXPDECAY = 2
HARMONIC = 3
ZERO = 4
RICCATI = 5
DIAG = 6
CONST = 7
SINT = 8
BRUSSELATOR = 9  # registered through include/bode_problem.cuh (csrc/problems_ext.cu)
USER_BASE = 1000

PROBLEM_NAMES = {
    "pleiades": PLEIADES, "heat": HEAT, "expdecay": EXPDECAY, "harmonic": HARMONIC,
    "zero": ZERO, "riccati": RICCATI, "diag": DIAG, "const": CONST, "sint": SINT,
    "brusselator": BRUSSELATOR,
}
SOLVER_NAMES = {"rkck": SOLVER_RKCK, "rkc": SOLVER_RKC}
ARITH_NAMES = {"exact": ARITH_EXACT, "fast": ARITH_FAST}


class Problem(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("dim", ctypes.c_int32),
                ("param_dim", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class Tol(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in (
        "eps", "abs_tol", "rel_tol", "uround", "tiny", "safety", "p1", "errcon",
        "pgrow", "pshrnk", "h_min_floor", "kappa")]


class Stats(ctypes.Structure):
    _fields_ = [("steps_accepted", ctypes.c_int64), ("steps_rejected", ctypes.c_int64),
                ("rhs_evals", ctypes.c_int64), ("spec_rad_evals", ctypes.c_int64),
                ("stages_total", ctypes.c_int64), ("h_min_seen", ctypes.c_double),
                ("h_max_seen", ctypes.c_double), ("underflow", ctypes.c_int32),
                ("budget_exhausted", ctypes.c_int32)]


assert ctypes.sizeof(Stats) == 64


STEP_DTYPE = np.dtype([("t", "<f8"), ("h", "<f8"), ("err", "<f8"), ("stages", "<i4"),
                       ("accepted", "<i4")])  # bode_step_record_t (StepRecord)
assert STEP_DTYPE.itemsize == 32


class StatsSummary(ctypes.Structure):  # bode_stats_summary_t
    _fields_ = [("num", ctypes.c_int64), ("attempts_total", ctypes.c_int64),
                ("attempts_max", ctypes.c_int64), ("attempts_argmax", ctypes.c_int64),
                ("attempts_mean", ctypes.c_double), ("rhs_evals_total", ctypes.c_int64),
                ("rhs_evals_max", ctypes.c_int64), ("underflow_count", ctypes.c_int64),
                ("budget_exhausted_count", ctypes.c_int64),
                ("lockstep_efficiency", ctypes.c_double)]

STATS_DTYPE = np.dtype([
    ("steps_accepted", "<i8"), ("steps_rejected", "<i8"), ("rhs_evals", "<i8"),
    ("spec_rad_evals", "<i8"), ("stages_total", "<i8"), ("h_min_seen", "<f8"),
    ("h_max_seen", "<f8"), ("underflow", "<i4"), ("budget_exhausted", "<i4")])
assert STATS_DTYPE.itemsize == 64


def default_tol(**overrides) -> Tol:
    """ToleranceSettings defaults (ode_problem.hpp:33-44)."""
    t = Tol(eps=1e-10, abs_tol=1e-10, rel_tol=1e-6, uround=2.22e-16, tiny=1e-30,
            safety=0.9, p1=0.1, errcon=1.89e-4, pgrow=-0.2, pshrnk=-0.25,
            h_min_floor=1e-20, kappa=2.0 / 13.0)
    for k, v in overrides.items():
        setattr(t, k, v)
    return t


def make_problem(kind, dim: int = 0) -> Problem:
    """Shape of each problem (problems.hpp:19-63)."""
    if isinstance(kind, str):
        kind = PROBLEM_NAMES[kind]
    fixed = {PLEIADES: (28, 0), EXPDECAY: (1, 1), HARMONIC: (2, 0), RICCATI: (1, 0),
             SINT: (1, 0)}
    if kind in fixed:
        d, p = fixed[kind]
    elif kind == HEAT:
        d, p = (dim or 64), 0
    elif kind == DIAG:
        d, p = dim, dim
    elif kind == BRUSSELATOR:
        d, p = (dim or 64), 3
    else:
        d, p = dim, 0
    return Problem(kind=kind, dim=d, param_dim=p, reserved=0)


def empty_stats(num: int) -> np.ndarray:
    st = np.zeros(num, dtype=STATS_DTYPE)
    st["h_min_seen"] = np.inf
    return st


def dptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if a is not None else None


def vptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_DIR = os.path.dirname(PKG_DIR)
# BODE_LIB_PATH: another in-tree build of the same library, for A/B timing
LIB_PATH = os.environ.get("BODE_LIB_PATH") or os.path.join(PKG_DIR, "lib", "libbode.so")
