"""Python host mirror of the reference's batch interface, over the C ABI.

Names, argument meaning and error behaviour follow batchode
(proj/include/batchode/*.hpp):

  BatchStates, pack, unpack, fill_params         batch.hpp:15-45
  integrate_batch  -> BatchResult                batch_driver.hpp:22-24
  outer_loop       -> OuterLoopResult            batch_driver.hpp:40-43
  ToleranceSettings / IntegrationStats           ode_problem.hpp:32-81
  problems.pleiades/heat_equation/exp_decay/...  problems.hpp:19-63
  InvalidShape / InvalidInterval / ...           errors.hpp:8-30

Every integration runs in libbode.so on the GPU. There is no CPU fallback:
a missing library raises at import, a missing device raises NoDevice.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
from typing import Callable, Optional, Sequence

import numpy as np

from . import _abi as A


class BodeError(RuntimeError):
    pass


class InvalidShape(BodeError, ValueError):
    pass


class InvalidInterval(BodeError, ValueError):
    pass


class InvalidStageCount(BodeError, ValueError):
    pass


class Unsupported(BodeError):
    pass


class CudaError(BodeError):
    pass


class NoDevice(BodeError):
    pass


_ERRORS = {A.E_INVALID_INTERVAL: InvalidInterval, A.E_INVALID_SHAPE: InvalidShape,
           A.E_INVALID_STAGE_COUNT: InvalidStageCount, A.E_UNSUPPORTED: Unsupported,
           A.E_CUDA: CudaError, A.E_NO_DEVICE: NoDevice}

_LIB = None
SINK = ctypes.CFUNCTYPE(None, ctypes.c_double, ctypes.POINTER(ctypes.c_double), ctypes.c_int64,
                        ctypes.c_int32, ctypes.c_void_p)


def lib():
    """Load libbode.so (built in-tree by paper_1611_02274_b200.build)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(A.LIB_PATH):
        raise ImportError(f"libbode.so not built at {A.LIB_PATH}; run "
                          "`python -m paper_1611_02274_b200.build` (no CPU fallback exists)")
    L = ctypes.CDLL(A.LIB_PATH)
    P = ctypes.POINTER
    c_d, c_i32, c_i64, c_u64, vp = (ctypes.c_double, ctypes.c_int32, ctypes.c_int64,
                                    ctypes.c_uint64, ctypes.c_void_p)
    PD = P(c_d)
    sig = {
        "bode_version": (ctypes.c_char_p, []),
        "bode_last_error": (ctypes.c_char_p, []),
        "bode_device_count": (ctypes.c_int, []),
        "bode_tol_default": (None, [P(A.Tol)]),
        "bode_tol_validate": (ctypes.c_int, [P(A.Tol)]),
        "bode_problem_init": (ctypes.c_int, [P(A.Problem), c_i32, c_i32]),
        "bode_problem_supported": (ctypes.c_int, [P(A.Problem), c_i32, c_i32]),
        "bode_int_driver": (ctypes.c_int, [P(A.Problem), c_i32, c_i32, c_d, c_d, c_i64, PD, PD,
                                           P(A.Tol), vp, c_i32]),
        "bode_outer_loop": (ctypes.c_int, [P(A.Problem), c_i32, c_i32, c_d, c_d, c_d, c_i64, PD,
                                           PD, P(A.Tol), vp, c_i32, SINK, vp, P(c_i32)]),
        "bode_int_driver_device": (ctypes.c_int, [P(A.Problem), c_i32, c_i32, c_d, c_d, c_i64,
                                                  vp, vp, P(A.Tol), vp, c_i32, vp]),
        "bode_num_windows": (c_i64, [c_d, c_d, c_d]),
        "bode_window_end": (c_d, [c_d, c_d, c_d, c_i64]),
        "bode_set_block_size": (ctypes.c_int, [c_i32]),
        "bode_launch_count": (c_i64, []),
        "bode_set_persistent": (ctypes.c_int, [c_i32]),
        "bode_set_wide": (ctypes.c_int, [c_i32]),
        "bode_use_device": (ctypes.c_int, [c_i32]),
        "bode_trace_steps": (ctypes.c_int, [P(A.Problem), c_i32, c_i32, c_d, c_d, PD, PD, P(A.Tol),
                                            vp, vp, c_i64, P(c_i64)]),
        "bode_set_shard_layout": (ctypes.c_int, [c_i32]),
        "bode_set_attempt_budget": (ctypes.c_int, [c_i64]),
        "bode_stats_summary": (ctypes.c_int, [vp, c_i64, P(A.StatsSummary)]),
        "bode_register_kernels": (ctypes.c_int, [vp, c_i32, c_i32]),
        "bode_order_init": (ctypes.c_int, [vp, c_i64, vp]),
        "bode_repack_by_cost": (ctypes.c_int, [P(A.Problem), c_i64, vp, vp, vp, vp, vp]),
        "bode_unpack": (ctypes.c_int, [P(A.Problem), c_i64, vp, vp, vp, vp, vp]),
        "bode_lockstep_efficiency": (ctypes.c_int, [P(A.Problem), c_i32, c_i32, c_i64, vp, P(c_d),
                                                    vp]),
        "bode_set_repack_threshold": (ctypes.c_int, [c_d]),
        "bode_repack_by_param": (ctypes.c_int, [P(A.Problem), c_i64, vp, vp, vp, vp, c_i32, vp]),
        "bode_set_presort_param": (ctypes.c_int, [c_i32]),
        "bode_registered_count": (ctypes.c_int, []),
        "bode_integrate_fixed": (ctypes.c_int, [P(A.Problem), c_i32, c_i32, c_d, c_d, c_i64,
                                                c_i32, c_d, c_i64, PD, PD]),
        "bode_splitmix64_at": (c_u64, [c_u64, c_u64]),
        "bode_unit_symmetric_at": (c_d, [c_u64, c_u64]),
        "bode_perturb_initial_conditions": (ctypes.c_int, [PD, c_i32, c_d, c_u64, c_i64, PD]),
        "bode_perturb_initial_conditions_range": (ctypes.c_int, [PD, c_i32, c_d, c_u64, c_i64,
                                                                 c_i64, PD]),
        "bode_pleiades_ic": (None, [PD]),
        "bode_heat_initial_condition": (None, [c_i32, PD]),
        "bode_selftest_cbrt": (ctypes.c_int, [PD, PD, c_i64]),
        "bode_selftest_fp64_peak": (ctypes.c_int, [PD, PD]),
        "bode_selftest_pow": (ctypes.c_int, [PD, PD, PD, c_i64]),
        "bode_pow_exact_available": (ctypes.c_int, []),
        "bode_selftest_exact_math": (ctypes.c_int, [PD, c_i64, c_i32, P(c_i64), P(c_i64)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _LIB = L
    return L


def load_problem_library(path: str) -> ctypes.CDLL:
    """Loads a problem library built against include/bode_problem.cuh (after
    libbode): its static initializer registers the problem's kernels with
    bode_register_kernels, so its kind is accepted everywhere afterwards."""
    L = lib()
    before = L.bode_registered_count()
    h = ctypes.CDLL(os.path.abspath(path))
    if L.bode_registered_count() <= before:
        raise Unsupported(f"{path}: no kernels registered "
                          f"({L.bode_last_error().decode(errors='replace')})")
    return h


def problem(kind: int, dim: int = 0) -> "OdeProblem":
    """OdeProblem for a built-in or registered kind (bode_problem_init)."""
    p = A.Problem()
    check(lib().bode_problem_init(ctypes.byref(p), int(kind), int(dim)))
    return OdeProblem(p.kind, p.dim, p.param_dim)


def check(rc: int):
    if rc != A.OK:
        msg = lib().bode_last_error().decode()
        raise _ERRORS.get(rc, BodeError)(msg)


# ---------------------------------------------------------------- types ----
ToleranceSettings = A.Tol
SolverChoice = {"RKCK": A.SOLVER_RKCK, "RKC": A.SOLVER_RKC}


def tolerance_settings(**kw) -> A.Tol:
    return A.default_tol(**kw)


@dataclasses.dataclass
class OdeProblem:
    """Problem tag + shape (ode_problem.hpp:23-28). The RHS is a compiled
    device functor selected by `kind`; arbitrary host callables cannot run on
    the GPU."""
    kind: int
    dim: int
    param_dim: int

    def c(self) -> A.Problem:
        return A.Problem(kind=self.kind, dim=self.dim, param_dim=self.param_dim, reserved=0)


@dataclasses.dataclass
class BatchStates:
    """SoA batch: variable j of system i at values[i + num_systems*j] (batch.hpp:15-29)."""
    num_systems: int
    dim: int
    param_dim: int
    values: np.ndarray
    params: np.ndarray

    def at(self, system: int, var: int) -> float:
        return float(self.values[system + self.num_systems * var])

    def state(self, system: int) -> np.ndarray:
        return self.values[system::self.num_systems][: self.dim].copy()

    def validate(self):  # batch.cpp:8-22
        if self.num_systems < 1 or self.dim < 1:
            raise InvalidShape("BatchStates: numSystems and dim must be positive")
        if self.param_dim < 0:
            raise InvalidShape("BatchStates: negative paramDim")
        if self.values.size != self.num_systems * self.dim:
            raise InvalidShape(f"BatchStates: values length {self.values.size} != "
                               f"numSystems*dim = {self.num_systems * self.dim}")
        if self.params.size != self.num_systems * self.param_dim:
            raise InvalidShape(f"BatchStates: params length {self.params.size} != "
                               f"numSystems*paramDim = {self.num_systems * self.param_dim}")

    def copy(self) -> "BatchStates":
        return BatchStates(self.num_systems, self.dim, self.param_dim, self.values.copy(),
                           self.params.copy())


def pack(states: Sequence[Sequence[float]], params: Sequence[Sequence[float]] = ()) -> BatchStates:
    """batch.cpp:24-50."""
    if len(states) == 0:
        raise InvalidShape("pack: no systems")
    dim = len(states[0])
    if dim == 0:
        raise InvalidShape("pack: zero-dimensional state")
    if any(len(s) != dim for s in states):
        raise InvalidShape("pack: ragged state vectors")
    if len(params) and len(params) != len(states):
        raise InvalidShape("pack: params count differs from state count")
    pdim = len(params[0]) if len(params) else 0
    if any(len(p) != pdim for p in params):
        raise InvalidShape("pack: ragged parameter vectors")
    n = len(states)
    vals = np.ascontiguousarray(np.asarray(states, dtype=np.float64).T).reshape(-1)
    prm = (np.ascontiguousarray(np.asarray(params, dtype=np.float64).T).reshape(-1)
           if pdim else np.zeros(0))
    return BatchStates(n, dim, pdim, vals, prm)


def unpack(batch: BatchStates) -> list:
    """batch.cpp:52-59."""
    batch.validate()
    return [list(batch.values[i::batch.num_systems][: batch.dim]) for i in range(batch.num_systems)]


def fill_params(batch: BatchStates, g: Sequence[float]):
    """batch.cpp:61-67."""
    g = np.asarray(g, dtype=np.float64)
    batch.param_dim = g.size
    batch.params = np.repeat(g, batch.num_systems)


@dataclasses.dataclass
class BatchResult:
    states: BatchStates
    stats: np.ndarray  # structured array, one IntegrationStats per system


@dataclasses.dataclass
class OuterLoopResult:
    states: BatchStates
    stats: np.ndarray
    outer_steps: int


def _arith(a) -> int:
    return A.ARITH_NAMES[a] if isinstance(a, str) else int(a)


def _solver(s) -> int:
    if isinstance(s, str):
        return A.SOLVER_NAMES.get(s.lower(), SolverChoice.get(s.upper(), -1))
    return int(s)


def _check_batch(problem: OdeProblem, batch: BatchStates):
    batch.validate()
    if batch.dim != problem.dim:
        raise InvalidShape("integrateBatch: batch dim does not match problem dim")
    if batch.param_dim != problem.param_dim:
        raise InvalidShape("integrateBatch: batch paramDim does not match problem")


def integrate_batch(problem: OdeProblem, batch: BatchStates, t: float, t_next: float,
                    solver="rkck", tol: Optional[A.Tol] = None, gpus: int = 1,
                    arith="exact") -> BatchResult:
    """batchode::integrateBatch on the GPU (value semantics: input untouched)."""
    if not (t_next > t):
        raise InvalidInterval("integrateBatch: tNext must exceed t")
    _check_batch(problem, batch)
    tol = tol or A.default_tol()
    out = batch.copy()
    stats = A.empty_stats(batch.num_systems)
    g = out.params if out.param_dim else None
    check(lib().bode_int_driver(ctypes.byref(problem.c()), _solver(solver), _arith(arith), t,
                                t_next, batch.num_systems, A.dptr(g), A.dptr(out.values),
                                ctypes.byref(tol), A.vptr(stats), gpus))
    return BatchResult(out, stats)


def outer_loop(problem: OdeProblem, initial: BatchStates, t0: float, t_end: float,
               h_outer: float, solver="rkck", tol: Optional[A.Tol] = None, gpus: int = 1,
               sink: Optional[Callable[[float, BatchStates], None]] = None,
               arith="exact") -> OuterLoopResult:
    """batchode::outerLoop with y resident on the device between windows."""
    if not (t_end > t0):
        raise InvalidInterval("outerLoop: tEnd must exceed t0")
    if not (h_outer > 0.0):
        raise InvalidInterval("outerLoop: hOuter must be positive")
    _check_batch(problem, initial)
    tol = tol or A.default_tol()
    out = initial.copy()
    stats = A.empty_stats(initial.num_systems)
    g = out.params if out.param_dim else None
    steps = ctypes.c_int32(0)
    cb = SINK()
    if sink is not None:
        def _cb(t, yptr, num, dim, _user):
            # an independent copy the sink may keep (batch_driver.hpp:26-28)
            snap = BatchStates(out.num_systems, out.dim, out.param_dim,
                               np.ctypeslib.as_array(yptr, shape=(num * dim,)).copy(),
                               out.params.copy())
            sink(t, snap)
        cb = SINK(_cb)
    check(lib().bode_outer_loop(ctypes.byref(problem.c()), _solver(solver), _arith(arith), t0,
                                t_end, h_outer, initial.num_systems, A.dptr(g),
                                A.dptr(out.values), ctypes.byref(tol), A.vptr(stats), gpus, cb,
                                None, ctypes.byref(steps)))
    return OuterLoopResult(out, stats, steps.value)


def integrate_fixed(problem: OdeProblem, batch: BatchStates, t0: float, t_end: float,
                    num_steps: int, solver="rkck", stages: int = 0,
                    kappa: float = 2.0 / 13.0, arith="exact") -> BatchStates:
    """rkck::integrateFixed / rkc::integrateFixed (rkck.cpp:168-181,
    rkc.cpp:290-306) over a whole batch on the GPU."""
    _check_batch(problem, batch)
    out = batch.copy()
    g = out.params if out.param_dim else None
    check(lib().bode_integrate_fixed(ctypes.byref(problem.c()), _solver(solver), _arith(arith),
                                     t0, t_end, num_steps, stages, kappa, batch.num_systems,
                                     A.dptr(g), A.dptr(out.values)))
    return out


def int_driver_device(problem: OdeProblem, solver, arith, t: float, t_end: float, num: int,
                      g_ptr: int, y_ptr: int, tol: A.Tol, stats_ptr: int, merge: bool,
                      stream: int):
    """Device-pointer intDriver (raw CUDA pointers, e.g. torch tensor data_ptr())."""
    check(lib().bode_int_driver_device(ctypes.byref(problem.c()), _solver(solver), _arith(arith),
                                       t, t_end, num, ctypes.c_void_p(g_ptr or None),
                                       ctypes.c_void_p(y_ptr), ctypes.byref(tol),
                                       ctypes.c_void_p(stats_ptr or None), int(bool(merge)),
                                       ctypes.c_void_p(stream or None)))


def order_init(order_ptr: int, num: int, stream: int = 0):
    """Identity position -> system map for re-packing (bode_order_init)."""
    check(lib().bode_order_init(ctypes.c_void_p(order_ptr), num, ctypes.c_void_p(stream or None)))


def repack_by_cost(problem: OdeProblem, num: int, y_ptr: int, g_ptr: int, stats_ptr: int,
                   order_ptr: int, stream: int = 0):
    """Sort a device-resident batch by last-window RHS cost so similar systems
    share warps (bode_repack_by_cost); results stay bitwise identical."""
    check(lib().bode_repack_by_cost(ctypes.byref(problem.c()), num, ctypes.c_void_p(y_ptr),
                                    ctypes.c_void_p(g_ptr or None), ctypes.c_void_p(stats_ptr),
                                    ctypes.c_void_p(order_ptr), ctypes.c_void_p(stream or None)))


def repack_by_param(problem: OdeProblem, num: int, y_ptr: int, g_ptr: int, stats_ptr: int,
                    order_ptr: int, param_row: int, stream: int = 0):
    """Sort a device-resident batch by |g[param_row]|, a stiffness proxy known
    before any window (bode_repack_by_param); results stay bitwise identical."""
    check(lib().bode_repack_by_param(ctypes.byref(problem.c()), num, ctypes.c_void_p(y_ptr),
                                     ctypes.c_void_p(g_ptr), ctypes.c_void_p(stats_ptr or None),
                                     ctypes.c_void_p(order_ptr), param_row,
                                     ctypes.c_void_p(stream or None)))


def unpack_order(problem: OdeProblem, num: int, y_ptr: int, g_ptr: int, stats_ptr: int,
                 order_ptr: int, stream: int = 0):
    """Restore the caller's order after repack_by_cost (bode_unpack). (Not to be
    confused with unpack(batch), the reference's BatchStates helper.)"""
    check(lib().bode_unpack(ctypes.byref(problem.c()), num, ctypes.c_void_p(y_ptr),
                            ctypes.c_void_p(g_ptr or None), ctypes.c_void_p(stats_ptr or None),
                            ctypes.c_void_p(order_ptr), ctypes.c_void_p(stream or None)))


def lockstep_efficiency(problem: OdeProblem, solver, arith, num: int, stats_ptr: int,
                        stream: int = 0) -> float:
    """SIMT lockstep efficiency implied by device stats (bode_lockstep_efficiency)."""
    eff = ctypes.c_double()
    check(lib().bode_lockstep_efficiency(ctypes.byref(problem.c()), _solver(solver),
                                         _arith(arith), num, ctypes.c_void_p(stats_ptr),
                                         ctypes.byref(eff), ctypes.c_void_p(stream or None)))
    return eff.value


def trace_steps(problem: OdeProblem, y, g=None, t: float = 0.0, t_end: float = 1.0,
                solver="rkck", arith="exact", tol: Optional[A.Tol] = None,
                capacity: int = 1 << 16):
    """rkck::driver / rkc::driver with a StepObserver (ode_problem.hpp:85-94) for one
    system on the device (bode_trace_steps). Returns (y, stats, records): the final
    state, the IntegrationStats and one StepRecord (t, h, err, stages, accepted)
    per attempt, bitwise the reference observer's under EXACT."""
    y = np.array(y, dtype=np.float64).reshape(-1)
    gg = None if g is None else np.ascontiguousarray(g, dtype=np.float64).reshape(-1)
    st = A.empty_stats(1)
    rec = np.zeros(capacity, dtype=A.STEP_DTYPE)
    n = ctypes.c_int64()
    check(lib().bode_trace_steps(ctypes.byref(problem.c()), _solver(solver), _arith(arith),
                                 t, t_end, A.dptr(gg), A.dptr(y),
                                 ctypes.byref(tol or A.default_tol()), A.vptr(st),
                                 rec.ctypes.data_as(ctypes.c_void_p), capacity, ctypes.byref(n)))
    return y, st[0], rec[:min(n.value, capacity)].copy()


def stats_summary(stats: np.ndarray) -> dict:
    """Straggler report over per-system stats (bode_stats_summary): attempt
    totals, the costliest system, underflow / budget counts and the lockstep
    efficiency of consecutive 32-system warps."""
    st = np.ascontiguousarray(stats, dtype=A.STATS_DTYPE)
    out = A.StatsSummary()
    check(lib().bode_stats_summary(st.ctypes.data_as(ctypes.c_void_p), st.size,
                                   ctypes.byref(out)))
    return {k: getattr(out, k) for k, _ in A.StatsSummary._fields_}


# ------------------------------------------------------------- problems ----
class problems:
    """problems.hpp:19-63."""

    @staticmethod
    def pleiades() -> OdeProblem:
        return OdeProblem(A.PLEIADES, 28, 0)

    @staticmethod
    def heat_equation(interior_points: int) -> OdeProblem:
        if interior_points < 2:
            raise InvalidShape("heatEquation: need at least two interior points")
        return OdeProblem(A.HEAT, interior_points, 0)

    @staticmethod
    def exp_decay() -> OdeProblem:
        return OdeProblem(A.EXPDECAY, 1, 1)

    @staticmethod
    def harmonic() -> OdeProblem:
        return OdeProblem(A.HARMONIC, 2, 0)

    @staticmethod
    def zero(dim: int) -> OdeProblem:
        return OdeProblem(A.ZERO, dim, 0)

    @staticmethod
    def riccati() -> OdeProblem:
        return OdeProblem(A.RICCATI, 1, 0)

    @staticmethod
    def diagonal(dim: int) -> OdeProblem:
        return OdeProblem(A.DIAG, dim, dim)

    @staticmethod
    def pleiades_initial_conditions() -> np.ndarray:
        out = np.empty(28)
        lib().bode_pleiades_ic(A.dptr(out))
        return out

    @staticmethod
    def heat_initial_condition(n: int) -> np.ndarray:
        out = np.empty(n)
        lib().bode_heat_initial_condition(n, A.dptr(out))
        return out

    @staticmethod
    def splitmix64_at(seed: int, k: int) -> int:
        return int(lib().bode_splitmix64_at(seed, k))

    @staticmethod
    def unit_symmetric_at(seed: int, k: int) -> float:
        return float(lib().bode_unit_symmetric_at(seed, k))

    @staticmethod
    def perturb_initial_conditions(base, magnitude: float, seed: int, count: int) -> BatchStates:
        base = np.ascontiguousarray(base, dtype=np.float64)
        if base.size == 0:
            raise InvalidShape("perturbInitialConditions: empty base state")
        out = np.empty(count * base.size) if count > 0 else np.empty(0)
        check(lib().bode_perturb_initial_conditions(A.dptr(base), base.size, magnitude, seed,
                                                    count, A.dptr(out)))
        return BatchStates(count, base.size, 0, out, np.zeros(0))


def stiffness_params(count: int, seed: int = 9) -> np.ndarray:
    """Config 4's per-system stiffness g0_i = 10^(2 + 2*unitSymmetricAt(9, i)),
    log-uniform in [1, 1e4]."""
    u = np.array([problems.unit_symmetric_at(seed, i) for i in range(count)]) if count < 4096 \
        else _unit_symmetric_vec(seed, count)
    return 10.0 ** (2.0 + 2.0 * u)


def _unit_symmetric_vec(seed: int, count: int) -> np.ndarray:
    k = np.arange(count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (k + np.uint64(1)) * np.uint64(0x9e3779b97f4a7c15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xbf58476d1ce4e5b9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94d049bb133111eb)
        z = z ^ (z >> np.uint64(31))
    u01 = (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return 2.0 * u01 - 1.0
