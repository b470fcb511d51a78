"""ctypes bindings to the CHECKERS under oracle/ -- test infrastructure only.

  Oracle    -> oracle/liboracle.so            (C restatement of the reference)
  RefLib    -> oracle/_ref/libbatchode_ref.so (reference sources compiled as-is)
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from paper_1611_02274_b200 import _abi as A

REPO = A.REPO_DIR
ORACLE_DIR = os.path.join(REPO, "oracle")
ORACLE_SO = os.path.join(ORACLE_DIR, "liboracle.so")
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libbatchode_ref.so")

P = ctypes.POINTER
c_d, c_i, c_i64, c_u64 = ctypes.c_double, ctypes.c_int, ctypes.c_int64, ctypes.c_uint64
PD = P(c_d)
PProb = P(A.Problem)
PTol = P(A.Tol)
PSt = ctypes.c_void_p
OBS = ctypes.CFUNCTYPE(None, c_d, c_d, c_i, c_d, c_i, ctypes.c_void_p)


def _ensure_oracle_built():
    if not os.path.exists(ORACLE_SO):
        subprocess.run(["make", "-C", ORACLE_DIR, "liboracle.so"], check=True,
                       capture_output=True)


class Oracle:
    """The plain-C restatement (oracle/bode_oracle.c)."""

    def __init__(self):
        _ensure_oracle_built()
        L = self.lib = ctypes.CDLL(ORACLE_SO)
        sig = {
            "orc_splitmix64_at": (c_u64, [c_u64, c_u64]),
            "orc_unit_symmetric_at": (c_d, [c_u64, c_u64]),
            "orc_perturb": (c_i, [PD, c_i, c_d, c_u64, c_i, PD]),
            "orc_rhs": (None, [PProb, c_d, PD, PD, PD]),
            "orc_heat_spectral_radius": (c_d, [c_i]),
            "orc_heat_initial_condition": (None, [c_i, PD]),
            "orc_pleiades_energy": (c_d, [PD]),
            "orc_pleiades_momentum": (None, [PD, PD]),
            "orc_rkck_step": (None, [PProb, c_d, PD, PD, PD, c_d, PD, PD]),
            "orc_rkck_error_norm": (None, [c_i, PD, PD, PD, c_d, c_d, c_d, PD, P(c_i)]),
            "orc_rkck_adjust_step": (None, [c_d, c_d, c_i, c_d, c_d, PTol, P(c_i), PD]),
            "orc_rkck_driver": (c_i, [PProb, c_d, c_d, PD, PD, PTol, PSt, OBS, ctypes.c_void_p]),
            "orc_rkck_integrate_fixed": (None, [PProb, c_d, c_d, ctypes.c_long, PD, PD]),
            "orc_chebyshev_eval": (None, [c_i, c_d, PD]),
            "orc_rkc_coefficients": (c_i, [c_i, c_d, PD, PD] + [PD] * 7),
            "orc_rkc_step": (c_i, [PProb, c_d, PD, PD, PD, c_d, c_i, c_d, PD]),
            "orc_rkc_error_norm": (c_d, [c_i, PD, PD, PD, PD, c_d, c_d, c_d]),
            "orc_rkc_stage_count": (None, [c_d, c_d, c_d, c_d, P(c_i), PD]),
            "orc_rkc_initial_step": (None, [PProb, c_d, PD, PD, PD, c_d, c_d, c_d, PTol, PD, PD]),
            "orc_rkc_next_step_accepted": (c_d, [c_d, c_d, c_d, c_d, c_i, c_d, c_d]),
            "orc_rkc_next_step_rejected": (c_d, [c_d, c_d]),
            "orc_rkc_driver": (c_i, [PProb, c_d, c_d, PD, PD, PTol, PSt, OBS, ctypes.c_void_p]),
            "orc_rkc_integrate_fixed": (None, [PProb, c_d, c_d, ctypes.c_long, c_i, c_d, PD, PD]),
            "orc_power_method": (c_i, [PProb, c_d, PD, PD, PD, c_d, PD, PD, PD, P(c_i), P(c_i)]),
            "orc_integrate_batch": (c_i, [PProb, c_i, c_d, c_d, c_i64, PD, PD, PTol, PSt, c_i]),
            "orc_outer_loop": (c_i, [PProb, c_i, c_d, c_d, c_d, c_i64, PD, PD, PTol, PSt, c_i, P(c_i)]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args

    # -- convenience wrappers (numpy in/out) --
    def rhs(self, prob, y, g=None, t=0.0):
        y = np.ascontiguousarray(y, dtype=np.float64)
        out = np.empty(prob.dim)
        g = None if g is None else np.ascontiguousarray(g, dtype=np.float64)
        self.lib.orc_rhs(ctypes.byref(prob), t, A.dptr(y), A.dptr(g), A.dptr(out))
        return out

    def driver(self, prob, solver, t, t_end, y, g=None, tol=None, observer=None):
        y = np.array(y, dtype=np.float64)
        g = None if g is None else np.ascontiguousarray(g, dtype=np.float64)
        st = A.empty_stats(1)
        tol = tol or A.default_tol()
        cb = OBS(observer) if observer else OBS()
        fn = self.lib.orc_rkck_driver if solver == A.SOLVER_RKCK else self.lib.orc_rkc_driver
        rc = fn(ctypes.byref(prob), t, t_end, A.dptr(y), A.dptr(g), ctypes.byref(tol),
                A.vptr(st), cb, None)
        return rc, y, st[0]

    def outer_loop(self, prob, solver, t0, t_end, h_outer, y_soa, g_soa=None, tol=None,
                   threads=None):
        num = y_soa.size // prob.dim
        y = np.array(y_soa, dtype=np.float64)
        g = None if g_soa is None else np.ascontiguousarray(g_soa, dtype=np.float64)
        st = A.empty_stats(num)
        steps = c_i(0)
        rc = self.lib.orc_outer_loop(ctypes.byref(prob), solver, t0, t_end, h_outer, num,
                                     A.dptr(y), A.dptr(g), ctypes.byref(tol or A.default_tol()),
                                     A.vptr(st), threads or os.cpu_count(), ctypes.byref(steps))
        return rc, y, st, steps.value

    def integrate_batch(self, prob, solver, t, t_next, y_soa, g_soa=None, tol=None,
                        threads=None):
        num = y_soa.size // prob.dim
        y = np.array(y_soa, dtype=np.float64)
        g = None if g_soa is None else np.ascontiguousarray(g_soa, dtype=np.float64)
        st = A.empty_stats(num)
        rc = self.lib.orc_integrate_batch(ctypes.byref(prob), solver, t, t_next, num,
                                          A.dptr(y), A.dptr(g),
                                          ctypes.byref(tol or A.default_tol()), A.vptr(st),
                                          threads or os.cpu_count())
        return rc, y, st

    def perturb(self, base, magnitude, seed, count):
        base = np.ascontiguousarray(base, dtype=np.float64)
        out = np.empty(count * base.size)
        rc = self.lib.orc_perturb(A.dptr(base), base.size, magnitude, seed, count, A.dptr(out))
        return rc, out

    def coefficients(self, s, kappa=2.0 / 13.0):
        arrs = [np.zeros(s + 1) for _ in range(7)]
        o0, o1 = c_d(), c_d()
        rc = self.lib.orc_rkc_coefficients(s, kappa, ctypes.byref(o0), ctypes.byref(o1),
                                           *[A.dptr(a) for a in arrs])
        names = ["mu", "nu", "muTilde", "gammaTilde", "b", "a", "c"]
        d = dict(zip(names, arrs))
        d.update(omega0=o0.value, omega1=o1.value, rc=rc)
        return d


def ref_available() -> bool:
    return os.path.exists(REF_SO)


class RefLib:
    """The unmodified reference sources compiled by oracle/Makefile."""

    def __init__(self):
        L = self.lib = ctypes.CDLL(REF_SO)
        sig = {
            "ref_outer_loop": (c_i, [PProb, c_i, c_d, c_d, c_d, c_i64, PD, PD, PTol, PSt, c_i, P(c_i)]),
            "ref_outer_loop_fn": (c_i, [ctypes.c_void_p, c_i, c_i, c_i, c_d, c_d, c_d, c_i64, PD,
                                        PD, PTol, PSt, c_i, P(c_i)]),
            "ref_integrate_batch": (c_i, [PProb, c_i, c_d, c_d, c_i64, PD, PD, PTol, PSt, c_i]),
            "ref_driver": (c_i, [PProb, c_i, c_d, c_d, PD, PD, PTol, PSt]),
            "ref_splitmix64_at": (c_u64, [c_u64, c_u64]),
            "ref_perturb": (c_i, [PD, c_i, c_d, c_u64, c_i, PD]),
            "ref_load_pleiades_ic": (c_i, [ctypes.c_char_p, PD]),
            "ref_fnv1a": (c_u64, [ctypes.c_char_p]),
            "ref_rhs": (None, [PProb, c_d, PD, PD, PD]),
            "ref_rkck_step": (None, [PProb, c_d, PD, PD, PD, c_d, PD, PD]),
            "ref_rkck_adjust_step": (None, [c_d, c_d, c_i, c_d, c_d, PTol, P(c_i), PD]),
            "ref_rkc_coefficients": (c_i, [c_i, c_d, PD, PD] + [PD] * 7),
            "ref_rkc_step": (c_i, [PProb, c_d, PD, PD, PD, c_d, c_i, c_d, PD]),
            "ref_rkc_stage_count": (None, [c_d, c_d, c_d, c_d, P(c_i), PD]),
            "ref_rkc_next_step_accepted": (c_d, [c_d, c_d, c_d, c_d, c_i, c_d, c_d]),
            "ref_rkc_next_step_rejected": (c_d, [c_d, c_d]),
            "ref_power_method": (c_i, [PProb, c_d, PD, PD, PD, c_d, PD, PD, PD, P(c_i), P(c_i)]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args

    def outer_loop(self, prob, solver, t0, t_end, h_outer, y_soa, g_soa=None, tol=None,
                   workers=None):
        num = y_soa.size // prob.dim
        y = np.array(y_soa, dtype=np.float64)
        g = None if g_soa is None else np.ascontiguousarray(g_soa, dtype=np.float64)
        st = A.empty_stats(num)
        steps = c_i(0)
        rc = self.lib.ref_outer_loop(ctypes.byref(prob), solver, t0, t_end, h_outer, num,
                                     A.dptr(y), A.dptr(g), ctypes.byref(tol or A.default_tol()),
                                     A.vptr(st), workers or os.cpu_count(), ctypes.byref(steps))
        return rc, y, st, steps.value

    def outer_loop_fn(self, rhs_addr, dim, param_dim, solver, t0, t_end, h_outer, y_soa,
                      g_soa=None, tol=None, workers=None):
        """outerLoop on an OdeProblem whose rhs is the C function at rhs_addr."""
        num = y_soa.size // dim
        y = np.array(y_soa, dtype=np.float64)
        g = None if g_soa is None else np.ascontiguousarray(g_soa, dtype=np.float64)
        st = A.empty_stats(num)
        steps = c_i(0)
        rc = self.lib.ref_outer_loop_fn(rhs_addr, dim, param_dim, solver, t0, t_end, h_outer,
                                        num, A.dptr(y), A.dptr(g),
                                        ctypes.byref(tol or A.default_tol()), A.vptr(st),
                                        workers or os.cpu_count(), ctypes.byref(steps))
        return rc, y, st, steps.value

    def driver(self, prob, solver, t, t_end, y, g=None, tol=None):
        y = np.array(y, dtype=np.float64)
        g = None if g is None else np.ascontiguousarray(g, dtype=np.float64)
        st = A.empty_stats(1)
        rc = self.lib.ref_driver(ctypes.byref(prob), solver, t, t_end, A.dptr(y), A.dptr(g),
                                 ctypes.byref(tol or A.default_tol()), A.vptr(st))
        return rc, y, st[0]
