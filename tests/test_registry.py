"""User-problem registry (include/bode_problem.cuh, bode_register_kernels):
host-side checks that need no GPU. The device parity of registered problems is
in test_gpu_user_problems.py."""
import ctypes
import os

import numpy as np
import pytest

import paper_1611_02274_b200 as B
from paper_1611_02274_b200 import _abi as A

USER_LIB = os.path.join(A.PKG_DIR, "lib", "libuser_problem.so")
LORENZ = A.USER_BASE + 96


def test_builtin_extension_registered_at_load():
    L = B.lib()
    assert L.bode_registered_count() >= 4  # Brusselator: RKCK/RKC x EXACT/FAST
    p = B.api.problem(A.BRUSSELATOR)
    assert (p.dim, p.param_dim) == (64, 3)
    prob = A.make_problem(A.BRUSSELATOR)
    for solver in (A.SOLVER_RKCK, A.SOLVER_RKC):
        for arith in (A.ARITH_EXACT, A.ARITH_FAST):
            assert L.bode_problem_supported(ctypes.byref(prob), solver, arith) == 1


def test_user_library_registers_its_kind():
    L = B.lib()
    n0 = L.bode_registered_count()
    h = B.api.load_problem_library(USER_LIB)
    assert L.bode_registered_count() >= n0 + 4 or n0 >= 8  # idempotent across test order
    p = B.api.problem(LORENZ)
    assert (p.dim, p.param_dim) == (40, 1)
    prob = A.Problem(kind=LORENZ, dim=40, param_dim=1, reserved=0)
    assert L.bode_problem_supported(ctypes.byref(prob), A.SOLVER_RKCK, A.ARITH_EXACT) == 1
    # the host form the parity oracle integrates
    f = h.bode_example_lorenz96_rhs
    f.restype = None
    f.argtypes = [ctypes.c_double] + [ctypes.POINTER(ctypes.c_double)] * 3
    y = np.linspace(-1.0, 2.0, 40)
    g = np.array([8.0])
    dy = np.empty(40)
    f(0.0, A.dptr(y), A.dptr(g), A.dptr(dy))
    ref = (np.roll(y, -1) - np.roll(y, 2)) * np.roll(y, 1) - y + 8.0
    assert np.array_equal(dy, ref)


def test_unknown_kind_rejected():
    p = A.Problem()
    assert B.lib().bode_problem_init(ctypes.byref(p), A.USER_BASE + 999, 0) == A.E_INVALID_SHAPE


def test_register_rejects_bad_tables():
    L = B.lib()
    assert L.bode_register_kernels(None, 1, 8) == A.E_INVALID_SHAPE
    buf = (ctypes.c_char * 4096)()
    assert L.bode_register_kernels(buf, 1, 7) == A.E_UNSUPPORTED  # layout mismatch


def test_repack_api_validation_without_device():
    """Argument checks come first; without a device the calls fail loudly
    (NO_DEVICE), never silently."""
    import pytest as _pt
    p = B.problems.pleiades()
    with _pt.raises(B.api.InvalidShape):
        B.api.repack_by_cost(p, 0, 1, 0, 1, 1)
    if B.lib().bode_device_count() == 0:
        with _pt.raises(B.api.NoDevice):
            B.api.repack_by_cost(p, 16, 1, 0, 1, 1)
        with _pt.raises(B.api.NoDevice):
            B.api.order_init(1, 16)
