"""The EXACT policy's pow must equal the host libm pow the reference calls in
rkck::adjustStep (rkck.cpp:105, :109) bit for bit: Pleiades trajectories with
close encounters amplify a 1-ulp step-size difference past the 1e-13 bar.
glibc 2.39's x86-64 FMA pow is restated in oracle/bode_oracle.c (CPU) and
paper_1611_02274_b200/csrc/arith.cuh (device), both over the loaded libm's tables."""
import ctypes
import ctypes.util

import numpy as np
import pytest

LIBM = ctypes.CDLL(ctypes.util.find_library("m"))
LIBM.pow.restype = ctypes.c_double
LIBM.pow.argtypes = [ctypes.c_double, ctypes.c_double]


def inputs(n, seed):
    rng = np.random.default_rng(seed)
    x = np.concatenate([10 ** rng.uniform(-4, 6, n), 1 + rng.uniform(-1e-3, 1e-3, n // 8),
                        10 ** rng.uniform(-300, 300, n // 8), [1.0, 2.0, 1.89e-4, 1e300]])
    y = np.concatenate([rng.choice([-0.2, -0.25], n), rng.uniform(-3, 3, n // 8),
                        rng.choice([-0.2, 0.5], n // 8), [-0.2, -0.25, -0.2, -0.25]])
    return x, y


def host_pow(x, y):
    return np.frompyfunc(LIBM.pow, 2, 1)(x, y).astype(np.float64)


def test_restated_glibc_pow_matches_libm(oracle):
    f = oracle.lib.orc_glibc_pow
    f.restype, f.argtypes = ctypes.c_double, [ctypes.c_double, ctypes.c_double]
    x, y = inputs(300_000, 1)
    with np.errstate(over="ignore"):
        got = np.frompyfunc(f, 2, 1)(x, y).astype(np.float64)
        ref = host_pow(x, y)
    assert np.array_equal(got.view(np.uint64), ref.view(np.uint64))


@pytest.mark.gpu
def test_device_pow_matches_host_libm(gpu):
    from paper_1611_02274_b200 import _abi as A
    assert gpu.lib().bode_pow_exact_available() == 1
    x, y = inputs(3_000_000, 2)
    out = np.empty_like(x)
    gpu.api.check(gpu.lib().bode_selftest_pow(A.dptr(x), A.dptr(y), A.dptr(out), x.size))
    with np.errstate(over="ignore"):
        ref = host_pow(x, y)
    bad = np.flatnonzero(out.view(np.uint64) != ref.view(np.uint64))
    assert bad.size == 0, f"{bad.size} mismatches, e.g. x={x[bad[:3]]} y={y[bad[:3]]}"
