"""The EXACT policy's cbrt must equal the host libm cbrt the reference calls
(rkc.cpp:177-190) bit for bit: RKC step-size control is chaotic at the
ulp level, so a 1-ulp cbrt difference breaks RKC parity."""
import ctypes
import ctypes.util

import numpy as np
import pytest

LIBM = ctypes.CDLL(ctypes.util.find_library("m"))
LIBM.cbrt.restype = ctypes.c_double
LIBM.cbrt.argtypes = [ctypes.c_double]


def sample_inputs(n, seed=1234):
    rng = np.random.default_rng(seed)
    x = 10.0 ** rng.uniform(-40, 6, n)             # controller range (err, errOld)
    bits = rng.integers(0, 2 ** 63, n // 4, dtype=np.uint64).view(np.float64)
    bits = bits[np.isfinite(bits)]
    special = np.array([0.0, -0.0, 1.0, -1.0, 8.0, 27.0, 1e-310, 5e-324, np.inf, -np.inf,
                        2.0 ** 1023, 1.0 - 2.0 ** -53])
    return np.concatenate([x, -x[: n // 8], bits, special])


def libm_cbrt(x):
    f = np.frompyfunc(LIBM.cbrt, 1, 1)
    return f(x).astype(np.float64)


def test_restated_glibc_cbrt_matches_libm(oracle):
    x = sample_inputs(400_000)
    f = oracle.lib.orc_glibc_cbrt
    f.restype, f.argtypes = ctypes.c_double, [ctypes.c_double]
    got = np.frompyfunc(f, 1, 1)(x).astype(np.float64)
    assert np.array_equal(got.view(np.uint64), libm_cbrt(x).view(np.uint64))


@pytest.mark.gpu
def test_device_cbrt_matches_host_libm(gpu):
    from paper_1611_02274_b200 import _abi as A
    x = sample_inputs(4_000_000, seed=77)
    out = np.empty_like(x)
    gpu.api.check(gpu.lib().bode_selftest_cbrt(A.dptr(x), A.dptr(out), x.size))
    ref = libm_cbrt(x)
    bad = np.flatnonzero(out.view(np.uint64) != ref.view(np.uint64))
    assert bad.size == 0, f"{bad.size} mismatches, first x={x[bad[:3]]}"
