"""The EXACT policy's branch-free sqrt / reciprocal / division (arith.cuh
sqrt_rn_bf, rcp_rn_bf on [2^-400, 2^400]; div_rn_nv wherever it reports the
intrinsic's fast path) must be bitwise the IEEE round-to-nearest results;
outside those domains the kernels fall back to the intrinsics. Checked on random bit patterns, log-uniform values, the
Pleiades r^2 range and mantissa edge cases."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def cases(n, seed):
    rng = np.random.default_rng(seed)
    lo, hi = 1023 - 400, 1023 + 400
    exps = rng.integers(lo, hi + 1, n, dtype=np.uint64)
    mant = rng.integers(0, 1 << 52, n, dtype=np.uint64)
    rand_bits = ((exps << np.uint64(52)) | mant).view(np.float64)
    edge_m = np.array([0, 1, 2, (1 << 52) - 1, (1 << 52) - 2, 1 << 51, (1 << 51) - 1,
                       (1 << 51) + 1], dtype=np.uint64)
    e2 = np.repeat(np.arange(lo, hi + 1, dtype=np.uint64), edge_m.size)
    edges = ((e2 << np.uint64(52)) | np.tile(edge_m, hi - lo + 1)).view(np.float64)
    pleiades = rng.uniform(1e-6, 400.0, n // 2)  # r2 = dx^2 + dy^2 of star pairs
    return np.concatenate([rand_bits, edges, pleiades, pleiades * np.sqrt(pleiades)])


def full_range_cases(n, seed):
    """Every exponent (subnormals, Inf, NaN included), random and edge
    significands, both signs: the EXACT sqrt_ / operator/ wrappers must equal
    the intrinsics everywhere, through their fallback where needed."""
    rng = np.random.default_rng(seed)
    bits = rng.integers(0, 1 << 63, n, dtype=np.uint64) | (rng.integers(0, 2, n, dtype=np.uint64) << np.uint64(63))
    x = bits.view(np.float64)
    edge = np.array([0.0, -0.0, 5e-324, -5e-324, 2.2250738585072014e-308, np.inf, -np.inf,
                     np.nan, 1.0, -1.0, 1.7976931348623157e308, 2.0 ** -970, 2.0 ** -971,
                     2.0 ** 1023])
    return np.concatenate([x, np.repeat(edge, 2), np.tile(edge, 2)])


@pytest.mark.parametrize("op", [3, 4], ids=["sqrt_policy", "div_policy"])
def test_policy_ops_match_ieee_everywhere(gpu, op):
    from paper_1611_02274_b200 import _abi as A
    bad, first = ctypes.c_int64(), ctypes.c_int64()
    for seed in range(4):
        x = full_range_cases(5_000_000, 50 + seed)
        gpu.api.check(gpu.lib().bode_selftest_exact_math(A.dptr(x), x.size, op,
                                                         ctypes.byref(bad), ctypes.byref(first)))
        assert bad.value == 0, f"{bad.value} mismatches, first x = {x[first.value]!r}"


@pytest.mark.parametrize("op", [0, 1, 2], ids=["sqrt", "rcp", "div"])
def test_branch_free_matches_ieee(gpu, op):
    from paper_1611_02274_b200 import _abi as A
    bad, first = ctypes.c_int64(), ctypes.c_int64()
    for seed in range(10):
        x = cases(10_000_000, seed)
        if op == 2:  # random (a, b) pairs, signs included
            rng = np.random.default_rng(100 + seed)
            x = x[rng.permutation(x.size)] * rng.choice([-1.0, 1.0], x.size)
        gpu.api.check(gpu.lib().bode_selftest_exact_math(A.dptr(x), x.size, op,
                                                         ctypes.byref(bad), ctypes.byref(first)))
        assert bad.value == 0, f"{bad.value} mismatches, first x = {x[first.value]!r}"


def test_div_zero_numerator(gpu):
    """+0 / b takes the straight-line division for every positive normal b
    (the padding of run-time-dimension systems); -0 / b, +0 / subnormal, Inf,
    NaN and negative b must still report the slow path or agree bitwise."""
    from paper_1611_02274_b200 import _abi as A
    bad, first = ctypes.c_int64(), ctypes.c_int64()
    b = np.concatenate([full_range_cases(2_000_000, 77), cases(1_000_000, 78)])
    for a in (0.0, -0.0):
        x = np.empty(2 * b.size)
        x[0::2], x[1::2] = a, b
        gpu.api.check(gpu.lib().bode_selftest_exact_math(A.dptr(x), x.size, 2,
                                                         ctypes.byref(bad), ctypes.byref(first)))
        assert bad.value == 0, f"{bad.value} mismatches, first pair at {first.value}"
