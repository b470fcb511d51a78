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
