"""Cost-aware re-packing (csrc/repack.cu, bode_repack_by_cost / bode_unpack /
bode_lockstep_efficiency) and its use inside bode_outer_loop. Re-packing moves
systems between positions only, so every result must stay bitwise the same."""
import ctypes

import numpy as np
import pytest

import paper_1611_02274_b200 as B
from paper_1611_02274_b200 import _abi as A
from golden_cases import CASES, build_inputs

pytestmark = pytest.mark.gpu


def vp(t):
    return ctypes.c_void_p(t.data_ptr())


def test_repack_unpack_roundtrip(gpu):
    import torch
    L = B.lib()
    num, dim, pdim = 5000, 6, 2
    rng = np.random.default_rng(3)
    y0 = rng.standard_normal(num * dim)
    g0 = rng.standard_normal(num * pdim)
    st0 = A.empty_stats(num)
    st0["rhs_evals"] = rng.integers(0, 1000, num)
    st0["steps_accepted"] = np.arange(num)
    prob = A.Problem(kind=A.DIAG, dim=dim, param_dim=pdim, reserved=0)
    y = torch.from_numpy(y0.copy()).cuda()
    g = torch.from_numpy(g0.copy()).cuda()
    st = torch.from_numpy(st0.view(np.uint8).copy()).cuda()
    order = torch.empty(num, dtype=torch.int64, device="cuda")
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    B.api.check(L.bode_order_init(vp(order), num, s))
    B.api.check(L.bode_repack_by_cost(ctypes.byref(prob), num, vp(y), vp(g), vp(st), vp(order), s))
    torch.cuda.synchronize()
    o = order.cpu().numpy()
    assert np.array_equal(np.sort(o), np.arange(num))
    sp = st.cpu().numpy().view(A.STATS_DTYPE)
    assert np.all(np.diff(sp["rhs_evals"]) >= 0)                   # sorted by cost
    assert np.array_equal(sp["steps_accepted"], o)                  # stats moved with systems
    # stable: equal costs keep their original relative order
    for c in np.unique(sp["rhs_evals"])[:20]:
        assert np.all(np.diff(o[sp["rhs_evals"] == c]) > 0)
    assert np.array_equal(y.cpu().numpy().reshape(dim, num), y0.reshape(dim, num)[:, o])
    assert np.array_equal(g.cpu().numpy().reshape(pdim, num), g0.reshape(pdim, num)[:, o])
    B.api.check(L.bode_unpack(ctypes.byref(prob), num, vp(y), vp(g), vp(st), vp(order), s))
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy(), y0)
    assert np.array_equal(g.cpu().numpy(), g0)
    assert np.array_equal(st.cpu().numpy().view(A.STATS_DTYPE), st0)
    assert np.array_equal(order.cpu().numpy(), np.arange(num))


def _config4(num):
    case = dict(CASES["cfg4_expdecay_rkc_stiff"])
    return build_inputs(case, num)


def test_lockstep_efficiency_natural_vs_sorted(gpu):
    import torch
    L = B.lib()
    num = 1 << 16
    prob, solver, y0, g = _config4(num)
    effs = {}
    for name, order in (("natural", np.arange(num)), ("sorted", np.argsort(g, kind="stable"))):
        y = torch.from_numpy(y0[order].copy()).cuda()
        gd = torch.from_numpy(g[order].copy()).cuda()
        st = torch.zeros(num * 8, dtype=torch.int64, device="cuda")
        s = torch.cuda.current_stream().cuda_stream
        B.int_driver_device(B.OdeProblem(prob.kind, prob.dim, prob.param_dim), "rkc", "exact",
                            0.0, 0.1, num, gd.data_ptr(), y.data_ptr(), A.default_tol(),
                            st.data_ptr(), False, s)
        e = ctypes.c_double()
        B.api.check(L.bode_lockstep_efficiency(ctypes.byref(prob), A.SOLVER_RKC, A.ARITH_EXACT,
                                               num, vp(st), ctypes.byref(e), ctypes.c_void_p(s)))
        effs[name] = e.value
    assert effs["natural"] < 0.6 < 0.9 < effs["sorted"], effs


def test_outer_loop_repack_is_bitwise_invisible(gpu):
    """Config 4 through bode_outer_loop with per-window snapshots: the automatic
    re-packing (default threshold 0.7 triggers on this batch) changes nothing."""
    L = B.lib()
    num = 1 << 15
    prob, solver, y0, g = _config4(num)
    runs = {}
    B.api.check(L.bode_set_presort_param(-1))  # the cost re-pack, not the g0 presort
    for thr in (0.0, 0.7):
        B.api.check(L.bode_set_repack_threshold(thr))
        snaps = []
        batch = B.BatchStates(num, prob.dim, prob.param_dim, y0.copy(), g.copy())
        r = B.outer_loop(B.OdeProblem(prob.kind, prob.dim, prob.param_dim), batch, 0.0, 1.0, 0.1,
                         solver="rkc", arith="exact",
                         sink=lambda t, b: snaps.append((t, b.values.copy())))
        runs[thr] = (r, snaps)
    B.api.check(L.bode_set_repack_threshold(0.7))
    B.api.check(L.bode_set_presort_param(-2))
    (r0, s0), (r1, s1) = runs[0.0], runs[0.7]
    assert np.array_equal(r0.states.values.view(np.uint64), r1.states.values.view(np.uint64))
    for k in A.STATS_DTYPE.names:
        assert np.array_equal(r0.stats[k], r1.stats[k]), k
    assert len(s0) == len(s1) == 10
    for (t0, a), (t1, b) in zip(s0, s1):
        assert t0 == t1 and np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.parametrize("with_sink,t_end", [(False, 1.0), (True, 1.0), (False, 0.1)])
def test_outer_loop_presort_by_param_is_bitwise_invisible(gpu, with_sink, t_end):
    """bode_set_presort_param(0): config 4 sorted by |g0| before the first
    window (bode_repack_by_param), snapshots and the result in the caller's
    order, bitwise the unsorted run's."""
    L = B.lib()
    num = 1 << 15
    prob, solver, y0, g = _config4(num)
    runs = {}
    for row in (-1, 0):
        B.api.check(L.bode_set_presort_param(row))
        snaps = []
        batch = B.BatchStates(num, prob.dim, prob.param_dim, y0.copy(), g.copy())
        sink = (lambda t, b: snaps.append((t, b.values.copy()))) if with_sink else None
        r = B.outer_loop(B.OdeProblem(prob.kind, prob.dim, prob.param_dim), batch, 0.0, t_end,
                         0.1, solver="rkc", arith="exact", sink=sink)
        runs[row] = (r, snaps)
    B.api.check(L.bode_set_presort_param(-2))  # back to the default
    (r0, s0), (r1, s1) = runs[-1], runs[0]
    assert np.array_equal(r0.states.values.view(np.uint64), r1.states.values.view(np.uint64))
    for k in A.STATS_DTYPE.names:
        assert np.array_equal(r0.stats[k], r1.stats[k]), k
    assert len(s0) == len(s1)
    for (t0, a), (t1, b) in zip(s0, s1):
        assert t0 == t1 and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_repack_by_param_sorts_and_unpacks(gpu):
    """bode_repack_by_param orders the batch by |g0| (stable), moves y and the
    order map with it, and bode_unpack restores the caller's order."""
    import torch
    num = 5000
    prob, solver, y0, g = _config4(num)
    y = torch.from_numpy(y0.copy()).cuda()
    gd = torch.from_numpy(g.copy()).cuda()
    order = torch.zeros(num, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    p = B.OdeProblem(prob.kind, prob.dim, prob.param_dim)
    B.api.order_init(order.data_ptr(), num, s)
    B.api.repack_by_param(p, num, y.data_ptr(), gd.data_ptr(), 0, order.data_ptr(), 0, s)
    torch.cuda.synchronize()
    perm = np.argsort(np.abs(g).astype(np.float32), kind="stable")
    assert np.array_equal(order.cpu().numpy(), perm)
    assert np.array_equal(gd.cpu().numpy(), g[perm])
    assert np.array_equal(y.cpu().numpy(), y0[perm])
    B.api.unpack_order(p, num, y.data_ptr(), gd.data_ptr(), 0, order.data_ptr(), s)
    torch.cuda.synchronize()
    assert np.array_equal(gd.cpu().numpy(), g) and np.array_equal(y.cpu().numpy(), y0)


@pytest.mark.parametrize("gpus", [1, 3])
def test_int_driver_presort_is_bitwise_invisible(gpu, gpus):
    """bode_int_driver sorts a config-4 batch by |g0| around its window (the
    default presort parameter) and restores the caller's order: bitwise the
    unsorted run, with one shard or three (several on one device)."""
    import time
    L = B.lib()
    num = 1 << 17
    prob, solver, y0, g = _config4(num)
    out, secs = {}, {}
    for row in (-1, -2):
        B.api.check(L.bode_set_presort_param(row))
        batch = B.BatchStates(num, prob.dim, prob.param_dim, y0.copy(), g.copy())
        t = time.perf_counter()
        out[row] = B.integrate_batch(B.OdeProblem(prob.kind, prob.dim, prob.param_dim), batch,
                                     0.0, 0.1, solver="rkc", arith="exact", gpus=gpus)
        secs[row] = time.perf_counter() - t
    B.api.check(L.bode_set_presort_param(-2))
    a, b = out[-1], out[-2]
    assert np.array_equal(a.states.values.view(np.uint64), b.states.values.view(np.uint64))
    for k in A.STATS_DTYPE.names:
        assert np.array_equal(a.stats[k], b.stats[k]), k
    print(f"int_driver config 4, {num} systems: natural {secs[-1] * 1e3:.1f} ms, "
          f"presorted {secs[-2] * 1e3:.1f} ms")


@pytest.mark.parametrize("merge", [False, True])
def test_int_driver_device_presort_is_bitwise_invisible(gpu, merge):
    """bode_int_driver_device sorts a config-4 batch by |g0| around its window
    in a stream-ordered scratch (the caller's g is only read) and copies the
    results back in the caller's order: bitwise the unsorted window, stats
    merged or not."""
    import torch
    L = B.lib()
    num = 100_003
    prob, solver, y0, g = _config4(num)
    out = {}
    for row in (-1, -2):
        B.api.check(L.bode_set_presort_param(row))
        yd = torch.from_numpy(y0.copy()).cuda()
        gd = torch.from_numpy(g.copy()).cuda()
        st = torch.zeros(num * 8, dtype=torch.int64, device="cuda")
        p = B.OdeProblem(prob.kind, prob.dim, prob.param_dim)
        for k in range(2 if merge else 1):
            B.int_driver_device(p, "rkc", "exact", 0.1 * k, 0.1 * (k + 1), num, gd.data_ptr(),
                                yd.data_ptr(), A.default_tol(), st.data_ptr(), merge and k > 0, 0)
        torch.cuda.synchronize()
        assert np.array_equal(gd.cpu().numpy().view(np.uint64), g.view(np.uint64))  # g untouched
        out[row] = (yd.cpu().numpy(), st.cpu().numpy().view(A.STATS_DTYPE))
    B.api.check(L.bode_set_presort_param(-2))
    (ya, sa), (yb, sb) = out[-1], out[-2]
    assert np.array_equal(ya.view(np.uint64), yb.view(np.uint64))
    for k in A.STATS_DTYPE.names:
        assert np.array_equal(sa[k], sb[k]), k
