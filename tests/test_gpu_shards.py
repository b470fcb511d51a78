"""Shards, leases and the asynchronous snapshot sink on the device.

* bode_int_driver / bode_outer_loop with `num_gpus` (the reference's
  `workers`) above the device count put several shards on one device; the
  results are bitwise those of one shard (test_batch.cpp:127-142), which also
  exercises the 2-D shard copies of the multi-GPU path on a one-GPU box.
* Outer-loop snapshots are staged on the device and copied to the host while
  the next window computes; every snapshot equals the state after that window
  from separate integrateBatch calls, in window order
  (batch_driver.cpp:104-114).
* Calls from several host threads, and a sink that itself integrates on the
  same device, get separate device buffers (no shared per-device state).
"""
import os
import subprocess
import sys
import threading
import time

import numpy as np
import pytest

import paper_1611_02274_b200 as B
from paper_1611_02274_b200 import _abi as A
from golden_cases import PLEIADES_IC, heat_ic, perturb

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIELDS = ("steps_accepted", "steps_rejected", "rhs_evals", "spec_rad_evals", "stages_total",
          "h_min_seen", "h_max_seen", "underflow")


def same(a, b):
    return np.array_equal(np.asarray(a).view(np.uint64), np.asarray(b).view(np.uint64))


def same_stats(a, b):
    return all(np.array_equal(a[k], b[k]) for k in FIELDS)


@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("solver", ["rkck", "rkc"])
def test_int_driver_worker_invariance(gpu, solver, pinned):
    import torch
    if solver == "rkck":
        prob, base, num = B.problems.pleiades(), PLEIADES_IC, 200_001
    else:
        prob, base, num = B.problems.heat_equation(64), heat_ic(64), 70_001
    y0 = perturb(base, 0.01, 5, num)
    outs = []
    for workers in (1, 2, 3, 8):
        yb = torch.from_numpy(y0.copy())
        if pinned:
            yb = yb.pin_memory()
        b = B.BatchStates(num, prob.dim, 0, yb.numpy(), np.zeros(0))
        st = A.empty_stats(num)
        B.api.check(B.lib().bode_int_driver(
            A.Problem(prob.kind, prob.dim, 0, 0), A.SOLVER_NAMES[solver], A.ARITH_EXACT, 0.0,
            0.1, num, None, A.dptr(b.values), A.default_tol(), A.vptr(st), workers))
        outs.append((b.values.copy(), st))
    for y, st in outs[1:]:
        assert same(y, outs[0][0]) and same_stats(st, outs[0][1])


@pytest.mark.parametrize("with_sink", [False, True])
def test_outer_loop_worker_invariance(gpu, with_sink):
    prob = B.problems.pleiades()
    num = 150_003
    b = B.problems.perturb_initial_conditions(PLEIADES_IC, 0.01, 9, num)
    res = []
    for workers in (1, 2, 5):
        snaps = []
        sink = (lambda t, s: snaps.append((t, s.values.copy()))) if with_sink else None
        r = B.outer_loop(prob, b, 0.0, 0.5, 0.1, solver="rkck", gpus=workers, sink=sink)
        res.append((r, snaps))
    r0, s0 = res[0]
    for r, s in res[1:]:
        assert same(r.states.values, r0.states.values) and same_stats(r.stats, r0.stats)
        assert [t for t, _ in s] == [t for t, _ in s0]
        assert all(same(a, c) for (_, a), (_, c) in zip(s, s0))


@pytest.mark.parametrize("solver,problem", [("rkck", "pleiades"), ("rkc", "heat64"),
                                            ("rkc", "expdecay")])
def test_async_snapshots_equal_windowed_integrate_batch(gpu, solver, problem):
    """Snapshot k == the state after k integrateBatch windows, bitwise; the
    snapshot is the caller's order even when the outer loop re-packs (expDecay
    is presorted by g0)."""
    if problem == "pleiades":
        prob = B.problems.pleiades()
        b = B.problems.perturb_initial_conditions(PLEIADES_IC, 0.01, 3, 100_000)
    elif problem == "heat64":
        prob = B.problems.heat_equation(64)
        b = B.problems.perturb_initial_conditions(heat_ic(64), 0.01, 3, 30_000)
    else:
        from paper_1611_02274_b200.api import stiffness_params
        prob = B.problems.exp_decay()
        b = B.problems.perturb_initial_conditions(np.array([1.0]), 0.01, 3, 100_000)
        b.param_dim, b.params = 1, stiffness_params(100_000)
    snaps, tids = [], []
    r = B.outer_loop(prob, b, 0.0, 1.0, 0.1, solver=solver,
                     sink=lambda t, s: (snaps.append((t, s.values.copy())),
                                        tids.append(threading.get_ident())))
    assert [t for t, _ in snaps] == [B.lib().bode_window_end(0.0, 1.0, 0.1, k)
                                     for k in range(1, 11)]
    assert len(set(tids[:-1])) == 1  # windows 1..n-1 from one library thread, in order
    cur = b
    for k in range(1, 11):
        w = B.integrate_batch(prob, cur, B.lib().bode_window_end(0.0, 1.0, 0.1, k - 1) if k > 1
                              else 0.0, B.lib().bode_window_end(0.0, 1.0, 0.1, k), solver=solver)
        cur = w.states
        assert same(snaps[k - 1][1], cur.values), k
    assert same(r.states.values, cur.values)


def test_async_sink_overlaps_the_next_window(gpu):
    """With a sink, each window's snapshot D2H runs under the next window's
    kernel: the loop costs about the same as without a sink, below the
    no-sink time plus one synchronous D2H per window. (C-level call with a
    no-op sink, so only the library's own snapshot path is timed.)"""
    import ctypes
    import torch
    num = 1 << 19
    prob = A.make_problem(A.HEAT, 64)
    y0 = B.problems.perturb_initial_conditions(heat_ic(64), 0.01, 4, num).values
    yh = torch.from_numpy(y0.copy()).pin_memory()
    yp = ctypes.cast(yh.data_ptr(), ctypes.POINTER(ctypes.c_double))
    st = A.empty_stats(num)
    L = B.lib()
    calls = [0]

    def noop(t, y, n, d, u):
        calls[0] += 1

    cb = B.api.SINK(noop)
    steps = ctypes.c_int32(0)

    def run(sink, t_end=1.0):
        yh.copy_(torch.from_numpy(y0))
        t = time.perf_counter()
        B.api.check(L.bode_outer_loop(ctypes.byref(prob), 1, 0, 0.0, t_end, 0.1, num, None, yp,
                                      ctypes.byref(A.default_tol()), A.vptr(st), 1, sink, None,
                                      ctypes.byref(steps)))
        return time.perf_counter() - t

    run(B.api.SINK(), 0.2)
    run(cb, 0.2)  # warm: pinned staging is cached after the first sink call
    calls[0] = 0
    t_plain = min(run(B.api.SINK()) for _ in range(2))
    t_sink = min(run(cb) for _ in range(2))
    d = torch.empty(num * 64, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(9):
        yh.copy_(d)
    torch.cuda.synchronize()
    t_d2h = time.perf_counter() - t
    print(f"outer loop 2^19 heat64: plain {t_plain*1e3:.1f} ms, with sink {t_sink*1e3:.1f} ms, "
          f"9 synchronous snapshot D2H {t_d2h*1e3:.1f} ms")
    assert calls[0] == 20
    assert t_sink < t_plain + 0.5 * t_d2h + 0.01


def test_concurrent_calls_and_nested_sink(gpu):
    """Two host threads run outer loops on the same device at once, and a sink
    integrates another batch on that device from inside the loop: each call
    has its own leased buffers, so every result equals its serial run."""
    prob = B.problems.pleiades()
    ba = B.problems.perturb_initial_conditions(PLEIADES_IC, 0.01, 21, 50_000)
    bb = B.problems.perturb_initial_conditions(PLEIADES_IC, 0.01, 22, 70_000)
    ref_a = B.outer_loop(prob, ba, 0.0, 0.5, 0.1, solver="rkck")
    ref_b = B.outer_loop(prob, bb, 0.0, 0.5, 0.1, solver="rkck")
    ref_w = B.integrate_batch(prob, bb, 0.0, 0.1, solver="rkck")
    got = {}

    def run(key, batch):
        got[key] = B.outer_loop(prob, batch, 0.0, 0.5, 0.1, solver="rkck")

    ths = [threading.Thread(target=run, args=("a", ba)), threading.Thread(target=run, args=("b", bb))]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    assert same(got["a"].states.values, ref_a.states.values)
    assert same(got["b"].states.values, ref_b.states.values)
    nested = []
    r = B.outer_loop(prob, ba, 0.0, 0.5, 0.1, solver="rkck",
                     sink=lambda t, s: nested.append(
                         B.integrate_batch(prob, bb, 0.0, 0.1, solver="rkck").states.values))
    assert same(r.states.values, ref_a.states.values)
    assert len(nested) == 5 and all(same(v, ref_w.states.values) for v in nested)


def test_multirank_bench_path_shared_gpu(gpu):
    """bench.py's multi-rank path (torchrun, 2 ranks, contiguous shards of a
    fixed batch, the final gather to rank 0) on one GPU with gloo plumbing;
    the gathered states equal the single-process run bitwise."""
    env = dict(os.environ, BODE_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533",
           os.path.join(REPO, "tools", "multirank_check.py"), "--systems", "300001"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=REPO)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert "MULTIRANK_OK" in out.stdout, out.stdout[-3000:]


@pytest.mark.parametrize("pinned", [False, True])
def test_block_cyclic_shards_bitwise(gpu, pinned):
    """bode_set_shard_layout(1): blocks dealt round robin over the shards (here
    several shards on one device); int_driver and the outer loop (with a sink,
    on a batch sorted by stiffness, presorted per shard) equal one shard bitwise."""
    import torch
    from paper_1611_02274_b200.api import stiffness_params
    L = B.lib()
    num = 300_001
    g = np.sort(stiffness_params(num))  # sorted by cost: contiguous shards would be unbalanced
    y0 = perturb(np.array([1.0]), 0.01, 5, num)
    prob = A.Problem(A.EXPDECAY, 1, 1, 0)

    def run(workers, layout):
        yb = torch.from_numpy(y0.copy())
        gb = torch.from_numpy(g.copy())
        if pinned:
            yb, gb = yb.pin_memory(), gb.pin_memory()
        st = A.empty_stats(num)
        L.bode_set_shard_layout(layout)
        snaps = []
        sink = B.api.SINK(lambda t, ys, n, d, u: snaps.append(
            np.ctypeslib.as_array(ys, shape=(n * d,)).copy()))
        steps = A.ctypes.c_int32(0)
        try:
            B.api.check(L.bode_outer_loop(prob, A.SOLVER_RKC, A.ARITH_EXACT, 0.0, 0.3, 0.1, num,
                                          A.dptr(gb.numpy()), A.dptr(yb.numpy()), A.default_tol(),
                                          A.vptr(st), workers, sink, None, A.ctypes.byref(steps)))
        finally:
            L.bode_set_shard_layout(0)
        y1 = yb.numpy().copy()
        yb.copy_(torch.from_numpy(y0))
        st1 = A.empty_stats(num)
        L.bode_set_shard_layout(layout)
        try:
            B.api.check(L.bode_int_driver(prob, A.SOLVER_RKC, A.ARITH_EXACT, 0.0, 0.1, num,
                                          A.dptr(gb.numpy()), A.dptr(yb.numpy()), A.default_tol(),
                                          A.vptr(st1), workers))
        finally:
            L.bode_set_shard_layout(0)
        return y1, st, snaps, yb.numpy().copy(), st1

    ref = run(1, 0)
    for workers in (2, 3, 8):
        got = run(workers, 1)
        assert same(got[0], ref[0]) and same_stats(got[1], ref[1])
        assert len(got[2]) == len(ref[2]) == 3
        assert all(same(a, b) for a, b in zip(got[2], ref[2]))
        assert same(got[3], ref[3]) and same_stats(got[4], ref[4])
