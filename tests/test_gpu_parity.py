"""GPU parity: the CUDA path (through the C ABI) against the reference.

Bars (BASELINE.json north_star):
  * EXACT policy: bitwise (states and every counter) for RKCK and RKC -- the
    device cbrt and pow reproduce the host glibc ones (tests/test_cbrt.py,
    tests/test_pow.py).
  * FAST policy (FMA, rsqrt): RKCK <= 1e-13 = 1e-3*eps per system with
    identical accepted/rejected/RHS counts on the bench workload (perturbation
    0.01); at the 0.1 stress perturbation close encounters amplify ulp
    differences, so the fraction within the bar is asserted instead. RKC fast is
    reported against the exact run with a looser bound, since RKC step
    selection is chaotic at the ulp level.
Per-system relative error: max_j |dy_j| / max_j |y_j^ref| (acceptance.cpp:142-147).
"""
import math
import os

import numpy as np
import pytest

import paper_1611_02274_b200 as B
from paper_1611_02274_b200 import _abi as A
from golden_cases import CASES, build_inputs, perturb, PLEIADES_IC, heat_ic

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
COUNTS = ("steps_accepted", "steps_rejected", "rhs_evals", "spec_rad_evals", "underflow")


def sysrel(y, yref, num, dim):
    a = y.reshape(dim, num)
    b = yref.reshape(dim, num)
    return np.max(np.abs(a - b), axis=0) / np.maximum(np.max(np.abs(b), axis=0), 1e-300)


def problem_of(p: A.Problem) -> B.OdeProblem:
    return B.OdeProblem(p.kind, p.dim, p.param_dim)


def run_gpu(prob, solver, y0, g, arith, t0=0.0, t1=1.0, hout=0.1, gpus=1):
    num = y0.size // prob.dim
    batch = B.BatchStates(num, prob.dim, prob.param_dim, y0.copy(),
                          g.copy() if g is not None else np.zeros(0))
    r = B.outer_loop(problem_of(prob), batch, t0, t1, hout, solver=solver, arith=arith, gpus=gpus)
    assert r.outer_steps == B.lib().bode_num_windows(t0, t1, hout)
    return r.states.values, r.stats


@pytest.mark.parametrize("name", sorted(CASES))
def test_exact_matches_golden(gpu, name):
    gold = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    prob, solver, y0, g = build_inputs(CASES[name])
    y, st = run_gpu(prob, solver, y0, g, "exact")
    for k in COUNTS:
        assert np.array_equal(st[k], gold[k]), k
    assert np.array_equal(y.view(np.uint64), gold["y"].view(np.uint64))
    assert np.array_equal(st["h_min_seen"], gold["h_min_seen"])
    assert np.array_equal(st["h_max_seen"], gold["h_max_seen"])


@pytest.mark.parametrize("name", ["cfg1_pleiades_rkck_s42", "cfg1_pleiades_rkck_s20140609"])
def test_fast_rkck_within_bar(gpu, name):
    gold = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    prob, solver, y0, g = build_inputs(CASES[name])
    y, st = run_gpu(prob, solver, y0, g, "fast")
    err = sysrel(y, gold["y"], y0.size // 28, 28)
    assert err.max() <= 1e-13, err.max()
    for k in ("steps_accepted", "steps_rejected", "rhs_evals"):
        assert np.array_equal(st[k], gold[k]), k


def test_fast_rkc_close_to_exact(gpu):
    prob, solver, y0, g = build_inputs(CASES["cfg3_heat64_rkc_s42"])
    ye, _ = run_gpu(prob, solver, y0, g, "exact")
    yf, _ = run_gpu(prob, solver, y0, g, "fast")
    err = sysrel(yf, ye, y0.size // 64, 64)
    assert err.max() <= 1e-4, err.max()  # O(relTol): a different, equally valid step sequence


@pytest.mark.parametrize("mag", [0.01, 0.1])
def test_pleiades_large_exact_bitwise(gpu, oracle, mag):
    """2^16 systems; perturbation 0.1 is the divergence stress."""
    num = 1 << 16
    prob = A.make_problem(A.PLEIADES)
    y0 = perturb(PLEIADES_IC, mag, 42, num)
    y, st = run_gpu(prob, A.SOLVER_RKCK, y0, None, "exact")
    rc, yo, so, _ = oracle.outer_loop(prob, A.SOLVER_RKCK, 0.0, 1.0, 0.1, y0)
    assert np.array_equal(y.view(np.uint64), yo.view(np.uint64))
    for k in COUNTS + ("stages_total",):
        assert np.array_equal(st[k], so[k]), k


@pytest.mark.parametrize("mag", [0.01, 0.1])
def test_pleiades_large_fast_within_bar(gpu, oracle, mag):
    num = 1 << 16
    prob = A.make_problem(A.PLEIADES)
    y0 = perturb(PLEIADES_IC, mag, 42, num)
    y, st = run_gpu(prob, A.SOLVER_RKCK, y0, None, "fast")
    rc, yo, so, _ = oracle.outer_loop(prob, A.SOLVER_RKCK, 0.0, 1.0, 0.1, y0)
    err = sysrel(y, yo, num, 28)
    same = np.ones(num, bool)
    for k in ("steps_accepted", "steps_rejected", "rhs_evals", "underflow"):
        same &= st[k] == so[k]
    ok = (err <= 1e-13) & same
    print(f"fast mag={mag}: within bar {ok.mean():.6f}, max rel err {err.max():.2e}, "
          f"count mismatches {(~same).sum()}")
    # at the bench perturbation (0.01) every system is within the bar with
    # identical counts. At the 0.1 stress, close encounters amplify FMA-level
    # differences past 1e-13 on part of the batch (measured 0.835 of systems
    # within the bar, max 5.8e-10) and flip an accept/reject decision on a few
    # (3 of 65536), which is why EXACT is the parity policy there
    if mag == 0.01:
        assert same.all(), (~same).sum()
        assert ok.all(), (err.max(), (~same).sum())
    else:
        assert (~same).mean() <= 1e-3, (~same).sum()
        assert ok.mean() >= 0.8 and err.max() <= 1e-8


def test_heat64_exact_bitwise_vs_oracle(gpu, oracle):
    num = 4096
    prob = A.make_problem(A.HEAT, 64)
    y0 = perturb(heat_ic(64), 0.01, 1234, num)
    y, st = run_gpu(prob, A.SOLVER_RKC, y0, None, "exact")
    rc, yo, so, _ = oracle.outer_loop(prob, A.SOLVER_RKC, 0.0, 1.0, 0.1, y0)
    assert np.array_equal(y.view(np.uint64), yo.view(np.uint64))
    for k in COUNTS + ("stages_total",):
        assert np.array_equal(st[k], so[k]), k


@pytest.mark.parametrize("n", [8, 16, 32])
def test_heat_other_sizes_exact(gpu, oracle, n):
    num = 1024
    prob = A.make_problem(A.HEAT, n)
    y0 = perturb(heat_ic(n), 0.01, 5, num)
    y, st = run_gpu(prob, A.SOLVER_RKC, y0, None, "exact")
    rc, yo, so, _ = oracle.outer_loop(prob, A.SOLVER_RKC, 0.0, 1.0, 0.1, y0)
    assert np.array_equal(y.view(np.uint64), yo.view(np.uint64))
    for k in COUNTS + ("stages_total",):
        assert np.array_equal(st[k], so[k]), k


def test_stiffness_varied_exact_bitwise(gpu, oracle):
    """Config 4 at 2^16 systems: g0 log-uniform in [1, 1e4]."""
    num = 1 << 16
    case = dict(CASES["cfg4_expdecay_rkc_stiff"])
    prob, solver, y0, g = build_inputs(case, num)
    y, st = run_gpu(prob, solver, y0, g, "exact")
    rc, yo, so, _ = oracle.outer_loop(prob, solver, 0.0, 1.0, 0.1, y0, g)
    assert np.array_equal(y.view(np.uint64), yo.view(np.uint64))
    for k in COUNTS + ("stages_total",):
        assert np.array_equal(st[k], so[k]), k


def test_stride_sample_at_2_20(gpu, oracle):
    """Full-size property check: 2^20 Pleiades on the GPU, every 64th system
    re-integrated by the oracle (systems are independent, batch_driver.hpp:16-21)."""
    num = 1 << 20
    prob = A.make_problem(A.PLEIADES)
    y0 = perturb(PLEIADES_IC, 0.01, 42, num)
    idx = np.arange(0, num, 64)
    sub = np.ascontiguousarray(y0.reshape(28, num)[:, idx]).reshape(-1)
    rc, yo, so, _ = oracle.outer_loop(prob, A.SOLVER_RKCK, 0.0, 1.0, 0.1, sub)
    for arith in ("exact", "fast"):
        y, st = run_gpu(prob, A.SOLVER_RKCK, y0, None, arith)
        got = np.ascontiguousarray(y.reshape(28, num)[:, idx]).reshape(-1)
        if arith == "exact":
            assert np.array_equal(got.view(np.uint64), yo.view(np.uint64))
        else:
            assert sysrel(got, yo, idx.size, 28).max() <= 1e-13
        assert np.array_equal(st["steps_accepted"][idx], so["steps_accepted"])
        assert np.array_equal(st["steps_rejected"][idx], so["steps_rejected"])


@pytest.mark.parametrize("solver", ["rkck", "rkc"])
def test_block_size_invariance(gpu, solver):
    """Results are bitwise independent of the launch shape (test_batch.cpp:127-142)."""
    if solver == "rkck":
        prob, y0, g = A.make_problem(A.PLEIADES), perturb(PLEIADES_IC, 0.01, 3, 3000), None
    else:
        prob, y0, g = A.make_problem(A.HEAT, 64), perturb(heat_ic(64), 0.01, 3, 1000), None
    L = B.lib()
    outs = []
    try:
        for bs in (64, 128, 256):
            assert L.bode_set_block_size(bs) == 0
            outs.append(run_gpu(prob, solver, y0, g, "exact")[0])
    finally:
        L.bode_set_block_size(0)
    assert all(np.array_equal(o.view(np.uint64), outs[0].view(np.uint64)) for o in outs[1:])


def test_outer_loop_equals_windowed_int_driver(gpu):
    """Device-resident outerLoop == 10 host-pointer integrateBatch windows."""
    prob = B.problems.heat_equation(64)
    b = B.problems.perturb_initial_conditions(heat_ic(64), 0.01, 11, 777)
    r = B.outer_loop(prob, b, 0.0, 1.0, 0.1, solver="rkc")
    cur = b
    acc = np.zeros(777, dtype=np.int64)
    for k in range(1, 11):
        t0 = 0.0 if k == 1 else 0.0 + (k - 1) * 0.1
        t1 = 1.0 if k == 10 else 0.0 + k * 0.1
        w = B.integrate_batch(prob, cur, t0, t1, solver="rkc")
        cur = w.states
        acc += w.stats["steps_accepted"]
    assert np.array_equal(cur.values.view(np.uint64), r.states.values.view(np.uint64))
    assert np.array_equal(acc, r.stats["steps_accepted"])


def test_device_pointer_entry_with_torch(gpu):
    import torch
    prob = A.make_problem(A.PLEIADES)
    num = 5000
    y0 = perturb(PLEIADES_IC, 0.01, 8, num)
    yd = torch.from_numpy(y0.copy()).cuda()
    st = torch.zeros(num * 8, dtype=torch.int64, device="cuda")
    tol = A.default_tol()
    s = torch.cuda.current_stream()
    B.int_driver_device(problem_of(prob), "rkck", "exact", 0.0, 0.1, num, 0, yd.data_ptr(), tol,
                        st.data_ptr(), False, s.cuda_stream)
    torch.cuda.synchronize()
    host = B.integrate_batch(problem_of(prob), B.BatchStates(num, 28, 0, y0.copy(), np.zeros(0)),
                             0.0, 0.1)
    assert np.array_equal(yd.cpu().numpy().view(np.uint64), host.states.values.view(np.uint64))


@pytest.mark.parametrize("arith", ["exact", "fast"])
def test_persistent_refill_is_bitwise_static(gpu, arith):
    """Dynamic refill changes which lane integrates which system, never the
    result: bitwise under EXACT; under FAST the two kernels may contract FMAs
    differently, so the tolerance bar applies."""
    import os as _os
    prob = A.make_problem(A.PLEIADES)
    y0 = perturb(PLEIADES_IC, 0.1, 17, 50_000)
    L = B.lib()
    outs = []
    try:
        for persistent in (0, 1):
            L.bode_set_persistent(persistent)
            outs.append(run_gpu(prob, A.SOLVER_RKCK, y0, None, arith))
    finally:
        L.bode_set_persistent(0)
    (ys, ss), (yp, sp) = outs
    if arith == "exact":
        assert np.array_equal(ys.view(np.uint64), yp.view(np.uint64))
        for k in COUNTS + ("stages_total", "h_min_seen", "h_max_seen"):
            assert np.array_equal(ss[k], sp[k]), k
    else:
        assert sysrel(yp, ys, y0.size // 28, 28).max() <= 1e-8
        assert np.array_equal(ss["steps_accepted"], sp["steps_accepted"])


def _stride_check(oracle, prob, solver, base, mag, num, stride, arith, seed=42):
    y0 = perturb(base, mag, seed, num)
    y, st = run_gpu(prob, solver, y0, None, arith)
    idx = np.arange(0, num, stride)
    sub = np.ascontiguousarray(y0.reshape(prob.dim, num)[:, idx]).reshape(-1)
    rc, yo, so, _ = oracle.outer_loop(prob, solver, 0.0, 1.0, 0.1, sub)
    got = np.ascontiguousarray(y.reshape(prob.dim, num)[:, idx]).reshape(-1)
    return got, yo, st, so, idx


@pytest.mark.parametrize("arith", ["exact", "fast"])
def test_rkck_full_size_2_22_stride(gpu, oracle, arith):
    """BASELINE configs[1] at its largest size: 2^22 systems on the GPU, every
    64th re-integrated by the oracle."""
    prob = A.make_problem(A.PLEIADES)
    got, yo, st, so, idx = _stride_check(oracle, prob, A.SOLVER_RKCK, PLEIADES_IC, 0.01, 1 << 22,
                                         64, arith)
    if arith == "exact":
        assert np.array_equal(got.view(np.uint64), yo.view(np.uint64))
    else:
        assert sysrel(got, yo, idx.size, 28).max() <= 1e-13
    for k in ("steps_accepted", "steps_rejected", "rhs_evals"):
        assert np.array_equal(st[k][idx], so[k]), k


def test_rkc_heat64_2_20_stride(gpu, oracle):
    """Config 3 at 2^20 systems, every 256th system re-integrated by the oracle."""
    prob = A.make_problem(A.HEAT, 64)
    got, yo, st, so, idx = _stride_check(oracle, prob, A.SOLVER_RKC, heat_ic(64), 0.01, 1 << 20,
                                         256, "exact")
    assert np.array_equal(got.view(np.uint64), yo.view(np.uint64))
    for k in COUNTS + ("stages_total",):
        assert np.array_equal(st[k][idx], so[k]), k


def test_very_stiff_generator_path_bitwise(gpu, oracle):
    """expDecay with g0 log-uniform in [1e9, 1e11]: about 1700 stages per step,
    far above the per-device coefficient table (s <= 160), so the chunked
    on-the-fly generator path of rkc.cuh runs; states and counters stay bitwise.
    (The oracle rebuilds the coefficients per stage like the reference, O(s^2)
    per step, hence the small batch.)"""
    num = 8
    prob = A.make_problem(A.EXPDECAY)
    u = np.linspace(-1.0, 1.0, num)
    g = 10.0 ** (10.0 + u)
    y0 = 1.0 + 0.5 * u
    y, st = run_gpu(prob, A.SOLVER_RKC, y0, g, "exact", t1=0.1)
    rc, yo, so, _ = oracle.outer_loop(prob, A.SOLVER_RKC, 0.0, 0.1, 0.1, y0, g)
    assert np.array_equal(y.view(np.uint64), yo.view(np.uint64))
    for k in COUNTS + ("stages_total",):
        assert np.array_equal(st[k], so[k]), k
    per_step = st["stages_total"] / np.maximum(st["steps_accepted"] + st["steps_rejected"], 1)
    assert per_step.max() > 160, per_step.max()


@pytest.mark.parametrize("env", [("4", "255"), ("4", "168"), ("8", "168"), ("8", "128"), ("8", "112"), ("8", "96"), ("16", "96"), ("16", "128")])
def test_heat64_lane_variants_bitwise(gpu, oracle, env):
    """Every compiled heat64 RKC instance (lanes per system x register cap,
    selected with BODE_LANES / BODE_MAXREG) gives the oracle's bits."""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, 'tests'); import numpy as np;"
            "from test_gpu_parity import run_gpu; from golden_cases import heat_ic, perturb;"
            "from paper_1611_02274_b200 import _abi as A;"
            "p = A.make_problem(A.HEAT, 64); y0 = perturb(heat_ic(64), 0.01, 42, 2048);"
            "y, st = run_gpu(p, A.SOLVER_RKC, y0, None, 'exact');"
            "np.save(sys.argv[1], y)")
    out = os.path.join(os.environ.get("TMPDIR", "/tmp"), f"heat_variant_{env[0]}_{env[1]}.npy")
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code, out], cwd=repo, capture_output=True, text=True,
                       env=dict(os.environ, BODE_LANES=env[0], BODE_MAXREG=env[1]))
    assert r.returncode == 0, r.stderr[-2000:]
    prob = A.make_problem(A.HEAT, 64)
    y0 = perturb(heat_ic(64), 0.01, 42, 2048)
    rc, yo, so, _ = oracle.outer_loop(prob, A.SOLVER_RKC, 0.0, 1.0, 0.1, y0)
    assert np.array_equal(np.load(out).view(np.uint64), yo.view(np.uint64))


@pytest.mark.parametrize("nwin_end", [0.1, 1.0])
def test_outer_loop_pinned_chunked_pipeline(gpu, nwin_end):
    """With pinned host buffers bode_outer_loop pipelines the first window's
    upload and the last window's download in column chunks (strided launches);
    the results equal the pageable (single-piece) path bit for bit."""
    import ctypes
    import torch
    L = B.lib()
    num = 1 << 18
    prob = A.make_problem(A.PLEIADES)
    y0 = perturb(PLEIADES_IC, 0.01, 42, num)
    tol = A.default_tol()
    outs = {}
    for pinned in (False, True):
        yh = torch.from_numpy(y0.copy())
        sth = torch.zeros(num * 8, dtype=torch.int64)
        if pinned:
            yh, sth = yh.pin_memory(), sth.pin_memory()
        n = ctypes.c_int32(0)
        B.api.check(L.bode_outer_loop(ctypes.byref(prob), A.SOLVER_RKCK, A.ARITH_FAST, 0.0,
                                      nwin_end, 0.1, num, None,
                                      ctypes.cast(yh.data_ptr(), ctypes.POINTER(ctypes.c_double)),
                                      ctypes.byref(tol), ctypes.c_void_p(sth.data_ptr()), 1,
                                      B.api.SINK(), None, ctypes.byref(n)))
        outs[pinned] = (yh.numpy().copy(), sth.numpy().copy())
    assert np.array_equal(outs[False][0].view(np.uint64), outs[True][0].view(np.uint64))
    assert np.array_equal(outs[False][1], outs[True][1])


@pytest.mark.parametrize("num", [1, 3, 33, 1001])
def test_ragged_batch_sizes_bitwise(gpu, oracle, num):
    """Batches that fill neither a warp nor a lane group evenly (1, 3, 33, 1001
    systems) on every default kernel shape: Pleiades RKCK (lane pair, EXACT),
    heat64 RKC (8 lanes per system), expDecay RKC (1 lane): bitwise the oracle."""
    cases = [(A.make_problem(A.PLEIADES), A.SOLVER_RKCK, PLEIADES_IC, None),
             (A.make_problem(A.HEAT, 64), A.SOLVER_RKC, heat_ic(64), None),
             (A.make_problem(A.EXPDECAY), A.SOLVER_RKC, np.array([1.0]),
              np.linspace(1.0, 1e3, num))]
    for prob, solver, base, g in cases:
        y0 = perturb(base, 0.01, 17, num)
        y, st = run_gpu(prob, solver, y0, g, "exact")
        rc, yo, so, _ = oracle.outer_loop(prob, solver, 0.0, 1.0, 0.1, y0, g)
        assert np.array_equal(y.view(np.uint64), yo.view(np.uint64)), (prob.kind, num)
        for k in COUNTS:
            assert np.array_equal(st[k], so[k]), (prob.kind, num, k)


@pytest.mark.parametrize("presort", [False, True])
def test_outer_loop_pinned_params_and_repack(gpu, presort):
    """Pinned buffers with per-system parameters (config 4, P = 1): chunked
    strided upload of y and g, automatic re-packing after window 1, unpack and
    whole download at the end -- bitwise the pageable path and the oracle.
    With presort, the batch is sorted by |g0| before window 1 instead (whole
    upload, bode_set_presort_param)."""
    import ctypes
    import torch
    L = B.lib()
    num = 1 << 18
    case = dict(CASES["cfg4_expdecay_rkc_stiff"])
    prob, solver, y0, g = build_inputs(case, num)
    tol = A.default_tol()
    outs = {}
    B.api.check(L.bode_set_presort_param(0 if presort else -1))
    for pinned in (False, True):
        yh = torch.from_numpy(y0.copy())
        gh = torch.from_numpy(g.copy())
        sth = torch.zeros(num * 8, dtype=torch.int64)
        if pinned:
            yh, gh, sth = yh.pin_memory(), gh.pin_memory(), sth.pin_memory()
        n = ctypes.c_int32(0)
        dp = lambda t: ctypes.cast(t.data_ptr(), ctypes.POINTER(ctypes.c_double))
        B.api.check(L.bode_outer_loop(ctypes.byref(prob), solver, A.ARITH_EXACT, 0.0, 1.0, 0.1,
                                      num, dp(gh), dp(yh), ctypes.byref(tol),
                                      ctypes.c_void_p(sth.data_ptr()), 1, B.api.SINK(), None,
                                      ctypes.byref(n)))
        outs[pinned] = (yh.numpy().copy(), sth.numpy().copy())
    B.api.check(L.bode_set_presort_param(-2))  # back to the default
    assert np.array_equal(outs[False][0].view(np.uint64), outs[True][0].view(np.uint64))
    assert np.array_equal(outs[False][1], outs[True][1])
    idx = np.arange(0, num, 97)
    rc, yo, so, _ = oracle_outer_sample(prob, solver, y0, g, num, idx)
    assert np.array_equal(outs[True][0].reshape(1, num)[:, idx].reshape(-1).view(np.uint64),
                          yo.view(np.uint64))


def oracle_outer_sample(prob, solver, y0, g, num, idx):
    from oracle_lib import Oracle
    sub_y = np.ascontiguousarray(y0.reshape(prob.dim, num)[:, idx]).reshape(-1)
    sub_g = np.ascontiguousarray(g.reshape(prob.param_dim, num)[:, idx]).reshape(-1)
    return Oracle().outer_loop(prob, solver, 0.0, 1.0, 0.1, sub_y, sub_g)


def test_heat64_mixed_groups_per_warp_bitwise(gpu, oracle):
    """The lane-group RKC driver is warp-uniform (rkc.cuh rkc_system): the four
    heat64 systems sharing a warp run every phase together and keep or drop
    the results by their own state. Neighbours here differ in amplitude (so in
    step sizes, stage counts and rejections), include all-zero systems
    (degenerate power method), a NaN system (underflow freeze) and a ragged
    last warp; every system must still be bitwise the oracle's."""
    num = 4 * 64 + 3
    y0 = perturb(heat_ic(64), 0.01, 99, num).reshape(64, num)
    scales = [1.0, 0.0, 1e-150, 1e3, 1e-6, -1.0, 5e2]
    for i in range(num):
        y0[:, i] *= scales[i % len(scales)]
    y0[5, 10] = np.nan
    y0 = np.ascontiguousarray(y0).reshape(-1)
    prob = A.make_problem(A.HEAT, 64)
    y, st = run_gpu(prob, A.SOLVER_RKC, y0, None, "exact")
    rc, yo, so, _ = oracle.outer_loop(prob, A.SOLVER_RKC, 0.0, 1.0, 0.1, y0)
    assert np.array_equal(y.view(np.uint64), yo.view(np.uint64))
    for k in COUNTS + ("stages_total",):
        assert np.array_equal(st[k], so[k]), k
    assert st["underflow"][10] == 1
    assert len(set(st["rhs_evals"].tolist())) > 3  # the groups really did differ


@pytest.mark.parametrize("scale", [2.0 ** 140, 2.0 ** -140])
def test_pleiades_exact_outside_fast_range_bitwise(gpu, oracle, scale):
    """EXACT Pleiades evaluates 1/(r2 sqrt r2) on a straight-line path only
    for r2 in [2^-266, 2^266) (arith.cuh r3_in_safe_range) and falls back to
    the IEEE intrinsics otherwise. Positions scaled by 2^+-140 put every r2
    outside that band; the results must still be the oracle's bits."""
    num = 96
    y0 = perturb(PLEIADES_IC, 0.01, 3, num).reshape(28, num)
    y0[:14] *= scale
    y0 = np.ascontiguousarray(y0).reshape(-1)
    prob = A.make_problem(A.PLEIADES)
    y, st = run_gpu(prob, A.SOLVER_RKCK, y0, None, "exact")
    rc, yo, so, _ = oracle.outer_loop(prob, A.SOLVER_RKCK, 0.0, 1.0, 0.1, y0)
    assert np.array_equal(y.view(np.uint64), yo.view(np.uint64))
    for k in COUNTS:
        assert np.array_equal(st[k], so[k]), k


def test_int_driver_pinned_32_chunk_pipeline(gpu):
    """bode_int_driver on pinned host buffers at 2^21 systems runs the full
    32-chunk H2D / kernel / D2H pipeline (strided column chunks); states and
    stats equal the device-pointer entry's bit for bit."""
    import ctypes
    import torch
    L = B.lib()
    num = 1 << 21
    prob = A.make_problem(A.PLEIADES)
    y0 = perturb(PLEIADES_IC, 0.01, 5, num)
    tol = A.default_tol()
    yh = torch.from_numpy(y0.copy()).pin_memory()
    sth = torch.zeros(num * 8, dtype=torch.int64).pin_memory()
    B.api.check(L.bode_int_driver(ctypes.byref(prob), A.SOLVER_RKCK, A.ARITH_FAST, 0.3, 0.4, num,
                                  None, ctypes.cast(yh.data_ptr(), ctypes.POINTER(ctypes.c_double)),
                                  ctypes.byref(tol), ctypes.c_void_p(sth.data_ptr()), 1))
    yd = torch.from_numpy(y0.copy()).cuda()
    std = torch.zeros(num * 8, dtype=torch.int64, device="cuda")
    B.int_driver_device(B.OdeProblem(prob.kind, prob.dim, prob.param_dim), "rkck", "fast", 0.3,
                        0.4, num, 0, yd.data_ptr(), tol, std.data_ptr(), False,
                        torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert np.array_equal(yh.numpy().view(np.uint64), yd.cpu().numpy().view(np.uint64))
    assert np.array_equal(sth.numpy(), std.cpu().numpy())
