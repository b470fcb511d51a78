"""The host-pointer pipeline's 40-byte stats transfer (csrc/host.cu,
CompactStats in dispatch.h): with pinned host arrays bode_int_driver moves the
per-system stats over PCIe as 32-bit counts plus the two step sizes and
expands them on the host in place; the result must be every field of the
64-byte bode_stats_t (ode_problem.hpp:57-81 plus stages_total), bitwise what
the full-record path (pageable host arrays) returns. Counts above 2^32 - 1
fall back to fetching the whole record; BODE_COMPACT_STATS_LIMIT lowers that
bound so the fallback runs here.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1611_02274_b200 as B
from paper_1611_02274_b200 import _abi as A
from golden_cases import PLEIADES_IC, heat_ic, perturb

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ALL = ("steps_accepted", "steps_rejected", "rhs_evals", "spec_rad_evals", "stages_total",
       "h_min_seen", "h_max_seen", "underflow", "budget_exhausted")


def run(case, num, pinned, budget=0):
    import torch
    if case == "pleiades":
        prob, y0, solver, t1 = A.make_problem(A.PLEIADES), perturb(PLEIADES_IC, 0.1, 5, num), 0, 0.6
    else:
        prob, y0, solver, t1 = A.make_problem(A.HEAT, 64), perturb(heat_ic(64), 0.01, 5, num), 1, 0.1
    y = torch.from_numpy(y0.copy())
    st = torch.zeros(num * 8, dtype=torch.int64)
    if pinned:
        y, st = y.pin_memory(), st.pin_memory()
    L = B.lib()
    assert L.bode_set_attempt_budget(budget) == 0
    try:
        B.api.check(L.bode_int_driver(prob, solver, A.ARITH_EXACT, 0.0, t1, num, None,
                                      A.dptr(y.numpy()), A.default_tol(),
                                      st.numpy().ctypes.data_as(A.ctypes.c_void_p), 1))
    finally:
        L.bode_set_attempt_budget(0)
    return y.numpy().copy(), st.numpy().view(A.STATS_DTYPE).copy()


@pytest.mark.parametrize("case,budget", [("pleiades", 0), ("heat64", 0), ("pleiades", 30)])
def test_compact_stats_equal_full_records(gpu, case, budget):
    num = 300_001  # 4 pipeline chunks, a ragged last one
    L = B.lib()
    n0 = L.bode_launch_count()
    yp, sp = run(case, num, True, budget)
    n1 = L.bode_launch_count()
    yf, sf = run(case, num, False, budget)
    n2 = L.bode_launch_count()
    # pinned: 4 chunk kernels + 4 stats packs; pageable: one launch, 64-byte records
    assert n1 - n0 == 8 and n2 - n1 == 1, (n1 - n0, n2 - n1)
    assert np.array_equal(yp.view(np.uint64), yf.view(np.uint64))
    for k in ALL:
        assert np.array_equal(np.ascontiguousarray(sp[k]).view(np.uint8),
                              np.ascontiguousarray(sf[k]).view(np.uint8)), k
    if budget:
        assert sp["budget_exhausted"].any()


def test_compact_stats_saturated_records_fetched_whole(gpu):
    """With the saturation bound lowered to 20, most records take the
    whole-record fallback; the stats still equal the full path's bitwise."""
    script = (
        "import sys, numpy as np; sys.path[:0] = [%r, %r];"
        "from test_gpu_compact_stats import run;"
        "y, s = run('pleiades', 140_000, True); np.save(sys.argv[1], s.view(np.uint8));"
        "np.save(sys.argv[2], y)" % (REPO, os.path.join(REPO, "tests")))
    out_s = os.path.join(os.environ.get("TMPDIR", "/tmp"), "compact_sat_stats.npy")
    out_y = os.path.join(os.environ.get("TMPDIR", "/tmp"), "compact_sat_y.npy")
    env = dict(os.environ, BODE_COMPACT_STATS_LIMIT="20")
    r = subprocess.run([sys.executable, "-c", script, out_s, out_y], env=env, capture_output=True,
                       text=True, timeout=600, cwd=REPO)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    sp = np.load(out_s).view(A.STATS_DTYPE)
    yp = np.load(out_y)
    yf, sf = run("pleiades", 140_000, False)
    att = sf["steps_accepted"] + sf["steps_rejected"]
    assert (sf["rhs_evals"] > 20).mean() > 0.9  # the fallback path really ran
    assert np.array_equal(yp.view(np.uint64), yf.view(np.uint64))
    for k in ALL:
        assert np.array_equal(np.ascontiguousarray(sp[k]).view(np.uint8),
                              np.ascontiguousarray(sf[k]).view(np.uint8)), k
    assert att.min() >= 1
