#!/usr/bin/env python3
"""Small runs of every main kernel family for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool memcheck python tools/sanitize_probe.py

RKCK Pleiades FAST (one lane, RKN) and EXACT (axis-split lane pair), the
persistent refill kernel, RKC heat n=64 EXACT and FAST (8-lane warp-uniform
groups), RKC expDecay (one lane, stiffness-varied, presort + re-pack), the
RKC coefficient-table kernel, heat at run-time dimensions (padded lane
groups, one system per block in shared or global memory), the step trace and
attempt-budget instances, the fixed-step harnesses, and the outer loop with
the asynchronous sink over two shards on one device. Prints PROBE_OK.
"""
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))

import paper_1611_02274_b200 as B  # noqa: E402
from paper_1611_02274_b200.api import stiffness_params  # noqa: E402
from golden_cases import PLEIADES_IC, heat_ic  # noqa: E402


def main():
    L = B.lib()
    n0 = L.bode_launch_count()
    pl = B.problems.pleiades()
    b = B.problems.perturb_initial_conditions(PLEIADES_IC, 0.1, 3, 1000)
    for arith in ("fast", "exact"):
        B.integrate_batch(pl, b, 0.0, 0.1, solver="rkck", arith=arith)
    L.bode_set_persistent(1)
    B.integrate_batch(pl, b, 0.0, 0.1, solver="rkck", arith="fast")
    L.bode_set_persistent(0)
    heat = B.problems.heat_equation(64)
    hb = B.problems.perturb_initial_conditions(heat_ic(64), 0.01, 3, 300)
    for arith in ("exact", "fast"):
        B.integrate_batch(heat, hb, 0.0, 0.1, solver="rkc", arith=arith)
    ed = B.problems.exp_decay()
    eb = B.problems.perturb_initial_conditions(np.array([1.0]), 0.01, 3, 5000)
    eb.param_dim, eb.params = 1, stiffness_params(5000)
    snaps = []
    B.outer_loop(ed, eb, 0.0, 0.3, 0.1, solver="rkc", gpus=2,
                 sink=lambda t, s: snaps.append(t))
    B.outer_loop(pl, b, 0.0, 0.3, 0.1, solver="rkck", arith="fast", gpus=2,
                 sink=lambda t, s: snaps.append(t))
    # heat with a run-time dimension: padded lane groups (n = 100 in HeatPad<104>
    # (RKC) / <128> (RKCK), n = 300 in <320> / <512> (RKCK: stages in shared
    # memory), n = 1000 in <1024>), one system per block with the vectors in shared
    # memory (n = 1500, and n = 100 forced onto the block kernels) and in the
    # per-block global scratch (n = 4000)
    for n, t1, force in ((100, 1e-3, 0), (300, 1e-4, 0), (1000, 1e-4, 0), (1500, 1e-5, 0),
                         (100, 1e-3, 1), (4000, 1e-5, 0)):
        hw = B.problems.heat_equation(n)
        wb = B.problems.perturb_initial_conditions(heat_ic(n), 0.01, 3, 20)
        L.bode_set_wide(force)
        for solver in ("rkc", "rkck"):
            B.integrate_batch(hw, wb, 0.0, t1, solver=solver, arith="exact")
        B.integrate_batch(hw, wb, 0.0, t1, solver="rkc", arith="fast")
        L.bode_set_wide(0)
    # the step trace (instrumented instances): RKCK EXACT lane pair, RKC heat64 lanes
    B.trace_steps(pl, b.values.reshape(28, -1)[:, 0].copy(), None, 0.0, 0.1, solver="rkck")
    B.trace_steps(heat, hb.values.reshape(64, -1)[:, 0].copy(), None, 0.0, 0.1, solver="rkc")
    L.bode_set_attempt_budget(5)
    B.integrate_batch(pl, b, 0.0, 0.1, solver="rkck", arith="fast")
    B.integrate_batch(heat, hb, 0.0, 0.1, solver="rkc", arith="exact")
    L.bode_set_attempt_budget(0)
    B.integrate_fixed(pl, b, 0.0, 0.1, 10, solver="rkck")
    B.integrate_fixed(heat, hb, 0.0, 0.01, 4, solver="rkc", stages=5)
    assert len(snaps) == 6
    print(f"PROBE_OK launches={L.bode_launch_count() - n0}", flush=True)


if __name__ == "__main__":
    main()
