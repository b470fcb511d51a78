#!/usr/bin/env python3
"""Throughput of heatEquation(n) at dimensions without an exact-size kernel
(padded lane groups for n <= 512, one system per block beyond), next to the reference CPU path (oracle/_ref, all host threads) on
the same systems, and the forced block kernel at n = 64 next to the 8-lane
kernel.

    python tests/experiments/wide_bench.py

One window [0, 0.01] of RKC EXACT from the perturbed initial condition
(problems.cpp:124-132, 0.01, seed 42); device time by CUDA events around
bode_int_driver_device on HBM-resident state, after one warm-up window.
Prints one JSON object per case."""
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [REPO, os.path.join(REPO, "tests")]

import torch  # noqa: E402

import paper_1611_02274_b200 as B  # noqa: E402
from paper_1611_02274_b200 import _abi as A  # noqa: E402
from golden_cases import heat_ic, perturb  # noqa: E402
from oracle_lib import RefLib, ref_available  # noqa: E402

T1 = 0.01


def gpu_time(n, num, force_wide=False):
    L = B.lib()
    y0 = perturb(heat_ic(n), 0.01, 42, num)
    yd = torch.from_numpy(y0).cuda()
    st = torch.zeros(num * 8, dtype=torch.int64, device="cuda")
    prob = B.OdeProblem(A.HEAT, n, 0)
    tol = A.default_tol()
    s = torch.cuda.Stream()
    L.bode_set_wide(1 if force_wide else 0)
    try:
        with torch.cuda.stream(s):
            B.int_driver_device(prob, "rkc", "exact", 0.0, T1, num, 0, yd.data_ptr(), tol,
                                st.data_ptr(), 0, s.cuda_stream)  # warm-up
            yd.copy_(torch.from_numpy(y0))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            B.int_driver_device(prob, "rkc", "exact", 0.0, T1, num, 0, yd.data_ptr(), tol,
                                st.data_ptr(), 0, s.cuda_stream)
            e1.record(s)
        torch.cuda.synchronize()
    finally:
        L.bode_set_wide(0)
    stats = st.cpu().numpy().view(A.STATS_DTYPE)
    return e0.elapsed_time(e1) / 1e3, yd.cpu().numpy(), stats, y0


def main():
    out = []
    ref = RefLib() if ref_available() else None
    for n, num in ((100, 1 << 16), (300, 1 << 15), (1000, 1 << 13), (2000, 1 << 12), (10000, 1 << 9)):
        secs, y, st, y0 = gpu_time(n, num)
        row = {"n": n, "systems": num, "window": T1, "gpu_s": secs,
               "gpu_system_windows_per_s": num / secs,
               "stages_per_system": float(st["stages_total"].mean()),
               "kernel": ("padded lane groups" if n <= 1024 else
                          "one system per block, shared memory" if 8 * n * 8 <= 200 * 1024 else
                          "one system per block, global scratch")}
        if ref is not None:
            k = min(num, {100: 8192, 300: 4096, 1000: 2048, 2000: 512}.get(n, 64))
            t = time.perf_counter()
            rc, yo, so, _ = ref.outer_loop(A.make_problem(A.HEAT, n), A.SOLVER_RKC, 0.0, T1, T1,
                                           np.ascontiguousarray(y0.reshape(n, num)[:, :k]).reshape(-1))
            cpu = time.perf_counter() - t
            row.update({"cpu_sample_systems": k, "cpu_threads": os.cpu_count(),
                        "cpu_system_windows_per_s": k / cpu,
                        "bitwise_on_sample": bool(np.array_equal(
                            y.reshape(n, num)[:, :k].view(np.uint64),
                            yo.reshape(n, k).view(np.uint64)))})
        out.append(row)
        print(json.dumps(row), flush=True)
    lane_s, yl, _, _ = gpu_time(64, 1 << 16)
    wide_s, yw, _, _ = gpu_time(64, 1 << 16, force_wide=True)
    print(json.dumps({"n": 64, "systems": 1 << 16, "lane_kernel_s": lane_s, "block_kernel_s": wide_s,
                      "block_over_lane_time": wide_s / lane_s,
                      "bitwise_equal": bool(np.array_equal(yl.view(np.uint64),
                                                           yw.view(np.uint64)))}), flush=True)


if __name__ == "__main__":
    main()
