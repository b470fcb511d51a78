#!/usr/bin/env python3
"""Where the time of bode_outer_loop goes (host buffers, 2^22 Pleiades, FAST):
whole 10-window call, 1-window call, and the per-window device-resident path."""
import ctypes
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))


def main():
    import torch
    import paper_1611_02274_b200 as P
    from paper_1611_02274_b200 import _abi as A
    from golden_cases import PLEIADES_IC, perturb
    L = P.lib()
    num = 1 << 22
    y0 = perturb(PLEIADES_IC, 0.01, 42, num)
    yh = torch.from_numpy(y0.copy()).pin_memory()
    sth = torch.zeros(num * 8, dtype=torch.int64).pin_memory()
    yp = ctypes.cast(yh.data_ptr(), ctypes.POINTER(ctypes.c_double))
    prob, tol = A.make_problem(A.PLEIADES), A.default_tol()
    out = {}

    def ol(t1, thr):
        L.bode_set_repack_threshold(thr)
        yh.copy_(torch.from_numpy(y0))
        n = ctypes.c_int32(0)
        t = time.perf_counter()
        P.api.check(L.bode_outer_loop(ctypes.byref(prob), 0, 1, 0.0, t1, 0.1, num, None, yp,
                                      ctypes.byref(tol), ctypes.c_void_p(sth.data_ptr()), 1,
                                      P.api.SINK(), None, ctypes.byref(n)))
        return (time.perf_counter() - t) * 1e3

    ol(0.2, 0.7)
    thrs = [float(x) for x in os.environ.get("PROBE_THRESHOLDS", "0.7 0.0").split()]
    for rep in range(int(os.environ.get("PROBE_REPS", "1"))):
        for thr in thrs:
            out.setdefault(f"outer10_thr{thr}_ms", []).append(ol(1.0, thr))
            if rep == 0:
                out[f"outer1_thr{thr}_ms"] = ol(0.1, thr)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
