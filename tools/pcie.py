#!/usr/bin/env python3
"""Pinned host <-> device copy bandwidth on this box (the e2e bound).

    python tools/pcie.py [--mb 940]

Times (CUDA events) H2D alone, D2H alone and both directions concurrently on
two streams, for the bench workload's per-window sizes (y: num*28*8 bytes in,
y + stats: num*(28*8+64) bytes out)."""
import argparse
import json

import torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--num", type=int, default=1 << 22)
    ap.add_argument("--stats-sweep", action="store_true")
    args = ap.parse_args()
    nin, nout = args.num * 28 * 8, args.num * (28 * 8 + 64)
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from bench import gpu_local_memory
    res = {}
    if args.stats_sweep:  # marginal cost of the per-system stats bytes on the D2H side
        with gpu_local_memory(torch, 0):
            hi = torch.zeros(nin, dtype=torch.uint8).pin_memory()
            for sb in (0, 40, 64):
                no = args.num * (28 * 8 + sb)
                ho = torch.zeros(no, dtype=torch.uint8).pin_memory()
                res[f"stats_{sb}B"] = measure(torch, hi, ho, nin, no)
                del ho
        print(json.dumps(res))
        return
    for placement in ("default", "gpu_local"):
        if placement == "gpu_local":
            with gpu_local_memory(torch, 0) as g:
                hi = torch.zeros(nin, dtype=torch.uint8).pin_memory()
                ho = torch.zeros(nout, dtype=torch.uint8).pin_memory()
                res["gpu_local_cpus"] = len(g.cpus or [])
        else:
            hi = torch.zeros(nin, dtype=torch.uint8).pin_memory()
            ho = torch.zeros(nout, dtype=torch.uint8).pin_memory()
        res[placement] = measure(torch, hi, ho, nin, nout)
    print(json.dumps(res))


def measure(torch, hi, ho, nin, nout):
    di = torch.empty(nin, dtype=torch.uint8, device="cuda")
    do = torch.empty(nout, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn, reps=5):
        best = 1e30
        for _ in range(reps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            torch.cuda.synchronize()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return best

    def h2d():
        with torch.cuda.stream(s1):
            di.copy_(hi, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            ho.copy_(do, non_blocking=True)

    def both():
        h2d()
        d2h()

    t_in, t_out, t_both = timed(h2d), timed(d2h), timed(both)
    return {"h2d_bytes": nin, "d2h_bytes": nout, "h2d_ms": t_in, "d2h_ms": t_out,
            "both_ms": t_both, "h2d_GBps": nin / t_in / 1e6, "d2h_GBps": nout / t_out / 1e6,
            "duplex_GBps": (nin + nout) / t_both / 1e6}


if __name__ == "__main__":
    main()
