#!/usr/bin/env python3
"""Benchmark: ODE system-windows integrated per second on B200 (FP64).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl bode|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU)

Workload (BASELINE.json configs[1]): RKCK on the Pleiades problem (N = 28),
2^22 systems per GPU with the reference's perturbed initial conditions
(perturbInitialConditions(pleiades_ic, 0.01, seed 42), problems.cpp:171-191).
A "step" is one outer window of 0.1 time units over all systems (a restart,
batch_driver.hpp:36-39); K = 10 steps is the paper's [0, 1] protocol
(PAPER.md:652). value = systems x windows / device time (max over ranks),
inputs resident in HBM; e2e = the same metric through the host-pointer C ABI
(bode_int_driver) with pinned host buffers, H2D + D2H inside every step.
The y array (940 MB) exceeds L2 (126 MB), so no L2 flush is needed.

Multi-GPU: systems are independent, so each rank integrates its own 2^22
systems with no collective on the data path (weak scaling); torch.distributed
only provides the barrier and the max-over-ranks of the device time.

Roofline: the path is FP64-compute bound (AI ~74 flop/B for RKCK-Pleiades);
achieved = algorithmic flops (SURVEY.md 8d formulas on the per-system
counters the kernel emits) / kernel time; peak = this device's DFMA
throughput measured in the same run (MEASURED_PEAKS.json has no FP64 entry).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))

METRIC = "ODE systems integrated/sec (RKCK, RKC) at 1/2/4/8 B200 vs CPU ref, %FP64 roof"
UNIT = "system-windows/s"
F_RHS = {"pleiades": 420, "heat": None, "expdecay": 1, "harmonic": 0}


def algorithmic_flops(problem: str, solver: str, dim: int, stats: np.ndarray, windows: int) -> float:
    """RKCK F = rhs*F_rhs + (acc+rej)*58*N;
    RKC F = rhs*F_rhs + N*(10*S + 6*I + 7*C + 8) per window, I = rhs - 2 - S."""
    if problem == "heat":
        f_rhs = 4 * dim - 2
    elif problem == "brusselator":  # 17 per grid point + 5 per call (csrc/problems_ext.cu)
        f_rhs = 17 * (dim // 2) + 5
    else:
        f_rhs = F_RHS[problem]
    rhs = float(stats["rhs_evals"].sum())
    if solver == "rkck":
        att = float(stats["steps_accepted"].sum() + stats["steps_rejected"].sum())
        return rhs * f_rhs + att * 58 * dim
    S = float(stats["stages_total"].sum())
    C = float(stats["spec_rad_evals"].sum())
    n_sys = stats.size
    I = rhs - 2.0 * windows * n_sys - S
    return rhs * f_rhs + dim * (10 * S + 6 * I + 7 * C + 8.0 * windows * n_sys)


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_reference_rate(problem, solver, base, mag, seed, num, windows, g=None, threads=None):
    """The reference CPU path (oracle/_ref = unmodified reference sources;
    fallback: the oracle restatement) on all host threads (or `threads`)."""
    from golden_cases import perturb
    from oracle_lib import Oracle, RefLib, ref_available
    from paper_1611_02274_b200 import _abi as A
    prob = A.make_problem(problem, base.size)
    solv = A.SOLVER_NAMES[solver]
    y0 = perturb(base, mag, seed, num)
    cores = threads or os.cpu_count()
    if ref_available():
        lib, kind = RefLib(), "reference"
        run = lambda y, t0, t1: lib.lib.ref_integrate_batch(
            ctypes.byref(prob), solv, t0, t1, num, A.dptr(y), A.dptr(g),
            ctypes.byref(A.default_tol()), None, cores)
    else:
        lib, kind = Oracle(), "port"
        run = lambda y, t0, t1: lib.lib.orc_integrate_batch(
            ctypes.byref(prob), solv, t0, t1, num, A.dptr(y), A.dptr(g),
            ctypes.byref(A.default_tol()), None, cores)
    y = y0.copy()
    run(y, 0.0, 0.1)  # warm-up window
    # the GPU arm's schedule: windows (k mod 10) of [0, 1], restarting from y0
    t = time.perf_counter()
    for k in range(windows):
        if k % 10 == 0:
            y = y0.copy()
        t0 = 0.0 + (k % 10) * 0.1
        rc = run(y, t0, 0.0 + (k % 10 + 1) * 0.1)
        assert rc == 0
    dt = time.perf_counter() - t
    return num * windows / dt, cores, kind, dt


def run_reference_arm(args):
    from golden_cases import PLEIADES_IC
    rate, cores, kind, dt = cpu_reference_rate("pleiades", "rkck", PLEIADES_IC, 0.01, 42,
                                               args.cpu_sample, args.steps)
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "RKCK Pleiades, perturb 0.01 seed 42, eps 1e-10, windows "
                               "(k mod 10) of [0, 1] as in the GPU arm",
                   "systems_sampled": args.cpu_sample, "window": 0.1},
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": f"{args.cpu_sample} systems x {args.steps} windows "
                                   f"(+1 warm-up window)"},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def measured_traffic(capture: str, num: int):
    """DRAM bytes per launch for `num` systems, from the newest committed ncu
    capture summary (profiles/*_ncu.json: dram read+write per system-window),
    plus that capture's FP64 pipe use, warp execution efficiency and DRAM GB/s."""
    import glob
    for path in sorted(glob.glob(os.path.join(REPO, "profiles", "*_ncu.json")), reverse=True):
        d = json.load(open(path)).get(capture)
        if d and d.get("dram_bytes_per_system"):
            tpi = d.get("thread_inst_per_inst")
            ncu = {"source": os.path.basename(path), "systems": d.get("systems"),
                   "fp64_pipe_pct": d.get("fp64_pipe_pct"),
                   "warp_execution_efficiency": tpi / 32.0 if tpi else None,
                   "dram_GBps": ((d["dram_read_bytes"] + d["dram_write_bytes"]) / d["duration_ns"]
                                 if d.get("duration_ns") else None),
                   "hbm_peak_GBps": 6534.8}
            return d["dram_bytes_per_system"] * num, os.path.basename(path), ncu
    return None, None, None


class gpu_local_memory:
    """Context: run on the CPUs of the GPU's own NUMA node while host buffers
    are allocated and first touched, so pinned pages land next to the GPU's
    PCIe root (a remote node costs ~30% of H2D/D2H bandwidth on these boxes).
    The previous affinity is restored on exit, so the CPU baseline still gets
    every host thread."""

    def __init__(self, torch, device):
        self.cpus = None
        try:
            p = torch.cuda.get_device_properties(device)
            bus = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            with open(f"/sys/bus/pci/devices/{bus}/local_cpulist") as f:
                self.cpus = _parse_cpulist(f.read())
        except (OSError, AttributeError, ValueError):
            self.cpus = None

    def __enter__(self):
        self.saved = os.sched_getaffinity(0)
        if self.cpus:
            try:
                os.sched_setaffinity(0, self.cpus & self.saved or self.saved)
            except OSError:
                pass
        return self

    def __exit__(self, *exc):
        os.sched_setaffinity(0, self.saved)


def _parse_cpulist(text):
    cpus = set()
    for part in text.strip().split(","):
        if "-" in part:
            a, b = part.split("-")
            cpus.update(range(int(a), int(b) + 1))
        elif part:
            cpus.add(int(part))
    return cpus


def measure_device(P, A, torch, problem, solver, arith, dim, y0, g0, steps, warmup, stream,
                   repack=False, presort_row=None):
    """K windows on HBM-resident state; per-launch CUDA events on `stream`.
    repack: after the first timed window, re-pack the batch by the cost each
    system showed (bode_repack_by_cost), and restore the caller's order after
    the last (bode_unpack); both inside the timed region. presort_row: sort by
    |g[presort_row]| before the first window instead (bode_repack_by_param)."""
    reorder = repack or presort_row is not None
    num = y0.size // dim
    yd = torch.from_numpy(y0).to("cuda")
    gd = torch.from_numpy(g0).to("cuda") if g0 is not None else None
    st = torch.zeros(num * 8, dtype=torch.int64, device="cuda")
    tol = A.default_tol()
    prob = P.OdeProblem(A.PROBLEM_NAMES[problem], dim, 0 if g0 is None else g0.size // num)
    gp = gd.data_ptr() if gd is not None else 0

    def window(k, merge):
        t0 = 0.0 + (k % 10) * 0.1
        P.int_driver_device(prob, solver, arith, t0, 0.0 + (k % 10 + 1) * 0.1, num, gp,
                            yd.data_ptr(), tol, st.data_ptr(), merge, stream.cuda_stream)

    L = P.lib()
    order = torch.empty(num, dtype=torch.int64, device="cuda") if reorder else None
    cprob = A.Problem(kind=prob.kind, dim=prob.dim, param_dim=prob.param_dim, reserved=0)
    with torch.cuda.stream(stream):
        for k in range(warmup):
            window(k, False)
            if reorder:  # warm the sort/gather kernels and the scratch allocation
                P.api.check(L.bode_order_init(ctypes.c_void_p(order.data_ptr()), num,
                                              ctypes.c_void_p(stream.cuda_stream)))
                for fn in (L.bode_repack_by_cost, L.bode_unpack):
                    P.api.check(fn(ctypes.byref(cprob), num, ctypes.c_void_p(yd.data_ptr()),
                                   ctypes.c_void_p(gp), ctypes.c_void_p(st.data_ptr()),
                                   ctypes.c_void_p(order.data_ptr()),
                                   ctypes.c_void_p(stream.cuda_stream)))
        yd.copy_(torch.from_numpy(y0))
        if gd is not None:
            gd.copy_(torch.from_numpy(g0))
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        n0 = P.lib().bode_launch_count()
        ev[0].record(stream)
        if reorder:
            P.api.check(L.bode_order_init(ctypes.c_void_p(order.data_ptr()), num,
                                          ctypes.c_void_p(stream.cuda_stream)))
        if presort_row is not None:
            P.api.check(L.bode_repack_by_param(
                ctypes.byref(cprob), num, ctypes.c_void_p(yd.data_ptr()), ctypes.c_void_p(gp),
                ctypes.c_void_p(st.data_ptr()), ctypes.c_void_p(order.data_ptr()), presort_row,
                ctypes.c_void_p(stream.cuda_stream)))
        for k in range(steps):
            window(k, k > 0)
            if repack and k == 0 and steps > 1:
                P.api.check(L.bode_repack_by_cost(
                    ctypes.byref(cprob), num, ctypes.c_void_p(yd.data_ptr()),
                    ctypes.c_void_p(gp), ctypes.c_void_p(st.data_ptr()),
                    ctypes.c_void_p(order.data_ptr()), ctypes.c_void_p(stream.cuda_stream)))
            if reorder and k == steps - 1:
                P.api.check(L.bode_unpack(
                    ctypes.byref(cprob), num, ctypes.c_void_p(yd.data_ptr()),
                    ctypes.c_void_p(gp), ctypes.c_void_p(st.data_ptr()),
                    ctypes.c_void_p(order.data_ptr()), ctypes.c_void_p(stream.cuda_stream)))
            ev[k + 1].record(stream)
        torch.cuda.synchronize()
    launches = P.lib().bode_launch_count() - n0
    per = [ev[k].elapsed_time(ev[k + 1]) for k in range(steps)]
    stats = st.cpu().numpy().view(A.STATS_DTYPE).copy()
    return sum(per) / 1e3, per, stats, launches, yd


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="bode", choices=["bode", "reference"])
    # (not --num: torchrun's own parser would take it for --numa-binding)
    ap.add_argument("--systems", dest="num", type=int, default=1 << 22, help="systems per GPU")
    ap.add_argument("--arith", default="fast", choices=["fast", "exact"])
    ap.add_argument("--rkc-systems", dest="rkc_num", type=int, default=1 << 22)
    ap.add_argument("--persistent", action="store_true",
                    help="persistent kernels with dynamic refill (default: static)")
    ap.add_argument("--no-secondary", dest="secondary", action="store_false",
                    help="skip the EXACT / RKC measurements")
    ap.add_argument("--cpu-sample", type=int, default=1 << 15)
    ap.add_argument("--block", type=int, default=0,
                    help="threads per block override (0: each kernel's default)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank == 0:
            run_reference_arm(args)
        return

    import torch
    import paper_1611_02274_b200 as P
    from paper_1611_02274_b200 import _abi as A
    from golden_cases import PLEIADES_IC, brusselator_ic, brusselator_params, heat_ic, perturb
    from paper_1611_02274_b200.api import stiffness_params

    # BODE_BENCH_SHARE_GPU=1 (functional test of the multi-rank path on one
    # GPU): ranks share cuda:0 and the barrier/max-over-ranks run on gloo
    share = os.environ.get("BODE_BENCH_SHARE_GPU") == "1"
    local = local % torch.cuda.device_count() if share else local
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    red_dev = "cpu" if share else "cuda"
    L = P.lib()
    L.bode_set_persistent(1 if args.persistent else 0)
    P.api.check(L.bode_set_block_size(args.block))
    stream = torch.cuda.Stream()

    peak = ctypes.c_double()
    psec = ctypes.c_double()
    P.api.check(L.bode_selftest_fp64_peak(ctypes.byref(peak), ctypes.byref(psec)))

    # ---- headline: RKCK Pleiades, per-rank shard of args.num systems ----
    num = args.num
    y0 = perturb(PLEIADES_IC, 0.01, 42 + rank, num)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        secs, per, stats, launches, _ = measure_device(P, A, torch, "pleiades", "rkck",
                                                       args.arith, 28, y0, None, args.steps,
                                                       args.warmup, stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
        tt = torch.tensor([secs], device=red_dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        secs = float(tt.item())
    value = world * num * args.steps / secs
    flops = algorithmic_flops("pleiades", "rkck", 28, stats, args.steps)
    achieved = flops / sum(p / 1e3 for p in per)

    # ---- e2e through the host-pointer C ABI (pinned buffers, H2D+D2H every window) ----
    e2e = None
    if not args.no_e2e:
        with gpu_local_memory(torch, local):
            yh = torch.from_numpy(y0.copy()).pin_memory()
            sth = torch.zeros(num * 8, dtype=torch.int64).pin_memory()
        yp = ctypes.cast(yh.data_ptr(), ctypes.POINTER(ctypes.c_double))
        prob = A.make_problem(A.PLEIADES)
        tol = A.default_tol()
        ar = A.ARITH_NAMES[args.arith]
        P.api.check(L.bode_int_driver(ctypes.byref(prob), 0, ar, 0.0, 0.1, num, None, yp,
                                      ctypes.byref(tol), ctypes.c_void_p(sth.data_ptr()), 1))
        yh.copy_(torch.from_numpy(y0))
        if dist:
            dist.barrier()
        t = time.perf_counter()
        for k in range(args.steps):
            P.api.check(L.bode_int_driver(ctypes.byref(prob), 0, ar, 0.0 + (k % 10) * 0.1,
                                          0.0 + (k % 10 + 1) * 0.1, num, None, yp,
                                          ctypes.byref(tol), ctypes.c_void_p(sth.data_ptr()), 1))
        e2e_s = time.perf_counter() - t
        if dist:
            tt = torch.tensor([e2e_s], device=red_dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_s = float(tt.item())
        e2e = {"value": world * num * args.steps / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": num * 28 * 8, "d2h_bytes_per_step": num * (28 * 8 + 64),
               "ms_per_step": e2e_s / args.steps * 1e3, "pinned_host": True}
        # the paper's intDriver(t, tEnd, numODE, gGlobal, yGlobal) exactly: y in and
        # out, no per-system stats requested (stats = NULL), same windows
        yh.copy_(torch.from_numpy(y0))
        if dist:
            dist.barrier()
        t = time.perf_counter()
        for k in range(args.steps):
            P.api.check(L.bode_int_driver(ctypes.byref(prob), 0, ar, 0.0 + (k % 10) * 0.1,
                                          0.0 + (k % 10 + 1) * 0.1, num, None, yp,
                                          ctypes.byref(tol), None, 1))
        pp_s = time.perf_counter() - t
        if dist:
            tt = torch.tensor([pp_s], device=red_dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            pp_s = float(tt.item())
        e2e["paper_protocol_no_stats"] = {
            "value": world * num * args.steps / pp_s, "unit": UNIT,
            "h2d_bytes_per_step": num * 28 * 8, "d2h_bytes_per_step": num * 28 * 8,
            "ms_per_step": pp_s / args.steps * 1e3}
        # the same 10-window protocol through bode_outer_loop (batchode::outerLoop's
        # drop-in): host buffers in and out, the state resident in HBM between
        # windows, so one H2D and one D2H per call instead of per window
        steps_out = ctypes.c_int32(0)
        P.api.check(L.bode_outer_loop(ctypes.byref(prob), 0, ar, 0.0, 0.2, 0.1, num, None, yp,
                                      ctypes.byref(tol), ctypes.c_void_p(sth.data_ptr()), 1,
                                      P.api.SINK(), None, ctypes.byref(steps_out)))  # warm-up
        yh.copy_(torch.from_numpy(y0))
        if dist:
            dist.barrier()
        t = time.perf_counter()
        P.api.check(L.bode_outer_loop(ctypes.byref(prob), 0, ar, 0.0, 1.0, 0.1, num, None, yp,
                                      ctypes.byref(tol), ctypes.c_void_p(sth.data_ptr()), 1,
                                      P.api.SINK(), None, ctypes.byref(steps_out)))
        ol_s = time.perf_counter() - t
        if dist:
            tt = torch.tensor([ol_s], device=red_dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ol_s = float(tt.item())
        e2e["outer_loop"] = {"value": world * num * steps_out.value / ol_s, "unit": UNIT,
                             "windows": steps_out.value, "ms_total": ol_s * 1e3,
                             "h2d_bytes_per_call": num * 28 * 8,
                             "d2h_bytes_per_call": num * (28 * 8 + 64)}

    def secondary(problem, solver, arith, dim, y0s, g0s, label, steps, repack=False,
                  presort_row=None):
        sec, perw, sts, _, _ = measure_device(P, A, torch, problem, solver, arith, dim, y0s, g0s,
                                               steps, 1, stream, repack=repack,
                                               presort_row=presort_row)
        f = algorithmic_flops(problem, solver, dim, sts, steps)
        n = y0s.size // dim
        return {"workload": label, "value": world * n * steps / secs_max(sec),
                "unit": UNIT, "ms_per_step": sec / steps * 1e3,
                "achieved_tflops": f / sec / 1e12, "frac_of_fp64_peak": f / sec / peak.value,
                "flop_per_system_window": f / (n * steps),
                "kernel_ms_per_window": [round(x, 4) for x in perw]}

    def secs_max(sec):
        if not dist:
            return sec
        tt = torch.tensor([sec], device=red_dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    extra = {}
    if args.secondary:
        extra["rkck_exact"] = secondary(
            "pleiades", "rkck", "exact", 28, y0, None,
            f"RKCK Pleiades, {num} systems, EXACT policy (bitwise reference arithmetic)",
            args.steps)
        if args.rkc_num > 0:
            yh0 = perturb(heat_ic(64), 0.01, 42 + rank, args.rkc_num)
            extra["rkc_heat64"] = secondary(
                "heat", "rkc", "exact", 64, yh0, None,
                f"RKC heat n=64 (config 3), {args.rkc_num} systems, EXACT", min(args.steps, 10))
            ye0 = perturb(np.array([1.0]), 0.01, 42 + rank, args.rkc_num)
            g0 = stiffness_params(args.rkc_num)
            extra["rkc_stiff_expdecay"] = secondary(
                "expdecay", "rkc", "exact", 1, ye0, g0,
                f"RKC expDecay, g0 log-uniform in [1,1e4] (config 4), {args.rkc_num} systems, EXACT",
                min(args.steps, 10))
            # the same natural-order batch, re-packed by its window-1 cost
            # (bode_repack_by_cost) and restored at the end, inside the timing
            extra["rkc_stiff_expdecay_repacked"] = secondary(
                "expdecay", "rkc", "exact", 1, ye0, g0,
                f"RKC expDecay, config 4 batch (natural order) re-packed by cost after window "
                f"1, {args.rkc_num} systems, EXACT", min(args.steps, 10), repack=True)
            # the same natural-order batch sorted by |g0| (its spectral radius, the
            # reference's specRadHint) before window 1 (bode_repack_by_param) and
            # restored at the end, inside the timing
            extra["rkc_stiff_expdecay_presorted"] = secondary(
                "expdecay", "rkc", "exact", 1, ye0, g0,
                f"RKC expDecay, config 4 batch (natural order) sorted by |g0| before window 1, "
                f"{args.rkc_num} systems, EXACT", min(args.steps, 10), presort_row=0)
            # the same batch with the systems sorted by stiffness (SURVEY 8d config 4:
            # shuffled and sorted): warps then hold similar stage counts
            order = np.argsort(g0, kind="stable")
            extra["rkc_stiff_expdecay_sorted"] = secondary(
                "expdecay", "rkc", "exact", 1, ye0[order], g0[order],
                f"RKC expDecay, config 4 batch sorted by g0, {args.rkc_num} systems, EXACT",
                min(args.steps, 10))
            yb0 = perturb(brusselator_ic(32), 0.01, 7 + rank, args.rkc_num)
            gb0 = brusselator_params(args.rkc_num, 0.02, 0.5)
            gbn = brusselator_params(args.rkc_num, 0.002, 0.02)
            extra["rkck_brusselator_fast"] = secondary(
                "brusselator", "rkck", "fast", 64, yb0, gbn,
                f"RKCK FAST Brusselator n=32 (registered problem, generic RKCK kernel), alpha "
                f"log-spaced in [0.002, 0.02], {args.rkc_num} systems", min(args.steps, 10))
            extra["rkc_brusselator"] = secondary(
                "brusselator", "rkc", "exact", 64, yb0, gb0,
                f"RKC Brusselator reaction-diffusion n=32 (dim 64, registered problem), alpha "
                f"log-spaced in [0.02, 0.5], {args.rkc_num} systems, EXACT", min(args.steps, 10))

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    traffic, traffic_src, ncu_evidence = measured_traffic(
        "rkck_fast" if args.arith == "fast" else "rkck_exact", num)
    cpu = None
    if not args.no_cpu:
        rate, cores, kind, dt = cpu_reference_rate("pleiades", "rkck", PLEIADES_IC, 0.01, 42,
                                                   args.cpu_sample, 10)
        rate1, _, _, dt1 = cpu_reference_rate("pleiades", "rkck", PLEIADES_IC, 0.01, 42,
                                              max(1024, args.cpu_sample // 16), 10, threads=1)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": kind,
               "sample": f"{args.cpu_sample} Pleiades systems x 10 windows ([0,1]), all host "
                         f"threads, {dt:.2f} s",
               "one_thread": {"value": rate1, "unit": UNIT, "cores": 1,
                              "sample": f"{max(1024, args.cpu_sample // 16)} systems x 10 "
                                        f"windows, {dt1:.2f} s"}}

    clocks = clk.summary()
    # nominal FP64 FMA peak at the SM clock observed during the timed region:
    # 64 DFMA/clk/SM x 2 flop x SMs (37.2 TF at 1965 MHz)
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    nominal = 64 * 2 * sms * (clocks["sm_mhz"] or 1965.0) * 1e6
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"RKCK Pleiades (N=28), {num} systems per GPU, perturb 0.01 "
                               f"seed 42+rank, eps 1e-10, window 0.1 (restart)",
                   "arith": args.arith, "systems_per_gpu": num, "window": 0.1,
                   "scheduling": "persistent refill" if args.persistent else "static",
                   "l2": "state (num*28*8 B) exceeds the 126 MB L2; no flush needed",
                   "parallelism": f"dp{world} (independent shards, no collective)"},
        "roofline": {"bound": "fp64", "achieved": achieved / 1e12, "peak": peak.value / 1e12,
                     "unit": "TFLOP/s", "frac": achieved / peak.value, "traffic": traffic,
                     "traffic_source": traffic_src, "ncu": ncu_evidence,
                     "algorithmic_bytes_per_launch": num * (28 * 8 * 2 + 64),
                     "peak_source": "DFMA microbenchmark on this device in this run "
                                    "(MEASURED_PEAKS.json has no FP64 entry)",
                     "peak_nominal": nominal / 1e12, "frac_of_nominal": achieved / nominal,
                     "flop_per_system_window": flops / (num * args.steps),
                     "kernel_ms_per_launch": sum(per) / len(per)},
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
        "clocks": clocks, **extra,
        "kernel_ms_per_window": [round(x, 4) for x in per],
        "systems_per_s_full_protocol": value / 10.0,
        "work_per_system_window": {
            "attempts": float((stats["steps_accepted"] + stats["steps_rejected"]).sum()) / (num * args.steps),
            "rhs_evals": float(stats["rhs_evals"].sum()) / (num * args.steps)},
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
