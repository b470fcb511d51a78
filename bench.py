#!/usr/bin/env python3
"""Benchmark: ODE system-windows integrated per second on B200 (FP64).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl bode|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU)

Workload (BASELINE.json configs[4] = config 5 at N GPUs; its RKCK leg is
configs[1]'s workload at 2^24): RKCK on the Pleiades problem (N = 28),
2^24 systems in total, with the reference's perturbed initial conditions
(perturbInitialConditions(pleiades_ic, 0.01, seed 42), problems.cpp:171-191).
A "step" is one outer window of 0.1 time units over all systems (a restart,
batch_driver.hpp:36-39). Step k integrates window (k mod 10) of the paper's
[0, 1] protocol and every 10th step restarts from y0 -- the
same schedule as the reference arm and the CPU baseline. The restore is a
device copy outside the timed intervals (per-window CUDA events).

value = systems x windows / device time (max over ranks), inputs resident in
HBM; e2e = the same metric through the host-pointer C ABI (bode_int_driver)
with pinned host buffers, H2D + D2H inside every step, and (N > 1) the final
result gather to rank 0 inside the timed region. The y array (3.76 GB)
exceeds L2 (126 MB), so no L2 flush is needed.

Multi-GPU (config 5): the 2^24 systems are split into contiguous shards, one
per rank (strong scaling; batch_driver.cpp:68-73 across GPUs). No collective
runs on the data path; the only exchange is the final gather of the shards to
rank 0 (paper_1611_02274_b200/dist.py, NCCL over NVLink).

Roofline: the path is FP64-compute bound (AI ~74 flop/B for RKCK-Pleiades);
achieved = algorithmic flops (SURVEY.md 8d formulas on the per-system
counters the kernel emits) / kernel time; peak = this device's DFMA
throughput measured in the same run (MEASURED_PEAKS.json has no FP64 entry),
with the nominal 64 DFMA/clk/SM figure beside it.
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
CYCLE = 10  # windows per [0, 1] protocol; the schedule restarts from y0 after each
T_START = time.monotonic()


def window_bounds(k: int):
    """Step k of the bench schedule: window (k mod 10) of [0, 1]."""
    j = k % CYCLE
    return 0.0 + j * 0.1, 0.0 + (j + 1) * 0.1


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


# ------------------------------------------------------------ inputs ----
def gen_states(L, base, mag, seed, first, count):
    """Systems [first, first+count) of perturbInitialConditions(base, mag, seed)
    as a local SoA array (bode_perturb_initial_conditions_range, threaded C)."""
    base = np.ascontiguousarray(base, dtype=np.float64)
    out = np.empty(count * base.size)
    dp = ctypes.POINTER(ctypes.c_double)
    rc = L.bode_perturb_initial_conditions_range(base.ctypes.data_as(dp), base.size, mag, seed,
                                                 first, count, out.ctypes.data_as(dp))
    assert rc == 0, L.bode_last_error()
    return out


def stiffness_range(first, count, seed=9):
    """Config 4's g0_i = 10^(2 + 2*unitSymmetricAt(9, i)) for i in [first, first+count)."""
    k = np.arange(first, first + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (k + np.uint64(1)) * np.uint64(0x9e3779b97f4a7c15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xbf58476d1ce4e5b9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94d049bb133111eb)
        z = z ^ (z >> np.uint64(31))
    u = 2.0 * ((z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53) - 1.0
    return 10.0 ** (2.0 + 2.0 * u)


# ------------------------------------------------------- CPU reference ----
def cpu_reference(problem, solver, base, mag, seed, num, g=None, threads=None, repeats=3):
    """The reference CPU path timed like timedOuterLoop (bench.cpp:196-214):
    batchode::outerLoop over [0, 1] in 10 windows of 0.1 (oracle/_ref = the
    unmodified reference sources; fallback: the oracle restatement), all host
    threads (or `threads`), one warm-up window, best of `repeats`.
    Returns (rate, cores, kind, best_seconds, y_final, stats)."""
    from oracle_lib import Oracle, RefLib, ref_available
    from paper_1611_02274_b200 import _abi as A
    prob = A.make_problem(problem, base.size)
    solv = A.SOLVER_NAMES[solver]
    y0 = gen_states(_lib(), base, mag, seed, 0, num)
    cores = threads or os.cpu_count()
    if ref_available():
        lib, kind = RefLib(), "reference"
        run = lambda y, t0, t1, h: lib.outer_loop(prob, solv, t0, t1, h, y, g, workers=cores)
    else:
        lib, kind = Oracle(), "port"
        run = lambda y, t0, t1, h: lib.outer_loop(prob, solv, t0, t1, h, y, g, threads=cores)
    run(y0, 0.0, 0.1, 0.1)  # warm-up window
    best, out = None, None
    for _ in range(repeats):
        t = time.perf_counter()
        rc, y, st, nwin = run(y0, 0.0, 1.0, 0.1)
        dt = time.perf_counter() - t
        assert rc == 0 and nwin == CYCLE
        if best is None or dt < best:
            best, out = dt, (y, st)
    return num * CYCLE / best, cores, kind, best, out[0], out[1]


_L = None


def _lib():
    global _L
    if _L is None:
        import paper_1611_02274_b200 as P
        _L = P.lib()
    return _L


def run_reference_arm(args):
    """--impl reference: the reference's own CPU path (oracle/_ref) on the host
    cores, on this arm's workload (RKCK Pleiades, perturb 0.01 seed 42) and
    step schedule; each step is one window over a bounded sample of systems."""
    from oracle_lib import Oracle, RefLib, ref_available
    from paper_1611_02274_b200 import _abi as A
    from golden_cases import PLEIADES_IC
    num = args.cpu_sample
    prob = A.make_problem(A.PLEIADES)
    y0 = gen_states(_lib(), PLEIADES_IC, 0.01, 42, 0, num)
    cores = os.cpu_count()
    if ref_available():
        lib, kind = RefLib(), "reference"
        run = lambda y, t0, t1: lib.lib.ref_integrate_batch(
            ctypes.byref(prob), A.SOLVER_RKCK, t0, t1, num, A.dptr(y), None,
            ctypes.byref(A.default_tol()), None, cores)
    else:
        lib, kind = Oracle(), "port"
        run = lambda y, t0, t1: lib.lib.orc_integrate_batch(
            ctypes.byref(prob), A.SOLVER_RKCK, t0, t1, num, A.dptr(y), None,
            ctypes.byref(A.default_tol()), None, cores)
    y = y0.copy()
    for k in range(args.warmup):
        if k % CYCLE == 0:
            y = y0.copy()
        assert run(y, *window_bounds(k)) == 0
    dt = 0.0
    for k in range(args.steps):
        if k % CYCLE == 0:
            y = y0.copy()  # outside the timed interval, as in the GPU arm
        t = time.perf_counter()
        rc = run(y, *window_bounds(k))
        dt += time.perf_counter() - t
        assert rc == 0
    rate = num * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "RKCK Pleiades (N=28), perturb 0.01 seed 42, eps 1e-10; step k "
                               "= window (k mod 10) of [0, 1], restart from y0 every 10 steps "
                               "(the GPU arm's schedule)",
                   "systems_sampled": num, "window": 0.1},
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": f"{num} systems x {args.steps} windows "
                                   f"(+{args.warmup} warm-up windows), integrateBatch per window"},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- device ----
def hbm_peak_gbps():
    """Measured HBM copy bandwidth of this pool (MEASURED_PEAKS.json, driver-written),
    else the profiling recipe's fallback (6.65 TB/s)."""
    try:
        return float(json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6650.0


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
                   "hbm_peak_GBps": hbm_peak_gbps()}
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
                   repack=False, presort_row=None, return_state=False):
    """K windows on HBM-resident state; per-window CUDA events on `stream`.
    Step k integrates window (k mod 10) of [0, 1]; the state restarts from y0
    before every 10th step with a device copy outside the timed intervals.
    repack: after the first timed window, re-pack the batch by the cost each
    system showed (bode_repack_by_cost), and restore the caller's order after
    the last (bode_unpack); both inside the timed region. presort_row: sort by
    |g[presort_row]| before the first window instead (bode_repack_by_param).
    Re-packing moves systems, so it is only used within one [0, 1] cycle."""
    reorder = repack or presort_row is not None
    assert not reorder or steps <= CYCLE
    num = y0.size // dim
    y0d = torch.from_numpy(y0).to("cuda")
    yd = y0d.clone()
    gd = torch.from_numpy(g0).to("cuda") if g0 is not None else None
    st = torch.zeros(num * 8, dtype=torch.int64, device="cuda")
    tol = A.default_tol()
    prob = P.OdeProblem(A.PROBLEM_NAMES[problem], dim, 0 if g0 is None else g0.size // num)
    gp = gd.data_ptr() if gd is not None else 0

    def window(k, merge):
        if k > 0 and k % CYCLE == 0:
            yd.copy_(y0d)
        t0, t1 = window_bounds(k)
        P.int_driver_device(prob, solver, arith, t0, t1, num, gp, yd.data_ptr(), tol,
                            st.data_ptr(), merge, stream.cuda_stream)

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
        yd.copy_(y0d)
        if gd is not None:
            gd.copy_(torch.from_numpy(g0))
        torch.cuda.synchronize()
        ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        n0 = P.lib().bode_launch_count()
        pre = torch.cuda.Event(enable_timing=True)
        pre.record(stream)
        if reorder:
            P.api.check(L.bode_order_init(ctypes.c_void_p(order.data_ptr()), num,
                                          ctypes.c_void_p(stream.cuda_stream)))
        if presort_row is not None:
            P.api.check(L.bode_repack_by_param(
                ctypes.byref(cprob), num, ctypes.c_void_p(yd.data_ptr()), ctypes.c_void_p(gp),
                ctypes.c_void_p(st.data_ptr()), ctypes.c_void_p(order.data_ptr()), presort_row,
                ctypes.c_void_p(stream.cuda_stream)))
        for k in range(steps):
            if k > 0 and k % CYCLE == 0:
                yd.copy_(y0d)  # restart from y0, outside [ev0[k], ev1[k]]
            ev0[k].record(stream)
            t0, t1 = window_bounds(k)
            P.int_driver_device(prob, solver, arith, t0, t1, num, gp, yd.data_ptr(), tol,
                                st.data_ptr(), k > 0, stream.cuda_stream)
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
            ev1[k].record(stream)
        torch.cuda.synchronize()
    launches = P.lib().bode_launch_count() - n0
    per = [ev0[k].elapsed_time(ev1[k]) for k in range(steps)]
    if presort_row is not None and steps:
        per[0] += pre.elapsed_time(ev0[0])  # the presort belongs to the timed region
    stats = st.cpu().numpy().view(A.STATS_DTYPE).copy()
    y_out = yd.cpu().numpy() if return_state else None
    del yd, y0d, gd, st, order
    torch.cuda.empty_cache()
    return sum(per) / 1e3, per, stats, launches, y_out


def sysrel(y, yo, num, dim):
    """Per-system max-norm relative error (acceptance.cpp:142-147)."""
    a, o = y.reshape(dim, num), yo.reshape(dim, num)
    den = np.max(np.abs(o), axis=0)
    return np.max(np.abs(a - o), axis=0) / np.where(den > 0, den, 1.0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="bode", choices=["bode", "reference"])
    # (not --num: torchrun's own parser would take it for --numa-binding)
    ap.add_argument("--systems", dest="num", type=int, default=1 << 24,
                    help="systems in total, split over the ranks (config 5: 2^24)")
    ap.add_argument("--arith", default="fast", choices=["fast", "exact"])
    ap.add_argument("--rkc-systems", dest="rkc_num", type=int, default=1 << 24,
                    help="RKC heat64 systems in total (config 5: 2^24)")
    ap.add_argument("--aux-systems", dest="aux_num", type=int, default=1 << 22,
                    help="systems for the config 2-stress / 4 / Brusselator secondaries")
    ap.add_argument("--persistent", action="store_true",
                    help="persistent kernels with dynamic refill (default: static)")
    ap.add_argument("--no-secondary", dest="secondary", action="store_false",
                    help="skip the EXACT / RKC measurements")
    ap.add_argument("--cpu-sample", type=int, default=1 << 16)
    ap.add_argument("--block", type=int, default=0,
                    help="threads per block override (0: each kernel's default)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--budget-s", type=float, default=1200.0,
                    help="wall-clock budget: secondaries that would start after it are skipped")
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
    from paper_1611_02274_b200 import dist as D
    from golden_cases import PLEIADES_IC, brusselator_ic, brusselator_params, heat_ic

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
    P.api.check(L.bode_use_device(local))  # this rank's GPU for the library's runtime too
    L.bode_set_persistent(1 if args.persistent else 0)
    P.api.check(L.bode_set_block_size(args.block))
    stream = torch.cuda.Stream()

    def secs_max(sec):
        if not dist:
            return sec
        tt = torch.tensor([sec], device=red_dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    def barrier():
        if dist:
            dist.barrier()

    peak = ctypes.c_double()
    psec = ctypes.c_double()
    P.api.check(L.bode_selftest_fp64_peak(ctypes.byref(peak), ctypes.byref(psec)))

    # ---- headline: RKCK Pleiades, this rank's contiguous shard of args.num ----
    total = args.num
    b, e = D.shard_range(total, world, rank)
    num = e - b
    y0 = gen_states(L, PLEIADES_IC, 0.01, 42, b, num)
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        secs, per, stats, launches, _ = measure_device(P, A, torch, "pleiades", "rkck",
                                                       args.arith, 28, y0, None, args.steps,
                                                       args.warmup, stream)
    torch.cuda.synchronize()
    barrier()
    secs = secs_max(secs)
    value = total * args.steps / secs
    flops = algorithmic_flops("pleiades", "rkck", 28, stats, args.steps)
    achieved = flops / sum(p / 1e3 for p in per)

    # ---- e2e through the host-pointer C ABI (pinned buffers, H2D+D2H every window) ----
    e2e = None
    if not args.no_e2e:
        with gpu_local_memory(torch, local):
            yh = torch.from_numpy(y0).pin_memory()
            sth = torch.zeros(num * 8, dtype=torch.int64).pin_memory()
            yg = (torch.empty(total * 28, dtype=torch.float64).pin_memory()
                  if world > 1 and rank == 0 else None)
        y0t = torch.from_numpy(y0)
        yp = ctypes.cast(yh.data_ptr(), ctypes.POINTER(ctypes.c_double))
        prob = A.make_problem(A.PLEIADES)
        tol = A.default_tol()
        ar = A.ARITH_NAMES[args.arith]

        def e2e_run(with_stats):
            """K windows through bode_int_driver with the bench schedule; the
            host restore of y0 every 10 steps is outside the timed calls. For
            N > 1 the final gather of every shard to rank 0 is timed too."""
            stp = ctypes.c_void_p(sth.data_ptr()) if with_stats else None
            for k in range(min(args.warmup, 1)):  # warm the pinned pipeline
                P.api.check(L.bode_int_driver(ctypes.byref(prob), 0, ar, *window_bounds(k), num,
                                              None, yp, ctypes.byref(tol), stp, 1))
            dt = 0.0
            for k in range(args.steps):
                if k % CYCLE == 0:
                    yh.copy_(y0t)
                barrier()
                t = time.perf_counter()
                P.api.check(L.bode_int_driver(ctypes.byref(prob), 0, ar, *window_bounds(k), num,
                                              None, yp, ctypes.byref(tol), stp, 1))
                dt += time.perf_counter() - t
            gather_s = 0.0
            if world > 1:
                barrier()
                t = time.perf_counter()
                D.gather_soa_to_rank0(torch, dist, yh, 28, total, yg)
                gather_s = time.perf_counter() - t
            return secs_max(dt + gather_s), gather_s

        e2e_s, gather_s = e2e_run(True)
        gbytes = total * 28 * 8 if world > 1 else 0
        e2e = {"value": total * args.steps / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": num * 28 * 8,
               "d2h_bytes_per_step": num * (28 * 8 + 64) + gbytes // max(args.steps, 1),
               "ms_per_step": e2e_s / args.steps * 1e3, "pinned_host": True,
               "api": "bode_int_driver (host pointers, per-window H2D/kernel/D2H pipeline)"}
        if world > 1:
            e2e["gather"] = {"ms": gather_s * 1e3, "bytes": gbytes,
                             "how": "shards to rank 0 over NCCL, one D2H of the global SoA"}
        # the paper's intDriver(t, tEnd, numODE, gGlobal, yGlobal) exactly: y in and
        # out, no per-system stats requested (stats = NULL), same windows
        pp_s, _ = e2e_run(False)
        e2e["paper_protocol_no_stats"] = {
            "value": total * args.steps / pp_s, "unit": UNIT,
            "h2d_bytes_per_step": num * 28 * 8, "d2h_bytes_per_step": num * 28 * 8,
            "ms_per_step": pp_s / args.steps * 1e3}
        # one [0, 1] protocol through bode_outer_loop (batchode::outerLoop's
        # drop-in): host buffers in and out, the state resident in HBM between
        # windows, so one H2D and one D2H per call instead of per window
        steps_out = ctypes.c_int32(0)
        P.api.check(L.bode_outer_loop(ctypes.byref(prob), 0, ar, 0.0, 0.2, 0.1, num, None, yp,
                                      ctypes.byref(tol), ctypes.c_void_p(sth.data_ptr()), 1,
                                      P.api.SINK(), None, ctypes.byref(steps_out)))  # warm-up
        yh.copy_(y0t)
        barrier()
        t = time.perf_counter()
        P.api.check(L.bode_outer_loop(ctypes.byref(prob), 0, ar, 0.0, 1.0, 0.1, num, None, yp,
                                      ctypes.byref(tol), ctypes.c_void_p(sth.data_ptr()), 1,
                                      P.api.SINK(), None, ctypes.byref(steps_out)))
        ol_s = secs_max(time.perf_counter() - t)
        e2e["outer_loop"] = {"value": total * steps_out.value / ol_s, "unit": UNIT,
                             "windows": steps_out.value, "ms_total": ol_s * 1e3,
                             "h2d_bytes_per_call": num * 28 * 8,
                             "d2h_bytes_per_call": num * (28 * 8 + 64)}
        del yh, sth, yg

    # ---- secondaries: the other configs, each over this rank's shard ----
    skipped = []

    def secondary(key, problem, solver, arith, dim, make, n_total, label, steps, repack=False,
                  presort_row=None, auto_presort=True):
        if time.monotonic() - T_START > args.budget_s:
            skipped.append(key)
            return
        sb, se = D.shard_range(n_total, world, rank)
        y0s, g0s = make(sb, se - sb)
        # auto_presort=False: the library's own sort by a stiffness parameter
        # around each window (bode_set_presort_param, default on) is switched off
        P.api.check(L.bode_set_presort_param(-2 if auto_presort else -1))
        try:
            sec, perw, sts, _, _ = measure_device(P, A, torch, problem, solver, arith, dim, y0s,
                                                  g0s, steps, 1, stream, repack=repack,
                                                  presort_row=presort_row)
        finally:
            P.api.check(L.bode_set_presort_param(-2))
        f = algorithmic_flops(problem, solver, dim, sts, steps)
        n = se - sb
        extra[key] = {"workload": label, "value": n_total * steps / secs_max(sec),
                      "unit": UNIT, "systems": n_total, "windows": steps,
                      "ms_per_step": sec / steps * 1e3,
                      "achieved_tflops": f / sec / 1e12, "frac_of_fp64_peak": f / sec / peak.value,
                      "flop_per_system_window": f / (n * steps),
                      "kernel_ms_per_window": [round(x, 4) for x in perw]}

    extra = {}
    w10 = min(args.steps, CYCLE)
    if args.secondary:
        pl = lambda mag, seed: (lambda b0, n: (gen_states(L, PLEIADES_IC, mag, seed, b0, n), None))
        secondary("rkck_exact", "pleiades", "rkck", "exact", 28, pl(0.01, 42), total,
                  f"RKCK Pleiades, {total} systems, EXACT policy (bitwise reference arithmetic)",
                  args.steps)
        heat = lambda b0, n: (gen_states(L, heat_ic(64), 0.01, 42, b0, n), None)
        if args.rkc_num > 0:
            secondary("rkc_heat64", "heat", "rkc", "exact", 64, heat, args.rkc_num,
                      f"RKC heat n=64 (config 3/5), {args.rkc_num} systems, EXACT", w10)
            secondary("rkc_heat64_fast", "heat", "rkc", "fast", 64, heat, args.rkc_num,
                      f"RKC heat n=64 (config 3/5), {args.rkc_num} systems, FAST", w10)
            # heatEquation(n) at dimensions without an exact-size kernel: padded
            # lane groups (n = 100 in HeatPad<128>) and one system per block (n = 2000)
            for hn, hk, hcap, label in ((100, "rkc_heat100_padded", 1 << 18,
                                         "padded 16-lane groups (HeatPad<128>)"),
                                        (2000, "rkc_heat2000_block", 1 << 10,
                                         "one system per thread block, vectors in shared memory")):
                hs = min(args.rkc_num, hcap)
                hmk = (lambda hn_: lambda b0, n: (gen_states(L, heat_ic(hn_), 0.01, 42, b0, n),
                                                  None))(hn)
                secondary(hk, "heat", "rkc", "exact", hn, hmk, hs,
                          f"RKC heat n={hn}, {label}, {hs} systems, EXACT", w10)
        if args.aux_num > 0:
            na = args.aux_num
            for ar_ in ("fast", "exact"):
                secondary(f"rkck_stress_{ar_}", "pleiades", "rkck", ar_, 28, pl(0.1, 42), na,
                          f"RKCK Pleiades perturb 0.1 (config 2 divergence stress), {na} "
                          f"systems, {ar_.upper()}", w10)
            expd = lambda b0, n: (gen_states(L, np.array([1.0]), 0.01, 42, b0, n),
                                  stiffness_range(b0, n))
            # natural input order through the default path: bode_int_driver_device
            # sorts each window by |g0| (the reference's specRadHint) on its own
            secondary("rkc_stiff_expdecay", "expdecay", "rkc", "exact", 1, expd, na,
                      f"RKC expDecay, g0 log-uniform in [1,1e4] (config 4), {na} systems, "
                      f"EXACT, natural input order, the library sorting each window by |g0| "
                      f"(default)", w10)
            # the same batch with that sort switched off: the raw lockstep cost
            secondary("rkc_stiff_expdecay_unsorted", "expdecay", "rkc", "exact", 1, expd, na,
                      f"RKC expDecay config 4, natural order, library sort off, {na} systems, "
                      f"EXACT", w10, auto_presort=False)
            # the natural-order batch re-packed by its window-1 cost
            # (bode_repack_by_cost) and restored at the end, inside the timing
            secondary("rkc_stiff_expdecay_repacked", "expdecay", "rkc", "exact", 1, expd, na,
                      f"RKC expDecay config 4 batch re-packed by cost after window 1 (library "
                      f"sort off), {na} systems, EXACT", w10, repack=True, auto_presort=False)
            # sorted once by |g0| before window 1 (bode_repack_by_param), restored
            # at the end, timed
            secondary("rkc_stiff_expdecay_presorted", "expdecay", "rkc", "exact", 1, expd, na,
                      f"RKC expDecay config 4 batch sorted by |g0| once before window 1 "
                      f"(library sort off), {na} systems, EXACT", w10, presort_row=0,
                      auto_presort=False)
            bru = lambda lo, hi: (lambda b0, n: (
                gen_states(L, brusselator_ic(32), 0.01, 7, b0, n),
                brusselator_params(na, lo, hi).reshape(3, na)[:, b0:b0 + n].copy().reshape(-1)))
            secondary("rkck_brusselator_fast", "brusselator", "rkck", "fast", 64,
                      bru(0.002, 0.02), na,
                      f"RKCK FAST Brusselator n=32 (registered problem, generic RKCK kernel), "
                      f"alpha log-spaced in [0.002, 0.02], {na} systems", w10)
            secondary("rkc_brusselator", "brusselator", "rkc", "exact", 64, bru(0.02, 0.5), na,
                      f"RKC Brusselator reaction-diffusion n=32 (dim 64, registered problem), "
                      f"alpha log-spaced in [0.02, 0.5], {na} systems, EXACT", w10)

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    traffic, traffic_src, ncu_evidence = measured_traffic(
        "rkck_fast" if args.arith == "fast" else "rkck_exact", num)
    cpu = None
    if not args.no_cpu and time.monotonic() - T_START < args.budget_s:
        cpu = cpu_leg(args, P, A, torch, stream, extra)

    clocks = clk.summary()
    # nominal FP64 FMA peak at the SM clock observed during the timed region:
    # 64 DFMA/clk/SM x 2 flop x SMs (37.2 TF at 1965 MHz)
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    nominal = 64 * 2 * sms * (clocks["sm_mhz"] or 1965.0) * 1e6
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"RKCK Pleiades (N=28), {total} systems in total (config 5; "
                               f"configs[1]'s workload at 2^24), perturb 0.01 seed 42, eps "
                               f"1e-10; step k = window (k mod 10) of [0, 1] (restart), y0 "
                               f"restored every 10 steps",
                   "arith": args.arith, "systems": total, "systems_per_gpu": num,
                   "window": 0.1,
                   "scheduling": "persistent refill" if args.persistent else "static",
                   "l2": "state (num*28*8 B) exceeds the 126 MB L2; no flush needed",
                   "parallelism": f"dp{world} (contiguous shards, no collective; final gather "
                                  f"to rank 0 in e2e)"},
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
        # bode_stats_summary over the headline's stats (merged over the timed windows)
        "straggler": {k: v for k, v in P.stats_summary(stats).items()
                      if k in ("attempts_max", "attempts_argmax", "attempts_mean",
                               "underflow_count", "budget_exhausted_count",
                               "lockstep_efficiency")},
        "skipped_over_budget": skipped,
        "wall_s": time.monotonic() - T_START,
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def cpu_leg(args, P, A, torch, stream, extra):
    """The reference CPU path on this host for every config the line reports
    (2^16 systems, [0, 1] in 10 windows, one warm-up window,
    best of 3), and -- as the checker, not as the thing measured -- the GPU's
    agreement with it on the config-2 stress sample under both policies."""
    from golden_cases import PLEIADES_IC, heat_ic
    n = args.cpu_sample
    rate, cores, kind, dt, _, _ = cpu_reference("pleiades", "rkck", PLEIADES_IC, 0.01, 42, n)
    n1 = max(1024, n // 16)
    rate1, _, _, dt1, _, _ = cpu_reference("pleiades", "rkck", PLEIADES_IC, 0.01, 42, n1,
                                           threads=1, repeats=1)
    cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": kind,
           "sample": f"{n} Pleiades systems x 10 windows ([0,1]) via outerLoop, all host "
                     f"threads, one warm-up window, best of 3: {dt:.2f} s",
           "one_thread": {"value": rate1, "unit": UNIT, "cores": 1,
                          "sample": f"{n1} systems x 10 windows, {dt1:.2f} s"},
           "configs": {}}
    heat_n = n
    for key, prob, solver, base, mag, ns, g, gpu_key in (
            ("rkc_heat64", "heat", "rkc", heat_ic(64), 0.01, heat_n, None, "rkc_heat64"),
            ("rkc_heat100_padded", "heat", "rkc", heat_ic(100), 0.01, max(64, n // 16), None,
             "rkc_heat100_padded"),
            ("rkc_heat2000_block", "heat", "rkc", heat_ic(2000), 0.01, max(16, n // 2048), None,
             "rkc_heat2000_block"),
            ("rkc_stiff_expdecay", "expdecay", "rkc", np.array([1.0]), 0.01, n,
             stiffness_range(0, n), "rkc_stiff_expdecay"),
            ("rkck_stress", "pleiades", "rkck", PLEIADES_IC, 0.1, n, None, "rkck_stress_fast")):
        if time.monotonic() - T_START > args.budget_s:
            break
        r, c, k, d, yref, sref = cpu_reference(prob, solver, base, mag, 42, ns, g=g)
        ent = {"value": r, "unit": UNIT, "cores": c, "kind": k,
               "sample": f"{ns} systems x 10 windows, one warm-up window, best of 3: {d:.2f} s"}
        if gpu_key in extra:
            ent["gpu_over_cpu"] = extra[gpu_key]["value"] / r
        if key == "rkck_stress":
            ent["parity"] = stress_parity(P, A, torch, stream, base, mag, ns, yref, sref)
        cpu["configs"][key] = ent
    return cpu


def stress_parity(P, A, torch, stream, base, mag, num, yref, sref):
    """Config-2 stress (perturb 0.1): per-system max-norm relative error of
    the GPU's [0, 1] result against the reference's, and count agreement,
    under both policies (north_star bar: 1e-3 * eps = 1e-13)."""
    out = {}
    y0 = gen_states(P.lib(), base, mag, 42, 0, num)
    for arith in ("fast", "exact"):
        _, _, st, _, y = measure_device(P, A, torch, "pleiades", "rkck", arith, 28, y0, None,
                                        CYCLE, 0, stream, return_state=True)
        err = sysrel(y, yref, num, 28)
        same = np.ones(num, bool)
        for k in ("steps_accepted", "steps_rejected", "rhs_evals", "underflow"):
            same &= st[k] == sref[k]
        out[arith] = {"systems": num, "within_1e-13": float(((err <= 1e-13) & same).mean()),
                      "max_rel_err": float(err.max()), "count_mismatches": int((~same).sum()),
                      "bitwise": bool(np.array_equal(y.view(np.uint64), yref.view(np.uint64)))}
    return out


if __name__ == "__main__":
    main()
