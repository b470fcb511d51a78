"""odebench on the GPU: the reference's benchmark/report front end
(proj/src/bench.cpp, proj/tools/odebench_main.cpp) over bode's kernels.

    python -m paper_1611_02274_b200.odebench --problem pleiades --solver rkck \\
        --mode integrate --num-systems 1024 --output run.csv --summary run.json

Same flags, defaults (bench.hpp:15-37), workloads (bench.cpp:89-119), CSV
layout with 17 significant digits (bench.cpp:23-28, :224-240, :296-301,
:357-363), JSON summary shape (configJson :140-157, statsJson :163-178) and
exit codes (0 ok, 1 IoError, 2 ConfigError, bench.cpp:382-397), so output
files can be diffed against the reference's. Differences: `--workers` is the
number of GPUs (scaling mode: the ladder 1, 2, 4, ... GPUs), `--arith`
selects the arithmetic policy, and --pleiades-ic defaults to the canonical
values built into the library (the asset's FNV-1a 0x5583feb418028048).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import math
import sys
import time

import numpy as np

from . import _abi as A
from . import api as B


class ConfigError(RuntimeError):
    pass


class IoError(RuntimeError):
    pass


def format17(v: float) -> str:
    """formatDouble17 (bench.cpp:23-28): 17 significant digits, general format."""
    return format(float(v), ".17g")


def config_json(cfg) -> dict:  # bench.cpp:140-157
    return {"problem": cfg.problem, "solver": cfg.solver, "mode": cfg.mode,
            "numSystems": cfg.num_systems, "t0": cfg.t0, "tEnd": cfg.t_end,
            "hOuter": cfg.outer_step, "eps": cfg.eps, "absTol": cfg.abs_tol,
            "relTol": cfg.rel_tol, "workers": cfg.workers, "seed": cfg.seed,
            "perturbMagnitude": cfg.perturb, "heatPoints": cfg.heat_points,
            "pleiadesIcPath": cfg.pleiades_ic}


def stats_json(stats: np.ndarray) -> dict:  # bench.cpp:163-178
    under = [int(i) for i in np.flatnonzero(stats["underflow"])]
    hmin = float(stats["h_min_seen"].min()) if stats.size else math.inf
    return {"stepsAccepted": int(stats["steps_accepted"].sum()),
            "stepsRejected": int(stats["steps_rejected"].sum()),
            "rhsEvals": int(stats["rhs_evals"].sum()),
            "specRadEvals": int(stats["spec_rad_evals"].sum()),
            "hMinSeen": hmin if math.isfinite(hmin) else 0.0,
            "hMaxSeen": float(stats["h_max_seen"].max()) if stats.size else 0.0,
            "underflowCount": len(under), "underflowSystems": under}


def load_pleiades_ic(path: str) -> np.ndarray:  # problems.cpp:39-52
    if path in ("", "builtin"):
        return B.problems.pleiades_initial_conditions()
    try:
        tokens = open(path).read().split()
    except OSError:
        raise IoError(f"cannot open Pleiades initial-condition file: {path}")
    try:
        vals = [float(x) for x in tokens]
    except ValueError:
        raise IoError(f"Pleiades initial-condition file is non-numeric: {path}")
    if len(vals) < 28:
        raise IoError(f"Pleiades initial-condition file ends early at line {len(vals) + 1}: {path}")
    if len(vals) > 28:
        raise IoError(f"Pleiades initial-condition file has more than 28 values: {path}")
    return np.array(vals)


def build_workload(cfg):  # bench.cpp:89-119
    if cfg.problem == "pleiades":
        problem, base = B.problems.pleiades(), load_pleiades_ic(cfg.pleiades_ic)
    elif cfg.problem == "heat":
        problem = B.problems.heat_equation(cfg.heat_points)
        base = B.problems.heat_initial_condition(cfg.heat_points)
    elif cfg.problem == "expdecay":
        problem, base = B.problems.exp_decay(), np.array([1.0])
    elif cfg.problem == "harmonic":
        problem, base = B.problems.harmonic(), np.array([1.0, 0.0])
    else:
        raise ConfigError(f"unknown problem: {cfg.problem}")
    batch = B.problems.perturb_initial_conditions(base, cfg.perturb, cfg.seed, cfg.num_systems)
    if cfg.problem == "expdecay":
        batch.param_dim = 1
        batch.params = np.ones(cfg.num_systems)
        problem = B.OdeProblem(A.EXPDECAY, 1, 1)
    return problem, batch


def tolerances(cfg):  # bench.cpp:120-127
    tol = A.default_tol(eps=cfg.eps, abs_tol=cfg.abs_tol, rel_tol=cfg.rel_tol)
    B.check(B.lib().bode_tol_validate(ctypes.byref(tol)))
    return tol


def timed_outer_loop(problem, batch, cfg, tol, gpus, keep):  # bench.cpp:196-214
    snaps, marks = [], []
    mark = [time.perf_counter()]

    def sink(t, snap):
        marks.append(time.perf_counter() - mark[0])
        if keep:
            snaps.append((t, snap))
        mark[0] = time.perf_counter()

    res = B.outer_loop(problem, batch, cfg.t0, cfg.t_end, cfg.outer_step, solver=cfg.solver,
                       tol=tol, gpus=gpus, sink=sink, arith=cfg.arith)
    return res, snaps, (sum(marks) / len(marks)) if marks else 0.0


def write(path, text):
    try:
        with open(path, "w", newline="") as f:
            f.write(text)
    except OSError:
        raise IoError(f"cannot open output file for writing: {path}")


def run_integrate(cfg):  # bench.cpp:218-249
    problem, batch = build_workload(cfg)
    tol = tolerances(cfg)
    res, snaps, per_window = timed_outer_loop(problem, batch, cfg, tol, cfg.workers, True)
    if cfg.output:
        lines = ["outerStepIndex,t,systemIndex" + "".join(f",var{j}" for j in range(problem.dim))]
        for k, (t, snap) in enumerate(snaps):
            vals = snap.values.reshape(problem.dim, snap.num_systems)
            tt = format17(t)
            for i in range(snap.num_systems):
                lines.append(f"{k + 1},{tt},{i}," + ",".join(format17(v) for v in vals[:, i]))
        write(cfg.output, "\n".join(lines) + "\n")
    if cfg.summary:
        write(cfg.summary, json.dumps({
            "config": config_json(cfg), "outerSteps": res.outer_steps,
            "wallClockPerOuterStepSeconds": per_window, "workers": cfg.workers,
            "stats": stats_json(res.stats)}, indent=2) + "\n")
    return 0


def run_convergence(cfg):  # bench.cpp:251-322
    if cfg.problem not in ("expdecay", "harmonic"):
        raise ConfigError("convergence mode needs an analytically solvable problem "
                          "(expdecay or harmonic)")
    span = cfg.t_end - cfg.t0
    if not span > 0.0:
        raise ConfigError("convergence mode: empty interval")
    if cfg.ladder_points < 2:
        raise ConfigError("convergence mode: need >= 2 ladder points")
    if cfg.problem == "expdecay":
        problem, batch = B.OdeProblem(A.EXPDECAY, 1, 1), B.pack([[1.0]], [[1.0]])
        exact = lambda y: abs(y[0] - math.exp(-span))
    else:
        problem, batch = B.problems.harmonic(), B.pack([[1.0, 0.0]])
        exact = lambda y: math.sqrt((y[0] - math.cos(span)) ** 2 + (y[1] + math.sin(span)) ** 2)
    h0 = cfg.ladder_h0 if cfg.ladder_h0 > 0 else (0.1 if cfg.solver == "rkck" else 0.05)
    hs, errs = [], []
    for k in range(cfg.ladder_points):
        h = h0 / float(1 << k)
        steps = int(math.floor(span / h + 0.5))  # std::lround
        y = B.integrate_fixed(problem, batch, cfg.t0, cfg.t_end, steps, solver=cfg.solver,
                              stages=5, arith=cfg.arith).values
        hs.append(span / float(steps))
        errs.append(exact(y))
    lx = np.log(hs)
    ly = np.log(np.maximum(errs, 5e-324))
    m = len(hs)
    slope = (m * np.sum(lx * ly) - lx.sum() * ly.sum()) / (m * np.sum(lx * lx) - lx.sum() ** 2)
    if cfg.output:
        write(cfg.output, "h,globalError\n" + "".join(
            f"{format17(h)},{format17(e)}\n" for h, e in zip(hs, errs)))
    if cfg.summary:
        write(cfg.summary, json.dumps({
            "config": config_json(cfg), "slope": float(slope),
            "points": [{"h": h, "globalError": e} for h, e in zip(hs, errs)]}, indent=2) + "\n")
    print(f"convergence slope: {format17(slope)}")
    return 0


def run_scaling(cfg):  # bench.cpp:324-380, ladder over GPUs
    if cfg.num_systems < cfg.workers:
        raise ConfigError("scaling mode requires numSystems >= workers")
    problem, batch = build_workload(cfg)
    tol = tolerances(cfg)
    ladder, n = [], 1
    while n <= cfg.workers:
        ladder.append(n)
        n *= 2
    rows, ref, identical, stats_out = [], None, True, None
    for gpus in ladder:
        res, _, wall = timed_outer_loop(problem, batch, cfg, tol, gpus, False)
        if gpus == 1:
            ref = res.states.values.copy()
            stats_out = stats_json(res.stats)
        elif not np.array_equal(res.states.values.view(np.uint64), ref.view(np.uint64)):
            identical = False
        rows.append([gpus, wall, 0.0])
    for r in rows:
        r[2] = rows[0][1] / r[1] if r[1] > 0 else 0.0
    rows[0][2] = 1.0
    if cfg.output:
        write(cfg.output, "workers,wallClockPerOuterStep,speedupVs1\n" + "".join(
            f"{w},{format17(t)},{format17(s)}\n" for w, t, s in rows))
    if cfg.summary:
        write(cfg.summary, json.dumps({
            "config": config_json(cfg),
            "rows": [{"workers": w, "wallClockPerOuterStepSeconds": t, "speedupVs1": s}
                     for w, t, s in rows],
            "bitwiseIdentical": identical, "stats": stats_out}, indent=2) + "\n")
    if not identical:
        print("warning: outputs differ across worker counts", file=sys.stderr)
    return 0


def run(cfg) -> int:  # bench.cpp:382-397
    try:
        if cfg.solver not in ("rkck", "rkc"):
            raise ConfigError(f"unknown solver: {cfg.solver}")
        modes = {"integrate": run_integrate, "convergence": run_convergence,
                 "scaling": run_scaling}
        if cfg.mode not in modes:
            raise ConfigError(f"unknown mode: {cfg.mode}")
        return modes[cfg.mode](cfg)
    except IoError as e:
        print(f"io error: {e}", file=sys.stderr)
        return 1
    except (ConfigError, B.InvalidShape, B.InvalidInterval) as e:
        print(f"config error: {e}", file=sys.stderr)
        return 2


def parser() -> argparse.ArgumentParser:  # odebench_main.cpp:16-51, bench.hpp:15-37
    ap = argparse.ArgumentParser(description="odebench: batched ODE integration benchmark (GPU)")
    ap.add_argument("--problem", default="pleiades")
    ap.add_argument("--solver", default="rkck")
    ap.add_argument("--mode", default="integrate")
    ap.add_argument("--num-systems", dest="num_systems", type=int, default=1024)
    ap.add_argument("--t0", type=float, default=0.0)
    ap.add_argument("--t-end", dest="t_end", type=float, default=1.0)
    ap.add_argument("--outer-step", dest="outer_step", type=float, default=0.1)
    ap.add_argument("--eps", type=float, default=1.0e-10)
    ap.add_argument("--abs-tol", dest="abs_tol", type=float, default=1.0e-10)
    ap.add_argument("--rel-tol", dest="rel_tol", type=float, default=1.0e-6)
    ap.add_argument("--workers", type=int, default=1, help="GPUs (scaling: ladder maximum)")
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--perturb", type=float, default=0.01)
    ap.add_argument("--output", default="")
    ap.add_argument("--summary", default="")
    ap.add_argument("--pleiades-ic", dest="pleiades_ic", default="builtin")
    ap.add_argument("--heat-points", dest="heat_points", type=int, default=64)
    ap.add_argument("--ladder-h0", dest="ladder_h0", type=float, default=0.0)
    ap.add_argument("--ladder-points", dest="ladder_points", type=int, default=4)
    ap.add_argument("--arith", default="exact", choices=["exact", "fast"])
    return ap


def main(argv=None) -> int:
    return run(parser().parse_args(argv))


if __name__ == "__main__":
    sys.exit(main())
