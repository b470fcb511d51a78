"""Parity configurations shared by the golden-fixture generator and the tests
(BASELINE.json configs 1, 3, 4)."""
import numpy as np

from paper_1611_02274_b200 import _abi as A

PLEIADES_IC = np.array([3.0, 3.0, -1.0, -3.0, 2.0, -2.0, 2.0, 3.0, -3.0, 2.0, 0.0, 0.0, -4.0, 4.0,
                        0.0, 0.0, 0.0, 0.0, 0.0, 1.75, -1.5, 0.0, 0.0, 0.0, -1.25, 1.0, 0.0, 0.0])

CASES = {
    # config 1: RKCK Pleiades, 1024 systems, bench seed and acceptance seed
    "cfg1_pleiades_rkck_s42": dict(problem="pleiades", solver="rkck", num=1024, seed=42, mag=0.01),
    "cfg1_pleiades_rkck_s20140609": dict(problem="pleiades", solver="rkck", num=1024,
                                         seed=20140609, mag=0.01),
    # config 3: RKC heat (n = 64)
    "cfg3_heat64_rkc_s42": dict(problem="heat", solver="rkc", num=256, seed=42, mag=0.01),
    # config 4: RKC expDecay with per-system stiffness g0 in [1, 1e4]
    "cfg4_expdecay_rkc_stiff": dict(problem="expdecay", solver="rkc", num=2048, seed=42, mag=0.01),
}


def unit_symmetric(seed, count):
    k = np.arange(count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (k + np.uint64(1)) * np.uint64(0x9e3779b97f4a7c15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xbf58476d1ce4e5b9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94d049bb133111eb)
        z = z ^ (z >> np.uint64(31))
    return 2.0 * ((z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53) - 1.0


def perturb(base, mag, seed, count):
    """perturbInitialConditions (problems.cpp:171-191), vectorised."""
    base = np.asarray(base, dtype=np.float64)
    u = unit_symmetric(seed, count * base.size).reshape(count, base.size)
    return np.ascontiguousarray((base[None, :] * (1.0 + u * mag)).T).reshape(-1)


def heat_ic(n):
    dx = 1.0 / (n + 1)
    x = (np.arange(n) + 1) * dx
    return 4.0 * x * (1.0 - x)


def brusselator_ic(n):
    """u = 1 + sin(2 pi x), v = 3 on the interior points x_i = i/(n+1), interleaved."""
    x = (np.arange(n) + 1) / (n + 1)
    y = np.empty(2 * n)
    y[0::2] = 1.0 + np.sin(2.0 * np.pi * x)
    y[1::2] = 3.0
    return y


def brusselator_params(num, alpha_lo, alpha_hi, A=1.0, B=3.0):
    """SoA params (A, B, alpha) with alpha log-spaced over the batch."""
    alpha = np.exp(np.linspace(np.log(alpha_lo), np.log(alpha_hi), num))
    return np.concatenate([np.full(num, A), np.full(num, B), alpha])


def build_inputs(case, num=None):
    num = num or case["num"]
    kind = case["problem"]
    solver = A.SOLVER_NAMES[case["solver"]]
    g = None
    if kind == "pleiades":
        prob, base = A.make_problem(A.PLEIADES), PLEIADES_IC
    elif kind == "heat":
        n = case.get("n", 64)
        prob, base = A.make_problem(A.HEAT, n), heat_ic(n)
    elif kind == "expdecay":
        prob, base = A.make_problem(A.EXPDECAY), np.array([1.0])
        g = 10.0 ** (2.0 + 2.0 * unit_symmetric(9, num))
    else:
        raise ValueError(kind)
    return prob, solver, perturb(base, case["mag"], case["seed"], num), g
