"""odebench-compatible report plumbing: bode's GPU
odebench writes the same CSV bytes and JSON stats as the reference's own
bench::run (proj/src/bench.cpp, compiled unmodified into oracle/_ref)."""
import ctypes
import json
import os

import numpy as np
import pytest

from paper_1611_02274_b200 import odebench
from paper_1611_02274_b200.odebench import format17
from oracle_lib import REF_SO, ref_available
from golden_cases import PLEIADES_IC


def test_format17_matches_reference_formatting():  # bench.cpp:23-28, test_bench.cpp:52-67
    rng = np.random.default_rng(0)
    for v in np.concatenate([rng.standard_normal(2000) * 10.0 ** rng.integers(-300, 300, 2000),
                             [0.0, 1.0, 0.1, 1e-10, 123456789.0]]):
        s = format17(v)
        assert float(s) == v
        assert len(s.replace("-", "").replace(".", "").split("e")[0].lstrip("0")) <= 17


def test_config_errors_map_to_exit_code_2(tmp_path):
    assert odebench.main(["--mode", "convergence", "--problem", "pleiades"]) == 2
    assert odebench.main(["--solver", "nope"]) == 2
    assert odebench.main(["--pleiades-ic", str(tmp_path / "missing.txt")]) == 1


def ref_bench(tmp, **kw):
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    lib = ctypes.CDLL(REF_SO)
    if not hasattr(lib, "ref_bench_run"):
        pytest.skip("reference bench.cpp not compiled (json.hpp absent)")
    f = lib.ref_bench_run
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_char_p] * 3 + [ctypes.c_int] + [ctypes.c_double] * 6 + \
        [ctypes.c_int, ctypes.c_uint64, ctypes.c_double] + [ctypes.c_char_p] * 3 + [ctypes.c_int]
    ic = os.path.join(tmp, "ic.txt")
    with open(ic, "w") as fh:
        fh.write("\n".join(format17(v) for v in PLEIADES_IC) + "\n")
    out, summ = os.path.join(tmp, "ref.csv"), os.path.join(tmp, "ref.json")
    rc = f(kw["problem"].encode(), kw["solver"].encode(), kw["mode"].encode(), kw["num"],
           0.0, 1.0, 0.1, 1e-10, 1e-10, 1e-6, 1, 42, 0.01, out.encode(), summ.encode(),
           ic.encode(), 64)
    assert rc == 0
    return out, summ, ic


@pytest.mark.gpu
@pytest.mark.parametrize("problem,solver,mode", [("pleiades", "rkck", "integrate"),
                                                 ("heat", "rkc", "integrate"),
                                                 ("harmonic", "rkck", "convergence"),
                                                 ("expdecay", "rkc", "convergence")])
def test_report_files_match_reference(gpu, tmp_path, problem, solver, mode):
    num = 48
    ref_csv, ref_json, ic = ref_bench(str(tmp_path), problem=problem, solver=solver, mode=mode,
                                      num=num)
    out, summ = str(tmp_path / "bode.csv"), str(tmp_path / "bode.json")
    rc = odebench.main(["--problem", problem, "--solver", solver, "--mode", mode,
                        "--num-systems", str(num), "--output", out, "--summary", summ,
                        "--pleiades-ic", ic])
    assert rc == 0
    assert open(out).read() == open(ref_csv).read()
    a, b = json.load(open(summ)), json.load(open(ref_json))
    if mode == "integrate":
        assert a["stats"] == b["stats"] and a["outerSteps"] == b["outerSteps"]
    else:
        assert a["points"] == b["points"]
        assert abs(a["slope"] - b["slope"]) <= 1e-12 * abs(b["slope"])
