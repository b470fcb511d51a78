"""The C++ drop-in (include/bode.hpp, examples/pleiades_drop_in.cpp) runs the
reference's Pleiades protocol and reproduces the oracle bit for bit."""
import os
import subprocess

import numpy as np
import pytest

from paper_1611_02274_b200 import _abi as A
from golden_cases import PLEIADES_IC, perturb

EXE = os.path.join(A.PKG_DIR, "lib", "pleiades_drop_in")


def test_example_is_built():
    assert os.path.exists(EXE), "run paper_1611_02274_b200.build (builds examples/)"


@pytest.mark.gpu
def test_cpp_drop_in_matches_oracle(gpu, oracle):
    num = 512
    out = subprocess.run([EXE, str(num)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    lines = out.stdout.strip().splitlines()
    assert sum(l.startswith("window") for l in lines) == 10
    fields = dict(kv.split("=") for kv in lines[-1].split())
    rc, y, st, _ = oracle.outer_loop(A.make_problem(A.PLEIADES), A.SOLVER_RKCK, 0.0, 1.0, 0.1,
                                     perturb(PLEIADES_IC, 0.01, 42, num))
    assert int(fields["accepted"]) == int(st["steps_accepted"].sum())
    assert int(fields["rejected"]) == int(st["steps_rejected"].sum())
    assert float(fields["x1[0]"]) == y[0]


BATCH_EXE = os.path.join(A.PKG_DIR, "lib", "test_batch_dropin")


def test_reference_batch_tests_host_cases():
    """test_batch.cpp's host-only cases (pack/unpack/validation) compiled
    against include/bode.hpp; without a device the program runs only those."""
    assert os.path.exists(BATCH_EXE), "run paper_1611_02274_b200.build (builds tests/cpp/)"
    out = subprocess.run([BATCH_EXE], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.startswith("PASS")


@pytest.mark.gpu
def test_reference_batch_tests_on_gpu(gpu):
    """All of test_batch.cpp:16-258, transcribed against the bode:: drop-in,
    including worker invariance (1, 2, 4, 8 shards on the available devices)
    and the NaN-freeze case on a registered device problem."""
    out = subprocess.run([BATCH_EXE], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.startswith("PASS") and "host-only" not in out.stdout, out.stdout
