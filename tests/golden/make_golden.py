"""Regenerate the golden fixtures from the UNMODIFIED reference.

    make -C oracle && python tests/golden/make_golden.py

Runs batchode::outerLoop (oracle/_ref/libbatchode_ref.so, compiled from
/root/reference/proj/src by oracle/Makefile) over [0, 1] in 10 restart
windows on the BASELINE.json parity configs and stores the final SoA states
and per-system stats. Inputs are regenerated at test time with the
reference generator (problems.cpp:158-191), which is itself pinned bitwise.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

from golden_cases import CASES, build_inputs  # noqa: E402
from oracle_lib import RefLib  # noqa: E402


def main():
    R = RefLib()
    for name, case in CASES.items():
        prob, solver, y0, g = build_inputs(case)
        rc, y, st, steps = R.outer_loop(prob, solver, 0.0, 1.0, 0.1, y0, g, workers=8)
        assert rc == 0 and steps == 10, (name, rc, steps)
        np.savez_compressed(
            os.path.join(HERE, name + ".npz"), y=y,
            steps_accepted=st["steps_accepted"].astype(np.int32),
            steps_rejected=st["steps_rejected"].astype(np.int32),
            rhs_evals=st["rhs_evals"].astype(np.int32),
            spec_rad_evals=st["spec_rad_evals"].astype(np.int32),
            h_min_seen=st["h_min_seen"], h_max_seen=st["h_max_seen"],
            underflow=st["underflow"].astype(np.int8))
        print(name, "written")


if __name__ == "__main__":
    main()
