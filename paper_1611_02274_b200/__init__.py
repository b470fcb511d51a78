"""B200-native batched RKCK / RKC ODE integration (arxiv/paper_1611_02274 hot path).

The hot path lives in libbode.so (CUDA sm_100a, FP64) behind the C ABI in
include/bode.h; this package is the Python mirror of the reference's batch
interface (api.py) plus the in-tree build (build.py).
"""
from . import _abi  # noqa: F401
from .api import (BatchResult, BatchStates, BodeError, CudaError, InvalidInterval,  # noqa: F401
                  InvalidShape, InvalidStageCount, NoDevice, OdeProblem, OuterLoopResult,
                  Unsupported, fill_params, int_driver_device, integrate_batch, integrate_fixed, lib,
                  outer_loop, pack, problems, stats_summary, stiffness_params, tolerance_settings,
                  trace_steps,
                  unpack)
