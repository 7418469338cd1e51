"""B200-native (sm_100a) RZF precoder update with WB-arSVD inverse maintenance.

Drop-in for the numerical core of the reference package ``leorzf`` 0.1.0
(pkg/src/leorzf/__init__.py:17-31): the same public names, signatures,
dataclasses and exceptions, computed by hand-written CUDA kernels through the
C ABI in include/leorzf_b200.h.  Plus the batched trajectory runner that
replaces the harness's per-trial loop (trajectory.py).
"""

from .errors import (DimensionMismatchError, NativeLibraryError, SimulationError,
                     SingularAuxiliaryError, SingularMatrixError, ZeroPrecoderError)
from .lowrank import (ArSvdConfig, GramState, LowRankFactor, UpdateReport, arsvd, cost_full,
                      cost_wb_arsvd, direct_inverse, gram_delta, gram_matrix, sketch_cost,
                      update_inverse, woodbury_update)
from .precoding import Precoder, RateReport, rzf_precoder, sum_rate
from .trajectory import TrajectoryConfig, TrajectoryRunner, run_trajectory

__version__ = "0.1.0"

__all__ = [
    "ArSvdConfig", "GramState", "LowRankFactor", "UpdateReport", "Precoder", "RateReport",
    "arsvd", "cost_full", "cost_wb_arsvd", "sketch_cost", "direct_inverse", "gram_delta",
    "gram_matrix", "update_inverse", "woodbury_update", "rzf_precoder", "sum_rate",
    "TrajectoryConfig", "TrajectoryRunner", "run_trajectory",
    "DimensionMismatchError", "NativeLibraryError", "SimulationError", "SingularAuxiliaryError",
    "SingularMatrixError", "ZeroPrecoderError",
]
