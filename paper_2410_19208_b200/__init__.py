"""paper_2410_19208_b200 — B200-native randomized projection onto the PSD cone.

Drop-in for the hot path of the reference ``psdcone`` package (arXiv
2410.19208): the same names, signatures, exceptions and RNG draw order, with
every numeric step in hand-written sm_100a kernels (libpsdproj.so, C ABI in
include/psdproj.h).  ``install()`` rebinds the reference modules so that
``psdcone.solve`` and friends run on this path.
"""

from .errors import (AlphaTooSmall, AsymmetricMatrixError, ConvergenceFailure, DeviceError,
                     DimensionMismatch, InvalidParams, NonSquareError, PsdconeError,
                     RankDeficientSample)
from ._tensors import DeviceRng
from .projection import (METHODS, ProjectionReport, ProjectorConfig, flops, project, ran_proj,
                         ran_proj_scal, set_fp64_engine)
from .sketch import (RangeParams, min_eig_magnitude, orthonormality_defect, power_iteration,
                     range_finder)
from .symmetric import (EigenDecomposition, eigh, exact_psd_projection, frobenius_norm,
                        gaussian_matrix, require_symmetric, rng_from_seed, symmetrize)
from .pipeline import ran_proj_many
from .sdls import SolveReport, SparseSdlsProblem, TrajectoryPoint, solve
from .install import install, uninstall
from . import workloads  # noqa: E402  (seeded HBM generators for the BASELINE configs)
from . import experiments  # noqa: E402  (Monte-Carlo projection-error harness, §8 f3)
from . import matrix_io  # noqa: E402  (Matrix Market / JSON problem files, §8 f4)
from .matrix_io import read_matrix_market, write_matrix_market  # noqa: E402
from .experiments import projection_error_sweep  # noqa: E402

__version__ = "0.1.0"

__all__ = [
    "experiments", "projection_error_sweep", "matrix_io", "read_matrix_market", "write_matrix_market",
    "AlphaTooSmall", "AsymmetricMatrixError", "ConvergenceFailure", "DeviceError",
    "DimensionMismatch", "InvalidParams", "NonSquareError", "PsdconeError", "RankDeficientSample",
    "DeviceRng", "METHODS", "ProjectionReport", "ProjectorConfig", "flops", "project", "ran_proj",
    "ran_proj_scal", "ran_proj_many", "set_fp64_engine", "RangeParams", "min_eig_magnitude", "orthonormality_defect",
    "power_iteration", "range_finder", "EigenDecomposition", "eigh", "exact_psd_projection",
    "frobenius_norm", "gaussian_matrix", "require_symmetric", "rng_from_seed", "symmetrize",
    "install", "uninstall", "solve", "SparseSdlsProblem", "SolveReport", "TrajectoryPoint",
]
