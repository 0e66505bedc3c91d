"""condkit-b200: B200-native Projected-Adam kappa_2 estimator (arXiv 2409.11515).

Drop-in for the reference's estimator / error-bound interface
(condkit/condest.hpp, error_bounds.hpp, sparse.hpp). Every numeric operation
runs in ``libcondkit_b200.so`` (sm_100a kernels behind a C ABI,
include/condkit_b200.h); there is no CPU fallback.
"""
from .condest import (AdamConfig, AdamState, AdamStepInfo, ExplicitOracle, GradientOracle,
                      NormEstimate, Session, estimate_norm, grad_explicit, loss_explicit, norm2,
                      projected_adam)
from .errors import (CondkitError, DegenerateDirection, DeviceUnavailable, DimensionMismatch,
                     InvalidArgument, LogicError, NativeLibraryMissing, NumericallySingular,
                     StructurallySingular, ZeroColumn, ZeroRHS, ZeroRow, ZeroSolution)
from .error_bounds import (Bounds, BoundsReport, Verdict, VerifyOptions, kEpsMach, loose_bounds,
                           propagate_bound, singularity_bound, tight_bounds, verify_solution)
from .inverse import (Cond2Result, InverseOracle, LUFactors, cond2, grad_inverse, inv_norm2,
                      lu_factorize, lu_solve, lu_transpose_solve)
from .rng import mix_seed, random_unit_vector, random_unit_vectors
from .sparse import (DeviceMatrix, ScalingDiagonal, SparseMatrix, column_norms, column_scale,
                     matvec, row_norms, row_scale, transpose_matvec, unscale_solution)

__all__ = [
    "AdamConfig", "AdamState", "AdamStepInfo", "ExplicitOracle", "GradientOracle",
    "NormEstimate", "Session", "estimate_norm", "grad_explicit", "loss_explicit", "norm2",
    "projected_adam", "CondkitError", "DegenerateDirection", "DeviceUnavailable",
    "DimensionMismatch", "InvalidArgument", "LogicError", "NativeLibraryMissing",
    "NumericallySingular", "StructurallySingular", "ZeroRHS", "ZeroSolution", "mix_seed",
    "random_unit_vector", "random_unit_vectors", "DeviceMatrix", "SparseMatrix", "matvec",
    "transpose_matvec", "Bounds", "BoundsReport", "Verdict", "VerifyOptions", "kEpsMach",
    "loose_bounds", "propagate_bound", "singularity_bound", "tight_bounds", "verify_solution",
    "Cond2Result", "InverseOracle", "LUFactors", "cond2", "grad_inverse", "inv_norm2",
    "lu_factorize", "lu_solve", "lu_transpose_solve", "ScalingDiagonal", "column_norms",
    "column_scale", "row_norms", "row_scale", "unscale_solution", "ZeroColumn", "ZeroRow",
]
