"""B200-native multilevel block-Toeplitz matvec + restarted GMRES
(hot path of arXiv 2506.04710). The product is libtbt.so (hand-written
sm_100a CUDA + C++ host behind the C ABI in include/tbt.h); this package is
its host-side mirror of the reference's operator/solver API."""
from .configs import CONFIGS, Config, rhs_for  # noqa: F401
from .toeplitz import (  # noqa: F401
    Correction, DeviceError, NumericError, SolveResult, SolverOptions, ToeplitzMatvec, ToeplitzRep,
    UserError, dist_plan, dist_unique_id, init_from_torch, loopback_group_id, iterative_solve, schur_solve, toeplitz_matvec, Margin, DenseMargin, generators_from_level1, read_ztoe1, port_network, tarc, array_farfield)

__all__ = ["CONFIGS", "Config", "rhs_for", "Correction", "DeviceError", "NumericError", "SolveResult",
           "SolverOptions", "ToeplitzMatvec", "ToeplitzRep", "UserError", "iterative_solve",
           "toeplitz_matvec", "dist_plan", "dist_unique_id", "init_from_torch", "loopback_group_id", "schur_solve", "Margin", "DenseMargin", "generators_from_level1", "read_ztoe1", "port_network", "tarc", "array_farfield"]
