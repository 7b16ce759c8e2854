"""B200-native MG-preconditioned CG with coarse-level telescoping (arxiv 1604.07163 hot path).

The product is the in-tree sm_100a library libtmgx.so behind the C-ABI in include/tmgx.h;
`tmgx` is the Python mirror of the reference's solver/preconditioner surface over it.
"""
from . import tmgx  # noqa: F401
from .tmgx import (ConfigError, CudaError, Error, GridHeader, KrylovConfig, MGConfig, Problem,  # noqa: F401
                   SolveReport, SolverNode, SplitResult, TelescopeStage, World)
