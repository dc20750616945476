"""B200-native multi-word Conjugate Gradient (FP64 / DW / QDW / TW / QTW).

Drop-in for the hot path of the reference package `mwcg` (cg_solve and the
operator table behind it), running on sm_100a through libmwcg_cuda.so.
"""
__version__ = "0.1.0"

from .sparse import CsrMatrix, identity, laplacian_2d, random_symmetric, scaled_laplacian_2d  # noqa: F401
from .cg import (ConvergenceRecord, Normalization, SolverConfig, SolverResult,  # noqa: F401
                 cg_solve)
from .kernels import MODES, MultiwordVector  # noqa: F401
